// TEST INFRASTRUCTURE — not product code.
//
// extern "C" shim over the UNMODIFIED reference library (/root/reference/proj/src,
// compiled by oracle/Makefile into oracle/_ref/libchebpr_ref.so).  Only tests/,
// __graft_entry__.smoke() and bench.py's CPU legs (cpu_baseline, --impl reference)
// load it, as the checker / the reference arm.  Status codes mirror
// include/chebpr_cuda.h so that the Python error mapping is shared.
#include <chrono>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <stdexcept>
#include <string>
#include <vector>

#include "chebpr/coefficients.hpp"
#include "chebpr/cpaa.hpp"
#include "chebpr/csv.hpp"
#include "chebpr/errors.hpp"
#include "chebpr/generate.hpp"
#include "chebpr/graph.hpp"
#include "chebpr/graph_io.hpp"
#include "chebpr/metrics.hpp"
#include "chebpr/power.hpp"

using namespace chebpr;

namespace {
thread_local std::string g_err;

template <class F>
int guard(F&& f) {
    try {
        f();
        return 0;
    } catch (const ValidationError& e) {
        g_err = e.what();
        return 1;
    } catch (const DomainError& e) {
        g_err = e.what();
        return 2;
    } catch (const NumericError& e) {
        g_err = e.what();
        return 3;
    } catch (const std::invalid_argument& e) {
        g_err = e.what();
        return 4;
    } catch (const CapacityError& e) {
        g_err = e.what();
        return 5;
    } catch (const ParseError& e) {
        g_err = e.what();
        return 8;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 9;
    }
}

EdgeList to_edges(const int64_t* e, int64_t E) {
    EdgeList out(static_cast<size_t>(E));
    for (int64_t i = 0; i < E; ++i) out[static_cast<size_t>(i)] = {e[2 * i], e[2 * i + 1]};
    return out;
}

int64_t* export_edges(const EdgeList& el, int64_t* count) {
    *count = static_cast<int64_t>(el.size());
    auto* out = static_cast<int64_t*>(std::malloc(sizeof(int64_t) * 2 * (el.size() + 1)));
    for (size_t i = 0; i < el.size(); ++i) {
        out[2 * i] = el[i].first;
        out[2 * i + 1] = el[i].second;
    }
    return out;
}

void export_trace(const std::vector<TraceRow>& tr, double* out) {
    if (!out) return;
    for (size_t i = 0; i < tr.size(); ++i) {
        double* r = out + 10 * i;
        r[0] = tr[i].k;
        r[1] = tr[i].c_k;
        r[2] = tr[i].S_k;
        r[3] = tr[i].residual_mass;
        r[4] = tr[i].l1_change;
        r[5] = tr[i].elapsed_ms;
        r[6] = tr[i].mass_T;
        r[7] = tr[i].err;
        r[8] = tr[i].err_l1;
        r[9] = 0.0;
    }
}

Vector from_ptr(const double* p, int64_t n) {
    Vector v(n);
    std::memcpy(v.data(), p, sizeof(double) * static_cast<size_t>(n));
    return v;
}
}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }
void ref_free(void* p) { std::free(p); }

int ref_gnp_edges(int64_t n, double p, uint64_t seed, int64_t** edges, int64_t* count) {
    return guard([&] { *edges = export_edges(gnp_edges(n, p, seed), count); });
}
int ref_ring_edges(int64_t n, int64_t** edges, int64_t* count) {
    return guard([&] { *edges = export_edges(ring_edges(n), count); });
}
int ref_star_edges(int64_t n, int64_t** edges, int64_t* count) {
    return guard([&] { *edges = export_edges(star_edges(n), count); });
}
int ref_regular_edges(int64_t n, int64_t k, int64_t** edges, int64_t* count) {
    return guard([&] { *edges = export_edges(regular_edges(n, k), count); });
}

// Graph handle = heap UndirectedGraph.
int ref_build_graph(const int64_t* edges, int64_t E, int dedup, int drop_isolated,
                    int64_t n_hint, void** handle, int64_t* stats /* n,m,nnz,dups,dropped */) {
    return guard([&] {
        BuildOptions o;
        o.dedup = dedup != 0;
        o.drop_isolated = drop_isolated != 0;
        o.n_hint = n_hint;
        BuildResult r = build_graph(to_edges(edges, E), o);
        stats[0] = r.graph.n;
        stats[1] = r.graph.m;
        stats[2] = static_cast<int64_t>(r.graph.neighbors.size());
        stats[3] = r.duplicates_removed;
        stats[4] = r.isolated_dropped;
        *handle = new UndirectedGraph(std::move(r.graph));
    });
}

// Graph from raw arrays (lets tests hand-build inconsistent or poisoned graphs,
// as /root/reference/proj/tests/test_cpaa.cpp:371-386 does).
void* ref_graph_from_arrays(int64_t n, int64_t m, const int64_t* offsets, int64_t n_off,
                            const int64_t* neighbors, int64_t nnz, const int64_t* degrees,
                            int64_t n_deg, const double* inv_degree, int64_t n_inv, int multi) {
    auto* g = new UndirectedGraph();
    g->n = n;
    g->m = m;
    g->offsets.assign(offsets, offsets + n_off);
    g->neighbors.assign(neighbors, neighbors + nnz);
    g->degrees.assign(degrees, degrees + n_deg);
    g->inv_degree.assign(inv_degree, inv_degree + n_inv);
    g->multi = multi != 0;
    return g;
}

// load_edge_list / load_matrix_market (graph_io.cpp:50-174) through the reference itself.
// stats: n, m, min_degree, max_degree, self_loops, duplicates_removed, isolated_dropped, nnz.
int ref_load(const char* path, int format, int dedup, int drop_isolated, int symmetrize, void** handle,
             int64_t* stats, double* avg_degree) {
    return guard([&] {
        LoadOptions o;
        o.dedup = dedup != 0;
        o.drop_isolated = drop_isolated != 0;
        o.symmetrize = symmetrize != 0;
        LoadedGraph lg = format == 0 ? load_edge_list(path, o) : load_matrix_market(path, o);
        stats[0] = lg.stats.n;
        stats[1] = lg.stats.m;
        stats[2] = lg.stats.min_degree;
        stats[3] = lg.stats.max_degree;
        stats[4] = lg.stats.self_loops;
        stats[5] = lg.stats.duplicates_removed;
        stats[6] = lg.stats.isolated_dropped;
        stats[7] = static_cast<int64_t>(lg.graph.neighbors.size());
        *avg_degree = lg.stats.avg_degree;
        *handle = new UndirectedGraph(std::move(lg.graph));
    });
}

void ref_graph_free(void* h) { delete static_cast<UndirectedGraph*>(h); }

void ref_graph_get(void* h, int64_t* offsets, int64_t* neighbors, int64_t* degrees,
                   double* inv_degree) {
    const auto& g = *static_cast<UndirectedGraph*>(h);
    if (offsets) std::memcpy(offsets, g.offsets.data(), sizeof(int64_t) * g.offsets.size());
    if (neighbors)
        std::memcpy(neighbors, g.neighbors.data(), sizeof(int64_t) * g.neighbors.size());
    if (degrees) std::memcpy(degrees, g.degrees.data(), sizeof(int64_t) * g.degrees.size());
    if (inv_degree)
        std::memcpy(inv_degree, g.inv_degree.data(), sizeof(double) * g.inv_degree.size());
}

int ref_validate(void* h, int64_t* stats /* n,m,min,max,loops */) {
    return guard([&] {
        GraphStats st = validate(*static_cast<UndirectedGraph*>(h));
        stats[0] = st.n;
        stats[1] = st.m;
        stats[2] = st.min_degree;
        stats[3] = st.max_degree;
        stats[4] = st.self_loops;
    });
}

// trace_out: rounds x 10 doubles (k,c_k,S_k,residual,l1,elapsed,mass_T,err,err_l1,0).
int ref_run_cpaa(void* h, double c, int rounds, double eps, int max_rounds, int parallelism,
                 const double* reference, double* ranks, double* trace_out, int* rounds_out,
                 double* total_mass, double* wall_ms) {
    return guard([&] {
        const auto& g = *static_cast<UndirectedGraph*>(h);
        SolverConfig cfg;
        cfg.c = c;
        cfg.rounds = rounds;
        cfg.eps = eps;
        cfg.max_rounds = max_rounds;
        cfg.parallelism = parallelism;
        Vector refv;
        if (reference) refv = from_ptr(reference, g.n);
        auto t0 = std::chrono::steady_clock::now();
        PageRankResult r = run_cpaa(g, cfg, reference ? &refv : nullptr);
        auto t1 = std::chrono::steady_clock::now();
        if (wall_ms) *wall_ms = std::chrono::duration<double, std::milli>(t1 - t0).count();
        std::memcpy(ranks, r.ranks.data(), sizeof(double) * static_cast<size_t>(g.n));
        export_trace(r.trace, trace_out);
        *rounds_out = r.rounds;
        *total_mass = r.total_mass;
    });
}

int ref_run_power(void* h, double c, int rounds, double tol, int max_rounds, int parallelism,
                  const double* reference, double* ranks, double* trace_out, int* rounds_out,
                  double* total_mass, double* wall_ms) {
    return guard([&] {
        const auto& g = *static_cast<UndirectedGraph*>(h);
        PowerConfig cfg;
        cfg.c = c;
        cfg.rounds = rounds;
        cfg.tol = tol;
        cfg.max_rounds = max_rounds;
        cfg.parallelism = parallelism;
        Vector refv;
        if (reference) refv = from_ptr(reference, g.n);
        auto t0 = std::chrono::steady_clock::now();
        PageRankResult r = run_power(g, cfg, reference ? &refv : nullptr);
        auto t1 = std::chrono::steady_clock::now();
        if (wall_ms) *wall_ms = std::chrono::duration<double, std::milli>(t1 - t0).count();
        std::memcpy(ranks, r.ranks.data(), sizeof(double) * static_cast<size_t>(g.n));
        export_trace(r.trace, trace_out);
        *rounds_out = r.rounds;
        *total_mass = r.total_mass;
    });
}

int ref_transition_apply(void* h, const double* x, int64_t nx, double* y) {
    return guard([&] {
        Vector out = transition_apply(*static_cast<UndirectedGraph*>(h), from_ptr(x, nx));
        std::memcpy(y, out.data(), sizeof(double) * static_cast<size_t>(out.size()));
    });
}

// Staged API: state arrays are caller-owned (n doubles each).
int ref_staged_run(void* h, double c, int M, double* acc_out, double* total_out) {
    return guard([&] {
        const auto& g = *static_cast<UndirectedGraph*>(h);
        CoefficientTable t = coefficients(c, M);
        IterationState st = init_state(g, t.c0);
        for (int k = 1; k <= M; ++k) {
            generate_stage(g, st);
            accumulate_stage(st, t.coeffs[static_cast<size_t>(k)]);
            st.T_prev.swap(st.T_curr);
            st.T_curr.swap(st.T_next);
            st.k = k + 1;
        }
        std::memcpy(acc_out, st.acc.data(), sizeof(double) * static_cast<size_t>(g.n));
        *total_out = kahan_sum(st.acc);
    });
}

int ref_dense_direct_solve(void* h, double c, double* out) {
    return guard([&] {
        Vector x = dense_direct_solve(*static_cast<UndirectedGraph*>(h), c);
        std::memcpy(out, x.data(), sizeof(double) * static_cast<size_t>(x.size()));
    });
}

int ref_coefficients(double c, int M, double* coeffs, double* beta_out, double* c0_out) {
    return guard([&] {
        CoefficientTable t = coefficients(c, M);
        std::memcpy(coeffs, t.coeffs.data(), sizeof(double) * t.coeffs.size());
        *beta_out = t.beta;
        *c0_out = t.c0;
    });
}

int ref_plan_iterations(double c, double eps, int* M, double* predicted) {
    return guard([&] {
        ApproxPlan p = plan_iterations(c, eps);
        *M = p.M;
        *predicted = p.predicted_err;
    });
}

int ref_err_bound(double c, int M, double* out) {
    return guard([&] { *out = err_bound(c, M); });
}

int ref_partition_vertices(void* h, int K, int64_t* cuts /* K+1 */) {
    return guard([&] {
        auto r = partition_vertices(*static_cast<UndirectedGraph*>(h), K);
        for (int j = 0; j < K; ++j) cuts[j] = r[static_cast<size_t>(j)].begin;
        cuts[K] = r.empty() ? 0 : r.back().end;
    });
}

double ref_kahan_sum(const double* x, int64_t n) { return kahan_sum(x, n); }

// The reference's own CSV writers (src/csv.cpp) and edge-list writer (src/generate.cpp:89-97),
// for byte-level parity of the CLI outputs.  algo 0 = run_cpaa, 1 = run_power.
int ref_solve_to_csv(void* h, int algo, double c, int rounds, double eps, int max_rounds,
                     const char* ranks_path, const char* trace_path) {
    return guard([&] {
        const auto& g = *static_cast<UndirectedGraph*>(h);
        PageRankResult r;
        if (algo == 0) {
            SolverConfig cfg;
            cfg.c = c;
            cfg.rounds = rounds;
            cfg.eps = eps;
            cfg.max_rounds = max_rounds;
            r = run_cpaa(g, cfg);
            if (trace_path && *trace_path) write_cpaa_trace_csv(trace_path, r.trace, r.has_err);
        } else {
            PowerConfig cfg;
            cfg.c = c;
            cfg.rounds = rounds;
            cfg.tol = eps;
            cfg.max_rounds = max_rounds;
            r = run_power(g, cfg);
            if (trace_path && *trace_path) write_power_trace_csv(trace_path, r.trace, r.has_err);
        }
        if (ranks_path && *ranks_path) write_ranks_csv(ranks_path, r.ranks);
    });
}

int ref_write_edges(const int64_t* edges, int64_t E, const char* path, const char* comment) {
    return guard([&] { write_edge_list(path, to_edges(edges, E), comment); });
}

}  // extern "C"
