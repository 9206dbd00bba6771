// C++ drop-in layer: the reference's public API (/root/reference/proj/include/chebpr/*.hpp)
// implemented over the C-ABI of libchebpr_b200 (include/chebpr_cuda.h).  Compute runs on
// the B200; host code here only marshals the reference's value types, re-throws the
// C-ABI status codes as the reference's exception types (errors.hpp:11-33), and provides
// the host-only pieces the reference keeps on the host (validate, the metrics test oracle,
// loaders, generators' writers).  Built as libchebpr_dropin.so.
#include <algorithm>
#include <cctype>
#include <charconv>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstddef>
#include <cstring>
#include <fstream>
#include <limits>
#include <sstream>
#include <string>
#include <type_traits>
#include <vector>

#include "chebpr/coefficients.hpp"
#include "chebpr/compare.hpp"
#include "chebpr/cpaa.hpp"
#include "chebpr/errors.hpp"
#include "chebpr/generate.hpp"
#include "chebpr/graph.hpp"
#include "chebpr/graph_io.hpp"
#include "chebpr/metrics.hpp"
#include "chebpr/power.hpp"
#include "chebpr_cuda.h"

namespace chebpr {

namespace {

[[noreturn]] void raise(cheb_status s, const char* msg_override = nullptr) {
    const std::string msg = msg_override ? msg_override : cheb_last_error();
    switch (s) {
        case CHEB_VALIDATION: throw ValidationError(msg);
        case CHEB_DOMAIN: throw DomainError(msg);
        case CHEB_NUMERIC: throw NumericError(msg);
        case CHEB_INVALID_ARG: throw std::invalid_argument(msg);
        case CHEB_CAPACITY: throw CapacityError(msg);
        case CHEB_PARSE: throw ParseError(msg);
        default: throw DeviceError(msg);
    }
}

void check(cheb_status s) {
    if (s != CHEB_OK) raise(s);
}

void check_gen(cheb_status s) {
    if (s != CHEB_OK) raise(s, cheb_gen_last_error());
}

// Device copy of a host graph for the duration of one call (the reference API is
// stateless and its graphs are mutable, so every call uploads).
struct Device {
    cheb_graph_t h = nullptr;
    Device(const UndirectedGraph& g, int device) {
        // the C-ABI reads a null inv_degree as "canonical 1/deg"; the reference's
        // essential_check (cpaa.cpp:18-22) rejects a graph whose inv_degree is missing
        if (g.n >= 1 && g.inv_degree.size() != static_cast<size_t>(g.n))
            throw ValidationError("inconsistent graph arrays");
        check(cheb_graph_upload_csr(g.offsets.data(), (int64_t)g.offsets.size(), g.neighbors.data(),
                                    (int64_t)g.neighbors.size(), g.degrees.data(), (int64_t)g.degrees.size(),
                                    g.inv_degree.data(), (int64_t)g.inv_degree.size(), g.n, g.m,
                                    g.multi ? 1 : 0, device, 0, &h));
    }
    ~Device() { cheb_graph_free(h); }
    Device(const Device&) = delete;
    Device& operator=(const Device&) = delete;
};

// Mode::Auto: bit-exact up to kAutoExactNnz entries, FAST above; the environment variable
// CHEBPR_MODE=fast|bitexact pins Auto to one schedule (so the reference's own suites can be
// run on the FAST kernel too, tests/test_reference_suites.py).
int resolve_mode(Mode m, const UndirectedGraph& g) {
    if (m == Mode::Fast) return CHEB_MODE_FAST;
    if (m == Mode::BitExact) return CHEB_MODE_BITEXACT;
    if (const char* env = std::getenv("CHEBPR_MODE")) {
        if (std::strcmp(env, "fast") == 0) return CHEB_MODE_FAST;
        if (std::strcmp(env, "bitexact") == 0) return CHEB_MODE_BITEXACT;
    }
    return (int64_t)g.neighbors.size() <= kAutoExactNnz ? CHEB_MODE_BITEXACT : CHEB_MODE_FAST;
}

TraceRow to_row(const cheb_trace_row& r) {
    TraceRow t;
    t.k = r.k;
    t.c_k = r.c_k;
    t.S_k = r.S_k;
    t.residual_mass = r.residual_mass;
    t.l1_change = r.l1_change;
    t.elapsed_ms = r.elapsed_ms;
    t.mass_T = r.mass_T;
    t.err = r.err;
    t.err_l1 = r.err_l1;
    return t;
}

EdgeList unpack(int64_t* e, int64_t E) {
    EdgeList out(static_cast<size_t>(E));
    for (int64_t i = 0; i < E; ++i) out[static_cast<size_t>(i)] = {e[2 * i], e[2 * i + 1]};
    cheb_free(e);
    return out;
}

}  // namespace

// ---------------------------------------------------------------- coefficients.hpp
double beta(double c) {
    double o;
    check(cheb_beta(c, &o));
    return o;
}
double sigma(double c) {
    double o;
    check(cheb_sigma(c, &o));
    return o;
}
double err_bound(double c, int M) {
    double o;
    check(cheb_err_bound(c, M, &o));
    return o;
}
ApproxPlan plan_iterations(double c, double eps) {
    ApproxPlan p;
    check(cheb_plan_iterations(c, eps, &p.M, &p.predicted_err));
    p.target_err = eps;
    return p;
}
CoefficientTable coefficients(double c, int M) {
    CoefficientTable t;
    t.c = c;
    if (M < 0) {  // domain errors come from the C-ABI with the reference's text
        double b, c0;
        check(cheb_coefficients(c, M, nullptr, &b, &c0));
    }
    t.coeffs.assign(static_cast<size_t>(std::max(M, 0)) + 1, 0.0);
    check(cheb_coefficients(c, M, t.coeffs.data(), &t.beta, &t.c0));
    return t;
}

namespace {
// Adaptive Simpson on f(t) = cos(k t) / (1 - c cos t) over [0, pi], with Richardson
// correction, a depth cap and a global evaluation budget (so an unreachable tolerance
// fails loudly instead of spinning).
struct Quad {
    double c;
    int k;
    int64_t evals = 0;
    double f(double t) const { return std::cos(k * t) / (1.0 - c * std::cos(t)); }
    double step(double a, double fa, double b, double fb, double m, double fm, double whole, double tol,
                int depth) {
        evals += 2;
        if (depth > 60 || evals > 50000000)
            throw NumericError("coefficient quadrature did not converge for k=" + std::to_string(k));
        const double lm = 0.5 * (a + m), rm = 0.5 * (m + b);
        const double flm = f(lm), frm = f(rm);
        const double left = (m - a) / 6.0 * (fa + 4.0 * flm + fm);
        const double right = (b - m) / 6.0 * (fm + 4.0 * frm + fb);
        const double diff = left + right - whole;
        if (std::abs(diff) <= 15.0 * tol) return left + right + diff / 15.0;
        return step(a, fa, m, fm, lm, flm, left, 0.5 * tol, depth + 1) +
               step(m, fm, b, fb, rm, frm, right, 0.5 * tol, depth + 1);
    }
};
}  // namespace

CoefficientTable coefficients_quadrature(double c, int M, double tol) {
    CoefficientTable t;
    t.beta = beta(c);  // domain check on c (DomainError)
    if (M < 0) throw DomainError("coefficient count must be non-negative");
    if (!(tol > 0.0)) throw DomainError("quadrature tolerance must be positive");
    t.c = c;
    t.coeffs.resize(static_cast<size_t>(M) + 1);
    const double pi = 3.14159265358979323846;
    int64_t budget = 0;
    for (int k = 0; k <= M; ++k) {
        Quad q{c, k, budget};
        const double fa = q.f(0.0), fb = q.f(pi), fm = q.f(0.5 * pi);
        const double whole = pi / 6.0 * (fa + 4.0 * fm + fb);
        t.coeffs[static_cast<size_t>(k)] = 2.0 / pi * q.step(0.0, fa, pi, fb, 0.5 * pi, fm, whole, tol, 0);
        budget = q.evals;
    }
    t.c0 = t.coeffs[0];
    return t;
}

// ---------------------------------------------------------------- graph.hpp
namespace {
// Host copy of a device graph (graph.hpp:21-31 arrays); frees the handle.
UndirectedGraph host_graph(cheb_graph_t h) {
    cheb_graph_info info;
    cheb_status s = cheb_graph_get_info(h, &info);
    if (s != CHEB_OK) {
        cheb_graph_free(h);
        check(s);
    }
    UndirectedGraph g;
    g.n = info.n;
    g.m = info.m;
    g.multi = info.multi != 0;
    g.offsets.resize(static_cast<size_t>(info.n) + 1);
    g.neighbors.resize(static_cast<size_t>(info.nnz));
    g.degrees.resize(static_cast<size_t>(info.n));
    s = cheb_graph_download_csr(h, g.offsets.data(), g.neighbors.data(), g.degrees.data());
    cheb_graph_free(h);
    check(s);
    if (info.n == 0) g.offsets.assign(1, 0);
    g.inv_degree.resize(static_cast<size_t>(info.n));
    for (size_t v = 0; v < g.degrees.size(); ++v) g.inv_degree[v] = 1.0 / static_cast<double>(g.degrees[v]);
    return g;
}
}  // namespace

BuildResult build_graph(const std::vector<std::pair<int64_t, int64_t>>& edges, const BuildOptions& opts) {
    // std::pair<int64_t, int64_t> is two adjacent int64 (standard layout, no padding): the
    // edge vector already is the interleaved (a0, b0, a1, b1, ...) array the C-ABI takes
    static_assert(std::is_standard_layout_v<std::pair<int64_t, int64_t>> &&
                      sizeof(std::pair<int64_t, int64_t>) == 2 * sizeof(int64_t),
                  "std::pair<int64_t, int64_t> must be two adjacent int64");
    static const int64_t none[2] = {0, 0};
    const int64_t* flat = edges.empty() ? none : &edges.front().first;
    cheb_build_opts o;
    cheb_build_opts_default(&o);
    o.dedup = opts.dedup ? 1 : 0;
    o.drop_isolated = opts.drop_isolated ? 1 : 0;
    o.n_hint = opts.n_hint;
    o.device = opts.device;
    cheb_graph_t h = nullptr;
    cheb_graph_info info;
    check(cheb_graph_build(flat, (int64_t)edges.size(), &o, &h, &info));
    BuildResult r;
    r.graph = host_graph(h);
    r.duplicates_removed = info.duplicates_removed;
    r.isolated_dropped = info.isolated_dropped;
    return r;
}

Vector transition_apply(const UndirectedGraph& g, const Vector& x) {
    if (x.size() != g.n)
        throw std::invalid_argument("vector length " + std::to_string(x.size()) +
                                    " does not match vertex count " + std::to_string(g.n));
    Vector y(g.n);
    if (g.n == 0) return y;
    Device d(g, 0);
    check(cheb_transition_apply(d.h, x.data(), (int64_t)x.size(), y.data(), resolve_mode(Mode::Auto, g)));
    return y;
}

GraphStats validate(const UndirectedGraph& g, int64_t duplicates_removed, int64_t isolated_dropped) {
    // graph.cpp:123-186 on the device (cheb_validate_csr): same check order and messages
    if (g.n < 0) throw ValidationError("negative vertex count");
    if (g.offsets.size() != static_cast<size_t>(g.n) + 1) throw ValidationError("offsets length is not n+1");
    cheb_graph_stats s;
    check(cheb_validate_csr(g.offsets.data(), (int64_t)g.offsets.size(), g.neighbors.data(),
                            (int64_t)g.neighbors.size(), g.degrees.data(), (int64_t)g.degrees.size(), g.n, g.m,
                            g.multi ? 1 : 0, duplicates_removed, isolated_dropped, 0, &s));
    GraphStats st;
    st.n = s.n;
    st.m = s.m;
    st.avg_degree = s.avg_degree;
    st.min_degree = s.min_degree;
    st.max_degree = s.max_degree;
    st.self_loops = s.self_loops;
    st.duplicates_removed = s.duplicates_removed;
    st.isolated_dropped = s.isolated_dropped;
    return st;
}

double kahan_sum(const double* x, int64_t n) { return cheb_kahan_sum(x, n); }
double kahan_sum(const Vector& x) { return cheb_kahan_sum(x.data(), (int64_t)x.size()); }

// ---------------------------------------------------------------- cpaa.hpp
std::vector<VertexRange> partition_vertices(const UndirectedGraph& g, int K) {
    std::vector<int64_t> cuts(static_cast<size_t>(std::max(K, 0)) + 1);
    check(cheb_partition_vertices(g.degrees.data(), g.n, K, cuts.data()));
    std::vector<VertexRange> r(static_cast<size_t>(K));
    for (int j = 0; j < K; ++j) r[j] = {cuts[j], cuts[j + 1]};
    return r;
}

Vector normalize(const Vector& v) {
    const double total = kahan_sum(v);
    if (!std::isfinite(total) || total <= 0.0) throw NumericError("normalization total is not positive and finite");
    Vector out(v.size());
    for (int64_t i = 0; i < (int64_t)v.size(); ++i) out[i] = v[i] / total;
    return out;
}

PageRankResult run_cpaa(const UndirectedGraph& g, const SolverConfig& cfg, const Vector* reference) {
    if (g.n < 1) throw ValidationError("graph has no vertices");
    Device d(g, cfg.device);
    cheb_cpaa_opts o;
    cheb_cpaa_opts_default(&o);
    o.c = cfg.c;
    o.rounds = cfg.rounds;
    o.eps = cfg.eps;
    o.max_rounds = cfg.max_rounds;
    o.parallelism = cfg.parallelism;
    o.mode = cfg.precision == 32 && cfg.mode == Mode::Auto ? CHEB_MODE_FAST : resolve_mode(cfg.mode, g);  // bit-exact is fp64 only
    o.precision = cfg.precision;
    const int cap = std::max({cfg.rounds, cfg.max_rounds, 1}) + 1;
    std::vector<cheb_trace_row> tr(static_cast<size_t>(cap));
    PageRankResult r;
    r.ranks.resize(g.n);
    check(cheb_cpaa(d.h, &o, reference ? reference->data() : nullptr, reference ? (int64_t)reference->size() : 0,
                    r.ranks.data(), tr.data(), &r.rounds, &r.total_mass));
    r.has_err = reference != nullptr;
    for (int k = 0; k < r.rounds; ++k) r.trace.push_back(to_row(tr[k]));
    return r;
}

IterationState init_state(const UndirectedGraph& g, double c0) {
    // the reference's essential_check (cpaa.cpp:16-26), then T_{-1} = T_0 = 1, acc = c0/2
    if (g.n < 1) throw ValidationError("graph has no vertices");
    if (g.offsets.size() != static_cast<size_t>(g.n) + 1 || g.degrees.size() != static_cast<size_t>(g.n) ||
        g.inv_degree.size() != static_cast<size_t>(g.n) || (int64_t)g.neighbors.size() != g.offsets[g.n])
        throw ValidationError("inconsistent graph arrays");
    for (int64_t v = 0; v < g.n; ++v)
        if (g.degrees[v] < 1) throw ValidationError("vertex " + std::to_string(v) + " is isolated (degree 0)");
    IterationState st;
    st.T_prev = Vector::Ones(g.n);
    st.T_curr = Vector::Ones(g.n);
    st.T_next = Vector::Zero(g.n);
    st.acc = Vector::Constant(g.n, c0 / 2.0);
    st.k = 1;
    return st;
}

void generate_stage(const UndirectedGraph& g, IterationState& state) {
    // one SpMV-shaped pass on the device with the fused solver's arithmetic (same mode
    // rule), so a staged loop reproduces run_cpaa bit for bit
    Device d(g, 0);
    check(cheb_state_init(d.h, 0.0, resolve_mode(Mode::Auto, g)));
    check(cheb_state_set(d.h, state.T_prev.data(), state.T_curr.data(), state.acc.data(), state.k));
    check(cheb_state_generate(d.h));
    state.T_next.resize(g.n);
    int k = 0;
    check(cheb_state_get(d.h, nullptr, nullptr, state.T_next.data(), nullptr, &k));
}

void accumulate_stage(IterationState& state, double c_k) {
    // acc += c_k T_next with a separate multiply and add: the device epilogue's rounding
    for (int64_t i = 0; i < (int64_t)state.acc.size(); ++i) {
        const double term = c_k * state.T_next[i];
        state.acc[i] = state.acc[i] + term;
    }
}

// ---------------------------------------------------------------- power.hpp
PageRankResult run_power(const UndirectedGraph& g, const PowerConfig& cfg, const Vector* reference) {
    if (g.n < 1) throw ValidationError("graph has no vertices");
    Device d(g, cfg.device);
    cheb_power_opts o;
    cheb_power_opts_default(&o);
    o.c = cfg.c;
    o.rounds = cfg.rounds;
    o.tol = cfg.tol;
    o.max_rounds = cfg.max_rounds;
    o.parallelism = cfg.parallelism;
    o.mode = resolve_mode(cfg.mode, g);
    const int cap = std::max(cfg.rounds >= 0 ? cfg.rounds : cfg.max_rounds, 1);
    std::vector<cheb_trace_row> tr(static_cast<size_t>(cap));
    PageRankResult r;
    r.ranks.resize(g.n);
    check(cheb_power(d.h, &o, reference ? reference->data() : nullptr, reference ? (int64_t)reference->size() : 0,
                     r.ranks.data(), tr.data(), cap, &r.rounds, &r.total_mass));
    r.has_err = reference != nullptr;
    for (int k = 0; k < r.rounds && k < cap; ++k) r.trace.push_back(to_row(tr[k]));
    return r;
}

Vector reference_pagerank(const UndirectedGraph& g, double c) {
    PowerConfig cfg;
    cfg.c = c;
    cfg.rounds = 210;
    cfg.parallelism = 1;
    return run_power(g, cfg).ranks;
}

// ---------------------------------------------------------------- metrics.hpp
ErrorReport max_relative_error(const Vector& est, const Vector& ref) {
    if (est.size() != ref.size()) throw std::invalid_argument("estimate and reference lengths differ");
    ErrorReport rep;
    double l1 = 0.0, lost = 0.0;
    for (int64_t i = 0; i < (int64_t)ref.size(); ++i) {
        if (!(ref[i] > 0.0)) throw DomainError("reference entry " + std::to_string(i) + " is not positive");
        const double d = std::abs(est[i] - ref[i]);
        rep.max_rel_err = std::max(rep.max_rel_err, d / ref[i]);
        const double y = d - lost, t = l1 + y;
        lost = (t - l1) - y;
        l1 = t;
    }
    rep.l1_err = l1;
    rep.mass_gap = std::abs(kahan_sum(est) - 1.0);
    return rep;
}

Vector dense_direct_solve(const UndirectedGraph& g, double c) {
    // (I - c P) x = (1-c)/n e by partial-pivot Gaussian elimination, then normalise
    if (g.n > 512) throw CapacityError("dense solve limited to n <= 512, got " + std::to_string(g.n));
    if (!(c > 0.0 && c < 1.0)) throw DomainError("damping factor must lie in (0,1)");
    const int64_t n = g.n;
    std::vector<double> A(static_cast<size_t>(n * n), 0.0);
    auto at = [&](int64_t i, int64_t j) -> double& { return A[static_cast<size_t>(i * n + j)]; };
    for (int64_t i = 0; i < n; ++i) at(i, i) = 1.0;
    for (int64_t u = 0; u < n; ++u)
        for (int64_t i = g.offsets[u]; i < g.offsets[u + 1]; ++i) at(u, g.neighbors[i]) -= c * g.inv_degree[g.neighbors[i]];
    const std::vector<double> A0 = A;
    std::vector<double> b(static_cast<size_t>(n), (1.0 - c) / static_cast<double>(n)), x = b;
    std::vector<int64_t> piv(static_cast<size_t>(n));
    for (int64_t k = 0; k < n; ++k) {
        int64_t p = k;
        for (int64_t i = k + 1; i < n; ++i)
            if (std::abs(at(i, k)) > std::abs(at(p, k))) p = i;
        if (p != k) {
            for (int64_t j = 0; j < n; ++j) std::swap(at(k, j), at(p, j));
            std::swap(x[k], x[p]);
        }
        for (int64_t i = k + 1; i < n; ++i) {
            const double f = at(k, k) != 0.0 ? at(i, k) / at(k, k) : 0.0;
            if (f == 0.0) continue;
            for (int64_t j = k; j < n; ++j) at(i, j) -= f * at(k, j);
            x[i] -= f * x[k];
        }
    }
    for (int64_t i = n - 1; i >= 0; --i) {
        double s = x[i];
        for (int64_t j = i + 1; j < n; ++j) s -= at(i, j) * x[j];
        x[i] = s / at(i, i);
    }
    double resid = 0.0;
    for (int64_t i = 0; i < n; ++i) {
        double s = 0.0;
        for (int64_t j = 0; j < n; ++j) s += A0[static_cast<size_t>(i * n + j)] * x[j];
        resid = std::max(resid, std::abs(s - b[i]));
    }
    if (!(resid <= 1e-10)) throw NumericError("dense solve residual " + std::to_string(resid) + " exceeds 1e-10");
    Vector out(n);
    for (int64_t i = 0; i < n; ++i) out[i] = x[i];
    const double total = kahan_sum(out);
    if (!std::isfinite(total) || total <= 0.0) throw NumericError("dense solve produced a non-normalizable vector");
    for (int64_t i = 0; i < n; ++i) out[i] /= total;
    return out;
}

double symmetry_similarity_check(const UndirectedGraph& g) {
    if (g.n > 2048) throw CapacityError("similarity check limited to n <= 2048, got " + std::to_string(g.n));
    const int64_t n = g.n;
    std::vector<double> S(static_cast<size_t>(n * n), 0.0);
    for (int64_t u = 0; u < n; ++u)
        for (int64_t i = g.offsets[u]; i < g.offsets[u + 1]; ++i) {
            const int64_t v = g.neighbors[i];
            const double d = static_cast<double>(g.degree(u)) * static_cast<double>(g.degree(v));
            S[static_cast<size_t>(u * n + v)] += 1.0 / std::sqrt(d);
        }
    double worst = 0.0;
    for (int64_t i = 0; i < n; ++i)
        for (int64_t j = i + 1; j < n; ++j)
            worst = std::max(worst, std::abs(S[static_cast<size_t>(i * n + j)] - S[static_cast<size_t>(j * n + i)]));
    return worst;
}

double mass_check(const Vector& vec, double expected) { return std::abs(kahan_sum(vec) - expected); }

// ---------------------------------------------------------------- compare.hpp
std::vector<CompareRow> compare_algorithms(const UndirectedGraph& g, const CompareOptions& opts) {
    if (!(opts.eps > 0.0)) throw DomainError("eps must be positive");
    if (opts.parallelism.empty()) throw DomainError("parallelism list is empty");
    const Vector ref = reference_pagerank(g, opts.c);
    auto summarize = [&](const std::string& algo, int K, const std::vector<TraceRow>& tr) {
        CompareRow row;
        row.algo = algo;
        row.parallelism = K;
        double elapsed = 0.0;
        for (const TraceRow& t : tr) {
            elapsed += t.elapsed_ms;
            row.err = t.err;
            row.l1 = t.err_l1;
            row.elapsed_ms = elapsed;
            if (t.err < opts.eps) {
                row.rounds = t.k;
                return row;
            }
        }
        row.rounds = -1;
        return row;
    };
    std::vector<CompareRow> rows;
    for (int K : opts.parallelism) {
        SolverConfig cfg;
        cfg.c = opts.c;
        cfg.rounds = opts.cpaa_budget;
        cfg.max_rounds = opts.cpaa_budget;
        cfg.parallelism = K;
        rows.push_back(summarize("cpaa", K, run_cpaa(g, cfg, &ref).trace));
    }
    for (int K : opts.parallelism) {
        PowerConfig cfg;
        cfg.c = opts.c;
        cfg.rounds = opts.power_budget;
        cfg.parallelism = K;
        rows.push_back(summarize("power", K, run_power(g, cfg, &ref).trace));
    }
    return rows;
}

// ---------------------------------------------------------------- generate.hpp
int64_t Rng::below(int64_t bound) {
    const uint64_t b = static_cast<uint64_t>(bound);
    const uint64_t limit = std::numeric_limits<uint64_t>::max() - std::numeric_limits<uint64_t>::max() % b;
    for (;;) {
        const uint64_t r = eng();
        if (r < limit) return static_cast<int64_t>(r % b);
    }
}

EdgeList ring_edges(int64_t n) {
    int64_t* e = nullptr;
    int64_t E = 0;
    check_gen(cheb_gen_ring(n, &e, &E));
    return unpack(e, E);
}
EdgeList star_edges(int64_t n) {
    int64_t* e = nullptr;
    int64_t E = 0;
    check_gen(cheb_gen_star(n, &e, &E));
    return unpack(e, E);
}
EdgeList regular_edges(int64_t n, int64_t k) {
    int64_t* e = nullptr;
    int64_t E = 0;
    check_gen(cheb_gen_regular(n, k, &e, &E));
    return unpack(e, E);
}
EdgeList gnp_edges(int64_t n, double p, uint64_t seed) {
    int64_t* e = nullptr;
    int64_t E = 0;
    check_gen(cheb_gen_gnp(n, p, seed, &e, &E));
    return unpack(e, E);
}

static EdgeList unpack32(void* e, int64_t E) {
    EdgeList out(static_cast<size_t>(E));
    const int32_t* p = static_cast<const int32_t*>(e);
    for (int64_t i = 0; i < E; ++i) out[static_cast<size_t>(i)] = {p[2 * i], p[2 * i + 1]};
    cheb_free(e);
    return out;
}
EdgeList rmat_edges(int scale, int64_t edge_factor, double a, double b, double c, uint64_t seed) {
    void* e = nullptr;
    int64_t E = 0;
    check_gen(cheb_gen_rmat(scale, edge_factor, a, b, c, seed, 0, 0, &e, &E));
    return unpack32(e, E);
}
EdgeList chung_lu_edges(int64_t n, double gamma, double wmin, double wmax, int64_t draws, uint64_t seed) {
    void* e = nullptr;
    int64_t E = 0;
    check_gen(cheb_gen_chung_lu(n, gamma, wmin, wmax, draws, seed, 0, 0, &e, &E));
    return unpack32(e, E);
}

void write_edge_list(const std::string& path, const EdgeList& edges, const std::string& comment) {
    std::FILE* f = std::fopen(path.c_str(), "wb");
    if (!f) throw ParseError("cannot write " + path);
    if (!comment.empty()) std::fprintf(f, "# %s\n", comment.c_str());
    for (const auto& [a, b] : edges) std::fprintf(f, "%lld %lld\n", (long long)a, (long long)b);
    if (std::fclose(f) != 0) throw ParseError("write failed for " + path);
}

// ---------------------------------------------------------------- graph_io.hpp
// The files are parsed on the GPU (csrc/ingest.cu, cheb_graph_load_*) and built by K1;
// finish()'s warnings (graph_io.cpp:38-40, 134-138) are printed here.
namespace {
LoadedGraph load_on_device(const std::string& path, const LoadOptions& opts, bool matrix_market) {
    cheb_load_opts o;
    cheb_load_opts_default(&o);
    o.dedup = opts.dedup ? 1 : 0;
    o.drop_isolated = opts.drop_isolated ? 1 : 0;
    o.symmetrize = opts.symmetrize ? 1 : 0;
    cheb_graph_t h = nullptr;
    cheb_graph_stats st;
    check(matrix_market ? cheb_graph_load_matrix_market(path.c_str(), &o, &h, &st)
                        : cheb_graph_load_edge_list(path.c_str(), &o, &h, &st));
    if (st.weights_ignored)
        std::fprintf(stderr, "warning: %s: real weights ignored, using pattern only\n", path.c_str());
    if (st.isolated_dropped > 0)
        std::fprintf(stderr, "warning: dropped %lld isolated vertices\n", (long long)st.isolated_dropped);
    LoadedGraph lg;
    lg.graph = host_graph(h);
    lg.stats.n = st.n;
    lg.stats.m = st.m;
    lg.stats.avg_degree = st.avg_degree;
    lg.stats.min_degree = st.min_degree;
    lg.stats.max_degree = st.max_degree;
    lg.stats.self_loops = st.self_loops;
    lg.stats.duplicates_removed = st.duplicates_removed;
    lg.stats.isolated_dropped = st.isolated_dropped;
    return lg;
}
}  // namespace

LoadedGraph load_edge_list(const std::string& path, const LoadOptions& opts) {
    return load_on_device(path, opts, false);
}

LoadedGraph load_matrix_market(const std::string& path, const LoadOptions& opts) {
    return load_on_device(path, opts, true);
}

}  // namespace chebpr
