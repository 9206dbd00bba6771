// extern "C" boundary of libchebpr_b200 (include/chebpr_cuda.h).
//
// Every entry converts internal exceptions into cheb_status + a thread-local message,
// and applies the reference's argument checks in the reference's order
// (/root/reference/proj/src/cpaa.cpp:79-94, power.cpp:28-47), so that the wrappers
// above the C-ABI raise exactly what the reference raises.
#include <algorithm>
#include <cmath>
#include <cstring>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include <nccl.h>

#include "common.cuh"

using namespace chebgpu;

struct cheb_comm {
    ncclComm_t nccl = nullptr;
    int nranks = 1, rank = 0, device = 0;
};

namespace {
thread_local std::string g_last_error;

template <class F>
cheb_status guarded(F&& f) {
    try {
        f();
        return CHEB_OK;
    } catch (const Error& e) {
        g_last_error = e.what();
        return e.code;
    } catch (const std::bad_alloc&) {
        g_last_error = "host allocation failed";
        return CHEB_CAPACITY;
    } catch (const std::exception& e) {
        g_last_error = e.what();
        return CHEB_CUDA;
    }
}

cheb_graph* new_graph(int device) {
    int count = 0;
    if (cudaGetDeviceCount(&count) != cudaSuccess || count == 0)
        fail(CHEB_CUDA, "no CUDA device available (libchebpr_b200 has no CPU fallback)");
    if (device < 0 || device >= count)
        fail(CHEB_INVALID_ARG, "device ordinal " + std::to_string(device) + " out of range");
    auto* g = new cheb_graph();
    g->device = device;
    DeviceGuard dg(device);
    g->stream = pooled_stream(device);
    CHEB_CUDA_CHECK(cudaEventCreate(&g->ev0));
    CHEB_CUDA_CHECK(cudaEventCreate(&g->ev1));
    return g;
}

void fill_info(cheb_graph* g, cheb_graph_info* info) {
    if (!info) return;
    info->n = g->n;
    info->m = g->m;
    info->nnz = g->nnz;
    info->duplicates_removed = g->duplicates_removed;
    info->isolated_dropped = g->isolated_dropped;
    info->max_degree = g->max_degree;
    info->min_degree = g->min_degree;
    info->multi = g->multi ? 1 : 0;
    info->row_ptr_64 = g->rp64 ? 1 : 0;
    info->inv_degree_array = g->inv_array ? 1 : 0;
    info->device = g->device;
}

void need_graph(cheb_graph* g) {
    if (!g) fail(CHEB_INVALID_ARG, "null graph handle");
}

void single_gpu_only(cheb_graph* g) {
    if (g->part.G > 1) fail(CHEB_INVALID_ARG, "operation not available on a partitioned (multi-GPU) handle");
}

// cpaa.cpp:16-26 essential_check, the parts that are not guaranteed by construction.
void essential(cheb_graph* g) {
    if (g->n < 1) fail(CHEB_VALIDATION, "graph has no vertices");
}
}  // namespace

namespace {
std::mutex& stream_pool_mu() {
    static std::mutex m;
    return m;
}
std::vector<std::pair<int, cudaStream_t>>& stream_pool() {
    static auto* v = new std::vector<std::pair<int, cudaStream_t>>();  // never destroyed (exit order)
    return *v;
}
}  // namespace

cudaStream_t chebgpu::pooled_stream(int device) {
    {
        std::lock_guard<std::mutex> lk(stream_pool_mu());
        auto& v = stream_pool();
        for (size_t i = 0; i < v.size(); ++i)
            if (v[i].first == device) {
                cudaStream_t s = v[i].second;
                v[i] = v.back();
                v.pop_back();
                return s;
            }
    }
    cudaStream_t s = nullptr;
    CHEB_CUDA_CHECK(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
    return s;
}

void chebgpu::release_stream(int device, cudaStream_t s) {
    if (!s) return;
    std::lock_guard<std::mutex> lk(stream_pool_mu());
    if (stream_pool().size() < 64) stream_pool().emplace_back(device, s);
    else cudaStreamDestroy(s);
}

void chebgpu::retain_pool_memory() {
    int dev = 0;
    cudaGetDevice(&dev);
    static std::atomic<uint64_t> done{0};
    if (dev < 0 || dev >= 64 || !first_on_device(done, dev)) return;
    cudaMemPool_t pool;
    if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
        uint64_t keep = UINT64_MAX;
        cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
    }
}

bool chebgpu::l2_window(const void* base, size_t bytes, cudaAccessPolicyWindow* w, size_t decide_bytes) {
    // Only when the vector does not fit L2 on its own (config 4: x = 136 MB): reserving
    // persisting L2 otherwise shrinks the normal L2 the other streams use (measured: C2 and
    // C5 slower, C4 12% faster).  The device-wide carve-out follows the decision.
    int dev = 0;
    cudaGetDevice(&dev);
    static size_t persist_max[64] = {}, window_max[64] = {}, l2_size[64] = {}, current[64] = {};
    static bool init[64] = {};
    static std::mutex mu;  // handles on different devices may launch from different threads
    if (dev < 0 || dev >= 64) return false;
    std::lock_guard<std::mutex> lk(mu);
    if (!init[dev]) {
        cudaDeviceProp prop;
        if (cudaGetDeviceProperties(&prop, dev) == cudaSuccess) {
            persist_max[dev] = prop.persistingL2CacheMaxSize;
            window_max[dev] = prop.accessPolicyMaxWindowSize;
            l2_size[dev] = prop.l2CacheSize;
        }
        init[dev] = true;
    }
    const bool use = persist_max[dev] > 0 && window_max[dev] > 0 && (decide_bytes ? decide_bytes : bytes) > l2_size[dev];
    const size_t want = use ? persist_max[dev] : 0;
    if (want != current[dev]) {
        cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, want);
        current[dev] = want;
    }
    if (!use) return false;
    w->base_ptr = const_cast<void*>(base);
    w->num_bytes = std::min({bytes, persist_max[dev], window_max[dev]});
    if (tuning().l2win_mb >= 0) w->num_bytes = std::min(w->num_bytes, (size_t)tuning().l2win_mb << 20);
    w->hitRatio = std::min(1.0f, std::max(0.0f, tuning().l2win_pct / 100.0f));
    w->hitProp = cudaAccessPropertyPersisting;
    w->missProp = cudaAccessPropertyStreaming;
    return true;
}

cheb_graph::~cheb_graph() {
    int prev = -1;
    cudaGetDevice(&prev);
    cudaSetDevice(device);
    if (aux) cudaStreamSynchronize(aux);
    if (stream) cudaStreamSynchronize(stream);
    if (peer) {
        peer->release();
        delete peer;
        peer = nullptr;
    }
    {   // return every buffer to the pool on this graph's stream while it still exists
        row_ptr.release();
        col.release();
        inv.release();
        view = chebgpu::SolverView{};
        if (ws.exec) {
            cudaGraphExecDestroy(ws.exec);
            ws.exec = nullptr;
        }
        ws.release_buffers();
        staged = chebgpu::StagedState{};
        bws = chebgpu::BatchWorkspace{};
    }
    if (ev0) cudaEventDestroy(ev0);
    if (ev1) cudaEventDestroy(ev1);
    release_stream(device, stream);  // idle: synchronised above, buffers returned on it
    release_stream(device, aux);
    if (prev >= 0) cudaSetDevice(prev);
}

extern "C" {

const char* cheb_last_error(void) { return g_last_error.c_str(); }

const char* cheb_version(void) { return "chebpr_b200 0.1 (sm_100a)"; }

int cheb_device_count(void) {
    int c = 0;
    if (cudaGetDeviceCount(&c) != cudaSuccess) return 0;
    return c;
}

cheb_status cheb_beta(double c, double* out) {
    return guarded([&] { *out = beta(c); });
}
cheb_status cheb_sigma(double c, double* out) {
    return guarded([&] { *out = sigma(c); });
}
cheb_status cheb_err_bound(double c, int M, double* out) {
    return guarded([&] { *out = err_bound(c, M); });
}
cheb_status cheb_plan_iterations(double c, double eps, int* M, double* predicted_err) {
    return guarded([&] { *M = plan_iterations(c, eps, predicted_err); });
}
cheb_status cheb_coefficients(double c, int M, double* coeffs, double* beta_out, double* c0) {
    return guarded([&] {
        NvtxRange nvtx_("cheb_coefficients");
        std::vector<double> t;
        coefficients(c, M, t, beta_out, c0);
        if (coeffs) std::memcpy(coeffs, t.data(), sizeof(double) * t.size());
    });
}
cheb_status cheb_resolve_rounds(double c, int rounds, double eps, int max_rounds, int* M) {
    return guarded([&] { *M = resolve_rounds(c, rounds, eps, max_rounds); });
}

double cheb_kahan_sum(const double* x, int64_t n) { return kahan_sum(x, n); }

void cheb_build_opts_default(cheb_build_opts* o) {
    o->dedup = 1;
    o->drop_isolated = 0;
    o->n_hint = 0;
    o->device = 0;
    o->row_ptr_64 = 0;
}

cheb_status cheb_graph_build(const int64_t* edges, int64_t E, const cheb_build_opts* opts,
                             cheb_graph_t* out, cheb_graph_info* info) {
    return guarded([&] {
        NvtxRange nvtx_("cheb_graph_build");
        if (E < 0) fail(CHEB_INVALID_ARG, "negative edge count");
        cheb_build_opts o;
        cheb_build_opts_default(&o);
        if (opts) o = *opts;
        // graph.cpp:27 — the host sees the ids first; reject negatives before any copy.
        for (int64_t i = 0; i < 2 * E; ++i)
            if (edges[i] < 0) fail(CHEB_VALIDATION, "negative vertex id in edge list");
        std::unique_ptr<cheb_graph> g(new_graph(o.device));
        GraphScope gs(g.get());
        DevMem d(sizeof(int64_t) * 2 * std::max<int64_t>(E, 1));
        if (E > 0)
            CHEB_CUDA_CHECK(cudaMemcpyAsync(d.get(), edges, sizeof(int64_t) * 2 * E,
                                            cudaMemcpyHostToDevice, g->stream));
        build_from_edges(g.get(), d.get(), E, 64, o);
        fill_info(g.get(), info);
        *out = g.release();
    });
}

cheb_status cheb_graph_build_device(const void* d_edges, int64_t E, int edge_bits,
                                    const cheb_build_opts* opts, cheb_graph_t* out,
                                    cheb_graph_info* info) {
    return guarded([&] {
        NvtxRange nvtx_("cheb_graph_build_device");
        if (edge_bits != 32 && edge_bits != 64) fail(CHEB_INVALID_ARG, "edge_bits must be 32 or 64");
        cheb_build_opts o;
        cheb_build_opts_default(&o);
        if (opts) o = *opts;
        std::unique_ptr<cheb_graph> g(new_graph(o.device));
        GraphScope gs(g.get());
        build_from_edges(g.get(), d_edges, E, edge_bits, o);
        fill_info(g.get(), info);
        *out = g.release();
    });
}

cheb_status cheb_graph_upload_csr(const int64_t* offsets, int64_t n_offsets,
                                  const int64_t* neighbors, int64_t nnz, const int64_t* degrees,
                                  int64_t n_degrees, const double* inv_degree, int64_t n_inv,
                                  int64_t n, int64_t m, int multi, int device, int row_ptr_64,
                                  cheb_graph_t* out) {
    return guarded([&] {
        NvtxRange nvtx_("cheb_graph_upload_csr");
        // cpaa.cpp:16-26 essential_check, in the reference's order.
        if (n < 1) fail(CHEB_VALIDATION, "graph has no vertices");
        if (n_offsets != n + 1 || n_degrees != n || (inv_degree && n_inv != n) ||
            nnz != offsets[n])
            fail(CHEB_VALIDATION, "inconsistent graph arrays");
        std::unique_ptr<cheb_graph> g(new_graph(device));
        GraphScope gs(g.get());
        g->m = m;
        g->multi = multi != 0;
        g->rp64 = row_ptr_64 != 0;
        g->duplicates_removed = 0;
        g->isolated_dropped = 0;
        // the remaining checks are O(n) host loops: they run while the CSR copies are in
        // flight, split over host threads (each chunk finds its first failing vertex; the
        // lowest one is reported, in the reference's check order)
        auto host_checks = [&] {
            struct Part {
                int64_t isolated = -1, nonmono = -1, dmin = INT64_MAX, dmax = 0;
                bool inv_differs = false;
            };
            const int hw = (int)std::max(1u, std::thread::hardware_concurrency());
            const int T = n >= (int64_t(1) << 18) ? std::min(16, hw) : 1;
            std::vector<Part> parts(T);
            auto scan = [&](int t) {  // one pass over the chunk: every check's first failure
                const int64_t lo = n * t / T, hi = n * (t + 1) / T;
                int64_t isolated = -1, nonmono = -1, dmin = INT64_MAX, dmax = 0;
                bool differs = false;
                for (int64_t v = lo; v < hi; ++v) {
                    if (degrees[v] < 1 && isolated < 0) isolated = v;
                    const int64_t d = offsets[v + 1] - offsets[v];
                    if (d < 0 && nonmono < 0) nonmono = v;
                    dmin = d < dmin ? d : dmin;
                    dmax = d > dmax ? d : dmax;
                    // inv_degree canonical iff every entry is 1.0/row length bitwise (IEEE
                    // division, as graph.cpp:97-99 stores it): then it is never uploaded
                    if (inv_degree) {
                        const double want = 1.0 / (double)d;
                        uint64_t a, b;
                        std::memcpy(&a, &want, 8);
                        std::memcpy(&b, inv_degree + v, 8);
                        differs |= a != b;
                    }
                }
                parts[t] = Part{isolated, nonmono, dmin, dmax, differs};  // locals: no false sharing
            };
            std::vector<std::thread> th;
            for (int t = 1; t < T; ++t) th.emplace_back(scan, t);
            scan(0);
            for (auto& x : th) x.join();
            for (const Part& p : parts)
                if (p.isolated >= 0)
                    fail(CHEB_VALIDATION, "vertex " + std::to_string(p.isolated) + " is isolated (degree 0)");
            if (offsets[0] != 0) fail(CHEB_VALIDATION, "offsets must start at 0");
            int64_t dmin = INT64_MAX, dmax = 0;
            for (const Part& p : parts) {
                if (p.nonmono >= 0)
                    fail(CHEB_VALIDATION, "offsets not monotone at vertex " + std::to_string(p.nonmono));
                dmin = std::min(dmin, p.dmin);
                dmax = std::max(dmax, p.dmax);
            }
            g->min_degree = dmin;
            g->max_degree = dmax;
            for (const Part& p : parts)
                if (p.inv_differs) return false;
            return true;
        };
        upload_csr(g.get(), offsets, neighbors, n, nnz, inv_degree, host_checks);
        *out = g.release();
    });
}

void cheb_load_opts_default(cheb_load_opts* o) {
    o->dedup = 1;
    o->drop_isolated = 0;
    o->symmetrize = 0;
    o->device = 0;
    o->row_ptr_64 = 0;
}

namespace {
void stats_of(cheb_graph* g, cheb_graph_stats* s) {  // graph.cpp:123-186 validate's numbers
    s->n = g->n;
    s->m = g->m;
    s->avg_degree = g->n > 0 ? static_cast<double>(g->m) / static_cast<double>(g->n) : 0.0;
    s->min_degree = g->n > 0 ? g->min_degree : 0;
    s->max_degree = g->n > 0 ? g->max_degree : 0;
    s->self_loops = count_self_loops(g);
    s->duplicates_removed = g->duplicates_removed;
    s->isolated_dropped = g->isolated_dropped;
}

cheb_status load_common(const char* path, const char* text, int64_t bytes, int format,
                        const cheb_load_opts* opts, cheb_graph_t* out, cheb_graph_stats* stats) {
    return guarded([&] {
        if (!path) fail(CHEB_INVALID_ARG, "null path");
        cheb_load_opts o;
        cheb_load_opts_default(&o);
        if (opts) o = *opts;
        std::unique_ptr<cheb_graph> g(new_graph(o.device));
        GraphScope gs(g.get());
        int64_t lines = 0;
        int wi = 0;
        load_graph_text(g.get(), path, text, bytes, format, o, &lines, &wi);
        if (stats) {
            stats_of(g.get(), stats);
            stats->lines = lines;
            stats->weights_ignored = wi;
        }
        *out = g.release();
    });
}
}  // namespace

cheb_status cheb_graph_load_edge_list(const char* path, const cheb_load_opts* opts, cheb_graph_t* out,
                                      cheb_graph_stats* stats) {
    return load_common(path, nullptr, 0, 0, opts, out, stats);
}

cheb_status cheb_graph_load_matrix_market(const char* path, const cheb_load_opts* opts, cheb_graph_t* out,
                                          cheb_graph_stats* stats) {
    return load_common(path, nullptr, 0, 1, opts, out, stats);
}

cheb_status cheb_graph_parse_text(const char* text, int64_t bytes, int format, const char* name,
                                  const cheb_load_opts* opts, cheb_graph_t* out, cheb_graph_stats* stats) {
    if (!text && bytes > 0) return guarded([] { fail(CHEB_INVALID_ARG, "null text"); });
    static const char empty = 0;
    return load_common(name ? name : "<memory>", text ? text : &empty, bytes, format, opts, out, stats);
}

cheb_status cheb_validate_csr(const int64_t* offsets, int64_t n_offsets, const int64_t* neighbors, int64_t nnz,
                              const int64_t* degrees, int64_t n_degrees, int64_t n, int64_t m, int multi,
                              int64_t duplicates_removed, int64_t isolated_dropped, int device,
                              cheb_graph_stats* stats) {
    return guarded([&] {
        NvtxRange nvtx_("cheb_validate_csr");
        if (!offsets || n_offsets < 1) fail(CHEB_VALIDATION, "offsets length is not n+1");
        int count = 0;
        if (cudaGetDeviceCount(&count) != cudaSuccess || count == 0)
            fail(CHEB_CUDA, "no CUDA device available (libchebpr_b200 has no CPU fallback)");
        cheb_graph_stats local;
        validate_csr(offsets, n_offsets, neighbors, nnz, degrees, n_degrees, n, m, multi, duplicates_removed,
                     isolated_dropped, device, stats ? stats : &local);
    });
}

cheb_status cheb_graph_validate_stats(cheb_graph_t g, cheb_graph_stats* stats) {
    return guarded([&] {
        NvtxRange nvtx_("cheb_graph_validate_stats");
        need_graph(g);
        GraphScope gs(g);
        if (!stats) fail(CHEB_INVALID_ARG, "null stats");
        stats_of(g, stats);
        stats->lines = 0;
        stats->weights_ignored = 0;
    });
}

cheb_status cheb_graph_download_csr(cheb_graph_t g, int64_t* offsets, int64_t* neighbors,
                                    int64_t* degrees) {
    return guarded([&] {
        NvtxRange nvtx_("cheb_graph_download_csr");
        need_graph(g);
        GraphScope gs(g);
        download_csr(g, offsets, neighbors, degrees);
    });
}

cheb_status cheb_graph_get_info(cheb_graph_t g, cheb_graph_info* info) {
    return guarded([&] {
        NvtxRange nvtx_("cheb_graph_get_info");
        need_graph(g);
        fill_info(g, info);
    });
}

void cheb_graph_free(cheb_graph_t g) {
    if (!g) return;
    GraphScope gs(g);
    cudaStreamSynchronize(g->stream);
    delete g;
}

int cheb_partition_block_rows(void) { return (int)kPartRows; }

cheb_status cheb_partition_vertices(const int64_t* degrees, int64_t n, int K, int64_t* cuts) {
    return guarded([&] { partition_cuts(degrees, n, K, cuts); });
}

cheb_status cheb_partition_plan(const int64_t* degrees, int64_t n, int G, int64_t* order,
                                int64_t* cuts, int64_t* max_rows) {
    // degree-descending relabel (ties by id; the view's order) + the reference cut rule on
    // the relabelled degrees; slot size = the largest slice.
    return guarded([&] {
        if (G < 1) fail(CHEB_DOMAIN, "parallelism must be >= 1");
        std::vector<int64_t> ids(n), dsorted(n);
        for (int64_t v = 0; v < n; ++v) ids[v] = v;
        std::stable_sort(ids.begin(), ids.end(), [&](int64_t a, int64_t b) { return degrees[a] > degrees[b]; });
        for (int64_t i = 0; i < n; ++i) dsorted[i] = degrees[ids[i]];
        partition_cuts(dsorted.data(), n, G, cuts);
        int64_t mr = 0;
        for (int r = 0; r < G; ++r) mr = std::max(mr, cuts[r + 1] - cuts[r]);
        if (order) std::memcpy(order, ids.data(), sizeof(int64_t) * n);
        if (max_rows) *max_rows = mr;
    });
}

void cheb_cpaa_opts_default(cheb_cpaa_opts* o) {
    o->c = 0.85;
    o->rounds = -1;
    o->eps = -1.0;
    o->max_rounds = 60;
    o->parallelism = 1;
    o->mode = CHEB_MODE_FAST;
    o->precision = CHEB_FP64;
    o->R = 1;
    o->personalization = nullptr;
    o->trace = 1;
}

// cheb_trace_row of a finished solve (cpaa.cpp:99,139-145 columns).
static void fill_trace(cheb_graph* g, const SolveSpec& s, const std::vector<double>& tr,
                       const std::vector<double>* errs, cheb_trace_row* trace) {
    if (!trace || s.M <= 0) return;
    std::vector<double> co;
    double b, c0;
    coefficients(s.c, s.M, co, &b, &c0);
    double residual = static_cast<double>(g->n) * c0 * b / (1.0 - b);  // cpaa.cpp:99
    const double per_term = g->last_loop_ms / s.M;
    for (int k = 1; k <= s.M; ++k) {
        cheb_trace_row& r = trace[k - 1];
        std::memset(&r, 0, sizeof r);
        r.k = k;
        r.c_k = co[k];
        r.mass_T = tr[2 * (k - 1)];
        r.S_k = tr[2 * (k - 1) + 1];
        residual *= b;
        r.residual_mass = residual;
        r.elapsed_ms = g->term_elapsed_ms.size() == (size_t)s.M ? g->term_elapsed_ms[(size_t)k - 1] : per_term;
        if (errs) {
            r.err = (*errs)[2 * (k - 1)];
            r.err_l1 = (*errs)[2 * (k - 1) + 1];
        }
    }
}

static SolveSpec checked_spec(cheb_graph* g, const cheb_cpaa_opts& o, const double* reference,
                              int64_t n_reference) {
    need_graph(g);
    essential(g);                                               // cpaa.cpp:81
    SolveSpec s;
    s.M = resolve_rounds(o.c, o.rounds, o.eps, o.max_rounds);   // cpaa.cpp:82
    std::vector<double> tmp;
    coefficients(o.c, s.M, tmp, nullptr, nullptr);              // cpaa.cpp:83 (DomainError on c)
    if (reference && n_reference != g->n)                       // cpaa.cpp:84-85
        fail(CHEB_INVALID_ARG, "reference length does not match vertex count");
    if (o.parallelism < 1) fail(CHEB_DOMAIN, "parallelism must be >= 1");  // cpaa.cpp:94
    if (o.mode != CHEB_MODE_FAST && o.mode != CHEB_MODE_BITEXACT)
        fail(CHEB_INVALID_ARG, "unknown mode");
    if (o.precision != CHEB_FP64 && o.precision != CHEB_FP32)
        fail(CHEB_INVALID_ARG, "precision must be 64 or 32");
    s.c = o.c;
    s.mode = o.mode;
    s.precision = o.precision;
    s.R = o.R < 1 ? 1 : o.R;
    s.p = o.personalization;
    s.trace = o.trace != 0;
    return s;
}

cheb_status cheb_cpaa(cheb_graph_t g, const cheb_cpaa_opts* opts, const double* reference,
                      int64_t n_reference, double* ranks, cheb_trace_row* trace,
                      int* rounds_out, double* total_mass_out) {
    return guarded([&] {
        NvtxRange nvtx_("cheb_cpaa");
        cheb_cpaa_opts o;
        cheb_cpaa_opts_default(&o);
        if (opts) o = *opts;
        SolveSpec s = checked_spec(g, o, reference, n_reference);
        if (reference && s.M > 0)  // metrics.cpp:18-19 (first call happens at round 1)
            for (int64_t i = 0; i < g->n; ++i)
                if (!(reference[i] > 0.0))
                    fail(CHEB_DOMAIN, "reference entry " + std::to_string(i) + " is not positive");
        std::vector<double> tr, errs;
        double total = 0.0;
        if (reference) cpaa_solve_ref(g, s, reference, &tr, &errs, &total);
        else cpaa_solve(g, s, true, &tr, &total);
        read_ranks(g, s.precision, ranks);
        fill_trace(g, s, tr, reference ? &errs : nullptr, trace);
        if (rounds_out) *rounds_out = s.M;
        if (total_mass_out) *total_mass_out = total;
    });
}

cheb_status cheb_cpaa_device(cheb_graph_t g, const cheb_cpaa_opts* opts, const void** d_ranks,
                             int sync) {
    return guarded([&] {
        NvtxRange nvtx_("cheb_cpaa_device");
        cheb_cpaa_opts o;
        cheb_cpaa_opts_default(&o);
        if (opts) o = *opts;
        SolveSpec s = checked_spec(g, o, nullptr, 0);
        if (sync) {
            double total;
            std::vector<double> tr;
            cpaa_solve(g, s, false, &tr, &total);
        } else {
            cpaa_solve(g, s, false, nullptr, nullptr);
        }
        if (d_ranks) *d_ranks = g->ws.out.get();
    });
}

cheb_status cheb_cpaa_profile(cheb_graph_t g, const cheb_cpaa_opts* opts, double* term_ms,
                              int capacity, int* terms) {
    return guarded([&] {
        NvtxRange nvtx_("cheb_cpaa_profile");
        cheb_cpaa_opts o;
        cheb_cpaa_opts_default(&o);
        if (opts) o = *opts;
        SolveSpec s = checked_spec(g, o, nullptr, 0);
        std::vector<double> ms;
        cpaa_profile(g, s, ms);
        for (int k = 0; k < s.M && k < capacity; ++k) term_ms[k] = ms[k];
        if (terms) *terms = s.M;
    });
}

// right-hand sides per SpMM pass (<= 128: 32 lanes x 4 values); tuning().batchblock
static int batch_block() { return std::max(1, std::min(tuning().batchblock, 128)); }

static BatchSpec batch_spec(cheb_graph* g, const cheb_cpaa_opts& o, const int64_t* seeds) {
    need_graph(g);
    single_gpu_only(g);
    essential(g);
    BatchSpec b;
    b.M = resolve_rounds(o.c, o.rounds, o.eps, o.max_rounds);
    std::vector<double> tmp;
    coefficients(o.c, b.M, tmp, nullptr, nullptr);
    if (o.parallelism < 1) fail(CHEB_DOMAIN, "parallelism must be >= 1");
    if (o.mode != CHEB_MODE_FAST) fail(CHEB_INVALID_ARG, "the batched path runs the FAST schedule only");
    if (o.precision != CHEB_FP64 && o.precision != CHEB_FP32)
        fail(CHEB_INVALID_ARG, "precision must be 64 or 32");
    if (o.R < 1) fail(CHEB_INVALID_ARG, "R must be >= 1");
    if (seeds && o.personalization) fail(CHEB_INVALID_ARG, "give seeds or a dense personalization, not both");
    if (seeds)
        for (int r = 0; r < o.R; ++r)
            if (seeds[r] < 0 || seeds[r] >= g->n)
                fail(CHEB_VALIDATION, "seed vertex " + std::to_string(seeds[r]) + " out of range");
    b.c = o.c;
    b.precision = o.precision;
    b.R = o.R;
    b.p = o.personalization;
    b.seeds = seeds;
    return b;
}

cheb_status cheb_cpaa_batch(cheb_graph_t g, const cheb_cpaa_opts* opts, const int64_t* seeds,
                            double* ranks, double* totals, cheb_trace_row* trace, int* rounds_out) {
    return guarded([&] {
        NvtxRange nvtx_("cheb_cpaa_batch");
        cheb_cpaa_opts o;
        cheb_cpaa_opts_default(&o);
        if (opts) o = *opts;
        BatchSpec b = batch_spec(g, o, seeds);
        std::vector<double> tr, tot;
        const int kBatchBlock = batch_block();
        if (b.R <= kBatchBlock) {
            cpaa_batch_solve(g, b, tr, tot, nullptr);
            if (ranks) read_batch_ranks(g, ranks, b.R);
        } else {
            // more right-hand sides than one SpMM pass carries: column blocks of kBatchBlock,
            // results scattered into the caller's n x R row-major block, traces summed
            const int64_t n = g->n;
            std::vector<double> blk, pblk;
            tot.assign(b.R, 0.0);
            for (int c0 = 0; c0 < b.R; c0 += kBatchBlock) {
                const int Rc = std::min(kBatchBlock, b.R - c0);
                BatchSpec bc = b;
                bc.R = Rc;
                bc.seeds = b.seeds ? b.seeds + c0 : nullptr;
                bc.record_start = c0 == 0;
                if (b.p) {
                    pblk.resize((size_t)n * Rc);
                    for (int64_t v = 0; v < n; ++v)
                        std::memcpy(&pblk[(size_t)v * Rc], b.p + (size_t)v * b.R + c0, sizeof(double) * Rc);
                    bc.p = pblk.data();
                }
                std::vector<double> trc, totc;
                cpaa_batch_solve(g, bc, trc, totc, nullptr);
                if (tr.empty()) tr.assign(trc.size(), 0.0);
                for (size_t i = 0; i < trc.size(); ++i) tr[i] += trc[i];
                std::memcpy(tot.data() + c0, totc.data(), sizeof(double) * Rc);
                if (ranks) {
                    blk.resize((size_t)n * Rc);
                    read_batch_ranks(g, blk.data(), Rc);
                    for (int64_t v = 0; v < n; ++v)
                        std::memcpy(ranks + (size_t)v * b.R + c0, &blk[(size_t)v * Rc], sizeof(double) * Rc);
                }
            }
        }
        if (totals) std::memcpy(totals, tot.data(), sizeof(double) * b.R);
        if (trace && b.M > 0) {
            std::vector<double> co;
            double be, c0;
            coefficients(b.c, b.M, co, &be, &c0);
            double residual = static_cast<double>(g->n) * b.R * c0 * be / (1.0 - be);
            for (int k = 1; k <= b.M; ++k) {
                cheb_trace_row& r = trace[k - 1];
                std::memset(&r, 0, sizeof r);
                r.k = k;
                r.c_k = co[k];
                r.mass_T = tr[2 * (k - 1)];
                r.S_k = tr[2 * (k - 1) + 1];
                residual *= be;
                r.residual_mass = residual;
                r.elapsed_ms = g->last_loop_ms / b.M;
            }
        }
        if (rounds_out) *rounds_out = b.M;
    });
}

cheb_status cheb_cpaa_batch_profile(cheb_graph_t g, const cheb_cpaa_opts* opts, const int64_t* seeds,
                                    double* term_ms, int capacity, int* terms) {
    return guarded([&] {
        NvtxRange nvtx_("cheb_cpaa_batch_profile");
        cheb_cpaa_opts o;
        cheb_cpaa_opts_default(&o);
        if (opts) o = *opts;
        BatchSpec b = batch_spec(g, o, seeds);
        std::vector<double> tr, tot, ms;
        cpaa_batch_solve(g, b, tr, tot, &ms);
        for (int k = 0; k < b.M && k < capacity; ++k) term_ms[k] = ms[k];
        if (terms) *terms = b.M;
    });
}

cheb_status cheb_nccl_unique_id(void* out, int out_bytes) {
    return guarded([&] {
        NvtxRange nvtx_("cheb_nccl_unique_id");
        if (out_bytes < (int)sizeof(ncclUniqueId)) fail(CHEB_INVALID_ARG, "unique id buffer too small");
        ncclUniqueId id;
        const ncclResult_t r = ncclGetUniqueId(&id);
        if (r != ncclSuccess) fail(CHEB_NCCL, std::string("ncclGetUniqueId: ") + ncclGetErrorString(r));
        std::memcpy(out, &id, sizeof id);
    });
}

cheb_status cheb_comm_create(const void* unique_id, int nranks, int rank, int device, cheb_comm_t* out) {
    return guarded([&] {
        NvtxRange nvtx_("cheb_comm_create");
        if (nranks < 1 || rank < 0 || rank >= nranks) fail(CHEB_INVALID_ARG, "bad rank / nranks");
        DeviceGuard dg(device);
        auto* c = new cheb_comm();
        c->nranks = nranks;
        c->rank = rank;
        c->device = device;
        ncclUniqueId id;
        std::memcpy(&id, unique_id, sizeof id);
        const ncclResult_t r = ncclCommInitRank(&c->nccl, nranks, id, rank);
        if (r != ncclSuccess) {
            delete c;
            fail(CHEB_NCCL, std::string("ncclCommInitRank: ") + ncclGetErrorString(r));
        }
        *out = c;
    });
}

void cheb_comm_destroy(cheb_comm_t c) {
    if (!c) return;
    DeviceGuard dg(c->device);
    if (c->nccl) ncclCommDestroy(c->nccl);
    delete c;
}

cheb_status cheb_graph_attach_comm(cheb_graph_t g, cheb_comm_t comm) {
    return guarded([&] {
        NvtxRange nvtx_("cheb_graph_attach_comm");
        need_graph(g);
        if (!comm) fail(CHEB_INVALID_ARG, "null communicator");
        if (comm->device != g->device) fail(CHEB_INVALID_ARG, "communicator and graph live on different devices");
        g->part.G = comm->nranks;
        g->part.rank = comm->rank;
        g->part.comm = comm->nccl;
        g->view.ready = false;  // rebuild the solver view as this rank's slice
        if (g->ws.exec) {
            cudaGraphExecDestroy(g->ws.exec);
            g->ws.exec = nullptr;
        }
        g->ws.exec_key.clear();
        g->ws.seen_key.clear();
    });
}

// ---------------- fused push exchange ---------------------------------------------------
void chebgpu::PeerGroup::release() {
    for (void* p : opened) cudaIpcCloseMemHandle(p);
    opened.clear();
    for (void* p : {X[0], X[1], trace_all, rbuf, static_cast<void*>(flags)})
        if (p) cudaFree(p);
    X[0] = X[1] = trace_all = rbuf = nullptr;
    flags = nullptr;
    table.release();
    if (signalled) cudaEventDestroy(signalled);
    signalled = nullptr;
}

struct cheb_group {
    std::vector<cheb_graph*> graphs;
};

namespace {
void drop_peer(cheb_graph* g) {
    if (!g->peer) return;
    DeviceGuard dg(g->device);
    cudaStreamSynchronize(g->stream);
    g->peer->release();
    delete g->peer;
    g->peer = nullptr;
}

void reset_partition(cheb_graph* g, int G, int rank) {
    g->part.G = G;
    g->part.rank = rank;
    g->part.comm = nullptr;
    g->view.ready = false;
    if (g->ws.exec) {
        cudaGraphExecDestroy(g->ws.exec);
        g->ws.exec = nullptr;
    }
    g->ws.exec_key.clear();
    g->ws.seen_key.clear();
}

// Make g rank `rank` of G with its own exchange buffers (view rebuilt as this rank's slice).
void make_peer(cheb_graph* g, int G, int rank, bool lockstep) {
    if (G < 1 || rank < 0 || rank >= G) fail(CHEB_INVALID_ARG, "bad group size / rank");
    essential(g);
    GraphScope gs(g);
    drop_peer(g);
    reset_partition(g, G, rank);
    g->peer = new PeerGroup();
    PeerGroup& pg = *g->peer;
    pg.G = G;
    pg.rank = rank;
    pg.lockstep = lockstep;
    ensure_view(g);
    pg.x_len = std::max<int64_t>(g->view.x_len, 1);
    const size_t xb = sizeof(double) * (size_t)pg.x_len;
    CHEB_CUDA_CHECK(cudaMalloc(&pg.X[0], xb));
    CHEB_CUDA_CHECK(cudaMalloc(&pg.X[1], xb));
    CHEB_CUDA_CHECK(cudaMalloc(&pg.rbuf, xb));
    CHEB_CUDA_CHECK(cudaMalloc(&pg.trace_all, sizeof(double) * 2 * (size_t)kMaxPushTerms * G));
    // G epoch slots written by the peers + one timeout flag raised by this rank's waits
    CHEB_CUDA_CHECK(cudaMalloc(reinterpret_cast<void**>(&pg.flags), sizeof(unsigned long long) * (G + 1)));
    CHEB_CUDA_CHECK(cudaMemset(pg.flags, 0, sizeof(unsigned long long) * (G + 1)));
    if (lockstep) CHEB_CUDA_CHECK(cudaEventCreateWithFlags(&pg.signalled, cudaEventDisableTiming));
    pg.pX0.assign(G, nullptr);
    pg.pX1.assign(G, nullptr);
    pg.ptrace.assign(G, nullptr);
    pg.prbuf.assign(G, nullptr);
    pg.pflags.assign(G, nullptr);
    pg.pX0[rank] = pg.X[0];
    pg.pX1[rank] = pg.X[1];
    pg.ptrace[rank] = pg.trace_all;
    pg.prbuf[rank] = pg.rbuf;
    pg.pflags[rank] = pg.flags;
}

void upload_table(cheb_graph* g) {
    PeerGroup& pg = *g->peer;
    std::vector<void*> t;
    for (auto* v : {&pg.pX0, &pg.pX1, &pg.ptrace, &pg.prbuf, &pg.pflags}) t.insert(t.end(), v->begin(), v->end());
    GraphScope gs(g);
    pg.table.alloc(sizeof(void*) * t.size());
    CHEB_CUDA_CHECK(cudaMemcpyAsync(pg.table.get(), t.data(), sizeof(void*) * t.size(), cudaMemcpyHostToDevice, g->stream));
    CHEB_CUDA_CHECK(cudaStreamSynchronize(g->stream));
    CHEB_CUDA_CHECK(cudaDeviceSynchronize());  // buffers and flags zeroed before any peer uses them
}
}  // namespace

cheb_status cheb_group_create(cheb_graph_t* graphs, int G, cheb_group_t* out) {
    return guarded([&] {
        NvtxRange nvtx_("cheb_group_create");
        if (!graphs || G < 1 || !out) fail(CHEB_INVALID_ARG, "bad group arguments");
        for (int r = 0; r < G; ++r) {
            need_graph(graphs[r]);
            for (int q = 0; q < r; ++q)
                if (graphs[q] == graphs[r]) fail(CHEB_INVALID_ARG, "a handle appears twice in the group");
            if (graphs[r]->n != graphs[0]->n || graphs[r]->nnz != graphs[0]->nnz || graphs[r]->m != graphs[0]->m)
                fail(CHEB_INVALID_ARG, "group members must hold the same graph");
        }
        for (int r = 0; r < G; ++r)  // peer access between distinct devices
            for (int q = 0; q < G; ++q) {
                const int a = graphs[r]->device, b = graphs[q]->device;
                if (a == b) continue;
                int ok = 0;
                CHEB_CUDA_CHECK(cudaDeviceCanAccessPeer(&ok, a, b));
                if (!ok) fail(CHEB_CUDA, "devices " + std::to_string(a) + " and " + std::to_string(b) +
                                             " have no peer access");
                DeviceGuard dg(a);
                const cudaError_t e = cudaDeviceEnablePeerAccess(b, 0);
                if (e != cudaSuccess && e != cudaErrorPeerAccessAlreadyEnabled) CHEB_CUDA_CHECK(e);
                cudaGetLastError();
            }
        for (int r = 0; r < G; ++r) make_peer(graphs[r], G, r, true);
        for (int r = 0; r < G; ++r) {
            PeerGroup& pg = *graphs[r]->peer;
            for (int q = 0; q < G; ++q) {
                const PeerGroup& o = *graphs[q]->peer;
                pg.pX0[q] = o.X[0];
                pg.pX1[q] = o.X[1];
                pg.ptrace[q] = o.trace_all;
                pg.prbuf[q] = o.rbuf;
                pg.pflags[q] = o.flags;
            }
            upload_table(graphs[r]);
        }
        auto* grp = new cheb_group();
        grp->graphs.assign(graphs, graphs + G);
        *out = grp;
    });
}

cheb_status cheb_group_cpaa(cheb_group_t grp, const cheb_cpaa_opts* opts, double* ranks, cheb_trace_row* trace,
                            int* rounds, double* total) {
    return guarded([&] {
        NvtxRange nvtx_("cheb_group_cpaa");
        if (!grp || grp->graphs.empty()) fail(CHEB_INVALID_ARG, "null group");
        cheb_graph* g0 = grp->graphs[0];
        cheb_cpaa_opts o;
        cheb_cpaa_opts_default(&o);
        if (opts) o = *opts;
        SolveSpec s = checked_spec(g0, o, nullptr, 0);
        std::vector<double> tr;
        double tot = 0.0;
        group_solve(grp->graphs, s, &tr, &tot);
        read_ranks(g0, s.precision, ranks);
        fill_trace(g0, s, tr, nullptr, trace);
        if (rounds) *rounds = s.M;
        if (total) *total = tot;
    });
}

cheb_status cheb_group_profile(cheb_group_t grp, const cheb_cpaa_opts* opts, double* rank_term_ms, int capacity) {
    return guarded([&] {
        NvtxRange nvtx_("cheb_group_profile");
        if (!grp || grp->graphs.empty()) fail(CHEB_INVALID_ARG, "null group");
        cheb_graph* g0 = grp->graphs[0];
        cheb_cpaa_opts o;
        cheb_cpaa_opts_default(&o);
        if (opts) o = *opts;
        SolveSpec s = checked_spec(g0, o, nullptr, 0);
        std::vector<double> tr, ms;
        double tot = 0.0;
        group_solve(grp->graphs, s, &tr, &tot, &ms);
        for (int r = 0; r < (int)ms.size() && r < capacity; ++r) rank_term_ms[r] = ms[(size_t)r];
    });
}

void cheb_group_destroy(cheb_group_t grp) {
    if (!grp) return;
    for (cheb_graph* g : grp->graphs) {
        drop_peer(g);
        reset_partition(g, 1, 0);
    }
    delete grp;
}

cheb_status cheb_peer_export(cheb_graph_t g, int G, int rank, void* out, size_t cap) {
    return guarded([&] {
        NvtxRange nvtx_("cheb_peer_export");
        need_graph(g);
        if (!out || cap < CHEB_PEER_EXPORT_BYTES) fail(CHEB_INVALID_ARG, "export buffer too small");
        make_peer(g, G, rank, false);
        PeerGroup& pg = *g->peer;
        std::memset(out, 0, CHEB_PEER_EXPORT_BYTES);
        auto* b = static_cast<unsigned char*>(out);
        int i = 0;
        for (void* p : {pg.X[0], pg.X[1], pg.trace_all, pg.rbuf, static_cast<void*>(pg.flags)}) {
            cudaIpcMemHandle_t h;
            CHEB_CUDA_CHECK(cudaIpcGetMemHandle(&h, p));
            std::memcpy(b + 64 * i++, &h, sizeof h);
        }
        const int64_t meta[2] = {pg.x_len, (int64_t)rank};
        std::memcpy(b + 320, meta, sizeof meta);
    });
}

cheb_status cheb_peer_import(cheb_graph_t g, const void* all, size_t bytes_per_rank) {
    return guarded([&] {
        NvtxRange nvtx_("cheb_peer_import");
        need_graph(g);
        if (!g->peer || g->peer->lockstep) fail(CHEB_INVALID_ARG, "cheb_peer_export first");
        if (!all || bytes_per_rank < CHEB_PEER_EXPORT_BYTES) fail(CHEB_INVALID_ARG, "bad import buffer");
        PeerGroup& pg = *g->peer;
        GraphScope gs(g);
        const auto* b = static_cast<const unsigned char*>(all);
        for (int q = 0; q < pg.G; ++q) {
            const unsigned char* e = b + bytes_per_rank * q;
            int64_t meta[2];
            std::memcpy(meta, e + 320, sizeof meta);
            if (meta[1] != q || meta[0] != pg.x_len) fail(CHEB_INVALID_ARG, "peer exports out of order or mismatched");
            if (q == pg.rank) continue;
            void* ptr[5];
            for (int i = 0; i < 5; ++i) {
                cudaIpcMemHandle_t h;
                std::memcpy(&h, e + 64 * i, sizeof h);
                CHEB_CUDA_CHECK(cudaIpcOpenMemHandle(&ptr[i], h, cudaIpcMemLazyEnablePeerAccess));
                pg.opened.push_back(ptr[i]);
            }
            pg.pX0[q] = ptr[0];
            pg.pX1[q] = ptr[1];
            pg.ptrace[q] = ptr[2];
            pg.prbuf[q] = ptr[3];
            pg.pflags[q] = ptr[4];
        }
        upload_table(g);
    });
}

cheb_status cheb_peer_detach(cheb_graph_t g) {
    return guarded([&] {
        NvtxRange nvtx_("cheb_peer_detach");
        need_graph(g);
        drop_peer(g);
        reset_partition(g, 1, 0);
    });
}

cheb_status cheb_graph_view_bins(cheb_graph_t g, int64_t* tiles, int64_t* rows, int64_t* nnz) {
    return guarded([&] {
        NvtxRange nvtx_("cheb_graph_view_bins");
        need_graph(g);
        GraphScope gs(g);
        ensure_view(g);
        for (int b = 0; b < 7; ++b) {
            if (tiles) tiles[b] = g->view.bin_tiles[b];
            if (rows) rows[b] = g->view.bin_rows[b];
            if (nnz) nnz[b] = g->view.bin_nnz[b];
        }
    });
}

cheb_status cheb_graph_view_download(cheb_graph_t g, int64_t* sizes, int64_t* row_ptr, int32_t* col,
                                     int32_t* order, int64_t* chunk_begin) {
    return guarded([&] {
        NvtxRange nvtx_("cheb_graph_view_download");
        need_graph(g);
        GraphScope gs(g);
        ensure_view(g);
        const SolverView& V = g->view;
        if (sizes) {
            sizes[0] = V.n_local;
            sizes[1] = V.nnz_local;
            sizes[2] = V.n_hub;
            sizes[3] = V.n_chunk_tiles;
            sizes[4] = kHotBytes / 8;
        }
        cudaStream_t st = g->stream;
        if (row_ptr) {
            std::vector<int32_t> r32;
            if (V.rp64) {
                CHEB_CUDA_CHECK(cudaMemcpyAsync(row_ptr, V.row_ptr.get(), sizeof(int64_t) * (V.n_local + 1),
                                                cudaMemcpyDeviceToHost, st));
            } else {
                r32.resize((size_t)V.n_local + 1);
                CHEB_CUDA_CHECK(cudaMemcpyAsync(r32.data(), V.row_ptr.get(), sizeof(int32_t) * (V.n_local + 1),
                                                cudaMemcpyDeviceToHost, st));
            }
            CHEB_CUDA_CHECK(cudaStreamSynchronize(st));
            for (size_t i = 0; i < r32.size(); ++i) row_ptr[i] = r32[i];
        }
        if (col && V.nnz_local > 0)
            CHEB_CUDA_CHECK(cudaMemcpyAsync(col, V.col.get(), sizeof(int32_t) * V.nnz_local, cudaMemcpyDeviceToHost, st));
        if (order && V.n_local > 0)
            CHEB_CUDA_CHECK(cudaMemcpyAsync(order, V.order.get(), sizeof(int32_t) * V.n_local, cudaMemcpyDeviceToHost, st));
        if (chunk_begin && V.n_chunk_tiles > 0) {
            std::vector<Tile> t((size_t)V.n_chunk_tiles + 1);
            CHEB_CUDA_CHECK(cudaMemcpyAsync(t.data(), V.tiles.get(), sizeof(Tile) * t.size(), cudaMemcpyDeviceToHost, st));
            CHEB_CUDA_CHECK(cudaStreamSynchronize(st));
            for (size_t i = 0; i < t.size(); ++i) chunk_begin[i] = t[i].nnz_begin;
        }
        CHEB_CUDA_CHECK(cudaStreamSynchronize(st));
    });
}

cheb_status cheb_graph_view_windows(cheb_graph_t g, int64_t* sizes, uint16_t* wcol, uint16_t* lane_meta,
                                    int32_t* block_base, int32_t* row_first, int32_t* piece_list) {
    return guarded([&] {
        NvtxRange nvtx_("cheb_graph_view_windows");
        need_graph(g);
        GraphScope gs(g);
        ensure_view(g);
        const SolverView& V = g->view;
        const SolverView::Windows& W = V.win;
        cudaStream_t st = g->stream;
        int listed = 0;
        if (W.ready)
            CHEB_CUDA_CHECK(cudaMemcpyAsync(&listed, W.kf.ptr<int>() + V.n_hub, sizeof(int), cudaMemcpyDeviceToHost, st));
        CHEB_CUDA_CHECK(cudaStreamSynchronize(st));
        if (sizes) {
            sizes[0] = W.ready ? W.NW : 0;
            sizes[1] = W.W;
            sizes[2] = W.H0;
            sizes[3] = W.n_blocks;
            sizes[4] = W.entries;
            sizes[5] = W.pieces;
            sizes[6] = W.MC;
            sizes[7] = listed;
        }
        if (!W.ready) return;
        if (wcol)
            CHEB_CUDA_CHECK(cudaMemcpyAsync(wcol, W.wcol.get(), sizeof(uint16_t) * (size_t)W.n_blocks * kWinBlock,
                                            cudaMemcpyDeviceToHost, st));
        if (lane_meta)
            CHEB_CUDA_CHECK(cudaMemcpyAsync(lane_meta, W.meta.get(), sizeof(uint16_t) * (size_t)W.n_blocks * 32,
                                            cudaMemcpyDeviceToHost, st));
        if (block_base)
            CHEB_CUDA_CHECK(cudaMemcpyAsync(block_base, W.bbase.get(), sizeof(int32_t) * (size_t)(W.n_blocks + 1),
                                            cudaMemcpyDeviceToHost, st));
        if (row_first)
            CHEB_CUDA_CHECK(cudaMemcpyAsync(row_first, W.kf.get(), sizeof(int32_t) * (size_t)(V.n_hub + 1),
                                            cudaMemcpyDeviceToHost, st));
        if (piece_list && listed > 0)
            CHEB_CUDA_CHECK(cudaMemcpyAsync(piece_list, W.klist.get(), sizeof(int32_t) * (size_t)listed,
                                            cudaMemcpyDeviceToHost, st));
        CHEB_CUDA_CHECK(cudaStreamSynchronize(st));
    });
}

cheb_status cheb_graph_view_tiles(cheb_graph_t g, int64_t* n_tiles, int64_t* nnz_begin, int32_t* row_begin,
                                  int32_t* meta, int32_t* n_launches) {
    return guarded([&] {
        NvtxRange nvtx_("cheb_graph_view_tiles");
        need_graph(g);
        GraphScope gs(g);
        ensure_view(g);
        const SolverView& V = g->view;
        if (n_tiles) *n_tiles = V.n_tiles;
        if (n_launches) *n_launches = V.phases.empty() ? 1 : (int32_t)V.phases.size();
        if (nnz_begin || row_begin || meta) {
            std::vector<Tile> t((size_t)V.n_tiles + 1);
            CHEB_CUDA_CHECK(cudaMemcpyAsync(t.data(), V.tiles.get(), sizeof(Tile) * t.size(), cudaMemcpyDeviceToHost,
                                            g->stream));
            CHEB_CUDA_CHECK(cudaStreamSynchronize(g->stream));
            for (size_t i = 0; i < t.size(); ++i) {
                if (nnz_begin) nnz_begin[i] = t[i].nnz_begin;
                if (row_begin) row_begin[i] = t[i].row_begin;
                if (meta) meta[i] = t[i].meta;
            }
        }
    });
}

cheb_status cheb_graph_partition_info(cheb_graph_t g, int64_t* lo, int64_t* hi, int64_t* nnz_local,
                                      int64_t* max_rows) {
    return guarded([&] {
        NvtxRange nvtx_("cheb_graph_partition_info");
        need_graph(g);
        GraphScope gs(g);
        ensure_view(g);
        // block-cyclic partition: the rank owns n_local sorted rows; lo = 0, hi = n_local
        if (lo) *lo = 0;
        if (hi) *hi = g->view.n_local;
        if (nnz_local) *nnz_local = g->view.nnz_local;
        if (max_rows) *max_rows = g->part.max_rows;
    });
}

cheb_status cheb_graph_exchange_info(cheb_graph_t g, int64_t* halo_stores, int64_t* all_stores) {
    return guarded([&] {
        NvtxRange nvtx_("cheb_graph_exchange_info");
        need_graph(g);
        GraphScope gs(g);
        ensure_view(g);
        if (halo_stores) *halo_stores = tuning().halo ? g->view.push_entries : g->view.push_entries_all;
        if (all_stores) *all_stores = g->view.push_entries_all;
    });
}

cheb_status cheb_set_tuning(const char* key, int value) {
    return guarded([&] {
        NvtxRange nvtx_("cheb_set_tuning");
        const std::string k = key ? key : "";
        if (k == "hot") tuning().hot = value;
        else if (k == "nogather") tuning().nogather = value;
        else if (k == "skip") tuning().skip = value;
        else if (k == "l2win") tuning().l2win = value;
        else if (k == "pdl") tuning().pdl = value;
        else if (k == "chunksched") tuning().chunksched = value;  // applies to views built afterwards
        else if (k == "l2win_mb") tuning().l2win_mb = value;
        else if (k == "l2win_pct") tuning().l2win_pct = value;
        else if (k == "streamcs") tuning().streamcs = value;
        else if (k == "xout_hint") tuning().xout_hint = value;
        else if (k == "xdiscard") tuning().xdiscard = value;
        else if (k == "packsched") tuning().packsched = value;  // applies to views built afterwards
        else if (k == "batchblock") tuning().batchblock = std::max(1, std::min(value, 128));
        else if (k == "halo") tuning().halo = value;
        else if (k == "prefetch") tuning().prefetch = value;
        else if (k == "skipwarm") tuning().skipwarm = value;
        else if (k == "spmm_hub_mb") tuning().spmm_hub_mb = value;
        else if (k == "spmm_xpol") tuning().spmm_xpol = value;
        else if (k == "sortrows") tuning().sortrows = value;
        else if (k == "hubwarp") tuning().hubwarp = value;
        else if (k == "colbufs") tuning().colbufs = value;
        else if (k == "colblocks") tuning().colblocks = value;  // applies to views built afterwards
        else if (k == "colsplit_pct") tuning().colsplit_pct = value;  // applies to views built afterwards
        else if (k == "windows") tuning().windows = value;    // applies to views built afterwards
        else if (k == "winsize") tuning().winsize = value;    // applies to views built afterwards
        else if (k == "winh0") tuning().winh0 = value;        // applies to views built afterwards
        else if (k == "winpw") tuning().winpw = value;        // applies to views built afterwards
        else if (k == "winbank") tuning().winbank = value;    // applies to views built afterwards
        else if (k == "winskip") tuning().winskip = value;
        else fail(CHEB_INVALID_ARG, "unknown tuning key " + k);
    });
}

cheb_status cheb_last_timing(cheb_graph_t g, double* loop_ms, double* term_kernel_ms, int* terms,
                             int* launches) {
    return guarded([&] {
        NvtxRange nvtx_("cheb_last_timing");
        need_graph(g);
        GraphScope gs(g);
        CHEB_CUDA_CHECK(cudaEventSynchronize(g->ev1));
        float ms = 0.f;
        CHEB_CUDA_CHECK(cudaEventElapsedTime(&ms, g->ev0, g->ev1));
        g->last_loop_ms = ms;
        if (loop_ms) *loop_ms = ms;
        if (term_kernel_ms) *term_kernel_ms = g->last_terms ? ms / g->last_terms : 0.0;
        if (terms) *terms = g->last_terms;
        if (launches) *launches = g->last_launches;
    });
}

void cheb_power_opts_default(cheb_power_opts* o) {
    o->c = 0.85;
    o->rounds = -1;
    o->tol = -1.0;
    o->max_rounds = 60;
    o->parallelism = 1;
    o->mode = CHEB_MODE_FAST;
}

cheb_status cheb_power(cheb_graph_t g, const cheb_power_opts* opts, const double* reference,
                       int64_t n_reference, double* ranks, cheb_trace_row* trace,
                       int trace_capacity, int* rounds_out, double* total_mass_out) {
    return guarded([&] {
        NvtxRange nvtx_("cheb_power");
        cheb_power_opts o;
        cheb_power_opts_default(&o);
        if (opts) o = *opts;
        need_graph(g);
        single_gpu_only(g);
        essential(g);                                                   // power.cpp:30
        if (!(o.c > 0.0 && o.c < 1.0)) fail(CHEB_DOMAIN, "damping factor must lie in (0,1)");
        const bool fixed = o.rounds >= 0, by_tol = o.tol > 0.0;         // power.cpp:33-37
        if (fixed == by_tol) fail(CHEB_INVALID_ARG, "set exactly one of rounds and tol");
        const int budget = fixed ? o.rounds : o.max_rounds;
        if (budget < 0) fail(CHEB_INVALID_ARG, "round budget must be non-negative");
        if (reference && n_reference != g->n)
            fail(CHEB_INVALID_ARG, "reference length does not match vertex count");
        if (o.parallelism < 1) fail(CHEB_DOMAIN, "parallelism must be >= 1");
        if (reference && budget > 0)
            for (int64_t i = 0; i < g->n; ++i)
                if (!(reference[i] > 0.0))
                    fail(CHEB_DOMAIN, "reference entry " + std::to_string(i) + " is not positive");
        int rounds = 0;
        double total = 0.0;
        power_solve(g, o.c, o.rounds, o.tol, o.max_rounds, o.mode, reference, ranks, trace,
                    trace_capacity, &rounds, &total);
        if (rounds_out) *rounds_out = rounds;
        if (total_mass_out) *total_mass_out = total;
    });
}

cheb_status cheb_transition_apply(cheb_graph_t g, const double* x, int64_t nx, double* y, int mode) {
    return guarded([&] {
        NvtxRange nvtx_("cheb_transition_apply");
        need_graph(g);
        single_gpu_only(g);
        if (nx != g->n)  // graph.cpp:105-107
            fail(CHEB_INVALID_ARG, "vector length " + std::to_string(nx) +
                                       " does not match vertex count " + std::to_string(g->n));
        if (g->n == 0) return;
        transition_apply(g, x, y, mode);
    });
}

cheb_status cheb_state_init(cheb_graph_t g, double c0, int mode) {
    return guarded([&] {
        NvtxRange nvtx_("cheb_state_init");
        need_graph(g);
        single_gpu_only(g);
        essential(g);  // cpaa.cpp:168
        staged_init(g, c0, mode);
    });
}
cheb_status cheb_state_set(cheb_graph_t g, const double* T_prev, const double* T_curr,
                           const double* acc, int k) {
    return guarded([&] {
        NvtxRange nvtx_("cheb_state_set");
        need_graph(g);
        staged_set(g, T_prev, T_curr, acc, k);
    });
}
cheb_status cheb_state_generate(cheb_graph_t g) {
    return guarded([&] {
        NvtxRange nvtx_("cheb_state_generate");
        need_graph(g);
        staged_generate(g);
    });
}
cheb_status cheb_state_accumulate(cheb_graph_t g, double c_k) {
    return guarded([&] {
        NvtxRange nvtx_("cheb_state_accumulate");
        need_graph(g);
        staged_accumulate(g, c_k);
    });
}
cheb_status cheb_state_rotate(cheb_graph_t g) {
    return guarded([&] {
        NvtxRange nvtx_("cheb_state_rotate");
        need_graph(g);
        staged_rotate(g);
    });
}
cheb_status cheb_state_get(cheb_graph_t g, double* T_prev, double* T_curr, double* T_next,
                           double* acc, int* k) {
    return guarded([&] {
        NvtxRange nvtx_("cheb_state_get");
        need_graph(g);
        staged_get(g, T_prev, T_curr, T_next, acc, k);
    });
}

}  // extern "C"
