/*
 * chebpr_cuda.h — C-ABI of the B200-native CPAA hot path (libchebpr_b200.so).
 *
 * Drop-in boundary for the reference's C++ API in /root/reference/proj/include/chebpr/
 * (every entry point below cites the reference interface it replaces).  Plain
 * pointers and sizes only; no exceptions cross this boundary: every call returns a
 * cheb_status and, on failure, cheb_last_error() holds the reference's message text
 * (e.g. "vertex 2 is isolated (degree 0)", "non-finite value at round 3").  The C++
 * wrapper (include/chebpr/ headers) re-throws them as the reference's exception types
 * (/root/reference/proj/include/chebpr/errors.hpp:11-33).
 *
 * Ownership: host buffers are caller-owned and copied synchronously.  Device memory,
 * streams and CUDA graphs are owned by the graph handle.  Calls on one handle are
 * serialised by the caller (one solve at a time); distinct handles are
 * independent.
 */
#ifndef CHEBPR_CUDA_H
#define CHEBPR_CUDA_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Status codes <-> reference exception taxonomy (errors.hpp:11-33). */
typedef enum {
    CHEB_OK = 0,
    CHEB_VALIDATION = 1,  /* chebpr::ValidationError */
    CHEB_DOMAIN = 2,      /* chebpr::DomainError */
    CHEB_NUMERIC = 3,     /* chebpr::NumericError */
    CHEB_INVALID_ARG = 4, /* std::invalid_argument */
    CHEB_CAPACITY = 5,    /* chebpr::CapacityError */
    CHEB_CUDA = 6,        /* CUDA runtime failure (new) */
    CHEB_NCCL = 7,        /* NCCL failure (new) */
    CHEB_PARSE = 8        /* chebpr::ParseError */
} cheb_status;

/* Thread-local text of the last failure on this thread. */
const char* cheb_last_error(void);
/* Library version string and the CUDA device count visible to it. */
const char* cheb_version(void);
int cheb_device_count(void);

/* ---- coefficient kit: coefficients.hpp:31-51 (host code, bit-identical) ---- */
cheb_status cheb_beta(double c, double* out);                               /* :31 */
cheb_status cheb_sigma(double c, double* out);                              /* :37 */
cheb_status cheb_err_bound(double c, int M, double* out);                   /* :40 */
cheb_status cheb_plan_iterations(double c, double eps, int* M, double* predicted_err); /* :43 */
cheb_status cheb_coefficients(double c, int M, double* coeffs /* M+1 */, double* beta,
                              double* c0);                                  /* :46 */
/* cpaa.cpp:28-36 resolve_rounds: exactly one of rounds>=0 / eps>0; clamp to max_rounds. */
cheb_status cheb_resolve_rounds(double c, int rounds, double eps, int max_rounds, int* M);

/* ---- graph handle: graph.hpp:21-31 UndirectedGraph, device-resident ---- */
typedef struct cheb_graph* cheb_graph_t;

typedef struct {
    int dedup;          /* BuildOptions::dedup (graph.hpp:45), default 1 */
    int drop_isolated;  /* BuildOptions::drop_isolated (graph.hpp:46), default 0 */
    int64_t n_hint;     /* BuildOptions::n_hint (graph.hpp:47), default 0 */
    int device;         /* CUDA ordinal (new) */
    int row_ptr_64;     /* 1: int64 row pointers (config 4); 0: int32 when nnz < 2^31 (new) */
} cheb_build_opts;

typedef struct {
    int64_t n;                  /* UndirectedGraph::n */
    int64_t m;                  /* UndirectedGraph::m (self-loops once) */
    int64_t nnz;                /* neighbors.size() = 2m - self_loops */
    int64_t duplicates_removed; /* BuildResult::duplicates_removed (graph.hpp:52) */
    int64_t isolated_dropped;   /* BuildResult::isolated_dropped (graph.hpp:53) */
    int64_t max_degree;
    int64_t min_degree;
    int multi;                  /* UndirectedGraph::multi */
    int row_ptr_64;
    int inv_degree_array;       /* 1 if a non-canonical inv_degree was uploaded */
    int device;
} cheb_graph_info;

void cheb_build_opts_default(cheb_build_opts* o);

/* K1 device CSR builder.  Replaces build_graph (graph.hpp:60-61, graph.cpp:23-102):
 * same n rule, canonical (min,max) dedup, self-loop counted once, isolated-vertex
 * error / order-preserving drop, rows sorted ascending — bit-exact arrays.
 * edges: E pairs interleaved (a0,b0,a1,b1,...) in HOST memory. */
cheb_status cheb_graph_build(const int64_t* edges, int64_t E, const cheb_build_opts* opts,
                             cheb_graph_t* out, cheb_graph_info* info);
/* Same, from DEVICE-resident int64 (or int32 when edge_bits==32) pairs on opts->device. */
cheb_status cheb_graph_build_device(const void* d_edges, int64_t E, int edge_bits,
                                    const cheb_build_opts* opts, cheb_graph_t* out,
                                    cheb_graph_info* info);

/* Upload a host CSR (UndirectedGraph arrays).  essential_check semantics of
 * cpaa.cpp:16-26 (n>=1, consistent sizes, every degree>=1).  inv_degree may be NULL;
 * when given it is compared bitwise with 1.0/deg on the host (threads, while the CSR
 * copies are in flight): if canonical it is never copied and the kernels use an
 * in-register reciprocal (no array traffic), else the array is uploaded and used
 * (the reference reads it, cpaa.cpp:107 — e.g. the poisoned test, test_cpaa.cpp:371). */
cheb_status cheb_graph_upload_csr(const int64_t* offsets, int64_t n_offsets,
                                  const int64_t* neighbors, int64_t nnz, const int64_t* degrees,
                                  int64_t n_degrees, const double* inv_degree, int64_t n_inv,
                                  int64_t n, int64_t m, int multi, int device, int row_ptr_64,
                                  cheb_graph_t* out);

/* Bit-exact readback of the CSR (offsets[n+1], neighbors[nnz], degrees[n]; any may be NULL). */
cheb_status cheb_graph_download_csr(cheb_graph_t g, int64_t* offsets, int64_t* neighbors,
                                    int64_t* degrees);
cheb_status cheb_graph_get_info(cheb_graph_t g, cheb_graph_info* info);
void cheb_graph_free(cheb_graph_t g);

/* ---- graph ingest (graph_io.hpp / graph_io.cpp:50-174), parsed on the device ---- */
typedef struct {
    int dedup;          /* LoadOptions::dedup (graph_io.hpp:25), default 1 */
    int drop_isolated;  /* LoadOptions::drop_isolated (graph_io.hpp:26), default 0 */
    int symmetrize;     /* LoadOptions::symmetrize (graph_io.hpp:27), default 0 */
    int device;         /* CUDA ordinal (new) */
    int row_ptr_64;     /* as cheb_build_opts (new) */
} cheb_load_opts;

typedef struct {        /* GraphStats (graph.hpp:33-42) + ingest facts */
    int64_t n, m;
    double avg_degree;  /* m / n */
    int64_t min_degree, max_degree, self_loops, duplicates_removed, isolated_dropped;
    int64_t lines;      /* text lines consumed */
    int weights_ignored; /* Matrix Market real field: the reference warns once (graph_io.cpp:134-138) */
} cheb_graph_stats;

void cheb_load_opts_default(cheb_load_opts* o);
/* load_edge_list (graph_io.cpp:50-70) / load_matrix_market (72-174): the file is streamed
 * to the device through a pinned ring, split into lines and parsed by GPU threads, then
 * built by K1 (build_graph + the validate stats of finish(), graph_io.cpp:31-46).  Errors:
 * CHEB_PARSE / CHEB_VALIDATION with the reference's message text naming the first failing
 * line.  The caller prints the reference's warnings (isolated_dropped > 0,
 * weights_ignored). */
cheb_status cheb_graph_load_edge_list(const char* path, const cheb_load_opts* opts, cheb_graph_t* out,
                                      cheb_graph_stats* stats);
cheb_status cheb_graph_load_matrix_market(const char* path, const cheb_load_opts* opts, cheb_graph_t* out,
                                          cheb_graph_stats* stats);
/* Same from an in-memory text (format 0 = edge list, 1 = Matrix Market); `name` stands in
 * for the path in messages. */
cheb_status cheb_graph_parse_text(const char* text, int64_t bytes, int format, const char* name,
                                  const cheb_load_opts* opts, cheb_graph_t* out, cheb_graph_stats* stats);
/* validate (graph.cpp:123-186) of a HOST CSR, run on the device: the reference's checks in
 * its order (shape, then per vertex: monotone offsets, degree, isolated, neighbour range,
 * sortedness, duplicates unless multi; entry counts; symmetry) with its messages naming the
 * first failing vertex; on success the GraphStats. */
cheb_status cheb_validate_csr(const int64_t* offsets, int64_t n_offsets, const int64_t* neighbors, int64_t nnz,
                              const int64_t* degrees, int64_t n_degrees, int64_t n, int64_t m, int multi,
                              int64_t duplicates_removed, int64_t isolated_dropped, int device,
                              cheb_graph_stats* stats);
/* validate (graph.cpp:123-186) statistics of a device graph built by K1 (whose invariants
 * hold by construction): n, m, avg/min/max degree, self loops, builder counts. */
cheb_status cheb_graph_validate_stats(cheb_graph_t g, cheb_graph_stats* stats);

/* cpaa.cpp:40-68 partition_vertices: degree-prefix cuts (host rule, the reference's; the
 * multi-GPU partition is block-cyclic instead, see cheb_partition_block_rows).  cuts has K+1
 * entries. */
cheb_status cheb_partition_vertices(const int64_t* degrees, int64_t n, int K, int64_t* cuts);

/* Row partition plan (host only): the view's degree-descending relabel (order[new] = old,
 * ties by id) — the order the device partition deals out block-cyclically — and, for
 * reference, the reference cut rule (cpaa.cpp:40-68) applied to the relabelled degree
 * sequence -> cuts[G+1] over new ids with max_rows = the largest such slice. */
cheb_status cheb_partition_plan(const int64_t* degrees, int64_t n, int G, int64_t* order,
                                int64_t* cuts, int64_t* max_rows);

/* Multi-GPU (one process per GPU): an NCCL communicator shared by G ranks.  Attaching
 * it to a graph handle (every rank holds the same graph) partitions the solver view
 * block-cyclically: cheb_cpaa then becomes a collective over the G ranks — each rank
 * runs the fused term kernel on its rows and all-gathers x_{k+1} (ncclAllGather of equal
 * slots, then back to the global sorted order) before the next term; trace sums are
 * combined in rank order and every
 * rank receives the full ranks vector.  FAST schedule only. */
typedef struct cheb_comm* cheb_comm_t;
cheb_status cheb_nccl_unique_id(void* out, int out_bytes); /* 128-byte ncclUniqueId */
cheb_status cheb_comm_create(const void* unique_id, int nranks, int rank, int device, cheb_comm_t* out);
void cheb_comm_destroy(cheb_comm_t c);
cheb_status cheb_graph_attach_comm(cheb_graph_t g, cheb_comm_t comm);
/* Rows per block of the block-cyclic (snake-order) row partition of a partitioned handle (new):
 * block b of the degree-sorted rows, cycle c = b / G, goes to rank b mod G on even cycles and
 * to G - 1 - (b mod G) on odd ones; x stays in the global sorted order on every rank. */
int cheb_partition_block_rows(void);
cheb_status cheb_graph_partition_info(cheb_graph_t g, int64_t* lo, int64_t* hi, int64_t* nnz_local,
                                      int64_t* max_rows);
/* Exchange volume of this rank's local rows per term (new; no reference counterpart): remote
 * x_{k+1} stores of the halo-only push (a row's value goes only to the ranks owning one of
 * its neighbours) and of replicate-to-every-rank ((G - 1) per local row). */
cheb_status cheb_graph_exchange_info(cheb_graph_t g, int64_t* halo_stores, int64_t* all_stores);
/* Solver-view introspection (new; tests and tools): sizes[5] = {n_local, nnz_local, n_hub,
 * n_chunk_tiles, hot-prefix capacity (fp64 entries)}; row_ptr[n_local + 1] (widened), col[nnz_local]
 * (renamed ids in storage order), order[n_local] (view row -> vertex), chunk_begin[n_chunk_tiles + 1]
 * (first entry of every hub-row chunk tile).  Any output may be NULL. */
cheb_status cheb_graph_view_download(cheb_graph_t g, int64_t* sizes, int64_t* row_ptr, int32_t* col,
                                     int32_t* order, int64_t* chunk_begin);
/* Column windows of the hub rows (new; tests and tools): sizes[8] = {windows NW (0: none), entries of
 * x per window W, first windowed id H0, stream blocks (256 entries each), windowed entries, pieces
 * (sums the window pass stores, padding included), chunk tiles left to the term kernel over the hub
 * rows, listed pieces}.  wcol[blocks * 256]: window-local ids, window-major; lane_meta[blocks * 32]:
 * per lane of a block (8 consecutive entries) its piece-start bits | pieces started in the block's
 * earlier lanes << 8; block_base[blocks + 1]: pieces before each block; row_first[n_hub + 1] and
 * piece_list[listed]: the pieces (stream indices) of every hub row.  Window w holds the ids
 * [H0 + w W, H0 + (w + 1) W) and starts at a block boundary.  Any output may be NULL. */
cheb_status cheb_graph_view_windows(cheb_graph_t g, int64_t* sizes, uint16_t* wcol, uint16_t* lane_meta,
                                    int32_t* block_base, int32_t* row_first, int32_t* piece_list);
/* Warp tiles of the solver view (new; tests and tools): *n_tiles, then per tile its first
 * entry, first row (a chunk tile: its hub row) and meta (log2 lanes per row, or 0x10 = chunk
 * of a hub row) for tiles [0, n_tiles] (tile n_tiles: the sentinel {nnz_local, n_local, 0});
 * *n_launches = term-kernel launches per term (1, or K with the opt-in column-blocked
 * schedule).  Arrays may be NULL (sizes only). */
cheb_status cheb_graph_view_tiles(cheb_graph_t g, int64_t* n_tiles, int64_t* nnz_begin, int32_t* row_begin,
                                  int32_t* meta, int32_t* n_launches);

/* ---- solvers ---- */
enum { CHEB_MODE_FAST = 0, CHEB_MODE_BITEXACT = 1 };
enum { CHEB_FP64 = 64, CHEB_FP32 = 32 };

typedef struct {
    double c;                    /* SolverConfig::c (cpaa.hpp:28) */
    int rounds;                  /* SolverConfig::rounds (cpaa.hpp:32), -1 = unset */
    double eps;                  /* SolverConfig::eps (cpaa.hpp:33), -1 = unset */
    int max_rounds;              /* SolverConfig::max_rounds (cpaa.hpp:34), default 60 */
    int parallelism;             /* SolverConfig::parallelism (cpaa.hpp:35): accepted, no effect
                                    on results (bit-identical for every K, as the reference) */
    int mode;                    /* CHEB_MODE_FAST (degree-binned, within 1e-12) or
                                    CHEB_MODE_BITEXACT (storage-order sums, bitwise = reference) */
    int precision;               /* CHEB_FP64 or CHEB_FP32 (new) */
    int R;                       /* number of right-hand sides (new; 1 = reference) */
    const double* personalization; /* n*R row-major host array or NULL = ones (new) */
    int trace;                   /* fill trace rows (default 1) */
} cheb_cpaa_opts;

/* One TraceRow (cpaa.hpp:38-49). */
typedef struct {
    int k;
    double c_k, S_k, residual_mass, l1_change, elapsed_ms, mass_T, err, err_l1;
} cheb_trace_row;

void cheb_cpaa_opts_default(cheb_cpaa_opts* o);

/* run_cpaa (cpaa.hpp:74-75, cpaa.cpp:79-165).  ranks: n*R host doubles (row-major).
 * trace: rounds rows (may be NULL; rounds <= max_rounds).  reference: optional vector of
 * n_reference entries (err/err_l1 columns, cpaa.cpp:149-154; length checked as cpaa.cpp:84-85).
 * rounds_out/total_mass_out may be NULL. */
cheb_status cheb_cpaa(cheb_graph_t g, const cheb_cpaa_opts* opts, const double* reference,
                      int64_t n_reference, double* ranks, cheb_trace_row* trace,
                      int* rounds_out, double* total_mass_out);

/* Device-resident variant for benchmarks: leaves ranks in the handle's device buffer
 * (returned via *d_ranks, n*R values of the solve precision), no host copies, enqueued on
 * the handle's stream.  Synchronises before returning iff sync != 0. */
cheb_status cheb_cpaa_device(cheb_graph_t g, const cheb_cpaa_opts* opts, const void** d_ranks,
                             int sync);
/* Device time (ms) of the last cheb_cpaa_device term loop, measured with CUDA events on the
 * handle's stream: loop_ms covers init+M terms+normalise, term_ms is loop_ms's per-term share
 * excluding init/normalise when measurable. */
cheb_status cheb_last_timing(cheb_graph_t g, double* loop_ms, double* term_kernel_ms,
                             int* terms, int* launches);

/* Batched personalised CPAA (K5, config 5): R right-hand sides in one SpMM-shaped pass per
 * term.  Column r starts from T_0 = e_{seeds[r]} (seeds: R vertex ids) or from the dense
 * opts->personalization (n x R row-major) or from ones.  ranks: n x R row-major host doubles
 * (column r normalised by totals[r]); trace rows carry sums over all R columns.  FAST only. */
cheb_status cheb_cpaa_batch(cheb_graph_t g, const cheb_cpaa_opts* opts, const int64_t* seeds,
                            double* ranks, double* totals, cheb_trace_row* trace, int* rounds_out);
cheb_status cheb_cpaa_batch_profile(cheb_graph_t g, const cheb_cpaa_opts* opts, const int64_t* seeds,
                                    double* term_ms, int capacity, int* terms);

/* Per-term kernel durations (ms) of one solve, CUDA events around every fused term launch
 * on the handle's stream (plain launches, no graph).  Used for the roofline figure. */
cheb_status cheb_cpaa_profile(cheb_graph_t g, const cheb_cpaa_opts* opts, double* term_ms,
                              int capacity, int* terms);

/* Experiment knobs for kernel studies (not for production use): "hot" caps the shared-memory
 * hot-prefix size in vertices (-1 = full capacity); "nogather" = 1 replaces x gathers by
 * constants (timing of everything but the gather; results are wrong).  "windows" / "winsize" /
 * "winh0" (views built afterwards): the number of column windows of the hub rows (0 off, -1 the
 * default policy: graphs of >= 48 M entries), the ids per window and the first windowed id.  The
 * full list is `Tuning` in csrc/common.cuh; an unknown key returns CHEB_INVALID_ARG. */
cheb_status cheb_set_tuning(const char* key, int value);

/* run_power (power.hpp:24-25, power.cpp:28-109). */
typedef struct {
    double c;       /* PowerConfig::c */
    int rounds;     /* PowerConfig::rounds, -1 = unset */
    double tol;     /* PowerConfig::tol, -1 = unset */
    int max_rounds; /* PowerConfig::max_rounds (60) */
    int parallelism;
    int mode;       /* CHEB_MODE_FAST / CHEB_MODE_BITEXACT */
} cheb_power_opts;
void cheb_power_opts_default(cheb_power_opts* o);
cheb_status cheb_power(cheb_graph_t g, const cheb_power_opts* opts, const double* reference,
                       int64_t n_reference, double* ranks, cheb_trace_row* trace,
                       int trace_capacity, int* rounds_out, double* total_mass_out);

/* transition_apply (graph.hpp:64, graph.cpp:104-121): y = P x. */
cheb_status cheb_transition_apply(cheb_graph_t g, const double* x, int64_t nx, double* y,
                                  int mode);

/* Staged API (cpaa.hpp:79-85, cpaa.cpp:167-196), device-backed with the SAME arithmetic as
 * cheb_cpaa in the given mode, so staged and fused results are bitwise equal
 * (test_cpaa.cpp:157-173).  The state lives on the device inside the handle. */
cheb_status cheb_state_init(cheb_graph_t g, double c0, int mode);      /* init_state */
cheb_status cheb_state_set(cheb_graph_t g, const double* T_prev, const double* T_curr,
                           const double* acc, int k);
cheb_status cheb_state_generate(cheb_graph_t g);                       /* generate_stage */
cheb_status cheb_state_accumulate(cheb_graph_t g, double c_k);         /* accumulate_stage */
cheb_status cheb_state_rotate(cheb_graph_t g);  /* T_prev<-T_curr<-T_next, k++ */
cheb_status cheb_state_get(cheb_graph_t g, double* T_prev, double* T_curr, double* T_next,
                           double* acc, int* k);

/* ---- generators: generate.hpp:27-40 (host, std::mt19937_64 as the reference) ---- */
/* Host outputs: E interleaved int64 pairs, malloc'ed; release with cheb_free. */
cheb_status cheb_gen_ring(int64_t n, int64_t** edges, int64_t* E);                /* :28 */
cheb_status cheb_gen_star(int64_t n, int64_t** edges, int64_t* E);                /* :31 */
cheb_status cheb_gen_regular(int64_t n, int64_t k, int64_t** edges, int64_t* E);  /* :35 */
cheb_status cheb_gen_gnp(int64_t n, double p, uint64_t seed, int64_t** edges, int64_t* E); /* :40 */
/* New, counter-based (host == device bit for bit).  Output: E interleaved int32 pairs,
 * on the device (cudaMalloc on `device`, release with cheb_device_free) when on_device,
 * else on the host (malloc, release with cheb_free). */
cheb_status cheb_gen_rmat(int scale, int64_t edge_factor, double a, double b, double c,
                          uint64_t seed, int on_device, int device, void** edges, int64_t* E);
cheb_status cheb_gen_chung_lu(int64_t n, double gamma, double wmin, double wmax, int64_t draws,
                              uint64_t seed, int on_device, int device, void** edges, int64_t* E);
const char* cheb_gen_last_error(void);
void cheb_free(void* p);
void cheb_device_free(void* p, int device);

/* kahan_sum (graph.hpp:75) on the host, exactly as graph.cpp:10-19. */
double cheb_kahan_sum(const double* x, int64_t n);

/* ---- fused push exchange: x_{k+1} stored by the term kernels straight
 * into every rank's buffer (NVLink peer memory), a release/acquire flag barrier per term;
 * replaces the NCCL all-gather of cheb_graph_attach_comm. ---- */
typedef struct cheb_group* cheb_group_t;
/* One process drives G partition ranks (graphs[r] = rank r; the same graph on every handle,
 * on one device or several peer-accessible devices). */
cheb_status cheb_group_create(cheb_graph_t* graphs, int G, cheb_group_t* out);
/* cheb_cpaa over the whole group: ranks (full vector, vertex order), trace, rounds, total
 * as cheb_cpaa.  FAST mode, no reference tracking. */
cheb_status cheb_group_cpaa(cheb_group_t grp, const cheb_cpaa_opts* opts, double* ranks,
                            cheb_trace_row* trace, int* rounds, double* total);
/* Per-rank balance of a lockstep group (new): the same solve with the ranks' term kernels
 * serialised (rank r's term after rank r-1's), so each rank's mean term time (ms, CUDA events)
 * is measured on the whole GPU; rank_term_ms[G]. */
cheb_status cheb_group_profile(cheb_group_t grp, const cheb_cpaa_opts* opts, double* rank_term_ms, int capacity);
void cheb_group_destroy(cheb_group_t grp); /* detaches the graphs (they become single-GPU) */
/* One process per GPU: make g rank `rank` of G and write its exchange-buffer IPC handles
 * (CHEB_PEER_EXPORT_BYTES) to out; gather every rank's bytes (rank order) and pass them to
 * cheb_peer_import; cheb_cpaa on g then runs the partitioned solve with the push exchange. */
#define CHEB_PEER_EXPORT_BYTES 384
cheb_status cheb_peer_export(cheb_graph_t g, int G, int rank, void* out, size_t cap);
cheb_status cheb_peer_import(cheb_graph_t g, const void* all, size_t bytes_per_rank);
cheb_status cheb_peer_detach(cheb_graph_t g);

/* Solver-view tile bins of the FAST schedule (for profiling): bin b = 0..5 pack tiles with
 * 2^b lanes per row, bin 6 chunk tiles of rows above the warp tile; per bin the number of
 * tiles, rows and CSR entries. */
cheb_status cheb_graph_view_bins(cheb_graph_t g, int64_t* tiles, int64_t* rows, int64_t* nnz);

#ifdef __cplusplus
}
#endif
#endif /* CHEBPR_CUDA_H */
