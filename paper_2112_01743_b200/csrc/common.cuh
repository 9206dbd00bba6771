// Internal header of libchebpr_b200: error plumbing, device buffers, the graph
// handle and the kernel-side helpers shared by the CSR builder and the term kernels.
#pragma once

#include <cuda_runtime.h>

#include <atomic>
#include <chrono>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <functional>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

#include <nvtx3/nvToolsExt.h>

#include "chebpr_cuda.h"

namespace chebgpu {

// Internal exception; converted to cheb_status at the C-ABI (capi.cu).
struct Error : std::runtime_error {
    cheb_status code;
    Error(cheb_status c, const std::string& m) : std::runtime_error(m), code(c) {}
};

[[noreturn]] inline void fail(cheb_status c, const std::string& m) { throw Error(c, m); }

#define CHEB_CUDA_CHECK(expr)                                                            \
    do {                                                                                 \
        cudaError_t _e = (expr);                                                         \
        if (_e != cudaSuccess)                                                           \
            ::chebgpu::fail(CHEB_CUDA, std::string("CUDA error ") + cudaGetErrorString(_e) + \
                                           " at " __FILE__ ":" + std::to_string(__LINE__) + \
                                           " (" #expr ")");                              \
    } while (0)

// Stream that device allocations of the current API call are ordered on (set by
// AllocScope).  Allocations come from the device's stream-ordered memory pool, whose
// release threshold is raised once per device so freed blocks are reused instead of
// returned to the driver (cheap per-call setup for the reference's stateless API).
inline cudaStream_t& alloc_stream() {
    thread_local cudaStream_t s = nullptr;
    return s;
}
struct AllocScope {
    cudaStream_t prev;
    explicit AllocScope(cudaStream_t s) : prev(alloc_stream()) { alloc_stream() = s; }
    ~AllocScope() { alloc_stream() = prev; }
};
void retain_pool_memory();  // capi.cu
// Non-blocking streams recycled across graph handles of the device (the reference API is
// stateless, so every drop-in call makes and frees a handle): a released stream must be idle.
cudaStream_t pooled_stream(int device);
void release_stream(int device, cudaStream_t s);

// L2 persistence for the gathered vector: an access-policy window over the first `bytes` of
// `base` (the degree-sorted hot prefix of x), sized to the device's persisting-L2 limit.
// Returns false when the device offers no persisting L2.
// decide_bytes: the size that decides whether a window is used at all (default: bytes)
bool l2_window(const void* base, size_t bytes, cudaAccessPolicyWindow* w, size_t decide_bytes = 0);

inline bool alloc_debug() {
    static const bool on = std::getenv("CHEB_DEBUG_ALLOC") != nullptr;
    return on;
}

// Owning device allocation (untyped bytes; typed views via ptr<T>()).
class DevMem {
public:
    DevMem() = default;
    explicit DevMem(size_t bytes) { alloc(bytes); }
    ~DevMem() { release(); }
    DevMem(const DevMem&) = delete;
    DevMem& operator=(const DevMem&) = delete;
    DevMem(DevMem&& o) noexcept : p_(o.p_), n_(o.n_), st_(o.st_), async_(o.async_) {
        o.p_ = nullptr;
        o.n_ = 0;
    }
    DevMem& operator=(DevMem&& o) noexcept {
        if (this != &o) {
            release();
            p_ = o.p_;
            n_ = o.n_;
            st_ = o.st_;
            async_ = o.async_;
            o.p_ = nullptr;
            o.n_ = 0;
        }
        return *this;
    }
    void alloc(size_t bytes) {
        release();
        if (bytes == 0) bytes = 16;
        st_ = alloc_stream();
        async_ = st_ != nullptr;
        const auto t0 = std::chrono::steady_clock::now();
        if (async_) {
            retain_pool_memory();
            CHEB_CUDA_CHECK(cudaMallocAsync(&p_, bytes, st_));
        } else {
            CHEB_CUDA_CHECK(cudaMalloc(&p_, bytes));
        }
        n_ = bytes;
        if (alloc_debug()) {
            const double ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
            if (ms > 1.0 || bytes > (size_t(1) << 30))
                std::fprintf(stderr, "[alloc] %s %.1f MB in %.2f ms\n", async_ ? "pool" : "cudaMalloc", bytes / 1e6, ms);
        }
    }
    // Grow-only reuse.
    void ensure(size_t bytes) {
        if (bytes > n_ || !p_) alloc(bytes);
    }
    void release() {
        if (p_) {
            if (async_) cudaFreeAsync(p_, st_);
            else cudaFree(p_);
        }
        p_ = nullptr;
        n_ = 0;
    }
    // Return the block to the pool on `s` from now on (a buffer built on an auxiliary
    // stream and joined into the owner's stream).
    void set_stream(cudaStream_t s) {
        if (async_) st_ = s;
    }
    template <class T>
    T* ptr() const { return static_cast<T*>(p_); }
    void* get() const { return p_; }
    size_t bytes() const { return n_; }
    explicit operator bool() const { return p_ != nullptr; }

private:
    void* p_ = nullptr;
    size_t n_ = 0;
    cudaStream_t st_ = nullptr;
    bool async_ = false;
};

// Scoped device selection.
struct DeviceGuard {
    int prev = -1;
    explicit DeviceGuard(int dev) {
        cudaGetDevice(&prev);
        if (prev != dev) CHEB_CUDA_CHECK(cudaSetDevice(dev));
    }
    ~DeviceGuard() {
        if (prev >= 0) cudaSetDevice(prev);
    }
};

// NVTX ranges (SURVEY.md §5 tracing): every C-ABI entry point is one named range, the
// phases inside (upload, solver view, solve enqueue) nested ranges, so an nsys / ncu
// timeline shows where a call's time goes.  nvtx3 is header-only: with no tool attached
// each push/pop is a cheap no-op.
struct NvtxRange {
    explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
    ~NvtxRange() { nvtxRangePop(); }
    NvtxRange(const NvtxRange&) = delete;
    NvtxRange& operator=(const NvtxRange&) = delete;
};

// Per-device one-time setup flags (function attributes, pool attributes): a context
// property must be set on every device a process uses, and handles on different devices
// may be driven from different host threads.  first_on_device(mask, dev) is true exactly
// once per (mask, dev); devices >= 64 always return true (the setup is idempotent).
inline bool first_on_device(std::atomic<uint64_t>& mask, int dev) {
    if (dev < 0 || dev >= 64) return true;
    const uint64_t bit = uint64_t(1) << dev;
    return (mask.fetch_or(bit, std::memory_order_acq_rel) & bit) == 0;
}

// --------------------------------------------------------------------------
// Degree-binned solver view (the hot-path layout, built once per graph).
//
// Rows are relabelled by degree (descending, ties by id) so that every bin is a
// contiguous row range and the most-gathered x entries (hubs) share cache lines.
// Column ids are renamed, but every row keeps its neighbours in the reference's
// storage order.  order[new] = old.
// --------------------------------------------------------------------------
// Warp tiles of the degree-sorted view.  meta: low 4 bits = log2(lanes per row) for
// pack tiles; kTileChunk marks a 256-nnz chunk of a row with degree > kWarpNnz (row_begin = the
// row).  tiles[n_tiles] is a sentinel {nnz, n}.
struct Tile {
    int64_t nnz_begin;
    int32_t row_begin;
    int32_t meta;
};
// A tile as stored in a warp's program (warp-major copy of the tiles the warp visits:
// tile t = w + i * (grid * kWarps) is entry i of warp w).
struct WTile {
    int64_t nnz_begin;
    int32_t row_begin;
    uint16_t cnt;
    uint8_t rows;
    uint8_t meta;
};
static_assert(sizeof(WTile) == 16, "WTile is 16 bytes");
constexpr int kWinSmemMax = 226 * 1024;            // dynamic shared memory of k_window_pass (+ its static mbarrier)
constexpr int kWinMaxIds = (kWinSmemMax / 8) & ~7;  // ids per window: an fp64 window must fit (28,928)
constexpr int kWinBlock = 256;       // entries per block of the window stream (a warp: 8 per lane)
constexpr int kDescBlock = 8;        // descriptors per TMA refill of a warp's program ring
constexpr int kThreads = 256;        // CTA size of the auxiliary kernels
#ifndef CHEB_WARPS
#define CHEB_WARPS 32
#endif
constexpr int kWarps = CHEB_WARPS;   // warps per CTA of the term kernel (1 CTA / SM)
constexpr int kWarpNnz = 248;        // nnz per tile: with <= 7 alignment slots, 8 per lane
constexpr int kWarpRows = 32;        // rows per pack tile (one per lane)
constexpr int kColBuf = 264;         // ints per TMA column buffer (256 + alignment slack)
#ifndef CHEB_HOT_KB
#define CHEB_HOT_KB 86
#endif
constexpr int kHotBytes = CHEB_HOT_KB * 1024;  // shared hot x prefix; sized so hot + scratch fit the 164 KB carve-out and L1 keeps ~64 KB (tools/variant_run.sh sweep)
constexpr int kTileChunk = 0x10;

// build.cu: cudaMalloc'ed blocks of the views' window arrays, recycled per device (a block
// given back may be handed to any later view of the device: give() waits for the device)
class DevMem;
void window_arena_take(DevMem& out, size_t bytes);
void window_arena_give(DevMem& blk);

struct SolverView {
    bool ready = false;
    bool rp64 = false;
    DevMem order;      // int32 [n_local]  local row -> old id
    DevMem rank;       // int32 [n]  old id -> view row (single-GPU views: the ranks are gathered in vertex order)
    DevMem order_full; // int32 [n]  global sorted row -> old id (partitioned runs only)
    int64_t n_local = 0, nnz_local = 0, x_len = 0;
    int part_G = 1, part_r = 0;  // local row i is sorted row part_global(i, part_r, part_G)
    DevMem row_ptr;    // int32/int64 [n+1] (new order)
    DevMem col;        // int32 [nnz] (renamed ids, storage order kept)
    DevMem inv;        // double [n] (new order) only when inv_degree is non-canonical
    DevMem tiles;      // Tile [n_tiles + 1]
    DevMem prog;       // WTile [grid * kWarps][prog_len]: per-warp tile programs
    int prog_len = 0;  // entries per warp (multiple of kDescBlock)
    int n_tiles = 0;
    int grid = 0;          // CTAs of one term launch (persistent: one per SM)
    int64_t n_hub = 0;     // rows [0, n_hub) with degree > kWarpNnz (chunk tiles)
    int64_t n_hub_wide = 0;  // rows [0, n_hub_wide): more than 32 chunk tiles (hub finalize: a warp each)
    int n_chunk_tiles = 0;
    DevMem hub_first;      // int32 [n_hub + 1]: first chunk tile of each hub row
    // Column-blocked schedule (x larger than L2): hub-row chunks never straddle a block of x
    // ids, and each term runs one launch per block (highest block first) whose program holds
    // that block's chunks, under an L2 window over that slice of x; the last launch (block 0)
    // also runs the pack tiles and the row epilogues.  Empty: one launch over `prog`.
    struct Phase {
        int64_t prog_off = 0;  // WTile offset of this launch's program inside `prog`
        int prog_len = 0, ntiles = 0;
        int64_t x_lo = 0, x_hi = 0;  // x ids this launch's chunks gather (its L2 window)
        bool epi = false;            // runs pack tiles (row epilogues, trace partials)
    };
    std::vector<Phase> phases;
    bool sorted_rows = false;  // rows hold their renamed ids in ascending order
    // Column windows of the hub rows (build.cu window_schedule): the x ids
    // [H0, H0 + NW W) are cut into NW windows of W entries.  Every hub row's entries inside a
    // window (a contiguous piece of the ascending row) are copied, as 16-bit window-local ids,
    // into one window-major stream cut into blocks of kWinBlock entries; k_window_pass loads a
    // window of x_k into shared memory and sums each piece from there, so these entries cost
    // no L2 sector.  A piece (cut again where it crosses a block) writes its sum to
    // hub_part[MC + k], k its index in stream order (coalesced stores); slots [0, MC) are the
    // chunk tiles over the entries left in the rows (hot prefix and cold ids).  k_hub_finalize
    // adds a row's chunk partials hub_part[hub_first[h] ..) and its pieces klist[kf[h] ..).
    // The term kernel then runs `prog` below instead of the view's own program (which, with
    // tiles / hub_first above, stays as built for the batched path and the introspection).
    struct Span {  // a piece of one of the two allocations below
        void* p = nullptr;
        template <class T>
        T* ptr() const { return static_cast<T*>(p); }
        void* get() const { return p; }
    };
    struct Windows {
        bool ready = false;
        int NW = 0, W = 0, H0 = 0;
        int64_t n_blocks = 0;      // stream blocks (kWinBlock entries each)
        int64_t n_slots = 0;       // hub_part slots: MC + pieces
        int MC = 0;                // main chunk tiles (slots [0, MC))
        int64_t n_wide = 0;        // hub rows [0, n_wide) finalized by a warp each
        int64_t entries = 0;       // windowed entries (statistics)
        int64_t pieces = 0;        // their slots
        Span wcol;               // uint16 [n_blocks * kWinBlock] window-local ids
        Span flags;              // uint8 [n_blocks * 32]: bit i of byte j = entry 8 j + i starts a piece
        Span meta;               // uint16 [n_blocks * 32]: per lane, its start bits | pieces in earlier lanes << 8
        Span bbase;              // int32 [n_blocks + 1]: pieces before each block
        Span kf;                 // int32 [n_hub + 1]: first klist entry of each hub row
        Span klist;              // int32: the rows' pieces (stream indices), row by row
        Span wblk;               // int64 [NW + 1]: first block of each window
        Span cta;                // int64 [grid + 1]: block range of each CTA of the window pass
        int grid = 0;
        Span prog;               // WTile programs of the term kernel (main chunk tiles + pack tiles)
        int prog_len = 0, n_tiles = 0;
        Span hub_first;          // int32 [n_hub + 1]: first main chunk tile (slot) of each hub row
        // The arrays above are carved from two blocks (the stream and its indices; the piece
        // lists and the program) of plain cudaMalloc memory recycled through a small per-device
        // cache (build.cu window_arena_take / _give): steady-state uploads allocate nothing for
        // the windows.  As ~18 separate pool allocations per upload they left the memory pool
        // unable to place the next upload's 4 GB buffers without remapping (config 4 e2e: uploads
        // of 176 ms with 240-1340 ms outliers); as two pool blocks, next to a resident graph's,
        // the outliers came back inside bench.py (e2e steps of 284-1520 ms).
        DevMem arena_a, arena_b;
        void release() {
            ready = false;
            for (Span* d : {&wcol, &flags, &meta, &bbase, &cta, &kf, &klist, &wblk, &prog, &hub_first}) d->p = nullptr;
            window_arena_give(arena_a);
            window_arena_give(arena_b);
        }
        Windows() = default;
        Windows(Windows&&) = default;
        Windows& operator=(Windows&& o) noexcept {
            if (this != &o) {
                release();  // the blocks go back to the cache, not to cudaFree
                ready = o.ready; NW = o.NW; W = o.W; H0 = o.H0; n_blocks = o.n_blocks; n_slots = o.n_slots;
                MC = o.MC; n_wide = o.n_wide; entries = o.entries; pieces = o.pieces; grid = o.grid;
                prog_len = o.prog_len; n_tiles = o.n_tiles;
                wcol = o.wcol; flags = o.flags; meta = o.meta; bbase = o.bbase; kf = o.kf; klist = o.klist;
                wblk = o.wblk; cta = o.cta; prog = o.prog; hub_first = o.hub_first;
                arena_a = std::move(o.arena_a);
                arena_b = std::move(o.arena_b);
                o.ready = false;
            }
            return *this;
        }
        ~Windows() { release(); }
    };
    Windows win;
    // Row partition (G > 1): bit r of push_mask[u] = rank r has a row with neighbour u, i.e.
    // needs x[u] (symmetric graph: u has a neighbour owned by r).  The halo-only push stores
    // x_{k+1}[u] only there.  push_entries = sum of popcounts over the local rows minus the
    // rows' own-rank bits (remote stores per term).
    DevMem push_mask;          // uint32 [n_local]
    DevMem col_sorted;         // batched path only: col with each row in ascending id order
    int64_t push_entries = 0, push_entries_all = 0;  // halo / replicate-everything remote stores
    // tile bins (host statistics): 0..5 = pack tiles with 2^b lanes per row, 6 = chunk tiles
    int64_t bin_tiles[7] = {}, bin_rows[7] = {}, bin_nnz[7] = {};
    void set_stream(cudaStream_t s) {
        for (DevMem* d : {&order, &rank, &order_full, &row_ptr, &col, &inv, &tiles, &prog, &hub_first, &push_mask,
                          &col_sorted})
            d->set_stream(s);
    }
};

// 1-D row partition of the degree-sorted view over G GPUs (one process per GPU), block-
// cyclic in snake order: sorted rows are cut into blocks of kPartRows; block b of cycle
// c = b / G goes to rank j = b mod G on even cycles and to G - 1 - j on odd ones.  Every rank
// thus holds the same mix of hub and leaf rows (nnz and row counts balanced to within a
// block per cycle), where contiguous degree-prefix ranges (the reference's partition_vertices
// rule, cpaa.cpp:40-68, measured round 2: tools/rank_balance.py) leave one rank with every
// low-degree row and cap 8-GPU scaling at ~1.6x on config 4.  x keeps the global sorted
// order on every rank (no padding): rank r's local row i is sorted row part_global(i, r, G),
// so the view's column ids, hot prefix and L2 window are the single-GPU ones.
constexpr int kPartLgRows = 6;
constexpr int64_t kPartRows = int64_t(1) << kPartLgRows;
__host__ __device__ __forceinline__ int part_owner(int64_t u, int G) {
    const int64_t b = u >> kPartLgRows, c = b / G;
    const int j = (int)(b - c * G);
    return (c & 1) ? G - 1 - j : j;
}
__host__ __device__ __forceinline__ int64_t part_global(int64_t i, int r, int G) {
    const int64_t c = i >> kPartLgRows;
    const int j = (c & 1) ? G - 1 - r : r;
    return ((c * G + j) << kPartLgRows) | (i & (kPartRows - 1));
}
__host__ __device__ __forceinline__ int64_t part_local(int64_t u, int G) {
    return (((u >> kPartLgRows) / G) << kPartLgRows) | (u & (kPartRows - 1));
}
struct Partition {
    int G = 1, rank = 0;
    std::vector<int64_t> rows{0};  // rows per rank
    int64_t max_rows = 0;          // largest rank's row count (NCCL slot size)
    void* comm = nullptr;  // ncclComm_t (owned by the cheb_comm handle, not by the graph)
};
// rows of an n-row view owned by each of G ranks
inline std::vector<int64_t> part_rows(int64_t n, int G) {
    std::vector<int64_t> rows((size_t)G, 0);
    const int64_t nb = (n + kPartRows - 1) / kPartRows;
    for (int64_t b = 0; b < nb; ++b) {
        const int64_t c = b / G;
        const int j = (int)(b - c * G);
        const int r = (c & 1) ? G - 1 - j : j;
        rows[(size_t)r] += std::min<int64_t>(kPartRows, n - b * kPartRows);
    }
    return rows;
}

// Fused push exchange of a row partition: every rank owns IPC-exportable
// exchange buffers and holds pointers to every peer's copies (IPC-opened or, when one
// process drives all ranks, plain/peer pointers).  The term epilogue stores x_{k+1} into
// all G buffers; a release/acquire flag barrier separates terms.
constexpr int kMaxPushTerms = 1024;  // trace slots per rank in the exchange buffer
struct PeerGroup {
    int G = 1, rank = 0;
    bool lockstep = false;  // all ranks driven by one host thread (cheb_group_*)
    int64_t x_len = 0;
    // this rank's own buffers (cudaMalloc: IPC-exportable)
    void* X[2] = {nullptr, nullptr};       // x_k in the global sorted order, x_len * 8 bytes each
    void* trace_all = nullptr;             // [G][2 * kMaxPushTerms] doubles
    void* rbuf = nullptr;                  // ranks in the global sorted order, x_len * 8 bytes
    unsigned long long* flags = nullptr;   // [G] barrier epochs written by the peers, [G] timeout flag
    // every rank's buffers as seen from this device ([rank] = own)
    std::vector<void*> pX0, pX1, ptrace, prbuf, pflags;
    std::vector<void*> opened;             // IPC-opened peer pointers (closed on release)
    DevMem table;                          // device copies: X0[G] X1[G] trace[G] rbuf[G] flags[G]
    unsigned long long epoch = 0;          // barriers passed (identical on every rank)
    cudaEvent_t signalled = nullptr;       // lockstep: this rank's last signal
    void release();
};

struct Workspace {
    int64_t n = 0;
    int R = 0;
    int vbytes = 0;
    int M = -1;
    DevMem T0, T1, X0, X1, acc, out;    // vectors (solve precision), out = ranks (orig order)
    DevMem part;                        // double [M][grid][2] block trace partials
    DevMem hub_part;                    // double [grid] chunk partials
    DevMem hub_ts;                      // double [M][n_hub][2]
    DevMem trace;                       // double [M][2] (mass_T, S_k)
    DevMem total;                       // double [1]
    DevMem coeffs;                      // double [M+1]
    DevMem snap;                        // BITEXACT: double [M][2][n] snapshots of T_k, acc_k
    DevMem stamps;                      // u64 [M + 1] term boundary stamps (%globaltimer, ns)
    DevMem done;                        // u32 [M + 1] CTAs finished per term (last one stamps)
    // CUDA graph of the whole solve for a given configuration.
    cudaGraphExec_t exec = nullptr;
    std::string exec_key;
    std::string seen_key;  // last configuration solved without a graph
    int launches = 0;
    // every buffer back to the pool on its stream (the owner calls this while the stream lives)
    void release_buffers() {
        for (DevMem* d : {&T0, &T1, &X0, &X1, &acc, &out, &part, &hub_part, &hub_ts, &trace, &total,
                          &coeffs, &snap, &stamps, &done})
            d->release();
    }
    ~Workspace() {
        if (exec) cudaGraphExecDestroy(exec);
    }
};

struct BatchWorkspace {
    DevMem T0, T1, X0, X1, acc, out, part, hub_part, hub_ts, trace, colpart, totals;
    const int* col = nullptr;  // the view's columns this batched solve gathers through
};

struct StagedState {
    bool active = false;
    int mode = 0;
    int k = 1;
    DevMem T_prev, T_curr, T_next, acc, x;
};

}  // namespace chebgpu

// The opaque handle of the C-ABI.
struct cheb_graph {
    int device = 0;
    cudaStream_t stream = nullptr;
    cudaStream_t aux = nullptr;    // solver-view build overlapped with the CSR upload
    cudaEvent_t ev0 = nullptr, ev1 = nullptr;
    int64_t n = 0, m = 0, nnz = 0;
    int64_t duplicates_removed = 0, isolated_dropped = 0;
    int64_t max_degree = 0, min_degree = 0;
    bool multi = false;
    bool rp64 = false;             // canonical row_ptr width
    bool inv_array = false;        // non-canonical inv_degree uploaded
    chebgpu::DevMem row_ptr;       // canonical CSR (reference order), int32/int64 [n+1]
    chebgpu::DevMem col;           // int32 [nnz]
    chebgpu::DevMem inv;           // double [n] iff inv_array
    chebgpu::SolverView view;
    chebgpu::Workspace ws;
    chebgpu::StagedState staged;
    chebgpu::BatchWorkspace bws;
    chebgpu::Partition part;
    chebgpu::PeerGroup* peer = nullptr;  // fused push exchange (instead of part.comm)
    double last_loop_ms = 0.0;
    int last_terms = 0;
    // device-clock time of each term of the last scalar solve (%globaltimer stamps taken by
    // the last CTA of each term's final kernel; TraceRow::elapsed_ms), empty if unavailable
    std::vector<double> term_elapsed_ms;
    int last_launches = 0;
    ~cheb_graph();
};

namespace chebgpu {
// Device + allocation-stream scope of an API call on a graph handle.
struct GraphScope {
    DeviceGuard dg;
    AllocScope as;
    explicit GraphScope(const cheb_graph* g) : dg(g->device), as(g->stream) {}
};
// Experiment knobs (cheb_set_tuning); defaults = the product configuration.
struct Tuning {
    int hot = -1;       // cap on the shared-memory hot prefix (vertices); -1 = capacity
    int nogather = 0;   // 1: skip the x gathers (timing experiments only; wrong results)
    int skip = 0;       // 1: skip chunk tiles, 2: skip pack tiles, 16+b: only tile bin b (experiments only)
    int l2win = 0;      // 1: persisting-L2 window over the hot prefix of x when x exceeds L2 (round 1:
                        // C4 5.21 -> 4.58 ms/term; with sorted rows + one column buffer it costs 1.6%: off)
    int pdl = 1;        // 1: programmatic dependent launch along the term chain (default on)
    int sortrows = -1;  // view rows in ascending id order: -1 when x exceeds L2, 0 never, 1 always, 2 hub rows only (experiment)
    int chunksched = 1; // hub chunks ordered for conflict-free hot gathers (k_permute_chunks); 2: also
                        // re-ordered after the config-4 row sort (k_schedule_chunks_inplace: no gain, ~57 ms of view build)
    int l2win_mb = -1;  // cap on the persisting window over x (MB); -1 = the device's persisting maximum
    int l2win_pct = 100; // hitRatio of that window (percent)
    int streamcs = 0;   // 1: per-row operands (row pointers, T, acc loads; T, acc stores) as streaming (.cs)
    int xout_hint = -1; // x_{k+1} stores: 0 plain, 1 L2 evict_first policy, 2 .cs, 3 L2 evict_last policy;
                        // -1: plain (config 4 without the window: evict_last 3503-3527 us/term, plain
                        // 3366-3393; with the round-1 window evict_last had won, 4.06 -> 3.95 ms)
    int xdiscard = 0;   // 1: the term kernel drops the x_out buffer's (dead) lines from L2 at its start.
                        // Off: neutral on the current kernel (C2/C3/C4 within 0.2%), and a CTA that
                        // starts late could discard lines other CTAs of the same launch already wrote
    int packsched = 0;  // pack-tile entries ordered for conflict-free hot gathers (k_schedule_pack);
                        // off: no measurable gain (C2 68.8 -> 68.5, C3 381.6 -> 380.2, C4 3953 -> 3950 us/term)
    int batchblock = 128; // right-hand sides per batched pass (column blocks of one call)
    int halo = 1;       // row partition, push exchange: store x_{k+1}[u] only on the ranks that read it
    int prefetch = 0;   // term kernel: L2 prefetch distance in tiles (0 off); slower on C2-C4
    int spmm_hub_mb = 64; // batched path: MB of X rows (the hub prefix) gathered under evict-last
    int spmm_xpol = 0;  // batched path x_{k+1} stores: 0 normal, 1 evict-last hub prefix + streaming rest
    int skipwarm = 0;   // experiment (wrong results): hub-row gathers of ids in [H, skipwarm) dropped
    int colblocks = 0;  // K > 1: hub-row chunks cut at K column blocks of x, one term launch per block
                        // under an L2 window over its slice (rows sorted by id only; C4: no gain, off)
    int upgroups = 16;  // groups of old rows an upload lands in, each permuted + sorted as it lands (C4: 4 -> 16 groups, upload 200 -> 163 ms)
    int colbufs = -1;   // term kernel column-id buffers per warp: -1 auto (1 when x exceeds L2), 1 or 2
    int hubwarp = 0;    // 1: every hub row finalized by a warp (the lane-per-row path off; tests)
    int pull = 1;       // view tiles / programs pulled from pinned host memory by a kernel (not the copy engine)
    int colsplit_pct = -1; // K = 2: first block boundary at this percent of x (-1: equal halves)
    int windows = -1;   // column windows of the hub rows (SolverView::Windows): NW > 0 windows,
                        // 0 off, -1 auto (64 when x exceeds L2, else 24, on graphs of >= 48 M entries)
    int winbank = 1;    // window stream entries ordered inside their pieces for conflict-free shared-memory gathers
    int winpw = 4;      // window pass CTA ranges: cost of a block = 256 + winpw * its pieces
    int winh0 = 0;      // first windowed id (0: the hub rows keep only ids past the last window; config 4 99.5 -> 94.3 ms per
                        // solve, config 3 11.58 -> 10.91); -1 = the fp64 hot-prefix capacity (the term kernel keeps ids below it)
    int bigscratch = 1; // view build: the permute target and the segmented sort's scratch (4 GB each on config 4) from
                        // per-device grow-only blocks instead of the memory pool
    int winskip = 0;    // timing experiments: 1 no window pass, 2 no term kernel, 3 no hub finalize (wrong results);
                        // bits: 4 window pass launched without PDL, 8 term kernel behind it WITH PDL, 16 hub finalize without
    int winsize = 28672; // entries of x per window (clamped to kWinMaxIds; 16-bit local ids; fp64 224 KB of shared memory; C4 24576 -> 28672: 94.1 -> 92.9 ms)
};
inline Tuning& tuning() {
    static Tuning t = [] {
        Tuning x;
        if (const char* e = std::getenv("CHEB_TUNE_HOT")) x.hot = std::atoi(e);
        if (const char* e = std::getenv("CHEB_TUNE_NOGATHER")) x.nogather = std::atoi(e);
        if (const char* e = std::getenv("CHEB_TUNE_SKIP")) x.skip = std::atoi(e);
        if (const char* e = std::getenv("CHEB_TUNE_L2WIN")) x.l2win = std::atoi(e);
        if (const char* e = std::getenv("CHEB_TUNE_PDL")) x.pdl = std::atoi(e);
        if (const char* e = std::getenv("CHEB_TUNE_SORTROWS")) x.sortrows = std::atoi(e);
        if (const char* e = std::getenv("CHEB_TUNE_CHUNKSCHED")) x.chunksched = std::atoi(e);
        if (const char* e = std::getenv("CHEB_TUNE_L2WIN_MB")) x.l2win_mb = std::atoi(e);
        if (const char* e = std::getenv("CHEB_TUNE_L2WIN_PCT")) x.l2win_pct = std::atoi(e);
        if (const char* e = std::getenv("CHEB_TUNE_STREAMCS")) x.streamcs = std::atoi(e);
        if (const char* e = std::getenv("CHEB_TUNE_XOUT_HINT")) x.xout_hint = std::atoi(e);
        if (const char* e = std::getenv("CHEB_TUNE_XDISCARD")) x.xdiscard = std::atoi(e);
        if (const char* e = std::getenv("CHEB_TUNE_PACKSCHED")) x.packsched = std::atoi(e);
        if (const char* e = std::getenv("CHEB_TUNE_BATCHBLOCK")) x.batchblock = std::atoi(e);
        if (const char* e = std::getenv("CHEB_TUNE_HALO")) x.halo = std::atoi(e);
        if (const char* e = std::getenv("CHEB_TUNE_PREFETCH")) x.prefetch = std::atoi(e);
        if (const char* e = std::getenv("CHEB_TUNE_SPMM_HUB_MB")) x.spmm_hub_mb = std::atoi(e);
        if (const char* e = std::getenv("CHEB_TUNE_SPMM_XPOL")) x.spmm_xpol = std::atoi(e);
        if (const char* e = std::getenv("CHEB_TUNE_COLBLOCKS")) x.colblocks = std::atoi(e);
        if (const char* e = std::getenv("CHEB_TUNE_PULL")) x.pull = std::atoi(e);
        if (const char* e = std::getenv("CHEB_TUNE_HUBWARP")) x.hubwarp = std::atoi(e);
        if (const char* e = std::getenv("CHEB_TUNE_COLBUFS")) x.colbufs = std::atoi(e);
        if (const char* e = std::getenv("CHEB_TUNE_UPGROUPS")) x.upgroups = std::atoi(e);
        if (const char* e = std::getenv("CHEB_TUNE_COLSPLIT_PCT")) x.colsplit_pct = std::atoi(e);
        if (const char* e = std::getenv("CHEB_TUNE_WINDOWS")) x.windows = std::atoi(e);
        if (const char* e = std::getenv("CHEB_TUNE_WINSIZE")) x.winsize = std::atoi(e);
        if (const char* e = std::getenv("CHEB_TUNE_WINSKIP")) x.winskip = std::atoi(e);
        if (const char* e = std::getenv("CHEB_TUNE_WINBANK")) x.winbank = std::atoi(e);
        if (const char* e = std::getenv("CHEB_TUNE_WINPW")) x.winpw = std::atoi(e);
        if (const char* e = std::getenv("CHEB_TUNE_WINH0")) x.winh0 = std::atoi(e);
        if (const char* e = std::getenv("CHEB_TUNE_BIGSCRATCH")) x.bigscratch = std::atoi(e);
        return x;
    }();
    return t;
}
// build.cu
void build_from_edges(cheb_graph* g, const void* d_edges, int64_t E, int edge_bits,
                      const cheb_build_opts& o);
// Upload of a host CSR: the H2D copies are enqueued first, `host_checks` (the reference's
// host-side validation; returns whether inv_degree is 1.0/row length bitwise) runs while
// they are in flight, and the solver view is built on an auxiliary stream as soon as the
// offsets have landed, overlapping the neighbour copy.  A canonical inv_degree is never
// copied (the kernels take the reciprocal of the row length, bit-identical).
void upload_csr(cheb_graph* g, const int64_t* offsets, const int64_t* neighbors, int64_t n,
                int64_t nnz, const double* inv_degree, const std::function<bool()>& host_checks);
void download_csr(cheb_graph* g, int64_t* offsets, int64_t* neighbors, int64_t* degrees);
void ensure_view(cheb_graph* g);
// The batched path's ascending-id copy of the view's columns (built on first use).
const int* batch_sorted_cols(cheb_graph* g);
void finalize_stats(cheb_graph* g);
// ingest.cu
void load_graph_text(cheb_graph* g, const std::string& path, const char* mem, int64_t mem_bytes, int format,
                     const cheb_load_opts& o, int64_t* lines, int* weights_ignored);
int64_t count_self_loops(cheb_graph* g);
// validate.cu
void validate_csr(const int64_t* offsets, int64_t n_off, const int64_t* neighbors, int64_t nnz,
                  const int64_t* degrees, int64_t n_deg, int64_t n, int64_t m, int multi, int64_t dup_removed,
                  int64_t iso_dropped, int device, cheb_graph_stats* st);

// host: partition_vertices rule (cpaa.cpp:40-68) over a degree sequence
void partition_cuts(const int64_t* degrees, int64_t n, int K, int64_t* cuts);

// coeffs.cpp (host coefficient kit, coefficients.cpp semantics)
double beta(double c);
double sigma(double c);
double err_bound(double c, int M);
int plan_iterations(double c, double eps, double* predicted);
void coefficients(double c, int M, std::vector<double>& out, double* beta_out, double* c0_out);
int resolve_rounds(double c, int rounds, double eps, int max_rounds);
double kahan_sum(const double* x, int64_t n);

// cpaa.cu
struct SolveSpec {
    double c = 0.85;
    int M = 0;
    int mode = CHEB_MODE_FAST;
    int precision = CHEB_FP64;
    int R = 1;
    const double* p = nullptr;  // host n*R or null
    bool trace = true;
};
// Runs the solve on the device; results stay in g->ws (out = ranks in original order).
// Fills trace (M rows of mass_T,S_k) and total on the host; throws on non-finite.
void cpaa_solve(cheb_graph* g, const SolveSpec& s, bool host_results, std::vector<double>* tr,
                double* total);
struct BatchSpec {
    double c = 0.85;
    int M = 0;
    int precision = CHEB_FP64;
    int R = 1;
    const double* p = nullptr;      // host n x R row-major, or null
    const int64_t* seeds = nullptr;  // host R vertex ids (one-hot columns), or null
    bool record_start = true;        // false: a later column block of one call (timing spans all)
};
void cpaa_batch_solve(cheb_graph* g, const BatchSpec& s, std::vector<double>& trace,
                      std::vector<double>& totals, std::vector<double>* term_ms);
void read_batch_ranks(cheb_graph* g, double* ranks, int R);
void cpaa_solve_ref(cheb_graph* g, const SolveSpec& s, const double* h_ref, std::vector<double>* tr,
                    std::vector<double>* errs, double* total);
void read_ranks(cheb_graph* g, int precision, double* ranks);
void group_solve(const std::vector<cheb_graph*>& gs, const SolveSpec& s, std::vector<double>* tr, double* total,
                 std::vector<double>* rank_ms = nullptr);
void dist_solve(cheb_graph* g, const SolveSpec& s, std::vector<double>* tr, double* total,
                std::vector<double>* term_ms);  // dist.cu: one rank of a partitioned solve
void cpaa_profile(cheb_graph* g, const SolveSpec& s, std::vector<double>& term_ms);
void power_solve(cheb_graph* g, double c, int rounds, double tol, int max_rounds, int mode,
                 const double* reference, double* ranks, cheb_trace_row* trace, int cap,
                 int* rounds_out, double* total);
void transition_apply(cheb_graph* g, const double* x, double* y, int mode);
void staged_init(cheb_graph* g, double c0, int mode);
void staged_set(cheb_graph* g, const double* Tp, const double* Tc, const double* acc, int k);
void staged_generate(cheb_graph* g);
void staged_accumulate(cheb_graph* g, double ck);
void staged_rotate(cheb_graph* g);
void staged_get(cheb_graph* g, double* Tp, double* Tc, double* Tn, double* acc, int* k);
}  // namespace chebgpu
