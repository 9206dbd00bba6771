// K1 — device-resident, pattern-only CSR builder, CSR upload/download, and the
// degree-binned solver view.
//
// Replaces build_graph (/root/reference/proj/src/graph.cpp:23-102) with the same
// observable result, bit for bit: n = max(n_hint, max id + 1) (:25-29); canonical
// (min,max) pairs sorted and deduplicated (:31-43); a self-loop adds 1 to its degree
// and one adjacency entry (:45-49, :88-92); isolated vertices are an error naming the
// lowest one (:70-75) or are dropped by an order-preserving renumbering (:51-69); rows
// hold their neighbours in ascending order (:93-95).  No values array and no
// inv_degree array are stored: the D^-1 scale is an in-register IEEE reciprocal of
// the row length, bit-identical to graph.cpp:97-99.
//
// Device algorithm: 64-bit keys (lo << s | hi) -> cub radix sort -> unique ->
// degree histogram -> (monotone remap) -> both directions emitted as (row << s | col)
// with the second copy of a self-loop emitted as a sentinel -> radix sort ->
// row_ptr = exclusive scan of degrees, col = low bits.
#include <cub/cub.cuh>

#include <algorithm>
#include <atomic>
#include <chrono>
#include <map>
#include <mutex>
#include <thread>
#include <cstring>

#include "common.cuh"

namespace chebgpu {

namespace {

constexpr int kBuildThreads = 256;

inline int grid_for(int64_t n, int threads = kBuildThreads) {
    int64_t b = (n + threads - 1) / threads;
    if (b < 1) b = 1;
    if (b > 148 * 32) b = 148 * 32;
    return static_cast<int>(b);
}

template <class T>
__device__ __forceinline__ int64_t load_id(const T* e, int64_t i) {
    return static_cast<int64_t>(e[i]);
}

// Min and max endpoint id over the edge list.
template <class T>
__global__ void k_minmax(const T* __restrict__ e, int64_t cnt, long long* out_min,
                         long long* out_max) {
    long long lo = LLONG_MAX, hi = LLONG_MIN;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < cnt;
         i += (int64_t)gridDim.x * blockDim.x) {
        long long v = load_id(e, i);
        lo = v < lo ? v : lo;
        hi = v > hi ? v : hi;
    }
    for (int o = 16; o; o >>= 1) {
        long long a = __shfl_xor_sync(0xffffffffu, lo, o);
        long long b = __shfl_xor_sync(0xffffffffu, hi, o);
        lo = a < lo ? a : lo;
        hi = b > hi ? b : hi;
    }
    if ((threadIdx.x & 31) == 0) {
        atomicMin(out_min, lo);
        atomicMax(out_max, hi);
    }
}

// Canonical undirected key (min << s) | max.
template <class T>
__global__ void k_canon(const T* __restrict__ e, int64_t E, int s, uint64_t* __restrict__ keys) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < E;
         i += (int64_t)gridDim.x * blockDim.x) {
        uint64_t a = (uint64_t)load_id(e, 2 * i), b = (uint64_t)load_id(e, 2 * i + 1);
        uint64_t lo = a < b ? a : b, hi = a < b ? b : a;
        keys[i] = (lo << s) | hi;
    }
}

__global__ void k_degree(const uint64_t* __restrict__ keys, int64_t m, int s,
                         unsigned int* __restrict__ deg) {
    const uint64_t mask = (1ull << s) - 1;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < m;
         i += (int64_t)gridDim.x * blockDim.x) {
        uint64_t k = keys[i];
        uint64_t a = k >> s, b = k & mask;
        atomicAdd(&deg[a], 1u);
        if (a != b) atomicAdd(&deg[b], 1u);
    }
}

// Lowest zero-degree vertex (or n if none) + degree extrema + flags for compaction.
__global__ void k_deg_scan(const unsigned int* __restrict__ deg, int64_t n,
                           unsigned long long* first_zero, unsigned int* dmin, unsigned int* dmax) {
    unsigned long long fz = ~0ull;
    unsigned int lo = 0xffffffffu, hi = 0;
    for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < n;
         v += (int64_t)gridDim.x * blockDim.x) {
        unsigned int d = deg[v];
        if (d == 0 && (unsigned long long)v < fz) fz = (unsigned long long)v;
        if (d) {
            lo = d < lo ? d : lo;
            hi = d > hi ? d : hi;
        }
    }
    for (int o = 16; o; o >>= 1) {
        fz = min(fz, __shfl_xor_sync(0xffffffffu, fz, o));
        lo = min(lo, __shfl_xor_sync(0xffffffffu, lo, o));
        hi = max(hi, __shfl_xor_sync(0xffffffffu, hi, o));
    }
    if ((threadIdx.x & 31) == 0) {
        atomicMin(first_zero, fz);
        atomicMin(dmin, lo);
        atomicMax(dmax, hi);
    }
}

__global__ void k_nonzero_flags(const unsigned int* __restrict__ deg, int64_t n,
                                int* __restrict__ flags) {
    for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < n;
         v += (int64_t)gridDim.x * blockDim.x)
        flags[v] = deg[v] > 0 ? 1 : 0;
}

// Order-preserving renumbering (graph.cpp:52-69): a monotone map keeps the sort.
__global__ void k_remap_keys(uint64_t* __restrict__ keys, int64_t m, int s,
                             const int* __restrict__ remap) {
    const uint64_t mask = (1ull << s) - 1;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < m;
         i += (int64_t)gridDim.x * blockDim.x) {
        uint64_t k = keys[i];
        uint64_t a = (uint64_t)remap[k >> s], b = (uint64_t)remap[k & mask];
        keys[i] = (a << s) | b;
    }
}

__global__ void k_compact_deg(const unsigned int* __restrict__ deg, const int* __restrict__ remap,
                              int64_t n, unsigned int* __restrict__ out) {
    for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < n;
         v += (int64_t)gridDim.x * blockDim.x) {
        unsigned int d = deg[v];
        if (d) out[remap[v]] = d;
    }
}

// Both directions of every canonical edge; the mirror of a self-loop becomes a
// sentinel that sorts past every real key (graph.cpp:88-92 stores a loop once).
__global__ void k_directed(const uint64_t* __restrict__ keys, int64_t m, int s,
                           uint64_t* __restrict__ out) {
    const uint64_t mask = (1ull << s) - 1;
    const uint64_t sentinel = ~0ull;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < m;
         i += (int64_t)gridDim.x * blockDim.x) {
        uint64_t k = keys[i];
        uint64_t a = k >> s, b = k & mask;
        out[2 * i] = k;
        out[2 * i + 1] = (a == b) ? sentinel : ((b << s) | a);
    }
}

__global__ void k_low_bits(const uint64_t* __restrict__ keys, int64_t nnz, int s,
                           int* __restrict__ col) {
    const uint64_t mask = (1ull << s) - 1;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nnz;
         i += (int64_t)gridDim.x * blockDim.x)
        col[i] = (int)(keys[i] & mask);
}

__global__ void k_widen_deg(const unsigned int* __restrict__ in, int64_t cnt, int64_t* __restrict__ out) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < cnt;
         i += (int64_t)gridDim.x * blockDim.x)
        out[i] = (int64_t)in[i];
}

template <class RP>
__global__ void k_narrow_rowptr(const int64_t* __restrict__ in, int64_t cnt, RP* __restrict__ out) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < cnt;
         i += (int64_t)gridDim.x * blockDim.x)
        out[i] = (RP)in[i];
}

template <class RP>
__global__ void k_widen_rowptr(const RP* __restrict__ in, int64_t cnt, int64_t* __restrict__ out) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < cnt;
         i += (int64_t)gridDim.x * blockDim.x)
        out[i] = (int64_t)in[i];
}

template <class RP>
__global__ void k_row_degrees(const RP* __restrict__ rp, int64_t n, int64_t* __restrict__ out) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x)
        out[i] = (int64_t)(rp[i + 1] - rp[i]);
}

__global__ void k_widen_col(const int* __restrict__ in, int64_t cnt, int64_t* __restrict__ out) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < cnt;
         i += (int64_t)gridDim.x * blockDim.x)
        out[i] = (int64_t)in[i];
}

// Upload path: int64 neighbours -> int32, flag out-of-range ids.
__global__ void k_narrow_col(const int64_t* __restrict__ in, int64_t cnt, int64_t n, int64_t base,
                             int* __restrict__ out, unsigned long long* bad) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < cnt;
         i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t v = in[i];
        const bool ok = v >= 0 && v < n;
        if (!ok) atomicMin(bad, (unsigned long long)(base + i));
        out[i] = ok ? (int)v : 0;  // never an out-of-range id on the device
    }
}

int bits_for(int64_t n) {  // smallest s with n <= 2^s - 1 (so a row field is never all-ones)
    int s = 1;
    while ((int64_t(1) << s) <= n) ++s;
    return s;
}

struct TempStore {
    DevMem mem;
    void* get(size_t bytes) {
        mem.ensure(bytes);
        return mem.get();
    }
};

void sort_keys(uint64_t*& keys, uint64_t*& alt, int64_t cnt, int end_bit, cudaStream_t st,
               TempStore& tmp) {
    cub::DoubleBuffer<uint64_t> db(keys, alt);
    size_t bytes = 0;
    CHEB_CUDA_CHECK(cub::DeviceRadixSort::SortKeys(nullptr, bytes, db, cnt, 0, end_bit, st));
    void* t = tmp.get(bytes);
    CHEB_CUDA_CHECK(cub::DeviceRadixSort::SortKeys(t, bytes, db, cnt, 0, end_bit, st));
    keys = db.Current();
    alt = db.Alternate();
}

template <class T>
T read_scalar(const T* d, cudaStream_t st) {
    T h;
    CHEB_CUDA_CHECK(cudaMemcpyAsync(&h, d, sizeof(T), cudaMemcpyDeviceToHost, st));
    CHEB_CUDA_CHECK(cudaStreamSynchronize(st));
    return h;
}

}  // namespace

namespace {
struct WindowArenaCache {
    std::mutex mu;
    std::map<int, std::vector<DevMem>> blocks;  // per device, free
};
WindowArenaCache& window_arena_cache() {
    static WindowArenaCache* c = new WindowArenaCache;  // never destroyed (no cudaFree at process exit)
    return *c;
}
constexpr size_t kWindowArenaKeep = 6;  // free blocks kept per device
}  // namespace

void window_arena_take(DevMem& out, size_t bytes) {
    int dev = 0;
    CHEB_CUDA_CHECK(cudaGetDevice(&dev));
    WindowArenaCache& c = window_arena_cache();
    {
        std::lock_guard<std::mutex> lk(c.mu);
        auto& v = c.blocks[dev];
        int best = -1;
        for (int i = 0; i < (int)v.size(); ++i)  // smallest block that fits without wasting more than half
            if (v[i].bytes() >= bytes && v[i].bytes() <= 2 * bytes + (size_t(1) << 20) &&
                (best < 0 || v[i].bytes() < v[best].bytes()))
                best = i;
        if (alloc_debug()) std::fprintf(stderr, "[arena] take %.1f MB: %zu cached, fit %d\n", bytes / 1e6, v.size(), best);
        if (best >= 0) {
            out = std::move(v[best]);
            v.erase(v.begin() + best);
            return;
        }
    }
    AllocScope plain(nullptr);
    out.alloc(bytes + bytes / 16);
}

void window_arena_give(DevMem& blk) {
    if (!blk.get() || blk.bytes() == 0) return;
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) return;
    cudaDeviceSynchronize();  // nothing in flight may still read the block
    WindowArenaCache& c = window_arena_cache();
    std::lock_guard<std::mutex> lk(c.mu);
    auto& v = c.blocks[dev];
    if (alloc_debug()) std::fprintf(stderr, "[arena] give %.1f MB (%zu cached)\n", blk.bytes() / 1e6, v.size());
    v.push_back(std::move(blk));
    if (v.size() > kWindowArenaKeep) {  // drop the smallest
        size_t small = 0;
        for (size_t i = 1; i < v.size(); ++i)
            if (v[i].bytes() < v[small].bytes()) small = i;
        v.erase(v.begin() + (long)small);
    }
}

void build_from_edges(cheb_graph* g, const void* d_edges, int64_t E, int edge_bits,
                      const cheb_build_opts& o) {
    cudaStream_t st = g->stream;
    TempStore tmp;
    const int64_t nid = 2 * E;

    // n and id checks (graph.cpp:25-29)
    int64_t n = std::max<int64_t>(o.n_hint, 0);
    if (E > 0) {
        DevMem mm(2 * sizeof(long long));
        long long init[2] = {LLONG_MAX, LLONG_MIN};
        CHEB_CUDA_CHECK(cudaMemcpyAsync(mm.get(), init, sizeof init, cudaMemcpyHostToDevice, st));
        if (edge_bits == 64)
            k_minmax<<<grid_for(nid), kBuildThreads, 0, st>>>(
                static_cast<const int64_t*>(d_edges), nid, mm.ptr<long long>(), mm.ptr<long long>() + 1);
        else
            k_minmax<<<grid_for(nid), kBuildThreads, 0, st>>>(
                static_cast<const int32_t*>(d_edges), nid, mm.ptr<long long>(), mm.ptr<long long>() + 1);
        CHEB_CUDA_CHECK(cudaGetLastError());
        long long h[2];
        CHEB_CUDA_CHECK(cudaMemcpyAsync(h, mm.get(), sizeof h, cudaMemcpyDeviceToHost, st));
        CHEB_CUDA_CHECK(cudaStreamSynchronize(st));
        if (h[0] < 0) fail(CHEB_VALIDATION, "negative vertex id in edge list");
        if (h[1] >= INT32_MAX - 1)  // before max id + 1 can overflow (graph.cpp:25-29)
            fail(CHEB_CAPACITY, "device CSR builder supports n < 2^31 (int32 column ids), got max id " +
                                    std::to_string(h[1]));
        n = std::max<int64_t>(n, h[1] + 1);
    }
    if (n > INT32_MAX - 1)
        fail(CHEB_CAPACITY, "device CSR builder supports n < 2^31 (int32 column ids), got n=" +
                                std::to_string(n));
    const int s = bits_for(n);

    // canonical keys, sort, dedup (graph.cpp:31-43)
    DevMem kbuf(sizeof(uint64_t) * std::max<int64_t>(E, 1));
    DevMem kalt(sizeof(uint64_t) * std::max<int64_t>(E, 1));
    uint64_t* keys = kbuf.ptr<uint64_t>();
    uint64_t* alt = kalt.ptr<uint64_t>();
    if (E > 0) {
        if (edge_bits == 64)
            k_canon<<<grid_for(E), kBuildThreads, 0, st>>>(static_cast<const int64_t*>(d_edges), E, s, keys);
        else
            k_canon<<<grid_for(E), kBuildThreads, 0, st>>>(static_cast<const int32_t*>(d_edges), E, s, keys);
        CHEB_CUDA_CHECK(cudaGetLastError());
        sort_keys(keys, alt, E, 2 * s, st, tmp);
    }
    int64_t m = E;
    if (o.dedup && E > 0) {
        DevMem cnt(sizeof(int64_t));
        size_t bytes = 0;
        CHEB_CUDA_CHECK(cub::DeviceSelect::Unique(nullptr, bytes, keys, alt, cnt.ptr<int64_t>(), E, st));
        void* t = tmp.get(bytes);
        CHEB_CUDA_CHECK(cub::DeviceSelect::Unique(t, bytes, keys, alt, cnt.ptr<int64_t>(), E, st));
        m = read_scalar(cnt.ptr<int64_t>(), st);
        std::swap(keys, alt);
    }
    g->duplicates_removed = E - m;

    // degrees, self-loop once (graph.cpp:45-49)
    DevMem deg(sizeof(unsigned int) * (n + 1));
    CHEB_CUDA_CHECK(cudaMemsetAsync(deg.get(), 0, sizeof(unsigned int) * (n + 1), st));
    if (m > 0) {
        k_degree<<<grid_for(m), kBuildThreads, 0, st>>>(keys, m, s, deg.ptr<unsigned int>());
        CHEB_CUDA_CHECK(cudaGetLastError());
    }
    DevMem scan(sizeof(unsigned long long) + 2 * sizeof(unsigned int));
    auto deg_stats = [&](const unsigned int* d, int64_t nn, unsigned long long* fz,
                         unsigned int* lo, unsigned int* hi) {
        unsigned char init[sizeof(unsigned long long) + 2 * sizeof(unsigned int)];
        unsigned long long a = ~0ull;
        unsigned int b = 0xffffffffu, c = 0;
        std::memcpy(init, &a, 8);
        std::memcpy(init + 8, &b, 4);
        std::memcpy(init + 12, &c, 4);
        CHEB_CUDA_CHECK(cudaMemcpyAsync(scan.get(), init, sizeof init, cudaMemcpyHostToDevice, st));
        if (nn > 0) {
            k_deg_scan<<<grid_for(nn), kBuildThreads, 0, st>>>(
                d, nn, scan.ptr<unsigned long long>(),
                reinterpret_cast<unsigned int*>(scan.ptr<char>() + 8),
                reinterpret_cast<unsigned int*>(scan.ptr<char>() + 12));
            CHEB_CUDA_CHECK(cudaGetLastError());
        }
        unsigned char out[16];
        CHEB_CUDA_CHECK(cudaMemcpyAsync(out, scan.get(), 16, cudaMemcpyDeviceToHost, st));
        CHEB_CUDA_CHECK(cudaStreamSynchronize(st));
        std::memcpy(fz, out, 8);
        std::memcpy(lo, out + 8, 4);
        std::memcpy(hi, out + 12, 4);
    };
    unsigned long long first_zero;
    unsigned int dmin, dmax;
    deg_stats(deg.ptr<unsigned int>(), n, &first_zero, &dmin, &dmax);

    g->isolated_dropped = 0;
    const bool any_isolated = n > 0 && first_zero != ~0ull;
    if (any_isolated && !o.drop_isolated)  // graph.cpp:70-75
        fail(CHEB_VALIDATION, "vertex " + std::to_string(first_zero) + " is isolated (degree 0)");
    if (any_isolated) {  // graph.cpp:51-69
        DevMem flags(sizeof(int) * n), remap(sizeof(int) * n);
        k_nonzero_flags<<<grid_for(n), kBuildThreads, 0, st>>>(deg.ptr<unsigned int>(), n, flags.ptr<int>());
        CHEB_CUDA_CHECK(cudaGetLastError());
        size_t bytes = 0;
        CHEB_CUDA_CHECK(cub::DeviceScan::ExclusiveSum(nullptr, bytes, flags.ptr<int>(), remap.ptr<int>(), n, st));
        void* t = tmp.get(bytes);
        CHEB_CUDA_CHECK(cub::DeviceScan::ExclusiveSum(t, bytes, flags.ptr<int>(), remap.ptr<int>(), n, st));
        int last_remap = read_scalar(remap.ptr<int>() + (n - 1), st);
        unsigned int last_deg = read_scalar(deg.ptr<unsigned int>() + (n - 1), st);
        const int64_t kept = (int64_t)last_remap + (last_deg > 0 ? 1 : 0);
        g->isolated_dropped = n - kept;
        if (m > 0) {
            k_remap_keys<<<grid_for(m), kBuildThreads, 0, st>>>(keys, m, s, remap.ptr<int>());
            CHEB_CUDA_CHECK(cudaGetLastError());
        }
        DevMem deg2(sizeof(unsigned int) * (kept + 1));
        CHEB_CUDA_CHECK(cudaMemsetAsync(deg2.get(), 0, sizeof(unsigned int) * (kept + 1), st));
        k_compact_deg<<<grid_for(n), kBuildThreads, 0, st>>>(deg.ptr<unsigned int>(), remap.ptr<int>(), n,
                                                             deg2.ptr<unsigned int>());
        CHEB_CUDA_CHECK(cudaGetLastError());
        deg = std::move(deg2);
        n = kept;
        deg_stats(deg.ptr<unsigned int>(), n, &first_zero, &dmin, &dmax);
    }

    // directed entries, sorted by (row, col): CSR with ascending rows (graph.cpp:77-95)
    const int64_t two_m = 2 * m;
    DevMem dir(sizeof(uint64_t) * std::max<int64_t>(two_m, 1));
    DevMem dalt(sizeof(uint64_t) * std::max<int64_t>(two_m, 1));
    uint64_t* dk = dir.ptr<uint64_t>();
    uint64_t* da = dalt.ptr<uint64_t>();
    if (m > 0) {
        k_directed<<<grid_for(m), kBuildThreads, 0, st>>>(keys, m, s, dk);
        CHEB_CUDA_CHECK(cudaGetLastError());
        CHEB_CUDA_CHECK(cudaStreamSynchronize(st));
    }
    kbuf.release();  // canonical keys are dead once the directed entries exist
    kalt.release();
    if (two_m > 0) sort_keys(dk, da, two_m, 2 * s, st, tmp);

    // row_ptr = exclusive scan of degrees (widened to int64; deg[n] == 0 so rp[n] = nnz)
    DevMem rp64((n + 1) * sizeof(int64_t));
    {
        DevMem deg64(sizeof(int64_t) * (n + 1));
        CHEB_CUDA_CHECK(cudaMemsetAsync(deg.ptr<unsigned int>() + n, 0, sizeof(unsigned int), st));
        k_widen_deg<<<grid_for(n + 1), kBuildThreads, 0, st>>>(deg.ptr<unsigned int>(), n + 1,
                                                               deg64.ptr<int64_t>());
        CHEB_CUDA_CHECK(cudaGetLastError());
        size_t bytes = 0;
        CHEB_CUDA_CHECK(cub::DeviceScan::ExclusiveSum(nullptr, bytes, deg64.ptr<int64_t>(), rp64.ptr<int64_t>(), n + 1, st));
        void* t = tmp.get(bytes);
        CHEB_CUDA_CHECK(cub::DeviceScan::ExclusiveSum(t, bytes, deg64.ptr<int64_t>(), rp64.ptr<int64_t>(), n + 1, st));
    }
    const int64_t nnz = n > 0 ? read_scalar(rp64.ptr<int64_t>() + n, st) : 0;

    g->n = n;
    g->m = m;
    g->nnz = nnz;
    g->multi = !o.dedup;
    g->max_degree = n > 0 ? dmax : 0;
    g->min_degree = n > 0 ? dmin : 0;
    g->rp64 = o.row_ptr_64 != 0 || nnz > INT32_MAX;
    g->col.alloc(sizeof(int) * std::max<int64_t>(nnz, 1));
    if (nnz > 0) {
        k_low_bits<<<grid_for(nnz), kBuildThreads, 0, st>>>(dk, nnz, s, g->col.ptr<int>());
        CHEB_CUDA_CHECK(cudaGetLastError());
    }
    if (g->rp64) {
        g->row_ptr = std::move(rp64);
    } else {
        g->row_ptr.alloc(sizeof(int) * (n + 1));
        k_narrow_rowptr<<<grid_for(n + 1), kBuildThreads, 0, st>>>(rp64.ptr<int64_t>(), n + 1,
                                                                   g->row_ptr.ptr<int>());
        CHEB_CUDA_CHECK(cudaGetLastError());
    }
    g->inv_array = false;
    g->view.ready = false;
    CHEB_CUDA_CHECK(cudaStreamSynchronize(st));
}

// Pageable neighbour arrays (a C++ caller's std::vector): the driver would stage them
// synchronously at ~11 GB/s.  Instead host threads narrow int64 -> int32 (with the range
// check) straight into a pinned ring and DMA each chunk as it is ready: half the bytes cross
// PCIe, the copies overlap, and no device narrowing pass is needed.
struct HostNarrowRing {
    static constexpr int kMaxThreads = 8;
    static constexpr int64_t kChunk = int64_t(1) << 21;  // int32 entries per buffer (8 MB)
    std::mutex mu;
    int* buf[2 * kMaxThreads] = {};
    cudaEvent_t done[2 * kMaxThreads] = {};
};
static HostNarrowRing& host_narrow_ring() {
    static HostNarrowRing* r = new HostNarrowRing();  // never destroyed: outlives every handle
    return *r;
}

struct HostNarrow {
    std::vector<std::thread> workers;
    std::atomic<int64_t> next{0};
    std::atomic<bool> stop{false};
    std::vector<int64_t> first_bad;  // per worker
    std::vector<std::string> errors;
    std::unique_lock<std::mutex> lock;

    void start(const int64_t* src, int64_t nnz, int64_t n, int* dst, cudaStream_t st, int device) {
        HostNarrowRing& R = host_narrow_ring();
        lock = std::unique_lock<std::mutex>(R.mu);
        const int64_t chunks = (nnz + HostNarrowRing::kChunk - 1) / HostNarrowRing::kChunk;
        const int hw = (int)std::max(1u, std::thread::hardware_concurrency());
        const int T = (int)std::max<int64_t>(1, std::min<int64_t>({(int64_t)HostNarrowRing::kMaxThreads, (int64_t)hw, chunks}));
        for (int b = 0; b < 2 * T; ++b) {
            if (!R.buf[b])
                CHEB_CUDA_CHECK(cudaHostAlloc(reinterpret_cast<void**>(&R.buf[b]), sizeof(int) * HostNarrowRing::kChunk,
                                              cudaHostAllocPortable));
            if (!R.done[b]) CHEB_CUDA_CHECK(cudaEventCreateWithFlags(&R.done[b], cudaEventDisableTiming));
        }
        first_bad.assign(T, -1);
        errors.assign(T, std::string());
        for (int w = 0; w < T; ++w)
            workers.emplace_back([this, w, chunks, src, nnz, n, dst, st, device, &R] {
                try {
                    CHEB_CUDA_CHECK(cudaSetDevice(device));
                    int parity = 0;
                    for (;;) {
                        const int64_t c = next.fetch_add(1);
                        if (c >= chunks || stop.load()) break;
                        const int b = 2 * w + parity;
                        parity ^= 1;
                        CHEB_CUDA_CHECK(cudaEventSynchronize(R.done[b]));  // its previous DMA is done
                        const int64_t off = c * HostNarrowRing::kChunk;
                        const int64_t len = std::min(HostNarrowRing::kChunk, nnz - off);
                        int* out = R.buf[b];
                        for (int64_t i = 0; i < len; ++i) {
                            const int64_t v = src[off + i];
                            const bool ok = v >= 0 && v < n;
                            if (!ok && first_bad[w] < 0) first_bad[w] = off + i;
                            out[i] = ok ? (int)v : 0;
                        }
                        CHEB_CUDA_CHECK(cudaMemcpyAsync(dst + off, out, sizeof(int) * len, cudaMemcpyHostToDevice, st));
                        CHEB_CUDA_CHECK(cudaEventRecord(R.done[b], st));
                    }
                } catch (const std::exception& e) {
                    errors[w] = e.what();
                    stop.store(true);
                }
            });
    }
    // first out-of-range entry over all workers (-1: none); rethrows a worker's CUDA error
    int64_t join() {
        for (auto& t : workers) t.join();
        workers.clear();
        for (auto& e : errors)
            if (!e.empty()) fail(CHEB_CUDA, e);
        int64_t bad = -1;
        for (int64_t b : first_bad)
            if (b >= 0 && (bad < 0 || b < bad)) bad = b;
        return bad;
    }
    ~HostNarrow() {
        stop.store(true);
        for (auto& t : workers) t.join();
    }
};

// Neighbour data of an upload landing on the device in groups of old rows: group i holds old
// rows [row_cut[i], row_cut[i + 1]) and is narrowed once ready[i] (upload stream) fires.  The
// view permutes (and sorts) each group as it lands, overlapping the rest of the copy.
struct ColGroups {
    std::vector<int64_t> row_cut;
    std::vector<cudaEvent_t> ready;
    ~ColGroups() {
        for (cudaEvent_t e : ready)
            if (e) cudaEventDestroy(e);
    }
};

template <class RPO, class RPN>
static void build_view_t(cheb_graph* g, cudaStream_t st, const std::function<void()>& before_col,
                         const ColGroups* groups = nullptr);

static bool dbg_on() {
    static const bool on = getenv("CHEB_DEBUG_UPLOAD") != nullptr;
    return on;
}
static std::chrono::steady_clock::time_point& dbg_t0() {
    static std::chrono::steady_clock::time_point t;
    return t;
}
static void dbg_mark(const char* what) {
    if (!dbg_on()) return;
    const auto t = std::chrono::steady_clock::now();
    fprintf(stderr, "[upload] %-24s %8.3f ms\n", what, std::chrono::duration<double, std::milli>(t - dbg_t0()).count());
}

void upload_csr(cheb_graph* g, const int64_t* offsets, const int64_t* neighbors, int64_t n,
                int64_t nnz, const double* inv_degree, const std::function<bool()>& host_checks) {
    cudaStream_t st = g->stream;
    const bool dbg = dbg_on();
    dbg_t0() = std::chrono::steady_clock::now();
    auto mark = dbg_mark;
    g->n = n;
    g->nnz = nnz;
    g->rp64 = g->rp64 || nnz > INT32_MAX;
    if (n > INT32_MAX - 1) fail(CHEB_CAPACITY, "device path supports n < 2^31");

    // 1. offsets: host int64 -> device (int32 narrowed when possible)
    DevMem rp64(sizeof(int64_t) * (n + 1));
    CHEB_CUDA_CHECK(cudaMemcpyAsync(rp64.get(), offsets, sizeof(int64_t) * (n + 1),
                                    cudaMemcpyHostToDevice, st));
    if (!g->rp64) {
        g->row_ptr.alloc(sizeof(int) * (n + 1));
        k_narrow_rowptr<<<grid_for(n + 1), kBuildThreads, 0, st>>>(rp64.ptr<int64_t>(), n + 1,
                                                                   g->row_ptr.ptr<int>());
        CHEB_CUDA_CHECK(cudaGetLastError());
    }
    // 2. first out-of-range neighbour entry (device verdict)
    DevMem flags(sizeof(unsigned long long));
    auto* bad = flags.ptr<unsigned long long>();
    CHEB_CUDA_CHECK(cudaMemsetAsync(bad, 0xff, sizeof(unsigned long long), st));
    g->inv_array = false;
    cudaEvent_t ev_rp = nullptr, ev_col = nullptr, ev_view = nullptr;
    struct Events {
        cudaEvent_t* e[3];
        ~Events() {
            for (auto* p : e)
                if (*p) cudaEventDestroy(*p);
        }
    } evs{{&ev_rp, &ev_col, &ev_view}};
    for (auto* p : evs.e) CHEB_CUDA_CHECK(cudaEventCreateWithFlags(p, cudaEventDisableTiming));
    CHEB_CUDA_CHECK(cudaEventRecord(ev_rp, st));

    // 3. neighbours: int64 -> int32, range-checked.  Chunked to bound the staging buffer.
    g->col.alloc(sizeof(int) * std::max<int64_t>(nnz, 1));
    bool pageable = false;
    if (nnz >= (int64_t(1) << 22)) {
        cudaPointerAttributes pa;
        if (cudaPointerGetAttributes(&pa, neighbors) != cudaSuccess) {
            cudaGetLastError();
            pageable = true;
        } else {
            pageable = pa.type == cudaMemoryTypeUnregistered;
        }
    }
    HostNarrow hn;
    struct CopyStream {  // the H2D copy stream, back to the pool once idle
        cudaStream_t s = nullptr;
        int device = 0;
        ~CopyStream() {
            if (s) {
                cudaStreamSynchronize(s);
                release_stream(device, s);
            }
        }
    } copy_stream;
    // Large pinned uploads land in groups of old rows (~nnz / 4 entries each), so that the view
    // permutes and sorts each group while the next one is still being copied.
    ColGroups groups;
    const bool view_here = g->part.G == 1 && !g->part.comm && !g->peer && n > 0;
    if (view_here && !pageable && nnz >= (int64_t(1) << 26)) {
        const int K = std::max(1, std::min(tuning().upgroups, 64));
        groups.row_cut.assign(K + 1, n);
        groups.row_cut[0] = 0;
        for (int i = 1; i < K; ++i)
            groups.row_cut[i] = std::lower_bound(offsets, offsets + n + 1, nnz * i / K) - offsets;
        for (int i = 1; i <= K; ++i) groups.row_cut[i] = std::max(groups.row_cut[i], groups.row_cut[i - 1]);
        groups.ready.assign(K, nullptr);
        for (auto& e : groups.ready) CHEB_CUDA_CHECK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    }
    if (pageable) {
        hn.start(neighbors, nnz, n, g->col.ptr<int>(), st, g->device);
    } else if (nnz > 0) {
        // The copy engine streams the int64 chunks back to back on its own stream into a ring
        // of staging buffers; each chunk is narrowed on `st` once it has landed, and a slot is
        // refilled once its narrowing is done.  (On one stream every copy would wait for the
        // previous chunk's narrowing, which queues behind the view build's kernels.)
        const int64_t chunk = std::min<int64_t>(nnz, int64_t(1) << 25);
        const int64_t nchunks = (nnz + chunk - 1) / chunk;
        const int ring = (int)std::min<int64_t>(nchunks, 4);
        copy_stream.s = pooled_stream(g->device);
        copy_stream.device = g->device;
        cudaStream_t cs = copy_stream.s;
        CHEB_CUDA_CHECK(cudaStreamWaitEvent(cs, ev_rp, 0));  // after the offsets (and flag reset)
        std::vector<DevMem> stage((size_t)ring);
        std::vector<cudaEvent_t> copied((size_t)ring, nullptr), narrowed((size_t)ring, nullptr);
        for (int r = 0; r < ring; ++r) {
            stage[(size_t)r].alloc(sizeof(int64_t) * chunk);
            CHEB_CUDA_CHECK(cudaEventCreateWithFlags(&copied[(size_t)r], cudaEventDisableTiming));
            CHEB_CUDA_CHECK(cudaEventCreateWithFlags(&narrowed[(size_t)r], cudaEventDisableTiming));
        }
        CHEB_CUDA_CHECK(cudaEventRecord(ev_col, st));  // staging allocated (stream-ordered on st)
        CHEB_CUDA_CHECK(cudaStreamWaitEvent(cs, ev_col, 0));
        size_t next_group = 0;
        for (int64_t i = 0; i < nchunks; ++i) {
            const int64_t off = i * chunk, c = std::min(chunk, nnz - off);
            const size_t r = (size_t)(i % ring);
            if (i >= ring) CHEB_CUDA_CHECK(cudaStreamWaitEvent(cs, narrowed[r], 0));
            CHEB_CUDA_CHECK(cudaMemcpyAsync(stage[r].get(), neighbors + off, sizeof(int64_t) * c,
                                            cudaMemcpyHostToDevice, cs));
            CHEB_CUDA_CHECK(cudaEventRecord(copied[r], cs));
            CHEB_CUDA_CHECK(cudaStreamWaitEvent(st, copied[r], 0));
            k_narrow_col<<<grid_for(c), kBuildThreads, 0, st>>>(stage[r].ptr<int64_t>(), c, n, off,
                                                                 g->col.ptr<int>() + off, bad);
            CHEB_CUDA_CHECK(cudaGetLastError());
            CHEB_CUDA_CHECK(cudaEventRecord(narrowed[r], st));
            while (next_group < groups.ready.size() && offsets[groups.row_cut[next_group + 1]] <= off + c)
                CHEB_CUDA_CHECK(cudaEventRecord(groups.ready[next_group++], st));
        }
        while (next_group < groups.ready.size()) CHEB_CUDA_CHECK(cudaEventRecord(groups.ready[next_group++], st));
        for (int r = 0; r < ring; ++r) {  // st has waited on every copy: the staging frees on st are safe
            cudaEventDestroy(copied[(size_t)r]);
            cudaEventDestroy(narrowed[(size_t)r]);
        }
    } else {
        for (auto& e : groups.ready) CHEB_CUDA_CHECK(cudaEventRecord(e, st));
    }
    if (!pageable) CHEB_CUDA_CHECK(cudaEventRecord(ev_col, st));
    mark("enqueued copies");

    // 4. the reference's host-side checks, while the copies are in flight; they also tell
    //    whether inv_degree is canonical (graph.cpp:97-99) — only a non-canonical one is
    //    uploaded (the reference's poisoned-array semantics, cpaa.cpp:107)
    const bool inv_canonical = host_checks ? host_checks() : inv_degree == nullptr;
    mark("host checks");
    int64_t host_bad = -1;
    bool joined = !pageable;
    auto finish_narrowing = [&] {  // every chunk enqueued: the column permute may wait on them
        if (joined) return;
        host_bad = hn.join();
        CHEB_CUDA_CHECK(cudaEventRecord(ev_col, st));
        joined = true;
        mark("host narrowing");
    };

    if (g->rp64) g->row_ptr = std::move(rp64);  // the view reads the canonical row_ptr

    // 5. solver view (single-GPU layout) on the auxiliary stream: the degree-only half
    //    overlaps the neighbour copy; the column permute waits for it.
    if (g->part.G == 1 && !g->part.comm && !g->peer && n > 0) {
        if (!g->aux) g->aux = pooled_stream(g->device);
        CHEB_CUDA_CHECK(cudaStreamWaitEvent(g->aux, ev_rp, 0));
        {
            AllocScope as(g->aux);
            g->view = SolverView{};
            const bool grouped = !groups.ready.empty();
            auto wait_col = [&] {  // the degree-only half of the view overlapped the narrowing
                finish_narrowing();
                if (!grouped) CHEB_CUDA_CHECK(cudaStreamWaitEvent(g->aux, ev_col, 0));  // else per group
            };
            if (g->rp64)
                build_view_t<int64_t, int64_t>(g, g->aux, wait_col, grouped ? &groups : nullptr);
            else
                build_view_t<int, int>(g, g->aux, wait_col, grouped ? &groups : nullptr);
        }
        mark("view enqueued");
        if (dbg) { cudaEventSynchronize(ev_col); mark("neighbours landed"); cudaStreamSynchronize(g->aux); mark("view done"); }
        CHEB_CUDA_CHECK(cudaEventRecord(ev_view, g->aux));
        CHEB_CUDA_CHECK(cudaStreamWaitEvent(st, ev_view, 0));
        g->view.set_stream(st);
    }
    finish_narrowing();
    rp64.release();  // (int32 graphs) stream-ordered after the narrowing and the inv check

    // 6. device-side verdict; a non-canonical inv_degree goes up now (the view, built
    //    without it, is rebuilt with it on first use)
    if (inv_degree && !inv_canonical) {
        g->inv.alloc(sizeof(double) * n);
        CHEB_CUDA_CHECK(cudaMemcpyAsync(g->inv.get(), inv_degree, sizeof(double) * n,
                                        cudaMemcpyHostToDevice, st));
    }
    unsigned long long b;
    CHEB_CUDA_CHECK(cudaMemcpyAsync(&b, flags.get(), sizeof b, cudaMemcpyDeviceToHost, st));
    CHEB_CUDA_CHECK(cudaStreamSynchronize(st));
    mark("synced");
    if (host_bad >= 0 && (b == ~0ull || (unsigned long long)host_bad < b)) b = (unsigned long long)host_bad;
    if (b != ~0ull) fail(CHEB_VALIDATION, "neighbor id out of range at entry " + std::to_string(b));
    g->inv_array = inv_degree && !inv_canonical;
    if (g->inv_array && g->view.ready) {  // the view gathers inv in its row order
        g->view.ready = false;
    }
    if (!g->inv_array) g->inv.release();
}

void download_csr(cheb_graph* g, int64_t* offsets, int64_t* neighbors, int64_t* degrees) {
    cudaStream_t st = g->stream;
    const int64_t n = g->n, nnz = g->nnz;
    if (offsets || degrees) {
        DevMem w(sizeof(int64_t) * (n + 1));
        if (offsets) {
            if (g->rp64)
                CHEB_CUDA_CHECK(cudaMemcpyAsync(offsets, g->row_ptr.get(), sizeof(int64_t) * (n + 1),
                                                cudaMemcpyDeviceToHost, st));
            else {
                k_widen_rowptr<<<grid_for(n + 1), kBuildThreads, 0, st>>>(g->row_ptr.ptr<int>(), n + 1,
                                                                          w.ptr<int64_t>());
                CHEB_CUDA_CHECK(cudaMemcpyAsync(offsets, w.get(), sizeof(int64_t) * (n + 1),
                                                cudaMemcpyDeviceToHost, st));
            }
            CHEB_CUDA_CHECK(cudaStreamSynchronize(st));
        }
        if (degrees && n > 0) {
            if (g->rp64)
                k_row_degrees<<<grid_for(n), kBuildThreads, 0, st>>>(g->row_ptr.ptr<int64_t>(), n, w.ptr<int64_t>());
            else
                k_row_degrees<<<grid_for(n), kBuildThreads, 0, st>>>(g->row_ptr.ptr<int>(), n, w.ptr<int64_t>());
            CHEB_CUDA_CHECK(cudaMemcpyAsync(degrees, w.get(), sizeof(int64_t) * n,
                                            cudaMemcpyDeviceToHost, st));
            CHEB_CUDA_CHECK(cudaStreamSynchronize(st));
        }
    }
    if (neighbors && nnz > 0) {
        const int64_t chunk = std::min<int64_t>(nnz, int64_t(1) << 26);
        DevMem w(sizeof(int64_t) * chunk);
        for (int64_t off = 0; off < nnz; off += chunk) {
            const int64_t c = std::min(chunk, nnz - off);
            k_widen_col<<<grid_for(c), kBuildThreads, 0, st>>>(g->col.ptr<int>() + off, c, w.ptr<int64_t>());
            CHEB_CUDA_CHECK(cudaMemcpyAsync(neighbors + off, w.get(), sizeof(int64_t) * c,
                                            cudaMemcpyDeviceToHost, st));
            CHEB_CUDA_CHECK(cudaStreamSynchronize(st));
        }
    }
}

// ---------------------------------------------------------------------------
// Solver view: degree-descending relabel + bins (see common.cuh).
// ---------------------------------------------------------------------------
namespace {

template <class RP>
__global__ void k_degree_keys(const RP* __restrict__ rp, int64_t n, unsigned int* __restrict__ key,
                              int* __restrict__ ids) {
    for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < n;
         v += (int64_t)gridDim.x * blockDim.x) {
        key[v] = ~(unsigned int)(rp[v + 1] - rp[v]);  // ascending sort of ~deg = descending deg
        ids[v] = (int)v;
    }
}

__global__ void k_scatter_rank(const int* __restrict__ order, int64_t n, int* __restrict__ rank) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x)
        rank[order[i]] = (int)i;
}

template <class RP>
__global__ void k_new_degrees(const RP* __restrict__ rp, const int* __restrict__ order, int64_t n,
                              int64_t* __restrict__ out) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        const int o = order[i];
        out[i] = (int64_t)(rp[o + 1] - rp[o]);
    }
}

// Copy the old neighbours of new rows [w0, w1) in storage order, renamed.  S lanes per row
// (S = 32: warp per row; S = 4 for the short rows, so that the ~1 M short rows of config 2
// are not each a warp waiting on four dependent loads); S = 0: a whole CTA per row (hubs).
template <int S, class RPO, class RPN>
__global__ void k_permute_rows(const RPO* __restrict__ rp_old, const int* __restrict__ col_old,
                               const RPN* __restrict__ rp_new, const int* __restrict__ order,
                               const int* __restrict__ rank, int64_t w0, int64_t w1, int* __restrict__ col_new,
                               int64_t oa, int64_t ob) {
    constexpr int kPer = S == 0 ? 1 : (int)(kBuildThreads / (S == 0 ? 1 : S));  // rows per CTA
    const int lane = S == 0 ? (int)threadIdx.x : (int)(threadIdx.x % (S == 0 ? 1 : S));
    const int stride = S == 0 ? (int)blockDim.x : S;
    for (int64_t w = w0 + (int64_t)blockIdx.x * kPer + (S == 0 ? 0 : threadIdx.x / (S == 0 ? 1 : S)); w < w1;
         w += (int64_t)gridDim.x * kPer) {
        const int o = order[w];
        if (o < oa || o >= ob) continue;  // another group of old rows
        const int64_t b = rp_old[o], e = rp_old[o + 1], d = rp_new[w];
        for (int64_t j = b + lane; j < e; j += stride) col_new[d + (j - b)] = rank[col_old[j]];
    }
}

// Bank-aware order of hub-row chunks (FAST schedule only).  A chunk tile is read as lane l
// of instruction q -> chunk position l + 32 q, so positions [16 w, 16 w + 16) are one
// half-warp: one conflict group of an fp64 shared-memory gather.  Each chunk is ordered so
// that every such window holds hot-prefix entries (ids < H) with distinct bank pairs
// (id mod 16): the k-th entry of bank pair r goes to window k, the hot entries of a window
// in bank-pair order, cold entries filling the remaining slots in their original order.
// A chunk where some bank pair has more entries than there are windows keeps its order.
// The entry set is unchanged (its partial sum is re-associated, deterministically).
// val[q] = entry at position lane + 32 q (cnt <= 256); returns dst[q] (or -1: no entry).
struct SchedScratch {
    int cnt[17], msk[16], f[16];
};
__device__ __forceinline__ void schedule_chunk(const int (&val)[8], int cnt, int H, SchedScratch& sc,
                                               int (&dst)[8]) {
    const int lane = threadIdx.x & 31;
    const unsigned lt = (1u << lane) - 1u;
    const int W = (cnt + 15) >> 4;
    if (lane < 17) sc.cnt[lane] = 0;
    __syncwarp();
    int key[8], rk[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) {  // key (bank pair 0..15, 16 = cold), stable rank within it
        const int p = lane + 32 * q;
        const bool live = p < cnt;
        key[q] = live ? ((unsigned)val[q] < (unsigned)H ? (val[q] & 15) : 16) : 17;
        const unsigned peers = __match_any_sync(0xffffffffu, key[q]);
        rk[q] = live ? sc.cnt[key[q]] + __popc(peers & lt) : 0;
        __syncwarp();
        if (live && (peers & lt) == 0) sc.cnt[key[q]] += __popc(peers);  // one leader per key
        __syncwarp();
    }
    // feasible iff every bank pair fits one entry per window, the last window included
    const int c = lane < 16 ? sc.cnt[lane] : 0;
    const int last_cap = cnt - 16 * (W - 1);
    const int h_last = __popc(__ballot_sync(0xffffffffu, lane < 16 && c > W - 1));
    if (!__all_sync(0xffffffffu, c <= W) || h_last > last_cap) {
#pragma unroll
        for (int q = 0; q < 8; ++q) dst[q] = lane + 32 * q < cnt ? lane + 32 * q : -1;
        return;
    }
    // window k: the bank pairs with more than k entries (mask; h_k of them first), then
    // free_k cold slots; F_k = cold entries placed before window k
    int Mk = 0;
    for (int k = 0; k < W; ++k) {
        const unsigned m = __ballot_sync(0xffffffffu, lane < 16 && c > k) & 0xffffu;
        if (lane == k) Mk = (int)m;
    }
    const int free_k = lane < W ? (lane == W - 1 ? last_cap : 16) - __popc(Mk) : 0;
    int F = free_k;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, F, o);
        if (lane >= o) F += y;
    }
    F -= free_k;
    if (lane < 16) {
        sc.msk[lane] = Mk;
        sc.f[lane] = lane < W ? F : 1 << 30;
    }
    __syncwarp();
#pragma unroll
    for (int q = 0; q < 8; ++q) {
        int d = -1;
        if (lane + 32 * q < cnt) {
            if (key[q] < 16) {  // hot: window rk, after the smaller bank pairs present there
                d = 16 * rk[q] + __popc(sc.msk[rk[q]] & ((1 << key[q]) - 1));
            } else {  // cold rank j: the last window whose first cold rank is <= j
                int k = 0;
#pragma unroll
                for (int step = 8; step; step >>= 1)
                    if (k + step < 16 && sc.f[k + step] <= rk[q]) k += step;
                d = 16 * k + __popc(sc.msk[k]) + (rk[q] - sc.f[k]);
            }
        }
        dst[q] = d;
    }
    __syncwarp();
}

// View columns of the hub rows (rows [0, n_hub), degree > kWarpNnz): one warp per chunk tile
// renames the old row's slice and writes it in bank-aware order (identity when sched == 0).
template <class RPO, class RPN>
__global__ void k_permute_chunks(const Tile* __restrict__ tiles, int n_chunk_tiles, const RPO* __restrict__ rp_old,
                                 const int* __restrict__ col_old, const RPN* __restrict__ rp_new,
                                 const int* __restrict__ order, const int* __restrict__ rank, int H, int sched,
                                 int* __restrict__ col_new, int64_t oa, int64_t ob) {
    __shared__ SchedScratch scr[8];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    for (int64_t t = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; t < n_chunk_tiles;
         t += ((int64_t)gridDim.x * blockDim.x) >> 5) {
        const Tile a = tiles[t];
        const int64_t z0 = a.nnz_begin;
        const int cnt = (int)(tiles[t + 1].nnz_begin - z0);
        const int h = a.row_begin;
        if (order[h] < oa || order[h] >= ob) continue;  // warp-uniform: another group of old rows
        const int64_t src = (int64_t)rp_old[order[h]] + (z0 - (int64_t)rp_new[h]);
        int val[8], dst[8];
#pragma unroll
        for (int q = 0; q < 8; ++q) {
            const int p = lane + 32 * q;
            val[q] = p < cnt ? rank[col_old[src + p]] : 0;
        }
        if (sched) {
            schedule_chunk(val, cnt, H, scr[w], dst);
        } else {
#pragma unroll
            for (int q = 0; q < 8; ++q) dst[q] = lane + 32 * q < cnt ? lane + 32 * q : -1;
        }
#pragma unroll
        for (int q = 0; q < 8; ++q)
            if (dst[q] >= 0) col_new[z0 + dst[q]] = val[q];
    }
}

// Bank-aware entry order inside PACK tiles (rows of <= kWarpNnz entries, L = 2^lg lanes per
// row; lane li of row g reads row offset li + s L at slot s, term.cuh term_step).  One
// instruction (slot s) serves a half-warp's 16 lanes at once, and its hot-prefix gathers
// (fp64 ids < H: bank pair id mod 16) conflict when two lanes hit the same bank pair.  Per
// half-warp, entries are redistributed within each row over that half-warp's offsets of the
// row: at every slot each lane takes, from its row's remaining entries, a hot entry on a
// bank pair still free at that slot, else a cold entry, else any.  Rows keep their entry
// sets (sums re-associated, deterministically).  One thread per (tile, half-warp).
template <class RPN>
__global__ void k_schedule_pack(const Tile* __restrict__ tiles, int t0, int t1, const RPN* __restrict__ rp, int H,
                                int* __restrict__ col) {
    for (int64_t job = t0 * 2 + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; job < (int64_t)t1 * 2;
         job += (int64_t)gridDim.x * blockDim.x) {
        const int t = (int)(job >> 1), hw = (int)(job & 1);
        const Tile a = tiles[t];
        if (a.meta & kTileChunk) continue;
        const int rows = tiles[t + 1].row_begin - a.row_begin;
        const int lg = a.meta & 0xf, L = 1 << lg;
        // rows of this half-warp and the lanes' offset classes
        int g0, g1, cls_lo, cls_hi;
        if (L <= 16) {
            g0 = hw * (16 >> lg);
            g1 = min(rows, g0 + (16 >> lg));
            cls_lo = 0;
            cls_hi = L;
        } else {  // one row over both half-warps: lanes li in [16 hw, 16 hw + 16)
            g0 = 0;
            g1 = rows > 0 ? 1 : 0;
            cls_lo = 16 * hw;
            cls_hi = 16 * hw + 16;
        }
        if (g0 >= g1) continue;
        int val[kWarpNnz];
        unsigned char rowof[kWarpNnz];
        bool used[kWarpNnz];
        int cnt = 0;
        int pstart[17], deg[16];
        int64_t base[16];
        for (int g = g0; g < g1; ++g) {
            const int k = g - g0;
            base[k] = (int64_t)rp[a.row_begin + g];
            deg[k] = (int)((int64_t)rp[a.row_begin + g + 1] - base[k]);
            pstart[k] = cnt;
            for (int o = 0; o < deg[k]; ++o) {
                const int li = o & (L - 1);
                if (li < cls_lo || li >= cls_hi) continue;
                val[cnt] = col[base[k] + o];
                rowof[cnt] = (unsigned char)k;
                used[cnt] = false;
                ++cnt;
            }
        }
        pstart[g1 - g0] = cnt;
        int out[kWarpNnz];
        for (int s = 0;; ++s) {
            bool any = false;
            unsigned banks = 0;
            for (int g = g0; g < g1; ++g) {
                const int k = g - g0;
                for (int li = cls_lo; li < cls_hi; ++li) {
                    const int o = li + s * L;
                    if (o >= deg[k]) continue;
                    any = true;
                    int pick = -1, cold = -1, anyi = -1;
                    for (int i = pstart[k]; i < pstart[k + 1]; ++i) {
                        if (used[i]) continue;
                        if (anyi < 0) anyi = i;
                        const int v = val[i];
                        if ((unsigned)v < (unsigned)H) {
                            if (!(banks >> (v & 15) & 1u)) {
                                pick = i;
                                break;
                            }
                        } else if (cold < 0) {
                            cold = i;
                        }
                    }
                    if (pick < 0) pick = cold >= 0 ? cold : anyi;
                    used[pick] = true;
                    if ((unsigned)val[pick] < (unsigned)H) banks |= 1u << (val[pick] & 15);
                    // slot (li, s) of row k: position among this half-warp's offsets of the row
                    out[pick] = o;  // entry `pick` goes to row offset o
                }
            }
            if (!any) break;
        }
        for (int i = 0; i < cnt; ++i) col[base[rowof[i]] + out[i]] = val[i];
    }
}

// Chunk tiles of rows whose ids were sorted ascending in place (x larger than L2): the
// same bank-aware chunk order as k_permute_chunks, applied to the sorted values (cold
// entries keep their ascending order in the free slots, so their gathers still walk x in
// address order).  One warp per chunk tile.
template <class RPN>
__global__ void k_schedule_chunks_inplace(const Tile* __restrict__ tiles, int n_chunk_tiles, int H,
                                          int* __restrict__ col) {
    __shared__ SchedScratch scr[8];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    for (int64_t t = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; t < n_chunk_tiles;
         t += ((int64_t)gridDim.x * blockDim.x) >> 5) {
        const int64_t z0 = tiles[t].nnz_begin;
        const int cnt = (int)(tiles[t + 1].nnz_begin - z0);
        int val[8], dst[8];
#pragma unroll
        for (int q = 0; q < 8; ++q) {
            const int p = lane + 32 * q;
            val[q] = p < cnt ? col[z0 + p] : 0;
        }
        __syncwarp();
        schedule_chunk(val, cnt, H, scr[w], dst);
#pragma unroll
        for (int q = 0; q < 8; ++q)
            if (dst[q] >= 0) col[z0 + dst[q]] = val[q];
        __syncwarp();
    }
}

// Halo masks of a row partition: bit r of mask[u] iff row u has a neighbour owned by rank r
// (column ids are global sorted ids, owner = part_owner).  Warp per row; also counts the
// remote stores per term (halo vs replicate-to-all) in int64.
template <class RPN>
__global__ void k_push_mask(const RPN* __restrict__ rp, const int* __restrict__ col, int64_t nl,
                            int G, int rank, unsigned* __restrict__ mask, unsigned long long* __restrict__ counts) {
    const int lane = threadIdx.x & 31;
    unsigned long long halo = 0;
    for (int64_t u = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; u < nl;
         u += ((int64_t)gridDim.x * blockDim.x) >> 5) {
        unsigned m = 0;
        for (int64_t j = (int64_t)rp[u] + lane; j < (int64_t)rp[u + 1]; j += 32) m |= 1u << part_owner(col[j], G);
        for (int o = 16; o; o >>= 1) m |= __shfl_xor_sync(0xffffffffu, m, o);
        if (lane == 0) {
            mask[u] = m;
            halo += (unsigned long long)__popc(m & ~(1u << rank));
        }
    }
    if (lane == 0 && halo) atomicAdd(counts, halo);
}

// View rows whose old row lies in [oa, ob): their [begin, end) entry ranges, appended in
// any order (each segment is sorted on its own, so the order of the list does not matter).
template <class RPN>
__global__ void k_group_segments(const int* __restrict__ order, const RPN* __restrict__ rp, int64_t nl, int64_t oa,
                                 int64_t ob, int64_t* __restrict__ seg_b, int64_t* __restrict__ seg_e,
                                 unsigned long long* __restrict__ cnt) {
    for (int64_t w = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; w < nl; w += (int64_t)gridDim.x * blockDim.x) {
        const int o = order[w];
        if (o < oa || o >= ob) continue;
        const unsigned long long i = atomicAdd(cnt, 1ull);
        seg_b[i] = (int64_t)rp[w];
        seg_e[i] = (int64_t)rp[w + 1];
    }
}

// This rank's rows of the block-cyclic partition: old ids and degrees of its local rows.
__global__ void k_gather_local(const int* __restrict__ order_g, const int64_t* __restrict__ deg_g, int64_t nl,
                               int rank, int G, int* __restrict__ order_l, int64_t* __restrict__ deg_l) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nl; i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t u = part_global(i, rank, G);
        order_l[i] = order_g[u];
        deg_l[i] = deg_g[u];
    }
}


__global__ void k_gather_inv(const double* __restrict__ inv, const int* __restrict__ order,
                             int64_t n, double* __restrict__ out) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x)
        out[i] = inv[order[i]];
}

}  // namespace

// Pinned staging for the view's small host<->device transfers.  Pageable copies are staged
// by the driver behind whatever the copy engine is doing — during an upload that is the
// neighbour array — so the view build would wait for it.  Grow-only slots, process-wide,
// held under a lock for one build (every build ends with a stream synchronize).
struct PinnedArena {
    std::mutex mu;
    void* p[5] = {};
    size_t n[5] = {};
    void* get(int slot, size_t bytes) {
        if (bytes > n[slot]) {
            if (p[slot]) CHEB_CUDA_CHECK(cudaFreeHost(p[slot]));
            p[slot] = nullptr;
            n[slot] = 0;
            const size_t want = std::max<size_t>(bytes + bytes / 4, 1 << 16);
            CHEB_CUDA_CHECK(cudaHostAlloc(&p[slot], want, cudaHostAllocPortable));
            n[slot] = want;
        }
        return p[slot];
    }
};
PinnedArena& pinned_arena() {
    static PinnedArena* a = new PinnedArena();  // never destroyed: outlives every handle
    return *a;
}
// Pinned (mapped) host memory -> device by a kernel reading it over the bus.  During an
// upload the copy engine is busy with the neighbour DMA (8.4 GB on config 4) and a
// cudaMemcpyAsync of the view's tiles and programs waited behind all of it (~150 ms); the
// kernel's reads interleave with the DMA instead.
__global__ void k_pull_host(const unsigned char* __restrict__ src, size_t bytes, unsigned char* __restrict__ dst) {
    const size_t n16 = bytes / 16;
    const size_t tid = blockIdx.x * (size_t)blockDim.x + threadIdx.x, nth = (size_t)gridDim.x * blockDim.x;
    for (size_t i = tid; i < n16; i += nth)
        reinterpret_cast<uint4*>(dst)[i] = reinterpret_cast<const uint4*>(src)[i];
    for (size_t i = n16 * 16 + tid; i < bytes; i += nth) dst[i] = src[i];
}
void h2d_pinned(void* dst, const void* pinned, size_t bytes, cudaStream_t st) {
    void* dsrc = nullptr;
    const bool aligned = ((uintptr_t)dst & 15) == 0 && ((uintptr_t)pinned & 15) == 0;
    if (bytes > 0 && aligned && tuning().pull && cudaHostGetDevicePointer(&dsrc, const_cast<void*>(pinned), 0) == cudaSuccess) {
        const int grid = (int)std::min<size_t>((bytes / 16 + kBuildThreads - 1) / kBuildThreads + 1, 148 * 8);
        k_pull_host<<<grid, kBuildThreads, 0, st>>>(static_cast<const unsigned char*>(dsrc), bytes,
                                                    static_cast<unsigned char*>(dst));
        CHEB_CUDA_CHECK(cudaGetLastError());
        return;
    }
    cudaGetLastError();
    if (bytes > 0) CHEB_CUDA_CHECK(cudaMemcpyAsync(dst, pinned, bytes, cudaMemcpyHostToDevice, st));
}
void h2d_staged(void* dst, const void* src, size_t bytes, int slot, cudaStream_t st) {
    void* h = pinned_arena().get(slot, bytes);
    std::memcpy(h, src, bytes);
    h2d_pinned(dst, h, bytes, st);
}

// Greedy tiling of the degree-sorted rows (runs of equal degree, descending), emitted per
// run rather than per tile: a run of hub rows (degree > kWarpNnz) is one segment of
// ceil(d / kWarpNnz) chunk tiles per row; a run of short rows is one segment of its whole
// tiles (kf = min(32, kWarpNnz / d) rows each) plus single tiles where a tile spans a run
// boundary.  k_expand_tiles writes the tiles on the device, so an upload does not push the
// tile list (16 B per tile, 67 MB on config 4) over a bus the neighbour DMA is saturating.
struct TileSeg {
    int64_t z0;     // nnz_begin of the segment's first tile
    int32_t row0;   // row_begin of its first tile
    int32_t tile0;  // id of its first tile
    int32_t count;  // tiles
    int32_t d;      // row degree (single tiles: unused)
    int32_t k;      // rows per tile (pack) | chunk tiles per row (kTileChunk)
    int32_t meta;   // pack: log2 lanes per row; chunk: kTileChunk
};

static std::vector<TileSeg> make_tile_segs(const std::vector<int64_t>& run_deg, const std::vector<int64_t>& run_cnt,
                                           int64_t n, int64_t nnz, SolverView& V) {
    std::vector<TileSeg> segs;
    int64_t row = 0, z = 0, tile = 0;
    int64_t cur_rows = 0, cur_nnz = 0, cur_row0 = 0, cur_z0 = 0, cur_dmax = 0;
    V.n_hub = 0;
    V.n_hub_wide = 0;
    V.n_chunk_tiles = 0;
    for (int b = 0; b < 7; ++b) V.bin_tiles[b] = V.bin_rows[b] = V.bin_nnz[b] = 0;
    auto lanes_log2 = [](int64_t dmax, int64_t rows) {
        // lanes per row: as many as 32 lanes allow for the tile's rows, but no more than
        // ~dmax/4 (each lane then walks >= 4 nnz; rows of a tile have similar degree)
        int lg = 0;
        while (lg < 5 && (rows << (lg + 1)) <= 32 && (int64_t(4) << (lg + 1)) <= dmax + 3) ++lg;
        return lg;
    };
    auto emit = [&](int64_t z0, int64_t r0, int64_t cnt, int64_t d, int64_t k, int meta, int64_t rows, int64_t nz) {
        segs.push_back(TileSeg{z0, (int32_t)r0, (int32_t)tile, (int32_t)cnt, (int32_t)d, (int32_t)k, meta});
        const int bin = (meta & kTileChunk) ? 6 : (meta & 0xf);
        V.bin_tiles[bin] += cnt;
        V.bin_rows[bin] += rows;
        V.bin_nnz[bin] += nz;
        tile += cnt;
    };
    auto close = [&] {
        if (cur_rows == 0) return;
        emit(cur_z0, cur_row0, 1, cur_dmax, cur_rows, lanes_log2(cur_dmax, cur_rows), cur_rows, cur_nnz);
        cur_rows = cur_nnz = 0;
    };
    for (size_t r = 0; r < run_deg.size(); ++r) {
        const int64_t d = run_deg[r];
        int64_t c = run_cnt[r];
        if (d > kWarpNnz) {
            close();
            const int64_t nch = (d + kWarpNnz - 1) / kWarpNnz;
            emit(z, row, c * nch, d, nch, kTileChunk, 0, c * d);
            V.n_chunk_tiles += (int)(c * nch);
            V.n_hub += c;
            if (nch > 32) V.n_hub_wide = V.n_hub;  // degree-descending: a prefix of the hub rows
            row += c;
            z += c * d;
            continue;
        }
        while (c > 0) {
            if (cur_rows == 0) {
                // whole tiles of kf rows: each closes as soon as it is full (32 rows, or no
                // room for another row of degree d)
                const int64_t kf = d > 0 ? std::min<int64_t>(kWarpRows, kWarpNnz / d) : 0;
                const int64_t m = kf > 0 ? c / kf : 0;
                if (m > 0) {
                    emit(z, row, m, d, kf, lanes_log2(d, kf), m * kf, m * kf * d);
                    row += m * kf;
                    z += m * kf * d;
                    c -= m * kf;
                    continue;
                }
                cur_row0 = row;
                cur_z0 = z;
                cur_dmax = d;
            }
            const int64_t room_rows = kWarpRows - cur_rows;
            const int64_t room_nnz = d > 0 ? (kWarpNnz - cur_nnz) / d : INT64_MAX;
            const int64_t k = std::min(c, std::min(room_rows, room_nnz));
            if (k == 0) {
                close();
                continue;
            }
            cur_rows += k;
            cur_nnz += k * d;
            row += k;
            z += k * d;
            c -= k;
            if (cur_rows == kWarpRows || kWarpNnz - cur_nnz < d) close();
        }
    }
    close();
    if (row != n || z != nnz) fail(CHEB_CUDA, "tiling does not cover the graph");
    if (tile >= INT32_MAX) fail(CHEB_CAPACITY, "too many tiles");
    V.bin_rows[6] = V.n_hub;
    V.n_tiles = (int)tile;
    return segs;
}

// Tiles (+ sentinel {nnz, n}) and hub_first (first chunk tile of each hub row, then
// n_chunk_tiles) from the run segments: thread per tile, segment by binary search on tile0.
__global__ void k_expand_tiles(const TileSeg* __restrict__ segs, int nseg, int n_tiles, int64_t nnz, int32_t n,
                               int n_hub, int n_chunk_tiles, Tile* __restrict__ tiles, int* __restrict__ hub_first) {
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t <= n_tiles; t += (int64_t)gridDim.x * blockDim.x) {
        if (t == n_tiles) {
            tiles[t] = Tile{nnz, n, 0};
            hub_first[n_hub] = n_chunk_tiles;
            continue;
        }
        int lo = 0, hi = nseg - 1;
        while (lo < hi) {  // last segment with tile0 <= t
            const int mid = (lo + hi + 1) >> 1;
            if (segs[mid].tile0 <= t) lo = mid;
            else hi = mid - 1;
        }
        const TileSeg sg = segs[lo];
        const int64_t i = t - sg.tile0;
        if (sg.meta & kTileChunk) {
            const int64_t r = i / sg.k, q = i % sg.k;
            tiles[t] = Tile{sg.z0 + r * sg.d + q * kWarpNnz, (int32_t)(sg.row0 + r), kTileChunk};
            if (q == 0) hub_first[sg.row0 + r] = (int)t;
        } else {
            tiles[t] = Tile{sg.z0 + i * sg.k * (int64_t)sg.d, (int32_t)(sg.row0 + i * sg.k), sg.meta};
        }
    }
}

// One launch's warp program from the tile list (identity order): tile t is entry t / S of
// warp t % S.  A chunk tile's WTile.row_begin holds its tile id (its hub_part slot).
__global__ void k_build_program(const Tile* __restrict__ tiles, int n_tiles, int S, int len, WTile* __restrict__ prog) {
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n_tiles; t += (int64_t)gridDim.x * blockDim.x) {
        const Tile a = tiles[t], b = tiles[t + 1];
        const bool chunk = (a.meta & kTileChunk) != 0;
        WTile w;
        w.nnz_begin = a.nnz_begin;
        w.row_begin = chunk ? (int32_t)t : a.row_begin;
        w.cnt = (uint16_t)(b.nnz_begin - a.nnz_begin);
        w.rows = (uint8_t)(chunk ? 1 : (b.row_begin - a.row_begin));
        w.meta = (uint8_t)a.meta;
        prog[(size_t)(t % S) * len + t / S] = w;
    }
}

// Tile-bin statistics of the view (host): 0..5 = pack tiles with 2^b lanes per row, 6 = chunk tiles.
static void tile_stats(SolverView& V, const std::vector<Tile>& tiles) {
    for (int b = 0; b < 7; ++b) V.bin_tiles[b] = V.bin_rows[b] = V.bin_nnz[b] = 0;
    for (int t = 0; t < V.n_tiles; ++t) {
        const Tile& a = tiles[t];
        const Tile& b = tiles[t + 1];
        const int bin = (a.meta & kTileChunk) ? 6 : (a.meta & 0xf);
        ++V.bin_tiles[bin];
        V.bin_nnz[bin] += b.nnz_begin - a.nnz_begin;
        V.bin_rows[bin] += (a.meta & kTileChunk) ? 0 : (int64_t)(b.row_begin - a.row_begin);
    }
    V.bin_rows[6] = V.n_hub;
}

// Per-warp tile programs (warp-major, each padded to whole descriptor blocks): entry i of
// a launch's tile list goes to warp i % S, position i / S.  lists == null: one launch over
// every tile in tile order; otherwise one launch per list (V.phases, ranges filled by the
// caller), the programs concatenated.  A chunk tile's WTile.row_begin holds its tile id:
// the slot of its partial in hub_part, whatever position it runs at.
static void upload_programs(SolverView& V, const std::vector<Tile>& tiles,
                            const std::vector<std::vector<int>>* lists, cudaStream_t st) {
    const int S = V.grid * kWarps;
    auto len_of = [&](int64_t cnt) {
        const int64_t per = (cnt + S - 1) / S;
        return (int)std::max<int64_t>(kDescBlock, (per + kDescBlock - 1) / kDescBlock * kDescBlock);
    };
    const int nl = lists ? (int)lists->size() : 1;
    std::vector<int> lens(nl);
    size_t np = 0;
    for (int p = 0; p < nl; ++p) {
        lens[p] = len_of(lists ? (int64_t)(*lists)[p].size() : (int64_t)V.n_tiles);
        np += (size_t)S * lens[p];
    }
    auto* prog = static_cast<WTile*>(pinned_arena().get(1, sizeof(WTile) * np));  // built in place
    std::memset(prog, 0, sizeof(WTile) * np);
    auto wtile = [&](int t) {
        const Tile& a = tiles[t];
        const Tile& b = tiles[t + 1];
        const bool chunk = (a.meta & kTileChunk) != 0;
        WTile w;
        w.nnz_begin = a.nnz_begin;
        w.row_begin = chunk ? t : a.row_begin;
        w.cnt = (uint16_t)(b.nnz_begin - a.nnz_begin);
        w.rows = (uint8_t)(chunk ? 1 : (b.row_begin - a.row_begin));
        w.meta = (uint8_t)a.meta;
        return w;
    };
    size_t off = 0;
    if (lists) V.phases.resize(nl);
    else V.phases.clear();
    for (int p = 0; p < nl; ++p) {
        WTile* pg = prog + off;
        const int L = lens[p];
        const int cnt = lists ? (int)(*lists)[p].size() : V.n_tiles;
        for (int i = 0; i < cnt; ++i) pg[(size_t)(i % S) * L + i / S] = wtile(lists ? (*lists)[p][i] : i);
        if (lists) {
            V.phases[p].prog_off = (int64_t)off;
            V.phases[p].prog_len = L;
            V.phases[p].ntiles = cnt;
        }
        off += (size_t)S * L;
    }
    V.prog_len = lens[0];
    V.prog.alloc(sizeof(WTile) * np);
    h2d_pinned(V.prog.get(), prog, sizeof(WTile) * np, st);
}

// Column-blocked chunk schedule (x larger than L2; rows hold ascending ids).  x ids are cut
// into K blocks; every hub row's entries are split where its ids cross a block boundary
// (binary search per (row, boundary): k_hub_splits) and each piece is cut into chunk tiles of
// <= kWarpNnz entries, so a chunk gathers from one block only.  A term then runs one launch
// per block, highest first, each under an L2 window over its slice of x: the gathers of a
// launch hit an L2-resident slice instead of missing across all of x (config 4: 136 MB of
// fp64 x against a 126 MB L2).  Block 0 (the hot prefix and the hubs) runs last, with the
// pack tiles.  Chunk partials are still combined in position order by k_hub_finalize
// (tile ids stay in row order), so the schedule is deterministic.
template <class RPN>
__global__ void k_hub_splits(const RPN* __restrict__ rp, const int* __restrict__ col, int64_t n_hub,
                             const int* __restrict__ bounds, int nb, int* __restrict__ out) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n_hub * nb;
         i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t h = i / nb;
        const int key = bounds[i % nb];
        int64_t lo = rp[h], hi = rp[h + 1];
        const int64_t b = lo;
        while (lo < hi) {
            const int64_t mid = (lo + hi) >> 1;
            if (col[mid] < key) lo = mid + 1;
            else hi = mid;
        }
        out[i] = (int)(lo - b);
    }
}

template <class RPN>
static void column_block_schedule(SolverView& V, int K, int64_t x_len, cudaStream_t st) {
    const int64_t n_hub = V.n_hub;
    std::vector<Tile> tiles((size_t)V.n_tiles + 1);
    CHEB_CUDA_CHECK(cudaMemcpyAsync(tiles.data(), V.tiles.get(), sizeof(Tile) * tiles.size(), cudaMemcpyDeviceToHost, st));
    const int nb = K - 1;
    std::vector<int> bounds(nb);
    for (int j = 1; j < K; ++j) {
        int64_t b = x_len * j / K;
        if (K == 2 && tuning().colsplit_pct > 0 && tuning().colsplit_pct < 100) b = x_len * tuning().colsplit_pct / 100;
        bounds[j - 1] = (int)(b & ~int64_t(31));  // whole 256-byte x segments per window
    }
    std::vector<int> splits((size_t)n_hub * nb);
    {
        DevMem d_b(sizeof(int) * nb), d_s(sizeof(int) * std::max<size_t>(splits.size(), 1));
        CHEB_CUDA_CHECK(cudaMemcpyAsync(d_b.get(), bounds.data(), sizeof(int) * nb, cudaMemcpyHostToDevice, st));
        k_hub_splits<RPN><<<grid_for(n_hub * nb), kBuildThreads, 0, st>>>(V.row_ptr.ptr<RPN>(), V.col.ptr<int>(), n_hub,
                                                                        d_b.ptr<int>(), nb, d_s.ptr<int>());
        CHEB_CUDA_CHECK(cudaGetLastError());
        CHEB_CUDA_CHECK(cudaMemcpyAsync(splits.data(), d_s.get(), sizeof(int) * splits.size(), cudaMemcpyDeviceToHost, st));
        CHEB_CUDA_CHECK(cudaStreamSynchronize(st));
    }
    const int old_chunks = V.n_chunk_tiles;
    std::vector<Tile> nt;
    std::vector<int> blk;  // block of each chunk tile
    std::vector<int> hub_first;
    nt.reserve(tiles.size() + (size_t)n_hub * nb);
    int h = -1;
    for (int t = 0; t < old_chunks;) {  // the old chunk tiles of row h are consecutive
        h = tiles[t].row_begin;
        int t1 = t;
        while (t1 < old_chunks && tiles[t1].row_begin == h) ++t1;
        const int64_t z = tiles[t].nnz_begin, d = tiles[t1].nnz_begin - z;
        hub_first.push_back((int)nt.size());
        int64_t a = 0;
        for (int j = 0; j < K; ++j) {
            const int64_t e = j < nb ? (int64_t)splits[(size_t)h * nb + j] : d;
            for (int64_t p = a; p < e; p += kWarpNnz) {
                nt.push_back(Tile{z + p, (int32_t)h, kTileChunk});
                blk.push_back(j);
            }
            a = std::max(a, e);
        }
        t = t1;
    }
    if ((int64_t)hub_first.size() != n_hub) fail(CHEB_CUDA, "column-block schedule: hub rows do not match");
    V.n_hub_wide = 0;  // rows with more than 32 chunks after the split: warp rows of the hub finalize
    for (int64_t r = 0; r < n_hub; ++r)
        if ((r + 1 < n_hub ? hub_first[(size_t)r + 1] : (int)nt.size()) - hub_first[(size_t)r] > 32) V.n_hub_wide = r + 1;
    const int new_chunks = (int)nt.size();
    hub_first.push_back(new_chunks);
    for (size_t t = (size_t)old_chunks; t < tiles.size(); ++t) nt.push_back(tiles[t]);  // pack tiles + sentinel
    tiles.swap(nt);
    V.n_chunk_tiles = new_chunks;
    V.n_tiles = (int)tiles.size() - 1;
    tile_stats(V, tiles);
    std::vector<std::vector<int>> lists(K);
    for (int t = 0; t < new_chunks; ++t) lists[(size_t)(K - 1 - blk[t])].push_back(t);
    for (int t = new_chunks; t < V.n_tiles; ++t) lists[(size_t)K - 1].push_back(t);
    upload_programs(V, tiles, &lists, st);
    for (int p = 0; p < K; ++p) {
        const int j = K - 1 - p;
        V.phases[p].x_lo = j == 0 ? 0 : bounds[j - 1];
        V.phases[p].x_hi = j == nb ? x_len : bounds[j];
        V.phases[p].epi = p == K - 1;
    }
    V.hub_first.alloc(sizeof(int) * hub_first.size());
    h2d_staged(V.hub_first.get(), hub_first.data(), sizeof(int) * hub_first.size(), 0, st);
    V.tiles.alloc(sizeof(Tile) * tiles.size());
    h2d_staged(V.tiles.get(), tiles.data(), sizeof(Tile) * tiles.size(), 2, st);
    CHEB_CUDA_CHECK(cudaStreamSynchronize(st));
}

// ---------------------------------------------------------------------------
// Column windows of the hub rows (SolverView::Windows; rows hold ascending ids)
// ---------------------------------------------------------------------------
// S[h][j], j = 0..NW: position inside hub row h of the first id >= H0 + j W.
template <class RPN>
__global__ void k_win_splits(const RPN* __restrict__ rp, const int* __restrict__ col, int64_t n_hub, int H0, int W,
                             int NW, int* __restrict__ S) {
    const int64_t total = n_hub * (NW + 1);
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t h = i / (NW + 1);
        const int j = (int)(i - h * (NW + 1));
        const int64_t key64 = (int64_t)H0 + (int64_t)j * W;
        const int key = key64 > INT32_MAX ? INT32_MAX : (int)key64;
        int64_t lo = rp[h], hi = rp[h + 1];
        const int64_t b = lo;
        while (lo < hi) {
            const int64_t mid = (lo + hi) >> 1;
            if (col[mid] < key) lo = mid + 1;
            else hi = mid;
        }
        S[i] = (int)(lo - b);
    }
}

// Piece sizes, window-major: csz[w n_hub + h] = entries of row h inside window w (tail: 0).
__global__ void k_win_sizes(const int* __restrict__ S, int64_t n_hub, int NW, int64_t* __restrict__ csz) {
    const int64_t total = n_hub * NW;
    for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q <= total; q += (int64_t)gridDim.x * blockDim.x) {
        if (q == total) {
            csz[q] = 0;
            continue;
        }
        const int64_t w = q / n_hub, h = q - w * n_hub;
        csz[q] = (int64_t)(S[h * (NW + 1) + w + 1] - S[h * (NW + 1) + w]);
    }
}

__global__ void k_win_gather_starts(const int64_t* __restrict__ off, int64_t n_hub, int NW, int64_t* __restrict__ out) {
    const int w = blockIdx.x * blockDim.x + threadIdx.x;
    if (w <= NW) out[w] = off[(int64_t)w * n_hub];
}

// Window-local 16-bit ids into the stream, and each piece's start bit: hub row h by `nt`
// cooperating threads.
template <class RPN>
__device__ __forceinline__ void win_copy_row(const RPN* __restrict__ rp, const int* __restrict__ col, int64_t n_hub,
                                             const int* __restrict__ S, const int64_t* __restrict__ off,
                                             const int64_t* __restrict__ delta, int H0, int W, int NW,
                                             unsigned short* __restrict__ wcol, unsigned* __restrict__ flags32,
                                             int64_t h, int t, int nt) {
    const int64_t base = rp[h];
    const int* Sh = S + h * (NW + 1);
    const int e0 = Sh[0], e1 = Sh[NW];
    for (int e = e0 + t; e < e1; e += nt) {
        const int id = col[base + e] - H0;
        const int w = id / W;
        const int64_t pos = off[(int64_t)w * n_hub + h] + delta[w] + (e - Sh[w]);
        wcol[pos] = (unsigned short)(id - w * W);
    }
    for (int w = t; w < NW; w += nt) {
        if (Sh[w + 1] > Sh[w]) {
            const int64_t pos = off[(int64_t)w * n_hub + h] + delta[w];
            atomicOr(&flags32[pos >> 5], 1u << (pos & 31));
        }
    }
}
constexpr int kWinBigRow = 4096;  // windowed entries above which a CTA copies the row (rows [0, kWinBigRows) only)
constexpr int kWinBigRows = 8192;
// A warp per hub row (rows a CTA takes are skipped) / a CTA per leading hub row.
template <class RPN, bool BIG>
__global__ void k_win_copy(const RPN* __restrict__ rp, const int* __restrict__ col, int64_t n_hub,
                           const int* __restrict__ S, const int64_t* __restrict__ off,
                           const int64_t* __restrict__ delta, int H0, int W, int NW,
                           unsigned short* __restrict__ wcol, unsigned* __restrict__ flags32) {
    if (BIG) {
        const int64_t h = blockIdx.x;
        if (S[h * (NW + 1) + NW] - S[h * (NW + 1)] > kWinBigRow)
            win_copy_row(rp, col, n_hub, S, off, delta, H0, W, NW, wcol, flags32, h, (int)threadIdx.x, (int)blockDim.x);
        return;
    }
    const int lane = threadIdx.x & 31;
    const int64_t gw = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t h = gw; h < n_hub; h += nw) {
        if (h < kWinBigRows && S[h * (NW + 1) + NW] - S[h * (NW + 1)] > kWinBigRow) continue;
        win_copy_row(rp, col, n_hub, S, off, delta, H0, W, NW, wcol, flags32, h, lane, 32);
    }
}

// Pieces starting inside block [blk 256, +256) before in-block position r (the block's
// first entry always starts one).
__device__ __forceinline__ int win_starts_before(const unsigned* __restrict__ flags32, int64_t blk, int r) {
    const unsigned* words = flags32 + blk * (kWinBlock / 32);
    int cnt = 0;
#pragma unroll
    for (int j = 0; j < kWinBlock / 32; ++j) {
        unsigned wd = words[j];
        if (j == 0) wd |= 1u;
        const int lo = j * 32;
        if (r >= lo + 32) cnt += __popc(wd);
        else if (r > lo) cnt += __popc(wd & ((1u << (r - lo)) - 1u));
    }
    return cnt;
}

// Padding between a window's last entry and its last block's end: one dummy piece.
__global__ void k_win_padflags(const int64_t* __restrict__ wend, int NW, unsigned* __restrict__ flags32) {
    const int w = blockIdx.x * blockDim.x + threadIdx.x;
    if (w < NW && (wend[w] & (kWinBlock - 1))) atomicOr(&flags32[wend[w] >> 5], 1u << (wend[w] & 31));
}

// Entries re-ordered inside their pieces (a piece is a sum: any order) so that the 16 lanes
// of a half-warp read distinct bank pairs of the fp64 window (id mod 16) in each of the 8
// gather instructions of a block: position p is read by lane p / 8 in instruction p % 8.
// Greedy: each position takes, among the next entries of its piece, one whose bank pair the
// instruction's half-warp has not used yet.
#ifndef CHEB_WIN_LOOK
#define CHEB_WIN_LOOK 24
#endif
constexpr int kBankLook = CHEB_WIN_LOOK;  // candidates a position may choose from (the next entries of its piece)
// A thread per half block (the half-warps of a gather instruction are independent: positions
// 0-127 belong to lanes 0-15), candidates never taken from the other half.
constexpr int kBankBlocks = 64, kBankThreads = 2 * kBankBlocks, kBankHalf = kWinBlock / 2;
constexpr int kBankStride = kBankHalf + 2;  // shorts per thread row (65 words: conflict-free)
__global__ void __launch_bounds__(kBankThreads)
k_win_bank_order(unsigned short* __restrict__ wcol, const unsigned* __restrict__ flags32, int64_t n_blocks) {
    __shared__ unsigned short sh[kBankThreads * kBankStride];
    for (int64_t b0 = (int64_t)blockIdx.x * kBankBlocks; b0 < n_blocks; b0 += (int64_t)gridDim.x * kBankBlocks) {
        const int nb = (int)min((int64_t)kBankBlocks, n_blocks - b0);
        __syncthreads();
        {  // the CTA's blocks into shared memory, 4 bytes per thread per step; row = (block, half)
            const unsigned* src = reinterpret_cast<const unsigned*>(wcol + b0 * kWinBlock);
            for (int i = threadIdx.x; i < nb * kBankHalf; i += kBankThreads) {
                const int r = i / (kBankHalf / 2), c = i % (kBankHalf / 2);
                *reinterpret_cast<unsigned*>(&sh[r * kBankStride + 2 * c]) = src[i];
            }
        }
        __syncthreads();
        if ((int)threadIdx.x < 2 * nb) {
            unsigned short* ids = sh + threadIdx.x * kBankStride;
            const int half = threadIdx.x & 1;
            const unsigned* fwp = flags32 + (b0 + (threadIdx.x >> 1)) * (kWinBlock / 32) + half * (kBankHalf / 32);
            unsigned fw[kBankHalf / 32 + 1];
#pragma unroll
            for (int j = 0; j < kBankHalf / 32; ++j) fw[j] = fwp[j];
            fw[kBankHalf / 32] = half ? 1u : fwp[kBankHalf / 32];  // the next block starts a piece
            unsigned used[8] = {0, 0, 0, 0, 0, 0, 0, 0};  // [instruction]: bank pairs taken by this half-warp
            int pe = 0;
#pragma unroll
            for (int wq = 0; wq < kBankHalf / 32; ++wq) {
                const unsigned fword = fw[wq], fnext = fw[wq + 1];
                for (int p4 = 0; p4 < 4; ++p4) {
#pragma unroll
                    for (int i = 0; i < 8; ++i) {
                        const int p = wq * 32 + p4 * 8 + i;  // position inside the half
                        if (p >= pe) {  // end of the piece holding p: next start bit, at most kBankLook positions on
                            const int q = p4 * 8 + i + 1;  // in-word bit of p + 1
                            const unsigned long long bits = ((unsigned long long)fnext << 32 | fword) >> q;
                            const int d = bits ? __ffsll((long long)bits) - 1 : 64;
                            pe = min(min(p + 1 + d, p + kBankLook), kBankHalf);
                        }
                        const unsigned mask = used[i];
                        int pick = p;
                        for (int j = p; j < pe; ++j)
                            if (!((mask >> (ids[j] & 15)) & 1u)) {
                                pick = j;
                                break;
                            }
                        const unsigned short v = ids[pick];
                        ids[pick] = ids[p];
                        ids[p] = v;
                        used[i] |= 1u << (v & 15);
                    }
                }
            }
        }
        __syncthreads();
        {
            unsigned* dst = reinterpret_cast<unsigned*>(wcol + b0 * kWinBlock);
            for (int i = threadIdx.x; i < nb * kBankHalf; i += kBankThreads) {
                const int r = i / (kBankHalf / 2), c = i % (kBankHalf / 2);
                dst[i] = *reinterpret_cast<const unsigned*>(&sh[r * kBankStride + 2 * c]);
            }
        }
    }
}

// Per lane of every block: its 8 start bits (block start forced) and the number of pieces
// started in the block's earlier lanes, as one 16-bit word (starts | before << 8).
__global__ void k_win_lanemeta(const unsigned char* __restrict__ flags8, int64_t n_blocks,
                               unsigned short* __restrict__ meta) {
    const int lane = threadIdx.x & 31;
    const int64_t gw = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t b = gw; b < n_blocks; b += nw) {
        unsigned m = flags8[b * 32 + lane];
        if (lane == 0) m |= 1u;
        const int mine = __popc(m);
        int pre = mine;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int t = __shfl_up_sync(0xffffffffu, pre, o);
            if (lane >= o) pre += t;
        }
        meta[b * 32 + lane] = (unsigned short)(m | ((unsigned)(pre - mine) << 8));
    }
}

__global__ void k_win_blockcount(const unsigned* __restrict__ flags32, int64_t n_blocks, int* __restrict__ pc) {
    for (int64_t b = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; b <= n_blocks; b += (int64_t)gridDim.x * blockDim.x)
        pc[b] = b < n_blocks ? win_starts_before(flags32, b, kWinBlock) : 0;
}

// Block ranges of the window pass's CTAs: equal shares of the cost 256 b + pw pieces(b)
// (blocks of short pieces store more sums and keep more bank conflicts).
__global__ void k_win_cta_starts(const int* __restrict__ bbase, int64_t n_blocks, int pw, int grid,
                                 int64_t* __restrict__ out) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i > grid) return;
    const double total = 256.0 * (double)n_blocks + (double)pw * (double)bbase[n_blocks];
    const double target = total * (double)i / (double)grid;
    int64_t lo = 0, hi = n_blocks;
    while (lo < hi) {  // first b with cost(b) >= target
        const int64_t mid = (lo + hi) >> 1;
        if (256.0 * (double)mid + (double)pw * (double)bbase[mid] < target) lo = mid + 1;
        else hi = mid;
    }
    out[i] = i == grid ? n_blocks : lo;
}

// Per hub row: its chunk tiles over the entries left in the row (ids < H0, then ids past the
// last window), its pieces before window w (subx), and its piece count.
template <class RPN>
__global__ void k_win_rows(const RPN* __restrict__ rp, int64_t n_hub, const int* __restrict__ S,
                           const int64_t* __restrict__ off, const int64_t* __restrict__ delta, int NW, int wide_min,
                           int drop_tail, int* __restrict__ mc, int* __restrict__ rowpieces, int* __restrict__ subx,
                           unsigned long long* __restrict__ wide) {
    for (int64_t h = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; h <= n_hub; h += (int64_t)gridDim.x * blockDim.x) {
        if (h == n_hub) {
            mc[h] = 0;
            rowpieces[h] = 0;
            continue;
        }
        const int64_t d = rp[h + 1] - rp[h];
        const int* Sh = S + h * (NW + 1);
        const int64_t sA = Sh[0], tail = d - Sh[NW];
        const int m = drop_tail ? 0 : (int)((sA + kWarpNnz - 1) / kWarpNnz + (tail + kWarpNnz - 1) / kWarpNnz);
        int s = 0;
        for (int w = 0; w < NW; ++w) {
            subx[h * NW + w] = s;
            const int64_t c = Sh[w + 1] - Sh[w];
            if (c > 0) {
                const int64_t pos = off[(int64_t)w * n_hub + h] + delta[w];
                s += (int)(((pos + c - 1) >> 8) - (pos >> 8)) + 1;
            }
        }
        mc[h] = m;
        rowpieces[h] = s;
        if (m + s > wide_min) atomicMax(wide, (unsigned long long)(h + 1));
    }
}
static_assert(kWinBlock == 256, "k_win_rows / k_win_klist shift by 8");

// Every hub row's pieces (stream indices), row by row in window order: klist[kf[h] ..).
__global__ void k_win_klist(int64_t n_hub, const int* __restrict__ S, const int64_t* __restrict__ off,
                            const int64_t* __restrict__ delta, int NW, const unsigned* __restrict__ flags32,
                            const int* __restrict__ bbase, const int* __restrict__ kf, const int* __restrict__ subx,
                            int* __restrict__ klist) {
    const int64_t total = n_hub * NW;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t h = i / NW;
        const int w = (int)(i - h * NW);
        const int64_t c = S[h * (NW + 1) + w + 1] - S[h * (NW + 1) + w];
        if (c <= 0) continue;
        const int64_t pos = off[(int64_t)w * n_hub + h] + delta[w];
        const int64_t blk = pos >> 8;
        const int nsub = (int)(((pos + c - 1) >> 8) - blk) + 1;
        int* dst = klist + kf[h] + subx[i];
        dst[0] = bbase[blk] + win_starts_before(flags32, blk, (int)(pos & 255));
        for (int q = 1; q < nsub; ++q) dst[q] = bbase[blk + q];  // cut at a block start: that block's first piece
    }
}

// The term kernel's program with windows: hub row h keeps chunk tiles over [0, S[h][0]) and
// [S[h][NW], d) (tile tb[h] + j = its partial's slot); pack tiles follow unchanged.
template <class RPN>
__global__ void k_win_prog_hub(const RPN* __restrict__ rp, int64_t n_hub, const int* __restrict__ S, int NW,
                               const int* __restrict__ tb, int Sw, int len, WTile* __restrict__ prog) {
    const int lane = threadIdx.x & 31;
    const int64_t gw = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t h = gw; h < n_hub; h += nw) {
        const int64_t base = rp[h], d = rp[h + 1] - base;
        const int64_t sA = S[h * (NW + 1)], sC = S[h * (NW + 1) + NW];
        const int nA = (int)((sA + kWarpNnz - 1) / kWarpNnz);
        const int m = tb[h + 1] - tb[h];
        for (int j = lane; j < m; j += 32) {
            int64_t p, end;
            if (j < nA) {
                p = (int64_t)j * kWarpNnz;
                end = sA;
            } else {
                p = sC + (int64_t)(j - nA) * kWarpNnz;
                end = d;
            }
            WTile wt;
            wt.nnz_begin = base + p;
            wt.row_begin = tb[h] + j;
            wt.cnt = (uint16_t)(end - p < kWarpNnz ? end - p : kWarpNnz);
            wt.rows = 1;
            wt.meta = (uint8_t)kTileChunk;
            const int64_t t = (int64_t)tb[h] + j;
            prog[(size_t)(t % Sw) * len + t / Sw] = wt;
        }
    }
}

__global__ void k_win_prog_pack(const Tile* __restrict__ tiles, int old_chunks, int n_tiles_old, int MC, int Sw,
                                int len, WTile* __restrict__ prog) {
    for (int64_t t0 = old_chunks + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t0 < n_tiles_old;
         t0 += (int64_t)gridDim.x * blockDim.x) {
        const Tile a = tiles[t0], b = tiles[t0 + 1];
        WTile wt;
        wt.nnz_begin = a.nnz_begin;
        wt.row_begin = a.row_begin;
        wt.cnt = (uint16_t)(b.nnz_begin - a.nnz_begin);
        wt.rows = (uint8_t)(b.row_begin - a.row_begin);
        wt.meta = (uint8_t)a.meta;
        const int64_t t = (int64_t)MC + (t0 - old_chunks);
        prog[(size_t)(t % Sw) * len + t / Sw] = wt;
    }
}

// Scratch of the window build: one grow-only cudaMalloc'ed block per device, reused by every
// upload (callers hold pinned_arena().mu), so the temporaries never touch the memory pool.
static char* window_scratch(size_t bytes, int slot = 0) {
    static std::map<std::pair<int, int>, DevMem> cache;
    int dev = 0;
    CHEB_CUDA_CHECK(cudaGetDevice(&dev));
    DevMem& d = cache[{dev, slot}];
    if (d.bytes() < bytes) {
        AllocScope plain(nullptr);
        d.alloc(bytes + bytes / 8);
    }
    return d.ptr<char>();
}
struct Carver {
    char* base;
    size_t off = 0;
    template <class T>
    T* take(size_t count) {
        T* p = base ? reinterpret_cast<T*>(base + off) : nullptr;
        off += (count * sizeof(T) + 255) & ~size_t(255);
        return p;
    }
};

// Builds SolverView::Windows on the device (hub rows ascending).  NW windows of W entries
// from id H0 (0, or the fp64 hot-prefix capacity: tuning().winh0).
template <class RPN>
static void window_schedule(SolverView& V, int NW_req, int W, cudaStream_t st) {
    SolverView::Windows& Wn = V.win;
    Wn.release();
    const int64_t n_hub = V.n_hub;
    const int H0 = tuning().winh0 >= 0 ? (tuning().winh0 & ~7) : kHotBytes / 8;
    W = std::max(256, std::min(W, kWinMaxIds)) & ~7;
    if (n_hub <= 0 || V.x_len <= H0) return;
    const int NW = (int)std::min<int64_t>(NW_req, (V.x_len - H0 + W - 1) / W);
    if (NW <= 0 || n_hub * (int64_t)(NW + 1) >= (int64_t)INT32_MAX * 4) return;
    const RPN* rp = V.row_ptr.ptr<RPN>();
    const int* col = V.col.ptr<int>();
    const int64_t nq = n_hub * NW;
    const int64_t max_blocks = V.nnz_local / kWinBlock + NW + 1;
    constexpr size_t kCubTemp = size_t(64) << 20;
    // scratch layout (sizes first, then the block)
    Carver sc{nullptr};
    int* S = nullptr;
    int64_t *csz = nullptr, *off = nullptr, *d_small = nullptr;
    int *pc = nullptr, *mc = nullptr, *rowpieces = nullptr, *subx = nullptr;
    unsigned long long* wide = nullptr;
    char* cub_tmp = nullptr;
    for (int pass = 0; pass < 2; ++pass) {
        if (pass == 1) {
            // the build's scratch + the view's arrays (~the same again) must leave the solver room:
            // otherwise the view keeps the plain schedule
            size_t free_b = 0, total_b = 0;
            if (cudaMemGetInfo(&free_b, &total_b) != cudaSuccess || 2 * sc.off > free_b / 2) return;
            sc = Carver{window_scratch(sc.off)};
        }
        S = sc.take<int>((size_t)n_hub * (NW + 1));
        csz = sc.take<int64_t>((size_t)nq + 1);
        off = sc.take<int64_t>((size_t)nq + 1);
        d_small = sc.take<int64_t>((size_t)4 * (NW + 1));
        pc = sc.take<int>((size_t)max_blocks + 1);
        mc = sc.take<int>((size_t)n_hub + 1);
        rowpieces = sc.take<int>((size_t)n_hub + 1);
        subx = sc.take<int>((size_t)nq);
        wide = sc.take<unsigned long long>(1);
        cub_tmp = sc.take<char>(kCubTemp);
    }
    auto scan = [&](auto* in, auto* out, int64_t cnt) {
        size_t bytes = 0;
        CHEB_CUDA_CHECK(cub::DeviceScan::ExclusiveSum(nullptr, bytes, in, out, cnt, st));
        if (bytes > kCubTemp) fail(CHEB_CAPACITY, "window build: scan scratch");
        CHEB_CUDA_CHECK(cub::DeviceScan::ExclusiveSum(cub_tmp, bytes, in, out, cnt, st));
    };
    k_win_splits<RPN><<<grid_for(n_hub * (NW + 1)), kBuildThreads, 0, st>>>(rp, col, n_hub, H0, W, NW, S);
    k_win_sizes<<<grid_for(nq + 1), kBuildThreads, 0, st>>>(S, n_hub, NW, csz);
    CHEB_CUDA_CHECK(cudaGetLastError());
    scan(csz, off, nq + 1);
    int64_t* d_starts = d_small;                        // [NW + 1] unpadded window starts
    int64_t* d_delta = d_starts + (NW + 1);             // [NW]
    int64_t* d_wend = d_delta + (NW + 1);               // [NW]
    int64_t* d_wblk = d_wend + (NW + 1);                // [NW + 1]
    k_win_gather_starts<<<(NW + 1 + 127) / 128, 128, 0, st>>>(off, n_hub, NW, d_starts);
    CHEB_CUDA_CHECK(cudaGetLastError());
    std::vector<int64_t> hs((size_t)4 * (NW + 1), 0);
    CHEB_CUDA_CHECK(cudaMemcpyAsync(hs.data(), d_starts, sizeof(int64_t) * (NW + 1), cudaMemcpyDeviceToHost, st));
    CHEB_CUDA_CHECK(cudaStreamSynchronize(st));
    int64_t* h_delta = hs.data() + (NW + 1);
    int64_t* h_wend = h_delta + (NW + 1);
    int64_t* h_wblk = h_wend + (NW + 1);
    int64_t cur = 0;
    for (int w = 0; w < NW; ++w) {
        const int64_t len = hs[(size_t)w + 1] - hs[(size_t)w];
        h_delta[w] = cur - hs[(size_t)w];
        h_wend[w] = cur + len;
        h_wblk[w] = cur / kWinBlock;
        cur = (cur + len + kWinBlock - 1) / kWinBlock * kWinBlock;
    }
    h_wblk[NW] = cur / kWinBlock;
    const int64_t entries = hs[(size_t)NW], stream_len = cur, n_blocks = cur / kWinBlock;
    if (entries == 0 || n_blocks >= INT32_MAX / 2 || n_blocks > max_blocks) return;
    CHEB_CUDA_CHECK(cudaMemcpyAsync(d_delta, h_delta, sizeof(int64_t) * 3 * (NW + 1), cudaMemcpyHostToDevice, st));
    // the view's own arrays, first allocation
    Wn.grid = (int)std::max<int64_t>(1, std::min<int64_t>(V.grid, n_blocks));
    Carver ca{nullptr};
    for (int pass = 0; pass < 2; ++pass) {
        if (pass == 1) {
            window_arena_take(Wn.arena_a, ca.off);
            ca = Carver{Wn.arena_a.ptr<char>()};
        }
        Wn.wcol.p = ca.take<unsigned short>((size_t)stream_len + 32);
        Wn.flags.p = ca.take<unsigned char>((size_t)stream_len / 8 + 64);
        Wn.meta.p = ca.take<unsigned short>((size_t)n_blocks * 32 + 32);
        Wn.bbase.p = ca.take<int>((size_t)n_blocks + 1);
        Wn.cta.p = ca.take<int64_t>((size_t)Wn.grid + 1);
        Wn.wblk.p = ca.take<int64_t>((size_t)NW + 1);
        Wn.hub_first.p = ca.take<int>((size_t)n_hub + 1);
        Wn.kf.p = ca.take<int>((size_t)n_hub + 1);
    }
    CHEB_CUDA_CHECK(cudaMemsetAsync(Wn.wcol.get(), 0, sizeof(unsigned short) * ((size_t)stream_len + 32), st));
    CHEB_CUDA_CHECK(cudaMemsetAsync(Wn.flags.get(), 0, (size_t)stream_len / 8 + 64, st));
    unsigned* flags32 = Wn.flags.ptr<unsigned>();
    if (dbg_on()) {
        CHEB_CUDA_CHECK(cudaStreamSynchronize(st));
        dbg_mark("    windows: splits + layout");
    }
    k_win_copy<RPN, true><<<(int)std::min<int64_t>(n_hub, kWinBigRows), 512, 0, st>>>(
        rp, col, n_hub, S, off, d_delta, H0, W, NW, Wn.wcol.ptr<unsigned short>(), flags32);
    k_win_copy<RPN, false><<<(int)std::min<int64_t>((n_hub * 32 + 255) / 256, 148 * 16), 256, 0, st>>>(
        rp, col, n_hub, S, off, d_delta, H0, W, NW, Wn.wcol.ptr<unsigned short>(), flags32);
    k_win_padflags<<<(NW + 127) / 128, 128, 0, st>>>(d_wend, NW, flags32);
    CHEB_CUDA_CHECK(cudaGetLastError());
    if (dbg_on()) {
        CHEB_CUDA_CHECK(cudaStreamSynchronize(st));
        dbg_mark("    windows: stream copied");
    }
    if (tuning().winbank)
        k_win_bank_order<<<(int)std::min<int64_t>((n_blocks + kBankBlocks - 1) / kBankBlocks, 148 * 32), kBankThreads, 0, st>>>(
            Wn.wcol.ptr<unsigned short>(), flags32, n_blocks);
    if (dbg_on()) {
        CHEB_CUDA_CHECK(cudaStreamSynchronize(st));
        dbg_mark("    windows: bank order");
    }
    k_win_lanemeta<<<(int)std::min<int64_t>((n_blocks * 32 + 255) / 256, 148 * 16), 256, 0, st>>>(
        Wn.flags.ptr<unsigned char>(), n_blocks, Wn.meta.ptr<unsigned short>());
    k_win_blockcount<<<grid_for(n_blocks + 1), kBuildThreads, 0, st>>>(flags32, n_blocks, pc);
    CHEB_CUDA_CHECK(cudaGetLastError());
    scan(pc, Wn.bbase.ptr<int>(), n_blocks + 1);
    k_win_cta_starts<<<(Wn.grid + 1 + 127) / 128, 128, 0, st>>>(Wn.bbase.ptr<int>(), n_blocks, tuning().winpw, Wn.grid,
                                                             Wn.cta.ptr<int64_t>());
    CHEB_CUDA_CHECK(cudaMemsetAsync(wide, 0, sizeof(unsigned long long), st));
    constexpr int kWideMin = 128;  // more partials than this: a warp per row in k_hub_finalize
    k_win_rows<RPN><<<grid_for(n_hub + 1), kBuildThreads, 0, st>>>(rp, n_hub, S, off, d_delta, NW, kWideMin,
                                                                  (tuning().winskip & 32) ? 1 : 0,  // timing experiment: the rows' cold tails dropped (wrong results)
                                                                  mc, rowpieces,
                                                                  subx, wide);
    CHEB_CUDA_CHECK(cudaGetLastError());
    int* tb = Wn.hub_first.ptr<int>();  // first main chunk tile (= slot) of each hub row
    scan(mc, tb, n_hub + 1);
    scan(rowpieces, Wn.kf.ptr<int>(), n_hub + 1);
    int h_tot[3] = {0, 0, 0};
    unsigned long long h_wide = 0;
    CHEB_CUDA_CHECK(cudaMemcpyAsync(&h_tot[0], Wn.bbase.ptr<int>() + n_blocks, sizeof(int), cudaMemcpyDeviceToHost, st));
    CHEB_CUDA_CHECK(cudaMemcpyAsync(&h_tot[1], tb + n_hub, sizeof(int), cudaMemcpyDeviceToHost, st));
    CHEB_CUDA_CHECK(cudaMemcpyAsync(&h_tot[2], Wn.kf.ptr<int>() + n_hub, sizeof(int), cudaMemcpyDeviceToHost, st));
    CHEB_CUDA_CHECK(cudaMemcpyAsync(&h_wide, wide, sizeof h_wide, cudaMemcpyDeviceToHost, st));
    CHEB_CUDA_CHECK(cudaStreamSynchronize(st));
    const int pieces = h_tot[0], MC = h_tot[1], listed = h_tot[2];  // pieces = listed + the padding's
    if ((int64_t)MC + pieces >= INT32_MAX) fail(CHEB_CAPACITY, "too many hub partials");
    // second allocation: the rows' piece lists and the term kernel's program (main chunk
    // tiles, then the view's pack tiles)
    const int npack = V.n_tiles - V.n_chunk_tiles;
    if ((int64_t)MC + npack >= INT32_MAX) fail(CHEB_CAPACITY, "too many tiles");
    Wn.n_tiles = MC + npack;
    const int Sw = V.grid * kWarps;
    const int per = (Wn.n_tiles + Sw - 1) / Sw;
    Wn.prog_len = std::max(kDescBlock, (per + kDescBlock - 1) / kDescBlock * kDescBlock);
    const size_t np = (size_t)Sw * Wn.prog_len;
    Carver cb{nullptr};
    for (int pass = 0; pass < 2; ++pass) {
        if (pass == 1) {
            window_arena_take(Wn.arena_b, cb.off);
            cb = Carver{Wn.arena_b.ptr<char>()};
        }
        Wn.klist.p = cb.take<int>((size_t)std::max(listed, 1));
        Wn.prog.p = cb.take<WTile>(np);
    }
    k_win_klist<<<grid_for(nq), kBuildThreads, 0, st>>>(n_hub, S, off, d_delta, NW, flags32, Wn.bbase.ptr<int>(),
                                                     Wn.kf.ptr<int>(), subx, Wn.klist.ptr<int>());
    CHEB_CUDA_CHECK(cudaGetLastError());
    CHEB_CUDA_CHECK(cudaMemsetAsync(Wn.prog.get(), 0, sizeof(WTile) * np, st));
    k_win_prog_hub<RPN><<<(int)std::min<int64_t>((n_hub * 32 + 255) / 256, 148 * 16), 256, 0, st>>>(
        rp, n_hub, S, NW, tb, Sw, Wn.prog_len, Wn.prog.ptr<WTile>());
    if (npack > 0)
        k_win_prog_pack<<<grid_for(npack), kBuildThreads, 0, st>>>(V.tiles.ptr<Tile>(), V.n_chunk_tiles, V.n_tiles, MC, Sw,
                                                                 Wn.prog_len, Wn.prog.ptr<WTile>());
    CHEB_CUDA_CHECK(cudaGetLastError());
    CHEB_CUDA_CHECK(cudaMemcpyAsync(Wn.wblk.get(), d_wblk, sizeof(int64_t) * (NW + 1), cudaMemcpyDeviceToDevice, st));
    CHEB_CUDA_CHECK(cudaStreamSynchronize(st));
    (void)h_wblk;
    Wn.NW = NW;
    Wn.W = W;
    Wn.H0 = H0;
    Wn.n_blocks = n_blocks;
    Wn.n_slots = (int64_t)MC + pieces;
    Wn.MC = MC;
    Wn.n_wide = (int64_t)h_wide;
    Wn.entries = entries;
    Wn.pieces = pieces;
    Wn.ready = true;
    if (dbg_on())
        dbg_mark(("  view: column windows (" + std::to_string(NW) + " x " + std::to_string(W) + ": " +
                  std::to_string(entries) + " entries, " + std::to_string(pieces) + " pieces, " +
                  std::to_string(MC) + " main chunk tiles, wide rows " + std::to_string(h_wide) + ")").c_str());
}

// Each of the first `segs` view rows' renamed ids in ascending order (cub segmented sort,
// in place over V.col).
template <class RPN>
static void sort_rows_of(const SolverView& V, int* col, int64_t segs, int64_t items, cudaStream_t st) {
    if (segs <= 0 || items <= 0) return;
    TempStore tmp;
    const RPN* offs = V.row_ptr.ptr<RPN>();
    DevMem alt(sizeof(int) * (size_t)items + 64);
    cub::DoubleBuffer<int> db(col, alt.ptr<int>());
    size_t bytes = 0;
    CHEB_CUDA_CHECK(cub::DeviceSegmentedSort::SortKeys(nullptr, bytes, db, (int)items, (int)segs, offs, offs + 1, st));
    void* t = tmp.get(bytes);
    CHEB_CUDA_CHECK(cub::DeviceSegmentedSort::SortKeys(t, bytes, db, (int)items, (int)segs, offs, offs + 1, st));
    if (db.Current() != col)
        CHEB_CUDA_CHECK(cudaMemcpyAsync(col, db.Current(), sizeof(int) * items, cudaMemcpyDeviceToDevice, st));
    CHEB_CUDA_CHECK(cudaStreamSynchronize(st));
}
template <class RPN>
static void sort_view_rows_t(SolverView& V, int64_t segs, int64_t items, cudaStream_t st) {
    sort_rows_of<RPN>(V, V.col.ptr<int>(), segs, items, st);
}

template <class RPO, class RPN>
static void build_view_t(cheb_graph* g, cudaStream_t st, const std::function<void()>& before_col,
                         const ColGroups* groups) {
    SolverView& V = g->view;
    const int64_t n = g->n;
    TempStore tmp;
    const RPO* rp_old = g->row_ptr.ptr<RPO>();
    V.col_sorted.release();  // the batched path's sorted copy follows the view

    DevMem keys(sizeof(unsigned) * n), keys2(sizeof(unsigned) * n), ids(sizeof(int) * n);
    V.order.alloc(sizeof(int) * n);
    k_degree_keys<<<grid_for(n), kBuildThreads, 0, st>>>(rp_old, n, keys.ptr<unsigned>(), ids.ptr<int>());
    CHEB_CUDA_CHECK(cudaGetLastError());
    {
        size_t bytes = 0;
        CHEB_CUDA_CHECK(cub::DeviceRadixSort::SortPairs(nullptr, bytes, keys.ptr<unsigned>(), keys2.ptr<unsigned>(),
                                                        ids.ptr<int>(), V.order.ptr<int>(), n, 0, 32, st));
        void* t = tmp.get(bytes);
        CHEB_CUDA_CHECK(cub::DeviceRadixSort::SortPairs(t, bytes, keys.ptr<unsigned>(), keys2.ptr<unsigned>(),
                                                        ids.ptr<int>(), V.order.ptr<int>(), n, 0, 32, st));
    }
    dbg_mark("  view: sort enqueued");
    DevMem rank(sizeof(int) * n);
    k_scatter_rank<<<grid_for(n), kBuildThreads, 0, st>>>(V.order.ptr<int>(), n, rank.ptr<int>());
    DevMem deg_new(sizeof(int64_t) * (n + 1));
    CHEB_CUDA_CHECK(cudaMemsetAsync(deg_new.get(), 0, sizeof(int64_t) * (n + 1), st));
    k_new_degrees<<<grid_for(n), kBuildThreads, 0, st>>>(rp_old, V.order.ptr<int>(), n, deg_new.ptr<int64_t>());
    CHEB_CUDA_CHECK(cudaGetLastError());

    // Row partition over G ranks (block-cyclic snake order, common.cuh): this
    // rank keeps its sorted rows (local row i = sorted row part_global(i, rank, G)); column
    // ids stay the global sorted ids.
    Partition& P = g->part;
    const int* colmap = rank.ptr<int>();
    DevMem deg_loc;  // this rank's row degrees (G > 1)
    const int64_t* deg_l = deg_new.ptr<int64_t>();
    if (P.G > 1) {
        P.rows = part_rows(n, P.G);
        P.max_rows = *std::max_element(P.rows.begin(), P.rows.end());
        const int64_t nloc = P.rows[(size_t)P.rank];
        V.order_full = std::move(V.order);
        V.order.alloc(sizeof(int) * (size_t)std::max<int64_t>(nloc, 1));
        deg_loc.alloc(sizeof(int64_t) * (size_t)(nloc + 1));
        CHEB_CUDA_CHECK(cudaMemsetAsync(deg_loc.get(), 0, sizeof(int64_t) * (nloc + 1), st));
        if (nloc > 0)
            k_gather_local<<<grid_for(nloc), kBuildThreads, 0, st>>>(V.order_full.ptr<int>(), deg_new.ptr<int64_t>(),
                                                                      nloc, P.rank, P.G, V.order.ptr<int>(),
                                                                      deg_loc.ptr<int64_t>());
        CHEB_CUDA_CHECK(cudaGetLastError());
        deg_l = deg_loc.ptr<int64_t>();
    } else {
        P.rows = {n};
        P.max_rows = n;
    }
    const int64_t nl = P.rows[(size_t)P.rank];
    V.n_local = nl;
    V.x_len = n;
    V.part_G = P.G;
    V.part_r = P.rank;
    const int64_t lo = 0;

    DevMem rp64(sizeof(int64_t) * (nl + 1));
    {
        // scan nl+1 entries of a copy with a zero tail
        DevMem dl(sizeof(int64_t) * (nl + 1));
        CHEB_CUDA_CHECK(cudaMemsetAsync(dl.get(), 0, sizeof(int64_t) * (nl + 1), st));
        if (nl > 0)
            CHEB_CUDA_CHECK(cudaMemcpyAsync(dl.get(), deg_l, sizeof(int64_t) * nl, cudaMemcpyDeviceToDevice, st));
        size_t bytes = 0;
        CHEB_CUDA_CHECK(cub::DeviceScan::ExclusiveSum(nullptr, bytes, dl.ptr<int64_t>(), rp64.ptr<int64_t>(), nl + 1, st));
        void* t = tmp.get(bytes);
        CHEB_CUDA_CHECK(cub::DeviceScan::ExclusiveSum(t, bytes, dl.ptr<int64_t>(), rp64.ptr<int64_t>(), nl + 1, st));
        CHEB_CUDA_CHECK(cudaStreamSynchronize(st));
    }
    dbg_mark("  view: scan synced");
    const int64_t nnz_l = nl > 0 ? read_scalar(rp64.ptr<int64_t>() + nl, st) : 0;
    dbg_mark("  view: nnz read");
    V.nnz_local = nnz_l;
    V.rp64 = sizeof(RPN) == 8;
    if (V.rp64) {
        V.row_ptr = std::move(rp64);
    } else {
        V.row_ptr.alloc(sizeof(int) * (nl + 1));
        k_narrow_rowptr<<<grid_for(nl + 1), kBuildThreads, 0, st>>>(rp64.ptr<int64_t>(), nl + 1, V.row_ptr.ptr<int>());
    }
    // Runs of equal degree (descending) -> greedy tiles on the host
    // (degree-only: overlaps the neighbour upload when built from upload_csr).
    std::lock_guard<std::mutex> staging_lock(pinned_arena().mu);
    std::vector<int64_t> run_deg, run_cnt;
    if (nl > 0) {
        DevMem uniq(sizeof(int64_t) * nl), cnts(sizeof(int64_t) * nl), nruns(sizeof(int64_t));
        size_t bytes = 0;
        CHEB_CUDA_CHECK(cub::DeviceRunLengthEncode::Encode(nullptr, bytes, deg_l, uniq.ptr<int64_t>(),
                                                           cnts.ptr<int64_t>(), nruns.ptr<int64_t>(), nl, st));
        void* t = tmp.get(bytes);
        CHEB_CUDA_CHECK(cub::DeviceRunLengthEncode::Encode(t, bytes, deg_l, uniq.ptr<int64_t>(),
                                                           cnts.ptr<int64_t>(), nruns.ptr<int64_t>(), nl, st));
        const int64_t R = read_scalar(nruns.ptr<int64_t>(), st);
        run_deg.resize(R);
        run_cnt.resize(R);
        auto* hd = static_cast<int64_t*>(pinned_arena().get(3, sizeof(int64_t) * R));
        auto* hc = static_cast<int64_t*>(pinned_arena().get(4, sizeof(int64_t) * R));
        CHEB_CUDA_CHECK(cudaMemcpyAsync(hd, uniq.get(), sizeof(int64_t) * R, cudaMemcpyDeviceToHost, st));
        CHEB_CUDA_CHECK(cudaMemcpyAsync(hc, cnts.get(), sizeof(int64_t) * R, cudaMemcpyDeviceToHost, st));
        CHEB_CUDA_CHECK(cudaStreamSynchronize(st));
        std::memcpy(run_deg.data(), hd, sizeof(int64_t) * R);
        std::memcpy(run_cnt.data(), hc, sizeof(int64_t) * R);
    }
    dbg_mark("  view: runs read");
    {
        const std::vector<TileSeg> segs = make_tile_segs(run_deg, run_cnt, nl, nnz_l, V);
        int dev = 0, sms = 148;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        V.grid = std::max(1, std::min(sms, (V.n_tiles + kWarps - 1) / kWarps));
        DevMem d_segs(sizeof(TileSeg) * std::max<size_t>(segs.size(), 1));
        if (!segs.empty()) h2d_staged(d_segs.get(), segs.data(), sizeof(TileSeg) * segs.size(), 0, st);
        V.tiles.alloc(sizeof(Tile) * ((size_t)V.n_tiles + 1));
        V.hub_first.alloc(sizeof(int) * ((size_t)V.n_hub + 1));
        k_expand_tiles<<<grid_for((int64_t)V.n_tiles + 1), kBuildThreads, 0, st>>>(
            d_segs.ptr<TileSeg>(), (int)segs.size(), V.n_tiles, nnz_l, (int32_t)nl, (int)V.n_hub, V.n_chunk_tiles,
            V.tiles.ptr<Tile>(), V.hub_first.ptr<int>());
        CHEB_CUDA_CHECK(cudaGetLastError());
        const int S = V.grid * kWarps;
        const int per = (V.n_tiles + S - 1) / S;
        V.prog_len = std::max(kDescBlock, (per + kDescBlock - 1) / kDescBlock * kDescBlock);
        const size_t np = (size_t)S * V.prog_len;
        V.prog.alloc(sizeof(WTile) * np);
        CHEB_CUDA_CHECK(cudaMemsetAsync(V.prog.get(), 0, sizeof(WTile) * np, st));
        if (V.n_tiles > 0)
            k_build_program<<<grid_for(V.n_tiles), kBuildThreads, 0, st>>>(V.tiles.ptr<Tile>(), V.n_tiles, S,
                                                                         V.prog_len, V.prog.ptr<WTile>());
        CHEB_CUDA_CHECK(cudaGetLastError());
        V.phases.clear();
        if (dbg_on()) {
            CHEB_CUDA_CHECK(cudaStreamSynchronize(st));
            dbg_mark(("  view: tiles + programs on the device (" + std::to_string(segs.size()) + " segments, " +
                      std::to_string(V.n_tiles) + " tiles)").c_str());
        }
    }
    V.col.alloc(sizeof(int) * std::max<int64_t>(nnz_l, 1) + 64);  // TMA reads round up to 16 B
    // When x does not fit L2 (config 4), ascending renamed ids within each row: a row's
    // gathers then walk x in address order (DRAM page / sector locality; C4 4.49 -> 3.95
    // ms/term).  When x fits L2 the storage order is kept (sorting cost C2 ~1%).  The
    // FAST sums are re-associated either way; results stay within 1e-12.
    int l2 = 0;
    {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&l2, cudaDevAttrL2CacheSize, dev);
    }
    const bool big_x = tuning().sortrows < 0 ? ((int64_t)V.x_len * 8 > (int64_t)l2) : tuning().sortrows > 0;
    // column windows need the hub rows in ascending id order
    // (partitioned views too: x keeps the global ids on every rank, and a rank's window pass runs
    // behind the term barrier like its term kernel; auto: views of >= 48 M entries, where the
    // extra launch per term is paid back: config 2,
    // 19 M entries, runs 65 -> 74 us/term with windows, config 3 362 -> 297, config 4 3447 -> 2554)
    int n_windows = tuning().windows;
    if (n_windows < 0) n_windows = nnz_l >= (int64_t(48) << 20) ? (big_x ? 64 : 24) : 0;
    const bool want_windows = n_windows > 0 && V.n_hub > 0 && tuning().chunksched <= 1 &&
                              V.x_len > kHotBytes / 8 && nnz_l < INT32_MAX;
    const bool hubs_only = (tuning().sortrows == 2 || (want_windows && !big_x)) && V.n_hub > 0;
    const bool sort_rows = (big_x || hubs_only) && nnz_l > 0 && nnz_l < INT32_MAX;
    const bool sort_grouped = sort_rows && !hubs_only;  // every row, group by group into V.col
    V.sorted_rows = sort_grouped;
    if (nl > 0) {
        cudaEvent_t dbg_ev[2] = {};
        // rows are degree-descending: hub rows [0, n_hub) by chunk tiles (in bank-aware
        // order), then [n_hub, n_huge) > 1024 entries, [n_huge, n_long) > 16, the rest <= 16
        int64_t n_huge = V.n_hub, n_long = V.n_hub, seen = 0;
        for (size_t r = 0; r < run_deg.size(); ++r) {
            const int64_t r0 = seen, r1 = seen + run_cnt[r];
            seen = r1;
            if (r1 <= V.n_hub) continue;
            const int64_t c = r1 - std::max(r0, V.n_hub);
            if (run_deg[r] > 1024) n_huge += c;
            if (run_deg[r] > 16) n_long += c;
        }
        const int* order_l = V.order.ptr<int>() + lo;
        const RPN* rp_l = V.row_ptr.ptr<RPN>();
        // permute target when the rows are sorted afterwards (sorted into V.col), and the
        // segmented sort's scratch: from the build's grow-only blocks (the staging lock is held
        // and the build ends synchronised), not two more 4 GB pool allocations per upload
        int* perm = sort_grouped && tuning().bigscratch
                        ? reinterpret_cast<int*>(window_scratch(sizeof(int) * (size_t)nnz_l + 64, 1)) : nullptr;
        DevMem perm_pool;
        if (sort_grouped && !perm) {
            perm_pool.alloc(sizeof(int) * (size_t)nnz_l + 64);
            perm = perm_pool.ptr<int>();
        }
        int* dst = sort_grouped ? perm : V.col.ptr<int>();
        const int K = groups ? (int)groups->row_cut.size() - 1 : 1;
        DevMem seg_b, seg_e, seg_n(sizeof(unsigned long long));
        TempStore sort_tmp;
        if (sort_grouped && K > 1) {
            seg_b.alloc(sizeof(int64_t) * (size_t)nl);
            seg_e.alloc(sizeof(int64_t) * (size_t)nl);
        }
        if (before_col) before_col();
        if (dbg_on()) {
            cudaEventCreate(&dbg_ev[0]);
            cudaEventCreate(&dbg_ev[1]);
            cudaEventRecord(dbg_ev[0], st);
        }
        for (int gi = 0; gi < K; ++gi) {
            const int64_t oa = groups ? groups->row_cut[gi] : 0;
            const int64_t ob = groups ? groups->row_cut[gi + 1] : INT64_MAX;
            if (groups) CHEB_CUDA_CHECK(cudaStreamWaitEvent(st, groups->ready[gi], 0));
            if (V.n_chunk_tiles > 0)
                k_permute_chunks<RPO, RPN><<<std::max(1, std::min((V.n_chunk_tiles + 7) / 8, 148 * 16)), 256, 0, st>>>(
                    V.tiles.ptr<Tile>(), V.n_chunk_tiles, rp_old, g->col.ptr<int>(), rp_l, order_l, colmap,
                    kHotBytes / 8, tuning().chunksched, dst, oa, ob);
            if (n_huge > V.n_hub)
                k_permute_rows<0><<<(int)std::min<int64_t>(n_huge - V.n_hub, 148 * 16), kBuildThreads, 0, st>>>(
                    rp_old, g->col.ptr<int>(), rp_l, order_l, colmap, V.n_hub, n_huge, dst, oa, ob);
            if (n_long > n_huge)
                k_permute_rows<32><<<grid_for((n_long - n_huge) * 32), kBuildThreads, 0, st>>>(
                    rp_old, g->col.ptr<int>(), rp_l, order_l, colmap, n_huge, n_long, dst, oa, ob);
            if (nl > n_long)
                k_permute_rows<4><<<grid_for((nl - n_long) * 4), kBuildThreads, 0, st>>>(
                    rp_old, g->col.ptr<int>(), rp_l, order_l, colmap, n_long, nl, dst, oa, ob);
            CHEB_CUDA_CHECK(cudaGetLastError());
            if (!sort_grouped) continue;
            // this group's rows, ascending ids, from the permute target into V.col
            size_t bytes = 0;
            if (K == 1) {
                CHEB_CUDA_CHECK(cub::DeviceSegmentedSort::SortKeys(nullptr, bytes, dst, V.col.ptr<int>(), (int)nnz_l,
                                                                   (int)nl, rp_l, rp_l + 1, st));
                void* t = tuning().bigscratch ? (void*)window_scratch(bytes, 2) : sort_tmp.get(bytes);
                CHEB_CUDA_CHECK(cub::DeviceSegmentedSort::SortKeys(t, bytes, dst, V.col.ptr<int>(), (int)nnz_l,
                                                                   (int)nl, rp_l, rp_l + 1, st));
            } else {
                CHEB_CUDA_CHECK(cudaMemsetAsync(seg_n.get(), 0, sizeof(unsigned long long), st));
                k_group_segments<RPN><<<grid_for(nl), kBuildThreads, 0, st>>>(order_l, rp_l, nl, oa, ob,
                                                                            seg_b.ptr<int64_t>(), seg_e.ptr<int64_t>(),
                                                                            seg_n.ptr<unsigned long long>());
                CHEB_CUDA_CHECK(cudaGetLastError());
                const int64_t nseg = (int64_t)read_scalar(seg_n.ptr<unsigned long long>(), st);
                if (nseg == 0) continue;
                CHEB_CUDA_CHECK(cub::DeviceSegmentedSort::SortKeys(nullptr, bytes, dst, V.col.ptr<int>(), (int)nnz_l,
                                                                   (int)nseg, seg_b.ptr<int64_t>(), seg_e.ptr<int64_t>(), st));
                void* t = tuning().bigscratch ? (void*)window_scratch(bytes, 2) : sort_tmp.get(bytes);
                CHEB_CUDA_CHECK(cub::DeviceSegmentedSort::SortKeys(t, bytes, dst, V.col.ptr<int>(), (int)nnz_l,
                                                                   (int)nseg, seg_b.ptr<int64_t>(), seg_e.ptr<int64_t>(), st));
            }
        }
        if (dbg_ev[0]) {  // CHEB_DEBUG_UPLOAD: neighbours landed + narrowed, then permuted (+ sorted)
            cudaEventRecord(dbg_ev[1], st);
            cudaEventSynchronize(dbg_ev[1]);
            float ms = 0.f;
            cudaEventElapsedTime(&ms, dbg_ev[0], dbg_ev[1]);
            dbg_mark(("  view: columns permuted/sorted (" + std::to_string(K) + " groups, " + std::to_string(ms) +
                      " ms after the first)").c_str());
            cudaEventDestroy(dbg_ev[0]);
            cudaEventDestroy(dbg_ev[1]);
        }
        if (sort_rows && hubs_only) {  // experiment: the hub rows only, in place
            const int64_t segs = V.n_hub;
            const int64_t items = (int64_t)read_scalar(V.row_ptr.ptr<RPN>() + segs, st);
            sort_view_rows_t<RPN>(V, segs, items, st);
        }
        if (sort_grouped && V.n_hub > 0 && tuning().colblocks > 1) {  // opt-in: measured no gain on C4
            CHEB_CUDA_CHECK(cudaStreamSynchronize(st));
            column_block_schedule<RPN>(V, tuning().colblocks, V.x_len, st);
            dbg_mark("  view: column-block schedule");
        }
        V.win.release();
        if (want_windows && sort_rows) {
            window_schedule<RPN>(V, n_windows, tuning().winsize, st);
            dbg_mark("  view: column windows");
        }
        if (sort_grouped && tuning().chunksched > 1 && V.n_chunk_tiles > 0) {  // the sort undid the chunk order
            k_schedule_chunks_inplace<RPN><<<std::max(1, std::min((V.n_chunk_tiles + 7) / 8, 148 * 16)), 256, 0, st>>>(
                V.tiles.ptr<Tile>(), V.n_chunk_tiles, kHotBytes / 8, V.col.ptr<int>());
            CHEB_CUDA_CHECK(cudaGetLastError());
        }
        CHEB_CUDA_CHECK(cudaStreamSynchronize(st));
        if (tuning().packsched && V.n_tiles > V.n_chunk_tiles) {
            const int jobs = 2 * (V.n_tiles - V.n_chunk_tiles);
            k_schedule_pack<RPN><<<std::max(1, std::min((jobs + 127) / 128, 148 * 8)), 128, 0, st>>>(
                V.tiles.ptr<Tile>(), V.n_chunk_tiles, V.n_tiles, V.row_ptr.ptr<RPN>(), kHotBytes / 8, V.col.ptr<int>());
            CHEB_CUDA_CHECK(cudaGetLastError());
        }
    }
    if (P.G > 1 && nl > 0) {
        if (P.G > 32) fail(CHEB_CAPACITY, "halo masks support at most 32 ranks");
        V.push_mask.alloc(sizeof(unsigned) * nl);
        DevMem cnt(sizeof(unsigned long long));
        CHEB_CUDA_CHECK(cudaMemsetAsync(cnt.get(), 0, sizeof(unsigned long long), st));
        k_push_mask<RPN><<<(int)std::min<int64_t>((nl * 32 + 255) / 256, 148 * 16), 256, 0, st>>>(
            V.row_ptr.ptr<RPN>(), V.col.ptr<int>(), nl, P.G, P.rank, V.push_mask.ptr<unsigned>(),
            cnt.ptr<unsigned long long>());
        CHEB_CUDA_CHECK(cudaGetLastError());
        unsigned long long c = 0;
        CHEB_CUDA_CHECK(cudaMemcpyAsync(&c, cnt.get(), sizeof c, cudaMemcpyDeviceToHost, st));
        CHEB_CUDA_CHECK(cudaStreamSynchronize(st));
        V.push_entries = (int64_t)c;
        V.push_entries_all = nl * (int64_t)(P.G - 1);
    } else {
        V.push_mask.release();
        V.push_entries = V.push_entries_all = 0;
    }
    if (g->inv_array) {
        V.inv.alloc(sizeof(double) * std::max<int64_t>(nl, 1));
        if (nl > 0)
            k_gather_inv<<<grid_for(nl), kBuildThreads, 0, st>>>(g->inv.ptr<double>(), V.order.ptr<int>() + lo, nl,
                                                                 V.inv.ptr<double>());
    } else {
        V.inv.release();
    }

    if (P.G == 1) V.rank = std::move(rank);  // k_normalize gathers acc[rank[v]] (coalesced writes)
    else V.rank.release();
    dbg_mark("  view: tiles staged");
    V.ready = true;
    CHEB_CUDA_CHECK(cudaStreamSynchronize(st));
    dbg_mark("  view: synced");
}

// The batched path's own ascending-id copy of the view's columns (same rows, tiles and row
// pointers), so that a batched solve never changes the scalar FAST schedule's bits.
const int* batch_sorted_cols(cheb_graph* g) {
    ensure_view(g);
    SolverView& V = g->view;
    if (V.sorted_rows || V.n_local == 0 || V.nnz_local >= INT32_MAX) return V.col.ptr<int>();
    if (!V.col_sorted) {
        V.col_sorted.alloc(sizeof(int) * (size_t)V.nnz_local + 64);
        CHEB_CUDA_CHECK(cudaMemcpyAsync(V.col_sorted.get(), V.col.get(), sizeof(int) * (size_t)V.nnz_local,
                                        cudaMemcpyDeviceToDevice, g->stream));
        if (V.rp64) sort_rows_of<int64_t>(V, V.col_sorted.ptr<int>(), V.n_local, V.nnz_local, g->stream);
        else sort_rows_of<int>(V, V.col_sorted.ptr<int>(), V.n_local, V.nnz_local, g->stream);
    }
    return V.col_sorted.ptr<int>();
}

void ensure_view(cheb_graph* g) {
    if (g->view.ready) return;
    NvtxRange nvtx_("solver view build");
    if (g->rp64)
        build_view_t<int64_t, int64_t>(g, g->stream, nullptr);
    else
        build_view_t<int, int>(g, g->stream, nullptr);
}

}  // namespace chebgpu
