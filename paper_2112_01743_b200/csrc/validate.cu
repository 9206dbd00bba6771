// validate on the device: the reference's structural re-check of a host
// CSR, /root/reference/proj/src/graph.cpp:123-186, with the same check order and messages.
// The reference walks vertices in order and throws at the first failing check; here every
// vertex is checked in parallel and the first failure is found with a 64-bit atomicMin over
// (vertex, check) keys — the same vertex and the same message.  Symmetry (v in N(u) iff u in
// N(v), binary search in the sorted lists) keys failures by (u, position in N(u)).
#include <climits>
#include <string>

#include "common.cuh"

namespace chebgpu {
namespace {

enum VCode : int {
    kVMonotone = 1,   // "offsets not monotone at vertex v"
    kVDegree = 2,     // "degree mismatch at vertex v"
    kVIsolated = 3,   // "vertex v is isolated (degree 0)"
    kVRange = 4,      // "neighbor id out of range at vertex v"
    kVUnsorted = 5,   // "neighbor list not sorted at vertex v"
    kVDuplicate = 6,  // "duplicate neighbor at vertex v"
    kVLength = 7,     // row runs past the neighbour array (the reference reads out of bounds)
};

struct VOut {
    unsigned long long first_bad;  // v * 8 + code
    unsigned long long self_loops;
    unsigned long long entries;
    long long min_deg, max_deg;
};

// Warp per vertex: the vertex's first failing check in the reference's order.
__global__ void k_validate_vertices(const int64_t* __restrict__ off, const int64_t* __restrict__ nb, int64_t nnz,
                                    const int64_t* __restrict__ deg, int64_t n, int multi, VOut* out) {
    const int lane = threadIdx.x & 31;
    unsigned long long loops = 0, entries = 0;
    long long dmin = LLONG_MAX, dmax = 0;
    for (int64_t v = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; v < n;
         v += ((int64_t)gridDim.x * blockDim.x) >> 5) {
        const int64_t lo = off[v], hi = off[v + 1];
        int code = 0;
        if (hi < lo) code = kVMonotone;
        else if (hi - lo != deg[v]) code = kVDegree;
        else if (hi - lo < 1) code = kVIsolated;
        if (code) {
            if (lane == 0) atomicMin(&out->first_bad, (unsigned long long)v * 8 + code);
            continue;
        }
        const int64_t d = hi - lo;
        if (lane == 0) {
            entries += (unsigned long long)d;
            dmin = d < dmin ? d : dmin;
            dmax = d > dmax ? d : dmax;
        }
        if (hi > nnz) {
            if (lane == 0) atomicMin(&out->first_bad, (unsigned long long)v * 8 + kVLength);
            continue;
        }
        // first failing entry of the row: (position, check) minimised over the lanes
        unsigned long long best = ~0ull;
        for (int64_t i = lo + lane; i < hi; i += 32) {
            const int64_t w = nb[i];
            int c = 0;
            if (w < 0 || w >= n) c = kVRange;
            else if (i > lo) {
                const int64_t prev = nb[i - 1];
                if (w < prev) c = kVUnsorted;
                else if (!multi && w == prev) c = kVDuplicate;
            }
            if (c) {
                best = min(best, (unsigned long long)(i - lo) * 8 + c);
                break;  // later entries of this lane cannot come first
            }
            if (w == v) ++loops;
        }
        for (int o = 16; o; o >>= 1) best = min(best, __shfl_xor_sync(0xffffffffu, best, o));
        if (lane == 0 && best != ~0ull) atomicMin(&out->first_bad, (unsigned long long)v * 8 + (best & 7));
    }
    for (int o = 16; o; o >>= 1) {
        loops += __shfl_xor_sync(0xffffffffu, loops, o);
        entries += __shfl_xor_sync(0xffffffffu, entries, o);
        dmin = min(dmin, __shfl_xor_sync(0xffffffffu, dmin, o));
        dmax = max(dmax, __shfl_xor_sync(0xffffffffu, dmax, o));
    }
    if (lane == 0) {
        if (loops) atomicAdd(&out->self_loops, loops);
        if (entries) atomicAdd(&out->entries, entries);
        atomicMin(&out->min_deg, dmin);
        atomicMax(&out->max_deg, dmax);
    }
}

// Warp per vertex u: every entry v of N(u) must have u in N(v); first failure by (u, pos).
__global__ void k_validate_symmetry(const int64_t* __restrict__ off, const int64_t* __restrict__ nb, int64_t n,
                                    unsigned long long* __restrict__ first_missing) {
    const int lane = threadIdx.x & 31;
    for (int64_t u = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; u < n;
         u += ((int64_t)gridDim.x * blockDim.x) >> 5) {
        const int64_t lo = off[u], hi = off[u + 1];
        for (int64_t i = lo + lane; i < hi; i += 32) {
            const int64_t v = nb[i];
            int64_t a = off[v], b = off[v + 1];
            while (a < b) {  // first position in N(v) not less than u (std::binary_search)
                const int64_t mid = a + (b - a) / 2;
                if (nb[mid] < u) a = mid + 1;
                else b = mid;
            }
            if (a == off[v + 1] || nb[a] != u) {
                atomicMin(first_missing, ((unsigned long long)u << 32) | (unsigned long long)(i - lo));
                break;
            }
        }
    }
}

}  // namespace

void validate_csr(const int64_t* offsets, int64_t n_off, const int64_t* neighbors, int64_t nnz,
                  const int64_t* degrees, int64_t n_deg, int64_t n, int64_t m, int multi, int64_t dup_removed,
                  int64_t iso_dropped, int device, cheb_graph_stats* st) {
    // graph.cpp:125-130, host-side shape checks in the reference's order
    if (n < 0) fail(CHEB_VALIDATION, "negative vertex count");
    if (n_off != n + 1) fail(CHEB_VALIDATION, "offsets length is not n+1");
    if (offsets[0] != 0) fail(CHEB_VALIDATION, "offsets must start at 0");
    if (n_deg != n) fail(CHEB_VALIDATION, "degrees length is not n");
    DeviceGuard dg(device);
    cudaStream_t st_ = nullptr;
    CHEB_CUDA_CHECK(cudaStreamCreateWithFlags(&st_, cudaStreamNonBlocking));
    struct StreamFree {
        cudaStream_t s;
        ~StreamFree() {
            cudaStreamSynchronize(s);
            cudaStreamDestroy(s);
        }
    } sf{st_};
    AllocScope as(st_);
    DevMem d_off(sizeof(int64_t) * (n + 1)), d_nb(sizeof(int64_t) * (size_t)std::max<int64_t>(nnz, 1)),
        d_deg(sizeof(int64_t) * (size_t)std::max<int64_t>(n, 1)), d_out(sizeof(VOut)), d_sym(sizeof(unsigned long long));
    CHEB_CUDA_CHECK(cudaMemcpyAsync(d_off.get(), offsets, sizeof(int64_t) * (n + 1), cudaMemcpyHostToDevice, st_));
    if (nnz > 0)
        CHEB_CUDA_CHECK(cudaMemcpyAsync(d_nb.get(), neighbors, sizeof(int64_t) * nnz, cudaMemcpyHostToDevice, st_));
    if (n > 0) CHEB_CUDA_CHECK(cudaMemcpyAsync(d_deg.get(), degrees, sizeof(int64_t) * n, cudaMemcpyHostToDevice, st_));
    VOut init{~0ull, 0ull, 0ull, LLONG_MAX, 0};
    CHEB_CUDA_CHECK(cudaMemcpyAsync(d_out.get(), &init, sizeof init, cudaMemcpyHostToDevice, st_));
    const int blocks = (int)std::max<int64_t>(1, std::min<int64_t>((n * 32 + 255) / 256, 148 * 64));
    if (n > 0) {
        k_validate_vertices<<<blocks, 256, 0, st_>>>(d_off.ptr<int64_t>(), d_nb.ptr<int64_t>(), nnz,
                                                    d_deg.ptr<int64_t>(), n, multi, d_out.ptr<VOut>());
        CHEB_CUDA_CHECK(cudaGetLastError());
    }
    VOut r;
    CHEB_CUDA_CHECK(cudaMemcpyAsync(&r, d_out.get(), sizeof r, cudaMemcpyDeviceToHost, st_));
    CHEB_CUDA_CHECK(cudaStreamSynchronize(st_));
    if (r.first_bad != ~0ull) {  // graph.cpp:144-164
        const std::string v = std::to_string(r.first_bad / 8);
        switch ((int)(r.first_bad % 8)) {
            case kVMonotone: fail(CHEB_VALIDATION, "offsets not monotone at vertex " + v);
            case kVDegree: fail(CHEB_VALIDATION, "degree mismatch at vertex " + v);
            case kVIsolated: fail(CHEB_VALIDATION, "vertex " + v + " is isolated (degree 0)");
            case kVRange: fail(CHEB_VALIDATION, "neighbor id out of range at vertex " + v);
            case kVUnsorted: fail(CHEB_VALIDATION, "neighbor list not sorted at vertex " + v);
            case kVDuplicate: fail(CHEB_VALIDATION, "duplicate neighbor at vertex " + v);
            default: fail(CHEB_VALIDATION, "neighbors length inconsistent with offsets");
        }
    }
    if ((int64_t)r.entries != nnz) fail(CHEB_VALIDATION, "neighbors length inconsistent with offsets");  // :166
    if ((int64_t)r.entries != 2 * m - (int64_t)r.self_loops)                                            // :168
        fail(CHEB_VALIDATION, "edge count inconsistent with adjacency entries");
    if (n > 0) {  // :172-182
        CHEB_CUDA_CHECK(cudaMemsetAsync(d_sym.get(), 0xff, sizeof(unsigned long long), st_));
        k_validate_symmetry<<<blocks, 256, 0, st_>>>(d_off.ptr<int64_t>(), d_nb.ptr<int64_t>(), n,
                                                    d_sym.ptr<unsigned long long>());
        CHEB_CUDA_CHECK(cudaGetLastError());
        unsigned long long miss;
        CHEB_CUDA_CHECK(cudaMemcpyAsync(&miss, d_sym.get(), sizeof miss, cudaMemcpyDeviceToHost, st_));
        CHEB_CUDA_CHECK(cudaStreamSynchronize(st_));
        if (miss != ~0ull) {
            const int64_t u = (int64_t)(miss >> 32);
            const int64_t v = neighbors[offsets[u] + (int64_t)(miss & 0xffffffffull)];
            fail(CHEB_VALIDATION, "adjacency not symmetric: " + std::to_string(v) + " in N(" + std::to_string(u) +
                                      ") but not conversely");
        }
    }
    st->n = n;
    st->m = m;
    st->avg_degree = n > 0 ? static_cast<double>(m) / static_cast<double>(n) : 0.0;
    st->min_degree = n > 0 ? std::min<int64_t>(degrees[0], r.min_deg) : 0;  // graph.cpp:137
    st->max_degree = r.max_deg;
    st->self_loops = (int64_t)r.self_loops;
    st->duplicates_removed = dup_removed;  // the builder's record (graph.hpp:69-71)
    st->isolated_dropped = iso_dropped;
    st->lines = 0;
    st->weights_ignored = 0;
}

}  // namespace chebgpu
