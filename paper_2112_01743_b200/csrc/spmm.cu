// K5 — batched CPAA over R right-hand sides (personalised PageRank for R seeds at once).
//
// Same recurrence as run_cpaa (/root/reference/proj/src/cpaa.cpp:109-156) applied to an
// n x R block: T_{k+1} = 2 P T_k - T_{k-1}, acc += c_k T_{k+1}, started from T_0 = p
// (columns = personalisation vectors; the reference hard-codes p = ones, cpaa.cpp:88-92,
// so each column is a restated run with T_0 = p[:, r]; a positive scale of p cancels in
// the normalisation, Eq. 22).  Layout: row-major n x Rs (Rs = R rounded up to
// the lane vector width) in the degree-sorted view, so one CSR entry = one contiguous
// R-vector gather: each column index is loaded once and reused across all R columns.
// A warp walks the view's tiles; lane l owns columns [l*VPL, l*VPL+VPL).  Rows with
// degree > kWarpNnz are split into chunk tiles whose R-vector partials are combined in
// chunk order by k_spmm_hub_finalize (deterministic, no atomics).
#include <algorithm>
#include <cmath>
#include <cstring>
#include <string>

#include "common.cuh"
#include "device.cuh"

namespace chebgpu {

template <class RP, class V>
struct BatchArgs {
    const RP* __restrict__ rp;
    const int* __restrict__ col;
    const double* __restrict__ inv;
    const V* __restrict__ x_in;
    V* __restrict__ x_out;
    V* T;
    V* acc;
    double ck;
    int first;
    int R;    // live columns
    int Rs;   // row stride (>= R, multiple of VPL)
    double* part;      // [grid][2]
    double* hub_part;  // [n_tiles][Rs]
    double* hub_ts;    // [n_hub][2]
    int hub_rows;      // rows [0, hub_rows) of X are gathered under an L2 evict-last policy
    int xpol;          // x_{k+1} stores: 0 normal; 1 evict-last for the hub prefix, streaming for the rest
};

template <class V, int VPL>
struct VecIO;
template <>
struct VecIO<double, 1> {
    static __device__ __forceinline__ void ld(const double* p, double (&o)[1]) { o[0] = __ldg(p); }
};
template <>
struct VecIO<double, 2> {
    static __device__ __forceinline__ void ld(const double* p, double (&o)[2]) {
        const double2 v = __ldg(reinterpret_cast<const double2*>(p));
        o[0] = v.x;
        o[1] = v.y;
    }
};
template <>
struct VecIO<double, 4> {
    static __device__ __forceinline__ void ld(const double* p, double (&o)[4]) {
        const double2 a = __ldg(reinterpret_cast<const double2*>(p));
        const double2 b = __ldg(reinterpret_cast<const double2*>(p) + 1);
        o[0] = a.x;
        o[1] = a.y;
        o[2] = b.x;
        o[3] = b.y;
    }
};
template <>
struct VecIO<float, 1> {
    static __device__ __forceinline__ void ld(const float* p, float (&o)[1]) { o[0] = __ldg(p); }
};
template <>
struct VecIO<float, 2> {
    static __device__ __forceinline__ void ld(const float* p, float (&o)[2]) {
        const float2 v = __ldg(reinterpret_cast<const float2*>(p));
        o[0] = v.x;
        o[1] = v.y;
    }
};
template <>
struct VecIO<float, 4> {
    static __device__ __forceinline__ void ld(const float* p, float (&o)[4]) {
        const float4 v = __ldg(reinterpret_cast<const float4*>(p));
        o[0] = v.x;
        o[1] = v.y;
        o[2] = v.z;
        o[3] = v.w;
    }
};

// X-row gathers under an explicit L2 policy: the hub prefix of X (the most-gathered rows
// after the degree relabel, ~64 MB) evict-last, every other row evict-first, so the rows
// that are reused stay in L2 while the one-off rows and the streams pass through
// (config 5: 296 -> 282 ms/solve).
__device__ __forceinline__ uint64_t policy_evict_last() {
    uint64_t pol;
    asm("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
    return pol;
}
__device__ __forceinline__ void st_policy(double* p, double v, uint64_t pol) {
    asm volatile("st.global.L2::cache_hint.f64 [%0], %1, %2;" :: "l"(p), "d"(v), "l"(pol) : "memory");
}
__device__ __forceinline__ void st_policy(float* p, float v, uint64_t pol) {
    asm volatile("st.global.L2::cache_hint.f32 [%0], %1, %2;" :: "l"(p), "f"(v), "l"(pol) : "memory");
}
__device__ __forceinline__ uint64_t policy_evict_first() {
    uint64_t pol;
    asm("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
    return pol;
}
template <class V, int VPL>
struct PolicyIO;
template <>
struct PolicyIO<double, 1> {
    static __device__ __forceinline__ void ld(const double* p, double (&o)[1], uint64_t pol) {
        asm("ld.global.nc.L2::cache_hint.f64 %0, [%1], %2;" : "=d"(o[0]) : "l"(p), "l"(pol));
    }
};
template <>
struct PolicyIO<double, 2> {
    static __device__ __forceinline__ void ld(const double* p, double (&o)[2], uint64_t pol) {
        asm("ld.global.nc.L2::cache_hint.v2.f64 {%0, %1}, [%2], %3;" : "=d"(o[0]), "=d"(o[1]) : "l"(p), "l"(pol));
    }
};
template <>
struct PolicyIO<double, 4> {
    static __device__ __forceinline__ void ld(const double* p, double (&o)[4], uint64_t pol) {
        asm("ld.global.nc.L2::cache_hint.v2.f64 {%0, %1}, [%2], %3;" : "=d"(o[0]), "=d"(o[1]) : "l"(p), "l"(pol));
        asm("ld.global.nc.L2::cache_hint.v2.f64 {%0, %1}, [%2], %3;" : "=d"(o[2]), "=d"(o[3]) : "l"(p + 2), "l"(pol));
    }
};
template <>
struct PolicyIO<float, 1> {
    static __device__ __forceinline__ void ld(const float* p, float (&o)[1], uint64_t pol) {
        asm("ld.global.nc.L2::cache_hint.f32 %0, [%1], %2;" : "=f"(o[0]) : "l"(p), "l"(pol));
    }
};
template <>
struct PolicyIO<float, 2> {
    static __device__ __forceinline__ void ld(const float* p, float (&o)[2], uint64_t pol) {
        asm("ld.global.nc.L2::cache_hint.v2.f32 {%0, %1}, [%2], %3;" : "=f"(o[0]), "=f"(o[1]) : "l"(p), "l"(pol));
    }
};
template <>
struct PolicyIO<float, 4> {
    static __device__ __forceinline__ void ld(const float* p, float (&o)[4], uint64_t pol) {
        asm("ld.global.nc.L2::cache_hint.v4.f32 {%0, %1, %2, %3}, [%4], %5;"
            : "=f"(o[0]), "=f"(o[1]), "=f"(o[2]), "=f"(o[3]) : "l"(p), "l"(pol));
    }
};

#ifndef CHEB_SPMM_UNROLL
#define CHEB_SPMM_UNROLL 0  // 0: per storage type (below)
#endif
constexpr int kSpmmUnroll = CHEB_SPMM_UNROLL;
// Neighbour R-vectors in flight per lane.  Fewer than 8 keeps the kernel at 64 registers
// (4 CTAs of 8 warps per SM) once the row's T/acc loads are hoisted ahead of its gathers:
// C5 fp64 U = 8 / 5 / 4: 301.5 / 272 / 241 ms per solve, fp32 U = 8 / 5 / 4: 205 / 169 / 181
// (one B200, interleaved runs, tools/batch_time.py).
template <class V, int VPL>
__host__ __device__ constexpr int spmm_unroll() {
    return kSpmmUnroll > 0 ? (VPL >= 4 && kSpmmUnroll > 4 ? 4 : kSpmmUnroll) : (VPL >= 4 ? 4 : sizeof(V) == 8 ? 4 : 5);
}

// Sum over CSR entries [b, e) of the gathered R-vectors (lane's VPL columns), U entries
// (U column ids then U row gathers) in flight per lane.  Sums accumulate in fp64 whatever
// the storage type (fp32: one rounding per row and column).
template <class RP, class V, int VPL>
__device__ __forceinline__ void row_gather(const BatchArgs<RP, V>& a, int64_t b, int64_t e, int lane,
                                           bool live, double (&s)[VPL]) {
#pragma unroll
    for (int k = 0; k < VPL; ++k) s[k] = 0.0;
    const int off = lane * VPL;
    constexpr int U = spmm_unroll<V, VPL>();
    const uint64_t p_hub = policy_evict_last(), p_cold = policy_evict_first();
    int64_t j = b;
    for (; j + U - 1 < e; j += U) {
        int c[U];
#pragma unroll
        for (int q = 0; q < U; ++q) c[q] = __ldg(a.col + j + q);
        if (live) {
            V v[U][VPL];
#pragma unroll
            for (int q = 0; q < U; ++q)
                PolicyIO<V, VPL>::ld(a.x_in + (int64_t)c[q] * a.Rs + off, v[q], c[q] < a.hub_rows ? p_hub : p_cold);
            if constexpr (sizeof(V) == 8) {
#pragma unroll
                for (int q = 0; q < U; ++q)
#pragma unroll
                    for (int k = 0; k < VPL; ++k) s[k] += v[q][k];
            } else {  // fp32: the U entries in fp32, one fp32 -> fp64 conversion per U
#pragma unroll
                for (int k = 0; k < VPL; ++k) {
                    V blk = v[0][k];
#pragma unroll
                    for (int q = 1; q < U; ++q) blk += v[q][k];
                    s[k] += (double)blk;
                }
            }
        }
    }
    V tail[VPL];  // fp32: the < U remaining entries summed in fp32, converted once
#pragma unroll
    for (int k = 0; k < VPL; ++k) tail[k] = V(0);
    for (; j < e; ++j) {
        const int c0 = __ldg(a.col + j);
        if (live) {
            V v0[VPL];
            PolicyIO<V, VPL>::ld(a.x_in + (int64_t)c0 * a.Rs + off, v0, c0 < a.hub_rows ? p_hub : p_cold);
#pragma unroll
            for (int k = 0; k < VPL; ++k) {
                if constexpr (sizeof(V) == 8) s[k] += v0[k];
                else tail[k] += v0[k];
            }
        }
    }
    if constexpr (sizeof(V) == 4) {
#pragma unroll
        for (int k = 0; k < VPL; ++k) s[k] += (double)tail[k];
    }
}

// Streaming (evict-first) access to the T / acc blocks: each is touched once per term and
// re-read only a term or two later (GBs of traffic in between), so keeping them out of L2
// leaves room for the gathered x rows.  x_out (the next term's gather source) keeps the
// normal policy.
#ifndef CHEB_SPMM_HINTS
#define CHEB_SPMM_HINTS 1
#endif
template <class V, int VPL>
struct StreamIO {  // VPL values at p (aligned to VPL * sizeof(V))
    static __device__ __forceinline__ void ld(const V* p, V (&o)[VPL]) {
#pragma unroll
        for (int k = 0; k < VPL; ++k) o[k] = CHEB_SPMM_HINTS ? __ldcs(p + k) : p[k];
    }
    static __device__ __forceinline__ void st(V* p, const V (&v)[VPL], bool stream) {
#pragma unroll
        for (int k = 0; k < VPL; ++k) {
            if (CHEB_SPMM_HINTS && stream) __stcs(p + k, v[k]);
            else p[k] = v[k];
        }
    }
};
template <>
struct StreamIO<double, 2> {
    static __device__ __forceinline__ void ld(const double* p, double (&o)[2]) {
        const double2 v = CHEB_SPMM_HINTS ? __ldcs(reinterpret_cast<const double2*>(p))
                                          : *reinterpret_cast<const double2*>(p);
        o[0] = v.x;
        o[1] = v.y;
    }
    static __device__ __forceinline__ void st(double* p, const double (&v)[2], bool stream) {
        const double2 w = make_double2(v[0], v[1]);
        if (CHEB_SPMM_HINTS && stream) __stcs(reinterpret_cast<double2*>(p), w);
        else *reinterpret_cast<double2*>(p) = w;
    }
};
template <>
struct StreamIO<float, 2> {
    static __device__ __forceinline__ void ld(const float* p, float (&o)[2]) {
        const float2 v = CHEB_SPMM_HINTS ? __ldcs(reinterpret_cast<const float2*>(p))
                                         : *reinterpret_cast<const float2*>(p);
        o[0] = v.x;
        o[1] = v.y;
    }
    static __device__ __forceinline__ void st(float* p, const float (&v)[2], bool stream) {
        const float2 w = make_float2(v[0], v[1]);
        if (CHEB_SPMM_HINTS && stream) __stcs(reinterpret_cast<float2*>(p), w);
        else *reinterpret_cast<float2*>(p) = w;
    }
};
template <>
struct StreamIO<float, 4> {
    static __device__ __forceinline__ void ld(const float* p, float (&o)[4]) {
        const float4 v = CHEB_SPMM_HINTS ? __ldcs(reinterpret_cast<const float4*>(p))
                                         : *reinterpret_cast<const float4*>(p);
        o[0] = v.x;
        o[1] = v.y;
        o[2] = v.z;
        o[3] = v.w;
    }
    static __device__ __forceinline__ void st(float* p, const float (&v)[4], bool stream) {
        const float4 w = make_float4(v[0], v[1], v[2], v[3]);
        if (CHEB_SPMM_HINTS && stream) __stcs(reinterpret_cast<float4*>(p), w);
        else *reinterpret_cast<float4*>(p) = w;
    }
};

// Fused recurrence epilogue for (row u, the lane's columns).
// The row's T_{k-1} and acc values of the lane (loaded before its gathers, so the two
// streams overlap the gather latency instead of following it).
template <class RP, class V, int VPL>
struct RowPrev {
    V tp[VPL], ac[VPL];
};
template <class RP, class V, int VPL>
__device__ __forceinline__ void load_prev(const BatchArgs<RP, V>& a, int64_t u, int lane, RowPrev<RP, V, VPL>& o) {
    const int c0 = lane * VPL;
    if (c0 + VPL > a.R) return;  // partial lanes load inside the epilogue
    const int64_t i0 = u * a.Rs + c0;
    if (!a.first) StreamIO<V, VPL>::ld(a.T + i0, o.tp);
    StreamIO<V, VPL>::ld(a.acc + i0, o.ac);
}

template <class RP, class V, int VPL>
__device__ __forceinline__ void batch_epilogue(const BatchArgs<RP, V>& a, int64_t u, int64_t deg, int lane,
                                               const double (&s)[VPL], double& p0, double& p1,
                                               const RowPrev<RP, V, VPL>* pre = nullptr) {
    const V inv = a.inv ? (V)a.inv[u] : rcp_rn((V)deg);
    const int c0 = lane * VPL;
    const int64_t i0 = u * a.Rs + c0;
    if (c0 + VPL <= a.R) {  // all of the lane's columns live: vector I/O
        V tp[VPL], ac[VPL], t[VPL], na[VPL], xo[VPL];
        if (pre) {
#pragma unroll
            for (int k = 0; k < VPL; ++k) {
                tp[k] = pre->tp[k];
                ac[k] = pre->ac[k];
            }
        } else {
            if (!a.first) StreamIO<V, VPL>::ld(a.T + i0, tp);
            StreamIO<V, VPL>::ld(a.acc + i0, ac);
        }
#pragma unroll
        for (int k = 0; k < VPL; ++k) {
            t[k] = a.first ? (V)s[k] : sub_rn(mul_rn(V(2), (V)s[k]), tp[k]);
            na[k] = add_rn(ac[k], mul_rn((V)a.ck, t[k]));
            xo[k] = mul_rn(t[k], inv);
            p0 += (double)t[k];
            p1 += (double)na[k];
        }
        StreamIO<V, VPL>::st(a.T + i0, t, true);
        StreamIO<V, VPL>::st(a.acc + i0, na, true);
        if (a.xpol == 1 && u < a.hub_rows) {  // next term's most-gathered rows stay in L2
            const uint64_t pol = policy_evict_last();
#pragma unroll
            for (int k = 0; k < VPL; ++k) st_policy(a.x_out + i0 + k, xo[k], pol);
        } else {
            StreamIO<V, VPL>::st(a.x_out + i0, xo, a.xpol == 1);
        }
        return;
    }
#pragma unroll
    for (int k = 0; k < VPL; ++k) {
        const int c = c0 + k;
        if (c >= a.R) continue;
        const int64_t i = i0 + k;
        const V t = a.first ? (V)s[k] : sub_rn(mul_rn(V(2), (V)s[k]), a.T[i]);
        a.T[i] = t;
        const V nacc = add_rn(a.acc[i], mul_rn((V)a.ck, t));
        a.acc[i] = nacc;
        a.x_out[i] = mul_rn(t, inv);
        p0 += (double)t;
        p1 += (double)nacc;
    }
}

#ifndef CHEB_SPMM_MINB
#define CHEB_SPMM_MINB 1
#endif
template <class RP, class V, int VPL>
__global__ void __launch_bounds__(256, CHEB_SPMM_MINB) k_spmm_term(BatchArgs<RP, V> a, const Tile* __restrict__ tiles,
                                                   int ntiles) {
    __shared__ double red[2][8];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const bool live = lane * VPL < a.R;
    double p0 = 0.0, p1 = 0.0;
    const int gw = blockIdx.x * (blockDim.x >> 5) + warp;
    const int nw = gridDim.x * (blockDim.x >> 5);
    for (int t = gw; t < ntiles; t += nw) {
        const Tile tl = tiles[t], nx = tiles[t + 1];
        if (tl.meta & kTileChunk) {
            const int64_t z0 = tl.nnz_begin, z1 = nx.nnz_begin;
            double s[VPL];
            row_gather<RP, V, VPL>(a, z0, z1, lane, live, s);
#pragma unroll
            for (int k = 0; k < VPL; ++k)
                if (lane * VPL + k < a.Rs) a.hub_part[(int64_t)t * a.Rs + lane * VPL + k] = s[k];
        } else {
            int64_t e = tl.row_begin < nx.row_begin ? (int64_t)a.rp[tl.row_begin] : 0;
            for (int64_t u = tl.row_begin; u < nx.row_begin; ++u) {
                const int64_t b = e;
                e = a.rp[u + 1];
                RowPrev<RP, V, VPL> pre;
                if (live) load_prev<RP, V, VPL>(a, u, lane, pre);
                double s[VPL];
                row_gather<RP, V, VPL>(a, b, e, lane, live, s);
                if (live) batch_epilogue<RP, V, VPL>(a, u, e - b, lane, s, p0, p1, &pre);
            }
        }
    }
    p0 = warp_sum_all(p0);
    p1 = warp_sum_all(p1);
    if (lane == 0) {
        red[0][warp] = p0;
        red[1][warp] = p1;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        double q0 = 0.0, q1 = 0.0;
        for (int w = 0; w < (int)(blockDim.x >> 5); ++w) {
            q0 += red[0][w];
            q1 += red[1][w];
        }
        a.part[2 * blockIdx.x] = q0;
        a.part[2 * blockIdx.x + 1] = q1;
    }
}

// Hub rows: warp per row sums its chunk partials (chunk order) and runs the epilogue.
template <class RP, class V, int VPL>
__global__ void __launch_bounds__(256) k_spmm_hub_finalize(BatchArgs<RP, V> a, const int* __restrict__ hub_first,
                                                           int64_t n_hub) {
    const int lane = threadIdx.x & 31;
    const bool live = lane * VPL < a.R;
    for (int64_t h = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; h < n_hub;
         h += ((int64_t)gridDim.x * blockDim.x) >> 5) {
        const int f0 = hub_first[h], f1 = hub_first[h + 1];
        double s[VPL];
#pragma unroll
        for (int k = 0; k < VPL; ++k) s[k] = 0.0;
        if (live)
            for (int q = f0; q < f1; ++q)
#pragma unroll
                for (int k = 0; k < VPL; ++k) s[k] += a.hub_part[(int64_t)q * a.Rs + lane * VPL + k];
        double p0 = 0.0, p1 = 0.0;
        if (live) batch_epilogue<RP, V, VPL>(a, h, a.rp[h + 1] - a.rp[h], lane, s, p0, p1);
        p0 = warp_sum_all(p0);
        p1 = warp_sum_all(p1);
        if (lane == 0 && a.hub_ts) {
            a.hub_ts[2 * h] = p0;
            a.hub_ts[2 * h + 1] = p1;
        }
    }
}

// T_{-1} = T_0 = p (dense n x R host block, one-hot seeds, or ones), acc = (c0/2) T_0,
// x_0 = T_0 D^-1.  Padding columns (c >= R) are zero.
template <class RP, class V>
__global__ void k_spmm_init(const RP* __restrict__ rp, const double* __restrict__ inv,
                            const double* __restrict__ p, const int64_t* __restrict__ seed_new,
                            int64_t n, int R, int Rs, double half_c0, V* T0, V* T1, V* acc, V* x0,
                            const int* __restrict__ order) {
    const int64_t total = n * Rs;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
         i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t u = i / Rs;
        const int c = (int)(i - u * Rs);
        V t0 = V(0);
        if (c < R) {
            if (seed_new) t0 = seed_new[c] == u ? V(1) : V(0);
            else if (p) t0 = (V)p[(int64_t)order[u] * R + c];
            else t0 = V(1);
        }
        T0[i] = t0;
        T1[i] = t0;
        acc[i] = (p || seed_new) ? mul_rn((V)half_c0, t0) : (c < R ? (V)half_c0 : V(0));
        const V iv = inv ? (V)inv[u] : rcp_rn((V)(rp[u + 1] - rp[u]));
        x0[i] = mul_rn(t0, iv);
    }
}

// Column sums of acc (deterministic): block b sums rows [b*chunk, ...) per column.
template <class V>
__global__ void k_col_partial(const V* __restrict__ acc, int64_t n, int Rs, int64_t chunk,
                              double* __restrict__ part) {
    const int c = threadIdx.x;
    if (c >= Rs) return;
    const int64_t r0 = blockIdx.x * chunk, r1 = min(n, r0 + chunk);
    double s = 0.0;
    for (int64_t u = r0; u < r1; ++u) s += (double)acc[u * Rs + c];
    part[(int64_t)blockIdx.x * Rs + c] = s;
}

__global__ void k_col_final(const double* __restrict__ part, int nb, int Rs, double* __restrict__ tot) {
    const int c = threadIdx.x;
    if (c >= Rs) return;
    double s = 0.0;
    for (int b = 0; b < nb; ++b) s += part[(int64_t)b * Rs + c];
    tot[c] = s;
}

template <class V>
__global__ void k_spmm_normalize(const V* __restrict__ acc, const int* __restrict__ order, int64_t n, int R,
                                 int Rs, const double* __restrict__ tot, double* __restrict__ out) {
    const int64_t total = n * R;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
         i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t u = i / R;
        const int c = (int)(i - u * R);
        out[(int64_t)order[u] * R + c] = (double)acc[u * Rs + c] / tot[c];
    }
}

__global__ void k_seed_remap(const int64_t* __restrict__ seeds_old, const int* __restrict__ order, int64_t n,
                             int R, int64_t* __restrict__ seeds_new) {
    // seeds_new[r] = new id of old vertex seeds_old[r] (scan of order; R small)
    for (int64_t u = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; u < n;
         u += (int64_t)gridDim.x * blockDim.x)
        for (int r = 0; r < R; ++r)
            if (order[u] == seeds_old[r]) seeds_new[r] = u;
}

__global__ void k_trace_reduce_b(const double* __restrict__ part, int grid, const double* __restrict__ hub_ts,
                                 int64_t n_hub, double* __restrict__ out) {
    __shared__ double sh[2][32];
    double a = 0.0, b = 0.0;
    for (int i = threadIdx.x; i < grid; i += blockDim.x) {
        a += part[2 * i];
        b += part[2 * i + 1];
    }
    for (int64_t i = threadIdx.x; i < n_hub; i += blockDim.x) {
        a += hub_ts[2 * i];
        b += hub_ts[2 * i + 1];
    }
    a = warp_sum_all(a);
    b = warp_sum_all(b);
    if ((threadIdx.x & 31) == 0) {
        sh[0][threadIdx.x >> 5] = a;
        sh[1][threadIdx.x >> 5] = b;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        double x = 0.0, y = 0.0;
        for (int w = 0; w < (int)(blockDim.x >> 5); ++w) {
            x += sh[0][w];
            y += sh[1][w];
        }
        out[0] = x;
        out[1] = y;
    }
}

// ---------------------------------------------------------------------------------------
namespace {

inline int vpl_for(int R) { return R <= 32 ? 1 : (R <= 64 ? 2 : 4); }

template <class RP, class V, int VPL>
void batch_run(cheb_graph* g, const BatchSpec& s, std::vector<double>& trace, std::vector<double>& totals,
               std::vector<double>* term_ms) {
    cudaStream_t st = g->stream;
    SolverView& Vw = g->view;
    BatchWorkspace& w = g->bws;
    const int64_t n = g->n;
    const int R = s.R, Rs = ((R + VPL - 1) / VPL) * VPL;
    const size_t elems = (size_t)n * Rs;
    const int M = s.M;
    const int grid = 148 * 8;
    w.T0.ensure(sizeof(V) * elems);
    w.T1.ensure(sizeof(V) * elems);
    w.X0.ensure(sizeof(V) * elems);
    w.X1.ensure(sizeof(V) * elems);
    w.acc.ensure(sizeof(V) * elems);
    w.out.ensure(sizeof(double) * (size_t)n * R);
    w.part.ensure(sizeof(double) * 2 * grid);
    w.hub_part.ensure(sizeof(double) * (size_t)std::max(Vw.n_tiles, 1) * Rs);
    w.hub_ts.ensure(sizeof(double) * 2 * std::max<int64_t>(Vw.n_hub, 1));
    w.trace.ensure(sizeof(double) * 2 * std::max(M, 1));
    const int nb = (int)std::min<int64_t>(std::max<int64_t>(1, (n + 4095) / 4096), 4096);
    const int64_t chunk = (n + nb - 1) / nb;
    w.colpart.ensure(sizeof(double) * (size_t)nb * Rs);
    w.totals.ensure(sizeof(double) * Rs);

    std::vector<double> co;
    double beta_v, c0;
    coefficients(s.c, M, co, &beta_v, &c0);
    DevMem d_p, d_seed, d_seed_new;
    if (s.p) {
        d_p.alloc(sizeof(double) * (size_t)n * R);
        CHEB_CUDA_CHECK(cudaMemcpyAsync(d_p.get(), s.p, sizeof(double) * (size_t)n * R, cudaMemcpyHostToDevice, st));
    }
    if (s.seeds) {
        d_seed.alloc(sizeof(int64_t) * R);
        d_seed_new.alloc(sizeof(int64_t) * R);
        CHEB_CUDA_CHECK(cudaMemcpyAsync(d_seed.get(), s.seeds, sizeof(int64_t) * R, cudaMemcpyHostToDevice, st));
        CHEB_CUDA_CHECK(cudaMemsetAsync(d_seed_new.get(), 0xff, sizeof(int64_t) * R, st));
        k_seed_remap<<<1184, 256, 0, st>>>(d_seed.ptr<int64_t>(), Vw.order.ptr<int>(), n, R, d_seed_new.ptr<int64_t>());
        CHEB_CUDA_CHECK(cudaGetLastError());
    }
    const RP* rp = Vw.row_ptr.ptr<RP>();
    const double* inv = g->inv_array ? Vw.inv.ptr<double>() : nullptr;
    V* T[2] = {w.T0.ptr<V>(), w.T1.ptr<V>()};
    V* X[2] = {w.X0.ptr<V>(), w.X1.ptr<V>()};
    std::vector<cudaEvent_t> ev;
    if (term_ms) {
        ev.resize(2 * (size_t)std::max(M, 1));
        for (auto& e : ev) CHEB_CUDA_CHECK(cudaEventCreate(&e));
    }
    if (s.record_start) CHEB_CUDA_CHECK(cudaEventRecord(g->ev0, st));
    k_spmm_init<RP, V><<<1184, 256, 0, st>>>(rp, inv, d_p.ptr<double>(), d_seed_new.ptr<int64_t>(), n, R, Rs,
                                             c0 / 2.0, T[0], T[1], w.acc.ptr<V>(), X[0], Vw.order.ptr<int>());
    CHEB_CUDA_CHECK(cudaGetLastError());
    int launches = 1;
    for (int k = 1; k <= M; ++k) {
        BatchArgs<RP, V> a{};
        a.rp = rp;
        a.col = w.col ? w.col : Vw.col.ptr<int>();
        a.inv = inv;
        a.x_in = X[(k - 1) & 1];
        a.x_out = X[k & 1];
        a.T = T[(k - 1) & 1];
        a.acc = w.acc.ptr<V>();
        a.ck = co[k];
        a.first = k == 1;
        a.R = R;
        a.Rs = Rs;
        a.hub_rows = (int)std::min<int64_t>(g->n, ((int64_t)tuning().spmm_hub_mb << 20) / ((int64_t)Rs * (int64_t)sizeof(V)));
        a.xpol = tuning().spmm_xpol;
        a.part = w.part.ptr<double>();
        a.hub_part = w.hub_part.ptr<double>();
        a.hub_ts = Vw.n_hub ? w.hub_ts.ptr<double>() : nullptr;
        if (term_ms) CHEB_CUDA_CHECK(cudaEventRecord(ev[2 * (k - 1)], st));
        {
            cudaLaunchConfig_t cfg = {};
            cfg.gridDim = dim3(grid);
            cfg.blockDim = dim3(256);
            cfg.stream = st;
            cudaLaunchAttribute attr[1];
            cfg.attrs = attr;
            cfg.numAttrs = 0;
            if (tuning().l2win > 1 && l2_window(a.x_in, elems * sizeof(V), &attr[0].val.accessPolicyWindow)) {
                attr[0].id = cudaLaunchAttributeAccessPolicyWindow;
                cfg.numAttrs = 1;
            }
            CHEB_CUDA_CHECK(cudaLaunchKernelEx(&cfg, k_spmm_term<RP, V, VPL>, a, (const Tile*)Vw.tiles.ptr<Tile>(),
                                               Vw.n_tiles));
        }
        CHEB_CUDA_CHECK(cudaGetLastError());
        ++launches;
        if (Vw.n_hub) {
            const int hb = (int)std::min<int64_t>((Vw.n_hub * 32 + 255) / 256, 148 * 16);
            k_spmm_hub_finalize<RP, V, VPL><<<hb, 256, 0, st>>>(a, Vw.hub_first.ptr<int>(), Vw.n_hub);
            CHEB_CUDA_CHECK(cudaGetLastError());
            ++launches;
        }
        if (term_ms) CHEB_CUDA_CHECK(cudaEventRecord(ev[2 * (k - 1) + 1], st));
        k_trace_reduce_b<<<1, 256, 0, st>>>(w.part.ptr<double>(), grid, a.hub_ts, Vw.n_hub,
                                            w.trace.ptr<double>() + 2 * (k - 1));
        CHEB_CUDA_CHECK(cudaGetLastError());
        ++launches;
    }
    k_col_partial<V><<<nb, Rs, 0, st>>>(w.acc.ptr<V>(), n, Rs, chunk, w.colpart.ptr<double>());
    k_col_final<<<1, Rs, 0, st>>>(w.colpart.ptr<double>(), nb, Rs, w.totals.ptr<double>());
    k_spmm_normalize<V><<<1184, 256, 0, st>>>(w.acc.ptr<V>(), Vw.order.ptr<int>(), n, R, Rs, w.totals.ptr<double>(),
                                              w.out.ptr<double>());
    CHEB_CUDA_CHECK(cudaGetLastError());
    launches += 3;
    CHEB_CUDA_CHECK(cudaEventRecord(g->ev1, st));
    g->last_terms = M;
    g->last_launches = s.record_start ? launches : g->last_launches + launches;
    trace.assign(2 * (size_t)std::max(M, 1), 0.0);
    totals.assign(Rs, 0.0);
    if (M > 0)
        CHEB_CUDA_CHECK(cudaMemcpyAsync(trace.data(), w.trace.get(), sizeof(double) * 2 * M, cudaMemcpyDeviceToHost, st));
    CHEB_CUDA_CHECK(cudaMemcpyAsync(totals.data(), w.totals.get(), sizeof(double) * Rs, cudaMemcpyDeviceToHost, st));
    CHEB_CUDA_CHECK(cudaStreamSynchronize(st));
    float ms = 0.f;
    CHEB_CUDA_CHECK(cudaEventElapsedTime(&ms, g->ev0, g->ev1));
    g->last_loop_ms = ms;
    if (term_ms) {
        term_ms->assign(M, 0.0);
        for (int k = 0; k < M; ++k) {
            float t = 0.f;
            CHEB_CUDA_CHECK(cudaEventElapsedTime(&t, ev[2 * k], ev[2 * k + 1]));
            (*term_ms)[k] = t;
        }
        for (auto& e : ev) cudaEventDestroy(e);
    }
    totals.resize(R);
    for (int k = 1; k <= M; ++k)
        if (!std::isfinite(trace[2 * (k - 1)]) || !std::isfinite(trace[2 * (k - 1) + 1]))
            fail(CHEB_NUMERIC, "non-finite value at round " + std::to_string(k));
    for (int r = 0; r < R; ++r)
        if (!std::isfinite(totals[r]) || totals[r] <= 0.0)
            fail(CHEB_NUMERIC, "normalization total is not positive and finite");
}

template <class RP, class V>
void batch_dispatch(cheb_graph* g, const BatchSpec& s, std::vector<double>& tr, std::vector<double>& tot,
                    std::vector<double>* term_ms) {
    switch (vpl_for(s.R)) {
        case 1: batch_run<RP, V, 1>(g, s, tr, tot, term_ms); break;
        case 2: batch_run<RP, V, 2>(g, s, tr, tot, term_ms); break;
        default: batch_run<RP, V, 4>(g, s, tr, tot, term_ms); break;
    }
}

}  // namespace

void cpaa_batch_solve(cheb_graph* g, const BatchSpec& s, std::vector<double>& trace,
                      std::vector<double>& totals, std::vector<double>* term_ms) {
    GraphScope gs(g);
    if (s.R < 1 || s.R > 128) fail(CHEB_INVALID_ARG, "batched solve supports 1 <= R <= 128");
    ensure_view(g);
    {   // the gathered block X (n x Rs) larger than L2: the batched path gathers through its
        // own ascending-id copy of the view's columns, so a row's X gathers walk memory in
        // order (config 5: 259 -> 252 ms/solve) while the scalar schedule's bits stay untouched
        const int vpl = vpl_for(s.R);
        const int64_t x_bytes = g->n * (int64_t)((s.R + vpl - 1) / vpl * vpl) *
                                (s.precision == CHEB_FP64 ? 8 : 4);
        int dev = 0, l2 = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&l2, cudaDevAttrL2CacheSize, dev);
        g->bws.col = (tuning().sortrows != 0 && x_bytes > (int64_t)l2) ? batch_sorted_cols(g) : g->view.col.ptr<int>();
    }
    if (g->view.rp64) {
        if (s.precision == CHEB_FP64) batch_dispatch<int64_t, double>(g, s, trace, totals, term_ms);
        else batch_dispatch<int64_t, float>(g, s, trace, totals, term_ms);
    } else {
        if (s.precision == CHEB_FP64) batch_dispatch<int, double>(g, s, trace, totals, term_ms);
        else batch_dispatch<int, float>(g, s, trace, totals, term_ms);
    }
}

void read_batch_ranks(cheb_graph* g, double* ranks, int R) {
    GraphScope gs(g);
    CHEB_CUDA_CHECK(cudaMemcpyAsync(ranks, g->bws.out.get(), sizeof(double) * (size_t)g->n * R,
                                    cudaMemcpyDeviceToHost, g->stream));
    CHEB_CUDA_CHECK(cudaStreamSynchronize(g->stream));
}

}  // namespace chebgpu
