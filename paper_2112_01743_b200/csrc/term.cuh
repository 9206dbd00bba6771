// Device side of the CPAA path, shared by the drivers (cpaa.cu single GPU, dist.cu row
// partition, power.cu Power / transition_apply / staged API): kernels, the launch helper
// and the solve workspace.  Everything here has internal linkage (each driver translation
// unit instantiates what it launches).
//
// The reference round (/root/reference/proj/src/cpaa.cpp:109-156) is a pre-scale pass
// contrib = T_k * D^-1 (:116), a CSR gather with the three-term recurrence
// T_{k+1} = (k==1 ? s : 2s - T_{k-1}) and the coefficient accumulation acc += c_k T_{k+1}
// (:126-132), two serial Kahan trace sums (:142-143) and a finite check (:147-148).  Here one
// term kernel does all of it:
//
//   s_u        = sum_{v in N(u)} x_k[v]                (warp-tiled gather)
//   t          = first ? s_u : 2 s_u - T_{k-1}[u]      (recurrence, in place over T_{k-1})
//   acc[u]    += c_k * t                               (separate mul/add: reference rounding)
//   x_{k+1}[u] = t * (1/deg u)                         (next term's D^-1 pre-scale, fused)
//   block partials of sum(t), sum(acc)                 (trace, fixed order, deterministic)
//
// Two schedules:
//  * FAST (the product path, k_term_warp): rows relabelled by degree (descending); a
//    persistent CTA of 32 warps per SM; every warp walks a static program of tiles (<= 32
//    rows and <= 248 entries with 2^b lanes per row, or 248-entry chunks of a hub row that
//    k_hub_finalize completes in chunk order), column ids by TMA, the hottest x entries
//    from a shared-memory prefix.  Sums differ from the reference only in association order
//    (<= 1e-12 max-abs, tests).
//  * BITEXACT (k_term_exact): thread-per-row storage-order sums on the reference-order CSR,
//    explicit round-to-nearest mul/add, the reference's serial Kahan trace sums: bitwise
//    equal to the reference (ranks and trace).
#pragma once
#include <cub/cub.cuh>

#include <algorithm>
#include <cmath>
#include <cstring>
#include <string>

#include <nccl.h>

#include "common.cuh"
#include "device.cuh"

#define CHEB_NCCL_CHECK(expr)                                                              \
    do {                                                                                   \
        ncclResult_t _r = (expr);                                                          \
        if (_r != ncclSuccess)                                                             \
            ::chebgpu::fail(CHEB_NCCL, std::string("NCCL error ") + ncclGetErrorString(_r) + \
                                           " at " __FILE__ ":" + std::to_string(__LINE__)); \
    } while (0)


namespace chebgpu {
namespace {

// Experiment knobs of the term kernel (cheb_set_tuning: nogather, skip, skipwarm, prefetch,
// streamcs) cost ~5% of its instructions when compiled in (ncu source page, C4): the product
// build leaves them out; `make EXP=1` builds the experiment variant the tools/ studies use.
#ifndef CHEB_TERM_EXPERIMENTS
#define CHEB_TERM_EXPERIMENTS 0
#endif
constexpr bool kExp = CHEB_TERM_EXPERIMENTS != 0;

enum Epi : int {
    EPI_CPAA = 0,   // fused CPAA term (cpaa.cpp:126-132 + :116 for the next round)
    EPI_GEN = 1,    // staged generate_stage (cpaa.cpp:178-190): T_next only
    EPI_POWER = 2,  // power round (power.cpp:60-86): y = c s + base
    EPI_PLAIN = 3   // transition_apply (graph.cpp:104-121): y = s
};

template <class RP, class V>
struct TermArgs {
    const RP* __restrict__ rp;
    const int* __restrict__ col;
    const double* __restrict__ inv;  // non-null iff non-canonical inv_degree
    const V* __restrict__ x_in;      // x_k = T_k D^-1
    V* __restrict__ x_out;           // x_{k+1}
    V* T;                            // CPAA: T_{k-1} in, T_{k+1} out (in place); POWER: x in (and out)
    const V* T_prev;                 // GEN: T_{k-1}
    V* out;                          // GEN: T_next; PLAIN: y; POWER: x_k if not in place
    V* acc;
    double ck;    // CPAA: c_k ; POWER: c
    double base;  // POWER: (1-c)/n
    int first;
    double* part;  // [grid][2] this term
    double* hub_part;  // [n_tiles] chunk partials
    double* hub_ts;  // [n_hub][2] this term
    int tune_nogather;  // experiments only (cheb_set_tuning): replace x gathers by 1.0
    int prefetch;       // > 0: tile i + prefetch's column ids and row operands are prefetched into L2
    int tune_skip;      // experiments only: 1 skip chunk tiles, 2 skip pack tiles, 16+b only bin b
    int tune_skipwarm;  // experiments only: chunk tiles drop their gathers of ids in [H, tune_skipwarm)
    int stream_cs;      // per-row operands loaded / stored with the streaming (.cs) policy
    int xout_hint;      // x_{k+1} store policy (tuning().xout_hint)
    int64_t xdiscard_len;  // > 0: drop x_out[0, len) from L2 at kernel start (dead x_{k-1} lines)
    // fused push exchange (partitioned runs): x_{k+1} of local row u is stored at
    // push[r][part_global(u, part_r, part_G)] for the ranks r that read it
    // for every rank r (peer memory over NVLink) instead of x_out[u]
    V* const* push;
    int push_n;
    int part_G, part_r;         // G > 1: x_{k+1} of local row u goes to sorted row part_global(u, r, G)
    const unsigned* push_mask;  // halo-only push: bit r = rank r reads x[u] (null: every rank)
    // per-term device clock (TraceRow::elapsed_ms): the first term stamps its start, the last
    // CTA of the term's final kernel stamps its end
    unsigned long long* stamp_start;
    unsigned long long* stamp_end;
    unsigned* done;
};

__device__ __forceinline__ unsigned long long global_ns() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}
// The last CTA of the grid to get here records the time (the kernel's end, to within one CTA).
__device__ __forceinline__ void stamp_last_cta(unsigned* done, unsigned long long* stamp) {
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence();
        if (atomicAdd(done, 1u) == gridDim.x - 1) *stamp = global_ns();
    }
}

// Row epilogue.  u is a row of the current layout; deg its row length.
template <int EPI, class RP, class V>
__device__ __forceinline__ void epilogue(const TermArgs<RP, V>& a, int64_t u, V s, int64_t deg,
                                         double& p0, double& p1) {
    if constexpr (EPI == EPI_PLAIN) {
        a.out[u] = s;
    } else {
        const V inv = a.inv ? (V)a.inv[u] : rcp_rn((V)deg);
        if constexpr (EPI == EPI_CPAA) {
            const V t = a.first ? s : sub_rn(mul_rn(V(2), s), a.T[u]);
            a.T[u] = t;
            const V nacc = add_rn(a.acc[u], mul_rn((V)a.ck, t));
            a.acc[u] = nacc;
            a.x_out[u] = mul_rn(t, inv);
            p0 += (double)t;
            p1 += (double)nacc;
        } else if constexpr (EPI == EPI_GEN) {
            const V t = a.first ? s : sub_rn(mul_rn(V(2), s), a.T_prev[u]);
            a.out[u] = t;
        } else {  // EPI_POWER
            const V y = add_rn(mul_rn((V)a.ck, s), (V)a.base);
            const V old = a.T[u];
            (a.out ? a.out : a.T)[u] = y;  // out: a separate x_k buffer (Power snapshots)
            a.x_out[u] = mul_rn(y, inv);
            p0 += fabs((double)y - (double)old);
            p1 += (double)y;
        }
    }
}

// ---------------- FAST: persistent warp-tiled schedule ---------------------------------
//
// The view's rows are sorted by degree (descending) and cut into WARP tiles (build.cu):
//  * pack tiles: <= 32 consecutive whole rows with <= kWarpNnz (256) nnz;
//  * chunk tiles: a slice of <= kWarpNnz (256) nnz of a row with degree > kWarpNnz;
//    a row with several chunks is finished by the last chunk to arrive, which combines
//    the chunk partials in chunk order (deterministic).
// One CTA of 32 warps per SM; each warp walks tiles blockIdx*32+warp, +gridDim*32, ...
// (static, deterministic) with no CTA barrier inside the term: per tile a lane issues
// its 8 column-id loads, the row end pointer, T_{k-1} and acc at once, then 8 gathers.
// Gathers of the hottest vertices (ids < H: the degree-sorted hub prefix, ~50% of all
// gathers on power-law graphs) hit a shared-memory copy of x_k[0..H) refreshed at the
// start of every term; the rest go through L1/L2.  Measured on B200
// (tools/micro_gather.cu): random LDS.64 876 G/s vs random LDG over an L2-resident
// table 256 G/s — the gather, not HBM, bounds this path.

// Cold x gathers: read-only path without L1 allocation (the L1 left next to the shared
// hot prefix is tiny; a random line would only evict another).
#ifndef CHEB_COLD_NOALLOC
#define CHEB_COLD_NOALLOC 0
#endif
__device__ __forceinline__ double ldg_cold(const double* p) {
#if CHEB_COLD_NOALLOC
    double v;
    asm volatile("ld.global.nc.L1::no_allocate.f64 %0, [%1];" : "=d"(v) : "l"(p));
    return v;
#else
    return __ldg(p);
#endif
}
__device__ __forceinline__ float ldg_cold(const float* p) {
#if CHEB_COLD_NOALLOC
    float v;
    asm volatile("ld.global.nc.L1::no_allocate.f32 %0, [%1];" : "=f"(v) : "l"(p));
    return v;
#else
    return __ldg(p);
#endif
}

template <class T>
__device__ __forceinline__ T ld_cs(const T* p) { return __ldcs(p); }
template <class T>
__device__ __forceinline__ void st_cs(T* p, T v) { __stcs(p, v); }

// Store with an L2 eviction-priority hint: 1 evict_first policy, 2 .cs, 3 evict_last policy.
__device__ __forceinline__ void st_hint(double* p, double v, int h) {
    if (h == 1 || h == 3) {
        uint64_t pol;
        if (h == 1) asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
        else asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
        asm volatile("st.global.L2::cache_hint.f64 [%0], %1, %2;" :: "l"(p), "d"(v), "l"(pol) : "memory");
    } else if (h == 2) {
        __stcs(p, v);
    } else {
        *p = v;
    }
}
__device__ __forceinline__ void st_hint(float* p, float v, int h) {
    if (h == 1 || h == 3) {
        uint64_t pol;
        if (h == 1) asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
        else asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
        asm volatile("st.global.L2::cache_hint.f32 [%0], %1, %2;" :: "l"(p), "f"(v), "l"(pol) : "memory");
    } else if (h == 2) {
        __stcs(p, v);
    } else {
        *p = v;
    }
}

__device__ __forceinline__ double lds_v(unsigned addr, double) {
    double v;
    asm volatile("ld.shared.f64 %0, [%1];" : "=d"(v) : "r"(addr));
    return v;
}
__device__ __forceinline__ float lds_v(unsigned addr, float) {
    float v;
    asm volatile("ld.shared.f32 %0, [%1];" : "=f"(v) : "r"(addr));
    return v;
}

// Gather x[c[q]] for a lane's column ids: cold ids (>= H) as predicated global loads
// issued back to back, hot ids from the shared-memory copy at 32-bit address hot_s;
// c < 0 = no element (0).
template <class V, int U>
__device__ __forceinline__ void gather8(const V* __restrict__ x, unsigned hot_s, int H, const int (&c)[U],
                                        V (&v)[U]) {
#pragma unroll
    for (int q = 0; q < U; ++q) {
        v[q] = V(0);
        if (c[q] >= H) v[q] = ldg_cold(x + c[q]);
    }
#pragma unroll
    for (int q = 0; q < U; ++q)
        if ((unsigned)c[q] < (unsigned)H) v[q] = lds_v(hot_s + (unsigned)c[q] * (unsigned)sizeof(V), V(0));
}

// Cold gathers through LDGSTS (cp.async.cg, 16 bytes: the aligned piece of x holding x[c])
// into per-lane staging slots in shared memory, then LDS.  An LDG stages every in-flight load
// in the L1 data array, and next to the shared hot prefix + warp scratch (164 KB) the L1 left
// over bounds the random gathers in flight: measured (tools/micro_ldgsts.cu, 32 warps/SM)
// LDG from a 64 MB table 266 -> 149 G/s and from a 136 MB table 108 -> 81 G/s once 164 KB of
// shared memory is reserved, while cp.async.cg gathers keep 240 / 108 G/s with up to 220 KB
// reserved (they land in shared memory and never allocate in L1).  In the term kernel itself
// the extra instructions (LDGSTS + commit/wait + LDS per cold gather, batches of 1-4 per lane)
// cost more than the in-flight capacity gains: C2 69.2 -> 75-81 us/term, C3 395 -> 434-464,
// C4 4051 -> 4001-4212 (profiles/r02_gather_paths.md); off by default, -DCHEB_GATHER_ASYNC=1.
#ifndef CHEB_GATHER_ASYNC
#define CHEB_GATHER_ASYNC 0
#endif
#ifndef CHEB_STAGE_SLOTS
#define CHEB_STAGE_SLOTS 2
#endif
constexpr bool kGatherAsync = CHEB_GATHER_ASYNC != 0;
constexpr int kStageSlots = CHEB_STAGE_SLOTS;  // 16-byte slots per lane (gathers in flight per lane)

__device__ __forceinline__ void cp_async16(unsigned dst, const void* src) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" :: "r"(dst), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() {
    asm volatile("cp.async.commit_group;\n\tcp.async.wait_group 0;" ::: "memory");
}

// gather8 with the cold ids through the lane's staging slots (slot j at stage_s + 512 j), in
// batches of kStageSlots.
template <class V, int U>
__device__ __forceinline__ void gather_staged(const V* __restrict__ x, unsigned hot_s, int H, unsigned stage_s,
                                              const int (&c)[U], V (&v)[U]) {
    constexpr int per16 = 16 / (int)sizeof(V);
#pragma unroll
    for (int b = 0; b < U; b += kStageSlots) {
#pragma unroll
        for (int q = b; q < b + kStageSlots && q < U; ++q)
            if (c[q] >= H) cp_async16(stage_s + (unsigned)(q - b) * 512u, x + (c[q] & ~(per16 - 1)));
        cp_async_wait_all();
#pragma unroll
        for (int q = b; q < b + kStageSlots && q < U; ++q) {
            v[q] = V(0);
            if ((unsigned)c[q] < (unsigned)H) v[q] = lds_v(hot_s + (unsigned)c[q] * (unsigned)sizeof(V), V(0));
            else if (c[q] >= H)
                v[q] = lds_v(stage_s + (unsigned)(q - b) * 512u + (unsigned)(c[q] & (per16 - 1)) * (unsigned)sizeof(V), V(0));
        }
    }
}

// Programmatic dependent launch: let the next kernel of the stream launch now (its CTAs
// take SMs as this grid drains), and wait for the previous kernel's completion + memory
// flush before reading anything it wrote.  Both are no-ops without the launch attribute.
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }

// TMA bulk copy global -> shared (cp.async.bulk), completion on an mbarrier.
__device__ __forceinline__ void bulk_g2s(void* smem_dst, const void* gsrc, unsigned bytes, uint64_t* mbar) {
    const unsigned dst = (unsigned)__cvta_generic_to_shared(smem_dst);
    const unsigned bar = (unsigned)__cvta_generic_to_shared(mbar);
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                 :: "r"(dst), "l"(gsrc), "r"(bytes), "r"(bar) : "memory");
}
// Column ids are read once per term: an L2 evict-first policy on their TMA copies keeps the
// per-term streams (~130 MB on C2, about the size of L2) from pushing x out of L2
// (C2 73.2 -> 70.1 us/term; profiles/r01_gather_microbench.md).
#ifndef CHEB_COL_EVICT_FIRST
#define CHEB_COL_EVICT_FIRST 1
#endif
__device__ __forceinline__ void bulk_g2s_stream(void* smem_dst, const void* gsrc, unsigned bytes, uint64_t* mbar) {
    if (!CHEB_COL_EVICT_FIRST) {  // experiments: no cache hint
        bulk_g2s(smem_dst, gsrc, bytes, mbar);
        return;
    }
    const unsigned dst = (unsigned)__cvta_generic_to_shared(smem_dst);
    const unsigned bar = (unsigned)__cvta_generic_to_shared(mbar);
    uint64_t pol;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;"
        :: "r"(dst), "l"(gsrc), "r"(bytes), "r"(bar), "l"(pol) : "memory");
}

__device__ __forceinline__ void mbar_init(uint64_t* mbar, unsigned count) {
    const unsigned bar = (unsigned)__cvta_generic_to_shared(mbar);
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" :: "r"(bar), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* mbar, unsigned bytes) {
    const unsigned bar = (unsigned)__cvta_generic_to_shared(mbar);
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" :: "r"(bar), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* mbar, unsigned parity) {
    const unsigned bar = (unsigned)__cvta_generic_to_shared(mbar);
    asm volatile(
        "{\n"
        ".reg .pred done;\n"
        "WAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 done, [%0], %1;\n"
        "@!done bra WAIT_%=;\n"
        "}\n" :: "r"(bar), "r"(parity) : "memory");
}

// Row epilogue with the row's operands already loaded (prev = T_{k-1} / old x).  SINGLE:
// one GPU, canonical inv_degree, no push exchange (the product case): those branches are
// compiled out of the term kernel.
template <int EPI, class RP, class V, bool SINGLE = false>
__device__ __forceinline__ void epilogue_v(const TermArgs<RP, V>& a, int64_t u, V s, int64_t deg,
                                           V prev, V accv, double& p0, double& p1) {
    if constexpr (EPI == EPI_PLAIN) {
        a.out[u] = s;
    } else {
        const V inv = (!SINGLE && a.inv) ? (V)a.inv[u] : rcp_rn((V)deg);
        if constexpr (EPI == EPI_CPAA) {
            const V t = a.first ? s : sub_rn(mul_rn(V(2), s), prev);
            const V nacc = add_rn(accv, mul_rn((V)a.ck, t));
            const V xn = mul_rn(t, inv);
            if (kExp && a.stream_cs) {
                st_cs(a.T + u, t);
                st_cs(a.acc + u, nacc);
            } else {
                a.T[u] = t;
                a.acc[u] = nacc;
            }
            const int64_t pos = (!SINGLE && a.part_G > 1) ? part_global(u, a.part_r, a.part_G) : u;
            if (!SINGLE && a.push) {  // fused exchange: straight into the copies of x_{k+1} that are read
                const unsigned m = a.push_mask ? __ldg(a.push_mask + u) : ~0u;
                for (int r = 0; r < a.push_n; ++r)
                    if (m >> r & 1u) a.push[r][pos] = xn;
            } else {
                st_hint(a.x_out + pos, xn, a.xout_hint);
            }
            p0 += (double)t;
            p1 += (double)nacc;
        } else if constexpr (EPI == EPI_GEN) {
            a.out[u] = a.first ? s : sub_rn(mul_rn(V(2), s), prev);
        } else {  // EPI_POWER
            const V y = add_rn(mul_rn((V)a.ck, s), (V)a.base);
            (a.out ? a.out : a.T)[u] = y;
            a.x_out[u] = mul_rn(y, inv);
            p0 += fabs((double)y - (double)prev);
            p1 += (double)y;
        }
    }
}

template <int EPI, class RP, class V>
__device__ __forceinline__ const V* prev_src(const TermArgs<RP, V>& a) {
    if constexpr (EPI == EPI_GEN) return a.T_prev;
    else return a.T;
}

template <class V>
__device__ __forceinline__ V warp_sum_v(V v) {
#pragma unroll
    for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

template <class V>
constexpr int hot_capacity() { return (kHotBytes / (int)sizeof(V)); }

// Per-warp shared scratch of the term kernel.
// Column-id landing buffers per warp (NB): 2 = the next tile's ids are copied while the
// current tile is read; 1 = one buffer, refilled as soon as the current tile's ids are in
// registers — 34 KB less shared memory per SM, so the carve-out drops from 164 to 132 KB and
// the L1 holds more in-flight gathers.  Chosen per graph at launch (launch_pass): 1 when x
// exceeds L2 (config 4 fp64: 3556 -> 3403-3456 us/term), 2 otherwise (config 2: 68.1 vs 72.2).
template <class V, int NB>
struct alignas(16) WarpScratch {
    int colb[NB][kColBuf];  // TMA landing buffers of column ids
    WTile desc[2][kDescBlock];  // TMA ring of this warp's tile program
    uint64_t colm[2];       // mbarriers of colb
    uint64_t descm[2];      // mbarriers of desc
    alignas(16) unsigned char stage[kGatherAsync ? kStageSlots : 0][32][16];  // cold-gather slots [slot][lane]
};

#ifndef CHEB_SMEM_PAD_KB
#define CHEB_SMEM_PAD_KB 0  // experiments: unused shared memory (shrinks the L1 carve-out)
#endif
template <class V, int NB>
constexpr size_t warp_smem_bytes() {
    return (size_t)kHotBytes + (size_t)kWarps * sizeof(WarpScratch<V, NB>) + 2 * 32 * sizeof(double) +
           (size_t)CHEB_SMEM_PAD_KB * 1024;
}

// Tile in registers.
struct TileR {
    int64_t z0;
    int r0, rows, cnt, meta;
};

// One 16-byte shared load per descriptor (field by field it was five loads per lane).
__device__ __forceinline__ TileR tile_of(const WTile& d) {
    const uint4 q = *reinterpret_cast<const uint4*>(&d);
    TileR r;
    r.z0 = (int64_t)(((uint64_t)q.y << 32) | q.x);  // nnz_begin
    r.r0 = (int)q.z;                               // row_begin
    r.cnt = (int)(q.w & 0xffffu);
    r.rows = (int)((q.w >> 16) & 0xffu);
    r.meta = (int)(q.w >> 24);
    return r;
}

// Lane 0: bulk-copy the tile's column ids from the 8-aligned position a0 = z0 & ~7 into buf.
__device__ __forceinline__ void issue_cols(const int* __restrict__ col, const TileR& t, int* buf,
                                           uint64_t* mbar) {
    const int64_t a0 = t.z0 & ~int64_t(7);
    const unsigned bytes = (unsigned)(((t.z0 - a0) + t.cnt + 3) & ~3) * 4u;
    mbar_expect_tx(mbar, bytes);
    bulk_g2s_stream(buf, col + a0, bytes, mbar);
}

// Row operands of a pack tile for the lane leading row g's lane group (L = 1 << lg lanes
// per row): tile-local row start/end, T_{k-1}, acc.
template <class V>
struct RowOps {
    int rs, re;
    V pv, av;
};

template <int EPI, class RP, class V>
__device__ __forceinline__ void load_rows(const TermArgs<RP, V>& a, const TileR& t, RowOps<V>& o) {
    const int lane = threadIdx.x & 31;
    o.rs = 0;
    o.re = 0;
    o.pv = V(0);
    o.av = V(0);
    if (t.meta & kTileChunk) return;
    const int lg = t.meta & 0xf;
    const int g = lane >> lg;
    if ((lane & ((1 << lg) - 1)) == 0 && g < t.rows) {
        if (kExp && a.stream_cs) {
            o.rs = (int)(ld_cs(a.rp + t.r0 + g) - t.z0);
            o.re = (int)(ld_cs(a.rp + t.r0 + g + 1) - t.z0);
            if constexpr (EPI != EPI_PLAIN) o.pv = ld_cs(prev_src<EPI>(a) + t.r0 + g);
            if constexpr (EPI == EPI_CPAA) o.av = ld_cs(a.acc + t.r0 + g);
        } else {
            o.rs = (int)(a.rp[t.r0 + g] - t.z0);
            o.re = (int)(a.rp[t.r0 + g + 1] - t.z0);
            if constexpr (EPI != EPI_PLAIN) o.pv = prev_src<EPI>(a)[t.r0 + g];
            if constexpr (EPI == EPI_CPAA) o.av = a.acc[t.r0 + g];
        }
    }
}

// Lane 0: bulk-copy descriptor block blk of this warp's program into ring slot blk & 1.
__device__ __forceinline__ void issue_desc(const WTile* my, int blk, void* unused,
                                           WTile* slot, uint64_t* mbar) {
    (void)unused;
    mbar_expect_tx(mbar, kDescBlock * sizeof(WTile));
    bulk_g2s(slot, my + (size_t)blk * kDescBlock, kDescBlock * sizeof(WTile), mbar);
}

#ifndef CHEB_PACK_UNROLL
#define CHEB_PACK_UNROLL 4
#endif
constexpr int kPackUnroll = CHEB_PACK_UNROLL;  // gathers in flight per lane in pack tiles

// One tile of the warp's program.  cur: this tile's row operands (loaded one tile ago);
// nxt receives the next tile's.  No register prefetched here is copied at the end.
template <int EPI, bool SINGLE, int NB, class RP, class V, class WS>
__device__ __forceinline__ void term_step(const TermArgs<RP, V>& a, unsigned hot_s, int H, WS& ws,
                                          const WTile* my, int w, int S, int nt, int i,
                                          const RowOps<V>& cur, RowOps<V>& nxt, double& p0, double& p1) {
    const int lane = threadIdx.x & 31;
    constexpr int U = 8;
    const TileR d = tile_of(ws.desc[(i / kDescBlock) & 1][i % kDescBlock]);
    TileR dn{};
    if (i + 1 < nt) {
        const int j = i + 1;
        if (j % kDescBlock == 0) mbar_wait(&ws.descm[(j / kDescBlock) & 1], ((j / kDescBlock) >> 1) & 1);
        dn = tile_of(ws.desc[(j / kDescBlock) & 1][j % kDescBlock]);
        if (NB == 2 && lane == 0) issue_cols(a.col, dn, ws.colb[j % NB], &ws.colm[j % NB]);
        load_rows<EPI>(a, dn, nxt);
    }
    // single buffer: the next tile's ids are copied once this tile's are in registers (`dep`:
    // an XOR of every id the lane read from the buffer).
    auto refill = [&](int dep) {
        if constexpr (NB == 1) {
            // a warp-wide OR of every lane's ids selects the copy's cache hint (either hint is
            // correct): the copy cannot issue before all of the warp's id loads have returned,
            // and the compiler cannot drop the dependency (an empty asm or a vote that does not
            // feed the copy is optimised away, and the copy then raced the reads: C3/C4 ranks
            // differed run to run)
            const unsigned all = __reduce_or_sync(0xffffffffu, (unsigned)dep);
            if (lane == 0 && i + 1 < nt) {
                const int64_t a0 = dn.z0 & ~int64_t(7);
                const unsigned bytes = (unsigned)(((dn.z0 - a0) + dn.cnt + 3) & ~3) * 4u;
                mbar_expect_tx(&ws.colm[0], bytes);
                if (all == 0x9e3779b9u) bulk_g2s(ws.colb[0], a.col + a0, bytes, &ws.colm[0]);
                else bulk_g2s_stream(ws.colb[0], a.col + a0, bytes, &ws.colm[0]);
            }
        }
    };
    // L2 prefetch of a tile further ahead (its descriptor lives in the current or the next
    // block of the ring): the per-warp double buffer keeps ~1 tile of column ids in flight,
    // too few bytes to cover DRAM latency on graphs whose streams miss L2 (config 4)
    if (kExp && a.prefetch > 0 && i + a.prefetch < nt && lane < 4) {
        const int j = i + a.prefetch;
        if ((j / kDescBlock) <= (i / kDescBlock) + 1) {
            if ((j / kDescBlock) != (i / kDescBlock)) mbar_wait(&ws.descm[(j / kDescBlock) & 1], ((j / kDescBlock) >> 1) & 1);
            const TileR dp = tile_of(ws.desc[(j / kDescBlock) & 1][j % kDescBlock]);
            if (lane == 0) {
                const int64_t a0 = dp.z0 & ~int64_t(3);
                const unsigned bytes = (unsigned)(((dp.z0 - a0) + dp.cnt + 3) & ~3) * 4u;
                asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" :: "l"(a.col + a0), "r"(bytes) : "memory");
            } else if (!(dp.meta & kTileChunk)) {  // row pointers, T_{k-1}, acc of its rows
                const void* p = lane == 1 ? (const void*)(a.rp + dp.r0)
                                          : lane == 2 ? (const void*)(prev_src<EPI>(a) + dp.r0) : (const void*)(a.acc + dp.r0);
                if (EPI == EPI_CPAA || lane == 1) asm volatile("prefetch.global.L2 [%0];" :: "l"(p));
            }
        }
    }
    // LSU-path variant (prefetch < 0): tile i + |prefetch|'s column-id lines and row operands
    // prefetched into L2 with prefetch.global.L2 by lanes 0-11 when its descriptor is in the
    // current block (no descriptor wait, no TMA-unit traffic)
    if (kExp && a.prefetch < 0 && lane < 12) {
        const int j = i - a.prefetch;
        if (j < nt && j / kDescBlock == i / kDescBlock) {
            const TileR dp = tile_of(ws.desc[(j / kDescBlock) & 1][j % kDescBlock]);
            const int64_t a0 = dp.z0 & ~int64_t(31);
            const int lines = (int)((dp.z0 + dp.cnt - a0 + 31) >> 5);
            if (lane < 9) {
                if (lane < lines) asm volatile("prefetch.global.L2 [%0];" :: "l"(a.col + a0 + 32 * lane));
            } else if (!(dp.meta & kTileChunk)) {
                const void* p = lane == 9 ? (const void*)(a.rp + dp.r0)
                                          : lane == 10 ? (const void*)(prev_src<EPI>(a) + dp.r0) : (const void*)(a.acc + dp.r0);
                asm volatile("prefetch.global.L2 [%0];" :: "l"(p));
            }
        }
    }
    mbar_wait(&ws.colm[i % NB], (i / NB) & 1);
    if (kExp && a.tune_skip &&
        (a.tune_skip >= 16 ? (((d.meta & kTileChunk) ? 6 : (d.meta & 0xf)) != a.tune_skip - 16)
                           : ((a.tune_skip & 1) ? (d.meta & kTileChunk) : !(d.meta & kTileChunk)))) {
        refill(0);
        __syncwarp();
        if (lane == 0 && i % kDescBlock == kDescBlock - 1) {
            const int blk = i / kDescBlock + 2;
            if (blk * kDescBlock < nt) issue_desc(my, blk, nullptr, ws.desc[blk & 1], &ws.descm[blk & 1]);
        }
        return;
    }
    const int* cb = ws.colb[i % NB] + (int)(d.z0 & 7);  // tile-local position p at cb[p]
    [[maybe_unused]] const unsigned stage_s = kGatherAsync ? (unsigned)__cvta_generic_to_shared(&ws.stage[0][lane][0]) : 0u;

    if (d.meta & kTileChunk) {
        // slice of a row with degree > kWarpNnz: partial only; completed by k_hub_finalize
        int c[U];
        if (d.cnt == kWarpNnz) {  // a full chunk (all but a row's last): only step 7 has empty lanes
#pragma unroll
            for (int q = 0; q < U - 1; ++q) c[q] = cb[lane + 32 * q];
            c[U - 1] = lane < kWarpNnz - 32 * (U - 1) ? cb[lane + 32 * (U - 1)] : -1;
        } else {
#pragma unroll
            for (int q = 0; q < U; ++q) {
                const int pp = lane + 32 * q;
                c[q] = pp < d.cnt ? cb[pp] : -1;
            }
        }
        {
            int dep = 0;
#pragma unroll
            for (int q = 0; q < U; ++q) dep ^= c[q];
            refill(dep);
        }
        V v[U];
        if (kExp && a.tune_nogather) {
#pragma unroll
            for (int q = 0; q < U; ++q) v[q] = c[q] >= 0 ? V(1) : V(0);
        } else {
            if (kExp && a.tune_skipwarm > 0) {  // experiment: hub-row gathers of ids in [H, skipwarm) dropped
#pragma unroll
                for (int q = 0; q < U; ++q)
                    if (c[q] >= H && c[q] < a.tune_skipwarm) c[q] = -1;
            }
            if constexpr (kGatherAsync) gather_staged(a.x_in, hot_s, H, stage_s, c, v);
            else gather8(a.x_in, hot_s, H, c, v);
        }
        double sum = 0.0;  // hub-row chunk sums in fp64 (fp32: a lane's U entries in fp32)
        if constexpr (sizeof(V) == 8) {
#pragma unroll
            for (int q = 0; q < U; ++q) sum += v[q];
        } else {
            V blk = v[0];
#pragma unroll
            for (int q = 1; q < U; ++q) blk += v[q];
            sum = (double)blk;
        }
        sum = warp_sum_v(sum);
        if (lane == 0) a.hub_part[d.r0] = (double)sum;  // a chunk tile's row_begin is its tile id
    } else {
        // rows of similar degree: L lanes per row, row g owned by lanes [g L, g L + L)
        const int lg = d.meta & 0xf;
        const int L = 1 << lg;
        const int li = lane & (L - 1), g = lane >> lg;
        int rb = cur.rs, rend = cur.re;
        if (lg) {
            const int leader = lane & ~(L - 1);
            rb = __shfl_sync(0xffffffffu, rb, leader);
            rend = __shfl_sync(0xffffffffu, rend, leader);
        }
        // pack rows: <= 8 entries per lane, summed in V; hub rows (chunk tiles) use fp64
        V sum = V(0);
        int jj0 = rb + li;
        if constexpr (NB == 1) {
            // the lane's first 2 kPackUnroll entries into registers, then the buffer is free;
            // the same per-lane order as the loop below
            int c8[2 * kPackUnroll];
#pragma unroll
            for (int q = 0; q < 2 * kPackUnroll; ++q) c8[q] = jj0 + q * L < rend ? cb[jj0 + q * L] : -1;
            const bool more = __any_sync(0xffffffffu, jj0 + 2 * kPackUnroll * L < rend);
            int dep = 0;
#pragma unroll
            for (int q = 0; q < 2 * kPackUnroll; ++q) dep ^= c8[q];
            if (!more) refill(dep);
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                if (jj0 + h * kPackUnroll * L < rend) {
                    int c[kPackUnroll];
#pragma unroll
                    for (int q = 0; q < kPackUnroll; ++q) c[q] = c8[h * kPackUnroll + q];
                    V v[kPackUnroll];
                    gather8(a.x_in, hot_s, H, c, v);
#pragma unroll
                    for (int q = 0; q < kPackUnroll; ++q) sum += v[q];
                }
            }
            jj0 += 2 * kPackUnroll * L;
            if (more) {  // a lane with more than 2 kPackUnroll entries (mixed-degree tile)
                int dep2 = dep;  // the first 2 kPackUnroll ids too
                for (int jj = jj0; jj < rend; jj += kPackUnroll * L) {
                    int c[kPackUnroll];
#pragma unroll
                    for (int q = 0; q < kPackUnroll; ++q) c[q] = jj + q * L < rend ? cb[jj + q * L] : -1;
#pragma unroll
                    for (int q = 0; q < kPackUnroll; ++q) dep2 ^= c[q];
                    V v[kPackUnroll];
                    gather8(a.x_in, hot_s, H, c, v);
#pragma unroll
                    for (int q = 0; q < kPackUnroll; ++q) sum += v[q];
                }
                refill(dep2);
            }
            jj0 = rend;  // done
        }
        for (int jj = jj0; jj < rend; jj += kPackUnroll * L) {
            int c[kPackUnroll];
#pragma unroll
            for (int q = 0; q < kPackUnroll; ++q) c[q] = jj + q * L < rend ? cb[jj + q * L] : -1;
            V v[kPackUnroll];
            if (kExp && a.tune_nogather) {
#pragma unroll
                for (int q = 0; q < kPackUnroll; ++q) v[q] = c[q] >= 0 ? V(1) : V(0);
            } else if constexpr (kGatherAsync) {
                gather_staged(a.x_in, hot_s, H, stage_s, c, v);
            } else {
                gather8(a.x_in, hot_s, H, c, v);
            }
#pragma unroll
            for (int q = 0; q < kPackUnroll; ++q) sum += v[q];
        }
        for (int o = L >> 1; o; o >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, o);
        if (li == 0 && g < d.rows)
            epilogue_v<EPI, RP, V, SINGLE>(a, (int64_t)d.r0 + g, sum, (int64_t)(rend - rb), cur.pv, cur.av, p0, p1);
    }
    __syncwarp();
    // descriptor block of tile i fully consumed: refill its slot two blocks ahead
    if (lane == 0 && i % kDescBlock == kDescBlock - 1) {
        const int blk = i / kDescBlock + 2;
        if (blk * kDescBlock < nt) issue_desc(my, blk, nullptr, ws.desc[blk & 1], &ws.descm[blk & 1]);
    }
}

template <int EPI, class RP, class V, bool SINGLE, int NB>
__global__ void __launch_bounds__(kWarps * 32, 1)
k_term_warp(TermArgs<RP, V> a, const WTile* __restrict__ prog, int P, int ntiles, int H) {
    extern __shared__ __align__(16) unsigned char smem[];
    V* hot = reinterpret_cast<V*>(smem);
    // shared-window address of the hot prefix, kept in a register: without the opaque move
    // the compiler rematerialises it (S2R SR_CgaCtaId + MOV + LEA) before every hot gather
    unsigned hot_s;
    asm volatile("mov.b32 %0, %1;" : "=r"(hot_s) : "r"((unsigned)__cvta_generic_to_shared(smem)));
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    WarpScratch<V, NB>& ws = reinterpret_cast<WarpScratch<V, NB>*>(smem + kHotBytes)[warp];
    double* red = reinterpret_cast<double*>(smem + kHotBytes + kWarps * sizeof(WarpScratch<V, NB>));
    __shared__ __align__(8) uint64_t mbar_hot;

    const int S = gridDim.x * kWarps;
    const int w = blockIdx.x * kWarps + warp;
    const int nt = w < ntiles ? (ntiles - w + S - 1) / S : 0;
    const WTile* my = prog + (size_t)w * P;

    // hot prefix x_k[0..H) -> shared memory (TMA bulk copies; sub-16-byte tail by loads)
    const unsigned hot_bytes = (unsigned)(H * sizeof(V)) & ~15u;
    if (threadIdx.x == 0) mbar_init(&mbar_hot, 1);
    if (lane == 0) {
        mbar_init(&ws.colm[0], 1);
        if (NB == 2) mbar_init(&ws.colm[1], 1);
        mbar_init(&ws.descm[0], 1);
        mbar_init(&ws.descm[1], 1);
    }
    if (threadIdx.x == 0) asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    __syncthreads();
    pdl_trigger();
    if (lane == 0) {  // this warp's tile program is static: fetch it before the dependency wait
        if (nt > 0) issue_desc(my, 0, nullptr, ws.desc[0], &ws.descm[0]);
        if (nt > kDescBlock) issue_desc(my, 1, nullptr, ws.desc[1], &ws.descm[1]);
    }
    pdl_wait();  // x_k, T, acc come from the previous kernels of the stream
    if (a.stamp_start && blockIdx.x == 0 && threadIdx.x == 0) *a.stamp_start = global_ns();
    if (a.xdiscard_len > 0) {
        // x_out holds x_{k-1}, dead once the previous term finished: drop its lines from L2
        // (no write-back) so they do not hold cache space (or the persisting carve-out)
        const int64_t lines = a.xdiscard_len * (int64_t)sizeof(V) / 128;
        const char* base = reinterpret_cast<const char*>(a.x_out);
        for (int64_t l = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; l < lines;
             l += (int64_t)gridDim.x * blockDim.x)
            asm volatile("discard.global.L2 [%0], 128;" :: "l"(base + l * 128) : "memory");
    }
    if (threadIdx.x == 0) {
        mbar_expect_tx(&mbar_hot, hot_bytes);
        constexpr unsigned kPiece = 32768;
        for (unsigned off = 0; off < hot_bytes; off += kPiece)
            bulk_g2s(smem + off, reinterpret_cast<const unsigned char*>(a.x_in) + off,
                     min(kPiece, hot_bytes - off), &mbar_hot);
    }
    for (int i = hot_bytes / sizeof(V) + threadIdx.x; i < H; i += blockDim.x) hot[i] = ldg_x(a.x_in + i);

    RowOps<V> A, B;
    if (nt > 0) {
        mbar_wait(&ws.descm[0], 0);
        const TileR d0 = tile_of(ws.desc[0][0]);
        if (lane == 0) issue_cols(a.col, d0, ws.colb[0], &ws.colm[0]);
        load_rows<EPI>(a, d0, A);
    }
    double p0 = 0.0, p1 = 0.0;
    mbar_wait(&mbar_hot, 0);
    __syncthreads();

    for (int i = 0; i < nt; i += 2) {
        term_step<EPI, SINGLE, NB>(a, hot_s, H, ws, my, w, S, nt, i, A, B, p0, p1);
        if (i + 1 >= nt) break;
        term_step<EPI, SINGLE, NB>(a, hot_s, H, ws, my, w, S, nt, i + 1, B, A, p0, p1);
    }
    if constexpr (EPI == EPI_CPAA || EPI == EPI_POWER) {
        if (a.part) {
            p0 = warp_sum_v(p0);
            p1 = warp_sum_v(p1);
            if (lane == 0) {
                red[warp] = p0;
                red[32 + warp] = p1;
            }
            __syncthreads();
            if (warp == 0) {
                double q0 = lane < kWarps ? red[lane] : 0.0;
                double q1 = lane < kWarps ? red[32 + lane] : 0.0;
                q0 = warp_sum_v(q0);
                q1 = warp_sum_v(q1);
                if (lane == 0) {
                    a.part[2 * blockIdx.x] = q0;
                    a.part[2 * blockIdx.x + 1] = q1;
                }
            }
        }
    }
    if (a.stamp_end) stamp_last_cta(a.done, a.stamp_end);
}

// Hub rows (degree > kWarpNnz, rows [0, n_hub) of the view, degree-descending): the row's
// chunk partials summed in the shuffle-tree order of a warp holding partial q in lane
// q mod 32, then the fused epilogue.  Chunk tiles of row h are the consecutive tiles
// [hub_first[h], hub_first[h+1]).  Rows [0, n_wide) (> 32 chunks) take a warp each; the
// rest take a lane each, 32 consecutive rows per warp, and replay the same tree for their
// <= 32 partials in registers (bitwise the warp result).  A warp per row left every warp
// walking ~50 rows one dependent load chain at a time (C4: ~1 M hub rows, 0.24 ms per term).
template <int EPI, class RP, class V>
__device__ __forceinline__ void hub_epilogue(const TermArgs<RP, V>& a, int64_t h, double tot) {
    const int64_t deg = a.rp[h + 1] - a.rp[h];
    double q0 = 0.0, q1 = 0.0;
    const V hp = EPI != EPI_PLAIN ? prev_src<EPI>(a)[h] : V(0);
    const V ha = EPI == EPI_CPAA ? a.acc[h] : V(0);
    epilogue_v<EPI>(a, h, (V)tot, deg, hp, ha, q0, q1);
    if (a.hub_ts) {
        a.hub_ts[2 * h] = q0;
        a.hub_ts[2 * h + 1] = q1;
    }
}

template <int EPI, class RP, class V>
__global__ void __launch_bounds__(256) k_hub_finalize(TermArgs<RP, V> a, const int* __restrict__ hub_first,
                                                      int64_t n_hub, int64_t n_wide, const int* __restrict__ kf,
                                                      const int* __restrict__ klist, const double* __restrict__ wpart) {
    const int lane = threadIdx.x & 31;
    pdl_trigger();
    pdl_wait();  // the term kernel's hub partials
    const int64_t gw = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t h = gw; h < n_wide; h += nw) {
        const int f0 = hub_first[h], f1 = hub_first[h + 1];
        double tot = 0.0;
        for (int q = f0 + lane; q < f1; q += 32) tot += a.hub_part[q];
        if (kf) {  // the row's window pieces (SolverView::Windows)
            const int g0 = kf[h], g1 = kf[h + 1];
            for (int q = g0 + lane; q < g1; q += 32) tot += wpart[klist[q]];
        }
        tot = warp_sum_v(tot);
        if (lane == 0) hub_epilogue<EPI>(a, h, tot);
    }
    const int64_t groups = (n_hub - n_wide + 31) >> 5;
    // lane groups continue the rotation where the wide rows stopped (group 0 goes to the warp
    // that would have taken row n_wide)
    for (int64_t gi = (gw + nw - n_wide % nw) % nw; gi < groups; gi += nw) {
        const int64_t h = n_wide + gi * 32 + lane;
        if (h >= n_hub) continue;
        const int f0 = hub_first[h], m = hub_first[h + 1] - f0;
        double tot;
        if (m <= 32) {
            double v[32];
#pragma unroll
            for (int i = 0; i < 32; ++i) v[i] = i < m ? __dadd_rn(0.0, a.hub_part[f0 + i]) : 0.0;
#pragma unroll
            for (int o = 16; o; o >>= 1)
#pragma unroll
                for (int i = 0; i < o; ++i) v[i] = __dadd_rn(v[i], v[i + o]);
            tot = v[0];
        } else {  // only after the opt-in column-block split (chunk counts no longer monotone)
            tot = 0.0;
            for (int q = 0; q < m; ++q) tot += a.hub_part[f0 + q];
        }
        if (kf) {
            const int g0 = kf[h], g1 = kf[h + 1];
            int q = g0;
            for (; q + 4 <= g1; q += 4) {  // four independent loads in flight, summed in list order
                const double p0 = wpart[klist[q]], p1 = wpart[klist[q + 1]], p2 = wpart[klist[q + 2]],
                             p3 = wpart[klist[q + 3]];
                tot += p0;
                tot += p1;
                tot += p2;
                tot += p3;
            }
            for (; q < g1; ++q) tot += wpart[klist[q]];
        }
        hub_epilogue<EPI>(a, h, tot);
    }
    if (a.stamp_end) stamp_last_cta(a.done, a.stamp_end);
}

// ---------------- column windows of the hub rows (SolverView::Windows) -----------------
// One CTA per SM over a contiguous range of the window-major stream's blocks.  A CTA loads the
// window of x_k its blocks belong to into shared memory (reloading when its range crosses into
// the next window); a warp takes one block of kWinBlock entries at a time, lane l the 8
// consecutive entries 8 l .. 8 l + 7 (one 16-byte load of 16-bit window-local ids), gathers
// them from shared memory and sums them piece by piece: runs that start and end inside the
// lane are stored directly, a run still open at the lane's end takes the following lanes'
// leading sums up to the next start (segmented suffix scan over the lanes, fixed order).  A
// block's first entry always starts a piece, so no sum crosses blocks.  Piece sums are in
// fp64; piece k of the stream goes to wpart[k] (consecutive pieces, coalesced stores), and
// k_hub_finalize adds a row's pieces (klist) to its chunk partials.  Every entry handled here
// costs one shared-memory load instead of an L2 sector.  The CTA block ranges (cta[]) are cut at
// build time by cost (256 + 4 pieces per block): blocks of short pieces store more sums.
// Reference loop this replaces for these entries: cpaa.cpp:126-132 (the neighbour sum).
struct WinBlock {
    uint4 ids;
    unsigned m;
    int kb;
};
__device__ __forceinline__ WinBlock win_load(const uint4* __restrict__ wcol, const unsigned short* __restrict__ meta,
                                             const int* __restrict__ bbase, int64_t blk, int64_t end, int lane) {
    WinBlock b{};
    if (blk < end) {
        b.ids = __ldcs(wcol + blk * 32 + lane);
        b.m = __ldcs(meta + blk * 32 + lane);  // start bits | pieces started in earlier lanes << 8
        b.kb = bbase[blk];
    }
    return b;
}

#ifndef CHEB_WIN_AHEAD
#define CHEB_WIN_AHEAD 3
#endif
constexpr int kWinAhead = CHEB_WIN_AHEAD;  // blocks of the stream in flight per warp (registers)

template <class V>
__global__ void __launch_bounds__(1024, 1)
k_window_pass(const V* __restrict__ x, int64_t x_len, int H0, int W, int NW, const int64_t* __restrict__ wblk,
              const uint4* __restrict__ wcol, const unsigned short* __restrict__ meta, const int* __restrict__ bbase,
              double* __restrict__ wpart, const int64_t* __restrict__ cta, unsigned long long* stamp_start) {
    extern __shared__ __align__(16) unsigned char smem[];
    V* win = reinterpret_cast<V*>(smem);
    __shared__ __align__(8) uint64_t mbar;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    if (threadIdx.x == 0) {
        mbar_init(&mbar, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    pdl_trigger();
    pdl_wait();  // x_k comes from the previous term's kernels
    if (stamp_start && blockIdx.x == 0 && threadIdx.x == 0) *stamp_start = global_ns();
    const int64_t b0 = cta[blockIdx.x], b1 = cta[blockIdx.x + 1];
    int w = 0;
    unsigned phase = 0;
    int64_t b = b0;
    while (b < b1) {
        while (wblk[w + 1] <= b) ++w;  // b < n_blocks = wblk[NW]
        const int64_t e = min(b1, wblk[w + 1]);
        const int64_t base = (int64_t)H0 + (int64_t)w * W;
        const int cnt = (int)min((int64_t)W, x_len - base);
        // this warp's first blocks of the window: issued before the window itself lands
        WinBlock q[kWinAhead];
#pragma unroll
        for (int j = 0; j < kWinAhead; ++j) q[j] = win_load(wcol, meta, bbase, b + warp + 32 * j, e, lane);
        __syncthreads();  // the previous window's gathers are done
        const unsigned bytes = (unsigned)(cnt * sizeof(V)) & ~15u;  // base is a multiple of 8 entries: 16-byte aligned
        if (threadIdx.x == 0) {
            mbar_expect_tx(&mbar, bytes);
            constexpr unsigned kPiece = 32768;
            for (unsigned o = 0; o < bytes; o += kPiece)
                bulk_g2s(smem + o, reinterpret_cast<const unsigned char*>(x + base) + o, min(kPiece, bytes - o), &mbar);
        }
        for (int i = bytes / sizeof(V) + threadIdx.x; i < cnt; i += blockDim.x) win[i] = x[base + i];
        mbar_wait(&mbar, phase);
        phase ^= 1u;
        __syncthreads();
        for (int64_t blk = b + warp; blk < e; blk += 32 * kWinAhead) {
#pragma unroll
            for (int j = 0; j < kWinAhead; ++j) {
                if (blk + 32 * j >= e) break;
                const WinBlock cb = q[j];
                q[j] = win_load(wcol, meta, bbase, blk + 32 * (j + kWinAhead), e, lane);
                const unsigned idw[4] = {cb.ids.x, cb.ids.y, cb.ids.z, cb.ids.w};
                double v[8];
#pragma unroll
                for (int i = 0; i < 4; ++i) {
                    v[2 * i] = (double)win[idw[i] & 0xffffu];
                    v[2 * i + 1] = (double)win[idw[i] >> 16];
                }
                int k = cb.kb + (int)(cb.m >> 8) - 1;  // index of the piece the current run belongs to (once started)
                double head = 0.0, run = 0.0;
                bool started = false;
#pragma unroll
                for (int i = 0; i < 8; ++i) {
                    if ((cb.m >> i) & 1u) {
                        if (started) wpart[k] = run;
                        else head = run;
                        started = true;
                        run = 0.0;
                        ++k;
                    }
                    run += v[i];
                }
                if (!started) head = run;
                // G = this lane's leading sum + those of the following lanes up to (and
                // including) the first lane that starts a piece
                double G = head;
                const unsigned ahead = __ballot_sync(0xffffffffu, started) >> lane;  // bit j: lane + j starts a piece
#pragma unroll
                for (int o = 1; o < 32; o <<= 1) {
                    const double nv = __shfl_down_sync(0xffffffffu, G, o);
                    if (lane + o < 32 && !(ahead & ((1u << o) - 1u))) G += nv;
                }
                double Gn = __shfl_down_sync(0xffffffffu, G, 1);
                if (lane == 31) Gn = 0.0;
                if (started) wpart[k] = run + Gn;
            }
        }
        b = e;
    }
}

// ---------------- BITEXACT: thread per row, storage order ----------------------------
template <int EPI, class RP>
__global__ void __launch_bounds__(kThreads) k_term_exact(TermArgs<RP, double> a, int64_t n) {
    if (a.stamp_start && blockIdx.x == 0 && threadIdx.x == 0) *a.stamp_start = global_ns();
    for (int64_t u = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; u < n;
         u += (int64_t)gridDim.x * blockDim.x) {
        const int64_t b = a.rp[u], e = a.rp[u + 1];
        double s = 0.0;
        for (int64_t j = b; j < e; ++j) s = __dadd_rn(s, a.x_in[a.col[j]]);
        double p0 = 0.0, p1 = 0.0;
        epilogue<EPI>(a, u, s, e - b, p0, p1);
    }
    if (a.stamp_end) stamp_last_cta(a.done, a.stamp_end);
}

// Serial Kahan sums exactly as graph.cpp:10-19 (single thread: bit-identical order).
// The reference's serial compensated sums, bit for bit (graph.cpp:10-19 order, one element
// at a time).  The recurrence is inherently sequential, so one thread runs it; warps 1..7
// stage the next chunk of both inputs into shared memory meanwhile, so the chain runs at
// FP64 add latency instead of waiting on global loads.
constexpr int kSerialChunk = 1024;

template <int MODE>  // 0: Kahan(x) [, Kahan(y)]   1: power: Kahan|y - x|, Kahan(y) (power.cpp:80-93)
__global__ void __launch_bounds__(256) k_serial_sums(const double* __restrict__ a, const double* __restrict__ b,
                                                     int64_t n, double* __restrict__ out) {
    __shared__ double sa[2][kSerialChunk], sb[2][kSerialChunk];
    const int tid = threadIdx.x;
    const bool two = b != nullptr;
    auto stage = [&](int buf, int64_t base) {  // warps 1..7
        const int64_t len = n - base < kSerialChunk ? n - base : (int64_t)kSerialChunk;
        for (int64_t i = tid - 32; i < len; i += blockDim.x - 32) {
            sa[buf][i] = a[base + i];
            if (two) sb[buf][i] = b[base + i];
        }
    };
    if (tid >= 32 && n > 0) stage(0, 0);
    __syncthreads();
    double s0 = 0.0, c0 = 0.0, s1 = 0.0, c1 = 0.0;
    for (int64_t base = 0; base < n; base += kSerialChunk) {
        const int cur = (int)((base / kSerialChunk) & 1);
        if (tid >= 32 && base + kSerialChunk < n) stage(cur ^ 1, base + kSerialChunk);
        if (tid == 0) {
            const int len = (int)(n - base < kSerialChunk ? n - base : (int64_t)kSerialChunk);
#pragma unroll 4
            for (int j = 0; j < len; ++j) {
                if constexpr (MODE == 0) {
                    const double av = __dsub_rn(sa[cur][j], c0);
                    const double t = __dadd_rn(s0, av);
                    c0 = __dsub_rn(__dsub_rn(t, s0), av);
                    s0 = t;
                    if (two) {
                        const double bv = __dsub_rn(sb[cur][j], c1);
                        const double u = __dadd_rn(s1, bv);
                        c1 = __dsub_rn(__dsub_rn(u, s1), bv);
                        s1 = u;
                    }
                } else {  // a = y (new), b = x (old)
                    const double y = sa[cur][j];
                    const double d = __dsub_rn(fabs(__dsub_rn(y, sb[cur][j])), c0);
                    const double t = __dadd_rn(s0, d);
                    c0 = __dsub_rn(__dsub_rn(t, s0), d);
                    s0 = t;
                    const double av = __dsub_rn(y, c1);
                    const double u = __dadd_rn(s1, av);
                    c1 = __dsub_rn(__dsub_rn(u, s1), av);
                    s1 = u;
                }
            }
        }
        __syncthreads();
    }
    if (tid == 0) {
        out[0] = s0;
        out[1] = s1;
    }
}

// Many independent serial Kahan sums (one per thread), each in the reference's element
// order: the BITEXACT trace of all M terms after the loop (mass_T = Kahan(T_k),
// S_k = Kahan(acc_k) from per-term snapshots).  Sums of different terms do not depend on
// each other, so they run side by side; within a sum the order is the reference's.
__global__ void k_kahan_many(const double* __restrict__ snaps, int64_t n, int count, double* __restrict__ out) {
    const int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= count) return;
    const double* __restrict__ x = snaps + (size_t)t * (size_t)n;
    double s = 0.0, c = 0.0;
    int64_t i = 0;
    constexpr int U = 16;
    for (; i + U <= n; i += U) {
        double v[U];
#pragma unroll
        for (int q = 0; q < U; ++q) v[q] = __ldg(x + i + q);
#pragma unroll
        for (int q = 0; q < U; ++q) {
            const double a = __dsub_rn(v[q], c);
            const double u = __dadd_rn(s, a);
            c = __dsub_rn(__dsub_rn(u, s), a);
            s = u;
        }
    }
    for (; i < n; ++i) {
        const double a = __dsub_rn(x[i], c);
        const double u = __dadd_rn(s, a);
        c = __dsub_rn(__dsub_rn(u, s), a);
        s = u;
    }
    out[t] = s;
}

// Power rounds j = 1..nb of a speculative batch (snapshots S[0..nb] of x): thread 2(j-1)
// runs the reference's Kahan L1 change |S[j] - S[j-1]|, thread 2(j-1)+1 the Kahan mass of
// S[j] (power.cpp:80-93), each in element order.
__global__ void k_power_many(const double* __restrict__ S, int64_t n, int nb, double* __restrict__ out) {
    const int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= 2 * nb) return;
    const int j = t / 2 + 1;
    const double* __restrict__ y = S + (size_t)j * (size_t)n;
    const double* __restrict__ x = S + (size_t)(j - 1) * (size_t)n;
    double s = 0.0, c = 0.0;
    constexpr int U = 16;  // loads of the next elements are independent of the chain
    int64_t i = 0;
    if (t & 1) {
        for (; i + U <= n; i += U) {
            double v[U];
#pragma unroll
            for (int q = 0; q < U; ++q) v[q] = __ldg(y + i + q);
#pragma unroll
            for (int q = 0; q < U; ++q) {
                const double a = __dsub_rn(v[q], c);
                const double u = __dadd_rn(s, a);
                c = __dsub_rn(__dsub_rn(u, s), a);
                s = u;
            }
        }
        for (; i < n; ++i) {
            const double a = __dsub_rn(__ldg(y + i), c);
            const double u = __dadd_rn(s, a);
            c = __dsub_rn(__dsub_rn(u, s), a);
            s = u;
        }
    } else {
        for (; i + U <= n; i += U) {
            double d[U];
#pragma unroll
            for (int q = 0; q < U; ++q) d[q] = fabs(__dsub_rn(__ldg(y + i + q), __ldg(x + i + q)));
#pragma unroll
            for (int q = 0; q < U; ++q) {
                const double e = __dsub_rn(d[q], c);
                const double u = __dadd_rn(s, e);
                c = __dsub_rn(__dsub_rn(u, s), e);
                s = u;
            }
        }
        for (; i < n; ++i) {
            const double e = __dsub_rn(fabs(__dsub_rn(__ldg(y + i), __ldg(x + i))), c);
            const double u = __dadd_rn(s, e);
            c = __dsub_rn(__dsub_rn(u, s), e);
            s = u;
        }
    }
    out[t] = s;
}

// ---------------- init / reductions / normalisation ----------------------------------
// T_{-1} = T_0 = p (or 1), acc = (c0/2) T_0, x_0 = T_0 D^-1   (cpaa.cpp:88-92, :116 at k=1)
template <class RP, class V>
__global__ void k_init(const RP* __restrict__ rp, const double* __restrict__ inv,
                       const double* __restrict__ p, const int* __restrict__ order, int64_t n,
                       double half_c0, V* __restrict__ T0, V* __restrict__ T1, V* __restrict__ acc,
                       V* __restrict__ x0) {
    for (int64_t u = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; u < n;
         u += (int64_t)gridDim.x * blockDim.x) {
        const V t0 = p ? (V)p[order ? order[u] : u] : V(1);
        T0[u] = t0;
        T1[u] = t0;
        acc[u] = p ? mul_rn((V)half_c0, t0) : (V)half_c0;
        const V iv = inv ? (V)inv[u] : rcp_rn((V)(rp[u + 1] - rp[u]));
        x0[u] = mul_rn(t0, iv);
    }
}

// trace[k] = sum of block partials (+ hub partials) of term k, fixed order: kTraceThreads
// threads, each with four independent accumulators over 16-byte loads (one CTA per term read
// C4's ~1 M hub-row pairs at ~10 GB/s with one 256-thread chain of dependent adds each).
constexpr int kTraceThreads = 1024;
__device__ __forceinline__ void trace_sums(const double* __restrict__ part, int grid, const double* __restrict__ hub_ts,
                                           int n_hub, int k, double* sh, double& A, double& B) {
    const double2* pk = reinterpret_cast<const double2*>(part + (size_t)k * grid * 2);
    double a[4] = {0.0, 0.0, 0.0, 0.0}, b[4] = {0.0, 0.0, 0.0, 0.0};
    auto sweep = [&](const double2* p, int cnt) {
        const int T = blockDim.x;
        int i = threadIdx.x;
        for (; i + 3 * T < cnt; i += 4 * T) {
            double2 v[4];
#pragma unroll
            for (int j = 0; j < 4; ++j) v[j] = __ldg(p + i + j * T);
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                a[j] += v[j].x;
                b[j] += v[j].y;
            }
        }
        for (int j = 0; i < cnt; i += T, ++j) {
            const double2 v = __ldg(p + i);
            a[j & 3] += v.x;
            b[j & 3] += v.y;
        }
    };
    sweep(pk, grid);
    if (hub_ts) sweep(reinterpret_cast<const double2*>(hub_ts + (size_t)k * n_hub * 2), n_hub);
    A = block_sum((a[0] + a[1]) + (a[2] + a[3]), sh);
    B = block_sum((b[0] + b[1]) + (b[2] + b[3]), sh);
}
__global__ void __launch_bounds__(kTraceThreads) k_trace_reduce(const double* __restrict__ part, int grid,
                                                                const double* __restrict__ hub_ts, int n_hub,
                                                                int k_first, double* __restrict__ trace) {
    __shared__ double sh[32];
    const int k = k_first + blockIdx.x;
    double A, B;
    trace_sums(part, grid, hub_ts, n_hub, k, sh, A, B);
    if (threadIdx.x == 0) {
        trace[2 * k] = A;
        trace[2 * k + 1] = B;
    }
}

template <class V>
__global__ void k_sum_blocks(const V* __restrict__ x, int64_t n, double* __restrict__ part) {
    __shared__ double sh[32];
    double a = 0.0;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x)
        a += (double)x[i];
    a = block_sum(a, sh);
    if (threadIdx.x == 0) part[blockIdx.x] = a;
}

__global__ void k_sum_final(const double* __restrict__ part, int cnt, double* __restrict__ out) {
    __shared__ double sh[32];
    double a = 0.0;
    for (int i = threadIdx.x; i < cnt; i += blockDim.x) a += part[i];
    a = block_sum(a, sh);
    if (threadIdx.x == 0) *out = a;
}

// ranks[order[u]] = acc[u] / total   (cpaa.cpp:159-163).  With the inverse permutation
// (rank = old id -> view row) the same values are gathered in vertex order instead:
// ranks[v] = acc[rank[v]] / total, coalesced writes (the scatter form wrote 8 random bytes per
// vertex: C4 1.14 ms per solve).
template <class V>
__global__ void k_normalize(const V* __restrict__ acc, const int* __restrict__ order, const int* __restrict__ rank,
                            int64_t n, const double* __restrict__ total, V* __restrict__ out) {
    const double tot = *total;
    for (int64_t u = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; u < n;
         u += (int64_t)gridDim.x * blockDim.x) {
        if (rank) {
            out[u] = (V)((double)acc[rank[u]] / tot);
        } else {
            const V r = (V)((double)acc[u] / tot);
            out[order ? order[u] : u] = r;
        }
    }
}

template <class V>
__global__ void k_permute_in(const double* __restrict__ src, const int* __restrict__ order, int64_t n,
                             V* __restrict__ dst) {
    for (int64_t u = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; u < n;
         u += (int64_t)gridDim.x * blockDim.x)
        dst[u] = (V)src[order ? order[u] : u];
}

template <class V>
__global__ void k_permute_out(const V* __restrict__ src, const int* __restrict__ order, const int* __restrict__ rank,
                              int64_t n, double* __restrict__ dst) {
    for (int64_t u = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; u < n;
         u += (int64_t)gridDim.x * blockDim.x) {
        if (rank) dst[u] = (double)src[rank[u]];  // gather in vertex order (coalesced writes)
        else dst[order ? order[u] : u] = (double)src[u];
    }
}

// x = T D^-1 (staged API / transition_apply pre-scale)
template <class RP, class V>
__global__ void k_prescale(const RP* __restrict__ rp, const double* __restrict__ inv,
                           const V* __restrict__ T, int64_t n, V* __restrict__ x) {
    for (int64_t u = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; u < n;
         u += (int64_t)gridDim.x * blockDim.x) {
        const V iv = inv ? (V)inv[u] : rcp_rn((V)(rp[u + 1] - rp[u]));
        x[u] = mul_rn(T[u], iv);
    }
}

// acc += c_k T_next (cpaa.cpp:192-194)
template <class V>
__global__ void k_accumulate(V* __restrict__ acc, const V* __restrict__ Tn, int64_t n, double ck) {
    for (int64_t u = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; u < n;
         u += (int64_t)gridDim.x * blockDim.x)
        acc[u] = add_rn(acc[u], mul_rn((V)ck, Tn[u]));
}

// Per-round error vs a reference (metrics.cpp:12-30 via cpaa.cpp:149-154):
// est = acc / S_k ; max |est-ref|/ref and sum |est-ref|.  ref in the same layout.
template <class V>
__global__ void k_err(const V* __restrict__ acc, const double* __restrict__ ref, int64_t n,
                      const double* __restrict__ S, int by_S, double* __restrict__ part) {
    __shared__ double sh[32];
    const double tot = by_S ? *S : 1.0;
    double mx = 0.0, l1 = 0.0;
    for (int64_t u = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; u < n;
         u += (int64_t)gridDim.x * blockDim.x) {
        const double est = by_S ? (double)acc[u] / tot : (double)acc[u];
        const double d = fabs(est - ref[u]);
        mx = fmax(mx, d / ref[u]);
        l1 += d;
    }
    for (int o = 16; o; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = mx;
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int w = 1; w < (int)(blockDim.x >> 5); ++w) mx = fmax(mx, sh[w]);
        part[2 * blockIdx.x] = mx;
    }
    __syncthreads();
    l1 = block_sum(l1, sh);
    if (threadIdx.x == 0) part[2 * blockIdx.x + 1] = l1;
}

__global__ void k_err_final(const double* __restrict__ part, int cnt, double* __restrict__ out) {
    __shared__ double sh[32];
    double mx = 0.0, l1 = 0.0;
    for (int i = threadIdx.x; i < cnt; i += blockDim.x) {
        mx = fmax(mx, part[2 * i]);
        l1 += part[2 * i + 1];
    }
    for (int o = 16; o; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = mx;
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int w = 1; w < (int)(blockDim.x >> 5); ++w) mx = fmax(mx, sh[w]);
        out[0] = mx;
    }
    __syncthreads();
    l1 = block_sum(l1, sh);
    if (threadIdx.x == 0) out[1] = l1;
}

// =====================================================================================
// Host drivers
// =====================================================================================

inline int grid1d(int64_t n) {
    int64_t b = (n + kThreads - 1) / kThreads;
    return (int)std::max<int64_t>(1, std::min<int64_t>(b, 148 * 16));
}

// Layout the solve runs on: FAST -> degree-binned view; BITEXACT -> reference order.
struct Layout {
    bool fast;
    bool rp64;
    const void* rp;
    const int* col;
    const double* inv;
    const int* order;  // new -> old (fast) or null
    const int* rank;   // old -> new (fast, single-GPU views) or null
};

Layout layout_of(cheb_graph* g, int mode) {
    Layout L{};
    if (mode == CHEB_MODE_FAST) {
        ensure_view(g);
        L.fast = true;
        L.rp64 = g->view.rp64;
        L.rp = g->view.row_ptr.get();
        L.col = g->view.col.ptr<int>();
        L.inv = g->inv_array ? g->view.inv.ptr<double>() : nullptr;
        L.order = g->view.order.ptr<int>();
        L.rank = g->view.rank ? g->view.rank.ptr<int>() : nullptr;
    } else {
        L.fast = false;
        L.rp64 = g->rp64;
        L.rp = g->row_ptr.get();
        L.col = g->col.ptr<int>();
        L.inv = g->inv_array ? g->inv.ptr<double>() : nullptr;
        L.order = nullptr;
        L.rank = nullptr;
    }
    return L;
}

template <class RP, class V>
TermArgs<RP, V> base_args(cheb_graph* /*g*/, const Layout& L) {
    TermArgs<RP, V> a{};
    a.rp = static_cast<const RP*>(L.rp);
    a.col = L.col;
    a.inv = L.inv;
    return a;
}

// Launch one SpMV-shaped pass with epilogue EPI on the given layout.
template <int EPI, class RP, class V>
int launch_pass(cheb_graph* g, const Layout& L, const TermArgs<RP, V>& a) {
    cudaStream_t st = g->stream;
    if (L.fast) {
        // the > 48 KB dynamic shared-memory opt-in is a per-device (per-context) attribute
        static std::atomic<uint64_t> attr_set{0};  // per template instance, bit per device
        constexpr size_t smem1 = warp_smem_bytes<V, 1>(), smem2 = warp_smem_bytes<V, 2>();
        if (first_on_device(attr_set, g->device)) {
            const std::pair<const void*, size_t> fs[] = {
                {(const void*)k_term_warp<EPI, RP, V, false, 2>, smem2}, {(const void*)k_term_warp<EPI, RP, V, true, 2>, smem2},
                {(const void*)k_term_warp<EPI, RP, V, false, 1>, smem1}, {(const void*)k_term_warp<EPI, RP, V, true, 1>, smem1}};
            for (const auto& f : fs) {
                const cudaError_t e = cudaFuncSetAttribute(f.first, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)f.second);
                if (e != cudaSuccess) {
                    attr_set.fetch_and(~(uint64_t(1) << (g->device & 63)));  // retry next launch
                    CHEB_CUDA_CHECK(e);
                }
            }
        }
        // single GPU, canonical inv_degree, no push: the specialised kernel
        const bool single = !a.push && !a.inv && !(g->part.G > 1);
        // one column-id buffer per warp (more L1) when x exceeds L2, two otherwise (us/term,
        // 1 vs 2 buffers: C2 8 MB 72.2 / 68.1, C3 19 MB 369 / 361, C4 fp32 68 MB 3072 / 3017,
        // C4 fp64 136 MB 3403-3456 / 3556-3561)
        int nbuf = tuning().colbufs;
        if (nbuf != 1 && nbuf != 2) {
            int l2 = 0;
            cudaDeviceGetAttribute(&l2, cudaDevAttrL2CacheSize, g->device);
            nbuf = (int64_t)g->view.x_len * (int64_t)sizeof(V) > (int64_t)l2 ? 1 : 2;
        }
        const size_t smem = nbuf == 1 ? smem1 : smem2;
        int H = (int)std::min<int64_t>(g->n, hot_capacity<V>());
        if (tuning().hot >= 0) H = (int)std::min<int64_t>(H, tuning().hot);
        TermArgs<RP, V> ab = a;
        ab.tune_nogather = tuning().nogather;
        ab.tune_skip = tuning().skip;
        ab.tune_skipwarm = tuning().skipwarm;
        ab.prefetch = tuning().prefetch;
        ab.stream_cs = tuning().streamcs;
        if (g->view.n_hub > 0) ab.stamp_end = nullptr;  // the hub finalize ends the term
        ab.xout_hint = tuning().xout_hint;
        if (ab.xout_hint < 0) ab.xout_hint = 0;  // plain stores (Tuning::xout_hint)
        // x buffers are cudaMalloc'ed (256-B aligned): whole 128-B lines of x_out only
        ab.xdiscard_len = (EPI == EPI_CPAA && tuning().xdiscard && !a.push && g->part.G == 1 && !g->part.comm)
                              ? (g->view.x_len * (int64_t)sizeof(V) / 128) * 128 / (int64_t)sizeof(V) : 0;
        const size_t x_bytes = (size_t)std::max<int64_t>(g->view.x_len, 1) * sizeof(V);
        const bool windows_on = g->view.win.ready;
        auto launch = [&](const TermArgs<RP, V>& args, const WTile* prog, int plen, int ntiles, const V* win,
                          size_t win_bytes) {
            cudaLaunchConfig_t cfg = {};
            cfg.gridDim = dim3(g->view.grid);
            cfg.blockDim = dim3(kWarps * 32);
            cfg.dynamicSmemBytes = smem;
            cfg.stream = st;
            cudaLaunchAttribute attr[2];
            cfg.attrs = attr;
            cfg.numAttrs = 0;
            // keep the hot (degree-sorted) prefix of x_k -- or this launch's block of it --
            // resident in L2 across the launch (only when x exceeds L2)
            if (tuning().l2win && l2_window(win, win_bytes, &attr[cfg.numAttrs].val.accessPolicyWindow, x_bytes))
                attr[cfg.numAttrs++].id = cudaLaunchAttributeAccessPolicyWindow;
            // (not after a window pass: a term CTA that takes over an SM the moment a window CTA
            // leaves it keeps that kernel's shared-memory carve-out, i.e. a ~28 KB L1, and the
            // cold gathers lose their in-flight capacity: config 4 3083 -> 3728 us/term)
            if (tuning().pdl && !(windows_on && !(tuning().winskip & 8))) {  // overlap this launch + prologue with the previous kernel's tail
                attr[cfg.numAttrs].id = cudaLaunchAttributeProgrammaticStreamSerialization;
                attr[cfg.numAttrs++].val.programmaticStreamSerializationAllowed = 1;
            }
            if (nbuf == 1) {
                if (single) CHEB_CUDA_CHECK(cudaLaunchKernelEx(&cfg, k_term_warp<EPI, RP, V, true, 1>, args, prog, plen, ntiles, H));
                else CHEB_CUDA_CHECK(cudaLaunchKernelEx(&cfg, k_term_warp<EPI, RP, V, false, 1>, args, prog, plen, ntiles, H));
            } else {
                if (single) CHEB_CUDA_CHECK(cudaLaunchKernelEx(&cfg, k_term_warp<EPI, RP, V, true, 2>, args, prog, plen, ntiles, H));
                else CHEB_CUDA_CHECK(cudaLaunchKernelEx(&cfg, k_term_warp<EPI, RP, V, false, 2>, args, prog, plen, ntiles, H));
            }
        };
        int launched = 0;
        const SolverView::Windows& Wn = g->view.win;
        const bool windows = windows_on;
        if (windows) {
            // the hub rows' window pieces first (their sums land in hub_part), then the term
            // kernel over the remaining entries, then the finalize
            static std::atomic<uint64_t> wattr_set{0};
            const size_t wsmem = (size_t)Wn.W * sizeof(V);
            if (wsmem > (size_t)kWinSmemMax) fail(CHEB_INVALID_ARG, "column window larger than shared memory");
            if (first_on_device(wattr_set, g->device)) {
                const cudaError_t e = cudaFuncSetAttribute((const void*)k_window_pass<V>,
                                                           cudaFuncAttributeMaxDynamicSharedMemorySize, kWinSmemMax);
                if (e != cudaSuccess) {
                    wattr_set.fetch_and(~(uint64_t(1) << (g->device & 63)));
                    CHEB_CUDA_CHECK(e);
                }
            }
            cudaLaunchConfig_t wc = {};
            wc.gridDim = dim3((unsigned)Wn.grid);
            wc.blockDim = dim3(1024);
            wc.dynamicSmemBytes = wsmem;
            wc.stream = st;
            cudaLaunchAttribute wattr[1];
            wattr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
            wattr[0].val.programmaticStreamSerializationAllowed = 1;
            wc.attrs = wattr;
            wc.numAttrs = (tuning().pdl && !(tuning().winskip & 4)) ? 1 : 0;
            if (tuning().winskip != 1)
            CHEB_CUDA_CHECK(cudaLaunchKernelEx(&wc, k_window_pass<V>, a.x_in, g->view.x_len, Wn.H0, Wn.W, Wn.NW,
                                               (const int64_t*)Wn.wblk.ptr<int64_t>(), (const uint4*)Wn.wcol.ptr<uint4>(),
                                               (const unsigned short*)Wn.meta.ptr<unsigned short>(),
                                               (const int*)Wn.bbase.ptr<int>(), a.hub_part + Wn.MC,
                                               (const int64_t*)Wn.cta.ptr<int64_t>(), ab.stamp_start));
            ab.stamp_start = nullptr;
            if (tuning().winskip != 2) launch(ab, Wn.prog.ptr<WTile>(), Wn.prog_len, Wn.n_tiles, a.x_in, x_bytes);
            launched = 2;
        } else if (g->view.phases.empty()) {
            launch(ab, g->view.prog.ptr<WTile>(), g->view.prog_len, g->view.n_tiles, a.x_in, x_bytes);
            launched = 1;
        } else {
            // column-blocked schedule (build.cu column_block_schedule): one launch per block
            // of x, chunk-only launches first; the last one runs the pack tiles and epilogues
            for (const SolverView::Phase& ph : g->view.phases) {
                if (ph.ntiles == 0 && !ph.epi) continue;
                TermArgs<RP, V> pa = ab;
                if (launched > 0) {  // once per term: start stamp, dead-line discard
                    pa.stamp_start = nullptr;
                    pa.xdiscard_len = 0;
                }
                if (!ph.epi) {
                    pa.part = nullptr;
                    pa.stamp_end = nullptr;
                }
                launch(pa, g->view.prog.ptr<WTile>() + ph.prog_off, ph.prog_len, ph.ntiles, a.x_in + ph.x_lo,
                       (size_t)(ph.x_hi - ph.x_lo) * sizeof(V));
                ++launched;
            }
        }
        if (g->view.n_hub > 0 && tuning().winskip != 3) {
            CHEB_CUDA_CHECK(cudaGetLastError());
            const int64_t n_wide = tuning().hubwarp ? g->view.n_hub : windows ? Wn.n_wide : g->view.n_hub_wide;
            const int64_t hub_warps = n_wide + (g->view.n_hub - n_wide + 31) / 32;
            const int hb = (int)std::max<int64_t>(1, std::min<int64_t>((hub_warps * 32 + 255) / 256, 148 * 16));
            cudaLaunchConfig_t hc = {};
            hc.gridDim = dim3(hb);
            hc.blockDim = dim3(256);
            hc.stream = st;
            cudaLaunchAttribute hattr[1];
            hattr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
            hattr[0].val.programmaticStreamSerializationAllowed = 1;
            hc.attrs = hattr;
            hc.numAttrs = (tuning().pdl && !(windows_on && (tuning().winskip & 16))) ? 1 : 0;
            CHEB_CUDA_CHECK(cudaLaunchKernelEx(&hc, k_hub_finalize<EPI, RP, V>, a,
                                               windows ? (const int*)Wn.hub_first.ptr<int>()
                                                       : (const int*)g->view.hub_first.ptr<int>(),
                                               g->view.n_hub, n_wide, windows ? (const int*)Wn.kf.ptr<int>() : (const int*)nullptr,
                                               windows ? (const int*)Wn.klist.ptr<int>() : (const int*)nullptr,
                                               (const double*)(a.hub_part + (windows ? Wn.MC : 0))));
            return launched + 1;
        }
        CHEB_CUDA_CHECK(cudaGetLastError());
        return launched;
    } else {
        if constexpr (std::is_same<V, double>::value) {
            k_term_exact<EPI, RP><<<grid1d(g->n), kThreads, 0, st>>>(a, g->n);
        } else {
            fail(CHEB_INVALID_ARG, "bitexact mode is fp64 only");
        }
    }
    CHEB_CUDA_CHECK(cudaGetLastError());
    return 1;
}

template <class V>
void ensure_workspace(cheb_graph* g, int M, int R) {
    Workspace& w = g->ws;
    const int64_t n = g->n;
    // Any reallocation invalidates the captured solve graph (it bakes in addresses).
    const void* before[] = {w.T0.get(), w.T1.get(), w.X0.get(), w.X1.get(), w.acc.get(), w.out.get(),
                            w.part.get(), w.hub_part.get(), w.hub_ts.get(),
                            w.trace.get(), w.total.get(), w.stamps.get(), w.done.get()};
    const int64_t vlen = std::max<int64_t>(std::max<int64_t>(n, g->view.x_len), 1);
    const size_t vb = sizeof(V) * (size_t)vlen * R;
    w.T0.ensure(vb);
    w.T1.ensure(vb);
    w.X0.ensure(vb);
    w.X1.ensure(vb);
    w.acc.ensure(vb);
    w.out.ensure(vb);
    const int grid = std::max(g->view.ready ? g->view.grid : 1, grid1d(n));
    w.part.ensure(sizeof(double) * 2 * (size_t)std::max(M, 1) * std::max(grid, 1));
    w.hub_part.ensure(sizeof(double) * (size_t)std::max<int64_t>(
                          std::max<int64_t>(g->view.n_tiles, g->view.win.ready ? g->view.win.n_slots : 0), 1));
    w.hub_ts.ensure(sizeof(double) * 2 * (size_t)std::max(M, 1) * std::max<int64_t>(g->view.n_hub, 1));
    w.trace.ensure(sizeof(double) * 2 * (size_t)std::max(M, 1));
    w.total.ensure(sizeof(double) * 4);
    w.stamps.ensure(sizeof(unsigned long long) * ((size_t)std::max(M, 1) + 1));
    w.done.ensure(sizeof(unsigned) * ((size_t)std::max(M, 1) + 1));
    w.n = n;
    w.R = R;
    w.vbytes = sizeof(V);
    const void* after[] = {w.T0.get(), w.T1.get(), w.X0.get(), w.X1.get(), w.acc.get(), w.out.get(),
                           w.part.get(), w.hub_part.get(), w.hub_ts.get(),
                           w.trace.get(), w.total.get(), w.stamps.get(), w.done.get()};
    if (std::memcmp(before, after, sizeof before) != 0) {
        if (w.exec) cudaGraphExecDestroy(w.exec);
        w.exec = nullptr;
        w.exec_key.clear();
        w.seen_key.clear();
    }
}

// BITEXACT trace snapshots (2 M n doubles) when they fit a quarter of the free memory (and
// 8 GB); otherwise the per-term serial sums run instead.
void ensure_snapshots(cheb_graph* g, int M) {
    Workspace& w = g->ws;
    const size_t need = sizeof(double) * 2 * (size_t)M * (size_t)g->n;
    if (w.snap.bytes() >= need) return;
    size_t free_b = 0, total_b = 0;
    if (cudaMemGetInfo(&free_b, &total_b) != cudaSuccess) return;
    if (need > free_b / 4 || need > (size_t(8) << 30)) return;
    w.snap.alloc(need);
    if (w.exec) cudaGraphExecDestroy(w.exec);  // a captured solve baked the old pointers in
    w.exec = nullptr;
    w.exec_key.clear();
    w.seen_key.clear();
}

// Enqueue the whole solve: init, M fused terms, trace reduction, normalisation.
}  // namespace
}  // namespace chebgpu
