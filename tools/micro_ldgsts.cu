// Micro-benchmark: does the L1 capacity left next to the shared-memory reservation bound the
// random-gather rate (LDG stages every in-flight load in the L1 data array), and do LDGSTS
// (cp.async global -> shared) gathers escape that bound?  148 persistent CTAs x 1024 threads,
// each lane keeps U gathers in flight; table of N doubles; index stream coalesced.
// Build: nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o build/micro_ldgsts tools/micro_ldgsts.cu
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <cuda_runtime.h>

#ifndef UU
#define UU 4
#endif
constexpr int U = UU;

__global__ void __launch_bounds__(1024, 1) k_ldg(const double* __restrict__ x, const int* __restrict__ idx, int64_t m,
                                                 double* out, int reserve) {
    extern __shared__ double pad[];
    if (reserve && threadIdx.x == 0) pad[0] = 0;
    const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    double s = 0;
    for (int64_t i = t; i < m; i += stride * U) {
        int c[U];
#pragma unroll
        for (int q = 0; q < U; ++q) { const int64_t j = i + q * stride; c[q] = j < m ? __ldcs(idx + j) : 0; }
        double v[U];
#pragma unroll
        for (int q = 0; q < U; ++q) v[q] = __ldg(x + c[q]);
#pragma unroll
        for (int q = 0; q < U; ++q) s += v[q];
    }
    out[t] = s;
}

__device__ __forceinline__ void cp16(unsigned dst, const void* src) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" :: "r"(dst), "l"(src) : "memory");
}
__device__ __forceinline__ void cp8(unsigned dst, const void* src) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" :: "r"(dst), "l"(src) : "memory");
}

// LDGSTS gathers into a per-lane staging ring of 2 x U slots (16 B each), double-buffered:
// batch b+1 is issued before batch b is consumed.  MODE 0: .cg 16-byte (aligned pair holding
// x[c]); MODE 1: .ca 8-byte.
template <int MODE>
__global__ void __launch_bounds__(1024, 1) k_ldgsts(const double* __restrict__ x, const int* __restrict__ idx, int64_t m,
                                                    double* out) {
    extern __shared__ __align__(16) unsigned char sm[];
    const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    // slot (buf, q) of this lane at sm + ((buf * U + q) * blockDim + tid) * 16: a warp's slots are contiguous
    const unsigned base = (unsigned)__cvta_generic_to_shared(sm);
    auto slot = [&](int buf, int q) { return base + (unsigned)(((buf * U + q) * blockDim.x + threadIdx.x) * 16); };
    double s = 0;
    int cprev[U];
    int buf = 0;
    int64_t i = t;
    bool have = false;
    for (;; i += stride * U) {
        const bool more = i < m;
        int c[U];
        if (more) {
#pragma unroll
            for (int q = 0; q < U; ++q) {
                const int64_t j = i + q * stride;
                c[q] = j < m ? __ldcs(idx + j) : 0;
                if (MODE == 0) cp16(slot(buf, q), x + (c[q] & ~1));
                else cp8(slot(buf, q), x + c[q]);
            }
        }
        asm volatile("cp.async.commit_group;" ::: "memory");
        if (have) {
            asm volatile("cp.async.wait_group 1;" ::: "memory");
#pragma unroll
            for (int q = 0; q < U; ++q) {
                double v;
                const unsigned a = slot(buf ^ 1, q) + (MODE == 0 ? (cprev[q] & 1) * 8 : 0);
                asm volatile("ld.shared.f64 %0, [%1];" : "=d"(v) : "r"(a));
                s += v;
            }
        }
        if (!more) break;
#pragma unroll
        for (int q = 0; q < U; ++q) cprev[q] = c[q];
        have = true;
        buf ^= 1;
    }
    asm volatile("cp.async.wait_group 0;" ::: "memory");
    out[t] = s;
}

int main() {
    const int64_t m = 40000000;
    std::vector<int> Ns = {1 << 20, 1 << 23, 17060846};
    int* d_idx; double* d_x; double* d_out;
    cudaMalloc(&d_idx, m * 4);
    cudaMalloc(&d_x, (size_t)17060846 * 8 + 64);
    cudaMalloc(&d_out, 148 * 1024 * 8);
    cudaMemset(d_x, 0, (size_t)17060846 * 8);
    std::vector<int> h(m);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    cudaFuncSetAttribute(k_ldg, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
    cudaFuncSetAttribute(k_ldgsts<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
    cudaFuncSetAttribute(k_ldgsts<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
    for (int N : Ns) {
        srand(1);
        for (int64_t i = 0; i < m; ++i) h[i] = (int)(((uint64_t)rand() * 2654435761ull + i * 40503ull) % N);
        cudaMemcpy(d_idx, h.data(), m * 4, cudaMemcpyHostToDevice);
        auto run = [&](const char* name, int kb, auto launch) {
            for (int w = 0; w < 3; ++w) launch();
            cudaEventRecord(a);
            for (int r = 0; r < 5; ++r) launch();
            cudaEventRecord(b);
            cudaEventSynchronize(b);
            float ms;
            cudaEventElapsedTime(&ms, a, b);
            const double us = ms * 1000.0 / 5;
            cudaError_t e = cudaGetLastError();
            printf("N=%9d %-14s smem %3d KB %9.1f us  %7.1f Ggather/s %s\n", N, name, kb, us, m / (us * 1e3),
                   e ? cudaGetErrorString(e) : "");
        };
        for (int kb : {0, 100, 164, 200})
            run("ldg", kb, [&] { k_ldg<<<148, 1024, kb * 1024>>>(d_x, d_idx, m, d_out, kb); });
        const int st = 2 * U * 1024 * 16 / 1024;  // staging KB (the rest of the reservation is padding)
        for (int kb : {st, 164, 200, 220}) {
            if (kb < st) continue;
            run("ldgsts.cg16", kb, [&] { k_ldgsts<0><<<148, 1024, kb * 1024>>>(d_x, d_idx, m, d_out); });
            run("ldgsts.ca8", kb, [&] { k_ldgsts<1><<<148, 1024, kb * 1024>>>(d_x, d_idx, m, d_out); });
        }
    }
    return 0;
}
