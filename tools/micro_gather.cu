// Microbenchmark: throughput of random 8-byte gathers on B200 through different paths.
// Each thread performs G gathers from a table of N doubles at precomputed random indices
// (index stream coalesced).  Reports giga-gathers/s.  Used to pick the x-gather path of
// the CPAA term kernel (profiles/ notes).
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <cuda_runtime.h>

constexpr int G = 16;

__global__ void k_ldg(const double* __restrict__ x, const int* __restrict__ idx, int64_t m, double* out) {
    int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    int64_t stride = (int64_t)gridDim.x * blockDim.x;
    double s = 0;
    for (int64_t i = t; i < m; i += stride * G) {
        int c[G];
#pragma unroll
        for (int q = 0; q < G; ++q) { int64_t j = i + q * stride; c[q] = j < m ? idx[j] : 0; }
#pragma unroll
        for (int q = 0; q < G; ++q) s += x[c[q]];
    }
    out[t] = s;
}
__global__ void k_ldg_nc(const double* __restrict__ x, const int* __restrict__ idx, int64_t m, double* out) {
    int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    int64_t stride = (int64_t)gridDim.x * blockDim.x;
    double s = 0;
    for (int64_t i = t; i < m; i += stride * G) {
        int c[G];
#pragma unroll
        for (int q = 0; q < G; ++q) { int64_t j = i + q * stride; c[q] = j < m ? __ldcs(idx + j) : 0; }
#pragma unroll
        for (int q = 0; q < G; ++q) s += __ldg(x + c[q]);
    }
    out[t] = s;
}
__global__ void k_ldg_cg(const double* __restrict__ x, const int* __restrict__ idx, int64_t m, double* out) {
    int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    int64_t stride = (int64_t)gridDim.x * blockDim.x;
    double s = 0;
    for (int64_t i = t; i < m; i += stride * G) {
        int c[G];
#pragma unroll
        for (int q = 0; q < G; ++q) { int64_t j = i + q * stride; c[q] = j < m ? __ldcs(idx + j) : 0; }
#pragma unroll
        for (int q = 0; q < G; ++q) s += __ldcg(x + c[q]);
    }
    out[t] = s;
}
__global__ void k_tex(cudaTextureObject_t tx, const int* __restrict__ idx, int64_t m, double* out) {
    int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    int64_t stride = (int64_t)gridDim.x * blockDim.x;
    double s = 0;
    for (int64_t i = t; i < m; i += stride * G) {
        int c[G];
#pragma unroll
        for (int q = 0; q < G; ++q) { int64_t j = i + q * stride; c[q] = j < m ? __ldcs(idx + j) : 0; }
#pragma unroll
        for (int q = 0; q < G; ++q) { int2 v = tex1Dfetch<int2>(tx, c[q]); s += __hiloint2double(v.y, v.x); }
    }
    out[t] = s;
}
// shared-memory table of S doubles, indices taken mod S
template <int S>
__global__ void k_lds(const double* __restrict__ x, const int* __restrict__ idx, int64_t m, double* out) {
    extern __shared__ double tab[];
    for (int i = threadIdx.x; i < S; i += blockDim.x) tab[i] = x[i];
    __syncthreads();
    int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    int64_t stride = (int64_t)gridDim.x * blockDim.x;
    double s = 0;
    for (int64_t i = t; i < m; i += stride * G) {
        int c[G];
#pragma unroll
        for (int q = 0; q < G; ++q) { int64_t j = i + q * stride; c[q] = j < m ? __ldcs(idx + j) : 0; }
#pragma unroll
        for (int q = 0; q < G; ++q) s += tab[c[q] & (S - 1)];
    }
    out[t] = s;
}
// float table
__global__ void k_ldg_f32(const float* __restrict__ x, const int* __restrict__ idx, int64_t m, double* out) {
    int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    int64_t stride = (int64_t)gridDim.x * blockDim.x;
    float s = 0;
    for (int64_t i = t; i < m; i += stride * G) {
        int c[G];
#pragma unroll
        for (int q = 0; q < G; ++q) { int64_t j = i + q * stride; c[q] = j < m ? __ldcs(idx + j) : 0; }
#pragma unroll
        for (int q = 0; q < G; ++q) s += __ldg(x + c[q]);
    }
    out[t] = s;
}
// sorted-within-warp indices (locality): same as k_ldg_nc but idx pre-sorted in blocks of 32
int main(int argc, char** argv) {
    const int64_t m = 20000000;
    std::vector<int> Ns = {1 << 14, 1 << 17, 1 << 20, 1 << 22, 1 << 24};
    int* d_idx; double* d_x; double* d_out; float* d_xf;
    cudaMalloc(&d_idx, m * 4);
    cudaMalloc(&d_x, (size_t)(1 << 24) * 8);
    cudaMalloc(&d_xf, (size_t)(1 << 24) * 4);
    cudaMalloc(&d_out, 148 * 2048 * 8 * 8);
    cudaMemset(d_x, 0, (size_t)(1 << 24) * 8);
    std::vector<int> h(m);
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    int grid = 148 * 8, threads = 256;
    for (int N : Ns) {
        srand(1);
        for (int64_t i = 0; i < m; ++i) h[i] = (int)(((uint64_t)rand() * 2654435761ull + i * 40503ull) % N);
        cudaMemcpy(d_idx, h.data(), m * 4, cudaMemcpyHostToDevice);
        cudaTextureObject_t tx;
        cudaResourceDesc rd = {}; rd.resType = cudaResourceTypeLinear; rd.res.linear.devPtr = d_x;
        rd.res.linear.desc = cudaCreateChannelDesc<int2>(); rd.res.linear.sizeInBytes = (size_t)N * 8;
        cudaTextureDesc td = {}; td.readMode = cudaReadModeElementType;
        cudaCreateTextureObject(&tx, &rd, &td, nullptr);
        auto run = [&](const char* name, auto launch) {
            for (int w = 0; w < 3; ++w) launch();
            cudaEventRecord(a);
            for (int r = 0; r < 10; ++r) launch();
            cudaEventRecord(b); cudaEventSynchronize(b);
            float ms; cudaEventElapsedTime(&ms, a, b);
            double us = ms * 100.0;
            printf("N=%9d %-10s %8.1f us/20M  %7.1f Ggather/s\n", N, name, us, m / (us * 1e3));
        };
        run("ldg", [&] { k_ldg<<<grid, threads>>>(d_x, d_idx, m, d_out); });
        run("ldg.nc", [&] { k_ldg_nc<<<grid, threads>>>(d_x, d_idx, m, d_out); });
        run("ldg.cg", [&] { k_ldg_cg<<<grid, threads>>>(d_x, d_idx, m, d_out); });
        run("tex", [&] { k_tex<<<grid, threads>>>(tx, d_idx, m, d_out); });
        run("ldg.f32", [&] { k_ldg_f32<<<grid, threads>>>(d_xf, d_idx, m, d_out); });
        cudaFuncSetAttribute(k_lds<16384>, cudaFuncAttributeMaxDynamicSharedMemorySize, 131072);
        run("lds16K", [&] { k_lds<16384><<<148, 1024, 131072>>>(d_x, d_idx, m, d_out); });
        cudaFuncSetAttribute(k_lds<4096>, cudaFuncAttributeMaxDynamicSharedMemorySize, 32768);
        run("lds4K", [&] { k_lds<4096><<<148 * 4, 512, 32768>>>(d_x, d_idx, m, d_out); });
        cudaDestroyTextureObject(tx);
        cudaError_t e = cudaGetLastError();
        if (e) printf("err %s\n", cudaGetErrorString(e));
    }
    return 0;
}
