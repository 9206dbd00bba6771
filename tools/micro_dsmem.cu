// Microbenchmark: random 8-byte gathers from a table distributed over the shared memory
// of a thread-block cluster (DSMEM), vs local shared memory and L2.  Informs whether a
// cluster-wide hot-x cache pays on B200.
#include <cooperative_groups.h>
#include <cstdint>
#include <cstdio>
#include <vector>
#include <cuda_runtime.h>
namespace cg = cooperative_groups;
constexpr int G = 16;
constexpr int S = 16384;  // doubles per CTA (128 KB)

template <int CL>
__global__ void __cluster_dims__(CL, 1, 1) k_dsmem(const double* __restrict__ x, const int* __restrict__ idx,
                                                   int64_t m, double* out) {
    extern __shared__ double tab[];
    cg::cluster_group cl = cg::this_cluster();
    const int rank = cl.block_rank();
    for (int i = threadIdx.x; i < S; i += blockDim.x) tab[i] = x[rank * S + i];
    cl.sync();
    double* parts[CL];
#pragma unroll
    for (int r = 0; r < CL; ++r) parts[r] = cl.map_shared_rank(tab, r);
    int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    int64_t stride = (int64_t)gridDim.x * blockDim.x;
    double s = 0;
    for (int64_t i = t; i < m; i += stride * G) {
        int c[G];
#pragma unroll
        for (int q = 0; q < G; ++q) { int64_t j = i + q * stride; c[q] = j < m ? __ldcs(idx + j) : 0; }
#pragma unroll
        for (int q = 0; q < G; ++q) {
            const int v = c[q] & (CL * S - 1);
            s += parts[v / S][v % S];
        }
    }
    out[t] = s;
    cl.sync();
}

int main() {
    const int64_t m = 20000000;
    int* d_idx; double* d_x; double* d_out;
    cudaMalloc(&d_idx, m * 4);
    cudaMalloc(&d_x, (size_t)8 * S * 8);
    cudaMalloc(&d_out, 148 * 2048 * 8 * 8);
    cudaMemset(d_x, 0, (size_t)8 * S * 8);
    std::vector<int> h(m);
    srand(1);
    for (int64_t i = 0; i < m; ++i) h[i] = (int)(((uint64_t)rand() * 2654435761ull + i * 40503ull) & 0x7fffffff);
    cudaMemcpy(d_idx, h.data(), m * 4, cudaMemcpyHostToDevice);
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    auto run = [&](const char* name, auto launch) {
        for (int w = 0; w < 3; ++w) launch();
        cudaEventRecord(a);
        for (int r = 0; r < 10; ++r) launch();
        cudaEventRecord(b); cudaEventSynchronize(b);
        float ms; cudaEventElapsedTime(&ms, a, b);
        double us = ms * 100.0;
        cudaError_t e = cudaGetLastError();
        printf("%-12s %8.1f us/20M  %7.1f Ggather/s %s\n", name, us, m / (us * 1e3), e ? cudaGetErrorString(e) : "");
    };
    const size_t smem = S * 8;
    cudaFuncSetAttribute(k_dsmem<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaFuncSetAttribute(k_dsmem<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaFuncSetAttribute(k_dsmem<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaFuncSetAttribute(k_dsmem<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    run("cluster1", [&] { k_dsmem<1><<<148, 1024, smem>>>(d_x, d_idx, m, d_out); });
    run("cluster2", [&] { k_dsmem<2><<<148, 1024, smem>>>(d_x, d_idx, m, d_out); });
    run("cluster4", [&] { k_dsmem<4><<<144, 1024, smem>>>(d_x, d_idx, m, d_out); });
    run("cluster8", [&] { k_dsmem<8><<<144, 1024, smem>>>(d_x, d_idx, m, d_out); });
    return 0;
}
