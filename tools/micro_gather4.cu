// Micro-benchmark: random-row gather throughput on one B200 from an L2-resident table.
//   (1) LDG: every lane gathers U random 8-byte elements per step (the term kernel's cold path)
//   (2) TMA tile::gather4: every lane issues one cp.async.bulk.tensor gather4 per step (4 random
//       16-byte rows -> 64 B of shared memory), STAGES steps in flight per lane
// Usage: micro_gather4 [rows_log2=19] [warps=32]
// Build: nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o build/micro_gather4 tools/micro_gather4.cu
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>

#include <cstdio>
#include <cstdlib>
#include <vector>

#define CK(x)                                                                                   \
    do {                                                                                        \
        cudaError_t e_ = (x);                                                                   \
        if (e_ != cudaSuccess) {                                                                \
            fprintf(stderr, "%s:%d %s: %s\n", __FILE__, __LINE__, #x, cudaGetErrorString(e_)); \
            exit(1);                                                                            \
        }                                                                                       \
    } while (0)

constexpr int STAGES = 2;

__device__ __forceinline__ unsigned smem_u32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }

__global__ void k_ldg(const double* __restrict__ x, const int* __restrict__ idx, long long n_idx, int steps,
                      double* out) {
    constexpr int U = 8;
    const long long tid = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    const long long nth = (long long)gridDim.x * blockDim.x;
    double acc = 0;
    for (int s = 0; s < steps; ++s) {
        const long long base = ((long long)s * nth + tid) * U % (n_idx - U);
        int c[U];
#pragma unroll
        for (int q = 0; q < U; ++q) c[q] = __ldg(idx + base + q);
        double v[U];
#pragma unroll
        for (int q = 0; q < U; ++q) v[q] = __ldg(x + 2 * (long long)c[q]);
#pragma unroll
        for (int q = 0; q < U; ++q) acc += v[q];
    }
    if (acc == 12345.0) out[0] = acc;
}

__global__ void k_gather4(const __grid_constant__ CUtensorMap tmap, const int* __restrict__ idx, long long n_idx,
                          int steps, double* out) {
    extern __shared__ __align__(128) unsigned char smem[];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int nwarps = blockDim.x >> 5;
    // per lane: STAGES slots of 64 B and STAGES mbarriers
    unsigned char* slots = smem + (size_t)(warp * 32 + lane) * STAGES * 128;  // TMA dst: 128 B aligned
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + (size_t)nwarps * 32 * STAGES * 128) + (warp * 32 + lane) * STAGES;
    for (int s = 0; s < STAGES; ++s)
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(bars + s)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    __syncwarp();
    const long long tid = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    const long long nth = (long long)gridDim.x * blockDim.x;
    double acc = 0;
    for (int s = 0; s < steps; ++s) {
        const int st = s % STAGES;
        if (s >= STAGES) {  // wait for this slot's previous gather, consume it
            const unsigned par = ((s / STAGES) - 1) & 1;
            asm volatile(
                "{\n.reg .pred p;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W_%=;\n}\n" ::"r"(
                    smem_u32(bars + st)),
                "r"(par)
                : "memory");
            acc += reinterpret_cast<const double*>(slots + st * 128)[0];
        }
        const long long base = ((long long)s * nth + tid) * 4 % (n_idx - 4);
        const int4 r = *reinterpret_cast<const int4*>(idx + (base & ~3ll));
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], 64;" ::"r"(smem_u32(bars + st)) : "memory");
        asm volatile(
            "cp.async.bulk.tensor.2d.shared::cluster.global.tile::gather4.mbarrier::complete_tx::bytes"
            " [%0], [%1, {%2, %3, %4, %5, %6}], [%7];" ::"r"(smem_u32(slots + st * 128)),
            "l"(reinterpret_cast<uint64_t>(&tmap)), "r"(0), "r"(r.x), "r"(r.y), "r"(r.z), "r"(r.w),
            "r"(smem_u32(bars + st))
            : "memory");
    }
    for (int s = steps; s < steps + STAGES && s >= STAGES; ++s) {
        const int st = s % STAGES;
        const unsigned par = ((s / STAGES) - 1) & 1;
        asm volatile(
            "{\n.reg .pred p;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W_%=;\n}\n" ::"r"(
                smem_u32(bars + st)),
            "r"(par)
            : "memory");
    }
    if (acc == 12345.0) out[0] = acc;
}

int main(int argc, char** argv) {
    const int lg = argc > 1 ? atoi(argv[1]) : 19;
    const int warps = argc > 2 ? atoi(argv[2]) : 32;
    const long long rows = 1ll << lg;  // 16-byte rows (2 doubles)
    const long long n_idx = 1ll << 26;
    double* x;
    int* idx;
    double* out;
    CK(cudaMalloc(&x, rows * 16));
    CK(cudaMalloc(&idx, n_idx * 4));
    CK(cudaMalloc(&out, 8));
    CK(cudaMemset(x, 0, rows * 16));
    std::vector<int> h(n_idx);
    unsigned long long s = 88172645463325252ull;
    for (auto& v : h) {
        s ^= s << 13;
        s ^= s >> 7;
        s ^= s << 17;
        v = (int)(s % rows);
    }
    CK(cudaMemcpy(idx, h.data(), n_idx * 4, cudaMemcpyHostToDevice));

    PFN_cuTensorMapEncodeTiled_v12000 encode = nullptr;
    cudaDriverEntryPointQueryResult q;
    CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", reinterpret_cast<void**>(&encode), cudaEnableDefault, &q));
    CUtensorMap tm;
    cuuint64_t gdim[2] = {2, (cuuint64_t)rows};
    cuuint64_t gstride[1] = {16};
    cuuint32_t box[2] = {2, 1};
    cuuint32_t estr[2] = {1, 1};
    CUresult cr = encode(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, x, gdim, gstride, box, estr,
                         CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE,
                         CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (cr != CUDA_SUCCESS) {
        fprintf(stderr, "cuTensorMapEncodeTiled failed: %d\n", (int)cr);
        return 1;
    }
    int sms = 0;
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
    cudaEvent_t a, b;
    CK(cudaEventCreate(&a));
    CK(cudaEventCreate(&b));
    const int threads = warps * 32;
    const int steps = 256;
    // LDG
    for (int rep = 0; rep < 3; ++rep) {
        CK(cudaEventRecord(a));
        k_ldg<<<sms, threads>>>(x, idx, n_idx, steps, out);
        CK(cudaEventRecord(b));
        CK(cudaEventSynchronize(b));
        float ms;
        CK(cudaEventElapsedTime(&ms, a, b));
        const double g = (double)sms * threads * steps * 8;
        if (rep) printf("LDG     rows=2^%d warps=%d: %.1f G gathers/s (%.3f ms)\n", lg, warps, g / ms / 1e6, ms);
    }
    const size_t smem = (size_t)threads * STAGES * 128 + (size_t)threads * STAGES * 8;
    CK(cudaFuncSetAttribute(k_gather4, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    for (int rep = 0; rep < 3; ++rep) {
        CK(cudaEventRecord(a));
        k_gather4<<<sms, threads, smem>>>(tm, idx, n_idx, steps, out);
        CK(cudaGetLastError());
        CK(cudaEventRecord(b));
        CK(cudaEventSynchronize(b));
        float ms;
        CK(cudaEventElapsedTime(&ms, a, b));
        const double g = (double)sms * threads * steps * 4;
        if (rep) printf("gather4 rows=2^%d warps=%d: %.1f G rows/s (%.3f ms)\n", lg, warps, g / ms / 1e6, ms);
    }
    return 0;
}
