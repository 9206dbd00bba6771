// Device helpers shared by the term kernels (cpaa.cu) and the batched kernels (spmm.cu).
#pragma once

#include <cuda_runtime.h>

namespace chebgpu {

// Arithmetic with the reference's rounding: explicit round-to-nearest, no contraction.
__device__ __forceinline__ double mul_rn(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ float mul_rn(float a, float b) { return __fmul_rn(a, b); }
__device__ __forceinline__ double add_rn(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ float add_rn(float a, float b) { return __fadd_rn(a, b); }
__device__ __forceinline__ double sub_rn(double a, double b) { return __dsub_rn(a, b); }
__device__ __forceinline__ float sub_rn(float a, float b) { return __fsub_rn(a, b); }
__device__ __forceinline__ double rcp_rn(double d) { return __drcp_rn(d); }
__device__ __forceinline__ float rcp_rn(float d) { return __frcp_rn(d); }

template <class V>
__device__ __forceinline__ V ldg_x(const V* p) { return __ldg(p); }
__device__ __forceinline__ int ld_stream(const int* p) { return __ldcs(p); }

__device__ __forceinline__ double warp_sum(double v) {
    for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}
__device__ __forceinline__ float warp_sum(float v) {
    for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

// Fixed-order block reduction; result valid in thread 0.  sh >= 32 doubles.
template <class T>
__device__ __forceinline__ T block_sum(T v, T* sh) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    v = warp_sum(v);
    if (lane == 0) sh[warp] = v;
    __syncthreads();
    if (warp == 0) {
        v = lane < (int)(blockDim.x >> 5) ? sh[lane] : T(0);
        v = warp_sum(v);
    }
    __syncthreads();
    return v;
}


template <class V>
__device__ __forceinline__ V warp_sum_all(V v) {
#pragma unroll
    for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

}  // namespace chebgpu
