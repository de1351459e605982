// profile.cu -- per-depth-bin total intensity (the paper's second output array,
// image_set.depth_intensity.v[i]; kernel argument image_depth_intensity,
// P:L373): profile[m] = sum over the plan's pixels of out[m][row][col].
// One CTA per depth plane, vectorised 16-byte loads, fp64 accumulation.
#include <cuda_runtime.h>
#include <stdint.h>

#include "daxm_internal.cuh"

namespace daxm {
namespace {

__global__ void __launch_bounds__(512) depth_profile_kernel(const float* __restrict__ out, size_t plane,
                                                            double* __restrict__ profile) {
    const float* p = out + (size_t)blockIdx.x * plane;
    double acc = 0.0;
    const size_t n4 = ((reinterpret_cast<uintptr_t>(p) & 15) == 0) ? plane / 4 : 0;
    const float4* p4 = reinterpret_cast<const float4*>(p);
    for (size_t i = threadIdx.x; i < n4; i += blockDim.x) {
        const float4 v = __ldcs(p4 + i);  // streamed once: evict-first
        acc += ((double)v.x + (double)v.y) + ((double)v.z + (double)v.w);
    }
    for (size_t i = n4 * 4 + threadIdx.x; i < plane; i += blockDim.x) acc += (double)p[i];
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    __shared__ double warp_sum[16];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (lane == 0) warp_sum[warp] = acc;
    __syncthreads();
    if (warp == 0) {
        acc = lane < (int)(blockDim.x >> 5) ? warp_sum[lane] : 0.0;
        for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
        if (lane == 0) profile[blockIdx.x] = acc;
    }
}

// The fused epilogue's second half: the row kernel leaves each row tile's per-plane sum in
// part[rt][m]; one thread per plane adds the tiles' sums in tile order (coalesced over m).
__global__ void __launch_bounds__(256) profile_reduce_kernel(const float* __restrict__ part, int rt0, int n, int M,
                                                             double* __restrict__ profile) {
    const int m = blockIdx.x * blockDim.x + threadIdx.x;
    if (m >= M) return;
    double acc = 0.0;
    const float* p = part + (size_t)rt0 * M + m;
    for (int t = 0; t < n; ++t) acc += (double)__ldcs(p + (size_t)t * M);
    profile[m] = acc;
}

}  // namespace

cudaError_t launch_profile_reduce(const float* part, int rt0, int n, int M, double* profile, cudaStream_t st) {
    if (M <= 0) return cudaSuccess;
    profile_reduce_kernel<<<(M + 255) / 256, 256, 0, st>>>(part, rt0, n, M, profile);
    return cudaGetLastError();
}

cudaError_t launch_depth_profile(const float* out, int M, size_t plane, double* profile, cudaStream_t st) {
    if (M <= 0) return cudaSuccess;
    depth_profile_kernel<<<M, 512, 0, st>>>(out, plane, profile);
    return cudaGetLastError();
}

}  // namespace daxm
