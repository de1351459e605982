// select.cu -- "pixel percentage": the intensity cutoff that keeps a given
// fraction of the plan's pixels, i.e. the k-th largest first-step intensity I_0(p)
// (reading R14), found exactly by a most-significant-digit radix select over an
// order-preserving integer key (8-bit digits, shared-memory histograms).
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>
#include <string.h>

#include "daxm_internal.cuh"

namespace daxm {
namespace {

// order-preserving key: u16 -> value; f32 -> sign-flipped bits (NaN ranks lowest)
__device__ __forceinline__ uint32_t key_of(uint16_t v) { return v; }
__device__ __forceinline__ uint32_t key_of(float v) {
    if (v != v) return 0u;
    const uint32_t b = __float_as_uint(v);
    return (b & 0x80000000u) ? ~b : (b | 0x80000000u);
}

template <typename T>
__global__ void __launch_bounds__(256) digit_histogram(const T* __restrict__ plane0, size_t n, uint32_t prefix,
                                                       uint32_t prefix_mask, int shift,
                                                       unsigned long long* __restrict__ hist) {
    __shared__ unsigned int h[256];
    h[threadIdx.x] = 0u;
    __syncthreads();
    for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
        const uint32_t k = key_of(plane0[i]);
        if ((k & prefix_mask) == prefix) atomicAdd(&h[(k >> shift) & 255u], 1u);
    }
    __syncthreads();
    if (h[threadIdx.x]) atomicAdd(&hist[threadIdx.x], (unsigned long long)h[threadIdx.x]);
}

}  // namespace

// k-th largest key (1-based) of plane0[0..n); returns the key, or sets *err.
template <typename T>
static cudaError_t select_kth(const T* plane0, size_t n, unsigned long long k, unsigned long long* d_hist,
                              cudaStream_t st, uint32_t* key_out) {
    constexpr int BITS = sizeof(T) == 2 ? 16 : 32;
    uint32_t prefix = 0u, mask = 0u;
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const int grid = (int)((n + 255) / 256 < (size_t)sms * 8 ? (n + 255) / 256 : (size_t)sms * 8);
    for (int shift = BITS - 8; shift >= 0; shift -= 8) {
        unsigned long long h[256];
        cudaError_t e = cudaMemsetAsync(d_hist, 0, sizeof(h), st);
        if (e != cudaSuccess) return e;
        digit_histogram<T><<<grid > 0 ? grid : 1, 256, 0, st>>>(plane0, n, prefix, mask, shift, d_hist);
        if ((e = cudaGetLastError()) != cudaSuccess) return e;
        if ((e = cudaMemcpyAsync(h, d_hist, sizeof(h), cudaMemcpyDeviceToHost, st)) != cudaSuccess) return e;
        if ((e = cudaStreamSynchronize(st)) != cudaSuccess) return e;
        int d = 255;
        for (; d > 0; --d) {  // walk digits from the top until k is reached
            if (h[d] >= k) break;
            k -= h[d];
        }
        prefix |= (uint32_t)d << shift;
        mask |= 255u << shift;
    }
    *key_out = prefix;
    return cudaSuccess;
}

cudaError_t select_cutoff(const void* plane0, int dtype, size_t n, unsigned long long k,
                          unsigned long long* d_hist, cudaStream_t st, double* cutoff) {
    uint32_t key = 0;
    cudaError_t e;
    if (dtype == DAXM_U16) {
        e = select_kth(static_cast<const uint16_t*>(plane0), n, k, d_hist, st, &key);
        *cutoff = (double)key;
    } else {
        e = select_kth(static_cast<const float*>(plane0), n, k, d_hist, st, &key);
        const uint32_t b = (key & 0x80000000u) ? (key & 0x7fffffffu) : ~key;
        float f;
        memcpy(&f, &b, 4);
        *cutoff = key == 0u ? -HUGE_VAL : (double)f;  // key 0: NaN ranks lowest -> -inf
    }
    return e;
}

}  // namespace daxm
