// select.cu -- "pixel percentage": the intensity cutoff that keeps a given
// fraction of the plan's pixels, i.e. the k-th largest first-step intensity I_0(p)
// (reading R14), found exactly by a most-significant-digit radix select over an
// order-preserving integer key (8-bit digits, shared-memory histograms).
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
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
// With `reduce`, each digit's 256-bin host histogram is summed over the shards (ranks) by the
// caller's callback before the digit is chosen, so every shard walks to the same global key.
template <typename T>
static cudaError_t select_kth(const T* plane0, size_t n, unsigned long long k, unsigned long long* d_hist,
                              cudaStream_t st, uint32_t* key_out, HistReduce reduce, void* ctx,
                              bool* reduce_failed) {
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
        if (reduce && reduce(h, 256, ctx) != 0) {
            *reduce_failed = true;
            return cudaSuccess;
        }
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
                          unsigned long long* d_hist, cudaStream_t st, double* cutoff, HistReduce reduce,
                          void* ctx, bool* reduce_failed) {
    uint32_t key = 0;
    cudaError_t e;
    *reduce_failed = false;
    if (dtype == DAXM_U16) {
        e = select_kth(static_cast<const uint16_t*>(plane0), n, k, d_hist, st, &key, reduce, ctx, reduce_failed);
        *cutoff = (double)key;
    } else {
        e = select_kth(static_cast<const float*>(plane0), n, k, d_hist, st, &key, reduce, ctx, reduce_failed);
        const uint32_t b = (key & 0x80000000u) ? (key & 0x7fffffffu) : ~key;
        float f;
        memcpy(&f, &b, 4);
        *cutoff = key == 0u ? -HUGE_VAL : (double)f;  // key 0: NaN ranks lowest -> -inf
    }
    return e;
}

// ---- intensity cutoff, tile granularity: a deposit tile none of whose pixels passes the cutoff
// has an all-zero output block (reading R14), so its deposit CTAs exit at once and zero_dead_tiles
// writes its planes as whole plane rows (coalesced, row-contiguous) instead of the tile's 32-byte
// row segments at a 16.8 MB plane stride interleaved with live neighbours' writes.

namespace {

template <typename T>
__global__ void __launch_bounds__(TILE_R) tile_live(const T* __restrict__ plane0, int row_begin, int row_end, int C,
                                                    int tr0, int tr_begin, int n_tc, float cutoff,
                                                    unsigned char* __restrict__ live, unsigned char* __restrict__ glive) {
    static_assert(LOCK_ROWS == 16, "one row group = half a warp");
    const int tile = tr_begin * n_tc + (int)blockIdx.x;
    const int tr = tile / n_tc, tc = tile % n_tc;
    const int j = (tr0 + tr) * TILE_R + (int)threadIdx.x;  // one detector row per thread
    bool on = false;
    if (j >= row_begin && j < row_end) {
        const T* s = plane0 + (size_t)(j - row_begin) * C + tc * TILE_C;
        for (int c = 0; c < TILE_C && tc * TILE_C + c < C; ++c) on |= (float)s[c] >= cutoff;  // as in the kernels
    }
    const unsigned b = __ballot_sync(0xffffffffu, on);
    if ((threadIdx.x & 15) == 0)  // row group = one warp of the step-locked kernels (LOCK_ROWS rows)
        glive[(size_t)tile * NG16 + threadIdx.x / 16] = ((b >> (threadIdx.x & 16)) & 0xffffu) ? 1 : 0;
    on = __syncthreads_or(on);
    if (threadIdx.x == 0) live[tile] = on ? 1 : 0;
}

// work item = (plane m, tile row tr): every row of the tile row inside [r_lo, r_hi), the columns
// whose 16-row group (one step-locked warp) has no pixel above the cutoff.  A thread holds its
// column quads' flags for a whole group, so the row loop is nothing but independent 16-byte
// streaming stores.  (Dead groups of a live tile that a non-locked kernel owns are written by both
// sides, with the same zeros.)
constexpr int ZQ = 4;  // column quads per thread and pass
__global__ void __launch_bounds__(256) zero_dead_tiles(float* __restrict__ out, const unsigned char* __restrict__ glive,
                                                       int M, int rows_band, int C, int row_begin, int tr0, int n_tc,
                                                       int tr_begin, int tr_end, int r_lo, int r_hi) {
    const int ntr = tr_end - tr_begin;
    const int nq = (C + 3) / 4;
    const bool vec = (C & 3) == 0;
    for (int it = blockIdx.x; it < M * ntr; it += gridDim.x) {
        const int m = it / ntr, tr = tr_begin + it % ntr;
        const unsigned char* lrow = glive + (size_t)tr * n_tc * NG16;
        for (int g = 0; g < NG16; ++g) {
            int rb = (tr0 + tr) * TILE_R + g * 16 - row_begin, re = rb + 16;
            rb = rb < r_lo ? r_lo : rb;
            re = re > r_hi ? r_hi : re;
            if (rb >= re) continue;
            float* o = out + ((size_t)m * rows_band + rb) * C;
            for (int q0 = 0; q0 < nq; q0 += ZQ * (int)blockDim.x) {
                bool dead[ZQ];
#pragma unroll
                for (int u = 0; u < ZQ; ++u) {
                    const int q = q0 + u * (int)blockDim.x + (int)threadIdx.x;
                    // TILE_C is a multiple of 4: a quad never straddles tiles
                    dead[u] = q < nq && !lrow[(4 * q / TILE_C) * NG16 + g];
                }
                if (vec) {
#pragma unroll 4
                    for (int r = rb; r < re; ++r) {
                        float* orow = o + (size_t)(r - rb) * C;
#pragma unroll
                        for (int u = 0; u < ZQ; ++u)
                            if (dead[u])
                                __stcs(reinterpret_cast<float4*>(orow + 4 * (q0 + u * (int)blockDim.x + (int)threadIdx.x)),
                                       make_float4(0.f, 0.f, 0.f, 0.f));
                    }
                } else {
                    for (int r = rb; r < re; ++r)
                        for (int u = 0; u < ZQ; ++u)
                            if (dead[u]) {
                                const int c = 4 * (q0 + u * (int)blockDim.x + (int)threadIdx.x);
                                for (int x = c; x < c + 4 && x < C; ++x) o[(size_t)(r - rb) * C + x] = 0.f;
                            }
                }
            }
        }
    }
}

}  // namespace

cudaError_t launch_cutoff_tiles(const DepositArgs& a, const void* plane0, int dtype, float* out, unsigned char* live,
                                int phase, cudaStream_t st) {
    const int n = (a.tr_end - a.tr_begin) * a.n_tc;
    if (n <= 0) return cudaSuccess;
    if (phase == 0) {  // per-tile flags from plane 0
        if (dtype == DAXM_U16)
            tile_live<uint16_t><<<n, TILE_R, 0, st>>>(static_cast<const uint16_t*>(plane0), a.row_begin, a.row_end,
                                                      a.C, a.tr0, a.tr_begin, a.n_tc, a.cutoff, live, live + (size_t)a.n_tr * a.n_tc);
        else
            tile_live<float><<<n, TILE_R, 0, st>>>(static_cast<const float*>(plane0), a.row_begin, a.row_end, a.C,
                                                   a.tr0, a.tr_begin, a.n_tc, a.cutoff, live, live + (size_t)a.n_tr * a.n_tc);
        return cudaGetLastError();
    }
    const int rows_band = a.row_end - a.row_begin;
    int r_lo = (a.tr0 + a.tr_begin) * TILE_R - a.row_begin, r_hi = (a.tr0 + a.tr_end) * TILE_R - a.row_begin;
    r_lo = r_lo < 0 ? 0 : r_lo;
    r_hi = r_hi > rows_band ? rows_band : r_hi;
    if (r_hi <= r_lo || a.M <= 0) return cudaSuccess;
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    // one block per SM by default (measured: 1 and 8 alike, 2 slower): the fill runs beside the
    // deposit launches, whose CTAs fill the rest
    static const int per_sm = getenv("DAXM_ZERO_PER_SM") ? atoi(getenv("DAXM_ZERO_PER_SM")) : 1;
    const long long work = (long long)a.M * (a.tr_end - a.tr_begin);
    const long long g = (long long)sms * (per_sm > 0 ? per_sm : 1);
    zero_dead_tiles<<<(int)(work < g ? work : g), 256, 0, st>>>(out, live + (size_t)a.n_tr * a.n_tc, a.M, rows_band, a.C, a.row_begin, a.tr0,
                                                                 a.n_tc, a.tr_begin, a.tr_end, r_lo, r_hi);
    return cudaGetLastError();
}

}  // namespace daxm
