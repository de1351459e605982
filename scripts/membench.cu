// membench.cu -- ceiling of the step-locked deposit kernel's memory pattern with no
// arithmetic (VERDICT r1 "next" 1, step 1).  C4 shape: output [401][2048][2048] fp32
// (6.73 GB), stack [801][2048][2048] u16 of which each warp streams ~200 wire steps of
// its own 16 x 8 pixel block (1.3 GB read), exactly as deposit_lock's TMA ring does.
//
// Variants (each timed with CUDA events, best of 5):
//   lock   : warp = 16 rows x 8 cols; per plane LDS.128 + st.global.cs.v4 per lane
//            (one 32-byte sector per lane pair) -- deposit_lock's copy-out; TMA input ring
//   lockw  : the same output pattern, no input
//   tma4   : output by TMA bulk-tensor stores of [4 planes][16 rows][8 cols] boxes; TMA input
//   tma8   : ... [8 planes][16][8]
//   wide   : warp = 16 rows x 16 cols (64-byte row segments), 4 lanes per row
//   copy   : fully coalesced streaming write of the output + read of 1.3 GB (reference)
//
// build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o membench scripts/membench.cu
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>

#define CK(x)                                                                              \
    do {                                                                                   \
        cudaError_t e_ = (x);                                                              \
        if (e_ != cudaSuccess) {                                                           \
            fprintf(stderr, "%s:%d %s: %s\n", __FILE__, __LINE__, #x, cudaGetErrorString(e_)); \
            exit(1);                                                                       \
        }                                                                                  \
    } while (0)

constexpr int R = 2048, C = 2048, S = 801, M = 401;
constexpr int NIT = 200;  // wire steps per warp (C4: ~22 % of 801 plus guards)

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t n) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(n) : "memory");
}
__device__ __forceinline__ void mbar_expect(uint64_t* b, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t par) {
    asm volatile(
        "{\n .reg .pred p;\nW_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra W_%=;\n}\n" ::"r"(
            smem_u32(b)),
        "r"(par)
        : "memory");
}
__device__ __forceinline__ void tma_load_3d(void* dst, const CUtensorMap* m, int c0, int c1, int c2, uint64_t* b) {
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], "
        "[%5];" ::"r"(smem_u32(dst)),
        "l"((uint64_t)m), "r"(c0), "r"(c1), "r"(c2), "r"(smem_u32(b))
        : "memory");
}
__device__ __forceinline__ void tma_store_3d(const CUtensorMap* m, int c0, int c1, int c2, const void* src) {
    asm volatile("cp.async.bulk.tensor.3d.global.shared::cta.tile.bulk_group [%0, {%1, %2, %3}], [%4];" ::"l"(
                     (uint64_t)m),
                 "r"(c0), "r"(c1), "r"(c2), "r"(smem_u32(src))
                 : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void bulk_wait() {
    asm volatile("cp.async.bulk.wait_group %0;" ::"n"(N) : "memory");
}
template <int N>
__device__ __forceinline__ void bulk_wait_read() {
    asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(N) : "memory");
}
__device__ __forceinline__ void fence_async() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }

// first wire step of tile column tc (windows shift across the detector like C4's)
__device__ __forceinline__ int k_first(int tc) { return (tc * (S - NIT - 4)) / (C / 8); }

// MODE 0: lock (LDS+STG), 1: output only, 2: TMA store boxes of PB planes, 3: wide (16 cols)
template <int MODE, int PB>
__global__ void __launch_bounds__(128, 4) pattern(const __grid_constant__ CUtensorMap in_map,
                                                  const __grid_constant__ CUtensorMap out_map, float* out) {
    constexpr int WCOLS = MODE == 3 ? 16 : 8;
    constexpr int IN_W = 16 * 16 * WCOLS * 2;                        // per warp: 16 steps x 16 rows x cols u16
    constexpr int OUT_W = (MODE == 2 ? 2 * PB : 2) * 16 * WCOLS;      // per warp, floats
    extern __shared__ __align__(128) unsigned char smem[];
    unsigned char(*s_in)[IN_W] = reinterpret_cast<unsigned char(*)[IN_W]>(smem);
    float(*s_out)[OUT_W] = reinterpret_cast<float(*)[OUT_W]>(smem + 4 * IN_W);
    uint64_t(*bars)[4] = reinterpret_cast<uint64_t(*)[4]>(smem + 4 * IN_W + 4 * OUT_W * 4);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int n_tc = C / WCOLS;
    const int tile = blockIdx.x / 2, sub = blockIdx.x % 2;
    const int tr = tile / n_tc, tc = tile % n_tc;
    const int row = tr * 128 + (sub * 4 + warp) * 16;
    const int col0 = tc * WCOLS;
    const int k0 = k_first(col0 / 8);
    if (lane == 0) {
        for (int g = 0; g < 4; ++g) mbar_init(&bars[warp][g], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    float* so = s_out[warp];
    for (int q = lane; q < OUT_W; q += 32) so[q] = (float)(q + row);
    __syncwarp();
    fence_async();
    const bool use_in = MODE != 1;
    constexpr int GB = 4 * 16 * WCOLS * 2;  // one group: 4 steps
    int issued = 0;
    auto issue = [&](int upto) {  // groups < upto
        for (; issued < upto && issued < NIT / 4; ++issued)
            if (lane == 0) {
                mbar_expect(&bars[warp][issued & 3], GB);
                tma_load_3d(&s_in[warp][(issued & 3) * GB], &in_map, col0, row, k0 + 4 * issued, &bars[warp][issued & 3]);
            }
    };
    if (use_in) issue(4);
    const size_t plane = (size_t)R * C;
    int done = 0;
    float acc = 0.f;
    int batch = 0;
    for (int it = 0; it < NIT; ++it) {
        if (use_in && (it & 3) == 0) {
            const int g = it >> 2;
            mbar_wait(&bars[warp][g & 3], (g >> 2) & 1);
            acc += (float)reinterpret_cast<const uint16_t*>(&s_in[warp][(g & 3) * GB])[lane];
            __syncwarp();
            issue(g + 4);  // slot of group g is consumed once the next group starts (approximation)
        }
        const int upto = ((it + 1) * M) / NIT;
        if (MODE == 0 || MODE == 1) {
            const int r = lane >> 1, h = lane & 1;
            float* gp = out + (size_t)(row + r) * C + col0 + 4 * h;
            for (; done < upto; ++done) {
                float4 v = reinterpret_cast<const float4*>(so)[(done & 1) * 32 + lane];
                v.x += acc;
                asm volatile("st.global.cs.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(gp + done * plane), "f"(v.x),
                             "f"(v.y), "f"(v.z), "f"(v.w)
                             : "memory");
            }
        } else if (MODE == 3) {
            const int r = lane >> 2, q = lane & 3;
            for (; done < upto; ++done) {
                float4 v = reinterpret_cast<const float4*>(so)[(done & 1) * 64 + lane];
                v.x += acc;
                for (int hh = 0; hh < 2; ++hh)
                    asm volatile("st.global.cs.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(
                                     out + (size_t)(row + r + 8 * hh) * C + col0 + 4 * q + done * plane),
                                 "f"(v.x), "f"(v.y), "f"(v.z), "f"(v.w)
                                 : "memory");
            }
        } else {  // TMA boxes of PB planes
            while (done + PB <= upto || (upto == M && done < M)) {
                if (lane == 0) {
                    bulk_wait_read<1>();
                    tma_store_3d(&out_map, col0, row, done, &so[(batch & 1) * PB * 128]);
                    bulk_commit();
                }
                ++batch;
                done += PB;
            }
        }
    }
    if (MODE == 2 && lane == 0) bulk_wait_read<0>();
    if (acc == -1.f) out[0] = acc;
}


// generic output-pattern variant: warp = WR rows x WC cols, output only or with input; each
// lane stores 16-byte chunks (row-major over the warp's WR x WC block), STAG: warps start at a
// column-dependent plane offset (mimics depth offsets across the detector) and wrap around
template <int WR, int WC, bool INPUT, bool STAG>
__global__ void __launch_bounds__(128, 4) generic(const __grid_constant__ CUtensorMap in_map, float* out) {
    constexpr int CH = WC / 4;                  // 16-byte chunks per row
    constexpr int NST = WR * CH / 32;           // stores per lane per plane
    static_assert(NST >= 1 && (WR * CH) % 32 == 0, "shape");
    constexpr int GB = 4 * WR * WC * 2;
    extern __shared__ __align__(128) unsigned char smem[];
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + 4 * 4 * GB);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int n_wc = C / WC;
    const int wg = blockIdx.x * 4 + warp;      // global warp index
    const int wr = wg / n_wc, wc = wg % n_wc;
    const int row = wr * WR, col0 = wc * WC;
    const int k0 = k_first(col0 / 8);
    unsigned char* s_in = smem + warp * 4 * GB;
    if (lane == 0) {
        for (int g = 0; g < 4; ++g) mbar_init(&bars[warp * 4 + g], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncwarp();
    int issued = 0;
    auto issue = [&](int upto) {
        for (; issued < upto && issued < NIT / 4; ++issued)
            if (lane == 0) {
                mbar_expect(&bars[warp * 4 + (issued & 3)], GB);
                tma_load_3d(s_in + (issued & 3) * GB, &in_map, col0, row, k0 + 4 * issued, &bars[warp * 4 + (issued & 3)]);
            }
    };
    if (INPUT) issue(4);
    const size_t plane = (size_t)R * C;
    const int off = STAG ? (col0 * 11 / 16) % M : 0;
    int done = 0;
    float acc = 0.f;
    for (int it = 0; it < NIT; ++it) {
        if (INPUT && (it & 3) == 0) {
            const int g = it >> 2;
            mbar_wait(&bars[warp * 4 + (g & 3)], (g >> 2) & 1);
            acc += (float)reinterpret_cast<const uint16_t*>(s_in + (g & 3) * GB)[lane];
            __syncwarp();
            issue(g + 4);
        }
        const int upto = ((it + 1) * M) / NIT;
        for (; done < upto; ++done) {
            int p = done + off;
            p = p >= M ? p - M : p;
#pragma unroll
            for (int q = 0; q < NST; ++q) {
                const int ch = q * 32 + lane, r = ch / CH, c = (ch % CH) * 4;
                asm volatile("st.global.cs.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(
                                 out + (size_t)p * plane + (size_t)(row + r) * C + col0 + c),
                             "f"(acc), "f"(acc), "f"(acc), "f"(acc)
                             : "memory");
            }
        }
    }
}


// generic with TMA output stores of [4 planes][WR][WC] boxes from a zeroed smem batch, 1 warp per CTA,
// occupancy set by the dynamic shared memory (sm_bytes)
template <int WR, int WC>
__global__ void __launch_bounds__(32) gen_tma(const __grid_constant__ CUtensorMap in_map,
                                              const __grid_constant__ CUtensorMap out_map) {
    constexpr int GB = 4 * WR * WC * 2;
    extern __shared__ __align__(128) unsigned char smem_raw2[];
    unsigned char* smem = smem_raw2 + ((128 - (smem_u32(smem_raw2) & 127)) & 127);
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + 4 * GB);
    float* so = reinterpret_cast<float*>(smem + 4 * GB + 128);
    const int lane = threadIdx.x;
    const int n_wc = C / WC;
    const int wg = blockIdx.x;
    const int wr = wg / n_wc, wc = wg % n_wc;
    const int row = wr * WR, col0 = wc * WC;
    const int k0 = k_first(col0 / 8);
    if (lane == 0) {
        for (int g = 0; g < 4; ++g) mbar_init(&bars[g], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    for (int q = lane; q < 4 * WR * WC; q += 32) so[q] = 0.f;
    __syncwarp();
    fence_async();
    int issued = 0;
    auto issue = [&](int upto) {
        for (; issued < upto && issued < NIT / 4; ++issued)
            if (lane == 0) {
                mbar_expect(&bars[issued & 3], GB);
                tma_load_3d(smem + (issued & 3) * GB, &in_map, col0, row, k0 + 4 * issued, &bars[issued & 3]);
            }
    };
    issue(4);
    int done = 0;
    for (int it = 0; it < NIT; ++it) {
        if ((it & 3) == 0) {
            const int g = it >> 2;
            mbar_wait(&bars[g & 3], (g >> 2) & 1);
            __syncwarp();
            issue(g + 4);
        }
        const int upto = ((it + 1) * M) / NIT;
        while (done + 4 <= upto || (upto == M && done < M)) {
            if (lane == 0) {
                tma_store_3d(&out_map, col0, row, done, so);
                bulk_commit();
            }
            done += 4;
        }
    }
    if (lane == 0) bulk_wait<0>();
}


// 2 x 64 output boxes, input as two [4][2][32] boxes per group (the column halves at different steps)
__global__ void __launch_bounds__(32) gen_split(const __grid_constant__ CUtensorMap in_map,
                                                const __grid_constant__ CUtensorMap out_map) {
    constexpr int WR = 2, WC = 64, GBH = 4 * WR * 32 * 2;  // one half-box
    extern __shared__ __align__(128) unsigned char smem_raw3[];
    unsigned char* smem = smem_raw3 + ((128 - (smem_u32(smem_raw3) & 127)) & 127);
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + 8 * GBH);
    float* so = reinterpret_cast<float*>(smem + 8 * GBH + 128);
    const int lane = threadIdx.x;
    const int n_wc = C / WC;
    const int wg = blockIdx.x;
    const int wr = wg / n_wc, wc = wg % n_wc;
    const int row = wr * WR, col0 = wc * WC;
    const int k0 = k_first(col0 / 8), k1 = k_first((col0 + 32) / 8);
    if (lane == 0) {
        for (int g = 0; g < 4; ++g) mbar_init(&bars[g], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    for (int q = lane; q < 4 * WR * WC; q += 32) so[q] = 0.f;
    __syncwarp();
    fence_async();
    int issued = 0;
    auto issue = [&](int upto) {
        for (; issued < upto && issued < NIT / 4; ++issued)
            if (lane == 0) {
                mbar_expect(&bars[issued & 3], 2 * GBH);
                tma_load_3d(smem + (issued & 3) * 2 * GBH, &in_map, col0, row, k0 + 4 * issued, &bars[issued & 3]);
                tma_load_3d(smem + (issued & 3) * 2 * GBH + GBH, &in_map, col0 + 32, row, k1 + 4 * issued, &bars[issued & 3]);
            }
    };
    issue(4);
    int done = 0;
    for (int it = 0; it < NIT; ++it) {
        if ((it & 3) == 0) {
            const int g = it >> 2;
            mbar_wait(&bars[g & 3], (g >> 2) & 1);
            __syncwarp();
            issue(g + 4);
        }
        const int upto = ((it + 1) * M) / NIT;
        while (done + 4 <= upto || (upto == M && done < M)) {
            if (lane == 0) {
                tma_store_3d(&out_map, col0, row, done, so);
                bulk_commit();
            }
            done += 4;
        }
    }
    if (lane == 0) bulk_wait<0>();
}

// coalesced reference: every thread writes 16-byte chunks of a contiguous span and reads the stack
__global__ void copy_ref(const uint4* __restrict__ in, size_t n_in, float4* __restrict__ out, size_t n_out) {
    uint32_t acc = 0;
    const size_t stride = (size_t)gridDim.x * blockDim.x;
    for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n_in; i += stride) acc ^= __ldcs(in + i).x;
    for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n_out; i += stride)
        __stcs(out + i, make_float4((float)acc, 0.f, 0.f, 0.f));
}

int main() {
    PFN_cuTensorMapEncodeTiled_v12000 enc = nullptr;
    cudaDriverEntryPointQueryResult q;
    CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&enc, cudaEnableDefault, &q));
    const size_t in_bytes = (size_t)S * R * C * 2, out_bytes = (size_t)M * R * C * 4;
    void *d_in, *d_out;
    CK(cudaMalloc(&d_in, in_bytes));
    CK(cudaMalloc(&d_out, out_bytes));
    CK(cudaMemset(d_in, 1, in_bytes));
    CK(cudaMemset(d_out, 0, out_bytes));
    auto mk_in = [&](int wcols) {
        CUtensorMap m;
        cuuint64_t dims[3] = {C, R, S}, str[2] = {C * 2ull, (cuuint64_t)C * R * 2};
        cuuint32_t box[3] = {(cuuint32_t)wcols, 16, 4}, es[3] = {1, 1, 1};
        if (enc(&m, CU_TENSOR_MAP_DATA_TYPE_UINT16, 3, d_in, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE))
            exit(2);
        return m;
    };
    auto mk_out = [&](int pb) {
        CUtensorMap m;
        cuuint64_t dims[3] = {C, R, M}, str[2] = {C * 4ull, (cuuint64_t)C * R * 4};
        cuuint32_t box[3] = {8, 16, (cuuint32_t)pb}, es[3] = {1, 1, 1};
        if (enc(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, d_out, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE))
            exit(3);
        return m;
    };
    const CUtensorMap in8 = mk_in(8), in16 = mk_in(16), out4 = mk_out(4), out8 = mk_out(8);
    const double rd8 = (double)(R / 16) * (C / 8) * NIT * 16 * 8 * 2;  // bytes the warps stream
    cudaEvent_t a, b;
    CK(cudaEventCreate(&a));
    CK(cudaEventCreate(&b));
    auto timeit = [&](const char* name, double bytes, auto&& launch) {
        float best = 1e30f;
        for (int rep = 0; rep < 6; ++rep) {
            CK(cudaEventRecord(a));
            launch();
            CK(cudaEventRecord(b));
            CK(cudaEventSynchronize(b));
            CK(cudaGetLastError());
            float ms;
            CK(cudaEventElapsedTime(&ms, a, b));
            if (rep > 0 && ms < best) best = ms;
        }
        printf("{\"variant\": \"%s\", \"ms\": %.4f, \"GB\": %.4f, \"GBps\": %.1f}\n", name, best, bytes / 1e9,
               bytes / (best * 1e-3) / 1e9);
        fflush(stdout);
    };
    const int grid8 = (R / 128) * (C / 8) * 2, grid16 = (R / 128) * (C / 16) * 2;
    auto smb = [](int mode, int pb) {
        const int wc = mode == 3 ? 16 : 8;
        return (size_t)4 * 16 * 16 * wc * 2 + (size_t)4 * (mode == 2 ? 2 * pb : 2) * 16 * wc * 4 + 4 * 4 * 8;
    };
    CK(cudaFuncSetAttribute(pattern<2, 8>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smb(2, 8)));
    CK(cudaFuncSetAttribute(pattern<2, 4>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smb(2, 4)));
    CK(cudaFuncSetAttribute(pattern<3, 4>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smb(3, 4)));
    // timeit("lock", out_bytes + rd8, [&] { pattern<0, 4><<<grid8, 128, smb(0, 4)>>>(in8, out4, (float*)d_out); });
    // timeit("lockw", out_bytes, [&] { pattern<1, 4><<<grid8, 128, smb(1, 4)>>>(in8, out4, (float*)d_out); });
    // timeit("tma4", out_bytes + rd8, [&] { pattern<2, 4><<<grid8, 128, smb(2, 4)>>>(in8, out4, (float*)d_out); });
    // timeit("tma8", out_bytes + rd8, [&] { pattern<2, 8><<<grid8, 128, smb(2, 8)>>>(in8, out8, (float*)d_out); });
    // timeit("wide", out_bytes + 2 * rd8, [&] { pattern<3, 4><<<grid16, 128, smb(3, 4)>>>(in16, out4, (float*)d_out); });

    auto mk_in2 = [&](int wr, int wc) {
        CUtensorMap m;
        cuuint64_t dims[3] = {C, R, S}, str[2] = {C * 2ull, (cuuint64_t)C * R * 2};
        cuuint32_t box[3] = {(cuuint32_t)wc, (cuuint32_t)wr, 4}, es[3] = {1, 1, 1};
        if (enc(&m, CU_TENSOR_MAP_DATA_TYPE_UINT16, 3, d_in, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE))
            exit(4);
        return m;
    };
#define GEN(NAME, WR, WC, IN, ST)                                                                          \
    {                                                                                                      \
        const CUtensorMap im = mk_in2(WR, WC);                                                             \
        const size_t sb = 4 * 4 * (4 * WR * WC * 2) + 4 * 4 * 8;                                           \
        CK(cudaFuncSetAttribute(generic<WR, WC, IN, ST>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sb)); \
        const int nw = (R / WR) * (C / WC);                                                                \
        timeit(NAME, out_bytes + (IN ? rd8 : 0.0), [&] { generic<WR, WC, IN, ST><<<nw / 4, 128, sb>>>(im, (float*)d_out); }); \
    }
    // GEN("g16x8_out", 16, 8, false, false)
    // GEN("g16x8_out_stag", 16, 8, false, true)
    // GEN("g16x16_out", 16, 16, false, false)
    // GEN("g8x32_out", 8, 32, false, false)
    // GEN("g4x32_out", 4, 32, false, false)
    // GEN("g4x32_out_stag", 4, 32, false, true)
    // GEN("g4x32_in", 4, 32, true, false)
    // GEN("g4x32_in_stag", 4, 32, true, true)
    // GEN("g8x32_in", 8, 32, true, false)
    // GEN("g2x64_in", 2, 64, true, false)

    auto mk_out2 = [&](int wr, int wc) {
        CUtensorMap m;
        cuuint64_t dims[3] = {C, R, M}, str[2] = {C * 4ull, (cuuint64_t)C * R * 4};
        cuuint32_t box[3] = {(cuuint32_t)wc, (cuuint32_t)wr, 4}, es[3] = {1, 1, 1};
        if (enc(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, d_out, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE))
            exit(5);
        return m;
    };
#define GTMA(NAME, WR, WC, SMB)                                                                               \
    {                                                                                                          \
        const CUtensorMap im = mk_in2(WR, WC), om = mk_out2(WR, WC);                                            \
        CK(cudaFuncSetAttribute(gen_tma<WR, WC>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)(SMB)));     \
        const int nw = (R / WR) * (C / WC);                                                                    \
        timeit(NAME, out_bytes + rd8, [&] { gen_tma<WR, WC><<<nw, 32, SMB>>>(im, om); });                       \
    }
    {
        const CUtensorMap im = mk_in2(2, 32), om = mk_out2(2, 64);
        for (int smb : {19700, 13500}) {
            CK(cudaFuncSetAttribute(gen_split, cudaFuncAttributeMaxDynamicSharedMemorySize, smb));
            timeit(smb > 15000 ? "split_2x64_11w" : "split_2x64_16w", out_bytes + rd8,
                   [&] { gen_split<<<(R / 2) * (C / 64), 32, smb>>>(im, om); });
        }
    }
    GTMA("tma_4x32_11w", 4, 32, 19700)
    GTMA("tma_4x32_16w", 4, 32, 13500)
    // GTMA("tma_8x16_11w", 8, 16, 19700)
    // GTMA("tma_8x16_15w", 8, 16, 14500)
    GTMA("tma_2x64_11w", 2, 64, 19700)
    GTMA("tma_2x64_16w", 2, 64, 13500)
    // GTMA("tma_16x8_11w", 16, 8, 19700)
    int sms = 148;
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
    timeit("copy", out_bytes + rd8, [&] {
        copy_ref<<<sms * 8, 512>>>((const uint4*)d_in, (size_t)(rd8 / 16), (float4*)d_out, out_bytes / 16);
    });
    return 0;
}
