// deposit_lock.cu -- step-locked gather deposit for
// tiles in the separated-span regime, plus the pre-pass that proves its per-warp
// output ring can never overflow.
//
// What is computed is exactly deposit_fast's: per pixel, with the
// step pairs visited in the order their trapezoids move deeper and c_q = dI_q / A_q,
// the intensity deposited below bin edge E is, inside zone q = (lo_q, lo_{q+1}],
//     F(E) = F(lo_q) + c_q x + xc (d_q + g_q xc),  x = E - lo_q, xc = min(x, w_q),
//     d_q = c_{q-1} - c_q,  g_q = -d_q / (2 w_q),  w_q = hi_q - lo_q,
// and bin m = [E_m, E_{m+1}) receives F(E_{m+1}) - F(E_m): the trapezoid overlaps of
// P:L320-331 (device_depth_resolve_pixel / device_get_trapezoid_height) summed over the
// pairs, one owner per (bin, pixel), no atomics.
//
// How it is scheduled differs: instead of walking bin edges and branching into a zone
// transition whenever a pixel crosses a knot (divergent, serialised per walk), every walk of
// a warp advances exactly ONE wire step per iteration -- all walks process visit vmin0 + j at
// iteration j, vmin0 the warp's first window start (from the geometry windows, so the cutoff
// cannot change an active walk's arithmetic) -- and then evaluates the bin edges of the zone
// that step closed in a warp-uniform, predicated loop.  Before its own window a walk's zones
// lie below the bins (they only offset F, which the bin differences cancel); after it they lie
// above (no edge left: pre-pass).  The wire travel and the input slot are warp-uniform, all
// control flow is warp-uniform, and walk pairs run in packed fp32x2 (FFMA2/FADD2/FMUL2).
//
// Warp = 16 detector rows x 8 columns, an independent pipeline (no CTA-level sync after
// setup): lane = (row group rg = lane / 8, column = lane % 8), walk w (0..3) = row
// 4 w + rg, so one walk's 32 lanes cover 4 consecutive rows x 8 columns = 128
// contiguous bytes of a staged plane (conflict-free scalar stores).
//   input : TMA loads of the warp's [LOCK_G steps][16 rows][8 cols] block into a 16-slot
//           ring, one mbarrier per group of LOCK_G steps (lane 0 produces);
//   output: a ring of RB staged planes indexed by bin edge e (plane e - 1); planes below
//           the slowest walk's frontier are TMA-stored in batches of SB, their slots
//           zeroed once the store has read them.  The pre-pass (lock_prepass_kernel)
//           replays the walks' edge frontiers with the same fp32 arithmetic and admits a
//           tile only if no iteration can write past the recycled part of the ring.
#include <cuda.h>
#include <cuda_runtime.h>
#include <limits.h>
#include <stdint.h>

#include "daxm_internal.cuh"
#include "ptx.cuh"

namespace daxm {
namespace {
using namespace ptx;

static_assert(NCOEF == 3, "lock kernel: quadratic depth model");
static_assert(TILE_C == 8 && TILE_R % (LOCK_ROWS * LOCK_WARPS) == 0, "lock kernel: tile shape");

#ifndef DAXM_LOCK_MINB
#define DAXM_LOCK_MINB 4  // CTAs per SM the register allocation targets (128 regs at 4)
#endif
#ifndef DAXM_LOCK_UNROLL
#define DAXM_LOCK_UNROLL 2  // iterations per loop body (2: no loop-carried register rotation)
#endif
#define DAXM_PRAGMA(x) _Pragma(#x)
#define DAXM_UNROLL(n) DAXM_PRAGMA(unroll n)
#ifndef DAXM_LOCK_KUNROLL
#define DAXM_LOCK_KUNROLL 1  // edge-loop trips per loop body
#endif
#ifndef DAXM_LOCK_DRAIN2
#define DAXM_LOCK_DRAIN2 1  // 1: copy-out loads two planes before storing either
#endif
#ifndef DAXM_LOCK_CHECK
#define DAXM_LOCK_CHECK 0  // 1: count ring-capacity violations (the pre-pass makes them impossible)
#endif

constexpr int LK_THREADS = LOCK_WARPS * 32;
constexpr int LK_PLANE = LOCK_ROWS * TILE_C * 4;  // bytes of one staged plane per warp

template <typename T, int RB>
struct LockSmem {
    static constexpr int OUT_BYTES = RB * LK_PLANE;                       // per warp
    static constexpr int IN_SLOT = LOCK_ROWS * TILE_C * (int)sizeof(T);    // per warp and step
    static constexpr int IN_GROUP = LOCK_G * IN_SLOT;                     // one TMA box
    static constexpr int IN_BYTES = LOCK_NB * IN_SLOT;                    // per warp
    static constexpr int OFF_OUT = 0;
    static constexpr int OFF_IN = OFF_OUT + LOCK_WARPS * OUT_BYTES;
    static constexpr int OFF_BAR = OFF_IN + LOCK_WARPS * IN_BYTES;
    static constexpr int OFF_TAU = OFF_BAR + LOCK_WARPS * LOCK_NB * 8;
    static size_t bytes(int max_nv) { return (size_t)OFF_TAU + sizeof(float) * (size_t)(max_nv + 4) + 128; }
};

// ---- packed fp32x2 helpers (sm_100a FADD2 / FMUL2 / FFMA2; per-component IEEE rn)
__device__ __forceinline__ float2 add2(float2 a, float2 b) { return __fadd2_rn(a, b); }
__device__ __forceinline__ float2 sub2(float2 a, float2 b) {
    float2 r;
    asm("{\n .reg .b64 ra, rb, rr;\n mov.b64 ra, {%2, %3};\n mov.b64 rb, {%4, %5};\n"
        " sub.rn.f32x2 rr, ra, rb;\n mov.b64 {%0, %1}, rr;\n}\n"
        : "=f"(r.x), "=f"(r.y)
        : "f"(a.x), "f"(a.y), "f"(b.x), "f"(b.y));
    return r;
}
__device__ __forceinline__ float2 mul2(float2 a, float2 b) { return __fmul2_rn(a, b); }
__device__ __forceinline__ float2 fma2(float2 a, float2 b, float2 c) { return __ffma2_rn(a, b, c); }
__device__ __forceinline__ float2 min2(float2 a, float2 b) { return make_float2(fminf(a.x, b.x), fminf(a.y, b.y)); }
__device__ __forceinline__ float2 max2(float2 a, float2 b) { return make_float2(fmaxf(a.x, b.x), fmaxf(a.y, b.y)); }
__device__ __forceinline__ float2 f2(float v) { return make_float2(v, v); }
__device__ __forceinline__ float2 poly2(const float2 c[3], float2 t) { return fma2(fma2(c[2], t, c[1]), t, c[0]); }
__device__ __forceinline__ float2 rcp2(float2 x) { return make_float2(rcp_approx(x.x), rcp_approx(x.y)); }

// Predicated edge store: if E <= Eb, st.shared [addr] = o and Fp = F (one FSETP, no branch).
__device__ __forceinline__ void edge_store(uint32_t addr, float o, float F, float E, float Eb, float& Fp) {
    asm volatile(
        "{\n .reg .pred q;\n setp.le.f32 q, %3, %4;\n @q st.shared.f32 [%1], %2;\n @q mov.f32 %0, %5;\n}\n"
        : "+f"(Fp)
        : "r"(addr), "f"(o), "f"(E), "f"(Eb), "f"(F)
        : "memory");
}
__device__ __forceinline__ void sts_zero4(uint32_t addr) {
    asm volatile("st.shared.v4.f32 [%0], {%1, %1, %1, %1};" ::"r"(addr), "f"(0.f) : "memory");
}

// Per-walk geometry shared by the kernel and its pre-pass: window, visit offset, the two
// edge-point polynomials of the pixel (back edge = column, front = column + 1 or the same
// column for POINT pixels).
struct LockWalk {
    int v0, npts;  // first visit (index into the tile's step list), points in the window (0: inactive)
};

__device__ __forceinline__ LockWalk lock_walk(const DepositArgs& a, const TileInfo& ti, int j, int i, bool act) {
    LockWalk lw{0, 0};
    if (!act || j >= a.row_end || j >= a.R || i >= a.C) return lw;
    const int2 win = a.win[(size_t)(j - a.pre_row0) * a.C + i];
    if (win.y <= win.x) return lw;
    lw.v0 = ti.dir > 0 ? win.x - ti.k_lo : ti.k_hi - win.y;
    lw.npts = win.y - win.x + 1;
    return lw;
}

__device__ __forceinline__ void lock_coef(const DepositArgs& a, int tile, int r, int c, bool point, float cb[3],
                                          float cf[3]) {
    const int ef = point ? c : c + 1;
#pragma unroll
    for (int m = 0; m < 3; ++m) {
        cb[m] = a.coef[(((size_t)tile * NCOEF + m) * TILE_E + c) * TILE_R + r];
        cf[m] = a.coef[(((size_t)tile * NCOEF + m) * TILE_E + ef) * TILE_R + r];
    }
}

// ------------------------------------------------------------------ kernel
__device__ __forceinline__ float4 lds128(uint32_t addr) {
    float4 v;
    asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "r"(addr)
                 : "memory");
    return v;
}
__device__ __forceinline__ void stg128_cs_if(bool ok, float* p, float4 v) {  // streaming (written once), predicated
    asm volatile("{\n .reg .pred q;\n setp.ne.u32 q, %5, 0;\n @q st.global.cs.v4.f32 [%0], {%1, %2, %3, %4};\n}\n" ::"l"(p),
                 "f"(v.x), "f"(v.y), "f"(v.z), "f"(v.w), "r"((unsigned)ok)
                 : "memory");
}

// The step-locked kernels share everything but the zone arithmetic: OV = false, separated spans
// (one zone quadratic per walk); OV = true, overlapping spans (ramp superposition).
template <typename T, bool POINT, int RB, bool OV>
__global__ void __launch_bounds__(LK_THREADS, OV ? 2 : DAXM_LOCK_MINB)
    deposit_lock(const __grid_constant__ CUtensorMap in_map, float* __restrict__ out, const DepositArgs a) {
    using L = LockSmem<T, RB>;
    extern __shared__ unsigned char smem_raw[];
    const uint32_t sbase = (smem_u32(smem_raw) + 127u) & ~127u;
    unsigned char* smem = smem_raw + (sbase - smem_u32(smem_raw));

    const int tile = a.tr_begin * a.n_tc + (int)blockIdx.x / LOCK_SUBS;
    const int sub = (int)blockIdx.x % LOCK_SUBS;
    const TileInfo ti = a.tiles[tile];
    if ((ti.lock & LOCK_CLASS_MASK) != (OV ? (RB | LOCK_OVB) : RB)) return;
    if (a.tile_live && !a.tile_live[tile]) return;  // cutoff: zero_dead_tiles writes this tile
    const int tr = tile / a.n_tc, tc = tile % a.n_tc;
    const int row0 = (a.tr0 + tr) * TILE_R;  // global row of tile row 0 (>= row_begin: pre-pass)
    const int col0 = tc * TILE_C;
    const int nv = ti.k_hi >= ti.k_lo ? ti.k_hi - ti.k_lo + 1 : 0;
    const int dir = ti.dir;

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int col = lane & 7, rg = lane >> 3;
    const int wrow = (sub * LOCK_WARPS + warp) * LOCK_ROWS;  // warp's first row in the tile
    const uint32_t s_out = sbase + L::OFF_OUT + warp * L::OUT_BYTES;
    const uint32_t s_in = sbase + L::OFF_IN + warp * L::IN_BYTES;
    const uint32_t s_bar = sbase + L::OFF_BAR + warp * LOCK_NB * 8;
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + L::OFF_BAR) + warp * LOCK_NB;
    float* tau = reinterpret_cast<float*>(smem + L::OFF_TAU);
    const uint32_t s_tau = sbase + L::OFF_TAU;

    for (int v = threadIdx.x; v < nv; v += blockDim.x) {
        const int k = dir > 0 ? ti.k_lo + v : ti.k_hi - v;
        tau[v] = (float)(a.t[k] - ti.t_ref);
    }
    if (lane == 0) {
        for (int s = 0; s < LOCK_NG; ++s) mbar_init(&bars[s], 1);
        fence_mbar_init();
    }
    // zero the output ring: RB planes x 512 B, 16 B per lane per plane
    const uint32_t s_copy = s_out + (uint32_t)lane * 16u;
#pragma unroll
    for (int s = 0; s < RB; ++s) sts_zero4(s_copy + s * LK_PLANE);
    __syncthreads();
    // a group without a pixel above the cutoff is written by zero_dead_tiles: its warp is done
    if (a.grp_live && !a.grp_live[tile * NG16 + wrow / LOCK_ROWS]) return;

    // ---- walks: rows wrow + 4w + rg, column col
    const int i = col0 + col;
    float cbs[4][3], cfs[4][3];
    bool act[4];
    int vmin0 = INT_MAX, vend = INT_MIN;
#pragma unroll
    for (int w = 0; w < 4; ++w) {
        const int r = wrow + 4 * w + rg;
        const int j = row0 + r;
        bool on = true;
        if (a.use_cutoff && j < a.row_end && i < a.C) {  // intensity cutoff (f1, reading R14)
            const T* s0 = static_cast<const T*>(a.stack) + (size_t)(j - a.row_begin) * a.C + i;
            on = (float)s0[0] >= a.cutoff;
        }
        // the warp's visit range comes from the geometry windows alone, so an active walk's
        // arithmetic (hence its output, bit for bit) does not depend on which others are active
        const LockWalk lw = lock_walk(a, ti, j, i, true);
        act[w] = on && lw.npts > 0;
        if (ti.lock & LOCK_FRONT_LO)  // the front edge is the shallower one over the whole tile (pre-pass)
            lock_coef(a, tile, r, col, POINT, cfs[w], cbs[w]);
        else
            lock_coef(a, tile, r, col, POINT, cbs[w], cfs[w]);
        if (lw.npts > 0) {
            vmin0 = min(vmin0, lw.v0);
            vend = max(vend, lw.v0 + lw.npts - 1);
        }
    }
    vmin0 = __reduce_min_sync(0xffffffffu, vmin0);
    vend = __reduce_max_sync(0xffffffffu, vend);
    // warp-locked walks: every walk visits vmin0 + jj at iteration jj (0 <= jj < niter)
    const bool any_act = __any_sync(0xffffffffu, act[0] || act[1] || act[2] || act[3]);
    const int niter = any_act && vend >= vmin0 ? vend - vmin0 + 1 : 0;

    const int rows_band = a.row_end - a.row_begin;
    const int row_local = row0 - a.row_begin + wrow;  // input / output row of the warp's first row
    const float E0 = (float)(-a.m_ref), EM = (float)(a.M - a.m_ref);
    const int M = a.M;

    // ---- output ring: plane P in slot P mod RB (edge e completes plane e - 1; "plane -1" of
    // edge 0 is scratch).  Planes [-1, done_p) are copied out and their slots zeroed; walks may
    // write planes < done_p + RB.  Copy-out: lane l moves row l/2, columns 4(l%2)..+3 of a plane
    // (LDS.128 -> st.global.cs.v4: every 32-byte output sector is written whole by one instruction).
    const size_t plane_stride = (size_t)rows_band * a.C;
    const int crow = row_local + (lane >> 1);
    const bool c_ok = crow < rows_band && col0 + (lane & 1) * 4 < a.C;
    float* const gout = out + (size_t)(c_ok ? crow : 0) * a.C + col0 + (lane & 1) * 4;
    int done_p = -1;
    float* gp = gout;  // output row chunk of plane done_p (>= 0)
    auto drain = [&](int upto) {  // warp-uniform: copy out and recycle planes [done_p, min(upto, M))
        upto = min(upto, M);
        if (done_p >= upto) return;
        __syncwarp();
        if (done_p < 0) {  // scratch slot of edge 0: every walk is past it
            sts_zero4(s_copy + (uint32_t)(RB - 1) * LK_PLANE);
            done_p = 0;
        }
        auto slot = [&](int p) { return s_copy + (uint32_t)(p & (RB - 1)) * LK_PLANE; };
#pragma unroll 1
        for (; DAXM_LOCK_DRAIN2 && done_p + 1 < upto; done_p += 2) {  // two planes per trip: both loads in flight
            const float4 va = lds128(slot(done_p)), vb = lds128(slot(done_p + 1));
            sts_zero4(slot(done_p));
            sts_zero4(slot(done_p + 1));
            stg128_cs_if(c_ok, gp, va);
            stg128_cs_if(c_ok, gp + plane_stride, vb);
            gp += 2 * plane_stride;
        }
#pragma unroll 1
        for (; done_p < upto; ++done_p) {
            const float4 v = lds128(slot(done_p));
            sts_zero4(slot(done_p));
            stg128_cs_if(c_ok, gp, v);
            gp += plane_stride;
        }
        __syncwarp();
    };

    if (niter > 0) {
        // ---- input ring: visit v (relative r = v - vmin0) in slot r % NB, parity (r / NB) & 1.
        // Loads are issued in groups of >= 4 and waited for in groups (warp-uniform bookkeeping).
        // Visits vmin0 + 4g .. + 3 form group g: one TMA box of LOCK_G consecutive wire steps
        // (ascending k, so for dir < 0 a group's visits land in reverse slot order: slot =
        // ((v - vmin0) ^ xr) mod NB) completing mbarrier g mod NG.  Group g reuses the slots of
        // group g - NG, free once every walk has read past it: at iteration jj the walks have
        // consumed the visits below vmin0 + jj, so groups up to (jj + NB - G) / G may be in
        // flight; the prefetch needs visit vmin0 + jj + 1.
        const int xr = dir > 0 ? 0 : LOCK_G - 1;
        const int ngroups = (vend - vmin0) / LOCK_G + 1;
        const int kbase = dir > 0 ? ti.k_lo + vmin0 : ti.k_hi - vmin0 - (LOCK_G - 1);
        int g_issue = 0, g_wait = 0;  // next group to load / to wait for
        auto issue = [&](int jj) {    // groups the ring can hold at iteration jj
            const int lim = min((jj + LOCK_NB - LOCK_G) / LOCK_G, ngroups - 1);
            if (g_issue > lim) return;
            if (lane == 0) {
                for (int g = g_issue; g <= lim; ++g) {
                    const int b = g & (LOCK_NG - 1);
                    mbar_arrive_expect_tx(&bars[b], L::IN_GROUP);
                    tma_load_3d(smem + (s_in - sbase) + b * L::IN_GROUP, &in_map, col0, row_local,
                                dir > 0 ? kbase + g * LOCK_G : kbase - g * LOCK_G, &bars[b]);
                }
            }
            g_issue = lim + 1;
        };
        auto wait_upto = [&](int v) {  // every group up to visit v's (clamped to the last) has landed
            const int g_need = (min(v, vend) - vmin0) / LOCK_G;
            if (g_wait > g_need) return;
            for (; g_wait <= g_need; ++g_wait) {  // compiler-visible retry loop: the warp reconverges after it
                while (!mbar_try(s_bar + (uint32_t)(g_wait & (LOCK_NG - 1)) * 8u, (uint32_t)(g_wait / LOCK_NG) & 1u)) {
                }
            }
            __syncwarp();
        };
        issue(0);

        // per-lane addresses
        const uint32_t in_lane = s_in + (uint32_t)(rg * TILE_C + col) * (uint32_t)sizeof(T);  // + w * 4 rows
        const uint32_t out_lane = s_out + (uint32_t)(rg * TILE_C + col) * 4u;                 // + w * 128

        // ---- walk state, packed by walk pairs (0,1), (2,3)
        float2 cb[2][3], cf[2][3];
#pragma unroll
        for (int p = 0; p < 2; ++p)
#pragma unroll
            for (int m = 0; m < 3; ++m) {
                cb[p][m] = make_float2(cbs[2 * p][m], cbs[2 * p + 1][m]);
                cf[p][m] = make_float2(cfs[2 * p][m], cfs[2 * p + 1][m]);
            }
        // wire travel (warp-uniform) and the 4 walks' intensities at visit vmin0 + jj; past the
        // last visit every walk re-reads it (its points lie above EM: pre-pass)
        auto fetch = [&](int jj, float& t, float2 I[2]) {
            const int vv = min(jj, niter - 1);
            t = lds_f32(s_tau + 4u * (uint32_t)(vmin0 + vv));
            const uint32_t sl = in_lane + (uint32_t)((vv ^ xr) & (LOCK_NB - 1)) * (uint32_t)L::IN_SLOT;
            constexpr uint32_t WB = 4 * TILE_C * sizeof(T);  // walk w: rows + 4 w
            I[0] = make_float2(lds_px<T>(sl), lds_px<T>(sl + WB));
            I[1] = make_float2(lds_px<T>(sl + 2 * WB), lds_px<T>(sl + 3 * WB));
        };

        wait_upto(vmin0 + 1);
        if constexpr (!OV) {
            float2 plo[2], phi[2], ps[2], pI[2], cq[2], zF[2], Fp[2], En[2], Iq[2];
            float tq;
            {
                float t0;
                fetch(0, t0, pI);
    #pragma unroll
                for (int p = 0; p < 2; ++p) {
                    plo[p] = poly2(cb[p], f2(t0));  // lo edge / hi edge: fixed order over the tile (pre-pass)
                    phi[p] = POINT ? plo[p] : poly2(cf[p], f2(t0));
                    ps[p] = add2(plo[p], phi[p]);
                    cq[p] = zF[p] = Fp[p] = f2(0.f);
                    // first edge: the first above point 0's lo (F = 0 below it); inactive walks never evaluate
                    En[p].x = act[2 * p] ? fmaxf(E0, floorf(plo[p].x) + 1.f) : EM + 1.f;
                    En[p].y = act[2 * p + 1] ? fmaxf(E0, floorf(plo[p].y) + 1.f) : EM + 1.f;
                }
                fetch(1, tq, Iq);
            }
            const float2 sdir2 = f2(2.f * a.sign * (float)dir);  // c = 2 s dir dI / (sum_{q+1} - sum_q)
            const int m_ref = a.m_ref;
            // bits(E + fbias) = 0x4B000000 + e - 1 + RB for edge index e: plane e - 1 mod RB in the low bits
            const float fbias = 8388608.f + (float)(m_ref - 1 + RB);
            // planes below the slowest walk's next edge are final; a finished or inactive walk sits at
            // edge M + 1 (its last point lies above the bins: pre-pass), so it never holds them back
            auto frontier = [&]() {
                const float fr = fminf(fminf(En[0].x, En[0].y), fminf(En[1].x, En[1].y));
                return __reduce_min_sync(0xffffffffu, (int)fr + m_ref) - 1;  // planes < edge - 1
            };
            drain(frontier());
    #if DAXM_LOCK_CHECK
            unsigned viol = 0u;
    #endif

            // iteration jj closes zone jj - 1 of every walk; before its own window a walk's zones lie
            // below the bins (F offset only), after it above them (no edge left: pre-pass)
            DAXM_UNROLL(DAXM_LOCK_UNROLL)
            for (int jj = 1; jj < niter; ++jj) {
                // point jj (prefetched); refill the ring below the slowest walk; prefetch point jj + 1
                issue(jj);
                wait_upto(vmin0 + jj + 1);
                float2 zlo[2], zw[2], zc[2], zd[2], zg[2], zF0[2], Eb[2];
                float tn;
                float2 In[2];
                fetch(jj + 1, tn, In);
    #pragma unroll
                for (int p = 0; p < 2; ++p) {
                    // past its window a walk re-reads its last point (lo >= EM, pre-pass): no edges
                    // remain below EM for it, whatever its zone arithmetic produces
                    const float2 lo = poly2(cb[p], f2(tq)), hi = POINT ? lo : poly2(cf[p], f2(tq));
                    const float2 s = add2(lo, hi);
                    const float2 c = mul2(mul2(sdir2, sub2(pI[p], Iq[p])), rcp2(sub2(s, ps[p])));
                    const float2 w = sub2(phi[p], plo[p]);
                    const float2 d = sub2(cq[p], c);
                    const float2 rw = rcp2(max2(w, f2(1e-30f)));
                    zlo[p] = plo[p];
                    zw[p] = w;
                    zc[p] = c;
                    zd[p] = d;
                    zg[p] = mul2(d, mul2(rw, f2(-0.5f)));
                    zF0[p] = zF[p];
                    Eb[p] = min2(lo, f2(EM));
                    // F at the next zone's start: F(lo) = F(plo) + c (lo - plo) + w d / 2
                    zF[p] = fma2(f2(0.5f), mul2(w, d), fma2(c, sub2(lo, plo[p]), zF[p]));
                    plo[p] = lo;
                    phi[p] = hi;
                    ps[p] = s;
                    pI[p] = Iq[p];
                    cq[p] = c;
                    Iq[p] = In[p];
                }
                tq = tn;
                // ---- edges of zone jj - 1: En .. floor(min(lo_jj, EM)), a warp-uniform trip count
                uint32_t es[4];
                float2 x[2], cm[2], fl[2];
                float kmax = 0.f;
    #pragma unroll
                for (int p = 0; p < 2; ++p) {
                    es[2 * p] = (uint32_t)__float_as_int(En[p].x + fbias) << 9;  // plane * plane bytes (mod RB)
                    es[2 * p + 1] = (uint32_t)__float_as_int(En[p].y + fbias) << 9;
                    fl[p] = add2(make_float2(floorf(Eb[p].x), floorf(Eb[p].y)), f2(1.f));  // first edge after the zone
                    const float2 cnt = sub2(fl[p], En[p]);  // edges of this zone (exact small integers)
                    kmax = fmaxf(kmax, fmaxf(cnt.x, cnt.y));
                    cm[p] = sub2(cnt, f2(1.f));  // trip k stores iff k <= cnt - 1
                    x[p] = sub2(En[p], zlo[p]);   // advanced by +1 per trip (the edge test is on k, exact)
                }
                const int K = __reduce_max_sync(0xffffffffu, (int)kmax);
                float kf = 0.f;
                DAXM_UNROLL(DAXM_LOCK_KUNROLL)
                for (int k = 0; k < K; ++k, kf += 1.f) {
    #pragma unroll
                    for (int p = 0; p < 2; ++p) {
                        const float2 xc = min2(x[p], zw[p]);
                        const float2 F = fma2(xc, fma2(zg[p], xc, zd[p]), fma2(zc[p], x[p], zF0[p]));
                        const float2 o = sub2(F, Fp[p]);
                        // predicated store + Fp update (setp inside the asm: no branch, no address remat)
                        edge_store(out_lane + (es[2 * p] & (uint32_t)((RB - 1) << 9)) + (2 * p) * 128, o.x, F.x, kf,
                                   cm[p].x, Fp[p].x);
                        edge_store(out_lane + (es[2 * p + 1] & (uint32_t)((RB - 1) << 9)) + (2 * p + 1) * 128, o.y, F.y,
                                   kf, cm[p].y, Fp[p].y);
                        x[p] = add2(x[p], f2(1.f));
                        es[2 * p] += 512u;
                        es[2 * p + 1] += 512u;
                    }
                }
                // next edge of each walk (edges <= Eb evaluated or, past the window, constant)
    #pragma unroll
                for (int p = 0; p < 2; ++p) En[p] = max2(En[p], fl[p]);
    #if DAXM_LOCK_CHECK
                {   // planes written this iteration must lie below done_p + RB (pre-pass guarantee)
                    const float lim = (float)(done_p + RB - m_ref + 1);  // edge bound: e - 1 < done_p + RB
    #pragma unroll
                    for (int p = 0; p < 2; ++p) {
                        if (cm[p].x >= 0.f && En[p].x - 1.f >= lim) viol = 1u;  // highest edge stored this iteration
                        if (cm[p].y >= 0.f && En[p].y - 1.f >= lim) viol = 1u;
                    }
                }
    #endif
                drain(frontier());
            }
    #if DAXM_LOCK_CHECK
            if (viol && a.lock_err) atomicAdd(a.lock_err, 1u);
    #endif
        } else {
            float2 plo[2], phi[2], ps[2], pI[2], cq[2], Fp[2], En[2], Iq[2];
            // ramp superposition: F(E) = Lr + A (E - plo) + sum over the last
            // LOCK_P ramps of d_s G_s(E); older ramps are retired into the linear part (Lr, A)
            float2 Lr[2], A[2], slo[2][LOCK_P], sw[2][LOCK_P], sk[2][LOCK_P], sd[2][LOCK_P];
            float tq;
            {
                float t0;
                fetch(0, t0, pI);
    #pragma unroll
                for (int p = 0; p < 2; ++p) {
                    plo[p] = poly2(cb[p], f2(t0));  // lo edge / hi edge: fixed order over the tile (pre-pass)
                    phi[p] = POINT ? plo[p] : poly2(cf[p], f2(t0));
                    ps[p] = add2(plo[p], phi[p]);
                    cq[p] = Fp[p] = Lr[p] = A[p] = f2(0.f);
    #pragma unroll
                    for (int u = 0; u < LOCK_P; ++u) {  // empty slots: zero coefficient, finite shape
                        slo[p][u] = plo[p];
                        sw[p][u] = f2(1.f);
                        sk[p][u] = sd[p][u] = f2(0.f);
                    }
                    // first edge: the first above point 0's lo (F = 0 below it); inactive walks never evaluate
                    En[p].x = act[2 * p] ? fmaxf(E0, floorf(plo[p].x) + 1.f) : EM + 1.f;
                    En[p].y = act[2 * p + 1] ? fmaxf(E0, floorf(plo[p].y) + 1.f) : EM + 1.f;
                }
                fetch(1, tq, Iq);
            }
            const float2 sdir2 = f2(2.f * a.sign * (float)dir);  // c = 2 s dir dI / (sum_{q+1} - sum_q)
            const int m_ref = a.m_ref;
            // bits(E + fbias) = 0x4B000000 + e - 1 + RB for edge index e: plane e - 1 mod RB in the low bits
            const float fbias = 8388608.f + (float)(m_ref - 1 + RB);
            // planes below the slowest walk's next edge are final; a finished or inactive walk sits at
            // edge M + 1 (its last point lies above the bins: pre-pass), so it never holds them back
            auto frontier = [&]() {
                const float fr = fminf(fminf(En[0].x, En[0].y), fminf(En[1].x, En[1].y));
                return __reduce_min_sync(0xffffffffu, (int)fr + m_ref) - 1;  // planes < edge - 1
            };
            drain(frontier());
    #if DAXM_LOCK_CHECK
            unsigned viol = 0u;
    #endif

            // iteration jj closes zone jj - 1 of every walk; before its own window a walk's zones lie
            // below the bins (F offset only), after it above them (no edge left: pre-pass)
            // blocks of LOCK_P steps so that ramp jj - 1 goes to the static slot (jj - 1) % LOCK_P;
            // steps past the last visit close no zone (every walk's last point lies above EM)
            float2 zlo_next[2];
    #pragma unroll 1
            for (int jb = 1; jb < niter; jb += LOCK_P)
    #pragma unroll
            for (int u = 0; u < LOCK_P; ++u) {
                const int jj = jb + u;
                // point jj (prefetched); refill the ring below the slowest walk; prefetch point jj + 1
                issue(jj);
                wait_upto(vmin0 + jj + 1);
                float2 Eb[2], off[2][LOCK_P];
                float tn;
                float2 In[2];
                fetch(jj + 1, tn, In);
    #pragma unroll
                for (int p = 0; p < 2; ++p) {
                    const float2 lo = poly2(cb[p], f2(tq)), hi = POINT ? lo : poly2(cf[p], f2(tq));
                    const float2 s = add2(lo, hi);
                    const float2 c = mul2(mul2(sdir2, sub2(pI[p], Iq[p])), rcp2(sub2(s, ps[p])));  // pair jj - 1
                    const float2 w = sub2(phi[p], plo[p]);          // ramp jj - 1 = point jj - 1's edge span
                    const float2 d = sub2(c, cq[p]);                // its coefficient c_{jj-1} - c_{jj-2}
                    // retire ramp jj - 1 - LOCK_P (finished below plo: pre-pass) into the linear part
                    const float2 h = sub2(sub2(plo[p], slo[p][u]), mul2(f2(0.5f), sw[p][u]));
                    Lr[p] = fma2(sd[p][u], h, Lr[p]);
                    A[p] = add2(A[p], sd[p][u]);
                    slo[p][u] = plo[p];
                    sw[p][u] = w;
                    sd[p][u] = d;
                    sk[p][u] = mul2(d, mul2(rcp2(max2(w, f2(1e-30f))), f2(0.5f)));
    #pragma unroll
                    for (int v = 0; v < LOCK_P; ++v) off[p][v] = sub2(plo[p], slo[p][v]);
                    Eb[p] = min2(lo, f2(EM));
                    ps[p] = s;
                    pI[p] = Iq[p];
                    cq[p] = c;
                    Iq[p] = In[p];
                    phi[p] = hi;
                    // (plo moves to lo after the zone's edges; the linear part follows it then)
                    zlo_next[p] = lo;
                }
                tq = tn;
                // ---- edges of zone jj - 1: En .. floor(min(lo_jj, EM)), a warp-uniform trip count
                uint32_t es[4];
                float2 x[2], cm[2], fl[2];
                float kmax = 0.f;
    #pragma unroll
                for (int p = 0; p < 2; ++p) {
                    es[2 * p] = (uint32_t)__float_as_int(En[p].x + fbias) << 9;  // plane * plane bytes (mod RB)
                    es[2 * p + 1] = (uint32_t)__float_as_int(En[p].y + fbias) << 9;
                    fl[p] = add2(make_float2(floorf(Eb[p].x), floorf(Eb[p].y)), f2(1.f));  // first edge after the zone
                    const float2 cnt = sub2(fl[p], En[p]);  // edges of this zone (exact small integers)
                    kmax = fmaxf(kmax, fmaxf(cnt.x, cnt.y));
                    cm[p] = sub2(cnt, f2(1.f));  // trip k stores iff k <= cnt - 1
                    x[p] = sub2(En[p], plo[p]);   // advanced by +1 per trip (the edge test is on k, exact)
                }
                const int K = __reduce_max_sync(0xffffffffu, (int)kmax);
                float kf = 0.f;
                DAXM_UNROLL(DAXM_LOCK_KUNROLL)
                for (int k = 0; k < K; ++k, kf += 1.f) {
    #pragma unroll
                    for (int p = 0; p < 2; ++p) {
                        float2 F = fma2(A[p], x[p], Lr[p]);
    #pragma unroll
                        for (int v = 0; v < LOCK_P; ++v) {  // ramp v: d (xs - xc) + d/(2w) xc^2, xs >= 0
                            const float2 xs = add2(x[p], off[p][v]);
                            const float2 xc = min2(xs, sw[p][v]);
                            F = fma2(sd[p][v], sub2(xs, xc), F);
                            F = fma2(mul2(sk[p][v], xc), xc, F);
                        }
                        const float2 o = sub2(F, Fp[p]);
                        // predicated store + Fp update (setp inside the asm: no branch, no address remat)
                        edge_store(out_lane + (es[2 * p] & (uint32_t)((RB - 1) << 9)) + (2 * p) * 128, o.x, F.x, kf,
                                   cm[p].x, Fp[p].x);
                        edge_store(out_lane + (es[2 * p + 1] & (uint32_t)((RB - 1) << 9)) + (2 * p + 1) * 128, o.y, F.y,
                                   kf, cm[p].y, Fp[p].y);
                        x[p] = add2(x[p], f2(1.f));
                        es[2 * p] += 512u;
                        es[2 * p + 1] += 512u;
                    }
                }
                // next edge of each walk (edges <= Eb evaluated or, past the window, constant)
    #pragma unroll
                for (int p = 0; p < 2; ++p) {
                    En[p] = max2(En[p], fl[p]);
                    Lr[p] = fma2(A[p], sub2(zlo_next[p], plo[p]), Lr[p]);  // linear part's origin -> lo_jj
                    plo[p] = zlo_next[p];
                }
    #if DAXM_LOCK_CHECK
                {   // planes written this iteration must lie below done_p + RB (pre-pass guarantee)
                    const float lim = (float)(done_p + RB - m_ref + 1);  // edge bound: e - 1 < done_p + RB
    #pragma unroll
                    for (int p = 0; p < 2; ++p) {
                        if (cm[p].x >= 0.f && En[p].x - 1.f >= lim) viol = 1u;  // highest edge stored this iteration
                        if (cm[p].y >= 0.f && En[p].y - 1.f >= lim) viol = 1u;
                    }
                }
    #endif
                drain(frontier());
            }
    #if DAXM_LOCK_CHECK
            if (viol && a.lock_err) atomicAdd(a.lock_err, 1u);
    #endif
        }
    }
    drain(M);
    // every issued input load has been waited for (wait_upto reached vend), so the CTA may exit
}
// ------------------------------------------------------------------ pre-pass
// Replays, per tile and lock warp, the kernel's warp-locked walks with its own fp32 arithmetic
// (lock_poly, fminf, floorf) and classifies the tile:
//   * the same pixel edge (back or front) is the shallower one at every point any walk of the
//     tile evaluates (the kernel then skips the per-point min/max; flag LOCK_FRONT_LO);
//   * consecutive points of a walk have distinct edge sums (finite zone densities, also before
//     and after the walk's own window);
//   * every window's last point lies at or above the top bin edge EM, so a walk past its
//     window has no edge left (the kernel needs no end-of-window case);
//   * the output-ring need, max over iterations j of
//       (furthest edge written at j) - (slowest walk's next edge after j - 1) + 1,
//     fits LOCK_RB_SMALL or LOCK_RB_LARGE planes -> lock = that class (0: not eligible).
// Inactive walks (intensity cutoff) only lower the need, so the plan-time answer holds for
// every cutoff.  d_stats: [0] small, [1] large, [2] fast-path tiles left to deposit_fast.
__global__ void __launch_bounds__(256) lock_prepass_kernel(DepositArgs a, TileInfo* __restrict__ tiles,
                                                           int* __restrict__ d_stats) {
    const int tile = blockIdx.x;
    TileInfo ti = tiles[tile];
    const int tr = tile / a.n_tc, tc = tile % a.n_tc;
    const int row0 = (a.tr0 + tr) * TILE_R;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;  // 8 warps = TILE_R / 16 lock warps
    const int col = lane & 7, rg = lane >> 3;
    const int wrow = warp * LOCK_ROWS;
    __shared__ int s_need, s_bad, s_back_lo, s_front_lo;
    if (threadIdx.x == 0) {
        s_need = s_bad = 0;
        s_back_lo = s_front_lo = 1;
    }
    __syncthreads();
    // overlapping tiles -> deposit_lock<..., OV = true> (ramp superposition); finite pixels only
    const bool ov = ti.separated == MODE_OVERLAP && a.lock_ov_enabled && !a.point_mode;
    const bool eligible = (ti.separated == MODE_SEPARATED || ov) && row0 >= a.row_begin && ti.k_hi >= ti.k_lo &&
                          a.table == nullptr && (ti.k_hi - ti.k_lo + 1) <= MAX_FAST_NV;
    if (eligible) {
        const int i = tc * TILE_C + col;
        const float E0 = (float)(-a.m_ref), EM = (float)(a.M - a.m_ref);
        float cb[4][3] = {}, cf[4][3] = {}, En[4], ps[4] = {}, hq[4][LOCK_P] = {};
        bool on[4];
        int vmin0 = INT_MAX, vend = INT_MIN;
        bool back_lo = true, front_lo = true, bad = false;
        auto point = [&](int w, int v, float& x0, float& x1) {
            const int k = ti.dir > 0 ? ti.k_lo + v : ti.k_hi - v;
            const float t = (float)(a.t[k] - ti.t_ref);
            x0 = lock_poly(cb[w][0], cb[w][1], cb[w][2], t);
            x1 = a.point_mode ? x0 : lock_poly(cf[w][0], cf[w][1], cf[w][2], t);
            back_lo &= x0 <= x1;
            front_lo &= x1 <= x0;
        };
        for (int w = 0; w < 4; ++w) {
            const int r = wrow + 4 * w + rg;
            const LockWalk lw = lock_walk(a, ti, row0 + r, i, true);
            on[w] = lw.npts > 0;
            lock_coef(a, tile, r, col, a.point_mode != 0, cb[w], cf[w]);
            if (on[w]) {
                vmin0 = min(vmin0, lw.v0);
                vend = max(vend, lw.v0 + lw.npts - 1);
                float x0, x1;
                point(w, lw.v0 + lw.npts - 1, x0, x1);
                bad |= !(fminf(x0, x1) >= EM);  // last point at or above the top bin edge
            }
        }
        vmin0 = __reduce_min_sync(0xffffffffu, vmin0);
        vend = __reduce_max_sync(0xffffffffu, vend);
        const int niter = vend >= vmin0 ? vend - vmin0 + 1 : 0;
        int need = 0;
        if (niter > 0) {
            for (int w = 0; w < 4; ++w) {
                En[w] = EM + 1.f;
                if (!on[w]) continue;
                float x0, x1;
                point(w, vmin0, x0, x1);
                En[w] = fmaxf(E0, floorf(fminf(x0, x1)) + 1.f);
                ps[w] = x0 + x1;
                hq[w][0] = fmaxf(x0, x1);
            }
            float fr = fminf(fminf(En[0], En[1]), fminf(En[2], En[3]));
            int fr_e = __reduce_min_sync(0xffffffffu, (int)fr + a.m_ref);
            for (int jj = 1; jj < niter; ++jj) {  // iterations >= niter close no edge (last points >= EM)
                float mx = -3.0e38f;
                for (int w = 0; w < 4; ++w) {
                    if (!on[w]) continue;
                    float x0, x1;
                    point(w, vmin0 + jj, x0, x1);
                    if (ov) {  // the ramp LOCK_P steps back has finished below this point's lo
                        if (jj >= LOCK_P) bad |= !(hq[w][jj % LOCK_P] <= fminf(x0, x1));
                        hq[w][jj % LOCK_P] = fmaxf(x0, x1);
                    }
                    const float sum = x0 + x1;
                    bad |= !(sum != ps[w]);  // the zone density needs a finite 1 / (sum - previous sum)
                    ps[w] = sum;
                    const float Eb = fminf(fminf(x0, x1), EM);
                    if (En[w] <= Eb) mx = fmaxf(mx, Eb);
                    En[w] = fmaxf(En[w], floorf(Eb) + 1.f);
                }
                const int wr = __reduce_max_sync(0xffffffffu, mx < -1.0e37f ? INT_MIN : (int)floorf(mx) + a.m_ref);
                if (wr != INT_MIN) need = max(need, wr - fr_e + 1);
                fr = fminf(fminf(En[0], En[1]), fminf(En[2], En[3]));
                fr_e = __reduce_min_sync(0xffffffffu, (int)fr + a.m_ref);
            }
        }
        if (lane == 0) atomicMax(&s_need, need);
        if (bad) atomicOr(&s_bad, 1);
        if (!back_lo) atomicAnd(&s_back_lo, 0);
        if (!front_lo) atomicAnd(&s_front_lo, 0);
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        int lock = 0;
        if (eligible && !s_bad && (s_back_lo || s_front_lo)) {
            if (s_need <= lock_need_max(LOCK_RB_SMALL))
                lock = LOCK_RB_SMALL;
            else if (s_need <= lock_need_max(LOCK_RB_LARGE))
                lock = LOCK_RB_LARGE;
            if (lock && ov) lock |= LOCK_OVB;
            if (lock && !s_back_lo) lock |= LOCK_FRONT_LO;
        }
        ti.lock = lock;
        tiles[tile] = ti;
        if ((lock & LOCK_CLASS_MASK) == LOCK_RB_SMALL) atomicAdd(&d_stats[0], 1);
        if ((lock & LOCK_CLASS_MASK) == LOCK_RB_LARGE) atomicAdd(&d_stats[1], 1);
        if ((lock & LOCK_CLASS_MASK) == (LOCK_RB_SMALL | LOCK_OVB)) atomicAdd(&d_stats[3], 1);
        if ((lock & LOCK_CLASS_MASK) == (LOCK_RB_LARGE | LOCK_OVB)) atomicAdd(&d_stats[4], 1);
        if (!lock && ti.separated != MODE_GENERAL) atomicAdd(&d_stats[2], 1);
    }
}

template <typename T, bool POINT, int RB, bool OV>
cudaError_t launch_lock_rb(const CUtensorMap* in_map, float* out, const DepositArgs& a, int n_tiles, cudaStream_t st) {
    const size_t sm = LockSmem<T, RB>::bytes(a.max_nv);
    auto kern = deposit_lock<T, POINT, RB, OV>;
    static std::atomic<unsigned long long> attr_done{0};  // per device (attributes are per device)
    cudaError_t ea = once_per_device(attr_done, [&]() {
        cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             (int)LockSmem<T, RB>::bytes(MAX_FAST_NV));
        if (e != cudaSuccess) return e;
        return cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout,
                                    (int)cudaSharedmemCarveoutMaxShared);
    });
    if (ea != cudaSuccess) return ea;
    kern<<<(unsigned)(n_tiles * LOCK_SUBS), LK_THREADS, sm, st>>>(*in_map, out, a);
    return cudaGetLastError();
}

template <typename T>
cudaError_t launch_lock_t(const DepositArgs& a, const CUtensorMap* in_map, float* out, int n_tiles,
                          const cudaStream_t* sts, int nst) {
    // one launch per tile class; class i goes to stream i mod nst (the classes own disjoint
    // tiles, so with nst > 1 they run concurrently and share each other's tails)
    cudaError_t e = cudaSuccess;
    int i = 0;
    if (a.lock_small > 0)
        e = a.point_mode ? launch_lock_rb<T, true, LOCK_RB_SMALL, false>(in_map, out, a, n_tiles, sts[i++ % nst])
                         : launch_lock_rb<T, false, LOCK_RB_SMALL, false>(in_map, out, a, n_tiles, sts[i++ % nst]);
    if (e != cudaSuccess) return e;
    if (a.lock_large > 0)
        e = a.point_mode ? launch_lock_rb<T, true, LOCK_RB_LARGE, false>(in_map, out, a, n_tiles, sts[i++ % nst])
                         : launch_lock_rb<T, false, LOCK_RB_LARGE, false>(in_map, out, a, n_tiles, sts[i++ % nst]);
    if (e != cudaSuccess) return e;
    // overlapping tiles (never POINT pixels: a point has no edge span)
    if (a.lock_ov_small > 0 && !a.point_mode)
        e = launch_lock_rb<T, false, LOCK_RB_SMALL, true>(in_map, out, a, n_tiles, sts[i++ % nst]);
    if (e != cudaSuccess) return e;
    if (a.lock_ov_large > 0 && !a.point_mode)
        e = launch_lock_rb<T, false, LOCK_RB_LARGE, true>(in_map, out, a, n_tiles, sts[i++ % nst]);
    return e;
}

}  // namespace

size_t lock_smem_bytes(int dtype, int rb, int max_nv) {
    if (dtype == DAXM_U16)
        return rb == LOCK_RB_SMALL ? LockSmem<uint16_t, LOCK_RB_SMALL>::bytes(max_nv)
                                   : LockSmem<uint16_t, LOCK_RB_LARGE>::bytes(max_nv);
    return rb == LOCK_RB_SMALL ? LockSmem<float, LOCK_RB_SMALL>::bytes(max_nv)
                               : LockSmem<float, LOCK_RB_LARGE>::bytes(max_nv);
}

cudaError_t launch_lock(const DepositArgs& a, const CUtensorMap* in_map, float* out, int dtype, int n_tiles,
                        const cudaStream_t* sts, int nst) {
    if (n_tiles <= 0) return cudaSuccess;
    return dtype == DAXM_U16 ? launch_lock_t<uint16_t>(a, in_map, out, n_tiles, sts, nst)
                             : launch_lock_t<float>(a, in_map, out, n_tiles, sts, nst);
}

cudaError_t launch_lock_prepass(const DepositArgs& a, int n_tiles, int* d_stats, cudaStream_t st) {
    if (n_tiles <= 0) return cudaSuccess;
    lock_prepass_kernel<<<(unsigned)n_tiles, 256, 0, st>>>(a, const_cast<TileInfo*>(a.tiles), d_stats);
    return cudaGetLastError();
}

}  // namespace daxm
