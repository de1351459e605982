// deposit_row.cu -- the production gather deposit and the pre-pass
// replay that admits a row tile to it.
//
// What is computed: per pixel, with the step pairs visited in the order their
// trapezoids move deeper and c_q = dI_q / A_q, the intensity deposited below bin edge E is,
// inside zone q = [lo_q, lo_{q+1}),
//     F(E) = F(lo_q) + c_q x + xc (d_q + g_q xc),  x = E - lo_q, xc = min(x, w_q),
//     d_q = c_{q-1} - c_q,  g_q = -d_q / (2 w_q),  w_q = hi_q - lo_q,
// (separated spans; the general-span variant keeps pairs v, v-1, v-2 open) and bin m = [E_m, E_{m+1})
// receives F(E_{m+1}) - F(E_m): the trapezoid overlaps of P:L320-331 (device_depth_resolve_pixel /
// device_get_trapezoid_height) summed over the pairs, one owner per (bin,
// pixel), no atomics.  dI_q = s (I_q - I_{q+1}) (readings R1, R2) is formed
// from the streamed planes.
//
// Schedule.  One warp = one row tile of 2 detector rows x 64 columns; lane l owns two adjacent
// columns of one column half (both rows): two walk pairs packed fp32x2.  All lanes advance one visit
// (wire step) per iteration in lock step, each from its own middle-aligned start, so the 128 walks
// of a warp stay within a few bins of each other; a point closes the zone of each walk and that
// zone's bin edges receive F through 3, 4 (+ a rare 5th) or 5 (+ a rare 6th) unrolled predicated
// stores (edge-trip class of the tile).  The schedule depends on geometry alone (inactive walks keep
// advancing, they just store nothing), so an active walk's output is bit-identical whatever the cutoff.
//
//   input : per column half, TMA loads of [4 steps][2 rows][32 cols] boxes into a 24-slot ring (32
//           for tiles whose lanes spread wider), one mbarrier per group; lane 0 refills the slots
//           every lane has read past, once per four iterations.
//   output: F staging -- a ring of RB planes [2][64] fp32 (+ trips - 1 overflow planes, so that the
//           unrolled edge stores use immediate offsets) holds F at each bin edge; once the slowest
//           walk has passed edge P + 1 every lane subtracts its 16 bytes of edges P and P + 1 and
//           writes plane P with one st.global.cs.v4 (the warp writes two 256-byte rows: the pattern
//           that reaches the copy ceiling, profiles/r02b_membench.md).
// The pre-pass (row_admit_kernel) replays every warp's schedule with the kernel's own fp32
// arithmetic and admits a tile only if the output ring, the unrolled edge loop and the input ring
// provably suffice; the rest goes to the general kernel.
#include <cuda.h>
#include <cuda_runtime.h>
#include <limits.h>
#include <stdint.h>
#include <stdlib.h>

#include <atomic>
#include <type_traits>

#include "daxm_internal.cuh"
#include "fp2.cuh"
#include "ptx.cuh"

#ifndef DAXM_ROW_TU
#define DAXM_ROW_TU 0  // which instance set this translation unit compiles (see the end of the file)
#endif
#define DAXM_PRAGMA_(x) _Pragma(#x)
#define DAXM_PRAGMA_UNROLL(n) DAXM_PRAGMA_(unroll n)
#ifndef DAXM_ROW_CHECK
#define DAXM_ROW_CHECK 0  // 1: count schedule violations in the kernel (the pre-pass makes them impossible)
#endif

namespace daxm {
namespace {
using namespace ptx;

constexpr int PLANE_B = RW_ROWS * RW_COLS * 4;  // one staged output plane (512 B)
template <typename T, int RB, int KT = RW_KT, int NB = RW_NB>
struct RowSmem {
    static constexpr int NG = NB / RW_G;  // input groups in the ring
    static constexpr int OUT_SLOTS = RB + KT - 1;
    static constexpr int IN_SLOT = RW_ROWS * 32 * (int)sizeof(T);  // one step of one column half
    static constexpr int IN_GROUP = RW_G * IN_SLOT;                // one TMA box
    static constexpr int IN_HALF = NB * IN_SLOT;                   // a half's ring
    static constexpr int OFF_OUT = 0;
    static constexpr int OFF_IN = OFF_OUT + OUT_SLOTS * PLANE_B;
    static constexpr int OFF_BAR = OFF_IN + RW_H * IN_HALF;
    static constexpr int OFF_TAU = OFF_BAR + NG * 8;
    static size_t bytes(int max_nv) { return (size_t)OFF_TAU + (DAXM_ROW_TAU_LINEAR ? 0 : 4 * (size_t)(max_nv + 4)) + 128; }
};

__device__ __forceinline__ void sts_zero4(uint32_t addr) {
    asm volatile("st.shared.v4.f32 [%0], {%1, %1, %1, %1};" ::"r"(addr), "f"(0.f) : "memory");
}
__device__ __forceinline__ float4 lds128(uint32_t addr) {
    float4 v;
    asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "r"(addr)
                 : "memory");
    return v;
}
__device__ __forceinline__ uint4 lds128u(uint32_t addr) {
    uint4 v;
    asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "r"(addr)
                 : "memory");
    return v;
}
__device__ __forceinline__ void sts128u(uint32_t addr, uint4 v) {
    asm volatile("st.shared.v4.u32 [%0], {%1, %2, %3, %4};" ::"r"(addr), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w)
                 : "memory");
}
constexpr uint32_t SENT = 0x7fbadbadu;  // overflow slot not written this lap (a NaN no arithmetic yields)
__device__ __forceinline__ void sts128(uint32_t addr, float4 v) {
    asm volatile("st.shared.v4.f32 [%0], {%1, %2, %3, %4};" ::"r"(addr), "f"(v.x), "f"(v.y), "f"(v.z), "f"(v.w)
                 : "memory");
}
// Edge store of trip k: if k < cnt, staged[addr + OFF] = o and Fp = F (one FSETP, no branch).
template <int OFF>
__device__ __forceinline__ void edge_st(uint32_t addr, float o, float F, float kf, float cnt, float& Fp) {
    asm volatile(
        "{\n .reg .pred q;\n setp.lt.f32 q, %3, %4;\n @q st.shared.f32 [%1+%6], %2;\n @q mov.f32 %0, %5;\n}\n"
        : "+f"(Fp)
        : "r"(addr), "f"(o), "f"(kf), "f"(cnt), "f"(F), "n"(OFF)
        : "memory");
}
__device__ __forceinline__ void stg_cs_v4(float* g, float4 v) {  // streaming store (evict first)
    asm volatile("st.global.cs.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(g), "f"(v.x), "f"(v.y), "f"(v.z), "f"(v.w)
                 : "memory");
}
__device__ __forceinline__ void stg_cs_v4_if(float* g, float2 a, float2 b, bool pred) {  // iff pred
    asm volatile("{\n .reg .pred q;\n setp.ne.u32 q, %5, 0;\n @q st.global.cs.v4.f32 [%0], {%1, %2, %3, %4};\n}\n" ::"l"(g),
                 "f"(a.x), "f"(a.y), "f"(b.x), "f"(b.y), "r"((unsigned)pred)
                 : "memory");
}
__device__ __forceinline__ void red_add_v4(float* g, float4 v) {  // one add per element (sm_90+)
    asm volatile("red.global.add.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(g), "f"(v.x), "f"(v.y), "f"(v.z), "f"(v.w)
                 : "memory");
}
__device__ __forceinline__ uint32_t lds_u32(uint32_t addr) {
    uint32_t v;
    asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(addr) : "memory");
    return v;
}
__device__ __forceinline__ float2 lds_f2(uint32_t addr) {
    float2 v;
    asm volatile("ld.shared.v2.f32 {%0, %1}, [%2];" : "=f"(v.x), "=f"(v.y) : "r"(addr) : "memory");
    return v;
}
// st.shared.f32 [addr + OFF] = v iff k < cnt (one FSETP, a predicated store)
template <int OFF>
__device__ __forceinline__ void st_if(uint32_t addr, float v, float kf, float cnt) {
    asm volatile("{\n .reg .pred q;\n setp.lt.f32 q, %2, %3;\n @q st.shared.f32 [%0+%4], %1;\n}\n" ::"r"(addr),
                 "f"(v), "f"(kf), "f"(cnt), "n"(OFF)
                 : "memory");
}
template <typename T, int OFF>
__device__ __forceinline__ float lds_in(uint32_t addr) {
    if constexpr (sizeof(T) == 2) {
        unsigned short v;
        asm volatile("ld.shared.u16 %0, [%1+%2];" : "=h"(v) : "r"(addr), "n"(OFF) : "memory");
        return (float)v;
    } else {
        float v;
        asm volatile("ld.shared.f32 %0, [%1+%2];" : "=f"(v) : "r"(addr), "n"(OFF) : "memory");
        return v;
    }
}

// Overflow fold of a staged slot at `ad` holding x: the value a walk wrote through the overflow slot
// (ad + RB planes) where one was written (not SENT), else x; written back to the direct slot (a later
// plane reads it as its lower edge) and the overflow slot re-armed.
template <int RB>
__device__ __forceinline__ uint4 fold_slot(uint32_t ad, uint4 x) {
    const uint4 y = lds128u(ad + RB * PLANE_B);
    x = make_uint4(y.x == SENT ? x.x : y.x, y.y == SENT ? x.y : y.y, y.z == SENT ? x.z : y.z, y.w == SENT ? x.w : y.w);
    sts128u(ad, x);
    sts128u(ad + RB * PLANE_B, make_uint4(SENT, SENT, SENT, SENT));
    return x;
}

// compile-time loop: f(integral_constant<int, k>) for k = K0 .. KN - 1 while f returns true
template <int K0, int KN, typename F>
__device__ __forceinline__ void static_for(F&& f) {
    if constexpr (K0 < KN) {
        if (f(std::integral_constant<int, K0>{})) static_for<K0 + 1, KN>(f);
    }
}

// ---- per-walk geometry shared by the kernel and its replay
struct RowWalk {
    int v0, npts;  // first visit (index into the tile's step list, ascending depth), points (0: none)
};
__device__ __forceinline__ RowWalk row_walk(const RowArgs& a, const RowTile& ti, int j, int i) {
    RowWalk w{0, 0};
    if (j < a.row_begin || j >= a.row_end || i >= a.C) return w;
    const int2 win = a.win[(size_t)(j - a.pre_row0) * a.C + i];
    if (win.y <= win.x) return w;
    w.v0 = ti.dir > 0 ? win.x - ti.k_lo : ti.k_hi - win.y;
    w.npts = win.y - win.x + 1;
    return w;
}
// depth polynomials of a walk's two pixel edges: edge column e (back) and e + 1 (front; POINT: e)
__device__ __forceinline__ void row_coef(const RowArgs& a, int rt, int row, int e, float c[3]) {
#pragma unroll
    for (int m = 0; m < 3; ++m) c[m] = a.coef[(((size_t)rt * NCOEF + m) * (RW_COLS + 1) + e) * RW_ROWS + row];
}

// ------------------------------------------------------------------ kernel
static_assert(RW_H == 2 && RW_ROWS == 2, "deposit_row: two column halves per lane, two rows");

// Loop-carried state of one lane: walk pair p = column half p (column col0 + lane + 32 p), rows
// row0 (x) and row0 + 1 (y); the point last visited (plo, phi, ps = lo + hi, pI) and the
// prefetched next one (tq, Iq).
struct RowState {
    float2 plo[2], phi[2], ps[2], pI[2], cq[2], zF[2], En[2], Iq[2];
    // general-span variant only (dead otherwise): c_{v-2}, hi_{v-1}, M_{v-2} (start of pair v-2's
    // falling ramp) and 1 / that ramp's width
    float2 cq2[2], phm[2], pM[2], if2[2];
    float tq;
};

// warp-wide integer min / max (redux.sync, full mask; the loop is convergent by construction)
__device__ __forceinline__ int warp_min(int x) {
    int r;
    asm volatile("redux.sync.min.s32 %0, %1, 0xffffffff;" : "=r"(r) : "r"(x));
    return r;
}
__device__ __forceinline__ int warp_max(int x) {
    int r;
    asm volatile("redux.sync.max.s32 %0, %1, 0xffffffff;" : "=r"(r) : "r"(x));
    return r;
}

// (a << 9) + b in one instruction (LEA): the byte offset of staged plane slot a
__device__ __forceinline__ uint32_t lea9(uint32_t a, uint32_t b) {
    uint32_t r;
    asm("{\n .reg .u32 t;\n shl.b32 t, %1, 9;\n add.u32 %0, t, %2;\n}\n" : "=r"(r) : "r"(a), "r"(b));
    return r;
}
// make a value opaque to the compiler, so that it stays in a register instead of being recomputed
// from constants inside the loop
__device__ __forceinline__ float opaque(float x) {
    asm volatile("" : "+f"(x));
    return x;
}
__device__ __forceinline__ uint32_t opaque(uint32_t x) {
    asm volatile("" : "+r"(x));
    return x;
}
__device__ __forceinline__ int opaque(int x) {
    asm volatile("" : "+r"(x));
    return x;
}

// Lane -> walks.  Lane l covers column half h = l / 16 of the tile's 64 columns, columns
// 32 h + 2 i and 32 h + 2 i + 1 (i = l % 16) of both rows: walk pair p = column 32 h + 2 i + (p ^ h)
// (the swap for h = 1 keeps the edge stores of one instruction on 32 distinct banks), rows 0 (x)
// and 1 (y).  Both columns of a lane are adjacent, so the lane reads one visit of its half per step.
__device__ __forceinline__ int rw_col(int lane, int p) { return 32 * (lane >> 4) + 2 * (lane & 15) + (p ^ (lane >> 4)); }

// Lock-step starts (kernel and replay).  A lane covers its four walks' windows [ws, we] (visits from
// the tile's first step).  All lanes advance one visit per iteration, but their depth per visit
// differs slightly across the 64 columns (2.6 % at C4), so lanes that started together drift apart
// by the end of their windows.  Aligning the windows' MIDDLES instead halves the largest spread:
// lane l starts (T - len_l) / 2 visits before its window, T = the warp's longest window (a point
// before a window lies below the bins: no edge), clamped at the tile's first step (row_tile_kernel
// extends the step range by RW_EXT for that).  Visits of column half h are then counted from
// vmin, the half's earliest start.
__device__ __forceinline__ void row_starts(const RowWalk wk[2][2], int lane, int& vmin, int& vs, int& ve, int& vs_max,
                                           int& vend) {
    int ws = INT_MAX, we = -1;
#pragma unroll
    for (int p = 0; p < 2; ++p)
#pragma unroll
        for (int r = 0; r < 2; ++r)
            if (wk[p][r].npts > 0) {
                ws = min(ws, wk[p][r].v0);
                we = max(we, wk[p][r].v0 + wk[p][r].npts - 1);
            }
    const int len = __reduce_max_sync(0xffffffffu, we >= 0 ? we - ws : -1);
    const int st = we >= 0 ? max(ws - ((len - (we - ws)) >> 1), 0) : INT_MAX;
    // per column half (16 lanes): the earliest start
    int m = st;
#pragma unroll
    for (int o = 8; o > 0; o >>= 1) m = min(m, __shfl_xor_sync(0xffffffffu, m, o));
    vmin = m == INT_MAX ? 0 : m;  // a half without windows
    vs = we >= 0 ? st - vmin : 0;  // no window in the lane's columns: done at once
    ve = we >= 0 ? we - vmin : 0;
    vs_max = __reduce_max_sync(0xffffffffu, vs);
    vend = __reduce_max_sync(0xffffffffu, ve);
}

#ifndef DAXM_RW_MINB
#define DAXM_RW_MINB 11  // resident CTAs (= warps) per SM the separated variant's registers allow
#endif
template <typename T, bool POINT, int RB, bool GEN, int NB, bool CLAMP, int KTS>
__global__ void __launch_bounds__(32, GEN ? 8 : DAXM_RW_MINB) deposit_row(const __grid_constant__ CUtensorMap in_map,
                                                            const __grid_constant__ CUtensorMap out_map,
                                                            const RowArgs a) {
    static_assert(!(GEN && POINT), "the general-span variant is for finite pixels");
    // max edges per zone and iteration: the separated variants by class (the tile's largest count,
    // admission replay; every trip unrolled), the general-span variant RW_KT_GEN (5 trips + a rare 6th)
    constexpr int KT = GEN ? RW_KT_GEN : KTS;
    using L = RowSmem<T, RB, KT, NB>;
    constexpr int NG = L::NG;
    static_assert(RB % RW_PB == 0 && (RB & (RB - 1)) == 0, "ring");
    extern __shared__ unsigned char smem_raw[];
    const uint32_t sbase = (smem_u32(smem_raw) + 127u) & ~127u;
    unsigned char* smem = smem_raw + (sbase - smem_u32(smem_raw));
    const int lane = threadIdx.x;
    const int rt = a.list[blockIdx.x];
    const RowTile ti = a.rt[rt];
    const int rr = rt / a.n_rc, rc = rt % a.n_rc;
    const int row0 = a.row_org + rr * RW_ROWS;  // global row of the tile's first row
    const int col0 = rc * RW_COLS;
    const int rowl = row0 - a.row_begin;           // band-local (< 0 for a band start inside the tile: TMA skips)
    const int nvt = ti.k_hi >= ti.k_lo ? ti.k_hi - ti.k_lo + 1 : 0;
    const int dir = ti.dir;
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + L::OFF_BAR);
    float* tau = reinterpret_cast<float*>(smem + L::OFF_TAU);

    if (!DAXM_ROW_TAU_LINEAR)
        for (int q = lane; q < nvt; q += 32) tau[q] = (float)(a.t[dir > 0 ? ti.k_lo + q : ti.k_hi - q] - ti.t_ref);
    if (lane == 0) {
        for (int g = 0; g < NG; ++g) mbar_init(&bars[g], 1);
        fence_mbar_init();
    }
#pragma unroll
    for (int s = 0; s < RB; ++s) sts_zero4(sbase + L::OFF_OUT + s * PLANE_B + lane * 16);
#pragma unroll
    for (int s = RB; s < L::OUT_SLOTS; ++s)
        sts128u(sbase + L::OFF_OUT + s * PLANE_B + lane * 16, make_uint4(SENT, SENT, SENT, SENT));
    __syncwarp();

    // ---- walks: pair p = column col0 + rw_col(lane, p), rows row0 (x) and row0 + 1 (y)
    const float E0 = (float)(-a.m_ref);
    float2 cb[2][3], cf[2][3], gate[2];
    bool any_act = false;
    RowWalk wk[2][2];
    const int hh = lane >> 4;  // the lane's column half
#pragma unroll
    for (int p = 0; p < 2; ++p) {
        const int e = rw_col(lane, p), c = col0 + e;
#pragma unroll
        for (int r = 0; r < 2; ++r) {
            const int j = row0 + r;
            wk[p][r] = row_walk(a, ti, j, c);
            bool on = wk[p][r].npts > 0;
            if (on && a.use_cutoff) {  // intensity cutoff (f1, reading R14)
                const T* s0 = static_cast<const T*>(a.stack) + (size_t)(j - a.row_begin) * a.C + c;
                on = (float)s0[0] >= a.cutoff;
            }
            any_act |= on;  // (a tile with constant intensities, row_live_kernel: none, zeros below)
            (r ? gate[p].y : gate[p].x) = on ? 0.f : 1.0e9f;  // inactive: edge counts below zero
            float cl[3], ch[3];
            row_coef(a, rt, r, (ti.cls & RW_CLS_FRONT_LO) && !POINT ? e + 1 : e, cl);
            row_coef(a, rt, r, (ti.cls & RW_CLS_FRONT_LO) || POINT ? e : e + 1, ch);
#pragma unroll
            for (int m = 0; m < 3; ++m) {
                (r ? cb[p][m].y : cb[p][m].x) = cl[m];
                (r ? cf[p][m].y : cf[p][m].x) = ch[m];
            }
        }
    }
    if (a.live && !a.live[rt]) any_act = false;  // every dI is 0 (exact zero-dI skip)
    if (!__any_sync(0xffffffffu, any_act)) {  // no active walk: the tile's output is zero
        fence_proxy_async_smem();
        __syncwarp();
        if (a.prof_part)  // fused depth profile: this tile adds nothing to any plane
            for (int m = lane; m < a.M; m += 32) a.prof_part[(size_t)rt * a.M + m] = 0.f;
        if (lane == 0 && !a.acc) {  // (adding zeros: nothing to do)
            for (int P = 0; P < a.M; P += RW_PB) tma_store_3d(&out_map, col0, rowl, P, smem + L::OFF_OUT);
            bulk_commit();
            bulk_wait<0>();
        }
        return;
    }
    // visits of the lane's half are counted from the half's earliest start (vmin); the lane starts at
    // vs and ends at ve; all lanes advance in lock step
    int vmin_h, vs, ve, vs_max, vend;
    row_starts(wk, lane, vmin_h, vs, ve, vs_max, vend);
    const int vmin0 = __shfl_sync(0xffffffffu, vmin_h, 0), vmin1 = __shfl_sync(0xffffffffu, vmin_h, 16);

    // ---- input rings, one per column half: visit v of half p in slot (v ^ xr) mod RW_NB; group g =
    // visits [RW_G g, RW_G g + RW_G) of both halves = two TMA boxes of consecutive steps on one
    // mbarrier (ascending k: for dir < 0 a group's visits land in reverse slot order)
    const int xr = dir > 0 ? 0 : RW_G - 1;
    const int ngroups = vend / RW_G + 1;
    const int kb0 = dir > 0 ? ti.k_lo + vmin0 : ti.k_hi - vmin0 - (RW_G - 1);
    const int kb1 = dir > 0 ? ti.k_lo + vmin1 : ti.k_hi - vmin1 - (RW_G - 1);
    int g_issue = 0, g_wait = 0;
    auto issue_upto = [&](int lim) {  // groups <= lim (clamped) may be in flight
        lim = min(lim, ngroups - 1);
        if (lim < g_issue) return;
        if (lane == 0)
#pragma unroll 1
            for (int g = g_issue; g <= lim; ++g) {  // (in the loop: one group per four steps)
                const int b = g % NG;
                const int dk = dir > 0 ? g * RW_G : -g * RW_G;
                mbar_arrive_expect_tx(&bars[b], 2 * L::IN_GROUP);
                tma_load_3d(smem + L::OFF_IN + b * L::IN_GROUP, &in_map, col0, rowl, kb0 + dk, &bars[b]);
                tma_load_3d(smem + L::OFF_IN + L::IN_HALF + b * L::IN_GROUP, &in_map, col0 + 32, rowl, kb1 + dk, &bars[b]);
            }
        g_issue = lim + 1;
    };
    const uint32_t s_bar = sbase + L::OFF_BAR;
    auto wait_for = [&](int v) {  // every group up to visit v's has landed (v warp-uniform, >= 0)
        const int gn = (int)((unsigned)v / RW_G);
        if (gn < g_wait) return;
#pragma unroll 1
        for (; g_wait <= gn; ++g_wait)
            while (!mbar_try(s_bar + (uint32_t)(g_wait % NG) * 8u, (uint32_t)(g_wait / NG) & 1u)) {
            }
        __syncwarp();
    };
    issue_upto(NG - 1);  // nothing consumed yet: visits below every pair's start are never read
    wait_for(__reduce_max_sync(0xffffffffu, min(vs + 1, ve)));

    // loop invariants, kept in registers
    const uint32_t s_copy = opaque(sbase + L::OFF_OUT + (uint32_t)lane * 16u);  // lane's 16 bytes of a plane
    // the lane's two columns of its half's ring (one 32-bit word per row for u16)
    const uint32_t in_lane =
        opaque(sbase + L::OFF_IN + (uint32_t)(hh * L::IN_HALF) + (uint32_t)(2 * (lane & 15)) * (uint32_t)sizeof(T));
    const uint32_t tau_l = opaque(sbase + L::OFF_TAU + 4u * (uint32_t)vmin_h);
    // (DAXM_ROW_TAU_LINEAR) wire travel of a visit: row_tau, the fit check bounds its depth error
    const float tAf = (float)(a.t[dir > 0 ? ti.k_lo : ti.k_hi] - ti.t_ref);
    const float tdh = dir > 0 ? a.dth : -a.dth, tdl = dir > 0 ? a.dtl : -a.dtl;
    const uint32_t ob = sbase + L::OFF_OUT + (uint32_t)(32 * hh + 2 * (lane & 15)) * 4u;  // column 2i of a plane
    const uint32_t ob0 = opaque(ob + 4u * (uint32_t)hh), ob1 = opaque(ob + 4u * (uint32_t)(hh ^ 1));  // pair 0 / 1
    // pair p's column is the (p ^ h)-th half-word of the lane's 32-bit input word
    const uint32_t sel0 = opaque(hh ? 0x5432u : 0x5410u), sel1 = opaque(hh ? 0x5410u : 0x5432u);
    const float2 sdir2 = f2(opaque(2.f * a.sign * (float)dir));
    const float2 dfl2 = f2(opaque(a.dI_floor));  // c = 2 s dir dI / (sum_{q+1} - sum_q)
    const float EM = opaque((float)(a.M - a.m_ref));
    const int m_ref = a.m_ref;
    // bits(E + fbias) = 0x4B000000 + e - 1 + RB for edge index e = E + m_ref: its plane's slot in the low bits
    const float fbias = opaque(8388608.f + (float)(m_ref - 1 + RB));
    const int xr_ = opaque(xr);
    const int ve_ = opaque(ve), vs_ = opaque(vs);
    const int need_hi = vs_max, need_end = vend;

    // wire travel and the two pairs' intensities (rows 0, 1) at visit v of the lane's half
    auto fetch = [&](int v, float& t, float2 I[2]) {
        if (DAXM_ROW_TAU_LINEAR)
            t = row_tau(tAf, tdh, tdl, vmin_h + v);
        else
            t = lds_f32(tau_l + 4u * (uint32_t)v);
        const uint32_t ad = in_lane + ((uint32_t)(v ^ xr_) % (uint32_t)NB) * (uint32_t)L::IN_SLOT;
        if constexpr (sizeof(T) == 2) {
            // u16 -> fp32 exactly: 0x4B00'xxxx is 2^23 + x, one PRMT builds it from the lane's
            // half-word (the pair's column), one packed FADD removes 2^23
            const uint32_t w0 = lds_u32(ad), w1 = lds_u32(ad + 64u);
            I[0] = add2(make_float2(__uint_as_float(__byte_perm(w0, 0x4B00u, sel0)),
                                    __uint_as_float(__byte_perm(w1, 0x4B00u, sel0))), f2(-8388608.f));
            I[1] = add2(make_float2(__uint_as_float(__byte_perm(w0, 0x4B00u, sel1)),
                                    __uint_as_float(__byte_perm(w1, 0x4B00u, sel1))), f2(-8388608.f));
        } else {
            const float2 a0 = lds_f2(ad), a1 = lds_f2(ad + 128u);
            I[0] = hh ? make_float2(a0.y, a1.y) : make_float2(a0.x, a1.x);
            I[1] = hh ? make_float2(a0.x, a1.x) : make_float2(a0.y, a1.y);
        }
    };

    RowState A, B;
    {
        float t0;
        float2 I0[2];
        fetch(vs_, t0, I0);
#pragma unroll
        for (int p = 0; p < 2; ++p) {
            A.pI[p] = I0[p];
            A.plo[p] = poly2(cb[p], f2(t0));
            A.phi[p] = POINT ? A.plo[p] : poly2(cf[p], f2(t0));
            A.ps[p] = add2(A.plo[p], A.phi[p]);
            A.cq[p] = A.zF[p] = f2(0.f);
            if constexpr (GEN) {  // no earlier pairs: zero coefficients, zero-width ramps
                A.cq2[p] = A.if2[p] = f2(0.f);
                A.phm[p] = A.pM[p] = A.plo[p];
            }
            A.En[p].x = wk[p][0].npts > 0 ? fmaxf(E0, floorf(A.plo[p].x) + 1.f) : EM + 1.f;
            A.En[p].y = wk[p][1].npts > 0 ? fmaxf(E0, floorf(A.plo[p].y) + 1.f) : EM + 1.f;
        }
        fetch(min(vs_ + 1, ve_), A.tq, A.Iq);
    }
    auto frontier = [&](const RowState& S) {  // slowest walk's next edge index (no window: EM + 1)
        return warp_min((int)fminf(fminf(S.En[0].x, S.En[0].y), fminf(S.En[1].x, S.En[1].y)) + m_ref);
    };
    // Output (F staging).  Slot (e - 1) mod RB of the staged ring holds F(E_e), the intensity a walk
    // deposits below bin edge e (edge e is the top of plane e - 1); plane P = F(E_{P+1}) - F(E_P).
    // Once the slowest walk has passed edge P + 1, every lane copies its 16 bytes of plane P out of
    // the ring: it reads F(E_{P+1}) and F(E_P) (both still staged) and writes their difference with
    // one st.global.cs.v4 (the warp writes the plane's two 256-byte rows: the
    // store geometry that reaches the copy ceiling, profiles/r02b_membench.md).  No slot is ever
    // zeroed: each walk writes each edge from its first one on exactly once, so the next lap simply
    // overwrites its position (positions a walk never writes keep their initial 0 = F below its
    // window).  The exception is an edge written through an overflow slot (RB + s): overflow slots
    // hold the sentinel SENT until a walk writes them; the copy takes the overflow value where one
    // was written, else the direct slot's, writes it back to the direct slot and re-arms SENT.  A
    // slot may be rewritten once the plane that reads it as its lower edge has been copied (the
    // replay's ring-need rule).
    const bool lane_out = rowl + (lane >> 4) >= 0 && row0 + (lane >> 4) < a.row_end && col0 + 4 * (lane & 15) < a.C;
    const size_t gplane = (size_t)(a.row_end - a.row_begin) * a.C;
    // the lane's 16 bytes of plane `copied` (advanced by one plane per copy)
    float* gnext = a.out + (ptrdiff_t)(rowl + (lane >> 4)) * a.C + col0 + 4 * (lane & 15);
    const bool plain = !a.acc && !a.prof_part;  // store only (the both-edges add and the fused profile: else)
    int copied = 0;  // planes [0, copied) written out
    auto copy_upto = [&](int final_planes) {  // planes [0, final_planes) hold their final values
        const int nf = min(final_planes, a.M);
        if (nf <= copied) return;
        __syncwarp();  // every lane's edge stores before the reads
        int P = copied;
        float* g = gnext;
        if (plain) {
            // plane P = F(E_{P+1}) (slot P mod RB) - F(E_P) (slot (P - 1) mod RB; E_0: slot RB - 1); the
            // upper edge of one plane is the lower edge of the next (two planes per trip, no copies)
            auto edge = [&](int Q) {  // F(E_{Q+1}) with the overflow fold
                const uint32_t ad = s_copy + ((uint32_t)Q & (RB - 1)) * PLANE_B;
                const uint4 x = lds128u(ad);
                return ((uint32_t)Q & (RB - 1)) < (uint32_t)(KT - 1) ? fold_slot<RB>(ad, x) : x;
            };
            auto put = [&](uint4 hi, uint4 lo) {
                stg_cs_v4_if(g, sub2(make_float2(__uint_as_float(hi.x), __uint_as_float(hi.y)),
                                     make_float2(__uint_as_float(lo.x), __uint_as_float(lo.y))),
                             sub2(make_float2(__uint_as_float(hi.z), __uint_as_float(hi.w)),
                                  make_float2(__uint_as_float(lo.z), __uint_as_float(lo.w))),
                             lane_out);
                g += gplane;
            };
            uint4 lo = lds128u(s_copy + ((uint32_t)(P - 1) & (RB - 1)) * PLANE_B);
#pragma unroll 1
            for (;;) {
                const uint4 hi = edge(P);
                put(hi, lo);
                if (++P == nf) break;
                lo = edge(P);
                put(lo, hi);
                if (++P == nf) break;
            }
        } else {
#pragma unroll 1
            do {
                const uint32_t ad = s_copy + ((uint32_t)P & (RB - 1)) * PLANE_B;
                uint4 x = lds128u(ad);
                if (((uint32_t)P & (RB - 1)) < (uint32_t)(KT - 1)) x = fold_slot<RB>(ad, x);
                const uint4 y = lds128u(s_copy + ((uint32_t)(P - 1) & (RB - 1)) * PLANE_B);
                const float4 v = make_float4(__uint_as_float(x.x) - __uint_as_float(y.x),
                                             __uint_as_float(x.y) - __uint_as_float(y.y),
                                             __uint_as_float(x.z) - __uint_as_float(y.z),
                                             __uint_as_float(x.w) - __uint_as_float(y.w));
                if (lane_out) {
                    if (a.acc)
                        red_add_v4(g, v);  // both-edges mode: the second edge adds
                    else
                        stg_cs_v4(g, v);
                }
                if (a.prof_part) {  // fused depth-profile epilogue: the tile's sum of the plane
                    float t = lane_out ? (v.x + v.y) + (v.z + v.w) : 0.f;
#pragma unroll
                    for (int o = 16; o > 0; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
                    if (lane == 0) a.prof_part[(size_t)rt * a.M + P] = t;
                }
                g += gplane;
            } while (++P < nf);
        }
        gnext = g;
        copied = nf;
        __syncwarp();  // every lane's reads before the next edge stores reuse the slots
    };
#if DAXM_ROW_CHECK
    unsigned viol = 0u;
#endif
    int fr_e = 0;

    // One iteration: every pair advances one point: point v + 1 closes the zone [lo_v, lo_{v+1}) of
    // each of its walks, whose bin edges are then evaluated.  A pair past its last visit re-reads it
    // (its points lie above EM: no edge, whatever the arithmetic yields).  S -> D, no register copies.
    // Lock step: at iteration it pair p of lane l sits at visit vs + it of its half and reads visit
    // vs + it + 2 (clamped to its last).  Every pair has read the visits below it + 2 of its half (the
    // smallest start is 0), and no pair reads beyond min(max vs + it + 2, last visit): warp-uniform
    // bounds the replay checks with the same formulas (deadlock-free iff the latter's group is loadable).
    int it2 = 2;  // it + 2 of the transition about to run (it reads visit vs + it2)
    // the next it2 at which group g_issue becomes loadable / group g_wait is needed (warp-uniform)
    int next_issue = g_issue >= ngroups ? INT_MAX : RW_G * g_issue + RW_G - NB;
    int next_wait = g_wait * RW_G > need_end ? INT_MAX : RW_G * g_wait - need_hi;
    // input rings: refill the slots every lane has read past (group g is loadable from it2 = 4 g + 4 -
    // NB on) and wait for what the next `ahead` + 1 transitions read (visit need_hi + it2 + ahead)
    auto input = [&](int ahead) {
        if (it2 >= next_issue) {
            issue_upto((int)((unsigned)(it2 + NB - RW_G) / RW_G));
            next_issue = g_issue >= ngroups ? INT_MAX : RW_G * g_issue + RW_G - NB;
        }
        if (it2 + ahead >= next_wait) {
            const int need = min(need_hi + it2 + ahead, need_end);
#if DAXM_ROW_CHECK
            if ((int)((unsigned)need / RW_G) >= g_issue) viol |= 1u;
#endif
            wait_for(need);
            next_wait = g_wait * RW_G > need_end ? INT_MAX : g_wait * RW_G - need_hi;
        }
    };
    // Zone [lo_v, lo_{v+1}) of a walk pair, everything its bin-edge stores need.  Inside the zone
    // F(E) = F0 + c x + xc (d + g xc), x = E - lo_v, xc = min(x, w); the admission replay checks
    // w < 2 bins, so from the zone's third edge on x > w and F(E) = h + c x, h = F0 + w d / 2: the
    // zone's edges En, En + 1, ... receive F(x0), F(x0 + 1) and then hc + k c, hc = h + c x0 (the
    // linear form at x0), k = 2, 3, ...
    struct Zone {
        float2 F0v, F1v, hc, c, cnt;
        float2 F2v, F3v;  // general-span variant: F at the zone's edges 2 and 3 (exact)
        uint32_t es[2];
    };
    // Transition S -> D: every pair advances one point; point v + 1 closes the zone [lo_v, lo_{v+1})
    // of each of its walks.  A pair past its last visit re-reads it (its points lie above EM: no
    // edge, whatever the arithmetic yields).
    auto trans = [&](const RowState& S, RowState& D, Zone Z[2]) {
        float2 In[2];
        fetch(min(vs_ + it2, ve_), D.tq, In);
        static_for<0, 2>([&](auto pc) {
            constexpr int p = decltype(pc)::value;
            const float2 lo = poly2(cb[p], f2(S.tq)), hi = POINT ? lo : poly2(cf[p], f2(S.tq));
            const float2 s = add2(lo, hi);
            // trapezoid height c = dI / area: twice the area is s - ps for separated spans and
            // (hi - lo_v) + |hi_v - lo| in general (the sorted corners' two parallel sides)
            const float2 dn = GEN ? add2(sub2(hi, S.plo[p]), abs2(sub2(S.phi[p], lo))) : sub2(s, S.ps[p]);
            // (both-edges mode: the clamp keeps this edge's sign of change, reading R16; -inf otherwise)
            const float2 sdI = mul2(sdir2, sub2(S.pI[p], S.Iq[p]));
            const float2 c = mul2(CLAMP ? max2(sdI, dfl2) : sdI, rcp2(dn));
            // edges of the zone [plo, lo): En .. floor(min(lo, EM))
            const float2 fl = add2(floor2(min2(lo, f2(EM))), f2(1.f));
            const float2 cnt = sub2(fl, add2(S.En[p], gate[p]));
            const float2 x0 = sub2(S.En[p], S.plo[p]);
            if constexpr (GEN) {
                // General spans ("general-span variant").  Pair q's trapezoid rises over
                // [lo_q, m_q], m_q = min(hi_q, lo_{q+1}), and falls over [M_q, hi_{q+1}], M_q = max(hi_q,
                // lo_{q+1}) (the sorted corners of P:L320-331).  In zone v = [lo_v, lo_{v+1}) only pairs v,
                // v-1 and v-2 are incomplete (replay), so with x = E - lo_v and the zone's linear form
                // h + c_v x (valid past every knot, x >= RW_NQ_GEN by the replay),
                //   F = h + c_v x + c_v (r - xc)^2 / 2r - c_{v-1} [(f1 - y1c)^2 / 2f1 - min(y1, 0)]
                //       - c_{v-2} (f2 - y2c)^2 / 2f2,
                // r = m_v - lo_v, xc = min(x, r); y1 = x - a1, a1 = M_{v-1} - lo_v, f1 = hi_v - M_{v-1},
                // y1c = clamp(y1, 0, f1); y2c = min(x + d2, f2), d2 = lo_v - M_{v-2}, f2 = hi_{v-1} - M_{v-2}.
                const float2 st = sub2(lo, S.plo[p]);
                const float2 r = min2(sub2(S.phi[p], S.plo[p]), st);
                const float2 ir = rcp2(r);
                const float2 M1 = max2(S.phm[p], S.plo[p]);
                const float2 a1 = sub2(M1, S.plo[p]);
                const float2 f1 = sub2(S.phi[p], M1);
                const float2 if1 = rcp2(f1);
                const float2 d2 = sub2(S.plo[p], S.pM[p]);
                const float2 f2v = sub2(S.phm[p], S.pM[p]);
                const float2 c1 = S.cq[p], c2 = S.cq2[p];
                const float2 ch = mul2(mul2(c, ir), f2(0.5f));
                const float2 nc1h = mul2(mul2(c1, if1), f2(-0.5f));
                const float2 c2h = mul2(mul2(c2, S.if2[p]), f2(0.5f));
                const float2 nc2h = mul2(c2h, f2(-1.f));
                const float2 t20 = sub2(f2v, min2(d2, f2v));
                // h = zF - c r / 2 + c1 (a1 + f1 / 2) + c2 (f2 - min(d2, f2))^2 / 2f2  (F = zF at x = 0)
                float2 h = fma2(c, mul2(r, f2(-0.5f)), S.zF[p]);
                h = fma2(c1, fma2(f1, f2(0.5f), a1), h);
                h = fma2(mul2(c2h, t20), t20, h);
                auto Fx = [&](float2 x) {
                    const float2 t = sub2(r, min2(x, r));
                    float2 e = fma2(c, x, h);
                    e = fma2(mul2(ch, t), t, e);
                    const float2 y1 = sub2(x, a1);
                    const float2 t1 = sub2(f1, min2(max2(y1, f2(0.f)), f1));
                    e = fma2(mul2(nc1h, t1), t1, e);
                    e = fma2(c1, min2(y1, f2(0.f)), e);
                    const float2 t2 = sub2(f2v, min2(add2(x, d2), f2v));
                    return fma2(mul2(nc2h, t2), t2, e);
                };
                const float2 F0v = Fx(x0), F1v = Fx(add2(x0, f2(1.f))), F2v = Fx(add2(x0, f2(2.f)));
                const float2 F3v = Fx(add2(x0, f2(3.f)));
                Z[p].F0v = F0v;
                Z[p].F1v = F1v;
                Z[p].F2v = F2v;
                Z[p].F3v = F3v;
                Z[p].hc = fma2(c, x0, h);
                Z[p].c = c;
                D.zF[p] = Fx(st);  // F at the next zone's start
                D.cq2[p] = c1;
                D.phm[p] = S.phi[p];
                D.pM[p] = M1;
                D.if2[p] = if1;
            } else {
            const float2 w = sub2(S.phi[p], S.plo[p]);
            const float2 d = sub2(S.cq[p], c);
            const float2 h = POINT ? S.zF[p] : fma2(f2(0.5f), mul2(w, d), S.zF[p]);
            const float2 x1 = add2(x0, f2(1.f));
            float2 F0v, F1v;
            if (POINT) {
                F0v = fma2(c, x0, S.zF[p]);
                F1v = fma2(c, x1, S.zF[p]);
            } else {
                const float2 g = mul2(d, mul2(rcp2(w), f2(-0.5f)));
                const float2 xc0 = min2(x0, w), xc1 = min2(x1, w);
                F0v = fma2(xc0, fma2(g, xc0, d), fma2(c, x0, S.zF[p]));
                F1v = fma2(xc1, fma2(g, xc1, d), fma2(c, x1, S.zF[p]));
            }
            Z[p].F0v = F0v;
            Z[p].F1v = F1v;
            Z[p].hc = fma2(c, x0, h);
            Z[p].c = c;
            D.zF[p] = fma2(c, sub2(lo, S.plo[p]), h);  // F at the next zone's start
            }
            Z[p].cnt = cnt;
            Z[p].es[0] = lea9((uint32_t)__float_as_int(S.En[p].x + fbias) & (uint32_t)(RB - 1), p ? ob1 : ob0);
            Z[p].es[1] = lea9((uint32_t)__float_as_int(S.En[p].y + fbias) & (uint32_t)(RB - 1), p ? ob1 : ob0);
            D.En[p] = max2(S.En[p], fl);
            D.plo[p] = lo;
            D.phi[p] = hi;
            D.ps[p] = s;
            D.pI[p] = S.Iq[p];
            D.cq[p] = c;
            D.Iq[p] = In[p];
            return true;
        });
        ++it2;
    };
    // The bin-edge stores of a zone: F at edge k of walk (p, r) goes to slot En + k - 1, staged slot
    // es + k planes (immediate offsets; row r, column half p), iff k < cnt.  Branch-free: RW_ST
    // predicated stores per walk, a rare extra trip when some zone holds more edges.
    // unrolled trips: every one of KT for the 3- and 4-edge classes; 4 + a rare 5th (warp vote) for the
    // 5-edge class (measured: all five unconditional cost C5 4 %); general spans 5 + a rare 6th
    constexpr int RW_ST = GEN ? 5 : (KT < 4 ? KT : 4);
    auto edges = [&](const Zone Z[2]) {
        static_for<0, 2>([&](auto pc) {
            constexpr int p = decltype(pc)::value;
            constexpr int O0 = 0, O1 = RW_COLS * 4;  // rows 0 / 1 (the column is in es)
            static_for<0, RW_ST>([&](auto kc) {
                constexpr int k = decltype(kc)::value;
                const float2 v = k == 0 ? Z[p].F0v : k == 1 ? Z[p].F1v : (GEN && k == 2) ? Z[p].F2v
                               : (GEN && k == 3) ? Z[p].F3v : fma2(Z[p].c, f2((float)k), Z[p].hc);
                st_if<O0 + k * PLANE_B>(Z[p].es[0], v.x, (float)k, Z[p].cnt.x);
                st_if<O1 + k * PLANE_B>(Z[p].es[1], v.y, (float)k, Z[p].cnt.y);
                return true;
            });
            return true;
        });
#if DAXM_ROW_CHECK
        if constexpr (RW_ST == KT) {
            const float cm = fmaxf(fmaxf(Z[0].cnt.x, Z[0].cnt.y), fmaxf(Z[1].cnt.x, Z[1].cnt.y));
            if (cm > (float)KT) viol |= 2u;
        }
#endif
        if constexpr (RW_ST < KT) {
        const float cmax = fmaxf(fmaxf(Z[0].cnt.x, Z[0].cnt.y), fmaxf(Z[1].cnt.x, Z[1].cnt.y));
        if (__any_sync(0xffffffffu, cmax > (float)RW_ST)) {  // rare: zones with more edges
            static_for<0, 2>([&](auto pc) {
                constexpr int p = decltype(pc)::value;
                constexpr int O0 = 0, O1 = RW_COLS * 4;
                static_for<RW_ST, KT>([&](auto kc) {
                    constexpr int k = decltype(kc)::value;
                    const float2 v = fma2(Z[p].c, f2((float)k), Z[p].hc);
                    st_if<O0 + k * PLANE_B>(Z[p].es[0], v.x, (float)k, Z[p].cnt.x);
                    st_if<O1 + k * PLANE_B>(Z[p].es[1], v.y, (float)k, Z[p].cnt.y);
                    return true;
                });
                return true;
            });
#if DAXM_ROW_CHECK
            if (cmax > (float)KT) viol |= 2u;
#endif
        }
        }
    };
    // Software pipeline: the stores of step n's zones and step n + 1's transition are independent,
    // so they form one block; the input waits, slot releases and batch stores sit between steps.
    Zone Z0[2], Z1[2];
    RowState& Bs = B;
    input(0);
    trans(A, Bs, Z0);  // step 0's zones; state after point 1
    fr_e = frontier(Bs);
    // the replay's iteration count, rounded up to a multiple of four (an extra step after every pair
    // has finished changes nothing: no edges, nothing left to load).  The input rings are refilled and
    // waited for once per four steps (for all four transitions).
    const int nquad = (ti.niter + 3) >> 2;
#pragma unroll 1
    for (int it = 0; it < nquad; ++it) {
        input(RW_G - 1);
        trans(Bs, A, Z1);
        edges(Z0);
        copy_upto(fr_e - 1);  // edge e completes plane e - 1: planes below the slowest walk's next are final
        fr_e = frontier(A);
        trans(A, Bs, Z0);
        edges(Z1);
        copy_upto(fr_e - 1);
        fr_e = frontier(Bs);
        trans(Bs, A, Z1);
        edges(Z0);
        copy_upto(fr_e - 1);
        fr_e = frontier(A);
        trans(A, Bs, Z0);
        edges(Z1);
        copy_upto(fr_e - 1);
        fr_e = frontier(Bs);
    }
    copy_upto(a.M);
    if (lane == 0) {
        // every issued input load must have landed before the CTA exits
        for (; g_wait < g_issue; ++g_wait)
            while (!mbar_try(s_bar + (uint32_t)(g_wait % NG) * 8u, (uint32_t)(g_wait / NG) & 1u)) {
            }
    }
#if DAXM_ROW_CHECK
    viol = __reduce_or_sync(0xffffffffu, viol);
    if (viol && lane == 0 && a.err) atomicOr(a.err, viol);
#endif
}

#if DAXM_ROW_TU == 0
// ------------------------------------------------------------------ exact zero-dI skip
// One warp per row tile of [rt0, rt0 + n).  A tile whose intensities are the same at every step of
// its range [k_lo, k_hi] has every dI = 0, so every bin value the row kernel would store is exactly 0:
// the warp clears the tile's live flag and the row kernel's CTA writes the zeros (its zero path,
// TMA stores interleaved with the live tiles' deposits) without running the deposit.  The scan reads
// 16-byte chunks, lanes on distinct (step, row, chunk), 8 loads in flight per lane, and stops at the
// first round with a change, so a live tile costs one round.  Tiles at the detector's edges, with
// misaligned rows, or not admitted to the row kernel stay live (no scan).
template <typename T>
__global__ void __launch_bounds__(256) row_live_kernel(const RowArgs a, int rt0, int n, unsigned char* __restrict__ live) {
    const int w = blockIdx.x * 8 + (threadIdx.x >> 5), lane = threadIdx.x & 31;
    if (w >= n) return;
    const int rt = rt0 + w;
    const RowTile ti = a.rt[rt];
    const int rr = rt / a.n_rc, rc = rt % a.n_rc;
    const int row0 = a.row_org + rr * RW_ROWS, col0 = rc * RW_COLS;
    const bool can = (ti.cls & RW_CLS_RB) != 0 && ti.k_hi >= ti.k_lo && row0 >= a.row_begin &&
                     row0 + RW_ROWS <= a.row_end && col0 + RW_COLS <= a.C && (a.C * (int)sizeof(T)) % 16 == 0;
    if (!can) {
        if (lane == 0) live[rt] = 1;
        return;
    }
    constexpr int CPR = RW_COLS * (int)sizeof(T) / 16;  // 16-byte chunks per row segment
    constexpr int CPS = CPR * RW_ROWS;                  // ... per step (16 or 32)
    constexpr int SPL = 32 / CPS;                       // steps per load instruction
    constexpr int U = 8;                                // loads in flight per lane
    const int ch = lane % CPS, sub = lane / CPS;
    const int r = ch / CPR, cc = ch % CPR;
    const size_t plane = (size_t)(a.row_end - a.row_begin) * a.C * sizeof(T);
    const char* base = static_cast<const char*>(a.stack) +
                       ((size_t)(row0 + r - a.row_begin) * a.C + col0) * sizeof(T) + (size_t)cc * 16;
    auto ld = [&](int k) { return __ldg(reinterpret_cast<const uint4*>(base + (size_t)k * plane)); };
    const uint4 ref = ld(ti.k_lo);
    unsigned var = 0;
    for (int k0 = ti.k_lo + 1; k0 <= ti.k_hi; k0 += U * SPL) {
        uint4 x[U];
#pragma unroll
        for (int u = 0; u < U; ++u) x[u] = ld(min(k0 + u * SPL + sub, ti.k_hi));
#pragma unroll
        for (int u = 0; u < U; ++u) var |= (x[u].x ^ ref.x) | (x[u].y ^ ref.y) | (x[u].z ^ ref.z) | (x[u].w ^ ref.w);
        if (__any_sync(0xffffffffu, var != 0)) break;
    }
    const bool changed = __any_sync(0xffffffffu, var != 0);
    if (lane == 0) live[rt] = changed ? 1 : 0;
}

// ------------------------------------------------------------------ admission replay
// One warp per row tile replays the kernel's schedule (lanes, pauses, frontier, drains) with the
// kernel's own fp32 arithmetic for the geometry (the intensities do not enter the schedule) and
// admits the tile (cls != 0) only if
//   * the same pixel edge is the shallower one at every evaluated point (RW_CLS_FRONT_LO),
//   * consecutive points of every walk have distinct edge sums and (finite pixels) edge spans
//     >= 1e-6 bins, so the zone density and ramp slope are finite,
//   * every window's last point lies at or above the top edge EM (a finished walk has no edge left),
//   * no iteration closes more than RW_KT edges of one walk,
//   * the input ring never waits for a group it could not yet load (no deadlock), and
//   * the planes written at every iteration lie below (zeroed batches) * RW_PB + RB: the ring holds
//     them (RB = RW_RB_SMALL or RW_RB_LARGE, the smaller that suffices).
// Walks with a window take part whatever the cutoff (the kernel's schedule is geometric), so the
// plan-time answer holds for every cutoff.  ti.niter = the schedule's iteration count.
// d_stats: [0] RB small, [1] RB large, [2] not admitted, [3] max ring need.
__global__ void __launch_bounds__(32) row_admit_kernel(RowArgs a, RowTile* __restrict__ rts, int n_rt,
                                                       int* __restrict__ d_stats) {
    const int rt = blockIdx.x;
    const int lane = threadIdx.x;
    RowTile ti = rts[rt];
    const int rr = rt / a.n_rc, rc = rt % a.n_rc;
    const int row0 = a.row_org + rr * RW_ROWS, col0 = rc * RW_COLS;
    const bool empty = ti.k_hi < ti.k_lo;  // no pixel window: the kernel streams zeros
    const bool eligible = !empty && ti.sep != MODE_GENERAL && ti.k_hi - ti.k_lo + 1 <= MAX_FAST_NV;
    unsigned bad = (!eligible && !empty) ? RW_WHY_MODE : 0u;  // reasons both variants share (RW_WHY_*)
    // reasons only the separated / only the general-span variant has
    unsigned bad_sep = (!empty && ti.sep != MODE_SEPARATED) ? RW_WHY_MODE : 0u;
    unsigned bad_gen = a.point_mode ? RW_WHY_MODE : 0u;
    unsigned bad_in[3] = {0u, 0u, 0u};  // input ring of RW_NB / RW_NB_WIDE / RW_NB_MID slots
    bool back_lo = true, front_lo = true;
    int need = 0, iters = 0, kmax_tile = 0;
    if (eligible) {
        const int nvt = ti.k_hi - ti.k_lo + 1;
        const float E0 = (float)(-a.m_ref), EM = (float)(a.M - a.m_ref);
        float cb[2][2][3], cf[2][2][3], En[2][2], ps[2][2];
        // general-span variant: the walk's last point (lo_v, hi_v), hi_{v-1}, hi_{v-2}, zones done
        float plo[2][2], phi[2][2], phm[2][2], phmm[2][2];
        int ndone[2][2];
        RowWalk wk[2][2];
        for (int p = 0; p < 2; ++p)
            for (int r = 0; r < 2; ++r) {
                const int e = rw_col(lane, p);
                wk[p][r] = row_walk(a, ti, row0 + r, col0 + e);
                row_coef(a, rt, r, e, cb[p][r]);
                row_coef(a, rt, r, a.point_mode ? e : e + 1, cf[p][r]);
            }
        int vmin_h, vs, ve, vs_max, vend;
        row_starts(wk, lane, vmin_h, vs, ve, vs_max, vend);
        const float tAf = (float)(a.t[ti.dir > 0 ? ti.k_lo : ti.k_hi] - ti.t_ref);
        const float tdh = ti.dir > 0 ? a.dth : -a.dth, tdl = ti.dir > 0 ? a.dtl : -a.dtl;
        auto tau_of = [&](int v) {  // v relative to the half's vmin, exactly as the kernel
            const int vv = vmin_h + v;
            return DAXM_ROW_TAU_LINEAR ? row_tau(tAf, tdh, tdl, vv)
                                       : (float)(a.t[ti.dir > 0 ? ti.k_lo + vv : ti.k_hi - vv] - ti.t_ref);
        };
        auto point = [&](int p, int r, int v, float& lo, float& hi) {  // walks with a window only
            const float t = tau_of(v);
            const float x0 = lock_poly(cb[p][r][0], cb[p][r][1], cb[p][r][2], t);
            const float x1 = a.point_mode ? x0 : lock_poly(cf[p][r][0], cf[p][r][1], cf[p][r][2], t);
            back_lo &= x0 <= x1;
            front_lo &= x1 <= x0;
            lo = fminf(x0, x1);
            hi = fmaxf(x0, x1);
        };
        int v = vs;
        for (int p = 0; p < 2; ++p)
            for (int r = 0; r < 2; ++r) {
                En[p][r] = EM + 1.f;  // a walk without a window never has an edge
                ps[p][r] = 0.f;
                if (wk[p][r].npts == 0) continue;
                float lo, hi;  // the window's last point at or above the top edge
                point(p, r, wk[p][r].v0 + wk[p][r].npts - 1 - vmin_h, lo, hi);
                if (!(lo >= EM)) bad |= RW_WHY_TOP;
                point(p, r, vs, lo, hi);
                En[p][r] = fmaxf(E0, floorf(lo) + 1.f);
                ps[p][r] = lo + hi;
                plo[p][r] = lo;
                phi[p][r] = hi;
                phm[p][r] = phmm[p][r] = lo;
                ndone[p][r] = 0;
            }
        // input ring of RW_NB (index 0), RW_NB_WIDE (1) or RW_NB_MID (2) slots per half: the same
        // schedule, loads issued further ahead with a wider ring.  The RW_NB ring must also keep
        // every needed group in flight RW_NB_MARGIN visits early (latency hiding: a ring that is just
        // deadlock-free makes the fastest lanes wait for their loads); the others only deadlock-free
        const int ngroups = vend / RW_G + 1;
        constexpr int NBs[3] = {RW_NB - RW_NB_MARGIN, RW_NB_WIDE, RW_NB_MID};
        int g_issue[3] = {min(NBs[0] / RW_G, ngroups), min(RW_NB_WIDE / RW_G, ngroups), min(RW_NB_MID / RW_G, ngroups)};
        for (int b = 0; b < 3; ++b)
            if (__reduce_max_sync(0xffffffffu, min(vs + 1, ve)) / RW_G >= g_issue[b]) bad_in[b] = RW_WHY_INPUT;
        auto frontier = [&]() {
            return __reduce_min_sync(
                0xffffffffu, (int)fminf(fminf(En[0][0], En[0][1]), fminf(En[1][0], En[1][1])) + a.m_ref);
        };
        int fr_e = frontier();
        int copied = 0;  // planes the kernel has copied out (F staging: edge e in slot (e - 1) mod RB)
        for (;;) {
            if (!__any_sync(0xffffffffu, v < ve)) break;
            if (++iters > 4 * nvt + 64) {  // cannot happen (every pair advances every iteration)
                bad |= RW_WHY_ITER;
                break;
            }
            // the kernel's lock-step input bounds for its transition n = iters - 1 (it reads visit
            // vs + n + 2): transition 0 alone, then blocks of four checked at their first transition
            const int n = iters - 1;
            if (n == 0 || (n - 1) % RW_G == 0) {
                const int it2 = n + 2, ahead = n == 0 ? 0 : RW_G - 1;
                const int nd_ = min(vs_max + it2 + ahead, vend);
                for (int b = 0; b < 3; ++b) {
                    g_issue[b] = max(g_issue[b], min((it2 + NBs[b] - RW_G) / RW_G, ngroups - 1) + 1);
                    if (nd_ / RW_G >= g_issue[b]) bad_in[b] = RW_WHY_INPUT;  // would wait for a group not yet loadable
                }
            }
            int kmax = 0, pmax = INT_MIN;
            for (int p = 0; p < 2; ++p) {
                if (v < ve)
                    for (int r = 0; r < 2; ++r) {
                        if (wk[p][r].npts == 0) continue;
                        float lo, hi;
                        point(p, r, v + 1, lo, hi);
                        const float s = lo + hi;
                        if (!(s != ps[p][r])) bad |= RW_WHY_DENSITY;
                        if (!a.point_mode) {
                            // finite ramp slope; separated variant: a span below two bins (from a zone's
                            // third edge on F is linear)
                            if (!(hi - lo >= 1e-6f)) bad |= RW_WHY_DENSITY;
                            if (!(hi - lo < 2.f)) bad_sep |= RW_WHY_DENSITY;
                            // general-span variant, zone v = [lo_v, lo): nonzero rise width r = min(w_v,
                            // lo - lo_v) and fall width f1 = hi_v - max(hi_{v-1}, lo_v) (finite reciprocals);
                            // where the zone can touch the bins, pair v-3 complete (hi_{v-2} <= lo_v) and
                            // every knot within RW_NQ_GEN bins of lo_v (exact edges 0 .. RW_NQ_GEN - 1)
                            const float lv = plo[p][r], hv = phi[p][r];
                            const float rr_ = fminf(hv - lv, lo - lv);
                            const float f1 = hv - fmaxf(phm[p][r], lv);
                            if (!(rr_ >= 1e-6f) || !(f1 >= 1e-6f)) bad_gen |= RW_WHY_GEN;
                            if (lo >= E0 - 1.f && lv <= EM + 1.f) {
                                if (ndone[p][r] >= 2 && !(phmm[p][r] <= lv)) bad_gen |= RW_WHY_GEN;
                                const float kn = fmaxf(hv, ndone[p][r] >= 1 ? phm[p][r] : hv) - lv;
                                if (!(kn <= (float)RW_NQ_GEN)) bad_gen |= RW_WHY_GEN;
                            }
                            phmm[p][r] = phm[p][r];
                            phm[p][r] = hv;
                            plo[p][r] = lo;
                            phi[p][r] = hi;
                            ++ndone[p][r];
                        }
                        ps[p][r] = s;
                        const float fl = floorf(fminf(lo, EM)) + 1.f;
                        const float cnt = fl - En[p][r];
                        if (cnt > 0.f) {
                            kmax = max(kmax, (int)cnt);
                            pmax = max(pmax, (int)fl - 2 + a.m_ref);  // plane of the last edge stored
                        }
                        En[p][r] = fmaxf(En[p][r], fl);
                    }
            }
            ++v;
            kmax = __reduce_max_sync(0xffffffffu, kmax);
            kmax_tile = max(kmax_tile, kmax);
            pmax = __reduce_max_sync(0xffffffffu, pmax);
            if (kmax > RW_KT) bad_sep |= RW_WHY_KT;
            if (kmax > RW_KT_GEN) bad_gen |= RW_WHY_KT;
            // edge e = pmax + 1 goes to slot pmax mod RB, whose previous occupant, edge e - RB, is free
            // once plane e - RB (which reads it as its lower edge) has been copied: pmax + 2 - copied <= RB
            if (pmax != INT_MIN) need = max(need, pmax + 2 - copied);
            fr_e = frontier();
            copied = max(copied, min(fr_e - 1, a.M));  // copy_upto, exactly as the kernel
        }
        // a finished schedule leaves every walk with a window past the top edge
        for (int p = 0; p < 2; ++p)
            for (int r = 0; r < 2; ++r)
                if (wk[p][r].npts > 0 && !(En[p][r] >= EM + 1.f)) bad |= RW_WHY_TOP;
    }
    bad = __reduce_or_sync(0xffffffffu, bad);
    bad_sep = __reduce_or_sync(0xffffffffu, bad_sep);
    bad_gen = __reduce_or_sync(0xffffffffu, bad_gen);
    bad_in[0] = __reduce_or_sync(0xffffffffu, bad_in[0]);
    bad_in[1] = __reduce_or_sync(0xffffffffu, bad_in[1]);
    bad_in[2] = __reduce_or_sync(0xffffffffu, bad_in[2]);
    back_lo = __all_sync(0xffffffffu, back_lo);
    front_lo = __all_sync(0xffffffffu, front_lo);
    if (lane == 0) {
        int cls = 0;
        if (!(back_lo || front_lo)) bad |= RW_WHY_ORDER;
        if (need > RW_RB_LARGE) bad |= RW_WHY_RING;
        // first that applies: separated variant, separated with the 32-slot input ring (one warp
        // fewer per SM), general-span variant, general-span with the wide input ring
        const int variant = !bad && !bad_sep && !bad_in[0] ? 0 : !bad && !bad_sep && !bad_in[2] ? 3
                          : !bad && !bad_gen && !bad_in[0] ? 1 : !bad && !bad_gen && !bad_in[1] ? 2 : -1;
        if (variant >= 0) {
            cls = need <= RW_RB_SMALL ? RW_RB_SMALL : RW_RB_LARGE;
            // edge-trip class of the separated variants (POINT plans: 5 only)
            const int ktc = (variant == 1 || variant == 2 || a.point_mode) ? 2 : kmax_tile <= 3 ? 0 : kmax_tile == 4 ? 1 : 2;
            cls |= ktc << RW_CLS_KT_SHIFT;
            if (!back_lo) cls |= RW_CLS_FRONT_LO;
            if (variant == 1 || variant == 2) cls |= RW_CLS_GEN;
            if (variant == 2) cls |= RW_CLS_NB_WIDE;
            if (variant == 3) cls |= RW_CLS_NB_MID;
        } else {
            bad |= bad_sep | bad_gen | bad_in[0] | bad_in[1] | bad_in[2];
        }
        ti.cls = cls;
        ti.why = (int)bad;
        ti.niter = iters;
        ti.kmax = kmax_tile;
        rts[rt] = ti;
        atomicAdd(&d_stats[(cls & RW_CLS_RB) == RW_RB_SMALL ? 0 : (cls & RW_CLS_RB) == RW_RB_LARGE ? 1 : 2], 1);
        atomicMax(&d_stats[3], need);
    }
}

#endif  // DAXM_ROW_TU == 0

// kernel variants: 0 separated, 1 general-span, 2 general-span with the wide input ring, 3 separated
// with the 32-slot input ring; CLAMP: the
// both-edges children (each edge keeps its sign of change, reading R16)
// KTS: edges per zone of the separated variants (3, 4 or 5 = RW_KT_CLASS[ktc])
template <typename T, bool POINT, int RB, int V, bool CLAMP, int KTS>
struct RowVariant {
    static constexpr bool GEN = V == 1 || V == 2;
    static constexpr int NB = V == 2 ? RW_NB_WIDE : V == 3 ? RW_NB_MID : RW_NB;
    using Smem = RowSmem<T, RB, GEN ? RW_KT_GEN : KTS, NB>;
    static constexpr auto kernel = deposit_row<T, POINT, RB, GEN, NB, CLAMP, GEN ? RW_KT : KTS>;
};

template <typename T, bool POINT, int RB, int V, bool CLAMP, int KTS>
cudaError_t set_attr_cl() {
    using K = RowVariant<T, POINT, RB, V, CLAMP, KTS>;
    cudaError_t e = cudaFuncSetAttribute(K::kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)K::Smem::bytes(MAX_FAST_NV));
    if (e != cudaSuccess) return e;
    return cudaFuncSetAttribute(K::kernel, cudaFuncAttributePreferredSharedMemoryCarveout,
                                (int)cudaSharedmemCarveoutMaxShared);
}

template <typename T, bool POINT, int RB, int V, int KTS = RW_KT>
cudaError_t set_attr_one() {
    cudaError_t e = set_attr_cl<T, POINT, RB, V, false, KTS>();
    return e != cudaSuccess ? e : set_attr_cl<T, POINT, RB, V, true, KTS>();
}

template <typename T, bool POINT, int RB, int V, bool CLAMP, int KTS>
cudaError_t launch_cl(const RowArgs& a, const CUtensorMap* in_map, const CUtensorMap* out_map,
                      cudaStream_t st) {
    using K = RowVariant<T, POINT, RB, V, CLAMP, KTS>;
    static const size_t extra = getenv("DAXM_ROW_EXTRA_SMEM") ? (size_t)atol(getenv("DAXM_ROW_EXTRA_SMEM")) : 0;
    K::kernel<<<(unsigned)a.n_list, 32, K::Smem::bytes(a.max_nv) + extra, st>>>(*in_map, *out_map, a);
    return cudaGetLastError();
}

template <typename T, bool POINT, int RB, int V, int KTS = RW_KT>
cudaError_t launch_one(const RowArgs& a, const CUtensorMap* in_map, const CUtensorMap* out_map,
                       cudaStream_t st) {
    return a.dI_floor > -INFINITY ? launch_cl<T, POINT, RB, V, true, KTS>(a, in_map, out_map, st)
                                  : launch_cl<T, POINT, RB, V, false, KTS>(a, in_map, out_map, st);
}

template <typename T, int RB, int V>
cudaError_t launch_kt(const RowArgs& a, const CUtensorMap* in_map, const CUtensorMap* out_map,
                      int ktc, cudaStream_t st) {  // separated variants: edge-trip class
    switch (ktc) {
        case 0: return launch_one<T, false, RB, V, 3>(a, in_map, out_map, st);
        case 1: return launch_one<T, false, RB, V, 4>(a, in_map, out_map, st);
        default: return launch_one<T, false, RB, V, 5>(a, in_map, out_map, st);
    }
}

template <typename T, int RB>
cudaError_t launch_rb(const RowArgs& a, const CUtensorMap* in_map, const CUtensorMap* out_map,
                      int variant, int ktc, cudaStream_t st) {
    if (a.point_mode)
        return variant == 3 ? launch_one<T, true, RB, 3>(a, in_map, out_map, st)
                            : launch_one<T, true, RB, 0>(a, in_map, out_map, st);
    switch (variant) {
        case 0: return launch_kt<T, RB, 0>(a, in_map, out_map, ktc, st);
        case 1: return launch_one<T, false, RB, 1>(a, in_map, out_map, st);
        case 2: return launch_one<T, false, RB, 2>(a, in_map, out_map, st);
        default: return launch_kt<T, RB, 3>(a, in_map, out_map, ktc, st);
    }
}

template <typename T, int RB>
cudaError_t set_attr_rb() {
    cudaError_t e;
    if ((e = set_attr_one<T, true, RB, 0>()) != cudaSuccess) return e;
    if ((e = set_attr_one<T, false, RB, 0, 3>()) != cudaSuccess) return e;
    if ((e = set_attr_one<T, false, RB, 0, 4>()) != cudaSuccess) return e;
    if ((e = set_attr_one<T, false, RB, 0, 5>()) != cudaSuccess) return e;
    if ((e = set_attr_one<T, false, RB, 1>()) != cudaSuccess) return e;
    if ((e = set_attr_one<T, false, RB, 2>()) != cudaSuccess) return e;
    if ((e = set_attr_one<T, true, RB, 3>()) != cudaSuccess) return e;
    if ((e = set_attr_one<T, false, RB, 3, 3>()) != cudaSuccess) return e;
    if ((e = set_attr_one<T, false, RB, 3, 4>()) != cudaSuccess) return e;
    return set_attr_one<T, false, RB, 3, 5>();
}

}  // namespace

// Instances are spread over four translation units (deposit_row.cu and deposit_row_{1,2,3}.cu, which
// include this file with DAXM_ROW_TU = 1, 2, 3) so that they compile in parallel:
// TU 0 u16 / ring 16 (+ the replay, the zero-dI scan and the dispatch), 1 u16 / ring 32, 2 f32 / ring 16,
// 3 f32 / ring 32.
using RowT = std::conditional_t<(DAXM_ROW_TU >= 2), float, uint16_t>;
constexpr int ROW_RB = (DAXM_ROW_TU & 1) ? RW_RB_LARGE : RW_RB_SMALL;
template <>
cudaError_t row_part_attributes_t<DAXM_ROW_TU>() {
    return set_attr_rb<RowT, ROW_RB>();
}
template <>
cudaError_t row_part_launch_t<DAXM_ROW_TU>(const RowArgs& a, const CUtensorMap* in_map, const CUtensorMap* out_map,
                                          int variant, int ktc, cudaStream_t st) {
    return launch_rb<RowT, ROW_RB>(a, in_map, out_map, variant, ktc, st);
}

#if DAXM_ROW_TU == 0
// The dynamic shared memory limit is a per-device function attribute: set it on the current
// device for every instance (daxm_create calls this on the plan's device).
cudaError_t row_set_attributes() {
    cudaError_t e;
    if ((e = row_part_attributes_t<0>()) != cudaSuccess) return e;
    if ((e = row_part_attributes_t<1>()) != cudaSuccess) return e;
    if ((e = row_part_attributes_t<2>()) != cudaSuccess) return e;
    return row_part_attributes_t<3>();
}

cudaError_t launch_row(const RowArgs& a, const CUtensorMap* in_map, const CUtensorMap* out_map, int dtype, int rb,
                       int variant, int ktc, cudaStream_t st) {
    if (a.n_list <= 0) return cudaSuccess;
    const int tu = (dtype == DAXM_U16 ? 0 : 2) + (rb == RW_RB_SMALL ? 0 : 1);
    switch (tu) {
        case 0: return row_part_launch_t<0>(a, in_map, out_map, variant, ktc, st);
        case 1: return row_part_launch_t<1>(a, in_map, out_map, variant, ktc, st);
        case 2: return row_part_launch_t<2>(a, in_map, out_map, variant, ktc, st);
        default: return row_part_launch_t<3>(a, in_map, out_map, variant, ktc, st);
    }
}

cudaError_t launch_row_live(const RowArgs& a, int rt0, int n, unsigned char* live, int dtype, cudaStream_t st) {
    if (n <= 0) return cudaSuccess;
    const unsigned grid = (unsigned)((n + 7) / 8);
    if (dtype == DAXM_U16)
        row_live_kernel<uint16_t><<<grid, 256, 0, st>>>(a, rt0, n, live);
    else
        row_live_kernel<float><<<grid, 256, 0, st>>>(a, rt0, n, live);
    return cudaGetLastError();
}

cudaError_t launch_row_admit(const RowArgs& a, RowTile* rt, int n_rt, int* d_stats, cudaStream_t st) {
    if (n_rt <= 0) return cudaSuccess;
    row_admit_kernel<<<(unsigned)n_rt, 32, 0, st>>>(a, rt, n_rt, d_stats);
    return cudaGetLastError();
}

#endif  // DAXM_ROW_TU == 0

}  // namespace daxm
