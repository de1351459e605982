// deposit.cu -- gather-form deposit kernels.
//
// Every output (depth bin m, pixel p) is owned by exactly one thread; there
// are no atomics (the paper's setTwo scatters with an fp64 CAS atomicAdd,
// P:L267-270).
//
// Deposit algebra.  For one pixel, visit the step pairs in the order in which
// their trapezoids move deeper and let F(E) be the intensity deposited below
// depth E (bin units).  Bin m receives F(m+1) - F(m): the trapezoid area inside
// [lo_m, hi_m) summed over pairs (device_depth_resolve_pixel P:L320-330,
// device_get_trapezoid_height P:L331), so computing F at the M+1 bin edges
// gives every bin exactly once.
//
//  * deposit_fast: when, for every pair, the pixel's edge span at one wire
//    step ends before the span at the next step begins ("separated", checked
//    in fp64 by the pre-pass), the sum of the pairs' trapezoids
//    f(z) = sum_q dI_q trap_q(z) / A_q is the piecewise-LINEAR function through
//    (lo_q, c_{q-1}) and (hi_q, c_q), c_q = dI_q / A_q, A_q = mid_{q+1} - mid_q:
//    on [lo_q, hi_q] pair q-1's falling ramp and pair q's rising ramp overlap,
//    on [hi_q, lo_{q+1}] only pair q's plateau.  F is then a running sum of
//    trapezoid-rule areas and F(E) inside a zone is one quadratic: 2 FMAs per
//    pixel per bin edge.  A tile of 128 rows x 8 columns: warp lanes are
//    detector rows (the depth-insensitive axis: lanes cross the same knots at
//    the same edge), each thread owns 4 adjacent columns.  A producer warp
//    streams the tile's wire-step planes with TMA into an mbarrier ring; the
//    consumers stage 4 depth planes at a time in shared memory (32B swizzle,
//    conflict-free 16-byte stores) and one thread writes them with a TMA
//    bulk-tensor store.
//  * deposit_general: any geometry (overlapping spans, degenerate trapezoids,
//    widths that TMA cannot describe): F(E) = sum of closed pairs' dI + sum over
//    open pairs of dI_q H_q(E)/A_q with the trapezoid CDF H, one thread per
//    pixel, plain loads.
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "daxm_internal.cuh"
#include "ptx.cuh"

namespace daxm {
namespace {
using namespace ptx;

__device__ __forceinline__ float poly3(const float c[NCOEF], float tau) {
    float p = c[NCOEF - 1];
#pragma unroll
    for (int m = NCOEF - 2; m >= 0; --m) p = fmaf(p, tau, c[m]);
    return p;
}

constexpr int CPT = COLS_PER_THREAD;                          // pixel walks (columns) per thread
constexpr int WPG = TILE_C / CPT;                             // warps per 32-row group
constexpr int N_PAIRS = TILE_R / 32;                          // 32-row warp groups (32 rows x 8 cols each)
constexpr int PAIR_BUF_BYTES = MC * 32 * TILE_C * 4;          // MC planes of a group's 32 x TILE_C block
constexpr int FAST_THREADS = N_CONSUMER_WARPS * 32;

template <typename T, int NB>
struct FastSmem {
    static constexpr int IN_SLOT_BYTES = TILE_R * TILE_C * (int)sizeof(T);
    static constexpr int OFF_OUT = 0;                                   // [pair][2][MC][32][8] f32
    static constexpr int OFF_IN = OFF_OUT + N_PAIRS * OUT_BUFS * PAIR_BUF_BYTES;
    static constexpr int OFF_BAR = OFF_IN + NB * IN_SLOT_BYTES;         // full[NB], empty[NB]
    static constexpr int OFF_OBAR = OFF_BAR + 2 * NB * 8;     // [pair][pfull[OUT_BUFS], pfree[OUT_BUFS]]
    static constexpr int OFF_SYNC = OFF_OBAR + 2 * OUT_BUFS * N_PAIRS * 8;  // v_issue, lock, cnt[pair][OB]
    static constexpr int OFF_TAU = OFF_SYNC + 64;
    static size_t bytes(int max_nv) { return (size_t)OFF_TAU + sizeof(float) * (size_t)(max_nv + 4) + 1024; }
};

// ------------------------------------------------------------------ fast kernel
// Eight warps: warp w covers tile rows 32*(w/2) .. +31 (lanes) and columns
// 4*(w%2) .. +3 (one pixel walk per column, all in registers).
//
// Per pixel, zone q = [lo_q, lo_{q+1}) holds pair q-1's falling ramp and pair
// q's rising ramp on [lo_q, hi_q] and pair q's plateau after it, so with
// x = E - lo_q, xc = min(x, w_q), w_q = hi_q - lo_q:
//     F(E) = F(lo_q) + c_q x + xc (d_q + g_q xc),  d_q = c_{q-1} - c_q,
//     g_q = (c_q - c_{q-1}) / (2 w_q)
// (exact for the linear interpolant through (lo_q, c_{q-1}), (hi_q, c_q),
// (lo_{q+1}, c_q)), one transition per wire step, 5 flops per pixel per edge.
//
// Pipeline: thread 0 is also the producer -- it issues the TMA loads of
// wire-step planes whenever a ring slot has been released by all eight warps,
// polling at every chunk start and inside every wait it performs, so no warp
// ever waits on a load that cannot be issued.  The two warps of a pair (same 32
// rows) stage MC depth planes of their 32x8 block in shared memory and the
// pair's first warp writes them with one TMA store; pairs never wait on each
// other.  Each warp waits for its input once per chunk, up to the furthest
// wire step its own pixels load in that chunk (pre-pass, a.vneed).
#ifndef DAXM_MINB
#define DAXM_MINB 2
#endif
#ifndef DAXM_SHPROD
#define DAXM_SHPROD 1
#endif
#ifndef DAXM_LASTSTORE
#define DAXM_LASTSTORE 1
#endif

template <typename T, int NB, bool POINT, int MODE>
__global__ void __launch_bounds__(FAST_THREADS, DAXM_MINB)
    deposit_fast(const __grid_constant__ CUtensorMap in_map, const __grid_constant__ CUtensorMap out_map,
                 const DepositArgs a) {
    static_assert((NB & (NB - 1)) == 0, "ring size must be a power of two");
    using L = FastSmem<T, NB>;
    extern __shared__ unsigned char smem_raw[];
    const uint32_t sbase = (smem_u32(smem_raw) + 1023u) & ~1023u;
    unsigned char* smem = smem_raw + (sbase - smem_u32(smem_raw));
    const int tile = a.tr_begin * a.n_tc + (int)blockIdx.x;
    const TileInfo ti = a.tiles[tile];
    const int tr = tile / a.n_tc, tc = tile % a.n_tc;
    const int row0 = (a.tr0 + tr) * TILE_R;  // global row of tile row 0
    // the general kernel owns this tile (same predicate as the plan's tile lists)
    if (!(ti.separated == MODE && row0 >= a.row_begin && ti.ring_need <= NB)) return;
    if (a.lock_enabled && ti.lock) return;  // the step-locked kernel owns this tile
    if (a.tile_live && !a.tile_live[tile]) return;  // cutoff: zero_dead_tiles writes this tile
    const int col0 = tc * TILE_C;
    const int row0_local = row0 - a.row_begin;
    const int nv_all = ti.k_hi >= ti.k_lo ? ti.k_hi - ti.k_lo + 1 : 0;
    int nv = nv_all;  // visits streamed: 0 when the intensity cutoff leaves no pixel of the tile
    const int dir = ti.dir;

    const uint32_t s_full = sbase + L::OFF_BAR, s_empty = s_full + NB * 8;
    const uint32_t s_obar = sbase + L::OFF_OBAR;
    const uint32_t s_tau = sbase + L::OFF_TAU, s_ring = sbase + L::OFF_IN;
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + L::OFF_BAR);
    uint64_t* empty = full + NB;
    uint64_t* obar = reinterpret_cast<uint64_t*>(smem + L::OFF_OBAR);  // [pair][pfull[OB], pfree[OB]]
    float* tau = reinterpret_cast<float*>(smem + L::OFF_TAU);

    const bool producer = threadIdx.x == 0;
    if (producer) {
        for (int s = 0; s < NB; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], N_CONSUMER_WARPS);
        }
        for (int pp = 0; pp < N_PAIRS; ++pp) {
            for (int bb = 0; bb < OUT_BUFS; ++bb) {
                mbar_init(&obar[pp * 2 * OUT_BUFS + bb], WPG);
                mbar_init(&obar[pp * 2 * OUT_BUFS + OUT_BUFS + bb], 1);
            }
        }
        fence_mbar_init();
    }
    int* sync_words = reinterpret_cast<int*>(smem + L::OFF_SYNC);  // [0] v_issue, [1] lock, [2..] cnt
    if (threadIdx.x < 16) sync_words[threadIdx.x] = 0;
    for (int v = threadIdx.x; v < nv_all; v += blockDim.x) {
        const int k = dir > 0 ? ti.k_lo + v : ti.k_hi - v;
        tau[v] = (float)(a.t[k] - ti.t_ref);
    }
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int pair = warp / WPG, h = warp % WPG;  // 32-row group, column group
    const int r = pair * 32 + lane;  // tile row
    const int j = row0 + r;          // global row
    // intensity cutoff (f1, reading R14): a walk runs only if its pixel's first-step
    // intensity reaches the cutoff; a tile with no such pixel streams no input at all
    unsigned act = (1u << CPT) - 1u;
    if (a.use_cutoff) {
        act = 0u;
        if (j < a.row_end) {
            const T* s0 = static_cast<const T*>(a.stack) + (size_t)(j - a.row_begin) * a.C + col0 + h * CPT;
#pragma unroll
            for (int w = 0; w < CPT; ++w)
                if (col0 + h * CPT + w < a.C && (float)s0[w] >= a.cutoff) act |= 1u << w;
        }
    }
    if (!__syncthreads_or(act != 0u)) nv = 0;
    // Producer: issue the TMA loads of every visit whose ring slot all warps have released.
#if DAXM_SHPROD
    // Shared producer state under a shared-memory lock: thread 0 polls at chunk starts and
    // lane 0 of ANY warp polls while it waits, so a starving warp fills the ring itself
    // instead of waiting for warp 0 to reach its next poll.
    volatile int* v_issue_sh = sync_words;
    auto issue_loads = [&]() {
        if (atomicCAS(&sync_words[1], 0, 1) != 0) return;  // another thread is issuing
        int v = *v_issue_sh;
        while (v < nv) {
            const int s = v & (NB - 1);
            if (v >= NB && !mbar_test(s_empty + s * 8, ((v / NB) - 1) & 1)) break;
            mbar_arrive_expect_tx(&full[s], L::IN_SLOT_BYTES);
            const int k = dir > 0 ? ti.k_lo + v : ti.k_hi - v;
            tma_load_3d(smem + L::OFF_IN + s * L::IN_SLOT_BYTES, &in_map, col0, row0_local, k, &full[s]);
            ++v;
        }
        *v_issue_sh = v;
        __threadfence_block();
        atomicExch(&sync_words[1], 0);
    };
    auto issued = [&]() { return *v_issue_sh; };
    auto wait_bar = [&](uint32_t bar, uint32_t parity) {
        while (!mbar_try(bar, parity))
            if (lane == 0) issue_loads();
    };
#else
    // producer state (thread 0 only): next visit index to load
    int v_issue = 0;
    auto issue_loads = [&]() {
        while (v_issue < nv) {
            const int s = v_issue & (NB - 1);
            if (v_issue >= NB && !mbar_test(s_empty + s * 8, ((v_issue / NB) - 1) & 1)) break;
            mbar_arrive_expect_tx(&full[s], L::IN_SLOT_BYTES);
            const int k = dir > 0 ? ti.k_lo + v_issue : ti.k_hi - v_issue;
            tma_load_3d(smem + L::OFF_IN + s * L::IN_SLOT_BYTES, &in_map, col0, row0_local, k, &full[s]);
            ++v_issue;
        }
    };
    auto issued = [&]() { return v_issue; };
    // wait on an mbarrier phase; in warp 0 the producer lane keeps issuing loads meanwhile
    // (warp-uniform split, so the other warps spin on a plain suspend-hinted try_wait)
    auto wait_bar = [&](uint32_t bar, uint32_t parity) {
        if (warp == 0) {
            while (!mbar_try(bar, parity))
                if (producer) issue_loads();
        } else {
            mbar_wait_u32(bar, parity);
        }
    };
#endif
    if (producer) issue_loads();

    const float sdir2 = 2.f * a.sign * (float)dir;  // c = 2 s dir dI / (sum_{q+1} - sum_q)
    const float INF = __int_as_float(0x7f800000);
    const uint32_t px_off = (uint32_t)(r * TILE_C + h * CPT) * (uint32_t)sizeof(T);
    const uint32_t s_pfull = s_obar + pair * 2 * OUT_BUFS * 8, s_pfree = s_pfull + OUT_BUFS * 8;

    float cb[CPT + 1][NCOEF];  // edge points h*CPT .. h*CPT+CPT of this row
#pragma unroll
    for (int e = 0; e <= CPT; ++e)
#pragma unroll
        for (int m = 0; m < NCOEF; ++m)
            cb[e][m] = a.coef[(((size_t)tile * NCOEF + m) * TILE_E + (h * CPT + e)) * TILE_R + r];

    // Zone state per walk (see above), the next point P1 = (nlo, nhi, nI) and the raw
    // inputs (tau, intensity) of the point after it, prefetched one transition ahead so
    // the shared-memory latency is off the transition's critical path.  Past the end of
    // the window the prefetch index is clamped and the point is replaced by +INF depths,
    // which makes c = 0 (rcp(inf) = 0) and stops further transitions: no branch.
    float zlo[CPT], zw[CPT], zF[CPT], zc[CPT], zd[CPT], zg[CPT], nlo[CPT], nhi[CPT], nI[CPT], Fp[CPT];
    float pt[CPT], pI[CPT];
    int vn[CPT], vlast[CPT];  // visit index of the prefetched point, last point of the window
#pragma unroll
    for (int w = 0; w < CPT; ++w) {
        zlo[w] = zw[w] = zF[w] = zc[w] = zd[w] = zg[w] = nI[w] = Fp[w] = pt[w] = pI[w] = 0.f;
        nlo[w] = nhi[w] = INF;
        vn[w] = 1;
        vlast[w] = 0;
    }
    // Input readiness is checked once per output chunk (warp-uniform): the
    // pre-pass recorded per tile, state and warp the furthest step loaded.
    int ready = -1;
    uint32_t ready_bar = s_full + (NB - 1) * 8, ready_par = 1;  // barrier / parity of visit `ready`
    constexpr int VN = N_CONSUMER_WARPS + 1;  // per state: 8 warps + the tile-wide max
    const int* vneed = a.vneed + (size_t)tile * (a.n_states + 1) * VN + warp;
    const int* vneed_tile = a.vneed + (size_t)tile * (a.n_states + 1) * VN + N_CONSUMER_WARPS;
    bool idle = false;  // all of this warp's walks finished: follow the tile-wide horizon
    auto wait_upto = [&](int vt) {
        vt = min(vt, nv - 1);
        while (ready < vt) {
            ++ready;
            ready_bar += 8;
            if (ready_bar == s_full + NB * 8) {
                ready_bar = s_full;
                ready_par ^= 1u;
            }
            wait_bar(ready_bar, ready_par);
        }
    };
    auto fetch_raw = [&](int w, int v) {
        pt[w] = lds_f32(s_tau + 4u * (uint32_t)v);
        pI[w] = lds_px<T>(s_ring + (uint32_t)(v & (NB - 1)) * (uint32_t)L::IN_SLOT_BYTES + px_off +
                          (uint32_t)(w * sizeof(T)));
    };
    auto depths = [&](int w, float t, float& lo, float& hi) {
        const float x0 = poly3(cb[w], t);
        const float x1 = POINT ? x0 : poly3(cb[w + 1], t);
        lo = fminf(x0, x1);
        hi = fmaxf(x0, x1);
    };
    auto evalF = [&](int w, float E) -> float {
        const float x = E - zlo[w];
        const float xc = fminf(x, zw[w]);
        return fmaf(xc, fmaf(zg[w], xc, zd[w]), fmaf(zc[w], x, zF[w]));
    };
    // one zone transition of walk w (E passed lo of the next point)
    auto transition = [&](int w) {
        // F(lo_{q+1}): x = lo_{q+1} - lo_q >= w_q in a separated zone, so
        // F = F0 + c x + w (d + g w) = F0 + c x + w d / 2
        zF[w] = fmaf(zc[w], nlo[w] - zlo[w], fmaf(0.5f * zw[w], zd[w], zF[w]));
        zlo[w] = nlo[w];
        zw[w] = nhi[w] - nlo[w];
        const float s_cur = nlo[w] + nhi[w], I_cur = nI[w];
        const bool more = vn[w] <= vlast[w];
        float lo, hi;
        depths(w, pt[w], lo, hi);
        nlo[w] = more ? lo : INF;
        nhi[w] = more ? hi : INF;
        nI[w] = pI[w];
        ++vn[w];
        fetch_raw(w, min(vn[w], vlast[w]));
        const float c = (sdir2 * (I_cur - nI[w])) * rcp_approx((nlo[w] + nhi[w]) - s_cur);
        zd[w] = zc[w] - c;
        zc[w] = c;
        // g = (c - c_prev) / (2 w); w == 0 (POINT pixels) -> huge g, but xc <= w keeps xc*g*xc ~ 0
        zg[w] = zd[w] * rcp_approx(-2.f * fmaxf(zw[w], 1e-30f));
    };
    auto advance = [&](int w, float E) {
        if (E > nlo[w]) {  // zones are longer than a bin in practice: one transition, rarely more
            transition(w);
            while (E > nlo[w]) transition(w);
        }
    };

    // ---- dual mode (MODE_OVERLAP tiles: any pixel whose spans overlap somewhere): for every
    // pair, trap_q = R_q - U_q with R_q a unit ramp over [lo_q, m_q], m_q = min(hi_q, lo_{q+1})
    // (= z1..z2) and U_q over [M_q, hi_{q+1}], M_q = max(hi_q, lo_{q+1}) (= z3..z4).  The R
    // ramps are disjoint and ordered, so are the U ramps: f = sum c_q R_q - sum c_q U_q is
    // walked by a "lo walk" (ramp / gap phases) and a "hi walk" sharing one quadratic
    // accumulator F = F0 + f0 x + (sL - sU) x^2 / 2 between consecutive events.
    float oz0[CPT], oF0[CPT], of0[CPT], osL[CPT], osU[CPT];
    float llo[CPT], lhi[CPT], lI[CPT], lev[CPT];         // lo walk: point A, next event
    float hlo[CPT], hhi[CPT], hI[CPT], hev[CPT], hsl[CPT];  // hi walk: point A, next event, pending slope
    int lvn[CPT], hvn[CPT];                              // next visit index to load
    bool lramp[CPT], hramp[CPT];                         // lo walk in a ramp / hi walk before a ramp
#pragma unroll
    for (int w = 0; w < CPT; ++w) {
        oz0[w] = oF0[w] = of0[w] = osL[w] = osU[w] = lI[w] = hI[w] = hsl[w] = 0.f;
        llo[w] = lhi[w] = hlo[w] = hhi[w] = lev[w] = hev[w] = INF;
        lvn[w] = hvn[w] = 1;
        lramp[w] = hramp[w] = false;
    }
    auto load_pt = [&](int w, int v, float& lo, float& hi, float& I) {
        depths(w, lds_f32(s_tau + 4u * (uint32_t)v), lo, hi);
        I = lds_px<T>(s_ring + (uint32_t)(v & (NB - 1)) * (uint32_t)L::IN_SLOT_BYTES + px_off +
                      (uint32_t)(w * sizeof(T)));
    };
    // load the point B after A = (alo, ahi, aI) (clamped; INF past the window) and return
    // c_AB / 2 * (...) pieces: c = s dir (I_A - I_B) / Area, Area = (hi_B + M - m - lo_A) / 2
    auto pair_load = [&](int w, float& alo, float& ahi, float& aI, int& vnx, float& m, float& M, float& hb,
                         float& c) -> bool {
        const bool more = vnx <= vlast[w];
        float blo, bhi, bI;
        load_pt(w, min(vnx, vlast[w]), blo, bhi, bI);
        ++vnx;
        m = fminf(ahi, blo);
        M = fmaxf(ahi, blo);
        hb = bhi;
        c = (sdir2 * (aI - bI)) * rcp_approx((bhi + M) - (m + alo));
        alo = more ? blo : INF;
        ahi = more ? bhi : INF;
        aI = bI;
        return more;
    };
    auto lo_event = [&](int w) {
        if (!lramp[w]) {  // ramp R_q starts at lo_A: it ends at m_q
            float m, M, hb, c;
            const float a_lo = llo[w];
            const bool more = pair_load(w, llo[w], lhi[w], lI[w], lvn[w], m, M, hb, c);
            osL[w] = more ? c * rcp_approx(m - a_lo) : 0.f;
            lev[w] = more ? m : INF;
            lramp[w] = more;
        } else {          // ramp ends: gap until the next ramp starts at lo_{q+1}
            osL[w] = 0.f;
            lev[w] = llo[w];
            lramp[w] = false;
        }
    };
    auto hi_event = [&](int w) {
        if (!hramp[w]) {  // U_{q-1} ended at hi_A: gap until M_q, then U_q rises to hi_{q+1}
            float m, M, hb, c;
            const bool more = pair_load(w, hlo[w], hhi[w], hI[w], hvn[w], m, M, hb, c);
            osU[w] = 0.f;
            hsl[w] = more ? c * rcp_approx(hb - M) : 0.f;
            hev[w] = more ? M : INF;
            hramp[w] = more;
        } else {          // U_q starts at M_q
            osU[w] = hsl[w];
            hev[w] = hhi[w];
            hramp[w] = false;
        }
    };
    auto advance_o = [&](int w, float E) {
        while (true) {
            const float k = fminf(lev[w], hev[w]);
            if (!(E > k)) break;
            const float Lz = k - oz0[w], sl = osL[w] - osU[w];
            oF0[w] = fmaf(Lz, fmaf(0.5f * sl, Lz, of0[w]), oF0[w]);
            of0[w] = fmaf(sl, Lz, of0[w]);
            oz0[w] = k;
            if (lev[w] <= hev[w])
                lo_event(w);
            else
                hi_event(w);
        }
    };
    auto evalF_o = [&](int w, float E) -> float {
        const float x = E - oz0[w];
        return fmaf(x, fmaf(0.5f * (osL[w] - osU[w]), x, of0[w]), oF0[w]);
    };

    wait_upto(vneed[0]);
    unsigned live = 0u;  // walks with a non-empty window (and above the cutoff)
    if constexpr (MODE == MODE_OVERLAP) {
#pragma unroll
        for (int w = 0; w < CPT; ++w) {
            const int i = col0 + h * CPT + w;
            int2 win = make_int2(0, 0);
            if (j < a.R && i < a.C) win = a.win[(size_t)(j - a.pre_row0) * a.C + i];
            if (win.y > win.x && ((act >> w) & 1u)) {
                const int v0 = dir > 0 ? win.x - ti.k_lo : ti.k_hi - win.y;
                vlast[w] = v0 + (win.y - win.x);
                load_pt(w, v0, llo[w], lhi[w], lI[w]);
                hlo[w] = llo[w];
                hhi[w] = lhi[w];
                hI[w] = lI[w];
                lvn[w] = hvn[w] = v0 + 1;
                live |= 1u << w;
                lev[w] = llo[w];  // first rising ramp starts at lo_0
                hev[w] = hhi[w];  // no falling ramp before hi_0
                oz0[w] = llo[w];  // F = 0 before the first event
            }
        }
    }
#pragma unroll
    for (int w = 0; w < CPT; ++w) {
        if constexpr (MODE != MODE_SEPARATED) break;
        const int i = col0 + h * CPT + w;
        int2 win = make_int2(0, 0);
        if (j < a.R && i < a.C) win = a.win[(size_t)(j - a.pre_row0) * a.C + i];
        if (win.y > win.x && ((act >> w) & 1u)) {
            const int v0 = dir > 0 ? win.x - ti.k_lo : ti.k_hi - win.y;
            vlast[w] = v0 + (win.y - win.x);
            fetch_raw(w, v0);
            depths(w, pt[w], nlo[w], nhi[w]);
            nI[w] = pI[w];
            vn[w] = v0 + 1;
            fetch_raw(w, v0 + 1);  // windows hold >= 2 points
            zlo[w] = nlo[w];       // virtual zone before point 0: F = 0
            live |= 1u << w;
        }
    }
    int vt_next = vneed[2 * VN], vt_next_tile = vneed_tile[2 * VN];  // prefetched bounds for chunk 0
    {
        wait_upto(vneed[VN]);
        const float E0 = (float)(0 - a.m_ref);
#pragma unroll
        for (int w = 0; w < CPT; ++w) {
            if constexpr (MODE == MODE_OVERLAP)
                advance_o(w, E0);
            else
                advance(w, E0);
        }
#pragma unroll
        for (int w = 0; w < CPT; ++w) Fp[w] = MODE == MODE_OVERLAP ? evalF_o(w, E0) : evalF(w, E0);
    }

    int released = 0;
    [[maybe_unused]] unsigned pending = 0u;  // output buffers this warp stored and has not handed back (LASTSTORE)
    const uint32_t out_base = sbase + L::OFF_OUT + pair * OUT_BUFS * PAIR_BUF_BYTES;
    // [q][32 rows][TILE_C cols] f32, 32- or 64-byte rows, SWIZZLE_32B / SWIZZLE_64B (16-byte
    // chunk index ^= bits 7.. of the offset); a plane (32 rows) is a whole number of swizzle
    // atoms, so the swizzled row offset is per-thread constant
    const uint32_t row_off = (uint32_t)(lane * (TILE_C * 4) + h * CPT * 4);
    const uint32_t sts_off = row_off ^ (((row_off >> 7) & (uint32_t)(TILE_C * 4 / 16 - 1)) << 4);
    const int n_chunks = (a.M + MC - 1) / MC;
    float E = (float)(1 - a.m_ref);
    // a warp none of whose pixels contributes (outside every window, or below the cutoff)
    // writes zeros into its slice of the staging buffers once and skips all per-plane work
    const bool wlive = __any_sync(0xffffffffu, live != 0u);
    if (!wlive) {
        for (int b = 0; b < OUT_BUFS; ++b)
#pragma unroll
            for (int q = 0; q < MC; ++q) {
                const uint32_t za = out_base + b * PAIR_BUF_BYTES + sts_off + q * (32 * TILE_C * 4);
                if constexpr (CPT == 4)
                    st_shared_v4(za, 0.f, 0.f, 0.f, 0.f);
                else if constexpr (CPT == 2)
                    asm volatile("st.shared.v2.f32 [%0], {%1, %1};" ::"r"(za), "f"(0.f) : "memory");
                else
                    asm volatile("st.shared.f32 [%0], %1;" ::"r"(za), "f"(0.f) : "memory");
            }
        fence_proxy_async_smem();
    }
    // A 32-row group none of whose warps has work streams its zero planes straight from the
    // (never rewritten) zero buffer -- no buffer hand-back, stores back to back -- and then
    // only keeps releasing ring slots for the other groups (final release loop below).
    int* group_live = sync_words + 2 + N_PAIRS * OUT_BUFS;  // [N_PAIRS], zeroed at start
    if (lane == 0 && wlive) atomicOr(&group_live[pair], 1);
    __syncthreads();
    const bool dead_group = group_live[pair] == 0;
    if (dead_group && h == 0 && lane == 0) {
        for (int ch = 0; ch < n_chunks; ++ch) {
            tma_store_3d(&out_map, col0, row0_local + pair * 32, ch * MC,
                         smem + L::OFF_OUT + (pair * OUT_BUFS) * PAIR_BUF_BYTES);
            bulk_commit();
        }
    }
    for (int ch = 0; ch < n_chunks && !dead_group; ++ch) {
        const int b = ch % OUT_BUFS;
        const int vt = idle ? vt_next_tile : vt_next;
        if (ch + 1 < n_chunks) {
            vt_next = vneed[(ch + 3) * VN];
            vt_next_tile = vneed_tile[(ch + 3) * VN];
        }
        if (ch >= OUT_BUFS) wait_bar(s_pfree + b * 8, ((ch / OUT_BUFS) - 1) & 1);  // store ch-OB left buffer b
        wait_upto(vt);
        if (producer) issue_loads();
        uint32_t sa = out_base + b * PAIR_BUF_BYTES + sts_off;
        // planes >= M (last chunk) are padding: their walks may read steps nobody waited for,
        // harmless -- the TMA store clips them and releases are capped at `ready` below
#pragma unroll 1
        for (int q = 0; q < MC && wlive; ++q, sa += 32 * TILE_C * 4) {
#pragma unroll
            for (int w = 0; w < CPT; ++w) {
                if constexpr (MODE == MODE_OVERLAP)
                    advance_o(w, E);
                else
                    advance(w, E);
            }
            float o[CPT];
#pragma unroll
            for (int w = 0; w < CPT; ++w) {
                const float F = MODE == MODE_OVERLAP ? evalF_o(w, E) : evalF(w, E);
                o[w] = F - Fp[w];
                Fp[w] = F;
            }
            if constexpr (CPT == 4)
                st_shared_v4(sa, o[0], o[1], o[2], o[3]);
            else if constexpr (CPT == 2)
                asm volatile("st.shared.v2.f32 [%0], {%1, %2};" ::"r"(sa), "f"(o[0]), "f"(o[1]) : "memory");
            else
                asm volatile("st.shared.f32 [%0], %1;" ::"r"(sa), "f"(o[0]) : "memory");
            E += 1.f;
        }
        fence_proxy_async_smem();
        // release wire-step slots no walk of this warp needs any more
        int my_min = INT_MAX;
#pragma unroll
        for (int w = 0; w < CPT; ++w)
            if constexpr (MODE == MODE_OVERLAP) {
                const int vmin = min(lvn[w], hvn[w]);
                if (vmin <= vlast[w]) my_min = min(my_min, vmin);
            } else {
                if (vn[w] <= vlast[w]) my_min = min(my_min, vn[w]);  // slot vn may still be in flight (LDS)
            }
        // never release a slot this warp has not waited for (a premature arrive would
        // complete the slot's previous phase for the producer)
        const int wmin = __reduce_min_sync(0xffffffffu, my_min);
        idle = wmin == INT_MAX;
        const int target = min(min(wmin, nv), ready + 1);
        __syncwarp();  // every lane's staging stores (and proxy fence) precede lane 0's signal
        if (lane == 0) {
            if (released < target) {
                uint32_t ea = s_empty + (uint32_t)(released & (NB - 1)) * 8;
                for (int v = released; v < target; ++v) {
                    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(ea) : "memory");
                    ea = (ea + 8 == s_empty + NB * 8) ? s_empty : ea + 8;
                }
            }
#if DAXM_LASTSTORE
            // The warp that completes chunk ch of its 32-row group last stores it, so no warp
            // waits for its partner here.  A buffer is handed back (pfree) by whoever stored it,
            // at that warp's next chunk end, once its bulk stores have been read out.
            if (pending) {
                bulk_wait_read<0>();
#pragma unroll
                for (int bb = 0; bb < OUT_BUFS; ++bb)
                    if (pending & (1u << bb)) mbar_arrive(&obar[pair * 2 * OUT_BUFS + OUT_BUFS + bb]);
                pending = 0u;
            }
            int old;
            asm volatile("atom.acq_rel.cta.shared::cta.add.u32 %0, [%1], 1;"
                         : "=r"(old)
                         : "r"(smem_u32(&sync_words[2 + pair * OUT_BUFS + b]))
                         : "memory");
            if (old % WPG == WPG - 1) {
                tma_store_3d(&out_map, col0, row0_local + pair * 32, ch * MC,
                             smem + L::OFF_OUT + (pair * OUT_BUFS + b) * PAIR_BUF_BYTES);
                bulk_commit();
                pending |= 1u << b;
            }
#else
            mbar_arrive(&obar[pair * 2 * OUT_BUFS + b]);  // pfull[b]
#endif
        }
        released = max(released, target);
#if !DAXM_LASTSTORE
        if (h == 0 && lane == 0) {  // the pair's storer
            bulk_wait_read<OUT_BUFS - 2>();  // store ch+1-OB has left its buffer ...
            if (ch + 1 >= OUT_BUFS)          // ... which chunk ch+1 reuses
                mbar_arrive(&obar[pair * 2 * OUT_BUFS + OUT_BUFS + (ch + 1) % OUT_BUFS]);
            wait_bar(s_pfull + b * 8, (ch / OUT_BUFS) & 1);  // partner has written chunk ch
            tma_store_3d(&out_map, col0, row0_local + pair * 32, ch * MC,
                         smem + L::OFF_OUT + (pair * OUT_BUFS + b) * PAIR_BUF_BYTES);
            bulk_commit();
        }
#endif
        __syncwarp();
    }
    // release the rest; an arrive for visit v must follow v's fill (else it would count toward
    // the slot's previous phase), so wait for each visit first
    for (int v = released; v < nv; ++v) {
        wait_upto(v);
        if (lane == 0) mbar_arrive(&empty[v & (NB - 1)]);
    }
#if DAXM_LASTSTORE
    if (lane == 0) bulk_wait<0>();  // stores this warp issued
#else
    if (h == 0 && lane == 0) bulk_wait<0>();
#endif
    if (producer) {
        while (issued() < nv) issue_loads();  // others may still need the tail
        // every issued load must land before the CTA may exit
        const int vi = issued();
        for (int v = vi > NB ? vi - NB : 0; v < vi; ++v) mbar_wait(&full[v & (NB - 1)], (v / NB) & 1);
    }
}

// ------------------------------------------------------------------ general kernel
__device__ __forceinline__ float trapezoid_fraction(float lo0, float hi0, float lo1, float hi1, float E) {
    const float z1 = fminf(lo0, lo1), z4 = fmaxf(hi0, hi1);
    const float ma = fmaxf(lo0, lo1), mb = fminf(hi0, hi1);
    const float z2 = fminf(ma, mb), z3 = fmaxf(ma, mb);
    const float w1 = z2 - z1, w2 = z3 - z2, w3 = z4 - z3;
    const float A = 0.5f * (w1 + w3) + w2;
    const float x1 = fminf(fmaxf(E - z1, 0.f), w1);
    const float x2 = fminf(fmaxf(E - z2, 0.f), w2);
    const float x3 = fminf(fmaxf(E - z3, 0.f), w3);
    float H = x2 + x3;
    if (w1 > 0.f) H += x1 * x1 / (2.f * w1);
    if (w3 > 0.f) H -= x3 * x3 / (2.f * w3);
    return H / A;
}

// One pixel (global row j, column i; position r, c in deposit tile `tile`), any geometry: bin edge
// by bin edge, F(E) = (dI of the pairs whose trapezoid lies below E) + sum over the open pairs of
// dI_q H_q(E) / A_q.  A pair with a NaN corner depth (the pixel edge inside the wire cylinder, or
// a tangent plane parallel to the beam) is skipped, as in the oracle (reading R8).
template <typename T>
__device__ void general_pixel(const DepositArgs& a, int tile, int r, int c, int j, int i, const T* __restrict__ stack,
                              float* __restrict__ out) {
    const TileInfo ti = a.tiles[tile];
    const int rows = a.row_end - a.row_begin;
    const size_t plane = (size_t)rows * a.C;
    const int jl = j - a.row_begin;
    const int2 w = a.win[(size_t)(j - a.pre_row0) * a.C + i];
    float cb[NCOEF], cf[NCOEF];
    const int eb = c, ef = a.point_mode ? c : c + 1;
#pragma unroll
    for (int m = 0; m < NCOEF; ++m) {
        cb[m] = a.coef[(((size_t)tile * NCOEF + m) * TILE_E + eb) * TILE_R + r];
        cf[m] = a.coef[(((size_t)tile * NCOEF + m) * TILE_E + ef) * TILE_R + r];
    }
    const bool act = !a.use_cutoff || (float)stack[(size_t)jl * a.C + i] >= a.cutoff;  // reading R14
    const int kb = w.x, ke = act ? w.y : w.x, n = ke - kb, dir = ti.dir;
    auto step_of = [&](int q) { return dir > 0 ? kb + q : ke - q; };
    // corner depths of point q (lo <= hi), false if either is NaN
    auto point = [&](int q, float& lo, float& hi) {
        float x0, x1;
        if (a.table) {  // exact per-step depths (general wire paths)
            const float* tb = a.table + a.toff[tile] + (size_t)(step_of(q) - ti.k_lo) * (TILE_E * TILE_R) + r;
            x0 = tb[eb * TILE_R];
            x1 = tb[ef * TILE_R];
        } else {
            const float tau = (float)(a.t[step_of(q)] - ti.t_ref);
            x0 = poly3(cb, tau);
            x1 = poly3(cf, tau);
        }
        lo = fminf(x0, x1);
        hi = fmaxf(x0, x1);
        return !(isnan(x0) || isnan(x1));
    };
    const T* px = stack + (size_t)jl * a.C + i;
    const float sgn = a.sign * (float)dir;
    auto Iw = [&](int k) -> float {  // the step's intensity, normalised by its weight (reading R17)
        const float v = (float)px[(size_t)k * plane];
        return a.w ? v * a.w[k] : v;
    };
    auto dI = [&](int q) -> float {
        return fmaxf(sgn * (Iw(step_of(q)) - Iw(step_of(q + 1))),
                     a.dI_floor);  // both-edges mode: this edge's sign of change only (R16)
    };
    int qc = 0, qo = 0;
    float P = 0.f, F_prev = 0.f;
    float* o = out + (size_t)jl * a.C + i;
    for (int e = 0; e <= a.M; ++e) {
        const float E = (float)(e - a.m_ref);
        while (qc < n) {  // close pairs whose trapezoid lies entirely below E (NaN pairs: at once, empty)
            float lo1, hi1, lo2, hi2;
            const bool ok = point(qc, lo1, hi1) & point(qc + 1, lo2, hi2);
            if (!ok) {
                ++qc;
            } else if (fmaxf(hi1, hi2) < E) {
                P += dI(qc);
                ++qc;
            } else {
                break;
            }
        }
        if (qo < qc) qo = qc;
        while (qo < n) {  // open pairs whose trapezoid starts below E
            float lo1, hi1, lo2, hi2;
            const bool ok = point(qo, lo1, hi1) & point(qo + 1, lo2, hi2);
            if (!ok || fminf(lo1, lo2) < E)
                ++qo;
            else
                break;
        }
        float F = P;
        for (int q = qc; q < qo; ++q) {
            float lo1, hi1, lo2, hi2;
            if (!(point(q, lo1, hi1) & point(q + 1, lo2, hi2))) continue;
            const float d = dI(q);
            if (d != 0.f) F += d * trapezoid_fraction(lo1, hi1, lo2, hi2, E);
        }
        if (e > 0) {
            float* q = o + (size_t)(e - 1) * plane;
            *q = a.acc ? *q + (F - F_prev) : F - F_prev;
        }
        F_prev = F;
    }
}

template <typename T>
__global__ void __launch_bounds__(256) deposit_general(DepositArgs a, const T* __restrict__ stack,
                                                       float* __restrict__ out) {
    const int tile = a.tile_list ? a.tile_list[blockIdx.x] : a.tr_begin * a.n_tc + (int)blockIdx.x;
    const int tr = tile / a.n_tc, tc = tile % a.n_tc;
    if (tr < a.tr_begin || tr >= a.tr_end) return;  // row-band launch: not this band
    if (a.tile_live && !a.tile_live[tile]) return;  // cutoff: zero_dead_tiles writes this tile
    for (int pix = threadIdx.x; pix < TILE_R * TILE_C; pix += blockDim.x) {
        const int r = pix / TILE_C, c = pix % TILE_C;
        const int j = (a.tr0 + tr) * TILE_R + r, i = tc * TILE_C + c;
        if (j < a.row_begin || j >= a.row_end || i >= a.C) continue;
        general_pixel<T>(a, tile, r, c, j, i, stack, out);
    }
}

// The general kernel over row tiles the row-segment kernel did not admit (one CTA per row tile,
// one thread per pixel); each pixel's depth polynomials come from its deposit tile.
template <typename T>
__global__ void __launch_bounds__(RW_ROWS * RW_COLS) deposit_general_rows(DepositArgs a, const int* __restrict__ list,
                                                                          int n_rc, int row_org,
                                                                          const T* __restrict__ stack,
                                                                          float* __restrict__ out) {
    const int rt = list[blockIdx.x];
    const int rr = rt / n_rc, rc = rt % n_rc;
    const int j = row_org + rr * RW_ROWS + (int)threadIdx.x / RW_COLS, i = rc * RW_COLS + (int)threadIdx.x % RW_COLS;
    if (j < a.row_begin || j >= a.row_end || i >= a.C) return;
    const int tile = (j / TILE_R - a.tr0) * a.n_tc + i / TILE_C;
    general_pixel<T>(a, tile, j % TILE_R, i % TILE_C, j, i, stack, out);
}

template <typename T, int NB, bool POINT, int MODE>
cudaError_t launch_fast(const CUtensorMap* in_map, const CUtensorMap* out_map, const DepositArgs& a, int n_tiles,
                        cudaStream_t st) {
    const size_t sm = FastSmem<T, NB>::bytes(a.max_nv);
    static std::atomic<unsigned long long> attr_done{0};  // per template instance and device
    cudaError_t ea = once_per_device(attr_done, []() {
        cudaError_t e = cudaFuncSetAttribute(deposit_fast<T, NB, POINT, MODE>,
                                             cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             (int)FastSmem<T, NB>::bytes(MAX_FAST_NV));
        if (e != cudaSuccess) return e;
        return cudaFuncSetAttribute(deposit_fast<T, NB, POINT, MODE>, cudaFuncAttributePreferredSharedMemoryCarveout,
                                    (int)cudaSharedmemCarveoutMaxShared);
    });
    if (ea != cudaSuccess) return ea;
    if (sm > FastSmem<T, NB>::bytes(MAX_FAST_NV)) return cudaErrorInvalidValue;
    deposit_fast<T, NB, POINT, MODE><<<n_tiles, FAST_THREADS, sm, st>>>(*in_map, *out_map, a);
    return cudaGetLastError();
}

template <typename T, int NB>
cudaError_t launch_fast_modes(const CUtensorMap* in_map, const CUtensorMap* out_map, const DepositArgs& a,
                              int n_tiles, cudaStream_t st) {
    cudaError_t e = a.point_mode ? launch_fast<T, NB, true, MODE_SEPARATED>(in_map, out_map, a, n_tiles, st)
                                 : launch_fast<T, NB, false, MODE_SEPARATED>(in_map, out_map, a, n_tiles, st);
    if (e != cudaSuccess || !a.has_overlap) return e;
    return a.point_mode ? launch_fast<T, NB, true, MODE_OVERLAP>(in_map, out_map, a, n_tiles, st)
                        : launch_fast<T, NB, false, MODE_OVERLAP>(in_map, out_map, a, n_tiles, st);
}

}  // namespace

size_t fast_smem_bytes(int dtype, int max_nv) {
    return dtype == DAXM_U16 ? FastSmem<uint16_t, NB_U16>::bytes(max_nv) : FastSmem<float, NB_F32>::bytes(max_nv);
}

cudaError_t launch_deposit(const DepositArgs& a, const CUtensorMap* in_map, const CUtensorMap* out_map,
                           const void* stack, int dtype, float* out, bool fast_enabled, cudaStream_t st,
                           const CUtensorMap* lock_in_map, const cudaStream_t* lock_sts, int n_lock_sts) {
    const int n_tiles = (a.tr_end - a.tr_begin) * a.n_tc;
    if (n_tiles <= 0) return cudaSuccess;
    cudaError_t e = cudaSuccess;
    if (fast_enabled) {
        if (a.lock_enabled) {
            e = launch_lock(a, lock_in_map, out, dtype, n_tiles, lock_sts, n_lock_sts);
            if (e != cudaSuccess) return e;
        }
        if (a.lock_rest > 0)
            e = dtype == DAXM_U16 ? launch_fast_modes<uint16_t, NB_U16>(in_map, out_map, a, n_tiles, st)
                                  : launch_fast_modes<float, NB_F32>(in_map, out_map, a, n_tiles, st);
        if (e != cudaSuccess) return e;
        if (a.n_list == 0) return cudaSuccess;
    }
    DepositArgs ga = a;
    if (!fast_enabled) {
        ga.tile_list = nullptr;
        ga.n_list = n_tiles;
    }
    if (dtype == DAXM_U16)
        deposit_general<uint16_t><<<ga.n_list, 256, 0, st>>>(ga, static_cast<const uint16_t*>(stack), out);
    else
        deposit_general<float><<<ga.n_list, 256, 0, st>>>(ga, static_cast<const float*>(stack), out);
    return cudaGetLastError();
}

cudaError_t launch_general_rows(const DepositArgs& a, const int* rt_list, int n, int n_rc, int row_org,
                                const void* stack, int dtype, float* out, cudaStream_t st) {
    if (n <= 0) return cudaSuccess;
    if (dtype == DAXM_U16)
        deposit_general_rows<uint16_t><<<n, RW_ROWS * RW_COLS, 0, st>>>(a, rt_list, n_rc, row_org,
                                                                        static_cast<const uint16_t*>(stack), out);
    else
        deposit_general_rows<float><<<n, RW_ROWS * RW_COLS, 0, st>>>(a, rt_list, n_rc, row_org,
                                                                     static_cast<const float*>(stack), out);
    return cudaGetLastError();
}

}  // namespace daxm
