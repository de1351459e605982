// plan.cu -- C ABI entry points, validation and the fp64 geometry pre-pass.
//
// Pre-pass (paper: device_pixel_xyz_to_depth,
// P:L306-319, called four times per thread in setTwo):
//   pixel_window_kernel  per pixel: exact fp64 tangent depths of both pixel
//                        edges at every wire step -> the window of step pairs
//                        whose trapezoid overlaps the bin range, the depth
//                        direction, monotonicity and NaN checks;
//   tile_kernel          per 32x32 tile: union step range and t_ref;
//   fit_kernel           per tile edge point: cubic in wire travel about t_ref
//                        (Chebyshev interpolation, fp64), stored fp32 in bin
//                        units, verified against the exact depth at every step
//                        the deposit kernel can read.
// The deposit kernel then evaluates corner depths with 3 FMAs instead of the
// paper's per-thread trig.
#include <cuda_runtime.h>
#include <limits.h>
#include <math.h>
#include <stdarg.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include <algorithm>
#include <new>
#include <string>
#include <vector>

#include "daxm.h"
#include "daxm_internal.cuh"

#include <cudaTypedefs.h>

using namespace daxm;

#ifndef DAXM_HOST_BANDS
#define DAXM_HOST_BANDS 32  // row bands of the in-core host pipeline (copy/compute overlap granularity)
#endif

struct daxm_plan {
    int device = 0;
    // both-edges mode (reading R16): the parent holds one plan per edge and runs both per call
    daxm_plan* child[2] = {nullptr, nullptr};
    bool is_child = false;
    float dI_floor = -INFINITY;  // children: 0 (each edge takes its own sign of change)
    int acc = 0;                 // children: 0 for the leading edge (stores), 1 for the trailing (adds)
    daxm_geometry g{};
    std::vector<double> wire;
    std::vector<double> t;        // wire travel t_k
    GeomConst gc{};
    int M = 0, rows = 0, C = 0, S = 0;
    int pre_row0 = 0, pre_rows = 0;   // global rows covered by the plan's tiles
    int tr0 = 0, n_tr = 0, n_tc = 0;
    double* d_t = nullptr;
    double* d_wire = nullptr;
    TileInfo* d_tiles = nullptr;
    int2* d_win = nullptr;
    float* d_coef = nullptr;
    signed char* d_pdir = nullptr;
    signed char* d_psep = nullptr;
    int* d_vneed = nullptr;     // [n_tiles][n_states + 1] furthest visit index needed (fast kernel)
    bool straight = true;       // wire centres on a line: travel-polynomial depth model possible
    float dt_h = 0.f, dt_l = 0.f;  // mean wire travel per step, hi + lo (row kernel's tau, row_tau)
    float* d_w = nullptr;          // per-step normalisation weights (daxm_set_step_weights), or NULL
    std::vector<double> step_w;    // ... their host copy (for band plans built later)
    float* d_table = nullptr;   // exact per-step depth table (general wire paths / model miss)
    long long* d_toff = nullptr;
    int n_states = 0;
    int* d_list_u16 = nullptr;  // general-kernel tile lists per dtype
    int* d_list_f32 = nullptr;
    int n_list_u16 = 0, n_list_f32 = 0;
    int max_nv = 0;
    // TMA descriptors, re-encoded when the caller's buffers change
    CUtensorMap in_map{}, out_map{};
    CUtensorMap lock_in_map{};  // step-locked kernel: one warp's [16 rows][8 cols] block of LOCK_G wire steps
    int lock_small = 0, lock_large = 0, lock_rest = 0;                // tile counts (lock pre-pass)
    int lock_ov_small = 0, lock_ov_large = 0;                         // ... overlapping tiles
    unsigned* d_lock_err = nullptr;                                   // ring-capacity violations
    const void* map_stack = nullptr;
    const float* map_out = nullptr;
    int map_dtype = -1;
    // end-to-end (host buffer) path scratch, allocated on first use
    void* d_stack_buf = nullptr;
    size_t stack_buf_bytes = 0;
    float* d_out_buf = nullptr;
    size_t out_buf_bytes = 0;
    cudaStream_t st_in = nullptr, st_out = nullptr;  // host-path pipeline streams
    // out-of-core host path (daxm_set_host_budget): band plans of ring_rows rows and a two-slot
    // device ring of [S][B][C] stacks and [M][B][C] outputs
    uint64_t host_budget = 0;
    int ring_rows = 0;                 // band rows the band plans were built for (0: none)
    std::vector<daxm_plan*> bands;     // band b: plan-local rows [band_r0[b], band_r0[b + 1])
    std::vector<int> band_r0;
    void* d_ring_in[2] = {nullptr, nullptr};
    float* d_ring_out[2] = {nullptr, nullptr};
    size_t ring_in_bytes = 0, ring_out_bytes = 0;
    cudaEvent_t ev_ring[6] = {nullptr, nullptr, nullptr, nullptr, nullptr, nullptr};
    int last_ring_rows = 0, last_ring_bands = 0;  // layout of the last host call (0: in core)
    static constexpr int N_FORK = 7;                 // forked streams for concurrent class launches
    cudaStream_t st_cls[N_FORK] = {};                 // (deposit-tile path: the first two)
    cudaEvent_t ev_cls[N_FORK + 1] = {};
    std::vector<cudaEvent_t> ev;
    int use_cutoff = 0;  // intensity cutoff (f1, reading R14)
    float cutoff = 0.f;
    unsigned long long* d_hist = nullptr;  // cutoff selection scratch (256 counters)
    unsigned char* d_live = nullptr;       // [n_tr][n_tc] cutoff: tile has a pixel above it
    // row-segment kernel (deposit_row.cu): row tiles of RW_ROWS x RW_COLS pixels
    bool row_ok = false;                   // the row path is available for this plan
    int row_org = 0, n_rr = 0, n_rc = 0;   // global row of row-tile row 0 (= row_begin), rows, columns
    int max_nv_row = 0;                    // largest row-tile step range
    RowTile* d_rt = nullptr;
    unsigned char* d_rlive = nullptr;  // row tiles' live flags of the last call (exact zero-dI skip)
    float* d_prof_part = nullptr;      // [n_rt][M] fused depth-profile partial sums (allocated on use)
    float* d_rcoef = nullptr;
    int* d_rlist = nullptr;                // class lists [small][large][general], each ascending
    std::vector<int> h_rlist;
    // row tiles per class, in h_rlist order: class 2 (variant + 4 ktc) + (ring 32): ring 16 / 32 x
    // variant (separated, general-span, general-span with the wide input ring, separated with the
    // 32-slot input ring) x edge-trip class ktc (3 / 4 / 5 edges per zone; separated variants), then
    // the not admitted ones (general kernel)
    static constexpr int N_RCLS = 25;
    int n_rcls[N_RCLS] = {};
    unsigned* d_row_err = nullptr;         // DAXM_ROW_CHECK builds: schedule violations
    CUtensorMap row_in_map{}, row_out_map{};
    daxm_plan_stats stats{};
    std::string err;
};

static thread_local std::string g_create_err;
static DepositArgs make_args(const daxm_plan* p, int dtype);
static RowArgs make_row_args(const daxm_plan* p);

namespace {

struct DeviceGuard {
    int prev = -1;
    explicit DeviceGuard(int dev) {
        if (cudaGetDevice(&prev) != cudaSuccess) prev = -1;
        cudaSetDevice(dev);
    }
    ~DeviceGuard() {
        if (prev >= 0) cudaSetDevice(prev);
    }
};

// ------------------------------------------------------------ fp64 geometry
__device__ __forceinline__ double dot3(const double* a, const double* b) {
    return a[0] * b[0] + a[1] * b[1] + a[2] * b[2];
}

// Lab position of detector point (column coordinate x, row j).
__device__ void detector_point(const GeomConst& g, double x, int j, double Q[3]) {
    double p0 = (x - 0.5 * (g.C - 1)) * g.pitch_col + g.trans[0];
    double p1 = ((double)j - 0.5 * (g.R - 1)) * g.pitch_row + g.trans[1];
    double p2 = g.trans[2];
    for (int r = 0; r < 3; ++r) Q[r] = g.rho[3 * r] * p0 + g.rho[3 * r + 1] * p1 + g.rho[3 * r + 2] * p2;
}

// Edge side: +1 when (a x (Q - W0)).d >= 0 for the leading edge (reading R3).
__device__ double edge_sigma(const GeomConst& g, const double Q[3]) {
    double q[3] = {Q[0] - g.w0[0], Q[1] - g.w0[1], Q[2] - g.w0[2]};
    double c[3] = {g.axis[1] * q[2] - g.axis[2] * q[1], g.axis[2] * q[0] - g.axis[0] * q[2],
                   g.axis[0] * q[1] - g.axis[1] * q[0]};
    double lead = dot3(c, g.d) >= 0.0 ? 1.0 : -1.0;
    return g.edge ? -lead : lead;
}

// Tangent depth in bin units relative to m_ref: u = (D - lo0)/dz - m_ref.
// D from the plane through Q tangent to the wire cylinder (contact normal n,
// n.(Q-W) = r) intersected with the beam: D = (n.(W-O) + r)/(n.k).  NaN if the
// pixel is inside the cylinder or the plane is parallel to the beam.
__device__ double tangent_u(const GeomConst& g, const double Q[3], double sigma, const double W[3]) {
    double qw[3] = {Q[0] - W[0], Q[1] - W[1], Q[2] - W[2]};
    double pa = dot3(qw, g.axis);
    double e[3] = {qw[0] - pa * g.axis[0], qw[1] - pa * g.axis[1], qw[2] - pa * g.axis[2]};
    double L2 = dot3(e, e);
    double r2 = g.r * g.r;
    if (!(L2 > r2)) return nan("");
    double s = sqrt(L2 - r2);
    double ae[3] = {g.axis[1] * e[2] - g.axis[2] * e[1], g.axis[2] * e[0] - g.axis[0] * e[2],
                    g.axis[0] * e[1] - g.axis[1] * e[0]};
    double n[3];
    for (int c = 0; c < 3; ++c) n[c] = (g.r * e[c] + sigma * s * ae[c]) / L2;
    double nk = dot3(n, g.beam);
    if (fabs(nk) < 1e-12) return nan("");
    double wo[3] = {W[0] - g.origin[0], W[1] - g.origin[1], W[2] - g.origin[2]};
    double D = (dot3(n, wo) + g.r) / nk;
    return (D - g.lo0) / g.dz - (double)g.m_ref;
}

__device__ __forceinline__ void edge_point(const GeomConst& g, int j, int edge_col, double Q[3]) {
    double x = g.point_mode ? (double)edge_col : (double)edge_col - 0.5;
    detector_point(g, x, j, Q);
}

__device__ __forceinline__ void atomic_max_pos_double(double* addr, double v) {
    // non-negative doubles order like their bit patterns
    atomicMax(reinterpret_cast<unsigned long long*>(addr), (unsigned long long)__double_as_longlong(v));
}

// ------------------------------------------------------------ pixel windows
// One warp per PW_PIX = 31 consecutive pixels of one row: lane l evaluates pixel edge point
// base + l (finite pixels: column base + l - 1/2; POINT: the pixel centre) at every wire step and
// pixel base + l (l < 31) takes its front edge from lane l + 1 (warp shuffle), so every edge point's
// tangent depth is computed once instead of twice.
constexpr int PW_PIX = 31;
__global__ void __launch_bounds__(128) pixel_window_kernel(GeomConst g, const double* __restrict__ wire, int pre_row0,
                                                           int pre_rows, int band_r0, int band_r1,
                                                           int2* __restrict__ win, signed char* __restrict__ pdir,
                                                           signed char* __restrict__ psep, unsigned* __restrict__ flags,
                                                           unsigned long long* __restrict__ counters) {
    const int lane = threadIdx.x & 31;
    const int wrow = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);  // warp index within the row
    const int jl = blockIdx.y;
    const int base = wrow * PW_PIX;
    if (base >= g.C || jl >= pre_rows) return;  // (warp-uniform)
    const int j = pre_row0 + jl;
    const int i = base + lane;  // this lane's pixel (lane < PW_PIX)
    const bool pix = lane < PW_PIX && i < g.C;
    if (j < band_r0 || j >= band_r1) {  // rows of a boundary tile outside the band: never output
        if (pix) {
            win[(size_t)jl * g.C + i] = make_int2(0, 0);
            pdir[(size_t)jl * g.C + i] = 0;
            psep[(size_t)jl * g.C + i] = 3;
        }
        return;
    }
    const int n_edges = g.point_mode ? g.C : g.C + 1;
    double Q[3];
    edge_point(g, j, min(i, n_edges - 1), Q);  // lane's edge point (lanes past the last edge: a copy)
    const double sg = edge_sigma(g, Q);
    const double upper = (double)(g.M - g.m_ref), lower = (double)(-g.m_ref);
    // back edge = this lane's point, front edge = the next lane's (POINT: the same point)
    auto depths = [&](int k, double& ub, double& uf) {
        ub = tangent_u(g, Q, sg, wire + 3 * k);
        const double nx = __shfl_down_sync(0xffffffffu, ub, 1);
        uf = g.point_mode ? ub : nx;
    };

    // pass 1: relevant pairs (trapezoid overlaps (0, M) bins), NaN bookkeeping
    double ub0, uf0;
    depths(0, ub0, uf0);
    int first = -1, last = -1;
    bool prev_nan = false, first_prev_nan = false, pending_nan = false, next_nan = false, nan_inside = false;
    bool any_valid = false;
    for (int k = 0; k + 1 < g.S; ++k) {
        double ub1, uf1;
        depths(k + 1, ub1, uf1);
        bool isn = isnan(ub0) || isnan(uf0) || isnan(ub1) || isnan(uf1);
        if (last >= 0 && k == last + 1) next_nan = isn;
        any_valid |= !isn;
        if (!isn) {
            double lo = fmin(fmin(ub0, uf0), fmin(ub1, uf1)), hi = fmax(fmax(ub0, uf0), fmax(ub1, uf1));
            if (hi > lower && lo < upper) {
                if (first < 0) {
                    first = k;
                    first_prev_nan = prev_nan;
                }
                if (pending_nan) nan_inside = true;
                last = k;
            }
        } else if (first >= 0) {
            pending_nan = true;
        }
        prev_nan = isn;
        ub0 = ub1;
        uf0 = uf1;
    }
    int2 w = make_int2(0, 0);
    signed char dir = 0, sep = 3;
    if (pix && any_valid) atomicAdd(&counters[4], 1ull);  // a pixel with every pair NaN is invalid (reading R8)
    int kb = INT_MAX, ke = -1;  // window points kb..ke (pairs [kb, ke))
    if (pix && first >= 0) {
        // NaN pairs inside the window (the pixel edge inside the wire cylinder at some step): the
        // pairs are skipped (reading R8) by the exact-table general kernel the host then selects
        if (nan_inside) atomicOr(flags, FLAG_NAN_IN_WINDOW);
        atomicAdd(&counters[2], (unsigned long long)(last - first + 1));
        atomicAdd(&counters[3], 1ull);
        kb = first;
        ke = last + 1;
        if (kb > 0 && !first_prev_nan) --kb;  // one guard pair each side (fp32 rounding)
        if (ke <= g.S - 2 && !next_nan) ++ke;
    }
    // pass 2: monotonicity and direction over each window's points kb..ke, and "separation":
    // consecutive points' edge spans [lo, hi] are disjoint (by a 1e-3-bin margin) and every trapezoid
    // has area >= 1e-3 bins, in either visiting order -- the condition for the fast deposit kernel's
    // piecewise-linear form.  The warp walks the union of its windows.
    const int KB = __reduce_min_sync(0xffffffffu, kb), KE = __reduce_max_sync(0xffffffffu, ke);
    bool pos = false, neg = false, sep_pos = true, sep_neg = true, ovl_pos = true, ovl_neg = true;
    double pb = 0.0, pf = 0.0;
    for (int k = KB; k <= KE; ++k) {
        double cb, cf;
        depths(k, cb, cf);
        if (k > kb && k <= ke) {
            double db = cb - pb, df = cf - pf;
            pos |= (db > 0.0) || (df > 0.0);
            neg |= (db < 0.0) || (df < 0.0);
            const double lo0 = fmin(pb, pf), hi0 = fmax(pb, pf), lo1 = fmin(cb, cf), hi1 = fmax(cb, cf);
            const double area = 0.5 * ((lo1 + hi1) - (lo0 + hi0));
            sep_pos &= (hi0 <= lo1 - 1e-3) && (area >= 1e-3);
            sep_neg &= (hi1 <= lo0 - 1e-3) && (-area >= 1e-3);
            // dual-walk mode (any span/sweep relation): rising ramp [lo_a, min(hi_a, lo_b)] and
            // falling ramp [max(hi_a, lo_b), hi_b] of nonzero length, area >= 1e-3 bins
            ovl_pos &= (fmin(hi0, lo1) >= lo0 + 1e-3) && (hi1 >= fmax(hi0, lo1) + 1e-3) &&
                       (0.5 * (hi1 + fmax(hi0, lo1) - fmin(hi0, lo1) - lo0) >= 1e-3);
            ovl_neg &= (fmin(hi1, lo0) >= lo1 + 1e-3) && (hi0 >= fmax(hi1, lo0) + 1e-3) &&
                       (0.5 * (hi0 + fmax(hi1, lo0) - fmin(hi1, lo0) - lo1) >= 1e-3);
        }
        pb = cb;
        pf = cf;
    }
    if (pix && ke >= 0) {
        if (pos && neg) atomicOr(flags, FLAG_NONMONOTONE);
        dir = neg ? -1 : 1;
        // bit 0: separated (single zone walk), bit 1: dual walk applicable
        sep = ((dir > 0 ? sep_pos : sep_neg) ? 1 : 0) | ((dir > 0 ? ovl_pos : ovl_neg) ? 2 : 0);
        w = make_int2(kb, ke);
    }
    if (pix) {
        win[(size_t)jl * g.C + i] = w;
        pdir[(size_t)jl * g.C + i] = dir;
        psep[(size_t)jl * g.C + i] = sep;
    }
}

// ------------------------------------------------------------ tiles
// One CTA (TILE_C x TILE_R threads) per tile: union step range, t_ref,
// separation, and the input-ring bound of the fast kernel.  ring_need bounds
// how far apart (in streamed steps) the tile's pixels can be between two
// consecutive output-chunk boundaries: with v_p(E) = v0_p + #{points of p with
// lo < E}, ring_need = max over c of [max_p v_p(E_{c+W}) - min_p v_p(E_c)] + 3 with
// W = RING_WINDOW_CHUNKS output chunks (the loads a warp may wait for are issued
// at most W chunks after the slowest pixel's frontier).
// A ring of at least that many slots can never deadlock.
__global__ void __launch_bounds__(1024) tile_kernel(GeomConst g, const double* __restrict__ t, const double* __restrict__ wire,
                            int pre_row0, int pre_rows, int tr0, int n_tc, int band_r0, int band_r1,
                            const int2* __restrict__ win, const signed char* __restrict__ pdir,
                            const signed char* __restrict__ psep, TileInfo* __restrict__ tiles,
                            unsigned* __restrict__ flags, unsigned long long* __restrict__ counters, int n_states,
                            int* __restrict__ vneed) {
    extern __shared__ int s_v[];  // [2][n_states + 1]: max, min of v_p at each state; then [n_states + 1][8] per warp
    const int tile = blockIdx.x;
    const int tr = tile / n_tc, tc = tile % n_tc;
    const int c = threadIdx.x, r = threadIdx.y;  // TILE_C x TILE_R
    const int tid = r * TILE_C + c;
    const int nthr = blockDim.x * blockDim.y;
    const int j = (tr0 + tr) * TILE_R + r, i = tc * TILE_C + c;
    int kb = INT_MAX, ke = INT_MIN, dpos = 0, dneg = 0, nsep = 0, novl = 0;
    long long pairs = 0;
    if (j < g.R && i < g.C && j >= pre_row0 && j < pre_row0 + pre_rows) {
        int2 w = win[(size_t)(j - pre_row0) * g.C + i];
        if (w.y > w.x) {
            kb = w.x;
            ke = w.y;  // last point read = ke
            signed char d = pdir[(size_t)(j - pre_row0) * g.C + i];
            dpos = d > 0;
            dneg = d < 0;
            const signed char m = psep[(size_t)(j - pre_row0) * g.C + i];
            nsep = (m & 1) ? 0 : 1;
            novl = (m & 2) ? 0 : 1;
            if (j >= band_r0 && j < band_r1) pairs = w.y - w.x;
        }
    }
    __shared__ int s_kb, s_ke, s_pos, s_neg, s_nsep, s_novl, s_need;
    __shared__ unsigned long long s_pairs;
    const bool track = n_states <= MAX_FAST_CHUNKS;
    if (tid == 0) {
        s_kb = INT_MAX;
        s_ke = INT_MIN;
        s_pos = s_neg = s_nsep = s_novl = 0;
        s_need = 0;
        s_pairs = 0;
    }
    int* s_w = s_v + 2 * (n_states + 1);  // per consumer warp of the fast kernel
    const int fwarp = (r / 32) * (TILE_C / COLS_PER_THREAD) + c / COLS_PER_THREAD;
    if (track) {
        for (int q = tid; q <= n_states; q += nthr) {
            s_v[q] = INT_MIN;
            s_v[n_states + 1 + q] = INT_MAX;
        }
        for (int q = tid; q < (n_states + 1) * N_CONSUMER_WARPS; q += nthr) s_w[q] = INT_MIN;
    }
    __syncthreads();
    if (kb != INT_MAX) {
        atomicMin(&s_kb, kb);
        atomicMax(&s_ke, ke);
        if (dpos) atomicOr(&s_pos, 1);
        if (dneg) atomicOr(&s_neg, 1);
        if (nsep) atomicOr(&s_nsep, 1);
        if (novl) atomicOr(&s_novl, 1);
        atomicAdd(&s_pairs, (unsigned long long)pairs);
    }
    __syncthreads();
    const int k_lo = s_kb, k_hi = s_ke;
    const int tdir = s_neg ? -1 : 1;
    // ring bound: state 0 = before any edge (v0), state 1 + c = after edge e = min(c*MC, M)
    if (track && kb != INT_MAX) {
        double Qb[3], Qf[3];
        edge_point(g, j, i, Qb);
        edge_point(g, j, g.point_mode ? i : i + 1, Qf);
        const double sb = edge_sigma(g, Qb), sf = edge_sigma(g, Qf);
        const int n_pts = ke - kb + 1;
        const int v0 = tdir > 0 ? kb - k_lo : k_hi - ke;
        atomicMax(&s_v[0], v0);
        atomicMin(&s_v[n_states + 1], v0);
        atomicMax(&s_w[fwarp], v0);
        int q = 0;  // points with lo < E seen so far
        double lo_q = 0.0;
        bool have = false;
        for (int st = 1; st <= n_states; ++st) {
            const int e = min((st - 1) * MC, g.M);
            const double E = (double)(e - g.m_ref);
            while (q < n_pts) {
                if (!have) {
                    const int k = tdir > 0 ? kb + q : ke - q;
                    lo_q = fmin(tangent_u(g, Qb, sb, wire + 3 * k), tangent_u(g, Qf, sf, wire + 3 * k));
                    have = true;
                }
                if (lo_q < E) {
                    ++q;
                    have = false;
                } else {
                    break;
                }
            }
            atomicMax(&s_v[st], v0 + q);
            atomicMin(&s_v[n_states + 1 + st], v0 + q);
            atomicMax(&s_w[st * N_CONSUMER_WARPS + fwarp], v0 + q);
        }
    }
    __syncthreads();
    // furthest visit index any pixel of the tile loads by the end of each state (+1: fp32 rounding),
    // so the fast kernel can wait for its input once per output chunk
    // [state][warp 0..7, tile-wide max]: a warp whose pixels are all finished (or that has none)
    // follows the tile-wide horizon so it keeps releasing ring slots in step with the others
    if (track)
        for (int q = tid; q < (n_states + 1) * (N_CONSUMER_WARPS + 1); q += nthr) {
            const int st = q / (N_CONSUMER_WARPS + 1), wq = q % (N_CONSUMER_WARPS + 1);
            const int hi = wq < N_CONSUMER_WARPS ? s_w[st * N_CONSUMER_WARPS + wq] : s_v[st];
            vneed[(size_t)tile * (n_states + 1) * (N_CONSUMER_WARPS + 1) + q] =
                (s_kb == INT_MAX || hi == INT_MIN) ? -1 : min(hi + 2, s_ke - s_kb);  // +1 prefetch, +1 fp32
        }
    if (track && s_kb != INT_MAX)
        for (int q = tid; q < n_states; q += nthr) {
            // states q -> q + RING_WINDOW_CHUNKS (clamped): the span of steps in flight
            const int q2 = min(q + RING_WINDOW_CHUNKS, n_states);
            const int hi = s_v[q2], lo = s_v[n_states + 1 + q];
            if (hi != INT_MIN && lo != INT_MAX) atomicMax(&s_need, hi - lo + 4);
        }
    __syncthreads();
    if (tid == 0) {
        TileInfo ti;
        ti.lock = 0;
        if (s_kb == INT_MAX) {
            ti.t_ref = 0.0;
            ti.k_lo = 0;
            ti.k_hi = -1;
            ti.dir = 1;
            ti.separated = MODE_SEPARATED;
            ti.ring_need = 0;
        } else {
            ti.k_lo = k_lo;
            ti.k_hi = k_hi;
            ti.t_ref = 0.5 * (t[k_lo] + t[k_hi]);
            ti.dir = tdir;
            ti.separated = !s_nsep ? MODE_SEPARATED : !s_novl ? MODE_OVERLAP : MODE_GENERAL;
            // the overlap walk's hi ramps lag the lo ramps by up to two points
            ti.ring_need = track ? s_need + (ti.separated == MODE_OVERLAP ? 2 : 0) : INT_MAX;
            if (s_pos && s_neg) atomicOr(flags, FLAG_MIXED_DIR);
            // staged steps, only for tiles that intersect the band
            int tj0 = (tr0 + tr) * TILE_R, tj1 = tj0 + TILE_R;
            if (tj1 > band_r0 && tj0 < band_r1) atomicAdd(&counters[1], (unsigned long long)(k_hi - k_lo + 1));
        }
        tiles[tile] = ti;
        atomicAdd(&counters[0], s_pairs);
    }
}

// ------------------------------------------------------------ depth polynomial fit
// One edge point Q (edge side sg): the depth u(t) in bins relative to m_ref as a polynomial of
// degree NCOEF-1 in tau = t - t_ref, Chebyshev-interpolated in fp64 over the tile's step range
// [t_{k_lo}, t_{k_hi}], stored fp32, and verified against the exact depth at every step the
// deposit kernels can read: model error (fp64 polynomial) and stored error (fp32 coefficients,
// fp32 tau, the kernels' evaluation).
__device__ void fit_point(const GeomConst& g, const double* __restrict__ t, const double* __restrict__ wire,
                          double t_ref, int k_lo, int k_hi, const double Q[3], double sg, unsigned* flags,
                          float cf[NCOEF], double& local_err, double& local_model, int lin_dir = 0,
                          float dth = 0.f, float dtl = 0.f) {
    const double h = 0.5 * (t[k_hi] - t[k_lo]);
    double b[NCOEF];
    for (int m = 0; m < NCOEF; ++m) b[m] = 0.0;
    if (h > 0.0) {
        // Chebyshev interpolation at the NCOEF first-kind nodes of [t_lo, t_hi]
        double a[NCOEF];
        for (int m = 0; m < NCOEF; ++m) a[m] = 0.0;
        for (int n = 0; n < NCOEF; ++n) {
            const double th = M_PI * (2 * n + 1) / (2.0 * NCOEF);
            const double x = cos(th);
            const double tn = t_ref + h * x;
            double W[3] = {g.w0[0] + tn * g.d[0], g.w0[1] + tn * g.d[1], g.w0[2] + tn * g.d[2]};
            const double u = tangent_u(g, Q, sg, W);
            if (isnan(u)) atomicOr(flags, FLAG_FIT_NAN);
            for (int m = 0; m < NCOEF; ++m) a[m] += u * cos(m * th);
        }
        for (int m = 0; m < NCOEF; ++m) a[m] *= (m == 0 ? 1.0 : 2.0) / NCOEF;
        // Chebyshev -> monomial in x (T_{n+1} = 2x T_n - T_{n-1}), then x = tau / h
        double Tm[NCOEF], Tc[NCOEF], Tn[NCOEF], bx[NCOEF];
        for (int m = 0; m < NCOEF; ++m) Tm[m] = Tc[m] = bx[m] = 0.0;
        Tm[0] = 1.0;                 // T_0
        if (NCOEF > 1) Tc[1] = 1.0;  // T_1
        for (int m = 0; m < NCOEF; ++m) bx[m] += a[0] * Tm[m];
        if (NCOEF > 1)
            for (int m = 0; m < NCOEF; ++m) bx[m] += a[1] * Tc[m];
        for (int n = 2; n < NCOEF; ++n) {
            for (int m = 0; m < NCOEF; ++m) Tn[m] = (m > 0 ? 2.0 * Tc[m - 1] : 0.0) - Tm[m];
            for (int m = 0; m < NCOEF; ++m) {
                bx[m] += a[n] * Tn[m];
                Tm[m] = Tc[m];
                Tc[m] = Tn[m];
            }
        }
        double hp = 1.0;
        for (int m = 0; m < NCOEF; ++m) {
            b[m] = bx[m] / hp;
            hp *= h;
        }
    } else {
        double W[3] = {g.w0[0] + t_ref * g.d[0], g.w0[1] + t_ref * g.d[1], g.w0[2] + t_ref * g.d[2]};
        b[0] = tangent_u(g, Q, sg, W);
        if (isnan(b[0])) atomicOr(flags, FLAG_FIT_NAN);
    }
    for (int m = 0; m < NCOEF; ++m) cf[m] = (float)b[m];
    for (int k = k_lo; k <= k_hi; ++k) {
        const double ex = tangent_u(g, Q, sg, wire + 3 * k);
        if (isnan(ex)) continue;
        const double td = t[k] - t_ref;
        // the kernel's fp32 tau: the tile table's rounding, or the row kernel's row_tau
        const double tau = lin_dir == 0 ? (double)(float)td
                         : (double)row_tau((float)(t[lin_dir > 0 ? k_lo : k_hi] - t_ref), lin_dir * dth, lin_dir * dtl,
                                           lin_dir > 0 ? k - k_lo : k_hi - k);
        double pm = b[NCOEF - 1], pp = (double)cf[NCOEF - 1];
        for (int m = NCOEF - 2; m >= 0; --m) {
            pm = b[m] + td * pm;
            pp = (double)cf[m] + tau * pp;
        }
        local_model = fmax(local_model, fabs(pm - ex));
        local_err = fmax(local_err, fabs(pp - ex));
    }
}

__global__ void __launch_bounds__(1024) fit_kernel(GeomConst g, const double* __restrict__ t, const double* __restrict__ wire, int tr0,
                           int n_tc, const TileInfo* __restrict__ tiles, float* __restrict__ coef,
                           unsigned* __restrict__ flags, double* __restrict__ max_err) {
    const int tile = blockIdx.x;
    const int tr = tile / n_tc, tc = tile % n_tc;
    const TileInfo ti = tiles[tile];
    const int r = threadIdx.x;  // row in tile
    const int j = (tr0 + tr) * TILE_R + r;
    double local_err = 0.0, local_model = 0.0;
    for (int e = threadIdx.y; e < TILE_E; e += blockDim.y) {
        const int eg = tc * TILE_C + e;  // global edge column
        const int n_edges = g.point_mode ? g.C : g.C + 1;
        float cf[NCOEF];
        for (int m = 0; m < NCOEF; ++m) cf[m] = 0.f;
        if (ti.k_hi >= ti.k_lo && j < g.R && eg < n_edges) {
            double Q[3];
            edge_point(g, j, eg, Q);
            fit_point(g, t, wire, ti.t_ref, ti.k_lo, ti.k_hi, Q, edge_sigma(g, Q), flags, cf, local_err, local_model);
        }
        for (int m = 0; m < NCOEF; ++m) coef[(((size_t)tile * NCOEF + m) * TILE_E + e) * TILE_R + r] = cf[m];
    }
    if (local_err > 0.0) atomic_max_pos_double(max_err, local_err);
    if (local_model > 0.0) atomic_max_pos_double(max_err + 1, local_model);
}

// ------------------------------------------------------------ row tiles (deposit_row.cu)
// One CTA per row tile (RW_ROWS x RW_COLS pixels): union of the band pixels' windows, direction,
// span regime, t_ref.  Rows outside the band carry no window (pixel_window_kernel).
__global__ void __launch_bounds__(RW_ROWS * RW_COLS) row_tile_kernel(
    GeomConst g, const double* __restrict__ t, int row_org, int n_rc, int pre_row0, int pre_rows,
    const int2* __restrict__ win, const signed char* __restrict__ pdir, const signed char* __restrict__ psep,
    RowTile* __restrict__ rts, unsigned* __restrict__ flags) {
    const int rt = blockIdx.x;
    const int rr = rt / n_rc, rc = rt % n_rc;
    const int j = row_org + rr * RW_ROWS + (int)threadIdx.y, i = rc * RW_COLS + (int)threadIdx.x;
    __shared__ int s_kb, s_ke, s_pos, s_neg, s_nsep, s_novl;
    if (threadIdx.x == 0 && threadIdx.y == 0) {
        s_kb = INT_MAX;
        s_ke = INT_MIN;
        s_pos = s_neg = s_nsep = s_novl = 0;
    }
    __syncthreads();
    if (i < g.C && j >= pre_row0 && j < pre_row0 + pre_rows) {
        const size_t q = (size_t)(j - pre_row0) * g.C + i;
        const int2 w = win[q];
        if (w.y > w.x) {
            atomicMin(&s_kb, w.x);
            atomicMax(&s_ke, w.y);
            if (pdir[q] > 0) atomicOr(&s_pos, 1);
            if (pdir[q] < 0) atomicOr(&s_neg, 1);
            if (!(psep[q] & 1)) atomicOr(&s_nsep, 1);
            if (!(psep[q] & 2)) atomicOr(&s_novl, 1);
        }
    }
    __syncthreads();
    if (threadIdx.x == 0 && threadIdx.y == 0) {
        RowTile ti;
        ti.cls = 0;
        ti.niter = 0;
        ti.why = 0;
        if (s_kb == INT_MAX) {
            ti.t_ref = 0.0;
            ti.k_lo = 0;
            ti.k_hi = -1;
            ti.dir = 1;
            ti.sep = MODE_SEPARATED;
        } else {
            ti.dir = s_neg ? -1 : 1;
            // room for the lock-step starts before the windows (deposit_row.cu row_starts)
            ti.k_lo = ti.dir > 0 ? max(s_kb - RW_EXT, 0) : s_kb;
            ti.k_hi = ti.dir > 0 ? s_ke : min(s_ke + RW_EXT, g.S - 1);
            ti.t_ref = 0.5 * (t[ti.k_lo] + t[ti.k_hi]);
            ti.sep = !s_nsep ? MODE_SEPARATED : !s_novl ? MODE_OVERLAP : MODE_GENERAL;
            if (s_pos && s_neg) atomicOr(flags, FLAG_MIXED_DIR);
        }
        rts[rt] = ti;
    }
}

// Depth polynomials of a row tile's edge points: [rt][NCOEF][RW_COLS + 1 edge columns][RW_ROWS].
__global__ void __launch_bounds__(RW_ROWS * (RW_COLS + 1)) row_fit_kernel(
    GeomConst g, const double* __restrict__ t, const double* __restrict__ wire, int row_org, int n_rc,
    const RowTile* __restrict__ rts, float* __restrict__ coef, unsigned* __restrict__ flags,
    double* __restrict__ max_err, float dth, float dtl) {
    const int rt = blockIdx.x;
    const RowTile ti = rts[rt];
    const int rr = rt / n_rc, rc = rt % n_rc;
    const int r = threadIdx.x, e = threadIdx.y;  // RW_ROWS x (RW_COLS + 1)
    const int j = row_org + rr * RW_ROWS + r, eg = rc * RW_COLS + e;
    const int n_edges = g.point_mode ? g.C : g.C + 1;
    double local_err = 0.0, local_model = 0.0;
    float cf[NCOEF];
    for (int m = 0; m < NCOEF; ++m) cf[m] = 0.f;
    if (ti.k_hi >= ti.k_lo && j < g.R && eg < n_edges) {
        double Q[3];
        edge_point(g, j, eg, Q);
        fit_point(g, t, wire, ti.t_ref, ti.k_lo, ti.k_hi, Q, edge_sigma(g, Q), flags, cf, local_err, local_model,
                  DAXM_ROW_TAU_LINEAR ? (ti.dir > 0 ? 1 : -1) : 0, dth, dtl);
    }
    for (int m = 0; m < NCOEF; ++m) coef[(((size_t)rt * NCOEF + m) * (RW_COLS + 1) + e) * RW_ROWS + r] = cf[m];
    if (local_err > 0.0) atomic_max_pos_double(max_err, local_err);
    if (local_model > 0.0) atomic_max_pos_double(max_err + 1, local_model);
}

daxm_status fail(daxm_plan* p, daxm_status s, const char* fmt, ...) {
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof buf, fmt, ap);
    va_end(ap);
    if (p)
        p->err = buf;
    else
        g_create_err = buf;
    return s;
}

bool finite3(const double* v) { return isfinite(v[0]) && isfinite(v[1]) && isfinite(v[2]); }
double norm3(const double* v) { return sqrt(v[0] * v[0] + v[1] * v[1] + v[2] * v[2]); }

void rodrigues(const double R[3], double rho[9]) {
    double th = norm3(R);
    for (int i = 0; i < 9; ++i) rho[i] = (i % 4 == 0) ? 1.0 : 0.0;
    if (th == 0.0) return;
    double k[3] = {R[0] / th, R[1] / th, R[2] / th};
    double K[9] = {0, -k[2], k[1], k[2], 0, -k[0], -k[1], k[0], 0};
    double s = sin(th), c1 = 1.0 - cos(th);
    for (int r = 0; r < 3; ++r)
        for (int c = 0; c < 3; ++c) {
            double k2 = 0;
            for (int q = 0; q < 3; ++q) k2 += K[3 * r + q] * K[3 * q + c];
            rho[3 * r + c] += s * K[3 * r + c] + c1 * k2;
        }
}

// out-of-core ring: band plans and slots
void free_ring(daxm_plan* p) {
    for (daxm_plan* b : p->bands) daxm_destroy(b);
    p->bands.clear();
    p->band_r0.clear();
    p->ring_rows = 0;
    for (int i = 0; i < 2; ++i) {
        cudaFree(p->d_ring_in[i]);
        cudaFree(p->d_ring_out[i]);
        p->d_ring_in[i] = nullptr;
        p->d_ring_out[i] = nullptr;
    }
    p->ring_in_bytes = p->ring_out_bytes = 0;
    for (cudaEvent_t& e : p->ev_ring) {
        if (e) cudaEventDestroy(e);
        e = nullptr;
    }
}

void free_plan_memory(daxm_plan* p) {
    cudaFree(p->d_t);
    cudaFree(p->d_wire);
    cudaFree(p->d_tiles);
    cudaFree(p->d_win);
    cudaFree(p->d_coef);
    cudaFree(p->d_pdir);
    cudaFree(p->d_psep);
    cudaFree(p->d_list_u16);
    cudaFree(p->d_vneed);
    cudaFree(p->d_list_f32);
    cudaFree(p->d_stack_buf);
    cudaFree(p->d_out_buf);
    p->d_stack_buf = nullptr;
    p->d_out_buf = nullptr;
    p->stack_buf_bytes = p->out_buf_bytes = 0;
    free_ring(p);
    cudaFree(p->d_hist);
    cudaFree(p->d_live);
    cudaFree(p->d_table);
    cudaFree(p->d_toff);
    cudaFree(p->d_lock_err);
    p->d_lock_err = nullptr;
    cudaFree(p->d_rt);
    cudaFree(p->d_rlive);
    cudaFree(p->d_prof_part);
    cudaFree(p->d_rcoef);
    cudaFree(p->d_w);
    p->d_w = nullptr;
    cudaFree(p->d_rlist);
    cudaFree(p->d_row_err);
    p->d_rt = nullptr;
    p->d_rlive = nullptr;
    p->d_prof_part = nullptr;
    p->d_rcoef = nullptr;
    p->d_rlist = nullptr;
    p->d_row_err = nullptr;
    for (cudaStream_t& x : p->st_cls) {
        if (x) cudaStreamDestroy(x);
        x = nullptr;
    }
    for (cudaEvent_t& x : p->ev_cls) {
        if (x) cudaEventDestroy(x);
        x = nullptr;
    }
    if (p->st_in) cudaStreamDestroy(p->st_in);
    if (p->st_out) cudaStreamDestroy(p->st_out);
    p->st_in = p->st_out = nullptr;
    for (cudaEvent_t ev : p->ev) cudaEventDestroy(ev);
    p->ev.clear();
    p->d_t = p->d_wire = nullptr;
    p->d_tiles = nullptr;
    p->d_win = nullptr;
    p->d_coef = nullptr;
    p->d_pdir = nullptr;
    p->d_psep = nullptr;
    p->d_list_u16 = p->d_list_f32 = nullptr;
    p->d_vneed = nullptr;
    p->d_stack_buf = nullptr;
    p->d_out_buf = nullptr;
}

#define CK(call)                                                                                  \
    do {                                                                                          \
        cudaError_t e_ = (call);                                                                  \
        if (e_ != cudaSuccess) {                                                                  \
            daxm_status s_ = e_ == cudaErrorMemoryAllocation ? DAXM_ERR_OUT_OF_MEMORY : DAXM_ERR_CUDA; \
            fail(nullptr, s_, "%s: %s (%s:%d)", #call, cudaGetErrorString(e_), __FILE__, __LINE__);     \
            cudaGetLastError();                                                                   \
            return s_;                                                                            \
        }                                                                                         \
    } while (0)

daxm_status host_prepare(daxm_plan* p) {
    const daxm_geometry& g = p->g;
    GeomConst& gc = p->gc;
    // ---- host geometry: rotation, unit vectors, scan line
    rodrigues(g.det_rot, gc.rho);
    for (int c = 0; c < 3; ++c) gc.trans[c] = g.det_trans[c];
    gc.pitch_col = g.pitch_col;
    gc.pitch_row = g.pitch_row;
    double na = norm3(g.wire_axis), nb = norm3(g.beam_dir);
    for (int c = 0; c < 3; ++c) {
        gc.axis[c] = g.wire_axis[c] / na;
        gc.beam[c] = g.beam_dir[c] / nb;
        gc.origin[c] = g.beam_origin[c];
    }
    const int S = g.n_steps;
    const double* W = p->wire.data();
    for (int c = 0; c < 3; ++c) gc.w0[c] = W[c];
    std::vector<double> v(3 * (size_t)S);
    for (int k = 0; k < S; ++k) {
        double q[3] = {W[3 * k] - W[0], W[3 * k + 1] - W[1], W[3 * k + 2] - W[2]};
        double pa = q[0] * gc.axis[0] + q[1] * gc.axis[1] + q[2] * gc.axis[2];
        for (int c = 0; c < 3; ++c) v[3 * k + c] = q[c] - pa * gc.axis[c];
    }
    double dl = norm3(&v[3 * (S - 1)]);
    if (!(dl > 0.0))
        return fail(nullptr, DAXM_ERR_NONMONOTONE_SCAN, "first and last wire positions coincide (perpendicular to the axis)");
    for (int c = 0; c < 3; ++c) gc.d[c] = v[3 * (S - 1) + c] / dl;
    p->t.assign(S, 0.0);
    p->straight = true;
    for (int k = 0; k < S; ++k) {
        double tk = v[3 * k] * gc.d[0] + v[3 * k + 1] * gc.d[1] + v[3 * k + 2] * gc.d[2];
        double res[3] = {v[3 * k] - tk * gc.d[0], v[3 * k + 1] - tk * gc.d[1], v[3 * k + 2] - tk * gc.d[2]};
        if (norm3(res) > 1e-6 + 1e-9 * fabs(tk)) p->straight = false;  // general path: exact depth table
        p->t[k] = tk;
    }
    {
        const double D = p->t[S - 1] / (double)(S - 1);
        p->dt_h = (float)D;
        p->dt_l = (float)(D - (double)p->dt_h);
    }
    for (int k = 1; k < S && p->straight; ++k)
        if (p->t[k] < p->t[k - 1])
            return fail(nullptr, DAXM_ERR_NONMONOTONE_SCAN, "wire travel decreases between steps %d and %d", k - 1, k);
    gc.r = g.wire_radius;
    gc.dz = g.depth_res;
    gc.lo0 = g.depth_start - 0.5 * g.depth_res;
    gc.R = g.n_rows;
    gc.C = g.n_cols;
    gc.S = S;
    gc.M = p->M;
    gc.edge = g.edge;
    gc.point_mode = g.pixel_model == DAXM_PIXEL_POINT;
    gc.m_ref = p->M / 2;
    return DAXM_OK;
}

// Exact per-step depth table (general wire paths, or where the polynomial model
// misses its tolerance): for every tile, edge point and step of the tile's step
// range, u = (D - lo0)/dz - m_ref in fp32.  One CTA per tile, TILE_R x 8 threads.
__global__ void __launch_bounds__(1024) table_kernel(GeomConst g, const double* __restrict__ wire, int tr0, int n_tc,
                             const TileInfo* __restrict__ tiles, const long long* __restrict__ toff,
                             float* __restrict__ table) {
    const int tile = blockIdx.x;
    const TileInfo ti = tiles[tile];
    if (ti.k_hi < ti.k_lo) return;
    const int tr = tile / n_tc, tc = tile % n_tc;
    const int r = threadIdx.x;
    const int j = (tr0 + tr) * TILE_R + r;
    const int nv = ti.k_hi - ti.k_lo + 1;
    float* tb = table + toff[tile];
    for (int e = threadIdx.y; e < TILE_E; e += blockDim.y) {
        double Q[3];
        edge_point(g, j, tc * TILE_C + e, Q);
        const double sg = edge_sigma(g, Q);
        for (int v = 0; v < nv; ++v)
            tb[((size_t)v * TILE_E + e) * TILE_R + r] = (float)tangent_u(g, Q, sg, wire + 3 * (ti.k_lo + v));
    }
}

// Row tiles of the row-segment kernel (deposit_row.cu): union windows, depth polynomials, and the
// admission replay; per-class lists (ascending row-tile index) for the launches.
daxm_status row_prepass(daxm_plan* p, int) {
    const daxm_geometry& g = p->g;
    GeomConst& gc = p->gc;
    // row tiles start at the band's first row (a band start inside a tile would need a negative TMA
    // row coordinate, which bulk-tensor stores reject); for even band starts they stay aligned to
    // global rows, so such a band reproduces the full-detector plan bit for bit
    p->row_org = g.row_begin;
    p->n_rr = (g.row_end - g.row_begin + RW_ROWS - 1) / RW_ROWS;
    p->n_rc = (g.n_cols + RW_COLS - 1) / RW_COLS;
    const size_t n_rt = (size_t)p->n_rr * p->n_rc;
    CK(cudaMalloc(&p->d_rt, sizeof(RowTile) * n_rt));
    CK(cudaMalloc(&p->d_rlive, n_rt));
    CK(cudaMalloc(&p->d_rcoef, sizeof(float) * n_rt * NCOEF * (RW_COLS + 1) * RW_ROWS));
    CK(cudaMalloc(&p->d_row_err, 64));
    CK(cudaMemset(p->d_row_err, 0, 64));
    unsigned* d_flags = p->d_row_err + 4;  // [4] flags, [6..9] fit errors (doubles), [10..13] stats
    double* d_err = reinterpret_cast<double*>(p->d_row_err + 6);
    int* d_stats = reinterpret_cast<int*>(p->d_row_err + 10);
    row_tile_kernel<<<(unsigned)n_rt, dim3(RW_COLS, RW_ROWS)>>>(gc, p->d_t, p->row_org, p->n_rc, p->pre_row0,
                                                                p->pre_rows, p->d_win, p->d_pdir, p->d_psep, p->d_rt,
                                                                d_flags);
    CK(cudaGetLastError());
    row_fit_kernel<<<(unsigned)n_rt, dim3(RW_ROWS, RW_COLS + 1)>>>(gc, p->d_t, p->d_wire, p->row_org, p->n_rc,
                                                                   p->d_rt, p->d_rcoef, d_flags, d_err, p->dt_h,
                                                                   p->dt_l);
    CK(cudaGetLastError());
    std::vector<RowTile> ht(n_rt);
    CK(cudaMemcpy(ht.data(), p->d_rt, sizeof(RowTile) * n_rt, cudaMemcpyDeviceToHost));
    p->max_nv_row = 1;
    for (const RowTile& t : ht)
        if (t.k_hi >= t.k_lo) p->max_nv_row = std::max(p->max_nv_row, t.k_hi - t.k_lo + 1);
    {
        RowArgs ra = make_row_args(p);
        CK(launch_row_admit(ra, p->d_rt, (int)n_rt, d_stats, 0));
    }
    unsigned char hb[64];
    CK(cudaMemcpy(hb, p->d_row_err, 64, cudaMemcpyDeviceToHost));
    unsigned flags;
    double ferr[2];
    int hs[4];
    memcpy(&flags, hb + 16, 4);
    memcpy(ferr, hb + 24, 16);
    memcpy(hs, hb + 40, 16);
    CK(cudaMemset(p->d_row_err, 0, 64));
    CK(cudaMemcpy(ht.data(), p->d_rt, sizeof(RowTile) * n_rt, cudaMemcpyDeviceToHost));
    // the row path needs the same depth-model tolerance as the deposit tiles' (else: old path)
    // (the fp32 error includes the row kernel's wire travel: non-uniformly stepped scans fail it)
    if ((flags & (FLAG_FIT_NAN | FLAG_MIXED_DIR)) || !(ferr[1] <= MODEL_ERR_MAX) || !(ferr[0] <= ROW_TAU_ERR_MAX))
        return DAXM_OK;
    std::vector<int> lists[daxm_plan::N_RCLS];
    p->stats.row_reject_bits = 0;
    for (size_t q = 0; q < n_rt; ++q) {
        p->stats.row_reject_bits |= ht[q].why;
        for (int b = 0; b < 8; ++b)
            if (ht[q].why & (1 << b)) ++p->stats.row_reject[b];
        if (ht[q].why & RW_WHY_GEN) ++p->stats.row_reject_more;
        const int rb = ht[q].cls & RW_CLS_RB;
        if (ht[q].cls & RW_CLS_RB) ++p->stats.row_kmax_hist[std::min(std::max(ht[q].kmax, 0), 7)];
        const int var = (ht[q].cls & RW_CLS_NB_MID) ? 3 : (ht[q].cls & RW_CLS_NB_WIDE) ? 2 : (ht[q].cls & RW_CLS_GEN) ? 1 : 0;
        const int ktc = (ht[q].cls >> RW_CLS_KT_SHIFT) & 3;
        const int c = 2 * (var + 4 * ktc);
        lists[rb == RW_RB_SMALL ? c : rb == RW_RB_LARGE ? c + 1 : daxm_plan::N_RCLS - 1].push_back((int)q);
    }
    p->h_rlist.clear();
    for (int c = 0; c < daxm_plan::N_RCLS; ++c) {
        p->n_rcls[c] = (int)lists[c].size();
        p->h_rlist.insert(p->h_rlist.end(), lists[c].begin(), lists[c].end());
    }
    CK(cudaMalloc(&p->d_rlist, sizeof(int) * std::max<size_t>(p->h_rlist.size(), 1)));
    CK(cudaMemcpy(p->d_rlist, p->h_rlist.data(), sizeof(int) * p->h_rlist.size(), cudaMemcpyHostToDevice));
    CK(row_set_attributes());
    for (int c = 0; c + 1 < daxm_plan::N_RCLS; ++c) {
        const int var = (c / 2) % 4;
        ((c & 1) ? p->stats.row_tiles_large : p->stats.row_tiles_small) += p->n_rcls[c];
        if (var == 1 || var == 2) p->stats.row_tiles_gen += p->n_rcls[c];
        if (var == 3) p->stats.row_tiles_nb_mid += p->n_rcls[c];
    }
    p->stats.row_tiles_general = p->n_rcls[daxm_plan::N_RCLS - 1];
    p->stats.row_launches = 0;
    for (int c = 0; c < daxm_plan::N_RCLS; ++c) p->stats.row_launches += p->n_rcls[c] > 0;
    p->stats.row_launches += 1;  // row_live_kernel (exact zero-dI skip)
    p->stats.row_ring_need_max = hs[3];
    // one path per plan: the row-segment kernel when it admits every row tile, else the deposit-tile
    // kernels (step-locked, fast, general) of round 1, which cover the overlapping-span regime
    // (both-edges children take the row path with the general kernel for the rest: the deposit-tile
    // kernels neither clamp nor accumulate)
    if (p->n_rcls[daxm_plan::N_RCLS - 1] > 0 && getenv("DAXM_ROW_PARTIAL") == nullptr && !p->is_child) return DAXM_OK;
    p->stats.fit_max_err_bins = std::max(p->stats.fit_max_err_bins, ferr[0]);
    p->stats.fit_model_err_bins = std::max(p->stats.fit_model_err_bins, ferr[1]);
    p->stats.device_bytes += (int64_t)(sizeof(RowTile) * n_rt + n_rt + sizeof(float) * n_rt * NCOEF * (RW_COLS + 1) * RW_ROWS +
                                       sizeof(int) * p->h_rlist.size());
    p->row_ok = true;
    p->stats.row_path = 1;
    if (p->stats.row_launches > 1 && !p->st_cls[0]) {  // class launches fork
        for (cudaStream_t& x : p->st_cls) CK(cudaStreamCreateWithFlags(&x, cudaStreamNonBlocking));
        for (cudaEvent_t& x : p->ev_cls) CK(cudaEventCreateWithFlags(&x, cudaEventDisableTiming));
    }
    return DAXM_OK;
}

daxm_status device_prepass(daxm_plan* p) {
    const daxm_geometry& g = p->g;
    GeomConst& gc = p->gc;
    const int S = g.n_steps;
    const double* W = p->wire.data();
    // ---- tiling (global-aligned)
    p->tr0 = g.row_begin / TILE_R;
    const int tr1 = (g.row_end + TILE_R - 1) / TILE_R;
    p->n_tr = tr1 - p->tr0;
    p->n_tc = (g.n_cols + TILE_C - 1) / TILE_C;
    p->pre_row0 = p->tr0 * TILE_R;
    p->pre_rows = (tr1 * TILE_R < g.n_rows ? tr1 * TILE_R : g.n_rows) - p->pre_row0;
    const size_t n_tiles = (size_t)p->n_tr * p->n_tc;

    // ---- device allocations
    CK(cudaMalloc(&p->d_t, sizeof(double) * S));
    CK(cudaMalloc(&p->d_wire, sizeof(double) * 3 * S));
    CK(cudaMalloc(&p->d_tiles, sizeof(TileInfo) * n_tiles));
    CK(cudaMalloc(&p->d_win, sizeof(int2) * (size_t)p->pre_rows * g.n_cols));
    CK(cudaMalloc(&p->d_pdir, (size_t)p->pre_rows * g.n_cols));
    CK(cudaMalloc(&p->d_psep, (size_t)p->pre_rows * g.n_cols));
    CK(cudaMalloc(&p->d_coef, sizeof(float) * n_tiles * NCOEF * TILE_E * TILE_R));
    unsigned* d_flags = nullptr;
    double* d_err = nullptr;
    unsigned long long* d_cnt = nullptr;
    CK(cudaMalloc(&d_flags, 64));
    d_err = reinterpret_cast<double*>(reinterpret_cast<char*>(d_flags) + 8);
    d_cnt = reinterpret_cast<unsigned long long*>(reinterpret_cast<char*>(d_flags) + 24);
    CK(cudaMemset(d_flags, 0, 64));
    CK(cudaMemcpy(p->d_t, p->t.data(), sizeof(double) * S, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(p->d_wire, W, sizeof(double) * 3 * S, cudaMemcpyHostToDevice));

    cudaEvent_t e0, e1;
    CK(cudaEventCreate(&e0));
    CK(cudaEventCreate(&e1));
    CK(cudaEventRecord(e0, 0));
    {
        const int warps_per_row = (g.n_cols + PW_PIX - 1) / PW_PIX;
        dim3 blk(128, 1), grd((warps_per_row + 3) / 4, p->pre_rows);
        pixel_window_kernel<<<grd, blk>>>(gc, p->d_wire, p->pre_row0, p->pre_rows, g.row_begin, g.row_end,
                                          p->d_win, p->d_pdir, p->d_psep, d_flags, d_cnt);
        CK(cudaGetLastError());
        const int n_states = (p->M + MC - 1) / MC + 1;
        p->n_states = n_states;
        const size_t tsm =
            n_states <= MAX_FAST_CHUNKS ? sizeof(int) * (2 + N_CONSUMER_WARPS) * (size_t)(n_states + 1) : 0;
        if (n_states <= MAX_FAST_CHUNKS)
            CK(cudaMalloc(&p->d_vneed, sizeof(int) * n_tiles * (n_states + 1) * (N_CONSUMER_WARPS + 1)));
        if (tsm > 48 * 1024)
            CK(cudaFuncSetAttribute(tile_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)tsm));
        tile_kernel<<<(unsigned)n_tiles, dim3(TILE_C, TILE_R), tsm>>>(
            gc, p->d_t, p->d_wire, p->pre_row0, p->pre_rows, p->tr0, p->n_tc, g.row_begin, g.row_end, p->d_win,
            p->d_pdir, p->d_psep, p->d_tiles, d_flags, d_cnt, n_states, p->d_vneed);
        CK(cudaGetLastError());
        fit_kernel<<<(unsigned)n_tiles, dim3(TILE_R, 8)>>>(gc, p->d_t, p->d_wire, p->tr0, p->n_tc, p->d_tiles,
                                                          p->d_coef, d_flags, d_err);
        CK(cudaGetLastError());
    }
    CK(cudaEventRecord(e1, 0));
    CK(cudaEventSynchronize(e1));
    float ms = 0.f;
    cudaEventElapsedTime(&ms, e0, e1);
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    unsigned char hb[64];
    CK(cudaMemcpy(hb, d_flags, 64, cudaMemcpyDeviceToHost));
    cudaFree(d_flags);
    unsigned flags;
    double max_err, model_err;
    unsigned long long cnt[5];
    memcpy(&flags, hb, 4);
    memcpy(&max_err, hb + 8, 8);
    memcpy(&model_err, hb + 16, 8);
    memcpy(cnt, hb + 24, 40);

    daxm_plan_stats& st = p->stats;
    st.n_bins = p->M;
    st.rows = p->rows;
    st.cols = g.n_cols;
    st.n_steps = S;
    st.window_pairs = (int64_t)cnt[0];
    st.contrib_pairs = (int64_t)cnt[2];
    st.contrib_pixels = (int64_t)cnt[3];
    st.staged_steps = (int64_t)cnt[1];
    st.n_tiles = (int64_t)n_tiles;
    st.tile_rows = TILE_R;
    st.tile_cols = TILE_C;
    st.fit_max_err_bins = max_err;
    st.fit_model_err_bins = model_err;
    st.prepass_ms = ms;
    st.device_bytes = (int64_t)(sizeof(double) * 4 * S + sizeof(TileInfo) * n_tiles +
                                (sizeof(int2) + 1) * (size_t)p->pre_rows * g.n_cols +
                                sizeof(float) * n_tiles * NCOEF * TILE_E * TILE_R);

    if (flags & (FLAG_NONMONOTONE | FLAG_MIXED_DIR))
        return fail(nullptr, DAXM_ERR_NONMONOTONE_SCAN,
                    "a pixel edge's tangent depth is not monotone in the wire step inside its window (flags 0x%x)", flags);
    if (cnt[4] == 0)
        return fail(nullptr, DAXM_ERR_GEOMETRY,
                    "every pixel is invalid: each pixel edge lies inside the wire cylinder or its tangent plane is "
                    "parallel to the beam at every wire step");
    // depth source: the travel polynomial where it holds its tolerance, else the exact table (also
    // when a pixel's window holds NaN pairs: the table keeps them NaN and the general kernel skips them)
    const bool use_table = !p->straight || (flags & (FLAG_FIT_NAN | FLAG_NAN_IN_WINDOW)) || !(model_err <= MODEL_ERR_MAX) ||
                           !(max_err <= 1e-3) || getenv("DAXM_FORCE_TABLE") != nullptr;
    {
        std::vector<TileInfo> ht(n_tiles);
        CK(cudaMemcpy(ht.data(), p->d_tiles, sizeof(TileInfo) * n_tiles, cudaMemcpyDeviceToHost));
        if (use_table) {
            std::vector<long long> off(n_tiles);
            long long tot = 0;
            for (size_t q = 0; q < n_tiles; ++q) {
                off[q] = tot;
                if (ht[q].k_hi >= ht[q].k_lo) tot += (long long)(ht[q].k_hi - ht[q].k_lo + 1) * TILE_E * TILE_R;
            }
            CK(cudaMalloc(&p->d_toff, sizeof(long long) * n_tiles));
            CK(cudaMemcpy(p->d_toff, off.data(), sizeof(long long) * n_tiles, cudaMemcpyHostToDevice));
            CK(cudaMalloc(&p->d_table, sizeof(float) * (size_t)(tot > 0 ? tot : 1)));
            table_kernel<<<(unsigned)n_tiles, dim3(TILE_R, 8)>>>(gc, p->d_wire, p->tr0, p->n_tc, p->d_tiles,
                                                                p->d_toff, p->d_table);
            CK(cudaGetLastError());
            CK(cudaDeviceSynchronize());
            st.depth_table_bytes = (int64_t)(sizeof(float) * (size_t)tot);
            st.device_bytes += st.depth_table_bytes + (int64_t)(sizeof(long long) * n_tiles);
        }
        std::vector<int> lu, lf;
        for (size_t q = 0; q < n_tiles; ++q) {
            const TileInfo& ti = ht[q];
            if (ti.separated != MODE_SEPARATED) ++st.nonseparated_tiles;
            if (ti.separated == MODE_OVERLAP) ++st.overlap_tiles;
            if (ti.k_hi >= ti.k_lo) st.ring_need_max = std::max<int64_t>(st.ring_need_max, ti.ring_need);
            if (ti.k_hi >= ti.k_lo) p->max_nv = std::max(p->max_nv, ti.k_hi - ti.k_lo + 1);
            // TMA boxes start at the tile's first row; a tile that starts above the band
            // (band start not a multiple of TILE_R) would need a negative coordinate -> general kernel
            const int tile_row0 = (p->tr0 + (int)(q / p->n_tc)) * TILE_R;
            const bool sep = ti.separated != MODE_GENERAL && tile_row0 >= g.row_begin && !use_table;
            if (!(sep && ti.ring_need <= NB_U16)) lu.push_back((int)q);
            if (!(sep && ti.ring_need <= NB_F32)) lf.push_back((int)q);
        }
        p->n_list_u16 = (int)lu.size();
        p->n_list_f32 = (int)lf.size();
        if (!lu.empty()) {
            CK(cudaMalloc(&p->d_list_u16, sizeof(int) * lu.size()));
            CK(cudaMemcpy(p->d_list_u16, lu.data(), sizeof(int) * lu.size(), cudaMemcpyHostToDevice));
        }
        if (!lf.empty()) {
            CK(cudaMalloc(&p->d_list_f32, sizeof(int) * lf.size()));
            CK(cudaMemcpy(p->d_list_f32, lf.data(), sizeof(int) * lf.size(), cudaMemcpyHostToDevice));
        }
        st.general_tiles_u16 = p->n_list_u16;
        st.general_tiles_f32 = p->n_list_f32;
    }
    // ---- step-locked kernel: per tile, replay the walks' edge frontiers in fp32 and admit the
    // tile if its per-warp output ring provably holds them (deposit_lock.cu)
    CK(cudaMalloc(&p->d_lock_err, 32));
    CK(cudaMemset(p->d_lock_err, 0, 32));
    CK(cudaMalloc(&p->d_live, n_tiles * (1 + NG16)));  // tile flags, then 16-row group flags
    if (!use_table) {
        int* d_ls = reinterpret_cast<int*>(p->d_lock_err) + 1;
        DepositArgs a = make_args(p, DAXM_U16);
        CK(launch_lock_prepass(a, (int)n_tiles, d_ls, 0));
        int hs[5];
        CK(cudaMemcpy(hs, d_ls, sizeof hs, cudaMemcpyDeviceToHost));
        p->lock_small = hs[0];
        p->lock_large = hs[1];
        p->lock_rest = hs[2];
        p->lock_ov_small = p->gc.point_mode ? 0 : hs[3];
        p->lock_ov_large = p->gc.point_mode ? 0 : hs[4];
        st.lock_tiles_small = hs[0];
        st.lock_tiles_large = hs[1];
        st.lock_tiles_overlap = p->lock_ov_small + p->lock_ov_large;
        // several tile classes: their launches run concurrently on forked streams
        const int ncls = (p->lock_small > 0) + (p->lock_large > 0) + (p->lock_ov_small > 0) + (p->lock_ov_large > 0);
        if (ncls >= 2) {
            for (cudaStream_t& x : p->st_cls) CK(cudaStreamCreateWithFlags(&x, cudaStreamNonBlocking));
            for (cudaEvent_t& x : p->ev_cls) CK(cudaEventCreateWithFlags(&x, cudaEventDisableTiming));
        }
    }
    if (!use_table) {
        daxm_status rs = row_prepass(p, 0);
        if (rs != DAXM_OK) return rs;
    }
    return DAXM_OK;
}

}  // namespace

extern "C" {

int daxm_abi_version(void) { return DAXM_ABI_VERSION; }

const char* daxm_status_string(daxm_status s) {
    switch (s) {
        case DAXM_OK: return "ok";
        case DAXM_ERR_INVALID_ARGUMENT: return "invalid argument";
        case DAXM_ERR_NONMONOTONE_SCAN: return "non-monotone scan";
        case DAXM_ERR_GEOMETRY: return "geometry error";
        case DAXM_ERR_OUT_OF_MEMORY: return "out of memory";
        case DAXM_ERR_CUDA: return "CUDA error";
    }
    return "unknown status";
}

const char* daxm_create_error(void) { return g_create_err.c_str(); }

const char* daxm_last_error(const daxm_plan* p) { return p ? p->err.c_str() : ""; }

static daxm_status create_one(const daxm_geometry* g, int cuda_device, bool child, daxm_plan** out);
static daxm_status create_both(const daxm_geometry* g, int cuda_device, daxm_plan** out);

daxm_status daxm_create(const daxm_geometry* g, int cuda_device, daxm_plan** out) {
    g_create_err.clear();
    if (!out) return fail(nullptr, DAXM_ERR_INVALID_ARGUMENT, "out is NULL");
    *out = nullptr;
    if (!g) return fail(nullptr, DAXM_ERR_INVALID_ARGUMENT, "geometry is NULL");
    if (g->n_steps < 2) return fail(nullptr, DAXM_ERR_INVALID_ARGUMENT, "n_steps = %d < 2", g->n_steps);
    if (g->n_rows < 1 || g->n_cols < 1)
        return fail(nullptr, DAXM_ERR_INVALID_ARGUMENT, "detector %d x %d", g->n_rows, g->n_cols);
    if (g->row_begin < 0 || g->row_end > g->n_rows || g->row_begin >= g->row_end)
        return fail(nullptr, DAXM_ERR_INVALID_ARGUMENT, "row band [%d, %d) outside [0, %d)", g->row_begin, g->row_end,
                    g->n_rows);
    if (!g->wire_xyz) return fail(nullptr, DAXM_ERR_INVALID_ARGUMENT, "wire_xyz is NULL");
    if (!(isfinite(g->pitch_col) && g->pitch_col > 0 && isfinite(g->pitch_row) && g->pitch_row > 0))
        return fail(nullptr, DAXM_ERR_INVALID_ARGUMENT, "pixel pitch must be finite and > 0");
    if (!finite3(g->det_rot) || !finite3(g->det_trans) || !finite3(g->beam_dir) || !finite3(g->beam_origin) ||
        !finite3(g->wire_axis))
        return fail(nullptr, DAXM_ERR_INVALID_ARGUMENT, "non-finite geometry vector");
    if (!(norm3(g->beam_dir) > 0) || !(norm3(g->wire_axis) > 0))
        return fail(nullptr, DAXM_ERR_INVALID_ARGUMENT, "zero-length beam or wire-axis vector");
    if (!(isfinite(g->wire_radius) && g->wire_radius > 0))
        return fail(nullptr, DAXM_ERR_INVALID_ARGUMENT, "wire radius must be finite and > 0");
    if (!(isfinite(g->depth_start) && isfinite(g->depth_end) && isfinite(g->depth_res) && g->depth_res > 0 &&
          g->depth_end >= g->depth_start))
        return fail(nullptr, DAXM_ERR_INVALID_ARGUMENT, "depth range/resolution invalid");
    const double nb = (g->depth_end - g->depth_start) / g->depth_res;
    if (fabs(nb - nearbyint(nb)) > 1e-6 || nb > 1e7)
        return fail(nullptr, DAXM_ERR_INVALID_ARGUMENT, "(depth_end - depth_start)/depth_res = %.9g is not an integer",
                    nb);
    if (g->edge != DAXM_EDGE_LEADING && g->edge != DAXM_EDGE_TRAILING && g->edge != DAXM_EDGE_BOTH)
        return fail(nullptr, DAXM_ERR_INVALID_ARGUMENT, "unknown edge %d", g->edge);
    if (g->pixel_model != DAXM_PIXEL_FINITE && g->pixel_model != DAXM_PIXEL_POINT)
        return fail(nullptr, DAXM_ERR_INVALID_ARGUMENT, "unknown pixel model %d", g->pixel_model);
    for (int k = 0; k < 3 * g->n_steps; ++k)
        if (!isfinite(g->wire_xyz[k])) return fail(nullptr, DAXM_ERR_INVALID_ARGUMENT, "non-finite wire position");
    {
        const double* a = g->wire_axis;
        const double* b = g->beam_dir;
        double c[3] = {a[1] * b[2] - a[2] * b[1], a[2] * b[0] - a[0] * b[2], a[0] * b[1] - a[1] * b[0]};
        if (norm3(c) < 1e-9 * norm3(a) * norm3(b))
            return fail(nullptr, DAXM_ERR_INVALID_ARGUMENT, "beam is parallel to the wire axis");
    }
    if (g->edge == DAXM_EDGE_BOTH) return create_both(g, cuda_device, out);
    return create_one(g, cuda_device, false, out);
}

// After daxm_create's validation: one plan (one edge).
static daxm_status create_one(const daxm_geometry* g, int cuda_device, bool child, daxm_plan** out) {
    daxm_plan* p = new (std::nothrow) daxm_plan();
    if (!p) return fail(nullptr, DAXM_ERR_OUT_OF_MEMORY, "host allocation failed");
    p->is_child = child;
    p->device = cuda_device;
    p->g = *g;
    p->wire.assign(g->wire_xyz, g->wire_xyz + 3 * (size_t)g->n_steps);
    p->g.wire_xyz = nullptr;
    p->M = (int)nearbyint((g->depth_end - g->depth_start) / g->depth_res) + 1;
    p->rows = g->row_end - g->row_begin;
    p->C = g->n_cols;
    p->S = g->n_steps;
    daxm_status s = host_prepare(p);  // scan line checks need no device
    if (s == DAXM_OK) {
        int n_dev = 0;
        if (cudaGetDeviceCount(&n_dev) != cudaSuccess || cuda_device < 0 || cuda_device >= n_dev) {
            cudaGetLastError();
            s = fail(nullptr, DAXM_ERR_CUDA, "CUDA device %d not available (%d devices)", cuda_device, n_dev);
        } else {
            DeviceGuard guard(cuda_device);
            s = device_prepass(p);
            if (s != DAXM_OK) free_plan_memory(p);
        }
    }
    if (s != DAXM_OK) {
        delete p;
        return s;
    }
    *out = p;
    return DAXM_OK;
}

// Both-edges mode (reading R16): one child plan per edge, same geometry; the leading child stores
// the reconstruction of the intensity decreases, the trailing child adds that of the increases.
static daxm_status create_both(const daxm_geometry* g, int cuda_device, daxm_plan** out) {
    daxm_plan* p = new (std::nothrow) daxm_plan();
    if (!p) return fail(nullptr, DAXM_ERR_OUT_OF_MEMORY, "host allocation failed");
    p->device = cuda_device;
    p->g = *g;
    p->g.wire_xyz = nullptr;
    for (int e = 0; e < 2; ++e) {
        daxm_geometry ge = *g;
        ge.edge = e == 0 ? DAXM_EDGE_LEADING : DAXM_EDGE_TRAILING;
        daxm_status s = create_one(&ge, cuda_device, true, &p->child[e]);
        if (s != DAXM_OK) {
            daxm_destroy(p);
            return s;
        }
        p->child[e]->dI_floor = 0.f;
        p->child[e]->acc = e;
    }
    const daxm_plan* c = p->child[0];
    p->M = c->M;
    p->rows = c->rows;
    p->C = c->C;
    p->S = c->S;
    p->tr0 = c->tr0;
    p->n_tr = c->n_tr;
    p->n_tc = c->n_tc;
    *out = p;
    return DAXM_OK;
}

daxm_status daxm_plan_info(const daxm_plan* p, int64_t* n_bins, int64_t* rows, int64_t* cols) {
    if (!p) return DAXM_ERR_INVALID_ARGUMENT;
    if (n_bins) *n_bins = p->M;
    if (rows) *rows = p->rows;
    if (cols) *cols = p->C;
    return DAXM_OK;
}

daxm_status daxm_plan_stats_get(const daxm_plan* p, daxm_plan_stats* st) {
    if (!p || !st) return DAXM_ERR_INVALID_ARGUMENT;
    if (p->child[0]) {  // both-edges mode: the leading child's numbers, sums of the per-plan counts
        daxm_plan_stats b;
        daxm_status s = daxm_plan_stats_get(p->child[0], st);
        if (s == DAXM_OK) s = daxm_plan_stats_get(p->child[1], &b);
        if (s != DAXM_OK) return s;
        st->contrib_pairs += b.contrib_pairs;
        st->contrib_pixels += b.contrib_pixels;
        st->window_pairs += b.window_pairs;
        st->general_tiles_u16 += b.general_tiles_u16;
        st->general_tiles_f32 += b.general_tiles_f32;
        st->prepass_ms += b.prepass_ms;
        st->device_bytes += b.device_bytes;
        st->lock_ring_violations += b.lock_ring_violations;
        st->row_tiles_small += b.row_tiles_small;
        st->row_tiles_large += b.row_tiles_large;
        st->row_tiles_general += b.row_tiles_general;
        st->row_tiles_gen += b.row_tiles_gen;
        st->row_launches += b.row_launches;
        st->row_path = st->row_path && b.row_path;
        st->fit_max_err_bins = std::max(st->fit_max_err_bins, b.fit_max_err_bins);
        st->fit_model_err_bins = std::max(st->fit_model_err_bins, b.fit_model_err_bins);
        return DAXM_OK;
    }
    *st = p->stats;
    st->row_path = p->row_ok && getenv("DAXM_NO_ROW") == nullptr ? 1 : 0;
    if (p->d_lock_err) {  // synchronous read of the step-locked kernel's violation counter
        DeviceGuard guard(p->device);
        unsigned v = 0;
        if (cudaMemcpy(&v, p->d_lock_err, sizeof v, cudaMemcpyDeviceToHost) != cudaSuccess) {
            cudaGetLastError();
            return DAXM_ERR_CUDA;
        }
        st->lock_ring_violations = v;
    }
    if (p->d_row_err) {  // row-segment kernel schedule violations (DAXM_ROW_CHECK builds)
        DeviceGuard guard(p->device);
        unsigned v = 0;
        if (cudaMemcpy(&v, p->d_row_err, sizeof v, cudaMemcpyDeviceToHost) != cudaSuccess) {
            cudaGetLastError();
            return DAXM_ERR_CUDA;
        }
        st->lock_ring_violations += v;
    }
    return DAXM_OK;
}

}  // extern "C"

static DepositArgs make_args(const daxm_plan* p, int dtype) {
    DepositArgs a;
    a.tile_list = dtype == DAXM_U16 ? p->d_list_u16 : p->d_list_f32;
    a.n_list = dtype == DAXM_U16 ? p->n_list_u16 : p->n_list_f32;
    a.nb = dtype == DAXM_U16 ? NB_U16 : NB_F32;
    a.has_overlap = p->stats.overlap_tiles > 0;
    a.max_nv = p->max_nv;
    a.vneed = p->d_vneed;
    a.n_states = p->n_states;
    a.t = p->d_t;
    a.tiles = p->d_tiles;
    a.win = p->d_win;
    a.coef = p->d_coef;
    a.R = p->g.n_rows;
    a.C = p->C;
    a.S = p->S;
    a.M = p->M;
    a.row_begin = p->g.row_begin;
    a.row_end = p->g.row_end;
    a.pre_row0 = p->pre_row0;
    a.tr0 = p->tr0;
    a.n_tr = p->n_tr;
    a.n_tc = p->n_tc;
    a.tr_begin = 0;
    a.tr_end = p->n_tr;
    a.m_ref = p->gc.m_ref;
    a.point_mode = p->gc.point_mode;
    a.sign = p->g.edge == DAXM_EDGE_TRAILING ? -1.f : 1.f;
    a.dI_floor = p->dI_floor;
    a.acc = p->acc;
    a.w = p->d_w;
    a.stack = nullptr;
    a.table = p->d_table;
    a.toff = p->d_toff;
    a.use_cutoff = p->use_cutoff;
    a.cutoff = p->cutoff;
    a.tile_live = nullptr;
    a.grp_live = nullptr;
    a.lock_enabled = (p->lock_small + p->lock_large + p->lock_ov_small + p->lock_ov_large) > 0 &&
                     getenv("DAXM_NO_LOCK") == nullptr;
    a.lock_small = p->lock_small;
    a.lock_large = p->lock_large;
    a.lock_ov_small = p->lock_ov_small;
    a.lock_ov_large = p->lock_ov_large;
    a.lock_ov_enabled = getenv("DAXM_NO_LOCK_OV") == nullptr;
    a.lock_rest = a.lock_enabled ? p->lock_rest : 1;
    a.lock_err = p->d_lock_err;
    return a;
}

static RowArgs make_row_args(const daxm_plan* p) {
    RowArgs a;
    a.t = p->d_t;
    a.rt = p->d_rt;
    a.win = p->d_win;
    a.coef = p->d_rcoef;
    a.list = nullptr;
    a.n_list = 0;
    a.R = p->g.n_rows;
    a.C = p->C;
    a.S = p->S;
    a.M = p->M;
    a.m_ref = p->gc.m_ref;
    a.row_begin = p->g.row_begin;
    a.row_end = p->g.row_end;
    a.pre_row0 = p->pre_row0;
    a.row_org = p->row_org;
    a.n_rc = p->n_rc;
    a.max_nv = p->max_nv_row;
    a.point_mode = p->gc.point_mode;
    a.sign = p->g.edge == DAXM_EDGE_TRAILING ? -1.f : 1.f;
    a.dI_floor = p->dI_floor;
    a.acc = p->acc;
    a.stack = nullptr;
    a.out = nullptr;
    a.dth = p->dt_h;
    a.dtl = p->dt_l;
    a.use_cutoff = p->use_cutoff;
    a.cutoff = p->cutoff;
    a.live = nullptr;
    a.prof_part = nullptr;
    a.err = p->d_row_err;
    return a;
}

extern "C" {

static PFN_cuTensorMapEncodeTiled_v12000 tensor_map_encoder() {
    static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
    static bool tried = false;
    if (!tried) {
        tried = true;
        cudaDriverEntryPointQueryResult q;
        void* f = nullptr;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(f);
        cudaGetLastError();
    }
    return fn;
}

// The fast kernel needs TMA-describable buffers: row pitch a multiple of 16 bytes.
static bool fast_possible(const daxm_plan* p, int dt) {
    const int es = dt == DAXM_U16 ? 2 : 4;
    return p->d_table == nullptr && (p->C * es) % 16 == 0 && (p->C * 4) % 16 == 0 && p->max_nv <= MAX_FAST_NV &&
           p->d_vneed != nullptr &&
           getenv("DAXM_FORCE_GENERAL") == nullptr && tensor_map_encoder() != nullptr;
}

static daxm_status encode_maps(daxm_plan* p, const void* d_stack, int dt, float* d_out) {
    if (p->map_stack == d_stack && p->map_out == d_out && p->map_dtype == dt) return DAXM_OK;
    auto enc = tensor_map_encoder();
    const cuuint64_t es = dt == DAXM_U16 ? 2 : 4;
    const cuuint64_t C = (cuuint64_t)p->C, R = (cuuint64_t)p->rows;
    {
        cuuint64_t dims[3] = {C, R, (cuuint64_t)p->S};
        cuuint64_t strides[2] = {C * es, C * R * es};
        cuuint32_t box[3] = {(cuuint32_t)TILE_C, (cuuint32_t)TILE_R, 1};
        cuuint32_t estr[3] = {1, 1, 1};
        CUresult r = enc(&p->in_map, dt == DAXM_U16 ? CU_TENSOR_MAP_DATA_TYPE_UINT16 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32,
                         3, const_cast<void*>(d_stack), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                         CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
                         CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        if (r != CUDA_SUCCESS) return fail(p, DAXM_ERR_CUDA, "cuTensorMapEncodeTiled(stack) failed: %d", (int)r);
    }
    {
        cuuint64_t dims[3] = {C, R, (cuuint64_t)p->M};
        cuuint64_t strides[2] = {C * 4, C * R * 4};
        cuuint32_t box[3] = {(cuuint32_t)TILE_C, 32u, (cuuint32_t)MC};  // one warp pair's rows
        cuuint32_t estr[3] = {1, 1, 1};
        CUresult r = enc(&p->out_map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, d_out, dims, strides, box, estr,
                         CU_TENSOR_MAP_INTERLEAVE_NONE, TILE_C == 16 ? CU_TENSOR_MAP_SWIZZLE_64B : CU_TENSOR_MAP_SWIZZLE_32B,
                         CU_TENSOR_MAP_L2_PROMOTION_NONE,
                         CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        if (r != CUDA_SUCCESS) return fail(p, DAXM_ERR_CUDA, "cuTensorMapEncodeTiled(out) failed: %d", (int)r);
    }
    {   // step-locked kernel: one warp's [16 rows][8 cols] block of LOCK_G consecutive wire steps
        cuuint64_t dims[3] = {C, R, (cuuint64_t)p->S};
        cuuint64_t strides[2] = {C * es, C * R * es};
        cuuint32_t box[3] = {(cuuint32_t)TILE_C, (cuuint32_t)LOCK_ROWS, (cuuint32_t)LOCK_G};
        cuuint32_t estr[3] = {1, 1, 1};
        CUresult r = enc(&p->lock_in_map, dt == DAXM_U16 ? CU_TENSOR_MAP_DATA_TYPE_UINT16 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32,
                         3, const_cast<void*>(d_stack), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                         CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
                         CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        if (r != CUDA_SUCCESS) return fail(p, DAXM_ERR_CUDA, "cuTensorMapEncodeTiled(lock stack) failed: %d", (int)r);
    }
    if (p->row_ok) {  // row-segment kernel: [RW_G steps][RW_ROWS][RW_COLS] loads, [RW_PB planes][...] stores
        cuuint64_t dims[3] = {C, R, (cuuint64_t)p->S};
        cuuint64_t strides[2] = {C * es, C * R * es};
        cuuint32_t box[3] = {32u, (cuuint32_t)RW_ROWS, (cuuint32_t)RW_G};  // one column half
        cuuint32_t estr[3] = {1, 1, 1};
        CUresult r = enc(&p->row_in_map, dt == DAXM_U16 ? CU_TENSOR_MAP_DATA_TYPE_UINT16 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32,
                         3, const_cast<void*>(d_stack), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                         CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
                         CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        if (r != CUDA_SUCCESS) return fail(p, DAXM_ERR_CUDA, "cuTensorMapEncodeTiled(row stack) failed: %d", (int)r);
        cuuint64_t odims[3] = {C, R, (cuuint64_t)p->M};
        cuuint64_t ostrides[2] = {C * 4, C * R * 4};
        cuuint32_t obox[3] = {(cuuint32_t)RW_COLS, (cuuint32_t)RW_ROWS, (cuuint32_t)RW_PB};
        r = enc(&p->row_out_map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, d_out, odims, ostrides, obox, estr,
                CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE,
                CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        if (r != CUDA_SUCCESS) return fail(p, DAXM_ERR_CUDA, "cuTensorMapEncodeTiled(row out) failed: %d", (int)r);
    }
    p->map_stack = d_stack;
    p->map_out = d_out;
    p->map_dtype = dt;
    return DAXM_OK;
}

// Row-segment path: one launch per admission class (ring of 16 / 32 planes) plus the general kernel
// for the row tiles not admitted, forked onto the plan's class streams and joined back into st.
// g0 / g1 (global rows of a host-pipeline band, g1 < 0: all) select the row tiles of those rows.
static daxm_status run_row(daxm_plan* p, const void* d_stack, int dt, float* d_out, cudaStream_t st, int g0,
                           int g1, double* d_profile = nullptr) {
    daxm_status s = encode_maps(p, d_stack, dt, d_out);
    if (s != DAXM_OK) return s;
    int ra = 0, rb = p->n_rr;
    if (g1 >= 0) {  // global rows [g0, g1) of a host-pipeline band
        // a row tile straddling a band boundary (odd band start) goes with the later band, whose rows
        // are copied after the earlier band's
        ra = g0 <= p->row_org ? 0 : (g0 - p->row_org) / RW_ROWS;
        rb = g1 >= p->g.row_end ? p->n_rr : std::max(0, (g1 - p->row_org) / RW_ROWS);
    }
    constexpr int NC = daxm_plan::N_RCLS;
    int seg[NC][2], n_launch = 0, off = 0;
    for (int c = 0; c < NC; ++c) {
        const int* b0 = p->h_rlist.data() + off;
        const int* b1 = b0 + p->n_rcls[c];
        seg[c][0] = (int)(std::lower_bound(b0, b1, ra * p->n_rc) - p->h_rlist.data());
        seg[c][1] = (int)(std::lower_bound(b0, b1, rb * p->n_rc) - p->h_rlist.data());
        n_launch += seg[c][1] > seg[c][0];
        off += p->n_rcls[c];
    }
    RowArgs a = make_row_args(p);
    a.stack = d_stack;
    a.out = d_out;
    a.prof_part = d_profile ? p->d_prof_part : nullptr;
    if (getenv("DAXM_NO_ZERO_SKIP") == nullptr) {  // exact zero-dI skip, before the class launches fork
        cudaError_t z = launch_row_live(a, ra * p->n_rc, (rb - ra) * p->n_rc, p->d_rlive, dt, st);
        if (z != cudaSuccess) {
            cudaGetLastError();
            return fail(p, DAXM_ERR_CUDA, "row live launch: %s", cudaGetErrorString(z));
        }
        a.live = p->d_rlive;
    }
    // every class launch on its own stream (up to N_FORK + 1): they run concurrently, so no launch
    // waits for another's tail; forked from st and joined back into it (graph-capturable)
    const int nfork = n_launch >= 2 && p->st_cls[0] != nullptr && getenv("DAXM_NO_FORK") == nullptr
                          ? std::min(n_launch - 1, (int)daxm_plan::N_FORK) : 0;
    cudaStream_t sts[daxm_plan::N_FORK + 1];
    sts[0] = st;
    for (int i = 0; i < daxm_plan::N_FORK; ++i) sts[1 + i] = i < nfork ? p->st_cls[i] : st;
    cudaError_t e = cudaSuccess;
    if (nfork) {
        e = cudaEventRecord(p->ev_cls[0], st);
        for (int i = 0; i < nfork && e == cudaSuccess; ++i) e = cudaStreamWaitEvent(p->st_cls[i], p->ev_cls[0], 0);
    }
    int li = 0;
    for (int c = 0; c < NC - 1 && e == cudaSuccess; ++c) {
        a.list = p->d_rlist + seg[c][0];
        a.n_list = seg[c][1] - seg[c][0];
        if (a.n_list <= 0) continue;
        e = launch_row(a, &p->row_in_map, &p->row_out_map, dt, (c & 1) == 0 ? RW_RB_SMALL : RW_RB_LARGE, (c / 2) % 4, c / 8,
                       sts[li++ % (nfork + 1)]);
    }
    if (e == cudaSuccess && seg[NC - 1][1] > seg[NC - 1][0]) {
        DepositArgs ga = make_args(p, dt);
        ga.stack = d_stack;
        e = launch_general_rows(ga, p->d_rlist + seg[NC - 1][0], seg[NC - 1][1] - seg[NC - 1][0], p->n_rc, p->row_org,
                                d_stack, dt, d_out, sts[li++ % (nfork + 1)]);
    }
    // join even after a failed launch, so a capture or the caller's stream stays consistent
    for (int i = 0; i < nfork; ++i) {
        cudaError_t j = cudaEventRecord(p->ev_cls[1 + i], p->st_cls[i]);
        if (j == cudaSuccess) j = cudaStreamWaitEvent(st, p->ev_cls[1 + i], 0);
        if (e == cudaSuccess) e = j;
    }
    if (e == cudaSuccess && d_profile) e = launch_profile_reduce(p->d_prof_part, ra * p->n_rc, (rb - ra) * p->n_rc, p->M,
                                                                d_profile, st);
    if (e != cudaSuccess) {
        cudaGetLastError();
        return fail(p, DAXM_ERR_CUDA, "row deposit launch: %s", cudaGetErrorString(e));
    }
    return DAXM_OK;
}

// Whether daxm_reconstruct runs the row kernel for this plan (both-edges: both children do).
static bool uses_row_path(const daxm_plan* p, int dt) {
    if (p->child[0]) return uses_row_path(p->child[0], dt) && uses_row_path(p->child[1], dt);
    return fast_possible(p, dt) && p->d_w == nullptr && p->row_ok && getenv("DAXM_NO_ROW") == nullptr;
}

// Band [g0, g1) of global rows (g1 < 0: the whole plan); the deposit-tile path needs band bounds
// on multiples of TILE_R (or the plan's ends), the row path on multiples of RW_ROWS.
static daxm_status run_deposit(daxm_plan* p, const void* d_stack, int dt, float* d_out, cudaStream_t st,
                               int g0 = 0, int g1 = -1) {
    if (p->child[0]) {  // both-edges mode: the leading child stores, the trailing child adds
        for (int e = 0; e < 2; ++e) {
            daxm_status s = run_deposit(p->child[e], d_stack, dt, d_out, st, g0, g1);
            if (s != DAXM_OK) {
                p->err = p->child[e]->err;
                return s;
            }
        }
        return DAXM_OK;
    }
    // (per-step weights: the general kernel normalises each intensity, the fast kernels do not)
    bool fast = fast_possible(p, dt) && p->d_w == nullptr;
    if (fast && p->row_ok && getenv("DAXM_NO_ROW") == nullptr)
        return run_row(p, d_stack, dt, d_out, st, g0, g1);
    // both-edges children off the row path: the general kernel alone clamps and accumulates
    if (p->is_child) fast = false;
    if (fast) {
        daxm_status s = encode_maps(p, d_stack, dt, d_out);
        if (s != DAXM_OK) return s;
    }
    DepositArgs a = make_args(p, dt);
    a.tr_begin = g1 < 0 ? 0 : std::max(0, g0 / TILE_R - p->tr0);
    a.tr_end = g1 < 0 ? p->n_tr : std::min(p->n_tr, (g1 + TILE_R - 1) / TILE_R - p->tr0);
    a.stack = d_stack;
    cudaError_t e = cudaSuccess;
    const bool live = a.use_cutoff && !p->is_child && getenv("DAXM_NO_TILE_LIVE") == nullptr;
    if (live) {  // dead tiles: flags here; their zero fill after the fork, beside the class launches
        e = launch_cutoff_tiles(a, d_stack, dt, d_out, p->d_live, 0, st);
        if (e != cudaSuccess) {
            cudaGetLastError();
            return fail(p, DAXM_ERR_CUDA, "cutoff tile launch: %s", cudaGetErrorString(e));
        }
        a.tile_live = p->d_live;
        if (getenv("DAXM_NO_GRP_LIVE") == nullptr) a.grp_live = p->d_live + (size_t)p->n_tr * p->n_tc;
    }
    // fork: class launches on {st, st_cls[0], st_cls[1]}, joined back into st (graph-capturable)
    const bool fork = fast && a.lock_enabled && p->st_cls[0] != nullptr && getenv("DAXM_NO_FORK") == nullptr;
    cudaStream_t sts[3] = {st, p->st_cls[0], p->st_cls[1]};
    if (fork) {
        e = cudaEventRecord(p->ev_cls[0], st);
        for (int i = 0; i < 2 && e == cudaSuccess; ++i) e = cudaStreamWaitEvent(p->st_cls[i], p->ev_cls[0], 0);
    }
    if (live && e == cudaSuccess) e = launch_cutoff_tiles(a, d_stack, dt, d_out, p->d_live, 1, st);
    if (e == cudaSuccess)
        e = launch_deposit(a, &p->in_map, &p->out_map, d_stack, dt, d_out, fast, st, &p->lock_in_map, sts,
                           fork ? 3 : 1);
    if (fork) {  // join even after a failed launch, so a capture or the caller's stream stays consistent
        for (int i = 0; i < 2; ++i) {
            cudaError_t j = cudaEventRecord(p->ev_cls[1 + i], p->st_cls[i]);
            if (j == cudaSuccess) j = cudaStreamWaitEvent(st, p->ev_cls[1 + i], 0);
            if (e == cudaSuccess) e = j;
        }
    }
    if (e != cudaSuccess) {
        cudaGetLastError();
        return fail(p, DAXM_ERR_CUDA, "deposit launch: %s", cudaGetErrorString(e));
    }
    return DAXM_OK;
}

daxm_status daxm_reconstruct(daxm_plan* p, const void* d_stack, daxm_dtype dt, float* d_out, void* cuda_stream) {
    if (!p) return DAXM_ERR_INVALID_ARGUMENT;
    p->err.clear();
    if (!d_stack || !d_out) return fail(p, DAXM_ERR_INVALID_ARGUMENT, "NULL stack or output pointer");
    if (dt != DAXM_U16 && dt != DAXM_F32) return fail(p, DAXM_ERR_INVALID_ARGUMENT, "unknown dtype %d", (int)dt);
    if ((reinterpret_cast<uintptr_t>(d_stack) | reinterpret_cast<uintptr_t>(d_out)) & 15)
        return fail(p, DAXM_ERR_INVALID_ARGUMENT, "stack and output must be 16-byte aligned");
    DeviceGuard guard(p->device);
    return run_deposit(p, d_stack, (int)dt, d_out, (cudaStream_t)cuda_stream);
}

daxm_status daxm_reconstruct_profile(daxm_plan* p, const void* d_stack, daxm_dtype dt, float* d_out, double* d_profile,
                                     void* cuda_stream) {
    if (!p) return DAXM_ERR_INVALID_ARGUMENT;
    p->err.clear();
    if (!d_stack || !d_out || !d_profile) return fail(p, DAXM_ERR_INVALID_ARGUMENT, "NULL stack, output or profile");
    if (dt != DAXM_U16 && dt != DAXM_F32) return fail(p, DAXM_ERR_INVALID_ARGUMENT, "unknown dtype %d", (int)dt);
    if ((reinterpret_cast<uintptr_t>(d_stack) | reinterpret_cast<uintptr_t>(d_out)) & 15)
        return fail(p, DAXM_ERR_INVALID_ARGUMENT, "stack and output must be 16-byte aligned");
    DeviceGuard guard(p->device);
    cudaStream_t st = (cudaStream_t)cuda_stream;
    // fused: every row tile in the row kernel (its epilogue sums each final plane per tile)
    const bool fused = !p->child[0] && p->row_ok && p->n_rcls[daxm_plan::N_RCLS - 1] == 0 &&
                       fast_possible(p, (int)dt) && getenv("DAXM_NO_ROW") == nullptr &&
                       getenv("DAXM_NO_FUSED_PROFILE") == nullptr;
    if (fused) {
        if (!p->d_prof_part) {
            const size_t n = (size_t)p->n_rr * p->n_rc * p->M;
            if (cudaMalloc(&p->d_prof_part, n * sizeof(float)) != cudaSuccess) {
                cudaGetLastError();
                return fail(p, DAXM_ERR_OUT_OF_MEMORY, "profile partial sums (%zu floats)", n);
            }
            p->stats.device_bytes += (int64_t)(n * sizeof(float));
        }
        return run_row(p, d_stack, (int)dt, d_out, st, 0, -1, d_profile);
    }
    daxm_status s = run_deposit(p, d_stack, (int)dt, d_out, st);
    if (s != DAXM_OK) return s;
    cudaError_t e = launch_depth_profile(d_out, p->M, (size_t)p->rows * p->C, d_profile, st);
    if (e != cudaSuccess) {
        cudaGetLastError();
        return fail(p, DAXM_ERR_CUDA, "depth profile launch: %s", cudaGetErrorString(e));
    }
    return DAXM_OK;
}

// Out-of-core host path (the paper's row chunking, P:L182-215 / Fig. 2, and
// its host<->device transfer stage): bands of B rows (B a multiple of TILE_R, band edges
// at global multiples of B, so every band plan's tiles are the whole plan's), one plan per band
// (built on first use), a two-slot device ring.  Band b (slot s = b & 1):
//   st_in : [wait: band b-2's deposit released in[s]]  H2D rows -> in[s]        record in-done
//   st    : [wait: in-done, band b-2's D2H released out[s]]  deposit in[s] -> out[s]  record dep-done
//   st_out: [wait: dep-done]  D2H out[s] -> host rows                          record out-done
// so H2D of band b + 1, the deposit of band b and the D2H of band b - 1 overlap.
static daxm_status host_ring(daxm_plan* p, const void* h_stack, daxm_dtype dt, float* h_out, cudaStream_t st) {
    const size_t es = dt == DAXM_U16 ? 2 : 4;
    const size_t row_in = (size_t)p->C * es, row_out = (size_t)p->C * sizeof(float);
    const size_t per_row = row_in * p->S + row_out * p->M;  // one detector row of one slot
    const uint64_t rows_fit = p->host_budget / (2 * per_row);
    // the largest band whose two slots fit, but at most 1/16 of the rows (a deeper pipeline: the first
    // band's copy in and the last one's copy out are not overlapped)
    const uint64_t b_pipe = std::max<uint64_t>(1, (uint64_t)p->rows / (16 * TILE_R));
    const int B = (int)std::min<uint64_t>(std::min<uint64_t>(rows_fit / TILE_R, b_pipe),
                                          (uint64_t)(p->g.n_rows / TILE_R + 1)) * TILE_R;
    if (rows_fit < (uint64_t)TILE_R)
        return fail(p, DAXM_ERR_OUT_OF_MEMORY,
                    "host budget %llu bytes holds no two %d-row ring slots (%zu bytes per row and slot)",
                    (unsigned long long)p->host_budget, TILE_R, per_row);
    cudaError_t e = cudaSuccess;
    if (p->ring_rows != B) {  // (re)build the band plans and the ring for this band height
        free_ring(p);
        const daxm_plan* src = p->child[0] ? p->child[0] : p;
        daxm_geometry ge = p->g;
        ge.wire_xyz = src->wire.data();
        for (int r = p->g.row_begin; r < p->g.row_end;) {
            const int r1 = std::min(p->g.row_end, (r / B + 1) * B);
            ge.row_begin = r;
            ge.row_end = r1;
            daxm_plan* bp = nullptr;
            daxm_status s = ge.edge == DAXM_EDGE_BOTH ? create_both(&ge, p->device, &bp)
                                                      : create_one(&ge, p->device, false, &bp);
            if (s != DAXM_OK) {
                free_ring(p);
                return fail(p, s, "band plan [%d, %d): %s", r, r1, g_create_err.c_str());
            }
            if (!p->step_w.empty()) daxm_set_step_weights(bp, p->step_w.data());
            p->bands.push_back(bp);
            p->band_r0.push_back(r - p->g.row_begin);
            r = r1;
        }
        p->band_r0.push_back(p->rows);
        for (cudaEvent_t& ev : p->ev_ring)
            if ((e = cudaEventCreateWithFlags(&ev, cudaEventDisableTiming)) != cudaSuccess) break;
        p->ring_rows = B;
    }
    int bmax = 0;
    for (size_t b = 0; b + 1 < p->band_r0.size(); ++b) bmax = std::max(bmax, p->band_r0[b + 1] - p->band_r0[b]);
    const size_t in_b = row_in * p->S * bmax, out_b = row_out * p->M * bmax;
    if (e == cudaSuccess && (p->ring_in_bytes < in_b || p->ring_out_bytes < out_b)) {
        for (int i = 0; i < 2; ++i) {
            cudaFree(p->d_ring_in[i]);
            cudaFree(p->d_ring_out[i]);
            p->d_ring_in[i] = nullptr;
            p->d_ring_out[i] = nullptr;
        }
        p->ring_in_bytes = p->ring_out_bytes = 0;
        for (int i = 0; i < 2 && e == cudaSuccess; ++i) {
            e = cudaMalloc(&p->d_ring_in[i], in_b);
            if (e == cudaSuccess) e = cudaMalloc(reinterpret_cast<void**>(&p->d_ring_out[i]), out_b);
        }
        if (e == cudaSuccess) {
            p->ring_in_bytes = in_b;
            p->ring_out_bytes = out_b;
        }
    }
    if (e == cudaSuccess && !p->st_in) {
        e = cudaStreamCreateWithFlags(&p->st_in, cudaStreamNonBlocking);
        if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&p->st_out, cudaStreamNonBlocking);
    }
    if (e != cudaSuccess) {
        cudaGetLastError();
        return fail(p, e == cudaErrorMemoryAllocation ? DAXM_ERR_OUT_OF_MEMORY : DAXM_ERR_CUDA, "host ring: %s",
                    cudaGetErrorString(e));
    }
    cudaEvent_t* ev_in = p->ev_ring;       // [slot] band's stack landed
    cudaEvent_t* ev_dep = p->ev_ring + 2;  // [slot] band's deposit done (in[s] free, out[s] ready)
    cudaEvent_t* ev_out = p->ev_ring + 4;  // [slot] band's output copied out (out[s] free)
    // the caller's stream must reach this point before the first copy
    e = cudaEventRecord(ev_dep[0], st);
    if (e == cudaSuccess) e = cudaStreamWaitEvent(p->st_in, ev_dep[0], 0);
    const int nb = (int)p->bands.size();
    for (int b = 0; b < nb && e == cudaSuccess; ++b) {
        const int s = b & 1, r0 = p->band_r0[b], nr = p->band_r0[b + 1] - r0;
        daxm_plan* bp = p->bands[b];
        if (b >= 2) e = cudaStreamWaitEvent(p->st_in, ev_dep[s], 0);
        if (e == cudaSuccess)
            e = cudaMemcpy2DAsync(p->d_ring_in[s], nr * row_in, static_cast<const char*>(h_stack) + r0 * row_in,
                                  p->rows * row_in, nr * row_in, p->S, cudaMemcpyHostToDevice, p->st_in);
        if (e == cudaSuccess) e = cudaEventRecord(ev_in[s], p->st_in);
        if (e == cudaSuccess) e = cudaStreamWaitEvent(st, ev_in[s], 0);
        if (e == cudaSuccess && b >= 2) e = cudaStreamWaitEvent(st, ev_out[s], 0);
        if (e != cudaSuccess) break;
        daxm_set_cutoff(bp, p->use_cutoff, p->cutoff);
        daxm_status ds = run_deposit(bp, p->d_ring_in[s], (int)dt, p->d_ring_out[s], st);
        if (ds != DAXM_OK) {
            p->err = bp->err;
            cudaStreamSynchronize(st);
            return ds;
        }
        e = cudaEventRecord(ev_dep[s], st);
        if (e == cudaSuccess) e = cudaStreamWaitEvent(p->st_out, ev_dep[s], 0);
        if (e == cudaSuccess)
            e = cudaMemcpy2DAsync(reinterpret_cast<char*>(h_out) + r0 * row_out, p->rows * row_out, p->d_ring_out[s],
                                  nr * row_out, nr * row_out, p->M, cudaMemcpyDeviceToHost, p->st_out);
        if (e == cudaSuccess) e = cudaEventRecord(ev_out[s], p->st_out);
    }
    // join: the caller's stream sees the last copy out, then completes
    if (e == cudaSuccess) e = cudaEventRecord(ev_out[0], p->st_out);
    if (e == cudaSuccess) e = cudaStreamWaitEvent(st, ev_out[0], 0);
    if (e == cudaSuccess) e = cudaStreamSynchronize(st);
    if (e != cudaSuccess) {
        cudaGetLastError();
        return fail(p, DAXM_ERR_CUDA, "host ring: %s", cudaGetErrorString(e));
    }
    p->last_ring_rows = B;
    p->last_ring_bands = nb;
    return DAXM_OK;
}

daxm_status daxm_set_step_weights(daxm_plan* p, const double* w) {
    if (!p) return DAXM_ERR_INVALID_ARGUMENT;
    p->err.clear();
    std::vector<float> hw;
    if (w) {
        hw.resize(p->S);
        for (int k = 0; k < p->S; ++k) {
            if (!(isfinite(w[k]) && w[k] > 0.0))
                return fail(p, DAXM_ERR_INVALID_ARGUMENT, "step weight %d = %g is not finite and > 0", k, w[k]);
            hw[k] = (float)w[k];
        }
    }
    for (daxm_plan* c : p->child)
        if (c) {
            daxm_status s = daxm_set_step_weights(c, w);
            if (s != DAXM_OK) return s;
        }
    for (daxm_plan* b : p->bands) {
        daxm_status s = daxm_set_step_weights(b, w);
        if (s != DAXM_OK) return s;
    }
    DeviceGuard guard(p->device);
    if (!w) {
        cudaFree(p->d_w);
        p->d_w = nullptr;
        p->step_w.clear();
        return DAXM_OK;
    }
    p->step_w.assign(w, w + p->S);
    if (!p->d_w) {
        cudaError_t e = cudaMalloc(&p->d_w, sizeof(float) * p->S);
        if (e != cudaSuccess) {
            cudaGetLastError();
            return fail(p, DAXM_ERR_OUT_OF_MEMORY, "step weights: %s", cudaGetErrorString(e));
        }
    }
    cudaError_t e = cudaMemcpy(p->d_w, hw.data(), sizeof(float) * p->S, cudaMemcpyHostToDevice);
    if (e != cudaSuccess) {
        cudaGetLastError();
        return fail(p, DAXM_ERR_CUDA, "step weights: %s", cudaGetErrorString(e));
    }
    return DAXM_OK;
}

daxm_status daxm_set_host_budget(daxm_plan* p, uint64_t device_bytes) {
    if (!p) return DAXM_ERR_INVALID_ARGUMENT;
    p->err.clear();
    p->host_budget = device_bytes;
    return DAXM_OK;
}

daxm_status daxm_host_ring_info(const daxm_plan* p, int64_t* band_rows, int64_t* n_bands, int64_t* ring_bytes) {
    if (!p) return DAXM_ERR_INVALID_ARGUMENT;
    if (band_rows) *band_rows = p->last_ring_rows;
    if (n_bands) *n_bands = p->last_ring_bands;
    if (ring_bytes) *ring_bytes = p->last_ring_rows ? (int64_t)(2 * (p->ring_in_bytes + p->ring_out_bytes)) : 0;
    return DAXM_OK;
}

daxm_status daxm_reconstruct_host(daxm_plan* p, const void* h_stack, daxm_dtype dt, float* h_out, void* cuda_stream) {
    if (!p) return DAXM_ERR_INVALID_ARGUMENT;
    p->err.clear();
    if (!h_stack || !h_out) return fail(p, DAXM_ERR_INVALID_ARGUMENT, "NULL stack or output pointer");
    if (dt != DAXM_U16 && dt != DAXM_F32) return fail(p, DAXM_ERR_INVALID_ARGUMENT, "unknown dtype %d", (int)dt);
    DeviceGuard guard(p->device);
    const size_t plane = (size_t)p->rows * p->C;
    const size_t in_bytes = plane * p->S * (dt == DAXM_U16 ? 2 : 4);
    const size_t out_bytes = plane * p->M * sizeof(float);
    cudaStream_t st = (cudaStream_t)cuda_stream;
    cudaError_t e = cudaSuccess;
    if (p->host_budget > 0 && in_bytes + out_bytes > p->host_budget) {  // out of core
        if (p->d_stack_buf || p->d_out_buf) {  // the in-core buffers would break the budget
            cudaStreamSynchronize(st);
            cudaFree(p->d_stack_buf);
            cudaFree(p->d_out_buf);
            p->d_stack_buf = nullptr;
            p->d_out_buf = nullptr;
            p->stack_buf_bytes = p->out_buf_bytes = 0;
        }
        return host_ring(p, h_stack, dt, h_out, st);
    }
    p->last_ring_rows = p->last_ring_bands = 0;
    if (p->stack_buf_bytes < in_bytes) {
        cudaFree(p->d_stack_buf);
        p->d_stack_buf = nullptr;
        p->stack_buf_bytes = 0;
        e = cudaMalloc(&p->d_stack_buf, in_bytes);
        if (e != cudaSuccess) goto fail_cuda;
        p->stack_buf_bytes = in_bytes;
    }
    if (p->out_buf_bytes < out_bytes) {
        cudaFree(p->d_out_buf);
        p->d_out_buf = nullptr;
        p->out_buf_bytes = 0;
        e = cudaMalloc(&p->d_out_buf, out_bytes);
        if (e != cudaSuccess) goto fail_cuda;
        p->out_buf_bytes = out_bytes;
    }
    // Row-band pipeline: band b's host->device copy, its deposit and its
    // device->host copy run on three streams, so the two PCIe directions and the GPU overlap.
    {
        if (!p->st_in) {
            e = cudaStreamCreateWithFlags(&p->st_in, cudaStreamNonBlocking);
            if (e != cudaSuccess) goto fail_cuda;
            e = cudaStreamCreateWithFlags(&p->st_out, cudaStreamNonBlocking);
            if (e != cudaSuccess) goto fail_cuda;
        }
        // bands of Q-row quanta: on the row path 64 rows counted from the plan's first row (its row
        // tiles start there, so no tile straddles two bands), else the deposit tiles' global 128
        const bool rowp = uses_row_path(p, (int)dt);
        const int Q = rowp ? 64 : TILE_R;
        const int base = rowp ? p->g.row_begin : 0;
        const int q0 = (p->g.row_begin - base) / Q, nq = (p->g.row_end - base + Q - 1) / Q - q0;
        const int n_bands = nq < DAXM_HOST_BANDS ? nq : DAXM_HOST_BANDS;
        while ((int)p->ev.size() < 2 * n_bands) {
            cudaEvent_t ev;
            e = cudaEventCreateWithFlags(&ev, cudaEventDisableTiming);
            if (e != cudaSuccess) goto fail_cuda;
            p->ev.push_back(ev);
        }
        // the caller's stream must reach this point before the copies start
        e = cudaEventRecord(p->ev[0], st);
        if (e != cudaSuccess) goto fail_cuda;
        e = cudaStreamWaitEvent(p->st_in, p->ev[0], 0);
        if (e != cudaSuccess) goto fail_cuda;
        const size_t es = dt == DAXM_U16 ? 2 : 4;
        const size_t row_in = (size_t)p->C * es, row_out = (size_t)p->C * sizeof(float);
        for (int b = 0; b < n_bands; ++b) {
            const int g0 = std::max(p->g.row_begin, base + (q0 + b * nq / n_bands) * Q);
            const int g1 = std::min(p->g.row_end, base + (q0 + (b + 1) * nq / n_bands) * Q);
            int r0 = g0 - p->g.row_begin, r1 = g1 - p->g.row_begin;
            r0 = r0 < 0 ? 0 : r0;
            r1 = r1 > p->rows ? p->rows : r1;
            if (r1 <= r0) continue;
            const size_t w_in = (size_t)(r1 - r0) * row_in, w_out = (size_t)(r1 - r0) * row_out;
            e = cudaMemcpy2DAsync(static_cast<char*>(p->d_stack_buf) + r0 * row_in, p->rows * row_in,
                                  static_cast<const char*>(h_stack) + r0 * row_in, p->rows * row_in, w_in, p->S,
                                  cudaMemcpyHostToDevice, p->st_in);
            if (e != cudaSuccess) goto fail_cuda;
            e = cudaEventRecord(p->ev[2 * b], p->st_in);
            if (e != cudaSuccess) goto fail_cuda;
            e = cudaStreamWaitEvent(st, p->ev[2 * b], 0);
            if (e != cudaSuccess) goto fail_cuda;
            {
                daxm_status s = run_deposit(p, p->d_stack_buf, (int)dt, p->d_out_buf, st, g0, g1);
                if (s != DAXM_OK) return s;
            }
            e = cudaEventRecord(p->ev[2 * b + 1], st);
            if (e != cudaSuccess) goto fail_cuda;
            e = cudaStreamWaitEvent(p->st_out, p->ev[2 * b + 1], 0);
            if (e != cudaSuccess) goto fail_cuda;
            e = cudaMemcpy2DAsync(reinterpret_cast<char*>(h_out) + r0 * row_out, p->rows * row_out,
                                  reinterpret_cast<char*>(p->d_out_buf) + r0 * row_out, p->rows * row_out, w_out,
                                  p->M, cudaMemcpyDeviceToHost, p->st_out);
            if (e != cudaSuccess) goto fail_cuda;
        }
        // join: the caller's stream sees the last copy; then wait for completion
        e = cudaEventRecord(p->ev[1], p->st_out);
        if (e != cudaSuccess) goto fail_cuda;
        e = cudaStreamWaitEvent(st, p->ev[1], 0);
        if (e != cudaSuccess) goto fail_cuda;
        e = cudaStreamSynchronize(st);
        if (e != cudaSuccess) goto fail_cuda;
    }
    (void)in_bytes;
    (void)out_bytes;
    return DAXM_OK;
fail_cuda:
    cudaGetLastError();
    return fail(p, e == cudaErrorMemoryAllocation ? DAXM_ERR_OUT_OF_MEMORY : DAXM_ERR_CUDA, "host path: %s",
                cudaGetErrorString(e));
}

daxm_status daxm_set_cutoff(daxm_plan* p, int enable, double cutoff) {
    if (!p) return DAXM_ERR_INVALID_ARGUMENT;
    p->err.clear();
    if (enable && !(cutoff == cutoff)) return fail(p, DAXM_ERR_INVALID_ARGUMENT, "cutoff is NaN");
    p->use_cutoff = enable ? 1 : 0;
    p->cutoff = (float)cutoff;
    for (daxm_plan* c : p->child)
        if (c) {
            c->use_cutoff = p->use_cutoff;
            c->cutoff = p->cutoff;
        }
    return DAXM_OK;
}

static daxm_status select_cutoff_impl(daxm_plan* p, const void* d_stack, daxm_dtype dt, double fraction,
                                      unsigned long long n_total, daxm_hist_reduce_fn reduce, void* ctx,
                                      double* cutoff, void* cuda_stream) {
    if (!p) return DAXM_ERR_INVALID_ARGUMENT;
    p->err.clear();
    if (!d_stack || !cutoff) return fail(p, DAXM_ERR_INVALID_ARGUMENT, "NULL stack or cutoff pointer");
    if (dt != DAXM_U16 && dt != DAXM_F32) return fail(p, DAXM_ERR_INVALID_ARGUMENT, "unknown dtype %d", (int)dt);
    if (!(fraction > 0.0 && fraction <= 1.0))
        return fail(p, DAXM_ERR_INVALID_ARGUMENT, "fraction %g outside (0, 1]", fraction);
    const size_t n = (size_t)p->rows * p->C;
    if (reduce && n_total < n)
        return fail(p, DAXM_ERR_INVALID_ARGUMENT, "n_total %llu below the plan's %zu pixels", n_total, n);
    DeviceGuard guard(p->device);
    if (!p->d_hist && cudaMalloc(&p->d_hist, 256 * sizeof(unsigned long long)) != cudaSuccess) {
        cudaGetLastError();
        return fail(p, DAXM_ERR_OUT_OF_MEMORY, "cutoff histogram");
    }
    const double nk = reduce ? (double)n_total : (double)n;
    unsigned long long k = (unsigned long long)ceil(fraction * nk);
    if (k < 1) k = 1;
    if (k > (unsigned long long)nk) k = (unsigned long long)nk;
    bool reduce_failed = false;
    cudaError_t e = select_cutoff(d_stack, (int)dt, n, k, p->d_hist, (cudaStream_t)cuda_stream, cutoff, reduce, ctx,
                                  &reduce_failed);
    if (e != cudaSuccess) {
        cudaGetLastError();
        return fail(p, DAXM_ERR_CUDA, "cutoff selection: %s", cudaGetErrorString(e));
    }
    if (reduce_failed) return fail(p, DAXM_ERR_INVALID_ARGUMENT, "histogram reduce callback failed");
    return DAXM_OK;
}

daxm_status daxm_select_cutoff(daxm_plan* p, const void* d_stack, daxm_dtype dt, double fraction, double* cutoff,
                               void* cuda_stream) {
    return select_cutoff_impl(p, d_stack, dt, fraction, 0, nullptr, nullptr, cutoff, cuda_stream);
}

daxm_status daxm_select_cutoff_sharded(daxm_plan* p, const void* d_stack, daxm_dtype dt, double fraction,
                                       unsigned long long n_total, daxm_hist_reduce_fn reduce, void* ctx,
                                       double* cutoff, void* cuda_stream) {
    if (!reduce) {
        if (p) p->err = "NULL reduce callback";
        return DAXM_ERR_INVALID_ARGUMENT;
    }
    return select_cutoff_impl(p, d_stack, dt, fraction, n_total, reduce, ctx, cutoff, cuda_stream);
}

daxm_status daxm_depth_profile(daxm_plan* p, const float* d_out, double* d_profile, void* cuda_stream) {
    if (!p) return DAXM_ERR_INVALID_ARGUMENT;
    p->err.clear();
    if (!d_out || !d_profile) return fail(p, DAXM_ERR_INVALID_ARGUMENT, "NULL output or profile pointer");
    DeviceGuard guard(p->device);
    cudaError_t e = launch_depth_profile(d_out, p->M, (size_t)p->rows * p->C, d_profile, (cudaStream_t)cuda_stream);
    if (e != cudaSuccess) {
        cudaGetLastError();
        return fail(p, DAXM_ERR_CUDA, "depth profile launch: %s", cudaGetErrorString(e));
    }
    return DAXM_OK;
}

void daxm_destroy(daxm_plan* p) {
    if (!p) return;
    for (daxm_plan*& c : p->child) {
        daxm_destroy(c);
        c = nullptr;
    }
    {
        DeviceGuard guard(p->device);
        cudaDeviceSynchronize();
        free_plan_memory(p);
    }
    delete p;
}

}  // extern "C"
