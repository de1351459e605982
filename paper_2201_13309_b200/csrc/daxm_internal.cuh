// daxm_internal.cuh -- internal data layout shared by the plan (pre-pass) and
// the deposit kernels.  Not part of the ABI.  See DESIGN.md "Data layout".
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <atomic>

#include "daxm.h"

namespace daxm {

// Deposit tile: TILE_R detector rows x TILE_C detector columns.  Rows are the
// warp lanes (the depth-insensitive detector axis: all 32 lanes of a warp walk
// their pixels in lock step); each thread owns 4 adjacent columns.  Tiles are
// aligned to GLOBAL detector rows/cols, so a row-band plan reproduces the
// full-detector plan bit for bit.
#ifndef DAXM_TILE_R
#define DAXM_TILE_R 128
#endif
#ifndef DAXM_TILE_C
#define DAXM_TILE_C 8
#endif
constexpr int TILE_R = DAXM_TILE_R;  // multiple of 32
constexpr int TILE_C = DAXM_TILE_C;  // 8 or 16: one tile row of output = 32 or 64 bytes
static_assert(TILE_R % 32 == 0 && (TILE_C == 8 || TILE_C == 16), "tile shape");
static_assert(TILE_R * TILE_C <= 1024, "pre-pass tile kernel: one thread per pixel");
constexpr int TILE_E = TILE_C + 1;  // pixel edge columns per tile (finite pixels)
constexpr int NCOEF = 3;            // depth model per edge point: polynomial of degree NCOEF-1 in wire travel
// fp64 approximation error allowed for the depth model (bins); the fp32 evaluation adds ~ulp(M/2)
constexpr double MODEL_ERR_MAX = NCOEF >= 4 ? 1e-6 : 2e-5;
constexpr double ROW_TAU_ERR_MAX = 2e-4;  // row path: max fp32 depth error (bins) incl. its wire travel
#ifndef DAXM_CPT
#define DAXM_CPT 4
#endif
constexpr int COLS_PER_THREAD = DAXM_CPT;  // pixel walks per fast-kernel thread (1, 2 or 4)
constexpr int N_CONSUMER_WARPS = (TILE_R / 32) * (TILE_C / COLS_PER_THREAD);
#ifndef DAXM_MC
#define DAXM_MC 4
#endif
#ifndef DAXM_PREFETCH
#define DAXM_PREFETCH 1
#endif
constexpr int MC = DAXM_MC;         // depth planes per output chunk (one TMA store)
#ifndef DAXM_NB_U16
#define DAXM_NB_U16 32
#endif
#ifndef DAXM_NB_F32
#define DAXM_NB_F32 16
#endif
#ifndef DAXM_OB
#define DAXM_OB 2
#endif
constexpr int NB_U16 = DAXM_NB_U16;  // input ring slots (wire steps) for uint16 stacks (power of 2)
constexpr int NB_F32 = DAXM_NB_F32;  // ... for float32 stacks
constexpr int OUT_BUFS = DAXM_OB;    // output staging buffers per 32-row warp group (slack between its warps)
constexpr int MAX_FAST_NV = 4096;   // fast path: steps streamed per tile (tau table in shared memory)
constexpr int MAX_FAST_CHUNKS = 1024;  // fast path needs (M + MC - 1) / MC + 1 <= this (M <= 4092)
constexpr int RING_WINDOW_CHUNKS = 1;  // a warp's input needs between two of its own chunk boundaries

// Geometry constants for the fp64 pre-pass (by value into kernels).
struct GeomConst {
    double rho[9];          // detector rotation (Rodrigues)
    double trans[3];        // det_trans
    double pitch_col, pitch_row;
    double axis[3];         // unit wire axis
    double beam[3];         // unit beam direction
    double origin[3];       // depth origin
    double w0[3];           // first wire centre
    double d[3];            // unit scan direction, perpendicular to the axis
    double r;               // wire radius
    double lo0;             // lower edge of bin 0 (um)
    double dz;              // bin width (um)
    int R, C, S, M;
    int edge;               // 0 leading, 1 trailing
    int point_mode;         // 1: POINT pixel model
    int m_ref;              // integer bin offset of the fp32 depth coordinate
};

// Per deposit tile (global tile index).
struct TileInfo {
    double t_ref;   // wire-travel reference (um) the cubic is expanded about
    int k_lo;       // first wire step (point) any pixel of the tile reads
    int k_hi;       // last wire step (point) any pixel of the tile reads (inclusive); k_hi < k_lo: empty
    int dir;        // +1: depth increases with the step index, -1: decreases
    int separated;  // deposit mode: MODE_SEPARATED / MODE_OVERLAP (fast kernel) or MODE_GENERAL
    int ring_need;  // input ring slots the fast kernel needs for this tile (deadlock-free bound)
    int lock;       // step-locked kernel: output ring class (LOCK_RB_SMALL / LOCK_RB_LARGE) or 0 (not eligible)
};

// Per-tile deposit mode (pre-pass, fp64): every pixel's consecutive edge spans are
// disjoint (SEPARATED) or every pixel's overlap (OVERLAP) -> fast kernel; else GENERAL.
enum : int { MODE_GENERAL = 0, MODE_SEPARATED = 1, MODE_OVERLAP = 2 };

// Pre-pass failure flags (device word, read back by the host).
enum : unsigned {
    FLAG_NONMONOTONE = 1u,
    FLAG_NAN_IN_WINDOW = 2u,
    FLAG_MIXED_DIR = 4u,
    FLAG_FIT_NAN = 8u,
};

// Device-side plan view passed to the deposit kernels by value.
struct DepositArgs {
    const double* t;          // [S] wire travel t_k (um)
    const TileInfo* tiles;    // [n_tr][n_tc]
    const int2* win;          // [pre_rows][C] pair window [kb, ke) per pixel (global pixel indexing)
    const float* coef;        // [n_tiles][NCOEF][TILE_E][TILE_R]
    const int* tile_list;     // tiles for the general kernel
    int n_list;
    int R, C, S, M;
    int row_begin, row_end;   // band (global rows)
    int pre_row0;             // first global row of win[]
    int tr0, n_tr, n_tc;      // tile rows covered (global tile-row index tr0 ..)
    int tr_begin, tr_end;     // tile rows (relative) this launch processes (row-band pipelining)
    int m_ref;
    int point_mode;
    int has_overlap;          // any MODE_OVERLAP tile (second fast-kernel launch)
    int nb;                   // input ring slots for this dtype (fast kernel)
    int max_nv;               // max steps any tile streams (tau table size)
    const int* vneed;         // [n_tiles][n_states + 1][8 warps] furthest visit index loaded by each state
    int n_states;             // (M + MC - 1) / MC + 1
    float sign;               // s: +1 leading, -1 trailing (reading R2)
    float dI_floor;           // s dI -> max(s dI, dI_floor): -inf, or 0 in the both-edges mode (R16)
    int acc;                  // 1: add into the output (both-edges mode, second edge) instead of storing
    const float* w;           // [S] per-step intensity normalisation weights (reading R17), or NULL
    const void* stack;        // band stack [S][rows][C] (plane 0 read for the intensity cutoff)
    const float* table;       // exact depth table (general kernel) or nullptr: per tile at toff[tile],
    const long long* toff;    //   [k - k_lo][TILE_E][TILE_R] fp32 bins relative to m_ref
    int use_cutoff;           // 1: only pixels with I_0 >= cutoff are reconstructed (reading R14)
    float cutoff;
    const unsigned char* tile_live;  // [n_tr][n_tc] cutoff on: 0 = no pixel of the tile passes (CTAs exit;
                                     //   zero_dead_tiles writes its planes), else nullptr
    const unsigned char* grp_live;   // [n_tr][n_tc][NG16] the same per 16-row group (one locked warp)
    int lock_enabled;         // step-locked kernel handles tiles with tiles[].lock != 0
    int lock_small, lock_large, lock_rest;  // tile counts: lock classes, fast tiles left to deposit_fast
    int lock_ov_small, lock_ov_large;       // ... overlapping tiles in deposit_lock_ov
    int lock_ov_enabled;                    // pre-pass: admit overlapping tiles (unset by DAXM_NO_LOCK_OV)
    unsigned* lock_err;       // device word: ring-capacity violations (must stay 0)
};

// Step-locked deposit kernel (deposit_lock.cu): one warp = 16 detector rows x 8 columns,
// lanes = 8 columns x 4 row groups, 4 pixel walks (rows) per thread.  Every walk of a warp
// visits the same wire step at the same iteration (warp-locked, from the warp's first window
// start); the edges of the zone the step closes are evaluated in a warp-uniform loop.  Output planes go through a per-warp
// ring of LOCK_RB planes indexed by bin edge.
constexpr int LOCK_ROWS = 16;       // detector rows per warp
constexpr int NG16 = TILE_R / LOCK_ROWS;  // 16-row groups per tile (cutoff liveness flags)
constexpr int LOCK_WARPS = 4;       // warps per CTA (independent pipelines)
constexpr int LOCK_SUBS = TILE_R / (LOCK_ROWS * LOCK_WARPS);  // CTAs per deposit tile
constexpr int LOCK_NB = 16;         // input ring slots (wire steps) per warp
constexpr int LOCK_G = 4;           // wire steps per TMA box and mbarrier (one group)
constexpr int LOCK_NG = LOCK_NB / LOCK_G;  // groups in the input ring
constexpr int LOCK_CLASS_MASK = 0xff;  // TileInfo.lock: ring class in the low byte
constexpr int LOCK_FRONT_LO = 0x100;   //   flag: the front pixel edge is the shallower over the whole tile
constexpr int LOCK_OVB = 0x40;         //   class bit: overlapping edge spans (deposit_lock_ov, ramp superposition)
constexpr int LOCK_P = 4;              // ramps deposit_lock_ov keeps quadratic: hi_q <= lo_{q+LOCK_P} (pre-pass)
constexpr int LOCK_RB_SMALL = 16;   // output ring planes per warp
constexpr int LOCK_RB_LARGE = 32;
// largest "need" (edges from the slowest walk's frontier to the furthest edge written in one
// iteration, inclusive) a ring of rb planes holds: planes below the frontier are copied out
// before the next iteration, so writes stay below frontier - 1 + rb
constexpr int lock_need_max(int rb) { return rb; }
static_assert(LOCK_NB % LOCK_G == 0 && (LOCK_NB / LOCK_G & (LOCK_NB / LOCK_G - 1)) == 0, "lock input ring shape");

// ---- Row-segment deposit kernel (deposit_row.cu), the production path.
// One warp = one "row tile" of RW_ROWS detector rows x RW_COLS columns, aligned to the band's first
// row and to global columns; lane l owns two adjacent columns of one column half, both rows: four
// pixel walks, packed in two pairs (two rows of one column).  Output planes leave as two 256-byte
// rows per warp (st.global.cs.v4 per lane; tiles without a change: TMA zero stores of
// [RW_PB planes][RW_ROWS][RW_COLS] boxes), the stack arrives as TMA loads of [RW_G steps][RW_ROWS]
// [32 cols] boxes per column half: the store geometry that reaches the copy ceiling
// (profiles/r02b_membench.md), where the round-1 16 x 8 warp block could not.
#ifndef DAXM_RW_ROWS
#define DAXM_RW_ROWS 2
#endif
#ifndef DAXM_RW_NB
#define DAXM_RW_NB 24
#endif
#ifndef DAXM_RW_KT
#define DAXM_RW_KT 5
#endif
constexpr int RW_ROWS = DAXM_RW_ROWS;  // 2 (tile 2 x 64) or 4 (tile 4 x 32)
constexpr int RW_COLS = 128 / RW_ROWS;
constexpr int RW_H = RW_COLS / 32;  // column halves per lane: pair p = half p (RW_H = 2) or rows 2p, 2p+1
constexpr int RW_NB = DAXM_RW_NB;   // input ring slots (wire steps) per column half (a multiple of RW_G)
constexpr int RW_G = 4;             // wire steps per TMA load box
#ifndef DAXM_RW_PB
#define DAXM_RW_PB 4
#endif
constexpr int RW_PB = DAXM_RW_PB;   // planes per TMA zero-store box (tiles without a change)
constexpr int RW_EXT = 16;          // steps a row tile's range extends below its windows (lock-step starts)
constexpr int RW_KT = DAXM_RW_KT;   // max bin edges one walk evaluates per iteration (unrolled trips)
constexpr int RW_RB_SMALL = 16, RW_RB_LARGE = 32;  // output ring planes (+ RW_KT - 1 overflow planes)
constexpr int RW_CLS_RB = 0xff;         // RowTile.cls: ring planes (0: not admitted -> general kernel)
constexpr int RW_CLS_FRONT_LO = 0x100;  //   the front pixel edge is the shallower one over the tile
constexpr int RW_CLS_GEN = 0x200;       //   general-span variant (overlapping spans, spans up to RW_NQ_GEN bins)
constexpr int RW_CLS_NB_WIDE = 0x400;   //   general-span variant with the RW_NB_WIDE-slot input ring
constexpr int RW_NB_WIDE = 64;          // input ring slots for tiles whose visits spread wider than RW_NB
constexpr int RW_CLS_NB_MID = 0x800;    //   separated variant with the RW_NB_MID-slot input ring
constexpr int RW_CLS_KT_SHIFT = 12;     //   bits 12-13: edge-trip class ktc of the separated variants
                                        //   (3, 4 or 5 edges per zone and step)
constexpr int RW_NB_MID = 32;           // input ring slots of that variant
#ifndef DAXM_RW_NB_MARGIN
#define DAXM_RW_NB_MARGIN 8
#endif
constexpr int RW_NB_MARGIN = DAXM_RW_NB_MARGIN;  // RW_NB ring: visits of load lookahead the admission keeps
static_assert(RW_NB_MARGIN % RW_G == 0 && RW_NB_MARGIN < RW_NB, "ring margin");
constexpr int RW_KT_GEN = 6;            // max bin edges per zone and iteration, general-span variant
constexpr int RW_NQ_GEN = 4;            // general-span variant: zone edges evaluated exactly (then linear)
static_assert(RW_ROWS * RW_COLS == 128 && RW_COLS % 32 == 0 && (RW_ROWS == 2 || RW_ROWS == 4),
              "row tile: 4 walks per lane, two per pair");
// pair p of a lane: column half and first row
__host__ __device__ constexpr int rw_half(int p) { return RW_H == 2 ? p : 0; }
__host__ __device__ constexpr int rw_row(int p) { return RW_H == 2 ? 0 : 2 * p; }
static_assert(RW_KT - 1 <= RW_RB_SMALL && RW_RB_SMALL % RW_PB == 0 && RW_NB % RW_G == 0, "row ring shapes");

struct RowTile {
    double t_ref;  // wire-travel reference the tile's depth polynomials are expanded about
    int k_lo, k_hi;  // union of the tile's pixel windows (points); k_hi < k_lo: empty
    int dir;         // +1: depth increases with the step index
    int sep;         // MODE_SEPARATED / MODE_OVERLAP / MODE_GENERAL over the tile's band pixels
    int cls;         // admission class (RW_CLS_*), 0 = general kernel
    int niter;       // iterations of the admitted schedule (pre-pass replay)
    int why;         // not admitted: RW_WHY_* bits
    int kmax;        // most bin edges one walk crosses in one step (admission replay)
};
enum : unsigned {
    RW_WHY_MODE = 1u,      // not every pixel in the separated-span regime
    RW_WHY_KT = 2u,        // a zone holds more than RW_KT bin edges
    RW_WHY_INPUT = 4u,     // the pairs' visits spread wider than the input ring
    RW_WHY_DENSITY = 8u,   // equal consecutive edge sums or a vanishing edge span (fp32)
    RW_WHY_TOP = 16u,      // a window's last point below the top bin edge
    RW_WHY_RING = 32u,     // output-ring need above RW_RB_LARGE
    RW_WHY_ORDER = 64u,    // neither pixel edge is the shallower one throughout
    RW_WHY_ITER = 128u,
    RW_WHY_GEN = 256u,     // general-span variant: a ramp reaching past the next zone, knots beyond
                           // RW_NQ_GEN bins or a vanishing rise / fall width
};

struct RowArgs {
    const double* t;       // [S] wire travel
    const RowTile* rt;     // [n_rt]
    const int2* win;       // [pre_rows][C] pixel windows (global pixel indexing, rows from pre_row0)
    const float* coef;     // [n_rt][NCOEF][RW_COLS + 1][RW_ROWS] depth polynomials (bins rel. m_ref)
    const int* list;       // row tiles of this launch (one class), ascending
    int n_list;
    int R, C, S, M, m_ref;
    int row_begin, row_end, pre_row0;
    int row_org;           // global row of row-tile row 0 (= row_begin: row tiles start at the band)
    int n_rc;              // row-tile columns
    int max_nv;            // largest tile step range (tau table size)
    int point_mode;
    float sign;            // s: +1 leading, -1 trailing (reading R2)
    float dI_floor;        // s dI -> max(s dI, dI_floor): -inf, or 0 in the both-edges mode (R16)
    int acc;               // 1: add into the output (both-edges mode, second edge)
    const void* stack;     // band stack (plane 0 read for the intensity cutoff)
    float* out;            // band output [M][rows][C] (the row kernel's plane copy-out)
    float dth, dtl;        // wire travel per step Delta = t_{S-1} / (S - 1), split hi + lo (row_tau)
    int use_cutoff;
    float cutoff;
    const unsigned char* live;  // [n_rt] per-call row_live_kernel flags (0: zeros written), or NULL
    float* prof_part;      // [n_rt][M] per-tile plane sums (fused depth-profile epilogue), or NULL
    unsigned* err;         // DAXM_ROW_CHECK builds: schedule violations (must stay 0)
};

#ifndef DAXM_ROW_TAU_LINEAR
#define DAXM_ROW_TAU_LINEAR 1  // row kernel: wire travel from row_tau (0: a per-warp shared-memory table)
#endif
// Wire travel of a row tile's visit v (its step k = k_lo + v, or k_hi - v for dir < 0) relative to
// the tile's t_ref, in fp32, as the row kernel, its admission replay and the row fit's error check
// all evaluate it: Af = (float)(t_{k_first} - t_ref), (dh, dl) = dir * (Delta_hi, Delta_lo) with
// Delta the mean step -- the scan's own travel for uniformly stepped scans; the fit check bounds the
// depth error of the approximation for any other straight scan (the row path is refused above it).
__device__ __forceinline__ float row_tau(float Af, float dh, float dl, int v) {
    const float fv = __int_as_float(0x4B000000 | v) - 8388608.f;  // (float)v, exact for v < 2^23
    return fmaf(fv, dh, fmaf(fv, dl, Af));
}

// Corner depth of one pixel edge at fp32 wire travel tau (bins relative to m_ref): the
// pre-pass ring check and the step-locked kernel evaluate exactly this expression.
__device__ __forceinline__ float lock_poly(float c0, float c1, float c2, float t) {
    return fmaf(fmaf(c2, t, c1), t, c0);
}

// One-time per DEVICE setup of a kernel's function attributes (cudaFuncSetAttribute acts on the
// current device): `done` holds one bit per device ordinal already set up.  Idempotent, so two
// threads racing on the same device both set the same attributes harmlessly.
template <typename F>
inline cudaError_t once_per_device(std::atomic<unsigned long long>& done, F&& set) {
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return e;
    const unsigned long long bit = dev < 64 ? 1ull << dev : 0ull;
    if (bit && (done.load(std::memory_order_acquire) & bit)) return cudaSuccess;
    if ((e = set()) != cudaSuccess) return e;
    done.fetch_or(bit, std::memory_order_acq_rel);
    return cudaSuccess;
}

// Launchers (deposit.cu, profile.cu, select.cu).
typedef int (*HistReduce)(unsigned long long* hist, int n, void* ctx);  // = daxm_hist_reduce_fn
cudaError_t select_cutoff(const void* plane0, int dtype, size_t n, unsigned long long k,
                          unsigned long long* d_hist, cudaStream_t st, double* cutoff, HistReduce reduce,
                          void* ctx, bool* reduce_failed);
cudaError_t launch_cutoff_tiles(const DepositArgs& a, const void* plane0, int dtype, float* out, unsigned char* live,
                                int phase, cudaStream_t st);  // phase 0: tile flags; 1: zero fill of dead tiles
cudaError_t launch_depth_profile(const float* out, int M, size_t plane, double* profile, cudaStream_t st);
// profile[m] = sum over row tiles [rt0, rt0 + n) of part[rt][m] (fp64, fixed order)
cudaError_t launch_profile_reduce(const float* part, int rt0, int n, int M, double* profile, cudaStream_t st);
size_t fast_smem_bytes(int dtype, int max_nv);
cudaError_t launch_deposit(const DepositArgs& a, const CUtensorMap* in_map, const CUtensorMap* out_map,
                           const void* stack, int dtype, float* out, bool fast_enabled, cudaStream_t st,
                           const CUtensorMap* lock_in_map, const cudaStream_t* lock_sts, int n_lock_sts);
size_t lock_smem_bytes(int dtype, int rb, int max_nv);
cudaError_t launch_lock(const DepositArgs& a, const CUtensorMap* in_map, float* out, int dtype, int n_tiles,
                        const cudaStream_t* sts, int nst);
cudaError_t launch_lock_prepass(const DepositArgs& a, int n_tiles, int* d_stats, cudaStream_t st);
// row-segment kernel (deposit_row.cu): pre-pass replay (admission) and the class launches
cudaError_t launch_row_admit(const RowArgs& a, RowTile* rt, int n_rt, int* d_stats, cudaStream_t st);
cudaError_t row_set_attributes();
cudaError_t launch_row_live(const RowArgs& a, int rt0, int n, unsigned char* live, int dtype,
                            cudaStream_t st);  // exact zero-dI skip flags of row tiles [rt0, rt0 + n)  // per device: dynamic shared memory of every instance
cudaError_t launch_row(const RowArgs& a, const CUtensorMap* in_map, const CUtensorMap* out_map, int dtype, int rb,
                       int variant, int ktc, cudaStream_t st);
// per-translation-unit instance sets of the row kernel (deposit_row.cu, deposit_row_{1,2,3}.cu)
template <int TU>
cudaError_t row_part_attributes_t();
template <int TU>
cudaError_t row_part_launch_t(const RowArgs& a, const CUtensorMap* in_map, const CUtensorMap* out_map, int variant,
                              int ktc, cudaStream_t st);  // variant: 0 separated, 1 general-span, 2 + wide input ring
cudaError_t launch_general_rows(const DepositArgs& a, const int* rt_list, int n, int n_rc, int row_org,
                                const void* stack, int dtype, float* out, cudaStream_t st);

}  // namespace daxm
