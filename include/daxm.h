/*
 * daxm.h -- C ABI of the B200 (sm_100a) wire-scan depth reconstruction library
 * (differential-aperture X-ray microscopy, "DAXM"; arXiv:2201.13309).
 *
 * The method (Fig. 6 P:L304-349 and Fig. 7): for every
 * detector pixel and every pair of consecutive wire steps k, k+1, take the
 * intensity difference dI = I_k - I_{k+1}; ray-trace
 * from the pixel's two edges, tangent to the wire edge, to the incident beam
 * ("depth is measured along the incident beam from the origin"),
 * which gives four corner depths of a trapezoidal depth response
 * (device_get_trapezoid_height); distribute dI over the fixed
 * depth bins (device_index_to_beam_depth P:L330/P:L344-345) in proportion to the
 * trapezoid area inside each bin (device_depth_resolve_pixel).
 * The result is one image per depth bin (image_set.depth_resolved).
 * Conventions the paper leaves open are fixed in DESIGN.md "Readings" (R1-R13)
 * and are identical to the CPU oracle's.
 *
 * Calls (all return daxm_status; no exceptions cross the ABI):
 *   daxm_create        geometry -> plan (validates, runs the fp64 geometry
 *                      pre-pass on the GPU, caches per-pixel windows and
 *                      per-edge-point depth polynomials in device memory)
 *   daxm_reconstruct   device stack [S][rows][C] -> device output [M][rows][C]
 *                      (stream-ordered, asynchronous, allocates nothing,
 *                      CUDA-graph capturable)
 *   daxm_reconstruct_host  the same from/to HOST buffers (copies included;
 *                      out of core under a device-memory budget,
 *                      daxm_set_host_budget / daxm_host_ring_info)
 *   daxm_reconstruct_profile  daxm_reconstruct + the depth profile (fused)
 *   daxm_set_cutoff / daxm_select_cutoff[_sharded]  intensity cutoff, pixel percentage
 *   daxm_set_step_weights  per-step intensity normalisation
 *   daxm_depth_profile  per-bin totals of an output
 *   daxm_plan_info / daxm_plan_stats / daxm_last_error / daxm_status_string
 *   daxm_destroy
 */
#ifndef DAXM_H_
#define DAXM_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define DAXM_ABI_VERSION 1

typedef struct daxm_plan daxm_plan; /* opaque; owned by the library */

typedef enum {
    DAXM_OK = 0,
    DAXM_ERR_INVALID_ARGUMENT = 1, /* bad sizes/enums/NaN/null pointers (see daxm_create)          */
    DAXM_ERR_NONMONOTONE_SCAN = 2, /* wire travel or a pixel's depth-vs-step not monotone           */
    DAXM_ERR_GEOMETRY = 3,         /* every pixel invalid (NaN tangent depth at every wire step)    */
    DAXM_ERR_OUT_OF_MEMORY = 4,
    DAXM_ERR_CUDA = 5              /* any CUDA runtime error; detail in daxm_last_error()            */
} daxm_status;

/* DAXM_EDGE_BOTH (reading R16): both wire edges in one reconstruction -- the leading
 * edge's geometry takes every step's intensity decrease max(I_k - I_{k+1}, 0), the trailing edge's
 * the increase max(I_{k+1} - I_k, 0) (its sign-normalised dI, reading R2), and the two add.  The
 * paper's wire_edge selector runs one edge per call; with BOTH a plan holds
 * one pre-pass per edge (twice the plan memory and pre-pass time) and a call runs both. */
typedef enum { DAXM_EDGE_LEADING = 0, DAXM_EDGE_TRAILING = 1, DAXM_EDGE_BOTH = 2 } daxm_edge;
typedef enum {
    DAXM_PIXEL_FINITE = 0, /* pixel of finite width along the column axis: trapezoid (the paper)   */
    DAXM_PIXEL_POINT = 1   /* pixel centre only: box response                                       */
} daxm_pixel_model;
typedef enum { DAXM_U16 = 0, DAXM_F32 = 1 } daxm_dtype;

/* Geometry (all lengths in um, lab frame).  Passed by pointer; copied. */
typedef struct {
    int32_t n_rows, n_cols;         /* full detector R x C; image layout [row][col], col fastest        */
    int32_t row_begin, row_end;     /* this plan's row band [begin, end) (0, R = whole detector)        */
    double pitch_col, pitch_row;    /* um per pixel along x' (col) and y' (row)                          */
    double det_rot[3];              /* Rodrigues vector (rad): |R| = angle, R/|R| = axis                 */
    double det_trans[3];            /* lab = rho * ((x', y', 0) + det_trans);                            */
                                    /* pixel centre (i, j): x' = (i-(C-1)/2) pitch_col, y' likewise      */
    double beam_dir[3];             /* incident beam direction k-hat (normalised by the library)         */
    double beam_origin[3];          /* depth origin O: depth D is the point O + D k-hat                  */
    double wire_axis[3];            /* wire axis a-hat (normalised by the library)                       */
    double wire_radius;             /* r > 0                                                             */
    int32_t n_steps;                /* S >= 2 wire steps                                                 */
    const double *wire_xyz;         /* host pointer, S x 3 wire-centre positions (copied at create).    */
                                    /* Any path along which every pixel edge's depth is monotone; a     */
                                    /* straight scan runs the fast kernels, any other path (jitter, a   */
                                    /* curved stage) an exact per-step depth table          */
    double depth_start, depth_end;  /* centres of the first / last depth bin                             */
    double depth_res;               /* bin width dz > 0; M = round((end-start)/dz) + 1 bins,            */
                                    /* bin m covers [start + (m-1/2) dz, start + (m+1/2) dz)             */
    int32_t edge;                   /* daxm_edge: which wire edge the tangent touches                    */
    int32_t pixel_model;            /* daxm_pixel_model                                                  */
} daxm_geometry;

/* Per-plan statistics (for roofline accounting and tests). */
typedef struct {
    int64_t n_bins, rows, cols, n_steps; /* M, rows in band, C, S                                       */
    int64_t contrib_pairs;     /* sum over band pixels of step pairs whose trapezoid overlaps the bins   */
                               /* (S_c, exact fp64; the algorithmic read count per pixel is S_c + 1)      */
    int64_t contrib_pixels;    /* band pixels with S_c > 0                                               */
    int64_t window_pairs;      /* pairs the deposit kernel visits (S_c plus one guard pair each side)     */
    int64_t staged_steps;      /* sum over band tiles of steps the deposit kernel streams for the tile    */
    int64_t n_tiles;           /* deposit tiles covering the band                                         */
    int64_t general_tiles_u16; /* tiles the general (non-separated) deposit kernel handles, uint16 stacks  */
    int64_t general_tiles_f32; /* ... float32 stacks (the rest run the TMA-pipelined fast kernel)          */
    int64_t nonseparated_tiles; /* tiles not in the separated-span regime                                */
    int64_t overlap_tiles;     /* of which every pixel's consecutive edge spans overlap (fast kernel, dual walk) */
    int64_t ring_need_max;     /* largest input-ring demand of a tile (fast path needs <= ring slots)     */
    int32_t tile_rows, tile_cols;
    double fit_max_err_bins;   /* max |fp32-stored cubic (fp32 tau) - exact fp64 depth| over every edge  */
                               /* point and every step the kernel can read, in bins (<= 1e-3 enforced)    */
    double fit_model_err_bins; /* the same for the fp64 cubic: approximation error (<= 1e-6 enforced)     */
    double prepass_ms;         /* GPU time of the geometry pre-pass                                       */
    int64_t device_bytes;      /* device memory owned by the plan                                         */
    int64_t depth_table_bytes; /* > 0: depths come from an exact per-step fp32 table (bins) over every    */
                               /* tile's step range and all tiles run the general kernel: the wire path */
                               /* is not straight, or the polynomial model missed its tolerance          */
    int64_t lock_tiles_small;  /* tiles the step-locked kernel handles with a 16-plane output ring        */
    int64_t lock_tiles_large;  /* ... with a 32-plane output ring                                         */
    int64_t lock_ring_violations; /* step-locked ring-capacity violations so far (read synchronously;    */
                               /* always 0: the pre-pass admits only tiles whose ring provably suffices) */
    int64_t lock_tiles_overlap; /* overlapping-span tiles the step-locked ramp-superposition kernel handles */
    int64_t row_tiles_small;   /* row tiles (2 rows x 64 columns) the row-segment kernel handles with a   */
    int64_t row_tiles_large;   /* 16- / 32-plane output ring; the rest run the general kernel             */
    int64_t row_tiles_general;
    int64_t row_ring_need_max; /* largest output-ring need (planes) the admission replay found          */
    int64_t row_reject_bits;   /* OR of the reasons row tiles were not admitted (RW_WHY_* bits,         */
    int64_t row_reject[8];     /* DESIGN.md §5.3) and the number of row tiles per reason bit            */
    int64_t row_path;          /* 1: daxm_reconstruct runs the row-segment kernel (every row tile          */
                               /* admitted), 0: the deposit-tile kernels                                   */
    int64_t row_tiles_gen;     /* of row_tiles_small + row_tiles_large: tiles the general-span variant    */
                               /* runs (overlapping edge spans or spans of 2-4 bins)      */
    int64_t row_reject_more;   /* row tiles not admitted for RW_WHY_GEN (bit 8)                          */
    int64_t row_launches;      /* kernel launches of one daxm_reconstruct on the row path: the zero-dI  */
                               /* scan, then one per non-empty class (separated / general-span / wide   */
                               /* input ring x ring 16 / 32, general)                                    */
    int64_t row_tiles_nb_mid;  /* of them: separated-variant tiles that need the 32-slot input ring        */
    int64_t row_kmax_hist[8];  /* admitted row tiles by the most bin edges one walk crosses in one wire    */
                               /* step (index = that count, 7 = 7 or more)                               */
} daxm_plan_stats;

/* daxm_create -- validate `g`, run the fp64 geometry pre-pass on `cuda_device`,
 * return a plan in *out (NULL on error).
 *   INVALID_ARGUMENT: g/out NULL; S < 2; R, C < 1 or band outside [0, R) or empty;
 *     pitch, r or dz <= 0 or non-finite; depth_end < depth_start; (end-start)/dz
 *     not an integer within 1e-6; zero-length or non-finite beam/axis vectors;
 *     any non-finite input; beam parallel to the axis; unknown enum value;
 *     wire_xyz NULL.
 *   NONMONOTONE_SCAN: first and last positions coincide (perpendicular to a-hat),
 *     the travel of a straight scan decreases, or a pixel edge's depth is not
 *     monotone in the step index inside its window.
 *   GEOMETRY: every pixel invalid: each pixel edge lies inside the wire cylinder, or its tangent
 *     plane is parallel to the beam, at every wire step.  Per-pixel degeneracies are not errors:
 *     a step pair with a NaN corner depth is skipped, as in the oracle (reading R8; such plans run
 *     the exact-depth-table general kernel).
 * Depth source: for a straight scan (centres within 1e-6 um + 1e-9 relative of
 * the line through the first and last) a quadratic per edge point in wire
 * travel, kept if its fp64 error is <= 2e-5 bins and its fp32 error <= 1e-3 bins;
 * otherwise (or with DAXM_FORCE_TABLE set in the environment) the exact per-step
 * table, see daxm_plan_stats.depth_table_bytes.
 *   OUT_OF_MEMORY / CUDA: allocation or runtime failure.
 * The calling thread's current device is restored before returning. */
daxm_status daxm_create(const daxm_geometry *g, int cuda_device, daxm_plan **out);

/* M, rows in the plan's band, C.  Any output pointer may be NULL. */
daxm_status daxm_plan_info(const daxm_plan *p, int64_t *n_bins, int64_t *rows, int64_t *cols);
daxm_status daxm_plan_stats_get(const daxm_plan *p, daxm_plan_stats *st);

/* daxm_reconstruct -- d_stack: device pointer, [S][rows][C] of `dt`, rows = the
 * plan's band (row_end - row_begin), C contiguous, 16-byte aligned.
 * d_out: device pointer, [M][rows][C] float32, fully overwritten (zeros
 * included), 16-byte aligned.  cuda_stream: cudaStream_t (NULL = legacy
 * default stream).  Asynchronous; no allocation; graph-capturable.  Caller
 * owns both buffers; they must stay valid until the stream reaches the work.
 * Errors: INVALID_ARGUMENT (NULL pointers, misalignment, unknown dtype), CUDA
 * (launch failure; detail in daxm_last_error).
 * Concurrency: at most ONE call on a plan may be in flight at a time.  Calls issued on one stream
 * are ordered by it; calls on different streams (or a captured graph replayed beside eager calls)
 * must be ordered by the caller, because the plan owns scratch they share (cutoff liveness flags,
 * the class-launch fork streams and events, the host-path buffers).  Use one plan per concurrent
 * stream.  A plan is not thread-safe: serialise calls from several host threads. */
daxm_status daxm_reconstruct(daxm_plan *p, const void *d_stack, daxm_dtype dt, float *d_out, void *cuda_stream);

/* daxm_reconstruct_host -- end-to-end path from HOST memory: copies h_stack
 * ([S][rows][C] of dt) to device buffers owned by the plan (allocated on first
 * use), reconstructs, copies the result to h_out ([M][rows][C] float32) and
 * synchronises `cuda_stream`.  Pinned host buffers give full PCIe/C2C speed;
 * pageable buffers work too.
 * Device memory: with no budget set (daxm_set_host_budget) or a budget that holds the whole stack
 * and output, the plan keeps one device copy of both and overlaps band copies with the deposit.
 * Otherwise the call runs OUT OF CORE (the paper's row chunking, Fig. 2, and its
 * transfer stage): the rows are cut into bands of B rows (B a multiple of 128, the
 * largest whose two ring slots fit the budget), each band has its own plan (built on the first
 * such call, cached), and band b goes H2D into ring slot b mod 2, is reconstructed there and
 * returns D2H while band b + 1 arrives -- device memory O(band), not O(stack).  Output of
 * 128-aligned bands equals the whole-plan output bit for bit (same tiles, same kernels).
 * Errors: as daxm_reconstruct; OUT_OF_MEMORY when the budget cannot hold two 128-row slots. */
daxm_status daxm_reconstruct_host(daxm_plan *p, const void *h_stack, daxm_dtype dt, float *h_out,
                                  void *cuda_stream);

/* daxm_set_step_weights -- per-step intensity normalisation (SURVEY §8(f)4 "per-step I0
 * normalisation"; the paper is silent, reading R17 in DESIGN.md): with w (host pointer, S
 * finite positive doubles, copied) later reconstructions use dI_k = s (w_k I_k - w_{k+1} I_{k+1}),
 * e.g. w_k = I0_ref / I0_k from the beam monitor; w = NULL switches it off.  The cutoff still
 * compares the raw first image (reading R14).  Normalised plans run the general kernel (one
 * thread per pixel; the fast kernels stream raw intensities).  Errors: INVALID_ARGUMENT (a weight
 * not finite or <= 0), OUT_OF_MEMORY, CUDA. */
daxm_status daxm_set_step_weights(daxm_plan *p, const double *w);

/* daxm_set_host_budget -- cap, in bytes, on the device memory daxm_reconstruct_host may hold for
 * stack and output buffers (0 = no cap, the default).  Takes effect at the next host call; band
 * plans already built for another band height are rebuilt.  Errors: INVALID_ARGUMENT (NULL plan). */
daxm_status daxm_set_host_budget(daxm_plan *p, uint64_t device_bytes);

/* daxm_host_ring_info -- the out-of-core layout of the last daxm_reconstruct_host call: band rows
 * B and band count (both 0 when the call ran in core) and the device bytes of the two ring slots.
 * Any output pointer may be NULL. */
daxm_status daxm_host_ring_info(const daxm_plan *p, int64_t *band_rows, int64_t *n_bands, int64_t *ring_bytes);

/* daxm_set_cutoff -- intensity cutoff ("d_cutoff", kernel setTwo argument; the
 * pixel-percentage experiment).  Reading R14: with enable != 0 a
 * pixel is reconstructed only if its intensity in the FIRST wire-step image, I_0(p),
 * compared in float32, is >= cutoff; every other pixel's output column is 0 and the
 * pixel's inputs are not processed (a deposit tile with no such pixel reads no wire-step
 * planes; its output block is written as zeros by a row-wise fill).
 * enable == 0 (the default) reconstructs every pixel.  Applies to later daxm_reconstruct /
 * daxm_reconstruct_host calls on this plan.  Errors: INVALID_ARGUMENT (NaN cutoff). */
daxm_status daxm_set_cutoff(daxm_plan *p, int enable, double cutoff);

/* daxm_select_cutoff -- the cutoff that keeps a fraction of the plan's pixels: *cutoff =
 * the k-th largest I_0(p) over the plan's rows x C pixels, k = ceil(fraction * n) (>= 1),
 * so that at least k pixels pass daxm_set_cutoff(p, 1, *cutoff) (more on ties).  NaN
 * intensities rank lowest.  d_stack: device stack as for daxm_reconstruct (only plane 0 is
 * read).  Exact (radix select on the value's bits, on the device); synchronises the stream.
 * Errors: INVALID_ARGUMENT (NULL pointers, dtype, fraction outside (0, 1]), OUT_OF_MEMORY,
 * CUDA. */
daxm_status daxm_select_cutoff(daxm_plan *p, const void *d_stack, daxm_dtype dtype, double fraction, double *cutoff,
                               void *cuda_stream);

/* Sum-over-shards callback of daxm_select_cutoff_sharded: on return hist[0..n) must hold the
 * element-wise sum of every shard's hist (an all-reduce of n uint64 in host memory).  Returns 0
 * on success; anything else aborts the selection with INVALID_ARGUMENT. */
typedef int (*daxm_hist_reduce_fn)(unsigned long long *hist, int n, void *ctx);

/* daxm_select_cutoff_sharded -- daxm_select_cutoff over a detector split into row bands, one
 * plan per band (one rank per GPU): *cutoff = the k-th largest I_0 over ALL
 * bands, k = ceil(fraction * n_total) clamped to [1, n_total], n_total = the whole detector's
 * pixel count.  The radix select runs on every shard in lock step; after each 8-bit digit's
 * device histogram of this plan's rows, `reduce(hist, 256, ctx)` must sum it over the shards
 * (every shard calls it the same number of times: 2 for u16, 4 for f32), so every shard
 * returns the same cutoff, equal to daxm_select_cutoff of one plan over the whole detector.
 * Synchronises the stream.  Errors: as daxm_select_cutoff; INVALID_ARGUMENT also for a NULL
 * reduce, n_total below the plan's pixel count, or a failing callback. */
daxm_status daxm_select_cutoff_sharded(daxm_plan *p, const void *d_stack, daxm_dtype dtype, double fraction,
                                       unsigned long long n_total, daxm_hist_reduce_fn reduce, void *ctx,
                                       double *cutoff, void *cuda_stream);

/* daxm_depth_profile -- per-depth-bin total intensity of a reconstruction (the paper's
 * second output, image_set.depth_intensity, P:L208 / image_depth_intensity):
 * d_profile[m] = sum over the plan's rows and all columns of d_out[m][row][col], in fp64.
 * d_out: device [M][rows][C] float32 as written by daxm_reconstruct; d_profile: device
 * double[M], overwritten.  Stream ordered, no allocation.  For a row-sharded multi-GPU run
 * the per-rank profiles add up (an all-reduce of M doubles).
 * Errors: INVALID_ARGUMENT (NULL pointers), CUDA. */
daxm_status daxm_depth_profile(daxm_plan *p, const float *d_out, double *d_profile, void *cuda_stream);

/* daxm_reconstruct_profile -- daxm_reconstruct plus the depth profile of its output (as
 * daxm_depth_profile: d_profile[m] = sum over the plan's pixels of d_out[m][row][col], fp64),
 * fused: when every row tile runs the row-segment kernel (stats.row_path = 1, no general tiles,
 * one edge), the kernel sums each final plane of its tile while the plane is staged in shared
 * memory (an fp32 sum of the tile's 128 values) and one short kernel adds the tiles' sums in
 * fixed order, so the output is not read back.  Otherwise it runs daxm_reconstruct and then
 * daxm_depth_profile.  The first fused call allocates rows/2 * C/64 * M floats of plan memory.
 * Arguments, layouts and errors as daxm_reconstruct plus d_profile: device double[M],
 * overwritten (NULL: INVALID_ARGUMENT). */
daxm_status daxm_reconstruct_profile(daxm_plan *p, const void *d_stack, daxm_dtype dtype, float *d_out,
                                     double *d_profile, void *cuda_stream);

/* Detail text for the last failing call on this plan ("" if none).  Valid until
 * the next call on the plan. */
const char *daxm_last_error(const daxm_plan *p);
/* Detail text of the last daxm_create failure on the calling thread. */
const char *daxm_create_error(void);
const char *daxm_status_string(daxm_status s);
/* Frees all plan-owned device memory (synchronises the device first).  NULL is a no-op. */
void daxm_destroy(daxm_plan *p);
int daxm_abi_version(void);

#ifdef __cplusplus
}
#endif
#endif /* DAXM_H_ */
