/*
 * daxm_oracle.c -- plain, slow, double-precision CPU ORACLE for wire-scan
 * (differential-aperture) depth reconstruction, arXiv:2201.13309.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and the
 * cpu_baseline / --impl reference legs of bench.py may load this library.
 * It shares no code, header, table or constant generator with the CUDA path
 * (paper_2201_13309_b200/), and neither side includes the other.
 *
 * What it computes follows the paper step by step (citations are
 * PAPER.md line numbers, "P:Lnnn", and the readings collected in SURVEY.md
 * §8(c) / DESIGN.md "Readings"):
 *
 *   for every pixel (row j, col i), every wire-step pair k = 0..S-2   [P:L255-262; reading R9]
 *     dI   = s * (I_k - I_{k+1})                                      [P:L264-266; R1, R2]
 *     four corner depths  D(back,W_k) D(front,W_k) D(back,W_k+1) D(front,W_k+1)
 *          by a ray from the pixel edge, tangent to the wire edge, to
 *          the incident beam ("depth measured along the beam")        [Fig.7; P:L342-343]
 *     sort -> z1<=z2<=z3<=z4, trapezoid of unit height, area A         [device_get_trapezoid_height P:L331,346; Area P:L321]
 *     for the depth bins it overlaps: out[m] += dI * (H(hi_m)-H(lo_m)) / A
 *                                                                    [device_depth_resolve_pixel P:L320-330, 338-341;
 *                                                                     device_index_to_beam_depth P:L330,344-345;
 *                                                                     device_add_pixel_intensity_at_index P:L332-333,347]
 *
 * Loop order is j, i, k, m; no blocking, no reordering.  OpenMP only splits
 * the outermost pixel loop across host threads (each pixel's arithmetic is
 * unchanged).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#ifdef _OPENMP
#include <omp.h>
#endif

/* ---- the oracle's own geometry struct (NOT the library's daxm_geometry) ---- */
typedef struct {
    int32_t n_rows, n_cols;
    double pitch_col, pitch_row;   /* um per pixel along x' (col) and y' (row)             */
    double det_rot[3];             /* Rodrigues vector, rad                                  */
    double det_trans[3];           /* um; lab = rho * ((x', y', 0) + det_trans)              */
    double beam_dir[3];            /* k-hat (normalised here)                                */
    double beam_origin[3];         /* depth origin O                                         */
    double wire_axis[3];           /* a-hat (normalised here)                                */
    double wire_radius;            /* r, um                                                  */
    int32_t n_steps;               /* S                                                      */
    const double *wire_xyz;        /* [S][3] wire-centre positions W_k                       */
    double depth_start, depth_end, depth_res;
    int32_t edge;                  /* 0 leading, 1 trailing, 2 both (reading R16)            */
    int32_t pixel_model;           /* 0 finite (trapezoid), 1 point (box)                    */
    int32_t raw_sign;              /* 1: s = +1 even for trailing (used by identity tests)   */
    const double *step_weight;     /* NULL, or [S] per-step intensity normalisation w_k      */
                                   /* (SURVEY §8(f)4 "per-step I0 normalisation"; the paper */
                                   /* is silent, reading R17: dI = s (w_k I_k - w_k+1 I_k+1)) */
} oracle_geometry;

enum { ORC_OK = 0, ORC_ERR_ARG = 1 };

/* ---------------------------------------------------------------- vectors */
static double dot3(const double *a, const double *b) { return a[0] * b[0] + a[1] * b[1] + a[2] * b[2]; }
static void cross3(const double *a, const double *b, double *c) {
    c[0] = a[1] * b[2] - a[2] * b[1];
    c[1] = a[2] * b[0] - a[0] * b[2];
    c[2] = a[0] * b[1] - a[1] * b[0];
}
static void unit3(const double *a, double *u) {
    double n = sqrt(dot3(a, a));
    u[0] = a[0] / n; u[1] = a[1] / n; u[2] = a[2] / n;
}

/* Step 1 (reading R5): rho = I + sin(th) K + (1-cos th) K^2. */
void oracle_rodrigues(const double R[3], double rho[9]) {
    double th = sqrt(dot3(R, R));
    if (th == 0.0) {
        for (int i = 0; i < 9; ++i) rho[i] = (i % 4 == 0) ? 1.0 : 0.0;
        return;
    }
    double k[3] = {R[0] / th, R[1] / th, R[2] / th};
    double K[9] = {0, -k[2], k[1], k[2], 0, -k[0], -k[1], k[0], 0};
    double K2[9];
    for (int r = 0; r < 3; ++r)
        for (int c = 0; c < 3; ++c) {
            double s = 0;
            for (int t = 0; t < 3; ++t) s += K[r * 3 + t] * K[t * 3 + c];
            K2[r * 3 + c] = s;
        }
    double s = sin(th), c1 = 1.0 - cos(th);
    for (int i = 0; i < 9; ++i) rho[i] = ((i % 4 == 0) ? 1.0 : 0.0) + s * K[i] + c1 * K2[i];
}

/* Lab-frame position of detector point (x, j): x = column coordinate (may be a
 * half-integer pixel edge), j = row.  Pixel centre i sits at
 * x' = (i - (C-1)/2) * pitch_col  (reading R5). */
void oracle_detector_point(const oracle_geometry *g, double x, double j, double out[3]) {
    double rho[9];
    oracle_rodrigues(g->det_rot, rho);
    double p[3] = {(x - 0.5 * (g->n_cols - 1)) * g->pitch_col + g->det_trans[0],
                   (j - 0.5 * (g->n_rows - 1)) * g->pitch_row + g->det_trans[1],
                   g->det_trans[2]};
    for (int r = 0; r < 3; ++r) out[r] = rho[r * 3 + 0] * p[0] + rho[r * 3 + 1] * p[1] + rho[r * 3 + 2] * p[2];
}

/* Step 3: tangent depth D(Q, W, sigma)  (paper's 2-D version
 * P:L306-319 `pixel_to_wireCenter_y/_z/_len`, `Dphi`, `Depth`).
 *   e = (Q-W) - ((Q-W).a) a,  L^2 = e.e
 *   n = (r e + sigma sqrt(L^2 - r^2) (a x e)) / L^2     (unit, n.(Q-W) = r)
 *   D = (n.(W-O) + r) / (n.k)
 * NaN if L <= r or |n.k| < 1e-12.  `axis`, `beam` must be unit vectors. */
double oracle_tangent_depth(const double Q[3], const double W[3], const double axis[3], double r,
                            double sigma, const double beam[3], const double origin[3]) {
    double qw[3] = {Q[0] - W[0], Q[1] - W[1], Q[2] - W[2]};
    double pa = dot3(qw, axis);
    double e[3] = {qw[0] - pa * axis[0], qw[1] - pa * axis[1], qw[2] - pa * axis[2]};
    double L2 = dot3(e, e);
    if (!(L2 > r * r)) return NAN;
    double s = sqrt(L2 - r * r);
    double axe[3];
    cross3(axis, e, axe);
    double n[3];
    for (int t = 0; t < 3; ++t) n[t] = (r * e[t] + sigma * s * axe[t]) / L2;
    double nk = dot3(n, beam);
    if (fabs(nk) < 1e-12) return NAN;
    double wo[3] = {W[0] - origin[0], W[1] - origin[1], W[2] - origin[2]};
    return (dot3(n, wo) + r) / nk;
}

/* Step 4: edge side sigma for an edge point Q (reading R3).
 * d = (W_{S-1} - W_0) projected perpendicular to a.  sigma_lead = sign((a x (Q-W_0)).d),
 * +1 when the product is >= 0; trailing uses -sigma_lead. */
double oracle_edge_sigma(const double Q[3], const double W0[3], const double Wlast[3], const double axis[3],
                         int edge) {
    double dd[3] = {Wlast[0] - W0[0], Wlast[1] - W0[1], Wlast[2] - W0[2]};
    double pa = dot3(dd, axis);
    double d[3] = {dd[0] - pa * axis[0], dd[1] - pa * axis[1], dd[2] - pa * axis[2]};
    double qw[3] = {Q[0] - W0[0], Q[1] - W0[1], Q[2] - W0[2]};
    double c[3];
    cross3(axis, qw, c);
    double lead = (dot3(c, d) >= 0.0) ? 1.0 : -1.0;
    return edge == 1 ? -lead : lead;
}

/* Step 5.5: unit-height trapezoid CDF H(z) with corners z1<=z2<=z3<=z4
 * (device_get_trapezoid_height, P:L331 / P:L346). */
double oracle_trapezoid_cdf(const double z[4], double x) {
    double z1 = z[0], z2 = z[1], z3 = z[2], z4 = z[3];
    if (x <= z1) return 0.0;
    if (x <= z2) return (x - z1) * (x - z1) / (2.0 * (z2 - z1));
    if (x <= z3) return 0.5 * (z2 - z1) + (x - z2);
    if (x <= z4) return 0.5 * (z2 - z1) + (z3 - z2) + 0.5 * (z4 - z3) - (z4 - x) * (z4 - x) / (2.0 * (z4 - z3));
    return 0.5 * (z4 + z3 - z2 - z1);
}

/* Steps 5.2-5.6 for one step pair: deposit dI with corner depths c[4] into
 * out[0..M-1] (stride `stride`).  Bins (reading R6): lo_m = start + (m - 1/2) dz,
 * hi_m = lo_m + dz.  Trapezoid parts outside [lo_0, hi_{M-1}] are dropped (R7).
 * Degenerate z4 == z1 -> all of dI into the bin containing z1 (R8). */
void oracle_deposit_pair(double dI, const double c[4], double start, double dz, int M, double *out,
                         long stride) {
    double z[4] = {c[0], c[1], c[2], c[3]};
    /* sort the four corners (insertion sort) */
    for (int a = 1; a < 4; ++a) {
        double v = z[a];
        int b = a - 1;
        while (b >= 0 && z[b] > v) { z[b + 1] = z[b]; --b; }
        z[b + 1] = v;
    }
    double lo0 = start - 0.5 * dz;
    double A = 0.5 * (z[3] + z[2] - z[1] - z[0]); /* `Area` */
    if (z[3] == z[0]) {
        double f = floor((z[0] - lo0) / dz);
        if (f >= 0.0 && f <= (double)(M - 1)) out[(long)f * stride] += dI;
        return;
    }
    double fl = floor((z[0] - lo0) / dz), fh = floor((z[3] - lo0) / dz);
    long m0 = fl < 0.0 ? 0 : (long)fl;
    long m1 = fh > (double)(M - 1) ? (long)(M - 1) : (long)fh;
    for (long m = m0; m <= m1; ++m) {
        double lo = start + ((double)m - 0.5) * dz; /* device_index_to_beam_depth */
        double hi = lo + dz;
        out[m * stride] += dI * (oracle_trapezoid_cdf(z, hi) - oracle_trapezoid_cdf(z, lo)) / A;
    }
}

static int geometry_ok(const oracle_geometry *g) {
    if (!g || g->n_rows < 1 || g->n_cols < 1 || g->n_steps < 2 || !g->wire_xyz) return 0;
    if (g->edge < 0 || g->edge > 2) return 0;
    if (!(g->depth_res > 0.0) || !(g->depth_end >= g->depth_start) || !(g->wire_radius > 0.0)) return 0;
    return 1;
}

int oracle_n_bins(const oracle_geometry *g) {
    return (int)lround((g->depth_end - g->depth_start) / g->depth_res) + 1;
}

/* Reconstruct a list of pixels.  series[p*S + k] = I_k at pixel (rows[p], cols[p])
 * (double), out[p*M + m] (double, overwritten). */
int oracle_reconstruct_pixels(const oracle_geometry *g, int n_pix, const int32_t *rows, const int32_t *cols,
                              const double *series, double *out, int n_threads) {
    if (!geometry_ok(g) || n_pix < 0 || (n_pix > 0 && (!rows || !cols || !series || !out))) return ORC_ERR_ARG;
    const int S = g->n_steps, M = oracle_n_bins(g);
    double axis[3], beam[3];
    unit3(g->wire_axis, axis);
    unit3(g->beam_dir, beam);
    const double *W0 = g->wire_xyz, *Wl = g->wire_xyz + 3 * (S - 1);
    /* edges run: the plan's one, or both (reading R16: leading takes the intensity decreases,
     * trailing the sign-normalised increases, and the two reconstructions add) */
    const int e_first = g->edge == 2 ? 0 : g->edge, e_last = g->edge == 2 ? 1 : g->edge;
#ifdef _OPENMP
    if (n_threads > 0) omp_set_num_threads(n_threads);
#pragma omp parallel for schedule(dynamic, 16)
#endif
    for (int p = 0; p < n_pix; ++p) {
        double *o = out + (long)p * M;
        for (int m = 0; m < M; ++m) o[m] = 0.0;
        const double *I = series + (long)p * S;
        /* Step 2 (reading R4): pixel edges along the column axis. */
        double back[3], front[3];
        if (g->pixel_model == 1) {
            oracle_detector_point(g, cols[p], rows[p], back);
            memcpy(front, back, sizeof back);
        } else {
            oracle_detector_point(g, cols[p] - 0.5, rows[p], back);
            oracle_detector_point(g, cols[p] + 0.5, rows[p], front);
        }
        for (int e = e_first; e <= e_last; ++e) {
        const double s = (e == 1 && !g->raw_sign) ? -1.0 : 1.0; /* reading R2 */
        double sb = oracle_edge_sigma(back, W0, Wl, axis, e);
        double sf = oracle_edge_sigma(front, W0, Wl, axis, e);
        for (int k = 0; k + 1 < S; ++k) {
            const double wa = g->step_weight ? g->step_weight[k] : 1.0, wb = g->step_weight ? g->step_weight[k + 1] : 1.0;
            double dI = s * (wa * I[k] - wb * I[k + 1]); /* reading R17 (w = 1 without normalisation) */
            if (g->edge == 2 && dI < 0.0) dI = 0.0; /* reading R16: each edge its own sign of change */
            if (dI == 0.0) continue;
            const double *Wa = g->wire_xyz + 3 * k, *Wb = g->wire_xyz + 3 * (k + 1);
            /* Fig. 7: full_start, partial_start, partial_end, full_end */
            double c[4] = {oracle_tangent_depth(back, Wa, axis, g->wire_radius, sb, beam, g->beam_origin),
                           oracle_tangent_depth(front, Wa, axis, g->wire_radius, sf, beam, g->beam_origin),
                           oracle_tangent_depth(back, Wb, axis, g->wire_radius, sb, beam, g->beam_origin),
                           oracle_tangent_depth(front, Wb, axis, g->wire_radius, sf, beam, g->beam_origin)};
            if (isnan(c[0]) || isnan(c[1]) || isnan(c[2]) || isnan(c[3])) continue; /* reading R8 */
            oracle_deposit_pair(dI, c, g->depth_start, g->depth_res, M, o, 1);
        }
        }
    }
    return ORC_OK;
}

/* Whole image: stack [S][R][C] of dtype (0 = uint16, 1 = float32, 2 = float64),
 * out [M][R][C] double.  Rows [row_begin, row_end) only (others untouched). */
int oracle_reconstruct(const oracle_geometry *g, const void *stack, int dtype, double *out, int row_begin,
                       int row_end, int n_threads) {
    if (!geometry_ok(g) || !stack || !out || row_begin < 0 || row_end > g->n_rows || row_begin > row_end)
        return ORC_ERR_ARG;
    const int S = g->n_steps, M = oracle_n_bins(g), C = g->n_cols;
    const long plane = (long)g->n_rows * C;
    const int nr = row_end - row_begin;
    const long n_pix = (long)nr * C;
    int32_t *rows = malloc(sizeof(int32_t) * n_pix), *cols = malloc(sizeof(int32_t) * n_pix);
    double *series = malloc(sizeof(double) * n_pix * S), *res = malloc(sizeof(double) * n_pix * M);
    if (!rows || !cols || !series || !res) {
        free(rows); free(cols); free(series); free(res);
        return ORC_ERR_ARG;
    }
    for (long p = 0; p < n_pix; ++p) {
        int j = row_begin + (int)(p / C), i = (int)(p % C);
        rows[p] = j; cols[p] = i;
        for (int k = 0; k < S; ++k) {
            long idx = (long)k * plane + (long)j * C + i;
            double v = dtype == 0 ? (double)((const uint16_t *)stack)[idx]
                     : dtype == 1 ? (double)((const float *)stack)[idx] : ((const double *)stack)[idx];
            series[p * S + k] = v;
        }
    }
    int st = oracle_reconstruct_pixels(g, (int)n_pix, rows, cols, series, res, n_threads);
    if (st == ORC_OK)
        for (long p = 0; p < n_pix; ++p)
            for (int m = 0; m < M; ++m) out[(long)m * plane + (long)rows[p] * C + cols[p]] = res[p * M + m];
    free(rows); free(cols); free(series); free(res);
    return st;
}

int oracle_max_threads(void) {
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}
