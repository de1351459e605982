// deposit.cu -- gather-form deposit kernel.
//
// One thread owns one pixel and writes all M depth bins of it; no atomics
// (the paper's setTwo scatters with an fp64 CAS atomicAdd, P:L267-270,
// P:L334).  With the wire-step pairs visited in the order in which
// their trapezoids move deeper, the deposited intensity up to a bin edge E is
//
//   F(E) = sum_{pairs q with z4_q < E} dI_q  +  sum_{open pairs} dI_q H_q(E)/A_q
//
// (H the unit-height trapezoid CDF of device_get_trapezoid_height, P:L331,
// A its area), and bin m receives F(m+1) - F(m) -- exactly the
// trapezoid's area inside [lo_m, hi_m) (device_depth_resolve_pixel,
// P:L320-330), summed over pairs.  Pairs are opened / closed by two monotone
// pointers (the "step-range search" of SURVEY §8(a) step 4).
//
// v1: straightforward, one pass per bin edge, corner depths recomputed from
// the per-edge-point cubic for every use, stack read with plain global loads.
#include <cuda_runtime.h>
#include <stdint.h>

#include "daxm_internal.cuh"

namespace daxm {
namespace {

__device__ __forceinline__ float poly3(const float c[NCOEF], float tau) {
    return fmaf(fmaf(fmaf(c[3], tau, c[2]), tau, c[1]), tau, c[0]);
}

template <typename T>
__device__ __forceinline__ float load_px(const T* __restrict__ p) {
    return (float)__ldg(p);
}

struct PixelWalk {
    float cb[NCOEF], cf[NCOEF];
    const double* t;
    double t_ref;
    int kb, ke, dir;

    __device__ __forceinline__ int step_of(int q) const { return dir > 0 ? kb + q : ke - q; }
    __device__ __forceinline__ void point(int q, float& lo, float& hi) const {
        const float tau = (float)(t[step_of(q)] - t_ref);
        const float a = poly3(cb, tau), b = poly3(cf, tau);
        lo = fminf(a, b);
        hi = fmaxf(a, b);
    }
};

// Unit-height trapezoid CDF at E divided by its area: corners from points q, q+1.
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

template <typename T>
__global__ void __launch_bounds__(256) deposit_v1(DepositArgs a, const T* __restrict__ stack, float* __restrict__ out) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    const int jl = blockIdx.y * blockDim.y + threadIdx.y;
    const int rows = a.row_end - a.row_begin;
    if (i >= a.C || jl >= rows) return;
    const int j = a.row_begin + jl;
    const size_t plane = (size_t)rows * a.C;
    const int tr = j / TILE_R - a.tr0, tc = i / TILE_C;
    const int tile = tr * a.n_tc + tc;
    const TileInfo ti = a.tiles[tile];
    const int2 w = a.win[(size_t)(j - a.pre_row0) * a.C + i];
    PixelWalk pw;
    const int r = j % TILE_R, eb = i % TILE_C, ef = a.point_mode ? eb : eb + 1;
#pragma unroll
    for (int m = 0; m < NCOEF; ++m) {
        pw.cb[m] = a.coef[(((size_t)tile * NCOEF + m) * TILE_E + eb) * TILE_R + r];
        pw.cf[m] = a.coef[(((size_t)tile * NCOEF + m) * TILE_E + ef) * TILE_R + r];
    }
    pw.t = a.t;
    pw.t_ref = ti.t_ref;
    pw.kb = w.x;
    pw.ke = w.y;
    pw.dir = ti.dir;
    const int n = w.y - w.x;  // pairs
    const T* px = stack + (size_t)jl * a.C + i;
    const float sgn = a.sign * (float)ti.dir;
    auto dI = [&](int q) -> float {
        return sgn * (load_px(px + (size_t)pw.step_of(q) * plane) - load_px(px + (size_t)pw.step_of(q + 1) * plane));
    };
    int qc = 0, qo = 0;
    float P = 0.f, F_prev = 0.f;
    float* o = out + (size_t)jl * a.C + i;
    for (int e = 0; e <= a.M; ++e) {
        const float E = (float)(e - a.m_ref);
        // close pairs whose trapezoid lies entirely below E
        while (qc < n) {
            float lo1, hi1, lo2, hi2;
            pw.point(qc, lo1, hi1);
            pw.point(qc + 1, lo2, hi2);
            if (fmaxf(hi1, hi2) < E) {
                P += dI(qc);
                ++qc;
            } else {
                break;
            }
        }
        // open pairs whose trapezoid starts below E
        if (qo < qc) qo = qc;
        while (qo < n) {
            float lo1, hi1, lo2, hi2;
            pw.point(qo, lo1, hi1);
            pw.point(qo + 1, lo2, hi2);
            if (fminf(lo1, lo2) < E)
                ++qo;
            else
                break;
        }
        float F = P;
        for (int q = qc; q < qo; ++q) {
            float lo1, hi1, lo2, hi2;
            pw.point(q, lo1, hi1);
            pw.point(q + 1, lo2, hi2);
            const float d = dI(q);
            if (d != 0.f) F += d * trapezoid_fraction(lo1, hi1, lo2, hi2, E);
        }
        if (e > 0) o[(size_t)(e - 1) * plane] = F - F_prev;
        F_prev = F;
    }
}

}  // namespace

cudaError_t launch_deposit(const DepositArgs& a, const void* stack, int dtype, float* out, cudaStream_t st) {
    const int rows = a.row_end - a.row_begin;
    dim3 blk(32, 8), grd((a.C + 31) / 32, (rows + 7) / 8);
    if (dtype == DAXM_U16)
        deposit_v1<uint16_t><<<grd, blk, 0, st>>>(a, static_cast<const uint16_t*>(stack), out);
    else
        deposit_v1<float><<<grd, blk, 0, st>>>(a, static_cast<const float*>(stack), out);
    return cudaGetLastError();
}

}  // namespace daxm
