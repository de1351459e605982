// fp2.cuh -- packed fp32x2 arithmetic (sm_100a FADD2 / FMUL2 / FFMA2, per-component IEEE
// round-to-nearest, so a packed result equals the two scalar results bit for bit) used by the
// deposit kernels to advance two pixel walks per instruction.  Internal; not part of the ABI.
#pragma once
#include <cuda_runtime.h>

namespace daxm {

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
__device__ __forceinline__ float2 abs2(float2 a) { return make_float2(fabsf(a.x), fabsf(a.y)); }
__device__ __forceinline__ float2 floor2(float2 a) { return make_float2(floorf(a.x), floorf(a.y)); }
__device__ __forceinline__ float2 f2(float v) { return make_float2(v, v); }
// depth of an edge point at wire travel t: c0 + t (c1 + t c2), the expression the pre-pass verifies
__device__ __forceinline__ float2 poly2(const float2 c[3], float2 t) { return fma2(fma2(c[2], t, c[1]), t, c[0]); }
__device__ __forceinline__ float rcp_approx_f(float x) {
    float y;
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}
__device__ __forceinline__ float2 rcp2(float2 x) { return make_float2(rcp_approx_f(x.x), rcp_approx_f(x.y)); }

}  // namespace daxm
