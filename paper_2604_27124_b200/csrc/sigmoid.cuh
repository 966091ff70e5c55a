// sigmoid.cuh -- the element-wise part of the hot loop: scale + bias + sigma, two elements at a time.
//
//   x = alpha s + b;   sigma(x) = 1 / (1 + 2^t),  t = -x log2(e) = s * (-alpha log2 e) + (-b log2 e)
//
// One MUFU op per element (ex2.approx); the reciprocal runs on the FMA pipe: a bit-trick seed
// (max rel. error 0.10) refined by two Newton steps r <- r + r (1 - y r)  (max rel. error 1.04e-4,
// always from below, mean bias -3e-6 -- far inside the bf16 rounding of P, 2^-9).  The sums use
// packed FFMA2 (fma.rn.f32x2) so a pair costs 5 FMA-pipe issues.  t is clamped at 126 so that
// y = 1 + 2^t stays finite (sigma(x) < 2^-126 there, i.e. 0 after rounding to bf16/fp16).
// Accuracy rationale: DESIGN.md "sigma evaluation" (the tanh.approx form of P:130 fails parity at
// b = -log N through cancellation; this form has no cancellation).
#pragma once
#include <stdint.h>

namespace sigattn {

__device__ __forceinline__ void ffma2(float& d0, float& d1, float a0, float a1, float b0, float b1, float c0,
                                      float c1) {
  asm("{.reg .b64 ra, rb, rc, rd;\n\t"
      "mov.b64 ra, {%2, %3};\n\tmov.b64 rb, {%4, %5};\n\tmov.b64 rc, {%6, %7};\n\t"
      "fma.rn.f32x2 rd, ra, rb, rc;\n\tmov.b64 {%0, %1}, rd;}"
      : "=f"(d0), "=f"(d1)
      : "f"(a0), "f"(a1), "f"(b0), "f"(b1), "f"(c0), "f"(c1));
}
__device__ __forceinline__ void fmul2(float& d0, float& d1, float a0, float a1, float b0, float b1) {
  asm("{.reg .b64 ra, rb, rd;\n\t"
      "mov.b64 ra, {%2, %3};\n\tmov.b64 rb, {%4, %5};\n\t"
      "mul.rn.f32x2 rd, ra, rb;\n\tmov.b64 {%0, %1}, rd;}"
      : "=f"(d0), "=f"(d1)
      : "f"(a0), "f"(a1), "f"(b0), "f"(b1));
}

__device__ __forceinline__ float ex2_ftz(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

// p = sigma(alpha s + b) for two scores; a2 = -alpha log2 e, b2 = -b log2 e.
__device__ __forceinline__ void sigma2(float s0, float s1, float a2, float b2, float& p0, float& p1) {
  float t0, t1;
  ffma2(t0, t1, s0, s1, a2, a2, b2, b2);
  t0 = fminf(t0, 126.0f);
  t1 = fminf(t1, 126.0f);
  const float e0 = ex2_ftz(t0), e1 = ex2_ftz(t1);
  float n0, n1;                                     // n = -(1 + e) = -y
  ffma2(n0, n1, e0, e1, -1.0f, -1.0f, -1.0f, -1.0f);
  // seed: bits(1/y) ~ 0x7EF311C3 - bits(y) = 0xFEF311C3 - bits(-y)
  float r0 = __uint_as_float(0xFEF311C3u - __float_as_uint(n0));
  float r1 = __uint_as_float(0xFEF311C3u - __float_as_uint(n1));
  float u0, u1;
  ffma2(u0, u1, n0, n1, r0, r1, 1.0f, 1.0f);        // u = 1 - y r
  ffma2(r0, r1, r0, r1, u0, u1, r0, r1);            // r = r + r u
  ffma2(u0, u1, n0, n1, r0, r1, 1.0f, 1.0f);
  ffma2(r0, r1, r0, r1, u0, u1, r0, r1);
  p0 = r0;
  p1 = r1;
}

}  // namespace sigattn
