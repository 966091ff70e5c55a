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

#ifndef SIGATTN_SIGMA_TIER4
#define SIGATTN_SIGMA_TIER4 1   // linear-R tier for chunks whose logits are all <= -4
#endif

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

// ---------------------------------------------------------------------------------------------
// Fast path for the common regime x <= -2 (sigma <= 0.12; with b = -log n almost every logit):
//   u = e^x = 2^(x log2 e)  (one MUFU op),  sigma(x) = u / (1 + u) = u R(u),
//   R(u) ~ c0 + c1 u + c2 u^2 on u in [0, e^-2]: minimax, max relative error 6.4e-5 (< 2^-14).
// No reciprocal, no clamp (u <= e^-2; u -> 0 as x -> -inf), 4 issue slots per element pair fewer
// than sigma2.  A warp takes it only when every logit of its chunk satisfies x <= -2 (max(t) test,
// t = x log2 e); otherwise the exact-range path sigma2 runs.
constexpr float kFastT = -2.8853900817779268f;   // -2 log2(e)
constexpr float kR0 = 0.9999361611215778f, kR1 = -0.9914453981504439f, kR2 = 0.8241421343752648f;
// Narrower regime x <= -4 (u <= e^-4; with b = -log n nearly every logit): sigma = u / (1 + u) =
// u - u^2 + u^3 - ...  ~  u - u^2, ONE fused multiply-add per element (u (-u) + u); relative error
// u^2 <= e^-8 = 3.4e-4 (at the tier boundary, far smaller for typical logits near b), below a sixth
// of the bf16 rounding of P (2^-9).  The sigma path is bound by the issue mix around the MUFU ex2,
// so every FMA-pipe op per pair counts.
constexpr float kFastT4 = -5.7707801635558535f;  // -4 log2(e)

__device__ __forceinline__ float fmax3(float a, float b, float c) {
  float d;
  asm("max.f32 %0, %1, %2, %3;" : "=f"(d) : "f"(a), "f"(b), "f"(c));
  return d;
}

// p = sigma(x) for t = x log2 e <= kFastT.
__device__ __forceinline__ void sigma2_fast(float t0, float t1, float& p0, float& p1) {
  const float u0 = ex2_ftz(t0), u1 = ex2_ftz(t1);
  float r0, r1;
  ffma2(r0, r1, u0, u1, kR2, kR2, kR1, kR1);        // c1 + c2 u
  ffma2(r0, r1, r0, r1, u0, u1, kR0, kR0);          // c0 + u (c1 + c2 u)
  fmul2(p0, p1, r0, r1, u0, u1);                    // u R(u)
}

__device__ __forceinline__ void fadd2(float& d0, float& d1, float a0, float a1, float b0, float b1) {
  asm("{.reg .b64 ra, rb, rd;\n\t"
      "mov.b64 ra, {%2, %3};\n\tmov.b64 rb, {%4, %5};\n\t"
      "add.rn.f32x2 rd, ra, rb;\n\tmov.b64 {%0, %1}, rd;}"
      : "=f"(d0), "=f"(d1)
      : "f"(a0), "f"(a1), "f"(b0), "f"(b1));
}

// 2^t on the FMA pipe (no MUFU), for t <= kFastT: t = j + f with j = rint(t) (magic-number
// rounding) and f in [-1/2, 1/2];  2^f ~ E(f), a degree-3 relative-minimax polynomial (max rel.
// error 7.5e-5);  the exponent j is added to E's bit pattern with one integer multiply-add.
// t is clamped at -125 so that the exponent field cannot underflow (sigma < 2^-125 rounds to 0).
// Used for a fixed subset of the element pairs so that the MUFU and FMA pipes share the exp2 work.
constexpr float kE0 = 0.9999280735404956f, kE1 = 0.6932609854573364f, kE2 = 0.24261112219433045f,
                kE3 = 0.05517166907486297f;
constexpr float kRoundMagic = 12582912.0f;   // 1.5 * 2^23
__device__ __forceinline__ void exp2_fma2(float t0, float t1, float& u0, float& u1) {
  t0 = fmaxf(t0, -125.0f);
  t1 = fmaxf(t1, -125.0f);
  float y0, y1, j0, j1, f0, f1, e0, e1;
  fadd2(y0, y1, t0, t1, kRoundMagic, kRoundMagic);          // low mantissa bits of y = rint(t)
  fadd2(j0, j1, y0, y1, -kRoundMagic, -kRoundMagic);        // rint(t)
  ffma2(f0, f1, j0, j1, -1.0f, -1.0f, t0, t1);              // f = t - rint(t)
  ffma2(e0, e1, f0, f1, kE3, kE3, kE2, kE2);
  ffma2(e0, e1, e0, e1, f0, f1, kE1, kE1);
  ffma2(e0, e1, e0, e1, f0, f1, kE0, kE0);
  // bits(2^t) = bits(E) + j << 23;  bits(y) = 0x4B400000 + j and 0x4B400000 << 23 == 0 (mod 2^32)
  u0 = __uint_as_float(__float_as_uint(y0) * (1u << 23) + __float_as_uint(e0));
  u1 = __uint_as_float(__float_as_uint(y1) * (1u << 23) + __float_as_uint(e1));
}

// sigma2_fast with the exp2 on the FMA pipe.
__device__ __forceinline__ void sigma2_fast_fma(float t0, float t1, float& p0, float& p1) {
  float u0, u1;
  exp2_fma2(t0, t1, u0, u1);
  float r0, r1;
  ffma2(r0, r1, u0, u1, kR2, kR2, kR1, kR1);
  ffma2(r0, r1, r0, r1, u0, u1, kR0, kR0);
  fmul2(p0, p1, r0, r1, u0, u1);
}

// p = sigma(x) for t = x log2 e <= kFastT4.
__device__ __forceinline__ void sigma2_fast4(float t0, float t1, float& p0, float& p1) {
  const float u0 = ex2_ftz(t0), u1 = ex2_ftz(t1);
  ffma2(p0, p1, u0, u1, -u0, -u1, u0, u1);          // u - u^2
}

// p = sigma(x) from t = x log2 e, any range (the reciprocal path of sigma2).
__device__ __forceinline__ void sigma2_from_t(float t0, float t1, float& p0, float& p1) {
  // 1 / (1 + 2^-t), with -t clamped at 126 so that 1 + 2^-t stays finite
  const float e0 = ex2_ftz(fminf(-t0, 126.0f)), e1 = ex2_ftz(fminf(-t1, 126.0f));
  float n0, n1;
  ffma2(n0, n1, e0, e1, -1.0f, -1.0f, -1.0f, -1.0f);
  float r0 = __uint_as_float(0xFEF311C3u - __float_as_uint(n0));
  float r1 = __uint_as_float(0xFEF311C3u - __float_as_uint(n1));
  float u0, u1;
  ffma2(u0, u1, n0, n1, r0, r1, 1.0f, 1.0f);
  ffma2(r0, r1, r0, r1, u0, u1, r0, r1);
  ffma2(u0, u1, n0, n1, r0, r1, 1.0f, 1.0f);
  ffma2(r0, r1, r0, r1, u0, u1, r0, r1);
  p0 = r0;
  p1 = r1;
}

// Speculative form of the common case: N scores of one row -> N values of the <= -4 tier (in place),
// (callers speculate only while the previous chunk of the warp took tier 4: when the bias is mild
// -- b = -log n for short sequences -- the vote fails often and speculation would double the work)
// evaluated BEFORE the warp vote, so the max/vote chain runs beside the MUFU work instead of in front
// of it.  Returns the vote: true iff every valid logit of the warp's chunk is <= -4, i.e. the values
// are the tier-4 sigma.  On false the caller must redo the chunk from its scores with sigma_row
// (the scores are gone: callers reload them from TMEM, where they are still intact).  The vote looks
// only at valid elements, as in sigma_row, so the choice never depends on pad content.
template <int N, bool kMask = false>
__device__ __forceinline__ bool sigma_row_spec4(float (&v)[N], float a, float c, bool lane_valid = true,
                                                int nvalid = N) {
  float m = -INFINITY;
#pragma unroll
  for (int e = 0; e < N; e += 2) {
    ffma2(v[e], v[e + 1], v[e], v[e + 1], a, a, c, c);
    if constexpr (kMask)
      m = fmax3(m, e < nvalid ? v[e] : -INFINITY, e + 1 < nvalid ? v[e + 1] : -INFINITY);
    else
      m = fmax3(m, v[e], v[e + 1]);
  }
#pragma unroll
  for (int e = 0; e < N; e += 2) {
    sigma2_fast4(v[e], v[e + 1], v[e], v[e + 1]);
    // materialise the speculative values here: keeps the compiler from sinking them into the branch
    // after the vote (which would put the vote back in front of the MUFU work)
    asm volatile("" : "+f"(v[e]), "+f"(v[e + 1]));
  }
  return __all_sync(0xffffffffu, !lane_valid || m <= kFastT4);
}

// N scores of one row -> N sigma values (in place), choosing the path warp-uniformly.
// a = alpha log2 e, c = b log2 e (so t = x log2 e = s a + c).  The path vote only looks at valid
// elements (lane_valid rows, columns < nvalid when kMask): padding can never change which
// arithmetic the valid outputs see, so results stay bitwise independent of pad content.
// kEmuEvery > 0: in the fast path, element pairs with index % kEmuEvery == kEmuEvery / 2 take the
// FMA-pipe exp2 (exp2_fma2) instead of MUFU ex2, off-loading the MUFU unit (16 ops/clk/SM).
// Returns the tier taken (warp-uniform): 4 (all valid logits <= -4), 2 (<= -2) or 0 (exact range).
template <int N, bool kMask = false, int kEmuEvery = 0>
__device__ __forceinline__ int sigma_row(float (&v)[N], float a, float c, bool lane_valid = true, int nvalid = N) {
  float m = -INFINITY;
#pragma unroll
  for (int e = 0; e < N; e += 2) {
    ffma2(v[e], v[e + 1], v[e], v[e + 1], a, a, c, c);
    if constexpr (kMask)
      m = fmax3(m, e < nvalid ? v[e] : -INFINITY, e + 1 < nvalid ? v[e + 1] : -INFINITY);
    else
      m = fmax3(m, v[e], v[e + 1]);
  }
  if (SIGATTN_SIGMA_TIER4 && __all_sync(0xffffffffu, !lane_valid || m <= kFastT4)) {
#pragma unroll
    for (int e = 0; e < N; e += 2) sigma2_fast4(v[e], v[e + 1], v[e], v[e + 1]);
    return 4;
  } else if (__all_sync(0xffffffffu, !lane_valid || m <= kFastT)) {
#pragma unroll
    for (int e = 0; e < N; e += 2) {
      if (kEmuEvery > 0 && (e / 2) % (kEmuEvery > 0 ? kEmuEvery : 1) == kEmuEvery / 2)
        sigma2_fast_fma(v[e], v[e + 1], v[e], v[e + 1]);
      else
        sigma2_fast(v[e], v[e + 1], v[e], v[e + 1]);
    }
    return 2;
  } else {
#pragma unroll
    for (int e = 0; e < N; e += 2) sigma2_from_t(v[e], v[e + 1], v[e], v[e + 1]);
    return 0;
  }
}


}  // namespace sigattn
