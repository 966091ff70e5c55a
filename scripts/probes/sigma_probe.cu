// sigma_probe.cu -- throughput of sigmoid formulations on sm_100a (debug tool).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I../../paper_2604_27124_b200/csrc sigma_probe.cu -o sigma_probe
#include <cstdio>
#include "sigmoid.cuh"
#include "sm100.cuh"
using namespace sigattn;

// variant 0: production sigma2 (ex2 MUFU + Newton FFMA2, FMNMX clamp)
// variant 1: ex2 MUFU + rcp MUFU
// variant 2: production without clamp
// variant 3: polynomial exp2 (degree 3, FFMA2) for all elements + Newton
// variant 4: half MUFU ex2, half polynomial
// variant 5: tanh.approx (1 MUFU, inaccurate: for reference)
__device__ __forceinline__ void exp2_poly2(float t0, float t1, float& e0, float& e1) {
  // 2^t = 2^floor(t) * p(f), f in [0,1): p = 1 + f(c1 + f(c2 + f c3)) (degree-3 minimax-ish)
  float f0 = floorf(t0), f1 = floorf(t1);
  float r0 = t0 - f0, r1 = t1 - f1;
  float p0, p1;
  ffma2(p0, p1, r0, r1, 0.0790199f, 0.0790199f, 0.2249162f, 0.2249162f);
  ffma2(p0, p1, p0, p1, r0, r1, 0.6957728f, 0.6957728f);
  ffma2(p0, p1, p0, p1, r0, r1, 1.0000000f, 1.0000000f);
  e0 = __int_as_float(__float_as_int(p0) + (__float2int_rz(f0) << 23));
  e1 = __int_as_float(__float_as_int(p1) + (__float2int_rz(f1) << 23));
}
__device__ __forceinline__ void sig_rcp(float s0, float s1, float a2, float b2, float& p0, float& p1) {
  float t0, t1, y0, y1;
  ffma2(t0, t1, s0, s1, a2, a2, b2, b2);
  const float e0 = ex2_ftz(t0), e1 = ex2_ftz(t1);
  ffma2(y0, y1, e0, e1, 1.0f, 1.0f, 1.0f, 1.0f);
  p0 = sm100::rcp_approx(y0);
  p1 = sm100::rcp_approx(y1);
}
__device__ __forceinline__ void ffma2_sat(float& d0, float& d1, float a0, float a1, float b0, float b1, float c0, float c1) {
  d0 = __saturatef(fmaf(a0, b0, c0));
  d1 = __saturatef(fmaf(a1, b1, c1));
}
__device__ __forceinline__ void sig_sat(float s0, float s1, float a2, float b2, float& p0, float& p1) {
  // t'' = sat(s a2/252 + b2/252 + 1/2) in [0,1];  t = 252 t'' - 126  in [-126, 126]
  float u0, u1, t0, t1;
  ffma2_sat(u0, u1, s0, s1, a2 * (1.f / 252.f), a2 * (1.f / 252.f), b2 * (1.f / 252.f) + 0.5f, b2 * (1.f / 252.f) + 0.5f);
  ffma2(t0, t1, u0, u1, 252.f, 252.f, -126.f, -126.f);
  const float e0 = ex2_ftz(t0), e1 = ex2_ftz(t1);
  float n0, n1;
  ffma2(n0, n1, e0, e1, -1.0f, -1.0f, -1.0f, -1.0f);
  float r0 = __uint_as_float(0xFEF311C3u - __float_as_uint(n0));
  float r1 = __uint_as_float(0xFEF311C3u - __float_as_uint(n1));
  float v0, v1;
  ffma2(v0, v1, n0, n1, r0, r1, 1.0f, 1.0f);
  ffma2(r0, r1, r0, r1, v0, v1, r0, r1);
  ffma2(v0, v1, n0, n1, r0, r1, 1.0f, 1.0f);
  ffma2(r0, r1, r0, r1, v0, v1, r0, r1);
  p0 = r0; p1 = r1;
}
template <int V>
__device__ __forceinline__ void sig(float s0, float s1, float a2, float b2, float& p0, float& p1) {
  if constexpr (V == 0) {
    sigma2(s0, s1, a2, b2, p0, p1);
  } else if constexpr (V == 1) {
    float t0, t1;
    ffma2(t0, t1, s0, s1, a2, a2, b2, b2);
    p0 = sm100::rcp_approx(1.0f + ex2_ftz(t0));
    p1 = sm100::rcp_approx(1.0f + ex2_ftz(t1));
  } else if constexpr (V == 2 || V == 3 || V == 4) {
    float t0, t1, e0, e1;
    ffma2(t0, t1, s0, s1, a2, a2, b2, b2);
    if constexpr (V == 2) { e0 = ex2_ftz(t0); e1 = ex2_ftz(t1); }
    else if constexpr (V == 3) { exp2_poly2(fminf(t0, 126.f), fminf(t1, 126.f), e0, e1); }
    else { e0 = ex2_ftz(t0); float d; exp2_poly2(t1, t1, e1, d); }
    float n0, n1;
    ffma2(n0, n1, e0, e1, -1.0f, -1.0f, -1.0f, -1.0f);
    float r0 = __uint_as_float(0xFEF311C3u - __float_as_uint(n0));
    float r1 = __uint_as_float(0xFEF311C3u - __float_as_uint(n1));
    float u0, u1;
    ffma2(u0, u1, n0, n1, r0, r1, 1.0f, 1.0f);
    ffma2(r0, r1, r0, r1, u0, u1, r0, r1);
    ffma2(u0, u1, n0, n1, r0, r1, 1.0f, 1.0f);
    ffma2(r0, r1, r0, r1, u0, u1, r0, r1);
    p0 = r0; p1 = r1;
  } else {
    float t0, t1;
    ffma2(t0, t1, s0, s1, a2, a2, b2, b2);
    float y0, y1;
    asm("tanh.approx.f32 %0, %1;" : "=f"(y0) : "f"(t0));
    asm("tanh.approx.f32 %0, %1;" : "=f"(y1) : "f"(t1));
    ffma2(p0, p1, y0, y1, 0.5f, 0.5f, 0.5f, 0.5f);
  }
}

template <int V>
__global__ void __launch_bounds__(512, 1) kern(const float* in, uint32_t* out, int iters, long long* cyc) {
  float x[32];
  for (int i = 0; i < 32; ++i) x[i] = in[(threadIdx.x * 32 + i) & 1023];
  uint32_t acc = 0;
  const float a2 = -0.18f, b2 = 13.0f;
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int e = 0; e < 32; e += 2) {
      float p0, p1;
      if constexpr (V == 6) { if ((e & 6) == 0) sig_rcp(x[e], x[e + 1], a2, b2, p0, p1); else sig<0>(x[e], x[e + 1], a2, b2, p0, p1); }
      else if constexpr (V == 7) { if ((e & 2) == 0) sig_rcp(x[e], x[e + 1], a2, b2, p0, p1); else sig<0>(x[e], x[e + 1], a2, b2, p0, p1); }
      else if constexpr (V == 8) { if ((e & 6) != 6) sig_rcp(x[e], x[e + 1], a2, b2, p0, p1); else sig<0>(x[e], x[e + 1], a2, b2, p0, p1); }
      else if constexpr (V == 9) sig_sat(x[e], x[e + 1], a2, b2, p0, p1);
      else if constexpr (V == 10) { if ((e & 2) == 0) sig_rcp(x[e], x[e + 1], a2, b2, p0, p1); else sig_sat(x[e], x[e + 1], a2, b2, p0, p1); }
      else sig<V>(x[e], x[e + 1], a2, b2, p0, p1);
      acc ^= sm100::pack_bf16(p0, p1);
    }
    x[it & 31] += 1e-3f;
  }
  __syncthreads();
  long long t1 = clock64();
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

int main() {
  float* in; uint32_t* out; long long* cyc;
  cudaMalloc(&in, 1024 * 4); cudaMemset(in, 0, 4096);
  cudaMalloc(&out, 148 * 512 * 4); cudaMalloc(&cyc, 148 * 8);
  const int iters = 2000;
  const char* names[11] = {"ex2 + Newton(FFMA2) + clamp [prod]", "ex2 + rcp (2 MUFU)", "ex2 + Newton, no clamp",
                          "poly exp2 (FMA) + Newton", "half ex2 / half poly + Newton", "tanh.approx (1 MUFU, inexact)",
                          "1/4 rcp MUFU + 3/4 Newton", "1/2 rcp MUFU + 1/2 Newton", "3/4 rcp MUFU + 1/4 Newton",
                          "sat-FFMA2 clamp + Newton", "1/2 rcp + 1/2 sat-Newton"};
  for (int threads : {256, 512}) {
    printf("threads/SM %d\n", threads);
    void (*ks[11])(const float*, uint32_t*, int, long long*) = {kern<0>, kern<1>, kern<2>, kern<3>, kern<4>, kern<5>,
                                                                 kern<6>, kern<7>, kern<8>, kern<9>, kern<10>};
    for (int v = 0; v < 11; ++v) {
      void (*k)(const float*, uint32_t*, int, long long*) = ks[v];
      k<<<148, threads>>>(in, out, iters, cyc);
      cudaDeviceSynchronize();
      long long c; cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
      double elems = (double)threads * 32 * iters;
      printf("  %-40s %6.2f elem/clk/SM\n", names[v], elems / c);
    }
  }
  return 0;
}
