// mufu_probe.cu -- MUFU ex2 throughput and the production sigma tiers in isolation (debug tool).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I../../paper_2604_27124_b200/csrc mufu_probe.cu -o mufu_probe
// Prints elements (sigma values or ex2 results) per clock per SM, for 256/512 threads per SM.
#include <cstdio>
#include <cuda_fp16.h>
#include "sigmoid.cuh"
#include "sm100.cuh"
using namespace sigattn;

template <int V>
__global__ void __launch_bounds__(512, 1) kern(const float* in, uint32_t* out, int iters, long long* cyc) {
  float x[32];
  for (int i = 0; i < 32; ++i) x[i] = in[(threadIdx.x * 32 + i) & 1023] - 9.0f;
  uint32_t acc = 0;
  const float a2 = 0.18f, b2 = -13.0f;
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
    if constexpr (V == 0) {          // bare MUFU.EX2, one per element
#pragma unroll
      for (int e = 0; e < 32; ++e) acc ^= __float_as_uint(ex2_ftz(x[e]));
    } else if constexpr (V == 1) {   // production tier-4 chunk: scale, max, vote, sigma2_fast4, pack
      float v[32];
#pragma unroll
      for (int e = 0; e < 32; ++e) v[e] = x[e];
      uint32_t pk[16];
      sigma_row<32, false, 0>(v, a2, b2, true, 32);
#pragma unroll
      for (int e = 0; e < 32; e += 2) pk[e >> 1] = sm100::pack2<true>(v[e], v[e + 1]);
#pragma unroll
      for (int e = 0; e < 16; ++e) acc ^= pk[e];
    } else if constexpr (V == 2) {   // ex2.approx.f16x2: two elements per MUFU op
#pragma unroll
      for (int e = 0; e < 32; e += 2) {
        uint32_t h, r;
        asm("cvt.rn.f16x2.f32 %0, %1, %2;" : "=r"(h) : "f"(x[e + 1]), "f"(x[e]));
        asm("ex2.approx.f16x2 %0, %1;" : "=r"(r) : "r"(h));
        acc ^= r;
      }
    } else if constexpr (V == 3) {   // ex2.approx.ftz.bf16x2
#pragma unroll
      for (int e = 0; e < 32; e += 2) {
        uint32_t h, r;
        asm("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(h) : "f"(x[e + 1]), "f"(x[e]));
        asm("ex2.approx.ftz.bf16x2 %0, %1;" : "=r"(r) : "r"(h));
        acc ^= r;
      }
    } else if constexpr (V == 4) {   // f16x2 ex2 only (inputs pre-packed): the raw MUFU rate
      uint32_t hx[16];
#pragma unroll
      for (int e = 0; e < 16; ++e) hx[e] = __float_as_uint(x[2 * e]) ^ it;
#pragma unroll
      for (int e = 0; e < 16; ++e) {
        uint32_t r;
        asm("ex2.approx.f16x2 %0, %1;" : "=r"(r) : "r"(hx[e]));
        acc ^= r;
      }
    } else if constexpr (V == 6) {   // speculative tier-4 (vote after the MUFU work)
      float v[32];
#pragma unroll
      for (int e = 0; e < 32; ++e) v[e] = x[e];
      uint32_t pk[16];
      if (!sigma_row_spec4<32>(v, a2, b2, true, 32)) {
#pragma unroll
        for (int e = 0; e < 32; ++e) v[e] = x[e];
        sigma_row<32, false, 0>(v, a2, b2, true, 32);
      }
#pragma unroll
      for (int e = 0; e < 32; e += 2) pk[e >> 1] = sm100::pack2<true>(v[e], v[e + 1]);
#pragma unroll
      for (int e = 0; e < 16; ++e) acc ^= pk[e];
    } else if constexpr (V == 5) {   // production tier-4 without the vote (fixed path)
#pragma unroll
      for (int e = 0; e < 32; e += 2) {
        float t0_, t1_, p0, p1;
        ffma2(t0_, t1_, x[e], x[e + 1], a2, a2, b2, b2);
        sigma2_fast4(t0_, t1_, p0, p1);
        acc ^= sm100::pack2<true>(p0, p1);
      }
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
  const int iters = 4000;
  const char* names[7] = {"bare MUFU.EX2 f32", "prod tier4 chunk (scale,max,vote,sigma,pack)", "cvt+ex2.f16x2",
                          "cvt+ex2.bf16x2", "ex2.f16x2 only", "prod tier4 no vote", "speculative tier4 (vote after MUFU)"};
  void (*ks[7])(const float*, uint32_t*, int, long long*) = {kern<0>, kern<1>, kern<2>, kern<3>, kern<4>, kern<5>, kern<6>};
  for (int threads : {128, 256, 512}) {
    printf("threads/SM %d\n", threads);
    for (int v = 0; v < 7; ++v) {
      ks[v]<<<148, threads>>>(in, out, 10, cyc);
      ks[v]<<<148, threads>>>(in, out, iters, cyc);
      cudaDeviceSynchronize();
      long long c; cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
      double elems = (double)threads * 32 * iters;
      printf("  %-48s %6.2f elem/clk/SM\n", names[v], elems / c);
    }
  }
  return 0;
}
