// tmem_cost.cu -- does tcgen05.ld block the issuing sub-partition?  (debug tool)
// per iteration and warp: A: ld 32x32b.x32 + wait + 32 integer adds; B: 64 independent FFMA2 only;
// C: ld + wait, then 64 FFMA2 on the loaded values; D: ld, 64 FFMA2 on other registers, then wait.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I../../paper_2604_27124_b200/csrc tmem_cost.cu -o tmem_cost
#include <cstdio>
#include "sm100.cuh"
#include "sigmoid.cuh"
using namespace sigattn;

template <int MODE, int kFma>
__global__ void __launch_bounds__(512, 1) probe(long long* out, int iters, float* sink) {
  __shared__ uint32_t tmem_holder;
  const int warp = threadIdx.x / 32;
  if (warp == 0) sm100::tmem_alloc<512>(&tmem_holder);
  sm100::tc_fence_before();
  __syncthreads();
  sm100::tc_fence_after();
  const uint32_t tmem = tmem_holder;
  const uint32_t lane_addr = ((warp & 3) * 32) << 16;
  const uint32_t col = (warp >> 2) * 32;
  float acc[32];
  for (int i = 0; i < 32; ++i) acc[i] = threadIdx.x * 1e-3f + i;
  uint32_t iacc = 0;
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
    if constexpr (MODE == 0) {
      uint32_t r[32];
      sm100::tmem_ld32_sync(tmem + lane_addr + col + (it & 3) * 128, r);
      for (int i = 0; i < 32; ++i) iacc += r[i];
    } else if constexpr (MODE == 1) {
#pragma unroll
      for (int k = 0; k < kFma; ++k)
#pragma unroll
        for (int i = 0; i < 32; i += 2) ffma2(acc[i], acc[i + 1], acc[i], acc[i + 1], 0.999f, 0.999f, 1e-3f, 1e-3f);
    } else if constexpr (MODE == 2) {
      float r[32];
      sm100::tmem_ld32_sync(tmem + lane_addr + col + (it & 3) * 128, r);
#pragma unroll
      for (int k = 0; k < kFma; ++k)
#pragma unroll
        for (int i = 0; i < 32; i += 2) ffma2(acc[i], acc[i + 1], r[i], r[i + 1], acc[i], acc[i + 1], 1e-3f, 1e-3f);
    } else if constexpr (MODE == 4) {   // MUFU on registers only
#pragma unroll
      for (int k = 0; k < kFma; ++k)
#pragma unroll
        for (int i = 0; i < 32; ++i) acc[i] = ex2_ftz(acc[i]) - 0.5f;
    } else if constexpr (MODE == 5) {   // ld + wait, then MUFU on loaded
      float r[32];
      sm100::tmem_ld32_sync(tmem + lane_addr + col + (it & 3) * 128, r);
#pragma unroll
      for (int k = 0; k < kFma; ++k)
#pragma unroll
        for (int i = 0; i < 32; ++i) acc[i] += ex2_ftz(r[i] * acc[i]);
    } else if constexpr (MODE == 6) {   // no TMEM: MUFU on fresh per-iteration values (same dataflow as 5)
      float r[32];
#pragma unroll
      for (int i = 0; i < 32; ++i) r[i] = (float)((it + i) & 7);
#pragma unroll
      for (int k = 0; k < kFma; ++k)
#pragma unroll
        for (int i = 0; i < 32; ++i) acc[i] += ex2_ftz(r[i] * acc[i]);
    } else {
      float r[32];
      sm100::tmem_ld32(tmem + lane_addr + col + (it & 3) * 128, r);
#pragma unroll
      for (int k = 0; k < kFma; ++k)
#pragma unroll
        for (int i = 0; i < 32; i += 2) ffma2(acc[i], acc[i + 1], acc[i], acc[i + 1], 0.999f, 0.999f, 1e-3f, 1e-3f);
      sm100::tmem_wait_ld_dep(r);
#pragma unroll
      for (int i = 0; i < 32; ++i) acc[i] += r[i];
    }
  }
  __syncthreads();
  long long t1 = clock64();
  if (threadIdx.x == 0) out[blockIdx.x] = t1 - t0;
  float s = 0;
  for (int i = 0; i < 32; ++i) s += acc[i];
  sink[blockIdx.x * blockDim.x + threadIdx.x] = s + iacc;
  sm100::tc_fence_before();
  __syncthreads();
  if (warp == 0) sm100::tmem_dealloc<512>(tmem);
}

template <int MODE, int kFma>
void run(const char* name, int threads, long long* d, float* sink) {
  const int iters = 2000;
  probe<MODE, kFma><<<148, threads>>>(d, iters, sink);
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) { printf("error %s\n", cudaGetErrorString(e)); return; }
  long long c;
  cudaMemcpy(&c, d, sizeof(c), cudaMemcpyDeviceToHost);
  printf("  %-52s warps %2d  %8.1f clk/iter (per warp)\n", name, threads / 32, (double)c / iters);
}

int main() {
  long long* d;
  float* sink;
  cudaMalloc(&d, 2048 * sizeof(long long));
  cudaMalloc(&sink, 148 * 512 * 4);
  for (int threads : {128, 512}) {
    run<0, 0>("A ld x32 + wait + 32 IADD", threads, d, sink);
    run<1, 2>("B 32 FFMA2 (2 x 16) independent", threads, d, sink);
    run<1, 4>("B 64 FFMA2", threads, d, sink);
    run<2, 2>("C ld + wait, then 32 FFMA2 on loaded", threads, d, sink);
    run<2, 4>("C ld + wait, then 64 FFMA2 on loaded", threads, d, sink);
    run<3, 2>("D ld, 32 FFMA2 other regs, wait", threads, d, sink);
    run<3, 4>("D ld, 64 FFMA2 other regs, wait", threads, d, sink);
    run<4, 1>("E 32 MUFU.EX2 (registers)", threads, d, sink);
    run<6, 1>("F 32 MUFU.EX2 + FFMA (fresh values, no TMEM)", threads, d, sink);
    run<5, 1>("G ld + wait, then 32 MUFU.EX2 + FFMA on loaded", threads, d, sink);
  }
  return 0;
}
