// tmem_ld_probe.cu -- SIMT tcgen05.ld throughput per SM by shape, 16 or 32 warps (debug tool).
// Each warp loads its lane quarter, 64 columns per iteration, as 2 x x32, 4 x x16 or 8 x x8, waits once.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I../../paper_2604_27124_b200/csrc tmem_ld_probe.cu -o tmem_ld_probe
#include <cstdio>
#include "sm100.cuh"

template <int W>
__global__ void __launch_bounds__(1024, 1) probe(long long* out, int iters) {
  __shared__ uint32_t tmem_holder;
  const int warp = threadIdx.x / 32;
  if (warp == 0) sm100::tmem_alloc<512>(&tmem_holder);
  sm100::tc_fence_before();
  __syncthreads();
  sm100::tc_fence_after();
  const uint32_t tmem = tmem_holder;
  const uint32_t lane_addr = ((warp & 3) * 32) << 16;
  const uint32_t col = ((warp >> 2) * 64) & 511;
  uint32_t acc = 0;
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
    uint32_t r[64];
    const uint32_t a = tmem + lane_addr + ((col + it * 64) & 511);
    if constexpr (W == 32) {
      sm100::tmem_ld32(a, *reinterpret_cast<uint32_t(*)[32]>(r));
      sm100::tmem_ld32(a + 32, *reinterpret_cast<uint32_t(*)[32]>(r + 32));
    } else if constexpr (W == 16) {
#pragma unroll
      for (int c = 0; c < 4; ++c) sm100::tmem_ld16(a + 16 * c, *reinterpret_cast<uint32_t(*)[16]>(r + 16 * c));
    } else {
#pragma unroll
      for (int c = 0; c < 8; ++c) sm100::tmem_ld8(a + 8 * c, *reinterpret_cast<uint32_t(*)[8]>(r + 8 * c));
    }
    sm100::tmem_wait_ld_dep(*reinterpret_cast<uint32_t(*)[32]>(r));
    sm100::tmem_wait_ld_dep(*reinterpret_cast<uint32_t(*)[32]>(r + 32));
#pragma unroll
    for (int i = 0; i < 64; i += 2) acc += r[i] ^ r[i + 1];
  }
  __syncthreads();
  long long t1 = clock64();
  if (threadIdx.x == 0) out[blockIdx.x] = t1 - t0;
  if (acc == 0x12345) out[1000] = acc;
  sm100::tc_fence_before();
  __syncthreads();
  if (warp == 0) sm100::tmem_dealloc<512>(tmem);
}

int main() {
  long long* d;
  cudaMalloc(&d, 2048 * sizeof(long long));
  const int iters = 4000;
  for (int threads : {256, 512, 1024}) {
    for (int w : {32, 16, 8}) {
      void (*k)(long long*, int) = w == 32 ? probe<32> : w == 16 ? probe<16> : probe<8>;
      k<<<148, threads>>>(d, iters);
      cudaError_t e = cudaDeviceSynchronize();
      if (e != cudaSuccess) { printf("error %s\n", cudaGetErrorString(e)); return 1; }
      long long c;
      cudaMemcpy(&c, d, sizeof(c), cudaMemcpyDeviceToHost);
      printf("warps %2d  64 columns as x%-2d loads, one wait: %7.1f B/clk/SM\n", threads / 32, w,
             256.0 * (threads / 32) * iters * 32 / (double)c);
    }
  }
  return 0;
}
