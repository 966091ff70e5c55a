// tmem_bw.cu -- SIMT tcgen05.ld / tcgen05.st throughput per SM (debug tool).
#include <cstdio>
#include "sm100.cuh"

template <int MODE>   // 0: ld32, 1: ld16, 2: st16, 3: ld32 x2 in flight, 4: ld32 + ld32 of a second lane block wait once
__global__ void __launch_bounds__(1024, 1) probe(long long* out, int iters) {
  __shared__ uint32_t tmem_holder;
  const int warp = threadIdx.x / 32;
  if (warp == 0) sm100::tmem_alloc<512>(&tmem_holder);
  sm100::tc_fence_before();
  __syncthreads();
  sm100::tc_fence_after();
  const uint32_t tmem = tmem_holder;
  const uint32_t lane_addr = ((warp & 3) * 32) << 16;
  const uint32_t col = ((warp >> 2) * 32) & 127;
  uint32_t acc = 0;
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
    if constexpr (MODE == 0) {
      uint32_t r[32];
      sm100::tmem_ld32_sync(tmem + lane_addr + col + (it & 3) * 128, r);
      for (int i = 0; i < 32; ++i) acc += r[i];
    } else if constexpr (MODE == 1) {
      float r[16];
      sm100::tmem_ld16(tmem + lane_addr + col + (it & 3) * 128, r);
      sm100::tmem_wait_ld_dep16(r);
      for (int i = 0; i < 16; ++i) acc += __float_as_uint(r[i]);
    } else if constexpr (MODE == 2) {
      uint32_t r[16];
      for (int i = 0; i < 16; ++i) r[i] = acc + i;
      sm100::tmem_st16(tmem + lane_addr + col + (it & 3) * 128, r);
      sm100::tmem_wait_st();
      acc += 1;
    } else {
      uint32_t a[32], b[32];
      sm100::tmem_ld32(tmem + lane_addr + (col & 127) + (it & 1) * 128, a);
      sm100::tmem_ld32(tmem + lane_addr + (col & 127) + 256 + (it & 1) * 128, b);
      sm100::tmem_wait_ld_dep(a);
      sm100::tmem_wait_ld_dep(b);
      for (int i = 0; i < 32; ++i) acc += a[i] ^ b[i];
    }
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
  const char* names[4] = {"ld 32x32b.x32 (4 KB/warp)", "ld 32x32b.x16 (2 KB/warp)", "st 32x32b.x16 (2 KB/warp)",
                          "2 x ld.x32 in flight (8 KB/warp)"};
  const double bytes[4] = {4096, 2048, 2048, 8192};
  for (int threads : {128, 256, 512, 1024}) {
    for (int m = 0; m < 4; ++m) {
      void (*k)(long long*, int) = m == 0 ? probe<0> : m == 1 ? probe<1> : m == 2 ? probe<2> : probe<3>;
      k<<<148, threads>>>(d, iters);
      cudaError_t e = cudaDeviceSynchronize();
      if (e != cudaSuccess) { printf("error %s\n", cudaGetErrorString(e)); return 1; }
      long long c;
      cudaMemcpy(&c, d, sizeof(c), cudaMemcpyDeviceToHost);
      printf("threads %3d  %-34s %7.1f B/clk/SM\n", threads, names[m], bytes[m] * (threads / 32) * iters / (double)c);
    }
  }
  return 0;
}
