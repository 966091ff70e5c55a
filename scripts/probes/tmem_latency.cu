// tmem_latency.cu -- latency of tcgen05.st / tcgen05.ld / st.shared from SIMT warps while the tensor
// core runs the backward MMA mix (debug tool).
#include <cstdio>
#include "sm100.cuh"

__global__ void __launch_bounds__(640, 1) probe(long long* out, int reps, int with_mma) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t bar;
  __shared__ uint32_t tmem_holder;
  __shared__ volatile int stop;
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  for (int i = threadIdx.x; i < 200 * 1024 / 16; i += blockDim.x) reinterpret_cast<uint4*>(smem)[i] = make_uint4(0, 0, 0, 0);
  if (threadIdx.x == 0) { sm100::mbar_init(&bar, 1); sm100::fence_barrier_init(); stop = 0; }
  if (warp == 16) sm100::tmem_alloc<512>(&tmem_holder);
  sm100::tc_fence_before();
  __syncthreads();
  sm100::tc_fence_after();
  const uint32_t tmem = tmem_holder;
  const uint32_t base = sm100::smem_u32(smem);
  if (warp == 17) {
    if (with_mma) {
      for (int r = 0; r < reps; ++r) {
        if (sm100::elect_one()) {
          constexpr uint32_t ids = sm100::make_idesc_f16(true, 128, 128, false, false);
          constexpr uint32_t idv = sm100::make_idesc_f16(true, 128, 64, false, true);
          constexpr uint32_t idq = sm100::make_idesc_f16(true, 128, 64, true, true);
          for (int kk = 0; kk < 4; ++kk)
            sm100::mma_ss(tmem, sm100::make_sdesc_sw128(base + kk * 32, 16, 1024), sm100::make_sdesc_sw128(base + 16384 + kk * 32, 16, 1024), ids, kk > 0);
          for (int kk = 0; kk < 4; ++kk)
            sm100::mma_ss(tmem + 128, sm100::make_sdesc_sw128(base + 32768 + kk * 32, 16, 1024), sm100::make_sdesc_sw128(base + 49152 + kk * 32, 16, 1024), ids, kk > 0);
          for (int kk = 0; kk < 8; ++kk)
            sm100::mma_ts(tmem + 320, tmem + 256 + kk * 8, sm100::make_sdesc_sw128(base + 65536 + kk * 2048, 16384, 1024), idv, 1);
          for (int kk = 0; kk < 8; ++kk)
            sm100::mma_ss(tmem + 384, sm100::make_sdesc_sw128(base + 98304 + (kk >> 2) * 16384 + (kk & 3) * 32, 16, 1024), sm100::make_sdesc_sw128(base + 81920 + kk * 2048, 16384, 1024), idv, 1);
          for (int kk = 0; kk < 8; ++kk)
            sm100::mma_ss(tmem + 448, sm100::make_sdesc_sw128(base + 98304 + kk * 2048, 16384, 1024), sm100::make_sdesc_sw128(base + kk * 2048, 16384, 1024), idq, kk > 0);
        }
        __syncwarp();
      }
      if (sm100::elect_one()) sm100::mma_commit(&bar);
      __syncwarp();
      sm100::mbar_wait(&bar, 0);
    } else {
      long long t0 = clock64();
      while (clock64() - t0 < 800000) {}
    }
    if (lane == 0) stop = 1;
  } else if (warp < 16) {
    const uint32_t lane_addr = ((warp & 3) * 32) << 16;
    long long t_st = 0, t_ld = 0, t_sts = 0, t_fence = 0;
    int n = 0;
    uint32_t acc = lane;
    while (!stop && n < 4000) {
      uint32_t pk[8];
      for (int i = 0; i < 8; ++i) pk[i] = acc + i;
      long long a = clock64();
      sm100::tmem_st8(tmem + lane_addr + 256 + (warp >> 2) * 16, pk);
      sm100::tmem_wait_st();
      long long b = clock64();
      float s[16];
      sm100::tmem_ld16(tmem + lane_addr + (warp >> 2) * 32, s);
      sm100::tmem_wait_ld_dep16(s);
      acc += __float_as_uint(s[3]);
      long long c = clock64();
      const uint32_t addr = base + 131072 + ((warp * 32 + lane) * 32) % 32768;
      sm100::st_shared_v4(addr, acc, acc + 1, acc + 2, acc + 3);
      sm100::st_shared_v4(addr + 16, acc, acc + 1, acc + 2, acc + 3);
      long long d = clock64();
      sm100::fence_proxy_async_smem();
      long long e = clock64();
      t_st += b - a; t_ld += c - b; t_sts += d - c; t_fence += e - d;
      ++n;
    }
    if (lane == 0 && blockIdx.x == 0) {
      out[warp * 4 + 0] = t_st / n; out[warp * 4 + 1] = t_ld / n; out[warp * 4 + 2] = t_sts / n; out[warp * 4 + 3] = t_fence / n;
    }
    if (acc == 0x12345678) out[1000] = acc;
  }
  sm100::tc_fence_before();
  __syncthreads();
  if (warp == 16) sm100::tmem_dealloc<512>(tmem);
}

int main() {
  long long* d;
  cudaMalloc(&d, 2048 * sizeof(long long));
  const int smem = 201 * 1024;
  cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  for (int with_mma = 0; with_mma < 2; ++with_mma) {
    probe<<<148, 640, smem>>>(d, 400, with_mma);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) { printf("error %s\n", cudaGetErrorString(e)); return 1; }
    long long h[64];
    cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
    double a[4] = {0, 0, 0, 0};
    for (int w = 0; w < 16; ++w) for (int k = 0; k < 4; ++k) a[k] += h[w * 4 + k] / 16.0;
    printf("%s: st8+wait::st %6.0f | ld16+wait %6.0f | 2x st.shared.v4 %6.0f | fence.proxy.async %6.0f clk\n",
           with_mma ? "with MMAs   " : "without MMAs", a[0], a[1], a[2], a[3]);
  }
  return 0;
}
