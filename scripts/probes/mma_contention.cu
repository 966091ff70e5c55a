// mma_contention.cu -- tcgen05.mma throughput of the backward's MMA mix with/without concurrent
// TMEM (tcgen05.ld/st) and shared-memory (st.shared) traffic from 16 other warps (debug tool).
#include <cstdio>
#include "sm100.cuh"

__global__ void __launch_bounds__(640, 1) probe(long long* out, int reps, int mode) {
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
    long long t0 = clock64();
    for (int r = 0; r < reps; ++r) {
      if (sm100::elect_one()) {
        constexpr uint32_t ids = sm100::make_idesc_f16(true, 128, 128, false, false);
        constexpr uint32_t idv = sm100::make_idesc_f16(true, 128, 64, false, true);
        constexpr uint32_t idq = sm100::make_idesc_f16(true, 128, 64, true, true);
        for (int kk = 0; kk < 4; ++kk)   // S^T
          sm100::mma_ss(tmem, sm100::make_sdesc_sw128(base + kk * 32, 16, 1024), sm100::make_sdesc_sw128(base + 16384 + kk * 32, 16, 1024), ids, kk > 0);
        for (int kk = 0; kk < 4; ++kk)   // dP^T
          sm100::mma_ss(tmem + 128, sm100::make_sdesc_sw128(base + 32768 + kk * 32, 16, 1024), sm100::make_sdesc_sw128(base + 49152 + kk * 32, 16, 1024), ids, kk > 0);
        for (int kk = 0; kk < 8; ++kk)   // dV (TS)
          sm100::mma_ts(tmem + 320, tmem + 256 + kk * 8, sm100::make_sdesc_sw128(base + 65536 + kk * 2048, 16384, 1024), idv, 1);
        for (int kk = 0; kk < 8; ++kk)   // dK (SS, A K-major)
          sm100::mma_ss(tmem + 384, sm100::make_sdesc_sw128(base + 98304 + (kk >> 2) * 16384 + (kk & 3) * 32, 16, 1024), sm100::make_sdesc_sw128(base + 81920 + kk * 2048, 16384, 1024), idv, 1);
        for (int kk = 0; kk < 8; ++kk)   // dQ (SS, MN/MN)
          sm100::mma_ss(tmem + 448, sm100::make_sdesc_sw128(base + 98304 + kk * 2048, 16384, 1024), sm100::make_sdesc_sw128(base + kk * 2048, 16384, 1024), idq, kk > 0);
      }
      __syncwarp();
    }
    if (sm100::elect_one()) sm100::mma_commit(&bar);
    __syncwarp();
    sm100::mbar_wait(&bar, 0);
    long long t1 = clock64();
    if (lane == 0) { out[blockIdx.x] = t1 - t0; stop = 1; }
  } else if (warp < 16) {
    const uint32_t lane_addr = ((warp & 3) * 32) << 16;
    uint32_t acc = 0;
    while (!stop) {
      if (mode & 1) {   // TMEM traffic: 2 x ld16 + st8 per iteration on the S / dP / P columns
        float s[16], dp[16];
        sm100::tmem_ld16(tmem + lane_addr + (warp >> 2) * 32, s);
        sm100::tmem_ld16(tmem + lane_addr + 128 + (warp >> 2) * 32, dp);
        sm100::tmem_wait_ld_dep16(s);
        sm100::tmem_wait_ld_dep16(dp);
        uint32_t pk[8];
        for (int i = 0; i < 8; ++i) pk[i] = __float_as_uint(s[2 * i] + dp[2 * i + 1]);
        sm100::tmem_st8(tmem + lane_addr + 256 + (warp >> 2) * 16, pk);
        acc += pk[0];
      }
      if (mode & 2) {   // shared-memory stores: 2 x 16B per thread per iteration into the dS area
        const uint32_t a = base + 131072 + ((warp * 32 + lane) * 32) % 32768;
        sm100::st_shared_v4(a, acc, acc + 1, acc + 2, acc + 3);
        sm100::st_shared_v4(a + 16, acc, acc + 1, acc + 2, acc + 3);
      }
      if (mode == 0) break;
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
  const int reps = 500, smem = 201 * 1024;
  cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  const char* names[4] = {"MMA only", "+ TMEM ld/st traffic (16 warps)", "+ st.shared traffic (16 warps)", "+ both"};
  for (int mode = 0; mode < 4; ++mode) {
    probe<<<148, 640, smem>>>(d, reps, mode);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) { printf("error %s\n", cudaGetErrorString(e)); return 1; }
    long long h;
    cudaMemcpy(&h, d, sizeof(h), cudaMemcpyDeviceToHost);
    printf("%-36s %8.1f clk per backward tile of MMAs (S,dP,dV,dK,dQ; ideal 1280)\n", names[mode], (double)h / reps);
  }
  return 0;
}
