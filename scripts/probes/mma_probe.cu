// mma_probe.cu -- microbenchmark of the tcgen05.mma shapes the attention kernels issue (debug tool).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I../../paper_2604_27124_b200/csrc mma_probe.cu -o mma_probe
#include <cstdio>
#include "sm100.cuh"

__global__ void __launch_bounds__(128, 1) probe(long long* out, int reps) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t bar, bar2, bar3;
  __shared__ uint32_t tmem_holder;
  const int warp = threadIdx.x / 32;
  for (int i = threadIdx.x; i < 160 * 1024 / 16; i += blockDim.x) reinterpret_cast<uint4*>(smem)[i] = make_uint4(0, 0, 0, 0);
  if (threadIdx.x == 0) { sm100::mbar_init(&bar, 1); sm100::mbar_init(&bar2, 1); sm100::mbar_init(&bar3, 1); sm100::fence_barrier_init(); }
  if (warp == 0) sm100::tmem_alloc<512>(&tmem_holder);
  sm100::tc_fence_before();
  __syncthreads();
  sm100::tc_fence_after();
  const uint32_t tmem = tmem_holder;
  const uint32_t base = sm100::smem_u32(smem);
  uint32_t phase = 0, ph2 = 0;
  if (warp == 0) {
    // variant v: 0 S(SS N128 K64) ; 1 PV(TS N64 K128) ; 2 half S(SS N64 K64) ; 3 TS N64 K64 ; 4 dq(SS MN/MN N64 K128)
    // 5 SS N128 K64 with B 2-CTA-free, A K-major (same as 0) but N=256; 6 TS N128 K128
    for (int v = 0; v < 14; ++v) {
      long long t_issue = 0;
      __syncwarp();
      long long t0 = clock64();
      for (int r = 0; r < reps; ++r) {
        long long a = clock64();
        if (sm100::elect_one()) {
          if (v == 0) {
            constexpr uint32_t id = sm100::make_idesc_f16(true, 128, 128, false, false);
            for (int kk = 0; kk < 4; ++kk)
              sm100::mma_ss(tmem, sm100::make_sdesc_sw128(base + kk * 32, 16, 1024), sm100::make_sdesc_sw128(base + 16384 + kk * 32, 16, 1024), id, kk > 0);
          } else if (v == 1) {
            constexpr uint32_t id = sm100::make_idesc_f16(true, 128, 64, false, true);
            for (int kk = 0; kk < 8; ++kk)
              sm100::mma_ts(tmem + 256, tmem + kk * 8, sm100::make_sdesc_sw128(base + 32768 + kk * 2048, 16384, 1024), id, 1);
          } else if (v == 2) {
            constexpr uint32_t id = sm100::make_idesc_f16(true, 128, 64, false, false);
            for (int kk = 0; kk < 4; ++kk)
              sm100::mma_ss(tmem, sm100::make_sdesc_sw128(base + kk * 32, 16, 1024), sm100::make_sdesc_sw128(base + 16384 + kk * 32, 16, 1024), id, kk > 0);
          } else if (v == 3) {
            constexpr uint32_t id = sm100::make_idesc_f16(true, 128, 64, false, true);
            for (int kk = 0; kk < 4; ++kk)
              sm100::mma_ts(tmem + 256, tmem + kk * 8, sm100::make_sdesc_sw128(base + 32768 + kk * 2048, 16384, 1024), id, 1);
          } else if (v == 4) {
            constexpr uint32_t id = sm100::make_idesc_f16(true, 128, 64, true, true);
            for (int kk = 0; kk < 8; ++kk)
              sm100::mma_ss(tmem + 384, sm100::make_sdesc_sw128(base + 65536 + kk * 2048, 16384, 1024), sm100::make_sdesc_sw128(base + kk * 2048, 16384, 1024), id, kk > 0);
          } else if (v == 5) {
            constexpr uint32_t id = sm100::make_idesc_f16(true, 128, 256, false, false);
            for (int kk = 0; kk < 4; ++kk)
              sm100::mma_ss(tmem, sm100::make_sdesc_sw128(base + kk * 32, 16, 1024), sm100::make_sdesc_sw128(base + 16384 + kk * 32, 16, 1024), id, kk > 0);
          } else if (v == 6) {
            constexpr uint32_t id = sm100::make_idesc_f16(true, 128, 128, false, true);
            for (int kk = 0; kk < 8; ++kk)
              sm100::mma_ts(tmem + 256, tmem + kk * 8, sm100::make_sdesc_sw128(base + 32768 + kk * 2048, 16384, 1024), id, 1);
          } else if (v == 7) {   // TS N64, two accumulators interleaved (dV / dK style)
            constexpr uint32_t id = sm100::make_idesc_f16(true, 128, 64, false, true);
            for (int kk = 0; kk < 8; ++kk)
              sm100::mma_ts(tmem + 256 + (kk & 1) * 64, tmem + (kk >> 1) * 8, sm100::make_sdesc_sw128(base + 32768 + (kk >> 1) * 2048, 16384, 1024), id, 1);
          } else if (v == 8) {   // SS N64 K64, two accumulators interleaved (S_q / dP_q style)
            constexpr uint32_t id = sm100::make_idesc_f16(true, 128, 64, false, false);
            for (int kk = 0; kk < 8; ++kk)
              sm100::mma_ss(tmem + (kk & 1) * 128, sm100::make_sdesc_sw128(base + (kk & 1) * 16384 + (kk >> 1) * 32, 16, 1024), sm100::make_sdesc_sw128(base + 32768 + (kk >> 1) * 32, 16, 1024), id, (kk >> 1) > 0);
          } else if (v == 9) {   // TS N64, four accumulators interleaved
            constexpr uint32_t id = sm100::make_idesc_f16(true, 128, 64, false, true);
            for (int kk = 0; kk < 8; ++kk)
              sm100::mma_ts(tmem + 256 + (kk & 3) * 64, tmem + (kk >> 2) * 8, sm100::make_sdesc_sw128(base + 32768 + (kk >> 2) * 2048, 16384, 1024), id, 1);
          } else if (v >= 11) {  // one backward tile: dV/dK(h0), S/dP(h0), dV/dK(h1), S/dP(h1), dQ (40 instr)
            constexpr uint32_t ids = sm100::make_idesc_f16(true, 128, 64, false, false);
            constexpr uint32_t ida = sm100::make_idesc_f16(true, 128, 64, false, true);
            constexpr uint32_t idq = sm100::make_idesc_f16(true, 128, 64, true, true);
            const uint32_t qa = base + 32768, da = base + 49152, ka = base, dsa = base + 65536;
            for (int q = 0; q < 2; ++q) {
              for (int kk = 0; kk < 4; ++kk)
                sm100::mma_ts(tmem + 256, tmem + q * 64 + kk * 16, sm100::make_sdesc_sw128(da + q * 8192 + kk * 2048, 16384, 1024), ida, 1);
              for (int kk = 0; kk < 4; ++kk)
                sm100::mma_ts(tmem + 320, tmem + 128 + q * 64 + kk * 16, sm100::make_sdesc_sw128(qa + q * 8192 + kk * 2048, 16384, 1024), ida, 1);
              for (int kk = 0; kk < 4; ++kk)
                sm100::mma_ts(tmem + q * 64, tmem + 448 + kk * 8, sm100::make_sdesc_sw128(qa + q * 8192 + kk * 32, 16, 1024), ids, kk > 0);
              for (int kk = 0; kk < 4; ++kk)
                sm100::mma_ts(tmem + 128 + q * 64, tmem + 480 + kk * 8, sm100::make_sdesc_sw128(da + q * 8192 + kk * 32, 16, 1024), ids, kk > 0);
              if (v >= 12) sm100::mma_commit(&bar3);
            }
            for (int kk = 0; kk < 8; ++kk)
              sm100::mma_ss(tmem + 384, sm100::make_sdesc_sw128(dsa + kk * 2048, 16384, 1024), sm100::make_sdesc_sw128(ka + kk * 2048, 16384, 1024), idq, kk > 0);
            if (v >= 12) sm100::mma_commit(&bar2);
          } else {               // TS N64 K64 with accumulate=0 on the first (fresh accumulator each group)
            constexpr uint32_t id = sm100::make_idesc_f16(true, 128, 64, false, true);
            for (int kk = 0; kk < 8; ++kk)
              sm100::mma_ts(tmem + 256, tmem + kk * 8, sm100::make_sdesc_sw128(base + 32768 + kk * 2048, 16384, 1024), id, kk > 0);
          }
        }
        __syncwarp();
        if (v == 13) {   // wait for the tile's last commit (3 arrivals per tile) before the next tile
          sm100::mbar_wait(&bar2, ph2); ph2 ^= 1;
        }
        t_issue += clock64() - a;
      }
      if (sm100::elect_one()) sm100::mma_commit(&bar);
      __syncwarp();
      sm100::mbar_wait(&bar, phase);
      phase ^= 1;
      long long t1 = clock64();
      if (threadIdx.x == 0) { out[2 * v] = t1 - t0; out[2 * v + 1] = t_issue; }
    }
    // latency of one S group: issue + commit + wait
    long long lat = 0;
    for (int r = 0; r < 64; ++r) {
      long long a = clock64();
      if (sm100::elect_one()) {
        constexpr uint32_t id = sm100::make_idesc_f16(true, 128, 128, false, false);
        for (int kk = 0; kk < 4; ++kk)
          sm100::mma_ss(tmem, sm100::make_sdesc_sw128(base + kk * 32, 16, 1024), sm100::make_sdesc_sw128(base + 16384 + kk * 32, 16, 1024), id, kk > 0);
        sm100::mma_commit(&bar);
      }
      __syncwarp();
      sm100::mbar_wait(&bar, phase);
      phase ^= 1;
      lat += clock64() - a;
    }
    if (threadIdx.x == 0) out[30] = lat / 64;
  }
  sm100::tc_fence_before();
  __syncthreads();
  if (warp == 0) sm100::tmem_dealloc<512>(tmem);
}

int main() {
  long long* d;
  cudaMalloc(&d, 64 * sizeof(long long));
  const int reps = 2000, smem = 160 * 1024 + 1024;
  cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  for (int grid : {1, 148}) {
    probe<<<grid, 128, smem>>>(d, reps);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) { printf("error %s\n", cudaGetErrorString(e)); return 1; }
    long long h[32];
    cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
    const char* names[14] = {"S: SS M128 N128 K64 (4 instr)", "PV: TS M128 N64 K128 (8)", "half S: SS M128 N64 K64 (4)",
                            "TS M128 N64 K64 (4)", "dQ: SS MN/MN M128 N64 K128 (8)", "SS M128 N256 K64 (4)", "TS M128 N128 K128 (8)",
                            "TS N64 x2 acc interleaved (8)", "SS N64 x2 acc interleaved (8)", "TS N64 x4 acc interleaved (8)",
                            "TS N64 K128 fresh acc (8)", "bwd tile, no commits (40)", "bwd tile + 3 commits (40)",
                            "bwd tile + commits, last waited (40)"};
    const double ideal[14] = {256, 256, 128, 128, 256, 512, 512, 256, 256, 256, 256, 1280, 1280, 1280};
    printf("grid %d\n", grid);
    for (int v = 0; v < 14; ++v)
      printf("  %-34s %8.1f clk/group (ideal %4.0f, %.0f%%)  issue %6.1f clk/group\n", names[v], (double)h[2 * v] / reps,
             ideal[v], 100.0 * ideal[v] / ((double)h[2 * v] / reps), (double)h[2 * v + 1] / reps);
    printf("  latency S group issue->commit->wait: %lld clk\n", h[30]);
  }
  return 0;
}
