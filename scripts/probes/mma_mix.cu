// mma_mix.cu -- clocks per tcgen05.mma for the shapes/operand sources the kernels use, alone and
// under concurrent TMEM / shared-memory traffic from 16 other warps (debug tool).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I../../paper_2604_27124_b200/csrc mma_mix.cu -o mma_mix
#include <cstdio>
#include "sm100.cuh"

constexpr int kSeqs = 12;
const char* kNames[kSeqs] = {
    "TS M128 N64  B K-major   x8", "TS M128 N64  B MN-major  x8", "TS M128 N128 B K-major   x8",
    "TS M128 N256 B K-major   x8", "SS M128 N64  K/K         x8", "SS M128 N128 K/K         x8",
    "SS M128 N64  MN/MN (dQ)  x8", "fwd tile: 4 SS N128 + 8 TS N64", "bwd tile: 32 TS N64 + 8 SS N64",
    "bwd tile + kernel's 6 commits", "bwd tile + commit after every MMA",
    "bwd tile, kernel's exact operands"};
constexpr int kInstr[kSeqs] = {8, 8, 8, 8, 8, 8, 8, 12, 40, 40, 40, 40};
constexpr double kFlopPerClk = 8192.0;   // dense bf16 per SM

__device__ __forceinline__ void run_seq(int seq, uint32_t tmem, uint32_t base, uint64_t* cb, int r = 0) {
  using namespace sm100;
  constexpr uint32_t i64k = make_idesc_f16(true, 128, 64, false, false);
  constexpr uint32_t i64m = make_idesc_f16(true, 128, 64, false, true);
  constexpr uint32_t i64mm = make_idesc_f16(true, 128, 64, true, true);
  constexpr uint32_t i128k = make_idesc_f16(true, 128, 128, false, false);
  constexpr uint32_t i256k = make_idesc_f16(true, 128, 256, false, false);
  const uint32_t a_t = tmem + 448;
  switch (seq) {
    case 0: for (int kk = 0; kk < 8; ++kk) mma_ts(tmem, a_t + (kk & 3) * 8, make_sdesc_sw128(base + (kk & 3) * 32, 16, 1024), i64k, 1); break;
    case 1: for (int kk = 0; kk < 8; ++kk) mma_ts(tmem, a_t + (kk & 3) * 8, make_sdesc_sw128(base + kk * 2048, 16384, 1024), i64m, 1); break;
    case 2: for (int kk = 0; kk < 8; ++kk) mma_ts(tmem, a_t + (kk & 3) * 8, make_sdesc_sw128(base + (kk & 3) * 32, 16, 1024), i128k, 1); break;
    case 3: for (int kk = 0; kk < 8; ++kk) mma_ts(tmem, a_t + (kk & 3) * 8, make_sdesc_sw128(base + (kk & 3) * 32, 16, 1024), i256k, 1); break;
    case 4: for (int kk = 0; kk < 8; ++kk) mma_ss(tmem, make_sdesc_sw128(base + 65536 + (kk & 3) * 32, 16, 1024), make_sdesc_sw128(base + (kk & 3) * 32, 16, 1024), i64k, 1); break;
    case 5: for (int kk = 0; kk < 8; ++kk) mma_ss(tmem, make_sdesc_sw128(base + 65536 + (kk & 3) * 32, 16, 1024), make_sdesc_sw128(base + (kk & 3) * 32, 16, 1024), i128k, 1); break;
    case 6: for (int kk = 0; kk < 8; ++kk) mma_ss(tmem, make_sdesc_sw128(base + 65536 + kk * 2048, 16384, 1024), make_sdesc_sw128(base + kk * 2048, 16384, 1024), i64mm, 1); break;
    case 7:
      for (int kk = 0; kk < 4; ++kk) mma_ss(tmem, make_sdesc_sw128(base + 65536 + kk * 32, 16, 1024), make_sdesc_sw128(base + kk * 32, 16, 1024), i128k, 1);
      for (int kk = 0; kk < 8; ++kk) mma_ts(tmem + 128, a_t + (kk & 3) * 8, make_sdesc_sw128(base + 32768 + kk * 2048, 16384, 1024), i64m, 1);
      break;
    case 8:
      for (int h = 0; h < 2; ++h) {
        for (int kk = 0; kk < 8; ++kk) mma_ts(tmem + (kk >> 2) * 64, a_t + (kk & 3) * 8, make_sdesc_sw128(base + (kk & 3) * 32, 16, 1024), i64k, 1);
        for (int kk = 0; kk < 8; ++kk) mma_ts(tmem + 128 + (kk >> 2) * 64, a_t + 32 + (kk & 3) * 8, make_sdesc_sw128(base + 32768 + (kk & 3) * 2048, 16384, 1024), i64m, 1);
      }
      for (int kk = 0; kk < 8; ++kk) mma_ss(tmem + 256, make_sdesc_sw128(base + 65536 + kk * 2048, 16384, 1024), make_sdesc_sw128(base + kk * 2048, 16384, 1024), i64mm, 1);
      break;
    case 9:
    case 10:
      for (int h = 0; h < 2; ++h) {
        for (int kk = 0; kk < 8; ++kk) {
          mma_ts(tmem + 128 + (kk >> 2) * 64, a_t + 32 + (kk & 3) * 8, make_sdesc_sw128(base + 32768 + (kk & 3) * 2048, 16384, 1024), i64m, 1);
          if (seq == 10) mma_commit(cb);
        }
        if (h == 1) { mma_commit(cb); }
        for (int kk = 0; kk < 8; ++kk) {
          mma_ts(tmem + (kk >> 2) * 64, a_t + (kk & 3) * 8, make_sdesc_sw128(base + (kk & 3) * 32, 16, 1024), i64k, 1);
          if (seq == 10) mma_commit(cb);
        }
        mma_commit(cb);
      }
      for (int kk = 0; kk < 8; ++kk) {
        mma_ss(tmem + 256, make_sdesc_sw128(base + 65536 + kk * 2048, 16384, 1024), make_sdesc_sw128(base + kk * 2048, 16384, 1024), i64mm, 1);
        if (seq == 10) mma_commit(cb);
      }
      mma_commit(cb); mma_commit(cb);
      break;
    case 11: {   // the d=64 backward kernel's per-tile sequence, BwdCfg smem / TMEM plan
      const uint32_t k_base = base, q_base = base + 65536, do_base = base + 98304, ds_base = base + 131072;
      const uint32_t st = r & 1;
      for (int q = 0; q < 2; ++q) {
        const uint32_t qa = q_base + st * 16384 + q * 8192, da = do_base + st * 16384 + q * 8192;
        for (int kk = 0; kk < 4; ++kk)   // dV += P^T dO
          mma_ts(tmem + 256, tmem + q * 64 + kk * 16, make_sdesc_sw128(da + kk * 2048, 16384, 1024), i64m, 1);
        for (int kk = 0; kk < 4; ++kk)   // dK += dS^T Q
          mma_ts(tmem + 320, tmem + 128 + q * 64 + kk * 16, make_sdesc_sw128(qa + kk * 2048, 16384, 1024), i64m, 1);
        const uint32_t qn = q_base + (st ^ 1) * 16384 + q * 8192, dn = do_base + (st ^ 1) * 16384 + q * 8192;
        for (int kk = 0; kk < 4; ++kk)   // S^T = K Q^T
          mma_ts(tmem + q * 64, tmem + 448 + kk * 8, make_sdesc_sw128(qn + kk * 32, 16, 1024), i64k, kk > 0);
        for (int kk = 0; kk < 4; ++kk)   // dP^T = V dO^T
          mma_ts(tmem + 128 + q * 64, tmem + 480 + kk * 8, make_sdesc_sw128(dn + kk * 32, 16, 1024), i64k, kk > 0);
        mma_commit(cb);
      }
      for (int kk = 0; kk < 8; ++kk)   // dQ = dS K
        mma_ss(tmem + 384, make_sdesc_sw128(ds_base + st * 32768 + kk * 2048, 16384, 1024),
               make_sdesc_sw128(k_base + kk * 2048, 16384, 1024), i64mm, kk > 0);
      mma_commit(cb); mma_commit(cb);
      break;
    }
  }
}

__global__ void __launch_bounds__(640, 1) probe(long long* out, int reps, int seq, int mode, int rnd) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t bar, cbar;
  __shared__ uint32_t tmem_holder;
  __shared__ volatile int stop;
  const int warp = threadIdx.x / 32;
  for (int i = threadIdx.x; i < 224 * 1024 / 4; i += blockDim.x) {
    // rnd: N(0,1)-like bf16 pairs (a cheap hash -> sum of uniforms), else zeros
    uint32_t h = (uint32_t)i * 2654435761u ^ 0x9e3779b9u;
    h ^= h >> 15; h *= 2246822519u; h ^= h >> 13;
    const float a = ((h & 0xffff) / 65536.f - 0.5f) * 3.4f, b = ((h >> 16) / 65536.f - 0.5f) * 3.4f;
    reinterpret_cast<uint32_t*>(smem)[i] = rnd ? sm100::pack_bf16(a, b) : 0u;
  }
  if (threadIdx.x == 0) { sm100::mbar_init(&bar, 1); sm100::mbar_init(&cbar, 1); sm100::fence_barrier_init(); stop = 0; }
  if (warp == 16) sm100::tmem_alloc<512>(&tmem_holder);
  sm100::tc_fence_before();
  __syncthreads();
  sm100::tc_fence_after();
  const uint32_t tmem = tmem_holder;
  const uint32_t base = sm100::smem_u32(smem);
  if (rnd && warp < 16) {   // random A operands / accumulators in TMEM
    const uint32_t lane_addr = ((warp & 3) * 32) << 16;
    for (int c0 = (warp >> 2) * 128; c0 < (warp >> 2) * 128 + 128; c0 += 8) {
      uint32_t pk[8];
      for (int i = 0; i < 8; ++i) pk[i] = sm100::pack_bf16(0.3f * ((threadIdx.x * 7 + c0 + i) % 13) - 1.8f, 0.25f * ((threadIdx.x + c0 * 3 + i) % 11) - 1.2f);
      sm100::tmem_st8(tmem + lane_addr + c0, pk);
    }
    sm100::tmem_wait_st();
  }
  sm100::tc_fence_before();
  __syncthreads();
  sm100::tc_fence_after();
  if (warp == 17) {
    long long t0 = clock64();
    for (int r = 0; r < reps; ++r) {
      if (sm100::elect_one()) run_seq(seq, tmem, base, &cbar, r);
      __syncwarp();
    }
    if (sm100::elect_one()) sm100::mma_commit(&bar);
    __syncwarp();
    sm100::mbar_wait(&bar, 0);
    long long t1 = clock64();
    if ((threadIdx.x & 31) == 0) { out[blockIdx.x] = t1 - t0; stop = 1; }
  } else if (warp < 16 && mode != 0) {
    const uint32_t tcol = (mode & 4) ? 0u : 384u;   // mode 5: TMEM traffic on the MMAs' own columns
    const uint32_t lane_addr = ((warp & 3) * 32) << 16;
    uint32_t acc = 0;
    while (!stop) {
      if (mode & 1) {   // TMEM traffic on columns the MMAs do not use (384..447)
        float s[16];
        sm100::tmem_ld16(tmem + lane_addr + tcol + (warp >> 2) * 16, s);
        sm100::tmem_wait_ld_dep16(s);
        uint32_t pk[8];
        for (int i = 0; i < 8; ++i) pk[i] = __float_as_uint(s[2 * i] + s[2 * i + 1]);
        sm100::tmem_st8(tmem + lane_addr + tcol + 64 + (warp >> 2) * 16, pk);
        acc += pk[0];
      }
      if (mode & 2) {   // shared-memory stores, 32 B per thread per iteration
        const uint32_t a = sm100::smem_u32(smem) + 131072 + ((warp * 32 + (threadIdx.x & 31)) * 32) % 65536;
        sm100::st_shared_v4(a, acc, acc + 1, acc + 2, acc + 3);
        sm100::st_shared_v4(a + 16, acc, acc + 1, acc + 2, acc + 3);
      }
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
  const int reps = 400, smem = 225 * 1024;
  cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  const char* modes[6] = {"alone", "+TMEM ld/st", "+st.shared", "+both", "random data", "+TMEM same cols"};
  printf("%-34s", "clk per MMA instruction");
  for (int m = 0; m < 6; ++m) printf(" %12s", modes[m]);
  printf("   (ideal clk/instr)\n");
  const int N[kSeqs] = {64, 64, 128, 256, 64, 128, 64, 0, 0, 0, 0, 0};
  for (int seq = 0; seq < kSeqs; ++seq) {
    printf("%-34s", kNames[seq]);
    for (int mode = 0; mode < 6; ++mode) {
      probe<<<148, 640, smem>>>(d, reps, seq, mode == 4 ? 0 : (mode == 5 ? 5 : mode), mode == 4);
      cudaError_t e = cudaDeviceSynchronize();
      if (e != cudaSuccess) { printf("error %s\n", cudaGetErrorString(e)); return 1; }
      long long h;
      cudaMemcpy(&h, d, sizeof(h), cudaMemcpyDeviceToHost);
      printf(" %12.1f", (double)h / reps / kInstr[seq]);
    }
    if (N[seq]) printf("   (%.0f)", 2.0 * 128 * N[seq] * 16 / kFlopPerClk);
    printf("\n");
  }
  return 0;
}
