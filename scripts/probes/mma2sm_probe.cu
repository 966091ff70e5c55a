// mma2sm_probe.cu -- per-SM tcgen05.mma throughput of cta_group::2 (M = 256 over a CTA pair) vs
// cta_group::1 (M = 128) for the backward's N = 64 shapes (debug tool; operands are zeros).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I../../paper_2604_27124_b200/csrc mma2sm_probe.cu -o mma2sm_probe
#include <cstdio>
#include "sm100.cuh"

__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ void mma2_ts(uint32_t d, uint32_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
               "tcgen05.mma.cta_group::2.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d), "r"(a), "l"(b), "r"(idesc),
               "r"(acc) : "memory");
}
__device__ __forceinline__ void mma2_ss(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
               "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d), "l"(a), "l"(b), "r"(idesc),
               "r"(acc) : "memory");
}
__device__ __forceinline__ void commit2(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::
                   "r"(sm100::smem_u32(bar)), "h"((uint16_t)1) : "memory");
}

#ifndef ONE_SM
#define CLUSTER_ATTR __cluster_dims__(2, 1, 1)
#else
#define CLUSTER_ATTR
#endif
__global__ void CLUSTER_ATTR __launch_bounds__(128, 1) probe(long long* out, int reps) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t bar;
  __shared__ uint32_t holder;
  const int warp = threadIdx.x / 32;
  for (int i = threadIdx.x; i < 96 * 1024 / 16; i += blockDim.x) reinterpret_cast<uint4*>(smem)[i] = make_uint4(0, 0, 0, 0);
  if (threadIdx.x == 0) { sm100::mbar_init(&bar, 1); sm100::fence_barrier_init(); }
#ifdef ONE_SM
  if (warp == 0) sm100::tmem_alloc<512>(&holder);
#else
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(sm100::smem_u32(&holder)), "r"(512));
  }
#endif
  sm100::tc_fence_before();
  __syncthreads();
#ifndef ONE_SM
  cluster_sync();
#endif
  sm100::tc_fence_after();
  const uint32_t tmem = holder;
  const uint32_t base = sm100::smem_u32(smem);
  uint32_t phase = 0;
#ifdef ONE_SM
  if (warp == 0) {
#else
  if (cluster_rank() == 0 && warp == 0) {
#endif
#ifdef ONE_SM
    for (int v = 0; v < 8; v += 2) {
#else
    for (int v = 0; v < 8; ++v) {
#endif
      const bool two = v & 1;
      const uint32_t id = sm100::make_idesc_f16(true, two ? 256 : 128, v >= 6 ? 128 : 64, false, v < 2);
      __syncwarp();
      long long t0 = clock64();
      if (sm100::elect_one()) {
        const uint64_t bmn0 = sm100::make_sdesc_sw128(base + 32768, 16384, 1024);
        const uint64_t bk0 = sm100::make_sdesc_sw128(base + 32768, 16, 1024);
        const uint64_t ak0 = sm100::make_sdesc_sw128(base, 16, 1024);
        for (int r = 0; r < reps; ++r) {
#pragma unroll
          for (int kk = 0; kk < 8; ++kk) {
            const uint64_t bmn = bmn0 + ((kk * 2048) >> 4), bk = bk0 + ((kk * 32) >> 4), ak = ak0 + ((kk * 32) >> 4);
            if (v == 0) sm100::mma_ts(tmem + 256, tmem + kk * 8, bmn, id, 1);
            else if (v == 1) mma2_ts(tmem + 256, tmem + kk * 8, bmn, id, 1);
            else if (v == 2 || v == 6) sm100::mma_ts(tmem + 256, tmem + kk * 8, bk, id, 1);
            else if (v == 3 || v == 7) mma2_ts(tmem + 256, tmem + kk * 8, bk, id, 1);
            else if (v == 4) sm100::mma_ss(tmem + 256, ak, bk, id, 1);
            else mma2_ss(tmem + 256, ak, bk, id, 1);
          }
        }
      }
      __syncwarp();
      if (sm100::elect_one()) {
        if (v & 1) commit2(&bar);
        else sm100::mma_commit(&bar);
      }
      __syncwarp();
      sm100::mbar_wait(&bar, phase);
      phase ^= 1;
      long long t1 = clock64();
      if (threadIdx.x == 0) out[blockIdx.x * 8 + v] = t1 - t0;
    }
  }
  sm100::tc_fence_before();
  __syncthreads();
#ifdef ONE_SM
  if (warp == 0) sm100::tmem_dealloc<512>(tmem);
#else
  cluster_sync();
  if (warp == 0) {
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::);
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512));
  }
#endif
}

int main() {
  long long* d;
  cudaMalloc(&d, 148 * 8 * sizeof(long long));
  cudaMemset(d, 0, 148 * 8 * sizeof(long long));
  const int reps = 200;
  cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024);
  probe<<<148, 128, 100 * 1024>>>(d, reps);
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) { printf("error %s\n", cudaGetErrorString(e)); return 1; }
  long long h[8];
  cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
  const char* names[8] = {"1SM TS M128 N64 (B MN-major)", "2SM TS M256 N64 (B MN-major)", "1SM TS M128 N64 (B K-major)",
                          "2SM TS M256 N64 (B K-major)", "1SM SS M128 N64", "2SM SS M256 N64", "1SM TS M128 N128",
                          "2SM TS M256 N128"};
  for (int v = 0; v < 8; ++v)
    if (h[v]) printf("  %-32s %7.1f clk per instruction (per SM: %s)\n", names[v], (double)h[v] / (8.0 * reps),
           (v & 1) ? "half of the pair's M" : "all of M");
  return 0;
}
