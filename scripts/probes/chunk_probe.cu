// chunk_probe.cu -- throughput of the forward's per-chunk sigma path on sm_100a (debug tool):
// tcgen05.ld 32 scores -> fwd64_chunk (scale, tier vote, sigma, pack) -> tcgen05.st 16 words, per warp
// in a loop, 8 or 16 warps per SM, one CTA per SM.  Prints elements per clock per SM (MUFU ex2 peak: 16).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I../../paper_2604_27124_b200/csrc chunk_probe.cu -o chunk_probe
#include <cstdio>
#include <type_traits>
#include "sigmoid.cuh"
#include "sm100.cuh"

// The forward chunk path measured here (the t-preserving speculative form tried for a two-query-tile
// d = 64 forward in round 2):
namespace sigattn {

// ---------------------------------------------------------------------------------------------
// Building blocks for callers that keep t (the scaled logits) alive across the tier vote, so a
// failed speculation recomputes from registers instead of reloading the scores (forward, d = 64).

// t = s a + c in place (t = x log2 e); returns the max over the valid columns (e < nvalid).
template <int N, bool kMask>
__device__ __forceinline__ float scale_row_max(float (&v)[N], float a, float c, int nvalid) {
  float m = -INFINITY;
#pragma unroll
  for (int e = 0; e < N; e += 2) {
    ffma2(v[e], v[e + 1], v[e], v[e + 1], a, a, c, c);
    if constexpr (kMask)
      m = fmax3(m, e < nvalid ? v[e] : -INFINITY, e + 1 < nvalid ? v[e + 1] : -INFINITY);
    else
      m = fmax3(m, v[e], v[e + 1]);
  }
  return m;
}

// sigma of one element pair from t in tier kTier (4: t <= kFastT4, 2: t <= kFastT, 0: any t).
// kFma: the exp2 of this pair runs on the FMA pipe (exp2_fma2) instead of the MUFU.
template <int kTier, bool kFma>
__device__ __forceinline__ void sigma_pair_t(float t0, float t1, float& p0, float& p1) {
  if constexpr (kTier == 0) {
    sigma2_from_t(t0, t1, p0, p1);
  } else {
    float u0, u1;
    if constexpr (kFma) {
      exp2_fma2(t0, t1, u0, u1);
    } else {
      u0 = ex2_ftz(t0);
      u1 = ex2_ftz(t1);
    }
    float r0, r1;
    if constexpr (kTier == 4) {
      r0 = 1.0f - u0;                                 // u (1 - u)
      r1 = 1.0f - u1;
    } else {
      ffma2(r0, r1, u0, u1, kR2, kR2, kR1, kR1);
      ffma2(r0, r1, r0, r1, u0, u1, kR0, kR0);        // R(u)
    }
    fmul2(p0, p1, r0, r1, u0, u1);
  }
}

// Whether pair index i (of a row chunk) takes the FMA-pipe exp2: kEmuEvery = 0 never, else one
// pair in kEmuEvery (the MUFU does 16 ex2/clk/SM; the FMA pipe has idle issue slots beside it).
template <int kEmuEvery>
__device__ __forceinline__ constexpr bool emu_pair(int i) {
  return kEmuEvery > 0 && (i % (kEmuEvery > 0 ? kEmuEvery : 1)) == (kEmuEvery > 0 ? kEmuEvery : 1) / 2;
}


template <bool kMask, bool kBf16, int kEmu>
__device__ __forceinline__ void fwd64_chunk(float (&v)[32], uint32_t (&pk)[16], float a, float c, bool row_valid,
                                            int nvalid, bool& spec) {
  const float m = scale_row_max<32, kMask>(v, a, c, nvalid);
  auto pack_tier = [&](auto tier_c) {
    constexpr int kT = decltype(tier_c)::value;
#pragma unroll
    for (int e = 0; e < 32; e += 2) {
      float p0, p1;
      if (emu_pair<kEmu>(e >> 1)) sigma_pair_t<kT, true>(v[e], v[e + 1], p0, p1);
      else sigma_pair_t<kT, false>(v[e], v[e + 1], p0, p1);
      if constexpr (kMask) {
        p0 = (e < nvalid) ? p0 : 0.0f;
        p1 = (e + 1 < nvalid) ? p1 : 0.0f;
      }
      pk[e >> 1] = sm100::pack2<kBf16>(p0, p1);
    }
  };
  if (spec) {
    pack_tier(std::integral_constant<int, 4>{});
#pragma unroll
    for (int i = 0; i < 16; ++i) asm volatile("" : "+r"(pk[i]));
  }
  const bool ok4 = __all_sync(0xffffffffu, !row_valid || m <= kFastT4);
  if (!(spec && ok4)) {
    if (ok4) pack_tier(std::integral_constant<int, 4>{});
    else if (__all_sync(0xffffffffu, !row_valid || m <= kFastT)) pack_tier(std::integral_constant<int, 2>{});
    else pack_tier(std::integral_constant<int, 0>{});
  }
  spec = ok4;
}
}  // namespace sigattn
using namespace sigattn;

template <int kEmu, bool kSpec, int kPairChunks, int kMode = 0>   // mode 0: ld+st, 1: no TMEM (registers), 2: st without wait, 3: ld only
__global__ void __launch_bounds__(512, 1) kern(int iters, long long* cyc, uint32_t* sink, float bias2) {
  __shared__ uint32_t tmem_holder;
  const uint32_t warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  if (warp == 0) sm100::tmem_alloc<512>(&tmem_holder);
  sm100::tc_fence_before();
  __syncthreads();
  sm100::tc_fence_after();
  const uint32_t tmem = tmem_holder;
  const uint32_t lane_addr = ((warp & 3) * 32) << 16;
  const uint32_t col = (warp >> 2) * 64;   // 64 columns per warp: 32 scores + room for P
  {   // fill scores ~ N(0, 8) pattern in TMEM
    uint32_t v[16];
    for (int i = 0; i < 16; ++i) v[i] = __float_as_uint(((lane * 7 + i * 13) % 31 - 15) * 0.5f);
    sm100::tmem_st16(tmem + lane_addr + col, v);
    sm100::tmem_st16(tmem + lane_addr + col + 16, v);
    sm100::tmem_wait_st();
  }
  __syncthreads();
  bool spec = kSpec;
  uint32_t acc = 0;
  const float a2 = 0.125f * 1.4426950408889634f;
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
    float r[kPairChunks][32];
    uint32_t pk[kPairChunks][16];
    if constexpr (kMode == 1) {
#pragma unroll
      for (int c = 0; c < kPairChunks; ++c)
#pragma unroll
        for (int i = 0; i < 32; ++i) r[c][i] = (float)((lane + i * 7 + it) & 15) * 0.5f;
    } else if constexpr (kMode == 5) {
      sm100::tmem_ld16(tmem + lane_addr + col, *reinterpret_cast<uint32_t(*)[16]>(&r[0][0]));
      sm100::tmem_ld16(tmem + lane_addr + col + 16, *reinterpret_cast<uint32_t(*)[16]>(&r[0][16]));
      sm100::tmem_wait_ld_dep(r[0]);
    } else if constexpr (kMode == 6) {
      uint32_t* u = reinterpret_cast<uint32_t*>(&r[0][0]);
      asm volatile("tcgen05.ld.sync.aligned.16x256b.x8.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, %15, "
                   "%16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31}, [%32];"
                   : "=r"(u[0]), "=r"(u[1]), "=r"(u[2]), "=r"(u[3]), "=r"(u[4]), "=r"(u[5]), "=r"(u[6]), "=r"(u[7]),
                     "=r"(u[8]), "=r"(u[9]), "=r"(u[10]), "=r"(u[11]), "=r"(u[12]), "=r"(u[13]), "=r"(u[14]), "=r"(u[15]),
                     "=r"(u[16]), "=r"(u[17]), "=r"(u[18]), "=r"(u[19]), "=r"(u[20]), "=r"(u[21]), "=r"(u[22]), "=r"(u[23]),
                     "=r"(u[24]), "=r"(u[25]), "=r"(u[26]), "=r"(u[27]), "=r"(u[28]), "=r"(u[29]), "=r"(u[30]), "=r"(u[31])
                   : "r"(tmem + ((warp & 3) * 32 << 16) + col));
      sm100::tmem_wait_ld_dep(r[0]);
    } else {
#pragma unroll
      for (int c = 0; c < kPairChunks; ++c) sm100::tmem_ld32(tmem + lane_addr + col, *reinterpret_cast<uint32_t(*)[32]>(&r[c]));
#pragma unroll
      for (int c = 0; c < kPairChunks; ++c) sm100::tmem_wait_ld_dep(r[c]);
    }
#pragma unroll
    for (int c = 0; c < kPairChunks; ++c) {
      bool sp = kSpec ? spec : false;
      fwd64_chunk<false, true, kEmu>(r[c], pk[c], a2, bias2, true, 32, sp);
      spec = kSpec ? sp : false;
    }
    if constexpr (kMode == 0 || kMode == 2) {
#pragma unroll
      for (int c = 0; c < kPairChunks; ++c) sm100::tmem_st16(tmem + lane_addr + col + 32 + (c & 1) * 16, pk[c]);
      if (kMode == 0 || (it & 3) == 3) sm100::tmem_wait_st();
    }
#pragma unroll
    for (int c = 0; c < kPairChunks; ++c)
#pragma unroll
      for (int i = 0; i < 16; ++i) acc ^= pk[c][i];
  }
  long long t1 = clock64();
  sink[blockIdx.x * blockDim.x + threadIdx.x] = acc;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
  sm100::tc_fence_before();
  __syncthreads();
  if (warp == 0) sm100::tmem_dealloc<512>(tmem);
}

template <int kEmu, bool kSpec, int kPC, int kMode = 0>
void run(const char* name, int threads, long long* cyc, uint32_t* sink, float bias2) {
  const int iters = 4000;
  kern<kEmu, kSpec, kPC, kMode><<<148, threads>>>(iters, cyc, sink, bias2);
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) { printf("error %s\n", cudaGetErrorString(e)); return; }
  long long c;
  cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
  printf("  %-44s warps %2d  %6.2f elem/clk/SM\n", name, threads / 32, (double)threads * 32 * kPC * iters / c);
}


// software-pipelined: the load of the next chunk is in flight while the current one is computed
template <int kEmu, bool kSpec>
__global__ void __launch_bounds__(512, 1) kern_pipe(int iters, long long* cyc, uint32_t* sink, float bias2) {
  __shared__ uint32_t tmem_holder;
  const uint32_t warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  if (warp == 0) sm100::tmem_alloc<512>(&tmem_holder);
  sm100::tc_fence_before();
  __syncthreads();
  sm100::tc_fence_after();
  const uint32_t tmem = tmem_holder;
  const uint32_t lane_addr = ((warp & 3) * 32) << 16;
  const uint32_t col = (warp >> 2) * 64;
  {
    uint32_t v[16];
    for (int i = 0; i < 16; ++i) v[i] = __float_as_uint(((lane * 7 + i * 13) % 31 - 15) * 0.5f);
    sm100::tmem_st16(tmem + lane_addr + col, v);
    sm100::tmem_st16(tmem + lane_addr + col + 16, v);
    sm100::tmem_wait_st();
  }
  __syncthreads();
  bool spec = kSpec;
  uint32_t acc = 0;
  const float a2 = 0.125f * 1.4426950408889634f;
  float ra[32], rb[32];
  uint32_t pk[16];
  sm100::tmem_ld32(tmem + lane_addr + col, ra);
  long long t0 = clock64();
  for (int it = 0; it < iters; it += 2) {
    sm100::tmem_wait_ld_dep(ra);
    sm100::tmem_ld32(tmem + lane_addr + col, rb);
    fwd64_chunk<false, true, kEmu>(ra, pk, a2, bias2, true, 32, spec);
    sm100::tmem_st16(tmem + lane_addr + col + 32, pk);
    sm100::tmem_wait_ld_dep(rb);
    sm100::tmem_ld32(tmem + lane_addr + col, ra);
    fwd64_chunk<false, true, kEmu>(rb, pk, a2, bias2, true, 32, spec);
    sm100::tmem_st16(tmem + lane_addr + col + 48, pk);
    if ((it & 7) == 6) sm100::tmem_wait_st();
#pragma unroll
    for (int i = 0; i < 16; ++i) acc ^= pk[i];
  }
  sm100::tmem_wait_ld_dep(ra);
  long long t1 = clock64();
  sink[blockIdx.x * blockDim.x + threadIdx.x] = acc + __float_as_uint(ra[3]);
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
  sm100::tc_fence_before();
  __syncthreads();
  if (warp == 0) sm100::tmem_dealloc<512>(tmem);
}
template <int kEmu, bool kSpec>
void run_pipe(const char* name, int threads, long long* cyc, uint32_t* sink, float bias2) {
  const int iters = 4000;
  kern_pipe<kEmu, kSpec><<<148, threads>>>(iters, cyc, sink, bias2);
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) { printf("error %s\n", cudaGetErrorString(e)); return; }
  long long c;
  cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
  printf("  %-44s warps %2d  %6.2f elem/clk/SM\n", name, threads / 32, (double)threads * 32 * iters / c);
}


// production forward chunk path (fwd.cuh sigmoid_chunk32 logic: spec tier 4, reload on vote failure)
// at chunk width kW (16 or 32 columns per load), any warp count up to 32
template <int kW>
__global__ void __launch_bounds__(1024, 1) kern_w(int iters, long long* cyc, uint32_t* sink, float bias2) {
  __shared__ uint32_t tmem_holder;
  const uint32_t warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  if (warp == 0) sm100::tmem_alloc<512>(&tmem_holder);
  sm100::tc_fence_before();
  __syncthreads();
  sm100::tc_fence_after();
  const uint32_t tmem = tmem_holder;
  const uint32_t lane_addr = ((warp & 3) * 32) << 16;
  const uint32_t col = (warp >> 2) * 64;
  {
    uint32_t v[16];
    for (int i = 0; i < 16; ++i) v[i] = __float_as_uint(((lane * 7 + i * 13) % 31 - 15) * 0.5f);
    sm100::tmem_st16(tmem + lane_addr + col, v);
    sm100::tmem_st16(tmem + lane_addr + col + 16, v);
    sm100::tmem_wait_st();
  }
  __syncthreads();
  bool spec = true;
  uint32_t acc = 0;
  const float a2 = 0.125f * 1.4426950408889634f;
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
    float r[kW];
    uint32_t pk[kW / 2];
    if constexpr (kW == 32) sm100::tmem_ld32_sync(tmem + lane_addr + col, r);
    else {
      sm100::tmem_ld16(tmem + lane_addr + col, r);
      sm100::tmem_wait_ld_dep16(r);
    }
    bool done = false;
    if (spec) {
      done = sigma_row_spec4<kW, false>(r, a2, bias2, true, kW);
      if (!done) {
        if constexpr (kW == 32) sm100::tmem_ld32_sync(tmem + lane_addr + col, r);
        else { sm100::tmem_ld16(tmem + lane_addr + col, r); sm100::tmem_wait_ld_dep16(r); }
      }
    }
    if (!done) spec = sigma_row<kW, false, 0>(r, a2, bias2, true, kW) == 4;
#pragma unroll
    for (int e = 0; e < kW; e += 2) pk[e >> 1] = sm100::pack2<true>(r[e], r[e + 1]);
    if constexpr (kW == 32) sm100::tmem_st16(tmem + lane_addr + col + 32, pk);
    else sm100::tmem_st8(tmem + lane_addr + col + 32, pk);
    if ((it & 3) == 3) sm100::tmem_wait_st();
#pragma unroll
    for (int i = 0; i < kW / 2; ++i) acc ^= pk[i];
  }
  long long t1 = clock64();
  sink[blockIdx.x * blockDim.x + threadIdx.x] = acc;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
  sm100::tc_fence_before();
  __syncthreads();
  if (warp == 0) sm100::tmem_dealloc<512>(tmem);
}
template <int kW>
void run_w(int warps, long long* cyc, uint32_t* sink, float bias2) {
  const int iters = 4000;
  kern_w<kW><<<148, warps * 32>>>(iters, cyc, sink, bias2);
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) { printf("error %s\n", cudaGetErrorString(e)); return; }
  long long c;
  cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
  printf("  production chunk path, %2d columns per load, warps %2d  %6.2f elem/clk/SM\n", kW, warps,
         (double)warps * 32 * kW * iters / c);
}


// instruction-class ablation of the tier-4 chunk path (16 warps): which part limits it
template <int kVar>
__global__ void __launch_bounds__(1024, 1) kern_ab(int iters, long long* cyc, uint32_t* sink, float bias2) {
  __shared__ uint32_t tmem_holder;
  const uint32_t warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  if (warp == 0) sm100::tmem_alloc<512>(&tmem_holder);
  sm100::tc_fence_before();
  __syncthreads();
  sm100::tc_fence_after();
  const uint32_t tmem = tmem_holder;
  const uint32_t lane_addr = ((warp & 3) * 32) << 16;
  const uint32_t col = (warp >> 2) * 64;
  {
    uint32_t v[16];
    for (int i = 0; i < 16; ++i) v[i] = __float_as_uint(((lane * 7 + i * 13) % 31 - 15) * 0.5f);
    sm100::tmem_st16(tmem + lane_addr + col, v);
    sm100::tmem_st16(tmem + lane_addr + col + 16, v);
    sm100::tmem_wait_st();
  }
  __syncthreads();
  uint32_t acc = 0;
  const float a2 = 0.125f * 1.4426950408889634f;
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
    float r[32];
    uint32_t pk[16];
    sm100::tmem_ld32_sync(tmem + lane_addr + col, r);
    float m = -INFINITY;
#pragma unroll
    for (int e = 0; e < 32; e += 2) {
      if (kVar != 3) ffma2(r[e], r[e + 1], r[e], r[e + 1], a2, a2, bias2, bias2);
      if (kVar != 1) m = fmax3(m, r[e], r[e + 1]);
    }
    bool ok = (kVar == 1) ? true : __all_sync(0xffffffffu, m <= kFastT4);
#pragma unroll
    for (int e = 0; e < 32; e += 2) {
      float p0, p1;
      float u0, u1;
      constexpr int kEmuK = kVar >= 5 ? kVar - 3 : 0;   // kVar 5..: pair e/2 % k == k/2 on the FMA pipe
      if (kEmuK > 0 && ((e >> 1) % (kEmuK > 0 ? kEmuK : 1)) == kEmuK / 2) exp2_fma2(r[e], r[e + 1], u0, u1);
      else { u0 = ex2_ftz(r[e]); u1 = ex2_ftz(r[e + 1]); }
      if (kVar == 4) { p0 = u0; p1 = u1; }
      else ffma2(p0, p1, u0, u1, -u0, -u1, u0, u1);
      if (kVar == 2) pk[e >> 1] = __float_as_uint(p0) ^ __float_as_uint(p1);
      else pk[e >> 1] = sm100::pack2<true>(p0, p1);
    }
    if (!ok) pk[0] ^= 1;
    sm100::tmem_st16(tmem + lane_addr + col + 32, pk);
    if ((it & 3) == 3) sm100::tmem_wait_st();
#pragma unroll
    for (int i = 0; i < 16; ++i) acc ^= pk[i];
  }
  long long t1 = clock64();
  sink[blockIdx.x * blockDim.x + threadIdx.x] = acc;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
  sm100::tc_fence_before();
  __syncthreads();
  if (warp == 0) sm100::tmem_dealloc<512>(tmem);
}
template <int kVar>
void run_ab(const char* name, long long* cyc, uint32_t* sink, float bias2) {
  const int iters = 4000, warps = 16;
  kern_ab<kVar><<<148, warps * 32>>>(iters, cyc, sink, bias2);
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) { printf("error %s\n", cudaGetErrorString(e)); return; }
  long long c;
  cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
  printf("  ablation %-40s %6.2f elem/clk/SM\n", name, (double)warps * 32 * 32 * iters / c);
}

int main() {
  long long* cyc;
  uint32_t* sink;
  cudaMalloc(&cyc, 148 * 8);
  cudaMalloc(&sink, 148 * 512 * 4);
  const float b4 = -13.0f, b0 = 0.0f;   // t = s a2 + b2: tier 4 (b = -log 8192 -> b2 ~ -13) / exact tier
  run_ab<0>("full tier-4 path", cyc, sink, b4);
  run_ab<1>("no max / vote", cyc, sink, b4);
  run_ab<2>("no bf16 pack (F2FP)", cyc, sink, b4);
  run_ab<3>("no scale FFMA2", cyc, sink, b4);
  run_ab<4>("no sigma FFMA2 (p = u)", cyc, sink, b4);
  run_ab<5>("exp2 on FMA pipe, 1 pair in 2", cyc, sink, b4);
  run_ab<6>("exp2 on FMA pipe, 1 pair in 3", cyc, sink, b4);
  run_ab<7>("exp2 on FMA pipe, 1 pair in 4", cyc, sink, b4);
  run_ab<8>("exp2 on FMA pipe, 1 pair in 5", cyc, sink, b4);
  run_ab<11>("exp2 on FMA pipe, 1 pair in 8", cyc, sink, b4);
  return 0;
}
