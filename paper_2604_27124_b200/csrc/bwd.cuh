// bwd.cuh -- sm_100a backward kernel of padding-aware sigmoid attention.
//
// The paper splits the backward into a dQ kernel (Alg. 2) and a dK/dV kernel
// (Alg. 3), each recomputing sigma.  Here the two are fused into ONE key-tile-owned
// pass: every (b, h, key tile) item keeps K_j, V_j resident and loops
// over the valid query tiles i, recomputing
//     S^T  = K_j Q_i^T,   dP^T = V_j dO_i^T                    (Alg. 3)
//     P^T  = mask . sigma(alpha S^T + b)
//     dS^T = alpha . P^T (1 - P^T) dP^T                         (alpha of P:669/P:727 folded in)
//     dV_j += P^T dO_i,  dK_j += dS^T Q_i  -- on chip, atomic-free
//     dQ_i += dS K_j  -- fp32 partial per key tile,
//                                                                 reduce-added into a workspace
// so sigma is evaluated once per element and the tensor work is the credited 10 d per pair.
//
// CTA roles (512 threads, persistent):
//   warp 0      TMA: K_j, V_j (2 slots), Q_i + dO_i ring (kQStages)
//   warp 1      MMA issuer (one thread)
//   warp 2      TMEM allocator
//   warps 4-11  two compute warpgroups; thread = key row (TMEM lane), WG g = query columns [64g, 64g+64)
//   warps 12-15 dQ reducer: tcgen05.ld dQ_i (thread = query row) -> red.global.add.v4.f32
// TMEM (d = 64): S^T [0,128) | dP^T [128,256) | dV [256,320) | dK [320,384) | dQ [384,448).
// P^T / dS^T (16-bit) are written back over the first half of each WG's own S^T / dP^T columns
// and feed the dV / dK MMAs straight from TMEM; dS^T is also written to shared memory (128B
// swizzled, keys as rows) where the same bytes serve as the MN-major A operand of dQ = dS K.
#pragma once
#include "fwd.cuh"

namespace sigattn {

struct BwdArgs {
  const int4* items;      // {b, h, key tile, query tiles}
  const int* n_items;
  const int32_t* seqlens_q;
  const int32_t* seqlens_k;
  const float* bias_per_seq;
  float bias;
  float scale;
  int B, H, Nq, Nk;
  float* dq_acc;          // fp32 [B,H,Nq,D], zero on valid rows at entry
  void* dk;               // [B,H,Nk,D]
  void* dv;
};

template <int D>
struct BwdCfg {
  static_assert(D == 64, "fused backward: d = 64 TMEM plan");
  static constexpr int kQStages = 2;
  static constexpr int kTileBytes = kTile * D * 2;           // 16 KB
  static constexpr int kKOff = 0;                            // K[2]
  static constexpr int kVOff = kKOff + 2 * kTileBytes;       // V[2]
  static constexpr int kQOff = kVOff + 2 * kTileBytes;       // Q[kQStages]
  static constexpr int kDOOff = kQOff + kQStages * kTileBytes;
  static constexpr int kDSOff = kDOOff + kQStages * kTileBytes;  // dS^T: 2 halves of [128 keys][64 q]
  static constexpr int kBarOff = kDSOff + 2 * kTile * 128;
  static constexpr int kNumBars = 2 + 2 + 2 * kQStages + 1 + 1 + 1 + 1 + 1 + 1 + 1;
  static constexpr int kSmemBytes = kBarOff + kNumBars * 8 + 16 + 1024;
  static constexpr int kThreads = 512;
  static constexpr uint32_t kTmemCols = 512;
  static constexpr uint32_t kColS = 0, kColDP = 128, kColDV = 256, kColDK = 256 + D, kColDQ = 256 + 2 * D;
};

__device__ __forceinline__ void red_add_v4(float* addr, float a, float b, float c, float d) {
  asm volatile("red.global.add.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(addr), "f"(a), "f"(b), "f"(c), "f"(d)
               : "memory");
}

template <int D, bool kBf16>
__global__ void __launch_bounds__(512, 1)
sigattn_bwd_kernel(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmK,
                   const __grid_constant__ CUtensorMap tmV, const __grid_constant__ CUtensorMap tmDO,
                   const BwdArgs args) {
  using C = BwdCfg<D>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + C::kBarOff);
  uint64_t* kv_full = bars + 0;        // [2]
  uint64_t* kv_empty = bars + 2;       // [2]
  uint64_t* qdo_full = bars + 4;       // [kQStages]
  uint64_t* qdo_empty = qdo_full + C::kQStages;
  uint64_t* s_full = qdo_empty + C::kQStages;
  uint64_t* p_full = s_full + 1;
  uint64_t* ds_free = p_full + 1;
  uint64_t* dq_full = ds_free + 1;
  uint64_t* dq_empty = dq_full + 1;
  uint64_t* acc_full = dq_empty + 1;
  uint64_t* acc_empty = acc_full + 1;
  uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(bars + C::kNumBars);

  const uint32_t warp = sm100::warp_id();
  const uint32_t lane = sm100::lane_id();

  if (threadIdx.x == 0) {
    for (int i = 0; i < 2; ++i) {
      sm100::mbar_init(&kv_full[i], 1);
      sm100::mbar_init(&kv_empty[i], 1);
    }
    for (int i = 0; i < C::kQStages; ++i) {
      sm100::mbar_init(&qdo_full[i], 1);
      sm100::mbar_init(&qdo_empty[i], 1);
    }
    sm100::mbar_init(s_full, 1);
    sm100::mbar_init(p_full, 8);
    sm100::mbar_init(ds_free, 1);
    sm100::mbar_init(dq_full, 1);
    sm100::mbar_init(dq_empty, 4);
    sm100::mbar_init(acc_full, 1);
    sm100::mbar_init(acc_empty, 8);
    sm100::fence_barrier_init();
  }
  if (warp == 0 && lane == 0) {
    sm100::tma_prefetch_desc(&tmQ);
    sm100::tma_prefetch_desc(&tmK);
    sm100::tma_prefetch_desc(&tmV);
    sm100::tma_prefetch_desc(&tmDO);
  }
  if (warp == 2) sm100::tmem_alloc<C::kTmemCols>(tmem_holder);
  sm100::tc_fence_before();
  __syncthreads();
  sm100::tc_fence_after();
  const uint32_t tmem = *tmem_holder;
  const int n_items = *args.n_items;

  if (warp == 0) {
    // ===================== TMA producer =====================
    if (lane == 0) {
      const uint64_t pol_kv = sm100::policy_evict_first();
      const uint64_t pol_q = sm100::policy_evict_last();
      uint32_t kv_c = 0, qi = 0;
      for (int it = blockIdx.x; it < n_items; it += gridDim.x) {
        const int4 item = args.items[it];
        const int b = item.x, h = item.y, kt = item.z, nqt = item.w;
        if (nqt <= 0) continue;
        const int zh = b * args.H + h;
        const uint32_t kvb = kv_c & 1;
        sm100::mbar_wait(&kv_empty[kvb], ((kv_c >> 1) & 1) ^ 1);
        sm100::mbar_arrive_expect_tx(&kv_full[kvb], 2 * C::kTileBytes);
        sm100::tma_load_3d(smem + C::kKOff + kvb * C::kTileBytes, &tmK, &kv_full[kvb], 0, kt * kTile, zh, pol_kv);
        sm100::tma_load_3d(smem + C::kVOff + kvb * C::kTileBytes, &tmV, &kv_full[kvb], 0, kt * kTile, zh, pol_kv);
        for (int i = 0; i < nqt; ++i, ++qi) {
          const uint32_t st = qi % C::kQStages;
          sm100::mbar_wait(&qdo_empty[st], ((qi / C::kQStages) & 1) ^ 1);
          sm100::mbar_arrive_expect_tx(&qdo_full[st], 2 * C::kTileBytes);
          sm100::tma_load_3d(smem + C::kQOff + st * C::kTileBytes, &tmQ, &qdo_full[st], 0, i * kTile, zh, pol_q);
          sm100::tma_load_3d(smem + C::kDOOff + st * C::kTileBytes, &tmDO, &qdo_full[st], 0, i * kTile, zh, pol_q);
        }
        ++kv_c;
      }
    }
  } else if (warp == 1) {
    // ===================== MMA issuer =====================
    if (lane == 0) {
      constexpr uint32_t idesc_st = sm100::make_idesc_f16(kBf16, 128, 128, false, false);  // S^T, dP^T
      constexpr uint32_t idesc_acc = sm100::make_idesc_f16(kBf16, 128, D, false, true);    // dV, dK (A tmem)
      constexpr uint32_t idesc_dq = sm100::make_idesc_f16(kBf16, 128, D, true, true);      // dQ (A = dS MN-major)
      const uint32_t k_base = sm100::smem_u32(smem + C::kKOff);
      const uint32_t v_base = sm100::smem_u32(smem + C::kVOff);
      const uint32_t q_base = sm100::smem_u32(smem + C::kQOff);
      const uint32_t do_base = sm100::smem_u32(smem + C::kDOOff);
      const uint32_t ds_base = sm100::smem_u32(smem + C::kDSOff);
      uint32_t kv_c = 0, qi = 0;
      for (int it = blockIdx.x; it < n_items; it += gridDim.x) {
        const int nqt = args.items[it].w;
        if (nqt <= 0) continue;
        const uint32_t kvb = kv_c & 1;
        sm100::mbar_wait(&kv_full[kvb], (kv_c >> 1) & 1);
        const uint32_t ka = k_base + kvb * C::kTileBytes;
        const uint32_t va = v_base + kvb * C::kTileBytes;
        for (int i = 0; i < nqt; ++i, ++qi) {
          const uint32_t st = qi % C::kQStages;
          sm100::mbar_wait(&qdo_full[st], (qi / C::kQStages) & 1);
          sm100::tc_fence_after();
          const uint32_t qa = q_base + st * C::kTileBytes;
          const uint32_t da = do_base + st * C::kTileBytes;
          // S^T = K Q^T  and  dP^T = V dO^T   (M = keys, N = queries, K = d; all K-major)
#pragma unroll
          for (int kk = 0; kk < D / 16; ++kk)
            sm100::mma_ss(tmem + C::kColS, sm100::make_sdesc_sw128(ka + kk * 32, 16, 1024),
                          sm100::make_sdesc_sw128(qa + kk * 32, 16, 1024), idesc_st, kk > 0);
#pragma unroll
          for (int kk = 0; kk < D / 16; ++kk)
            sm100::mma_ss(tmem + C::kColDP, sm100::make_sdesc_sw128(va + kk * 32, 16, 1024),
                          sm100::make_sdesc_sw128(da + kk * 32, 16, 1024), idesc_st, kk > 0);
          sm100::mma_commit(s_full);
          sm100::mbar_wait(p_full, qi & 1);
          if (i == 0) sm100::mbar_wait(acc_empty, (kv_c & 1) ^ 1);
          sm100::tc_fence_after();
          // dV += P^T dO ;  dK += dS^T Q   (M = keys, N = d, K = queries; A from TMEM, B MN-major)
#pragma unroll
          for (int kk = 0; kk < kTile / 16; ++kk) {
            const uint32_t a_off = (kk >> 2) * 64 + (kk & 3) * 8;
            sm100::mma_ts(tmem + C::kColDV, tmem + C::kColS + a_off,
                          sm100::make_sdesc_sw128(da + kk * 2048, kTile * 128, 1024), idesc_acc,
                          (i > 0 || kk > 0) ? 1u : 0u);
          }
#pragma unroll
          for (int kk = 0; kk < kTile / 16; ++kk) {
            const uint32_t a_off = (kk >> 2) * 64 + (kk & 3) * 8;
            sm100::mma_ts(tmem + C::kColDK, tmem + C::kColDP + a_off,
                          sm100::make_sdesc_sw128(qa + kk * 2048, kTile * 128, 1024), idesc_acc,
                          (i > 0 || kk > 0) ? 1u : 0u);
          }
          // dQ_i = dS K_j   (M = queries, N = d, K = keys; A = dS MN-major smem, B = K MN-major smem)
          sm100::mbar_wait(dq_empty, (qi & 1) ^ 1);
          sm100::tc_fence_after();
#pragma unroll
          for (int kk = 0; kk < kTile / 16; ++kk)
            sm100::mma_ss(tmem + C::kColDQ, sm100::make_sdesc_sw128(ds_base + kk * 2048, kTile * 128, 1024),
                          sm100::make_sdesc_sw128(ka + kk * 2048, kTile * 128, 1024), idesc_dq, kk > 0);
          sm100::mma_commit(&qdo_empty[st]);
          sm100::mma_commit(ds_free);
          sm100::mma_commit(dq_full);
        }
        sm100::mma_commit(&kv_empty[kvb]);
        sm100::mma_commit(acc_full);
        ++kv_c;
      }
    }
  } else if (warp >= 4 && warp < 12) {
    // ===================== compute warpgroups =====================
    const uint32_t g = (warp - 4) >> 2;
    const uint32_t quarter = warp & 3;
    const uint32_t row = quarter * 32 + lane;          // key row within the tile = TMEM lane
    const uint32_t lane_addr = (quarter * 32) << 16;
    uint8_t* ds_row = smem + C::kDSOff + g * (kTile * 128) + (row >> 3) * 1024 + (row & 7) * 128;
    uint32_t kv_c = 0, qi = 0;
    for (int it = blockIdx.x; it < n_items; it += gridDim.x) {
      const int4 item = args.items[it];
      const int b = item.x, h = item.y, kt = item.z, nqt = item.w;
      if (nqt <= 0) continue;
      const int nq = clampi(args.seqlens_q ? args.seqlens_q[b] : args.Nq, 0, args.Nq);
      const int nk = clampi(args.seqlens_k ? args.seqlens_k[b] : args.Nk, 0, args.Nk);
      const float bias = args.bias_per_seq ? args.bias_per_seq[b] : args.bias;
      const float a2 = -args.scale * kLog2e;
      const float b2 = -bias * kLog2e;
      const float alpha = args.scale;
      const int key = kt * kTile + (int)row;
      const bool key_valid = key < nk;
      for (int i = 0; i < nqt; ++i, ++qi) {
        sm100::mbar_wait(s_full, qi & 1);
        sm100::mbar_wait(ds_free, (qi & 1) ^ 1);
        sm100::tc_fence_after();
        const int q0 = i * kTile + (int)g * 64;
#pragma unroll
        for (int ch = 0; ch < 2; ++ch) {
          uint32_t s[32], dp[32];
          sm100::tmem_ld32(tmem + lane_addr + C::kColS + g * 64 + ch * 32, s);
          sm100::tmem_ld32(tmem + lane_addr + C::kColDP + g * 64 + ch * 32, dp);
          sm100::tmem_wait_ld_dep(s);
          sm100::tmem_wait_ld_dep(dp);
          const int qc = q0 + ch * 32;
          const bool need_mask = !key_valid || (qc + 32 > nq);
          uint32_t pp[16], dd[16];
#pragma unroll
          for (int e = 0; e < 32; e += 2) {
            float p0 = sm100::rcp_approx(1.0f + sm100::ex2_approx(fmaf(__uint_as_float(s[e]), a2, b2)));
            float p1 = sm100::rcp_approx(1.0f + sm100::ex2_approx(fmaf(__uint_as_float(s[e + 1]), a2, b2)));
            float d0 = (p0 - p0 * p0) * __uint_as_float(dp[e]) * alpha;
            float d1 = (p1 - p1 * p1) * __uint_as_float(dp[e + 1]) * alpha;
            if (need_mask) {
              const bool v0 = key_valid && (qc + e < nq);
              const bool v1 = key_valid && (qc + e + 1 < nq);
              p0 = v0 ? p0 : 0.0f;
              d0 = v0 ? d0 : 0.0f;
              p1 = v1 ? p1 : 0.0f;
              d1 = v1 ? d1 : 0.0f;
            }
            pp[e >> 1] = sm100::pack2<kBf16>(p0, p1);
            dd[e >> 1] = sm100::pack2<kBf16>(d0, d1);
          }
          sm100::tmem_st16(tmem + lane_addr + C::kColS + g * 64 + ch * 16, pp);
          sm100::tmem_st16(tmem + lane_addr + C::kColDP + g * 64 + ch * 16, dd);
          // dS^T row into the swizzled smem tile: 32 queries = 64 B = 16-byte chunks 4ch..4ch+3
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            const uint32_t chunk = (uint32_t)(ch * 4 + u) ^ (row & 7);
            *reinterpret_cast<uint4*>(ds_row + chunk * 16) =
                make_uint4(dd[4 * u], dd[4 * u + 1], dd[4 * u + 2], dd[4 * u + 3]);
          }
        }
        sm100::tmem_wait_st();
        sm100::fence_proxy_async_smem();
        sm100::tc_fence_before();
        __syncwarp();
        if (lane == 0) sm100::mbar_arrive(p_full);
      }
      // ---- epilogue: dV, dK rows of this key tile, columns [g*D/2, g*D/2 + D/2)
      sm100::mbar_wait(acc_full, kv_c & 1);
      sm100::tc_fence_after();
      constexpr int kHalf = D / 2;
      uint32_t rv[32], rk[32];
      static_assert(kHalf == 32, "d = 64");
      sm100::tmem_ld32(tmem + lane_addr + C::kColDV + g * kHalf, rv);
      sm100::tmem_ld32(tmem + lane_addr + C::kColDK + g * kHalf, rk);
      sm100::tmem_wait_ld_dep(rv);
      sm100::tmem_wait_ld_dep(rk);
      sm100::tc_fence_before();
      __syncwarp();
      if (lane == 0) sm100::mbar_arrive(acc_empty);
      if (key < args.Nk) {
        const size_t off = ((size_t)(b * args.H + h) * args.Nk + key) * D + g * kHalf;
        uint4* dvp = reinterpret_cast<uint4*>(reinterpret_cast<uint16_t*>(args.dv) + off);
        uint4* dkp = reinterpret_cast<uint4*>(reinterpret_cast<uint16_t*>(args.dk) + off);
#pragma unroll
        for (int e = 0; e < kHalf; e += 8) {
          uint4 wv, wk;
          wv.x = key_valid ? sm100::pack2<kBf16>(__uint_as_float(rv[e]), __uint_as_float(rv[e + 1])) : 0u;
          wv.y = key_valid ? sm100::pack2<kBf16>(__uint_as_float(rv[e + 2]), __uint_as_float(rv[e + 3])) : 0u;
          wv.z = key_valid ? sm100::pack2<kBf16>(__uint_as_float(rv[e + 4]), __uint_as_float(rv[e + 5])) : 0u;
          wv.w = key_valid ? sm100::pack2<kBf16>(__uint_as_float(rv[e + 6]), __uint_as_float(rv[e + 7])) : 0u;
          wk.x = key_valid ? sm100::pack2<kBf16>(__uint_as_float(rk[e]), __uint_as_float(rk[e + 1])) : 0u;
          wk.y = key_valid ? sm100::pack2<kBf16>(__uint_as_float(rk[e + 2]), __uint_as_float(rk[e + 3])) : 0u;
          wk.z = key_valid ? sm100::pack2<kBf16>(__uint_as_float(rk[e + 4]), __uint_as_float(rk[e + 5])) : 0u;
          wk.w = key_valid ? sm100::pack2<kBf16>(__uint_as_float(rk[e + 6]), __uint_as_float(rk[e + 7])) : 0u;
          dvp[e >> 3] = wv;
          dkp[e >> 3] = wk;
        }
      }
      ++kv_c;
    }
  } else if (warp >= 12) {
    // ===================== dQ reducer =====================
    const uint32_t quarter = warp & 3;
    const uint32_t row = quarter * 32 + lane;      // query row within the tile
    const uint32_t lane_addr = (quarter * 32) << 16;
    uint32_t qi = 0;
    for (int it = blockIdx.x; it < n_items; it += gridDim.x) {
      const int4 item = args.items[it];
      const int b = item.x, h = item.y, nqt = item.w;
      if (nqt <= 0) continue;
      const int nq = clampi(args.seqlens_q ? args.seqlens_q[b] : args.Nq, 0, args.Nq);
      const size_t zrow0 = (size_t)(b * args.H + h) * args.Nq;
      for (int i = 0; i < nqt; ++i, ++qi) {
        sm100::mbar_wait(dq_full, qi & 1);
        sm100::tc_fence_after();
        uint32_t r0[32], r1[32];
        sm100::tmem_ld32(tmem + lane_addr + C::kColDQ, r0);
        sm100::tmem_ld32(tmem + lane_addr + C::kColDQ + 32, r1);
        sm100::tmem_wait_ld_dep(r0);
        sm100::tmem_wait_ld_dep(r1);
        sm100::tc_fence_before();
        __syncwarp();
        if (lane == 0) sm100::mbar_arrive(dq_empty);
        const int q = i * kTile + (int)row;
        if (q < nq) {
          float* dst = args.dq_acc + (zrow0 + q) * D;
#pragma unroll
          for (int e = 0; e < 32; e += 4)
            red_add_v4(dst + e, __uint_as_float(r0[e]), __uint_as_float(r0[e + 1]), __uint_as_float(r0[e + 2]),
                       __uint_as_float(r0[e + 3]));
#pragma unroll
          for (int e = 0; e < 32; e += 4)
            red_add_v4(dst + 32 + e, __uint_as_float(r1[e]), __uint_as_float(r1[e + 1]), __uint_as_float(r1[e + 2]),
                       __uint_as_float(r1[e + 3]));
        }
      }
    }
  }

  sm100::tc_fence_before();
  __syncthreads();
  if (warp == 2) sm100::tmem_dealloc<C::kTmemCols>(tmem);
}

}  // namespace sigattn
