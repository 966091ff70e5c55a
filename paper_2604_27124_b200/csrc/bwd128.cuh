// bwd128.cuh -- sm_100a backward kernel for head dimension d = 128 (same method as bwd.cuh).
//
// With d = 128 the d-wide accumulators dV, dK (128 TMEM columns each) leave no room for full
// 128x128 score tiles, so each key tile (128 keys, owned by the CTA; K_j, V_j resident in smem)
// loops over 64-query tiles i and dQ is produced transposed (M = d) so that it needs only 64
// columns:
//     S^T  = K_j Q_i^T,   dP^T = V_j dO_i^T          SS, M = 128 keys, N = 64 queries, K = d
//     P^T  = mask . sigma(alpha S^T + b),  dS^T = P^T (1 - P^T) dP^T
//     dV_j += P^T dO_i,   dK_j += dS^T Q_i           TS (P^T, dS^T in TMEM), N = d = 128
//     dQ_i^T = K_j^T dS_i^T                          SS, M = d, N = 64 queries, K = keys
//                                                    (A = K read MN-major, B = dS^T smem MN-major)
// dQ^T is drained lane = d index into a swizzled fp32 smem tile [64 q][128 d] (four SW128 boxes of
// 32 columns) and added into the fp32 workspace by four TMA bulk tensor reduce-adds (in L2); alpha
// is applied in the epilogues.  MMA order per tile: dV/dK(i) | S,dP(i+1) | dQ(i), so
// the compute warps start on tile i+1 while dQ(i) runs.
// Roles as in bwd.cuh (768 threads): warps 0-15 compute (warpgroup w: queries [16w, 16w+16) of the
// 64-query tile), 16-19 epilogue, 20 TMA, 21 MMA, 22 TMEM allocator.
// TMEM: S^T [0,64) dP^T [64,128) dV [128,256) dK [256,384) dQ^T [384,448).
// Shared memory: K, V (single slot, 2 x 32 KB), Q_i + dO_i ring (3 x 2 x 16 KB), dS^T (2 x 16 KB).
#pragma once
#include <type_traits>
#include "bwd.cuh"

namespace sigattn {

struct Bwd128Cfg {
  static constexpr int D = 128;
  static constexpr int kQT = 64;                             // queries per tile
  static constexpr int kKVBytes = kTile * D * 2;             // 32 KB: [128 keys][2 x 64 d]
  static constexpr int kQBytes = kQT * D * 2;                // 16 KB: [64 q][2 x 64 d]
  static constexpr int kQStages = 3;
  static constexpr int kKOff = 0;
  static constexpr int kVOff = kKOff + kKVBytes;
  static constexpr int kQOff = kVOff + kKVBytes;
  static constexpr int kDOOff = kQOff + kQStages * kQBytes;
  static constexpr int kDSOff = kDOOff + kQStages * kQBytes;
  static constexpr int kDSBytes = kTile * 128;               // [128 keys][64 q] 16-bit = 16 KB
  static constexpr int kDQOff = kDSOff + 2 * kDSBytes;       // fp32 dQ staging: 4 boxes [64 q][32 d] SW128
  static constexpr int kDQBytes = kQT * D * 4;               // 32 KB
  static constexpr int kBarOff = kDQOff + kDQBytes;
  static constexpr int kNumBars = 2 + 2 * kQStages + 1 + 1 + 2 + 1 + 1 + 1 + 1 + 1;
  static constexpr int kSmemBytes = kBarOff + kNumBars * 8 + 16 + 1024;
  static constexpr int kWarpEpi = 16, kWarpTMA = 20, kWarpMMA = 21, kWarpAlloc = 22, kWarpFill = 23;
  static constexpr int kThreads = 768;
  static constexpr uint32_t kTmemCols = 512;
  static constexpr uint32_t kColS = 0, kColDP = 64, kColDV = 128, kColDK = 256, kColDQ = 384;
};

// kDQ = false: dK, dV only (deterministic backward, Alg. 3); see bwd.cuh.
template <bool kBf16, bool kDQ = true, bool kDB = false, bool kBSHD = false>
__global__ void __launch_bounds__(Bwd128Cfg::kThreads, 1)
sigattn_bwd128_kernel(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmK,
                      const __grid_constant__ CUtensorMap tmV, const __grid_constant__ CUtensorMap tmDO,
                      const __grid_constant__ CUtensorMap tmDQ, const BwdArgs args) {
  using C = Bwd128Cfg;
  constexpr int D = C::D;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + C::kBarOff);
  uint64_t* kv_full = bars + 0;
  uint64_t* kv_empty = bars + 1;
  uint64_t* qdo_full = bars + 2;                  // [kQStages]
  uint64_t* qdo_empty = qdo_full + C::kQStages;
  uint64_t* s_full = qdo_empty + C::kQStages;
  uint64_t* p_full = s_full + 1;
  uint64_t* ds_free = p_full + 1;                 // [2]
  uint64_t* dq_full = ds_free + 2;
  uint64_t* dq_empty = dq_full + 1;
  uint64_t* acc_full = dq_empty + 1;
  uint64_t* acc_empty = acc_full + 1;
  uint64_t* dp_full = acc_empty + 1;              // dP^T landed (S^T lands first: s_full)
  uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(bars + C::kNumBars);

  const uint32_t warp = sm100::warp_id();
  const uint32_t lane = sm100::lane_id();

  if (threadIdx.x == 0) {
    sm100::mbar_init(kv_full, 1);
    sm100::mbar_init(kv_empty, 1);
    for (int i = 0; i < C::kQStages; ++i) {
      sm100::mbar_init(&qdo_full[i], 1);
      sm100::mbar_init(&qdo_empty[i], 1);
    }
    sm100::mbar_init(s_full, 1);
    sm100::mbar_init(dp_full, 1);
    sm100::mbar_init(p_full, 16);
    sm100::mbar_init(&ds_free[0], 1);
    sm100::mbar_init(&ds_free[1], 1);
    sm100::mbar_init(dq_full, 1);
    sm100::mbar_init(dq_empty, 4);
    sm100::mbar_init(acc_full, 1);
    sm100::mbar_init(acc_empty, 4);
    sm100::fence_barrier_init();
  }
  if (warp == C::kWarpTMA && lane == 0) {
    sm100::tma_prefetch_desc(&tmQ);
    sm100::tma_prefetch_desc(&tmK);
    sm100::tma_prefetch_desc(&tmV);
    sm100::tma_prefetch_desc(&tmDO);
  }
  if (warp == C::kWarpAlloc) sm100::tmem_alloc<C::kTmemCols>(tmem_holder);
  sm100::tc_fence_before();
  __syncthreads();
  sm100::tc_fence_after();
  const uint32_t tmem = *tmem_holder;
  const int n_items = *args.n_items;
  auto item_tiles = [&](int b) {   // 64-query tiles of sequence b
    const int nq = clampi(args.seqlens_q ? args.seqlens_q[b] : args.Nq, 0, args.Nq);
    return (nq + C::kQT - 1) / C::kQT;
  };

  if (warp == C::kWarpTMA) {
    // ===================== TMA producer =====================
    const uint64_t pol_kv = sm100::policy_evict_first();
    const uint64_t pol_q = sm100::policy_evict_last();
    uint32_t kv_c = 0, t = 0;
    for (int it = first_item(); it < n_items; it = next_item(it)) {
      const int4 item = args.items[it];
      if (item.w <= 0) continue;
      const int b = item.x, h = item.y, kt = item.z, nqt = item_tiles(b);
      const int zh = b * args.H + h;
      sm100::mbar_wait_backoff(kv_empty, (kv_c & 1) ^ 1);
      if (sm100::elect_one()) {
        sm100::mbar_arrive_expect_tx(kv_full, 2 * C::kKVBytes);
#pragma unroll
        for (int s = 0; s < 2; ++s) {
          sm100::tma_load_bh(smem + C::kKOff + s * (kTile * 128), &tmK, kv_full, s * 64, kt * kTile, zh, pol_kv, kBSHD ? args.H : 0);
          sm100::tma_load_bh(smem + C::kVOff + s * (kTile * 128), &tmV, kv_full, s * 64, kt * kTile, zh, pol_kv, kBSHD ? args.H : 0);
        }
      }
      __syncwarp();
      for (int i = 0; i < nqt; ++i, ++t) {
        const uint32_t st = t % C::kQStages;
        sm100::mbar_wait_backoff(&qdo_empty[st], ((t / C::kQStages) & 1) ^ 1);
        if (sm100::elect_one()) {
          sm100::mbar_arrive_expect_tx(&qdo_full[st], 2 * C::kQBytes);
#pragma unroll
          for (int s = 0; s < 2; ++s) {
            sm100::tma_load_bh(smem + C::kQOff + st * C::kQBytes + s * (C::kQT * 128), &tmQ, &qdo_full[st], s * 64,
                               i * C::kQT, zh, pol_q, kBSHD ? args.H : 0);
            sm100::tma_load_bh(smem + C::kDOOff + st * C::kQBytes + s * (C::kQT * 128), &tmDO, &qdo_full[st],
                               s * 64, i * C::kQT, zh, pol_q, kBSHD ? args.H : 0);
          }
        }
        __syncwarp();
      }
      ++kv_c;
    }
  } else if (warp == C::kWarpMMA) {
    // ===================== MMA issuer =====================
    constexpr uint32_t idesc_s = sm100::make_idesc_f16(kBf16, 128, C::kQT, false, false);   // S^T, dP^T
    constexpr uint32_t idesc_acc = sm100::make_idesc_f16(kBf16, 128, D, false, true);       // dV, dK
    constexpr uint32_t idesc_dq = sm100::make_idesc_f16(kBf16, 128, C::kQT, true, true);    // dQ^T
    const uint32_t k_base = sm100::smem_u32(smem + C::kKOff);
    const uint32_t v_base = sm100::smem_u32(smem + C::kVOff);
    const uint32_t q_base = sm100::smem_u32(smem + C::kQOff);
    const uint32_t do_base = sm100::smem_u32(smem + C::kDOOff);
    const uint32_t ds_base = sm100::smem_u32(smem + C::kDSOff);
    // S^T then dP^T, each on its own barrier: the compute warps start sigma while dP^T is computed
    auto mma_s_only = [&](uint32_t st) {
      const uint32_t qa = q_base + st * C::kQBytes;
#pragma unroll
      for (int kk = 0; kk < D / 16; ++kk) {
        const uint32_t ko = (kk >> 2) * (kTile * 128) + (kk & 3) * 32, qo = (kk >> 2) * (C::kQT * 128) + (kk & 3) * 32;
        sm100::mma_ss(tmem + C::kColS, sm100::sdesc_add(sm100::make_sdesc_sw128(k_base, 16, 1024), ko),
                      sm100::sdesc_add(sm100::make_sdesc_sw128(qa, 16, 1024), qo), idesc_s, kk > 0);
      }
      sm100::mma_commit(s_full);
    };
    auto mma_dp_only = [&](uint32_t st) {
      const uint32_t da = do_base + st * C::kQBytes;
#pragma unroll
      for (int kk = 0; kk < D / 16; ++kk) {
        const uint32_t ko = (kk >> 2) * (kTile * 128) + (kk & 3) * 32, qo = (kk >> 2) * (C::kQT * 128) + (kk & 3) * 32;
        sm100::mma_ss(tmem + C::kColDP, sm100::sdesc_add(sm100::make_sdesc_sw128(v_base, 16, 1024), ko),
                      sm100::sdesc_add(sm100::make_sdesc_sw128(da, 16, 1024), qo), idesc_s, kk > 0);
      }
      sm100::mma_commit(dp_full);
    };
    auto mma_s = [&](uint32_t st) {
      mma_s_only(st);
      mma_dp_only(st);
    };
    auto mma_dq = [&](uint32_t buf) {
      const uint32_t dsa = ds_base + buf * C::kDSBytes;
      // dQ^T = K^T dS^T: A = K read MN-major (M = d: 64-wide atoms at LBO = 16 KB), B = dS^T MN-major
#pragma unroll
      for (int kk = 0; kk < kTile / 16; ++kk)
        sm100::mma_ss(tmem + C::kColDQ, sm100::sdesc_add(sm100::make_sdesc_sw128(k_base, kTile * 128, 1024), kk * 2048),
                      sm100::sdesc_add(sm100::make_sdesc_sw128(dsa, 16, 1024), kk * 2048), idesc_dq, kk > 0);
    };

    uint32_t t = 0, item_c = 0;
    bool primed = false;   // S/dP of the current tile already issued
    for (int it = first_item(); it < n_items; it = next_item(it)) {
      const int4 item = args.items[it];
      if (item.w <= 0) continue;
      const int nqt = item_tiles(item.x);
      sm100::mbar_wait(kv_full, item_c & 1);
      if (!primed) {
        sm100::mbar_wait(&qdo_full[t % C::kQStages], (t / C::kQStages) & 1);
        sm100::tc_fence_after();
        if (sm100::elect_one()) mma_s(t % C::kQStages);
        __syncwarp();
      }
      for (int i = 0; i < nqt; ++i, ++t) {
        const uint32_t st = t % C::kQStages, buf = t & 1;
        sm100::mbar_wait_backoff(p_full, t & 1);
        if (i == 0) sm100::mbar_wait(acc_empty, (item_c & 1) ^ 1);
        sm100::tc_fence_after();
        // dV(i) | S(i+1) | dK(i) | dP(i+1) | dQ(i): S(i+1) overwrites the S^T columns right after dV(i)
        // has read P^T(i) from them, dP(i+1) the dP^T columns after dK(i) has read dS^T(i) (in-order
        // tcgen05 execution), so the compute warps get the next scores four MMAs earlier
        const bool has_next_here = i + 1 < nqt;
        const uint32_t st1 = (t + 1) % C::kQStages;
        if (sm100::elect_one()) {
          const uint32_t da = do_base + st * C::kQBytes;
#pragma unroll
          for (int kk = 0; kk < C::kQT / 16; ++kk)   // dV += P^T dO  (queries 16kk: warpgroup kk's columns)
            sm100::mma_ts(tmem + C::kColDV, tmem + C::kColS + kk * 16,
                          sm100::sdesc_add(sm100::make_sdesc_sw128(da, C::kQT * 128, 1024), kk * 2048), idesc_acc,
                          (i == 0 && kk == 0) ? 0u : 1u);
        }
        __syncwarp();
        if (has_next_here) {
          sm100::mbar_wait(&qdo_full[st1], ((t + 1) / C::kQStages) & 1);
          sm100::tc_fence_after();
          if (sm100::elect_one()) mma_s_only(st1);
          __syncwarp();
        }
        if (sm100::elect_one()) {
          const uint32_t qa = q_base + st * C::kQBytes;
#pragma unroll
          for (int kk = 0; kk < C::kQT / 16; ++kk)   // dK += dS^T Q
            sm100::mma_ts(tmem + C::kColDK, tmem + C::kColDP + kk * 16,
                          sm100::sdesc_add(sm100::make_sdesc_sw128(qa, C::kQT * 128, 1024), kk * 2048), idesc_acc,
                          (i == 0 && kk == 0) ? 0u : 1u);
          sm100::mma_commit(&qdo_empty[st]);
          if (i == nqt - 1) sm100::mma_commit(acc_full);
          if (i == 0 && args.counters) atomicAdd(args.counters + 1, (unsigned long long)nqt);
          if (has_next_here) mma_dp_only(st1);
        }
        __syncwarp();
        if constexpr (kDQ) {
          sm100::mbar_wait(dq_empty, (t & 1) ^ 1);
          sm100::tc_fence_after();
          if (sm100::elect_one()) {
            mma_dq(buf);
            sm100::mma_commit(&ds_free[buf]);
            sm100::mma_commit(dq_full);
            if (i == nqt - 1) sm100::mma_commit(kv_empty);
          }
        } else {
          if (sm100::elect_one() && i == nqt - 1) sm100::mma_commit(kv_empty);
        }
        __syncwarp();
      }
      primed = false;   // the next item's K/V arrive only after this item's last dQ (single K/V slot)
      ++item_c;
    }
  } else if (warp < C::kWarpEpi) {
    // ===================== compute warps: warpgroup w4 = queries [16 w4, 16 w4 + 16) =====================
    const uint32_t w4 = warp >> 2;
    const uint32_t quarter = warp & 3;
    const uint32_t row = quarter * 32 + lane;
    const uint32_t lane_addr = (quarter * 32) << 16;
    const uint32_t s_col = C::kColS + w4 * 16, dp_col = C::kColDP + w4 * 16;
    const uint32_t ds_row = sm100::smem_u32(smem + C::kDSOff + (row >> 3) * 1024 + (row & 7) * 128);
    uint32_t t = 0;
    for (int it = first_item(); it < n_items; it = next_item(it)) {
      const int4 item = args.items[it];
      if (item.w <= 0) continue;
      const int b = item.x, kt = item.z, nqt = item_tiles(b);
      const int nq = clampi(args.seqlens_q ? args.seqlens_q[b] : args.Nq, 0, args.Nq);
      const int nk = clampi(args.seqlens_k ? args.seqlens_k[b] : args.Nk, 0, args.Nk);
      const float bias = args.bias_per_seq ? args.bias_per_seq[b] : args.bias;
      const float a2 = args.scale * kLog2e;
      const float b2 = bias * kLog2e;
      const bool key_valid = kt * kTile + (int)row < nk;
      const bool warp_keys_valid = __all_sync(0xffffffffu, key_valid);
      float db_acc = 0.f;
      bool spec = true;   // speculate while the last chunk took the speculated tier
      // the query loop, instantiated for the item's speculative sigma tier (one hot copy per item)
      auto query_loop = [&](auto tier_c) {
        constexpr int kT = decltype(tier_c)::value;
        for (int i = 0; i < nqt; ++i, ++t) {
          SIGATTN_COMPUTE_WAIT(s_full, t & 1);
          if (kDQ) sm100::mbar_wait(&ds_free[t & 1], ((t >> 1) & 1) ^ 1);
          sm100::tc_fence_after();
          float s[16], dp[16];
          sm100::tmem_ld16(tmem + lane_addr + s_col, s);
          sm100::tmem_wait_ld_dep16(s);
          const int ncol = nq - (i * C::kQT + (int)w4 * 16);
          const bool full = warp_keys_valid && ncol >= 16;
          const int nv = full ? 16 : (key_valid ? ncol : 0);
          if (full) bwd_sigma16<false, true, kT>(s, a2, b2, true, 16, tmem + lane_addr + s_col, spec);
          else bwd_sigma16<true, true, kT>(s, a2, b2, key_valid, nv, tmem + lane_addr + s_col, spec);
          // dP^T lands after S^T: sigma above overlaps the dP^T MMAs
          SIGATTN_COMPUTE_WAIT(dp_full, t & 1);
          sm100::tc_fence_after();
          sm100::tmem_ld16(tmem + lane_addr + dp_col, dp);
          sm100::tmem_wait_ld_dep16(dp);
          uint32_t pp[8], dd[8];
          if (full) bwd_ds16<false, kBf16, kDB>(s, dp, pp, dd, 16, &db_acc);
          else bwd_ds16<true, kBf16, kDB>(s, dp, pp, dd, nv, &db_acc);
          sm100::tmem_st8(tmem + lane_addr + s_col, pp);
          sm100::tmem_st8(tmem + lane_addr + dp_col, dd);
          if constexpr (kDQ) {
            const uint32_t dsr = ds_row + (t & 1) * C::kDSBytes;
#pragma unroll
            for (int u = 0; u < 2; ++u) {
              const uint32_t chunk = (uint32_t)(w4 * 2 + u) ^ (row & 7);
              sm100::st_shared_v4(dsr + chunk * 16, dd[4 * u], dd[4 * u + 1], dd[4 * u + 2], dd[4 * u + 3]);
            }
          }
          sm100::tmem_wait_st();
          if (kDQ) sm100::fence_proxy_async_smem();
          sm100::tc_fence_before();
          __syncwarp();
          if (lane == 0) sm100::mbar_arrive(p_full);
        }
      };
      if (bias <= kSpec4MaxBias) query_loop(std::integral_constant<int, 4>{});
      else query_loop(std::integral_constant<int, 2>{});
      if constexpr (kDB) dbias_flush(args.dbias, b, db_acc, lane);
    }
  } else if (warp < C::kWarpTMA) {
    // ===================== epilogue: dQ^T drain (lane = d index) + dK/dV =====================
    constexpr uint32_t kEpiThread0 = 32 * C::kWarpEpi;
    const uint32_t quarter = warp & 3;
    const uint32_t row = quarter * 32 + lane;          // d index for dQ^T, key row for dK/dV
    const uint32_t lane_addr = (quarter * 32) << 16;
    const float alpha = args.scale;
    uint32_t t = 0, item_c = 0;
    for (int it = first_item(); it < n_items; it = next_item(it)) {
      const int4 item = args.items[it];
      if (item.w <= 0) continue;
      const int b = item.x, h = item.y, kt = item.z, nqt = item_tiles(b);
      const int nq = clampi(args.seqlens_q ? args.seqlens_q[b] : args.Nq, 0, args.Nq);
      const int nk = clampi(args.seqlens_k ? args.seqlens_k[b] : args.Nk, 0, args.Nk);
      const size_t zh = (size_t)(b * args.H + h);
      for (int i = 0; i < nqt * kDQ; ++i, ++t) {
        sm100::mbar_wait_backoff(dq_full, t & 1);
        sm100::tc_fence_after();
        float r[4][16];
#pragma unroll
        for (int c4 = 0; c4 < 4; ++c4) sm100::tmem_ld16(tmem + lane_addr + C::kColDQ + c4 * 16, r[c4]);
#pragma unroll
        for (int c4 = 0; c4 < 4; ++c4) sm100::tmem_wait_ld_dep16(r[c4]);
        sm100::tc_fence_before();
        __syncwarp();
        if (lane == 0) sm100::mbar_arrive(dq_empty);
        // alpha dQ^T -> the fp32 staging tile [64 q][128 d] as four SW128 [64][32] boxes (thread = d
        // index: every store of a warp hits 32 distinct banks), then one thread reduce-adds the boxes
        // into the accumulator through the TMA (rows past Nq clipped; padded query rows add zeros).
        uint8_t* dqs = smem + C::kDQOff;
        if (threadIdx.x == kEpiThread0) sm100::bulk_wait_group_read<0>();   // previous tile's reduce read it
        sm100::named_bar_sync(1, 128);
        {
          const uint32_t hh = row >> 5, j = row & 31;   // box, float within the 128-byte row
          const uint32_t bbase = sm100::smem_u32(dqs) + hh * (C::kQT * 128) + (j & 3) * 4;
#pragma unroll
          for (int c4 = 0; c4 < 4; ++c4)
#pragma unroll
            for (int e = 0; e < 16; ++e) {
              const uint32_t q = c4 * 16 + e;
              sm100::st_shared_f32(bbase + q * 128 + (((j >> 2) ^ (q & 7)) * 16), alpha * r[c4][e]);
            }
        }
        sm100::fence_proxy_async_smem();
        sm100::named_bar_sync(1, 128);
        if (threadIdx.x == kEpiThread0) {
#pragma unroll
          for (int hh = 0; hh < 4; ++hh)
            sm100::tma_reduce_add_3d(&tmDQ, dqs + hh * (C::kQT * 128), hh * 32, i * C::kQT, (int)zh);
          sm100::bulk_commit_group();
        }
      }
      sm100::mbar_wait_backoff(acc_full, item_c & 1);
      sm100::tc_fence_after();
      const int key = kt * kTile + (int)row;
      const bool key_valid = key < nk;
      const size_t off = kBSHD ? row_off(1, args.H, args.Nk, D, b, h, key) : (zh * args.Nk + key) * D;
#pragma unroll 1
      for (int which = 0; which < 2; ++which) {
        const uint32_t col0 = which == 0 ? C::kColDV : C::kColDK;
        const float sc = which == 0 ? 1.0f : alpha;
        uint4* dst = reinterpret_cast<uint4*>(reinterpret_cast<uint16_t*>(which == 0 ? args.dv : args.dk) + off);
#pragma unroll 1
        for (int hh = 0; hh < 4; ++hh) {
          float r[2][16];
          sm100::tmem_ld16(tmem + lane_addr + col0 + hh * 32, r[0]);
          sm100::tmem_ld16(tmem + lane_addr + col0 + hh * 32 + 16, r[1]);
          sm100::tmem_wait_ld_dep16(r[0]);
          sm100::tmem_wait_ld_dep16(r[1]);
          if (which == 1 && hh == 3) {
            sm100::tc_fence_before();
            __syncwarp();
            if (lane == 0) sm100::mbar_arrive(acc_empty);
          }
          if (key < args.Nk) {
#pragma unroll
            for (int c4 = 0; c4 < 2; ++c4)
#pragma unroll
              for (int e = 0; e < 16; e += 8) {
                uint4 w;
                w.x = key_valid ? sm100::pack2<kBf16>(sc * r[c4][e], sc * r[c4][e + 1]) : 0u;
                w.y = key_valid ? sm100::pack2<kBf16>(sc * r[c4][e + 2], sc * r[c4][e + 3]) : 0u;
                w.z = key_valid ? sm100::pack2<kBf16>(sc * r[c4][e + 4], sc * r[c4][e + 5]) : 0u;
                w.w = key_valid ? sm100::pack2<kBf16>(sc * r[c4][e + 6], sc * r[c4][e + 7]) : 0u;
                dst[hh * 4 + c4 * 2 + (e >> 3)] = w;
              }
          }
        }
      }
      ++item_c;
    }
  }

  if ((warp == C::kWarpFill || warp == C::kWarpAlloc)) {   // padded dK / dV rows no tile epilogue writes
    pad_fill_warp(args.dk, D * 2, args.B, args.H, args.Nk, args.seqlens_k, args.seqlens_q, args.Nq, kTile, lane, kBSHD ? 1 : 0, args.fill_pad, warp == C::kWarpFill ? 0 : 1, 2);
    pad_fill_warp(args.dv, D * 2, args.B, args.H, args.Nk, args.seqlens_k, args.seqlens_q, args.Nq, kTile, lane, kBSHD ? 1 : 0, args.fill_pad, warp == C::kWarpFill ? 0 : 1, 2);
    if (args.dq_pad)   // dq_finalize_kernel covers the rows below
      pad_fill_warp(args.dq_pad, D * 2, args.B, args.H, args.Nq, args.seqlens_q, args.seqlens_k, args.Nk, kTile, lane, kBSHD ? 1 : 0, args.fill_pad, warp == C::kWarpFill ? 0 : 1, 2);
  }

  if (kDQ && threadIdx.x == 32 * C::kWarpEpi) sm100::bulk_wait_group<0>();   // reduce-adds complete before exit
  sm100::tc_fence_before();
  __syncthreads();
  if (warp == C::kWarpAlloc) sm100::tmem_dealloc<C::kTmemCols>(tmem);
}

}  // namespace sigattn
