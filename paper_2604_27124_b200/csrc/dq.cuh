// dq.cuh -- the query-tile-owned dQ pass of the deterministic backward (Alg. 2).
//
// For one 128-query tile of one (b, h), loop over the valid key tiles in order:
//   S = Q K_j^T,  dP = dO V_j^T          (recomputed)
//   dS = P (1 - P) dP,  P = mask * sigma(alpha S + b)
//   dQ += dS K_j
// and write dQ = rn(alpha dQ).  The key tiles are summed in a fixed order in one TMEM
// accumulator, so dQ is bitwise reproducible (no atomics).  Together with the backward kernel in its
// no-dQ mode (Alg. 3: dK, dV) this is SIGATTN_F_BWD_DETERMINISTIC; the default backward fuses both
// passes (10d instead of 14d FLOP per pair) but reduces dQ across key tiles in L2.
//
// Structure (640 threads, persistent, LPT work list of (b, h, q-tile) items as the forward):
//   warps 0-15  two warpgroup pairs take alternate 64-key half tiles u (pair = u % 2); within a pair
//               warpgroup gp owns keys [32 gp, +32) of the half (two 16-column chunks), thread = query
//               row = TMEM lane.  They turn S, dP into packed dS written over the S columns they read.
//   warp 16     TMA: Q + dO per item (double-buffered at d = 64), K and V rings
//   warp 17     MMA: S_u, dP_u (SS, M=128 N=64) into a ring of 3 half-tile buffers, issued two halves
//               ahead; dQ += dS_u K (TS, A = packed dS in TMEM, B = K rows MN-major)
//   warp 18     TMEM allocator; warp 19 padded-row fill of dQ
// TMEM: buffer b at [128 b, +128): S_u in [0, 64), dP_u in [64, 128); dQ at [384, 384 + D).
#pragma once
#include "bwd.cuh"

namespace sigattn {

struct DqArgs {
  const int4* items;      // {b, h, q tile, key tiles}
  const int* n_items;
  const int32_t* seqlens_q;
  const int32_t* seqlens_k;
  const float* bias_per_seq;
  float bias;
  float scale;
  int B, H, Nq, Nk;
  void* dq;               // bf16/fp16 [B,H,Nq,D], or fp32 when kOutF32 (context-parallel partial)
  int bshd;               // 1: tensors are [B, N, H, d], else [B, H, N, d]
  unsigned long long* counters;   // skip accounting (sigattn_set_debug_counters) or nullptr
  int fill_pad;           // as BwdArgs::fill_pad
};

template <int D>
struct DqCfg {
  static constexpr int kStages = (D == 64) ? 4 : 2;   // K / V ring, one key tile per slot
  static constexpr int kQBufs = (D == 64) ? 2 : 1;    // Q + dO tiles per work item
  static constexpr int kSub = D / 64;                 // 64-column swizzle atoms per row
  static constexpr int kTileBytes = kTile * D * 2;
  static constexpr int kQOff = 0;                               // Q[kQBufs]
  static constexpr int kDOOff = kQOff + kQBufs * kTileBytes;    // dO[kQBufs]
  static constexpr int kKOff = kDOOff + kQBufs * kTileBytes;    // K[kStages]
  static constexpr int kVOff = kKOff + kStages * kTileBytes;    // V[kStages]
  static constexpr int kBarOff = kVOff + kStages * kTileBytes;
  static constexpr int kSBuf = 3;                               // S|dP half-tile buffers
  static constexpr int kNumBars = 2 * kQBufs + 4 * kStages + 2 * kSBuf + 2;
  static constexpr int kSmemBytes = kBarOff + kNumBars * 8 + 16 + 1024;
  static constexpr int kNumWG = 4;
  static constexpr int kWarpTMA = 4 * kNumWG, kWarpMMA = kWarpTMA + 1, kWarpAlloc = kWarpTMA + 2,
                       kWarpFill = kWarpTMA + 3;
  static constexpr int kThreads = 32 * (4 * kNumWG + 4);
  static constexpr uint32_t kTmemCols = 512;
  static constexpr uint32_t kColDQ = 128 * kSBuf;
  static_assert(kColDQ + D <= kTmemCols, "TMEM budget");
  static_assert(kSmemBytes <= 227 * 1024, "shared memory budget");
};

template <int D, bool kBf16, bool kOutF32, bool kBSHD = false>
__global__ void __launch_bounds__(DqCfg<D>::kThreads, 1)
sigattn_dq_kernel(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmK,
                  const __grid_constant__ CUtensorMap tmV, const __grid_constant__ CUtensorMap tmDO,
                  const DqArgs args) {
  using C = DqCfg<D>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + C::kBarOff);
  uint64_t* q_full = bars;                          // [kQBufs] Q + dO of the item landed
  uint64_t* q_empty = q_full + C::kQBufs;           // [kQBufs]
  uint64_t* k_full = q_empty + C::kQBufs;           // [kStages]
  uint64_t* v_full = k_full + C::kStages;
  uint64_t* k_empty = v_full + C::kStages;          // K slot free: last dQ MMA of the tile done
  uint64_t* v_empty = k_empty + C::kStages;         // V slot free: last dP MMA of the tile done
  uint64_t* s_full = v_empty + C::kStages;          // [kSBuf] S_u, dP_u in TMEM
  uint64_t* p_full = s_full + C::kSBuf;             // [kSBuf] dS_u packed in TMEM
  uint64_t* o_full = p_full + C::kSBuf;             // dQ of the item complete
  uint64_t* o_empty = o_full + 1;                   // epilogue read dQ
  uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(bars + C::kNumBars);

  const uint32_t warp = sm100::warp_id();
  const uint32_t lane = sm100::lane_id();

  if (threadIdx.x == 0) {
    for (int i = 0; i < C::kQBufs; ++i) {
      sm100::mbar_init(&q_full[i], 1);
      sm100::mbar_init(&q_empty[i], 1);
    }
    for (int i = 0; i < C::kStages; ++i) {
      sm100::mbar_init(&k_full[i], 1);
      sm100::mbar_init(&v_full[i], 1);
      sm100::mbar_init(&k_empty[i], 1);
      sm100::mbar_init(&v_empty[i], 1);
    }
    for (int i = 0; i < C::kSBuf; ++i) {
      sm100::mbar_init(&s_full[i], 1);
      sm100::mbar_init(&p_full[i], 2 * C::kNumWG);   // the 8 warps of the pair owning the half tile
    }
    sm100::mbar_init(o_full, 1);
    sm100::mbar_init(o_empty, 4 * C::kNumWG);
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

  if (warp == C::kWarpTMA) {
    // ===================== TMA producer =====================
    const uint64_t pol_q = sm100::policy_evict_first();
    const uint64_t pol_kv = sm100::policy_evict_last();
    uint32_t kv_it = 0, c = 0;
    for (int it = first_item(); it < n_items; it = next_item(it)) {
      const int4 item = args.items[it];
      const int b = item.x, h = item.y, qt = item.z, nkt = item.w;
      if (nkt <= 0) continue;
      const int zh = b * args.H + h;
      const uint32_t qb = c % C::kQBufs;
      sm100::mbar_wait_backoff(&q_empty[qb], ((c / C::kQBufs) & 1) ^ 1);
      if (sm100::elect_one()) {
        sm100::mbar_arrive_expect_tx(&q_full[qb], 2 * C::kTileBytes);
#pragma unroll
        for (int s = 0; s < C::kSub; ++s) {
          sm100::tma_load_bh(smem + C::kQOff + qb * C::kTileBytes + s * (kTile * 128), &tmQ, &q_full[qb], s * 64,
                             qt * kTile, zh, pol_q, kBSHD ? args.H : 0);
          sm100::tma_load_bh(smem + C::kDOOff + qb * C::kTileBytes + s * (kTile * 128), &tmDO, &q_full[qb],
                             s * 64, qt * kTile, zh, pol_q, kBSHD ? args.H : 0);
        }
      }
      __syncwarp();
      for (int j = 0; j < nkt; ++j, ++kv_it) {
        const uint32_t st = kv_it % C::kStages, ph = (kv_it / C::kStages) & 1;
        sm100::mbar_wait_backoff(&k_empty[st], ph ^ 1);
        if (sm100::elect_one()) {
          sm100::mbar_arrive_expect_tx(&k_full[st], C::kTileBytes);
#pragma unroll
          for (int s = 0; s < C::kSub; ++s)
            sm100::tma_load_bh(smem + C::kKOff + st * C::kTileBytes + s * (kTile * 128), &tmK, &k_full[st], s * 64,
                               j * kTile, zh, pol_kv, kBSHD ? args.H : 0);
        }
        __syncwarp();
        sm100::mbar_wait_backoff(&v_empty[st], ph ^ 1);
        if (sm100::elect_one()) {
          sm100::mbar_arrive_expect_tx(&v_full[st], C::kTileBytes);
#pragma unroll
          for (int s = 0; s < C::kSub; ++s)
            sm100::tma_load_bh(smem + C::kVOff + st * C::kTileBytes + s * (kTile * 128), &tmV, &v_full[st], s * 64,
                               j * kTile, zh, pol_kv, kBSHD ? args.H : 0);
        }
        __syncwarp();
      }
      ++c;
    }
  } else if (warp == C::kWarpMMA) {
    // ===================== MMA issuer =====================
    constexpr uint32_t idesc_s = sm100::make_idesc_f16(kBf16, 128, 64, false, false);   // S_u, dP_u
    constexpr uint32_t idesc_dq = sm100::make_idesc_f16(kBf16, 128, D, false, true);    // dQ += dS K
    const uint32_t q_base = sm100::smem_u32(smem + C::kQOff);
    const uint32_t do_base = sm100::smem_u32(smem + C::kDOOff);
    const uint32_t k_base = sm100::smem_u32(smem + C::kKOff);
    const uint32_t v_base = sm100::smem_u32(smem + C::kVOff);
    uint32_t kv_it = 0, u_it = 0, c = 0;
    for (int it = first_item(); it < n_items; it = next_item(it)) {
      const int nkt = args.items[it].w;
      if (nkt <= 0) continue;
      if (args.counters && sm100::elect_one()) atomicAdd(args.counters + 2, (unsigned long long)nkt);
      __syncwarp();
      const uint32_t qb = c % C::kQBufs;
      sm100::mbar_wait(&q_full[qb], (c / C::kQBufs) & 1);
      const uint32_t qa = q_base + qb * C::kTileBytes, da = do_base + qb * C::kTileBytes;
      const int U = 2 * nkt;   // 64-key half tiles of this item
      // S_u = Q K_h^T and dP_u = dO V_h^T for half tile ul of this item (u = u_it + ul globally)
      auto issue_sd = [&](int ul) {
        const uint32_t u = u_it + ul, kvi = kv_it + (ul >> 1), st = kvi % C::kStages, hh = ul & 1;
        if (hh == 0) {
          sm100::mbar_wait(&k_full[st], (kvi / C::kStages) & 1);
          sm100::mbar_wait(&v_full[st], (kvi / C::kStages) & 1);
        }
        sm100::tc_fence_after();
        const uint32_t ka = k_base + st * C::kTileBytes + hh * 8192, va = v_base + st * C::kTileBytes + hh * 8192;
        const uint32_t d_s = tmem + (u % C::kSBuf) * 128;
        if (sm100::elect_one()) {
#pragma unroll
          for (int kk = 0; kk < D / 16; ++kk) {
            const uint32_t off = (kk >> 2) * (kTile * 128) + (kk & 3) * 32;
            sm100::mma_ss(d_s, sm100::sdesc_add(sm100::make_sdesc_sw128(qa, 16, 1024), off), sm100::sdesc_add(sm100::make_sdesc_sw128(ka, 16, 1024), off),
                          idesc_s, kk > 0);
          }
#pragma unroll
          for (int kk = 0; kk < D / 16; ++kk) {
            const uint32_t off = (kk >> 2) * (kTile * 128) + (kk & 3) * 32;
            sm100::mma_ss(d_s + 64, sm100::sdesc_add(sm100::make_sdesc_sw128(da, 16, 1024), off),
                          sm100::sdesc_add(sm100::make_sdesc_sw128(va, 16, 1024), off), idesc_s, kk > 0);
          }
          sm100::mma_commit(&s_full[u % C::kSBuf]);
          if (hh == 1) sm100::mma_commit(&v_empty[st]);   // last reader of V_j
        }
        __syncwarp();
      };
      // S|dP run two half tiles ahead: buffer (u+2) % 3 held dS(u-1), consumed by the dQ MMA of
      // u-1 issued earlier (tcgen05 ops of one thread execute in order).
      issue_sd(0);
      issue_sd(1);
      for (int ul = 0; ul < U; ++ul) {
        if (ul + 2 < U) issue_sd(ul + 2);
        const uint32_t u = u_it + ul, kvi = kv_it + (ul >> 1), st = kvi % C::kStages, hh = ul & 1;
        sm100::mbar_wait_backoff(&p_full[u % C::kSBuf], (u / C::kSBuf) & 1);
        if (ul == 0) sm100::mbar_wait(o_empty, (c & 1) ^ 1);   // epilogue read the previous dQ
        sm100::tc_fence_after();
        const uint32_t ka = k_base + st * C::kTileBytes + hh * 8192;
        const uint32_t ds_col = (u % C::kSBuf) * 128;
        if (sm100::elect_one()) {
#pragma unroll
          for (int kk = 0; kk < 4; ++kk) {
            // keys [16 kk, +16) of the half: warpgroup kk/2 packed its 32 keys at columns [32 (kk/2), +16)
            const uint32_t a_col = ds_col + (kk >> 1) * 32 + (kk & 1) * 8;
            sm100::mma_ts(tmem + C::kColDQ, tmem + a_col, sm100::sdesc_add(sm100::make_sdesc_sw128(ka, kTile * 128, 1024), kk * 2048),
                          idesc_dq, (ul > 0 || kk > 0) ? 1u : 0u);
          }
          if (hh == 1) sm100::mma_commit(&k_empty[st]);   // last reader of K_j
        }
        __syncwarp();
      }
      if (sm100::elect_one()) {
        sm100::mma_commit(&q_empty[qb]);
        sm100::mma_commit(o_full);
      }
      __syncwarp();
      kv_it += nkt;
      u_it += U;
      ++c;
    }
  } else if (warp < C::kWarpTMA) {
    // ===================== dS warps + epilogue =====================
    const uint32_t g = warp >> 2;
    const uint32_t pair = warp >> 3;
    const uint32_t gp = g & 1;
    const uint32_t quarter = warp & 3;
    const uint32_t row = quarter * 32 + lane;
    const uint32_t lane_addr = (quarter * 32) << 16;
    uint32_t u_it = 0, c = 0;
    for (int it = first_item(); it < n_items; it = next_item(it)) {
      const int4 item = args.items[it];
      const int b = item.x, h = item.y, qt = item.z, nkt = item.w;
      if (nkt <= 0) continue;
      const int nq = clampi(args.seqlens_q ? args.seqlens_q[b] : args.Nq, 0, args.Nq);
      const int nk = clampi(args.seqlens_k ? args.seqlens_k[b] : args.Nk, 0, args.Nk);
      const float bias = args.bias_per_seq ? args.bias_per_seq[b] : args.bias;
      const float a2 = args.scale * kLog2e;
      const float b2 = bias * kLog2e;
      const bool row_valid = qt * kTile + (int)row < nq;
      const bool warp_rows_valid = __all_sync(0xffffffffu, row_valid);
      bool spec = true;   // speculate tier 4 while the last chunk took it
      const int U = 2 * nkt;
      for (int ul = 0; ul < U; ++ul) {
        const uint32_t u = u_it + ul;
        if ((u & 1) != pair) continue;   // the other pair takes this half tile
        sm100::mbar_wait(&s_full[u % C::kSBuf], (u / C::kSBuf) & 1);
        sm100::tc_fence_after();
        const uint32_t sb = (u % C::kSBuf) * 128;
#pragma unroll
        for (int ch = 0; ch < 2; ++ch) {
          const uint32_t s_col = sb + gp * 32 + ch * 16, dp_col = sb + 64 + gp * 32 + ch * 16;
          const int ncol = nk - ((ul >> 1) * kTile + (ul & 1) * 64 + (int)gp * 32 + ch * 16);   // valid keys here
          float s[16], dp[16];
          sm100::tmem_ld16(tmem + lane_addr + s_col, s);
          sm100::tmem_ld16(tmem + lane_addr + dp_col, dp);
          sm100::tmem_wait_ld_dep16(s);
          sm100::tmem_wait_ld_dep16(dp);
          uint32_t pp[8], dd[8];
          if (warp_rows_valid && ncol >= 16) bwd_row16<false, kBf16>(s, dp, pp, dd, a2, b2, true, 16, tmem + lane_addr + s_col, spec);
          else bwd_row16<true, kBf16>(s, dp, pp, dd, a2, b2, row_valid, row_valid ? ncol : 0, tmem + lane_addr + s_col, spec);
          // packed dS over this warpgroup's own, already-read S columns: [32 gp + 8 ch, +8)
          sm100::tmem_st8(tmem + lane_addr + sb + gp * 32 + ch * 8, dd);
        }
        sm100::tmem_wait_st();
        sm100::tc_fence_before();
        __syncwarp();
        if (lane == 0) sm100::mbar_arrive(&p_full[u % C::kSBuf]);
      }
      u_it += U;
      // ---- epilogue: dQ = rn(alpha dQ) for rows of this q tile, columns [g D/4, +D/4)
      sm100::mbar_wait(o_full, c & 1);
      sm100::tc_fence_after();
      constexpr int kPart = D / C::kNumWG;
      uint32_t ov[kPart];
      if constexpr (kPart == 32) sm100::tmem_ld32_sync(tmem + lane_addr + C::kColDQ + g * kPart, ov);
      else sm100::tmem_ld16_sync(tmem + lane_addr + C::kColDQ + g * kPart, ov);
      sm100::tc_fence_before();
      __syncwarp();
      if (lane == 0) sm100::mbar_arrive(o_empty);
      const int qrow = qt * kTile + (int)row;
      if (qrow < args.Nq) {
        const bool valid = qrow < nq;
        const float alpha = args.scale;
        const size_t off = row_off(kBSHD ? 1 : 0, args.H, args.Nq, D, b, h, qrow) + g * kPart;
        if constexpr (kOutF32) {
          float4* dst = reinterpret_cast<float4*>(reinterpret_cast<float*>(args.dq) + off);
#pragma unroll
          for (int e = 0; e < kPart; e += 4)
            dst[e >> 2] = valid ? make_float4(alpha * __uint_as_float(ov[e]), alpha * __uint_as_float(ov[e + 1]),
                                              alpha * __uint_as_float(ov[e + 2]), alpha * __uint_as_float(ov[e + 3]))
                                : make_float4(0.f, 0.f, 0.f, 0.f);
        } else {
          uint4* dst = reinterpret_cast<uint4*>(reinterpret_cast<uint16_t*>(args.dq) + off);
#pragma unroll
          for (int e = 0; e < kPart; e += 8) {
            uint4 w;
            w.x = valid ? sm100::pack2<kBf16>(alpha * __uint_as_float(ov[e]), alpha * __uint_as_float(ov[e + 1])) : 0u;
            w.y = valid ? sm100::pack2<kBf16>(alpha * __uint_as_float(ov[e + 2]), alpha * __uint_as_float(ov[e + 3])) : 0u;
            w.z = valid ? sm100::pack2<kBf16>(alpha * __uint_as_float(ov[e + 4]), alpha * __uint_as_float(ov[e + 5])) : 0u;
            w.w = valid ? sm100::pack2<kBf16>(alpha * __uint_as_float(ov[e + 6]), alpha * __uint_as_float(ov[e + 7])) : 0u;
            dst[e >> 3] = w;
          }
        }
      }
      ++c;
    }
  }

  if (!SIGATTN_DBG_NOFILL && (warp == C::kWarpFill || warp == C::kWarpAlloc))   // padded dQ rows beyond the last valid tile
    pad_fill_warp(args.dq, D * (kOutF32 ? 4 : 2), args.B, args.H, args.Nq, args.seqlens_q, args.seqlens_k, args.Nk,
                  kTile, lane, kBSHD ? 1 : 0, args.fill_pad, warp == C::kWarpFill ? 0 : 1, 2);

  sm100::tc_fence_before();
  __syncthreads();
  if (warp == C::kWarpAlloc) sm100::tmem_dealloc<C::kTmemCols>(tmem);
}

}  // namespace sigattn
