// fwd2.cuh -- forward kernel with two query tiles per CTA (Alg. 1).
//
// A work item is a PAIR of consecutive 128-query tiles (A = 2p, B = 2p + 1) of one (b, h); both
// tiles walk the same key tiles, so K_j / V_j are loaded once for the two.  Each query tile has
// its own S buffer (P aliased onto it) and its own O accumulator in TMEM, and its own warpgroup
// pair of sigma warps:
//   warps 0-7   pair A: sigma for tile A (warpgroup gp owns key columns [64 gp, +64), two chunks
//               of 32; thread = query row = TMEM lane); then tile A's O epilogue
//   warps 8-15  pair B: the same for tile B (idle when the sequence has an odd tile count)
//   warp 16     TMA: the Q pair, then K_j / V_j rings
//   warp 17     MMA: S_A(0), S_B(0); per key tile j: PV_A(j), S_A(j+1) as soon as P_A(j) is
//               ready, then PV_B(j), S_B(j+1).  The two tiles' chains are independent, so while
//               one pair evaluates sigma the tensor core works on the other tile's PV and S.
//   warp 18     TMEM allocator; warp 19 padded-row fill of O
// TMEM: S_A [0,128), S_B [128,256), O_A [256, 256+D), O_B [256+D, 256+2D).
// Compared with fwd.cuh (one query tile, the two pairs alternating key tiles through a 3-deep S
// ring), a pair's next S never waits for the other pair's P, which is what serialised sigma and
// the MMAs there.
#pragma once
#include <type_traits>
#include "fwd.cuh"

namespace sigattn {

template <int D>
struct Fwd2Cfg {
  static constexpr int kStages = (D == 64) ? 4 : 2;     // K / V ring
  static constexpr int kQBufs = (D == 64) ? 2 : 1;      // Q-pair buffers
  static constexpr int kSub = D / 64;
  static constexpr int kTileBytes = kTile * D * 2;
  static constexpr int kQOff = 0;                                   // Q[kQBufs][2 tiles]
  static constexpr int kKOff = kQOff + kQBufs * 2 * kTileBytes;     // K[kStages]
  static constexpr int kVOff = kKOff + kStages * kTileBytes;        // V[kStages]
  static constexpr int kBarOff = kVOff + kStages * kTileBytes;
  static constexpr int kNumBars = 2 * kQBufs + 4 * kStages + 2 + 2 + 2 + 2 + 2 + 2;
  // d = 64: P gets its own TMEM columns so a pair releases S_x(j) once it has READ it (mid-sigma)
  // and S_x(j+1) is computed while the pair still works on sigma(j); d = 128 has no room (P aliased).
  static constexpr bool kSepP = (D == 64);
  // d = 128: per sigma warp a 2 KB staging tile (32 rows x 32 columns of 16-bit O) through which
  // the epilogue turns row-per-lane stores into 64-byte row segments (8 rows per store instruction)
  static constexpr int kStgOff = (kBarOff + kNumBars * 8 + 16 + 127) / 128 * 128;
  static constexpr int kStgBytes = (D == 128) ? 16 * 2048 : 0;
  static constexpr int kSmemBytes = kStgOff + kStgBytes + 1024;
  static constexpr int kWarpTMA = 16, kWarpMMA = 17, kWarpAlloc = 18, kWarpFill = 19;
  static constexpr int kThreads = 32 * 20;
  static constexpr uint32_t kTmemCols = 512;
  static constexpr uint32_t kColP = 256;                            // kSepP: P_A, P_B (64 cols each)
  static constexpr uint32_t kColO = kSepP ? 384 : 256;              // O_A, then O_B at kColO + D
  static_assert(kColO + 2 * D <= kTmemCols, "TMEM budget");
  static_assert(kSmemBytes <= 227 * 1024, "shared memory budget");
};

template <int D, bool kBf16, bool kOutF32>
__global__ void __launch_bounds__(Fwd2Cfg<D>::kThreads, 1)
sigattn_fwd2_kernel(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmK,
                    const __grid_constant__ CUtensorMap tmV, const FwdArgs args) {
  using C = Fwd2Cfg<D>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + C::kBarOff);
  uint64_t* q_full = bars;                     // [kQBufs]
  uint64_t* q_empty = q_full + C::kQBufs;      // [kQBufs]
  uint64_t* k_full = q_empty + C::kQBufs;      // [kStages]
  uint64_t* v_full = k_full + C::kStages;
  uint64_t* k_empty = v_full + C::kStages;     // K slot free: S of both tiles done
  uint64_t* v_empty = k_empty + C::kStages;    // V slot free: PV of both tiles done
  uint64_t* s_full = v_empty + C::kStages;     // [2] per query tile X
  uint64_t* p_full = s_full + 2;               // [2]
  uint64_t* o_full = p_full + 2;               // [2]
  uint64_t* o_empty = o_full + 2;              // [2]
  uint64_t* s_free = o_empty + 2;              // [2] kSepP: pair x has read S_x(j)
  uint64_t* pv_done = s_free + 2;              // [2] kSepP: PV_x(j) has read P_x(j)
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
    for (int x = 0; x < 2; ++x) {
      sm100::mbar_init(&s_full[x], 1);
      sm100::mbar_init(&p_full[x], 8);     // the 8 warps of pair x
      sm100::mbar_init(&o_full[x], 1);
      sm100::mbar_init(&o_empty[x], 8);
      sm100::mbar_init(&s_free[x], 8);
      sm100::mbar_init(&pv_done[x], 1);
    }
    sm100::fence_barrier_init();
  }
  if (warp == C::kWarpTMA && lane == 0) {
    sm100::tma_prefetch_desc(&tmQ);
    sm100::tma_prefetch_desc(&tmK);
    sm100::tma_prefetch_desc(&tmV);
  }
  if (warp == C::kWarpAlloc) sm100::tmem_alloc<C::kTmemCols>(tmem_holder);
  sm100::tc_fence_before();
  __syncthreads();
  sm100::tc_fence_after();
  const uint32_t tmem = *tmem_holder;
  if (threadIdx.x == 0) sm100::trace_globaltime(args.trace, 4094);
  const int n_items = *args.n_items;
  // tiles of this item that hold a valid query: A always, B when 2p + 1 < ceil(n_q / 128)
  auto has_b = [&](int b, int pi) {
    const int nq = clampi(args.seqlens_q ? args.seqlens_q[b] : args.Nq, 0, args.Nq);
    return 2 * pi + 1 < (nq + kTile - 1) / kTile;
  };
  // work item (b, h, query-tile pair) over key tiles [kb, kb + nkt); piece >= 0: one key-range piece
  // of a split tail item (split_tail_block), whose fp32 partial O goes to the piece buffer
  struct Item2 {
    int b, h, pi, kb, nkt, piece;
  };
  auto decode = [](int4 it) { return Item2{it.x & 0xFFFF, it.y, it.z & 0xFFFF, it.z >> 16, it.w, (it.x >> 16) - 1}; };

  if (warp == C::kWarpTMA) {
    // ===================== TMA producer =====================
    const uint64_t pol_q = sm100::policy_evict_first();
    const uint64_t pol_kv = sm100::policy_evict_last();
    uint32_t kv_it = 0, c = 0;
    for (int it = first_item(); it < n_items; it = next_item(it)) {
      const Item2 item = decode(args.items[it]);
      const int b = item.b, h = item.h, pi = item.pi, nkt = item.nkt, kb = item.kb;
      if (nkt <= 0) continue;
      const int zh = b * args.H + h;
      const int ntq = has_b(b, pi) ? 2 : 1;
      const uint32_t qb = c % C::kQBufs;
      sm100::mbar_wait_backoff(&q_empty[qb], ((c / C::kQBufs) & 1) ^ 1);
      if (sm100::elect_one()) {
        sm100::mbar_arrive_expect_tx(&q_full[qb], ntq * C::kTileBytes);
        for (int x = 0; x < ntq; ++x)
#pragma unroll
          for (int s = 0; s < C::kSub; ++s)
            sm100::tma_load_bh(smem + C::kQOff + (qb * 2 + x) * C::kTileBytes + s * (kTile * 128), &tmQ, &q_full[qb],
                               s * 64, (2 * pi + x) * kTile, zh, pol_q, args.bshd ? args.H : 0);
      }
      __syncwarp();
      for (int j = 0; j < nkt; ++j, ++kv_it) {
        const uint32_t st = kv_it % C::kStages, ph = (kv_it / C::kStages) & 1;
        sm100::mbar_wait_backoff(&k_empty[st], ph ^ 1);
        if (sm100::elect_one()) {
          if (SIGATTN_DBG_FWD_NOTMA_KV && kv_it >= (uint32_t)C::kStages) {
            sm100::mbar_arrive(&k_full[st]);
          } else {
            sm100::mbar_arrive_expect_tx(&k_full[st], C::kTileBytes);
#pragma unroll
            for (int s = 0; s < C::kSub; ++s)
              sm100::tma_load_bh(smem + C::kKOff + st * C::kTileBytes + s * (kTile * 128), &tmK, &k_full[st], s * 64,
                                 (kb + j) * kTile, zh, pol_kv, args.bshd ? args.H : 0);
          }
        }
        __syncwarp();
        sm100::mbar_wait_backoff(&v_empty[st], ph ^ 1);
        if (sm100::elect_one()) {
          if (SIGATTN_DBG_FWD_NOTMA_KV && kv_it >= (uint32_t)C::kStages) {
            sm100::mbar_arrive(&v_full[st]);
          } else {
            sm100::mbar_arrive_expect_tx(&v_full[st], C::kTileBytes);
#pragma unroll
            for (int s = 0; s < C::kSub; ++s)
              sm100::tma_load_bh(smem + C::kVOff + st * C::kTileBytes + s * (kTile * 128), &tmV, &v_full[st], s * 64,
                                 (kb + j) * kTile, zh, pol_kv, args.bshd ? args.H : 0);
          }
        }
        __syncwarp();
      }
      ++c;
    }
  } else if (warp == C::kWarpMMA) {
    // ===================== MMA issuer =====================
    constexpr uint32_t idesc_s = sm100::make_idesc_f16(kBf16, 128, 128, false, false);
    constexpr uint32_t idesc_o = sm100::make_idesc_f16(kBf16, 128, D, false, true);
    const uint32_t q_base = sm100::smem_u32(smem + C::kQOff);
    const uint32_t k_base = sm100::smem_u32(smem + C::kKOff);
    const uint32_t v_base = sm100::smem_u32(smem + C::kVOff);
    uint32_t kv_it = 0, c = 0;
    uint32_t xs[2] = {0, 0};   // S / P phase counter per query-tile slot
    uint32_t xo[2] = {0, 0};   // O phase counter per slot
    for (int it = first_item(); it < n_items; it = next_item(it)) {
      const Item2 item = decode(args.items[it]);
      const int nkt = item.nkt;
      if (nkt <= 0) continue;
      const int ntq = has_b(item.b, item.pi) ? 2 : 1;
      if (args.counters && sm100::elect_one()) atomicAdd(args.counters, (unsigned long long)(ntq * nkt));
      __syncwarp();
      const uint32_t qb = c % C::kQBufs;
      if (lane == 0) sm100::trace_event(args.trace, c, 512);                // item c: Q wait start
      sm100::mbar_wait(&q_full[qb], (c / C::kQBufs) & 1);
      if (lane == 0) sm100::trace_event(args.trace, 512 + c, 1024);         // item c: Q ready
      // S_x(j) = Q_x K_j^T into slot x's buffer; the last S of key tile j releases K_j
      auto issue_s = [&](int x, int j) {
        const uint32_t kvi = kv_it + j, st = kvi % C::kStages;
        if (x == 0) sm100::mbar_wait(&k_full[st], (kvi / C::kStages) & 1);
        sm100::tc_fence_after();
        const uint32_t qa = q_base + (qb * 2 + x) * C::kTileBytes, ka = k_base + st * C::kTileBytes;
        if (sm100::elect_one()) {
#pragma unroll
          for (int kk = 0; kk < D / 16; ++kk) {
            const uint32_t off = (kk >> 2) * (kTile * 128) + (kk & 3) * 32;
            sm100::mma_ss(tmem + x * 128, sm100::sdesc_add(sm100::make_sdesc_sw128(qa, 16, 1024), off),
                          sm100::sdesc_add(sm100::make_sdesc_sw128(ka, 16, 1024), off), idesc_s, kk > 0);
          }
          sm100::mma_commit(&s_full[x]);
          if (x == ntq - 1) sm100::mma_commit(&k_empty[st]);
        }
        __syncwarp();
      };
      // O_x += P_x(j) V_j; the last PV of key tile j releases V_j
      auto issue_pv = [&](int x, int j) {
        const uint32_t kvi = kv_it + j, st = kvi % C::kStages;
        SIGATTN_FWD_MMA_WAIT(&p_full[x], xs[x] & 1);
        if (j == 0) sm100::mbar_wait(&o_empty[x], (xo[x] & 1) ^ 1);   // epilogue drained O_x
        if (x == 0) sm100::mbar_wait(&v_full[st], (kvi / C::kStages) & 1);
        sm100::tc_fence_after();
        const uint32_t va = v_base + st * C::kTileBytes;
        if (sm100::elect_one()) {
#pragma unroll
          for (int kk = 0; kk < kTile / 16; ++kk) {
            // P for keys [16kk, 16kk+16): warpgroup kk/4 packed its 64 keys at S cols [64 (kk/4), +32)
            const uint32_t a_col = C::kSepP ? C::kColP + x * 64 + (kk >> 2) * 32 + (kk & 3) * 8
                                            : x * 128 + (kk >> 2) * 64 + (kk & 3) * 8;
            sm100::mma_ts(tmem + C::kColO + x * D, tmem + a_col,
                          sm100::sdesc_add(sm100::make_sdesc_sw128(va, kTile * 128, 1024), kk * 2048), idesc_o,
                          (j > 0 || kk > 0) ? 1u : 0u);
          }
          if (x == ntq - 1) sm100::mma_commit(&v_empty[st]);
          if (C::kSepP) sm100::mma_commit(&pv_done[x]);
        }
        __syncwarp();
        ++xs[x];
      };
      // the Q pair is released once the item's LAST S MMAs complete (PV does not read Q), so the next
      // item's Q loads during the last key tiles' sigma and PV instead of after them
      auto release_q = [&]() {
        if (sm100::elect_one()) sm100::mma_commit(&q_empty[qb]);
        __syncwarp();
      };
      for (int x = 0; x < ntq; ++x) issue_s(x, 0);
      if (lane == 0) sm100::trace_event(args.trace, 1024 + c, 1536);        // item c: first S issued
      if (nkt == 1) release_q();
      if constexpr (C::kSepP) {
        // events arrive as s_free_A(j), s_free_B(j), p_full_A(j), p_full_B(j): issue in that order
        for (int j = 0; j < nkt; ++j) {
          if (j + 1 < nkt) {
            for (int x = 0; x < ntq; ++x) {
              sm100::mbar_wait(&s_free[x], xs[x] & 1);   // pair x has read S_x(j)
              issue_s(x, j + 1);
            }
            if (j + 2 == nkt) release_q();
          }
          for (int x = 0; x < ntq; ++x) issue_pv(x, j);
        }
      } else {
        for (int j = 0; j < nkt; ++j) {
          for (int x = 0; x < ntq; ++x) {
            issue_pv(x, j);                      // reads P_x(j) out of the S_x buffer ...
            if (j + 1 < nkt) issue_s(x, j + 1);  // ... which S_x(j+1) then overwrites (in-order)
          }
          if (j + 2 == nkt) release_q();
        }
      }
      if (sm100::elect_one()) {
        for (int x = 0; x < ntq; ++x) sm100::mma_commit(&o_full[x]);
      }
      __syncwarp();
      if (lane == 0) sm100::trace_event(args.trace, 1536 + c, 2048);        // item c: last PV issued
      for (int x = 0; x < ntq; ++x) ++xo[x];
      kv_it += nkt;
      ++c;
    }
  } else if (warp < C::kWarpTMA) {
    // ===================== sigma warps + epilogue, pair x = query tile slot =====================
    const uint32_t x = warp >> 3;
    const uint32_t gp = (warp >> 2) & 1;         // key columns [64 gp, +64) of the tile
    const uint32_t quarter = warp & 3;
    const uint32_t row = quarter * 32 + lane;
    const uint32_t lane_addr = (quarter * 32) << 16;
    bool spec = true;   // speculate while the last chunk took the speculated tier
    uint32_t xs = 0, xo = 0;
    for (int it = first_item(); it < n_items; it = next_item(it)) {
      const Item2 item = decode(args.items[it]);
      const int b = item.b, h = item.h, pi = item.pi, nkt = item.nkt, kb = item.kb;
      if (nkt <= 0) continue;
      if (x == 1 && !has_b(b, pi)) continue;     // odd tile count: no second tile in this item
      const int qt = 2 * pi + (int)x;
      const int nq = clampi(args.seqlens_q ? args.seqlens_q[b] : args.Nq, 0, args.Nq);
      const int nk = clampi(args.seqlens_k ? args.seqlens_k[b] : args.Nk, 0, args.Nk);
      const float bias = args.bias_per_seq ? args.bias_per_seq[b] : args.bias;
      const float a2 = args.scale * kLog2e;
      const float b2 = bias * kLog2e;
      const bool spec4 = bias <= kSpec4MaxBias;   // speculative sigma tier of this item
      const bool row_valid = qt * kTile + (int)row < nq;
      // the key loop, instantiated for the item's speculative sigma tier (one hot copy per item)
      auto key_loop = [&](auto tier_c) {
        constexpr int kT = decltype(tier_c)::value;
        for (int j = 0; j < nkt; ++j, ++xs) {
          SIGATTN_COMPUTE_WAIT(&s_full[x], xs & 1);
          sm100::tc_fence_after();
#pragma unroll
          for (int ch = 0; ch < 2; ++ch) {
            const uint32_t col = x * 128 + gp * 64 + ch * 32;
            const int nvalid = nk - ((kb + j) * kTile + (int)gp * 64 + ch * 32);
            float r[32];
            uint32_t pk[16];
            sm100::tmem_ld32_sync(tmem + lane_addr + col, r);
            if (C::kSepP && ch == 1) {   // all of this warp's S_x(j) columns are read: release the buffer
              sm100::tc_fence_before();
              __syncwarp();
              if (lane == 0) sm100::mbar_arrive(&s_free[x]);
            }
            if (SIGATTN_DBG_FWD_NOSIGMA) {   // timing experiments only: P = bits of S, no sigma work
#pragma unroll
              for (int e = 0; e < 16; ++e) pk[e] = __float_as_uint(r[2 * e]) ^ __float_as_uint(r[2 * e + 1]);
            } else if (C::kSepP) {   // S already released: no reload possible, vote-first tiers
              if (nvalid >= 32) sigmoid_row32<false, kBf16>(r, pk, a2, b2, row_valid, nvalid);
              else sigmoid_row32<true, kBf16>(r, pk, a2, b2, row_valid, nvalid);
            } else {
              if (nvalid >= 32) sigmoid_chunk32<false, kBf16, kT>(tmem + lane_addr + col, r, pk, a2, b2, row_valid, nvalid, spec);
              else sigmoid_chunk32<true, kBf16, kT>(tmem + lane_addr + col, r, pk, a2, b2, row_valid, nvalid, spec);
            }
            if (C::kSepP) {
              if (ch == 0) {   // PV_x(j-1) has read the previous P_x
                sm100::mbar_wait(&pv_done[x], (xs & 1) ^ 1);
                sm100::tc_fence_after();
              }
              sm100::tmem_st16(tmem + lane_addr + C::kColP + x * 64 + gp * 32 + ch * 16, pk);
            } else {
              sm100::tmem_st16(tmem + lane_addr + x * 128 + gp * 64 + ch * 16, pk);
            }
          }
          sm100::tmem_wait_st();
          sm100::tc_fence_before();
          __syncwarp();
          if (lane == 0) sm100::mbar_arrive(&p_full[x]);
        }
      };
      if (spec4) key_loop(std::integral_constant<int, 4>{});
      else key_loop(std::integral_constant<int, 2>{});
      // ---- epilogue: O_x rows, columns [gp D/2, +D/2) in 32-column pieces
      if (lane == 0 && warp == 0) sm100::trace_event(args.trace, 3584 + 3 * xo, 4092);
      sm100::mbar_wait(&o_full[x], xo & 1);
      if (lane == 0 && warp == 0) sm100::trace_event(args.trace, 3584 + 3 * xo + 1, 4092);
      sm100::tc_fence_after();
      const int qrow = qt * kTile + (int)row;
      const bool valid = qrow < nq;
      const size_t rowoff = row_off(args.bshd, args.H, args.Nq, D, b, h, qrow);
#pragma unroll
      for (int pc = 0; pc < D / 64; ++pc) {
        const int c0 = (int)gp * (D / 2) + pc * 32;
        uint32_t ov[32];
        sm100::tmem_ld32_sync(tmem + lane_addr + C::kColO + x * D + c0, ov);
        if (pc == D / 64 - 1) {
          sm100::tc_fence_before();
          __syncwarp();
          if (lane == 0) sm100::mbar_arrive(&o_empty[x]);
        }
        if (kOutF32 && args.peer_o) {
          if (valid) peer_red_row32(args, D, b, h, qrow, c0, ov);
        } else if (item.piece >= 0) {   // a piece of a split tail item: fp32 partial into its slot
          float4* dst = reinterpret_cast<float4*>(args.split_acc + ((size_t)(item.piece * 2 + x) * kTile + row) * D + c0);
#pragma unroll
          for (int e = 0; e < 32; e += 4)
            dst[e >> 2] = valid ? make_float4(__uint_as_float(ov[e]), __uint_as_float(ov[e + 1]),
                                              __uint_as_float(ov[e + 2]), __uint_as_float(ov[e + 3]))
                                : make_float4(0.f, 0.f, 0.f, 0.f);
        } else if (C::kStgBytes > 0 && !kOutF32) {
          // stage the warp's 32 rows x 32 columns (64 bytes per row; 16-byte chunk c of row r at slot
          // c ^ ((r >> 1) & 3): conflict-free both ways), then store 8 rows x 64 bytes per instruction
          const uint32_t stg = sm100::smem_u32(smem + C::kStgOff + warp * 2048);
#pragma unroll
          for (int c = 0; c < 4; ++c) {
            const int e = 8 * c;
            sm100::st_shared_v4(stg + lane * 64 + ((c ^ ((lane >> 1) & 3)) * 16),
                                sm100::pack2<kBf16>(__uint_as_float(ov[e + 0]), __uint_as_float(ov[e + 1])),
                                sm100::pack2<kBf16>(__uint_as_float(ov[e + 2]), __uint_as_float(ov[e + 3])),
                                sm100::pack2<kBf16>(__uint_as_float(ov[e + 4]), __uint_as_float(ov[e + 5])),
                                sm100::pack2<kBf16>(__uint_as_float(ov[e + 6]), __uint_as_float(ov[e + 7])));
          }
          __syncwarp();
#pragma unroll
          for (int k = 0; k < 4; ++k) {
            const int rr = 8 * k + (int)(lane >> 2), cc = (int)(lane & 3);
            const uint4 w = sm100::ld_shared_v4(stg + rr * 64 + ((cc ^ ((rr >> 1) & 3)) * 16));
            const int grow = qt * kTile + (int)quarter * 32 + rr;
            if (grow < args.Nq && !SIGATTN_DBG_EPI_NOSTORE) {
              const uint4 z = grow < nq ? w : make_uint4(0u, 0u, 0u, 0u);
              *reinterpret_cast<uint4*>(reinterpret_cast<uint16_t*>(args.o) +
                                        row_off(args.bshd, args.H, args.Nq, D, b, h, grow) + c0 + cc * 8) = z;
            }
          }
          __syncwarp();   // the next piece overwrites the staging tile
        } else if (qrow < args.Nq && !SIGATTN_DBG_EPI_NOSTORE) {
          if constexpr (kOutF32) {
            float4* dst = reinterpret_cast<float4*>(reinterpret_cast<float*>(args.o) + rowoff + c0);
#pragma unroll
            for (int e = 0; e < 32; e += 4)
              dst[e >> 2] = valid ? make_float4(__uint_as_float(ov[e]), __uint_as_float(ov[e + 1]),
                                                __uint_as_float(ov[e + 2]), __uint_as_float(ov[e + 3]))
                                  : make_float4(0.f, 0.f, 0.f, 0.f);
          } else {
            uint4* dst = reinterpret_cast<uint4*>(reinterpret_cast<uint16_t*>(args.o) + rowoff + c0);
#pragma unroll
            for (int e = 0; e < 32; e += 8) {
              uint4 w;
              w.x = valid ? sm100::pack2<kBf16>(__uint_as_float(ov[e + 0]), __uint_as_float(ov[e + 1])) : 0u;
              w.y = valid ? sm100::pack2<kBf16>(__uint_as_float(ov[e + 2]), __uint_as_float(ov[e + 3])) : 0u;
              w.z = valid ? sm100::pack2<kBf16>(__uint_as_float(ov[e + 4]), __uint_as_float(ov[e + 5])) : 0u;
              w.w = valid ? sm100::pack2<kBf16>(__uint_as_float(ov[e + 6]), __uint_as_float(ov[e + 7])) : 0u;
              dst[e >> 3] = w;
            }
          }
        }
      }
      if (lane == 0 && warp == 0) sm100::trace_event(args.trace, 3584 + 3 * xo + 2, 4092);
      ++xo;
    }
  }

  if (!SIGATTN_DBG_NOFILL && (warp == C::kWarpFill || warp == C::kWarpAlloc) && args.o)   // padded O rows beyond the last valid tile
    pad_fill_warp(args.o, D * (kOutF32 ? 4 : 2), args.B, args.H, args.Nq, args.seqlens_q, args.seqlens_k, args.Nk,
                  kTile, lane, args.bshd, args.fill_pad, warp == C::kWarpFill ? 0 : 1, 2);

  if (kOutF32 && args.peer_o) sm100::fence_sys();   // this CTA's peer reductions before kernel completion
  if (lane == 0) sm100::trace_event(args.trace, 4064 + (int)warp, 4092);   // per-warp end (trace builds)
  sm100::tc_fence_before();
  __syncthreads();
  if (threadIdx.x == 0) sm100::trace_globaltime(args.trace, 4095);
  if (warp == C::kWarpAlloc) sm100::tmem_dealloc<C::kTmemCols>(tmem);
}

}  // namespace sigattn
