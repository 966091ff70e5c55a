// fwd.cuh -- sm_100a forward kernel of padding-aware sigmoid attention (Alg. 1).
//
//   O[z, M, h, :] = sum over key tiles N < n_k[z] of  sigma(alpha Q_M K_N^T + b_z) masked  . V_N
//
// One CTA per SM (persistent), warp-specialised:
//   warps 0-15  four sigmoid warpgroups in two pairs that take alternate key tiles (ping-pong: one
//               pair computes while the other synchronises); within a pair warpgroup g owns key
//               columns [64g, 64g+64): tcgen05.ld S -> x = alpha s + b -> sigma -> key mask -> bf16
//               -> tcgen05.st P (aliased onto the first half of its own S columns).  The pair
//               that evaluated an item's last key tile runs its epilogue, half of the O columns
//               per warpgroup (padded query rows written as exact 0), while the other
//               pair already evaluates the next item's first tile.
//   warp 16     TMA producer: Q tile (double-buffered) and a K/V ring of kStages tiles
//   warp 17     MMA issuer (one elected thread): S = Q K^T (SS, both K-major) -> TMEM S[3] ring
//                                                O += P V  (TS, P from TMEM, V MN-major) -> TMEM O[2]
//               one stream of key tiles across items: S runs two tiles ahead of PV, also over
//               item boundaries, and O is double-buffered (D = 64), so nothing drains per q tile
//   warp 18     TMEM allocator
// Work items (b, h, q-tile) come from a device work list sorted longest-first (LPT), built
// by sched.cuh from the device seqlens, so fully padded query tiles are never visited
// and the key loop stops at ceil(n_k / 128) tiles.
#pragma once
#include <type_traits>
#include "sched.cuh"
#include "sigmoid.cuh"
#include "sm100.cuh"

#ifndef SIGATTN_FWD_SPEC
#define SIGATTN_FWD_SPEC 1  // tier-4 sigma evaluated before the warp vote (sigma_row_spec4)
#endif

namespace sigattn {

constexpr int kTile = 128;           // B_M = B_N = 128 (UMMA M = 128, one TMEM lane per row)
constexpr float kLog2e = 1.4426950408889634f;

struct FwdArgs {
  const int4* items;      // {b, h, tile, cost}
  const int* n_items;
  const int32_t* seqlens_q;
  const int32_t* seqlens_k;
  const float* bias_per_seq;
  float bias;
  float scale;
  int B, H, Nq, Nk;
  void* o;                // bf16/fp16 [B,H,Nq,D] or fp32 partial
  int fill_pad;           // zero the O rows no tile epilogue writes (pad_fill_warp)
  long long* trace;       // SIGATTN_TRACE builds: [grid][4096] clock64 event slots
  int bshd;               // 1: tensors are [B, N, H, d], else [B, H, N, d]
  unsigned long long* counters;   // skip accounting (sigattn_set_debug_counters) or nullptr
  // key-split context parallelism with the reduction fused into the epilogue (sigattn_fwd_cp):
  // peer_o[g] is rank g's fp32 accumulator [B, H, peer_rows, D] (peer_rows = Nq / world); the
  // partial O row of query q is reduce-added into peer_o[q / peer_rows] at row q % peer_rows
  float* const* peer_o;
  int peer_rows;
  // two-tile forward (fwd2.cuh) with a tail split (split_tail_block): fp32 piece buffer
  // [pieces][2 tiles][128][D], or nullptr when the work list has no split items
  float* split_acc;
};

// fp32 partial O row -> the owning rank's accumulator (context parallelism, A4: P:121).  32 values
// of row qrow, columns [c0, c0 + 32).
__device__ __forceinline__ void peer_red_row32(const FwdArgs& args, int D, int b, int h, int qrow, int c0,
                                               const uint32_t (&v)[32]) {
  const int owner = qrow / args.peer_rows, lr = qrow - owner * args.peer_rows;
  float* dst = args.peer_o[owner] + ((size_t)(b * args.H + h) * args.peer_rows + lr) * D + c0;
#pragma unroll
  for (int e = 0; e < 32; e += 4)
    sm100::red_add_v4_sys(dst + e, __uint_as_float(v[e]), __uint_as_float(v[e + 1]), __uint_as_float(v[e + 2]),
                          __uint_as_float(v[e + 3]));
}

template <int D>
struct FwdCfg {
#ifndef SIGATTN_FWD_STAGES
#define SIGATTN_FWD_STAGES 4
#endif
  static constexpr int kStages = (D == 64) ? SIGATTN_FWD_STAGES : 2;
  static constexpr int kSub = D / 64;                       // 64-column (128 B) swizzle atoms per row
  static constexpr int kTileBytes = kTile * D * 2;          // one 128-row tile of Q, K or V
  static constexpr int kQOff = 0;                           // Q[2]
  static constexpr int kKOff = kQOff + 2 * kTileBytes;      // K[kStages]
  static constexpr int kVOff = kKOff + kStages * kTileBytes;
  static constexpr int kBarOff = kVOff + kStages * kTileBytes;
  // O accumulators: two when TMEM has room (D = 64), so the epilogue of one item overlaps the
  // first PV of the next
  static constexpr int kOBufs = (128 * 3 + 2 * D <= 512) ? 2 : 1;
  static constexpr int kNumBars = 2 + 2 + 4 * kStages + 3 + 3 + 2 * kOBufs;
  static constexpr int kSmemBytes = kBarOff + kNumBars * 8 + 16 + 1024;  // + alignment slack
  static constexpr int kNumWG = 4;                          // sigmoid warpgroups: warps [0, 4 kNumWG)
  // Single-thread roles sit in the HIGHEST warp ids: the warp scheduler favours high warp ids, so
  // the MMA / TMA issuers are never starved by the sigmoid warps sharing their sub-partition.
  static constexpr int kWarpTMA = 4 * kNumWG, kWarpMMA = kWarpTMA + 1, kWarpAlloc = kWarpTMA + 2,
                       kWarpFill = kWarpTMA + 3;
  static constexpr int kThreads = 32 * (4 * kNumWG + 4);
  static constexpr uint32_t kTmemCols = 512;
  // TMEM columns
  // S ring of kSBuf 128-column fp32 buffers (P aliased inside each), then O.
  static constexpr uint32_t kSBuf = 3;
  static constexpr uint32_t kColO = 128 * kSBuf;
  static_assert(kColO + kOBufs * D <= kTmemCols, "TMEM budget");
};

__device__ __forceinline__ int clampi(int v, int lo, int hi) { return v < lo ? lo : (v > hi ? hi : v); }

// 32 scores of one row -> 16 packed 16-bit P values; kMask zeroes columns e >= nvalid (padded keys).
template <bool kMask, bool kBf16>
__device__ __forceinline__ void sigmoid_row32(float (&v)[32], uint32_t (&pk)[16], float a, float c, bool row_valid,
                                              int nvalid) {
  sigma_row<32, kMask, 0>(v, a, c, row_valid, nvalid);
#pragma unroll
  for (int e = 0; e < 32; e += 2) {
    float p0 = v[e], p1 = v[e + 1];
    if constexpr (kMask) {
      p0 = (e < nvalid) ? p0 : 0.0f;
      p1 = (e + 1 < nvalid) ? p1 : 0.0f;
    }
    pk[e >> 1] = sm100::pack2<kBf16>(p0, p1);
  }
}

// sigmoid_row32 for a chunk loaded from TMEM address taddr.  SIGATTN_FWD_SPEC: the tier-4 sigma is
// evaluated speculatively before the warp vote; on a failed vote (some valid logit > -4, rare with
// b = -log n) the scores are reloaded -- the chunk's S columns are not yet overwritten by P -- and
// the exact tiers of sigma_row run.
// Speculative tier of sigmoid_chunk32, chosen per work item from the sequence's bias: with
// b = -log n and logits alpha s of unit spread, some logit of a 32 x 32 chunk exceeds -4 in ~0.03% of
// the chunks at n = 8192 (b = -9) but ~15% at n = 2048 (b = -7.6), and a failed speculation (reload +
// exact redo) holds up the whole pair's P for that key tile.  Items with b <= kSpec4MaxBias speculate
// the <= -4 tier (one FFMA2 per pair after the ex2), the others the <= -2 tier (three FMA-pipe ops
// per pair).  Measured (d = 128): n = 2048 forward 0.31 -> 0.25 ms with the <= -2 tier, n = 8192
// 0.91 -> 0.97 ms; the two tie at n = 4096 (b = -8.3).
constexpr float kSpec4MaxBias = -8.3f;

// 32 scores of one row (loaded from TMEM address taddr) -> 16 packed 16-bit P values.  SIGATTN_FWD_SPEC:
// the kTier sigma is evaluated before the warp vote while `spec` holds (the last chunk of the warp
// took a tier >= kTier); on a failed vote the scores are reloaded -- the chunk's S columns are not
// yet overwritten by P -- and the exact tiers of sigma_row run.
template <bool kMask, bool kBf16, int kTier>
__device__ __forceinline__ void sigmoid_chunk32(uint32_t taddr, float (&v)[32], uint32_t (&pk)[16], float a, float c,
                                                bool row_valid, int nvalid, bool& spec) {
#if SIGATTN_FWD_SPEC
  if (spec) {
    // t = x log2 e and the max of the valid t; the speculative tier's sigma of every element packed
    // straight to 16 bits (the scores are dead afterwards, so the MUFU ex2 and the FMA-pipe work
    // interleave freely); the vote only decides whether to redo the chunk from the reloaded scores
    float m = -INFINITY;
#pragma unroll
    for (int e = 0; e < 32; e += 2) {
      ffma2(v[e], v[e + 1], v[e], v[e + 1], a, a, c, c);
      if constexpr (kMask)
        m = fmax3(m, e < nvalid ? v[e] : -INFINITY, e + 1 < nvalid ? v[e + 1] : -INFINITY);
      else
        m = fmax3(m, v[e], v[e + 1]);
    }
#pragma unroll
    for (int e = 0; e < 32; e += 2) {
      float p0, p1;
      if constexpr (kTier == 4) sigma2_fast4(v[e], v[e + 1], p0, p1);
      else sigma2_fast(v[e], v[e + 1], p0, p1);
      if constexpr (kMask) {
        p0 = (e < nvalid) ? p0 : 0.0f;
        p1 = (e + 1 < nvalid) ? p1 : 0.0f;
      }
      pk[e >> 1] = sm100::pack2<kBf16>(p0, p1);
    }
    if (__all_sync(0xffffffffu, !row_valid || m <= (kTier == 4 ? kFastT4 : kFastT))) return;
    sm100::tmem_ld32_sync(taddr, v);   // rare: the speculative tier failed
  }
  spec = sigma_row<32, kMask, 0>(v, a, c, row_valid, nvalid) >= kTier;
#pragma unroll
  for (int e = 0; e < 32; e += 2) {
    float p0 = v[e], p1 = v[e + 1];
    if constexpr (kMask) {
      p0 = (e < nvalid) ? p0 : 0.0f;
      p1 = (e + 1 < nvalid) ? p1 : 0.0f;
    }
    pk[e >> 1] = sm100::pack2<kBf16>(p0, p1);
  }
#else
  (void)taddr;
  (void)spec;
  sigmoid_row32<kMask, kBf16>(v, pk, a, c, row_valid, nvalid);
#endif
}

template <int D, bool kBf16, bool kOutF32>
__global__ void __launch_bounds__(FwdCfg<D>::kThreads, 1)
sigattn_fwd_kernel(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmK,
                   const __grid_constant__ CUtensorMap tmV, const FwdArgs args) {
  using C = FwdCfg<D>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + C::kBarOff);
  uint64_t* q_full = bars + 0;          // [2]
  uint64_t* q_empty = bars + 2;         // [2]
  uint64_t* k_full = bars + 4;          // [kStages]
  uint64_t* v_full = k_full + C::kStages;
  uint64_t* k_empty = v_full + C::kStages;   // K slot free: its S MMA completed
  uint64_t* v_empty = k_empty + C::kStages;  // V slot free: its PV MMA completed
  uint64_t* s_full = v_empty + C::kStages;   // [kSBuf]
  uint64_t* p_full = s_full + C::kSBuf;      // [kSBuf]
  uint64_t* o_full = p_full + C::kSBuf;      // [kOBufs]
  uint64_t* o_empty = o_full + C::kOBufs;    // [kOBufs]
  uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(bars + C::kNumBars);

  const uint32_t warp = sm100::warp_id();
  const uint32_t lane = sm100::lane_id();

  if (threadIdx.x == 0) {
    for (int i = 0; i < 2; ++i) {
      sm100::mbar_init(&q_full[i], 1);
      sm100::mbar_init(&q_empty[i], 1);
    }
    for (int i = 0; i < (int)C::kSBuf; ++i) {
      sm100::mbar_init(&s_full[i], 1);
      sm100::mbar_init(&p_full[i], 2 * C::kNumWG);   // the 8 warps of the pair that owns the tile
    }
    for (int i = 0; i < C::kStages; ++i) {
      sm100::mbar_init(&k_full[i], 1);
      sm100::mbar_init(&v_full[i], 1);
      sm100::mbar_init(&k_empty[i], 1);
      sm100::mbar_init(&v_empty[i], 1);
    }
    for (int i = 0; i < C::kOBufs; ++i) {
      sm100::mbar_init(&o_full[i], 1);
      sm100::mbar_init(&o_empty[i], 2 * C::kNumWG);   // the 8 warps of the pair that runs the epilogue
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
  const int BH = args.B * args.H;
  (void)BH;

  if (warp == C::kWarpTMA) {
    // ===================== TMA producer (whole warp waits, one elected lane issues) =====================
    const uint64_t pol_q = sm100::policy_evict_first();
    const uint64_t pol_kv = sm100::policy_evict_last();
    uint32_t kv_it = 0, c = 0;
    for (int it = first_item(); it < n_items; it = next_item(it)) {
      const int4 item = args.items[it];
      const int b = item.x, h = item.y, qt = item.z, nkt = item.w;
      if (nkt <= 0) continue;
      const int zh = b * args.H + h;
      const uint32_t qb = c & 1, qph = (c >> 1) & 1;
      sm100::mbar_wait_backoff(&q_empty[qb], qph ^ 1);
      if (sm100::elect_one()) {
        sm100::mbar_arrive_expect_tx(&q_full[qb], C::kTileBytes);
        uint8_t* qs = smem + C::kQOff + qb * C::kTileBytes;
#pragma unroll
        for (int s = 0; s < C::kSub; ++s)
          sm100::tma_load_bh(qs + s * (kTile * 128), &tmQ, &q_full[qb], s * 64, qt * kTile, zh, pol_q, args.bshd ? args.H : 0);
      }
      __syncwarp();
      for (int j = 0; j < nkt; ++j, ++kv_it) {
        const uint32_t st = kv_it % C::kStages, ph = (kv_it / C::kStages) & 1;
        // K and V slots are released separately (K after its S MMA, V after its PV MMA), so the
        // S look-ahead never waits for a PV that is itself waiting for sigma.
        sm100::mbar_wait_backoff(&k_empty[st], ph ^ 1);
        if (sm100::elect_one()) {
          sm100::trace_event(args.trace, kv_it, 512);
          uint8_t* ks = smem + C::kKOff + st * C::kTileBytes;
          if (SIGATTN_DBG_FWD_NOTMA_KV && kv_it >= (uint32_t)C::kStages) {
            sm100::mbar_arrive(&k_full[st]);
          } else {
            sm100::mbar_arrive_expect_tx(&k_full[st], C::kTileBytes);
#pragma unroll
            for (int s = 0; s < C::kSub; ++s)
              sm100::tma_load_bh(ks + s * (kTile * 128), &tmK, &k_full[st], s * 64, j * kTile, zh, pol_kv, args.bshd ? args.H : 0);
          }
        }
        __syncwarp();
        sm100::mbar_wait_backoff(&v_empty[st], ph ^ 1);
        if (sm100::elect_one()) {
          uint8_t* vs = smem + C::kVOff + st * C::kTileBytes;
          if (SIGATTN_DBG_FWD_NOTMA_KV && kv_it >= (uint32_t)C::kStages) {
            sm100::mbar_arrive(&v_full[st]);
          } else {
            sm100::mbar_arrive_expect_tx(&v_full[st], C::kTileBytes);
#pragma unroll
            for (int s = 0; s < C::kSub; ++s)
              sm100::tma_load_bh(vs + s * (kTile * 128), &tmV, &v_full[st], s * 64, j * kTile, zh, pol_kv, args.bshd ? args.H : 0);
          }
        }
        __syncwarp();
      }
      ++c;
    }
  } else if (warp == C::kWarpMMA) {
    // ===================== MMA issuer (whole warp waits, one elected lane issues) =====================
    constexpr uint32_t idesc_s = sm100::make_idesc_f16(kBf16, 128, 128, false, false);
    constexpr uint32_t idesc_o = sm100::make_idesc_f16(kBf16, 128, D, false, true);
    const uint32_t q_base = sm100::smem_u32(smem + C::kQOff);
    const uint32_t k_base = sm100::smem_u32(smem + C::kKOff);
    const uint32_t v_base = sm100::smem_u32(smem + C::kVOff);
    // One stream of key tiles over all of this CTA's items: S runs two tiles ahead of PV ACROSS item
    // boundaries (the next item's Q is double-buffered), so the tensor pipe and the sigmoid warps see
    // no pipeline drain at the end of a query tile.
    struct Cur {
      int it, j, nkt;
      uint32_t c;   // item ordinal (Q buffer / O buffer parity)
    };
    auto skip_empty = [&](Cur& x) {
      while (x.it < n_items && (x.nkt = args.items[x.it].w) <= 0) x.it = next_item(x.it);
    };
    auto advance = [&](Cur& x) {
      if (++x.j >= x.nkt) {
        x.j = 0;
        ++x.c;
        x.it = next_item(x.it);
        skip_empty(x);
      }
    };
    Cur sc{first_item(), 0, 0, 0};   // next S to issue
    skip_empty(sc);
    Cur pc = sc;                     // next PV to issue
    uint32_t s_it = 0;               // global index of the next S (= K/V ring index, TMEM S buffer)
    auto issue_s = [&]() {
      if (sc.it >= n_items) return;
      const uint32_t qb = sc.c & 1;
      if (sc.j == 0) sm100::mbar_wait(&q_full[qb], (sc.c >> 1) & 1);
      const uint32_t qa = q_base + qb * C::kTileBytes;
      const uint32_t st = s_it % C::kStages;
      sm100::mbar_wait(&k_full[st], (s_it / C::kStages) & 1);
      sm100::tc_fence_after();
      const uint32_t ka = k_base + st * C::kTileBytes;
      const uint32_t d_s = tmem + (s_it % C::kSBuf) * 128;
      if (sm100::elect_one()) {
        // stage-base descriptors; a K step adds (offset >> 4) to the start-address field (no carry:
        // every operand lies inside the CTA's shared window)
        const uint64_t dq0 = sm100::make_sdesc_sw128(qa, 16, 1024), dk0 = sm100::make_sdesc_sw128(ka, 16, 1024);
#pragma unroll
        for (int kk = 0; kk < D / 16; ++kk) {
          const uint32_t off = (kk >> 2) * (kTile * 128) + (kk & 3) * 32;
          sm100::mma_ss(d_s, dq0 + (off >> 4), dk0 + (off >> 4), idesc_s, kk > 0);
        }
        sm100::mma_commit(&s_full[s_it % C::kSBuf]);
        sm100::mma_commit(&k_empty[st]);
        sm100::trace_event(args.trace, 512 + s_it, 1024);
      }
      __syncwarp();
      ++s_it;
      advance(sc);
    };
    // S(g+2) reuses the buffer of P(g-1), read by PV(g-1) issued earlier (tcgen05 ops of one thread
    // execute in order), so it never waits for sigma(g).
    issue_s();
    issue_s();
    for (uint32_t si = 0; pc.it < n_items; ++si) {
      issue_s();
      SIGATTN_FWD_MMA_WAIT(&p_full[si % C::kSBuf], (si / C::kSBuf) & 1);
      const uint32_t ob = pc.c % C::kOBufs;
      if (pc.j == 0) sm100::mbar_wait(&o_empty[ob], ((pc.c / C::kOBufs) & 1) ^ 1);   // epilogue drained this O
      const uint32_t st = si % C::kStages;
      sm100::mbar_wait(&v_full[st], (si / C::kStages) & 1);
      sm100::tc_fence_after();
      const uint32_t va = v_base + st * C::kTileBytes;
      const uint32_t p_col = (si % C::kSBuf) * 128;
      if (sm100::elect_one()) {
        sm100::trace_event(args.trace, 1024 + si, 1536);
        const uint64_t dv0 = sm100::make_sdesc_sw128(va, kTile * 128, 1024);
#pragma unroll
        for (int kk = 0; kk < kTile / 16; ++kk) {
          // P for keys [16kk, 16kk+16): pair warpgroup kk/4 packed its 64 keys at S cols [64 (kk/4), +32)
          const uint32_t a_col = p_col + (kk >> 2) * 64 + (kk & 3) * 8;
          sm100::mma_ts(tmem + C::kColO + ob * D, tmem + a_col, dv0 + ((kk * 2048) >> 4), idesc_o,
                        (pc.j > 0 || kk > 0) ? 1u : 0u);
        }
        sm100::mma_commit(&v_empty[st]);
        if (pc.j == 0 && args.counters) atomicAdd(args.counters, (unsigned long long)pc.nkt);
        if (pc.j == pc.nkt - 1) {
          sm100::mma_commit(&q_empty[pc.c & 1]);
          sm100::mma_commit(&o_full[ob]);
        }
        sm100::trace_event(args.trace, 1536 + si, 2048);
      }
      __syncwarp();
      advance(pc);
    }
  } else if (warp < C::kWarpTMA) {
    // ===================== sigmoid warpgroups + epilogue =====================
    const uint32_t g = warp >> 2;                // warpgroup
    const uint32_t pair = warp >> 3;             // warpgroup pair: takes the key tiles with si % 2 == pair
    const uint32_t gp = g & 1;                   // within the pair: key columns [64 gp, 64 gp + 64)
    const uint32_t quarter = warp & 3;           // TMEM lane quarter this warp may access
    const uint32_t row = quarter * 32 + lane;    // tile row = TMEM lane
    const uint32_t lane_addr = (quarter * 32) << 16;
    bool spec = true;                            // speculate while the last chunk took the speculated tier
    uint32_t s_it = 0, c = 0;
    for (int it = first_item(); it < n_items; it = next_item(it)) {
      const int4 item = args.items[it];
      const int b = item.x, h = item.y, qt = item.z, nkt = item.w;
      if (nkt <= 0) continue;
      const int nq = clampi(args.seqlens_q ? args.seqlens_q[b] : args.Nq, 0, args.Nq);
      const int nk = clampi(args.seqlens_k ? args.seqlens_k[b] : args.Nk, 0, args.Nk);
      const float bias = args.bias_per_seq ? args.bias_per_seq[b] : args.bias;
      const float a2 = args.scale * kLog2e;    // t = x log2 e = s (alpha log2 e) + b log2 e
      const float b2 = bias * kLog2e;
      const bool spec4 = bias <= kSpec4MaxBias;   // speculative sigma tier of this item
      const bool row_valid = qt * kTile + (int)row < nq;
      // the key loop, instantiated for the item's speculative sigma tier (one hot copy per item)
      auto key_loop = [&](auto tier_c) {
        constexpr int kT = decltype(tier_c)::value;
        for (int j = 0; j < nkt; ++j) {
          const uint32_t si = s_it + j;
          if ((si & 1) != pair) continue;          // the other warpgroup pair takes this key tile
          if (lane == 0 && warp == pair * 8) sm100::trace_event(args.trace, 3072 + si, 3584);
          SIGATTN_COMPUTE_WAIT(&s_full[si % C::kSBuf], (si / C::kSBuf) & 1);
          if (lane == 0 && warp == pair * 8) sm100::trace_event(args.trace, 2048 + si, 2560);
          sm100::tc_fence_after();
#pragma unroll
          for (int ch = 0; ch < 2; ++ch) {
            const uint32_t col = (si % C::kSBuf) * 128 + gp * 64 + ch * 32;
            const int nvalid = nk - (j * kTile + (int)gp * 64 + ch * 32);   // valid keys in these 32 columns
            float r[32];
            uint32_t pk[16];
            sm100::tmem_ld32_sync(tmem + lane_addr + col, r);
  #if SIGATTN_DBG_FWD_NOSIGMA   // timing experiments only: P = bits of S, no sigma work
#pragma unroll
            for (int e = 0; e < 16; ++e) pk[e] = __float_as_uint(r[2 * e]) ^ __float_as_uint(r[2 * e + 1]);
  #else
            if (nvalid >= 32) sigmoid_chunk32<false, kBf16, kT>(tmem + lane_addr + col, r, pk, a2, b2, row_valid, nvalid, spec);
            else sigmoid_chunk32<true, kBf16, kT>(tmem + lane_addr + col, r, pk, a2, b2, row_valid, nvalid, spec);
  #endif
            // P over the first half of this warpgroup's 64 columns (chunk 0's columns are already read)
            sm100::tmem_st16(tmem + lane_addr + (si % C::kSBuf) * 128 + gp * 64 + ch * 16, pk);
          }
          sm100::tmem_wait_st();
          sm100::tc_fence_before();
          __syncwarp();
          if (lane == 0) sm100::mbar_arrive(&p_full[si % C::kSBuf]);
          if (lane == 0 && warp == pair * 8) sm100::trace_event(args.trace, 2560 + si, 3072);
        }
      };
      if (spec4) key_loop(std::integral_constant<int, 4>{});
      else key_loop(std::integral_constant<int, 2>{});
      // ---- epilogue, run by the pair that evaluated the item's last key tile (the other pair goes
      // straight on to the next item's first tile): O rows of this q tile, columns [gp D/2, +D/2)
      const uint32_t epi_pair = (s_it + nkt - 1) & 1;
      s_it += nkt;
      if (pair == epi_pair) {
        const uint32_t ob = c % C::kOBufs;
        if (lane == 0 && warp == pair * 8) sm100::trace_event(args.trace, 3584 + 3 * c, 4094);
        sm100::mbar_wait(&o_full[ob], (c / C::kOBufs) & 1);
        if (lane == 0 && warp == pair * 8) sm100::trace_event(args.trace, 3584 + 3 * c + 1, 4094);
        sm100::tc_fence_after();
        constexpr int kPart = D / 2;   // columns per warpgroup of the pair
        const uint32_t ocol = C::kColO + ob * D + gp * kPart;
        const int qrow = qt * kTile + (int)row;
        const bool valid = qrow < nq;
#pragma unroll
        for (int h0 = 0; h0 < kPart; h0 += 32) {
          uint32_t ov[32];
          sm100::tmem_ld32_sync(tmem + lane_addr + ocol + h0, ov);
          if (h0 + 32 >= kPart) {
            sm100::tc_fence_before();
            __syncwarp();
            if (lane == 0) sm100::mbar_arrive(&o_empty[ob]);
          }
          if (kOutF32 && args.peer_o) {
            if (valid) peer_red_row32(args, D, b, h, qrow, gp * kPart + h0, ov);
          } else if (qrow < args.Nq) {
            const size_t off = row_off(args.bshd, args.H, args.Nq, D, b, h, qrow) + gp * kPart + h0;
            if constexpr (kOutF32) {
              float4* dst = reinterpret_cast<float4*>(reinterpret_cast<float*>(args.o) + off);
#pragma unroll
              for (int e = 0; e < 32; e += 4) {
                float4 w = valid ? make_float4(__uint_as_float(ov[e]), __uint_as_float(ov[e + 1]),
                                               __uint_as_float(ov[e + 2]), __uint_as_float(ov[e + 3]))
                                 : make_float4(0.f, 0.f, 0.f, 0.f);
                dst[e >> 2] = w;
              }
            } else {
              uint4* dst = reinterpret_cast<uint4*>(reinterpret_cast<uint16_t*>(args.o) + off);
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
        if (lane == 0 && warp == pair * 8) sm100::trace_event(args.trace, 3584 + 3 * c + 2, 4094);
      }
      ++c;
    }
  }

  if (!SIGATTN_DBG_NOFILL && (warp == C::kWarpFill || warp == C::kWarpAlloc) && args.o)   // padded O rows beyond the last valid tile
    pad_fill_warp(args.o, D * (kOutF32 ? 4 : 2), args.B, args.H, args.Nq, args.seqlens_q, args.seqlens_k, args.Nk,
                  128, lane, args.bshd, args.fill_pad, warp == C::kWarpFill ? 0 : 1, 2);

  if (kOutF32 && args.peer_o) sm100::fence_sys();   // this CTA's peer reductions before kernel completion
  sm100::tc_fence_before();
  __syncthreads();
  if (threadIdx.x == 0) sm100::trace_globaltime(args.trace, 4095);
  if (warp == C::kWarpAlloc) sm100::tmem_dealloc<C::kTmemCols>(tmem);
}

}  // namespace sigattn
