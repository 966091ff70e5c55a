// bwd.cuh -- sm_100a backward kernel of padding-aware sigmoid attention.
//
// The paper splits the backward into a dQ kernel (Alg. 2) and a dK/dV kernel
// (Alg. 3), each recomputing sigma.  Here the two are fused into ONE key-tile-owned
// pass: every (b, h, key tile j) item keeps K_j, V_j resident (in shared
// memory and, copied once by tcgen05.cp, in TMEM) and loops over the valid 128-query tiles i, each
// processed as two 64-query halves q:
//     S^T_q  = K_j Q_iq^T,  dP^T_q = V_j dO_iq^T     (Alg. 3)   TS: A = K_j / V_j in TMEM
//     P^T_q  = mask . sigma(alpha S^T_q + b)
//     dS^T_q = P^T_q (1 - P^T_q) dP^T_q
//     dV_j  += P^T_q dO_iq,  dK_j += dS^T_q Q_iq          TS: A = P^T / dS^T in TMEM
//     dQ_i   = dS_i K_j (both halves)                 SS: A = dS^T smem (MN-major)
// dQ_i is an fp32 partial per key tile, reduce-added into a workspace; alpha is
// applied once in the epilogues.  sigma is evaluated once per element; the tensor work is the
// credited 10 d per (query, key) pair.
//
// Pipelining: the MMA warp issues, per tile i,   dV/dK(i, q0) | S,dP(i+1, q0) | dV/dK(i, q1) |
// S,dP(i+1, q1) | dQ(i)   so while the compute warps work on one half, the tensor core finishes the
// other half and prepares the next tile's scores for it.
//
// CTA roles (768 threads, persistent, one CTA per SM; single-thread roles in the highest warp ids,
// which the warp scheduler favours):
//   warps 0-15  compute: thread = key row (TMEM lane); all 16 warps process query half 0, then half 1;
//               warpgroup w takes 16 queries [64q + 16w, +16) of half q
//   warps 16-19 epilogue warpgroup: dQ_i drain (tcgen05.ld -> x alpha -> swizzled fp32 smem tile ->
//               two TMA bulk tensor reduce-adds into the fp32 workspace, in L2), dK/dV of a finished
//               key tile (x alpha for dK, round, store; padded rows = 0)
//   warp 20     TMA: K_j, V_j (2 slots), Q_i + dO_i (2 stages)
//   warp 21     MMA issuer (one elected thread); also tcgen05.cp of K_j, V_j into TMEM
//   warp 22     TMEM allocator
// TMEM (d = 64): S^T [0,128) dP^T [128,256) dV [256,320) dK [320,384) dQ [384,448) K [448,480) V [480,512)
// P^T / dS^T (16-bit) overwrite the first half of each warpgroup's own S^T / dP^T columns.
// Shared memory: dS^T (16-bit, 128B-swizzled, keys as rows, double-buffered) is read MN-major as
// the A operand of dQ = dS K.
#pragma once
#include "fwd.cuh"
#include "sigmoid.cuh"

#ifndef SIGATTN_BWD_MMA_SPIN
#define SIGATTN_BWD_MMA_SPIN 0    // 1: the MMA warp spins (no nanosleep back-off) on p_full
#endif
#if SIGATTN_BWD_MMA_SPIN
#define MMA_WAIT_P(b, p) sm100::mbar_wait(b, p)
#else
#define MMA_WAIT_P(b, p) sm100::mbar_wait_backoff(b, p)
#endif
#ifndef SIGATTN_BWD_SPEC
#define SIGATTN_BWD_SPEC 1        // tier-4 sigma evaluated before the warp vote (sigma_row_spec4)
#endif
#ifndef SIGATTN_BWD_SPEC_V2
#define SIGATTN_BWD_SPEC_V2 1     // speculative tier 4 without the ordering barrier (sigmoid_chunk32 style)
#endif
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
  float* dq_acc;          // fp32 [B,H,Nq,D], zero on valid rows at entry; receives alpha dS K
  void* dk;               // [B,H,Nk,D]
  void* dv;
  void* dq_pad;           // 16-bit dQ output whose rows >= ceil128(n_q) the fill warp zeroes, or nullptr
  int fill_pad;           // 1: zero the padded output rows no tile epilogue writes; 0 (NO_ZERO_PAD_OUT):
                          //    only the valid rows of sequences with an empty key / query set
  float* dbias;           // [B] fp32, zeroed at entry, += sum of dS (learnable bias gradient); or nullptr
  long long* trace;       // SIGATTN_TRACE builds: [grid][4096] clock64 event slots (8 events x 512 tiles)
  int bshd;               // 1: tensors are [B, N, H, d], else [B, H, N, d]
  unsigned long long* counters;   // skip accounting (sigattn_set_debug_counters) or nullptr
};

template <int D>
struct BwdCfg {
  static_assert(D == 64, "fused backward: d = 64 TMEM plan");
  static constexpr int kTileBytes = kTile * D * 2;           // 16 KB
  static constexpr int kQStages = 2;                         // Q_i + dO_i ring
  static constexpr int kKOff = 0;                            // K[2]
  static constexpr int kVOff = kKOff + 2 * kTileBytes;       // V[2]
  static constexpr int kQOff = kVOff + 2 * kTileBytes;       // Q[kQStages]
  static constexpr int kDOOff = kQOff + kQStages * kTileBytes;      // dO[kQStages]
  static constexpr int kDSOff = kDOOff + kQStages * kTileBytes;     // dS^T[2]: 2 halves of [128 keys][64 q]
  static constexpr int kDSBytes = 2 * kTile * 128;
  static constexpr int kDQOff = kDSOff + 2 * kDSBytes;      // fp32 dQ staging tile for the TMA reduce-add
  static constexpr int kBarOff = kDQOff + kTile * D * 4;
  static constexpr int kNumBars = 2 + 2 + 2 * kQStages + 2 + 2 + 2 + 1 + 1 + 1 + 1 + 2;
  static constexpr int kSmemBytes = kBarOff + kNumBars * 8 + 16 + 1024;
  static constexpr int kNumWG = 4;                           // compute warpgroups
  static constexpr int kWarpEpi = 4 * kNumWG, kWarpTMA = kWarpEpi + 4, kWarpMMA = kWarpTMA + 1,
                       kWarpAlloc = kWarpTMA + 2, kWarpFill = kWarpTMA + 3;
  static constexpr int kThreads = 32 * (kWarpEpi + 8);
  static constexpr uint32_t kTmemCols = 512;
  static constexpr uint32_t kColS = 0, kColDP = 128, kColDV = 256, kColDK = 320, kColDQ = 384, kColK = 448,
                            kColV = 480;
};


// Query tile visited at step i of key tile kt's sweep: odd key tiles sweep backwards, so the CTAs of
// one (b, h) split into two streams that meet in the middle instead of all reduce-adding their dQ
// partials into the same query tile at the same time (L2 atomics on the same lines serialise);
// each stream still shares its Q / dO tiles in L2.
#ifndef SIGATTN_BWD_ALT_SWEEP
#define SIGATTN_BWD_ALT_SWEEP 1
#endif
__device__ __forceinline__ int sweep_tile(int kt, int i, int nqt) {
  return (SIGATTN_BWD_ALT_SWEEP && (kt & 1)) ? nqt - 1 - i : i;
}

// Walks this CTA's non-empty work items (first_item / next_item order) and their query tiles.
struct TileIter {
  int it, n_items, i, nqt;
  uint32_t item_c;   // index of the current item among this CTA's non-empty items
  bool valid;
  __device__ __forceinline__ void seek(const int4* items) {
    while (it < n_items && items[it].w <= 0) it = next_item(it);
    valid = it < n_items;
    nqt = valid ? items[it].w : 0;
  }
  __device__ __forceinline__ void init(const int4* items, int n) {
    it = first_item();
    n_items = n;
    i = 0;
    item_c = 0;
    seek(items);
  }
  __device__ __forceinline__ void advance(const int4* items) {
    if (++i >= nqt) {
      i = 0;
      it = next_item(it);
      ++item_c;
      seek(items);
    }
  }
};

// 16 query columns of one key row: P^T and dS^T = P^T (1 - P^T) dP^T, packed to 16 bits.
// kMask: columns e >= nvalid (padded queries) give P = dS = 0 (nvalid = 0 for a padded key row).
// kSum: also accumulate the fp32 dS values into *dsum (learnable-bias gradient).
// 16 query columns of one key row, step 1: scores -> P^T (fp32, in place).
// s_taddr: TMEM address the 16 scores were loaded from (still intact: each warp packs P / dS over its
// own columns only after this call).  SIGATTN_BWD_SPEC: the tier-4 sigma is evaluated before the warp
// vote; on a failed vote the scores are reloaded from s_taddr and the exact tiers run.  spec:
// speculate tier 4 (updated to whether this chunk took tier 4, so a warp stops speculating while its
// logits keep failing the vote).
// kTier: the speculated tier (4: <= -4, one FFMA2 per pair; 2: <= -2, three FMA-pipe ops), chosen per
// work item from the bias as in the forward (kSpec4MaxBias).
template <bool kMask, bool kSpec = true, int kTier = 4>
__device__ __forceinline__ void bwd_sigma16(float (&v)[16], float a2, float b2, bool key_valid, int nvalid,
                                            uint32_t s_taddr, bool& spec) {
  if constexpr (!kSpec) {   // vote first (measured better for the d = 64 fused backward)
    (void)s_taddr;
    (void)spec;
    sigma_row<16, kMask, 0>(v, a2, b2, key_valid, nvalid);
    return;
  }
#if SIGATTN_BWD_SPEC
  if (spec) {
#if SIGATTN_BWD_SPEC_V2
    // scale, max and the tier-4 sigma in place with no ordering barrier; the vote only gates a
    // reload-and-redo (as in the forward's sigmoid_chunk32)
    float m = -INFINITY;
#pragma unroll
    for (int e = 0; e < 16; e += 2) {
      ffma2(v[e], v[e + 1], v[e], v[e + 1], a2, a2, b2, b2);
      if constexpr (kMask)
        m = fmax3(m, e < nvalid ? v[e] : -INFINITY, e + 1 < nvalid ? v[e + 1] : -INFINITY);
      else
        m = fmax3(m, v[e], v[e + 1]);
    }
#pragma unroll
    for (int e = 0; e < 16; e += 2) {
      if constexpr (kTier == 4) sigma2_fast4(v[e], v[e + 1], v[e], v[e + 1]);
      else sigma2_fast(v[e], v[e + 1], v[e], v[e + 1]);
    }
    if (__all_sync(0xffffffffu, !key_valid || m <= (kTier == 4 ? kFastT4 : kFastT))) return;
#else
    if (sigma_row_spec4<16, kMask>(v, a2, b2, key_valid, nvalid)) return;   // v: scores in, P out
#endif
    sm100::tmem_ld16(s_taddr, v);   // rare: some valid logit > -4
    sm100::tmem_wait_ld_dep16(v);
  }
  spec = sigma_row<16, kMask, 0>(v, a2, b2, key_valid, nvalid) >= kTier;   // one inlined copy
#else
  (void)s_taddr;
  (void)spec;
  sigma_row<16, kMask, 0>(v, a2, b2, key_valid, nvalid);   // v: scores in, P out
#endif
}

// Step 2: dS^T = P^T (1 - P^T) dP^T, both packed to 16 bits.  kMask: columns e >= nvalid (padded
// queries) give P = dS = 0 (nvalid = 0 for a padded key row).  kSum: also accumulate the fp32 dS
// values into *dsum (learnable-bias gradient).
template <bool kMask, bool kBf16, bool kSum = false>
__device__ __forceinline__ void bwd_ds16(const float (&v)[16], const float (&dp)[16], uint32_t (&pp)[8],
                                         uint32_t (&dd)[8], int nvalid, float* dsum = nullptr) {
  float s0 = 0.f, s1 = 0.f;
#pragma unroll
  for (int e = 0; e < 16; e += 2) {
    float p0 = v[e], p1 = v[e + 1], u0, u1, d0, d1;
    ffma2(u0, u1, p0, p1, -p0, -p1, p0, p1);                   // p (1 - p)
    fmul2(d0, d1, u0, u1, dp[e], dp[e + 1]);
    if constexpr (kMask) {
      p0 = (e < nvalid) ? p0 : 0.0f;
      d0 = (e < nvalid) ? d0 : 0.0f;
      p1 = (e + 1 < nvalid) ? p1 : 0.0f;
      d1 = (e + 1 < nvalid) ? d1 : 0.0f;
    }
    if constexpr (kSum) fadd2(s0, s1, s0, s1, d0, d1);
    pp[e >> 1] = sm100::pack2<kBf16>(p0, p1);
    dd[e >> 1] = sm100::pack2<kBf16>(d0, d1);
  }
  if constexpr (kSum) *dsum += s0 + s1;
}

// Both steps on 16 query columns of one key row (scores and dP^T already loaded).
template <bool kMask, bool kBf16, bool kSum = false, bool kSpec = true, int kTier = 4>
__device__ __forceinline__ void bwd_row16(float (&v)[16], const float (&dp)[16], uint32_t (&pp)[8], uint32_t (&dd)[8],
                                          float a2, float b2, bool key_valid, int nvalid, uint32_t s_taddr,
                                          bool& spec, float* dsum = nullptr) {
  bwd_sigma16<kMask, kSpec, kTier>(v, a2, b2, key_valid, nvalid, s_taddr, spec);
  bwd_ds16<kMask, kBf16, kSum>(v, dp, pp, dd, nvalid, dsum);
}

// Adds a warp's per-lane partial sums of dS into dbias[b] (one atomic per warp).
__device__ __forceinline__ void dbias_flush(float* dbias, int b, float acc, uint32_t lane) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  if (lane == 0 && acc != 0.0f) atomicAdd(dbias + b, acc);
}

// kDQ = false: dK, dV only (the key-tile-owned pass of the deterministic backward, Alg. 3;
// dQ then comes from sigattn_dq_kernel, Alg. 2): no dQ MMA, no dS staging, no dQ reduction.
// kBSHD: tensors are [B, N, H, d] -- a template flag here (the d = 64 backward runs at the
// register limit; a runtime layout test cost 2% through extra spills)
template <int D, bool kBf16, bool kDQ = true, bool kDB = false, bool kBSHD = false>
__global__ void __launch_bounds__(BwdCfg<D>::kThreads, 1)
sigattn_bwd_kernel(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmK,
                   const __grid_constant__ CUtensorMap tmV, const __grid_constant__ CUtensorMap tmDO,
                   const __grid_constant__ CUtensorMap tmDQ, const BwdArgs args) {
  using C = BwdCfg<D>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + C::kBarOff);
  uint64_t* kv_full = bars + 0;                   // [2]
  uint64_t* kv_empty = bars + 2;                  // [2]
  uint64_t* qdo_full = bars + 4;                  // [kQStages]
  uint64_t* qdo_empty = qdo_full + C::kQStages;   // [kQStages]
  uint64_t* s_full = qdo_empty + C::kQStages;     // [2] per query half: S^T, dP^T in TMEM
  uint64_t* p_full = s_full + 2;                  // [2] per query half: P^T, dS^T in TMEM, dS^T in smem
  uint64_t* ds_free = p_full + 2;                 // [2] dQ MMA finished reading dS^T buffer
  uint64_t* dq_full = ds_free + 2;                // dQ(t) in TMEM
  uint64_t* dq_empty = dq_full + 1;               // epilogue read dQ(t) out of TMEM
  uint64_t* acc_full = dq_empty + 1;
  uint64_t* acc_empty = acc_full + 1;
  uint64_t* dp_full = acc_empty + 1;              // [2] per query half: dP^T in TMEM (S^T: s_full)
  uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(bars + C::kNumBars);

  const uint32_t warp = sm100::warp_id();
  const uint32_t lane = sm100::lane_id();
  constexpr uint32_t kComputeWarps = 4 * C::kNumWG;

  if (threadIdx.x == 0) {
    for (int i = 0; i < 2; ++i) {
      sm100::mbar_init(&kv_full[i], 1);
      sm100::mbar_init(&kv_empty[i], 1);
      sm100::mbar_init(&ds_free[i], 1);
      sm100::mbar_init(&s_full[i], 1);
      sm100::mbar_init(&dp_full[i], 1);
      sm100::mbar_init(&p_full[i], kComputeWarps);       // every compute warp works on every half
    }
    for (int i = 0; i < C::kQStages; ++i) {
      sm100::mbar_init(&qdo_full[i], 1);
      sm100::mbar_init(&qdo_empty[i], 1);
    }
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
  if (threadIdx.x == 0) sm100::trace_globaltime(args.trace, 4094);
  const int n_items = *args.n_items;

  if (warp == C::kWarpTMA) {
    // ===================== TMA producer (whole warp waits, one elected lane issues) =====================
    const uint64_t pol_kv = sm100::policy_evict_first();
    const uint64_t pol_q = sm100::policy_evict_last();
    uint32_t kv_c = 0, t = 0;
    for (int it = first_item(); it < n_items; it = next_item(it)) {
      const int4 item = args.items[it];
      const int b = item.x, h = item.y, kt = item.z, nqt = item.w;
      if (nqt <= 0) continue;
      const int zh = b * args.H + h;
      const uint32_t kvb = kv_c & 1;
      sm100::mbar_wait_backoff(&kv_empty[kvb], ((kv_c >> 1) & 1) ^ 1);
      if (sm100::elect_one()) {
        sm100::mbar_arrive_expect_tx(&kv_full[kvb], 2 * C::kTileBytes);
        sm100::tma_load_bh(smem + C::kKOff + kvb * C::kTileBytes, &tmK, &kv_full[kvb], 0, kt * kTile, zh, pol_kv, kBSHD ? args.H : 0);
        sm100::tma_load_bh(smem + C::kVOff + kvb * C::kTileBytes, &tmV, &kv_full[kvb], 0, kt * kTile, zh, pol_kv, kBSHD ? args.H : 0);
      }
      __syncwarp();
      for (int i = 0; i < nqt; ++i, ++t) {
        const uint32_t st = t % C::kQStages;
        sm100::mbar_wait_backoff(&qdo_empty[st], ((t / C::kQStages) & 1) ^ 1);
        if (sm100::elect_one()) {
          if (SIGATTN_DBG_NOTMA_QDO && t >= C::kQStages) {   // timing experiments only: stale Q/dO tiles
            sm100::mbar_arrive(&qdo_full[st]);
          } else {
            sm100::mbar_arrive_expect_tx(&qdo_full[st], 2 * C::kTileBytes);
            const int qi = sweep_tile(kt, i, nqt);
            sm100::tma_load_bh(smem + C::kQOff + st * C::kTileBytes, &tmQ, &qdo_full[st], 0, qi * kTile, zh, pol_q, kBSHD ? args.H : 0);
            sm100::tma_load_bh(smem + C::kDOOff + st * C::kTileBytes, &tmDO, &qdo_full[st], 0, qi * kTile, zh, pol_q, kBSHD ? args.H : 0);
          }
        }
        __syncwarp();
      }
      ++kv_c;
    }
  } else if (warp == C::kWarpMMA) {
    // ===================== MMA issuer (whole warp waits, one elected lane issues) =====================
    constexpr uint32_t idesc_s = sm100::make_idesc_f16(kBf16, 128, 64, false, false);    // S^T_q, dP^T_q
    constexpr uint32_t idesc_acc = sm100::make_idesc_f16(kBf16, 128, D, false, true);    // dV, dK
    constexpr uint32_t idesc_dq = sm100::make_idesc_f16(kBf16, 128, D, true, true);      // dQ
    const uint32_t k_base = sm100::smem_u32(smem + C::kKOff);
    const uint32_t v_base = sm100::smem_u32(smem + C::kVOff);
    const uint32_t q_base = sm100::smem_u32(smem + C::kQOff);
    const uint32_t do_base = sm100::smem_u32(smem + C::kDOOff);
    const uint32_t ds_base = sm100::smem_u32(smem + C::kDSOff);

    // K_j, V_j (smem, SW128 K-major) -> TMEM A-operand layout (16 elements per 8 columns)
    auto copy_kv = [&](uint32_t kvb) {
      const uint32_t ka = k_base + kvb * C::kTileBytes, va = v_base + kvb * C::kTileBytes;
#pragma unroll
      for (int kk = 0; kk < D / 16; ++kk) {
        sm100::tmem_cp_128x256b(tmem + C::kColK + kk * 8, sm100::sdesc_add(sm100::make_sdesc_sw128(ka, 16, 1024), kk * 32));
        sm100::tmem_cp_128x256b(tmem + C::kColV + kk * 8, sm100::sdesc_add(sm100::make_sdesc_sw128(va, 16, 1024), kk * 32));
      }
    };
    // S^T_q = K Q_q^T, then dP^T_q = V dO_q^T  (M = 128 keys, N = 64 queries, K = d; A from TMEM),
    // each signalled on its own barrier: sigma needs only S^T
    auto mma_s = [&](uint32_t st, uint32_t q) {
      const uint32_t qa = q_base + st * C::kTileBytes + q * 8192;
#pragma unroll
      for (int kk = 0; kk < D / 16; ++kk)
        sm100::mma_ts(tmem + C::kColS + q * 64, tmem + C::kColK + kk * 8,
                      sm100::sdesc_add(sm100::make_sdesc_sw128(qa, 16, 1024), kk * 32), idesc_s, kk > 0);
      sm100::mma_commit(&s_full[q]);
    };
    auto mma_dp = [&](uint32_t st, uint32_t q) {
      const uint32_t da = do_base + st * C::kTileBytes + q * 8192;
#pragma unroll
      for (int kk = 0; kk < D / 16; ++kk)
        sm100::mma_ts(tmem + C::kColDP + q * 64, tmem + C::kColV + kk * 8,
                      sm100::sdesc_add(sm100::make_sdesc_sw128(da, 16, 1024), kk * 32), idesc_s, kk > 0);
      sm100::mma_commit(&dp_full[q]);
    };
    // dV += P^T_q dO_q ; dK += dS^T_q Q_q   (M = keys, N = d, K = 64 queries; A from TMEM)
    auto mma_dv = [&](uint32_t st, uint32_t q, bool first) {
      const uint32_t da = do_base + st * C::kTileBytes + q * 8192;
#pragma unroll
      for (int kk = 0; kk < 4; ++kk) {
        // queries [64q + 16kk, +16): warpgroup kk packed them at S cols 64q + 16kk + [0, 8)
        const uint32_t a_col = q * 64 + kk * 16;
        sm100::mma_ts(tmem + C::kColDV, tmem + C::kColS + a_col,
                      sm100::sdesc_add(sm100::make_sdesc_sw128(da, kTile * 128, 1024), kk * 2048), idesc_acc,
                      (first && kk == 0) ? 0u : 1u);
      }
    };
    auto mma_dk = [&](uint32_t st, uint32_t q, bool first) {
      const uint32_t qa = q_base + st * C::kTileBytes + q * 8192;
#pragma unroll
      for (int kk = 0; kk < 4; ++kk) {
        const uint32_t a_col = q * 64 + kk * 16;
        sm100::mma_ts(tmem + C::kColDK, tmem + C::kColDP + a_col,
                      sm100::sdesc_add(sm100::make_sdesc_sw128(qa, kTile * 128, 1024), kk * 2048), idesc_acc,
                      (first && kk == 0) ? 0u : 1u);
      }
    };

    TileIter cur;
    cur.init(args.items, n_items);
    if (cur.valid) {
      sm100::mbar_wait(&kv_full[cur.item_c & 1], (cur.item_c >> 1) & 1);
      sm100::mbar_wait(&qdo_full[0], 0);
      sm100::tc_fence_after();
      if (sm100::elect_one()) {
        copy_kv(cur.item_c & 1);
        mma_s(0, 0);
        mma_dp(0, 0);
        mma_s(0, 1);
        mma_dp(0, 1);
      }
      __syncwarp();
    }
    // dQ(t) = dS(t) K after both halves' next-tile score MMAs (one tile later, between the halves of
    // tile t+1, measured slower: 3.03 vs 2.57 ms on C3; a second issuer warp for the gradient MMAs,
    // 2% slower).
    uint32_t prev_kvb = 0;
    bool prev_last = false;      // the tile dQ is pending for was its item's last (frees its K/V slot)
    auto issue_dq = [&](uint32_t tq) {
      if constexpr (!kDQ) {
        if (sm100::elect_one() && prev_last) sm100::mma_commit(&kv_empty[prev_kvb]);   // K/V smem slot free
        __syncwarp();
        return;
      }
      const uint32_t b2 = tq & 1;
#if !SIGATTN_DBG_MMAONLY
      sm100::mbar_wait(dq_empty, (tq & 1) ^ 1);                  // epilogue drained the accumulator
      // dS(tq) in smem: p_full of both halves (waited by the caller) covers the compute warps' stores
#endif
      if (lane == 0 && tq >= 40 && tq < 48) sm100::trace_event(args.trace, 3328 + (tq - 40) * 8 + 3, 4094);
      sm100::tc_fence_after();
      if (sm100::elect_one()) {
        const uint32_t ka = k_base + prev_kvb * C::kTileBytes;
        const uint32_t dsa = ds_base + b2 * C::kDSBytes;
        // dQ = dS K   (M = 128 queries, N = d, K = 128 keys; A = dS MN-major, B = K MN-major)
#pragma unroll
        for (int kk = 0; kk < kTile / 16; ++kk)
          sm100::mma_ss(tmem + C::kColDQ, sm100::sdesc_add(sm100::make_sdesc_sw128(dsa, kTile * 128, 1024), kk * 2048),
                        sm100::sdesc_add(sm100::make_sdesc_sw128(ka, kTile * 128, 1024), kk * 2048), idesc_dq, kk > 0);
        sm100::mma_commit(&ds_free[b2]);
        sm100::mma_commit(dq_full);
        if (prev_last) sm100::mma_commit(&kv_empty[prev_kvb]);   // K/V smem slot free
      }
      __syncwarp();
    };
    uint32_t t = 0;
    while (cur.valid) {
      TileIter nxt = cur;
      nxt.advance(args.items);
      const uint32_t st = t % C::kQStages, kvb = cur.item_c & 1;
      const uint32_t st1 = (t + 1) % C::kQStages;
#define MMA_TR(e) if (lane == 0 && t >= 40 && t < 48) sm100::trace_event(args.trace, 3328 + (t - 40) * 8 + (e), 4094)
      MMA_TR(4);
      // long wait (a compute phase): poll with back-off so the MMA warp does not steal issue slots
#if !SIGATTN_DBG_MMAONLY
      MMA_WAIT_P(&p_full[0], t & 1);
#endif
      if (lane == 0) sm100::trace_event(args.trace, 0 * 512 + t, 0 * 512 + 512);
#if !SIGATTN_DBG_MMAONLY
      if (cur.i == 0) sm100::mbar_wait(acc_empty, (cur.item_c & 1) ^ 1);   // epilogue read previous dV/dK
#endif
      // Per half q: dV(t, q) | S(t+1, q) | dK(t, q) | dP(t+1, q).  S(t+1, q) overwrites the S^T columns
      // holding P^T(t, q) right after dV(t, q) has read them, and dP(t+1, q) the dP^T columns holding
      // dS^T(t, q) after dK(t, q) (tcgen05 ops of one thread execute in order), so the compute warps
      // get S(t+1, q) eight MMAs after P(t, q) instead of sixteen, and start sigma before dP lands.
      sm100::tc_fence_after();
      if (sm100::elect_one()) mma_dv(st, 0, cur.i == 0);
      __syncwarp();
      MMA_TR(0);
      if (nxt.valid) {
        if (nxt.i == 0) sm100::mbar_wait(&kv_full[nxt.item_c & 1], (nxt.item_c >> 1) & 1);
        MMA_TR(5);
        sm100::mbar_wait(&qdo_full[st1], ((t + 1) / C::kQStages) & 1);
        MMA_TR(6);
        sm100::tc_fence_after();
        if (sm100::elect_one()) {
          // the copy executes after every earlier MMA (tcgen05 ops of one thread run in order), so
          // S/dP(t, q1) have finished reading the previous K/V columns
          if (nxt.i == 0) copy_kv(nxt.item_c & 1);
          mma_s(st1, 0);
        }
        __syncwarp();
      }
      MMA_TR(7);
      if (sm100::elect_one()) {
        mma_dk(st, 0, cur.i == 0);
        if (nxt.valid) mma_dp(st1, 0);
      }
      __syncwarp();
      if (lane == 0) sm100::trace_event(args.trace, 1 * 512 + t, 1 * 512 + 512);
#if !SIGATTN_DBG_MMAONLY
      MMA_WAIT_P(&p_full[1], t & 1);
#endif
      if (lane == 0) sm100::trace_event(args.trace, 2 * 512 + t, 2 * 512 + 512);
      sm100::tc_fence_after();
      if (sm100::elect_one()) {
        mma_dv(st, 1, false);
        if (nxt.valid) mma_s(st1, 1);
        mma_dk(st, 1, false);
        sm100::mma_commit(&qdo_empty[st]);                       // last readers of Q_i, dO_i
        if (cur.i == cur.nqt - 1) sm100::mma_commit(acc_full);   // dV, dK of this key tile are final
        if (cur.i == 0 && args.counters) atomicAdd(args.counters + 1, (unsigned long long)cur.nqt);
        if (nxt.valid) mma_dp(st1, 1);
      }
      __syncwarp();
      MMA_TR(1);
      MMA_TR(2);
      prev_kvb = kvb;
      prev_last = cur.i == cur.nqt - 1;
      issue_dq(t);
      if (lane == 0) sm100::trace_event(args.trace, 3 * 512 + t, 3 * 512 + 512);
      cur = nxt;
      ++t;
    }
  } else if (warp < kComputeWarps && !SIGATTN_DBG_MMAONLY) {
    // ===================== compute warps: all 16 work on each query half in turn =====================
    // warpgroup w4 owns queries [16 w4, 16 w4 + 16) of each 64-query half
    const uint32_t w4 = warp >> 2;
    const uint32_t quarter = warp & 3;
    const uint32_t row = quarter * 32 + lane;          // key row within the tile = TMEM lane
    const uint32_t lane_addr = (quarter * 32) << 16;
    const uint32_t ds_row = sm100::smem_u32(smem + C::kDSOff + (row >> 3) * 1024 + (row & 7) * 128);
    uint32_t t = 0;
    for (int it = first_item(); it < n_items; it = next_item(it)) {
      const int4 item = args.items[it];
      const int b = item.x, kt = item.z, nqt = item.w;
      if (nqt <= 0) continue;
      const int nq = clampi(args.seqlens_q ? args.seqlens_q[b] : args.Nq, 0, args.Nq);
      const int nk = clampi(args.seqlens_k ? args.seqlens_k[b] : args.Nk, 0, args.Nk);
      const float bias = args.bias_per_seq ? args.bias_per_seq[b] : args.bias;
      const float a2 = args.scale * kLog2e;    // t = x log2 e
      const float b2 = bias * kLog2e;
      const bool key_valid = kt * kTile + (int)row < nk;
      const bool warp_keys_valid = __all_sync(0xffffffffu, key_valid);
      float db_acc = 0.f;
      bool spec = true;   // speculate tier 4 while the last chunk took it
      // vote first (measured 1.5% faster than speculating the <= -4 tier on C3, and 2-3% faster than
      // speculating the <= -2 tier for b > kSpec4MaxBias at N = 1-2K)
      for (int i = 0; i < nqt; ++i, ++t) {
#pragma unroll
        for (int qh = 0; qh < 2; ++qh) {
          SIGATTN_COMPUTE_WAIT(&s_full[qh], t & 1);
#define BWD_TR(e) if (lane == 0 && t >= 40 && t < 48) sm100::trace_event(args.trace, 4 * 512 + (warp * 8 + (t - 40)) * 8 + (e), 6 * 512)
          BWD_TR(qh == 0 ? 0 : 3);
          sm100::tc_fence_after();
          const uint32_t s_col = C::kColS + qh * 64 + w4 * 16, dp_col = C::kColDP + qh * 64 + w4 * 16;
#if SIGATTN_DBG_NOCOMPUTE
          if (true) {
            __syncwarp();
            if (lane == 0) sm100::mbar_arrive(&p_full[qh]);
            continue;
          }
#endif
          float s[16], dp[16];
          sm100::tmem_ld16(tmem + lane_addr + s_col, s);
          sm100::tmem_wait_ld_dep16(s);
          // valid query columns here; the masked variant is chosen warp-uniformly (it also zeroes the
          // rows of padded keys)
          const int ncol = nq - (sweep_tile(kt, i, nqt) * kTile + qh * 64 + (int)w4 * 16);
          const bool full = warp_keys_valid && ncol >= 16;
          const int nv = full ? 16 : (key_valid ? ncol : 0);
          if (full) bwd_sigma16<false, false>(s, a2, b2, true, 16, tmem + lane_addr + s_col, spec);
          else bwd_sigma16<true, false>(s, a2, b2, key_valid, nv, tmem + lane_addr + s_col, spec);
          if (qh == 0) BWD_TR(6);
          // dP^T(t, q) lands after S^T(t, q): sigma above overlaps the dP^T MMAs
          SIGATTN_COMPUTE_WAIT(&dp_full[qh], t & 1);
          sm100::tc_fence_after();
          sm100::tmem_ld16(tmem + lane_addr + dp_col, dp);
          sm100::tmem_wait_ld_dep16(dp);
          if (qh == 0) BWD_TR(7);
          uint32_t pp[8], dd[8];
          if (full) bwd_ds16<false, kBf16, kDB>(s, dp, pp, dd, 16, &db_acc);
          else bwd_ds16<true, kBf16, kDB>(s, dp, pp, dd, nv, &db_acc);
          BWD_TR(qh == 0 ? 1 : 4);
          // P^T / dS^T over the first half of this warp's own (already read) columns, and dS^T into
          // the dQ MMA's shared-memory operand
          sm100::tmem_st8(tmem + lane_addr + s_col, pp);
          sm100::tmem_st8(tmem + lane_addr + dp_col, dd);
          if constexpr (kDQ) {
            // queries [64 qh + 16 w4, +16) of key row `row` = 16-byte chunks 2 w4, 2 w4 + 1 of the
            // half's 128-byte row, SW128 swizzle (chunk c at slot c ^ (row & 7))
            if (qh == 0) sm100::mbar_wait(&ds_free[t & 1], ((t >> 1) & 1) ^ 1);   // dQ(t-2) MMA done with the buffer
            const uint32_t dsr = ds_row + (t & 1) * C::kDSBytes + qh * (kTile * 128);
            sm100::st_shared_v4(dsr + (((2 * w4) ^ (row & 7)) * 16), dd[0], dd[1], dd[2], dd[3]);
            sm100::st_shared_v4(dsr + (((2 * w4 + 1) ^ (row & 7)) * 16), dd[4], dd[5], dd[6], dd[7]);
            // the dQ MMA reading both halves is issued after p_full[1]: one proxy fence there orders
            // this thread's stores of both halves
            if (qh == 1) sm100::fence_proxy_async_smem();
          }
          sm100::tmem_wait_st();
          sm100::tc_fence_before();
          __syncwarp();
          if (lane == 0) sm100::mbar_arrive(&p_full[qh]);
          BWD_TR(qh == 0 ? 2 : 5);
#undef BWD_TR
        }
      }
      if constexpr (kDB) dbias_flush(args.dbias, b, db_acc, lane);
    }
  } else if (warp < C::kWarpTMA && !SIGATTN_DBG_MMAONLY && warp >= kComputeWarps) {
    // ===================== epilogue warpgroup: dQ drain, dK/dV =====================
    // The compute warps store dS^T into the dQ MMA's shared-memory operand themselves (beside the TMEM
    // copy the dK MMA reads), so the tile's score MMAs never wait on a TMEM read-back; this warpgroup
    // drains dQ(t) as soon as it lands and writes dK/dV when a key tile is finished.
    const uint32_t quarter = warp & 3;
    const uint32_t row = quarter * 32 + lane;
    const uint32_t lane_addr = (quarter * 32) << 16;
    const float alpha = args.scale;
    // dQ(tq) += alpha * TMEM dQ through the TMA: the fp32 tile is written (SW128, two 32-column
    // boxes) into a dedicated staging buffer, then one thread issues two bulk tensor reduce-adds
    // into the fp32 accumulator (the adds happen in L2; no per-lane atomics).
    constexpr uint32_t kEpiThread0 = 32 * kComputeWarps;
#define EPI_TR(tt, e) if (threadIdx.x == kEpiThread0 && (tt) >= 40 && (tt) < 48) sm100::trace_event(args.trace, 3072 + ((tt) - 40) * 16 + (e), 4094)
    auto drain_dq = [&](uint32_t tq, int zh, int i) {
      sm100::mbar_wait(dq_full, tq & 1);
      EPI_TR(tq + 1, 7);
      sm100::tc_fence_after();
      uint8_t* buf = smem + C::kDQOff;
      const uint32_t sb = sm100::smem_u32(buf) + row * 128;
      // the previous tile's reduce-add has finished reading the staging buffer
      if (threadIdx.x == kEpiThread0) sm100::bulk_wait_group_read<0>();
      sm100::named_bar_sync(1, 128);
#pragma unroll
      for (int hh = 0; hh < 2; ++hh) {     // columns [32 hh, 32 hh + 32) -> box hh
        float r[2][16];
        if (SIGATTN_DBG_EPI_NOLD) {
          if (hh == 1 && lane == 0) sm100::mbar_arrive(dq_empty);
          continue;
        }
        sm100::tmem_ld16(tmem + lane_addr + C::kColDQ + hh * 32, r[0]);
        sm100::tmem_ld16(tmem + lane_addr + C::kColDQ + hh * 32 + 16, r[1]);
        sm100::tmem_wait_ld_dep16(r[0]);
        sm100::tmem_wait_ld_dep16(r[1]);
        if (hh == 1) {
          sm100::tc_fence_before();
          __syncwarp();
          if (lane == 0) sm100::mbar_arrive(dq_empty);
          EPI_TR(tq + 1, 8);
        }
#pragma unroll
        for (int c = 0; c < 8; ++c)   // 16-byte chunk c (columns 4c..4c+3) at slot c ^ (row & 7)
          sm100::st_shared_v4(sb + hh * (kTile * 128) + ((c ^ (row & 7)) * 16),
                              __float_as_uint(alpha * r[c >> 2][(c & 3) * 4]),
                              __float_as_uint(alpha * r[c >> 2][(c & 3) * 4 + 1]),
                              __float_as_uint(alpha * r[c >> 2][(c & 3) * 4 + 2]),
                              __float_as_uint(alpha * r[c >> 2][(c & 3) * 4 + 3]));
      }
      sm100::fence_proxy_async_smem();
      sm100::named_bar_sync(1, 128);
      EPI_TR(tq + 1, 9);
      if (threadIdx.x == kEpiThread0 && !SIGATTN_DBG_NORED) {
        // rows past Nq are clipped by the TMA; padded query rows add exact zeros (dS = 0 there)
        sm100::tma_reduce_add_3d(&tmDQ, buf, 0, i * kTile, zh);
        sm100::tma_reduce_add_3d(&tmDQ, buf + kTile * 128, 32, i * kTile, zh);
        sm100::bulk_commit_group();
      }
      EPI_TR(tq + 1, 10);
    };
    uint32_t t = 0, item_c = 0;
    for (int it = first_item(); it < n_items; it = next_item(it)) {
      const int4 item = args.items[it];
      const int b = item.x, h = item.y, kt = item.z, nqt = item.w;
      if (nqt <= 0) continue;
      const int nq = clampi(args.seqlens_q ? args.seqlens_q[b] : args.Nq, 0, args.Nq);
      const int nk = clampi(args.seqlens_k ? args.seqlens_k[b] : args.Nk, 0, args.Nk);
      const size_t zh = (size_t)(b * args.H + h);
      for (int i = 0; i < nqt * kDQ; ++i, ++t) {
        drain_dq(t, (int)zh, sweep_tile(kt, i, nqt));   // dQ(t) as soon as it lands
      }
      // ---- dV, dK rows of this key tile (dK scaled by alpha)
      sm100::mbar_wait_backoff(acc_full, item_c & 1);
      sm100::tc_fence_after();
      const int key = kt * kTile + (int)row;
      const bool key_valid = key < nk;
      const size_t off = kBSHD ? row_off(1, args.H, args.Nk, D, b, h, key) : (zh * args.Nk + key) * D;
#pragma unroll
      for (int which = 0; which < 2; ++which) {
        const uint32_t col = which == 0 ? C::kColDV : C::kColDK;
        const float sc = which == 0 ? 1.0f : alpha;
        uint4* dst = reinterpret_cast<uint4*>(reinterpret_cast<uint16_t*>(which == 0 ? args.dv : args.dk) + off);
#pragma unroll
        for (int hh = 0; hh < 2; ++hh) {
          float r[2][16];
          if (SIGATTN_DBG_EPI_NOLD) {
            if (which == 1 && hh == 1 && lane == 0) sm100::mbar_arrive(acc_empty);
            continue;
          }
          sm100::tmem_ld16(tmem + lane_addr + col + hh * 32, r[0]);
          sm100::tmem_ld16(tmem + lane_addr + col + hh * 32 + 16, r[1]);
          sm100::tmem_wait_ld_dep16(r[0]);
          sm100::tmem_wait_ld_dep16(r[1]);
          if (which == 1 && hh == 1) {
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
    if (kDQ && threadIdx.x == kEpiThread0) sm100::bulk_wait_group<0>();   // reduce-adds complete before exit
  }

  if (!SIGATTN_DBG_NOFILL && (warp == C::kWarpFill || warp == C::kWarpAlloc)) {   // padded dK / dV rows no tile epilogue writes
    pad_fill_warp(args.dk, D * 2, args.B, args.H, args.Nk, args.seqlens_k, args.seqlens_q, args.Nq, kTile, lane, kBSHD ? 1 : 0, args.fill_pad, warp == C::kWarpFill ? 0 : 1, 2);
    pad_fill_warp(args.dv, D * 2, args.B, args.H, args.Nk, args.seqlens_k, args.seqlens_q, args.Nq, kTile, lane, kBSHD ? 1 : 0, args.fill_pad, warp == C::kWarpFill ? 0 : 1, 2);
    if (args.dq_pad)   // dq_finalize_kernel covers the rows below
      pad_fill_warp(args.dq_pad, D * 2, args.B, args.H, args.Nq, args.seqlens_q, args.seqlens_k, args.Nk, kTile, lane, kBSHD ? 1 : 0, args.fill_pad, warp == C::kWarpFill ? 0 : 1, 2);
  }

  if (lane == 0) sm100::trace_event(args.trace, 4064 + (int)warp, 4092);   // per-warp end (trace builds)
  sm100::tc_fence_before();
  __syncthreads();
  if (threadIdx.x == 0) sm100::trace_globaltime(args.trace, 4095);
  if (warp == C::kWarpAlloc) sm100::tmem_dealloc<C::kTmemCols>(tmem);
}

}  // namespace sigattn
