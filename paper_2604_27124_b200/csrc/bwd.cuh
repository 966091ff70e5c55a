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
// Pipelining: two MMA issuers.  Warp 21 issues S,dP(i, q) as soon as dV/dK(i-1, q) have read the
// previous tile's P^T/dS^T out of those TMEM columns; warp 22 issues dV/dK(i, q) once the compute warps
// stored P^T/dS^T(i, q), then dQ(i).  While the compute warps work on one half, the tensor core finishes
// the other half and prepares the next tile's scores for it.
//
// CTA roles (768 threads, persistent, one CTA per SM; single-thread roles in the highest warp ids,
// which the warp scheduler favours):
//   warps 0-15  compute: thread = key row (TMEM lane); all 16 warps process query half 0, then half 1;
//               warpgroup w takes 16 queries [64q + 16w, +16) of half q
//   warps 16-19 epilogue warpgroup: dS^T staging into shared memory for the dQ MMA, dQ_i drain
//               (tcgen05.ld -> x alpha -> swizzled fp32 smem tile -> TMA bulk reduce-add into the
//               fp32 workspace), dK/dV of a finished key tile (x alpha for dK, round, store; padded rows = 0)
//   warp 20     TMA: K_j, V_j (2 slots), Q_i + dO_i (3 stages)
//   warp 21     score MMA issuer (one elected thread); also tcgen05.cp of K_j, V_j into TMEM
//   warp 22     TMEM allocator, then gradient MMA issuer (dV, dK, dQ)
// TMEM (d = 64): S^T [0,128) dP^T [128,256) dV [256,320) dK [320,384) dQ [384,448) K [448,480) V [480,512)
// P^T / dS^T (16-bit) overwrite the first half of each warpgroup's own S^T / dP^T columns.
// Shared memory: dS^T (16-bit, 128B-swizzled, keys as rows, double-buffered) is read MN-major as
// the A operand of dQ = dS K.
#pragma once
#include "fwd.cuh"
#include "sigmoid.cuh"

#ifndef SIGATTN_BWD_MMA_SPIN
#define SIGATTN_BWD_MMA_SPIN 0    // 1: the gradient-MMA warp spins (no nanosleep back-off) on p_full
#endif
#if SIGATTN_BWD_MMA_SPIN
#define MMA_WAIT_P(b, p) sm100::mbar_wait(b, p)
#else
#define MMA_WAIT_P(b, p) sm100::mbar_wait_backoff(b, p)
#endif
#ifndef SIGATTN_DBG_NOCOMPUTE
#define SIGATTN_DBG_NOCOMPUTE 0   // timing experiments only (wrong results): compute warps skip sigma + TMEM I/O
#endif
#ifndef SIGATTN_DBG_EPI_NOLD
#define SIGATTN_DBG_EPI_NOLD 0    // timing experiments only: epilogue skips TMEM loads and global writes
#endif
#ifndef SIGATTN_DBG_NORED
#define SIGATTN_DBG_NORED 0       // timing experiments only: skip the dQ reduce-add into global memory
#endif
#ifndef SIGATTN_DBG_NOSTAGE
#define SIGATTN_DBG_NOSTAGE 0     // timing experiments only (wrong results): epilogue skips the dS smem staging
#endif
#ifndef SIGATTN_BWD_SPEC
#define SIGATTN_BWD_SPEC 1        // tier-4 sigma evaluated before the warp vote (sigma_row_spec4)
#endif
#ifndef SIGATTN_BWD64_SPEC
#define SIGATTN_BWD64_SPEC false  // ... in the d = 64 fused backward: vote first measured 1.5-8% faster
#endif
#ifndef SIGATTN_BWD_EMU
#define SIGATTN_BWD_EMU 0         // every k-th element pair takes the FMA-pipe exp2 (0: all on MUFU)
#endif
#ifndef SIGATTN_DBG_NOTMA_QDO
#define SIGATTN_DBG_NOTMA_QDO 0   // timing experiments only: Q/dO tiles loaded once, then reused (stale)
#endif
#ifndef SIGATTN_DBG_MMAONLY
#define SIGATTN_DBG_MMAONLY 0     // timing experiments only: MMA + TMA pipeline alone (no compute/epilogue waits)
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
  // key-split context parallelism with the dQ reduction fused into the epilogue (sigattn_bwd_cp):
  // peer_dq[g] is rank g's fp32 accumulator [B, H, peer_rows, D]; alpha dS K of query q is
  // reduce-added into peer_dq[q / peer_rows] at row q % peer_rows instead of into dq_acc
  float* const* peer_dq;
  int peer_rows;
};

// A staged fp32 dQ tile (n_boxes SW128 boxes of [box_rows][32 floats], 16-byte chunk c of row r at
// slot c ^ (r & 7)) -> reduce-adds into the owning ranks' accumulators, 8 threads per 128-byte box
// row so every warp writes 4 full rows (context parallelism, A4: P:121).  tid in [0, 128).
__device__ __forceinline__ void peer_red_staged(const BwdArgs& args, const uint8_t* tile, int n_boxes, int box_rows,
                                                int D, int zh, int row0, int nq, uint32_t tid) {
  for (int hh = 0; hh < n_boxes; ++hh)
    for (int idx = (int)tid; idx < box_rows * 8; idx += 128) {
      const int r = idx >> 3, c = idx & 7, qrow = row0 + r;
      if (qrow >= nq) continue;   // padded query rows carry exact zeros (dS = 0)
      const float4 v = *reinterpret_cast<const float4*>(tile + hh * box_rows * 128 + r * 128 + ((c ^ (r & 7)) * 16));
      const int owner = qrow / args.peer_rows, lr = qrow - owner * args.peer_rows;
      float* dst = args.peer_dq[owner] + ((size_t)zh * args.peer_rows + lr) * D + hh * 32 + c * 4;
      sm100::red_add_v4_sys(dst, v.x, v.y, v.z, v.w);
    }
}

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
  static constexpr int kNumBars = 2 + 2 + 2 * kQStages + 2 + 2 + 2 + 2 + 1 + 1 + 2 + 2 + 2;
  static constexpr int kSmemBytes = kBarOff + kNumBars * 8 + 16 + 1024;
  static constexpr int kNumWG = 4;                           // compute warpgroups
  // kWarpMMA issues the score MMAs (S^T, dP^T) and the K/V TMEM copies, kWarpGrad the gradient MMAs
  // (dV, dK, dQ); kWarpGrad also allocates TMEM before the roles start
  static constexpr int kWarpEpi = 4 * kNumWG, kWarpTMA = kWarpEpi + 4, kWarpMMA = kWarpTMA + 1,
                       kWarpGrad = kWarpTMA + 2, kWarpAlloc = kWarpTMA + 2, kWarpFill = kWarpTMA + 3;
  static constexpr int kThreads = 32 * (kWarpEpi + 8);
  static constexpr uint32_t kTmemCols = 512;
  static constexpr uint32_t kColS = 0, kColDP = 128, kColDV = 256, kColDK = 320, kColDQ = 384, kColK = 448,
                            kColV = 480;
};


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
template <bool kMask, bool kSpec = true>
__device__ __forceinline__ void bwd_sigma16(float (&v)[16], float a2, float b2, bool key_valid, int nvalid,
                                            uint32_t s_taddr, bool& spec) {
  if constexpr (!kSpec) {   // vote first (measured better for the d = 64 fused backward)
    (void)s_taddr;
    (void)spec;
    sigma_row<16, kMask, SIGATTN_BWD_EMU>(v, a2, b2, key_valid, nvalid);
    return;
  }
#if SIGATTN_BWD_SPEC
  bool done = false;
  if (spec) {
    done = sigma_row_spec4<16, kMask>(v, a2, b2, key_valid, nvalid);   // v: scores in, P out
    if (!done) {
      sm100::tmem_ld16(s_taddr, v);
      sm100::tmem_wait_ld_dep16(v);
    }
  }
  if (!done) spec = sigma_row<16, kMask, 0>(v, a2, b2, key_valid, nvalid) == 4;   // one inlined copy
#else
  (void)s_taddr;
  (void)spec;
  sigma_row<16, kMask, SIGATTN_BWD_EMU>(v, a2, b2, key_valid, nvalid);   // v: scores in, P out
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
template <bool kMask, bool kBf16, bool kSum = false, bool kSpec = true>
__device__ __forceinline__ void bwd_row16(float (&v)[16], const float (&dp)[16], uint32_t (&pp)[8], uint32_t (&dd)[8],
                                          float a2, float b2, bool key_valid, int nvalid, uint32_t s_taddr,
                                          bool& spec, float* dsum = nullptr) {
  bwd_sigma16<kMask, kSpec>(v, a2, b2, key_valid, nvalid, s_taddr, spec);
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
  uint64_t* ds_copied = acc_empty + 1;            // [2] per query half: epilogue read dS^T from TMEM
  uint64_t* ds_full = ds_copied + 2;              // [2] per dS smem buffer: both halves staged + fenced
  uint64_t* dvdk_done = ds_full + 2;              // [2] per query half: dV/dK MMAs have read P^T / dS^T
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
      sm100::mbar_init(&p_full[i], kComputeWarps);       // every compute warp works on every half
      sm100::mbar_init(&ds_copied[i], 4);
      sm100::mbar_init(&ds_full[i], 4);                  // the 4 epilogue warps, after both halves
      sm100::mbar_init(&dvdk_done[i], 1);
    }
    for (int i = 0; i < C::kQStages; ++i) {
      sm100::mbar_init(&qdo_full[i], 1);
      sm100::mbar_init(&qdo_empty[i], 2);                // both MMA warps read Q_i, dO_i
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
            sm100::tma_load_bh(smem + C::kQOff + st * C::kTileBytes, &tmQ, &qdo_full[st], 0, i * kTile, zh, pol_q, kBSHD ? args.H : 0);
            sm100::tma_load_bh(smem + C::kDOOff + st * C::kTileBytes, &tmDO, &qdo_full[st], 0, i * kTile, zh, pol_q, kBSHD ? args.H : 0);
          }
        }
        __syncwarp();
      }
      ++kv_c;
    }
  } else if (warp == C::kWarpMMA || warp == C::kWarpGrad) {
    // ===================== MMA issuers (whole warp waits, one elected lane issues) =====================
    // A tcgen05.mma issue blocks while the tensor pipe is busy (the queue holds about one MMA), so an
    // issuer's barrier waits (~100 clk each, even when already complete) drain the pipe.  Two issuers
    // whose streams only meet through barriers keep it fed while either one waits:
    //   kWarpMMA   per tile i, half q: S^T, dP^T(i, q)     (after dV/dK(i-1, q) read P^T/dS^T there)
    //   kWarpGrad  per tile i: dV, dK(i, q0), dV, dK(i, q1), then dQ(i) = dS(i) K
    constexpr uint32_t idesc_s = sm100::make_idesc_f16(kBf16, 128, 64, false, false);    // S^T_q, dP^T_q
    constexpr uint32_t idesc_acc = sm100::make_idesc_f16(kBf16, 128, D, false, true);    // dV, dK
    constexpr uint32_t idesc_dq = sm100::make_idesc_f16(kBf16, 128, D, true, true);      // dQ
    const uint32_t k_base = sm100::smem_u32(smem + C::kKOff);
    const uint32_t v_base = sm100::smem_u32(smem + C::kVOff);
    const uint32_t q_base = sm100::smem_u32(smem + C::kQOff);
    const uint32_t do_base = sm100::smem_u32(smem + C::kDOOff);
    const uint32_t ds_base = sm100::smem_u32(smem + C::kDSOff);
    TileIter cur;
    cur.init(args.items, n_items);
    if (warp == C::kWarpMMA) {
      for (uint32_t t = 0; cur.valid; cur.advance(args.items), ++t) {
        const uint32_t st = t % C::kQStages, kvb = cur.item_c & 1;
        if (cur.i == 0) sm100::mbar_wait(&kv_full[kvb], (cur.item_c >> 1) & 1);
        sm100::mbar_wait(&qdo_full[st], (t / C::kQStages) & 1);
#pragma unroll
        for (int q = 0; q < 2; ++q) {
          if (t > 0) {   // the previous tile's P^T / dS^T in these columns are consumed
            sm100::mbar_wait(&dvdk_done[q], (t - 1) & 1);
            if (kDQ && !SIGATTN_DBG_MMAONLY) sm100::mbar_wait(&ds_copied[q], (t - 1) & 1);
          }
          sm100::tc_fence_after();
          if (sm100::elect_one()) {
            if (q == 0 && cur.i == 0) {
              // K_j, V_j (smem, SW128 K-major) -> TMEM A-operand layout (16 elements per 8 columns); in
              // order after this warp's last S^T / dP^T MMAs of the previous item, which read them
              const uint32_t ka = k_base + kvb * C::kTileBytes, va = v_base + kvb * C::kTileBytes;
#pragma unroll
              for (int kk = 0; kk < D / 16; ++kk) {
                sm100::tmem_cp_128x256b(tmem + C::kColK + kk * 8, sm100::sdesc_add(sm100::make_sdesc_sw128(ka, 16, 1024), kk * 32));
                sm100::tmem_cp_128x256b(tmem + C::kColV + kk * 8, sm100::sdesc_add(sm100::make_sdesc_sw128(va, 16, 1024), kk * 32));
              }
            }
            // S^T_q = K Q_q^T and dP^T_q = V dO_q^T  (M = 128 keys, N = 64 queries, K = d; A from TMEM)
            const uint32_t qa = q_base + st * C::kTileBytes + q * 8192, da = do_base + st * C::kTileBytes + q * 8192;
            const uint64_t dq0 = sm100::make_sdesc_sw128(qa, 16, 1024), dd0 = sm100::make_sdesc_sw128(da, 16, 1024);
#pragma unroll
            for (int kk = 0; kk < D / 16; ++kk)
              sm100::mma_ts(tmem + C::kColS + q * 64, tmem + C::kColK + kk * 8, dq0 + ((kk * 32) >> 4), idesc_s, kk > 0);
#pragma unroll
            for (int kk = 0; kk < D / 16; ++kk)
              sm100::mma_ts(tmem + C::kColDP + q * 64, tmem + C::kColV + kk * 8, dd0 + ((kk * 32) >> 4), idesc_s, kk > 0);
            sm100::mma_commit(&s_full[q]);
            if (q == 1) sm100::mma_commit(&qdo_empty[st]);   // this warp's reads of Q_i, dO_i
          }
          __syncwarp();
          if (lane == 0 && t > 0) sm100::trace_event(args.trace, (q == 0 ? 512 : 3328) + t - 1, q == 0 ? 1024 : 4000);
        }
      }
    } else {
      for (uint32_t t = 0; cur.valid; cur.advance(args.items), ++t) {
        const uint32_t st = t % C::kQStages, kvb = cur.item_c & 1;
        const bool last = cur.i == cur.nqt - 1;
#pragma unroll
        for (int q = 0; q < 2; ++q) {
          // dV += P^T_q dO_q ; dK += dS^T_q Q_q   (M = keys, N = d, K = 64 queries; A from TMEM)
#if !SIGATTN_DBG_MMAONLY
          MMA_WAIT_P(&p_full[q], t & 1);
          if (lane == 0) sm100::trace_event(args.trace, q * 1024 + t, q * 1024 + 512);
          if (q == 0 && cur.i == 0) sm100::mbar_wait(acc_empty, (cur.item_c & 1) ^ 1);   // epilogue read previous dV/dK
#endif
          sm100::tc_fence_after();
          if (sm100::elect_one()) {
            const uint32_t qa = q_base + st * C::kTileBytes + q * 8192, da = do_base + st * C::kTileBytes + q * 8192;
            const uint64_t dq0 = sm100::make_sdesc_sw128(qa, kTile * 128, 1024), dd0 = sm100::make_sdesc_sw128(da, kTile * 128, 1024);
            const bool first = cur.i == 0 && q == 0;
#pragma unroll
            for (int kk = 0; kk < 4; ++kk)   // queries [64q + 16kk, +16): warpgroup kk packed them at cols 64q + 16kk + [0, 8)
              sm100::mma_ts(tmem + C::kColDV, tmem + C::kColS + q * 64 + kk * 16, dd0 + ((kk * 2048) >> 4), idesc_acc,
                            (first && kk == 0) ? 0u : 1u);
#pragma unroll
            for (int kk = 0; kk < 4; ++kk)
              sm100::mma_ts(tmem + C::kColDK, tmem + C::kColDP + q * 64 + kk * 16, dq0 + ((kk * 2048) >> 4), idesc_acc,
                            (first && kk == 0) ? 0u : 1u);
            sm100::mma_commit(&dvdk_done[q]);
            if (q == 1) {
              sm100::mma_commit(&qdo_empty[st]);                 // this warp's reads of Q_i, dO_i
              if (last) sm100::mma_commit(acc_full);             // dV, dK of this key tile are final
              if (cur.i == 0 && args.counters) atomicAdd(args.counters + 1, (unsigned long long)cur.nqt);
            }
          }
          __syncwarp();
        }
        if constexpr (kDQ) {
          // dQ(t) = dS(t) K   (M = 128 queries, N = d, K = 128 keys; A = dS MN-major, B = K MN-major)
#if !SIGATTN_DBG_MMAONLY
          sm100::mbar_wait(dq_empty, (t & 1) ^ 1);              // epilogue drained the accumulator
          sm100::mbar_wait(&ds_full[t & 1], (t >> 1) & 1);      // dS(t) staged in smem, proxy-fenced
#endif
          sm100::tc_fence_after();
          if (sm100::elect_one()) {
            const uint32_t ka = k_base + kvb * C::kTileBytes;
            const uint64_t ds0 = sm100::make_sdesc_sw128(ds_base + (t & 1) * C::kDSBytes, kTile * 128, 1024);
            const uint64_t k0 = sm100::make_sdesc_sw128(ka, kTile * 128, 1024);
#pragma unroll
            for (int kk = 0; kk < kTile / 16; ++kk)
              sm100::mma_ss(tmem + C::kColDQ, ds0 + ((kk * 2048) >> 4), k0 + ((kk * 2048) >> 4), idesc_dq, kk > 0);
            sm100::mma_commit(&ds_free[t & 1]);
            sm100::mma_commit(dq_full);
            if (last) sm100::mma_commit(&kv_empty[kvb]);        // K/V smem slot free
          }
          __syncwarp();
          if (lane == 0) sm100::trace_event(args.trace, 1536 + t, 2048);
        } else {
          if (sm100::elect_one() && last) sm100::mma_commit(&kv_empty[kvb]);
          __syncwarp();
        }
      }
    }
  } else if (warp < kComputeWarps && !SIGATTN_DBG_MMAONLY) {
    // ===================== compute warps: all 16 work on each query half in turn =====================
    // warpgroup w4 owns queries [16 w4, 16 w4 + 16) of each 64-query half (splitting the halves between
    // two warp sets instead was measured 2-3% slower)
    const uint32_t w4 = warp >> 2;
    const uint32_t quarter = warp & 3;
    const uint32_t row = quarter * 32 + lane;          // key row within the tile = TMEM lane
    const uint32_t lane_addr = (quarter * 32) << 16;
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
          sm100::tmem_ld16(tmem + lane_addr + dp_col, dp);
          sm100::tmem_wait_ld_dep16(s);
          sm100::tmem_wait_ld_dep16(dp);
          // valid query columns here; the masked variant is chosen warp-uniformly (it also zeroes the
          // rows of padded keys)
          const int ncol = nq - (i * kTile + qh * 64 + (int)w4 * 16);
          uint32_t pp[8], dd[8];
          if (warp_keys_valid && ncol >= 16) bwd_row16<false, kBf16, kDB, SIGATTN_BWD64_SPEC>(s, dp, pp, dd, a2, b2, true, 16, tmem + lane_addr + s_col, spec, &db_acc);
          else bwd_row16<true, kBf16, kDB, SIGATTN_BWD64_SPEC>(s, dp, pp, dd, a2, b2, key_valid, key_valid ? ncol : 0, tmem + lane_addr + s_col, spec, &db_acc);
          BWD_TR(qh == 0 ? 1 : 4);
          // P^T / dS^T over the first half of this warp's own (already read) columns; the epilogue
          // warpgroup stages dS^T into shared memory for the dQ MMA
          sm100::tmem_st8(tmem + lane_addr + s_col, pp);
          sm100::tmem_st8(tmem + lane_addr + dp_col, dd);
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
    // ===================== epilogue warpgroup: dS^T staging, dQ drain, dK/dV =====================
    // Per query tile t: for each half, copy the packed dS^T the compute warps left in TMEM into the
    // swizzled smem operand of the dQ MMA (so the compute warps never wait on shared-memory stores or
    // proxy fences), then drain dQ(t-1) -- one tile behind, so the drain never delays the copies the
    // MMA warp is waiting for.
    const uint32_t quarter = warp & 3;
    const uint32_t row = quarter * 32 + lane;
    const uint32_t lane_addr = (quarter * 32) << 16;
    const uint32_t ds_row = sm100::smem_u32(smem + C::kDSOff + (row >> 3) * 1024 + (row & 7) * 128);
    const float alpha = args.scale;
    // dQ(tq) += alpha * TMEM dQ through the TMA: the fp32 tile is written (SW128, two 32-column
    // boxes) into a dedicated staging buffer, then one thread issues two bulk tensor reduce-adds
    // into the fp32 accumulator (the adds happen in L2; no per-lane atomics).  (Reusing the dS
    // buffer instead put the reduce's smem read on the dS staging path: +2000 clk per tile.)
    constexpr uint32_t kEpiThread0 = 32 * kComputeWarps;
#define EPI_TR(tt, e) if (threadIdx.x == kEpiThread0 && (tt) >= 40 && (tt) < 48) sm100::trace_event(args.trace, 3072 + ((tt) - 40) * 16 + (e), 4094)
    auto drain_dq = [&](uint32_t tq, int zh, int i, int nq_) {
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
      if (args.peer_dq) {
        peer_red_staged(args, buf, 2, kTile, D, zh, i * kTile, nq_, threadIdx.x - kEpiThread0);
      } else if (threadIdx.x == kEpiThread0 && !SIGATTN_DBG_NORED) {
        // rows past Nq are clipped by the TMA; padded query rows add exact zeros (dS = 0 there)
        sm100::tma_reduce_add_3d(&tmDQ, buf, 0, i * kTile, zh);
        sm100::tma_reduce_add_3d(&tmDQ, buf + kTile * 128, 32, i * kTile, zh);
        sm100::bulk_commit_group();
      }
      EPI_TR(tq + 1, 10);
    };
    uint32_t t = 0, item_c = 0;
    bool pend = false;            // a dQ tile waiting to be drained
    int pend_zh = 0, pend_i = 0, pend_nq = 0;
    for (int it = first_item(); it < n_items; it = next_item(it)) {
      const int4 item = args.items[it];
      const int b = item.x, h = item.y, kt = item.z, nqt = item.w;
      if (nqt <= 0) continue;
      const int nq = clampi(args.seqlens_q ? args.seqlens_q[b] : args.Nq, 0, args.Nq);
      const int nk = clampi(args.seqlens_k ? args.seqlens_k[b] : args.Nk, 0, args.Nk);
      const size_t zh = (size_t)(b * args.H + h);
      for (int i = 0; i < nqt * kDQ; ++i, ++t) {
        const uint32_t dsr = ds_row + (t & 1) * C::kDSBytes;
#pragma unroll 1
        for (int qh = 0; qh < 2; ++qh) {
          sm100::mbar_wait(&p_full[qh], t & 1);
          EPI_TR(t, qh == 0 ? 0 : 4);
          sm100::tc_fence_after();
          uint32_t d[4][8];   // packed dS^T of queries [64 qh + 16 g, +16) at columns 64 qh + 16 g + [0, 8)
#pragma unroll
          for (int g = 0; g < 4 * !SIGATTN_DBG_EPI_NOLD; ++g)
            sm100::tmem_ld8(tmem + lane_addr + C::kColDP + qh * 64 + g * 16, d[g]);
          sm100::tmem_wait_ld_dep4x8(d);
          sm100::tc_fence_before();
          __syncwarp();
          if (lane == 0) sm100::mbar_arrive(&ds_copied[qh]);
          EPI_TR(t, qh == 0 ? 1 : 5);
          if (qh == 0) {
            sm100::mbar_wait(&ds_free[t & 1], ((t >> 1) & 1) ^ 1);   // dQ(t-2) MMA done with the buffer
            EPI_TR(t, 2);
          }
#pragma unroll
          for (int c = 0; c < 8 * !SIGATTN_DBG_NOSTAGE; ++c)   // 16-byte chunk c = queries [8c, 8c + 8) of this half, SW128 swizzle
            sm100::st_shared_v4(dsr + qh * (kTile * 128) + ((c ^ (row & 7)) * 16), d[c >> 1][(c & 1) * 4],
                                d[c >> 1][(c & 1) * 4 + 1], d[c >> 1][(c & 1) * 4 + 2], d[c >> 1][(c & 1) * 4 + 3]);
          if (qh == 1) {   // one proxy fence covers both halves' stores
            sm100::fence_proxy_async_smem();
            __syncwarp();
            if (lane == 0) sm100::mbar_arrive(&ds_full[t & 1]);
          }
          EPI_TR(t, qh == 0 ? 3 : 6);
        }
        if (pend) drain_dq(t - 1, pend_zh, pend_i, pend_nq);
        pend = true;
        pend_zh = (int)zh;
        pend_i = i;
        pend_nq = nq;
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
    if (kDQ && pend) drain_dq(t - 1, pend_zh, pend_i, pend_nq);
    if (kDQ && args.peer_dq) sm100::fence_sys();   // peer reductions before kernel completion
    if (kDQ && threadIdx.x == kEpiThread0) sm100::bulk_wait_group<0>();   // reduce-adds complete before exit
  }

  if (!SIGATTN_DBG_NOFILL && warp == C::kWarpFill) {   // padded dK / dV rows no tile epilogue writes
    pad_fill_warp(args.dk, D * 2, args.B, args.H, args.Nk, args.seqlens_k, args.seqlens_q, args.Nq, kTile, lane, kBSHD ? 1 : 0, args.fill_pad);
    pad_fill_warp(args.dv, D * 2, args.B, args.H, args.Nk, args.seqlens_k, args.seqlens_q, args.Nq, kTile, lane, kBSHD ? 1 : 0, args.fill_pad);
    if (args.dq_pad)   // dq_finalize_kernel covers the rows below
      pad_fill_warp(args.dq_pad, D * 2, args.B, args.H, args.Nq, args.seqlens_q, args.seqlens_k, args.Nk, kTile, lane, kBSHD ? 1 : 0, args.fill_pad);
  }

  sm100::tc_fence_before();
  __syncthreads();
  if (threadIdx.x == 0) sm100::trace_globaltime(args.trace, 4095);
  if (warp == C::kWarpAlloc) sm100::tmem_dealloc<C::kTmemCols>(tmem);
}

}  // namespace sigattn
