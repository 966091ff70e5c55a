// sched.cuh -- small device kernels around the two attention kernels:
//   * the work-list builder (padded-tile skipping + longest-first order),
//   * the backward prologue (work list + dQ-accumulator zeroing, one launch) and dQ finalisation,
//   * the padded-row zero fill the attention kernels run in their idle warp,
//   * key-padding-mask -> valid lengths conversion.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "debug.cuh"
#include "sm100.cuh"


namespace sigattn {

constexpr int kSchedThreads = 1024;
constexpr int kMaxSchedB = 4096;      // sequences per batch the single-block builder supports
constexpr int kMaxTail = 128;         // tail items the kind-2 split handles (m <= G / 2, G <= 256 CTAs)
constexpr int kMinPiece = 8;          // key tiles per piece of a split tail item (at least)

// Work items of this CTA in a persistent grid: rounds of gridDim.x consecutive items of the
// longest-first list, dealt boustrophedon (even rounds by CTA index, odd rounds reversed), so the
// CTA that gets the largest item of one round gets the smallest of the next.  On C3 this lifts the
// load balance (mean / max CTA work) from 96.4% (plain stride) to 98.3%.
__device__ __forceinline__ int first_item() { return (int)blockIdx.x; }
__device__ __forceinline__ int next_item(int it) {
  const int G = (int)gridDim.x, r = it / G, p = it - r * G;
  const int c = (r & 1) ? G - 1 - p : p;          // this CTA
  return (r + 1) * G + (((r + 1) & 1) ? G - 1 - c : c);
}

__device__ __forceinline__ int clamp_len(const int32_t* lens, int b, int N) {
  int n = lens ? lens[b] : N;
  return n < 0 ? 0 : (n > N ? N : n);
}

// Work items: kind 0 (forward)  -> (b, h, q-tile) for q-tiles holding a valid query, cost = key tiles
//             kind 1 (backward) -> (b, h, k-tile) for k-tiles holding a valid key,  cost = query tiles
//             kind 2 (forward, two query tiles per item) -> (b, h, q-tile pair), cost = key tiles
// Items with cost 0 are not emitted (their outputs are all padding and are zero-filled).
// Order: sequences by cost descending (ties: b ascending); within a sequence h-major, tile-minor.
// One CTA of kSchedThreads threads; B <= kMaxSchedB.  Shared memory: 4 B + 1 ints.
__device__ __forceinline__ void build_worklist_block(int kind, int B, int H, int Nq, int Nk,
                                                     const int32_t* __restrict__ seqlens_q,
                                                     const int32_t* __restrict__ seqlens_k, int4* __restrict__ items,
                                                     int* __restrict__ n_items, int* sh) {
  int* cost = sh;           // [B]
  int* ntile = sh + B;      // [B]
  int* order = sh + 2 * B;  // [B] rank -> b
  int* offs = sh + 3 * B;   // [B + 1] rank -> first item
  for (int b = threadIdx.x; b < B; b += blockDim.x) {
    const int nq = clamp_len(seqlens_q, b, Nq);
    const int nk = clamp_len(seqlens_k, b, Nk);
    const int tq = (nq + 127) / 128, tk = (nk + 127) / 128;
    int c = kind == 1 ? tq : tk;
    int t = kind == 0 ? tq : (kind == 1 ? tk : (tq + 1) / 2);   // kind 2: pairs of query tiles
    if (c == 0) t = 0;
    cost[b] = c;
    ntile[b] = t;
  }
  __syncthreads();
  for (int b = threadIdx.x; b < B; b += blockDim.x) {
    const int cb = cost[b];
    int rank = 0;
    for (int o = 0; o < B; ++o) {
      const int co = cost[o];
      rank += (co > cb) || (co == cb && o < b);
    }
    order[rank] = b;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    int acc = 0;
    for (int r = 0; r < B; ++r) {
      offs[r] = acc;
      acc += H * ntile[order[r]];
    }
    offs[B] = acc;
    *n_items = acc;
  }
  __syncthreads();
  const int total = offs[B];
  for (int i = threadIdx.x; i < total; i += blockDim.x) {   // parallel emission
    int lo = 0, hi = B;                                    // last rank with offs[r] <= i
    while (hi - lo > 1) {
      const int mid = (lo + hi) >> 1;
      if (offs[mid] <= i) lo = mid; else hi = mid;
    }
    while (lo + 1 < B && offs[lo + 1] <= i) ++lo;           // skip empty sequences
    const int b = order[lo], nt = ntile[b], local = i - offs[lo];
    items[i] = make_int4(b, local / nt, local % nt, cost[b]);
  }
}

// Tail split of a kind-2 list for a persistent grid of G CTAs (the d = 128 forward).  Items are
// dealt in rounds of G; with R full rounds and m < G/2 items left, the last round would keep only m
// CTAs busy (equal-cost items -- e.g. a uniformly padded batch -- leave up to a whole item of tail).
// Each of the m tail items is cut along its KEY range into up to G/m pieces, so the last round fills
// the grid with short pieces.  Sigmoid attention is additive over key blocks, so a piece
// writes its partial O (fp32, both query tiles) into its own slot of a piece buffer and
// fwd_split_finalize_kernel sums the pieces of each split item: plain stores, no atomics, no zeroing,
// deterministic.  Encoding of a piece: x = b | (piece + 1) << 16, z = pair | first key tile << 16,
// w = key tiles of the piece; map[slot] = (b, h, pair, first piece | pieces << 16).
__device__ __forceinline__ void split_tail_block(int G, int4* __restrict__ items, int* __restrict__ n_items,
                                                 int4* __restrict__ map, int* __restrict__ n_split) {
  __syncthreads();
  if (threadIdx.x != 0) return;
  const int n = *n_items, R = n / G, m = n - R * G;
  int nsplit = 0;
  if (R >= 1 && m > 0 && 2 * m <= G) {
    const int s = G / m;
    int4 tail[kMaxTail];
    for (int t = 0; t < m; ++t) tail[t] = items[R * G + t];
    int pos = R * G, piece = 0;
    for (int t = 0; t < m; ++t) {
      const int4 it = tail[t];
      // pieces of at least kMinPiece key tiles: a piece pays a Q load, a pipeline fill and drain and an
      // fp32 round trip, which short items do not recover (measured: d = 128, 12-tile items -4%)
      const int nkt = it.w, si = max(1, min(s, nkt / kMinPiece)), c = (nkt + si - 1) / si, p = (nkt + c - 1) / c;
      if (p <= 1) {
        items[pos++] = it;
        continue;
      }
      map[nsplit++] = make_int4(it.x, it.y, it.z, piece | (p << 16));
      for (int q = 0; q < p; ++q, ++piece) {
        const int kb = q * c;
        items[pos++] = make_int4(it.x | ((piece + 1) << 16), it.y, it.z | (kb << 16), min(c, nkt - kb));
      }
    }
    *n_items = pos;
  }
  *n_split = nsplit;
}

__global__ void __launch_bounds__(kSchedThreads)
build_worklist_kernel(int kind, int B, int H, int Nq, int Nk, const int32_t* __restrict__ seqlens_q,
                      const int32_t* __restrict__ seqlens_k, int4* __restrict__ items, int* __restrict__ n_items,
                      int split_grid, int4* __restrict__ split_map, int* __restrict__ n_split) {
  extern __shared__ int sh[];
  build_worklist_block(kind, B, H, Nq, Nk, seqlens_q, seqlens_k, items, n_items, sh);
  if (kind == 2 && split_grid > 0) split_tail_block(split_grid, items, n_items, split_map, n_split);
}


// Backward prologue, one launch: CTA 0 builds the backward work list while CTAs 1.. zero the fp32
// dQ accumulator on valid query rows [0, n_q[b]).  Padded accumulator rows are never read (the
// finaliser writes zeros there).
__global__ void __launch_bounds__(kSchedThreads)
bwd_prep_kernel(int B, int H, int Nq, int Nk, int D, const int32_t* __restrict__ seqlens_q,
                const int32_t* __restrict__ seqlens_k, int4* __restrict__ items, int* __restrict__ n_items,
                float* __restrict__ dq_acc, float* __restrict__ dbias) {
  extern __shared__ int sh[];
  if (blockIdx.x == 0) {
    if (dbias)
      for (int i = threadIdx.x; i < B; i += blockDim.x) dbias[i] = 0.f;
    build_worklist_block(1, B, H, Nq, Nk, seqlens_q, seqlens_k, items, n_items, sh);
    return;
  }
  const int nblk = gridDim.x - 1, blk = blockIdx.x - 1;
  if (!dq_acc) return;
  // (b, h) slabs split into kParts pieces each; pieces strided over the zeroing CTAs
  constexpr int kParts = 8;
  const int vec_per_row = D / 4;
  const float4 z = make_float4(0.f, 0.f, 0.f, 0.f);
  for (int task = blk; task < B * H * kParts; task += nblk) {
    const int zh = task / kParts, part = task % kParts;
    const int n = clamp_len(seqlens_q, zh / H, Nq);
    const long long total = (long long)n * vec_per_row;
    const long long lo = total * part / kParts, hi = total * (part + 1) / kParts;
    float4* base = reinterpret_cast<float4*>(dq_acc + (size_t)zh * Nq * D);
    for (long long i = lo + threadIdx.x; i < hi; i += blockDim.x) base[i] = z;
  }
}

// Element offset of row `row` of the (b, h) slab of a [B, H, N, D] (bshd = 0) or [B, N, H, D]
// (bshd = 1, the paper's [Z, L, H, D] layout) tensor.
__device__ __forceinline__ size_t row_off(int bshd, int H, int N, int D, int b, int h, int row) {
  return bshd ? ((size_t)((size_t)b * N + row) * H + h) * D : ((size_t)((size_t)b * H + h) * N + row) * D;
}

// One warp zeroes, for every (b, h) slab it is given, rows [r0, r1) of a [B, H, N, row] (or, with
// bshd, [B, N, H, row]) tensor of row_bytes-long rows.
//   pad_rows = 1: r1 = N; r0 = 0 when the sequence has no work item (n_own == 0 or n_other == 0),
//                 else min(ceil_gran(n_own), N) -- the rows below r0 are written (padded rows as
//                 zeros) by the tile epilogues.
//   pad_rows = 0 (SIGATTN_F_NO_ZERO_PAD_OUT: padded rows are left as they are): only the VALID rows
//                 no epilogue writes, [0, n_own) of a sequence with n_other == 0 -- an empty key (or
//                 query) set gives exact-zero valid outputs (empty sums, Eq. 2).
// The rows of every slab are spread over all workers -- the grid's CTAs times the `nworkers` idle
// warps of each persistent attention CTA (worker `k` of this CTA) -- in round-robin 512-byte blocks,
// so a batch whose padding sits in a few long sequences (C3: 74% padding) is zeroed evenly by every
// SM alongside the main work instead of by the few CTAs that own those slabs.
__device__ __forceinline__ void pad_fill_warp(void* out, int row_bytes, int B, int H, int N,
                                              const int32_t* __restrict__ lens_own,
                                              const int32_t* __restrict__ lens_other, int N_other, int gran,
                                              uint32_t lane, int bshd = 0, int pad_rows = 1, int k = 0,
                                              int nworkers = 1) {
  const uint4 z = make_uint4(0, 0, 0, 0);
  const int cpr = row_bytes / 16;   // 16-byte chunks per row
  const long long W = (long long)gridDim.x * nworkers, w = (long long)blockIdx.x * nworkers + k;
  // The 16-byte chunks to zero, concatenated over the slabs in (b, h) order, are cut into 512-byte
  // blocks dealt round-robin to the W workers.  A step covers 32 slabs, one per lane: lengths loaded
  // in parallel, chunk counts prefix-summed across the warp, and each lane tests whether this
  // worker owns a block reaching into its slab; the warp then stores only into those slabs.  (A walk
  // over every slab by every worker cost ~100 clk per slab: 60-140 us past the main work at
  // B H = 512-1024.)  Rows are a power of two of chunks, so no division in the store loop.
  const int lg = __ffs(cpr) - 1;
  long long run = 0;   // chunks of the earlier steps
  for (int zh0 = 0; zh0 < B * H; zh0 += 32) {
    const int zl = zh0 + (int)lane;
    int r0 = 0, r1 = 0;
    if (zl < B * H) {
      const int b = zl / H;
      const int n = clamp_len(lens_own, b, N), m = clamp_len(lens_other, b, N_other);
      if (pad_rows) {
        r0 = (n == 0 || m == 0) ? 0 : min((n + gran - 1) / gran * gran, N);
        r1 = N;
      } else {
        r0 = 0;
        r1 = m == 0 ? n : 0;
      }
      r1 = max(r1, r0);
    }
    const long long c = (long long)(r1 - r0) << lg;
    long long incl = c;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const long long v = __shfl_up_sync(0xffffffffu, incl, o);
      if ((int)lane >= o) incl += v;
    }
    const long long lo = run + incl - c, hi = run + incl;   // this lane's slab: global chunks [lo, hi)
    const long long b0 = lo >> 5;
    const long long bw = b0 + ((w - b0 % W) % W + W) % W;   // this worker's first block at or after b0
    unsigned todo = __ballot_sync(0xffffffffu, c > 0 && (bw << 5) < hi);
    while (todo) {
      const int sl = __ffs(todo) - 1;
      todo &= todo - 1;
      const long long slo = __shfl_sync(0xffffffffu, lo, sl), shi = __shfl_sync(0xffffffffu, hi, sl);
      const long long sbw = __shfl_sync(0xffffffffu, bw, sl);
      const int a0 = __shfl_sync(0xffffffffu, r0, sl);
      const int zh = zh0 + sl, b = zh / H, h = zh - b * H;
      uint8_t* slab = reinterpret_cast<uint8_t*>(out) +
                      (bshd ? ((size_t)b * N * H + h) * row_bytes : ((size_t)zh * N + a0) * row_bytes);
      for (long long blk = sbw; (blk << 5) < shi; blk += W) {
        const long long g = (blk << 5) + lane;
        if (g >= slo && g < shi) {
          const long long i = g - slo;
          if (!bshd) reinterpret_cast<uint4*>(slab)[i] = z;
          else reinterpret_cast<uint4*>(slab + ((size_t)(a0 + (i >> lg)) * H) * row_bytes)[i & (cpr - 1)] = z;
        }
      }
    }
    run = __shfl_sync(0xffffffffu, hi, 31);
  }
}

// SIGATTN_F_SANITIZE_PAD: zero rows [n, min(ceil128(n), N)) of one (b, h) slab per CTA of a 16-bit
// [B, H, N, D] (or [B, N, H, D]) tensor -- the padded rows that share a tile with valid rows.
__global__ void sanitize_pad_kernel(void* t, int H, int N, int D, const int32_t* __restrict__ lens, int bshd) {
  const int zh = blockIdx.x, b = zh / H, h = zh % H;
  const int n = clamp_len(lens, b, N);
  const int r1 = min((n + 127) / 128 * 128, N);
  const int cpr = D * 2 / 16;   // 16-byte chunks per row
  uint16_t* base = reinterpret_cast<uint16_t*>(t);
  for (int i = threadIdx.x; i < (r1 - n) * cpr; i += blockDim.x) {
    const int r = n + i / cpr, c = i % cpr;
    reinterpret_cast<uint4*>(base + row_off(bshd, H, N, D, b, h, r))[c] = make_uint4(0, 0, 0, 0);
  }
}

// Warp-cooperative dQ finalisation of rows [r0, r1) of one (b, h) slab:
// dq[r] = r < n_q ? round(acc[r]) : 0.  (acc rows are read through L2, ld.global.cg.)
template <bool kBf16>
__device__ __forceinline__ void dq_finalize_rows(const float* __restrict__ acc, uint16_t* __restrict__ dq, int D,
                                                 int r0, int r1, int nq, uint32_t lane, size_t dq_rs) {
  const int v8 = D / 8;
  const long long total = (long long)(r1 - r0) * v8;
  for (long long i = lane; i < total; i += 32) {
    const int r = r0 + (int)(i / v8);
    const long long e = (long long)r * D + (i % v8) * 8;
    uint4 w = make_uint4(0, 0, 0, 0);
    if (r < nq) {
      const float4 a = __ldcg(reinterpret_cast<const float4*>(acc + e));
      const float4 c = __ldcg(reinterpret_cast<const float4*>(acc + e) + 1);
      if constexpr (kBf16) {
        asm("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(w.x) : "f"(a.y), "f"(a.x));
        asm("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(w.y) : "f"(a.w), "f"(a.z));
        asm("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(w.z) : "f"(c.y), "f"(c.x));
        asm("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(w.w) : "f"(c.w), "f"(c.z));
      } else {
        asm("cvt.rn.f16x2.f32 %0, %1, %2;" : "=r"(w.x) : "f"(a.y), "f"(a.x));
        asm("cvt.rn.f16x2.f32 %0, %1, %2;" : "=r"(w.y) : "f"(a.w), "f"(a.z));
        asm("cvt.rn.f16x2.f32 %0, %1, %2;" : "=r"(w.z) : "f"(c.y), "f"(c.x));
        asm("cvt.rn.f16x2.f32 %0, %1, %2;" : "=r"(w.w) : "f"(c.w), "f"(c.z));
      }
    }
    *reinterpret_cast<uint4*>(dq + (size_t)r * dq_rs + (i % v8) * 8) = w;
  }
}

// dQ finalisation, launched after the backward (finalising inside it needs a gpu-scope fence per
// query tile to publish the red.global.add contributions; measured 2.7 ms -> 6.5 ms on C3):
// dq[b,h,i,:] = i < n_q[b] ? round(acc[b,h,i,:]) : 0    (acc already holds alpha * dS K)
template <bool kBf16>
__global__ void dq_finalize_kernel(const float* __restrict__ acc, uint16_t* __restrict__ dq, int H, int N, int D,
                                   const int32_t* __restrict__ lens, const int32_t* __restrict__ lens_k, int Nk,
                                   int bshd, int pad_rows) {
  const int zh = blockIdx.y;
  const int nq = clamp_len(lens, zh / H, N), nk = clamp_len(lens_k, zh / H, Nk);
  // rows from ceil128(n_q) on (all rows if the sequence has no work) are zeroed by the backward
  // kernel's fill warp; finalise the rest
  // (pad_rows = 0, SIGATTN_F_NO_ZERO_PAD_OUT: the valid rows only)
  const int rlim = (nq == 0 || nk == 0) ? 0 : (pad_rows ? min((nq + 127) & ~127, N) : nq);
  const int rows = (rlim + gridDim.x - 1) / gridDim.x;
  const int r0 = blockIdx.x * rows, r1 = min(rlim, r0 + rows);
  const int warp = threadIdx.x >> 5, nwarps = blockDim.x >> 5;
  const int per = (r1 - r0 + nwarps - 1) / nwarps;
  const int w0 = r0 + warp * per, w1 = min(r1, w0 + per);
  if (w0 < w1)
    dq_finalize_rows<kBf16>(acc + (size_t)zh * N * D, dq + row_off(bshd, H, N, D, zh / H, zh % H, 0), D, w0, w1, nq,
                            threadIdx.x & 31, bshd ? (size_t)H * D : (size_t)D);
}


// Context-parallel finalize: rank `rank`'s fp32 accumulator [B, H, rows, D] (the sum over every
// rank's key block, A4 P:121) -> out [B, H, rows, D] 16-bit; local row r is global query row
// rank * rows + r and is written as exact 0 when that row is padded (>= n_q[b]).
template <bool kBf16>
__global__ void cp_finalize_kernel(const float* __restrict__ acc, uint16_t* __restrict__ out, int H, int rows, int D,
                                   int Nq, const int32_t* __restrict__ lens, int rank) {
  const int zh = blockIdx.y;
  const int nq = clamp_len(lens, zh / H, Nq);
  const int nloc = max(0, min(rows, nq - rank * rows));   // valid rows of this block
  const int per = (rows + gridDim.x - 1) / gridDim.x;
  const int r0 = blockIdx.x * per, r1 = min(rows, r0 + per);
  const int warp = threadIdx.x >> 5, nwarps = blockDim.x >> 5;
  const int wper = (r1 - r0 + nwarps - 1) / nwarps;
  const int w0 = r0 + warp * wper, w1 = min(r1, w0 + wper);
  if (w0 < w1)
    dq_finalize_rows<kBf16>(acc + (size_t)zh * rows * D, out + (size_t)zh * rows * D, D, w0, w1, nloc,
                            threadIdx.x & 31, (size_t)D);
}


// Context-parallel push: this rank's complete fp32 partial acc [B, H, Nq, D] (summed over its key
// tiles) -> reduce-added into the owners' accumulators peer[g] [B, H, rows, D] (g = row / rows),
// valid rows only; each warp covers whole 256/512-byte rows (coalesced, one float4 per lane).  Ends
// with a system-scope fence so the adds are performed before the kernel completes.
__global__ void cp_push_kernel(const float* __restrict__ acc, float* const* __restrict__ peer, int rows, int H,
                               int Nq, int D, const int32_t* __restrict__ lens) {
  const int zh = blockIdx.y;
  const int nq = clamp_len(lens, zh / H, Nq);
  const int v4 = D / 4;   // float4 per row
  const long long total = (long long)nq * v4;
  const float4* src = reinterpret_cast<const float4*>(acc + (size_t)zh * Nq * D);
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < total; i += (long long)gridDim.x * blockDim.x) {
    const int r = (int)(i / v4), c = (int)(i % v4);
    const int owner = r / rows, lr = r - owner * rows;
    const float4 a = __ldcg(src + i);
    sm100::red_add_v4_sys(peer[owner] + ((size_t)zh * rows + lr) * D + c * 4, a.x, a.y, a.z, a.w);
  }
  sm100::fence_sys();
}

// General (non-prefix) key_padding_mask [B, N] (1 = pad) -> a stable compaction per sequence:
// index[b, r] = position of the r-th valid token for r < n_b, then of the (r - n_b)-th padded one;
// seqlens[b] = n_b.  One CTA of 1024 threads per sequence; chunks of 1024 positions scanned with
// warp ballots.  Attention is equivariant under a joint permutation of the queries and keys of a
// sequence, so compacting, attending with prefix lengths and scattering back is exact.
__global__ void __launch_bounds__(1024) mask_to_index_kernel(const uint8_t* __restrict__ mask, int N,
                                                             int32_t* __restrict__ index,
                                                             int32_t* __restrict__ seqlens) {
  const int b = blockIdx.x, warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  __shared__ int s_warp[32];
  __shared__ int s_total;
  // pass 1: number of valid tokens
  int valid = 0;
  for (int i = threadIdx.x; i < N; i += blockDim.x) valid += mask[(size_t)b * N + i] == 0;
  for (int o = 16; o > 0; o >>= 1) valid += __shfl_xor_sync(0xffffffffu, valid, o);
  if (lane == 0) s_warp[warp] = valid;
  __syncthreads();
  if (threadIdx.x == 0) {
    int t = 0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += s_warp[w];
    s_total = t;
    seqlens[b] = t;
  }
  __syncthreads();
  const int n = s_total;
  int base_v = 0, base_p = 0;   // valid / padded tokens before this chunk
  for (int c0 = 0; c0 < N; c0 += blockDim.x) {
    const int i = c0 + threadIdx.x;
    const bool in = i < N;
    const bool v = in && mask[(size_t)b * N + i] == 0;
    const unsigned bv = __ballot_sync(0xffffffffu, v), bp = __ballot_sync(0xffffffffu, in && !v);
    __syncthreads();
    if (lane == 0) s_warp[warp] = __popc(bv) | (__popc(bp) << 16);
    __syncthreads();
    int pv = 0, pp = 0;
    for (int w = 0; w < warp; ++w) {
      pv += s_warp[w] & 0xffff;
      pp += s_warp[w] >> 16;
    }
    const unsigned lt = (1u << lane) - 1u;
    if (v) index[(size_t)b * N + base_v + pv + __popc(bv & lt)] = i;
    else if (in) index[(size_t)b * N + n + base_p + pp + __popc(bp & lt)] = i;
    int tv = 0, tp = 0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) {
      tv += s_warp[w] & 0xffff;
      tp += s_warp[w] >> 16;
    }
    base_v += tv;
    base_p += tp;
  }
}

// Row gather / scatter of a [B, H, N, D] 16-bit tensor along N by index [B, N]:
// scatter = 0: dst[b, h, r] = src[b, h, index[b, r]];  scatter = 1: dst[b, h, index[b, r]] = src[b, h, r].
// Grid (B*H, ceil(N / 8)), 128 threads: 8 rows per CTA, 16-byte chunks.
__global__ void permute_rows_kernel(const uint16_t* __restrict__ src, uint16_t* __restrict__ dst,
                                    const int32_t* __restrict__ index, int H, int N, int D, int scatter) {
  const int zh = blockIdx.x, b = zh / H;
  const int cpr = D / 8;
  const size_t slab = (size_t)zh * N * D;
  for (int i = threadIdx.x; i < 8 * cpr; i += blockDim.x) {
    const int r = blockIdx.y * 8 + i / cpr, c = i % cpr;
    if (r >= N) continue;
    const int j = index[(size_t)b * N + r];
    const int rs = scatter ? r : j, rd = scatter ? j : r;
    reinterpret_cast<uint4*>(dst + slab + (size_t)rd * D)[c] = reinterpret_cast<const uint4*>(src + slab + (size_t)rs * D)[c];
  }
}

// key_padding_mask [B, N] (1 = pad) -> seqlens[b] = number of valid tokens; flags non-prefix masks.
__global__ void mask_to_seqlens_kernel(const uint8_t* __restrict__ mask, int N, int32_t* __restrict__ seqlens,
                                       int32_t* __restrict__ nonprefix) {
  const int b = blockIdx.x;
  int valid = 0, first_pad = N;
  for (int i = threadIdx.x; i < N; i += blockDim.x) {
    const bool pad = mask[(size_t)b * N + i] != 0;
    valid += pad ? 0 : 1;
    if (pad && i < first_pad) first_pad = i;
  }
  for (int o = 16; o > 0; o >>= 1) {
    valid += __shfl_xor_sync(0xffffffffu, valid, o);
    first_pad = min(first_pad, __shfl_xor_sync(0xffffffffu, first_pad, o));
  }
  __shared__ int s_valid[32], s_first[32];
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  if (l == 0) { s_valid[w] = valid; s_first[w] = first_pad; }
  __syncthreads();
  if (threadIdx.x == 0) {
    int v = 0, f = N;
    for (int i = 0; i < (int)(blockDim.x + 31) / 32; ++i) { v += s_valid[i]; f = min(f, s_first[i]); }
    seqlens[b] = v;
    if (v != f) atomicExch(nonprefix, 1);
  }
}

// Sum of the pieces of every split item (split_tail_block) -> the 16-bit O rows of its two query
// tiles (rows >= n_q exact 0).  One CTA per split slot; acc: [pieces][2 tiles][128][D] fp32.
template <bool kBf16>
__global__ void fwd_split_finalize_kernel(const float* __restrict__ acc, const int4* __restrict__ map,
                                          const int* __restrict__ n_split, uint16_t* __restrict__ out, int H, int Nq,
                                          int D, const int32_t* __restrict__ lens, int bshd) {
  const int slot = blockIdx.x;
  if (slot >= *n_split) return;
  const int4 mp = map[slot];
  const int b = mp.x & 0xFFFF, h = mp.y, pi = mp.z & 0xFFFF, first = mp.w & 0xFFFF, np = mp.w >> 16;
  const int nq = clamp_len(lens, b, Nq);
  const int v8 = D / 8;
  for (int i = threadIdx.x; i < 2 * 128 * v8; i += blockDim.x) {
    const int x = i / (128 * v8), r = (i / v8) % 128, c = (i % v8) * 8;
    const int qrow = (2 * pi + x) * 128 + r;
    if (qrow >= Nq) continue;
    float a[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
    if (qrow < nq)
      for (int p = 0; p < np; ++p) {
        const float4* src = reinterpret_cast<const float4*>(acc + ((size_t)((first + p) * 2 + x) * 128 + r) * D + c);
        const float4 u = __ldcg(src), w = __ldcg(src + 1);
        a[0] += u.x; a[1] += u.y; a[2] += u.z; a[3] += u.w;
        a[4] += w.x; a[5] += w.y; a[6] += w.z; a[7] += w.w;
      }
    uint4 o;
    o.x = sm100::pack2<kBf16>(a[0], a[1]);
    o.y = sm100::pack2<kBf16>(a[2], a[3]);
    o.z = sm100::pack2<kBf16>(a[4], a[5]);
    o.w = sm100::pack2<kBf16>(a[6], a[7]);
    *reinterpret_cast<uint4*>(out + row_off(bshd, H, Nq, D, b, h, qrow) + c) = o;
  }
}

}  // namespace sigattn
