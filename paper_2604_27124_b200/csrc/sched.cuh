// sched.cuh -- small device kernels around the two attention kernels:
//   * the work-list builder (padded-tile skipping + longest-first order),
//   * padded-row zero fill, dQ-accumulator zeroing and dQ finalisation,
//   * key-padding-mask -> valid lengths conversion.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace sigattn {

constexpr int kSchedThreads = 1024;
constexpr int kMaxSchedB = 4096;      // sequences per batch the single-block builder supports

__device__ __forceinline__ int clamp_len(const int32_t* lens, int b, int N) {
  int n = lens ? lens[b] : N;
  return n < 0 ? 0 : (n > N ? N : n);
}

// Work items: kind 0 (forward)  -> (b, h, q-tile) for q-tiles holding a valid query, cost = key tiles
//             kind 1 (backward) -> (b, h, k-tile) for k-tiles holding a valid key,  cost = query tiles
// Items with cost 0 are not emitted (their outputs are all padding and are zero-filled).
// Order: sequences by cost descending (ties: b ascending); within a sequence h-major, tile-minor.
// Single CTA; B <= kMaxSchedB.  Shared memory: 4 * B ints.
__global__ void __launch_bounds__(kSchedThreads)
build_worklist_kernel(int kind, int B, int H, int Nq, int Nk, const int32_t* __restrict__ seqlens_q,
                      const int32_t* __restrict__ seqlens_k, int4* __restrict__ items, int* __restrict__ n_items) {
  extern __shared__ int sh[];
  int* cost = sh;           // [B]
  int* ntile = sh + B;      // [B]
  int* order = sh + 2 * B;  // [B] rank -> b
  int* offs = sh + 3 * B;   // [B] rank -> first item
  for (int b = threadIdx.x; b < B; b += blockDim.x) {
    const int nq = clamp_len(seqlens_q, b, Nq);
    const int nk = clamp_len(seqlens_k, b, Nk);
    const int tq = (nq + 127) / 128, tk = (nk + 127) / 128;
    int c = kind == 0 ? tk : tq;
    int t = kind == 0 ? tq : tk;
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
    *n_items = acc;
  }
  __syncthreads();
  for (int r = threadIdx.x; r < B; r += blockDim.x) {
    const int b = order[r];
    const int nt = ntile[b], c = cost[b];
    int base = offs[r];
    for (int h = 0; h < H; ++h)
      for (int t = 0; t < nt; ++t) items[base++] = make_int4(b, h, t, c);
  }
}

// Zero rows of a [B, H, N, row_elems] tensor.  mode 0: rows [n_b, N) where n_b = lens[b], or all
// rows if gate[b] == 0 (the other side has no valid token);  mode 1: rows [0, n_b).
// row_bytes must be a multiple of 16.
__global__ void zero_rows_kernel(void* __restrict__ out, int row_bytes, int B, int H, int N,
                                 const int32_t* __restrict__ lens, const int32_t* __restrict__ gate,
                                 int gate_N, int mode) {
  const int zh = blockIdx.y;
  const int b = zh / H;
  const int n = clamp_len(lens, b, N);
  int lo, hi;
  if (mode == 0) {
    const bool all = gate_N >= 0 && clamp_len(gate, b, gate_N) == 0;
    lo = all ? 0 : n;
    hi = N;
  } else {
    lo = 0;
    hi = n;
  }
  if (hi <= lo) return;
  const int vec_per_row = row_bytes / 16;
  const long long total = (long long)(hi - lo) * vec_per_row;
  uint4* base = reinterpret_cast<uint4*>(reinterpret_cast<uint8_t*>(out) + ((size_t)zh * N + lo) * row_bytes);
  const uint4 z = make_uint4(0, 0, 0, 0);
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += (long long)gridDim.x * blockDim.x)
    base[i] = z;
}

// dq[b,h,i,:] = i < n_q[b] ? round(ws[b,h,i,:]) : 0    (ws already holds alpha * dS K)
template <bool kBf16>
__global__ void dq_finalize_kernel(const float* __restrict__ ws, uint16_t* __restrict__ dq, int H, int N, int D,
                                   const int32_t* __restrict__ lens, long long total8) {
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < total8; i += (long long)gridDim.x * blockDim.x) {
    const long long e = i * 8;
    const long long row = e / D;
    const int r = (int)(row % N);
    const int b = (int)(row / N / H);
    const bool valid = r < clamp_len(lens, b, N);
    uint4 w = make_uint4(0, 0, 0, 0);
    if (valid) {
      const float4 a = reinterpret_cast<const float4*>(ws + e)[0];
      const float4 c = reinterpret_cast<const float4*>(ws + e)[1];
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
    reinterpret_cast<uint4*>(dq + e)[0] = w;
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

}  // namespace sigattn
