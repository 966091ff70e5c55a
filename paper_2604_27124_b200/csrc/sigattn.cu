// sigattn.cu -- C-ABI host side of libsigattn.so (declared in include/sigattn.h).
// Validation, TMA descriptor encoding, workspace layout and kernel launches.  No computation of
// the method happens on the host; every step runs in the kernels of fwd.cuh / bwd.cuh / sched.cuh.
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>
#include <cstring>
#include <atomic>
#include <map>
#include <mutex>
#include <string>
#include <vector>

#include "../../include/sigattn.h"
#include "bwd.cuh"
#include "bwd128.cuh"
#include "dq.cuh"
#include "fwd2.cuh"

// Forward kernel per head dimension: two query tiles per CTA (fwd2.cuh) at d = 128 -- 1.55x the
// one-tile kernel on C2 at N=16K (1195 vs 773 TFLOPS) -- and the one-tile kernel with alternating
// key tiles (fwd.cuh) at d = 64, where it is 12% faster (741 vs 650 TFLOPS, sigma-bound).
#ifndef SIGATTN_FWD2_MIN_D
#define SIGATTN_FWD2_MIN_D 128
#endif
constexpr bool use_fwd2(int d) { return d >= SIGATTN_FWD2_MIN_D; }
// work-list kind of the forward: pairs of query tiles (2) or single query tiles (0)
constexpr int fwd_item_kind(int d) { return use_fwd2(d) ? 2 : 0; }
#include "fwd.cuh"
#include "sched.cuh"

using namespace sigattn;

namespace {

thread_local std::string g_err;

// Key-split context parallelism with the reduction fused into the kernels' epilogues: the device
// table of every rank's fp32 accumulator and the rows each rank owns (Nq / world).
struct CpTarget {
  float* const* peer;
  int rows;
};
std::atomic<long long> g_launches{0};
thread_local cudaEvent_t g_prof[4] = {nullptr, nullptr, nullptr, nullptr};
thread_local long long* g_trace = nullptr;
thread_local unsigned long long* g_counters = nullptr;

void count_launch(int n = 1) { g_launches.fetch_add(n, std::memory_order_relaxed); }

void prof_record(int idx, cudaStream_t s) {
  if (g_prof[idx]) cudaEventRecord(g_prof[idx], s);
}

sigattn_status fail(sigattn_status s, const std::string& msg) {
  g_err = msg;
  return s;
}

#define CUDA_TRY(expr)                                                                        \
  do {                                                                                        \
    cudaError_t e_ = (expr);                                                                  \
    if (e_ != cudaSuccess)                                                                    \
      return fail(SIGATTN_ECUDA, std::string(#expr) + ": " + cudaGetErrorString(e_));         \
  } while (0)

// cuTensorMapEncodeTiled through the runtime's driver entry point (no -lcuda link dependency).
typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiledFn get_encode() {
  static EncodeTiledFn fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeTiledFn>(p);
  });
  return fn;
}

// [B, H, rows, d] tensor: 3-D view {d (inner), rows, B H}.  With bshd, the paper's [B, rows, H, d]
// layout: 4-D view {d, rows, H, B}.  Box {64 elements = 128 B, box_rows, 1(, 1)}, 128-byte
// swizzle: exactly the UMMA K-major / MN-major SWIZZLE_128B atom whichever the layout.  Rows past
// `rows` read as zero (OOB fill), so a ragged last tile never touches another head's or sequence's data.
sigattn_status encode_tmap(CUtensorMap* m, const void* ptr, CUtensorMapDataType dt, int elem_bytes, int d, int rows,
                           int B, int H, bool bshd, int box_rows) {
  EncodeTiledFn enc = get_encode();
  if (!enc) return fail(SIGATTN_ECUDA, "cuTensorMapEncodeTiled unavailable (driver too old?)");
  const cuuint64_t e = (cuuint64_t)elem_bytes, dd = (cuuint64_t)d, n = (cuuint64_t)rows, hh = (cuuint64_t)H;
  cuuint64_t dims[4] = {dd, n, bshd ? hh : hh * (cuuint64_t)B, (cuuint64_t)B};
  cuuint64_t strides[3] = {bshd ? hh * dd * e : dd * e,    // next row
                           bshd ? dd * e : n * dd * e,     // next head ((b, h) slab without bshd)
                           n * hh * dd * e};               // next sequence (bshd only)
  cuuint32_t box[4] = {(cuuint32_t)(128 / elem_bytes), (cuuint32_t)box_rows, 1, 1};
  cuuint32_t estr[4] = {1, 1, 1, 1};
  CUresult r = enc(m, dt, bshd ? 4 : 3, const_cast<void*>(ptr), dims, strides, box, estr,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(SIGATTN_ECUDA, "cuTensorMapEncodeTiled failed: " + std::to_string((int)r));
  return SIGATTN_OK;
}

// Small cache of encoded tensor maps keyed by (pointer, geometry): a training loop calls the
// library with the same buffers step after step, and encoding 3-5 maps per call costs host time
// on the launch path.  The map is a pure function of its key (it holds no other state), so a hit
// is exactly the map encode_tmap would produce.  Bounded: kTmapCacheSize entries, replaced round
// robin; guarded by a mutex (calls are reentrant).
struct TmapKey {
  const void* ptr;
  int dt, elem_bytes, d, rows, B, H, bshd, box_rows;
  bool operator==(const TmapKey& o) const {
    return ptr == o.ptr && dt == o.dt && elem_bytes == o.elem_bytes && d == o.d && rows == o.rows && B == o.B &&
           H == o.H && bshd == o.bshd && box_rows == o.box_rows;
  }
};
constexpr int kTmapCacheSize = 64;

sigattn_status make_tmap(CUtensorMap* m, const void* ptr, CUtensorMapDataType dt, int elem_bytes, int d, int rows,
                         int B, int H, bool bshd, int box_rows = 128) {
  static std::mutex mu;
  static TmapKey keys[kTmapCacheSize];
  static CUtensorMap maps[kTmapCacheSize];
  static int used = 0, next = 0;
  const TmapKey key{ptr, (int)dt, elem_bytes, d, rows, B, H, bshd ? 1 : 0, box_rows};
  {
    std::lock_guard<std::mutex> lock(mu);
    for (int i = 0; i < used; ++i)
      if (keys[i] == key) {
        *m = maps[i];
        return SIGATTN_OK;
      }
  }
  sigattn_status st = encode_tmap(m, ptr, dt, elem_bytes, d, rows, B, H, bshd, box_rows);
  if (st != SIGATTN_OK) return st;
  std::lock_guard<std::mutex> lock(mu);
  const int slot = used < kTmapCacheSize ? used++ : (next++ % kTmapCacheSize);
  keys[slot] = key;
  maps[slot] = *m;
  return SIGATTN_OK;
}

bool layout_bshd(const sigattn_params* p) { return (p->flags & SIGATTN_F_LAYOUT_BSHD) != 0; }

int num_sms() {
  int dev = 0, n = 148;
  if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
  return n;
}

bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; }

int cdiv(long long a, long long b) { return (int)((a + b - 1) / b); }

sigattn_status check_params(const sigattn_params* p) {
  if (!p) return fail(SIGATTN_EINVAL, "params is NULL");
  if (p->B <= 0 || p->H <= 0 || p->Nq <= 0 || p->Nk <= 0)
    return fail(SIGATTN_EINVAL, "B, H, Nq, Nk must be positive");
  if (p->d != 64 && p->d != 128) return fail(SIGATTN_EINVAL, "d must be 64 or 128");
  if (p->dtype != SIGATTN_BF16 && p->dtype != SIGATTN_FP16) return fail(SIGATTN_EINVAL, "dtype must be bf16 or fp16");
  if (p->B > kMaxSchedB) return fail(SIGATTN_EUNSUPPORTED, "B > 4096 sequences per call");
  const long long bh = (long long)p->B * p->H;
  if (bh > 65535) return fail(SIGATTN_EUNSUPPORTED, "B*H > 65535");
  if (bh * std::max(p->Nq, p->Nk) * (long long)p->d >= (1ll << 40)) return fail(SIGATTN_EINVAL, "tensor too large");
  if (!(p->scale == p->scale)) return fail(SIGATTN_EINVAL, "scale is NaN");
  return SIGATTN_OK;
}

// cudaFuncSetAttribute once per (kernel, device, size): it is a host call on every launch path otherwise.
template <typename K>
sigattn_status set_smem(K kernel, int bytes) {
  static std::mutex mu;
  static std::vector<std::pair<const void*, std::pair<int, int>>> done;
  int dev = 0;
  CUDA_TRY(cudaGetDevice(&dev));
  const void* key = reinterpret_cast<const void*>(kernel);
  {
    std::lock_guard<std::mutex> lock(mu);
    for (auto& e : done)
      if (e.first == key && e.second.first == dev && e.second.second >= bytes) return SIGATTN_OK;
  }
  CUDA_TRY(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes));
  std::lock_guard<std::mutex> lock(mu);
  done.push_back({key, {dev, bytes}});
  return SIGATTN_OK;
}

int sched_smem(const sigattn_params* p) { return (4 * p->B + 1) * (int)sizeof(int); }

// split_grid > 0 (kind 2): cut the last round's items along their key range (split_tail_block)
sigattn_status launch_worklist(int kind, const sigattn_params* p, int4* items, int* n_items, cudaStream_t s,
                               int split_grid = 0, int4* split_map = nullptr, int* n_split = nullptr) {
  const int smem = sched_smem(p);
  if (smem > 48 * 1024) {
    sigattn_status st = set_smem(build_worklist_kernel, (4 * kMaxSchedB + 1) * (int)sizeof(int));
    if (st != SIGATTN_OK) return st;
  }
  build_worklist_kernel<<<1, kSchedThreads, smem, s>>>(kind, p->B, p->H, p->Nq, p->Nk, p->seqlens_q, p->seqlens_k,
                                                        items, n_items, split_grid, split_map, n_split);
  count_launch();
  CUDA_TRY(cudaGetLastError());
  return SIGATTN_OK;
}

sigattn_status launch_bwd_prep(const sigattn_params* p, int4* items, int* n_items, float* dq_acc, cudaStream_t s) {
  // (also zeroes p->dbias when the bias gradient is requested)
  const int smem = sched_smem(p);
  if (smem > 48 * 1024) {
    sigattn_status st = set_smem(bwd_prep_kernel, (4 * kMaxSchedB + 1) * (int)sizeof(int));
    if (st != SIGATTN_OK) return st;
  }
  const int zero_ctas = dq_acc ? num_sms() : 0;
  bwd_prep_kernel<<<1 + zero_ctas, kSchedThreads, smem, s>>>(p->B, p->H, p->Nq, p->Nk, p->d, p->seqlens_q,
                                                              p->seqlens_k, items, n_items, dq_acc, p->dbias);
  count_launch();
  CUDA_TRY(cudaGetLastError());
  return SIGATTN_OK;
}

template <int D, bool kBf16, bool kF32>
sigattn_status launch_fwd(const sigattn_params* p, const void* q, const void* k, const void* v, void* o,
                          const int4* items, const int* n_items, int max_items, cudaStream_t s,
                          const CpTarget* cp = nullptr, float* split_acc = nullptr) {
  const CUtensorMapDataType dt = kBf16 ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16 : CU_TENSOR_MAP_DATA_TYPE_FLOAT16;
  CUtensorMap tq, tk, tv;
  sigattn_status st;
  if ((st = make_tmap(&tq, q, dt, 2, D, p->Nq, p->B, p->H, layout_bshd(p))) != SIGATTN_OK) return st;
  if ((st = make_tmap(&tk, k, dt, 2, D, p->Nk, p->B, p->H, layout_bshd(p))) != SIGATTN_OK) return st;
  if ((st = make_tmap(&tv, v, dt, 2, D, p->Nk, p->B, p->H, layout_bshd(p))) != SIGATTN_OK) return st;
  FwdArgs a;
  a.items = items;
  a.n_items = n_items;
  a.seqlens_q = p->seqlens_q;
  a.seqlens_k = p->seqlens_k;
  a.bias_per_seq = p->bias_per_seq;
  a.bias = p->bias;
  a.scale = p->scale;
  a.B = p->B;
  a.H = p->H;
  a.Nq = p->Nq;
  a.Nk = p->Nk;
  a.o = o;
  a.fill_pad = (p->flags & SIGATTN_F_NO_ZERO_PAD_OUT) ? 0 : 1;
  a.trace = g_trace;
  a.counters = g_counters;
  a.bshd = layout_bshd(p) ? 1 : 0;
  a.peer_o = cp ? cp->peer : nullptr;
  a.peer_rows = cp ? cp->rows : 0;
  a.split_acc = split_acc;
  const int grid = std::max(1, std::min(num_sms(), max_items));
  if constexpr (use_fwd2(D)) {
    using C = Fwd2Cfg<D>;
    auto kern = sigattn_fwd2_kernel<D, kBf16, kF32>;
    if ((st = set_smem(kern, C::kSmemBytes)) != SIGATTN_OK) return st;
    prof_record(0, s);
    kern<<<grid, C::kThreads, C::kSmemBytes, s>>>(tq, tk, tv, a);
  } else {
    using C = FwdCfg<D>;
    auto kern = sigattn_fwd_kernel<D, kBf16, kF32>;
    if ((st = set_smem(kern, C::kSmemBytes)) != SIGATTN_OK) return st;
    prof_record(0, s);
    kern<<<grid, C::kThreads, C::kSmemBytes, s>>>(tq, tk, tv, a);
  }
  prof_record(1, s);
  count_launch();
  CUDA_TRY(cudaGetLastError());
  return SIGATTN_OK;
}

template <int D, bool kBf16, bool kDQ = true, bool kDB = false>
sigattn_status launch_bwd_t(const sigattn_params* p, const void* q, const void* k, const void* v, const void* dout,
                          float* dq_acc, void* dk, void* dv,
                          const int4* items, const int* n_items, int max_items, cudaStream_t s,
                          void* dq_pad = nullptr) {
  const CUtensorMapDataType dt = kBf16 ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16 : CU_TENSOR_MAP_DATA_TYPE_FLOAT16;
  CUtensorMap tq, tk, tv, tdo;
  sigattn_status st;
  if ((st = make_tmap(&tq, q, dt, 2, D, p->Nq, p->B, p->H, layout_bshd(p))) != SIGATTN_OK) return st;
  if ((st = make_tmap(&tk, k, dt, 2, D, p->Nk, p->B, p->H, layout_bshd(p))) != SIGATTN_OK) return st;
  if ((st = make_tmap(&tv, v, dt, 2, D, p->Nk, p->B, p->H, layout_bshd(p))) != SIGATTN_OK) return st;
  if ((st = make_tmap(&tdo, dout, dt, 2, D, p->Nq, p->B, p->H, layout_bshd(p))) != SIGATTN_OK) return st;
  CUtensorMap tdq;   // fp32 dQ accumulator, 32-column boxes for the TMA reduce-add
  std::memset(&tdq, 0, sizeof(tdq));
  if (kDQ && (st = make_tmap(&tdq, dq_acc, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, D, p->Nq, p->B, p->H, false)) != SIGATTN_OK)
    return st;
  BwdArgs a;
  a.items = items;
  a.n_items = n_items;
  a.seqlens_q = p->seqlens_q;
  a.seqlens_k = p->seqlens_k;
  a.bias_per_seq = p->bias_per_seq;
  a.bias = p->bias;
  a.scale = p->scale;
  a.B = p->B;
  a.H = p->H;
  a.Nq = p->Nq;
  a.Nk = p->Nk;
  a.dq_acc = dq_acc;
  a.dk = dk;
  a.dv = dv;
  a.dq_pad = dq_pad;
  a.fill_pad = (p->flags & SIGATTN_F_NO_ZERO_PAD_OUT) ? 0 : 1;
  a.dbias = p->dbias;
  a.trace = g_trace;
  a.counters = g_counters;
  a.bshd = layout_bshd(p) ? 1 : 0;
  using C = BwdCfg<D>;
  auto kern = layout_bshd(p) ? sigattn_bwd_kernel<D, kBf16, kDQ, kDB, true> : sigattn_bwd_kernel<D, kBf16, kDQ, kDB, false>;
  if ((st = set_smem(kern, C::kSmemBytes)) != SIGATTN_OK) return st;
  const int grid = std::max(1, std::min(num_sms(), max_items));
  prof_record(2, s);
  kern<<<grid, C::kThreads, C::kSmemBytes, s>>>(tq, tk, tv, tdo, tdq, a);
  prof_record(3, s);
  count_launch();
  CUDA_TRY(cudaGetLastError());
  return SIGATTN_OK;
}

template <bool kBf16, bool kDQ = true, bool kDB = false>
sigattn_status launch_bwd128_t(const sigattn_params* p, const void* q, const void* k, const void* v, const void* dout,
                             float* dq_acc, void* dk, void* dv,
                             const int4* items, const int* n_items, int max_items, cudaStream_t s,
                             void* dq_pad = nullptr) {
  const CUtensorMapDataType dt = kBf16 ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16 : CU_TENSOR_MAP_DATA_TYPE_FLOAT16;
  CUtensorMap tq, tk, tv, tdo;
  sigattn_status st;
  if ((st = make_tmap(&tq, q, dt, 2, 128, p->Nq, p->B, p->H, layout_bshd(p), Bwd128Cfg::kQT)) != SIGATTN_OK) return st;
  if ((st = make_tmap(&tk, k, dt, 2, 128, p->Nk, p->B, p->H, layout_bshd(p))) != SIGATTN_OK) return st;
  if ((st = make_tmap(&tv, v, dt, 2, 128, p->Nk, p->B, p->H, layout_bshd(p))) != SIGATTN_OK) return st;
  if ((st = make_tmap(&tdo, dout, dt, 2, 128, p->Nq, p->B, p->H, layout_bshd(p), Bwd128Cfg::kQT)) != SIGATTN_OK) return st;
  CUtensorMap tdq;   // fp32 dQ accumulator [B, H, Nq, 128], 32-column x 64-row boxes for the TMA reduce-add
  std::memset(&tdq, 0, sizeof(tdq));
  if (kDQ && (st = make_tmap(&tdq, dq_acc, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, 128, p->Nq, p->B, p->H, false,
                                    Bwd128Cfg::kQT)) != SIGATTN_OK)
    return st;
  BwdArgs a;
  a.items = items;
  a.n_items = n_items;
  a.seqlens_q = p->seqlens_q;
  a.seqlens_k = p->seqlens_k;
  a.bias_per_seq = p->bias_per_seq;
  a.bias = p->bias;
  a.scale = p->scale;
  a.B = p->B;
  a.H = p->H;
  a.Nq = p->Nq;
  a.Nk = p->Nk;
  a.dq_acc = dq_acc;
  a.dk = dk;
  a.dv = dv;
  a.dq_pad = dq_pad;
  a.fill_pad = (p->flags & SIGATTN_F_NO_ZERO_PAD_OUT) ? 0 : 1;
  a.dbias = p->dbias;
  a.trace = g_trace;
  a.counters = g_counters;
  a.bshd = layout_bshd(p) ? 1 : 0;
  auto kern = layout_bshd(p) ? sigattn_bwd128_kernel<kBf16, kDQ, kDB, true> : sigattn_bwd128_kernel<kBf16, kDQ, kDB, false>;
  if ((st = set_smem(kern, Bwd128Cfg::kSmemBytes)) != SIGATTN_OK) return st;
  const int grid = std::max(1, std::min(num_sms(), max_items));
  prof_record(2, s);
  kern<<<grid, Bwd128Cfg::kThreads, Bwd128Cfg::kSmemBytes, s>>>(tq, tk, tv, tdo, tdq, a);
  prof_record(3, s);
  count_launch();
  CUDA_TRY(cudaGetLastError());
  return SIGATTN_OK;
}

// runtime dispatch of the bias-gradient variant (kDB: the compute warps also sum dS)
template <int D, bool kBf16, bool kDQ = true>
sigattn_status launch_bwd(const sigattn_params* p, const void* q, const void* k, const void* v, const void* dout,
                          float* dq_acc, void* dk, void* dv, const int4* items, const int* n_items, int max_items,
                          cudaStream_t s, void* dq_pad = nullptr) {
  return p->dbias ? launch_bwd_t<D, kBf16, kDQ, true>(p, q, k, v, dout, dq_acc, dk, dv, items, n_items, max_items, s, dq_pad)
                  : launch_bwd_t<D, kBf16, kDQ, false>(p, q, k, v, dout, dq_acc, dk, dv, items, n_items, max_items, s, dq_pad);
}
template <bool kBf16, bool kDQ = true>
sigattn_status launch_bwd128(const sigattn_params* p, const void* q, const void* k, const void* v, const void* dout,
                             float* dq_acc, void* dk, void* dv, const int4* items, const int* n_items, int max_items,
                             cudaStream_t s, void* dq_pad = nullptr) {
  return p->dbias ? launch_bwd128_t<kBf16, kDQ, true>(p, q, k, v, dout, dq_acc, dk, dv, items, n_items, max_items, s, dq_pad)
                  : launch_bwd128_t<kBf16, kDQ, false>(p, q, k, v, dout, dq_acc, dk, dv, items, n_items, max_items, s, dq_pad);
}

template <int D, bool kBf16, bool kF32>
sigattn_status launch_dq(const sigattn_params* p, const void* q, const void* k, const void* v, const void* dout,
                         void* dq, const int4* items, const int* n_items, int max_items, cudaStream_t s) {
  const CUtensorMapDataType dt = kBf16 ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16 : CU_TENSOR_MAP_DATA_TYPE_FLOAT16;
  CUtensorMap tq, tk, tv, tdo;
  sigattn_status st;
  if ((st = make_tmap(&tq, q, dt, 2, D, p->Nq, p->B, p->H, layout_bshd(p))) != SIGATTN_OK) return st;
  if ((st = make_tmap(&tk, k, dt, 2, D, p->Nk, p->B, p->H, layout_bshd(p))) != SIGATTN_OK) return st;
  if ((st = make_tmap(&tv, v, dt, 2, D, p->Nk, p->B, p->H, layout_bshd(p))) != SIGATTN_OK) return st;
  if ((st = make_tmap(&tdo, dout, dt, 2, D, p->Nq, p->B, p->H, layout_bshd(p))) != SIGATTN_OK) return st;
  DqArgs a;
  a.items = items;
  a.n_items = n_items;
  a.seqlens_q = p->seqlens_q;
  a.seqlens_k = p->seqlens_k;
  a.bias_per_seq = p->bias_per_seq;
  a.bias = p->bias;
  a.scale = p->scale;
  a.B = p->B;
  a.H = p->H;
  a.Nq = p->Nq;
  a.Nk = p->Nk;
  a.dq = dq;
  a.bshd = layout_bshd(p) ? 1 : 0;
  a.counters = g_counters;
  a.fill_pad = (p->flags & SIGATTN_F_NO_ZERO_PAD_OUT) ? 0 : 1;
  using C = DqCfg<D>;
  auto kern = layout_bshd(p) ? sigattn_dq_kernel<D, kBf16, kF32, true> : sigattn_dq_kernel<D, kBf16, kF32, false>;
  if ((st = set_smem(kern, C::kSmemBytes)) != SIGATTN_OK) return st;
  const int grid = std::max(1, std::min(num_sms(), max_items));
  kern<<<grid, C::kThreads, C::kSmemBytes, s>>>(tq, tk, tv, tdo, a);
  count_launch();
  CUDA_TRY(cudaGetLastError());
  return SIGATTN_OK;
}

// SIGATTN_F_SANITIZE_PAD: zero the padded rows inside each sequence's last valid tile, in place.
sigattn_status sanitize_pad(const sigattn_params* p, const void* t, int N, const int32_t* lens, cudaStream_t s) {
  if (!(p->flags & SIGATTN_F_SANITIZE_PAD) || !lens) return SIGATTN_OK;
  sanitize_pad_kernel<<<p->B * p->H, 128, 0, s>>>(const_cast<void*>(t), p->H, N, p->d, lens, layout_bshd(p) ? 1 : 0);
  count_launch();
  CUDA_TRY(cudaGetLastError());
  return SIGATTN_OK;
}

size_t align_up(size_t x, size_t a) { return (x + a - 1) / a * a; }

size_t ws_acc_bytes(const sigattn_params* p) { return align_up((size_t)p->B * p->H * p->Nq * p->d * sizeof(float), 256); }
size_t ws_items_bytes(const sigattn_params* p) {
  return align_up(16 + (size_t)p->B * p->H * cdiv(p->Nk, 128) * sizeof(int4), 256);
}
size_t ws_items_q_bytes(const sigattn_params* p) {   // query-tile work list (deterministic dQ pass)
  return align_up(16 + (size_t)p->B * p->H * cdiv(p->Nq, 128) * sizeof(int4), 256);
}
// Forward workspace: {count, split count, pad} + items (+ grid spare entries for the pieces of a
// tail split), then, for the two-tile forward, the split map [grid] and the fp32 piece buffer
// [grid][2][128][d] (split_tail_block).
int fwd_split_grid(const sigattn_params* p) { return use_fwd2(p->d) ? num_sms() : 0; }
size_t ws_fwd_items_bytes(const sigattn_params* p) {
  return align_up(16 + ((size_t)p->B * p->H * cdiv(p->Nq, 128) + fwd_split_grid(p)) * sizeof(int4), 256);
}
size_t ws_fwd_bytes(const sigattn_params* p) {
  const size_t G = (size_t)fwd_split_grid(p);
  return ws_fwd_items_bytes(p) + align_up(G * sizeof(int4), 256) + G * 2 * 128 * p->d * sizeof(float);
}

}  // namespace

extern "C" {

const char* sigattn_last_error(void) { return g_err.c_str(); }

int64_t sigattn_launch_count(void) { return g_launches.load(); }

void sigattn_set_trace_buffer(void* device_buffer) { g_trace = reinterpret_cast<long long*>(device_buffer); }
void sigattn_set_debug_counters(void* device_counters) {
  g_counters = reinterpret_cast<unsigned long long*>(device_counters);
}

void sigattn_set_profile_events(void* fwd_start, void* fwd_stop, void* bwd_start, void* bwd_stop) {
  g_prof[0] = reinterpret_cast<cudaEvent_t>(fwd_start);
  g_prof[1] = reinterpret_cast<cudaEvent_t>(fwd_stop);
  g_prof[2] = reinterpret_cast<cudaEvent_t>(bwd_start);
  g_prof[3] = reinterpret_cast<cudaEvent_t>(bwd_stop);
}

const char* sigattn_version(void) { return "sigattn-b200 0.1 (sm_100a tcgen05/TMEM/TMA)"; }

int64_t sigattn_valid_flops(int B, int H, int d, const int32_t* host_nq, const int32_t* host_nk, int forward) {
  if (B <= 0 || H <= 0 || d <= 0 || !host_nq || !host_nk) return -1;
  const int64_t c = forward ? 4 : 10;  // App. B.1: fwd 4 b h n^2 d, bwd 2.5x
  int64_t s = 0;
  for (int b = 0; b < B; ++b) {
    if (host_nq[b] < 0 || host_nk[b] < 0) return -1;
    s += (int64_t)host_nq[b] * (int64_t)host_nk[b];
  }
  return c * (int64_t)H * (int64_t)d * s;
}

int64_t sigattn_worklist_host(int kind, int B, int H, int Nq, int Nk, const int32_t* host_nq, const int32_t* host_nk,
                              int32_t* items, int64_t max_items) {
  if (kind < 0 || kind > 2 || B <= 0 || H <= 0 || Nq <= 0 || Nk <= 0) return -1;
  std::vector<int> cost(B), nt(B), order(B);
  for (int b = 0; b < B; ++b) {
    int nq = host_nq ? host_nq[b] : Nq, nk = host_nk ? host_nk[b] : Nk;
    nq = std::min(std::max(nq, 0), Nq);
    nk = std::min(std::max(nk, 0), Nk);
    const int tq = (nq + 127) / 128, tk = (nk + 127) / 128;
    cost[b] = kind == 1 ? tq : tk;
    nt[b] = cost[b] == 0 ? 0 : (kind == 0 ? tq : (kind == 1 ? tk : (tq + 1) / 2));
    order[b] = b;
  }
  std::stable_sort(order.begin(), order.end(), [&](int x, int y) { return cost[x] > cost[y]; });
  int64_t n = 0;
  for (int r = 0; r < B; ++r) {
    const int b = order[r];
    for (int h = 0; h < H; ++h)
      for (int t = 0; t < nt[b]; ++t, ++n)
        if (items && n < max_items) {
          items[4 * n + 0] = b;
          items[4 * n + 1] = h;
          items[4 * n + 2] = t;
          items[4 * n + 3] = cost[b];
        }
  }
  return n;
}

size_t sigattn_fwd_workspace_bytes(const sigattn_params* p) {
  if (check_params(p) != SIGATTN_OK) return 0;
  return ws_fwd_bytes(p);
}

sigattn_status sigattn_fwd(const sigattn_params* p, const void* q, const void* k, const void* v, void* o,
                           void* workspace, size_t workspace_bytes, void* stream) {
  sigattn_status st = check_params(p);
  if (st != SIGATTN_OK) return st;
  if (!q || !k || !v || !o || !workspace) return fail(SIGATTN_EINVAL, "null pointer");
  if (!aligned16(q) || !aligned16(k) || !aligned16(v) || !aligned16(o) || !aligned16(workspace))
    return fail(SIGATTN_EINVAL, "pointers must be 16-byte aligned");
  if (workspace_bytes < ws_fwd_bytes(p))
    return fail(SIGATTN_EWORKSPACE, "workspace too small: need " + std::to_string(ws_fwd_bytes(p)) + " bytes");
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  {   // every host-detectable error is reported above, before anything is launched
    const int32_t* lk = p->seqlens_k;   // NULL: all keys valid
    if ((st = sanitize_pad(p, q, p->Nq, p->seqlens_q, s)) != SIGATTN_OK) return st;
    if ((st = sanitize_pad(p, k, p->Nk, lk, s)) != SIGATTN_OK) return st;
    if ((st = sanitize_pad(p, v, p->Nk, lk, s)) != SIGATTN_OK) return st;
  }
  const bool f32 = (p->flags & SIGATTN_F_OUT_F32_PARTIAL) != 0;
  const int max_items = p->B * p->H * cdiv(p->Nq, 128);
  uint8_t* ws = reinterpret_cast<uint8_t*>(workspace);
  int* n_items = reinterpret_cast<int*>(ws);
  int* n_split = n_items + 1;
  int4* items = reinterpret_cast<int4*>(ws + 16);
  // tail split: the two-tile forward with 16-bit output (fp32 partials keep whole items)
  const int G = f32 ? 0 : fwd_split_grid(p);
  int4* split_map = reinterpret_cast<int4*>(ws + ws_fwd_items_bytes(p));
  float* split_acc = G ? reinterpret_cast<float*>(ws + ws_fwd_items_bytes(p) + align_up((size_t)G * sizeof(int4), 256))
                       : nullptr;
  st = launch_worklist(fwd_item_kind(p->d), p, items, n_items, s, G, split_map, n_split);
  if (st == SIGATTN_OK) {
    const bool bf = p->dtype == SIGATTN_BF16;
    if (p->d == 64) {
      if (bf) st = f32 ? launch_fwd<64, true, true>(p, q, k, v, o, items, n_items, max_items, s)
                       : launch_fwd<64, true, false>(p, q, k, v, o, items, n_items, max_items, s);
      else st = f32 ? launch_fwd<64, false, true>(p, q, k, v, o, items, n_items, max_items, s)
                    : launch_fwd<64, false, false>(p, q, k, v, o, items, n_items, max_items, s);
    } else {
      if (bf) st = f32 ? launch_fwd<128, true, true>(p, q, k, v, o, items, n_items, max_items, s)
                       : launch_fwd<128, true, false>(p, q, k, v, o, items, n_items, max_items, s, nullptr, split_acc);
      else st = f32 ? launch_fwd<128, false, true>(p, q, k, v, o, items, n_items, max_items, s)
                    : launch_fwd<128, false, false>(p, q, k, v, o, items, n_items, max_items, s, nullptr, split_acc);
    }
  }
  if (st == SIGATTN_OK && G) {   // sum the pieces of the split tail items into their O rows
    if (p->dtype == SIGATTN_BF16)
      fwd_split_finalize_kernel<true><<<G, 256, 0, s>>>(split_acc, split_map, n_split, reinterpret_cast<uint16_t*>(o),
                                                        p->H, p->Nq, p->d, p->seqlens_q, layout_bshd(p) ? 1 : 0);
    else
      fwd_split_finalize_kernel<false><<<G, 256, 0, s>>>(split_acc, split_map, n_split, reinterpret_cast<uint16_t*>(o),
                                                         p->H, p->Nq, p->d, p->seqlens_q, layout_bshd(p) ? 1 : 0);
    count_launch();
    CUDA_TRY(cudaGetLastError());
  }
  return st;
}

// Workspace: fp32 dQ accumulator | work list (256-B aligned parts).

size_t sigattn_bwd_workspace_bytes(const sigattn_params* p) {
  if (check_params(p) != SIGATTN_OK) return 0;
  if (p->flags & SIGATTN_F_BWD_DETERMINISTIC) return ws_items_bytes(p) + ws_items_q_bytes(p);
  return ws_acc_bytes(p) + ws_items_bytes(p);
}

sigattn_status sigattn_bwd(const sigattn_params* p, const void* q, const void* k, const void* v, const void* dout,
                           void* dq, void* dk, void* dv, void* workspace, size_t workspace_bytes, void* stream) {
  sigattn_status st = check_params(p);
  if (st != SIGATTN_OK) return st;
  if (!q || !k || !v || !dout || !dq || !dk || !dv || !workspace) return fail(SIGATTN_EINVAL, "null pointer");
  if (!aligned16(q) || !aligned16(k) || !aligned16(v) || !aligned16(dout) || !aligned16(dq) || !aligned16(dk) ||
      !aligned16(dv) || !aligned16(workspace))
    return fail(SIGATTN_EINVAL, "pointers must be 16-byte aligned");
  const size_t need = sigattn_bwd_workspace_bytes(p);
  if (workspace_bytes < need)
    return fail(SIGATTN_EWORKSPACE, "workspace too small: need " + std::to_string(need) + " bytes");
  const bool dq_f32 = (p->flags & SIGATTN_F_DQ_F32_PARTIAL) != 0;
  if (dq_f32 && layout_bshd(p))
    return fail(SIGATTN_EUNSUPPORTED, "SIGATTN_F_DQ_F32_PARTIAL needs the [B, H, N, d] layout");
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  {   // every host-detectable error is reported above, before anything is launched
    const int32_t* lk = p->seqlens_k;   // NULL: all keys valid
    if ((st = sanitize_pad(p, q, p->Nq, p->seqlens_q, s)) != SIGATTN_OK) return st;
    if ((st = sanitize_pad(p, dout, p->Nq, p->seqlens_q, s)) != SIGATTN_OK) return st;
    if ((st = sanitize_pad(p, k, p->Nk, lk, s)) != SIGATTN_OK) return st;
    if ((st = sanitize_pad(p, v, p->Nk, lk, s)) != SIGATTN_OK) return st;
  }
  uint8_t* ws = reinterpret_cast<uint8_t*>(workspace);
  const bool bf = p->dtype == SIGATTN_BF16;
  if (p->flags & SIGATTN_F_BWD_DETERMINISTIC) {
    // Alg. 3 (dK, dV; key-tile-owned) then Alg. 2 (dQ; query-tile-owned) -- no atomics anywhere
    int* n_items = reinterpret_cast<int*>(ws);
    int4* items = reinterpret_cast<int4*>(ws + 16);
    int* nq_items = reinterpret_cast<int*>(ws + ws_items_bytes(p));
    int4* q_items = reinterpret_cast<int4*>(ws + ws_items_bytes(p) + 16);
    if ((st = launch_bwd_prep(p, items, n_items, nullptr, s)) != SIGATTN_OK) return st;
    const int max_items = p->B * p->H * cdiv(p->Nk, 128);
    if (p->d == 64)
      st = bf ? launch_bwd<64, true, false>(p, q, k, v, dout, nullptr, dk, dv, items, n_items, max_items, s)
              : launch_bwd<64, false, false>(p, q, k, v, dout, nullptr, dk, dv, items, n_items, max_items, s);
    else
      st = bf ? launch_bwd128<true, false>(p, q, k, v, dout, nullptr, dk, dv, items, n_items, max_items, s)
              : launch_bwd128<false, false>(p, q, k, v, dout, nullptr, dk, dv, items, n_items, max_items, s);
    if (st != SIGATTN_OK) return st;
    if ((st = launch_worklist(0, p, q_items, nq_items, s)) != SIGATTN_OK) return st;
    const int max_q_items = p->B * p->H * cdiv(p->Nq, 128);
    if (p->d == 64) {
      if (bf) st = dq_f32 ? launch_dq<64, true, true>(p, q, k, v, dout, dq, q_items, nq_items, max_q_items, s)
                          : launch_dq<64, true, false>(p, q, k, v, dout, dq, q_items, nq_items, max_q_items, s);
      else st = dq_f32 ? launch_dq<64, false, true>(p, q, k, v, dout, dq, q_items, nq_items, max_q_items, s)
                       : launch_dq<64, false, false>(p, q, k, v, dout, dq, q_items, nq_items, max_q_items, s);
    } else {
      if (bf) st = dq_f32 ? launch_dq<128, true, true>(p, q, k, v, dout, dq, q_items, nq_items, max_q_items, s)
                          : launch_dq<128, true, false>(p, q, k, v, dout, dq, q_items, nq_items, max_q_items, s);
      else st = dq_f32 ? launch_dq<128, false, true>(p, q, k, v, dout, dq, q_items, nq_items, max_q_items, s)
                       : launch_dq<128, false, false>(p, q, k, v, dout, dq, q_items, nq_items, max_q_items, s);
    }
    return st;
  }
  const size_t acc_bytes = ws_acc_bytes(p);
  float* dq_acc = dq_f32 ? reinterpret_cast<float*>(dq) : reinterpret_cast<float*>(ws);
  int* n_items = reinterpret_cast<int*>(ws + acc_bytes);
  int4* items = reinterpret_cast<int4*>(ws + acc_bytes + 16);
  const int max_items = p->B * p->H * cdiv(p->Nk, 128);
  // fp32 dQ output (context-parallel partials): plain zero-init, the kernel accumulates into it
  if (dq_f32) CUDA_TRY(cudaMemsetAsync(dq, 0, (size_t)p->B * p->H * p->Nq * p->d * sizeof(float), s));
  if ((st = launch_bwd_prep(p, items, n_items, dq_f32 ? nullptr : dq_acc, s)) != SIGATTN_OK)
    return st;
  void* dq_pad = dq_f32 ? nullptr : dq;   // 16-bit dQ: the kernel's fill warp zeroes rows >= ceil128(n_q)
  if (p->d == 64)
    st = bf ? launch_bwd<64, true>(p, q, k, v, dout, dq_acc, dk, dv, items, n_items, max_items, s, dq_pad)
            : launch_bwd<64, false>(p, q, k, v, dout, dq_acc, dk, dv, items, n_items, max_items, s, dq_pad);
  else
    st = bf ? launch_bwd128<true>(p, q, k, v, dout, dq_acc, dk, dv, items, n_items, max_items, s, dq_pad)
            : launch_bwd128<false>(p, q, k, v, dout, dq_acc, dk, dv, items, n_items, max_items, s, dq_pad);
  if (st != SIGATTN_OK || dq_f32) return st;
  const dim3 grid(std::max(1, std::min(32, cdiv(p->Nq, 512))), p->B * p->H);
  if (bf)
    dq_finalize_kernel<true><<<grid, 256, 0, s>>>(dq_acc, reinterpret_cast<uint16_t*>(dq), p->H, p->Nq, p->d,
                                                  p->seqlens_q, p->seqlens_k, p->Nk, layout_bshd(p) ? 1 : 0,
                                                  (p->flags & SIGATTN_F_NO_ZERO_PAD_OUT) ? 0 : 1);
  else
    dq_finalize_kernel<false><<<grid, 256, 0, s>>>(dq_acc, reinterpret_cast<uint16_t*>(dq), p->H, p->Nq, p->d,
                                                   p->seqlens_q, p->seqlens_k, p->Nk, layout_bshd(p) ? 1 : 0,
                                                  (p->flags & SIGATTN_F_NO_ZERO_PAD_OUT) ? 0 : 1);
  count_launch();
  CUDA_TRY(cudaGetLastError());
  return SIGATTN_OK;
}

sigattn_status sigattn_mask_to_index(const uint8_t* key_padding_mask, int B, int N, int32_t* index,
                                     int32_t* seqlens, void* stream) {
  if (!key_padding_mask || !index || !seqlens || B <= 0 || N <= 0 || N > 65535)
    return fail(SIGATTN_EINVAL, "bad mask_to_index arguments");
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  mask_to_index_kernel<<<B, 1024, 0, s>>>(key_padding_mask, N, index, seqlens);
  count_launch();
  CUDA_TRY(cudaGetLastError());
  return SIGATTN_OK;
}

sigattn_status sigattn_permute_rows(const void* src, void* dst, const int32_t* index, int B, int H, int N, int d,
                                    int scatter, void* stream) {
  if (!src || !dst || !index || src == dst || B <= 0 || H <= 0 || N <= 0 || (d != 64 && d != 128))
    return fail(SIGATTN_EINVAL, "bad permute_rows arguments");
  if (!aligned16(src) || !aligned16(dst)) return fail(SIGATTN_EINVAL, "tensor pointers must be 16-byte aligned");
  if ((long long)B * H > 65535 * 1024ll) return fail(SIGATTN_EUNSUPPORTED, "B*H too large");
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  const dim3 grid(B * H, (N + 7) / 8);
  permute_rows_kernel<<<grid, 128, 0, s>>>(reinterpret_cast<const uint16_t*>(src), reinterpret_cast<uint16_t*>(dst),
                                           index, H, N, d, scatter);
  count_launch();
  CUDA_TRY(cudaGetLastError());
  return SIGATTN_OK;
}

sigattn_status sigattn_copy_valid_rows(const void* src, void* dst, int B, int H, int N, int row_bytes,
                                       const int32_t* host_lens, int layout_bshd, int kind, void* stream,
                                       int64_t* bytes_out) {
  if (!src || !dst || !host_lens || B <= 0 || H <= 0 || N <= 0 || row_bytes <= 0 || row_bytes % 16 != 0 ||
      kind < 1 || kind > 3)
    return fail(SIGATTN_EINVAL, "bad copy_valid_rows arguments");
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  const cudaMemcpyKind k = static_cast<cudaMemcpyKind>(kind);
  const size_t rb = (size_t)row_bytes, slab = (size_t)N * rb;
  int64_t bytes = 0;
  for (int b = 0; b < B; ++b) {
    const int n = std::min(std::max(host_lens[b], 0), N);
    if (n == 0) continue;
    if (layout_bshd) {   // sequence b: rows [0, n) of all heads are one block of n * H rows
      const size_t off = (size_t)b * N * H * rb, len = (size_t)n * H * rb;
      CUDA_TRY(cudaMemcpyAsync(static_cast<uint8_t*>(dst) + off, static_cast<const uint8_t*>(src) + off, len, k, s));
      bytes += (int64_t)len;
    } else {             // H slabs of N rows: n rows each, pitch N rows
      const size_t off = (size_t)b * H * slab;
      CUDA_TRY(cudaMemcpy2DAsync(static_cast<uint8_t*>(dst) + off, slab, static_cast<const uint8_t*>(src) + off, slab,
                                 (size_t)n * rb, (size_t)H, k, s));
      bytes += (int64_t)n * H * (int64_t)rb;
    }
  }
  if (bytes_out) *bytes_out = bytes;
  return SIGATTN_OK;
}

sigattn_status sigattn_mask_to_seqlens(const uint8_t* key_padding_mask, int B, int N, int32_t* seqlens,
                                       int32_t* nonprefix_flag, void* stream) {
  if (!key_padding_mask || !seqlens || !nonprefix_flag || B <= 0 || N <= 0)
    return fail(SIGATTN_EINVAL, "bad mask_to_seqlens arguments");
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  CUDA_TRY(cudaMemsetAsync(nonprefix_flag, 0, sizeof(int32_t), s));
  mask_to_seqlens_kernel<<<B, 256, 0, s>>>(key_padding_mask, N, seqlens, nonprefix_flag);
  count_launch();
  CUDA_TRY(cudaGetLastError());
  return SIGATTN_OK;
}

}  // extern "C"

// ------------------------------------------------------------------ key-split context parallelism
// with the partial-sum reduction fused into the kernels (A4)

namespace {
sigattn_status check_cp(const sigattn_params* p, const sigattn_cp_params* cp) {
  if (!cp || cp->world < 1 || cp->rank < 0 || cp->rank >= cp->world || !cp->peer_acc)
    return fail(SIGATTN_EINVAL, "bad sigattn_cp_params");
  if (p->Nq % cp->world) return fail(SIGATTN_EINVAL, "context parallelism needs Nq divisible by world");
  if (layout_bshd(p)) return fail(SIGATTN_EUNSUPPORTED, "context parallelism needs the [B, H, N, d] layout");
  if (!aligned16(cp->peer_acc)) return fail(SIGATTN_EINVAL, "peer_acc must be 16-byte aligned");
  return SIGATTN_OK;
}
}  // namespace

extern "C" {

size_t sigattn_bwd_cp_workspace_bytes(const sigattn_params* p) {
  if (check_params(p) != SIGATTN_OK) return 0;
  return ws_acc_bytes(p) + ws_items_bytes(p);
}

sigattn_status sigattn_fwd_cp(const sigattn_params* p, const sigattn_cp_params* cp, const void* q, const void* k,
                              const void* v, void* workspace, size_t workspace_bytes, void* stream) {
  sigattn_status st = check_params(p);
  if (st != SIGATTN_OK) return st;
  if ((st = check_cp(p, cp)) != SIGATTN_OK) return st;
  if (!q || !k || !v || !workspace) return fail(SIGATTN_EINVAL, "null pointer");
  if (!aligned16(q) || !aligned16(k) || !aligned16(v) || !aligned16(workspace))
    return fail(SIGATTN_EINVAL, "pointers must be 16-byte aligned");
  if (workspace_bytes < ws_fwd_bytes(p))
    return fail(SIGATTN_EWORKSPACE, "workspace too small: need " + std::to_string(ws_fwd_bytes(p)) + " bytes");
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  if ((st = sanitize_pad(p, q, p->Nq, p->seqlens_q, s)) != SIGATTN_OK) return st;
  if ((st = sanitize_pad(p, k, p->Nk, p->seqlens_k, s)) != SIGATTN_OK) return st;
  if ((st = sanitize_pad(p, v, p->Nk, p->seqlens_k, s)) != SIGATTN_OK) return st;
  const CpTarget t{cp->peer_acc, p->Nq / cp->world};
  const int max_items = p->B * p->H * cdiv(p->Nq, 128);
  int* n_items = reinterpret_cast<int*>(workspace);
  int4* items = reinterpret_cast<int4*>(reinterpret_cast<uint8_t*>(workspace) + 16);
  if ((st = launch_worklist(fwd_item_kind(p->d), p, items, n_items, s)) != SIGATTN_OK) return st;
  const bool bf = p->dtype == SIGATTN_BF16;
  if (p->d == 64)
    return bf ? launch_fwd<64, true, true>(p, q, k, v, nullptr, items, n_items, max_items, s, &t)
              : launch_fwd<64, false, true>(p, q, k, v, nullptr, items, n_items, max_items, s, &t);
  return bf ? launch_fwd<128, true, true>(p, q, k, v, nullptr, items, n_items, max_items, s, &t)
            : launch_fwd<128, false, true>(p, q, k, v, nullptr, items, n_items, max_items, s, &t);
}

sigattn_status sigattn_bwd_cp(const sigattn_params* p, const sigattn_cp_params* cp, const void* q, const void* k,
                              const void* v, const void* dout, void* dk, void* dv, void* workspace,
                              size_t workspace_bytes, void* stream) {
  sigattn_status st = check_params(p);
  if (st != SIGATTN_OK) return st;
  if ((st = check_cp(p, cp)) != SIGATTN_OK) return st;
  if (p->flags & SIGATTN_F_BWD_DETERMINISTIC)
    return fail(SIGATTN_EUNSUPPORTED, "the fused context-parallel backward has no deterministic mode");
  if (!q || !k || !v || !dout || !dk || !dv || !workspace) return fail(SIGATTN_EINVAL, "null pointer");
  if (!aligned16(q) || !aligned16(k) || !aligned16(v) || !aligned16(dout) || !aligned16(dk) || !aligned16(dv) ||
      !aligned16(workspace))
    return fail(SIGATTN_EINVAL, "pointers must be 16-byte aligned");
  const size_t need = ws_acc_bytes(p) + ws_items_bytes(p);
  if (workspace_bytes < need)
    return fail(SIGATTN_EWORKSPACE, "workspace too small: need " + std::to_string(need) + " bytes");
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  if ((st = sanitize_pad(p, q, p->Nq, p->seqlens_q, s)) != SIGATTN_OK) return st;
  if ((st = sanitize_pad(p, dout, p->Nq, p->seqlens_q, s)) != SIGATTN_OK) return st;
  if ((st = sanitize_pad(p, k, p->Nk, p->seqlens_k, s)) != SIGATTN_OK) return st;
  if ((st = sanitize_pad(p, v, p->Nk, p->seqlens_k, s)) != SIGATTN_OK) return st;
  // dQ over this rank's keys accumulates in the local fp32 workspace (TMA reduce-adds in L2: every key
  // tile adds a partial, so sending those over NVLink would multiply the traffic by the key-tile
  // count), then one push kernel reduce-adds each valid row into its owner: the same bytes as a
  // reduce-scatter, issued by our kernel over peer memory.
  uint8_t* ws = reinterpret_cast<uint8_t*>(workspace);
  float* dq_acc = reinterpret_cast<float*>(ws);
  int* n_items = reinterpret_cast<int*>(ws + ws_acc_bytes(p));
  int4* items = reinterpret_cast<int4*>(ws + ws_acc_bytes(p) + 16);
  const int max_items = p->B * p->H * cdiv(p->Nk, 128);
  if ((st = launch_bwd_prep(p, items, n_items, dq_acc, s)) != SIGATTN_OK) return st;
  const bool bf = p->dtype == SIGATTN_BF16;
  if (p->d == 64)
    st = bf ? launch_bwd<64, true>(p, q, k, v, dout, dq_acc, dk, dv, items, n_items, max_items, s)
            : launch_bwd<64, false>(p, q, k, v, dout, dq_acc, dk, dv, items, n_items, max_items, s);
  else
    st = bf ? launch_bwd128<true>(p, q, k, v, dout, dq_acc, dk, dv, items, n_items, max_items, s)
            : launch_bwd128<false>(p, q, k, v, dout, dq_acc, dk, dv, items, n_items, max_items, s);
  if (st != SIGATTN_OK) return st;
  const int rows = p->Nq / cp->world;
  const dim3 grid(std::max(1, std::min(64, cdiv(p->Nq, 256))), p->B * p->H);
  cp_push_kernel<<<grid, 256, 0, s>>>(dq_acc, cp->peer_acc, rows, p->H, p->Nq, p->d, p->seqlens_q);
  count_launch();
  CUDA_TRY(cudaGetLastError());
  return SIGATTN_OK;
}

sigattn_status sigattn_cp_finalize(const sigattn_params* p, int world, int rank, const float* acc, void* out,
                                   void* stream) {
  sigattn_status st = check_params(p);
  if (st != SIGATTN_OK) return st;
  if (world < 1 || rank < 0 || rank >= world || p->Nq % world) return fail(SIGATTN_EINVAL, "bad world / rank");
  if (!acc || !out) return fail(SIGATTN_EINVAL, "null pointer");
  if (!aligned16(acc) || !aligned16(out)) return fail(SIGATTN_EINVAL, "pointers must be 16-byte aligned");
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  const int rows = p->Nq / world;
  const dim3 grid(std::max(1, std::min(32, cdiv(rows, 512))), p->B * p->H);
  if (p->dtype == SIGATTN_BF16)
    cp_finalize_kernel<true><<<grid, 256, 0, s>>>(acc, reinterpret_cast<uint16_t*>(out), p->H, rows, p->d, p->Nq,
                                                  p->seqlens_q, rank);
  else
    cp_finalize_kernel<false><<<grid, 256, 0, s>>>(acc, reinterpret_cast<uint16_t*>(out), p->H, rows, p->d, p->Nq,
                                                   p->seqlens_q, rank);
  count_launch();
  CUDA_TRY(cudaGetLastError());
  return SIGATTN_OK;
}

// CUDA IPC: a handle is the cudaIpcMemHandle_t of the allocation containing the pointer, followed by
// the pointer's byte offset in it (int64), so interior pointers of a caching allocator's blocks work.
namespace {
std::mutex g_ipc_mu;
std::map<void*, void*> g_ipc_bases;   // imported pointer -> mapped allocation base
}  // namespace

size_t sigattn_ipc_handle_bytes(void) { return sizeof(cudaIpcMemHandle_t) + sizeof(int64_t); }

sigattn_status sigattn_ipc_export(const void* dev_ptr, void* handle) {
  if (!dev_ptr || !handle) return fail(SIGATTN_EINVAL, "null pointer");
  CUdeviceptr base = 0;
  size_t size = 0;
  {
    cudaPointerAttributes attr;
    CUDA_TRY(cudaPointerGetAttributes(&attr, dev_ptr));
    if (attr.type != cudaMemoryTypeDevice) return fail(SIGATTN_EINVAL, "ipc export needs device memory");
  }
  void* fn = nullptr;
  cudaDriverEntryPointQueryResult q;
  CUDA_TRY(cudaGetDriverEntryPoint("cuMemGetAddressRange", &fn, cudaEnableDefault, &q));
  if (!fn) return fail(SIGATTN_ECUDA, "cuMemGetAddressRange unavailable");
  using F = CUresult (*)(CUdeviceptr*, size_t*, CUdeviceptr);
  if (reinterpret_cast<F>(fn)(&base, &size, reinterpret_cast<CUdeviceptr>(dev_ptr)) != CUDA_SUCCESS)
    return fail(SIGATTN_ECUDA, "cuMemGetAddressRange failed");
  cudaIpcMemHandle_t h;
  CUDA_TRY(cudaIpcGetMemHandle(&h, reinterpret_cast<void*>(base)));
  const int64_t off = (int64_t)(reinterpret_cast<CUdeviceptr>(dev_ptr) - base);
  std::memcpy(handle, &h, sizeof(h));
  std::memcpy(reinterpret_cast<uint8_t*>(handle) + sizeof(h), &off, sizeof(off));
  return SIGATTN_OK;
}

sigattn_status sigattn_ipc_import(const void* handle, void** dev_ptr) {
  if (!handle || !dev_ptr) return fail(SIGATTN_EINVAL, "null pointer");
  cudaIpcMemHandle_t h;
  int64_t off;
  std::memcpy(&h, handle, sizeof(h));
  std::memcpy(&off, reinterpret_cast<const uint8_t*>(handle) + sizeof(h), sizeof(off));
  void* base = nullptr;
  CUDA_TRY(cudaIpcOpenMemHandle(&base, h, cudaIpcMemLazyEnablePeerAccess));
  *dev_ptr = reinterpret_cast<uint8_t*>(base) + off;
  std::lock_guard<std::mutex> lk(g_ipc_mu);
  g_ipc_bases[*dev_ptr] = base;
  return SIGATTN_OK;
}

sigattn_status sigattn_ipc_close(void* dev_ptr) {
  void* base = nullptr;
  {
    std::lock_guard<std::mutex> lk(g_ipc_mu);
    auto it = g_ipc_bases.find(dev_ptr);
    if (it == g_ipc_bases.end()) return fail(SIGATTN_EINVAL, "pointer was not imported by sigattn_ipc_import");
    base = it->second;
    g_ipc_bases.erase(it);
  }
  CUDA_TRY(cudaIpcCloseMemHandle(base));
  return SIGATTN_OK;
}

}  // extern "C"
