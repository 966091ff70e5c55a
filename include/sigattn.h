/*
 * sigattn.h -- C ABI of libsigattn.so: padding-aware bidirectional sigmoid attention on B200
 * (sm_100a), forward and backward.
 *
 * Operation (Eq. 2; Alg. 1-3):
 *   O     = sigma(alpha * Q K^T + b) V                    per (batch z, head h)
 *   P_ij  = sigma(alpha <q_i,k_j> + b_z) if i < n_q[z] and j < n_k[z], else 0   (Alg. 1)
 *   dV    = P^T dO                                        (Alg. 3)
 *   dS    = P (1 - P) (dO V^T)                            (Alg. 2; diagonal Jacobian P:358-365)
 *   dQ    = alpha dS K,   dK = alpha dS^T Q               (Alg. 2; Alg. 3)
 *   Rows i >= n_q[z] of O and dQ, and rows j >= n_k[z] of dK and dV, are written as exact 0
 *   (P:593).
 *
 * Conventions shared by every entry point:
 *   - Tensors are [B, H, N, d] contiguous (row-major), N = Nq for Q, O, dO, dQ and N = Nk for
 *     K, V, dK, dV.  d in {64, 128}.  Element type bf16 or fp16 (sigattn_dtype).  All tensor
 *     pointers are DEVICE pointers, 16-byte aligned, owned by the caller; the library never
 *     frees or retains them beyond the call's stream work.
 *   - seqlens_q / seqlens_k are DEVICE int32 [B] valid lengths (validity is a prefix).
 *     NULL means "all valid".  Values are clamped to [0, N] on the device; n = 0 gives all-zero
 *     rows.  Pad CONTENT must be finite (a tensor core computes 0 * NaN = NaN); with finite pad
 *     the outputs are independent of it.
 *   - All calls are asynchronous on `stream` (a cudaStream_t passed as void*; NULL = legacy
 *     default stream).  No host synchronisation happens inside a call.  The library allocates no
 *     device memory: every buffer, workspaces included, is the caller's.  Calls are reentrant
 *     and may run concurrently from several host threads (internal host caches -- encoded TMA
 *     descriptors, kernel attributes -- are mutex-guarded); two calls in flight at once must not
 *     share a workspace unless they are ordered on one stream.  Calls are CUDA-graph capturable
 *     (no allocation, no synchronisation, no host reads of device data).
 *   - Errors: a status code is returned and no exception crosses the ABI.  Host-detectable
 *     argument errors return SIGATTN_EINVAL before anything is launched; launch failures return
 *     SIGATTN_ECUDA.  sigattn_last_error() gives a thread-local message for the last failure.
 */
#ifndef SIGATTN_H_
#define SIGATTN_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum { SIGATTN_BF16 = 0, SIGATTN_FP16 = 1 } sigattn_dtype;

typedef enum {
  SIGATTN_OK = 0,
  SIGATTN_EINVAL = 1,        /* bad argument (shape, dtype, alignment, null pointer, ws size) */
  SIGATTN_EUNSUPPORTED = 2,  /* valid request this build does not implement                 */
  SIGATTN_ECUDA = 3,         /* a CUDA runtime / driver call or a launch failed             */
  SIGATTN_EWORKSPACE = 4     /* workspace too small                                          */
} sigattn_status;

/* flags bitfield */
enum {
  SIGATTN_F_BWD_DETERMINISTIC = 1u << 0, /* bwd: the paper's two-pass split -- a query-tile-owned
                                          dQ pass (Alg. 2) + a key-tile-owned dK/dV
                                          pass (Alg. 3).  No atomics: bitwise
                                          reproducible dQ; 14d instead of 10d FLOP per pair.  */
  SIGATTN_F_OUT_F32_PARTIAL = 1u << 1, /* fwd: o is float* (fp32, no cast) -- a partial O
                                          for key-split context parallelism (A4)     */
  SIGATTN_F_DQ_F32_PARTIAL = 1u << 2,  /* bwd: dq is float* fp32 alpha*dS K, not finalised
                                          (for the CP reduce-scatter)                        */
  SIGATTN_F_NO_ZERO_PAD_OUT = 1u << 3, /* fwd and bwd: padded output rows (i >= n_q of O, dQ;
                                          j >= n_k of dK, dV) are left unspecified instead of
                                          zeroed (saves the fill writes; C3 is 74% padding).
                                          Valid rows are always written, including the exact
                                          zeros of a sequence whose key (or query) set is empty. */
  SIGATTN_F_SANITIZE_PAD = 1u << 5,    /* NaN-safe padding: before reading them, the library
                                          zeroes IN PLACE the padded rows of q, k, v (and dout)
                                          that share a 128-row tile with valid rows (rows
                                          [n, ceil128(n)) of each sequence) -- the only padded
                                          rows the kernels load.  Without it pad content must be
                                          finite: a tensor core computes 0 * NaN = NaN (DESIGN R3).
                                          The inputs are modified.                           */
  SIGATTN_F_LAYOUT_BSHD = 1u << 4      /* every tensor argument (q, k, v, o, dout, dq, dk, dv)
                                          is [B, N, H, d] -- the paper's [Z, L, H, D] layout
                                          (Alg. 1-3 Require lines) --
                                          instead of [B, H, N, d]; read and written in place
                                          through strided TMA views, no transposes.  Not
                                          combinable with SIGATTN_F_DQ_F32_PARTIAL (the CP
                                          partial dQ is always [B, H, Nq, d]).              */
};

typedef struct {
  int B, H;          /* batch, heads                                                     */
  int Nq, Nk;        /* padded query / key lengths (Nq == Nk for self-attention)         */
  int d;             /* head dimension: 64 or 128                                        */
  int dtype;         /* sigattn_dtype                                                    */
  const int32_t* seqlens_q; /* device [B] or NULL (all Nq valid)                          */
  const int32_t* seqlens_k; /* device [B] or NULL (all Nk valid)                          */
  float scale;       /* alpha; callers pass 1/sqrt(d) by convention              */
  float bias;        /* scalar b, used when bias_per_seq == NULL (b = -log n)     */
  const float* bias_per_seq; /* device [B] or NULL: per-sequence b in R^Z (Alg. 1)  */
  unsigned flags;    /* SIGATTN_F_*                                                      */
  float* dbias;      /* sigattn_bwd only: device [B] fp32 or NULL.  When set, receives
                        d loss / d b_z = sum over heads and valid (i, j) of dS_ij (the gradient
                        of a learnable per-sequence bias); overwritten, not accumulated.
                        Summed with fp32 atomics: not bitwise reproducible run to run.      */
} sigattn_params;

/* Bytes of device workspace sigattn_fwd needs (the device work list of visited query tiles:
 * 16 + 16 * B * H * ceil(Nq / 128) bytes, rounded up to 256).  Returns 0 for invalid params.   */
size_t sigattn_fwd_workspace_bytes(const sigattn_params* p);

/* Forward (Alg. 1).  q [B,H,Nq,d], k/v [B,H,Nk,d], o [B,H,Nq,d] (fp32 if OUT_F32_PARTIAL).
 * Fully padded query tiles are skipped and the key loop stops at n_k.
 * workspace: device, >= sigattn_fwd_workspace_bytes(p), 16-byte aligned, caller-owned; it is
 * written and read by this call's stream work only (calls on different streams need different
 * workspaces; calls on one stream may share one).  Returns SIGATTN_EWORKSPACE if too small.    */
sigattn_status sigattn_fwd(const sigattn_params* p, const void* q, const void* k, const void* v,
                           void* o, void* workspace, size_t workspace_bytes, void* stream);

/* Bytes of device workspace sigattn_bwd needs (an fp32 dQ accumulator [B,H,Nq,d] plus a
 * small scheduling area).  Returns 0 for invalid params.                                     */
size_t sigattn_bwd_workspace_bytes(const sigattn_params* p);

/* Backward (Alg. 2 + Alg. 3, fused into one key-tile-owned pass: dK/dV accumulate on chip
 * without atomics, dQ partials are reduced into the fp32 workspace, then finalised; with
 * SIGATTN_F_BWD_DETERMINISTIC the paper's two passes run instead, see above).
 * dout [B,H,Nq,d]; dq [B,H,Nq,d] (fp32 if DQ_F32_PARTIAL); dk, dv [B,H,Nk,d].
 * workspace: device, >= sigattn_bwd_workspace_bytes(p), 16-byte aligned, caller-owned.       */
sigattn_status sigattn_bwd(const sigattn_params* p, const void* q, const void* k, const void* v,
                           const void* dout, void* dq, void* dk, void* dv, void* workspace,
                           size_t workspace_bytes, void* stream);

/* key_padding_mask [B,N] uint8 (1 = PAD, PyTorch convention) -> seqlens [B] int32 (device).
 * Only prefix masks reduce to lengths: *nonprefix_flag (device int32) is set to 1 if any row
 * has a valid token after a pad token, else 0.                                               */
sigattn_status sigattn_mask_to_seqlens(const uint8_t* key_padding_mask, int B, int N,
                                       int32_t* seqlens, int32_t* nonprefix_flag, void* stream);

/* Valid-token FLOP credit (App. B.1): sum_b c * H * d * nq[b] * nk[b] with c = 4
 * (forward) or 10 (backward).  HOST arrays, no GPU needed.  Returns -1 on bad arguments.      */
int64_t sigattn_valid_flops(int B, int H, int d, const int32_t* host_nq, const int32_t* host_nk,
                            int forward);

/* Host mirror of the device work-list builder, for tests and schedulers: writes the items the
 * forward (kind = 0, items = (b,h,q-tile), cost = key tiles; kind = 2, items = (b,h,pair of
 * q-tiles 2t and 2t+1), cost = key tiles -- the two-tile forward) or backward (kind = 1, items =
 * (b,h,k-tile), cost = query tiles) kernel visits, in visiting order (longest first, ties by
 * b then h then tile).  Each item is 4 int32: {b, h, tile, cost}.  Returns the item count, or
 * -1 on bad arguments; writes at most max_items.  tile = 128 rows.  (The device list of the
 * two-tile forward additionally cuts the items of a short last round of the persistent grid along
 * their key range -- sched.cuh split_tail_block; this mirror returns the uncut list.)           */
int64_t sigattn_worklist_host(int kind, int B, int H, int Nq, int Nk, const int32_t* host_nq,
                              const int32_t* host_nk, int32_t* items, int64_t max_items);

/* General (non-prefix) key_padding_mask [B, N] uint8 (1 = PAD) -> a stable compaction of every
 * sequence: index [B, N] int32 (device) lists the valid positions in order, then the padded ones;
 * seqlens [B] int32 (device) receives the valid counts.  Attention is equivariant under a joint
 * permutation of a sequence's queries and keys (sigma is element-wise, Eq. 2), so
 * permute_rows(gather) -> sigattn_fwd/bwd with seqlens -> permute_rows(scatter) is exact for any
 * mask (self-attention, the same mask on queries and keys).                                      */
sigattn_status sigattn_mask_to_index(const uint8_t* key_padding_mask, int B, int N, int32_t* index,
                                     int32_t* seqlens, void* stream);
/* Row permutation of a [B, H, N, d] 16-bit tensor (device, src != dst) by index [B, N]:
 * scatter == 0: dst[b,h,r] = src[b,h,index[b,r]];  scatter == 1: dst[b,h,index[b,r]] = src[b,h,r].  */
sigattn_status sigattn_permute_rows(const void* src, void* dst, const int32_t* index, int B, int H, int N,
                                    int d, int scatter, void* stream);

/* Padding-aware host <-> device transfer (the end-to-end path of a padded batch): copies only the
 * VALID rows [0, lens[b]) of every (b, h) slab of a 16- or 32-bit [B, H, N, d] tensor (layout_bshd:
 * [B, N, H, d], whose valid rows of sequence b are one contiguous block) from src to dst, as
 * cudaMemcpy2DAsync / cudaMemcpyAsync on `stream` -- one call per sequence; rows past lens[b] of dst
 * are not touched.  The kernels never read padded input rows beyond the last valid 128-row tile
 * and write padded output rows as zeros, so a caller that keeps persistent
 * buffers whose padded rows are zero (or passes SIGATTN_F_SANITIZE_PAD) moves only the valid
 * bytes across PCIe.  host_lens: HOST int32 [B], clamped to [0, N].  kind: 1 host -> device,
 * 2 device -> host, 3 device -> device (cudaMemcpyKind values).  row_bytes = d * element size, a
 * multiple of 16.  Returns the bytes copied through *bytes_out when it is non-NULL.  Argument
 * errors return SIGATTN_EINVAL before any copy is enqueued.                                       */
sigattn_status sigattn_copy_valid_rows(const void* src, void* dst, int B, int H, int N, int row_bytes,
                                       const int32_t* host_lens, int layout_bshd, int kind, void* stream,
                                       int64_t* bytes_out);

/* Instrumentation (bench / tests).  sigattn_launch_count(): number of kernels this library has
 * launched in this process so far (all entry points).  sigattn_set_profile_events(): thread-local;
 * when an event pair is non-NULL, the next sigattn_fwd / sigattn_bwd calls on this thread record
 * `start` immediately before and `stop` immediately after their main attention kernel, on the
 * call's stream (cudaEvent_t passed as void*).  Pass NULLs to disable.                          */
int64_t sigattn_launch_count(void);
void sigattn_set_profile_events(void* fwd_start, void* fwd_stop, void* bwd_start, void* bwd_stop);
/* Debug builds compiled with -DSIGATTN_TRACE=1 only: device buffer of grid x 4096 int64 that the
 * kernels fill with clock64() pipeline timestamps (thread-local setting; NULL disables).  A no-op
 * in release builds.                                                                            */
void sigattn_set_trace_buffer(void* device_buffer);
/* Skip accounting: thread-local; when non-NULL, the attention kernels add
 * the (query tile, key tile) pairs they actually execute to device uint64 counters:
 * counters[0] forward (128 x 128 pairs), counters[1] backward key-tile pass (128 keys x its query
 * tile: 128 rows for d = 64, 64 rows for d = 128), counters[2] deterministic dQ pass (128 x 128).
 * The caller zeroes them; one atomic per work item.  NULL disables.                               */
void sigattn_set_debug_counters(void* device_counters);

/* ---------------------------------------------------------------------------------------------
 * Key-split context parallelism with the reduction fused into the kernels.
 * Sigmoid weights are additive over key blocks (sec. 3): with the SAME bias b,
 *   O = sum_r sigma(alpha Q K_r^T + b) V_r,   dQ = sum_r alpha dS_r K_r,
 * so G ranks that each hold one key block need no log-sum-exp merge -- only a sum.  Rank g owns
 * query rows [g Nq/G, (g+1) Nq/G) and an fp32 accumulator [B, H, Nq/G, d] for them.  The fused
 * calls below reduce-add (red.global.add.v4.f32, system scope) every partial row straight into the
 * owner's accumulator -- over NVLink when the owner is another GPU -- instead of materialising a
 * partial tensor and reduce-scattering it with a separate collective: the forward straight from the
 * kernel epilogue (each O row is final for this rank's keys once its query tile's key loop ends),
 * the backward from a push kernel after the key-tile pass (every key tile adds a dQ partial, which
 * is summed in L2 first so that each row crosses NVLink once).
 *
 * Per-rank problem in sigattn_params: Nq = the full query length (all queries, e.g. all-gathered
 * Q), Nk = this rank's key block length, seqlens_q = global valid lengths, seqlens_k = the valid
 * keys of this rank's block, bias = the GLOBAL b (e.g. -log of the global length, never the block
 * length; DESIGN reading R1).  Layout [B, H, N, d] only.
 * Protocol (the caller's, e.g. paper_2604_27124_b200.parallel): every rank zeroes its accumulator,
 * all ranks synchronise, each rank runs the fused call, all ranks synchronise again (the kernels end
 * with a system-scope fence), then each rank runs sigattn_cp_finalize on its own accumulator.    */
typedef struct {
  int world;               /* G >= 1; Nq must be a multiple of G                                   */
  int rank;                /* this rank, 0 <= rank < G                                             */
  float* const* peer_acc;  /* DEVICE array [G] of device pointers: rank g's fp32 accumulator
                              [B, H, Nq/G, d] (this rank's own at [rank]), mapped on this device
                              (sigattn_ipc_import for other processes' buffers)                    */
} sigattn_cp_params;

/* Forward partial over this rank's keys, reduce-added into the owners' accumulators (unscaled fp32
 * sums of P V, padded query rows contribute nothing).  workspace >= sigattn_fwd_workspace_bytes(p). */
sigattn_status sigattn_fwd_cp(const sigattn_params* p, const sigattn_cp_params* cp, const void* q,
                              const void* k, const void* v, void* workspace, size_t workspace_bytes,
                              void* stream);
/* Bytes of workspace sigattn_bwd_cp needs (a local fp32 dQ partial [B, H, Nq, d] + scheduling).  */
size_t sigattn_bwd_cp_workspace_bytes(const sigattn_params* p);
/* Backward over this rank's keys: dk, dv [B, H, Nk, d] of this rank's block are complete on return
 * (keys are owned; padded rows 0 as in sigattn_bwd); alpha dS K summed over this rank's key tiles is
 * reduce-added, row by row, into the owners' fp32 dQ accumulators.  dout is the full [B, H, Nq, d]. */
sigattn_status sigattn_bwd_cp(const sigattn_params* p, const sigattn_cp_params* cp, const void* q,
                              const void* k, const void* v, const void* dout, void* dk, void* dv,
                              void* workspace, size_t workspace_bytes, void* stream);
/* acc [B, H, Nq/G, d] fp32 (this rank's accumulator, complete) -> out [B, H, Nq/G, d] in p->dtype;
 * rows whose global index rank * Nq/G + r is >= n_q[b] are written as exact 0.                   */
sigattn_status sigattn_cp_finalize(const sigattn_params* p, int world, int rank, const float* acc, void* out,
                                   void* stream);

/* CUDA IPC of a device buffer between processes (for sigattn_cp_params.peer_acc): export writes
 * sigattn_ipc_handle_bytes() bytes (the allocation's cudaIpcMemHandle_t and the pointer's offset in
 * it); import maps it on the current device (peer access over NVLink when it lives on another
 * GPU) and returns the pointer; close unmaps a pointer returned by import.                       */
size_t sigattn_ipc_handle_bytes(void);
sigattn_status sigattn_ipc_export(const void* dev_ptr, void* handle);
sigattn_status sigattn_ipc_import(const void* handle, void** dev_ptr);
sigattn_status sigattn_ipc_close(void* dev_ptr);

const char* sigattn_last_error(void); /* thread-local message of the last failing call */
const char* sigattn_version(void);

#ifdef __cplusplus
}
#endif

#endif /* SIGATTN_H_ */
