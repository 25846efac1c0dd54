/*
 * lags_b200.h -- C ABI of the B200-native LAGS-SGD sparsify -> exchange -> decode -> update path.
 *
 * The reference (arxiv 1911.08727, /root/reference/pkg/src/lagsgd) is pure Python/numpy and has
 * no FFI; each entry point below replaces one reference function (cited as R: file:line).  The
 * Python package `paper_1911_08727_b200` binds these with ctypes and keeps the reference's Python
 * names (top_k, decompress, lags_step, ...).  See INTEGRATION.md for binding stubs.
 *
 * Conventions
 *  - Buffer pointers are DEVICE pointers owned by the caller; the library never allocates device
 *    memory (a bucket lives in caller-provided device memory; its handle is a small host struct).
 *  - Every call is stream-ordered on `stream` and does not synchronise the host, except
 *    lags_bucket_create (one-time table upload) and lags_bucket_stats (diagnostic read-back).
 *  - Return value: LAGS_OK (0) or a negative lags_status_t; lags_last_error() gives a message
 *    (thread-local).  No C++ exception crosses the ABI.
 *  - A bucket is a contiguous run of layers of the flat per-worker buffers (the reference's
 *    LayeredVector layout, R: layered.py:46-107): layer j occupies [offset_j, offset_j + dim_j),
 *    offsets being the prefix sums of dims.  Flat buffers need only their element alignment
 *    (4 bytes fp32, 8 bytes fp64); 16-byte aligned buffers take the vector path throughout.
 */
#ifndef LAGS_B200_H
#define LAGS_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct CUstream_st* lags_stream_t; /* == cudaStream_t */
typedef struct lags_bucket lags_bucket_t;  /* opaque host handle */

typedef enum {
  LAGS_OK = 0,
  LAGS_ERR_INVALID_ARG = -1,    /* null pointer, bad sizes, misaligned buffer -> ValueError            */
  LAGS_ERR_K_OUT_OF_RANGE = -2, /* k outside 1..dim                            -> ValueError (R: sparsify.py:82-83) */
  LAGS_ERR_STRUCTURE = -3,      /* inconsistent layer layout                   -> StructureError (R: training.py:172-173) */
  LAGS_ERR_WORKSPACE = -4,      /* caller memory too small                                              */
  LAGS_ERR_CUDA = -5            /* CUDA launch / runtime error                                          */
} lags_status_t;

/* Storage / arithmetic modes (R: training.py:250 under numpy's NEP 50 promotion rules).
 *  LAGS_F32        g, r, v float32; acc = fl32(r + fl32(fl32(alpha) * g)); values float32
 *  LAGS_F64        everything float64 (the reference's default LayeredVector dtype)
 *  LAGS_F32_ACC64  g, r, v float32 with a numpy-float64 alpha: acc and values float64,
 *                  residual stored back as float32 (R: training.py:63-64 + :250-252)        */
typedef enum { LAGS_F32 = 0, LAGS_F64 = 1, LAGS_F32_ACC64 = 2 } lags_dtype_t;

/* Status bits OR-ed into the caller's device status word. */
#define LAGS_STATUS_P2P_TIMEOUT 0x100u /* lags_p2p_wait: a peer's message did not arrive in time */
#define LAGS_STATUS_NONFINITE 0x1u /* a gradient entry was inf/nan -> DivergenceError (R: training.py:174-175) */

/* lags_bucket_compress flags */
#define LAGS_COMPRESS_EXACT 0x1u     /* skip the predicted-threshold fast path (dense exact selection) */
#define LAGS_COMPRESS_ZERO_GRAD 0x2u /* clear g after reading it (fused zero_grad of the optimizer)   */

int lags_abi_version(void);
const char* lags_last_error(void);
/* Number of kernels this library has launched in the process (diagnostic / bench evidence). */
unsigned long long lags_kernel_launches(void);

/* ---- bucket: the per-layer hot path ------------------------------------------------------- */

/* Device bytes for a bucket of `nlayers` layers (host arrays dims[], ks[]) exchanged among up to
 * `max_world` ranks (tables, selection state, candidate lists, decode planes). */
size_t lags_bucket_device_bytes(int32_t dtype, const int64_t* dims, const int32_t* ks, int32_t nlayers,
                                int32_t max_world);

/* Build a bucket in `device_mem` (>= lags_bucket_device_bytes): uploads the layer/task tables and
 * zeroes the selection state (synchronises `stream` once).  Validates 1 <= k_l <= d_l
 * (R: sparsify.py:82-83, LAGS_ERR_K_OUT_OF_RANGE) and d_l < 2^31. */
int lags_bucket_create(int32_t dtype, const int64_t* dims, const int32_t* ks, int32_t nlayers, int32_t max_world,
                       void* device_mem, size_t bytes, lags_stream_t stream, lags_bucket_t** out);
void lags_bucket_destroy(lags_bucket_t* bucket);

/* Byte layout of one worker's sparse message for this bucket:
 *   counts int32[nlayers] @ off_counts | idx int32[sum k] @ off_idx | values @ off_val (float32 for
 *   LAGS_F32, float64 otherwise); msg_bytes is a multiple of 16.  Layer j's entries occupy slots
 *   [slot_j, slot_j + counts[j]) with slot_j = k_1 + ... + k_{j-1}; indices are layer-local,
 *   strictly ascending. */
int lags_bucket_message_layout(const lags_bucket_t* bucket, int64_t* off_counts, int64_t* off_idx,
                               int64_t* off_val, int64_t* msg_bytes);

/* One worker's compress of the bucket -- per layer l replaces R: training.py:250-252
 *   acc = r + alpha*g;  chunk = top_k(acc, k_l);  r = acc - decompress(chunk)
 * plus the finiteness check of R: training.py:174 (fused; ORs LAGS_STATUS_NONFINITE into
 * *status, never clears it).  Writes the message (layout above) to `msg`.  g is read-only unless
 * LAGS_COMPRESS_ZERO_GRAD is set. */
int lags_bucket_compress(lags_bucket_t* bucket, void* g, void* r, double alpha, void* msg, uint32_t* status,
                         uint32_t flags, lags_stream_t stream);

/* Compress with the exchange fused into the selection (LAGS_F32 buckets): every finished layer's
 * count and (index, value) pairs are also stored into slot `rank` of every rank's receive area
 * (the lags_p2p_push layout and epoch parity, own area included) by the CTA that produced them,
 * so the NVLink transfer overlaps the rest of the selection; the last CTA publishes the flags.
 * Follow it with lags_p2p_wait on the receive area, exactly as after lags_p2p_push (which this
 * replaces).  Replaces R: training.py:245-248 (the all-gather) together with the compress. */
typedef struct {
  const void* bases;          /* device uint64[P]: every rank's receive area (lags_ipc_open) */
  int32_t P, rank, ctas_per_peer;
  uint64_t flags_bytes;       /* as lags_p2p_push */
  const void* epoch;          /* device uint32 epoch counter (advanced by lags_p2p_wait) */
} lags_peer_push_t;
int lags_bucket_compress_push(lags_bucket_t* bucket, void* g, void* r, double alpha, void* msg, uint32_t* status,
                              uint32_t flags, const lags_peer_push_t* peer, lags_stream_t stream);

/* Single-rank step (P = 1, no exchange): lags_bucket_compress plus the update v = v - total / 1,
 * fused into the selection epilogue for LAGS_F32 buckets of up to 49152 selected entries (no
 * separate decode pass); larger selections and the fp64 / mixed modes run the ordinary decode
 * after the compress.  The message is still written.  Equivalent to lags_bucket_compress followed
 * by lags_bucket_decode_update(..., P = 1, ...). */
int lags_bucket_step_local(lags_bucket_t* bucket, void* g, void* r, double alpha, void* v, void* msg,
                           uint32_t* status, uint32_t flags, lags_stream_t stream);

/* Decode + update after the exchange -- replaces R: training.py:248,253-254:
 *   total = fp64 zeros; for p = 1..P (rank order): total[idx] += val;   v = v - total / P
 * `msgs` holds P messages, rank p's at byte offset p * msg_stride.  mu == 0 is the reference
 * (parity) mode and touches only selected weights; mu > 0 applies heavy-ball momentum over the
 * whole bucket, m = mu*m + total/P, v -= m (parity unpinned: momentum is a non-goal of the
 * reference, R: SPEC.md:366).  `momentum` may be NULL when mu == 0.  P <= max_world.
 * flags: LAGS_DECODE_V64 -- v (and momentum) are float64 whatever the bucket dtype, v = fl64(v -
 * total/P) without rounding to the storage type (the reference's slgs_step returns its float32
 * parameters promoted to float64, R: training.py:224). */
#define LAGS_DECODE_V64 0x1u
int lags_bucket_decode_update(lags_bucket_t* bucket, const void* msgs, int64_t msg_stride, int32_t P, void* v,
                              void* momentum, double mu, uint32_t flags, lags_stream_t stream);

/* Diagnostics: when set (non-NULL cudaEvent_t handles), every fp32 compress records `before` and
 * `after` around its streaming kernel (K1) so callers can time the dominant kernel live. */
int lags_bucket_set_probe_events(lags_bucket_t* bucket, void* before, void* after);

/* Gradient pointer table (LAGS_F32): `table` is a DEVICE array of nlayers pointers, layer j's
 * gradient (dim_j contiguous floats, e.g. a framework's per-parameter .grad tensor), read by
 * every later compress / step_local instead of the flat g (which may then be NULL).  Lets an
 * autograd engine hand its gradient tensors over without accumulating into a flat buffer.  The
 * table's contents are read when the kernels run (stream-ordered); NULL switches back to flat g. */
int lags_bucket_set_grad_table(lags_bucket_t* bucket, const void* table);

/* Diagnostics: per layer {threshold key, fallbacks, last candidate count, calls, last select
 * cycles, last path (0 small dense, 1 candidates, 2 dense after a failed prediction), phase
 * cycles, select start / end / CTA launch (%globaltimer ns, low 32 bits), 0} (synchronous).
 * LAGS_F64 / LAGS_F32_ACC64 buckets: {threshold key >> 32, fallbacks, last candidate count, calls,
 * 0, last path (0 small layer, 1 candidates, 2 dense), 0...}. */
#define LAGS_STATS_WORDS 12
int lags_bucket_stats(const lags_bucket_t* bucket, uint32_t* out /* [nlayers * 12] */, lags_stream_t stream);

/* ---- diagnostics -------------------------------------------------------------------------------
 * acc_p = r_p with message p's pairs written back (the accumulated vector before selection, as
 * R: training.py:329 forms it): P planes of n_total elements, plane_stride elements apart.  r and
 * acc may not alias.  LAGS_F32 / LAGS_F64 buckets. */
int lags_bucket_reconstruct(const lags_bucket_t* bucket, const void* msgs, int64_t msg_stride, int32_t P,
                            const void* r, void* acc, int64_t plane_stride, lags_stream_t stream);

/* Aggregation-quality ratio per layer -- R: analysis.py:24-56 (topk_aggregation_ratio) as the
 * train loop logs it (R: training.py:320-337): total = sum_p acc_p, agg = sum_p (acc_p - r_p)
 * (fp64, worker order), out[j] = ||total - agg||^2 / ((1 - k_j/d_j) ||total||^2), NaN where the
 * denominator vanishes (the reference's None).  out: device double[nlayers]. */
int lags_bucket_delta(const lags_bucket_t* bucket, const void* acc, const void* r, int64_t plane_stride, int32_t P,
                      double* out, lags_stream_t stream);

/* Residual-identity monitor -- the dense shadow sequence of R: training.py:197-200 and the
 * identity check of R: training.py:356-369 (Eq. 10: v - x equals the mean error-feedback residual).
 * lags_bucket_shadow_step: x = x - (alpha * g_sum) / P in fp64 (x: float64[n_total]; g_sum: the
 * sum of the P workers' gradients in the bucket's storage dtype).
 * lags_bucket_identity: out[j] = ||mean residual of layer j||^2 (j < nlayers), out[nlayers] =
 * ||v - x||^2, out[nlayers + 1] = max_i |(v - x)_i - r_sum_i / P| (out: device double[nlayers + 2];
 * v and r_sum in the storage dtype). */
int lags_bucket_shadow_step(const lags_bucket_t* bucket, const void* g_sum, double* x, double alpha, int32_t P,
                            lags_stream_t stream);
int lags_bucket_identity(const lags_bucket_t* bucket, const void* v, const double* x, const void* r_sum, int32_t P,
                         double* out, lags_stream_t stream);

/* ---- single-vector operators ---------------------------------------------------------------- */

/* Finiteness of x[0:n) (R: training.py:174); ORs LAGS_STATUS_NONFINITE into *status. */
int lags_check_finite(int32_t dtype, const void* x, int64_t n, uint32_t* status, lags_stream_t stream);

/* Exact magnitude top-k of one dense vector -- R: sparsify.py:71-90.  x is not modified.
 * Writes min(k, nnz) ascending int32 indices + values and the count. */
size_t lags_top_k_workspace_bytes(int32_t dtype, int64_t dim);
int lags_top_k(int32_t dtype, const void* x, int64_t dim, int32_t k, int32_t* idx_out, void* val_out,
               int32_t* count_out, void* workspace, size_t workspace_bytes, lags_stream_t stream);

/* Dense reconstruction -- R: sparsify.py:63-68.  out[0:dim] = 0; out[idx[j]] = val[j], j < *count. */
int lags_decompress(int32_t dtype, const int32_t* idx, const void* val, const int32_t* count, int64_t dim,
                    void* out, lags_stream_t stream);

/* ---- sparse wire format -- R: sparsify.py:260-310 --------------------------------------------
 *   chunk   = u32 layer_id, u32 dim, u32 count, count x (u32 index, f64 value)   little-endian, packed
 *   message = u32 chunk count, then the chunks back to back
 * A chunk table names the chunks to encode / receives the decoded ones: device arrays layer_ids,
 * dims, counts and first (the chunk's first entry in idx / val).  A bucket message
 * (lags_bucket_message_layout) is a chunk table whose first[j] is layer j's slot offset.
 * Errors are reported in *error (device u64): ~0 = none, else (chunk << 8) | LAGS_WIRE_ERR_*,
 * the first failing chunk in stream order (the reference raises at the first bad chunk). */
#define LAGS_WIRE_MESSAGE 0u /* with the u32 chunk-count header (encode_message / decode_message) */
#define LAGS_WIRE_CHUNK 1u   /* exactly one chunk, no header (encode_chunk / decode_chunk)         */

#define LAGS_WIRE_ERR_TRUNCATED_MESSAGE 1u /* < 4 bytes                  -> StructureError (R: sparsify.py:301-302) */
#define LAGS_WIRE_ERR_TRUNCATED_HEADER 2u  /* chunk header past the end  -> StructureError (R: sparsify.py:281-282) */
#define LAGS_WIRE_ERR_TRUNCATED_PAYLOAD 3u /* chunk payload past the end -> StructureError (R: sparsify.py:286-287) */
#define LAGS_WIRE_ERR_INDEX_RANGE 4u       /* last index >= dim          -> StructureError (R: sparsify.py:48-49)   */
#define LAGS_WIRE_ERR_INDEX_ORDER 5u       /* not strictly increasing    -> StructureError (R: sparsify.py:50-51)   */
#define LAGS_WIRE_ERR_TRAILING 6u          /* bytes after the last chunk -> StructureError (R: sparsify.py:308-309) */
#define LAGS_WIRE_ERR_CAPACITY 7u          /* output / wire buffers too small                                        */

/* Encode nchunks chunks (R: encode_chunk / encode_message, sparsify.py:269-296).  val_dtype
 * LAGS_F32 or LAGS_F64 (widened exactly to f64).  *wire_len receives the length; nothing is
 * written (error LAGS_WIRE_ERR_CAPACITY) when it exceeds wire_capacity. */
int lags_wire_encode(uint32_t mode, int32_t nchunks, const uint32_t* layer_ids, const uint32_t* dims,
                     const int32_t* counts, const int64_t* first, const int32_t* idx, const void* val,
                     int32_t val_dtype, void* wire, int64_t wire_capacity, int64_t* wire_len, uint64_t* error,
                     lags_stream_t stream);

/* Decode wire[offset:wire_len] (R: decode_chunk / decode_message, sparsify.py:279-310) into a
 * chunk table of at most max_chunks (<= 4096) chunks.  Entries of chunk c go to first[c] with
 * room caps[c]; with first == NULL they are packed in chunk order into entry_capacity slots.
 * *end_out = offset after the last decoded chunk (decode_chunk's returned offset). */
int lags_wire_decode(uint32_t mode, const void* wire, int64_t wire_len, int64_t offset, int32_t max_chunks,
                     const int64_t* first, const int32_t* caps, int64_t entry_capacity, uint32_t* layer_ids,
                     uint32_t* dims, int32_t* counts, int32_t* idx, void* val, int32_t val_dtype,
                     int32_t* nchunks_out, int64_t* end_out, uint64_t* error, lags_stream_t stream);

/* ---- peer-memory exchange (one process per GPU, CUDA IPC over NVLink / NVSwitch) -------------
 * Replaces the all-gather of the fixed-size bucket messages (R: training.py:245-248 gathers every
 * worker's sparse chunks) with direct stores into every peer's receive area:
 *   area = [flags: P * G u32, padded to flags_bytes (multiple of 256)] [parity 0: P messages] [parity 1: P messages]
 * lags_ipc_malloc allocates a zeroed area and its 64-byte IPC handle; peers map it with
 * lags_ipc_open.  lags_p2p_push (G = ctas_per_peer CTAs per destination; bases = device array of
 * the P areas, own included) writes the message into slot `rank` of parity (epoch & 1) of every
 * area and publishes the epoch in flag [rank * G + g] (system-scope release).  lags_p2p_wait
 * acquires the local P * G flags (>= epoch, wrap-safe); on timeout it ORs LAGS_STATUS_P2P_TIMEOUT
 * into *status.  The decode that follows on the stream then reads the parity's P messages in rank order.
 * The epoch lives in device memory (*epoch, u32, starts at 0): the push uses *epoch + 1, the wait
 * waits for it and then stores it, so a step's launches have fixed arguments (graph-capturable);
 * the receiving parity is then (exchange count) & 1. */
int lags_ipc_malloc(size_t bytes, void** ptr, void* handle64);
int lags_ipc_open(const void* handle64, void** ptr);
int lags_ipc_close(void* ptr);
int lags_ipc_free(void* ptr);
int lags_p2p_push(const void* msg, int64_t msg_bytes, const uint64_t* bases, int P, int rank, int ctas_per_peer,
                  uint64_t flags_bytes, const uint32_t* epoch, lags_stream_t stream);
int lags_p2p_wait(const uint32_t* flags, int nflags, uint32_t* epoch, int32_t* status, uint64_t timeout_ns,
                  lags_stream_t stream);

#ifdef __cplusplus
}
#endif
#endif /* LAGS_B200_H */
