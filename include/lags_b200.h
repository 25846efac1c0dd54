/*
 * lags_b200.h -- C ABI of the B200-native LAGS-SGD sparsify -> exchange -> decode -> update path.
 *
 * The reference (arxiv 1911.08727, /root/reference/pkg/src/lagsgd) is pure Python/numpy and has
 * no FFI; each entry point below replaces one reference function (cited as R: file:line).  The
 * Python package `paper_1911_08727_b200` binds these with ctypes and keeps the reference's Python
 * names (top_k, decompress, lags_step, ...).  See INTEGRATION.md for the binding stubs.
 *
 * Conventions
 *  - All buffer pointers are DEVICE pointers owned by the caller.  Nothing here allocates.
 *  - Every call is stream-ordered on `stream` and never synchronises the host.
 *  - Return value: LAGS_OK (0) or a negative lags_status_t; lags_last_error() gives a message
 *    (thread-local).  No C++ exception crosses the ABI.
 *  - No global mutable device state: calls on distinct (stream, workspace) pairs are independent.
 *  - dtype selects storage / accumulation types (see lags_dtype_t).
 *  - A "bucket" is a contiguous run of layers inside flat per-worker buffers (the reference's
 *    LayeredVector layout, R: layered.py:46-107): layer j occupies [offset_j, offset_j + dim_j).
 *    Selected entries of layer j go to output slots [slot_j, slot_j + k_j); indices are
 *    layer-local int32, strictly ascending, values are the accumulated entries.
 */
#ifndef LAGS_B200_H
#define LAGS_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct CUstream_st* lags_stream_t; /* == cudaStream_t */

typedef enum {
  LAGS_OK = 0,
  LAGS_ERR_INVALID_ARG = -1,   /* null pointer, bad sizes            -> ValueError      */
  LAGS_ERR_K_OUT_OF_RANGE = -2,/* k outside 1..dim                   -> ValueError      (R: sparsify.py:82-83) */
  LAGS_ERR_STRUCTURE = -3,     /* layer table inconsistent           -> StructureError  (R: training.py:172-173) */
  LAGS_ERR_WORKSPACE = -4,     /* workspace too small                                    */
  LAGS_ERR_CUDA = -5           /* CUDA launch / runtime error                            */
} lags_status_t;

/* Storage / arithmetic modes (R: training.py:250 under numpy's NEP 50 promotion rules).
 *  LAGS_F32        g, r, v float32; acc = fl32(r + fl32(fl32(alpha) * g)); values float32
 *  LAGS_F64        everything float64 (the reference's default LayeredVector dtype)
 *  LAGS_F32_ACC64  g, r, v float32 with a numpy-float64 alpha: acc and values float64,
 *                  residual stored back as float32 (R: training.py:63-64 + :250-252)        */
typedef enum { LAGS_F32 = 0, LAGS_F64 = 1, LAGS_F32_ACC64 = 2 } lags_dtype_t;

/* Status bits written (OR-ed) into the caller's device status word. */
#define LAGS_STATUS_NONFINITE 0x1u /* some gradient entry was inf/nan -> DivergenceError (R: training.py:174-175) */

/* One layer of a bucket.  Lives in device memory (an array of these). */
typedef struct {
  int64_t offset; /* first element of the layer inside the flat g / r / v buffers */
  int64_t dim;    /* d_l >= 1                                                      */
  int32_t k;      /* selection budget 1 <= k_l <= d_l (R: sparsify.py:182-184)     */
  int32_t slot;   /* first output slot of the layer (prefix sum of k)              */
} lags_layer_t;

/* Per-bucket persistent selection state (device memory, one per layer, zero-initialise once).
 * Holds the predicted magnitude threshold used by the fast path; opaque to callers. */
typedef struct {
  uint64_t pred_key;   /* predicted threshold key (0 = no prediction yet)  */
  uint32_t flags;      /* internal                                         */
  uint32_t last_cands; /* candidates seen at the last call (diagnostic)    */
} lags_layer_state_t;

int lags_abi_version(void);
const char* lags_last_error(void);
/* Number of kernels this library has launched in the process (diagnostic / bench evidence). */
unsigned long long lags_kernel_launches(void);

/* Bytes of workspace lags_compress needs for a bucket of `n_total` elements / `nlayers`
 * layers / `total_k` slots. */
size_t lags_compress_workspace_bytes(int32_t dtype, int32_t nlayers, int64_t n_total, int64_t total_k);

/* Per-worker compress of one bucket -- replaces, per worker p and layer l, R: training.py:250-252
 * (acc = r + alpha*g; top_k(acc, k); r = acc - sent) and the finiteness check of
 * R: training.py:174 (fused; sets LAGS_STATUS_NONFINITE in *status, never clears it).
 *   g, r        flat worker buffers (dtype storage type), bucket starts at element 0
 *   idx_out     int32 [total_k]        val_out  acc type [total_k]     count_out int32 [nlayers]
 *   state       lags_layer_state_t [nlayers] or NULL (NULL = exact path every call)
 */
int lags_compress(int32_t dtype, const lags_layer_t* layers, int32_t nlayers, int64_t n_total,
                  int64_t total_k, const void* g, void* r, double alpha, int32_t* idx_out,
                  void* val_out, int32_t* count_out, uint32_t* status, lags_layer_state_t* state,
                  void* workspace, size_t workspace_bytes, lags_stream_t stream);

/* Finiteness of x[0:n) (R: training.py:174); ORs LAGS_STATUS_NONFINITE into *status. */
int lags_check_finite(int32_t dtype, const void* x, int64_t n, uint32_t* status, lags_stream_t stream);

/* Exact magnitude top-k of one dense vector -- R: sparsify.py:71-90.  x is not modified.
 * Writes min(k, nnz) ascending int32 indices + values and the count. */
int lags_top_k(int32_t dtype, const void* x, int64_t dim, int32_t k, int32_t* idx_out,
               void* val_out, int32_t* count_out, void* workspace, size_t workspace_bytes,
               lags_stream_t stream);
size_t lags_top_k_workspace_bytes(int32_t dtype, int64_t dim);

/* Dense reconstruction -- R: sparsify.py:63-68.  out[0:dim] = 0; out[idx[j]] = val[j]. */
int lags_decompress(int32_t dtype, const int32_t* idx, const void* val, const int32_t* count,
                    int64_t dim, void* out, lags_stream_t stream);

/* Decode + update of one bucket after the exchange -- replaces R: training.py:248,253-254:
 *   total = fp64 zeros; for p = 1..P (rank order): total[idx] += val;  v = v - total / P
 * Rank p's message is at byte offset p*rank_stride_bytes from idx0 / val0 / cnt0.
 * mu == 0 is the reference (parity) mode and touches only selected positions; mu > 0 adds
 * heavy-ball momentum m = mu*m + total/P; v -= m over the whole bucket (parity unpinned,
 * R: SPEC.md:366 lists momentum as a non-goal).  `momentum` may be NULL when mu == 0.
 * The decode workspace must be zero-filled before the first call; every call leaves it zeroed. */
size_t lags_decode_workspace_bytes(int32_t dtype, int64_t n_total, int32_t P);
int lags_decode_update(int32_t dtype, const lags_layer_t* layers, int32_t nlayers, int64_t n_total,
                       int64_t total_k, const int32_t* idx0, const void* val0, const int32_t* cnt0,
                       int64_t rank_stride_bytes, int32_t P, void* v, void* momentum, double mu,
                       void* workspace, size_t workspace_bytes, lags_stream_t stream);

#ifdef __cplusplus
}
#endif
#endif /* LAGS_B200_H */
