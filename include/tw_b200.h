/*
 * tw_b200.h -- C ABI of the B200-native tile-wise (TW) sparse GEMM library
 * (libtw_b200.so).  Plain pointers and sizes; no torch or numpy types.
 *
 * Each entry point names the reference interface it replaces
 * (reference = arxiv/paper_2008_13006 package `tilewise`,
 *  /root/reference/pkg/src/tilewise/<file>:<line>).
 *
 * Conventions
 *   - Every function returns an int status: TW_OK (0) or a TW_ERR_* code;
 *     tw_last_error() returns a thread-local message for the last failure.
 *     TW_ERR_DIMENSION maps to the reference's DimensionError
 *     (matrix.py:34-35), TW_ERR_FORMAT to FormatError (matrix.py:38-39),
 *     everything else to RuntimeError.
 *   - Matrices follow the reference's engine layout (engine.py:4-7, :102,
 *     :129, :164): activations are passed TRANSPOSED, at = A^T (K x M, M
 *     contiguous, row stride lda elements), and the output is written
 *     TRANSPOSED, ct = C^T (N x M, row stride ldc) -- i.e. the buffer of a
 *     COL_MAJOR C.  ROW_MAJOR fp32 activations are converted by
 *     tw_prep_activations (the reference's `at = a.array().T` copy,
 *     engine.py:129, with the bf16/fp16 cast fused in).
 *   - Device pointers are CUDA device memory on the current device; `stream`
 *     is a cudaStream_t (NULL = legacy default stream).  Launches are
 *     asynchronous; concurrent calls on distinct streams are safe (plans are
 *     read-only after creation).  No hidden allocations happen in the
 *     compute calls.
 *   - There is no CPU fallback: compute entry points require an sm_100 GPU
 *     and return TW_ERR_CUDA otherwise.
 */
#ifndef TW_B200_H
#define TW_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define TW_OK 0
#define TW_ERR_DIMENSION 1
#define TW_ERR_FORMAT 2
#define TW_ERR_CUDA 3
#define TW_ERR_ARG 4
#define TW_ERR_NOMEM 5
#define TW_ERR_UNSUPPORTED 6

/* element types */
#define TW_F32 0
#define TW_BF16 1
#define TW_F16 2

/* dense layout tags == matrix.py:29-31 Layout */
#define TW_ROW_MAJOR 0
#define TW_COL_MAJOR 1

const char *tw_last_error(void);
int tw_version(void);

/* ------------------------------------------------------------------------
 * Host-side metadata packer (CPU only; bit-exact with the reference)
 * ---------------------------------------------------------------------- */

/* pattern.py:169-177 pack_mask_words: keep[length] (0/1 bytes) ->
 * words[ceil(length/32)], bit b of word w = index 32w+b, 1 = keep. */
int tw_pack_mask_words(const uint8_t *keep, int64_t length, uint32_t *words);

/* pattern.py:180-185 unpack_mask_words.  TW_ERR_DIMENSION if the words do
 * not cover `length` bits (same condition as the reference). */
int tw_unpack_mask_words(const uint32_t *words, int64_t nwords, int64_t length, uint8_t *keep);

/* pattern.py:188-189 mask_words_to_indices: ascending kept indices. */
int tw_mask_words_to_indices(const uint32_t *words, int64_t nwords, int64_t length,
                             int64_t *idx, int64_t *count);

/* pattern.py:223-241 compact.  b: K x N fp32 with layout tag; tile t owns
 * col_ids[col_off[t] .. col_off[t+1]) and row mask words
 * row_mask_words[t*nwords .. (t+1)*nwords), nwords = ceil(K/32).
 * Writes every tile's sub-matrix COL_MAJOR (subs[sub_off[t] + j*k_t + r] =
 * B[rows_t[r], col_ids_t[j]]) and sub_off[0..n_tiles]. */
int tw_compact(const float *b, int64_t k, int64_t n, int layout, int64_t n_tiles,
               const int64_t *col_off, const int32_t *col_ids, const uint32_t *row_mask_words,
               float *subs, int64_t *sub_off);

/* pruning.py:257-258 _pruned_columns_of: ascending columns of [0,N) owned by
 * no tile (the C^T rows that must be exactly 0). */
int tw_pruned_columns(int64_t n, int64_t n_tiles, const int64_t *col_off, const int32_t *col_ids,
                      int64_t *out, int64_t *count);

/* ------------------------------------------------------------------------
 * Plans: the packed, device-resident form of a CompactTileSet
 * (pattern.py:145-158) consumed by the persistent kernel.
 * ---------------------------------------------------------------------- */
typedef struct tw_plan tw_plan;

typedef struct tw_plan_info {
  int64_t k, n, g;             /* pattern dims (CompactTileSet.k/.n/.g) */
  int64_t col_begin, col_end;  /* output column range this plan writes (shards) */
  int64_t n_tiles;             /* tiles in the CompactTileSet */
  int64_t n_live;              /* tiles with k_i > 0 and n_i > 0 (engine.py:134-135) */
  int64_t n_zero_rows;         /* C^T rows written as zeros (pruned + dead-tile columns) */
  int64_t kept_elems;          /* sum k_i*n_i over tiles in range: kept FLOPs = 2*M*kept_elems */
  int64_t union_k;             /* |union of kept rows| (A rows read at least once) */
  int64_t sum_k;               /* sum k_i over live tiles (index-list length) */
  int64_t sum_n;               /* sum n_i over live tiles */
  int64_t block_n;             /* MMA N tile (128 or 256) */
  int64_t wimg_bytes;          /* packed weight image bytes on device */
  int in_dtype;                /* TW_BF16 or TW_F16 */
  int flags;                   /* TW_PLAN_* the plan was built with */
  int64_t a_rows;              /* rows of the A^T operand tw_gemm reads: K, or 2K (TW_PLAN_SPLIT3) */
} tw_plan_info;

/* Plan flags (tw_plan_create_ex).
 * TW_PLAN_SPLIT3: fp32-faithful tensor-core mode.  Weights and activations
 *   are split into bf16 high/low parts, x = hi + lo with hi = rn_bf16(x),
 *   lo = rn_bf16(x - hi); the plan computes A.W as Ah.Wh + Al.Wh + Ah.Wl (3
 *   k_i kept rows per tile) from the 2K-row operand [Ah; Al] that
 *   tw_prep_activations_split writes.  Relative error per product ~2^-17:
 *   the reference's fp32 acceptance bar (1e-4*K max-abs,
 *   test_acceptance.py:63-81) on unrounded fp32 inputs.  Needs TW_BF16.
 * TW_PLAN_F32_WEIGHTS: keep the fp32 weights (the reference's sub_matrix
 *   values, pattern.py:233) on the device so tw_gemm_exact reproduces
 *   gemm_tw bit for bit on ANY fp32 weights, not only bf16-representable ones. */
#define TW_PLAN_SPLIT3 1
#define TW_PLAN_F32_WEIGHTS 2
/* TW_PLAN_DENSE_PAD: every live tile keeps ALL K rows, the pruned ones with
 *   zero weights (the same products: a pruned weight contributes 0 * a).
 *   Such a plan runs on the 2-SM kernel (tcgen05 cta_group::2, 256 output
 *   columns x 256 tokens per CTA pair, A^T by TMA tiles): the choice for
 *   near-dense patterns, where gathering the kept rows costs more than the
 *   MMAs on the pruned ones.  Non-finite activations in a
 *   tile's pruned rows give NaN there (0 * Inf), as in any dense GEMM. */
#define TW_PLAN_DENSE_PAD 4

/* Build a plan from the reference's compact form (the same arrays as
 * tw_compact's outputs plus the pattern) and upload it to the current
 * device.  subs are fp32 (the reference dtype); they are rounded to
 * in_dtype (RNE) here.  [col_begin, col_end) selects the output columns this
 * plan computes (0, N for the whole layer; a contiguous shard for the
 * N-sharded multi-GPU path -- tiles straddling the range are split, rows of
 * the output are re-based to col - col_begin).  G must be <= 256. */
int tw_plan_create(int64_t k, int64_t n, int64_t g, int64_t n_tiles, const int64_t *col_off,
                   const int32_t *col_ids, const uint32_t *row_mask_words, const float *subs,
                   const int64_t *sub_off, int in_dtype, int64_t col_begin, int64_t col_end,
                   tw_plan **out);
/* Same packing as tw_plan_create without touching the GPU (no device
 * buffers; tw_gemm on such a plan fails).  For inspecting / testing the
 * packed layout on a CPU-only host. */
int tw_plan_build_host(int64_t k, int64_t n, int64_t g, int64_t n_tiles, const int64_t *col_off,
                       const int32_t *col_ids, const uint32_t *row_mask_words, const float *subs,
                       const int64_t *sub_off, int in_dtype, int64_t col_begin, int64_t col_end,
                       tw_plan **out);
/* tw_plan_create with TW_PLAN_* flags (0 = tw_plan_create). */
int tw_plan_create_ex(int64_t k, int64_t n, int64_t g, int64_t n_tiles, const int64_t *col_off,
                      const int32_t *col_ids, const uint32_t *row_mask_words, const float *subs,
                      const int64_t *sub_off, int in_dtype, int64_t col_begin, int64_t col_end, int flags,
                      tw_plan **out);
int tw_plan_destroy(tw_plan *plan);
int tw_plan_get_info(const tw_plan *plan, tw_plan_info *info);

/* Copy the host image of the packed plan (for bit-exact layout tests):
 * which = 0 kept-K index lists (int32, padded with K), 1 col ids (int32,
 * block_n per live tile, padded with -1), 2 zero rows (int32), 3 weight
 * image (bytes, swizzled), 4 tile table (int64 x 8 per live tile:
 * src tile, kidx_off, col_off, n_i, k_i, k16, nkb, w_off).
 * *bytes is in/out: capacity in, size out (size only if dst == NULL). */
int tw_plan_export(const tw_plan *plan, int which, void *dst, int64_t *bytes);

/* Host-side view of the static launch schedule tw_gemm would use for M
 * tokens on a GPU with `sms` SMs (per-CTA unit lists + zero-row ranges; the
 * replacement for group_by_shape/execute_batched's LPT bins, engine.py:72-123).
 * which = 0 units (int32 x 4 per unit: live tile, first token, 64-token
 * quarters, 0), 1 per-CTA unit offsets (grid + 1), 2 per-CTA zero-row offsets
 * (grid + 1).  Same size protocol as tw_plan_export. */
int tw_schedule_export(const tw_plan *plan, int64_t m, int out_dtype, int accumulate, int sms, int which,
                       void *dst, int64_t *bytes);

/* ------------------------------------------------------------------------
 * Device compute (sm_100a)
 * ---------------------------------------------------------------------- */

/* engine.py:152-164 gemm_tw (+ _plan_tasks/gather_rows/group_by_shape/
 * execute_batched/mm_accum, engine.py:61-149, _kernels.py:13-27) as ONE
 * persistent tcgen05 kernel.  at: K x M (in_dtype, row stride lda, lda % 8
 * == 0, 16-byte aligned), ct: (col_end-col_begin) x M in out_dtype
 * (TW_F32 | TW_BF16 | TW_F16), row stride ldc.  accumulate = 0 writes
 * every output row (pruned columns as exact zeros, like the zero-filled
 * buffer of engine.py:102); accumulate = 1 adds into ct and leaves pruned
 * rows untouched (used by gemm_tew).  m == 0 is a no-op. */
int tw_gemm(const tw_plan *plan, const void *at, int64_t m, int64_t lda, void *ct, int64_t ldc,
            int out_dtype, int accumulate, void *stream);

/* trainer.py:232-250 engine_logits layer: tw_gemm with the bias + ReLU
 * epilogue fused -- ct[j, m] = relu?(C[m, j] + bias[j]) for every output
 * column j of the plan's range, pruned columns included (they become the
 * constant relu?(bias[j])).  fp32 add then max, rounded once to out_dtype.
 * bias: DEVICE fp32 array indexed by global output column (length N). */
int tw_gemm_bias(const tw_plan *plan, const void *at, int64_t m, int64_t lda, void *ct, int64_t ldc,
                 int out_dtype, const float *bias, int relu, void *stream);

/* General form of tw_gemm / tw_gemm_bias.  flags: TW_GEMM_ACCUMULATE (add
 * into ct, pruned rows untouched -- gemm_tew's second pass) and/or
 * TW_GEMM_KEEP_PRUNED (write only the kept columns' rows and leave the
 * pruned-column rows of ct as they are: for a resident output buffer whose
 * pruned rows already hold their value -- 0, or relu?(bias) with the bias
 * epilogue -- from an earlier full call, e.g. layer-chain activations).
 * bias may be NULL. */
#define TW_GEMM_ACCUMULATE 1
#define TW_GEMM_KEEP_PRUNED 2
/* Launch without programmatic dependent launch: the kernel starts only after
 * the previous work in the stream has completed (for isolated timing next to
 * library GEMMs, which are launched that way). */
#define TW_GEMM_NO_PDL 4
/* Run a K4-eligible plan (tw_plan_kernel) on K4 even when the layer does not
 * fill a wave of CTA pairs (TwPlan(dense_pad=True): the caller's choice). */
#define TW_GEMM_FORCE_PAIR 8
int tw_gemm_ex(const tw_plan *plan, const void *at, int64_t m, int64_t lda, void *ct, int64_t ldc, int out_dtype,
               int flags, const float *bias, int relu, void *stream);

/* Fused compute + all-gather for the N-sharded layer: the
 * plan's C^T rows are written to cts[0] (this GPU's full C^T buffer, offset to
 * the plan's first row) AND to every cts[1 .. n_ct-1] -- the same rows of the
 * other ranks' C^T replicas, as NVLink peer pointers (tw_ipc_open) -- from
 * the kernel's epilogue, so the reassembly rides on the stores instead of a
 * separate ncclAllGather.  No accumulate / bias.  The caller orders the call
 * against the peers' reads of their replicas (a barrier before and after). */
#define TW_MAX_PEERS 7
int tw_gemm_peers(const tw_plan *plan, const void *at, int64_t m, int64_t lda, void *const *cts, int n_ct,
                  int64_t ldc, int out_dtype, void *stream);

/* CUDA IPC for the peer replicas: a device allocation plus its 64-byte
 * cudaIpcMemHandle_t, opening a peer's handle (peer access enabled lazily),
 * and the matching releases. */
int tw_ipc_alloc(int64_t bytes, void **ptr, void *handle);
int tw_ipc_free(void *ptr);
int tw_ipc_open(const void *handle, void **ptr);
int tw_ipc_close(void *ptr);

/* Bit-exact CUDA-core variant of tw_gemm: fp32 multiply then fp32 add, in
 * ascending k per element (exactly mm_accum's rounding sequence,
 * _kernels.py:13-27).  Weights: the plan's fp32 copy when it was built with
 * TW_PLAN_F32_WEIGHTS (bit-exact with the reference for any fp32 input --
 * the drop-in's precision="exact"), else the 16-bit image (bit-exact for
 * bf16-representable weights, which proves the packed layout).  Same
 * arguments as tw_gemm; activations are fp32; not for TW_PLAN_SPLIT3 plans. */
int tw_gemm_exact(const tw_plan *plan, const float *at, int64_t m, int64_t lda, float *ct,
                  int64_t ldc, void *stream);

/* engine.py:129 (at = A^T copy) with the cast fused: a is M x K fp32 in
 * `layout` (ROW_MAJOR: a[i*K+j]; COL_MAJOR: a[j*M+i]), written as
 * at: K x M in out_dtype (TW_BF16 | TW_F16 | TW_F32) with row stride ldat. */
int tw_prep_activations(const float *a, int64_t m, int64_t k, int layout, void *at, int64_t ldat,
                        int out_dtype, void *stream);
/* tw_prep_activations for TW_PLAN_SPLIT3 plans: at2 is 2K x M bf16 (row
 * stride ldat), rows 0..K-1 = rn_bf16(A^T) and rows K..2K-1 =
 * rn_bf16(A^T - rn_bf16(A^T)) -- the high and low parts. */
int tw_prep_activations_split(const float *a, int64_t m, int64_t k, int layout, void *at2, int64_t ldat,
                              void *stream);

/* engine.py:167-181 spmm_csc (+ spmm_accum, _kernels.py:30-41): for each
 * CSC column j, ct[j, :] (+)= sum_p values[p] * at[row_idx[p], :], p in
 * ascending order, fp32 multiply then fp32 add (bit-exact with the
 * reference when at_dtype is TW_F32, or on bf16-representable inputs).
 * col_ptr/row_idx int32 and values fp32 are DEVICE arrays (N+1 / nnz).
 * accumulate = 0 overwrites every row j in [0, N) (zeros where empty). */
int tw_spmm_csc(const void *at, int at_dtype, int64_t k, int64_t m, int64_t lda, int64_t n,
                const int32_t *col_ptr, const int32_t *row_idx, const float *values, void *ct,
                int64_t ldc, int out_dtype, int accumulate, void *stream);

/* engine.py:184-198 gemm_tew: C = gemm_tw + spmm_csc (TEW overlay over all N
 * columns, including pruned ones -- pruning.py:548-549).  Implemented as
 * the SpMM writing every row followed by the TW kernel accumulating into
 * the kept rows.  nnz == 0 is exactly tw_gemm (engine.py:194-195). */
int tw_gemm_tew(const tw_plan *plan, const void *at, int64_t m, int64_t lda, const int32_t *col_ptr,
                const int32_t *row_idx, const float *values, int64_t nnz, void *ct, int64_t ldc,
                int out_dtype, void *stream);

/* Which kernel tw_gemm(plan, M, out_dtype, accumulate = 0, 16-byte aligned
 * output) runs on this device: 2 = K2 (kept-row gathers, one CTA per
 * 128-column unit), 4 = K4 (CTA pairs; plans whose tiles keep every row in
 * order, when the layer has at least one wave of 256 x 256 pair units). */
int tw_plan_kernel(const tw_plan *plan, int64_t m, int out_dtype, int *kernel);

/* Profiling hook: tw_gemm (accumulate = 0) that also records %globaltimer
 * stamps into the device buffer trace[grid * 8 units * 8 slots] (int64, ns;
 * slots: producer unit start / issued, MMA start / committed, epilogue zero
 * rows done / accumulator ready / unit stored).  Not for production use. */
int tw_gemm_traced(const tw_plan *plan, const void *at, int64_t m, int64_t lda, void *ct, int64_t ldc,
                   int out_dtype, int64_t *trace, void *stream);

/* Strided (2-D) async copy for the reference-signature API's pipelined
 * host round trip (token chunks of A in, token columns of C^T out):
 * kind 0 host->device, 1 device->host, 2 device->device. */
int tw_copy_2d(void *dst, int64_t dpitch, const void *src, int64_t spitch, int64_t width_bytes, int64_t height,
               int kind, void *stream);

/* Pruning unit scores on the GPU (pruning.py:293, :316-318; SURVEY §8(f)
 * row 4).  scores: device K x N float64, row-major (ScoreMap.scores).
 * tw_prune_col_means: out[j] = mean over rows of column j (s.mean(axis=0)).
 * tw_prune_row_means: for tile t with columns cols[off[t] .. off[t+1]),
 * out[t*K + r] = mean of s[r, cols_t] (s[:, cols].mean(axis=1)).  Both sum
 * sequentially in numpy's order, so the means are bit-identical. */
int tw_prune_col_means(const double *scores, int64_t k, int64_t n, double *out, void *stream);
int tw_prune_row_means(const double *scores, int64_t k, int64_t n, const int32_t *cols, const int64_t *off,
                       int64_t n_tiles, double *out, void *stream);

/* Number of SMs used by the persistent grid on the current device. */
int tw_device_sm_count(int *sms);

#ifdef __cplusplus
}
#endif
#endif /* TW_B200_H */
