/*
 * tw_oracle.c -- CPU restatement of the reference's TW-GEMM arithmetic.
 *
 * TEST INFRASTRUCTURE ONLY.  This file is the parity checker (and the
 * `cpu_baseline` / `--impl reference` arm of bench.py).  Nothing in the
 * product package `paper_2008_13006_b200/` links, loads or calls it; the
 * product path runs only the sm_100a CUDA kernels in libtw_b200.so.
 *
 * Restates (reference = /root/reference/pkg/src/tilewise):
 *   oracle_mm_accum    <- _kernels.py:13-27  mm_accum   (loop order k -> j -> m)
 *   oracle_spmm_accum  <- _kernels.py:30-41  spmm_accum (loop order j -> p -> m)
 *   oracle_gemm_tw     <- engine.py:126-164  _plan_tasks + gather_rows + gemm_tw
 *   oracle_gemm_dense  <- matrix.py:149-166  gemm_dense (128-column blocks)
 *
 * Arithmetic contract (the reason this is bit-identical to the numba code):
 * every `ct[r][m] += b * at[k][m]` rounds the product to fp32 and then the
 * sum to fp32 -- no FMA contraction (compile with -ffp-contract=off), no
 * reassociation (no -ffast-math), ascending k per output element.  The numba
 * kernels are compiled without fastmath and emit vmulps + vaddps, so the
 * per-element operation sequence is the same.
 *
 * Parallelism: the reference schedules whole shape-groups on threads
 * (engine.py:89-123); output rows of different tiles are disjoint, so
 * running tiles concurrently (OpenMP below, `threads` argument) gives the
 * bit-identical result.  threads <= 1 runs the exact serial order.
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

/* _kernels.py:13-27 */
void oracle_mm_accum(const float *at, int64_t lda_at, int64_t k_dim, int64_t m_dim,
                     const float *b_colmajor, int64_t ldb, int64_t n_dim,
                     const int64_t *out_rows, float *ct, int64_t ldc) {
  for (int64_t k = 0; k < k_dim; ++k) {
    const float *arow = at + k * lda_at;
    for (int64_t j = 0; j < n_dim; ++j) {
      const float bv = b_colmajor[j * ldb + k];
      float *crow = ct + out_rows[j] * ldc;
      for (int64_t m = 0; m < m_dim; ++m) {
        float p = bv * arow[m];
        crow[m] = crow[m] + p;
      }
    }
  }
}

/* _kernels.py:30-41 : CSC column j accumulates into ct row j */
void oracle_spmm_accum(const float *at, int64_t lda_at, int64_t m_dim, int64_t n_dim,
                       const int64_t *col_ptr, const int64_t *row_idx, const float *values,
                       float *ct, int64_t ldc) {
  for (int64_t j = 0; j < n_dim; ++j) {
    float *crow = ct + j * ldc;
    for (int64_t p = col_ptr[j]; p < col_ptr[j + 1]; ++p) {
      const float *arow = at + row_idx[p] * lda_at;
      const float v = values[p];
      for (int64_t m = 0; m < m_dim; ++m) {
        float t = v * arow[m];
        crow[m] = crow[m] + t;
      }
    }
  }
}

/*
 * engine.py:126-164.  Inputs are the reference's own compacted form:
 *   at          : K x M, row-contiguous (the transposed activations)
 *   tile i      : kept row indices rows[row_off[i] .. row_off[i+1])  (ascending)
 *                 col ids cols[col_off[i] .. col_off[i+1])
 *                 sub-matrix subs + sub_off[i], COL_MAJOR k_i x n_i
 *                 (data[j*k_i + r] = B[rows[r], cols[j]], pattern.py:233)
 *   ct          : N x M, zero-filled here (engine.py:102)
 * gather_rows (engine.py:61-69) packs kept rows into a k_i x M buffer; the
 * product of the packed rows equals indexing at[rows[r]] directly, so the
 * gather is folded into the row pointer below (same values, same order).
 */
void oracle_gemm_tw(const float *at, int64_t k_total, int64_t m_dim, int64_t n_total,
                    int64_t n_tiles, const int64_t *row_off, const int64_t *rows,
                    const int64_t *col_off, const int64_t *cols,
                    const int64_t *sub_off, const float *subs, float *ct, int threads) {
  (void)k_total;
  memset(ct, 0, sizeof(float) * (size_t)(n_total * m_dim));
#ifdef _OPENMP
  if (threads < 1) threads = 1;
#pragma omp parallel for schedule(dynamic, 1) num_threads(threads)
#endif
  for (int64_t i = 0; i < n_tiles; ++i) {
    const int64_t ki = row_off[i + 1] - row_off[i];
    const int64_t ni = col_off[i + 1] - col_off[i];
    if (ki == 0 || ni == 0) continue; /* engine.py:134-135 */
    const int64_t *r = rows + row_off[i];
    const int64_t *c = cols + col_off[i];
    const float *b = subs + sub_off[i];
    for (int64_t k = 0; k < ki; ++k) {
      const float *arow = at + r[k] * m_dim;
      for (int64_t j = 0; j < ni; ++j) {
        const float bv = b[j * ki + k];
        float *crow = ct + c[j] * m_dim;
        for (int64_t m = 0; m < m_dim; ++m) {
          float p = bv * arow[m];
          crow[m] = crow[m] + p;
        }
      }
    }
  }
}

/* matrix.py:149-166: b is K x N ROW_MAJOR; out ct N x M */
void oracle_gemm_dense(const float *at, int64_t k_dim, int64_t m_dim, const float *b,
                       int64_t n_dim, float *ct, int threads) {
  memset(ct, 0, sizeof(float) * (size_t)(n_dim * m_dim));
#ifdef _OPENMP
  if (threads < 1) threads = 1;
#pragma omp parallel for schedule(dynamic, 1) num_threads(threads)
#endif
  for (int64_t c0 = 0; c0 < n_dim; c0 += 128) {
    const int64_t c1 = c0 + 128 < n_dim ? c0 + 128 : n_dim;
    for (int64_t k = 0; k < k_dim; ++k) {
      const float *arow = at + k * m_dim;
      for (int64_t j = c0; j < c1; ++j) {
        const float bv = b[k * n_dim + j];
        float *crow = ct + j * m_dim;
        for (int64_t m = 0; m < m_dim; ++m) {
          float p = bv * arow[m];
          crow[m] = crow[m] + p;
        }
      }
    }
  }
}

/* engine.py:167-181 (zero-filled output, then spmm_accum) */
void oracle_spmm_csc(const float *at, int64_t m_dim, int64_t n_dim, const int64_t *col_ptr,
                     const int64_t *row_idx, const float *values, float *ct, int threads) {
  memset(ct, 0, sizeof(float) * (size_t)(n_dim * m_dim));
#ifdef _OPENMP
  if (threads < 1) threads = 1;
#pragma omp parallel for schedule(dynamic, 16) num_threads(threads)
#endif
  for (int64_t j = 0; j < n_dim; ++j) {
    float *crow = ct + j * m_dim;
    for (int64_t p = col_ptr[j]; p < col_ptr[j + 1]; ++p) {
      const float *arow = at + row_idx[p] * m_dim;
      const float v = values[p];
      for (int64_t m = 0; m < m_dim; ++m) {
        float t = v * arow[m];
        crow[m] = crow[m] + t;
      }
    }
  }
}

int oracle_max_threads(void) {
#ifdef _OPENMP
  return omp_get_max_threads();
#else
  return 1;
#endif
}
