/*
 * dfss_oracle.c -- C restatement of the reference DFSS hot loops.
 * TEST INFRASTRUCTURE ONLY: used by tests/ as a bitwise checker and by
 * bench.py as the CPU baseline ("kind": "port").  Never linked into, loaded
 * by, or called from the product package paper_2203_00091_b200.
 *
 * Each function restates one numba kernel of the reference package
 * nmattn 0.1.0 (/root/reference/pkg/src/nmattn/_kernels_numba.py) with the
 * same per-element operation order, float64 throughout.  Built with
 * -ffp-contract=off so that no multiply-add is fused (the reference runs
 * numba with fastmath off, _kernels_numba.py:1-8); results are then bitwise
 * equal to the reference, which tests/test_oracle_golden.py pins.
 */
#include <math.h>
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

/* _kernels_numba.py:16-36 -- tiled out = scale * a b^T, ascending-k accumulation. */
void oracle_gemm_abt(const double* a, const double* b, int64_t n, int64_t m, int64_t kdim,
                     double scale, double* out) {
  memset(out, 0, sizeof(double) * (size_t)(n * m));
  for (int64_t i = 0; i < n; ++i)
    for (int64_t j = 0; j < m; ++j) {
      double acc = 0.0;
      for (int64_t k = 0; k < kdim; ++k) acc += a[i * kdim + k] * b[j * kdim + k];
      out[i * m + j] = acc;
    }
  for (int64_t i = 0; i < n * m; ++i) out[i] = out[i] * scale;
}

/* _kernels_numba.py:43-59 -- dense row softmax (full-attention comparator). */
void oracle_row_softmax_dense(const double* x, int64_t rows, int64_t cols, double* out) {
  for (int64_t i = 0; i < rows; ++i) {
    const double* xr = x + i * cols;
    double* o = out + i * cols;
    double mx = xr[0];
    for (int64_t j = 1; j < cols; ++j)
      if (xr[j] > mx) mx = xr[j];
    double s = 0.0;
    for (int64_t j = 0; j < cols; ++j) {
      double e = exp(xr[j] - mx);
      o[j] = e;
      s += e;
    }
    for (int64_t j = 0; j < cols; ++j) o[j] = o[j] / s;
  }
}

/* _kernels_numba.py:66-84 -- softmax over present nonzeros (present may be NULL = all). */
void oracle_softmax_nonzeros(const double* nz, const uint8_t* present, int64_t rows, int64_t cols,
                             double* out) {
  for (int64_t i = 0; i < rows; ++i) {
    const double* x = nz + i * cols;
    const uint8_t* p = present ? present + i * cols : NULL;
    double* o = out + i * cols;
    double mx = -INFINITY;
    for (int64_t j = 0; j < cols; ++j)
      if ((!p || p[j]) && x[j] > mx) mx = x[j];
    double s = 0.0;
    for (int64_t j = 0; j < cols; ++j) {
      if (!p || p[j]) {
        double e = exp(x[j] - mx);
        o[j] = e;
        s += e;
      } else {
        o[j] = 0.0;
      }
    }
    for (int64_t j = 0; j < cols; ++j)
      if (!p || p[j]) o[j] = o[j] / s;
  }
}

/* _kernels_numba.py:91-103 -- out[i,:] += nz[i,c] * v[col[i,c],:], ascending c. */
void oracle_spmm_gather(const double* nz, const int64_t* cols, const uint8_t* present, int64_t rows,
                        int64_t nzc, const double* v, int64_t d, double* out) {
  memset(out, 0, sizeof(double) * (size_t)(rows * d));
  for (int64_t i = 0; i < rows; ++i)
    for (int64_t c = 0; c < nzc; ++c) {
      if (present && !present[i * nzc + c]) continue;
      double val = nz[i * nzc + c];
      const double* vr = v + cols[i * nzc + c] * d;
      double* o = out + i * d;
      for (int64_t j = 0; j < d; ++j) o[j] += val * vr[j];
    }
}

/* codec.py:346-360 -- nibble -> dense column of every stored nonzero (logical layout). */
void oracle_nonzero_columns(const uint8_t* meta, int64_t rows, int64_t dense_cols, int gs,
                            int64_t* cols) {
  int64_t groups = dense_cols / gs;
  for (int64_t i = 0; i < rows; ++i)
    for (int64_t g = 0; g < groups; ++g) {
      uint8_t nib = meta[i * groups + g];
      if (gs == 2) {
        cols[i * groups + g] = 2 * g + (nib == 0xE);
      } else {
        cols[i * (dense_cols / 2) + 2 * g] = 4 * g + (nib & 3);
        cols[i * (dense_cols / 2) + 2 * g + 1] = 4 * g + ((nib >> 2) & 3);
      }
    }
}

/*
 * _kernels_numba.py:110-185 -- fused score tile + prune/encode epilogue.
 * keep: [grid_rows * grid_cols] tile mask (NULL = all tiles kept).  Outputs are
 * zero-initialised here (the reference allocates with np.zeros, :115-116).
 * stats (nullable): {peak, nnz_written, nib_written}.
 */
void oracle_sddmm_compress(const double* q, const double* kmat, int64_t n, int64_t m, int64_t kdim,
                           double scale, int gs, int tile_rows, int tile_cols, const uint8_t* keep,
                           double* nonzeros, uint8_t* meta, int64_t* stats) {
  memset(nonzeros, 0, sizeof(double) * (size_t)(n * (m / 2)));
  memset(meta, 0, (size_t)(n * (m / gs)));
  int64_t grid_rows = (n + tile_rows - 1) / tile_rows;
  int64_t grid_cols = (m + tile_cols - 1) / tile_cols;
  double* tile = (double*)malloc(sizeof(double) * (size_t)tile_rows * (size_t)tile_cols);
  int64_t peak = 0, nnz = 0, nib = 0;
  for (int64_t ti = 0; ti < grid_rows; ++ti) {
    int64_t i0 = ti * tile_rows;
    int64_t ih = (i0 + tile_rows < n ? i0 + tile_rows : n) - i0;
    for (int64_t tj = 0; tj < grid_cols; ++tj) {
      if (keep && !keep[ti * grid_cols + tj]) continue;
      int64_t j0 = tj * tile_cols;
      int64_t jw = (j0 + tile_cols < m ? j0 + tile_cols : m) - j0;
      if (ih * jw > peak) peak = ih * jw;
      for (int64_t a = 0; a < ih; ++a)
        for (int64_t b = 0; b < jw; ++b) tile[a * tile_cols + b] = 0.0;
      for (int64_t k = 0; k < kdim; ++k)
        for (int64_t a = 0; a < ih; ++a) {
          double qv = q[(i0 + a) * kdim + k];
          for (int64_t b = 0; b < jw; ++b) tile[a * tile_cols + b] += qv * kmat[(j0 + b) * kdim + k];
        }
      for (int64_t a = 0; a < ih; ++a)
        for (int64_t b = 0; b < jw; ++b) tile[a * tile_cols + b] = tile[a * tile_cols + b] * scale;
      if (gs == 2) {
        int64_t g0 = j0 / 2;
        for (int64_t a = 0; a < ih; ++a) {
          int64_t r = i0 + a;
          const double* t = tile + a * tile_cols;
          for (int64_t g = 0; g < jw / 2; ++g) {
            int64_t b = 2 * g;
            if (t[b + 1] > t[b]) {
              nonzeros[r * (m / 2) + g0 + g] = t[b + 1];
              meta[r * (m / 2) + g0 + g] = 0xE;
            } else {
              nonzeros[r * (m / 2) + g0 + g] = t[b];
              meta[r * (m / 2) + g0 + g] = 0x4;
            }
            nnz += 1;
            nib += 1;
          }
        }
      } else {
        int64_t g0 = j0 / 4;
        for (int64_t a = 0; a < ih; ++a) {
          int64_t r = i0 + a;
          const double* t = tile + a * tile_cols;
          for (int64_t g = 0; g < jw / 4; ++g) {
            int64_t b = 4 * g;
            int best = 0;
            for (int u = 1; u < 4; ++u)
              if (t[b + u] > t[b + best]) best = u;
            int second = -1;
            for (int u = 0; u < 4; ++u) {
              if (u == best) continue;
              if (second < 0 || t[b + u] > t[b + second]) second = u;
            }
            int lo = best < second ? best : second;
            int hi = best < second ? second : best;
            int64_t gg = g0 + g;
            nonzeros[r * (m / 2) + 2 * gg] = t[b + lo];
            nonzeros[r * (m / 2) + 2 * gg + 1] = t[b + hi];
            meta[r * (m / 4) + gg] = (uint8_t)(lo | (hi << 2));
            nnz += 2;
            nib += 1;
          }
        }
      }
    }
  }
  free(tile);
  if (stats) {
    stats[0] = peak;
    stats[1] = nnz;
    stats[2] = nib;
  }
}

/* pipeline.py:15-32 for one (batch, head): sddmm(1/sqrt d) -> softmax_rows -> spmm. */
void oracle_nm_attention(const double* q, const double* k, const double* v, int64_t n, int64_t d,
                         int gs, double* out) {
  int64_t half = n / 2;
  double* nz = (double*)malloc(sizeof(double) * (size_t)(n * half));
  double* p = (double*)malloc(sizeof(double) * (size_t)(n * half));
  uint8_t* meta = (uint8_t*)malloc((size_t)(n * (n / gs)));
  int64_t* cols = (int64_t*)malloc(sizeof(int64_t) * (size_t)(n * half));
  oracle_sddmm_compress(q, k, n, n, d, 1.0 / sqrt((double)d), gs, 32, 64, NULL, nz, meta, NULL);
  oracle_softmax_nonzeros(nz, NULL, n, half, p);
  oracle_nonzero_columns(meta, n, n, gs, cols);
  oracle_spmm_gather(p, cols, NULL, n, half, v, d, out);
  free(nz);
  free(p);
  free(meta);
  free(cols);
}

/* dense.py:118-122 for one (batch, head): the CPU dense comparator. */
void oracle_full_attention(const double* q, const double* k, const double* v, int64_t n, int64_t d,
                           double* out) {
  double* s = (double*)malloc(sizeof(double) * (size_t)(n * n));
  double* w = (double*)malloc(sizeof(double) * (size_t)(n * n));
  double* vt = (double*)malloc(sizeof(double) * (size_t)(n * d));
  oracle_gemm_abt(q, k, n, n, d, 1.0 / sqrt((double)d), s);
  oracle_row_softmax_dense(s, n, n, w);
  for (int64_t i = 0; i < n; ++i)
    for (int64_t j = 0; j < d; ++j) vt[j * n + i] = v[i * d + j];
  oracle_gemm_abt(w, vt, n, d, n, 1.0, out);
  free(s);
  free(w);
  free(vt);
}

/* ---- batched, multi-threaded driver over independent (batch, head) slices ---- */

typedef struct {
  const double *q, *k, *v;
  double* out;
  int64_t n, d, begin, end;
  int gs, dense;
} oracle_job;

static void* oracle_worker(void* arg) {
  oracle_job* j = (oracle_job*)arg;
  int64_t nd = j->n * j->d;
  for (int64_t h = j->begin; h < j->end; ++h) {
    if (j->dense)
      oracle_full_attention(j->q + h * nd, j->k + h * nd, j->v + h * nd, j->n, j->d, j->out + h * nd);
    else
      oracle_nm_attention(j->q + h * nd, j->k + h * nd, j->v + h * nd, j->n, j->d, j->gs,
                          j->out + h * nd);
  }
  return NULL;
}

/* q,k,v,out: [bh, n, d] float64.  dense=0 -> nm_attention, dense=1 -> full_attention. */
int oracle_attention_batched(const double* q, const double* k, const double* v, int64_t bh, int64_t n,
                             int64_t d, int gs, int dense, int nthreads, double* out) {
  if (nthreads < 1) nthreads = 1;
  if (nthreads > bh) nthreads = (int)bh;
  pthread_t* th = (pthread_t*)malloc(sizeof(pthread_t) * (size_t)nthreads);
  oracle_job* jobs = (oracle_job*)malloc(sizeof(oracle_job) * (size_t)nthreads);
  for (int t = 0; t < nthreads; ++t) {
    jobs[t] = (oracle_job){q, k, v, out, n, d, bh * t / nthreads, bh * (t + 1) / nthreads, gs, dense};
    pthread_create(&th[t], NULL, oracle_worker, &jobs[t]);
  }
  for (int t = 0; t < nthreads; ++t) pthread_join(th[t], NULL);
  free(th);
  free(jobs);
  return 0;
}
