/*
 * sliceblur_oracle.c - TEST INFRASTRUCTURE ONLY (the parity checker and the
 * CPU baseline).  Nothing in the product path links or calls this file.
 *
 * A plain-C restatement of the reference running-sum slice filter,
 * /root/reference/pkg/src/sliceblur/filtering.py, op-for-op in float64 so
 * its results are bit-identical to the numpy reference (pinned against
 * tests/golden/filter_cases.npz, which was produced by running the reference):
 *
 *   oracle_filter_rows     <- filtering.py:48-64  _filter_rows
 *   oracle_separable_2d    <- filtering.py:76-104 separable_filter_2d
 *                             (rows, then columns; rows/columns are spread over
 *                             pthreads, which is bit-identical because every
 *                             row/column is independent - the reference's own
 *                             parallel=True argument, filtering.py:91-101)
 *   oracle_prefix_sum      <- filtering.py:31-36  prefix_sum
 *   oracle_filter_at       <- filtering.py:107-148 filter_at
 *
 * Build with -ffp-contract=off: numpy never fuses w*(hi-lo) + out into an FMA.
 */
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

/* One row, numpy order of operations (filtering.py:51-63):
 *   cum = cumsum(row)                        (sequential, :51)
 *   out = 0                                  (:53)
 *   for (p, w): hi = cum[min(x+p, n-1)] + max(x+p-(n-1), 0) * last   (:57-59)
 *               lo = x-p-1 < 0 ? min(x-p, 0) * first : cum[x-p-1]    (:60-62)
 *               out += w * (hi - lo)                                  (:63)      */
static void filter_one_row(const double* in, int64_t in_step, double* out, int64_t out_step, int64_t n,
                           const int64_t* radii, const double* weights, int k, double* cum, double* acc) {
  double run = 0.0;
  for (int64_t j = 0; j < n; ++j) {
    run = run + in[j * in_step];
    cum[j] = run;
  }
  const double first = in[0];
  const double last = in[(n - 1) * in_step];
  for (int64_t x = 0; x < n; ++x) acc[x] = 0.0;
  for (int i = 0; i < k; ++i) {
    const int64_t p = radii[i];
    const double w = weights[i];
    for (int64_t x = 0; x < n; ++x) {
      const int64_t hi_idx = x + p;
      const double over = (double)(hi_idx - (n - 1) > 0 ? hi_idx - (n - 1) : 0);
      const double hi = cum[hi_idx < n - 1 ? hi_idx : n - 1] + over * last;
      const int64_t lo_idx = x - p - 1;
      double lo;
      if (lo_idx < 0) {
        const double under = (double)(lo_idx + 1 < 0 ? lo_idx + 1 : 0);
        lo = under * first;
      } else {
        lo = cum[lo_idx];
      }
      acc[x] = acc[x] + w * (hi - lo);
    }
  }
  for (int64_t x = 0; x < n; ++x) out[x * out_step] = acc[x];
}

typedef struct {
  const double* in;
  double* out;
  int64_t lines, n;
  int64_t in_line, in_step, out_line, out_step;
  const int64_t* radii;
  const double* weights;
  int k;
  int64_t begin, end;
} job_t;

static void* run_job(void* arg) {
  job_t* j = (job_t*)arg;
  double* cum = (double*)malloc(sizeof(double) * (size_t)j->n);
  double* acc = (double*)malloc(sizeof(double) * (size_t)j->n);
  if (!cum || !acc) {
    free(cum);
    free(acc);
    return (void*)1;
  }
  for (int64_t l = j->begin; l < j->end; ++l)
    filter_one_row(j->in + l * j->in_line, j->in_step, j->out + l * j->out_line, j->out_step, j->n, j->radii,
                   j->weights, j->k, cum, acc);
  free(cum);
  free(acc);
  return NULL;
}

/* Filter `lines` independent 1D lines of length n (strided), over `threads` threads. */
static int filter_lines(const double* in, int64_t in_line, int64_t in_step, double* out, int64_t out_line,
                        int64_t out_step, int64_t lines, int64_t n, const int64_t* radii, const double* weights,
                        int k, int threads) {
  if (threads < 1) threads = 1;
  if (threads > 256) threads = 256;
  if (threads > lines) threads = (int)lines;
  if (threads < 1) threads = 1;
  pthread_t tid[256];
  job_t jobs[256];
  int rc = 0;
  for (int t = 0; t < threads; ++t) {
    job_t* j = &jobs[t];
    j->in = in;
    j->out = out;
    j->lines = lines;
    j->n = n;
    j->in_line = in_line;
    j->in_step = in_step;
    j->out_line = out_line;
    j->out_step = out_step;
    j->radii = radii;
    j->weights = weights;
    j->k = k;
    j->begin = lines * t / threads;
    j->end = lines * (t + 1) / threads;
    if (threads == 1) return run_job(j) ? -1 : 0;
    if (pthread_create(&tid[t], NULL, run_job, j)) return -1;
  }
  for (int t = 0; t < threads; ++t) {
    void* r = NULL;
    pthread_join(tid[t], &r);
    if (r) rc = -1;
  }
  return rc;
}

/* filtering.py:48-64 on an (m, n) row-major array. */
int oracle_filter_rows(const double* in, double* out, int64_t m, int64_t n, const int64_t* radii,
                       const double* weights, int k, int threads) {
  return filter_lines(in, n, 1, out, n, 1, m, n, radii, weights, k, threads);
}

/* filtering.py:76-104: rows into `tmp` (h*w doubles, caller-provided), then
 * columns of tmp into out.  The reference's column pass is _filter_rows on
 * rows.T; walking each column with stride w performs the same arithmetic. */
int oracle_separable_2d(const double* img, double* out, double* tmp, int64_t h, int64_t w, const int64_t* radii,
                        const double* weights, int k, int threads) {
  if (filter_lines(img, w, 1, tmp, w, 1, h, w, radii, weights, k, threads)) return -1;
  return filter_lines(tmp, 1, w, out, 1, w, w, h, radii, weights, k, threads);
}

/* filtering.py:31-36 */
void oracle_prefix_sum(const double* in, double* out, int64_t n) {
  double run = 0.0;
  for (int64_t j = 0; j < n; ++j) {
    run = run + in[j];
    out[j] = run;
  }
}

/* filtering.py:107-148: the row-filtered value of column x for every row
 * (same arithmetic as _filter_rows restricted to one column, :130-143), then
 * the 1D filter of that column (:147), gathered at each requested (x, y).
 * `cum` needs h*w doubles, `col` and `colout` need h doubles each. */
int oracle_filter_at(const double* img, int64_t h, int64_t w, const int64_t* radii, const double* weights, int k,
                     const int64_t* xs, const int64_t* ys, int64_t npts, double* values, double* cum, double* col,
                     double* colout) {
  for (int64_t y = 0; y < h; ++y) {
    double run = 0.0;
    for (int64_t x = 0; x < w; ++x) {
      run = run + img[y * w + x];
      cum[y * w + x] = run;
    }
  }
  double* lcum = (double*)malloc(sizeof(double) * (size_t)h);
  double* lacc = (double*)malloc(sizeof(double) * (size_t)h);
  if (!lcum || !lacc) {
    free(lcum);
    free(lacc);
    return -1;
  }
  for (int64_t q = 0; q < npts; ++q) {
    const int64_t x = xs[q];
    /* row_filtered_column(x), filtering.py:130-143 */
    for (int64_t y = 0; y < h; ++y) col[y] = 0.0;
    for (int i = 0; i < k; ++i) {
      const int64_t p = radii[i];
      const double wt = weights[i];
      const int64_t hi_idx = x + p;
      const double over = (double)(hi_idx - (w - 1) > 0 ? hi_idx - (w - 1) : 0);
      const int64_t lo_idx = x - p - 1;
      for (int64_t y = 0; y < h; ++y) {
        const double last = img[y * w + (w - 1)];
        const double first = img[y * w];
        const double hi = cum[y * w + (hi_idx < w - 1 ? hi_idx : w - 1)] + over * last;
        double lo;
        if (lo_idx < 0) {
          lo = (double)(lo_idx + 1 < 0 ? lo_idx + 1 : 0) * first;
        } else {
          lo = cum[y * w + lo_idx];
        }
        col[y] = col[y] + wt * (hi - lo);
      }
    }
    filter_one_row(col, 1, colout, 1, h, radii, weights, k, lcum, lacc);
    values[q] = colout[ys[q]];
  }
  free(lcum);
  free(lacc);
  return 0;
}

/* ------------------------------------------------------------------ large-image helpers
 * The BASELINE's biggest configs (32768^2 f32) do not fit the reference's
 * full-image float64 temporaries comfortably, so parity there is checked on
 * (a) full output COLUMNS - bit-identical to separable_filter_2d because they
 *     are exactly filter_at's arithmetic (filtering.py:126-148), computed with
 *     O(width) memory per thread;
 * (b) full output ROW BANDS - the column pass of rows [y0, y1) only reads
 *     row-filtered rows [y0-pmax-1, y1+pmax], so the band is filtered with the
 *     same float64 arithmetic restricted to those rows.  The column prefix then
 *     starts at the band instead of row 0, which changes float64 rounding only
 *     (|diff| ~ 1e-12 of the pixel scale; tests/test_oracle.py bounds it).
 * Sources are read in their own dtype (0 = u8, 2 = f32, 3 = f64) and
 * converted to float64 exactly, as np.asarray(image, float64) does. */

static double load_px(const void* src, int dtype, int64_t idx) {
  switch (dtype) {
    case 0: return (double)((const uint8_t*)src)[idx];
    case 1: return (double)((const uint16_t*)src)[idx];
    case 2: return (double)((const float*)src)[idx];
    default: return ((const double*)src)[idx];
  }
}

typedef struct {
  const void* src;
  int dtype;
  int64_t h, w, px_stride;
  const int64_t* radii;
  const double* weights;
  int k;
  const int64_t* xs;
  int64_t nx;
  double* cols; /* nx * h, column x_j at cols + j*h */
  int64_t y_begin, y_end;
} coljob_t;

static void* run_coljob(void* arg) {
  coljob_t* j = (coljob_t*)arg;
  const int64_t w = j->w;
  double* row = (double*)malloc(sizeof(double) * (size_t)w);
  double* cum = (double*)malloc(sizeof(double) * (size_t)w);
  if (!row || !cum) {
    free(row);
    free(cum);
    return (void*)1;
  }
  for (int64_t y = j->y_begin; y < j->y_end; ++y) {
    double run = 0.0;
    for (int64_t x = 0; x < w; ++x) {
      row[x] = load_px(j->src, j->dtype, (y * w + x) * j->px_stride);
      run = run + row[x];
      cum[x] = run;
    }
    for (int64_t q = 0; q < j->nx; ++q) {
      const int64_t x = j->xs[q];
      double acc = 0.0;
      for (int i = 0; i < j->k; ++i) {
        const int64_t p = j->radii[i];
        const int64_t hi_idx = x + p;
        const double over = (double)(hi_idx - (w - 1) > 0 ? hi_idx - (w - 1) : 0);
        const double hi = cum[hi_idx < w - 1 ? hi_idx : w - 1] + over * row[w - 1];
        const int64_t lo_idx = x - p - 1;
        const double lo = lo_idx < 0 ? (double)(lo_idx + 1 < 0 ? lo_idx + 1 : 0) * row[0] : cum[lo_idx];
        acc = acc + j->weights[i] * (hi - lo);
      }
      j->cols[q * j->h + y] = acc;
    }
  }
  free(row);
  free(cum);
  return NULL;
}

/* Full output columns xs[0..nx) of separable_filter_2d(image) for an (h, w)
 * image with pixel stride px_stride (interleaved channel c: src advanced by c).
 * out: nx * h doubles (column q at out + q*h); scratch: nx * h doubles. */
int oracle_filter_columns(const void* src, int dtype, int64_t h, int64_t w, int64_t px_stride, const int64_t* radii,
                          const double* weights, int k, const int64_t* xs, int64_t nx, double* out, double* scratch,
                          int threads) {
  if (threads < 1) threads = 1;
  if (threads > 256) threads = 256;
  if (threads > h) threads = (int)h;
  pthread_t tid[256];
  coljob_t jobs[256];
  int rc = 0;
  for (int t = 0; t < threads; ++t) {
    coljob_t* j = &jobs[t];
    j->src = src;
    j->dtype = dtype;
    j->h = h;
    j->w = w;
    j->px_stride = px_stride;
    j->radii = radii;
    j->weights = weights;
    j->k = k;
    j->xs = xs;
    j->nx = nx;
    j->cols = scratch;
    j->y_begin = h * t / threads;
    j->y_end = h * (t + 1) / threads;
    if (pthread_create(&tid[t], NULL, run_coljob, j)) return -1;
  }
  for (int t = 0; t < threads; ++t) {
    void* r = NULL;
    pthread_join(tid[t], &r);
    if (r) rc = -1;
  }
  if (rc) return rc;
  return filter_lines(scratch, h, 1, out, h, 1, nx, h, radii, weights, k, threads);
}

/* Output rows [y0, y1) (all columns) of separable_filter_2d for an (h, w)
 * image, using only input rows [y0-pmax-1, y1+pmax] (clamped).
 * out: (y1-y0) * w doubles; scratch: (y1-y0+2*pmax+2) * w doubles. */
int oracle_filter_band(const void* src, int dtype, int64_t h, int64_t w, int64_t px_stride, const int64_t* radii,
                       const double* weights, int k, int64_t y0, int64_t y1, double* out, double* scratch,
                       int threads) {
  const int64_t pmax = radii[k - 1];
  int64_t a = y0 - pmax - 1, b = y1 + pmax;
  if (a < 0) a = 0;
  if (b > h) b = h;
  const int64_t n = b - a;
  /* row pass over rows [a, b) into scratch (n x w) */
  double* rowbuf = (double*)malloc(sizeof(double) * (size_t)(n * w));
  if (!rowbuf) return -1;
  for (int64_t y = a; y < b; ++y)
    for (int64_t x = 0; x < w; ++x) rowbuf[(y - a) * w + x] = load_px(src, dtype, (y * w + x) * px_stride);
  int rc = filter_lines(rowbuf, w, 1, scratch, w, 1, n, w, radii, weights, k, threads);
  free(rowbuf);
  if (rc) return rc;
  /* column pass over the band: outputs [y0, y1) never read outside [a, b)
   * except through the true image edges, where a == 0 / b == h */
  double* colout = (double*)malloc(sizeof(double) * (size_t)(n * w));
  if (!colout) return -1;
  rc = filter_lines(scratch, 1, w, colout, 1, w, w, n, radii, weights, k, threads);
  if (!rc)
    for (int64_t y = y0; y < y1; ++y) memcpy(out + (y - y0) * w, colout + (y - a) * w, sizeof(double) * (size_t)w);
  free(colout);
  return rc;
}
