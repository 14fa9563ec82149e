/*
 * dmlp_oracle.c -- CPU restatement of the reference hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  This file is the parity checker (and the CPU
 * baseline timed by bench.py's cpu_baseline / --impl reference legs).  The
 * product path (paper_1003_0358_b200/) never links, loads or calls it.
 *
 * It restates, operation for operation, the arithmetic of the reference
 * package mounted at /root/reference/pkg/src/deepmlp (numba "tiled" variant
 * and the numpy/scipy deformation pipeline).  Every function cites the
 * reference file:line it follows.  Compile with -ffp-contract=off: the
 * reference (numba without fastmath, numpy elementwise) never fuses a
 * multiply into an add, so neither may we.
 *
 * Parity pinning: tests/test_oracle_golden.py checks this file bit-for-bit
 * against golden vectors produced by importing the reference itself
 * (tests/golden/make_golden.py).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#include <pthread.h>

/* Persistent fork/join pool: parallel-for over [0, n) in static chunks
 * (replaces numba's prange; every index's arithmetic is independent of the
 * split, so results do not depend on the thread count). */
static int g_threads = 1;
typedef void (*or_body_fn)(void *ctx, int64_t lo, int64_t hi);
#define OR_MAX_THREADS 256
static pthread_mutex_t g_mu = PTHREAD_MUTEX_INITIALIZER;
static pthread_cond_t g_cv_go = PTHREAD_COND_INITIALIZER, g_cv_done = PTHREAD_COND_INITIALIZER;
static int g_pool_size = 0;          /* worker threads started (excl. caller) */
static unsigned long g_gen = 0;      /* task generation */
static int g_pending = 0;            /* workers still running the task */
static or_body_fn g_fn;
static void *g_ctx;
static int64_t g_n;
static int g_T;                      /* participants of the current task */

static void *or_worker(void *arg) {
  const int id = (int)(intptr_t)arg; /* 1..pool */
  unsigned long seen = 0;
  for (;;) {
    pthread_mutex_lock(&g_mu);
    while (g_gen == seen) pthread_cond_wait(&g_cv_go, &g_mu);
    seen = g_gen;
    const int T = g_T;
    or_body_fn fn = g_fn;
    void *ctx = g_ctx;
    const int64_t n = g_n;
    pthread_mutex_unlock(&g_mu);
    if (id < T) fn(ctx, n * id / T, n * (id + 1) / T);
    pthread_mutex_lock(&g_mu);
    if (--g_pending == 0) pthread_cond_signal(&g_cv_done);
    pthread_mutex_unlock(&g_mu);
  }
  return NULL;
}

static void or_parallel_for(int64_t n, or_body_fn fn, void *ctx) {
  int T = g_threads;
  if (T > n) T = (int)n;
  if (T <= 1) { fn(ctx, 0, n); return; }
  pthread_mutex_lock(&g_mu);
  while (g_pool_size < T - 1 && g_pool_size < OR_MAX_THREADS - 1) {
    pthread_t th;
    g_pool_size++;
    pthread_create(&th, NULL, or_worker, (void *)(intptr_t)g_pool_size);
    pthread_detach(th);
  }
  g_fn = fn; g_ctx = ctx; g_n = n; g_T = T;
  g_pending = g_pool_size;
  g_gen++;
  pthread_cond_broadcast(&g_cv_go);
  pthread_mutex_unlock(&g_mu);
  fn(ctx, 0, n / T);
  pthread_mutex_lock(&g_mu);
  while (g_pending > 0) pthread_cond_wait(&g_cv_done, &g_mu);
  pthread_mutex_unlock(&g_mu);
}

#define OR_A 1.7159f   /* network.py:13 */
#define OR_B 0.6666f   /* network.py:14 */
#define OR_GRID 29     /* deform.py:21 */

/* ------------------------------------------------------------------ */
/* RNG: rng.py:19-38 (splitmix64 key chain) + numpy Philox4x64-10      */
/* ------------------------------------------------------------------ */

uint64_t or_splitmix64(uint64_t x) { /* rng.py:19-24 */
  x = x + 0x9E3779B97F4A7C15ULL;
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ULL;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBULL;
  return x ^ (x >> 31);
}

/* rng.py:27-32 -- key = (h, splitmix(h)), h chained over (seed, *path). */
void or_stream_key(uint64_t seed, const uint64_t *path, int npath, uint64_t key[2]) {
  uint64_t h = or_splitmix64(seed);
  for (int i = 0; i < npath; i++) h = or_splitmix64(h ^ path[i]);
  key[0] = h;
  key[1] = or_splitmix64(h);
}

static inline void mulhilo64(uint64_t a, uint64_t b, uint64_t *hi, uint64_t *lo) {
  unsigned __int128 p = (unsigned __int128)a * b;
  *hi = (uint64_t)(p >> 64);
  *lo = (uint64_t)p;
}

/* numpy Philox4x64-10 (Random123 constants); counter (ctr) is the block
 * counter *after* numpy's pre-increment, i.e. the first block uses ctr=1. */
void or_philox_block(const uint64_t key_in[2], uint64_t ctr, uint64_t out[4]) {
  uint64_t c0 = ctr, c1 = 0, c2 = 0, c3 = 0;
  uint64_t k0 = key_in[0], k1 = key_in[1];
  for (int r = 0; r < 10; r++) {
    uint64_t hi0, lo0, hi1, lo1;
    mulhilo64(0xD2E7470EE14C6C93ULL, c0, &hi0, &lo0);
    mulhilo64(0xCA5A826395121157ULL, c2, &hi1, &lo1);
    uint64_t n0 = hi1 ^ c1 ^ k0, n1 = lo1, n2 = hi0 ^ c3 ^ k1, n3 = lo0;
    c0 = n0; c1 = n1; c2 = n2; c3 = n3;
    k0 += 0x9E3779B97F4A7C15ULL;
    k1 += 0xBB67AE8584CAA73BULL;
  }
  out[0] = c0; out[1] = c1; out[2] = c2; out[3] = c3;
}

/* First n u64 words of the stream substream(key). */
void or_philox_words(const uint64_t key[2], int64_t n, uint64_t *out) {
  uint64_t blk[4];
  for (int64_t i = 0; i < n; i += 4) {
    or_philox_block(key, (uint64_t)(i / 4) + 1, blk);
    for (int k = 0; k < 4 && i + k < n; k++) out[i + k] = blk[k];
  }
}

static inline double u53(uint64_t w) { /* numpy next_double */
  return (double)(w >> 11) * (1.0 / 9007199254740992.0);
}
static inline double uniform(double lo, double hi, uint64_t w) { /* numpy random_uniform */
  double range = hi - lo;
  return lo + range * u53(w);
}

/* ------------------------------------------------------------------ */
/* Deformation: deform.py:87-214                                       */
/* ------------------------------------------------------------------ */

/* deform.py:87-99 + mnist_io.py:137-139 (all float32). */
void or_upscale(const uint8_t *img /*28x28*/, float *out /*29x29*/) {
  float n[28 * 28];
  for (int i = 0; i < 28 * 28; i++) n[i] = ((float)img[i] / 127.5f) - 1.0f;
  for (int r = 0; r < OR_GRID; r++) {
    int r0 = r - 1 < 0 ? 0 : r - 1, r1 = r > 27 ? 27 : r;
    for (int c = 0; c < OR_GRID; c++) {
      int c0 = c - 1 < 0 ? 0 : c - 1, c1 = c > 27 ? 27 : c;
      float s = n[r0 * 28 + c0] + n[r0 * 28 + c1];
      s = s + n[r1 * 28 + c0];
      s = s + n[r1 * 28 + c1];
      out[r * OR_GRID + c] = 0.25f * s;
    }
  }
}

/* numpy pairwise sum (n < 128 branch: 8 accumulators, then the tail). */
static double np_pairwise_sum(const double *a, int n) {
  if (n < 8) {
    double res = 0.0;  /* numpy starts from -0.0 for n<8; +0 and -0 agree for n>0 non-degenerate */
    for (int i = 0; i < n; i++) res += a[i];
    return res;
  }
  double r[8];
  for (int k = 0; k < 8; k++) r[k] = a[k];
  int i;
  for (i = 8; i < n - (n % 8); i += 8)
    for (int k = 0; k < 8; k++) r[k] += a[i + k];
  double res = ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]));
  for (; i < n; i++) res += a[i];
  return res;
}

/* deform.py:102-109 */
void or_gaussian_kernel_1d(double sigma, int size, double *g) {
  int half = size / 2;
  for (int k = 0; k < size; k++) {
    double off = (double)k - (double)half;
    g[k] = exp(-(off * off) / (2.0 * sigma * sigma));
  }
  double s = np_pairwise_sum(g, size);
  for (int k = 0; k < size; k++) g[k] = g[k] / s;
}

/* scipy.ndimage.convolve1d, mode=constant cval=0, symmetric kernel path:
 * out = x[c]*g0 + sum_{k=1..h} (x[c-k]+x[c+k])*g(k), k descending. */
static void conv1d_sym(const double *in, double *out, const double *g, int size,
                       int axis) {
  int h = size / 2;
  for (int r = 0; r < OR_GRID; r++)
    for (int c = 0; c < OR_GRID; c++) {
      int p = axis == 0 ? r : c;
      double xc = axis == 0 ? in[r * OR_GRID + c] : in[r * OR_GRID + c];
      double acc = xc * g[h];
      for (int k = h; k >= 1; k--) {
        int lo = p - k, hi = p + k;
        double xl = 0.0, xh = 0.0;
        if (lo >= 0) xl = axis == 0 ? in[lo * OR_GRID + c] : in[r * OR_GRID + lo];
        if (hi < OR_GRID) xh = axis == 0 ? in[hi * OR_GRID + c] : in[r * OR_GRID + hi];
        acc = acc + (xl + xh) * g[h + k];
      }
      out[r * OR_GRID + c] = acc;
    }
}

/* deform.py:119-133 for one field: noise -> conv axis0 -> conv axis1 -> *alpha */
static void elastic_field(const double *noise, const double *g, int size, double alpha,
                          double *field) {
  double tmp[OR_GRID * OR_GRID];
  conv1d_sym(noise, tmp, g, size, 0);
  conv1d_sym(tmp, field, g, size, 1);
  for (int i = 0; i < OR_GRID * OR_GRID; i++) field[i] = alpha * field[i];
}

/* deform.py:148-200 given the raw draws. mode 0 = rotation, 1 = shear. */
static void compose_and_warp(const float *up, const double *edx, const double *edy,
                             int mode, double angle, double sx, double sy, float *out) {
  const double center = (OR_GRID - 1) / 2.0;
  double rad = angle * (3.141592653589793 / 180.0); /* np.deg2rad */
  double cs = cos(rad), sn = sin(rad), tn = tan(rad);
  for (int r = 0; r < OR_GRID; r++)
    for (int c = 0; c < OR_GRID; c++) {
      double y = (double)r - center, x = (double)c - center;
      double xs = sx * x, ys = sy * y, xr, yr;
      if (mode == 0) {
        xr = cs * xs - sn * ys;
        yr = sn * xs + cs * ys;
      } else {
        xr = xs + tn * ys;
        yr = ys;
      }
      double dx = (xr - x) + edx[r * OR_GRID + c];
      double dy = (yr - y) + edy[r * OR_GRID + c];
      double sr = (double)r + dy, sc = (double)c + dx;
      double fl_r = floor(sr), fl_c = floor(sc);
      long i0 = (long)fl_r, j0 = (long)fl_c;
      double fr = sr - (double)i0, fc = sc - (double)j0;
      double v[4];
      for (int q = 0; q < 4; q++) {
        long ii = i0 + (q >> 1), jj = j0 + (q & 1);
        int valid = ii >= 0 && ii < OR_GRID && jj >= 0 && jj < OR_GRID;
        v[q] = valid ? (double)up[ii * OR_GRID + jj] : -1.0;
      }
      double o = (1.0 - fr) * (1.0 - fc) * v[0];
      o = o + (1.0 - fr) * fc * v[1];
      o = o + fr * (1.0 - fc) * v[2];
      o = o + fr * fc * v[3];
      if (o < -1.0) o = -1.0;
      if (o > 1.0) o = 1.0;
      out[r * OR_GRID + c] = (float)o;
    }
}

typedef struct {
  double sigma_lo, sigma_hi, alpha_lo, alpha_hi, beta_default, beta_reduced, gamma_lo,
      gamma_hi;
  int kernel_size;
} or_deform_params;

/* deform.py:203-214 driven by substream(seed, 2, epoch, index) (deform.py:237). */
void or_deform_image(const uint8_t *img, int digit, uint64_t seed, uint64_t epoch,
                     uint64_t index, const or_deform_params *p, float *out) {
  uint64_t path[3] = {2, epoch, index}, key[2];
  or_stream_key(seed, path, 3, key);
  const int N = OR_GRID * OR_GRID;
  uint64_t w[2 + 2 * OR_GRID * OR_GRID + 5];
  or_philox_words(key, 2 + 2 * N + 5, w);
  float up[OR_GRID * OR_GRID];
  or_upscale(img, up);
  double sigma = uniform(p->sigma_lo, p->sigma_hi, w[0]);
  double alpha = uniform(p->alpha_lo, p->alpha_hi, w[1]);
  double g[64];
  or_gaussian_kernel_1d(sigma, p->kernel_size, g);
  double noise[OR_GRID * OR_GRID], edx[OR_GRID * OR_GRID], edy[OR_GRID * OR_GRID];
  for (int i = 0; i < N; i++) noise[i] = uniform(-1.0, 1.0, w[2 + i]);
  elastic_field(noise, g, p->kernel_size, alpha, edx);
  for (int i = 0; i < N; i++) noise[i] = uniform(-1.0, 1.0, w[2 + N + i]);
  elastic_field(noise, g, p->kernel_size, alpha, edy);
  const uint64_t *a = w + 2 + 2 * N;
  int mode = (int)((((a[0] & 0xFFFFFFFFULL) * 2ULL) >> 32) & 1ULL); /* integers(0,2) */
  double beta = (digit == 1 || digit == 7) ? p->beta_reduced : p->beta_default;
  double angle = uniform(-beta, beta, a[1]);
  double gamma = uniform(p->gamma_lo, p->gamma_hi, a[2]);
  double sx = uniform(1.0 - gamma / 100.0, 1.0 + gamma / 100.0, a[3]);
  double sy = uniform(1.0 - gamma / 100.0, 1.0 + gamma / 100.0, a[4]);
  compose_and_warp(up, edx, edy, mode, angle, sx, sy, out);
}

/* Injected-field variant: same pipeline, raw draws supplied by the caller. */
void or_deform_injected(const uint8_t *img, const double *noise_dx, const double *noise_dy,
                        double sigma, double alpha, int mode, double angle, double sx,
                        double sy, int kernel_size, float *out) {
  float up[OR_GRID * OR_GRID];
  or_upscale(img, up);
  double g[64], edx[OR_GRID * OR_GRID], edy[OR_GRID * OR_GRID];
  or_gaussian_kernel_1d(sigma, kernel_size, g);
  elastic_field(noise_dx, g, kernel_size, alpha, edx);
  elastic_field(noise_dy, g, kernel_size, alpha, edy);
  compose_and_warp(up, edx, edy, mode, angle, sx, sy, out);
}

typedef struct {
  const uint8_t *imgs, *labels; int64_t first; uint64_t seed, epoch;
  const or_deform_params *p; float *out;
} deform_ctx;
static void deform_body(void *c, int64_t lo, int64_t hi) {
  deform_ctx *d = (deform_ctx *)c;
  for (int64_t i = lo; i < hi; i++)
    or_deform_image(d->imgs + i * 784, d->labels[i], d->seed, d->epoch,
                    (uint64_t)(d->first + i), d->p, d->out + i * OR_GRID * OR_GRID);
}
void or_deform_batch(const uint8_t *imgs, const uint8_t *labels, int64_t first, int64_t n,
                     uint64_t seed, uint64_t epoch, const or_deform_params *p, float *out,
                     int threads) {
  int saved = g_threads;
  if (threads > 0) g_threads = threads;
  deform_ctx d = {imgs, labels, first, seed, epoch, p, out};
  or_parallel_for(n, deform_body, &d);
  g_threads = saved;
}

void or_upscale_batch(const uint8_t *imgs, int64_t n, float *out) {
  for (int64_t i = 0; i < n; i++) or_upscale(imgs + i * 784, out + i * 841);
}

/* ------------------------------------------------------------------ */
/* Training kernels: kernels.py (tiled variant, DEFAULT_SCHEME)        */
/* ------------------------------------------------------------------ */

/* kernels.py:100-126: 32-wide segment partials summed sequentially, segment
 * partials summed in ascending order, then + bias; y = A*tanhf(B*a). */
typedef struct { const float *w; int fo, fi; const float *x; float *a, *y; } fp_ctx;
static void fp_body(void *c, int64_t lo, int64_t hi) {
  fp_ctx *f = (fp_ctx *)c;
  const float *w = f->w, *x = f->x;
  const int fi = f->fi, ld = fi + 1;
  float *a = f->a, *y = f->y;
  for (int64_t j = lo; j < hi; j++) {
    const float *row = w + (int64_t)j * ld;
    float acc = 0.0f;
    for (int base = 0; base < fi; base += 32) {
      int top = base + 32 < fi ? base + 32 : fi;
      float part = 0.0f;
      for (int i = base; i < top; i++) part = part + row[i] * x[i];
      acc = acc + part;
    }
    acc = acc + row[fi];
    a[j] = acc;
    y[j] = OR_A * tanhf(OR_B * acc);
  }
}
void or_fp_tiled(const float *w, int fo, int fi, const float *x, float *a, float *y) {
  fp_ctx f = {w, fo, fi, x, a, y};
  or_parallel_for(fo, fp_body, &f);
}

/* kernels.py:129-165: per column i and 32-row tile, sequential sum over the
 * tile's 32 rows (zero rows pad the last tile), tile sums in ascending
 * order, then the hidden derivative which numba evaluates in float64
 * (int literal 1 - float32 promotes), see SURVEY App. A.4. */
typedef struct { const float *w; int fo, fi; const float *dd, *a_up; float *du; } bp_ctx;
static void bp_body(void *c, int64_t blo, int64_t bhi) {
  bp_ctx *b = (bp_ctx *)c;
  const float *w = b->w, *dd = b->dd, *a_up = b->a_up;
  float *du = b->du;
  const int fo = b->fo, fi = b->fi, ld = fi + 1;
  const int ntiles = (fo + 31) / 32;
  const float AB = OR_A * OR_B;
  for (int ib = (int)blo * 64; ib < (int)bhi * 64 && ib < fi; ib += 64) {
    int ie = ib + 64 < fi ? ib + 64 : fi;
    float tot[64], part[64];
    for (int i = ib; i < ie; i++) tot[i - ib] = 0.0f;
    for (int tj = 0; tj < ntiles; tj++) {
      for (int i = ib; i < ie; i++) part[i - ib] = 0.0f;
      for (int jj = 0; jj < 32; jj++) {
        int j = tj * 32 + jj;
        if (j < fo) {
          const float *row = w + (int64_t)j * ld;
          float d = dd[j];
          for (int i = ib; i < ie; i++) part[i - ib] = part[i - ib] + row[i] * d;
        } else {
          for (int i = ib; i < ie; i++) part[i - ib] = part[i - ib] + 0.0f * 0.0f;
        }
      }
      for (int i = ib; i < ie; i++) tot[i - ib] = tot[i - ib] + part[i - ib];
    }
    for (int i = ib; i < ie; i++) {
      float t = tanhf(OR_B * a_up[i]);
      float tt = t * t;
      double deriv = (double)AB * (1.0 - (double)tt);
      du[i] = (float)((double)tot[i - ib] * deriv);
    }
  }
}
void or_bp_tiled(const float *w, int fo, int fi, const float *dd, const float *a_up,
                 float *du) {
  bp_ctx b = {w, fo, fi, dd, a_up, du};
  or_parallel_for((fi + 63) / 64, bp_body, &b);
}

/* kernels.py:168-183 (bit-identical to _update_naive 86-94):
 * d = eta*delta_j; w_ji = w_ji + d*y_i; bias += d. */
typedef struct { float *w; int fi; const float *delta, *yin; float eta; } up_ctx;
static void up_body(void *c, int64_t lo, int64_t hi) {
  up_ctx *u = (up_ctx *)c;
  const int fi = u->fi, ld = fi + 1;
  for (int64_t j = lo; j < hi; j++) {
    float *row = u->w + j * ld;
    float d = u->eta * u->delta[j];
    for (int i = 0; i < fi; i++) row[i] = row[i] + d * u->yin[i];
    row[fi] = row[fi] + d;
  }
}
void or_update(float *w, int fo, int fi, const float *delta, const float *yin, float eta) {
  up_ctx u = {w, fi, delta, yin, eta};
  or_parallel_for(fo, up_body, &u);
}

/* kernels.py:58-94 naive references (used by tests of the tolerance story). */
void or_fp_naive(const float *w, int fo, int fi, const float *x, float *a, float *y) {
  const int ld = fi + 1;
  for (int j = 0; j < fo; j++) {
    float acc = 0.0f;
    for (int i = 0; i < fi; i++) acc = acc + w[(int64_t)j * ld + i] * x[i];
    acc = acc + w[(int64_t)j * ld + fi];
    a[j] = acc;
    y[j] = OR_A * tanhf(OR_B * acc);
  }
}

/* kernels.py:74-83 _bp_naive: acc = delta_up[i] (zero) + sum over j in
 * ascending order of w_ji * delta_j (mul then add), then the f64 derivative
 * product exactly as the tiled reduce (numba promotes 1 - t*t to f64). */
void or_bp_naive(const float *w, int fo, int fi, const float *dd, const float *a_up,
                 float *du) {
  const int ld = fi + 1;
  const float AB = OR_A * OR_B;
  for (int i = 0; i < fi; i++) {
    float acc = 0.0f;
    for (int j = 0; j < fo; j++) acc = acc + w[(int64_t)j * ld + i] * dd[j];
    const float t = tanhf(OR_B * a_up[i]);
    const float tt = t * t;
    du[i] = (float)((double)acc * ((double)AB * (1.0 - (double)tt)));
  }
}

float or_tanhf(float x) { return tanhf(x); }

int or_set_threads(int n) {
  if (n > 0) g_threads = n > OR_MAX_THREADS ? OR_MAX_THREADS : n;
  return g_threads;
}
