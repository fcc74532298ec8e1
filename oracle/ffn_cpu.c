/*
 * CPU restatement of the executed expert FFN, for the bench's cpu_baseline /
 * --impl reference legs ONLY (test infrastructure; never linked into the
 * product).  Same packed expert format as the device path (256-byte header +
 * group-64 affine codes with fp32 scale/zero, or bf16), same math:
 *   y = sum_j w_j * W2_j (silu(W1_j x) * (W3_j x))
 * dequantizing on the fly (zero + code * scale) with fp32 accumulation,
 * a persistent pthread pool over output rows (this image has no libgomp).
 * The reference itself has no expert FFN (pipeline.py:477-479 charges a
 * constant), so this is the repo's CPU port.
 */
#include <math.h>
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <unistd.h>

typedef struct {
  int64_t c1, c3, c2, s1, s3, s2;
} layout_t;

static layout_t make_layout(int H, int I, int bits) {
  layout_t L;
  const int64_t n = (int64_t)H * I;
  if (bits == 16) {
    L.c1 = 0, L.c3 = 2 * n, L.c2 = 4 * n, L.s1 = L.s3 = L.s2 = 6 * n;
  } else {
    const int64_t cb = n * bits / 8, sb = n / 64 * 8;
    L.c1 = 0, L.c3 = cb, L.c2 = 2 * cb, L.s1 = 3 * cb, L.s3 = 3 * cb + sb, L.s2 = 3 * cb + 2 * sb;
  }
  return L;
}

static float row_dot(const uint8_t *codes, const float *sz, int bits, int64_t row, int K, const float *x) {
  float acc = 0.f;
  if (bits == 16) {
    const uint16_t *w = (const uint16_t *)codes + row * K;
    for (int i = 0; i < K; ++i) {
      uint32_t u = (uint32_t)w[i] << 16;
      float f;
      memcpy(&f, &u, 4);
      acc += f * x[i];
    }
    return acc;
  }
  const int per = 8 / bits, mask = (1 << bits) - 1, gpr = K / 64;
  const uint8_t *c = codes + row * K / per;
  for (int g = 0; g < gpr; ++g) {
    const float s = sz[2 * (row * gpr + g)], z = sz[2 * (row * gpr + g) + 1];
    float p = 0.f, sx = 0.f;
    for (int i = g * 64; i < g * 64 + 64; ++i) {
      const int q = (c[i / per] >> ((i % per) * bits)) & mask;
      p += (float)q * x[i];
      sx += x[i];
    }
    acc += s * p + z * sx;
  }
  return acc;
}


/* ---- persistent worker pool ------------------------------------------- */
typedef void (*task_fn)(void *ctx, int lo, int hi);
static pthread_mutex_t mu = PTHREAD_MUTEX_INITIALIZER;
static pthread_cond_t cv_go = PTHREAD_COND_INITIALIZER, cv_done = PTHREAD_COND_INITIALIZER;
static int n_workers = 0, gen = 0, pending = 0;
static task_fn cur_fn;
static void *cur_ctx;
static int cur_n;

static void *worker(void *arg) {
  const int id = (int)(intptr_t)arg;
  int seen = 0;
  for (;;) {
    pthread_mutex_lock(&mu);
    while (gen == seen) pthread_cond_wait(&cv_go, &mu);
    seen = gen;
    task_fn fn = cur_fn;
    void *ctx = cur_ctx;
    const int n = cur_n, nw = n_workers + 1;
    pthread_mutex_unlock(&mu);
    const int lo = (int)((int64_t)n * id / nw), hi = (int)((int64_t)n * (id + 1) / nw);
    fn(ctx, lo, hi);
    pthread_mutex_lock(&mu);
    if (--pending == 0) pthread_cond_signal(&cv_done);
    pthread_mutex_unlock(&mu);
  }
  return NULL;
}

int fate_cpu_threads(int n) {
  if (n_workers) return n_workers + 1;
  if (n <= 0) n = (int)sysconf(_SC_NPROCESSORS_ONLN);
  for (int i = 1; i < n; ++i) {
    pthread_t t;
    pthread_create(&t, NULL, worker, (void *)(intptr_t)i);
    pthread_detach(t);
  }
  n_workers = n - 1;
  return n;
}

static void parallel_for(int n, task_fn fn, void *ctx) {
  if (!n_workers) fate_cpu_threads(0);
  pthread_mutex_lock(&mu);
  cur_fn = fn, cur_ctx = ctx, cur_n = n, pending = n_workers;
  ++gen;
  pthread_cond_broadcast(&cv_go);
  pthread_mutex_unlock(&mu);
  fn(ctx, 0, (int)((int64_t)n / (n_workers + 1)));
  pthread_mutex_lock(&mu);
  while (pending) pthread_cond_wait(&cv_done, &mu);
  pthread_mutex_unlock(&mu);
}

/* ---- the FFN ------------------------------------------------------------ */
typedef struct {
  const float *x;
  int H, n;
  const uint8_t *const *bufs;
  const int *I, *bits;
  const float *w;
  float *y, *a;
  int j, off;
} ctx_t;

static void up_rows(void *p, int lo, int hi) {
  ctx_t *c = (ctx_t *)p;
  const layout_t L = make_layout(c->H, c->I[c->j], c->bits[c->j]);
  const uint8_t *b = c->bufs[c->j] + 256;
  for (int r = lo; r < hi; ++r) {
    const float u = row_dot(b + L.c1, (const float *)(b + L.s1), c->bits[c->j], r, c->H, c->x);
    const float v = row_dot(b + L.c3, (const float *)(b + L.s3), c->bits[c->j], r, c->H, c->x);
    c->a[c->off + r] = u / (1.0f + expf(-u)) * v;
  }
}

static void down_rows(void *p, int lo, int hi) {
  ctx_t *c = (ctx_t *)p;
  for (int r = lo; r < hi; ++r) {
    float acc = 0.f;
    int o = 0;
    for (int j = 0; j < c->n; ++j) {
      const layout_t L = make_layout(c->H, c->I[j], c->bits[j]);
      const uint8_t *b = c->bufs[j] + 256;
      acc += c->w[j] * row_dot(b + L.c2, (const float *)(b + L.s2), c->bits[j], r, c->I[j], c->a + o);
      o += c->I[j];
    }
    c->y[r] = acc;
  }
}

/* bufs[j]: packed expert buffer (header + payload); I[j], bits[j], w[j]. */
void fate_cpu_ffn(const float *x, int H, int n, const uint8_t *const *bufs, const int *I, const int *bits,
                  const float *w, float *y, float *scratch) {
  ctx_t c = {x, H, n, bufs, I, bits, w, y, scratch, 0, 0};
  for (int j = 0; j < n; ++j) {
    c.j = j;
    parallel_for(I[j], up_rows, &c);
    c.off += I[j];
  }
  parallel_for(H, down_rows, &c);
}
