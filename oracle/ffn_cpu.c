/*
 * CPU restatement of the executed expert FFN, for the bench's cpu_baseline /
 * --impl reference legs ONLY (test infrastructure; never linked into the
 * product).  Same packed expert format as the device path (256-byte header +
 * group-64 affine codes with fp32 scale/zero, or bf16; W2 slab-major, see
 * paper_2502_12224_b200/csrc/fate_internal.cuh), same math:
 *   y = sum_j w_j * W2_j (silu(W1_j x) * (W3_j x))
 * dequantizing on the fly with fp32 accumulation.
 *
 * Vectorised explicitly with AVX2 + FMA (8 fp32 lanes): codes are unpacked
 * 8 at a time into exact small-integer floats, each lane keeps its own
 * partial sum over the elements i = 8m + lane of a group, and the 8 lanes are
 * reduced in a fixed pairwise order ((0+4)+(2+6)) + ((1+5)+(3+7)) at the end of
 * every group.  The affine map is folded per group: s * sum(c x) + z * sum(x).
 * A persistent pthread pool splits rows over the host cores (this image has
 * no libgomp).  The reference itself has no expert FFN (pipeline.py:477-479
 * charges a constant), so this is the repo's CPU port.
 */
#include <immintrin.h>
#include <math.h>
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <unistd.h>

#define W2_SLAB_Q 64  /* quantized W2 slab width (one group) */
#define W2_SLAB_BF 8  /* bf16 W2 slab width */

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

/* fixed-order horizontal sum of 8 lanes */
static inline float hsum8(__m256 v) {
  const __m128 lo = _mm256_castps256_ps128(v), hi = _mm256_extractf128_ps(v, 1);
  const __m128 a = _mm_add_ps(lo, hi);             /* (0+4, 1+5, 2+6, 3+7) */
  const __m128 b = _mm_add_ps(a, _mm_movehl_ps(a, a)); /* ((0+4)+(2+6), (1+5)+(3+7)) */
  return _mm_cvtss_f32(_mm_add_ss(b, _mm_movehdup_ps(b)));
}

/* 8 consecutive codes (uint8 values 0..255, already unpacked) -> floats */
static inline __m256 u8x8_to_ps(const uint8_t *p) {
  return _mm256_cvtepi32_ps(_mm256_cvtepu8_epi32(_mm_loadl_epi64((const __m128i *)p)));
}

/* Unpack the 64 codes of one group into bytes, element order (element i of a
 * byte at bit i*bits, quant.py:30-39). */
static inline void unpack64(const uint8_t *c, int bits, uint8_t *out) {
  if (bits == 8) {
    memcpy(out, c, 64);
  } else if (bits == 4) {
    const __m256i v = _mm256_loadu_si256((const __m256i *)c); /* 32 bytes = 64 nibbles */
    const __m256i m = _mm256_set1_epi8(0x0F);
    const __m256i lo = _mm256_and_si256(v, m), hi = _mm256_and_si256(_mm256_srli_epi16(v, 4), m);
    /* interleave per 128-bit half: bytes b -> (lo b, hi b) */
    const __m256i a = _mm256_unpacklo_epi8(lo, hi), b = _mm256_unpackhi_epi8(lo, hi);
    /* a = [half0: elems 0..15 | half1: elems 32..47], b = [16..31 | 48..63] */
    _mm_storeu_si128((__m128i *)(out + 0), _mm256_castsi256_si128(a));
    _mm_storeu_si128((__m128i *)(out + 16), _mm256_castsi256_si128(b));
    _mm_storeu_si128((__m128i *)(out + 32), _mm256_extracti128_si256(a, 1));
    _mm_storeu_si128((__m128i *)(out + 48), _mm256_extracti128_si256(b, 1));
  } else { /* 2 bits: 16 bytes = 64 crumbs */
    const __m128i v = _mm_loadu_si128((const __m128i *)c);
    const __m128i m = _mm_set1_epi8(0x03);
    const __m128i f0 = _mm_and_si128(v, m), f1 = _mm_and_si128(_mm_srli_epi16(v, 2), m);
    const __m128i f2 = _mm_and_si128(_mm_srli_epi16(v, 4), m), f3 = _mm_and_si128(_mm_srli_epi16(v, 6), m);
    const __m128i p01l = _mm_unpacklo_epi8(f0, f1), p01h = _mm_unpackhi_epi8(f0, f1);
    const __m128i p23l = _mm_unpacklo_epi8(f2, f3), p23h = _mm_unpackhi_epi8(f2, f3);
    _mm_storeu_si128((__m128i *)(out + 0), _mm_unpacklo_epi16(p01l, p23l));
    _mm_storeu_si128((__m128i *)(out + 16), _mm_unpackhi_epi16(p01l, p23l));
    _mm_storeu_si128((__m128i *)(out + 32), _mm_unpacklo_epi16(p01h, p23h));
    _mm_storeu_si128((__m128i *)(out + 48), _mm_unpackhi_epi16(p01h, p23h));
  }
}

/* one quantized group of 64 against x[64]: s * sum(c x) + z * sx (sx = sum x, precomputed) */
static inline float group_dot(const uint8_t *codes, int bits, float s, float z, const float *x, float sx) {
  uint8_t u[64] __attribute__((aligned(32)));
  unpack64(codes, bits, u);
  __m256 acc = _mm256_setzero_ps();
  for (int m = 0; m < 8; ++m) acc = _mm256_fmadd_ps(u8x8_to_ps(u + 8 * m), _mm256_loadu_ps(x + 8 * m), acc);
  return s * hsum8(acc) + z * sx;
}

/* 8 bf16 against 8 floats */
static inline __m256 bf16x8_fma(const uint16_t *w, const float *x, __m256 acc) {
  const __m256i v = _mm256_slli_epi32(_mm256_cvtepu16_epi32(_mm_loadu_si128((const __m128i *)w)), 16);
  return _mm256_fmadd_ps(_mm256_castsi256_ps(v), _mm256_loadu_ps(x), acc);
}

/* row r of a row-major [rows x K] projection (W1 / W3) against x[K] */
static float row_dot(const uint8_t *codes, const float *sz, int bits, int64_t row, int K, const float *x,
                     const float *xsum) {
  if (bits == 16) {
    const uint16_t *w = (const uint16_t *)codes + row * K;
    __m256 acc = _mm256_setzero_ps();
    for (int i = 0; i < K; i += 8) acc = bf16x8_fma(w + i, x + i, acc);
    return hsum8(acc);
  }
  const int gpr = K / 64, gb = 64 * bits / 8;
  const uint8_t *c = codes + row * (int64_t)gpr * gb;
  float acc = 0.f;
  for (int g = 0; g < gpr; ++g)
    acc += group_dot(c + (int64_t)g * gb, bits, sz[2 * (row * gpr + g)], sz[2 * (row * gpr + g) + 1], x + 64 * g,
                     xsum[g]);
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
  const float *x, *xsum;
  int H, n;
  const uint8_t *const *bufs;
  const int *I, *bits;
  const float *w;
  float *y, *a, *asum;
  int j, off;
} ctx_t;

static void up_rows(void *p, int lo, int hi) {
  ctx_t *c = (ctx_t *)p;
  const layout_t L = make_layout(c->H, c->I[c->j], c->bits[c->j]);
  const uint8_t *b = c->bufs[c->j] + 256;
  for (int r = lo; r < hi; ++r) {
    const float u = row_dot(b + L.c1, (const float *)(b + L.s1), c->bits[c->j], r, c->H, c->x, c->xsum);
    const float v = row_dot(b + L.c3, (const float *)(b + L.s3), c->bits[c->j], r, c->H, c->x, c->xsum);
    c->a[c->off + r] = c->w[c->j] * (u / (1.0f + expf(-u)) * v);
  }
}

/* rows [lo, hi) of y: every expert's W2 slabs (slab-major, contiguous per slab) */
static void down_rows(void *p, int lo, int hi) {
  ctx_t *c = (ctx_t *)p;
  const int H = c->H;
  for (int r = lo; r < hi; ++r) c->y[r] = 0.f;
  int o = 0;
  for (int j = 0; j < c->n; ++j) {
    const int I = c->I[j], bits = c->bits[j];
    const layout_t L = make_layout(H, I, bits);
    const uint8_t *b = c->bufs[j] + 256;
    const float *a = c->a + o;
    if (bits == 16) {
      const uint16_t *w2 = (const uint16_t *)(b + L.c2);
      for (int s = 0; s < I / W2_SLAB_BF; ++s) {
        const __m256 av = _mm256_loadu_ps(a + s * W2_SLAB_BF);
        const uint16_t *slab = w2 + (int64_t)s * H * W2_SLAB_BF;
        for (int r = lo; r < hi; ++r) {
          const __m256i v = _mm256_slli_epi32(
              _mm256_cvtepu16_epi32(_mm_loadu_si128((const __m128i *)(slab + (int64_t)r * W2_SLAB_BF))), 16);
          c->y[r] += hsum8(_mm256_mul_ps(_mm256_castsi256_ps(v), av));
        }
      }
    } else {
      const int gb = 64 * bits / 8;
      const uint8_t *w2 = b + L.c2;
      const float *sz = (const float *)(b + L.s2);
      for (int s = 0; s < I / W2_SLAB_Q; ++s) {
        const float *as = a + s * W2_SLAB_Q;
        const float sa = c->asum[o / 64 + s];
        for (int r = lo; r < hi; ++r) {
          const int64_t g = (int64_t)s * H + r;
          c->y[r] += group_dot(w2 + g * gb, bits, sz[2 * g], sz[2 * g + 1], as, sa);
        }
      }
    }
    o += I;
  }
}

/* bufs[j]: packed expert buffer (header + payload); I[j], bits[j], w[j].
 * scratch: >= sum(I) + sum(I)/64 + H/64 floats. */
void fate_cpu_ffn(const float *x, int H, int n, const uint8_t *const *bufs, const int *I, const int *bits,
                  const float *w, float *y, float *scratch) {
  int tot = 0;
  for (int j = 0; j < n; ++j) tot += I[j];
  float *a = scratch, *asum = scratch + tot, *xsum = asum + tot / 64;
  for (int g = 0; g < H / 64; ++g) {
    __m256 acc = _mm256_setzero_ps();
    for (int m = 0; m < 8; ++m) acc = _mm256_add_ps(acc, _mm256_loadu_ps(x + 64 * g + 8 * m));
    xsum[g] = hsum8(acc);
  }
  ctx_t c = {x, xsum, H, n, bufs, I, bits, w, y, a, asum, 0, 0};
  for (int j = 0; j < n; ++j) {
    c.j = j;
    parallel_for(I[j], up_rows, &c);
    c.off += I[j];
  }
  for (int g = 0; g < tot / 64; ++g) {
    __m256 acc = _mm256_setzero_ps();
    for (int m = 0; m < 8; ++m) acc = _mm256_add_ps(acc, _mm256_loadu_ps(a + 64 * g + 8 * m));
    asum[g] = hsum8(acc);
  }
  parallel_for(H, down_rows, &c);
}
