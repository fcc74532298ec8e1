// K2: ARC on the device, executed by one warp over a shared-memory copy of a
// layer's lists (cache.py:104-179).  Lengths and p are kept replicated in
// every lane's registers so control flow is warp-uniform; list edits are
// warp-parallel shifts separated by __syncwarp().
#pragma once

#include "engine_dev.cuh"

namespace fate {

struct WarpArc {
  ArcLayer *s;  // shared-memory copy
  int c, n1, n2, nb1, nb2;
  double p;

  __device__ void load(const ArcLayer *g, ArcLayer *sm) {
    s = sm;
    const int lane = threadIdx.x & 31;
    const int4 *src = reinterpret_cast<const int4 *>(g);
    int4 *dst = reinterpret_cast<int4 *>(sm);
    for (int i = lane; i < (int)(sizeof(ArcLayer) / 16); i += 32) dst[i] = src[i];
    __syncwarp();
    c = sm->c, n1 = sm->n1, n2 = sm->n2, nb1 = sm->nb1, nb2 = sm->nb2, p = sm->p;
  }

  // lists already copied into shared memory (by the whole block)
  __device__ void attach(ArcLayer *sm) {
    s = sm;
    c = sm->c, n1 = sm->n1, n2 = sm->n2, nb1 = sm->nb1, nb2 = sm->nb2, p = sm->p;
  }

  __device__ void store(ArcLayer *g) {
    const int lane = threadIdx.x & 31;
    if (lane == 0) s->n1 = n1, s->n2 = n2, s->nb1 = nb1, s->nb2 = nb2, s->p = p;
    __syncwarp();
    const int4 *src = reinterpret_cast<const int4 *>(s);
    int4 *dst = reinterpret_cast<int4 *>(g);
    for (int i = lane; i < (int)(sizeof(ArcLayer) / 16); i += 32) dst[i] = src[i];
    __syncwarp();
  }

  __device__ static int find(const int32_t *lst, int n, int x) {
    const int lane = threadIdx.x & 31;
    for (int base = 0; base < n; base += 32) {
      const int i = base + lane;
      const unsigned m = __ballot_sync(0xffffffffu, i < n && lst[i] == x);
      if (m) return base + __ffs(m) - 1;
    }
    return -1;
  }

  __device__ static void remove_at(int32_t *lst, int &n, int i) {
    const int lane = threadIdx.x & 31;
    for (int base = i; base < n - 1; base += 32) {
      const int j = base + lane;
      const int v = j < n - 1 ? lst[j + 1] : 0;
      __syncwarp();
      if (j < n - 1) lst[j] = v;
      __syncwarp();
    }
    --n;
  }

  __device__ static void push(int32_t *lst, int &n, int x) {
    if ((threadIdx.x & 31) == 0) lst[n] = x;
    __syncwarp();
    ++n;
  }

  __device__ int pop_front(int32_t *lst, int &n) {
    const int v = lst[0];
    remove_at(lst, n, 0);
    return v;
  }

  // REPLACE (cache.py:128-135); returns the expert demoted to a ghost list.
  __device__ int replace(bool x_in_b2) {
    if (n1 > 0 && ((double)n1 > p || (x_in_b2 && (double)n1 == p))) {
      const int v = pop_front(s->t1, n1);
      push(s->b1, nb1, v);
      return v;
    }
    if (n2 > 0) {
      const int v = pop_front(s->t2, n2);
      push(s->b2, nb2, v);
      return v;
    }
    if (n1 > 0) {
      const int v = pop_front(s->t1, n1);
      push(s->b1, nb1, v);
      return v;
    }
    return -1;
  }

  // ARC access (cache.py:137-179).  Returns 1 on a resident hit; *victim is
  // the expert that left T1 u T2 (or -1).
  __device__ int access(int x, int *victim) {
    *victim = -1;
    if (c < 1) return 0;
    int i = find(s->t1, n1, x);
    if (i >= 0) {
      remove_at(s->t1, n1, i);
      push(s->t2, n2, x);
      return 1;
    }
    i = find(s->t2, n2, x);
    if (i >= 0) {
      remove_at(s->t2, n2, i);
      push(s->t2, n2, x);
      return 1;
    }
    i = find(s->b1, nb1, x);
    if (i >= 0) {
      const double d = fmax(1.0, __ddiv_rn((double)nb2, (double)nb1));
      p = fmin((double)c, __dadd_rn(p, d));
      *victim = replace(false);
      remove_at(s->b1, nb1, find(s->b1, nb1, x));
      push(s->t2, n2, x);
      return 0;
    }
    i = find(s->b2, nb2, x);
    if (i >= 0) {
      const double d = fmax(1.0, __ddiv_rn((double)nb1, (double)nb2));
      p = fmax(0.0, __dsub_rn(p, d));
      *victim = replace(true);
      remove_at(s->b2, nb2, find(s->b2, nb2, x));
      push(s->t2, n2, x);
      return 0;
    }
    // full miss: case IV-A / IV-B
    if (n1 + nb1 == c) {
      if (n1 < c) {
        pop_front(s->b1, nb1);
        *victim = replace(false);
      } else {
        *victim = pop_front(s->t1, n1);
      }
    } else {
      const int tot = n1 + nb1 + n2 + nb2;
      if (tot >= c) {
        if (tot == 2 * c) pop_front(s->b2, nb2);
        *victim = replace(false);
      }
    }
    push(s->t1, n1, x);
    return 0;
  }
};

}  // namespace fate
