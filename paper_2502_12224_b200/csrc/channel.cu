// The transfer channel (C1) as a standalone C-ABI object: the reference's
// _Channel (pipeline.py:163-264) over real copies.  A host FIFO of pending
// transfers (enqueue, promote_ondemand, drop_stale reorder / discard them
// until they start, as in the reference); "settling" submits them in queue
// order as cudaMemcpyAsync on the channel's copy stream, at most max_inflight
// at a time, each followed by an event; a consumer stream waits for a
// transfer's event (completion) without blocking the host.  The decode engine
// runs the same discipline internally (engine.cu, Channel); this object is the
// export a caller building its own step loop binds.  device < 0 keeps the
// bookkeeping only (no CUDA calls), for host-side tests of the queue semantics.
#include <deque>
#include <vector>

#include "fate_internal.cuh"

struct fate_channel {
  struct T {
    int kind, token, layer, expert, bits;
    const void *src;
    void *dst;
    int64_t bytes;
    int64_t id;
    int state;  // 0 pending, 1 submitted, 2 complete
    cudaEvent_t ev;
  };
  int device = -1, max_inflight = 2;
  cudaStream_t stream = nullptr;
  std::deque<T> pending;
  std::vector<T> started;  // submitted or complete, submission order
  int64_t next_id = 0;
  std::vector<cudaEvent_t> ev_free;
};

namespace {

using fate::set_error;

bool step_le(int t0, int l0, int t1, int l1) { return t0 < t1 || (t0 == t1 && l0 <= l1); }

int submit_front(fate_channel *c) {
  fate_channel::T t = c->pending.front();
  c->pending.pop_front();
  t.state = 1;
  t.ev = nullptr;
  if (c->device >= 0) {
    if (!c->ev_free.empty()) {
      t.ev = c->ev_free.back();
      c->ev_free.pop_back();
    } else {
      FATE_CUDA(cudaEventCreateWithFlags(&t.ev, cudaEventDisableTiming));
    }
    FATE_CUDA(cudaMemcpyAsync(t.dst, t.src, (size_t)t.bytes, cudaMemcpyDefault, c->stream));
    FATE_CUDA(cudaEventRecord(t.ev, c->stream));
  }
  c->started.push_back(t);
  return FATE_OK;
}

// retire submitted transfers whose event completed
void retire(fate_channel *c) {
  for (auto &t : c->started)
    if (t.state == 1 && (c->device < 0 || cudaEventQuery(t.ev) == cudaSuccess)) {
      t.state = 2;
      if (t.ev) c->ev_free.push_back(t.ev);  // a completed transfer needs no event
      t.ev = nullptr;
    }
}

int in_flight(const fate_channel *c) {
  int n = 0;
  for (const auto &t : c->started) n += t.state == 1;
  return n;
}

}  // namespace

using fate::set_error;

extern "C" int fate_channel_create(int device, int max_inflight, fate_channel **out) {
  if (!out || max_inflight < 1) {
    set_error("fate_channel_create: bad arguments");
    return FATE_EINVAL;
  }
  auto *c = new fate_channel();
  c->device = device;
  c->max_inflight = max_inflight;
  if (device >= 0) {
    cudaError_t e = cudaSetDevice(device);
    if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking);
    if (e != cudaSuccess) {
      delete c;
      return fate::cuda_status(e, "fate_channel_create");
    }
  }
  *out = c;
  return FATE_OK;
}

extern "C" int fate_channel_destroy(fate_channel *c) {
  if (!c) return FATE_OK;
  if (c->device >= 0) {
    cudaSetDevice(c->device);
    cudaStreamSynchronize(c->stream);
    for (auto &t : c->started)
      if (t.ev) cudaEventDestroy(t.ev);
    for (auto e : c->ev_free) cudaEventDestroy(e);
    cudaStreamDestroy(c->stream);
  }
  delete c;
  return FATE_OK;
}

// _Channel.enqueue (pipeline.py:196-202)
extern "C" int fate_channel_enqueue(fate_channel *c, int kind, int token, int layer, int expert, int bits,
                                    const void *src, void *dst, int64_t bytes, int64_t *id_out) {
  if (!c || (kind != 0 && kind != 1) || bytes < 0 || (c->device >= 0 && bytes > 0 && (!src || !dst))) {
    set_error("fate_channel_enqueue: bad arguments (kind 0 prefetch, 1 on-demand)");
    return FATE_EINVAL;
  }
  fate_channel::T t{kind, token, layer, expert, bits, src, dst, bytes, c->next_id++, 0, nullptr};
  c->pending.push_back(t);
  if (id_out) *id_out = t.id;
  return FATE_OK;
}

// _Channel.promote_ondemand (pipeline.py:241-245): on-demand ahead of prefetch, stably
extern "C" int fate_channel_promote(fate_channel *c) {
  std::deque<fate_channel::T> urgent, rest;
  for (auto &t : c->pending) (t.kind == 1 ? urgent : rest).push_back(t);
  c->pending = urgent;
  for (auto &t : rest) c->pending.push_back(t);
  return FATE_OK;
}

// _Channel.drop_stale (pipeline.py:247-253): pending prefetches whose step <= (token, layer)
extern "C" int fate_channel_drop_stale(fate_channel *c, int token, int layer, int *n_dropped) {
  std::deque<fate_channel::T> keep;
  int n = 0;
  for (auto &t : c->pending) {
    if (t.kind == 0 && step_le(t.token, t.layer, token, layer)) ++n;
    else keep.push_back(t);
  }
  c->pending = keep;
  if (n_dropped) *n_dropped = n;
  return FATE_OK;
}

// _Channel.settle (pipeline.py:214-220) on a real copy engine: retire completed
// transfers, then start pending ones in queue order while fewer than
// max_inflight are in flight
extern "C" int fate_channel_pump(fate_channel *c) {
  if (c->device >= 0) cudaSetDevice(c->device);
  retire(c);
  while (!c->pending.empty() && in_flight(c) < c->max_inflight)
    if (int st = submit_front(c)) return st;
  return FATE_OK;
}

// _Channel.completion (pipeline.py:222-230) + the consumer's wait: start every
// transfer up to `id` in queue order, then make `stream` wait for its event
extern "C" int fate_channel_wait(fate_channel *c, int64_t id, void *stream) {
  if (c->device >= 0) cudaSetDevice(c->device);
  retire(c);
  for (auto &t : c->started)
    if (t.id == id) {
      if (t.state == 1 && c->device >= 0 && stream) FATE_CUDA(cudaStreamWaitEvent((cudaStream_t)stream, t.ev, 0));
      return FATE_OK;
    }
  bool present = false;
  for (auto &t : c->pending) present = present || t.id == id;
  if (!present) {
    set_error("fate_channel_wait: transfer vanished from the channel queue (dropped or unknown id)");
    return FATE_EINVAL;
  }
  while (!c->pending.empty()) {
    const bool last = c->pending.front().id == id;
    if (int st = submit_front(c)) return st;
    if (last) break;
  }
  if (c->device >= 0 && stream) FATE_CUDA(cudaStreamWaitEvent((cudaStream_t)stream, c->started.back().ev, 0));
  return FATE_OK;
}

// _Channel.find (pipeline.py:232-239): state -1 none, 0 pending, 1 submitted, 2 complete
extern "C" int fate_channel_find(fate_channel *c, int token, int layer, int expert, int *state, int64_t *id_out) {
  if (c->device >= 0) cudaSetDevice(c->device);
  retire(c);
  *state = -1;
  for (auto &t : c->pending)
    if (t.expert == expert && t.token == token && t.layer == layer) {
      *state = 0;
      if (id_out) *id_out = t.id;
      return FATE_OK;
    }
  for (auto it = c->started.rbegin(); it != c->started.rend(); ++it)
    if (it->expert == expert && it->token == token && it->layer == layer) {
      *state = it->state;
      if (id_out) *id_out = it->id;
      return FATE_OK;
    }
  return FATE_OK;
}

// the pending queue in order (ids) and the number of transfers in flight
extern "C" int fate_channel_pending(fate_channel *c, int64_t *ids, int max, int *n, int *n_inflight) {
  if (c->device >= 0) cudaSetDevice(c->device);
  retire(c);
  int i = 0;
  for (auto &t : c->pending) {
    if (i < max && ids) ids[i] = t.id;
    ++i;
  }
  *n = i;
  if (n_inflight) *n_inflight = in_flight(c);
  return FATE_OK;
}
