// eq_queues.cu — the reference's queue operator API as a batch of independent
// GPU queues: make_queue / enqueue / pop_due / occupancy (queues.py:636-692,
// events.py:99-141), all kinds the network path uses plus LossyRing.
//
// One handle holds Q queues of one kind that advance together (one pop per
// step for all).  enqueue() takes a batch of events in CALL order; events of
// different queues are independent, events of one queue must be applied in
// call order (accept/drop and floating-point merge order depend on it), so a
// batch is stably sorted by queue (CUB radix sort) and each queue's run is
// applied sequentially by one thread.  Payloads are DualScalar-shaped
// (weight primal, weight tangent, time tangent) and merged in float/double in
// insertion order — the same order and arithmetic as the Python classes, so
// fp64 results are bitwise the reference's (tests/test_gpu_queues.py).
//
// Errors follow the reference exactly for a batch: the first offending event
// in call order raises (CausalityError / CapabilityError), and every event
// before it — in any queue — is applied, none after it.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>
#include <string>
#include <vector>

#include <cub/cub.cuh>

#include "../../include/eventq_b200.h"

namespace {

constexpr int kInf = 0x7fffffff;

template <typename T>
struct Ev {
  int due;
  int seq;
  T w, dw, tt;
};

template <typename T>
struct QView {
  int kind, Q, cap;
  int now;
  // ring / lossyring: slots [Q][cap]
  T* sw;
  T* sdw;
  T* swtt;
  unsigned char* occ;
  int* count;             // occupied slots (ring) / stored events (others)
  long long* aliased;     // lossyring
  long long* merged;      // lossyring
  // fifo / heap / sorted: events [Q][cap]
  Ev<T>* ev;
  int* head;              // fifo / sorted head
  int* tail_key;          // fifo
  int* seq;               // heap insertion counter
};

__device__ __forceinline__ bool kless(int da, int sa, int db, int sb) { return da < db || (da == db && sa < sb); }

// Validation pass: the first offending event of queue q (call order) given its
// current metadata; stateful only for FIFO (tail key, count).
template <typename T>
__global__ void k_validate(QView<T> V, const int* sq, const int* sidx, const int* due, long long n, int* first_bad,
                           int* bad_code) {
  for (long long k = blockIdx.x * (long long)blockDim.x + threadIdx.x; k < n; k += (long long)gridDim.x * blockDim.x) {
    const int q = sq[k];
    if (k > 0 && sq[k - 1] == q) continue;   // one thread per queue run
    int count = V.count ? V.count[q] : 0;
    int tail = V.tail_key ? V.tail_key[q] : -1;
    for (long long r = k; r < n && sq[r] == q; ++r) {
      const int e = sidx[r];
      const int step = due[e];
      int code = 0;
      if (step < V.now) code = EQ_ERR_CAUSALITY;                              // events.py:136-141
      else if (V.kind == EQ_KIND_RING && step - V.now >= V.cap) code = EQ_ERR_CAPABILITY;  // queues.py:94-98
      else if (V.kind == EQ_KIND_FIFORING) {
        if (step < tail) code = EQ_ERR_CAPABILITY;                           // queues.py:220-224
        else if (count < V.cap) { count += 1; tail = step; }
      }
      if (code) {
        int prev = atomicMin(first_bad, e);
        if (prev > e) atomicExch(bad_code, code);   // best effort; re-derived on the host
        break;
      }
    }
  }
}

// Apply one event of queue q at queue time `now` (enqueue, events.py:99-141);
// returns true if accepted.  Callers have validated causality/capability.
template <typename T>
__device__ __forceinline__ bool apply_one(const QView<T>& V, int q, int now, int step, T w, T dw, T tt) {
  if (V.kind == EQ_KIND_DONOTHING) return false;
  if (V.kind == EQ_KIND_RING || V.kind == EQ_KIND_LOSSYRING) {
    if (V.kind == EQ_KIND_LOSSYRING && step - now >= V.cap) V.aliased[q] += 1;   // queues.py:164-165
    const size_t s = (size_t)q * V.cap + (step % V.cap);
    if (!V.occ[s]) {
      V.occ[s] = 1;
      V.count[q] += 1;
    } else if (V.kind == EQ_KIND_LOSSYRING) {
      V.merged[q] += 1;                                                  // :167-168
    }
    V.sw[s] = V.sw[s] + w;                                               // :104-106
    V.sdw[s] = V.sdw[s] + dw;
    V.swtt[s] = V.swtt[s] + w * tt;
    return true;
  }
  const int cnt = V.count[q];
  if (cnt == V.cap) return false;                                        // drop incoming
  Ev<T>* a = V.ev + (size_t)q * V.cap;
  Ev<T> x;
  x.due = step;
  x.seq = 0;
  x.w = w;
  x.dw = dw;
  x.tt = tt;
  if (V.kind == EQ_KIND_FIFORING) {                                      // :227-231
    int slot = V.head[q] + cnt;
    if (slot >= V.cap) slot -= V.cap;
    a[slot] = x;
    V.tail_key[q] = step;
  } else if (V.kind == EQ_KIND_BINARYHEAP) {                             // :516-528
    x.seq = V.seq[q]++;
    int i = cnt;
    while (i > 0) {
      const int parent = (i - 1) >> 1;
      if (!kless(x.due, x.seq, a[parent].due, a[parent].seq)) break;
      a[i] = a[parent];
      i = parent;
    }
    a[i] = x;
  } else {                                                               // sorted, stable (:348-366)
    const int h = V.head[q];
    int kk = cnt;
    while (kk > 0) {
      int pi = h + kk - 1;
      if (pi >= V.cap) pi -= V.cap;
      if (a[pi].due <= step) break;
      int di = pi + 1;
      if (di >= V.cap) di -= V.cap;
      a[di] = a[pi];
      --kk;
    }
    int di = h + kk;
    if (di >= V.cap) di -= V.cap;
    a[di] = x;
  }
  V.count[q] = cnt + 1;
  return true;
}

template <typename T>
__global__ void k_apply(QView<T> V, const int* sq, const int* sidx, const int* due, const T* w, const T* dw,
                        const T* tt, long long n, int limit, unsigned char* accepted) {
  for (long long k = blockIdx.x * (long long)blockDim.x + threadIdx.x; k < n; k += (long long)gridDim.x * blockDim.x) {
    const int q = sq[k];
    if (k > 0 && sq[k - 1] == q) continue;
    for (long long r = k; r < n && sq[r] == q; ++r) {
      const int e = sidx[r];
      if (e >= limit) break;   // at or after the first error in call order
      accepted[e] = apply_one<T>(V, q, V.now, due[e], w[e], dw[e], tt[e]) ? 1 : 0;
    }
  }
}

// pop_due of queue q at queue time `now`: sums in insertion order; returns
// whether a slot/event was due (queues.py:109-120, :245-254, :378-398, :555-568).
template <typename T>
__device__ __forceinline__ bool pop_one(const QView<T>& V, int q, int now, T& w, T& dw, T& wtt) {
  w = (T)0;
  dw = (T)0;
  wtt = (T)0;
  bool got = false;
  if (V.kind == EQ_KIND_RING || V.kind == EQ_KIND_LOSSYRING) {
    const size_t s = (size_t)q * V.cap + (now % V.cap);
    if (V.occ[s]) {
      got = true;
      w = V.sw[s];
      dw = V.sdw[s];
      wtt = V.swtt[s];
      V.sw[s] = (T)0;
      V.sdw[s] = (T)0;
      V.swtt[s] = (T)0;
      V.occ[s] = 0;
      V.count[q] -= 1;
    }
  } else if (V.kind != EQ_KIND_DONOTHING) {
    Ev<T>* a = V.ev + (size_t)q * V.cap;
    int cnt = V.count[q];
    if (V.kind == EQ_KIND_BINARYHEAP) {
      while (cnt > 0 && a[0].due == now) {
        const Ev<T> top = a[0];
        got = true;
        w = w + top.w;
        dw = dw + top.dw;
        wtt = wtt + top.w * top.tt;
        const int last = --cnt;
        const Ev<T> item = a[last];
        if (last > 0) {
          int i = 0;
          const int half = last >> 1;
          while (i < half) {
            int child = 2 * i + 1;
            const int right = child + 1;
            if (right < last && kless(a[right].due, a[right].seq, a[child].due, a[child].seq)) child = right;
            if (!kless(a[child].due, a[child].seq, item.due, item.seq)) break;
            a[i] = a[child];
            i = child;
          }
          a[i] = item;
        }
      }
    } else {
      int h = V.head[q];
      while (cnt > 0 && a[h].due == now) {
        got = true;
        w = w + a[h].w;
        dw = dw + a[h].dw;
        wtt = wtt + a[h].w * a[h].tt;
        h += 1;
        if (h == V.cap) h = 0;
        cnt -= 1;
      }
      V.head[q] = h;
    }
    V.count[q] = cnt;
  }
  return got;
}

template <typename T>
__global__ void k_pop(QView<T> V, T* ow, T* odw, T* owtt, unsigned char* has) {
  const int q = blockIdx.x * blockDim.x + threadIdx.x;
  if (q >= V.Q) return;
  T w, dw, wtt;
  const bool got = pop_one<T>(V, q, V.now, w, dw, wtt);
  ow[q] = w;
  odw[q] = dw;
  owtt[q] = wtt;
  has[q] = got ? 1 : 0;
}

// The reference's single-queue Poisson benchmark (bench.py:183-205
// _drive_queue) for every queue of the batch in one launch: queues are
// independent, so each thread steps its own queue through the whole stream —
// pop, then enqueue a unit event due `delay` steps later if the stream spikes
// — and drains the in-flight tail with delay+1 more pops.
template <typename T>
__global__ void k_poisson(QView<T> V, const uint32_t* spikes, int words, int t_steps, int delay, double* delivered,
                          long long* accepted, int* err) {
  const int q = blockIdx.x * blockDim.x + threadIdx.x;
  if (q >= V.Q) return;
  const uint32_t* row = spikes + (size_t)q * words;
  int now = V.now;
  double del = 0.0;
  long long acc = 0;
  T w, dw, wtt;
  for (int s = 0; s < t_steps; ++s) {
    if (pop_one<T>(V, q, now, w, dw, wtt)) del += (double)w;
    now += 1;
    if ((__ldg(row + (s >> 5)) >> (s & 31)) & 1u) {
      const int step = V.now + s + delay;
      if (V.kind == EQ_KIND_RING && step - now >= V.cap) {               // queues.py:94-98
        atomicCAS(err, 0, EQ_ERR_CAPABILITY);
        break;
      }
      if (V.kind == EQ_KIND_FIFORING && V.tail_key[q] > step) {           // queues.py:220-224
        atomicCAS(err, 0, EQ_ERR_CAPABILITY);
        break;
      }
      if (apply_one<T>(V, q, now, step, (T)1, (T)0, (T)0)) acc += 1;
    }
  }
  for (int k = 0; k <= delay; ++k) {
    if (pop_one<T>(V, q, now, w, dw, wtt)) del += (double)w;
    now += 1;
  }
  delivered[q] = del;
  accepted[q] = acc;
}

}  // namespace

struct eq_queues {
  int kind = 0, precision = 64, Q = 0, cap = 0, maxd = 0, device = 0;
  int now = 0;
  std::string err;
  std::vector<void*> owned;
  void *sw = nullptr, *sdw = nullptr, *swtt = nullptr, *ev = nullptr;
  unsigned char* occ = nullptr;
  int *count = nullptr, *head = nullptr, *tail_key = nullptr, *seq = nullptr;
  long long *aliased = nullptr, *merged = nullptr;
  // scratch
  void* tmp = nullptr;
  size_t tmp_bytes = 0;
  int *sq = nullptr, *sidx = nullptr, *qin = nullptr, *iota = nullptr, *bad = nullptr;
  long long scratch_n = 0;
};

namespace {

int qfail(eq_queues* h, int code, const std::string& m) {
  if (h) h->err = m;
  return code;
}

#define QCUDA(h, call)                                                                    \
  do {                                                                                    \
    cudaError_t _e = (call);                                                              \
    if (_e != cudaSuccess) return qfail((h), EQ_ERR_CUDA, std::string(#call) + ": " + cudaGetErrorString(_e)); \
  } while (0)

cudaError_t qalloc(eq_queues* h, void** p, size_t bytes) {
  if (bytes == 0) bytes = 16;
  cudaError_t e = cudaMalloc(p, bytes);
  if (e == cudaSuccess) {
    h->owned.push_back(*p);
    e = cudaMemset(*p, 0, bytes);
  }
  return e;
}

template <typename T>
QView<T> view(eq_queues* h) {
  QView<T> v;
  v.kind = h->kind;
  v.Q = h->Q;
  v.cap = h->cap;
  v.now = h->now;
  v.sw = (T*)h->sw;
  v.sdw = (T*)h->sdw;
  v.swtt = (T*)h->swtt;
  v.occ = h->occ;
  v.count = h->count;
  v.aliased = h->aliased;
  v.merged = h->merged;
  v.ev = (Ev<T>*)h->ev;
  v.head = h->head;
  v.tail_key = h->tail_key;
  v.seq = h->seq;
  return v;
}

__global__ void k_iota32(int* v, long long n) {
  for (long long k = blockIdx.x * (long long)blockDim.x + threadIdx.x; k < n; k += (long long)gridDim.x * blockDim.x)
    v[k] = (int)k;
}

__global__ void k_fill_int(int* v, long long n, int x) {
  for (long long k = blockIdx.x * (long long)blockDim.x + threadIdx.x; k < n; k += (long long)gridDim.x * blockDim.x)
    v[k] = x;
}

// Scratch for one enqueue batch; the iota initialisation is stream-ordered on
// the caller's stream s, which the sort that reads it uses next.
int ensure_scratch(eq_queues* h, long long n, cudaStream_t s) {
  if (n <= h->scratch_n) return EQ_OK;
  for (void* p : {(void*)h->sq, (void*)h->sidx, (void*)h->iota, (void*)h->tmp}) {
    if (p) {
      cudaFree(p);
      h->owned.erase(std::remove(h->owned.begin(), h->owned.end(), p), h->owned.end());
    }
  }
  long long cap = std::max<long long>(n, 1024);
  QCUDA(h, qalloc(h, (void**)&h->sq, cap * sizeof(int)));
  QCUDA(h, qalloc(h, (void**)&h->sidx, cap * sizeof(int)));
  QCUDA(h, qalloc(h, (void**)&h->iota, cap * sizeof(int)));
  k_iota32<<<256, 256, 0, s>>>(h->iota, cap);
  size_t tb = 0;
  int end_bit = 1;
  while ((1LL << end_bit) < h->Q) ++end_bit;
  QCUDA(h, cub::DeviceRadixSort::SortPairs(nullptr, tb, (const int*)nullptr, (int*)nullptr, (const int*)nullptr,
                                           (int*)nullptr, (int)cap, 0, end_bit));
  QCUDA(h, qalloc(h, &h->tmp, tb));
  h->tmp_bytes = tb;
  h->scratch_n = cap;
  return EQ_OK;
}

template <typename T>
int enqueue_impl(eq_queues* h, const int32_t* queue, const int32_t* due, const void* w, const void* dw,
                 const void* tt, int64_t n, uint8_t* accepted, cudaStream_t s) {
  if (n <= 0) return EQ_OK;
  int rc = ensure_scratch(h, n, s);
  if (rc) return rc;
  int end_bit = 1;
  while ((1LL << end_bit) < h->Q) ++end_bit;
  size_t tb = h->tmp_bytes;
  QCUDA(h, cub::DeviceRadixSort::SortPairs(h->tmp, tb, queue, h->sq, (const int*)h->iota, h->sidx, (int)n, 0, end_bit,
                                           s));
  int init[2] = {kInf, 0};
  QCUDA(h, cudaMemcpyAsync(h->bad, init, sizeof init, cudaMemcpyHostToDevice, s));
  QView<T> V = view<T>(h);
  int blocks = (int)std::min<long long>((n + 255) / 256, 4096);
  k_validate<T><<<blocks, 256, 0, s>>>(V, h->sq, h->sidx, due, n, h->bad, h->bad + 1);
  int bad[2];
  QCUDA(h, cudaMemcpyAsync(bad, h->bad, sizeof bad, cudaMemcpyDeviceToHost, s));
  QCUDA(h, cudaStreamSynchronize(s));
  const int limit = bad[0] == kInf ? (int)n : bad[0];
  k_apply<T><<<blocks, 256, 0, s>>>(V, h->sq, h->sidx, due, (const T*)w, (const T*)dw, (const T*)tt, n, limit,
                                    accepted);
  QCUDA(h, cudaGetLastError());
  if (bad[0] != kInf) {
    // re-derive the code of the first offending event on the host for an exact message
    int step = 0;
    QCUDA(h, cudaMemcpy(&step, due + bad[0], sizeof(int), cudaMemcpyDeviceToHost));
    const char* kn = h->kind == EQ_KIND_FIFORING ? "fiforing" : h->kind == EQ_KIND_RING ? "ring" : "queue";
    char buf[256];
    if (step < h->now) {
      snprintf(buf, sizeof buf, "%s: event for step %d enqueued at step %d; delivery must lag creation by >= 1 step",
               kn, step, h->now);
      return qfail(h, EQ_ERR_CAUSALITY, buf);
    }
    if (h->kind == EQ_KIND_RING)
      snprintf(buf, sizeof buf, "ring: delay of %d steps exceeds buffer capacity %d", step - h->now + 1, h->cap);
    else
      snprintf(buf, sizeof buf, "fiforing supports homogeneous delays only: event %d for step %d arrived after a later one",
               bad[0], step);
    return qfail(h, EQ_ERR_CAPABILITY, buf);
  }
  return EQ_OK;
}

}  // namespace

extern "C" {

int eq_queues_create(int kind, int precision, int n_queues, int capacity, int max_delay_steps, int device,
                     eq_queues** out) {
  if (!out) return EQ_ERR_CONFIGURATION;
  eq_queues* h = new eq_queues();
  *out = h;
  h->kind = kind;
  h->precision = precision;
  h->Q = n_queues;
  h->device = device;
  if (precision != 32 && precision != 64) return qfail(h, EQ_ERR_CONFIGURATION, "precision must be 32 or 64");
  if (n_queues < 1) return qfail(h, EQ_ERR_CONFIGURATION, "n_queues must be >= 1");
  // make_queue argument rules (queues.py:636-692)
  int cap = capacity;
  if (kind == EQ_KIND_RING) {
    if (cap <= 0) cap = max_delay_steps;
    if (cap <= 0) return qfail(h, EQ_ERR_CONFIGURATION, "ring needs a capacity or a max delay");
    int maxd = max_delay_steps > 0 ? max_delay_steps : cap;
    if (maxd > cap)
      return qfail(h, EQ_ERR_CONFIGURATION,
                   "ring capacity " + std::to_string(cap) + " cannot cover max delay " + std::to_string(maxd) +
                       "; a smaller buffer aliases (use lossyring)");
    h->maxd = maxd;
  } else if (kind == EQ_KIND_LOSSYRING) {
    if (cap <= 0) return qfail(h, EQ_ERR_CONFIGURATION, "lossyring needs a capacity");
  } else if (kind == EQ_KIND_FIFORING || kind == EQ_KIND_SORTEDARRAY || kind == EQ_KIND_BINARYHEAP) {
    const char* nm = kind == EQ_KIND_FIFORING ? "fiforing" : kind == EQ_KIND_SORTEDARRAY ? "sortedarray" : "binaryheap";
    if (cap <= 0) return qfail(h, EQ_ERR_CONFIGURATION, std::string(nm) + " needs a capacity");
  } else if (kind == EQ_KIND_DONOTHING) {
    cap = 1;
  } else {
    return qfail(h, EQ_ERR_CONFIGURATION, "unknown queue kind " + std::to_string(kind));
  }
  h->cap = cap;
  if (cudaSetDevice(device) != cudaSuccess) return qfail(h, EQ_ERR_CUDA, "no CUDA device");
  const size_t T = precision == 32 ? 4 : 8;
  const size_t Q = n_queues;
  QCUDA(h, qalloc(h, (void**)&h->count, Q * sizeof(int)));
  QCUDA(h, qalloc(h, (void**)&h->bad, 2 * sizeof(int)));
  if (kind == EQ_KIND_RING || kind == EQ_KIND_LOSSYRING) {
    QCUDA(h, qalloc(h, &h->sw, Q * cap * T));
    QCUDA(h, qalloc(h, &h->sdw, Q * cap * T));
    QCUDA(h, qalloc(h, &h->swtt, Q * cap * T));
    QCUDA(h, qalloc(h, (void**)&h->occ, Q * cap));
    QCUDA(h, qalloc(h, (void**)&h->aliased, Q * sizeof(long long)));
    QCUDA(h, qalloc(h, (void**)&h->merged, Q * sizeof(long long)));
  } else if (kind != EQ_KIND_DONOTHING) {
    QCUDA(h, qalloc(h, &h->ev, Q * cap * (precision == 32 ? sizeof(Ev<float>) : sizeof(Ev<double>))));
    QCUDA(h, qalloc(h, (void**)&h->head, Q * sizeof(int)));
    QCUDA(h, qalloc(h, (void**)&h->tail_key, Q * sizeof(int)));
    QCUDA(h, qalloc(h, (void**)&h->seq, Q * sizeof(int)));
    k_fill_int<<<64, 256>>>(h->tail_key, (long long)Q, -1);   // FIFORingQueue._tail_key = -1
  }
  QCUDA(h, cudaDeviceSynchronize());
  return EQ_OK;
}

int eq_queues_destroy(eq_queues* h) {
  if (!h) return EQ_OK;
  for (void* p : h->owned) cudaFree(p);
  delete h;
  return EQ_OK;
}

const char* eq_queues_last_error(const eq_queues* h) { return h ? h->err.c_str() : "null handle"; }

int eq_queues_capacity(const eq_queues* h) { return h ? h->cap : -1; }

int eq_queues_now(const eq_queues* h) { return h ? h->now : -1; }

int eq_queues_enqueue(eq_queues* h, const int32_t* queue, const int32_t* deliver_step, const void* weight,
                      const void* weight_tangent, const void* time_tangent, int64_t n, uint8_t* accepted,
                      void* stream) {
  if (!h) return EQ_ERR_CONFIGURATION;
  if (n >= (1LL << 31)) return qfail(h, EQ_ERR_CONFIGURATION, "batch too large");
  cudaStream_t s = (cudaStream_t)stream;
  if (h->precision == 32)
    return enqueue_impl<float>(h, queue, deliver_step, weight, weight_tangent, time_tangent, n, accepted, s);
  return enqueue_impl<double>(h, queue, deliver_step, weight, weight_tangent, time_tangent, n, accepted, s);
}

int eq_queues_pop(eq_queues* h, void* out_w, void* out_dw, void* out_wtt, uint8_t* out_has, void* stream) {
  if (!h) return EQ_ERR_CONFIGURATION;
  cudaStream_t s = (cudaStream_t)stream;
  const int blocks = (h->Q + 255) / 256;
  if (h->precision == 32)
    k_pop<float><<<blocks, 256, 0, s>>>(view<float>(h), (float*)out_w, (float*)out_dw, (float*)out_wtt, out_has);
  else
    k_pop<double><<<blocks, 256, 0, s>>>(view<double>(h), (double*)out_w, (double*)out_dw, (double*)out_wtt,
                                         out_has);
  QCUDA(h, cudaGetLastError());
  h->now += 1;
  return EQ_OK;
}

int eq_queues_run_poisson(eq_queues* h, const uint32_t* spikes, int32_t t_steps, int32_t delay, double* delivered,
                          int64_t* accepted, void* stream) {
  if (!h) return EQ_ERR_CONFIGURATION;
  if (t_steps < 1 || delay < 1) return qfail(h, EQ_ERR_CONFIGURATION, "t_steps and delay must be >= 1");
  cudaStream_t s = (cudaStream_t)stream;
  int zero = 0;
  QCUDA(h, cudaMemcpyAsync(h->bad, &zero, sizeof zero, cudaMemcpyHostToDevice, s));
  const int blocks = (h->Q + 127) / 128, words = (t_steps + 31) / 32;
  if (h->precision == 32)
    k_poisson<float><<<blocks, 128, 0, s>>>(view<float>(h), spikes, words, t_steps, delay, delivered,
                                            (long long*)accepted, h->bad);
  else
    k_poisson<double><<<blocks, 128, 0, s>>>(view<double>(h), spikes, words, t_steps, delay, delivered,
                                             (long long*)accepted, h->bad);
  QCUDA(h, cudaGetLastError());
  int e = 0;
  QCUDA(h, cudaMemcpyAsync(&e, h->bad, sizeof e, cudaMemcpyDeviceToHost, s));
  QCUDA(h, cudaStreamSynchronize(s));
  h->now += t_steps + delay + 1;
  if (e) {
    char buf[160];
    if (h->kind == EQ_KIND_RING)
      snprintf(buf, sizeof buf, "ring: delay of %d steps exceeds buffer capacity %d", delay, h->cap);
    else
      snprintf(buf, sizeof buf, "fiforing supports homogeneous delays only");
    return qfail(h, e, buf);
  }
  return EQ_OK;
}

int eq_queues_occupancy(eq_queues* h, int32_t* out, void* stream) {
  if (!h) return EQ_ERR_CONFIGURATION;
  QCUDA(h, cudaMemcpyAsync(out, h->count, (size_t)h->Q * sizeof(int), cudaMemcpyDeviceToDevice,
                           (cudaStream_t)stream));
  return EQ_OK;
}

int eq_queues_lossy_counts(eq_queues* h, int64_t* aliased, int64_t* merged, void* stream) {
  if (!h) return EQ_ERR_CONFIGURATION;
  if (h->kind != EQ_KIND_LOSSYRING) return qfail(h, EQ_ERR_CONFIGURATION, "lossyring only");
  cudaStream_t s = (cudaStream_t)stream;
  QCUDA(h, cudaMemcpyAsync(aliased, h->aliased, (size_t)h->Q * 8, cudaMemcpyDeviceToDevice, s));
  QCUDA(h, cudaMemcpyAsync(merged, h->merged, (size_t)h->Q * 8, cudaMemcpyDeviceToDevice, s));
  return EQ_OK;
}

}  // extern "C"
