// eq_ring.cuh — persistent fused step kernels (forward + reverse) for the ring
// queue (RingQueue, queues.py:55-123) and DoNothing (queues.py:26-52).
//
// Geometry: a cooperative grid of G CTAs.  Neuron-trials are flattened to
// idx = trial*N + neuron and CTA c owns the contiguous range
// [c*per, (c+1)*per).  One grid barrier per simulated step:
//
//   phase m (forward):  pop slot m + synapse + LIF for the owned neurons
//                       (network.py:547-580), then fan the CTA's own crossings
//                       out as fixed-point red.add into slot (dstep mod R) of
//                       each target (network.py:583-611).
//   phase m (reverse):  R-fanout(m) for the CTA's own spikes of step m (gather
//                       of the reverse slots, dL/dw, dL/dd, dL/dt_spk), then
//                       R-neuron(m) for the owned neurons.
//
// Ring rows are R = horizon + 1 slots: a fan-out of step m writes delivery
// steps in [m+2, m+horizon] while other CTAs may still pop slot m in the same
// phase, so (m+horizon) mod R must differ from m mod R.  Any R >= horizon gives
// the reference's results (slot = step % capacity never aliases a live step).
#pragma once

#include "eq_device.cuh"

namespace eq {

template <typename T>
struct StepConsts {
  T dt, tau_m, tau_s, v_th, v_reset, k_m, k_s, cc;
  double scale, inv_scale;  // 2^F, 2^-F
};

template <typename T>
struct NetView {
  const int64_t* rowptr;
  const int32_t* col;
  const T* w;
  const T* d;
  const uint32_t* mask;  // [B][t_mask][words]
  const T* amp;          // [N]
  int words, t_mask;
};

template <typename T>
struct FwdArgs {
  int N, B, G;
  long long total, per;
  int m0, m1;         // steps [m0, m1)
  int R, kind, refractory, exact;
  StepConsts<T> c;
  NetView<T> net;
  T* I;
  T* V;
  int32_t* refr;
  long long* ring;    // fp32: [B][R][N]; fp64: [B][R][N][2]
  SpikeRec<T>* scratch;  // [G][per] per-CTA spill area for the step's spikes
  SpikeRec<T>* log;
  long long log_cap;
  unsigned long long* log_count;
  long long* chunk_off;  // [m][G]
  int* chunk_cnt;        // [m][G]
  long long* counters;   // [B][3]
  T* v_trace;            // [m1-m0][B][N] or null
  unsigned long long* tl;  // debug timeline [m][G][4] (globaltimer ns) or null
  int* err;
  unsigned* bar;
};

template <int NT>
struct FwdShared {
  static constexpr int kCap = 1024;   // spikes staged in smem per step per CTA
  static constexpr int kTrials = 8;   // per-CTA trial counters kept in smem
};

__device__ __forceinline__ void tl_mark(unsigned long long* tl, int m, int G, int cta, int k) {
  if (tl && threadIdx.x == 0) tl[((size_t)m * G + cta) * 8 + k] = globaltimer();
}

// Exclusive prefix over a staged spike batch's row lengths, by warp 0.
// On entry pre[k+1] = len[k] (k < n); on exit pre[0..n] is the exclusive scan.
__device__ __forceinline__ void warp0_scan(int* pre, int n) {
  if (threadIdx.x < 32) {
    const int lane = threadIdx.x;
    int carry = 0;
    for (int base = 0; base < n; base += 32) {
      const int k = base + lane;
      int v = k < n ? pre[k + 1] : 0;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        int t = __shfl_up_sync(0xffffffffu, v, o);
        if (lane >= o) v += t;
      }
      if (k < n) pre[k + 1] = carry + v;
      carry += __shfl_sync(0xffffffffu, v, 31);
    }
    if (lane == 0) pre[0] = 0;
  }
}

// Row of flat event f: the largest k < n with pre[k] <= f.
__device__ __forceinline__ int find_row(const int* pre, int n, int f) {
  int lo = 0, hi = n;
  while (hi - lo > 1) {
    int mid = (lo + hi) >> 1;
    if (pre[mid] <= f) lo = mid;
    else hi = mid;
  }
  return lo;
}

// One neuron-step of PrimalRSNN.step (network.py:559-580) after the pop.
// Returns true on a threshold crossing; t_spk is NaN for a grazing crossing
// (slope below 1e-9, neuro.py:194-199), which the caller turns into an error.
template <typename T>
__device__ __forceinline__ bool lif_step(const StepConsts<T>& c, bool exact, int refractory, int m, T ps, T pm,
                                         T I, T V, T drive, int& rf, T& i_out, T& v_out, T& a_out, T& vh_out,
                                         T& t_out) {
  const T i = (I + ps) * c.k_s;                       // :559
  const T a = i + drive;                              // :561
  T v = V;
  if (exact) v = v + c.cc * (pm - ps);                // :564
  T v_new = a + (v - a) * c.k_m;                      // :565
  bool spike = false;
  if (rf > 0) {                                       // :566-567
    rf -= 1;
  } else if (v < c.v_th && c.v_th <= v_new) {         // :568
    const T v_dot = (a - c.v_th) / c.tau_m;           // :569
    if (v_dot < (T)1e-9) {
      t_out = (T)NAN;
    } else {
      const T r = (c.v_th - a) / (v - a);             // :574
      const T t_spk = (T)m * c.dt - c.tau_m * eq_log_t(r);  // :575
      const T uu = (T)(m + 1) * c.dt - t_spk;         // :576
      v_new = a + (c.v_reset - a) * eq_exp_t(-uu / c.tau_m);  // :577
      rf = refractory;                                // :578
      t_out = t_spk;
    }
    spike = true;
  }
  i_out = i;
  v_out = v_new;
  a_out = a;
  vh_out = v;
  return spike;
}

template <typename T>
__device__ __forceinline__ bool drive_bit(const NetView<T>& net, int b, int m, int j) {
  int mm = m < net.t_mask ? m : net.t_mask - 1;   // network.py:155 rows[-1]
  const uint32_t* row = net.mask + ((size_t)b * net.t_mask + mm) * net.words;
  return (__ldg(row + (j >> 5)) >> (j & 31)) & 1u;
}

template <typename T, int NT, int U>
__global__ void __launch_bounds__(NT) k_forward(FwdArgs<T> A) {
  typedef Prec<T> P;
  constexpr int kCap = FwdShared<NT>::kCap;
  constexpr int kTr = FwdShared<NT>::kTrials;
  __shared__ SpikeRec<T> s_spk[kCap];
  __shared__ long long s_r0[kCap];
  __shared__ int s_pre[kCap + 1];
  __shared__ int s_n;
  __shared__ long long s_off;
  __shared__ unsigned long long s_ctr[kTr][2];

  const int tid = threadIdx.x;
  const int cta = blockIdx.x;
  const long long begin = (long long)cta * A.per;
  const long long end = begin + A.per < A.total ? begin + A.per : A.total;
  const int b_first = (int)(begin / A.N);
  const StepConsts<T> c = A.c;
  SpikeRec<T>* spill = A.scratch + (size_t)cta * A.per;

  if (tid < kTr * 2) (&s_ctr[0][0])[tid] = 0ULL;

  for (int m = A.m0; m < A.m1; ++m) {
    if (tid == 0) s_n = 0;
    __syncthreads();
    tl_mark(A.tl, m, A.G, cta, 0);
    // ---------------- neuron update: pop, synapse, membrane, crossing
    for (long long base = begin; base < end; base += (long long)NT * U) {
      long long slot_v[U][2];
      T Iv[U], Vv[U];
      int rf[U];
      bool on[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int idx = (int)base + u * NT + tid;
        slot_v[u][0] = slot_v[u][1] = 0;
        if (idx < end) {
          const int b = idx / A.N;
          const int j = idx - b * A.N;
          size_t so = ((size_t)b * A.R + (size_t)(m % A.R)) * A.N + j;
          if (A.kind == EQ_KIND_RING) {
            if (P::kSlotWords == 1) {
              slot_v[u][0] = ld_slot(A.ring + so);
            } else {
              slot_v[u][0] = ld_slot(A.ring + 2 * so);
              slot_v[u][1] = ld_slot(A.ring + 2 * so + 1);
            }
          }
          Iv[u] = A.I[idx];
          Vv[u] = A.V[idx];
          rf[u] = A.refractory ? A.refr[idx] : 0;
          on[u] = drive_bit(A.net, b, m, j);
        }
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int idx = (int)base + u * NT + tid;
        if (idx >= end) continue;
        const int b = idx / A.N;
        const int j = idx - b * A.N;
        T ps, pm;
        if (P::kSlotWords == 1) {
          long long qs, qm;
          unpack2(slot_v[u][0], qs, qm);
          ps = P::deq(qs, c.inv_scale);
          pm = P::deq(qm, c.inv_scale);
        } else {
          ps = P::deq(slot_v[u][0], c.inv_scale);
          pm = P::deq(slot_v[u][1], c.inv_scale);
        }
        if (!A.exact) pm = (T)0;
        const T drive = on[u] ? __ldg(A.net.amp + j) : (T)0;
        T i, v_new, a, v, t_spk;
        if (lif_step(c, A.exact != 0, A.refractory, m, ps, pm, Iv[u], Vv[u], drive, rf[u], i, v_new, a, v, t_spk)) {
          if (t_spk != t_spk) {
            raise_error(A.err, EQ_ERR_GRAZING, m + 1, b, j);
          } else {
            int pos = atomicAdd(&s_n, 1);
            SpikeRec<T> rec;
            rec.idx = idx;
            rec.t = t_spk;
            rec.a = a;
            rec.vh = v;
            if (pos < kCap) s_spk[pos] = rec;
            else spill[pos - kCap] = rec;
          }
        }
        A.I[idx] = i;
        A.V[idx] = v_new;
        if (A.refractory) A.refr[idx] = rf[u];
        if (A.v_trace) A.v_trace[(size_t)(m - A.m0) * A.total + idx] = v_new;
      }
    }
    __syncthreads();
    tl_mark(A.tl, m, A.G, cta, 1);
    // Clear the popped slot row (RingQueue._pop_raw zeroes it, queues.py:114-117).
    // Done here, not next to the load: a store to the line a pending load is
    // filling stalled the pop loop ~8x.  Row m mod R receives no red.add in
    // this phase (fan-out targets rows m+2 .. m+horizon, R = horizon + 1).
    if (A.kind == EQ_KIND_RING) {
      const int row = m % A.R;
      for (int idx = (int)begin + tid; idx < end; idx += NT) {
        const int b = idx / A.N;
        const size_t so = ((size_t)b * A.R + row) * A.N + (idx - b * A.N);
        if (P::kSlotWords == 1) {
          st_slot(A.ring + so, 0);
        } else {
          st_slot(A.ring + 2 * so, 0);
          st_slot(A.ring + 2 * so + 1, 0);
        }
      }
    }
    __syncthreads();
    tl_mark(A.tl, m, A.G, cta, 4);
    const int nspk = s_n;
    // ---------------- spike log for the reverse pass: one chunk per (step, CTA)
    if (tid == 0) {
      unsigned long long off = nspk ? atomicAdd(A.log_count, (unsigned long long)nspk) : 0ULL;
      if (nspk && (long long)(off + nspk) > A.log_cap) {
        raise_error(A.err, EQ_ERR_CAPACITY, m, -1, -1);
        off = 0;
      }
      s_off = (long long)off;
      A.chunk_off[(size_t)m * A.G + cta] = (long long)off;
      A.chunk_cnt[(size_t)m * A.G + cta] = nspk;
    }
    __syncthreads();
    if (s_off + nspk <= A.log_cap) {
      for (int k = tid; k < nspk; k += NT) A.log[s_off + k] = k < kCap ? s_spk[k] : spill[k - kCap];
    }
    __syncthreads();
    tl_mark(A.tl, m, A.G, cta, 5);
    // ---------------- fan-out (network.py:583-611), flattened over (spike, edge)
    // so every lane carries an event: batch of <= kCap spikes, prefix of their
    // row lengths, then flat events f -> (spike, x) with EV events per thread in
    // flight.  Slot sums are fixed-point, so the order of the red.adds is free.
    for (int k0 = 0; k0 < nspk; k0 += kCap) {
      const int nb = nspk - k0 < kCap ? nspk - k0 : kCap;
      __syncthreads();
      if (k0 > 0)
        for (int k = tid; k < nb; k += NT) s_spk[k] = spill[k0 - kCap + k];
      __syncthreads();
      for (int k = tid; k < nb; k += NT) {
        const int b = s_spk[k].idx / A.N;
        const int i = s_spk[k].idx - b * A.N;
        const long long r0 = __ldg(A.net.rowptr + i);
        const int len = (int)(__ldg(A.net.rowptr + i + 1) - r0);
        s_r0[k] = r0;
        s_pre[k + 1] = len;
        const int tb = b - b_first;
        if (tb < kTr) {
          atomicAdd(&s_ctr[tb][0], 1ULL);
          atomicAdd(&s_ctr[tb][1], (unsigned long long)len);
        } else {
          atomicAdd(reinterpret_cast<unsigned long long*>(A.counters + 3 * b), 1ULL);
          atomicAdd(reinterpret_cast<unsigned long long*>(A.counters + 3 * b + 1), (unsigned long long)len);
        }
        if (A.kind == EQ_KIND_DONOTHING)
          atomicAdd(reinterpret_cast<unsigned long long*>(A.counters + 3 * b + 2), (unsigned long long)len);
      }
      __syncthreads();
      warp0_scan(s_pre, nb);
      __syncthreads();
      if (k0 == 0) tl_mark(A.tl, m, A.G, cta, 6);
      if (A.kind != EQ_KIND_RING) continue;
      const int total = s_pre[nb];
      constexpr int EV = 4;
      for (int f0 = tid; f0 < total; f0 += EV * NT) {
        int jj[EV], kk[EV];
        T ww[EV], dd[EV];
#pragma unroll
        for (int e = 0; e < EV; ++e) {
          const int f = f0 + e * NT;
          kk[e] = -1;
          if (f < total) {
            const int k = find_row(s_pre, nb, f);
            const long long x = s_r0[k] + (f - s_pre[k]);
            kk[e] = k;
            jj[e] = __ldg(A.net.col + x);
            ww[e] = __ldg(A.net.w + x);
            dd[e] = __ldg(A.net.d + x);
          }
        }
#pragma unroll
        for (int e = 0; e < EV; ++e) {
          if (kk[e] < 0) continue;
          const SpikeRec<T> rec = s_spk[kk[e]];
          const int b = rec.idx / A.N;
          const T w = ww[e], d = dd[e];
          const T t_post = rec.t + d;                        // :588
          const int ds = delivery_step(t_post, d, c.dt, m);  // jumps.py:96
          T ws, wm;
          if (A.exact) {
            const T phi = (T)ds * c.dt - t_post;             // :599
            ws = w * eq_exp_t(-phi / c.tau_s);               // :601
            wm = w * eq_exp_t(-phi / c.tau_m);               // :606
          } else {
            ws = w;
            wm = (T)0;
          }
          const size_t so = ((size_t)b * A.R + (size_t)(ds % A.R)) * A.N + jj[e];
          const long long qs = P::q(ws, c.scale), qm = P::q(wm, c.scale);
          if (P::kSlotWords == 1) {
            red_add(A.ring + so, pack2(qs, qm));
          } else {
            red_add(A.ring + 2 * so, qs);
            if (A.exact) red_add(A.ring + 2 * so + 1, qm);
          }
        }
      }
    }
    __syncthreads();
    tl_mark(A.tl, m, A.G, cta, 2);
    if (!grid_sync(A.bar, A.G, A.err)) break;
    tl_mark(A.tl, m, A.G, cta, 3);
    if (ld_volatile(A.err) != 0) break;
  }
  __syncthreads();
  if (tid < kTr) {
    int b = b_first + tid;
    if (b < A.B && (long long)b * A.N < end) {
      if (s_ctr[tid][0]) atomicAdd(reinterpret_cast<unsigned long long*>(A.counters + 3 * b), s_ctr[tid][0]);
      if (s_ctr[tid][1]) atomicAdd(reinterpret_cast<unsigned long long*>(A.counters + 3 * b + 1), s_ctr[tid][1]);
    }
  }
}

// ------------------------------------------------------------------ reverse

template <typename T>
struct BwdArgs {
  int N, B, G;
  long long total, per;
  int m_run;          // steps simulated since reset (reverse walks m_run-1 .. 0)
  int R, refractory;
  StepConsts<T> c;
  NetView<T> net;
  T* lamV;
  T* lamI;
  typename Prec<T>::T2* lam;   // [B][R][N] (Lambda_s, Lambda_m)
  double* gw;
  double* gd;
  double* gamp_bt;             // [B][N] or null
  const SpikeRec<T>* log;
  T* lt_log;                   // dL/dt_spk per log record
  const long long* chunk_off;
  const int* chunk_cnt;
  const long long* ev_base;     // bounded kinds: flat event id of each log record's first edge
  const unsigned* drop_bits;    // bounded kinds: dropped events (contribute nothing); null for ring
  int no_events;                // donothing: every event was dropped
  unsigned long long* tl;  // debug timeline [m][G][4] or null
  int* err;
  unsigned* bar;
};

template <typename T, int NT, int U>
__global__ void __launch_bounds__(NT) k_backward(BwdArgs<T> A) {
  typedef typename Prec<T>::T2 T2;
  constexpr int kCapB = sizeof(T) == 4 ? 512 : 256;   // spikes per batch
  constexpr int kEv = sizeof(T) == 4 ? 4096 : 2048;    // events per reduction window
  __shared__ SpikeRec<T> s_rec[kCapB];
  __shared__ long long s_r0[kCapB];
  __shared__ int s_pre[kCapB + 1];
  __shared__ T s_lt[kCapB];
  __shared__ T s_gtp[kEv];
  extern __shared__ unsigned int s_bits[];   // one bit per owned neuron-trial
  const int tid = threadIdx.x;
  const int cta = blockIdx.x;
  const long long begin = (long long)cta * A.per;
  const long long end = begin + A.per < A.total ? begin + A.per : A.total;
  const int nwords = (int)((A.per + 31) / 32);
  const StepConsts<T> c = A.c;
  for (int k = tid; k < nwords; k += NT) s_bits[k] = 0u;
  __syncthreads();

  for (int m = A.m_run - 1; m >= 0; --m) {
    tl_mark(A.tl, m, A.G, cta, 0);
    const long long off = A.chunk_off[(size_t)m * A.G + cta];
    const int cnt = A.chunk_cnt[(size_t)m * A.G + cta];
    // ---------------- R-fanout(m): own spikes of step m, flattened over
    // (spike, edge).  dL/dt_spk of a spike is the SEQUENTIAL sum of its edges'
    // g_tp in row order (zeros for events never popped), staged through s_gtp
    // in windows of kEv events; the oracle sums in the same order.
    for (int k0 = 0; k0 < cnt; k0 += kCapB) {
      const int nb = cnt - k0 < kCapB ? cnt - k0 : kCapB;
      __syncthreads();
      for (int k = tid; k < nb; k += NT) {
        const SpikeRec<T> rec = A.log[off + k0 + k];
        s_rec[k] = rec;
        const int b = rec.idx / A.N;
        const int i = rec.idx - b * A.N;
        const long long r0 = __ldg(A.net.rowptr + i);
        s_r0[k] = r0;
        s_pre[k + 1] = (int)(__ldg(A.net.rowptr + i + 1) - r0);
        s_lt[k] = (T)0;
      }
      __syncthreads();
      warp0_scan(s_pre, nb);
      __syncthreads();
      const int total = s_pre[nb];
      for (int w0 = 0; w0 < total; w0 += kEv) {
        const int wend = total - w0 < kEv ? total : w0 + kEv;
        constexpr int EV = 4;
        for (int f0 = w0 + tid; f0 < wend; f0 += EV * NT) {
          int jj[EV], kk[EV];
          long long xx[EV];
          T ww[EV], dd[EV];
#pragma unroll
          for (int e = 0; e < EV; ++e) {
            const int f = f0 + e * NT;
            kk[e] = -1;
            if (f < wend) {
              const int k = find_row(s_pre, nb, f);
              const long long x = s_r0[k] + (f - s_pre[k]);
              kk[e] = k;
              xx[e] = x;
              jj[e] = __ldg(A.net.col + x);
              ww[e] = __ldg(A.net.w + x);
              dd[e] = __ldg(A.net.d + x);
            }
          }
#pragma unroll
          for (int e = 0; e < EV; ++e) {
            if (kk[e] < 0) continue;
            const int f = f0 + e * NT;
            const SpikeRec<T> rec = s_rec[kk[e]];
            const int b = rec.idx / A.N;
            const T w = ww[e], d = dd[e];
            const T t_post = rec.t + d;
            const int st = delivery_step(t_post, d, c.dt, m);
            T g_tp = (T)0;
            bool live = st < A.m_run && !A.no_events;        // never popped / dropped: no effect
            if (live && A.drop_bits) {                       // dropped by a bounded queue
              const long long id = A.ev_base[off + k0 + kk[e]] + (f - s_pre[kk[e]]);
              live = !((A.drop_bits[id >> 5] >> (id & 31)) & 1u);
            }
            if (live) {
              const T phi = (T)st * c.dt - t_post;
              const T es = eq_exp_t(-phi / c.tau_s);
              const T em = eq_exp_t(-phi / c.tau_m);
              const T2 L = A.lam[((size_t)b * A.R + (size_t)(st % A.R)) * A.N + jj[e]];
              const T g_w = es * L.x + em * L.y;
              g_tp = w * (es * L.x / c.tau_s + em * L.y / c.tau_m);
              atomicAdd(A.gw + xx[e], (double)g_w);
              atomicAdd(A.gd + xx[e], (double)g_tp);
            }
            s_gtp[f - w0] = g_tp;
          }
        }
        __syncthreads();
        const int ka = find_row(s_pre, nb, w0);
        const int kb = find_row(s_pre, nb, wend - 1);
        for (int k = ka + tid; k <= kb; k += NT) {
          const int lo = s_pre[k] > w0 ? s_pre[k] : w0;
          const int hi = s_pre[k + 1] < wend ? s_pre[k + 1] : wend;
          T acc = s_lt[k];
          for (int q = lo; q < hi; ++q) acc = acc + s_gtp[q - w0];
          s_lt[k] = acc;
        }
        __syncthreads();
      }
      for (int k = tid; k < nb; k += NT) {
        A.lt_log[off + k0 + k] = s_lt[k];
        const int loc = s_rec[k].idx - (int)begin;
        atomicOr(&s_bits[loc >> 5], 1u << (loc & 31));
      }
    }
    __syncthreads();
    tl_mark(A.tl, m, A.G, cta, 1);
    // ---------------- R-neuron(m)
    for (long long base = begin; base < end; base += (long long)NT * U) {
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int idx = (int)base + u * NT + tid;
        if (idx >= end) continue;
        const int b = idx / A.N;
        const int j = idx - b * A.N;
        T lv = A.lamV[idx];
        T la, lvh;
        const int loc = idx - (int)begin;
        if ((s_bits[loc >> 5] >> (loc & 31)) & 1u) {
          int k = 0;
          while (k < cnt && A.log[off + k].idx != idx) ++k;
          SpikeRec<T> rec = A.log[off + k];
          T lt0 = A.lt_log[off + k];
          T t = rec.t, a = rec.a, vh = rec.vh;
          T uu = (T)(m + 1) * c.dt - t;
          T ku = eq_exp_t(-uu / c.tau_m);
          T r = (c.v_th - a) / (vh - a);
          T lt = lt0 + lv * (c.v_reset - a) * ku / c.tau_m;
          T lr = -c.tau_m * lt / r;
          T den = vh - a;
          T den2 = den * den;
          la = lv * ((T)1 - ku) + lr * (c.v_th - vh) / den2;
          lvh = -lr * (c.v_th - a) / den2;
        } else {
          la = lv * ((T)1 - c.k_m);
          lvh = lv * c.k_m;
        }
        T lip = A.lamI[idx] + la;
        if (A.gamp_bt && drive_bit(A.net, b, m, j)) A.gamp_bt[idx] += (double)la;
        T2 L;
        L.x = c.k_s * lip - c.cc * lvh;
        L.y = c.cc * lvh;
        A.lam[((size_t)b * A.R + (size_t)(m % A.R)) * A.N + j] = L;
        A.lamI[idx] = c.k_s * lip;
        A.lamV[idx] = lvh;
      }
    }
    __syncthreads();
    for (int k = tid; k < cnt; k += NT) {
      long long loc = (long long)A.log[off + k].idx - begin;
      s_bits[loc >> 5] = 0u;
    }
    __syncthreads();
    tl_mark(A.tl, m, A.G, cta, 2);
    if (!grid_sync(A.bar, A.G, A.err)) break;
    tl_mark(A.tl, m, A.G, cta, 3);
    if (ld_volatile(A.err) != 0) break;
  }
}

}  // namespace eq
