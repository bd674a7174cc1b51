/*
 * oracle/eq_oracle.cpp — CPU restatement of the EventQueues hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  Nothing in paper_2512_05906_b200/ links, loads or
 * calls this file; only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs do, and only as the checker.
 *
 * What it restates (file:line in /root/reference):
 *   primal step ........ pkg/src/eventq/network.py:547-611 (PrimalRSNN.step),
 *                        expression order copied term by term so that reference
 *                        mode is bitwise identical to the Python reference
 *   synapse ............ neuro.py:33-47 + jumps.py:116-126 + dual.py:72-84
 *   LIF + crossing ..... neuro.py:125-210 (refractory gate before the crossing
 *                        test :155-158, grazing error :194-199)
 *   fan-out ............ network.py:412-443 with compose_delay / delivery_step
 *                        (jumps.py:83-96) and exact-delivery payloads
 *                        (network.py:429-437)
 *   ring ............... queues.py:55-123 (slot = step % capacity, capability
 *                        error when step - now >= capacity :94-98)
 *   lossy ring ......... queues.py:126-181 (slot = step % capacity with no
 *                        capability check: a delay past the buffer aliases to
 *                        an earlier step), wired by network.py:321-328 with
 *                        capacity `queue_capacity or horizon*(n-1)+1`
 *   fifo/heap/sorted ... queues.py:184-260, 481-571, 308-403: all three drop the
 *                        INCOMING event when full and pop every due event; their
 *                        accepted sets are identical, so one
 *                        "pool" restatement covers all three; FIFO keeps its
 *                        tail-key capability check (queues.py:220-224)
 *   donothing .......... queues.py:26-52 (drops everything)
 *   reverse mode ....... SURVEY.md Appendix B — the transpose of the reference's
 *                        forward-mode tangent recurrences (the reference has no
 *                        VJP; its JVP, network.py:668-683, is the pin); with
 *                        exact_delivery=False the transpose of the plain
 *                        delivery tangents: synapse jump W' + Q/tau_s
 *                        (jumps.py:116-126), membrane -Q/tau_m (neuro.py:146-149,
 *                        network.py:403-408), Q = sum w * (t_spk' + d')
 *
 * Two arithmetic modes:
 *   mode 0 "reference": double, glibc exp/log, slot sums in the reference's
 *          insertion order (emit step, source ascending, CSR row order).  Pinned
 *          bitwise against the Python reference in tests/test_oracle_pin.py.
 *   mode 1 "device": T = float or double, exp/log from include/eq_math.h, slot
 *          sums in fixed point (int32 for float, int64 for double) with
 *          frac_bits fraction bits, which makes them order-independent.  This
 *          is the arithmetic contract of the CUDA kernels; the GPU is compared
 *          with this mode bit for bit.
 */
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>
#ifdef _OPENMP
#include <omp.h>
#endif

#include "../include/eq_math.h"

namespace {

enum Kind { K_RING = 0, K_FIFO = 1, K_HEAP = 2, K_SORTED = 3, K_LOSSY = 4, K_DONOTHING = 5 };
enum Status { OK = 0, E_CONFIG = 1, E_CAPABILITY = 2, E_CAUSALITY = 3, E_GRAZING = 4, E_INTERNAL = 5 };

struct Cfg {
  int32_t kind, n, n_trials, t_steps, refractory_steps, exact_delivery, capacity, frac_bits;
  int32_t mode, precision, record_v, pad;
  double dt, tau_m, tau_syn, v_th, v_reset;
};

struct Spike {
  int32_t step, trial, neuron;
  double t, a, vh;       // exact copies of the T values
  int64_t ev_off;        // offset of this spike's first event in its trial's accept list
};

template <typename T> struct FixedOf;
template <> struct FixedOf<float> { typedef int32_t type; };
template <> struct FixedOf<double> { typedef int64_t type; };

struct Error {
  int code = OK;
  std::string msg;
};

template <typename T, bool DEV>
struct Trial;

struct Session {
  Cfg cfg;
  // network (double copies; cast to T at use)
  std::vector<int64_t> rowptr;
  std::vector<int32_t> col;
  std::vector<double> w, d;
  std::vector<uint32_t> mask;  // [B][T][W]
  std::vector<double> amp;     // [N]
  int words = 0;
  int horizon = 0;
  int capacity = 0;            // bounded kinds
  // outputs
  std::vector<double> v_out, i_out, v_trace;
  std::vector<Spike> spikes;
  std::vector<int64_t> counters;   // [B][3]
  std::vector<std::vector<uint8_t>> accepted;  // per trial, per event in fan-out order
  std::vector<int64_t> pending;    // [B][N][horizon][2] fixed (device mode)
  std::vector<double> pending_ref; // [B][N][horizon][2] (reference mode)
  std::string err;
  bool forward_done = false;
};

inline bool drive_on(const Session& s, int b, int m, int j) {
  const uint32_t* row = s.mask.data() + ((size_t)b * s.cfg.t_steps + m) * s.words;
  return (row[j >> 5] >> (j & 31)) & 1u;
}

template <typename T, bool DEV> inline T xexp(T x) {
  if (DEV) return eq_exp_t(x);
  return (T)std::exp((double)x);
}
template <typename T, bool DEV> inline T xlog(T x) {
  if (DEV) return eq_log_t(x);
  return (T)std::log((double)x);
}

/*
 * delivery_step (jumps.py:90-96) for a spike emitted in loop step m:
 * max(ceil(t_post/dt), m+2).  For t_spk in (m dt, (m+1) dt] exact arithmetic
 * bounds ceil(t_post/dt) to [m+1+floor(d/dt), m+1+ceil(d/dt)] — one value when
 * d is grid-aligned (|d/dt - k| <= tol*k, tol 1e-5 fp32 / 1e-12 fp64).  Device
 * mode clamps to those bounds so rounding of t_post/dt (frequent in fp32 near
 * a step edge) cannot move an event by a step; reference mode is literal.
 */
template <typename T, bool DEV>
inline int32_t delivery(T t_post, T d, T dt, int m) {
  int32_t q = (int32_t)std::ceil(t_post / dt);
  if (DEV) {
    const T tol = sizeof(T) == 4 ? (T)1e-5 : (T)1e-12;
    const T kd = d / dt;
    const T kr = std::rint(kd);
    int32_t lo, hi;
    if (std::fabs(kd - kr) <= tol * (kr > (T)1 ? kr : (T)1)) {
      lo = hi = m + 1 + (int32_t)kr;
    } else {
      lo = m + 1 + (int32_t)std::floor(kd);
      hi = m + 1 + (int32_t)std::ceil(kd);
    }
    q = std::min(std::max(q, lo), hi);
  }
  return std::max(q, (int32_t)(m + 2));
}

// fixed-point helpers (device mode): q = rint(v * 2^F), v = q * 2^-F
template <typename A> inline A to_fixed(double v, int F) {
  return (A)std::llrint(std::ldexp(v, F));
}
template <typename T, typename A> inline T from_fixed(A q, int F) {
  return (T)std::ldexp((double)q, -F);
}

/* One trial of the primal simulation. */
template <typename T, bool DEV>
struct Trial {
  typedef typename FixedOf<T>::type A;
  struct Ev { int32_t due; A fs, fm; double rs, rm; };

  const Session& S;
  const Cfg& c;
  int b;
  int N, R;
  std::vector<T> I, V;
  std::vector<int32_t> refr;
  // ring storage: [R][N] pairs
  std::vector<A> ring_f;       // device mode
  std::vector<double> ring_r;  // reference mode
  std::vector<uint8_t> ring_occ;
  // bounded storage
  std::vector<std::vector<Ev>> pool;
  std::vector<int32_t> tail_key;
  int64_t n_spk = 0, n_enq = 0, n_drop = 0;
  std::vector<uint8_t> acc;        // accepted flag per event, fan-out order
  Error e;

  Trial(const Session& s, int trial) : S(s), c(s.cfg), b(trial) {
    N = c.n;
    // lossy ring: slot = step % capacity; any capacity >= horizon behaves as a
    // horizon-slot ring (no step in flight aliases), so storage is min of both
    R = c.kind == K_LOSSY ? std::min(S.capacity, S.horizon) : S.horizon;
    I.assign(N, (T)0);
    V.assign(N, (T)c.v_reset);
    refr.assign(N, 0);
    if (c.kind == K_RING || c.kind == K_LOSSY) {
      if (DEV) ring_f.assign((size_t)R * N * 2, 0);
      else ring_r.assign((size_t)R * N * 2, 0.0);
      ring_occ.assign((size_t)R * N, 0);
    } else if (c.kind != K_DONOTHING) {
      pool.resize(N);
      tail_key.assign(N, -1);
    }
  }

  // pop slot `now` for neuron j -> (ps, pm)
  inline void pop(int j, int now, T& ps, T& pm) {
    ps = (T)0; pm = (T)0;
    if (c.kind == K_RING || c.kind == K_LOSSY) {
      size_t k = (size_t)(now % R) * N + j;
      if (DEV) {
        ps = from_fixed<T, A>(ring_f[2 * k], c.frac_bits);
        pm = from_fixed<T, A>(ring_f[2 * k + 1], c.frac_bits);
        ring_f[2 * k] = 0; ring_f[2 * k + 1] = 0;
      } else {
        ps = (T)ring_r[2 * k]; pm = (T)ring_r[2 * k + 1];
        ring_r[2 * k] = 0.0; ring_r[2 * k + 1] = 0.0;
      }
      ring_occ[k] = 0;
    } else if (c.kind != K_DONOTHING) {
      std::vector<Ev>& q = pool[j];
      A fs = 0, fm = 0;
      double rs = 0.0, rm = 0.0;
      size_t keep = 0;
      for (size_t x = 0; x < q.size(); ++x) {
        if (q[x].due == now) {   // merged in insertion order (= (due, seq) order)
          fs += q[x].fs; fm += q[x].fm;
          rs += q[x].rs; rm += q[x].rm;
        } else {
          q[keep++] = q[x];
        }
      }
      q.resize(keep);
      if (DEV) { ps = from_fixed<T, A>(fs, c.frac_bits); pm = from_fixed<T, A>(fm, c.frac_bits); }
      else { ps = (T)rs; pm = (T)rm; }
    }
  }

  // enqueue one event; returns false when dropped
  inline bool enqueue(int j, int now, int32_t dstep, T ws, T wm) {
    if (dstep < now) {
      e.code = E_CAUSALITY;
      e.msg = "event for step " + std::to_string(dstep) + " enqueued at step " + std::to_string(now);
      return false;
    }
    if (c.kind == K_DONOTHING) return false;
    if (c.kind == K_RING || c.kind == K_LOSSY) {
      if (c.kind == K_RING && dstep - now >= R) {
        e.code = E_CAPABILITY;
        e.msg = "ring: delay of " + std::to_string(dstep - now + 1) + " steps exceeds buffer capacity " + std::to_string(R);
        return false;
      }
      size_t k = (size_t)(dstep % R) * N + j;
      if (DEV) {
        ring_f[2 * k] += to_fixed<A>((double)ws, c.frac_bits);
        ring_f[2 * k + 1] += to_fixed<A>((double)wm, c.frac_bits);
      } else {
        ring_r[2 * k] += (double)ws;
        ring_r[2 * k + 1] += (double)wm;
      }
      ring_occ[k] = 1;
      return true;
    }
    if (c.kind == K_FIFO && dstep < tail_key[j]) {
      e.code = E_CAPABILITY;
      e.msg = "fiforing supports homogeneous delays only: event for step " + std::to_string(dstep) +
              " arrived after one for step " + std::to_string(tail_key[j]);
      return false;
    }
    std::vector<Ev>& q = pool[j];
    if ((int)q.size() == S.capacity) return false;
    Ev ev;
    ev.due = dstep;
    ev.fs = DEV ? to_fixed<A>((double)ws, c.frac_bits) : 0;
    ev.fm = DEV ? to_fixed<A>((double)wm, c.frac_bits) : 0;
    ev.rs = (double)ws; ev.rm = (double)wm;
    q.push_back(ev);
    if (c.kind == K_FIFO) tail_key[j] = dstep;
    return true;
  }

  void run(std::vector<Spike>& out, double* vtrace) {
    const T dt = (T)c.dt, tau_m = (T)c.tau_m, tau_s = (T)c.tau_syn;
    const T v_th = (T)c.v_th, v_reset = (T)c.v_reset;
    // constants as the reference computes them (network.py:527-528, 183-185)
    const T k_m = (T)std::exp(-c.dt / c.tau_m);
    const T k_s = (T)std::exp(-c.dt / c.tau_syn);
    const T cc = c.exact_delivery ? (T)(c.tau_syn / (c.tau_m - c.tau_syn)) : (T)0;
    const bool exact = c.exact_delivery != 0;
    const T inv_s = (T)(1.0 / c.tau_syn), inv_m = (T)(1.0 / c.tau_m);
    std::vector<int> crossing;
    std::vector<T> cross_t;
    for (int m = 0; m < c.t_steps && e.code == OK; ++m) {
      crossing.clear(); cross_t.clear();
      for (int j = 0; j < N; ++j) {
        T ps, pm;
        pop(j, m, ps, pm);
        if (!exact) pm = (T)0;
        T i = (I[j] + ps) * k_s;                              // network.py:559
        I[j] = i;
        T drive = drive_on(S, b, m, j) ? (T)S.amp[j] : (T)0;
        T a = i + drive;                                       // :561
        T v = V[j];
        if (exact) v = v + cc * (pm - ps);                      // :564
        T v_new = a + (v - a) * k_m;                            // :565
        if (refr[j] > 0) {                                      // :566-567
          refr[j] -= 1;
        } else if (v < v_th && v_th <= v_new) {                 // :568
          T v_dot = (a - v_th) / tau_m;                         // :569
          if (v_dot < (T)1e-9) {
            e.code = E_GRAZING;
            e.msg = "grazing crossing at step " + std::to_string(m + 1);
            return;
          }
          T r = (v_th - a) / (v - a);                           // :574
          T t_spk = (T)m * dt - tau_m * xlog<T, DEV>(r);        // :575
          T u = (T)(m + 1) * dt - t_spk;                        // :576
          v_new = a + (v_reset - a) * xexp<T, DEV>(-u / tau_m); // :577
          refr[j] = c.refractory_steps;                         // :578
          crossing.push_back(j);
          cross_t.push_back(t_spk);
          Spike sp;
          sp.step = m; sp.trial = b; sp.neuron = j;
          sp.t = (double)t_spk; sp.a = (double)a; sp.vh = (double)v;
          out.push_back(sp);
        }
        V[j] = v_new;                                           // :580
      }
      if (vtrace) for (int j = 0; j < N; ++j) vtrace[(size_t)m * N + j] = (double)V[j];
      // fan-out in ascending source order, CSR row order (network.py:583-611)
      const int now = m + 1;  // queues were popped for step m
      const size_t first = out.size() - crossing.size();
      for (size_t k = 0; k < crossing.size() && e.code == OK; ++k) {
        int i = crossing[k];
        T t_spk = cross_t[k];
        n_spk += 1;
        out[first + k].ev_off = (int64_t)acc.size();
        for (int64_t x = S.rowptr[i]; x < S.rowptr[i + 1]; ++x) {
          int j = S.col[x];
          T d = (T)S.d[x];
          T t_post = t_spk + d;                                 // :588
          int32_t dstep = delivery<T, DEV>(t_post, d, dt, m);   // jumps.py:96
          n_enq += 1;
          T w = (T)S.w[x];
          T ws, wm;
          if (exact) {
            T phi = (T)dstep * dt - t_post;                     // :599
            // device mode multiplies by (T)(1/tau) per event
            ws = w * xexp<T, DEV>(DEV ? -phi * inv_s : -phi / tau_s);  // :601
            wm = w * xexp<T, DEV>(DEV ? -phi * inv_m : -phi / tau_m);  // :606
          } else {
            ws = w; wm = (T)0;
          }
          bool ok = enqueue(j, now, dstep, ws, wm);
          if (e.code != OK) return;
          if (!ok) n_drop += 1;
          acc.push_back(ok || c.kind == K_RING || c.kind == K_LOSSY ? 1 : 0);
        }
      }
    }
  }
};

template <typename T, bool DEV>
int run_forward(Session& s) {
  const Cfg& c = s.cfg;
  int B = c.n_trials, N = c.n;
  s.v_out.assign((size_t)B * N, 0.0);
  s.i_out.assign((size_t)B * N, 0.0);
  s.counters.assign((size_t)B * 3, 0);
  if (c.record_v) s.v_trace.assign((size_t)B * c.t_steps * N, 0.0);
  else s.v_trace.clear();
  s.pending.assign(DEV ? (size_t)B * N * s.horizon * 2 : 0, 0);
  s.pending_ref.assign(DEV ? 0 : (size_t)B * N * s.horizon * 2, 0.0);
  std::vector<std::vector<Spike>> per_trial(B);
  std::vector<Error> errs(B);
  s.accepted.assign(B, std::vector<uint8_t>());
#pragma omp parallel for schedule(dynamic, 1)
  for (int b = 0; b < B; ++b) {
    Trial<T, DEV> tr(s, b);
    tr.run(per_trial[b], c.record_v ? s.v_trace.data() + (size_t)b * c.t_steps * N : nullptr);
    errs[b] = tr.e;
    s.accepted[b].swap(tr.acc);
    for (int j = 0; j < N; ++j) {
      s.v_out[(size_t)b * N + j] = (double)tr.V[j];
      s.i_out[(size_t)b * N + j] = (double)tr.I[j];
    }
    s.counters[3 * b] = tr.n_spk;
    s.counters[3 * b + 1] = tr.n_enq;
    s.counters[3 * b + 2] = tr.n_drop;
    // canonical pending contents: due steps T .. T+horizon-1
    int H = s.horizon;
    if (c.kind == K_FIFO || c.kind == K_HEAP || c.kind == K_SORTED) {   // one pass over each pool
      for (int j = 0; j < N; ++j) {
        for (auto& ev : tr.pool[j]) {
          const int k = ev.due - c.t_steps;
          if (k < 0 || k >= H) continue;
          size_t o = (((size_t)b * N + j) * H + k) * 2;
          if (DEV) { s.pending[o] += ev.fs; s.pending[o + 1] += ev.fm; }
          else { s.pending_ref[o] += ev.rs; s.pending_ref[o + 1] += ev.rm; }
        }
      }
      continue;
    }
    for (int j = 0; j < N; ++j) {
      for (int k = 0; k < H; ++k) {
        int due = c.t_steps + k;
        typename FixedOf<T>::type fs = 0, fm = 0;
        double rs = 0.0, rm = 0.0;
        if (c.kind == K_RING || (c.kind == K_LOSSY && k < tr.R)) {
          // (a lossy ring's slot k >= R would alias an earlier due step)
          size_t q = (size_t)(due % tr.R) * N + j;
          if (DEV) { fs = tr.ring_f[2 * q]; fm = tr.ring_f[2 * q + 1]; }
          else { rs = tr.ring_r[2 * q]; rm = tr.ring_r[2 * q + 1]; }
        } else if (c.kind == K_LOSSY) {
        } else if (c.kind != K_DONOTHING) {
          for (auto& ev : tr.pool[j]) if (ev.due == due) { fs += ev.fs; fm += ev.fm; rs += ev.rs; rm += ev.rm; }
        }
        size_t o = (((size_t)b * N + j) * H + k) * 2;
        if (DEV) { s.pending[o] = fs; s.pending[o + 1] = fm; }
        else { s.pending_ref[o] = rs; s.pending_ref[o + 1] = rm; }
      }
    }
  }
  for (int b = 0; b < B; ++b) {
    if (errs[b].code != OK) { s.err = errs[b].msg; return errs[b].code; }
  }
  s.spikes.clear();
  for (int b = 0; b < B; ++b) s.spikes.insert(s.spikes.end(), per_trial[b].begin(), per_trial[b].end());
  s.forward_done = true;
  return OK;
}

/*
 * Reverse mode.  For each trial, walking m = T-1 .. 0:
 *   R-fanout(m): every spike of step m gathers the reverse slot adjoints
 *     Lambda_s, Lambda_m at its events' delivery steps s (zero for s >= T) and
 *     produces dL/dw_e, dL/dd_e and dL/dt_spk.
 *   R-neuron(m): per neuron, the adjoint of F1..F6 of PrimalRSNN.step.
 * dL/dt_spk of one spike is the sequential sum over its row in CSR order (the
 * order the kernel's per-spike reduction uses), so lambda_t matches bitwise.
 * Gradients accumulate in double.
 */
template <typename T, bool DEV>
int run_backward(Session& s, const double* vbar, const double* ibar, double* gw, double* gd, double* gamp) {
  const Cfg& c = s.cfg;
  if (c.kind == K_DONOTHING) { /* every event dropped: only the neuron recurrences remain */ }
  const bool exact = c.exact_delivery != 0;
  int B = c.n_trials, N = c.n, TT = c.t_steps;
  size_t E = s.col.size();
  const T dt = (T)c.dt, tau_m = (T)c.tau_m, tau_s = (T)c.tau_syn;
  const T v_th = (T)c.v_th, v_reset = (T)c.v_reset;
  const T k_m = (T)std::exp(-c.dt / c.tau_m);
  const T k_s = (T)std::exp(-c.dt / c.tau_syn);
  // exact delivery: Lambda_m = c * lambda_vhat is the membrane twin payload's
  // adjoint; plain delivery: Lambda_m = -lambda_vhat carries the membrane's
  // -Q/tau_m tangent term, and there is no bump (c = 0)
  const T cc = exact ? (T)(c.tau_syn / (c.tau_m - c.tau_syn)) : (T)0;
  const T cm = exact ? cc : (T)-1;
  const T inv_s = (T)(1.0 / c.tau_syn), inv_m = (T)(1.0 / c.tau_m);
  const int R = s.horizon + 1;
  const int lossy_cap = c.kind == K_LOSSY ? s.capacity : 0;
  std::fill(gw, gw + E, 0.0);
  std::fill(gd, gd + E, 0.0);
  std::fill(gamp, gamp + N, 0.0);
  // spikes grouped by (trial, step)
  std::vector<std::vector<std::vector<int>>> by(B, std::vector<std::vector<int>>(TT));
  for (size_t k = 0; k < s.spikes.size(); ++k) by[s.spikes[k].trial][s.spikes[k].step].push_back((int)k);

  int P = 1;
#ifdef _OPENMP
  P = omp_get_max_threads();
#endif
  std::vector<std::vector<double>> pw(P, std::vector<double>(E)), pd(P, std::vector<double>(E)),
      pa(P, std::vector<double>(N));
  for (int b0 = 0; b0 < B; b0 += P) {
    int nb = std::min(P, B - b0);
#pragma omp parallel for schedule(dynamic, 1)
    for (int q = 0; q < nb; ++q) {
      int b = b0 + q;
      std::vector<double>& lw = pw[q];
      std::vector<double>& ld = pd[q];
      std::vector<double>& la_acc = pa[q];
      std::fill(lw.begin(), lw.end(), 0.0);
      std::fill(ld.begin(), ld.end(), 0.0);
      std::fill(la_acc.begin(), la_acc.end(), 0.0);
      std::vector<T> lV(N), lI(N);
      for (int j = 0; j < N; ++j) {
        lV[j] = (T)vbar[(size_t)b * N + j];
        lI[j] = ibar ? (T)ibar[(size_t)b * N + j] : (T)0;
      }
      std::vector<T> Ls((size_t)R * N, (T)0), Lm((size_t)R * N, (T)0);
      std::vector<T> spk_lt(N, (T)0);
      std::vector<int> spk_of(N, -1);
      for (int m = TT - 1; m >= 0; --m) {
        const std::vector<int>& list = by[b][m];
        // R-fanout(m)
        for (int k : list) {
          const Spike& sp = s.spikes[k];
          int i = sp.neuron;
          T t = (T)sp.t;
          // dL/dt_spk: sequential sum over the row in CSR order, zeros for
          // events delivered at or after T (the kernel's reduction order)
          T lt_sum = (T)0;
          int64_t r0 = s.rowptr[i], r1 = s.rowptr[i + 1];
          const uint8_t* okv = s.accepted[b].data() + sp.ev_off;
          for (int64_t x = r0; x < r1; ++x) {
            int j = s.col[x];
            T w = (T)s.w[x];
            T dd = (T)s.d[x];
            T t_post = t + dd;
            int32_t st = delivery<T, DEV>(t_post, dd, dt, m);
            // the step the event is popped at: st, or for a lossy ring the
            // first step >= m+1 in st's residue class mod capacity
            int32_t sp = st;
            if (lossy_cap > 0 && st - (m + 1) >= lossy_cap) sp = (m + 1) + (st - (m + 1)) % lossy_cap;
            if (sp >= TT || !okv[x - r0]) { lt_sum = lt_sum + (T)0; continue; }
            T es = (T)1, em = (T)1;
            if (exact) {
              T phi = (T)st * dt - t_post;
              es = xexp<T, DEV>(DEV ? -phi * inv_s : -phi / tau_s);
              em = xexp<T, DEV>(DEV ? -phi * inv_m : -phi / tau_m);
            }
            size_t o = (size_t)(sp % R) * N + j;
            T as = Ls[o], am = Lm[o];
            T g_w = exact ? es * as + em * am : as;
            T g_tp = DEV ? w * (es * as * inv_s + em * am * inv_m) : w * (es * as / tau_s + em * am / tau_m);
            lw[x] += (double)g_w;
            ld[x] += (double)g_tp;
            lt_sum = lt_sum + g_tp;
          }
          spk_lt[i] = lt_sum;
          spk_of[i] = k;
        }
        // R-neuron(m)
        for (int j = 0; j < N; ++j) {
          T lv = lV[j];
          T la, lvh;
          if (spk_of[j] >= 0) {
            const Spike& sp = s.spikes[spk_of[j]];
            T t = (T)sp.t, a = (T)sp.a, vh = (T)sp.vh;
            T u = (T)(m + 1) * dt - t;
            T ku = xexp<T, DEV>(-u / tau_m);
            T r = (v_th - a) / (vh - a);
            T lt = spk_lt[j] + lv * (v_reset - a) * ku / tau_m;
            T lr = -tau_m * lt / r;
            T den = vh - a;
            T den2 = den * den;
            la = lv * ((T)1 - ku) + lr * (v_th - vh) / den2;
            lvh = -lr * (v_th - a) / den2;
            spk_of[j] = -1;
          } else {
            la = lv * ((T)1 - k_m);
            lvh = lv * k_m;
          }
          T lip = lI[j] + la;
          if (drive_on(s, b, m, j)) la_acc[j] += (double)la;
          size_t o = (size_t)(m % R) * N + j;
          Lm[o] = cm * lvh;
          Ls[o] = k_s * lip - cc * lvh;
          lI[j] = k_s * lip;
          lV[j] = lvh;
        }
      }
    }
    // fixed-order reduction over trials (deterministic regardless of threads)
#pragma omp parallel for schedule(static)
    for (int64_t x = 0; x < (int64_t)E; ++x)
      for (int q = 0; q < nb; ++q) { gw[x] += pw[q][x]; gd[x] += pd[q][x]; }
    for (int j = 0; j < N; ++j)
      for (int q = 0; q < nb; ++q) gamp[j] += pa[q][j];
  }
  return OK;
}

}  // namespace

extern "C" {

struct eqo_cfg {
  int32_t kind, n, n_trials, t_steps, refractory_steps, exact_delivery, capacity, frac_bits;
  int32_t mode, precision, record_v, pad;
  double dt, tau_m, tau_syn, v_th, v_reset;
};

void* eqo_create(const eqo_cfg* cfg) {
  Session* s = new Session();
  std::memcpy(&s->cfg, cfg, sizeof(Cfg));
  s->words = (cfg->n + 31) / 32;
  return s;
}

void eqo_destroy(void* h) { delete (Session*)h; }

const char* eqo_error(void* h) { return ((Session*)h)->err.c_str(); }

int eqo_set_network(void* h, const int64_t* rowptr, const int32_t* col, const double* w, const double* d) {
  Session* s = (Session*)h;
  const Cfg& c = s->cfg;
  int N = c.n;
  s->rowptr.assign(rowptr, rowptr + N + 1);
  int64_t E = rowptr[N];
  s->col.assign(col, col + E);
  s->w.assign(w, w + E);
  s->d.assign(d, d + E);
  // horizon = max ceil(d/dt) + 1 in the working precision (network.py:188-198)
  int hmax = 1;
  for (int64_t x = 0; x < E; ++x) {
    int q;
    if (c.mode == 1 && c.precision == 32) q = (int)std::ceil((float)d[x] / (float)c.dt);
    else q = (int)std::ceil(d[x] / c.dt);
    hmax = std::max(hmax, q);
  }
  s->horizon = hmax + 1;
  if (c.kind == K_FIFO || c.kind == K_HEAP || c.kind == K_SORTED || c.kind == K_LOSSY)
    s->capacity = c.capacity > 0 ? c.capacity : s->horizon * (N - 1) + 1;  // network.py:327
  return OK;
}

int eqo_horizon(void* h) { return ((Session*)h)->horizon; }

int eqo_set_drive(void* h, const uint32_t* mask, const double* amp) {
  Session* s = (Session*)h;
  const Cfg& c = s->cfg;
  s->mask.assign(mask, mask + (size_t)c.n_trials * c.t_steps * s->words);
  s->amp.assign(amp, amp + c.n);
  return OK;
}

int eqo_forward(void* h) {
  Session* s = (Session*)h;
  const Cfg& c = s->cfg;
  if (c.mode == 0) return run_forward<double, false>(*s);
  if (c.precision == 32) return run_forward<float, true>(*s);
  return run_forward<double, true>(*s);
}

int eqo_backward(void* h, const double* vbar, const double* ibar, double* gw, double* gd, double* gamp) {
  Session* s = (Session*)h;
  const Cfg& c = s->cfg;
  if (!s->forward_done) { s->err = "backward before forward"; return E_CONFIG; }
  if (c.mode == 0) return run_backward<double, false>(*s, vbar, ibar, gw, gd, gamp);
  if (c.precision == 32) return run_backward<float, true>(*s, vbar, ibar, gw, gd, gamp);
  return run_backward<double, true>(*s, vbar, ibar, gw, gd, gamp);
}

int64_t eqo_spike_count(void* h) { return (int64_t)((Session*)h)->spikes.size(); }

void eqo_get_spikes(void* h, int32_t* step, int32_t* trial, int32_t* neuron, double* t, double* a, double* vh) {
  Session* s = (Session*)h;
  for (size_t k = 0; k < s->spikes.size(); ++k) {
    const Spike& sp = s->spikes[k];
    step[k] = sp.step; trial[k] = sp.trial; neuron[k] = sp.neuron;
    t[k] = sp.t; a[k] = sp.a; vh[k] = sp.vh;
  }
}

void eqo_get_state(void* h, double* v, double* i) {
  Session* s = (Session*)h;
  std::copy(s->v_out.begin(), s->v_out.end(), v);
  std::copy(s->i_out.begin(), s->i_out.end(), i);
}

void eqo_get_vtrace(void* h, double* out) {
  Session* s = (Session*)h;
  std::copy(s->v_trace.begin(), s->v_trace.end(), out);
}

void eqo_get_counters(void* h, int64_t* out) {
  Session* s = (Session*)h;
  std::copy(s->counters.begin(), s->counters.end(), out);
}

void eqo_get_pending(void* h, int64_t* fixed_out, double* ref_out) {
  Session* s = (Session*)h;
  if (fixed_out) std::copy(s->pending.begin(), s->pending.end(), fixed_out);
  if (ref_out) std::copy(s->pending_ref.begin(), s->pending_ref.end(), ref_out);
}

int eqo_threads(void) {
#ifdef _OPENMP
  return omp_get_max_threads();
#else
  return 1;
#endif
}

}  // extern "C"

extern "C" {
/* Vectorised access to the shared eq_math.h functions (accuracy tests):
 * which = 0 exp, 1 log (double); 2 expf, 3 logf (float, carried in double). */
void eqo_math(int which, const double* in, double* out, int64_t n) {
  for (int64_t k = 0; k < n; ++k) {
    switch (which) {
      case 0: out[k] = eq_exp(in[k]); break;
      case 1: out[k] = eq_log(in[k]); break;
      case 2: out[k] = (double)eq_expf((float)in[k]); break;
      default: out[k] = (double)eq_logf((float)in[k]); break;
    }
  }
}
}

extern "C" {
/* On-device PoissonDrive restated (paper_2512_05906_b200/csrc/eq_drive.cu):
 * the reference's pulse-train walk (pkg/src/eventq/network.py:113-120) and
 * grid sampling (:138-143) with per-(trial, neuron) Philox4x32-10 streams
 * (Salmon et al., SC'11; Random123 round constants) instead of numpy's PCG64. */
void eqo_philox4x32_10(const uint32_t* ctr_in, const uint32_t* key, uint32_t* out) {
  uint32_t x0 = ctr_in[0], x1 = ctr_in[1], x2 = ctr_in[2], x3 = ctr_in[3];
  uint32_t k0 = key[0], k1 = key[1];
  for (int r = 0; r < 10; ++r) {
    const uint64_t p0 = (uint64_t)0xD2511F53u * x0;
    const uint64_t p1 = (uint64_t)0xCD9E8D57u * x2;
    const uint32_t y0 = (uint32_t)(p1 >> 32) ^ x1 ^ k0;
    const uint32_t y1 = (uint32_t)p1;
    const uint32_t y2 = (uint32_t)(p0 >> 32) ^ x3 ^ k1;
    const uint32_t y3 = (uint32_t)p0;
    x0 = y0; x1 = y1; x2 = y2; x3 = y3;
    k0 += 0x9E3779B9u;
    k1 += 0xBB67AE85u;
  }
  out[0] = x0; out[1] = x1; out[2] = x2; out[3] = x3;
}

void eqo_poisson_drive(int32_t n, int32_t n_trials, int32_t t_steps, double dt, double mean, double dur,
                       uint64_t seed, uint32_t* mask) {
  const int words = (n + 31) / 32;
  const uint32_t key[2] = {(uint32_t)seed, (uint32_t)(seed >> 32)};
  const double t_total = (double)t_steps * dt;
  std::fill(mask, mask + (size_t)n_trials * t_steps * words, 0u);
  for (int b = 0; b < n_trials; ++b)
    for (int i = 0; i < n; ++i) {
      uint32_t call = 0;
      std::vector<double> pend;   // draws of the current Philox call not yet used
      auto draw = [&]() {
        if (pend.empty()) {
          const uint32_t c[4] = {call++, (uint32_t)i, (uint32_t)b, 0x5d0f1eedu};
          uint32_t o[4];
          eqo_philox4x32_10(c, key, o);
          const double inv53 = 1.0 / 9007199254740992.0;
          const double ua = ((double)(o[0] >> 5) * 67108864.0 + (double)(o[1] >> 6) + 0.5) * inv53;
          const double ub = ((double)(o[2] >> 5) * 67108864.0 + (double)(o[3] >> 6) + 0.5) * inv53;
          pend.push_back(-mean * eq_log(ub));
          pend.push_back(-mean * eq_log(ua));
        }
        const double v = pend.back();
        pend.pop_back();
        return v;
      };
      double t = draw();                                   // network.py:116
      while (t < t_total) {                                // :117
        const double s = t, e = s + dur;
        const long long lo = std::min<long long>(t_steps, std::max<long long>(0, (long long)std::ceil(s / dt)));
        const long long hi = std::min<long long>(t_steps, std::max<long long>(0, (long long)std::ceil(e / dt)));
        for (long long m = lo; m < hi; ++m)
          mask[((size_t)b * t_steps + m) * words + (i >> 5)] |= 1u << (i & 31);
        t += dur + draw();                                 // :118
      }
    }
}
}  // extern "C"
