// eq_jvp.cuh — batched forward-mode (JVP) run: the reference's native gradient
// mode (forward_gradient, network.py:668-683; build_rsnn seeding :273-291;
// PoissonDrive.materialize seeded_neuron :123-155) for D seeded directions at
// once, as extra tangent lanes of one primal trajectory.
//
// fp64, ring kind, exact or plain delivery.  The primal arithmetic is the engine's
// (lif_step, fixed-point slot sums in the DRAM ring rows), so the raster is
// the forward kernel's; each direction d carries the reference's dual parts:
//   synapse    I' += W_s' + Q_s/tau_s; I' *= k_s            (neuro.py:33-47, jumps.py:116-126)
//   membrane   v' = V' + c (W_m' + Q_m/tau_m - W_s' - Q_s/tau_s)      (network.py:392-401)
//              (plain delivery: v' = V' - Q_s/tau_m, neuro.py:146-149 delivered_wtt;
//               payloads w with no phase factor, network.py:403-408, 438)
//              v_new' = a' + (v' - a') k_m                  (neuro.py:150-154)
//   crossing   r' = (num' den - num den') / den^2, tdot = -tau_m r'/r (neuro.py:200-210)
//   reset      v_new' = a' + (-a') ku + (v_r - a) ku tdot / tau_m     (neuro.py:161-175)
//   fan-out    tt = tdot + d'_e, W' = w'_e e^{-phi/tau}, Q += (w e^{-phi/tau}) tt
//                                                           (network.py:429-437, jumps.py:83-87)
// Tangent slot sums are double atomics (order-dependent in the last bits; the
// JVP is compared with a tolerance).  Five kernels per step (primal update,
// tangent update per (neuron, direction), offsets, fan-out per (event,
// direction), next) read the step from device memory; the host captures a block
// of steps once as a CUDA graph and replays it (the run is launch-bound
// otherwise: ~6 us of host time per kernel at C1).
#pragma once

#include "eq_ring.cuh"

namespace eq {

struct JvpArgs {
  int N, B, D, R, refractory;
  int exact;              // exact delivery (else plain)
  int* m_dev;             // current step (device-side, so a CUDA graph of steps replays unchanged)
  long long total;
  StepConsts<double> c;
  NetView<double> net;
  double* I;
  double* V;
  int32_t* refr;
  long long* ring;        // [B][R][N][2] primal fixed-point slots
  double* tI;             // [B][D][N]
  double* tV;             // [B][D][N]
  double* tslot;          // [B][D][R][N][4]: W_s', Q_s, W_m', Q_m
  const int* dkind;       // [D] 0 weight, 1 delay, 2 drive
  const long long* dindex;  // [D] edge index (weight/delay) or neuron (drive)
  int* spk_idx;           // [cap] flat neuron-trial of each spike of this step
  double* spk_t;          // [cap]
  double* spk_tdot;       // [cap][D]
  double *pa, *pv, *pr, *pku;   // [total] primal intermediates of this step (a, v-hat, r, e^{-u/tau_m})
  int2* pinfo;            // [total] {on | crossed << 1, spike slot}
  int* spk_n;             // spikes of this step
  int spk_cap;
  long long* counters;    // [B][3]
  int* err;
};

// Primal step of every neuron (one thread each); the quantities the tangent
// recurrences need are kept per neuron for k_jvp_tangent.
__global__ void k_jvp_update(JvpArgs A) {
  typedef Prec<double> P;
  const long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (idx >= A.total) return;
  const StepConsts<double>& c = A.c;
  const int m = *A.m_dev;
  const int b = (int)(idx / A.N);
  const int j = (int)(idx - (long long)b * A.N);
  // primal pop + clear (RingQueue._pop_raw, queues.py:109-120)
  const size_t so = ((size_t)b * A.R + (size_t)(m % A.R)) * A.N + j;
  const double ps = P::deq(A.ring[2 * so], c.inv_scale), pm = P::deq(A.ring[2 * so + 1], c.inv_scale);
  A.ring[2 * so] = 0;
  A.ring[2 * so + 1] = 0;
  const bool on = drive_bit(A.net, b, m, j);
  const double drive = on ? A.net.amp[j] : 0.0;
  int rf = A.refractory ? A.refr[idx] : 0;
  double i, v_new, a, v, t_spk;
  const bool spike = lif_step<double>(c, A.exact != 0, A.refractory, m, ps, A.exact ? pm : 0.0, A.I[idx], A.V[idx],
                                      drive, rf, i, v_new, a, v, t_spk);
  if (spike && t_spk != t_spk) {
    raise_error(A.err, EQ_ERR_GRAZING, m + 1, b, j);
    return;
  }
  const bool crossed = spike;   // lif_step reports a crossing only outside refractoriness
  double ku = 0.0, r = 0.0;
  int slot = -1;
  if (crossed) {
    r = (c.v_th - a) / (v - a);                             // neuro.py:196-201 (same ops as lif_step)
    const double uu = (double)(m + 1) * c.dt - t_spk;
    ku = eq_exp_t(-uu / c.tau_m);
    slot = atomicAdd(A.spk_n, 1);
    if (slot < A.spk_cap) {
      A.spk_idx[slot] = (int)idx;
      A.spk_t[slot] = t_spk;
    } else {
      raise_error(A.err, EQ_ERR_CAPACITY, m, b, j);
      slot = -1;
    }
  }
  A.pa[idx] = a;
  A.pv[idx] = v;
  A.pr[idx] = r;
  A.pku[idx] = ku;
  A.pinfo[idx] = make_int2((on ? 1 : 0) | (crossed ? 2 : 0), slot);
  A.I[idx] = i;
  A.V[idx] = v_new;
  if (A.refractory) A.refr[idx] = rf;
}

// Tangent step: one thread per (trial, direction, neuron), neuron fastest
// (coalesced tangent state and slots).
__global__ void k_jvp_tangent(JvpArgs A) {
  const long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (t >= A.total * A.D) return;
  const StepConsts<double>& c = A.c;
  const int m = *A.m_dev;
  const int j = (int)(t % A.N);
  const long long bd = t / A.N;                             // b * D + d
  const int d = (int)(bd % A.D);
  const int b = (int)(bd / A.D);
  const long long idx = (long long)b * A.N + j;
  const int2 info = A.pinfo[idx];
  const bool on = info.x & 1, crossed = info.x & 2;
  const size_t ts = (size_t)bd * A.N + j;
  double* sl = A.tslot + (((size_t)bd * A.R + (size_t)(m % A.R)) * A.N + j) * 4;
  const double Ws = sl[0], Qs = sl[1], Wm = sl[2], Qm = sl[3];
  sl[0] = sl[1] = sl[2] = sl[3] = 0.0;
  double tI = A.tI[ts];
  tI = (tI + Ws + Qs / c.tau_s) * c.k_s;                    // apply_jump_pulse + dual_exp_decay
  const double ta = tI + ((on && A.dkind[d] == 2 && A.dindex[d] == j) ? 1.0 : 0.0);
  const double tv = A.exact ? A.tV[ts] + c.cc * (Wm + Qm / c.tau_m - Ws - Qs / c.tau_s)
                            : A.tV[ts] - Qs / c.tau_m;
  double tvn = ta + (tv - ta) * c.k_m;
  if (crossed) {
    const double a = A.pa[idx], v = A.pv[idx], r = A.pr[idx], ku = A.pku[idx];
    const double num_p = c.v_th - a, num_t = -ta;
    const double den_p = v - a, den_t = tv - ta;
    const double r_t = (num_t * den_p - num_p * den_t) / (den_p * den_p);
    const double tdot = -c.tau_m * r_t / r;
    const double rest_p = c.v_reset - a, rest_t = -ta;
    tvn = ta + (rest_t * ku + rest_p * (ku * tdot / c.tau_m));
    if (info.y >= 0) A.spk_tdot[(size_t)info.y * A.D + d] = tdot;
  }
  A.tI[ts] = tI;
  A.tV[ts] = tvn;
}

// One thread per (spike, out-edge) of this step's spikes.
__global__ void k_jvp_fanout(JvpArgs A, const long long* n_events_p, const long long* ev_off) {
  typedef Prec<double> P;
  const StepConsts<double>& c = A.c;
  const int n = *A.spk_n < A.spk_cap ? *A.spk_n : A.spk_cap;
  const long long n_items = *n_events_p * A.D;
  for (long long it = blockIdx.x * (long long)blockDim.x + threadIdx.x; it < n_items;
       it += (long long)gridDim.x * blockDim.x) {
    const long long f = it / A.D;                           // event; direction fastest across lanes
    const int dd = (int)(it - f * A.D);
    int lo = 0, hi = n;                                     // spike k: ev_off[k] <= f < ev_off[k+1]
    while (hi - lo > 1) {
      const int mid = (lo + hi) >> 1;
      if (ev_off[mid] <= f) lo = mid;
      else hi = mid;
    }
    const int k = lo;
    const int idx = A.spk_idx[k];
    const int b = idx / A.N, i = idx - b * A.N;
    const long long x = A.net.rowptr[i] + (f - ev_off[k]);
    const int j = A.net.col[x];
    const double w = A.net.w[x], d = A.net.d[x];
    const double t_post = A.spk_t[k] + d;                   // jumps.py:83-87
    const int ds = delivery_step_coded(t_post, A.net.dcode[x], c.dt, *A.m_dev);
    double es = 1.0, em = 0.0;                              // plain delivery: payload w, no twin
    if (A.exact) {
      const double phi = (double)ds * c.dt - t_post;
      es = eq_exp_t(-phi * c.inv_tau_s);
      em = eq_exp_t(-phi * c.inv_tau_m);
    }
    const double ws = w * es, wm = w * em;
    if (dd == 0) {
      const size_t so = ((size_t)b * A.R + (size_t)(ds % A.R)) * A.N + j;
      red_add(A.ring + 2 * so, P::q(ws, c.scale));
      red_add(A.ring + 2 * so + 1, P::q(wm, c.scale));
    }
    const double tt = A.spk_tdot[(size_t)k * A.D + dd] + ((A.dkind[dd] == 1 && A.dindex[dd] == x) ? 1.0 : 0.0);
    const double wt = (A.dkind[dd] == 0 && A.dindex[dd] == x) ? 1.0 : 0.0;
    double* sl = A.tslot + ((((size_t)b * A.D + dd) * A.R + (size_t)(ds % A.R)) * A.N + j) * 4;
    if (wt != 0.0) {
      atomicAdd(sl + 0, wt * es);                           // DualScalar.scale: (p c, t c)
      atomicAdd(sl + 2, wt * em);
    }
    if (tt != 0.0) {
      atomicAdd(sl + 1, ws * tt);                           // wtt += p * time_tangent
      atomicAdd(sl + 3, wm * tt);
    }
  }
}

// End of a step: advance the device-side step and empty the spike list.
__global__ void k_jvp_next(JvpArgs A) {
  *A.m_dev += 1;
  *A.spk_n = 0;
}

// Exclusive prefix of the step's spikes' out-degrees (one block).
__global__ void k_jvp_offsets(JvpArgs A, long long* ev_off, long long* n_events) {
  __shared__ long long s_sum[1024];
  const int n = *A.spk_n < A.spk_cap ? *A.spk_n : A.spk_cap;
  long long run = 0;
  for (int base = 0; base < n; base += blockDim.x) {
    const int k = base + threadIdx.x;
    long long len = 0;
    if (k < n) {
      const int idx = A.spk_idx[k];
      const int i = idx % A.N;
      len = A.net.rowptr[i + 1] - A.net.rowptr[i];
    }
    s_sum[threadIdx.x] = len;
    __syncthreads();
    for (int o = 1; o < (int)blockDim.x; o <<= 1) {        // inclusive scan (Hillis-Steele)
      const long long t = threadIdx.x >= o ? s_sum[threadIdx.x - o] : 0;
      __syncthreads();
      s_sum[threadIdx.x] += t;
      __syncthreads();
    }
    if (k < n) ev_off[k] = run + s_sum[threadIdx.x] - len;
    const long long blk = s_sum[blockDim.x - 1];
    __syncthreads();
    run += blk;
  }
  if (threadIdx.x == 0) {
    ev_off[n] = run;
    *n_events = run;
  }
}

}  // namespace eq
