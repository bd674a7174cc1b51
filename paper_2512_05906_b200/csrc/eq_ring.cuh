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

// Forward delivery into the L2-resident fixed-point accumulator (2 x B x N x 8 B,
// 38 MB at C3 x 24).  An evict-last policy on these reds measured no gain
// (profiles/r1g_ab_fwd_policies.txt): the accumulator stays in L2 anyway.
__device__ __forceinline__ void red_acc(long long* p, long long v) {
  asm volatile("red.relaxed.gpu.global.add.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

template <typename T>
struct StepConsts {
  T dt, tau_m, tau_s, v_th, v_reset, k_m, k_s, cc;
  T cm;                     // reverse: Lambda_m = cm * lambda_vhat (cc exact, -1 plain delivery)
  T inv_tau_m, inv_tau_s;   // (T)(1/tau) for the per-event exponents (device-mode contract)
  T scale, inv_scale;       // 2^F, 2^-F (exact powers of two)
  FastDiv divN;             // idx -> trial
};

// calendar bucket entry: fp32 {target, packed pair} = one 16-byte access;
// fp64 {target, qs, qm, pad} = two
template <typename T>
__host__ __device__ constexpr int bk_words() { return Prec<T>::kSlotWords == 1 ? 2 : 4; }

template <typename T>
struct NetView {
  const int64_t* rowptr;
  const int32_t* col;
  const T* w;
  const T* d;
  const unsigned short* dcode;  // [E] delivery_code(d, dt)
  const EdgeRec<T>* er;         // [E] packed {col, w, d, code}
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
  long long* log_r0;     // CSR row start of each logged spike's source (written by its owner)
  int* log_len;          // its row length
  long long log_cap;
  unsigned long long* log_count;
  long long* chunk_off;  // [m][G]
  int* chunk_cnt;        // [m][G]
  long long* step_start; // [m] first log record of step m (published at each barrier)
  long long* counters;   // [B][3]
  T* v_trace;            // [m1-m0][B][N] or null
  unsigned long long* tl;  // debug timeline [m][G][4] (globaltimer ns) or null
  int* err;
  unsigned* bar;
  // calendar (ring kind): events due at step s wait in bucket s % NB until phase
  // s-1 delivers them into the L2-resident accumulator acc[s & 1]
  long long* acc;        // [2][total] x words
  long long* bk;         // [G][NB][cap_b] entries {target, payload} (bk_words<T>() int64 each; per-CTA private)
  int* bk_cnt;           // [G][NB] fill (kept in smem inside a launch)
  long long cap_b;
  int NB;
  int* ring_dirty;       // [R] a bucket overflowed into ring row r
  // partitioned network (eq_set_partition): owned neuron j is CSR row
  // src_off + j; spikes imported from other partitions (emitted in the
  // previous exchange window) are fanned out in the launch's first phase
  int src_off;
  int smem_state;            // I, V of the owned range kept in shared memory for the launch
  const SpikeRec<T>* imp;    // idx = trial*N (flat base of the trial), a = (T)emit step
  const long long* imp_r0;
  const int* imp_len;
  long long imp_n;
  const long long* imp_dev;  // peer exchange: {first, count} of the import block on the device (overrides imp_n)
  int no_pause;              // asynchronous windows: a full spike log is an error, not a pause
  int cal;                   // the calendar path runs (ring kind, or a bounded kind by admission)
  // bounded kinds by admission (binaryheap / sortedarray, eq_adm.cuh): the
  // calendar carries the accepted events; a per-target record counts them
  int adm_cap;               // accept while the queue holds fewer events
  int* aw;                   // [2][totp] E | pc << 16 by phase parity
  unsigned short* ac;        // [2][totp] events accepted for the step with that parity (popped at it)
  unsigned short* aa;        // [3][totp] arrivals of the phase (step % 3)
  long long totp;            // total rounded up to a multiple of 8
  int* fl;                   // [2][G][per] targets whose step needs the reference order
  int* fl_cnt;               // [2][G]
  int* lpos;                 // [3][total] log position of the spike of step s (s % 3)
  const int2* csc;           // [E] in-edges {x, source} by target, ascending x
  const long long* csc_off;  // [N+1]
  unsigned* drop_bits;       // event id = log position * maxdeg + row offset
  long long drop_cap;
  int maxdeg;
  FastDiv divPer;            // flat target -> owner CTA
  int* cring;                // [B][R][N] event counts of the DRAM ring rows (bucket overflow)
  int2* slots;               // [2][total][kAdmSlots] {x, log position} of a phase's first arrivals
  int adm_slots;             // keys recorded while free < adm_slots (<= kAdmSlots; 0: every fix-up walks the CSC)
};

// Arrivals whose key is recorded per target and phase (when 0 < free < kAdmSlots):
// a fix-up with at most this many arrivals ranks them without the CSC walk.
constexpr int kAdmSlots = 8;

template <int NT, typename T = float>
struct FwdShared {
  static constexpr int kCap = sizeof(T) == 4 ? 1024 : 512;   // spikes staged in smem per batch
  static constexpr int kTrials = 8;   // per-CTA trial counters kept in smem
  static constexpr int kBins = 512;   // calendar buckets (horizon + 1 <= kBins)
};

__device__ __forceinline__ void tl_mark(unsigned long long* tl, int m, int G, int cta, int k) {
  if (tl && threadIdx.x == 0) tl[((size_t)m * G + cta) * 8 + k] = globaltimer();
}
// same, from whichever thread calls it (warp-group leaders)
__device__ __forceinline__ void tl_mark_any(unsigned long long* tl, int m, int G, int cta, int k) {
  if (tl) tl[((size_t)m * G + cta) * 8 + k] = globaltimer();
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

// Row of flat event f at or after row k0 (pre[k0] <= f): exponential search
// from k0, then bisection.  A thread's events come in increasing f a few rows
// apart, so this takes ~4 shared loads where find_row takes log2(n) (find_row
// was 12% of the forward's executed instructions, profiles/r2af_fwd_lines.txt).
__device__ __forceinline__ int find_row_from(const int* pre, int n, int f, int k0) {
  int lo = k0, hi = k0 + 1, step = 1;
  while (hi < n && pre[hi] <= f) {
    lo = hi;
    step <<= 1;
    hi = lo + step;
  }
  if (hi > n) hi = n;
  while (hi - lo > 1) {
    const int mid = (lo + hi) >> 1;
    if (pre[mid] <= f) lo = mid;
    else hi = mid;
  }
  return lo;
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

// Named barrier for a warp group (ids 1..15; 0 is __syncthreads).
__device__ __forceinline__ void group_sync(int id, int nthreads) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}

// Exclusive prefix over a staged batch's row lengths by the group's first warp.
// On entry pre[k+1] = len[k] (k < n); on exit pre[0..n] is the exclusive scan.
__device__ __forceinline__ void group_scan(int* pre, int n, int gtid) {
  if (gtid < 32) {
    const int lane = gtid;
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

// Stage log records [k0, k0+nb) in smem with their CSR row starts and the
// exclusive prefix of their row lengths (s_pre[nb] = events in the batch).
// Executed by one warp group (gtid in [0, gsize), named barrier bar_id).
template <typename T>
__device__ __forceinline__ void stage_spikes(const SpikeRec<T>* log, const long long* log_r0, const int* log_len,
                                             long long k0, int nb, SpikeRec<T>* s_rec, long long* s_r0, int* s_pre,
                                             int gtid, int gsize, int bar_id) {
  group_sync(bar_id, gsize);
  for (int k = gtid; k < nb; k += gsize) {
    s_rec[k] = log[k0 + k];
    s_r0[k] = log_r0[k0 + k];        // row start/length stored by the owner: no dependent rowptr load
    s_pre[k + 1] = log_len[k0 + k];
  }
  group_sync(bar_id, gsize);
  group_scan(s_pre, nb, gtid);
  group_sync(bar_id, gsize);
}

// Warp specialisation of the persistent kernels: in every phase the first NF
// threads run the event side (delivery + fan-out of step m-1, or R-fanout of
// step m-1), the other NT-NF threads the neuron side (update / R-neuron of
// step m).  The two sides touch disjoint data within a phase, so they overlap
// their memory latencies instead of running back to back.
template <int NT, int NF_ = NT / 2>
struct Roles {
  static constexpr int NF = NF_;
  static constexpr int NN = NT - NF_;
  static constexpr int kBarF = 1, kBarN = 2;
};

// ------------------------------------------------------------------ admission
//
// Bounded kinds by admission (BinaryHeapQueue queues.py:481-571, SortedArrayQueue
// :308-403).  Both drop the INCOMING event when the queue holds `capacity`
// events and pop every event due now, so a queue's effect on
// the network is fixed by two numbers per step: how many events it holds and,
// among a step's arrivals, which come first in the reference order (emit step,
// then ascending CSR edge index x).  The events themselves ride the ring kind's
// calendar (buckets + L2 accumulator, fixed point); the structure is replaced by
// admission counters per queue, each in its own array so the owner's per-step
// pass over them is coalesced (16 bytes per queue and step):
//
//   aw[2]  E | pc << 16 of the phase with that parity: E = events held before
//          the phase's admissions, pc = events popped at its step
//   ac[2]  signed 16-bit: events accepted for the step with that parity (counted
//          where the payload is delivered into the accumulator; read and zeroed
//          at pop; decoded pairwise with the borrow, like the payload pairs)
//   aa[3]  16-bit: arrivals of the phase (step % 3)
//
// (16-bit counters are updated with 32-bit atomics on the word holding two
// queues' counters: arrivals stay in [0, 65535]; pop counts in [-cap, cap]
// are decoded with the borrow.)
//
// Phase m admits the arrivals of step m-1's spikes: an event takes a ticket t
// (atomic on its target's arrival word); with occ = min(E + n, cap) - pc of phase
// m-1, the first free = cap - occ tickets are accepted.  Tickets come in
// arbitrary order, so when 0 < free < n the target goes on its owner's fix-up
// list: at the start of phase m+1 the owner ranks the arrivals by x — from the
// keys {x, log position} they recorded by ticket while free < kAdmSlots, or by
// walking the target's in-edges in ascending x (CSC, one warp) when there were
// more arrivals than slots — and swaps any ticket winner that is not among the
// first `free` in the reference order for the one that is (payload and count
// moved with the exact fixed-point negation, drop bits flipped).  The accepted
// SET then equals the reference's; accepted COUNTS never change.  Queue
// contents, pops and the reverse pass's drop bits are therefore the reference's;
// a queue full before the phase drops every arrival whatever the ticket order.

constexpr long long kNegEntry = 1LL << 62;   // bucket entry flag: a withdrawn event (count -1)

__device__ __forceinline__ void red_i32(int* p, int v) {
  asm volatile("red.relaxed.gpu.global.add.s32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

// count word of target tgt in DRAM ring row `row` (the ring's [B][R][N] layout)
template <typename T>
__device__ __forceinline__ int* cring_at(const FwdArgs<T>& A, int row, long long tgt) {
  const int b = A.c.divN.div((int)tgt);
  return A.cring + ((size_t)b * A.R + row) * A.N + (tgt - (long long)b * A.N);
}

// Occupancy before the admissions of phase m (from phase m-1's counters).
template <typename T>
__device__ __forceinline__ int adm_occ(const FwdArgs<T>& A, int m, long long tgt) {
  const int ep = A.aw[(size_t)((m - 1) & 1) * A.totp + tgt];
  const int n = A.aa[(size_t)((m + 2) % 3) * A.totp + tgt];
  const int e = (ep & 0xffff) + n;
  return (e < A.adm_cap ? e : A.adm_cap) - (ep >> 16);
}
// Ticket of an arrival in phase m (its rank among the target's arrivals so far).
template <typename T>
__device__ __forceinline__ int adm_ticket(const FwdArgs<T>& A, int m, long long tgt) {
  unsigned* w = reinterpret_cast<unsigned*>(A.aa + (size_t)(m % 3) * A.totp) + (tgt >> 1);
  const int sh = (int)(tgt & 1) * 16;
  return (int)((atomicAdd(w, 1u << sh) >> sh) & 0xffffu);
}
// +-1 accepted event for the step with parity par.
template <typename T>
__device__ __forceinline__ void adm_count(const FwdArgs<T>& A, int par, long long tgt, int sign) {
  red_i32(reinterpret_cast<int*>(A.ac + (size_t)par * A.totp) + (tgt >> 1), sign * (1 << ((int)(tgt & 1) * 16)));
}

// Add (sign +1) or withdraw (-1) one event's payload and count at due step ds
// during phase p (in_kernel) or after the launch that ended with phase p-1.
template <typename T>
__device__ __forceinline__ void adm_apply(const FwdArgs<T>& A, int p, bool in_kernel, int ds, int tgt, long long q1,
                                          long long q2, int sign, int* bins, int cta) {
  typedef Prec<T> P;
  if (ds == p || (in_kernel && ds == p + 1)) {
    long long* a = A.acc + (size_t)(ds & 1) * A.total * P::kSlotWords;
    if (P::kSlotWords == 1) {
      red_add(a + tgt, pack2(q1, q2));
    } else {
      red_add(a + 2 * (size_t)tgt, q1);
      red_add(a + 2 * (size_t)tgt + 1, q2);
    }
    adm_count(A, ds & 1, tgt, sign);
    return;
  }
  const int bn = ds % A.NB;
  const int pos = atomicAdd(bins + bn, 1);
  if (pos < A.cap_b) {
    long long* bk = A.bk + (((size_t)cta * A.NB + bn) * A.cap_b + pos) * bk_words<T>();
    const long long tg = sign < 0 ? (tgt | kNegEntry) : tgt;
    longlong2* o = reinterpret_cast<longlong2*>(bk);
    if (P::kSlotWords == 1) {
      *o = make_longlong2(tg, pack2(q1, q2));
    } else {
      o[0] = make_longlong2(tg, q1);
      o[1] = make_longlong2(q2, 0);
    }
  } else {
    const int b = A.c.divN.div(tgt);
    const size_t so = ((size_t)b * A.R + (size_t)(ds % A.R)) * A.N + (tgt - b * A.N);
    if (P::kSlotWords == 1) {
      red_add(A.ring + so, pack2(q1, q2));
    } else {
      red_add(A.ring + 2 * so, q1);
      red_add(A.ring + 2 * so + 1, q2);
    }
    red_i32(cring_at(A, ds % A.R, tgt), sign);
    if (A.ring_dirty[ds % A.R] == 0) atomicExch(A.ring_dirty + ds % A.R, 1);
  }
}

// One arrival of a fix-up target: swap it in (canon) or out of the accepted
// set if its ticket decided otherwise (drop bit = the ticket's decision).
template <typename T>
__device__ __forceinline__ void adm_settle(const FwdArgs<T>& A, const int p, const bool in_kernel, const int tgt,
                                           const int x, const int pos, const bool canon, int* bins, const int cta) {
  typedef Prec<T> P;
  const StepConsts<T>& c = A.c;
  const long long id = (long long)pos * A.maxdeg + (x - A.log_r0[pos]);
  const unsigned bit = 1u << (id & 31);
  const bool tent = !(A.drop_bits[id >> 5] & bit);
  if (canon == tent) return;
  const int me = p - 2;
  const SpikeRec<T> rec = A.log[pos];
  const EdgeRec<T> ed = ld_edge(A.net.er + x);
  const T t_post = rec.t + ed.d;
  const int ds = delivery_step_coded(t_post, (unsigned short)ed.code, c.dt, me);
  T ws, wm;
  if (A.exact) {
    const T phi = (T)ds * c.dt - t_post;
    ws = ed.w * eq_exp_t(-phi * c.inv_tau_s);
    wm = ed.w * eq_exp_t(-phi * c.inv_tau_m);
  } else {
    ws = ed.w;
    wm = (T)0;
  }
  long long q1 = P::q(ws, c.scale), q2 = A.exact ? P::q(wm, c.scale) : 0;
  if (canon) {
    atomicAnd(A.drop_bits + (id >> 5), ~bit);
  } else {
    atomicOr(A.drop_bits + (id >> 5), bit);
    q1 = -q1;
    q2 = -q2;
  }
  adm_apply<T>(A, p, in_kernel, ds, tgt, q1, q2, canon ? 1 : -1, bins, cta);
}

// Free room and arrival count of a fix-up target's admissions of phase p-1.
template <typename T>
__device__ __forceinline__ int2 adm_room(const FwdArgs<T>& A, int p, int tgt) {
  const int q = p - 1;
  return make_int2(A.adm_cap - adm_occ(A, q, tgt), A.aa[(size_t)(q % 3) * A.totp + tgt]);
}

// Fix-up from the recorded keys (n <= kAdmSlots arrivals), by one thread:
// rank = number of arrivals with a smaller x.
template <typename T>
__device__ __forceinline__ void adm_fixup_slots(const FwdArgs<T>& A, const int p, const bool in_kernel, const int tgt,
                                                const int fr, const int n, int* bins, const int cta) {
  const int2* sl = A.slots + ((size_t)((p - 1) & 1) * A.total + tgt) * kAdmSlots;
  int2 k[kAdmSlots];
#pragma unroll
  for (int e = 0; e < kAdmSlots; ++e)
    if (e < n) k[e] = sl[e];
#pragma unroll
  for (int e = 0; e < kAdmSlots; ++e) {
    if (e >= n) continue;
    int rank = 0;
#pragma unroll
    for (int g = 0; g < kAdmSlots; ++g) rank += (g < n && k[g].x < k[e].x) ? 1 : 0;
    adm_settle<T>(A, p, in_kernel, tgt, k[e].x, k[e].y, rank < fr, bins, cta);
  }
}

// Reference-order fix-up of one target's admissions of phase p-1 (arrivals from
// the spikes of step p-2) with more arrivals than recorded keys, by one warp:
// in-edges in ascending x, 32 per round, arrival = the source's spike of that
// step is in the log (lpos).
template <typename T>
__device__ __forceinline__ void adm_fixup(const FwdArgs<T>& A, const int p, const bool in_kernel, const int tgt,
                                          const int lane, int* bins, const int cta) {
  const StepConsts<T>& c = A.c;
  const int me = p - 2;
  const int b = c.divN.div(tgt), j = tgt - b * A.N;
  const int2 rn = adm_room(A, p, tgt);
  const int fr = rn.x, n = rn.y;
  const long long L0 = A.step_start[me], L1 = A.step_start[me + 1];
  const int* lp = A.lpos + (size_t)(me % 3) * A.total + (size_t)b * A.N;
  const long long cs = A.csc_off[j], ce = A.csc_off[j + 1];
  int rank = 0;
  for (long long k0 = cs; k0 < ce && rank < n; k0 += 32) {
    const long long k = k0 + lane;
    bool arr = false;
    int2 xi = make_int2(0, 0);
    int pos = 0;
    if (k < ce) {
      xi = A.csc[k];
      pos = lp[xi.y];
      arr = pos >= L0 && pos < L1;
    }
    const unsigned bal = __ballot_sync(0xffffffffu, arr);
    if (arr) adm_settle<T>(A, p, in_kernel, tgt, xi.x, pos, rank + __popc(bal & ((1u << lane) - 1u)) < fr, bins, cta);
    rank += __popc(bal);
  }
}

// The fix-ups listed for this CTA by the admissions of phase p-1, one warp per
// target; the list is emptied for its next use (phase p+1).
// Targets with recorded keys: one thread each; the rest (more arrivals than
// slots, or room beyond the slots) then one warp each over the CSC.
template <typename T>
__device__ __noinline__ void adm_fixups(const FwdArgs<T>& A, const int p, const bool in_kernel, const int cta,
                                        const int gtid, const int nthreads, int* bins) {   // out of line: rare path
  const int par = (p - 1) & 1;
  const int n = A.fl_cnt[par * A.G + cta];
  const int* lst = A.fl + ((size_t)par * A.G + cta) * A.per;
  bool walk = false;
  for (int k = gtid; k < n; k += nthreads) {
    const int tgt = lst[k];
    const int2 rn = adm_room(A, p, tgt);
    if (rn.x < A.adm_slots && rn.y <= A.adm_slots) adm_fixup_slots<T>(A, p, in_kernel, tgt, rn.x, rn.y, bins, cta);
    else walk = true;
  }
  if (!__any_sync(0xffffffffu, walk)) return;     // warp-uniform: each warp walks the targets of its own lanes
  const int lane = gtid & 31;
  for (int k0 = gtid - lane; k0 < n; k0 += nthreads) {
    const int k = k0 + lane;
    bool w = false;
    int tgt = 0;
    if (k < n) {
      tgt = lst[k];
      const int2 rn = adm_room(A, p, tgt);
      w = !(rn.x < A.adm_slots && rn.y <= A.adm_slots);
    }
    unsigned bal = __ballot_sync(0xffffffffu, w);
    while (bal) {
      const int src = __ffs(bal) - 1;
      bal &= bal - 1;
      adm_fixup<T>(A, p, in_kernel, __shfl_sync(0xffffffffu, tgt, src), lane, bins, cta);
    }
  }
}

// After a forward launch: the fix-ups of its last admissions (phase err[4],
// the step it reached), so the next launch and the queue contents read now see
// them applied.
template <typename T, int NT>
__global__ void __launch_bounds__(NT) k_adm_fixup(FwdArgs<T> A) {
  if (ld_volatile(A.err) != 0) return;
  const int p = ld_volatile(A.err + 4) + 1;
  const int cta = blockIdx.x;
  adm_fixups<T>(A, p, false, cta, threadIdx.x, NT, A.bk_cnt + (size_t)cta * A.NB);
  __syncthreads();
  if (threadIdx.x == 0) A.fl_cnt[((p - 1) & 1) * A.G + cta] = 0;
}

// Fan-out (network.py:583-611) of log records [s0, s1): the CTA's share of
// step m-1's own spikes (kImp = false) or, in a launch's first phase, of the
// spikes imported from other partitions (kImp = true: per-spike emit steps in
// rec.a, flat trial base in rec.idx).  An event due at m+1 goes straight into
// acc[(m+1)&1]; a later one is appended to this CTA's bucket of its delivery
// step (rank from a shared-memory counter).  No read-modify-write touches
// DRAM; a full bucket spills into the DRAM ring row (flagged), never losing
// events.  Executed by the event-side warp group.
constexpr int kDropTr = 64;   // per-trial drop counts of a phase's admissions kept in smem

template <typename T, int NT, int NF, bool kImp, bool kAdm = false, int kAdmEv = 2>
__device__ __forceinline__ void fwd_fanout(const FwdArgs<T>& A, const int m, const int cta, const int gtid,
                                           const long long s0, const long long s1, SpikeRec<T>* s_spk,
                                           long long* s_r0, int* s_pre, int* s_bin, unsigned* s_drop = nullptr) {
  typedef Prec<T> P;
  typedef Roles<NT, NF> Ro;
  constexpr int kCap = FwdShared<NT, T>::kCap;
  const StepConsts<T>& c = A.c;
  const SpikeRec<T>* lg = kImp ? A.imp : A.log;
  const long long* lr0 = kImp ? A.imp_r0 : A.log_r0;
  const int* llen = kImp ? A.imp_len : A.log_len;
  const int me_fixed = m - 1;
  long long* accn = A.acc + (size_t)((m + 1) & 1) * A.total * P::kSlotWords;
  long long* bk_cta = A.bk + (size_t)cta * A.NB * A.cap_b * bk_words<T>();
  const int me_bin = kImp ? 0 : me_fixed % A.NB;
  for (long long k0 = s0; k0 < s1; k0 += kCap) {
    const int nb = (int)(s1 - k0 < kCap ? s1 - k0 : kCap);
    stage_spikes<T>(lg, lr0, llen, k0, nb, s_spk, s_r0, s_pre, gtid, Ro::NF, Ro::kBarF);
    const int total = s_pre[nb];
    if (kImp) {                                           // imported: count their events here
      for (int k = gtid; k < nb; k += Ro::NF) {
        const int b = c.divN.div(s_spk[k].idx);
        atomicAdd(reinterpret_cast<unsigned long long*>(A.counters + 3 * b + 1),
                  (unsigned long long)(s_pre[k + 1] - s_pre[k]));
      }
    }
#ifndef EQ_FWD_EV
#define EQ_FWD_EV 3
#endif
    constexpr int EV = kAdm ? kAdmEv : EQ_FWD_EV;
    int krow = 0;                                          // row of this thread's last event
    for (int f0 = gtid; f0 < total; f0 += EV * Ro::NF) {
      int jj[EV], kk[EV];
      T ww[EV], dd[EV];
      unsigned short cc[EV];
      int xs[kAdm ? EV : 1];
#pragma unroll
      for (int e = 0; e < EV; ++e) {
        const int f = f0 + e * Ro::NF;
        kk[e] = -1;
        if (f < total) {
          const int k = find_row_from(s_pre, nb, f, krow);
          krow = k;
          const long long x = s_r0[k] + (f - s_pre[k]);
          kk[e] = k;
          if constexpr (kAdm) xs[e] = (int)x;
          const EdgeRec<T> ed = ld_edge(A.net.er + x);   // one 16-byte streamed load per event
          jj[e] = ed.col;
          ww[e] = ed.w;
          dd[e] = ed.d;
          cc[e] = (unsigned short)ed.code;
        }
      }
      // admission: every event's ticket and its target's occupancy, issued
      // back to back before any is consumed
      int tk[kAdm ? EV : 1], fr[kAdm ? EV : 1];
      if constexpr (kAdm) {
#pragma unroll
        for (int e = 0; e < EV; ++e) {
          if (kk[e] < 0) continue;
          const int tgt = c.divN.div(s_spk[kk[e]].idx) * A.N + jj[e];
          tk[e] = adm_ticket(A, m, tgt);
          fr[e] = A.adm_cap - adm_occ(A, m, tgt);
        }
#pragma unroll
        for (int e = 0; e < EV; ++e) {                      // keys for a possible fix-up
          if (kk[e] < 0 || fr[e] <= 0 || fr[e] >= A.adm_slots || tk[e] >= A.adm_slots) continue;
          const int tgt = c.divN.div(s_spk[kk[e]].idx) * A.N + jj[e];
          A.slots[((size_t)(m & 1) * A.total + tgt) * kAdmSlots + tk[e]] = make_int2(xs[e], (int)(k0 + kk[e]));
        }
      }
#pragma unroll
      for (int e = 0; e < EV; ++e) {
        if (kk[e] < 0) continue;
        const SpikeRec<T> rec = s_spk[kk[e]];
        const int b = c.divN.div(rec.idx);
        const int tgt = b * A.N + jj[e];                    // flat target
        if constexpr (kAdm) {
          if (tk[e] >= fr[e]) {                             // queue full at this ticket: dropped (no payload)
            const int f = f0 + e * Ro::NF;
            const long long id = (k0 + kk[e]) * (long long)A.maxdeg + (f - s_pre[kk[e]]);
            atomicOr(A.drop_bits + (id >> 5), 1u << (id & 31));
            if (b < kDropTr) atomicAdd(s_drop + b, 1u);
            else atomicAdd(reinterpret_cast<unsigned long long*>(A.counters + 3 * b + 2), 1ULL);
            if (tk[e] == fr[e] && fr[e] > 0) {              // more arrivals than room: reference order needed
              const int owner = A.divPer.div(tgt);
              const int slot = atomicAdd(A.fl_cnt + (m & 1) * A.G + owner, 1);
              A.fl[((size_t)(m & 1) * A.G + owner) * A.per + slot] = tgt;
            }
            continue;
          }
        }
        const int me = kImp ? (int)rec.a : me_fixed;
        const T w = ww[e], d = dd[e];
        const T t_post = rec.t + d;                              // :588
        const int ds = delivery_step_coded(t_post, cc[e], c.dt, me);  // jumps.py:96
        T ws, wm;
        if (A.exact) {
          const T phi = (T)ds * c.dt - t_post;              // :599
          ws = w * eq_exp_t(-phi * c.inv_tau_s);            // :601 (x 1/tau)
          wm = w * eq_exp_t(-phi * c.inv_tau_m);            // :606
        } else {
          ws = w;
          wm = (T)0;
        }
        const long long q1 = P::q(ws, c.scale);
        const long long q2 = A.exact ? P::q(wm, c.scale) : 0;
        if (ds == m + 1) {
          if (P::kSlotWords == 1) {
            red_add(accn + tgt, pack2(q1, q2));
          } else {
            red_add(accn + 2 * (size_t)tgt, q1);
            red_add(accn + 2 * (size_t)tgt + 1, q2);
          }
          if constexpr (kAdm) adm_count(A, (m + 1) & 1, tgt, 1);
          continue;
        }
        int bn;
        if (!kImp) {
          bn = me_bin + (ds - me);                          // ds % NB, ds - me in [2, H]
          if (bn >= A.NB) bn -= A.NB;
        } else {
          if (ds <= m) {                                    // exchange window longer than D_min
            raise_error(A.err, EQ_ERR_CAUSALITY, m, b, jj[e]);
            continue;
          }
          bn = ds % A.NB;
        }
        // one shared atomic per event (a warp-aggregated variant with
        // __match_any_sync measured slower: fwd 32.2 -> 37.7 ms, profiles/r1h_ab_bin_agg.txt)
        const int pos = atomicAdd(&s_bin[bn], 1);
        if (pos < A.cap_b) {
          longlong2* o = reinterpret_cast<longlong2*>(bk_cta + ((size_t)bn * A.cap_b + pos) * bk_words<T>());
          if (P::kSlotWords == 1) {                         // read once, ~H/2 steps later: streaming
            __stcs(o, make_longlong2(tgt, pack2(q1, q2)));
          } else {
            __stcs(o, make_longlong2(tgt, q1));
            __stcs(o + 1, make_longlong2(q2, 0));
          }
        } else {                                            // bucket full: DRAM ring row
          const size_t so = ((size_t)b * A.R + (size_t)(ds % A.R)) * A.N + jj[e];
          if (P::kSlotWords == 1) {
            red_add(A.ring + so, pack2(q1, q2));
          } else {
            red_add(A.ring + 2 * so, q1);
            red_add(A.ring + 2 * so + 1, q2);
          }
          if constexpr (kAdm) red_i32(cring_at(A, ds % A.R, tgt), 1);
          if (A.ring_dirty[ds % A.R] == 0) atomicExch(A.ring_dirty + ds % A.R, 1);
        }
      }
    }
  }
}

// Spikes imported from other partitions, fanned out by a plain launch just
// before the persistent kernel's first phase m0 (stream-ordered): the same
// per-CTA buckets (fill levels round-trip through bk_cnt) and acc[(m0+1)&1]
// for events due at m0+1.  Kept out of the persistent kernel so its register
// allocation is that of the own-spike path alone.
template <typename T, int NT>
__global__ void __launch_bounds__(NT) k_import_fanout(FwdArgs<T> A) {
  constexpr int kCap = FwdShared<NT, T>::kCap;
  __shared__ SpikeRec<T> s_spk[kCap];
  __shared__ long long s_r0[kCap];
  __shared__ int s_pre[kCap + 1];
  __shared__ int s_bin[FwdShared<NT>::kBins];
  const int cta = blockIdx.x;
  for (int k = threadIdx.x; k < A.NB; k += NT) s_bin[k] = A.bk_cnt[(size_t)cta * A.NB + k];
  __syncthreads();
  long long first = 0, n = A.imp_n;
  if (A.imp_dev) {
    first = A.imp_dev[0];
    n = A.imp_dev[1];
  }
  fwd_fanout<T, NT, NT, true>(A, A.m0, cta, threadIdx.x, first + n * cta / A.G, first + n * (cta + 1) / A.G, s_spk,
                              s_r0, s_pre, s_bin);
  __syncthreads();
  for (int k = threadIdx.x; k < A.NB; k += NT) A.bk_cnt[(size_t)cta * A.NB + k] = s_bin[k];
}

// Per-trial counters of this CTA (spikes, events, drops) are counted per phase
// in 32-bit shared memory (64-bit shared atomics are compare-and-swap loops on
// sm_100a) and flushed into the 64-bit device counters once per phase.
template <int kTr>
__device__ __forceinline__ void flush_counters(unsigned (*s_ctr)[3], long long* counters, int b_first, int B,
                                               long long end, int N) {
  const int t = threadIdx.x;
  if (t < kTr * 3) {
    const int tb = t / 3, q = t % 3;
    const unsigned v = s_ctr[tb][q];
    const int b = b_first + tb;
    if (v && b < B && (long long)b * N < end)
      atomicAdd(reinterpret_cast<unsigned long long*>(counters + 3 * b + q), (unsigned long long)v);
    s_ctr[tb][q] = 0u;
  }
}

// Neuron side of one forward phase m (network.py:547-580): pop (the slot sums
// waiting in acc[m&1] when acc_pop — ring, and bounded kinds whose queue stage
// wrote them), synapse + LIF + exact crossing for the CTA's neuron-trials, clear
// the popped slots, then the spike log (one chunk per (step, CTA)) and the
// per-trial counters.  Executed by the neuron-side warp group (gtid < NN).
template <typename T, int NT, int U, int NF, bool kAdm = false>
__device__ __forceinline__ void neuron_side(const FwdArgs<T>& A, const int m, const int cta, const int gtid,
                                            const long long begin, const long long end, const int b_first,
                                            const bool acc_pop, SpikeRec<T>* s_own, int& s_n, long long& s_off,
                                            unsigned (*s_ctr)[3], SpikeRec<T>* spill, T* s_st = nullptr,
                                            int* s_bin = nullptr) {
  // s_st: the CTA's I and V kept in shared memory across the launch ([per] I,
  // then [per] V, indexed by idx - begin), or null (state in HBM)
  T* const gI = s_st ? s_st - begin : A.I;
  T* const gV = s_st ? s_st + A.per - begin : A.V;
  typedef Prec<T> P;
  typedef Roles<NT, NF> Ro;
  constexpr int kCapN = FwdShared<NT, T>::kCap / 2;
  constexpr int kTr = FwdShared<NT>::kTrials;
  const StepConsts<T>& c = A.c;
  const bool dirty = A.cal && ld_volatile(A.ring_dirty + m % A.R) != 0;
  if constexpr (kAdm) {
    // (a) reference-order fix-ups of the last phase's admissions (they may
    // move events due now, so before the pop), then this phase's record words
    adm_fixups<T>(A, m, true, cta, gtid, Ro::NN, s_bin);
    __threadfence();   // their reds into acc / counts, before this group's plain loads of them
    group_sync(Ro::kBarN, Ro::NN);
    if (gtid == 0) A.fl_cnt[((m - 1) & 1) * A.G + cta] = 0;
    // E|pc of this phase from the last one's counters, pops of step m read and
    // zeroed, next phase's arrival counters zeroed: four queues per thread with
    // 16- / 8-byte accesses (begin and per are multiples of 32)
    const int* wp = A.aw + (size_t)((m - 1) & 1) * A.totp;
    int* wc = A.aw + (size_t)(m & 1) * A.totp;
    const unsigned short* np = A.aa + (size_t)((m + 2) % 3) * A.totp;
    unsigned short* nz = A.aa + (size_t)((m + 1) % 3) * A.totp;
    unsigned short* cp = A.ac + (size_t)(m & 1) * A.totp;
    for (long long i0 = begin + 4 * gtid; i0 < end; i0 += 4 * Ro::NN) {
      const int4 w4 = *reinterpret_cast<const int4*>(wp + i0);
      const ushort4 n4 = *reinterpret_cast<const ushort4*>(np + i0);
      // pop counts: signed 16-bit pairs (a withdrawal may sit here while its
      // event went to a DRAM ring row: -1 borrows from the pair's other half)
      const uint2 c2 = *reinterpret_cast<const uint2*>(cp + i0);
      const int wv[4] = {w4.x, w4.y, w4.z, w4.w};
      const int nv[4] = {n4.x, n4.y, n4.z, n4.w};
      int cv[4];
      cv[0] = (short)(c2.x & 0xffffu);
      cv[1] = (int)(c2.x - (unsigned)cv[0]) >> 16;
      cv[2] = (short)(c2.y & 0xffffu);
      cv[3] = (int)(c2.y - (unsigned)cv[2]) >> 16;
      int out[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        if (dirty && i0 + u < end) {                   // events that overflowed a bucket into ring row m
          int* cr = cring_at(A, m % A.R, i0 + u);
          cv[u] += *cr;
          *cr = 0;
        }
        const int e = (wv[u] & 0xffff) + nv[u];
        out[u] = ((e < A.adm_cap ? e : A.adm_cap) - (wv[u] >> 16)) | (cv[u] << 16);
      }
      *reinterpret_cast<int4*>(wc + i0) = make_int4(out[0], out[1], out[2], out[3]);   // (tail lanes past
      *reinterpret_cast<ushort4*>(cp + i0) = make_ushort4(0, 0, 0, 0);                // `end` are padding)
      *reinterpret_cast<ushort4*>(nz + i0) = make_ushort4(0, 0, 0, 0);
    }
    if (gtid == 0) tl_mark_any(A.tl, m, A.G, cta, 7);
  }
  // ---------------- (b) neuron update: pop, synapse, membrane, crossing.
  // Walked per trial segment of the owned range so the row pointers are
  // computed once per segment, not per neuron.
  const int mm = m < A.net.t_mask ? m : A.net.t_mask - 1;   // network.py:155 rows[-1]
  const long long* accm = A.acc + (size_t)(m & 1) * A.total * P::kSlotWords;
  const int b_last = (int)((end - 1) / A.N);
  for (int b = b_first; b <= b_last; ++b) {
    const int tb0 = b * A.N;
    const int j0 = (int)(begin > tb0 ? begin - tb0 : 0);
    const int j1 = (int)(end < (long long)tb0 + A.N ? end - tb0 : A.N);
    const uint32_t* mrow = A.net.mask + ((size_t)b * A.net.t_mask + mm) * A.net.words;
    if (P::kSlotWords == 1 && acc_pop && (A.N & 3) == 0 && !dirty) {
      // fp32 fast path: four neurons per thread with 16-byte accesses
      // (segment bounds are multiples of 4 when N % 4 == 0: ranges are
      // warp-aligned).  Same per-neuron arithmetic as the scalar path.
      for (int jq = j0 + 4 * gtid; jq < j1; jq += 4 * Ro::NN) {
        const int idx = tb0 + jq;
        const longlong2 a01 = *reinterpret_cast<const longlong2*>(accm + idx);
        const longlong2 a23 = *reinterpret_cast<const longlong2*>(accm + idx + 2);
        const float4 I4 = *reinterpret_cast<const float4*>(gI + idx);
        const float4 V4 = *reinterpret_cast<const float4*>(gV + idx);
        const float4 M4 = __ldg(reinterpret_cast<const float4*>(A.net.amp + jq));
        const unsigned mw = __ldg(mrow + (jq >> 5)) >> (jq & 31);
        int4 R4 = make_int4(0, 0, 0, 0);
        if (A.refractory) R4 = *reinterpret_cast<const int4*>(A.refr + idx);
        const long long av[4] = {a01.x, a01.y, a23.x, a23.y};
        const float Iv4[4] = {I4.x, I4.y, I4.z, I4.w};
        const float Vv4[4] = {V4.x, V4.y, V4.z, V4.w};
        const float Av4[4] = {M4.x, M4.y, M4.z, M4.w};
        int rf4[4] = {R4.x, R4.y, R4.z, R4.w};
        float In[4], Vn[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          long long qs, qm;
          unpack2(av[q], qs, qm);
          const T ps = P::deq(qs, c.inv_scale);
          const T pm = A.exact ? P::deq(qm, c.inv_scale) : (T)0;
          const T drive = ((mw >> q) & 1u) ? (T)Av4[q] : (T)0;
          T i, v_new, a, v, t_spk;
          if (lif_step(c, A.exact != 0, A.refractory, m, ps, pm, (T)Iv4[q], (T)Vv4[q], drive, rf4[q], i, v_new,
                       a, v, t_spk)) {
            if (t_spk != t_spk) {
              raise_error(A.err, EQ_ERR_GRAZING, m + 1, b, jq + q);
            } else {
              int pos = atomicAdd(&s_n, 1);
              SpikeRec<T> rec;
              rec.idx = idx + q;
              rec.t = t_spk;
              rec.a = a;
              rec.vh = v;
              if (pos < kCapN) s_own[pos] = rec;
              else spill[pos - kCapN] = rec;
            }
          }
          In[q] = (float)i;
          Vn[q] = (float)v_new;
        }
        *reinterpret_cast<float4*>(gI + idx) = make_float4(In[0], In[1], In[2], In[3]);
        *reinterpret_cast<float4*>(gV + idx) = make_float4(Vn[0], Vn[1], Vn[2], Vn[3]);
        // RingQueue._pop_raw zeroes the slot (queues.py:114-117): the load has been
        // consumed, so this store does not wait behind it
        long long* accz = const_cast<long long*>(accm) + idx;
        *reinterpret_cast<longlong2*>(accz) = make_longlong2(0, 0);
        *reinterpret_cast<longlong2*>(accz + 2) = make_longlong2(0, 0);
        if (A.refractory)
          *reinterpret_cast<int4*>(A.refr + idx) = make_int4(rf4[0], rf4[1], rf4[2], rf4[3]);
        if (A.v_trace)
          *reinterpret_cast<float4*>(A.v_trace + (size_t)(m - A.m0) * A.total + idx) =
              make_float4(Vn[0], Vn[1], Vn[2], Vn[3]);
      }
      continue;
    }
    if (P::kSlotWords == 2 && acc_pop && (A.N & 1) == 0 && !dirty) {
      // fp64 fast path: two neurons per thread with 16-byte accesses (a neuron's
      // two int64 slot words are one longlong2); same per-neuron arithmetic
      for (int jq = j0 + 2 * gtid; jq < j1; jq += 2 * Ro::NN) {
        const int idx = tb0 + jq;
        long long* accz = const_cast<long long*>(accm) + 2 * (size_t)idx;
        const longlong2 s0 = *reinterpret_cast<const longlong2*>(accz);
        const longlong2 s1 = *reinterpret_cast<const longlong2*>(accz + 2);
        const double2 I2 = *reinterpret_cast<const double2*>(A.I + idx);
        const double2 V2 = *reinterpret_cast<const double2*>(A.V + idx);
        const double2 M2 = __ldg(reinterpret_cast<const double2*>(A.net.amp + jq));
        const unsigned mw = __ldg(mrow + (jq >> 5)) >> (jq & 31);
        int2 R2 = make_int2(0, 0);
        if (A.refractory) R2 = *reinterpret_cast<const int2*>(A.refr + idx);
        const long long qs2[2] = {s0.x, s1.x}, qm2[2] = {s0.y, s1.y};
        const double Iv2[2] = {I2.x, I2.y}, Vv2[2] = {V2.x, V2.y}, Av2[2] = {M2.x, M2.y};
        int rf2[2] = {R2.x, R2.y};
        double In[2], Vn[2];
#pragma unroll
        for (int q = 0; q < 2; ++q) {
          const T ps = P::deq(qs2[q], c.inv_scale);
          const T pm = A.exact ? P::deq(qm2[q], c.inv_scale) : (T)0;
          const T drive = ((mw >> q) & 1u) ? (T)Av2[q] : (T)0;
          T i, v_new, a, v, t_spk;
          if (lif_step(c, A.exact != 0, A.refractory, m, ps, pm, (T)Iv2[q], (T)Vv2[q], drive, rf2[q], i, v_new,
                       a, v, t_spk)) {
            if (t_spk != t_spk) {
              raise_error(A.err, EQ_ERR_GRAZING, m + 1, b, jq + q);
            } else {
              int pos = atomicAdd(&s_n, 1);
              SpikeRec<T> rec;
              rec.idx = idx + q;
              rec.t = t_spk;
              rec.a = a;
              rec.vh = v;
              if (pos < kCapN) s_own[pos] = rec;
              else spill[pos - kCapN] = rec;
            }
          }
          In[q] = (double)i;
          Vn[q] = (double)v_new;
        }
        *reinterpret_cast<double2*>(A.I + idx) = make_double2(In[0], In[1]);
        *reinterpret_cast<double2*>(A.V + idx) = make_double2(Vn[0], Vn[1]);
        // RingQueue._pop_raw zeroes the slot (queues.py:114-117)
        *reinterpret_cast<longlong2*>(accz) = make_longlong2(0, 0);
        *reinterpret_cast<longlong2*>(accz + 2) = make_longlong2(0, 0);
        if (A.refractory) *reinterpret_cast<int2*>(A.refr + idx) = make_int2(rf2[0], rf2[1]);
        if (A.v_trace)
          *reinterpret_cast<double2*>(A.v_trace + (size_t)(m - A.m0) * A.total + idx) = make_double2(Vn[0], Vn[1]);
      }
      continue;
    }
    for (int jb = j0; jb < j1; jb += Ro::NN * U) {
      long long slot_v[U][2];
      T Iv[U], Vv[U], Am[U];
      int rf[U];
      unsigned mw[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int j = jb + u * Ro::NN + gtid;
        slot_v[u][0] = slot_v[u][1] = 0;
        if (j < j1) {
          const int idx = tb0 + j;
          if (acc_pop) {
            if (P::kSlotWords == 1) {
              slot_v[u][0] = ld_slot(accm + idx);
            } else {
              slot_v[u][0] = ld_slot(accm + 2 * (size_t)idx);
              slot_v[u][1] = ld_slot(accm + 2 * (size_t)idx + 1);
            }
            if (dirty) {                       // a bucket overflowed into the DRAM row
              size_t so = ((size_t)b * A.R + (size_t)(m % A.R)) * A.N + j;
              if (P::kSlotWords == 1) {
                slot_v[u][0] += ld_slot(A.ring + so);
              } else {
                slot_v[u][0] += ld_slot(A.ring + 2 * so);
                slot_v[u][1] += ld_slot(A.ring + 2 * so + 1);
              }
            }
          }
          Iv[u] = gI[idx];
          Vv[u] = gV[idx];
          rf[u] = A.refractory ? A.refr[idx] : 0;
          mw[u] = __ldg(mrow + (j >> 5));
          Am[u] = __ldg(A.net.amp + j);
        }
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int j = jb + u * Ro::NN + gtid;
        if (j >= j1) continue;
        const int idx = tb0 + j;
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
        const T drive = ((mw[u] >> (j & 31)) & 1u) ? Am[u] : (T)0;
        T i, v_new, a, v, t_spk;
        if (lif_step(c, A.exact != 0, A.refractory, m, ps, pm, Iv[u], Vv[u], drive, rf[u], i, v_new, a, v,
                     t_spk)) {
          if (t_spk != t_spk) {
            raise_error(A.err, EQ_ERR_GRAZING, m + 1, b, j);
          } else {
            int pos = atomicAdd(&s_n, 1);
            SpikeRec<T> rec;
            rec.idx = idx;
            rec.t = t_spk;
            rec.a = a;
            rec.vh = v;
            if (pos < kCapN) s_own[pos] = rec;
            else spill[pos - kCapN] = rec;
          }
        }
        gI[idx] = i;
        gV[idx] = v_new;
        if (A.refractory) A.refr[idx] = rf[u];
        if (A.v_trace) A.v_trace[(size_t)(m - A.m0) * A.total + idx] = v_new;
      }
    }
  }
  group_sync(Ro::kBarN, Ro::NN);
  if (gtid == 0) tl_mark_any(A.tl, m, A.G, cta, 4);
  // Clear the popped accumulator (RingQueue._pop_raw zeroes the slot,
  // queues.py:114-117), in a separate pass: a store next to the pending
  // load of the same line stalled the pop loop ~8x.  acc[m&1] receives no
  // red.add in this phase (the event side writes acc[(m+1)&1]).
  const bool cleared = acc_pop && !dirty && (P::kSlotWords == 1 ? (A.N & 3) == 0 : (A.N & 1) == 0);   // by the vector update
  if (acc_pop && !cleared) {
    long long* accm = A.acc + (size_t)(m & 1) * A.total * P::kSlotWords;
    if (P::kSlotWords == 1 && ((begin | end) & 1) == 0) {
      for (long long idx = begin + 2 * gtid; idx < end; idx += 2 * Ro::NN)
        *reinterpret_cast<longlong2*>(accm + idx) = make_longlong2(0, 0);
    } else {
      for (int idx = (int)begin + gtid; idx < end; idx += Ro::NN) {
        if (P::kSlotWords == 1) {
          st_slot(accm + idx, 0);
        } else {
          st_slot(accm + 2 * (size_t)idx, 0);
          st_slot(accm + 2 * (size_t)idx + 1, 0);
        }
      }
    }
    if (dirty) {
      const int row = m % A.R;
      for (int idx = (int)begin + gtid; idx < end; idx += Ro::NN) {
        const int b = c.divN.div(idx);   // rare path (bucket overflow)
        const size_t so = ((size_t)b * A.R + row) * A.N + (idx - b * A.N);
        if (P::kSlotWords == 1) {
          st_slot(A.ring + so, 0);
        } else {
          st_slot(A.ring + 2 * so, 0);
          st_slot(A.ring + 2 * so + 1, 0);
        }
      }
    }
  }
  const int nspk = s_n;
  // ---------------- spike log: one chunk per (step, CTA); the chunks of a
  // step are contiguous because every reservation of step m happens between
  // the two barriers around phase m.  Counters per trial (spikes, events;
  // donothing drops every event, queues.py:42-45).
  if (gtid == 0) {
    unsigned long long off = nspk ? atomicAdd(A.log_count, (unsigned long long)nspk) : 0ULL;
    if (nspk && (long long)(off + nspk) > A.log_cap) {
      raise_error(A.err, EQ_ERR_CAPACITY, m, -1, -1);
      off = 0;
    }
    s_off = (long long)off;
    A.chunk_off[(size_t)m * A.G + cta] = (long long)off;
    A.chunk_cnt[(size_t)m * A.G + cta] = nspk;
  }
  group_sync(Ro::kBarN, Ro::NN);
  if (!kAdm && gtid == 0) tl_mark_any(A.tl, m, A.G, cta, 7);
  const bool log_ok = s_off + nspk <= A.log_cap;
  for (int k = gtid; k < nspk; k += Ro::NN) {
    const SpikeRec<T> rec = k < kCapN ? s_own[k] : spill[k - kCapN];
    const int b = c.divN.div(rec.idx);
    const int i = rec.idx - b * A.N;
    const long long r0 = __ldg(A.net.rowptr + A.src_off + i);
    const unsigned long long len = (unsigned long long)(__ldg(A.net.rowptr + A.src_off + i + 1) - r0);
    if (log_ok) {
      A.log[s_off + k] = rec;
      A.log_r0[s_off + k] = r0;
      A.log_len[s_off + k] = (int)len;
      if constexpr (kAdm) A.lpos[(size_t)(m % 3) * A.total + rec.idx] = (int)(s_off + k);
    }
    const int tb = b - b_first;
    if (tb < kTr) {
      atomicAdd(&s_ctr[tb][0], 1u);
      atomicAdd(&s_ctr[tb][1], (unsigned)len);
      if (A.kind == EQ_KIND_DONOTHING) atomicAdd(&s_ctr[tb][2], (unsigned)len);
    } else {
      atomicAdd(reinterpret_cast<unsigned long long*>(A.counters + 3 * b), 1ULL);
      atomicAdd(reinterpret_cast<unsigned long long*>(A.counters + 3 * b + 1), len);
      if (A.kind == EQ_KIND_DONOTHING)
        atomicAdd(reinterpret_cast<unsigned long long*>(A.counters + 3 * b + 2), len);
    }
  }
  group_sync(Ro::kBarN, Ro::NN);
  if (gtid == 0) {
    s_n = 0;
    tl_mark_any(A.tl, m, A.G, cta, 6);
  }
}

// Delivery of this CTA's calendar bucket m+1 into acc[(m+1)&1] (events due at
// m+1 it appended in earlier phases; the bucket receives no appends in phase
// m), shared by both warp groups: each warp claims 256-entry chunks from a
// shared counter as soon as its own side's work is done, so the delivery
// fills whichever side finishes first instead of lengthening the event side.
template <typename T, bool kAdm = false>
__device__ __forceinline__ void deliver_bucket(const FwdArgs<T>& A, const int m, const int cta, const int n,
                                               int* s_dq) {
  typedef Prec<T> P;
  constexpr int DV = 8;
  const int lane = threadIdx.x & 31;
  const int bin = (m + 1) % A.NB;
  const longlong2* bk = reinterpret_cast<const longlong2*>(A.bk + ((size_t)cta * A.NB + bin) * A.cap_b * bk_words<T>());
  long long* accn = A.acc + (size_t)((m + 1) & 1) * A.total * P::kSlotWords;
  while (true) {
    int base = 0;
    if (lane == 0) base = atomicAdd(s_dq, DV * 32);
    base = __shfl_sync(0xffffffffu, base, 0);
    if (base >= n) break;
    longlong2 ev[DV], ev2[DV];
#pragma unroll
    for (int e = 0; e < DV; ++e) {
      const int k = base + e * 32 + lane;
      ev[e] = make_longlong2(-1, 0);
      if (k < n) {
        if (P::kSlotWords == 1) {
          ev[e] = __ldcs(bk + k);
        } else {
          ev[e] = __ldcs(bk + 2 * (size_t)k);
          ev2[e] = __ldcs(bk + 2 * (size_t)k + 1);
        }
      }
    }
#pragma unroll
    for (int e = 0; e < DV; ++e) {
      if (ev[e].x < 0) continue;
      long long tg = ev[e].x;
      if constexpr (kAdm) {
        const int sign = (tg & kNegEntry) ? -1 : 1;
        tg &= kNegEntry - 1;
        adm_count(A, (m + 1) & 1, tg, sign);
      }
      if (P::kSlotWords == 1) {
        red_acc(accn + tg, ev[e].y);
      } else {
        red_acc(accn + 2 * (size_t)tg, ev[e].y);
        red_acc(accn + 2 * (size_t)tg + 1, ev2[e].x);
      }
    }
  }
}

// After the barrier of phase m: could the next step overflow the spike log?
// (one step logs at most `total` spikes).  Read from the value the barrier
// published, so every CTA decides the same.
template <typename T>
__device__ __forceinline__ bool pause_due(const FwdArgs<T>& A, int m) {
  return ld_published(A.step_start + m + 1) + A.total > A.log_cap;
}

// kAdmEv: admission events in flight per thread — 2, or 1 when the neuron state
// stays in HBM (C4 heap[16] fwd 129.5 -> 127.2-128.3 ms; C2, state in shared
// memory, prefers 2: profiles/r2bo_ab_admission_ev_split320.txt)
template <typename T, int NT, int U, int NF = NT / 2, bool kAdm = false, int kAdmEv = 2>
__global__ void __launch_bounds__(NT, 2) k_forward(const __grid_constant__ FwdArgs<T> A) {
  // (__grid_constant__: the out-of-line admission fix-ups take A by reference
  // without a local copy)
  typedef Prec<T> P;
  typedef Roles<NT, NF> Ro;
  constexpr int kCap = FwdShared<NT, T>::kCap;
  constexpr int kCapN = kCap / 2;
  constexpr int kTr = FwdShared<NT>::kTrials;
  // event side
  __shared__ SpikeRec<T> s_spk[kCap];
  __shared__ long long s_r0[kCap];
  __shared__ int s_pre[kCap + 1];
  __shared__ int s_bin[FwdShared<NT>::kBins];   // this CTA's bucket fill levels
  // neuron side
  __shared__ SpikeRec<T> s_own[kCapN];
  __shared__ int s_n;
  __shared__ long long s_off;
  __shared__ unsigned s_ctr[kTr][3];   // per-phase counts (32-bit: native smem atomics), flushed every phase
  __shared__ int s_dq;                            // next unclaimed entry of the bucket being delivered
  __shared__ unsigned s_drop[kAdm ? kDropTr : 1];  // admission drops per trial, flushed every phase

  const int tid = threadIdx.x;
  const int cta = blockIdx.x;
  const long long begin = (long long)cta * A.per;
  const long long end = begin + A.per < A.total ? begin + A.per : A.total;
  const int b_first = (int)(begin / A.N);
  const StepConsts<T> c = A.c;
  SpikeRec<T>* spill = A.scratch + (size_t)cta * A.per;
  if (A.no_pause && ld_volatile(A.err) != 0) return;   // an earlier asynchronous window failed

  if (tid < kTr * 3) (&s_ctr[0][0])[tid] = 0u;
  if (tid == 0) s_dq = 0;
  if (kAdm && tid < kDropTr) s_drop[tid] = 0u;
  if (A.cal)
    for (int k = tid; k < A.NB; k += NT) s_bin[k] = A.bk_cnt[(size_t)cta * A.NB + k];
  if (tid == 0) s_n = 0;
  // state in shared memory for the launch (A.smem_state): I then V of the owned range
  extern __shared__ __align__(16) unsigned char s_dynf[];
  T* s_st = A.smem_state ? reinterpret_cast<T*>(s_dynf) : nullptr;
  if (s_st)
    for (long long k = tid; k < end - begin; k += NT) {
      s_st[k] = A.I[begin + k];
      s_st[A.per + k] = A.V[begin + k];
    }
  __syncthreads();

  // Phase m: (a) [event side] deliver this CTA's bucket m+1 and fan out its
  // share of the crossings of step m-1 — the whole grid shares them evenly
  // (they are in the log, contiguous per step); (b) [neuron side] pop + update
  // step m for the owned neurons and log their crossings.  Events of step m-1
  // land at steps >= m+1, never in acc[m&1], and acc[(m+1)&1] is popped only
  // after the barrier.  A last pass m = m1 fans out the final step so the
  // queue contents after the run are complete.
  // m1 may be lowered at a barrier (pause_due): the launch then ends at a step
  // boundary with the spike log one step short of full, the host grows it and
  // relaunches from there (eq_run resumes bitwise, tests/test_gpu_parity.py)
  int m1 = A.m1;
  for (int m = A.m0; m <= m1; ++m) {
    tl_mark(A.tl, m < m1 ? m : m1 - 1, A.G, cta, m < m1 ? 0 : 7);
    // bucket m+1 (complete: phase m appends only to later buckets), delivered
    // by both sides once their own work is done (deliver_bucket)
    int dn = 0;
    if (m > A.m0 && A.cal) {
      dn = s_bin[(m + 1) % A.NB];
      dn = dn < A.cap_b ? dn : (int)A.cap_b;
    }
    // fp64: the neuron side (two neurons per thread, 16-byte slots) finishes
    // well before the fan-out, so both sides share the delivery (fwd 81.9 ->
    // 76.8 ms at C3 x 24); fp32: the sides already finish together and the
    // delivery goes first on the event side (sharing measured 32.8 -> 33.6 ms)
    constexpr bool kShare = sizeof(T) == 8;
    if (tid < Ro::NF) {
      // ======================== event side
      const int gtid = tid;
      if (!kShare) deliver_bucket<T, kAdm>(A, m, cta, dn, &s_dq);
      // ---------------- fan-out of step m-1: fwd_fanout
      if (A.cal && m > A.m0) {
        const int me = m - 1;                          // emitting step
        const long long L0 = ld_published(A.step_start + me), S = ld_published(A.step_start + me + 1) - L0;
        fwd_fanout<T, NT, NF, false, kAdm, kAdmEv>(A, m, cta, gtid, L0 + S * cta / A.G, L0 + S * (cta + 1) / A.G, s_spk,
                                           s_r0, s_pre, s_bin, s_drop);
      }
      if (m < m1) tl_mark(A.tl, m, A.G, cta, 1);
      if (kShare) deliver_bucket<T, kAdm>(A, m, cta, dn, &s_dq);
      if (m < m1) tl_mark(A.tl, m, A.G, cta, 5);
    } else {
      // ======================== neuron side
      const int gtid = tid - Ro::NF;
      if (m < m1) {
        neuron_side<T, NT, U, NF, kAdm>(A, m, cta, gtid, begin, end, b_first, A.cal != 0, s_own, s_n, s_off,
                                        s_ctr, spill, s_st, s_bin);
      } else if constexpr (kAdm) {                    // last pass: the last phase's fix-ups only
        adm_fixups<T>(A, m, true, cta, gtid, Ro::NN, s_bin);
        group_sync(Ro::kBarN, Ro::NN);
        if (gtid == 0) A.fl_cnt[((m - 1) & 1) * A.G + cta] = 0;
      }
      if (kShare) deliver_bucket<T, kAdm>(A, m, cta, dn, &s_dq);
    }
    __syncthreads();
    if (tid == 0) {
      s_dq = 0;
      if (dn > 0 || (m > A.m0 && A.cal)) s_bin[(m + 1) % A.NB] = 0;
    }
    if constexpr (kAdm) {
      if (tid < kDropTr) {
        if (s_drop[tid] && tid < A.B)
          atomicAdd(reinterpret_cast<unsigned long long*>(A.counters + 3 * tid + 2), (unsigned long long)s_drop[tid]);
        s_drop[tid] = 0u;
      }
    }
    if (m == m1) break;
    flush_counters<kTr>(s_ctr, A.counters, b_first, A.B, end, A.N);
    tl_mark(A.tl, m, A.G, cta, 2);
    if (!grid_sync(A.bar, A.G, A.err, A.step_start + m + 1, A.log_count, nullptr,
                   A.cal ? A.ring_dirty + m % A.R : nullptr))
      break;
    tl_mark(A.tl, m, A.G, cta, 3);
    if (ld_volatile(A.err) != 0) break;
    if (m + 1 < m1 && pause_due(A, m)) {             // same published value on every CTA
      if (A.no_pause) {
        raise_error(A.err, EQ_ERR_CAPACITY, m + 1, -1, -1);
        break;
      }
      m1 = m + 1;
    }
  }
  if (cta == 0 && tid == 0) A.err[4] = m1;            // the step this launch reached
  __syncthreads();
  if (s_st)
    for (long long k = tid; k < end - begin; k += NT) {
      A.I[begin + k] = s_st[k];
      A.V[begin + k] = s_st[A.per + k];
    }
  if (A.cal)
    for (int k = tid; k < A.NB; k += NT) A.bk_cnt[(size_t)cta * A.NB + k] = s_bin[k];
  if (tid < kTr) {
    int b = b_first + tid;
    if (b < A.B && (long long)b * A.N < end) {
      for (int q = 0; q < 3; ++q)
        if (s_ctr[tid][q]) atomicAdd(reinterpret_cast<unsigned long long*>(A.counters + 3 * b + q), (unsigned long long)s_ctr[tid][q]);
    }
  }
}

// ------------------------------------------------------------------ reverse

template <typename T>
struct BwdArgs {
  int N, B, G;
  long long total, per;
  int m_run;          // steps simulated since reset (the reverse pass walks m_run-1 .. 0)
  int m_hi, m_lo;     // this launch's phases: m_hi-1 .. m_lo (one exchange window, or all)
  int R, refractory;
  int exact;          // exact delivery (else plain: payload w, Lambda_m = -lambda_vhat)
  int lossy_cap;      // lossy ring: the reference's capacity (events pop at the first step
                      // >= m+1 in the due step's residue class), 0 otherwise
  int serial;         // R-fanout(m-1) after R-neuron(m) behind a grid barrier (lossy ring:
                      // an event of step m-1 may pop at step m, whose reverse row R-neuron(m) writes)
  StepConsts<T> c;
  NetView<T> net;
  T* lamV;
  T* lamI;
  typename Prec<T>::T2* lam;   // [B][R][N] (Lambda_s, Lambda_m)
  double* gw;
  double* gd;
  double* gamp_bt;             // [B][N] or null
  const SpikeRec<T>* log;
  const long long* log_r0;
  const int* log_len;
  T* lt_log;                   // dL/dt_spk per log record
  const long long* chunk_off;
  const int* chunk_cnt;
  const long long* step_start;  // [m] first log record of step m
  int maxdeg;                   // bounded kinds: event id = log position * maxdeg + row offset
  const unsigned* drop_bits;    // bounded kinds: dropped events (contribute nothing); null for ring
  int no_events;                // donothing: every event was dropped
  // partitioned network: dL/dt_spk contributions of the other partitions'
  // edges to this partition's spikes (added at R-neuron), and the imported
  // spikes whose partial dL/dt_spk over this partition's edges the last phase
  // computes (R-fanout of the import block of forward launch m_lo)
  const T* lt_rem;              // [log] or null
  const SpikeRec<T>* imp;
  const long long* imp_r0;
  const int* imp_len;
  long long imp_n;
  const long long* imp_dev;     // peer exchange: {first, count} of the import block on the device
  T* imp_lt;
  unsigned long long* tl;  // debug timeline [m][G][4] or null
  int* err;
  unsigned* bar;
};

// Random 8/16-byte reverse-slot gather: a 64-byte L2 fill instead of the
// default 128 (fewer DRAM bytes per useful byte), marked evict-first: the
// gathered line is rarely hit again before eviction (1.2 GB live ring), so it
// must not displace the per-edge gradient accumulators.  Per-edge gradient
// reductions (dL/dw, dL/dd: 2 x 8 B x E, 160 MB at C3) are evict-last.
// A/B on one box, C3 x 24 trials: no policy 49.1 ms, gathers evict-first
// 45.95, both 45.53 (profiles/r1g_ab_hint.txt).
__device__ __forceinline__ float2 ld_gather(const float2* p) {
  float2 v;
  unsigned long long pol;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  asm volatile("ld.global.L2::cache_hint.L2::64B.v2.f32 {%0, %1}, [%2], %3;"
               : "=f"(v.x), "=f"(v.y) : "l"(p), "l"(pol));
  return v;
}
__device__ __forceinline__ double2 ld_gather(const double2* p) {
  double2 v;
  unsigned long long pol;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  asm volatile("ld.global.L2::cache_hint.L2::64B.v2.f64 {%0, %1}, [%2], %3;"
               : "=d"(v.x), "=d"(v.y) : "l"(p), "l"(pol));
  return v;
}
__device__ __forceinline__ void red_grad(double* p, double v) {
  unsigned long long pol;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
  asm volatile("red.relaxed.gpu.global.add.L2::cache_hint.f64 [%0], %1, %2;" ::"l"(p), "d"(v), "l"(pol)
               : "memory");
}

template <typename T>
struct BwdShared {
  static constexpr int kCapB = sizeof(T) == 4 ? 512 : 256;   // spikes per batch
#ifndef EQ_REV_WIN
#define EQ_REV_WIN 4096
#endif
  static constexpr int kEv = sizeof(T) == 4 ? EQ_REV_WIN : 2048;    // events per reduction window
};

// R-fanout of log records [s0, s1): the CTA's share of step
// m-1's own spikes (kImp = false, dL/dt_spk into lt_log) or of the spikes
// imported before forward launch m_lo (kImp = true, partial dL/dt_spk over
// this partition's edges into imp_lt).  dL/dt_spk of a spike is the SEQUENTIAL
// sum of its edges' g_tp in row order (zeros for events never popped or
// dropped), staged through s_gtp in windows of kEv events; the oracle sums in
// the same order.  Executed by the event-side warp group.
template <typename T, int NT, int NF, bool kImp, int kCapB, int kEv>
__device__ __forceinline__ void bwd_rfanout(const BwdArgs<T>& A, const int m, const int cta, const int gtid,
                                            const long long s0, const long long s1, SpikeRec<T>* s_rec,
                                            long long* s_r0, int* s_pre, T* s_lt, T* s_gtp,
                                            const bool prestaged = false) {
  typedef typename Prec<T>::T2 T2;
  typedef Roles<NT, NF> Ro;
  const StepConsts<T>& c = A.c;
  const SpikeRec<T>* lg = kImp ? A.imp : A.log;
  const long long* lr0 = kImp ? A.imp_r0 : A.log_r0;
  const int* llen = kImp ? A.imp_len : A.log_len;
  T* lt_out = kImp ? A.imp_lt : A.lt_log;
  const int me_fixed = m - 1;
  for (long long k0 = s0; k0 < s1; k0 += kCapB) {
    const int nb = (int)(s1 - k0 < kCapB ? s1 - k0 : kCapB);
    // a single-batch share may have been staged by the neuron side during the previous phase
    if (!prestaged) stage_spikes<T>(lg, lr0, llen, k0, nb, s_rec, s_r0, s_pre, gtid, Ro::NF, Ro::kBarF);
    for (int k = gtid; k < nb; k += Ro::NF) s_lt[k] = (T)0;
    group_sync(Ro::kBarF, Ro::NF);
    if (k0 == s0) tl_mark(A.tl, m, A.G, cta, 4);
    const int total = s_pre[nb];
    for (int w0 = 0; w0 < total; w0 += kEv) {
      const int wend = total - w0 < kEv ? total : w0 + kEv;
#ifndef EQ_REV_EV
#define EQ_REV_EV 2
#endif
      constexpr int EV = EQ_REV_EV;   // events in flight per thread (2: bwd 45.9 -> 43.6 ms vs 3, profiles/r1g_ab_rev*.txt)
      int krow = w0 > 0 ? find_row(s_pre, nb, w0) : 0;     // row of this thread's last event
      for (int f0 = w0 + gtid; f0 < wend; f0 += EV * Ro::NF) {
        int jj[EV], kk[EV];
        long long xx[EV];
        T ww[EV], dd[EV];
        unsigned short cc[EV];
#pragma unroll
        for (int e = 0; e < EV; ++e) {
          const int f = f0 + e * Ro::NF;
          kk[e] = -1;
          if (f < wend) {
            const int k = find_row_from(s_pre, nb, f, krow);
            krow = k;
            const long long x = s_r0[k] + (f - s_pre[k]);
            kk[e] = k;
            xx[e] = x;
            const EdgeRec<T> ed = ld_edge(A.net.er + x);   // one 16-byte streamed load per event
            jj[e] = ed.col;
            ww[e] = ed.w;
            dd[e] = ed.d;
            cc[e] = (unsigned short)ed.code;
          }
        }
#pragma unroll
        for (int e = 0; e < EV; ++e) {
          if (kk[e] < 0) continue;
          const int f = f0 + e * Ro::NF;
          const SpikeRec<T> rec = s_rec[kk[e]];
          const int b = c.divN.div(rec.idx);
          const int me = kImp ? (int)rec.a : me_fixed;
          const T w = ww[e], d = dd[e];
          const T t_post = rec.t + d;
          const int st = delivery_step_coded(t_post, cc[e], c.dt, me);
          int sp = st;                                     // the step the event is popped at
          if (A.lossy_cap > 0 && st - (me + 1) >= A.lossy_cap) sp = me + 1 + (st - (me + 1)) % A.lossy_cap;
          T g_tp = (T)0;
          bool live = sp < A.m_run && !A.no_events;        // never popped / dropped: no effect
          if (live && A.drop_bits) {                       // dropped by a bounded queue
            const long long id = (k0 + kk[e]) * (long long)A.maxdeg + (f - s_pre[kk[e]]);
            live = !((A.drop_bits[id >> 5] >> (id & 31)) & 1u);
          }
          if (live) {
            T es = (T)1, em = (T)1;
            if (A.exact) {
              const T phi = (T)st * c.dt - t_post;
              es = eq_exp_t(-phi * c.inv_tau_s);
              em = eq_exp_t(-phi * c.inv_tau_m);
            }
            const T2 L = ld_gather(A.lam + ((size_t)b * A.R + (size_t)(sp % A.R)) * A.N + jj[e]);
            // plain delivery: W' enters the synapse jump alone, Q = sum w tt
            // enters synapse (+Q/tau_s) and membrane (-Q/tau_m, in Lambda_m)
            const T g_w = A.exact ? es * L.x + em * L.y : L.x;
            g_tp = w * (es * L.x * c.inv_tau_s + em * L.y * c.inv_tau_m);
            red_grad(A.gw + xx[e], (double)g_w);
            red_grad(A.gd + xx[e], (double)g_tp);
          }
          s_gtp[f - w0] = g_tp;
        }
      }
      group_sync(Ro::kBarF, Ro::NF);
      if (k0 == s0 && w0 == 0) tl_mark(A.tl, m, A.G, cta, 5);
      const int ka = find_row(s_pre, nb, w0);
      const int kb = find_row(s_pre, nb, wend - 1);
      for (int k = ka + gtid; k <= kb; k += Ro::NF) {
        const int lo = s_pre[k] > w0 ? s_pre[k] : w0;
        const int hi = s_pre[k + 1] < wend ? s_pre[k + 1] : wend;
        T acc = s_lt[k];
        for (int q = lo; q < hi; ++q) acc = acc + s_gtp[q - w0];
        s_lt[k] = acc;
      }
      group_sync(Ro::kBarF, Ro::NF);
    }
    for (int k = gtid; k < nb; k += Ro::NF) lt_out[k0 + k] = s_lt[k];
  }
}

template <typename T, int NT, int U, int NF = NT / 2>
__global__ void __launch_bounds__(NT, 2) k_backward(BwdArgs<T> A) {
  typedef typename Prec<T>::T2 T2;
  typedef Roles<NT, NF> Ro;
  constexpr int kCapB = BwdShared<T>::kCapB;
  constexpr int kEv = BwdShared<T>::kEv;
  // staging of the event side's spike batch, double-buffered by phase parity:
  // the neuron side pre-stages the next phase's share when it finishes early
  __shared__ SpikeRec<T> s_rec[2][kCapB];
  __shared__ long long s_r0[2][kCapB];
  __shared__ int s_pre[2][kCapB + 1];
  __shared__ int s_ready[2];                  // phase whose share buffer k holds (or -1)
  __shared__ T s_lt[kCapB];
  __shared__ T s_gtp[kEv];
  extern __shared__ unsigned int s_bits[];   // one bit per owned neuron-trial, then uint16 chunk positions
  const int tid = threadIdx.x;
  const int cta = blockIdx.x;
  const long long begin = (long long)cta * A.per;
  const long long end = begin + A.per < A.total ? begin + A.per : A.total;
  const int nwords = (int)((A.per + 31) / 32);
  unsigned short* s_pos = reinterpret_cast<unsigned short*>(s_bits + nwords);
  const StepConsts<T> c = A.c;
  for (int k = tid; k < nwords; k += NT) s_bits[k] = 0u;
  if (tid < 2) s_ready[tid] = -1;
  __syncthreads();

  // Phase m (m = m_run-1 .. 0): [event side] R-fanout of step m-1 (its events
  // read reverse slots of steps >= m+1, all final); [neuron side] R-neuron(m),
  // which writes reverse slot m only and reads dL/dt_spk of its own spikes of
  // step m, produced by the event side of phase m+1.
  bool ok = true;
  for (int m = A.m_hi - 1; m >= A.m_lo && ok; --m) {
    tl_mark(A.tl, m, A.G, cta, 0);
    // serial mode (lossy ring): pass 0 = R-neuron(m), grid barrier, pass 1 =
    // R-fanout(m-1); otherwise one pass with both sides concurrent
    for (int pass = A.serial ? 0 : 1; pass < 2; ++pass) {
    const bool ev_pass = pass == 1, nr_pass = !A.serial || pass == 0;
    if (tid < Ro::NF && ev_pass) {
      // ======================== event side: R-fanout(m-1), shared evenly by
      // the whole grid (whole spikes per CTA): bwd_rfanout
      const int gtid = tid;
      if (m >= 1) {
        const int me = m - 1;
        const int cur = m & 1;
        const long long L0 = A.step_start[me], S = A.step_start[me + 1] - L0;
        bwd_rfanout<T, NT, NF, false, kCapB, kEv>(A, m, cta, gtid, L0 + S * cta / A.G, L0 + S * (cta + 1) / A.G,
                                                  s_rec[cur], s_r0[cur], s_pre[cur], s_lt, s_gtp,
                                                  s_ready[cur] == m);
      }
      tl_mark(A.tl, m, A.G, cta, 1);
    } else if (tid >= Ro::NF && nr_pass) {
      // ======================== neuron side: R-neuron(m)
      const int gtid = tid - Ro::NF;
      const long long off = A.chunk_off[(size_t)m * A.G + cta];
      const int cnt = A.chunk_cnt[(size_t)m * A.G + cta];
      // own spikers of step m -> bitmap (looked up in the own log chunk)
      for (int k = gtid; k < cnt; k += Ro::NN) {
        const int loc = A.log[off + k].idx - (int)begin;
        atomicOr(&s_bits[loc >> 5], 1u << (loc & 31));
        s_pos[loc] = (unsigned short)(k < 0xffff ? k : 0xffff);
      }
      group_sync(Ro::kBarN, Ro::NN);
      const int mm = m < A.net.t_mask ? m : A.net.t_mask - 1;
      const int b_first = (int)(begin / A.N);
      const int b_last = (int)((end - 1) / A.N);
      for (int b = b_first; b <= b_last; ++b) {
        const int tb0 = b * A.N;
        const int j0 = (int)(begin > tb0 ? begin - tb0 : 0);
        const int j1 = (int)(end < (long long)tb0 + A.N ? end - tb0 : A.N);
        const uint32_t* mrow = A.net.mask + ((size_t)b * A.net.t_mask + mm) * A.net.words;
        T2* lam_row = A.lam + ((size_t)b * A.R + (size_t)(m % A.R)) * A.N;
        if (sizeof(T) == 4 && (A.N & 3) == 0 && ((j0 | j1) & 3) == 0) {
          // fp32 fast path: four neurons per thread, 16-byte accesses
          for (int jq = j0 + 4 * gtid; jq < j1; jq += 4 * Ro::NN) {
            const int idx = tb0 + jq;
            const float4 LV4 = *reinterpret_cast<const float4*>(A.lamV + idx);
            const float4 LI4 = *reinterpret_cast<const float4*>(A.lamI + idx);
            const float lvv[4] = {LV4.x, LV4.y, LV4.z, LV4.w};
            const float liv[4] = {LI4.x, LI4.y, LI4.z, LI4.w};
            float nv[4], ni[4], ls[4], lm[4];
            unsigned mw = 0;
            if (A.gamp_bt) mw = __ldg(mrow + (jq >> 5)) >> (jq & 31);
            const int loc0 = idx - (int)begin;
            const unsigned sb = (s_bits[loc0 >> 5] >> (loc0 & 31)) & 0xfu;
#pragma unroll
            for (int q = 0; q < 4; ++q) {
              const T lv = (T)lvv[q];
              T la, lvh;
              if ((sb >> q) & 1u) {
                int k = s_pos[loc0 + q];
                if (k == 0xffff) {
                  k = 0;
                  while (k < cnt && A.log[off + k].idx != idx + q) ++k;
                }
                SpikeRec<T> rec = A.log[off + k];
                const T lt0 = (m + 1 < A.m_run ? A.lt_log[off + k] : (T)0) + (A.lt_rem ? A.lt_rem[off + k] : (T)0);
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
              const T lip = (T)liv[q] + la;
              if (A.gamp_bt && ((mw >> q) & 1u)) A.gamp_bt[idx + q] += (double)la;
              ls[q] = (float)(c.k_s * lip - c.cc * lvh);
              lm[q] = (float)(c.cm * lvh);
              ni[q] = (float)(c.k_s * lip);
              nv[q] = (float)lvh;
            }
            float4* lr4 = reinterpret_cast<float4*>(lam_row + jq);
            // read back only by random gathers 1..H phases later (from DRAM): streaming stores
            __stcs(lr4, make_float4(ls[0], lm[0], ls[1], lm[1]));
            __stcs(lr4 + 1, make_float4(ls[2], lm[2], ls[3], lm[3]));
            *reinterpret_cast<float4*>(A.lamI + idx) = make_float4(ni[0], ni[1], ni[2], ni[3]);
            *reinterpret_cast<float4*>(A.lamV + idx) = make_float4(nv[0], nv[1], nv[2], nv[3]);
          }
          continue;
        }
        if (sizeof(T) == 8 && (A.N & 1) == 0 && ((j0 | j1) & 1) == 0) {
          // fp64 fast path: two neurons per thread, 16-byte accesses
          for (int jq = j0 + 2 * gtid; jq < j1; jq += 2 * Ro::NN) {
            const int idx = tb0 + jq;
            const double2 LV2 = *reinterpret_cast<const double2*>(A.lamV + idx);
            const double2 LI2 = *reinterpret_cast<const double2*>(A.lamI + idx);
            const double lvv[2] = {LV2.x, LV2.y};
            const double liv[2] = {LI2.x, LI2.y};
            double nv[2], ni[2], ls[2], lm[2];
            unsigned mw = 0;
            if (A.gamp_bt) mw = __ldg(mrow + (jq >> 5)) >> (jq & 31);
            const int loc0 = idx - (int)begin;
            const unsigned sb = (s_bits[loc0 >> 5] >> (loc0 & 31)) & 0x3u;
#pragma unroll
            for (int q = 0; q < 2; ++q) {
              const T lv = (T)lvv[q];
              T la, lvh;
              if ((sb >> q) & 1u) {
                int k = s_pos[loc0 + q];
                if (k == 0xffff) {
                  k = 0;
                  while (k < cnt && A.log[off + k].idx != idx + q) ++k;
                }
                SpikeRec<T> rec = A.log[off + k];
                const T lt0 = (m + 1 < A.m_run ? A.lt_log[off + k] : (T)0) + (A.lt_rem ? A.lt_rem[off + k] : (T)0);
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
              const T lip = (T)liv[q] + la;
              if (A.gamp_bt && ((mw >> q) & 1u)) A.gamp_bt[idx + q] += (double)la;
              ls[q] = (double)(c.k_s * lip - c.cc * lvh);
              lm[q] = (double)(c.cm * lvh);
              ni[q] = (double)(c.k_s * lip);
              nv[q] = (double)lvh;
            }
            double2* lr2 = reinterpret_cast<double2*>(lam_row + jq);
            __stcs(lr2, make_double2(ls[0], lm[0]));
            __stcs(lr2 + 1, make_double2(ls[1], lm[1]));
            *reinterpret_cast<double2*>(A.lamI + idx) = make_double2(ni[0], ni[1]);
            *reinterpret_cast<double2*>(A.lamV + idx) = make_double2(nv[0], nv[1]);
          }
          continue;
        }
        for (int jb = j0; jb < j1; jb += Ro::NN * U) {
          T LV[U], LI[U];
#pragma unroll
          for (int u = 0; u < U; ++u) {
            const int j = jb + u * Ro::NN + gtid;
            if (j < j1) {
              LV[u] = A.lamV[tb0 + j];
              LI[u] = A.lamI[tb0 + j];
            }
          }
#pragma unroll
          for (int u = 0; u < U; ++u) {
            const int j = jb + u * Ro::NN + gtid;
            if (j >= j1) continue;
            const int idx = tb0 + j;
            const T lv = LV[u];
            T la, lvh;
            const int loc = idx - (int)begin;
            if ((s_bits[loc >> 5] >> (loc & 31)) & 1u) {
              int k = s_pos[loc];
              if (k == 0xffff) {
                k = 0;
                while (k < cnt && A.log[off + k].idx != idx) ++k;
              }
              SpikeRec<T> rec = A.log[off + k];
              const T lt0 = (m + 1 < A.m_run ? A.lt_log[off + k] : (T)0) + (A.lt_rem ? A.lt_rem[off + k] : (T)0);
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
            T lip = LI[u] + la;
            if (A.gamp_bt && ((__ldg(mrow + (j >> 5)) >> (j & 31)) & 1u)) A.gamp_bt[idx] += (double)la;
            T2 L;
            L.x = c.k_s * lip - c.cc * lvh;
            L.y = c.cm * lvh;
            lam_row[j] = L;
            A.lamI[idx] = c.k_s * lip;
            A.lamV[idx] = lvh;
          }
        }
      }
      group_sync(Ro::kBarN, Ro::NN);
      for (int k = gtid; k < cnt; k += Ro::NN) {
        const int loc = A.log[off + k].idx - (int)begin;
        s_bits[loc >> 5] = 0u;
      }
      if (gtid == 0) tl_mark_any(A.tl, m, A.G, cta, 6);
      // pre-stage the event side's share of the next phase (R-fanout of step
      // m-2) into the other buffer: the event side is the critical path
      if (m - 1 >= A.m_lo && m - 1 >= 1) {
        const int nxt = (m - 1) & 1;
        const long long L0 = A.step_start[m - 2], S = A.step_start[m - 1] - L0;
        const long long s0 = L0 + S * cta / A.G, s1 = L0 + S * (cta + 1) / A.G;
        if (s1 - s0 <= kCapB) {
          stage_spikes<T>(A.log, A.log_r0, A.log_len, s0, (int)(s1 - s0), s_rec[nxt], s_r0[nxt], s_pre[nxt], gtid,
                          Ro::NN, Ro::kBarN);
          if (gtid == 0) s_ready[nxt] = m - 1;
        }
      }
    }
    if (A.serial && pass == 0 && !grid_sync(A.bar, A.G, A.err)) ok = false;
    if (!ok) break;
    }
    if (!ok) break;
    __syncthreads();
    tl_mark(A.tl, m, A.G, cta, 2);
    if (!grid_sync(A.bar, A.G, A.err)) break;
    tl_mark(A.tl, m, A.G, cta, 3);
    if (ld_volatile(A.err) != 0) break;
  }
}

// Reverse of k_import_fanout: after a reverse window's launch (phases down to
// m_lo, so reverse slots >= m_lo are final), the partial dL/dt_spk over this
// partition's edges of the spikes imported before forward launch m_lo — their
// events are due >= m_lo + 1 because the exchange window is <= D_min.
template <typename T, int NT>
__global__ void __launch_bounds__(NT) k_import_rfanout(BwdArgs<T> A) {
  constexpr int kCapB = BwdShared<T>::kCapB;
  constexpr int kEv = BwdShared<T>::kEv;
  __shared__ SpikeRec<T> s_rec[kCapB];
  __shared__ long long s_r0[kCapB];
  __shared__ int s_pre[kCapB + 1];
  __shared__ T s_lt[kCapB];
  __shared__ T s_gtp[kEv];
  const int cta = blockIdx.x;
  long long first = 0, n = A.imp_n;
  if (A.imp_dev) {
    first = A.imp_dev[0];
    n = A.imp_dev[1];
  }
  bwd_rfanout<T, NT, NT, true, kCapB, kEv>(A, A.m_lo, cta, threadIdx.x, first + n * cta / A.G,
                                           first + n * (cta + 1) / A.G, s_rec, s_r0, s_pre, s_lt, s_gtp);
}

}  // namespace eq
