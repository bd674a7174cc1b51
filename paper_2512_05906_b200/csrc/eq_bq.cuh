// eq_bq.cuh — the bounded queue kinds, FIFORing (queues.py:184-260),
// BinaryHeap (queues.py:481-571) and SortedArray (queues.py:308-403), for
// capacities up to kBqMaxCap: per-neuron queues kept in HBM between steps and
// STAGED IN SHARED MEMORY for each step's operations, arrivals grouped by an
// in-kernel counting sort.  Opt-in (eq_config.staged_queues): parity-green
// like the HBM-resident structures of eq_bounded.cuh, but measured slower on
// B200 (C2 heap[64] fwd 76 vs 44 ms, C4 heap[16] 506 vs 317 ms: the inbox
// atomics and the per-round stalls of the queue pass cost more than the
// dependent HBM round trips they replace — DESIGN.md §6.4).
//
// Queue q = trial * N + j, storage capacity C (the capacity rounded up to 4):
//   keys[q][C]  uint32 (due mod 2^24) << 8 | slot, entries [0, count):
//               binary min-heap on due / array sorted by due (stable) / FIFO
//               in arrival order — only these 4-byte keys move
//   pay[q][C]   fixed-point payload of slot s (fp32: packed (qm << 32) + qs;
//               fp64: {qs, qm}), written once at insert, read once at pop
//   meta[q]     int4 {count, occupied-slot mask lo, mask hi, FIFO tail key}
//   qdue[q]     the queue's next due step (INT_MAX when empty)
//
// Phase m of k_forward_bq, one grid barrier per step:
//   0. arrival sort: the arrivals of step m-1 sit in this CTA's inbox in
//      arrival order (every producer appended with one atomic on the owner's
//      counter, and counted the target); an in-kernel counting sort — one
//      radix pass on the target, a block scan of the per-target counts, a
//      scatter of inbox positions — groups them by target (the segmented
//      sort; the edge order inside a target's segment is the insertion order
//      below).  Inbox, counts and index stay L2-resident (one step's arrivals).
//   1. queue pass, over the CTA's queues in chunks: a vectorised scan of qdue
//      and the arrival counters finds the busy queues (a pop due at m, or
//      arrivals of step m-1) and compacts them into a shared-memory list;
//      rounds of one busy queue per thread then stage its keys with cp.async
//      (every thread's copies in flight at once), insert the arrivals in
//      ascending edge order with the reference's accept-while-not-full rule
//      (queues.py:225-226, :514-515, :344-345), pop every event due at m, sum
//      the popped payloads into the step's accumulator acc[m & 1] and write
//      the keys back.  A full queue drops its arrivals without being staged.
//   2. neuron pass: eq_ring.cuh's neuron_side (vectorised LIF over all owned
//      neurons, popping acc[m & 1]) — the ring kind's code, unchanged.
//   3. fan-out of the CTA's own crossings of step m (from its log chunk) into
//      the owners' inboxes, for insertion at phase m+1.
// Pops sum fixed-point payloads, so ties among equal due steps may sit in any
// order: accepted sets, popped sums and pending contents equal the reference's.
#pragma once

#include "eq_bounded.cuh"

namespace eq {

constexpr int kBqMaxCap = 64;         // largest capacity staged in shared memory

template <typename T> struct BqPay;
template <> struct BqPay<float> { typedef long long type; };    // packed (qm << 32) + qs
template <> struct BqPay<double> { typedef longlong2 type; };   // {qs, qm}

__device__ __forceinline__ unsigned bq_key(int due, int slot) { return ((unsigned)due << 8) | (unsigned)slot; }
// due - m for a key whose due is in [m, m + 2^23): the heap / sorted order key
__device__ __forceinline__ unsigned bq_rel(unsigned key, int m) { return ((key >> 8) - (unsigned)m) & 0xFFFFFFu; }
__device__ __forceinline__ int bq_slot(unsigned key) { return (int)(key & 0xFFu); }

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
  const unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(sa), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;" ::: "memory"); }

// One arrival in an owner's inbox: edge x (the reference's arrival order
// within a step is ascending x), due step, flat target, drop-bit id (log
// position * maxdeg + row offset), fixed-point payload.
template <typename T> struct InArr;
template <> struct alignas(32) InArr<float> {
  int x, due, tgt, pad;
  long long id;
  long long p;
};
template <> struct alignas(8) InArr<double> {
  int x, due, tgt, pad;
  long long id;
  long long ps, pm;
};

struct BqState {
  int count, tail;            // tail: FIFO tail key (queues.py:220-224)
  unsigned long long mask;    // occupied payload slots
};

__device__ __forceinline__ void bq_add(long long v, long long& qs, long long& qm) { qs += v; }
__device__ __forceinline__ void bq_add(longlong2 v, long long& qs, long long& qm) {
  qs += v.x;
  qm += v.y;
}

// Insert one event (called in reference order) into the staged keys.  0
// accepted, 1 dropped (full), 2 capability error (FIFO order).  The payload
// goes straight to its slot in HBM.
template <typename PT>
__device__ __forceinline__ int bq_insert(int kind, int cap, unsigned* sk, BqState& st, int m, int due, PT p,
                                         PT* pay) {
  if (kind == EQ_KIND_FIFORING && due < st.tail) return 2;     // queues.py:220-224
  if (st.count == cap) return 1;                               // :225-226, :514-515, :344-345
  const int slot = __ffsll((long long)~st.mask) - 1;           // a free slot: count < cap <= C <= 64
  st.mask |= 1ull << slot;
  pay[slot] = p;
  const unsigned key = bq_key(due, slot);
  const unsigned rk = bq_rel(key, m);
  int i = st.count++;
  if (kind == EQ_KIND_FIFORING) {                              // append (queues.py:227-231)
    st.tail = due;
  } else if (kind == EQ_KIND_BINARYHEAP) {                     // sift up (queues.py:521-528)
    while (i > 0) {
      const int parent = (i - 1) >> 1;
      const unsigned pk = sk[parent];
      if (bq_rel(pk, m) <= rk) break;
      sk[i] = pk;
      i = parent;
    }
  } else {                                                     // sorted: insertion sweep (:351-366), stable
    while (i > 0 && bq_rel(sk[i - 1], m) > rk) {
      sk[i] = sk[i - 1];
      --i;
    }
  }
  sk[i] = key;
  return 0;
}

// Pop every event due at m (the minimum) from the staged keys; returns the
// popped slots (freed in st.mask).
__device__ __forceinline__ unsigned long long bq_pop(int kind, unsigned* sk, BqState& st, int m) {
  unsigned long long popped = 0;
  if (kind == EQ_KIND_BINARYHEAP) {
    while (st.count > 0 && bq_rel(sk[0], m) == 0) {            // :555-568
      popped |= 1ull << bq_slot(sk[0]);
      const int last = --st.count;
      if (last > 0) {
        const unsigned item = sk[last];
        const unsigned ri = bq_rel(item, m);
        int i = 0;
        while (true) {                                         // sift down (:531-553)
          int ch = 2 * i + 1;
          if (ch >= last) break;
          unsigned ck = sk[ch], cr = bq_rel(ck, m);
          if (ch + 1 < last) {
            const unsigned k1 = sk[ch + 1], r1 = bq_rel(k1, m);
            if (r1 < cr) {
              ch += 1;
              ck = k1;
              cr = r1;
            }
          }
          if (cr >= ri) break;
          sk[i] = ck;
          i = ch;
        }
        sk[i] = item;
      }
    }
  } else {                                                     // due run at the head (:245-254, :378-398)
    int p = 0;
    while (p < st.count && bq_rel(sk[p], m) == 0) {
      popped |= 1ull << bq_slot(sk[p]);
      ++p;
    }
    if (p > 0) {
      for (int k = p; k < st.count; ++k) sk[k - p] = sk[k];
      st.count -= p;
    }
  }
  st.mask &= ~popped;
  return popped;
}

// Sum the payloads of the popped slots, four independent loads per group.
template <typename PT>
__device__ __forceinline__ void bq_sum(unsigned long long popped, const PT* pay, long long& qs, long long& qm) {
  while (popped) {
    int s[4];
    int n = 0;
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      s[e] = 0;
      if (popped) {
        s[e] = __ffsll((long long)popped) - 1;
        popped &= popped - 1;
        n = e + 1;
      }
    }
    PT v[4];
#pragma unroll
    for (int e = 0; e < 4; ++e)
      if (e < n) v[e] = pay[s[e]];
#pragma unroll
    for (int e = 0; e < 4; ++e)
      if (e < n) bq_add(v[e], qs, qm);
  }
}

constexpr int kBqChunk = 2048;        // queues scanned per chunk (4 per thread at 512 threads)
constexpr int kBqPoolWords = 8192;    // key staging (32 KB): kBqPoolWords / C queues per round

// Block-wide exclusive scan of one int per thread; returns the total.
template <int NT>
__device__ __forceinline__ int block_exclusive_scan(int v, int& excl, int* s_warp) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  int x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) s_warp[warp] = x;
  __syncthreads();
  if (warp == 0) {
    int w = lane < NT / 32 ? s_warp[lane] : 0;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, w, o);
      if (lane >= o) w += y;
    }
    if (lane < NT / 32) s_warp[lane] = w;   // inclusive warp prefix
  }
  __syncthreads();
  const int before = warp > 0 ? s_warp[warp - 1] : 0;
  excl = before + x - v;
  const int total = s_warp[NT / 32 - 1];
  __syncthreads();
  return total;
}

template <typename T>
struct BqView {                 // the staged-queue arrays of BndArgs, typed
  unsigned* keys;
  typename BqPay<T>::type* pay;
  int4* meta;
  int* qdue;
};

// One busy queue of phase m (insert the arrivals of step m-1, pop m), keys
// staged at sk.  Returns nothing; writes acc[m & 1][idx] when events popped.
template <typename T>
__device__ __forceinline__ void bq_process(const BndArgs<T>& A, const BqView<T>& Q, int m, bool last, int idx,
                                           unsigned* sk, int b_first, unsigned (*s_ctr)[3]) {
  typedef typename BqPay<T>::type PT;
  const FwdArgs<T>& F = A.f;
  const int C = A.C, kind = F.kind;
  constexpr int kTr = FwdShared<512>::kTrials;
  const int b = F.c.divN.div(idx);
  const int j = idx - b * F.N;
  const int4 mt = Q.meta[idx];
  const int qd = Q.qdue[idx];
  const bool ins = m - 1 >= A.insert_first && m >= 1;
  const int par = (m - 1) & 1;
  int* cntp = A.acnt + ((size_t)par * F.B + b) * F.N + j;
  const int narr = ins ? *cntp : 0;
  const int a_end = narr > 0 ? A.aoff[idx] : 0;
  BqState st;
  st.count = mt.x;
  st.mask = ((unsigned long long)(unsigned)mt.z << 32) | (unsigned long long)(unsigned)mt.y;
  st.tail = mt.w;
  const bool pop_due = !last && st.count > 0 && qd == m;
  const bool can_ins = narr > 0 && st.count < A.cap;
  unsigned* gk = A.keys + (size_t)idx * C;
  const int cta = blockIdx.x;
  const InArr<T>* inb = reinterpret_cast<const InArr<T>*>(A.inbox) + ((size_t)par * F.G + cta) * A.in_cap;
  const int* ai = A.aidx + (size_t)cta * A.in_cap + (a_end - narr);
  if (pop_due || can_ins) {                          // stage the occupied keys
    for (int k = 0; k < st.count; k += 4) cp_async16(sk + k, gk + k);
  }
  cp_async_wait_all();
  PT* const pay = Q.pay + (size_t)idx * C;
  bool dirty = false;
  if (narr > 0) {
    *cntp = 0;
    unsigned long long drops = 0;
    int last_x = -1;
    for (int r = 0; r < narr; ++r) {                 // ascending x = the reference's arrival order
      int best = r;
      if (can_ins) {
        int bx = 0x7fffffff;
        for (int k = 0; k < narr; ++k) {
          const int x = inb[ai[k]].x;
          if (x > last_x && x < bx) {
            bx = x;
            best = k;
          }
        }
        last_x = bx;
      }
      const InArr<T> a = inb[ai[best]];
      int rc;
      if (can_ins) {
        PT p;
        if constexpr (sizeof(T) == 4) p = a.p;
        else p = make_longlong2(a.ps, a.pm);
        rc = bq_insert<PT>(kind, A.cap, sk, st, m, a.due, p, pay);
        dirty = true;
      } else {                                       // full: every arrival dropped (FIFO order still checked)
        rc = (kind == EQ_KIND_FIFORING && a.due < st.tail) ? 2 : 1;
      }
      if (rc == 2) {
        raise_error(F.err, EQ_ERR_CAPABILITY, m, b, j);
      } else if (rc == 1) {
        drops += 1;
        const long long id = a.id;
        if (id < A.drop_cap) atomicOr(A.drop_bits + (id >> 5), 1u << (id & 31));
        else raise_error(F.err, EQ_ERR_CAPACITY, m - 1, b, j);
      }
    }
    if (drops) {
      const int tb = b - b_first;
      if (tb < kTr) atomicAdd(&s_ctr[tb][2], (unsigned)drops);
      else atomicAdd(reinterpret_cast<unsigned long long*>(F.counters + 3 * b + 2), drops);
    }
  }
  if (pop_due) {
    const unsigned long long popped = bq_pop(kind, sk, st, m);
    long long qs = 0, qm = 0;
    bq_sum<PT>(popped, pay, qs, qm);
    if (Prec<T>::kSlotWords == 1) {                  // packed pair, summed mod 2^64
      F.acc[(size_t)(m & 1) * F.total + idx] = qs;
    } else {
      long long* o = F.acc + ((size_t)(m & 1) * F.total + idx) * 2;
      o[0] = qs;
      o[1] = qm;
    }
    dirty = true;
  }
  if (dirty) {
    for (int k = 0; k < st.count; k += 4)
      *reinterpret_cast<uint4*>(gk + k) = *reinterpret_cast<const uint4*>(sk + k);
    Q.meta[idx] = make_int4(st.count, (int)(unsigned)(st.mask & 0xffffffffull), (int)(unsigned)(st.mask >> 32),
                            st.tail);
    Q.qdue[idx] = st.count ? m + (int)bq_rel(sk[0], m) : 0x7fffffff;
  }
}

// Fan-out of this CTA's crossings of step m (its log chunk) into the owners'
// inboxes: one record {edge, due, target, drop id, payload} per event at a
// position from the owner's counter, plus the target's arrival count; the
// owner sorts and inserts them in edge order at phase m+1.
template <typename T, int NT>
__device__ __forceinline__ void bq_fanout(const BndArgs<T>& A, int m, int cta, int tid, SpikeRec<T>* s_spk,
                                          long long* s_r0, int* s_pre) {
  typedef Prec<T> P;
  constexpr int kCap = FwdShared<NT, T>::kCap;
  const FwdArgs<T>& F = A.f;
  const StepConsts<T>& c = F.c;
  const long long L0 = F.chunk_off[(size_t)m * F.G + cta];
  const int n = F.chunk_cnt[(size_t)m * F.G + cta];
  if (L0 + n > F.log_cap) return;                    // (the log overflow is already an error)
  const int par = m & 1;
  for (int k0 = 0; k0 < n; k0 += kCap) {
    const int nb = n - k0 < kCap ? n - k0 : kCap;
    stage_spikes<T>(F.log, F.log_r0, F.log_len, L0 + k0, nb, s_spk, s_r0, s_pre, tid, NT, 3);
    const int total = s_pre[nb];
    for (int f = tid; f < total; f += NT) {
      const int k = find_row(s_pre, nb, f);
      const int ro = f - s_pre[k];
      const long long x = s_r0[k] + ro;
      const SpikeRec<T> rec = s_spk[k];
      const int b = c.divN.div(rec.idx);
      const EdgeRec<T> ed = ld_edge(F.net.er + x);
      const int jt = ed.col;
      const T t_post = rec.t + ed.d;
      const int ds = delivery_step_coded(t_post, (unsigned short)ed.code, c.dt, m);
      T ws, wm;
      if (F.exact) {
        const T phi = (T)ds * c.dt - t_post;
        ws = ed.w * eq_exp_t(-phi * c.inv_tau_s);
        wm = ed.w * eq_exp_t(-phi * c.inv_tau_m);
      } else {
        ws = ed.w;
        wm = (T)0;
      }
      const long long q1 = P::q(ws, c.scale), q2 = P::q(wm, c.scale);
      const int tgt = b * F.N + jt;
      const int owner = A.divPer.div(tgt);
      InArr<T> ar;
      ar.x = (int)x;
      ar.due = ds;
      ar.tgt = tgt;
      ar.pad = 0;
      ar.id = (L0 + k0 + k) * (long long)A.maxdeg + ro;
      if constexpr (sizeof(T) == 4) {
        ar.p = pack2(q1, q2);
      } else {
        ar.ps = q1;
        ar.pm = q2;
      }
      const int pos = atomicAdd(A.in_cnt + par * F.G + owner, 1);
      if (pos < A.in_cap)
        reinterpret_cast<InArr<T>*>(A.inbox)[((size_t)par * F.G + owner) * A.in_cap + pos] = ar;
      else
        raise_error(F.err, EQ_ERR_CAPACITY, m, b, jt);
      atomicAdd(A.acnt + (size_t)par * F.B * F.N + tgt, 1);    // the owner's counting sort
    }
  }
}

template <typename T, int NT, int U>
__global__ void __launch_bounds__(NT, 2) k_forward_bq(BndArgs<T> A) {
  constexpr int kCap = FwdShared<NT, T>::kCap;
  constexpr int kCapN = kCap / 2;
  constexpr int kTr = FwdShared<NT>::kTrials;
  __shared__ SpikeRec<T> s_spk[kCap];             // fan-out staging
  __shared__ long long s_r0[kCap];
  __shared__ int s_pre[kCap + 1];
  __shared__ SpikeRec<T> s_own[kCapN];            // neuron pass
  __shared__ int s_n;
  __shared__ long long s_off;
  __shared__ unsigned s_ctr[kTr][3];   // per-phase counts (32-bit: native smem atomics), flushed every phase
  __shared__ int s_warp[NT / 32];
  extern __shared__ __align__(16) unsigned s_dyn[];
  int* s_busy = reinterpret_cast<int*>(s_dyn);                 // [kBqChunk]
  unsigned* s_pool = s_dyn + kBqChunk;                         // [kBqPoolWords]
  const FwdArgs<T>& F = A.f;
  BqView<T> Q;
  Q.keys = A.keys;
  Q.pay = reinterpret_cast<typename BqPay<T>::type*>(A.pay);
  Q.meta = A.meta;
  Q.qdue = A.qdue;

  const int tid = threadIdx.x;
  const int cta = blockIdx.x;
  const long long begin = (long long)cta * F.per;
  const long long end = begin + F.per < F.total ? begin + F.per : F.total;
  const int b_first = (int)(begin / F.N);
  SpikeRec<T>* spill = F.scratch + (size_t)cta * F.per;
  const int C = A.C;
  const int per_round = kBqPoolWords / C < NT ? kBqPoolWords / C : NT;
  unsigned* const sk = s_pool + (tid < per_round ? tid : 0) * C;
  if (tid < kTr * 3) (&s_ctr[0][0])[tid] = 0u;
  if (tid == 0) s_n = 0;
  __syncthreads();

  int m1 = F.m1;   // lowered at a barrier when the spike log could overflow (pause_due)
  for (int m = F.m0; m <= m1; ++m) {
    const bool last = (m == m1);   // extra pass: insert the final step's arrivals only
    if (!last) tl_mark(F.tl, m, F.G, cta, 0);
    const bool ins = m - 1 >= A.insert_first && m >= 1;
    const int* acnt = A.acnt + (size_t)((m - 1) & 1) * F.B * F.N;
    // ---------------- 0. arrival sort (counting sort of the inbox by target)
    if (ins) {
      int carry = 0;
      for (long long cb = begin; cb < end; cb += kBqChunk) {
        int c4[4], sum = 0;
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const long long q = cb + 4 * tid + e;
          c4[e] = (q < end && q < cb + kBqChunk) ? acnt[q] : 0;
          sum += c4[e];
        }
        int off;
        const int tot = block_exclusive_scan<NT>(sum, off, s_warp);
        off += carry;
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const long long q = cb + 4 * tid + e;
          if (q < end && q < cb + kBqChunk) A.aoff[q] = off;   // run start; the scatter advances it to the end
          off += c4[e];
        }
        carry += tot;
      }
      __syncthreads();
      const int par = (m - 1) & 1;
      const int n_in = A.in_cnt[par * F.G + cta];
      const InArr<T>* inb = reinterpret_cast<const InArr<T>*>(A.inbox) + ((size_t)par * F.G + cta) * A.in_cap;
      int* aix = A.aidx + (size_t)cta * A.in_cap;
      for (int r = tid; r < n_in && r < A.in_cap; r += NT) aix[atomicAdd(A.aoff + inb[r].tgt, 1)] = r;
      __syncthreads();
      if (tid == 0) A.in_cnt[par * F.G + cta] = 0;
    }
    // ---------------- 1. queue pass
    for (long long cb = begin; cb < end; cb += kBqChunk) {
      int flags = 0;
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const long long q = cb + 4 * tid + e;
        if (q < end && q < cb + kBqChunk) {
          const bool busy = (!last && Q.qdue[q] == m) || (ins && acnt[q] > 0);
          flags |= (int)busy << e;
        }
      }
      int off;
      const int nb = block_exclusive_scan<NT>(__popc(flags), off, s_warp);
#pragma unroll
      for (int e = 0; e < 4; ++e)
        if ((flags >> e) & 1) s_busy[off++] = (int)(cb + 4 * tid + e);
      __syncthreads();
      for (int r0 = 0; r0 < nb; r0 += per_round)
        if (tid < per_round && r0 + tid < nb) bq_process<T>(A, Q, m, last, s_busy[r0 + tid], sk, b_first, s_ctr);
      __syncthreads();
    }
    if (last) break;
    tl_mark(F.tl, m, F.G, cta, 1);
    // ---------------- 2. neuron pass: pop acc[m & 1], LIF, spike log (eq_ring.cuh)
    neuron_side<T, NT, U, 0>(F, m, cta, tid, begin, end, b_first, true, s_own, s_n, s_off, s_ctr, spill, nullptr);
    __syncthreads();
    // ---------------- 3. fan-out of the crossings of step m
    bq_fanout<T, NT>(A, m, cta, tid, s_spk, s_r0, s_pre);
    __syncthreads();
    flush_counters<kTr>(s_ctr, F.counters, b_first, F.B, end, F.N);
    tl_mark(F.tl, m, F.G, cta, 2);
    if (!grid_sync(F.bar, F.G, F.err, F.step_start + m + 1, F.log_count)) break;
    tl_mark(F.tl, m, F.G, cta, 3);
    if (ld_volatile(F.err) != 0) break;
    if (m + 1 < m1 && pause_due(F, m)) m1 = m + 1;
  }
  if (cta == 0 && tid == 0) F.err[4] = m1;
  __syncthreads();
  if (tid < kTr) {
    const int b = b_first + tid;
    if (b < F.B && (long long)b * F.N < end) {
      for (int q = 0; q < 3; ++q)
        if (s_ctr[tid][q]) atomicAdd(reinterpret_cast<unsigned long long*>(F.counters + 3 * b + q), (unsigned long long)s_ctr[tid][q]);
    }
  }
}

__global__ void k_meta_init_bq(int4* meta, int* qdue, long long n) {
  for (long long k = blockIdx.x * (long long)blockDim.x + threadIdx.x; k < n; k += (long long)gridDim.x * blockDim.x) {
    meta[k] = make_int4(0, 0, 0, -1);                  // FIFORingQueue._tail_key = -1
    qdue[k] = 0x7fffffff;
  }
}

// Pending contents (canonical int64 [B*N][H][2], due now .. now+H-1).
template <typename T>
__global__ void k_pending_bq(const unsigned* keys, const typename BqPay<T>::type* pay, const int4* meta, int C,
                             long long total, int H, int now, long long* out) {
  for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < total;
       idx += (long long)gridDim.x * blockDim.x) {
    long long* o = out + idx * H * 2;
    for (int k = 0; k < 2 * H; ++k) o[k] = 0;
    const int count = meta[idx].x;
    for (int k = 0; k < count; ++k) {
      const unsigned key = keys[idx * C + k];
      const int h = (int)bq_rel(key, now);
      if (h >= H) continue;
      long long qs = 0, qm = 0;
      bq_add(pay[idx * C + bq_slot(key)], qs, qm);
      if (sizeof(T) == 4) {
        const long long packed = qs;
        unpack2(packed, qs, qm);
      }
      o[2 * h] += qs;
      o[2 * h + 1] += qm;
    }
  }
}

}  // namespace eq
