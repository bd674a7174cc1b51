// eq_bounded.cuh — persistent fused forward kernel for the bounded queue kinds:
// FIFORing (queues.py:184-260), BinaryHeap (queues.py:481-571) and SortedArray
// (queues.py:308-403).
//
// All three drop the INCOMING event when the queue holds `capacity` events and
// pop every event due now, so their accepted sets are identical (SURVEY App.
// A.6); only the data structure — and so the cost profile — differs.  The
// accept decision depends on arrival order, which the reference fixes as
// (emit step, source ascending, CSR row order) = ascending CSR edge index.
// Parallel fan-out cannot produce that order, so an arrival is not inserted by
// its producer.  Instead:
//
//   phase m, producer (the CTA that detected the crossing): each event of
//     edge x -> target j is appended to j's arrival list (a slot from an
//     atomic per-target counter, inside j's in-edge segment csc_off[j]..: it
//     cannot overflow) as one 32-byte record {x, log position, due, row
//     offset, payload} — one full sector per event, no partial writes;
//   phase m+1, owner of j, before pop(m+1): read j's (few) arrivals and insert
//     them in ascending x, exactly the reference order — FIFO tail-key check
//     (CapabilityError), drop when full, structure insert.
//
// Lists and counters are double-buffered by step parity (phase m+1 producers
// write step m+1 while owners read step m).  The final step's arrivals are
// inserted after a last barrier so the queue contents after a run equal the
// reference's.  Pops and sums are fixed point (order-free), as for the ring.
#pragma once

#include "eq_ring.cuh"

namespace eq {

// staging / queue entry.  `tag` = log position of the source spike (staging)
// or insertion sequence number (heap).  due_off = due - emit step (<= horizon);
// row_off = edge offset within the source's CSR row (drop bookkeeping).
template <typename T> struct QEv;
template <> struct alignas(16) QEv<float> {
  int tag;
  int due;
  long long p;        // packed fixed-point pair (qm << 32) + qs
  __device__ __forceinline__ void add_to(long long& s, long long& m) const {
    long long a, b;
    unpack2(p, a, b);
    s += a;
    m += b;
  }
};
template <> struct alignas(16) QEv<double> {
  int tag;
  int due;
  long long ps, pm;
  long long pad;
  __device__ __forceinline__ void add_to(long long& s, long long& m) const {
    s += ps;
    m += pm;
  }
};

// one arrival (32 bytes, one sector): edge x (the reference's arrival order
// within a step is ascending x), log position of the source spike, due step,
// row offset of x in the source's CSR row (drop bookkeeping), payload
template <typename T> struct Arrival;
template <> struct alignas(32) Arrival<float> {
  int x, tag, due, ro;
  long long p;
  long long pad;
};
template <> struct alignas(32) Arrival<double> {
  int x, tag, due, ro;
  long long ps, pm;
};

template <typename T>
struct BndArgs {
  FwdArgs<T> f;
  int cap;                    // events per queue (lossy ring: physical slots = min(capacity, horizon) + 1)
  int cap_ref;                // lossy ring: the reference's capacity (aliasing modulus)
  const long long* csc_off;   // [N+1] in-edge segment offsets
  long long E;
  Arrival<T>* alist;          // [2][B][E] arrival lists, target j at csc_off[j]
  int* acnt;                  // [2][B][N] arrivals per target
  QEv<T>* q;                  // [B*N][cap]
  int4* meta;                 // [B*N] {count, head|seq, tail_key, next_due}
  int maxdeg;                 // event id = log position * maxdeg + row offset
  unsigned* drop_bits;        // [drop_cap/32]
  long long drop_cap;
  int insert_first;           // first step whose arrivals this launch inserts
  // shared-memory staged queues (eq_bq.cuh, capacity <= kBqMaxCap)
  unsigned* keys;             // [B*N][C]
  void* pay;                  // [B*N][C] fixed-point payloads
  int C;                      // storage capacity (capacity rounded up to 4)
  int* qdue;                  // [B*N] next due step of each queue
  // owner inboxes (eq_bq.cuh): arrivals appended per owner CTA, counting-sorted by target
  void* inbox;                // [2][G][in_cap] InArr<T>
  int* in_cnt;                // [2][G]
  long long in_cap;
  int* aoff;                  // [B*N] end of each queue's arrival run in its CTA's sorted index
  int* aidx;                  // [G][in_cap] inbox positions sorted by target
  FastDiv divPer;             // flat target -> owner CTA
};

__device__ __forceinline__ bool key_less(int da, int sa, int db, int sb) {
  return da < db || (da == db && sa < sb);
}

// Per-target queues in HBM.  Every structure operation is a chain of
// dependent memory round trips, so the device structures are laid out to keep
// the chains short (the accepted sets and popped sums do not depend on the
// structure: pops sum fixed-point payloads, acceptance depends on the count):
//   heap    — min-heap on (due, insertion seq), 8-ary: a level's children are
//             8 adjacent entries read in one round trip, depth log8(cap);
//   sorted  — circular array, stable insertion (:351-366) (a chunked shift,
//             8 keys per round trip, measured no faster at capacity 64);
//   FIFO    — circular buffer, pops read 4 head entries per round trip.
constexpr int kHeapD = 8;

template <typename T>
__device__ __forceinline__ int2 qkey(const QEv<T>* p) {   // {tag, due}: the entry's first 8 bytes
  return *reinterpret_cast<const int2*>(p);
}

// Insert one event (reference order) into the owner's queue.
// Returns 0 accepted, 1 dropped (full), 2 capability error (FIFO order).
template <typename T>
__device__ __forceinline__ int queue_insert(int kind, int cap, QEv<T>* q, int4& mt, QEv<T> ev) {
  if (kind == EQ_KIND_FIFORING && ev.due < mt.z) return 2;      // queues.py:220-224
  if (mt.x == cap) return 1;                                     // :225-226, :514-515, :344-345
  if (kind == EQ_KIND_FIFORING) {
    int slot = mt.y + mt.x;
    if (slot >= cap) slot -= cap;
    q[slot] = ev;
    mt.x += 1;
    mt.z = ev.due;
    if (mt.x == 1) mt.w = ev.due;
  } else if (kind == EQ_KIND_BINARYHEAP) {
    ev.tag = mt.y++;                                             // insertion seq, :517-518
    int i = mt.x++;
    while (i > 0) {                                              // sift up (:522-528), 8-ary
      const int parent = (i - 1) / kHeapD;
      const QEv<T> pv = q[parent];
      if (!key_less(ev.due, ev.tag, pv.due, pv.tag)) break;
      q[i] = pv;
      i = parent;
    }
    q[i] = ev;
    mt.w = i == 0 ? ev.due : mt.w;
  } else {  // sorted array, circular with head mt.y; stable for equal due (:351-366)
    int k = mt.x;
    while (k > 0) {
      int pi = mt.y + k - 1;
      if (pi >= cap) pi -= cap;
      const QEv<T> pv = q[pi];
      if (pv.due <= ev.due) break;
      int di = pi + 1;
      if (di >= cap) di -= cap;
      q[di] = pv;
      --k;
    }
    int di = mt.y + k;
    if (di >= cap) di -= cap;
    q[di] = ev;
    mt.x += 1;
    if (k == 0) mt.w = ev.due;
  }
  return 0;
}

// Pop every event due at step `now` (the minimum), summing fixed-point payloads.
template <typename T>
__device__ __forceinline__ void queue_pop(int kind, int cap, QEv<T>* q, int4& mt, int now, long long& s,
                                          long long& mm) {
  if (mt.x == 0 || mt.w != now) return;
  if (kind == EQ_KIND_BINARYHEAP) {
    while (mt.x > 0 && q[0].due == now) {                        // :555-568
      q[0].add_to(s, mm);
      const int last = --mt.x;
      if (last > 0) {
        const QEv<T> item = q[last];
        int i = 0;
        while (true) {                                           // sift down (:541-551), 8-ary
          const int c0 = kHeapD * i + 1;
          if (c0 >= last) break;
          const int cn = last - c0 < kHeapD ? last - c0 : kHeapD;
          int2 kk[kHeapD];
#pragma unroll
          for (int e = 0; e < kHeapD; ++e) kk[e] = e < cn ? qkey(q + c0 + e) : make_int2(0x7fffffff, 0x7fffffff);
          int best = 0, bd = kk[0].y, bt = kk[0].x;
#pragma unroll
          for (int e = 1; e < kHeapD; ++e)
            if (key_less(kk[e].y, kk[e].x, bd, bt)) {
              best = e;
              bd = kk[e].y;
              bt = kk[e].x;
            }
          if (!key_less(bd, bt, item.due, item.tag)) break;
          q[i] = q[c0 + best];                                   // L1 hit: its line was just read
          i = c0 + best;
        }
        q[i] = item;
      }
    }
    mt.w = mt.x ? q[0].due : 0x7fffffff;
  } else {  // FIFO and sorted: due run at the head (:245-254, :378-386), 4 entries per round trip
    while (mt.x > 0) {
      const int nb = mt.x < 4 ? mt.x : 4;
      QEv<T> ev[4];
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        int pi = mt.y + e;
        if (pi >= cap) pi -= cap;
        if (e < nb) ev[e] = q[pi];
      }
      int taken = 0, next = 0x7fffffff;
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        if (e < nb && e == taken && ev[e].due == now) {
          ev[e].add_to(s, mm);
          ++taken;
        } else if (e < nb && e == taken) {
          next = ev[e].due;                                      // first entry not due: the new head
        }
      }
      mt.y += taken;
      if (mt.y >= cap) mt.y -= cap;
      mt.x -= taken;
      if (taken < nb) {
        mt.w = next;
        return;
      }
      if (nb < 4) break;                                         // emptied
    }
    mt.w = mt.x ? q[mt.y].due : 0x7fffffff;
  }
}

// Owner-side insertion of target j's `n` arrivals of step `ms` (parity ms & 1)
// in ascending x (= the reference's source order): each round takes the
// smallest x above the last one (the list is read once; rounds hit L1).
template <typename T>
__device__ __forceinline__ void insert_arrivals(const BndArgs<T>& A, int b, int j, int idx, int ms, int n,
                                                long long cs, int4& mt, unsigned long long& drops) {
  const Arrival<T>* lst = A.alist + ((size_t)(ms & 1) * A.f.B + b) * A.E + cs;
  QEv<T>* q = A.q + (size_t)idx * A.cap;
  int last_x = -1;
  for (int r = 0; r < n; ++r) {
    int best = -1, bx = 0x7fffffff;
    for (int k = 0; k < n; ++k) {
      const int x = lst[k].x;
      if (x > last_x && x < bx) {
        bx = x;
        best = k;
      }
    }
    last_x = bx;
    const Arrival<T> a = lst[best];
    QEv<T> ev;
    ev.tag = a.tag;
    ev.due = a.due;
    if constexpr (sizeof(T) == 4) {
      ev.p = a.p;
    } else {
      ev.ps = a.ps;
      ev.pm = a.pm;
      ev.pad = 0;
    }
    const int rc = queue_insert<T>(A.f.kind, A.cap, q, mt, ev);
    if (rc == 2) {
      raise_error(A.f.err, EQ_ERR_CAPABILITY, ms + 1, b, j);
    } else if (rc == 1) {
      drops += 1;
      const long long id = (long long)a.tag * A.maxdeg + a.ro;
      if (id < A.drop_cap) atomicOr(A.drop_bits + (id >> 5), 1u << (id & 31));
      else raise_error(A.f.err, EQ_ERR_CAPACITY, ms, b, j);
    }
  }
}

// Spike log of step m for this CTA (one chunk per (step, CTA)) and the fan-out
// of its crossings: every event of edge x -> target j is appended to j's
// arrival list for insertion by j's owner at phase m+1 (lossy ring: added
// straight into the target's slot).  Shared by the bounded-kind kernels.
template <typename T, int NT>
__device__ __forceinline__ void bounded_log_fanout(const BndArgs<T>& A, const int m, const int cta, const int tid,
                                                   const int nspk, const int b_first, SpikeRec<T>* s_spk,
                                                   long long* s_r0, int* s_pre, SpikeRec<T>* spill, long long& s_off,
                                                   unsigned (*s_ctr)[3]) {
  typedef Prec<T> P;
  constexpr int kCap = FwdShared<NT, T>::kCap;
  constexpr int kTr = FwdShared<NT>::kTrials;
  const FwdArgs<T>& F = A.f;
  const StepConsts<T>& c = F.c;
    // ---------------- spike log + event-id range for this (step, CTA)
    if (tid == 0) {
      unsigned long long off = nspk ? atomicAdd(F.log_count, (unsigned long long)nspk) : 0ULL;
      if (nspk && (long long)(off + nspk) > F.log_cap) {
        raise_error(F.err, EQ_ERR_CAPACITY, m, -1, -1);
        off = 0;
      }
      s_off = (long long)off;
      F.chunk_off[(size_t)m * F.G + cta] = (long long)off;
      F.chunk_cnt[(size_t)m * F.G + cta] = nspk;
    }
    __syncthreads();
    const bool log_ok = s_off + nspk <= F.log_cap;
    if (log_ok)
      for (int k = tid; k < nspk; k += NT) F.log[s_off + k] = k < kCap ? s_spk[k] : spill[k - kCap];
    // ---------------- fan-out: stage each event at its in-edge slot
    for (int k0 = 0; k0 < nspk; k0 += kCap) {
      const int nb = nspk - k0 < kCap ? nspk - k0 : kCap;
      __syncthreads();
      if (k0 > 0)
        for (int k = tid; k < nb; k += NT) s_spk[k] = spill[k0 - kCap + k];
      __syncthreads();
      for (int k = tid; k < nb; k += NT) {
        const int b = c.divN.div(s_spk[k].idx);
        const int i = s_spk[k].idx - b * F.N;
        const long long r0 = __ldg(F.net.rowptr + i);
        const int len = (int)(__ldg(F.net.rowptr + i + 1) - r0);
        s_r0[k] = r0;
        s_pre[k + 1] = len;
        if (log_ok) {
          F.log_r0[s_off + k0 + k] = r0;
          F.log_len[s_off + k0 + k] = len;
        }
        const int tb = b - b_first;
        if (tb < kTr) {
          atomicAdd(&s_ctr[tb][0], 1u);
          atomicAdd(&s_ctr[tb][1], (unsigned)len);
        } else {
          atomicAdd(reinterpret_cast<unsigned long long*>(F.counters + 3 * b), 1ULL);
          atomicAdd(reinterpret_cast<unsigned long long*>(F.counters + 3 * b + 1), (unsigned long long)len);
        }
      }
      __syncthreads();
      warp0_scan(s_pre, nb);
      __syncthreads();
      const int total = s_pre[nb];
      const int par = m & 1;
      // EV events in flight per thread: their edge-record loads, then their
      // slot atomics (the returned slots) are issued back to back
      constexpr int EV = 1;   // 2 or 3 in flight spill at the 64-register budget and
                              // measured slower (C4 heap[16] fwd 317 -> 345 ms at 2)
      for (int f0 = tid; f0 < total; f0 += EV * NT) {
        int kk[EV], jt[EV], ds[EV], ro[EV], bb[EV];
        long long xx[EV], q1[EV], q2[EV];
#pragma unroll
        for (int e = 0; e < EV; ++e) {
          const int f = f0 + e * NT;
          kk[e] = -1;
          if (f >= total) continue;
          const int k = find_row(s_pre, nb, f);
          kk[e] = k;
          ro[e] = f - s_pre[k];
          xx[e] = s_r0[k] + ro[e];
          const EdgeRec<T> ed = ld_edge(F.net.er + xx[e]);
          const SpikeRec<T> rec = s_spk[k];
          bb[e] = c.divN.div(rec.idx);
          jt[e] = ed.col;
          const T t_post = rec.t + ed.d;
          ds[e] = delivery_step_coded(t_post, (unsigned short)ed.code, c.dt, m);
          T ws, wm;
          if (F.exact) {
            const T phi = (T)ds[e] * c.dt - t_post;
            ws = ed.w * eq_exp_t(-phi * c.inv_tau_s);
            wm = ed.w * eq_exp_t(-phi * c.inv_tau_m);
          } else {
            ws = ed.w;
            wm = (T)0;
          }
          q1[e] = P::q(ws, c.scale);
          q2[e] = P::q(wm, c.scale);
        }
        if (F.kind == EQ_KIND_LOSSYRING) {
#pragma unroll
          for (int e = 0; e < EV; ++e) {
            if (kk[e] < 0) continue;
            // LossyRingQueue.enqueue (queues.py:160-176): slot = step % capacity,
            // i.e. the event is popped at the first step >= now = m+1 in its due
            // step's residue class; add straight into that slot (order-free fixed
            // point).  The ring has capacity+1 physical slots so slot m, popped
            // in this phase by other CTAs, is never a target here.
            int off = ds[e] - (m + 1);
            if (off >= A.cap_ref) off %= A.cap_ref;
            const int se = m + 1 + off;
            long long* sl = F.ring + ((size_t)bb[e] * A.cap + (size_t)(se % A.cap)) * F.N * P::kSlotWords +
                            (size_t)jt[e] * P::kSlotWords;
            if (P::kSlotWords == 1) {
              red_add(sl, pack2(q1[e], q2[e]));
            } else {
              red_add(sl, q1[e]);
              red_add(sl + 1, q2[e]);
            }
          }
          continue;
        }
        // append to the target's arrival list (slot from its counter; the
        // segment holds all in-edges, so it cannot overflow)
        int slot[EV];
        long long cs[EV];
#pragma unroll
        for (int e = 0; e < EV; ++e)
          if (kk[e] >= 0) {
            slot[e] = atomicAdd(A.acnt + ((size_t)par * F.B + bb[e]) * F.N + jt[e], 1);
            cs[e] = __ldg(A.csc_off + jt[e]);
          }
#pragma unroll
        for (int e = 0; e < EV; ++e) {
          if (kk[e] < 0) continue;
          Arrival<T> ar;
          ar.x = (int)xx[e];
          ar.tag = (int)(s_off + k0 + kk[e]);
          ar.due = ds[e];
          ar.ro = ro[e];
          if constexpr (sizeof(T) == 4) {
            ar.p = pack2(q1[e], q2[e]);
            ar.pad = 0;
          } else {
            ar.ps = q1[e];
            ar.pm = q2[e];
          }
          A.alist[((size_t)par * F.B + bb[e]) * A.E + cs[e] + slot[e]] = ar;
        }
      }
    }
}

template <typename T, int NT, int U>
__global__ void __launch_bounds__(NT, 2) k_forward_bounded(BndArgs<T> A) {
  typedef Prec<T> P;
  constexpr int kCap = FwdShared<NT, T>::kCap;
  constexpr int kTr = FwdShared<NT>::kTrials;
  __shared__ SpikeRec<T> s_spk[kCap];
  __shared__ long long s_r0[kCap];
  __shared__ int s_pre[kCap + 1];
  __shared__ int s_n;
  __shared__ long long s_off;
  __shared__ unsigned s_ctr[kTr][3];   // per-phase counts (32-bit: native smem atomics), flushed every phase
  FwdArgs<T>& F = A.f;

  const int tid = threadIdx.x;
  const int cta = blockIdx.x;
  const long long begin = (long long)cta * F.per;
  const long long end = begin + F.per < F.total ? begin + F.per : F.total;
  const int b_first = (int)(begin / F.N);
  const StepConsts<T> c = F.c;
  SpikeRec<T>* spill = F.scratch + (size_t)cta * F.per;
  if (tid < kTr * 3) (&s_ctr[0][0])[tid] = 0u;

  int m1 = F.m1;   // lowered at a barrier when the spike log could overflow (pause_due)
  for (int m = F.m0; m <= m1; ++m) {
    const bool last = (m == m1);   // extra pass: insert the final step's arrivals only
    if (tid == 0) s_n = 0;
    __syncthreads();
    if (!last) tl_mark(F.tl, m, F.G, cta, 0);
    // ---------------- owner phase: insert arrivals(m-1), pop(m), neuron update
    for (long long base = begin; base < end; base += NT) {
      const int idx = (int)base + tid;
      if (idx >= end) continue;
      const int b = c.divN.div(idx);
      const int j = idx - b * F.N;
      long long qs = 0, qm = 0;
      if (F.kind == EQ_KIND_LOSSYRING) {
        // LossyRingQueue._pop_raw (queues.py:109-120 via :178): read and zero
        // slot m of the target's ring; producers added into it directly
        if (last) continue;
        long long* sl = F.ring + ((size_t)b * A.cap + (size_t)(m % A.cap)) * F.N * P::kSlotWords + (size_t)j * P::kSlotWords;
        if (P::kSlotWords == 1) {
          unpack2(sl[0], qs, qm);
          sl[0] = 0;
        } else {
          qs = sl[0];
          qm = sl[1];
          sl[0] = 0;
          sl[1] = 0;
        }
      }
      const T I0 = F.I[idx], V0 = F.V[idx];
      int rf = F.refractory ? F.refr[idx] : 0;
      const bool drv = !last && drive_bit(F.net, b, m, j);
      const T ampj = __ldg(F.net.amp + j);
      if (F.kind != EQ_KIND_LOSSYRING) {
      // every load that does not depend on the queue first: one round trip
      int4 mt = A.meta[idx];
      const bool ins = m - 1 >= A.insert_first && m >= 1;
      int* cntp = A.acnt + ((size_t)((m - 1) & 1) * F.B + b) * F.N + j;
      const int narr = ins ? *cntp : 0;
      const long long acs = __ldg(A.csc_off + j);
      bool dirty = false;
      // the queue lines a step's inserts and pops will walk, fetched into L2
      // together: the structure's dependent chains then miss DRAM once
      auto prefetch_queue = [&](int qidx, const int4& qm, int qn) {
        // a full queue drops its arrivals without reading the structure:
        // only pops and accepting inserts walk its lines
        if ((qn > 0 && qm.x < A.cap) || (!last && qm.x > 0 && qm.w == m)) {
          const char* qb = reinterpret_cast<const char*>(A.q + (size_t)qidx * A.cap);
          const int span = qm.x + qn < A.cap ? qm.x + qn : A.cap;
          const int first = F.kind == EQ_KIND_BINARYHEAP ? 0 : qm.y;
          for (int e = 0; e < span; e += 128 / (int)sizeof(QEv<T>)) {
            int k = first + e;
            if (k >= A.cap) k -= A.cap;
            asm volatile("prefetch.global.L2 [%0];" ::"l"(qb + (size_t)k * sizeof(QEv<T>)));
          }
        }
      };
      // (prefetching the NEXT owned queue one iteration ahead measured slower:
      // C3 x 16 heap fwd 163 -> 188 ms, profiles/r1g_ab_prefetch_next.txt)
      prefetch_queue(idx, mt, narr);
      if (narr > 0) {
        {
          *cntp = 0;
          unsigned long long d = 0;
          insert_arrivals<T>(A, b, j, idx, m - 1, narr, acs, mt, d);
          const int tb = b - b_first;
          if (d) {
            if (tb < kTr) atomicAdd(&s_ctr[tb][2], (unsigned)d);
            else atomicAdd(reinterpret_cast<unsigned long long*>(F.counters + 3 * b + 2), d);
          }
          dirty = true;
        }
      }
      if (last) {
        if (dirty) A.meta[idx] = mt;
        continue;
      }
      if (mt.x > 0 && mt.w == m) {
        queue_pop<T>(F.kind, A.cap, A.q + (size_t)idx * A.cap, mt, m, qs, qm);
        dirty = true;
      }
      if (dirty) A.meta[idx] = mt;
      }
      T ps = P::deq(qs, c.inv_scale), pm = P::deq(qm, c.inv_scale);
      if (!F.exact) pm = (T)0;
      const T drive = drv ? ampj : (T)0;
      T i, v_new, a, v, t_spk;
      if (lif_step(c, F.exact != 0, F.refractory, m, ps, pm, I0, V0, drive, rf, i, v_new, a, v, t_spk)) {
        if (t_spk != t_spk) {
          raise_error(F.err, EQ_ERR_GRAZING, m + 1, b, j);
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
      F.I[idx] = i;
      F.V[idx] = v_new;
      if (F.refractory) F.refr[idx] = rf;
      if (F.v_trace) F.v_trace[(size_t)(m - F.m0) * F.total + idx] = v_new;
    }
    __syncthreads();
    if (last) break;
    tl_mark(F.tl, m, F.G, cta, 1);
    const int nspk = s_n;
    bounded_log_fanout<T, NT>(A, m, cta, tid, nspk, b_first, s_spk, s_r0, s_pre, spill, s_off, s_ctr);
    __syncthreads();
    flush_counters<kTr>(s_ctr, F.counters, b_first, F.B, end, F.N);
    tl_mark(F.tl, m, F.G, cta, 2);
    if (!grid_sync(F.bar, F.G, F.err, F.step_start + m + 1, F.log_count)) break;
    tl_mark(F.tl, m, F.G, cta, 3);
    if (ld_volatile(F.err) != 0) break;
    if (m + 1 < m1 && pause_due(F, m)) m1 = m + 1;
  }
  if (cta == 0 && tid == 0) F.err[4] = m1;
  // per-trial counters
  __syncthreads();
  if (tid < kTr) {
    int b = b_first + tid;
    if (b < F.B && (long long)b * F.N < end) {
      for (int q = 0; q < 3; ++q)
        if (s_ctr[tid][q]) atomicAdd(reinterpret_cast<unsigned long long*>(F.counters + 3 * b + q), (unsigned long long)s_ctr[tid][q]);
    }
  }
}

}  // namespace eq
