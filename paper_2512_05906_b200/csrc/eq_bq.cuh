// eq_bq.cuh — the bounded queue kinds, FIFORing (queues.py:184-260),
// BinaryHeap (queues.py:481-571) and SortedArray (queues.py:308-403), as
// per-neuron queues STAGED IN SHARED MEMORY for each step's operations and
// kept in HBM between steps (capacities up to kBqMaxCap; larger ones use the
// HBM-resident structures of eq_bounded.cuh).
//
// Queue q = trial * N + j, storage capacity C (the capacity rounded up to 4):
//   keys[q][C]  uint32 (due mod 2^24) << 8 | slot   — the structure itself
//                (binary min-heap on due / circular sorted array / circular FIFO)
//   pay[q][C]   fixed-point payload of slot s (fp32: packed (qm << 32) + qs;
//                fp64: {qs, qm}); heap and sorted keep payloads in place and move
//                only 4-byte keys; FIFO's slot is its circular position
//   meta[q]     int4 {count | head << 16, next due, free-slot mask lo / FIFO tail
//                key, free-slot mask hi}
//
// Phase m, warp-cooperative: a warp takes a batch of L consecutive queues (one
// per lane).  The lanes whose queue will change this step (arrivals that can
// be accepted, or a pop due) copy its key array into the warp's shared-memory
// staging area with cp.async, all at once — one memory round trip for the
// batch instead of one per heap level / shifted entry — then insert the
// arrivals of step m-1 in ascending edge order (the reference's source order,
// with its accept-while-not-full rule: queues.py:225-226, :514-515, :344-345),
// pop every event due at m, sum the popped payloads (loaded in groups, not one
// dependent load per entry) and write the staged keys back.  A full queue
// drops its arrivals without being staged.  Because pops sum fixed-point
// payloads, ties among equal due steps may sit in any order: the accepted sets,
// popped sums and pending contents equal the reference's (tests/).
#pragma once

#include "eq_bounded.cuh"

namespace eq {

constexpr int kBqMaxCap = 64;         // largest capacity staged in shared memory
constexpr int kBqWarpWords = 1024;    // staging words per warp (4 KB)

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

struct BqState {
  int count, head, tail;      // tail: FIFO tail key (queues.py:220-224)
  unsigned long long mask;    // heap / sorted: occupied payload slots
};

__device__ __forceinline__ void bq_add(long long v, long long& qs, long long& qm) { qs += v; }
__device__ __forceinline__ void bq_add(longlong2 v, long long& qs, long long& qm) {
  qs += v.x;
  qm += v.y;
}

// Insert one event (called in reference order).  0 accepted, 1 dropped
// (full), 2 capability error (FIFO order).  The payload goes straight to HBM.
template <typename PT>
__device__ __forceinline__ int bq_insert(int kind, int cap, int C, unsigned* sk, BqState& st, int m, int due, PT p,
                                         PT* pay) {
  if (kind == EQ_KIND_FIFORING && due < st.tail) return 2;     // queues.py:220-224
  if (st.count == cap) return 1;                               // :225-226, :514-515, :344-345
  if (kind == EQ_KIND_FIFORING) {
    int pos = st.head + st.count;
    if (pos >= C) pos -= C;
    sk[pos] = bq_key(due, pos);
    pay[pos] = p;
    st.count += 1;
    st.tail = due;
    return 0;
  }
  const int slot = __ffsll((long long)~st.mask) - 1;           // a free slot: count < cap <= C <= 64
  st.mask |= 1ull << slot;
  pay[slot] = p;
  const unsigned key = bq_key(due, slot);
  const unsigned rk = bq_rel(key, m);
  if (kind == EQ_KIND_BINARYHEAP) {                            // sift up (queues.py:521-528)
    int i = st.count++;
    while (i > 0) {
      const int parent = (i - 1) >> 1;
      const unsigned pk = sk[parent];
      if (bq_rel(pk, m) <= rk) break;
      sk[i] = pk;
      i = parent;
    }
    sk[i] = key;
  } else {                                                     // sorted: insertion sweep (:351-366)
    int k = st.count;
    while (k > 0) {
      int pi = st.head + k - 1;
      if (pi >= C) pi -= C;
      const unsigned pk = sk[pi];
      if (bq_rel(pk, m) <= rk) break;
      int di = pi + 1;
      if (di >= C) di -= C;
      sk[di] = pk;
      --k;
    }
    int di = st.head + k;
    if (di >= C) di -= C;
    sk[di] = key;
    st.count += 1;
  }
  return 0;
}

// Pop every event due at m (the minimum); returns the popped slots.
__device__ __forceinline__ unsigned long long bq_pop(int kind, int C, unsigned* sk, BqState& st, int m) {
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
    st.mask &= ~popped;
  } else {                                                     // due run at the head (:245-254, :378-398)
    while (st.count > 0 && bq_rel(sk[st.head], m) == 0) {
      popped |= 1ull << bq_slot(sk[st.head]);
      st.head = st.head + 1 == C ? 0 : st.head + 1;
      st.count -= 1;
    }
    if (kind != EQ_KIND_FIFORING) st.mask &= ~popped;
  }
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

__device__ __forceinline__ int bq_next_due(int kind, const unsigned* sk, const BqState& st, int m) {
  if (st.count == 0) return 0x7fffffff;
  return m + (int)bq_rel(sk[kind == EQ_KIND_BINARYHEAP ? 0 : st.head], m);
}

template <typename T, int NT, int U>
__global__ void __launch_bounds__(NT, 2) k_forward_bq(BndArgs<T> A) {
  typedef Prec<T> P;
  typedef typename BqPay<T>::type PT;
  constexpr int kCap = FwdShared<NT, T>::kCap;
  constexpr int kTr = FwdShared<NT>::kTrials;
  constexpr int NW = NT / 32;
  __shared__ SpikeRec<T> s_spk[kCap];
  __shared__ long long s_r0[kCap];
  __shared__ int s_pre[kCap + 1];
  __shared__ int s_n;
  __shared__ long long s_off;
  __shared__ unsigned long long s_ctr[kTr][3];
  extern __shared__ __align__(16) unsigned s_keys[];   // [NW][kBqWarpWords] staging
  const FwdArgs<T>& F = A.f;

  const int tid = threadIdx.x;
  const int cta = blockIdx.x;
  const int warp = tid >> 5, lane = tid & 31;
  const long long begin = (long long)cta * F.per;
  const long long end = begin + F.per < F.total ? begin + F.per : F.total;
  const int b_first = (int)(begin / F.N);
  const StepConsts<T> c = F.c;
  SpikeRec<T>* spill = F.scratch + (size_t)cta * F.per;
  const int C = A.C, L = A.lanes, kind = F.kind;
  unsigned* const sk = s_keys + warp * kBqWarpWords + lane * C;
  PT* const payb = reinterpret_cast<PT*>(A.pay);
  if (tid < kTr * 3) (&s_ctr[0][0])[tid] = 0ULL;

  int m1 = F.m1;   // lowered at a barrier when the spike log could overflow (pause_due)
  for (int m = F.m0; m <= m1; ++m) {
    const bool last = (m == m1);   // extra pass: insert the final step's arrivals only
    if (tid == 0) s_n = 0;
    __syncthreads();
    if (!last) tl_mark(F.tl, m, F.G, cta, 0);
    const bool ins = m - 1 >= A.insert_first && m >= 1;
    // ---------------- owner phase, one batch of L consecutive queues per warp
    for (long long base = begin + (long long)warp * L; base < end; base += (long long)NW * L) {
      const long long qi = base + lane;
      const bool act = lane < L && qi < end;
      const int idx = (int)qi;
      int b = 0, j = 0, narr = 0, rf = 0;
      int4 mt = make_int4(0, 0x7fffffff, 0, 0);
      int* cntp = nullptr;
      T I0 = (T)0, V0 = (T)0, ampj = (T)0;
      bool drv = false;
      if (act) {                                    // independent loads of the lane: one round trip
        b = c.divN.div(idx);
        j = idx - b * F.N;
        mt = A.meta[idx];
        cntp = A.acnt + ((size_t)((m - 1) & 1) * F.B + b) * F.N + j;
        narr = ins ? *cntp : 0;
        if (!last) {
          I0 = F.I[idx];
          V0 = F.V[idx];
          rf = F.refractory ? F.refr[idx] : 0;
          drv = drive_bit(F.net, b, m, j);
          ampj = __ldg(F.net.amp + j);
        }
      }
      BqState st;
      st.count = mt.x & 0xffff;
      st.head = (int)((unsigned)mt.x >> 16);
      st.tail = kind == EQ_KIND_FIFORING ? mt.z : 0;
      st.mask = kind == EQ_KIND_FIFORING ? 0ull
                                         : ((unsigned long long)(unsigned)mt.w << 32) | (unsigned long long)(unsigned)mt.z;
      const bool pop_due = act && !last && st.count > 0 && mt.y == m;
      const bool can_ins = narr > 0 && st.count < A.cap;
      const unsigned* gk = A.keys + (size_t)idx * C;
      if (pop_due || can_ins)                       // stage the key array (all lanes' copies in flight at once)
        for (int k = 0; k < C; k += 4) cp_async16(sk + k, gk + k);
      cp_async_wait_all();
      bool dirty = false;
      PT* const pay = payb + (size_t)idx * C;
      if (narr > 0) {
        *cntp = 0;
        unsigned long long drops = 0;
        const Arrival<T>* lst = A.alist + ((size_t)((m - 1) & 1) * F.B + b) * A.E + __ldg(A.csc_off + j);
        int last_x = -1;
        for (int r = 0; r < narr; ++r) {             // ascending x = the reference's arrival order
          int best = 0;
          if (can_ins) {
            int bx = 0x7fffffff;
            for (int k = 0; k < narr; ++k) {
              const int x = lst[k].x;
              if (x > last_x && x < bx) {
                bx = x;
                best = k;
              }
            }
            last_x = bx;
          } else {
            best = r;                                // full queue: order only matters for FIFO's error
          }
          const Arrival<T> a = lst[best];
          PT p;
          if constexpr (sizeof(T) == 4) p = a.p;
          else p = make_longlong2(a.ps, a.pm);
          int rc;
          if (can_ins) {
            rc = bq_insert<PT>(kind, A.cap, C, sk, st, m, a.due, p, pay);
            dirty = true;
          } else {
            rc = (kind == EQ_KIND_FIFORING && a.due < st.tail) ? 2 : 1;
          }
          if (rc == 2) {
            raise_error(F.err, EQ_ERR_CAPABILITY, m, b, j);
          } else if (rc == 1) {
            drops += 1;
            const long long id = (long long)a.tag * A.maxdeg + a.ro;
            if (id < A.drop_cap) atomicOr(A.drop_bits + (id >> 5), 1u << (id & 31));
            else raise_error(F.err, EQ_ERR_CAPACITY, m - 1, b, j);
          }
        }
        if (drops) {
          const int tb = b - b_first;
          if (tb < kTr) atomicAdd(&s_ctr[tb][2], drops);
          else atomicAdd(reinterpret_cast<unsigned long long*>(F.counters + 3 * b + 2), drops);
        }
      }
      long long qs = 0, qm = 0;
      if (pop_due) {
        const unsigned long long popped = bq_pop(kind, C, sk, st, m);
        bq_sum<PT>(popped, pay, qs, qm);
        dirty = true;
      }
      if (dirty) {
        unsigned* gkw = const_cast<unsigned*>(gk);
        for (int k = 0; k < C; k += 4)
          *reinterpret_cast<uint4*>(gkw + k) = *reinterpret_cast<const uint4*>(sk + k);
        int4 o;
        o.x = st.count | (st.head << 16);
        o.y = bq_next_due(kind, sk, st, m);
        o.z = kind == EQ_KIND_FIFORING ? st.tail : (int)(unsigned)(st.mask & 0xffffffffull);
        o.w = kind == EQ_KIND_FIFORING ? 0 : (int)(unsigned)(st.mask >> 32);
        A.meta[idx] = o;
      }
      if (!act || last) continue;
      if (P::kSlotWords == 1) {
        const long long packed = qs;
        unpack2(packed, qs, qm);
      }
      T ps = P::deq(qs, c.inv_scale), pm = P::deq(qm, c.inv_scale);
      if (!F.exact) pm = (T)0;
      const T drive = drv ? ampj : (T)0;
      T i, v_new, a, v, t_spk;
      if (lif_step(c, F.exact != 0, F.refractory, m, ps, pm, I0, V0, drive, rf, i, v_new, a, v, t_spk)) {
        if (t_spk != t_spk) {
          raise_error(F.err, EQ_ERR_GRAZING, m + 1, b, j);
        } else {
          const int pos = atomicAdd(&s_n, 1);
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
        if (s_ctr[tid][q]) atomicAdd(reinterpret_cast<unsigned long long*>(F.counters + 3 * b + q), s_ctr[tid][q]);
    }
  }
}

__global__ void k_meta_init_bq(int4* meta, long long n, int fifo) {
  for (long long k = blockIdx.x * (long long)blockDim.x + threadIdx.x; k < n; k += (long long)gridDim.x * blockDim.x)
    meta[k] = make_int4(0, 0x7fffffff, fifo ? -1 : 0, 0);   // FIFORingQueue._tail_key = -1
}

// Pending contents (canonical int64 [B*N][H][2], due now .. now+H-1).
template <typename T>
__global__ void k_pending_bq(const unsigned* keys, const typename BqPay<T>::type* pay, const int4* meta, int kind,
                             int C, long long total, int H, int now, long long* out) {
  for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < total;
       idx += (long long)gridDim.x * blockDim.x) {
    long long* o = out + idx * H * 2;
    for (int k = 0; k < 2 * H; ++k) o[k] = 0;
    const int4 mt = meta[idx];
    const int count = mt.x & 0xffff, head = (int)((unsigned)mt.x >> 16);
    for (int k = 0; k < count; ++k) {
      int pos = k;
      if (kind != EQ_KIND_BINARYHEAP) {
        pos = head + k;
        if (pos >= C) pos -= C;
      }
      const unsigned key = keys[idx * C + pos];
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
