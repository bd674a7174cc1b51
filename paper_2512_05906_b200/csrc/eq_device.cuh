// eq_device.cuh — device primitives shared by the EventQueues kernels.
//
// Everything here is sm_100a-only code (no arch dispatch).  The arithmetic that
// must agree bit-for-bit with the CPU oracle lives in include/eq_math.h and in
// the step helpers below, compiled with -fmad=false so no a*b+c is fused
// behind the source's back.
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

#include "../../include/eq_math.h"
#include "../../include/eventq_b200.h"

namespace eq {

constexpr int kWarp = 32;

// ---------------------------------------------------------------- precision

template <typename T> struct Prec;

// fp32: slot = one int64 holding two int32 fixed-point sums (membrane << 32 | synapse).
// q = rint(v * 2^F) and v = q * 2^-F are evaluated in float: scaling by a power
// of two is exact and |q| < 2^31, so they round exactly like the oracle's
// double-precision ldexp/llrint (no FP64 in the fp32 hot loops).
template <> struct Prec<float> {
  typedef float2 T2;
  static constexpr int kSlotWords = 1;
  __device__ __forceinline__ static long long q(float v, float scale) {
    return (long long)__float2int_rn(v * scale);
  }
  __device__ __forceinline__ static float deq(long long q, float inv) {
    return __int2float_rn((int)q) * inv;
  }
};
template <> struct Prec<double> {
  typedef double2 T2;
  static constexpr int kSlotWords = 2;
  __device__ __forceinline__ static long long q(double v, double scale) {
    return __double2ll_rn(v * scale);
  }
  __device__ __forceinline__ static double deq(long long q, double inv) {
    return __ll2double_rn(q) * inv;
  }
};

// n / d for 0 <= n < 2^31 without an integer divide: M = ceil(2^(31+L)/d),
// L = ceil(log2 d), q = (n*M) >> (31+L) (Granlund-Montgomery, exact here).
struct FastDiv {
  unsigned d, M, S;
  __host__ __device__ FastDiv() : d(1), M(1u << 31), S(31) {}
  __host__ explicit FastDiv(unsigned dd) : d(dd) {
    unsigned L = 0;
    while ((1ull << L) < dd) ++L;
    S = 31 + L;
    M = (unsigned)(((1ull << S) + dd - 1) / dd);
  }
  __device__ __forceinline__ int div(int n) const {
    return (int)(((unsigned long long)(unsigned)n * M) >> S);
  }
};

// pack/unpack the fp32 slot: P = qm * 2^32 + qs, summed mod 2^64; each field's
// true sum fits int32 by the frac-bits bound, so the low word sign-extends to qs.
__device__ __forceinline__ long long pack2(long long qs, long long qm) {
  return qm * 4294967296LL + qs;
}
__device__ __forceinline__ void unpack2(long long p, long long& qs, long long& qm) {
  int lo = (int)(unsigned int)(p & 0xffffffffLL);
  qs = lo;
  qm = (p - (long long)lo) >> 32;
}

// ---------------------------------------------------------------- memory

// Slot rows are written by other CTAs' red.add (at L2) in earlier phases; every
// phase starts after grid_sync's acquire fence, which invalidates L1, so plain
// (weak) accesses observe them.  __ldcg/__stcg compile to STRONG.GPU accesses on
// sm_100a and were 5x slower in the pop loop.
__device__ __forceinline__ long long ld_slot(const long long* p) { return *p; }
__device__ __forceinline__ void st_slot(long long* p, long long v) { *p = v; }

__device__ __forceinline__ unsigned ld_acquire(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release(unsigned* p, unsigned v) {
  asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ int ld_volatile(const int* p) { return *(volatile const int*)p; }
__device__ __forceinline__ unsigned long long globaltimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// Fire-and-forget reductions (no return value travels back to the SM).
__device__ __forceinline__ void red_add(long long* p, long long v) {
  asm volatile("red.relaxed.gpu.global.add.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ void red_add_f64(double* p, double v) {
  asm volatile("red.relaxed.gpu.global.add.f64 [%0], %1;" ::"l"(p), "d"(v) : "memory");
}

// error word: [0] code, [1] step, [2] trial, [3] neuron
__device__ __forceinline__ void raise_error(int* err, int code, int step, int trial, int neuron) {
  if (atomicCAS(err, 0, code) == 0) {
    err[1] = step;
    err[2] = trial;
    err[3] = neuron;
  }
}

__device__ __forceinline__ unsigned ld_relaxed(const unsigned* p) {
  unsigned v;
  asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ unsigned atom_add_acq_rel(unsigned* p, unsigned v) {
  unsigned old;
  asm volatile("atom.acq_rel.gpu.global.add.u32 %0, [%1], %2;" : "=r"(old) : "l"(p), "r"(v) : "memory");
  return old;
}
__device__ __forceinline__ void st_relaxed(unsigned* p, unsigned v) {
  asm volatile("st.relaxed.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ void fence_acq_rel_gpu() { asm volatile("fence.acq_rel.gpu;" ::: "memory"); }

// `bar` holds kBarWords words (only bar[0] is used by grid_sync; the rest
// keeps the word on its own 128-byte line).
constexpr unsigned kBarWords = 64;

// Grid barrier: one arrival atomic per CTA on a single word whose top bit
// flips when the last CTA arrives (CTA 0 adds 2^31 - (G-1), the others 1), a
// relaxed spin on that bit, one acquire fence.  1.2 us per barrier at 296 CTAs
// on B200 (scripts/micro/barrier.cu; a two-level tree with a separate release
// word took 3.2 us).  The CTA whose arrival flips the bit publishes
// *publish_src to *publish_dst AFTER the release, so readers of the published
// value spin on its sentinel (-1, see ld_published); the zero hooks run there too.
__device__ __forceinline__ bool grid_sync(unsigned* bar, unsigned nblocks, int* err,
                                          long long* publish_dst = nullptr,
                                          const unsigned long long* publish_src = nullptr,
                                          unsigned long long* zero_u64 = nullptr, int* zero_i32 = nullptr) {
  __shared__ int s_ok;
  __syncthreads();
  if (threadIdx.x == 0) {
    s_ok = 1;
    const unsigned inc = blockIdx.x == 0 ? 0x80000000u - (nblocks - 1) : 1u;
    const unsigned old = atom_add_acq_rel(bar, inc);
    if (((old ^ (old + inc)) & 0x80000000u) != 0) {        // this arrival completed the barrier
      if (publish_dst) *(volatile long long*)publish_dst = (long long)*(volatile const unsigned long long*)publish_src;
      if (zero_u64) *(volatile unsigned long long*)zero_u64 = 0ULL;
      if (zero_i32) *(volatile int*)zero_i32 = 0;
    } else {
      unsigned long long t0 = 0;
      int spins = 0;
      while (((ld_relaxed(bar) ^ old) & 0x80000000u) == 0) {
        if (++spins > 1024) {
          spins = 0;
          if (t0 == 0) t0 = globaltimer();
          else if (globaltimer() - t0 > 20000000000ULL) {   // 20 s watchdog
            atomicCAS(err, 0, EQ_ERR_CUDA);
            s_ok = 0;
            break;
          }
        }
      }
    }
    fence_acq_rel_gpu();
  }
  __syncthreads();
  return s_ok;
}

// A value published by grid_sync's last arriver (sentinel -1 until then).
__device__ __forceinline__ long long ld_published(const long long* p) {
  long long v;
  while ((v = *(volatile const long long*)p) == -1LL) {
  }
  return v;
}

template <typename T>
__device__ __forceinline__ T warp_sum_butterfly(T v) {
#pragma unroll
  for (int off = 16; off >= 1; off >>= 1) v = v + __shfl_xor_sync(0xffffffffu, v, off);
  return v;
}

// ---------------------------------------------------------------- step math
//
// Mirrors network.py:547-611 (PrimalRSNN.step) with the device-mode delivery
// clamp of oracle/eq_oracle.cpp::delivery.

// Exact-arithmetic bounds of ceil((t_spk + d)/dt) for t_spk in (m dt, (m+1) dt]:
// [m+1+floor(d/dt), m+1+ceil(d/dt)], a single value when d is grid-aligned
// (|d/dt - k| <= tol*k; tol 1e-5 in fp32, 1e-12 in fp64).  Clamping to them
// removes rounding artefacts of t_post/dt (fp32 near a step edge) that would
// otherwise move an event one step (spurious CapabilityError on the ring
// horizon, spurious FIFO order violations for homogeneous delays).
template <typename T>
__device__ __forceinline__ int delivery_step(T t_post, T d, T dt, int m) {
  const T tol = sizeof(T) == 4 ? (T)1e-5 : (T)1e-12;
  const T kd = d / dt;
  const T kr = rint(kd);
  int lo, hi;
  if (fabs(kd - kr) <= tol * (kr > (T)1 ? kr : (T)1)) {
    lo = hi = m + 1 + (int)kr;
  } else {
    lo = m + 1 + (int)floor(kd);
    hi = m + 1 + (int)ceil(kd);
  }
  int q = (int)ceil(t_post / dt);
  q = q < lo ? lo : (q > hi ? hi : q);
  return q > m + 2 ? q : m + 2;
}

// Per-edge delivery offset, precomputed once per network (eq_set_network):
// bit 15 set = delay not grid-aligned; bits 0..14 = m+1+floor(d/dt) - m (or
// the rounded value when aligned), i.e. the exact-arithmetic lower bound of
// dstep - m.  For an aligned delay dstep = m + max(lo, 2) with no division.
template <typename T>
__device__ __forceinline__ unsigned short delivery_code(T d, T dt) {
  const T tol = sizeof(T) == 4 ? (T)1e-5 : (T)1e-12;
  const T kd = d / dt;
  const T kr = rint(kd);
  if (fabs(kd - kr) <= tol * (kr > (T)1 ? kr : (T)1)) return (unsigned short)(1 + (int)kr);
  return (unsigned short)(0x8000 | (1 + (int)floor(kd)));
}

template <typename T>
__device__ __forceinline__ int delivery_step_coded(T t_post, unsigned short code, T dt, int m) {
  const int lo = m + (code & 0x7fff);
  int q = lo;
  if (code & 0x8000) {                   // not grid-aligned: ceil within [lo, lo + 1]
    q = (int)ceil(t_post / dt);
    q = q < lo ? lo : (q > lo + 1 ? lo + 1 : q);
  }
  return q > m + 2 ? q : m + 2;
}

// One packed record per CSR edge (built by eq_set_network): the fan-outs read
// a whole edge with one vector load instead of four scalar ones, so the loads
// of several events stay in flight without spilling (the 64-register budget
// of the 2-CTA/SM persistent kernels).  code = delivery_code(d, dt).
template <typename T>
struct EdgeRec;
template <>
struct alignas(16) EdgeRec<float> {
  int col;
  float w, d;
  int code;
};
template <>
struct alignas(8) EdgeRec<double> {
  int col;
  int code;
  double w, d;
};
__device__ __forceinline__ EdgeRec<float> ld_edge(const EdgeRec<float>* p) {
  const int4 v = __ldcs(reinterpret_cast<const int4*>(p));   // streamed once per event: evict-first
  EdgeRec<float> e;
  e.col = v.x;
  e.w = __int_as_float(v.y);
  e.d = __int_as_float(v.z);
  e.code = v.w;
  return e;
}
__device__ __forceinline__ EdgeRec<double> ld_edge(const EdgeRec<double>* p) {
  const int2 h = __ldcs(reinterpret_cast<const int2*>(p));
  EdgeRec<double> e;
  e.col = h.x;
  e.code = h.y;
  e.w = __ldcs(&p->w);
  e.d = __ldcs(&p->d);
  return e;
}

template <typename T>
struct alignas(16) SpikeRec;
template <>
struct alignas(16) SpikeRec<float> {
  int idx;      // trial * N + neuron
  float t, a, vh;
};
template <>
struct alignas(16) SpikeRec<double> {
  int idx;
  int pad;
  double t, a, vh;
};

}  // namespace eq
