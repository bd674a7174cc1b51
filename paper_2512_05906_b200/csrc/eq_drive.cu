// eq_drive.cu — on-device PoissonDrive.
//
// The reference's drive (PoissonDrive, pkg/src/eventq/network.py:98-155):
// neuron i of a trial gets pulse trains defined in physical time,
//     t = Exp(mean_interval); while t < t_total: pulse [t, t + duration);
//                             t += duration + Exp(mean_interval)     (:113-120)
// sampled onto the step grid as active steps [ceil(s/dt), ceil(e/dt)) clipped
// to [0, T) (materialize, :138-143).  The reference draws the exponentials
// from numpy's sequential PCG64 stream, which cannot be split across threads;
// here every (trial, neuron) pair owns a counter-based Philox4x32-10 stream
// (Salmon et al., SC'11), so a warp generates 32 neurons' trains in parallel
// and writes the packed mask [B][T][ceil(n/32)] that eq_set_drive consumes —
// no T x n host materialisation and no host-to-device copy.  Same statistics
// as the reference's drive, not the same draws; the host-materialised mask
// stays the parity path.  oracle/eq_oracle.cpp restates this generator (its
// own Philox) bit for bit.
//
// Draw k of (trial b, neuron i): Philox call c = k >> 1 with counter
// {c, i, b, 0x5d0f1eed} and key {seed lo, seed hi}; words (w0, w1) give draw
// 2c and (w2, w3) draw 2c+1 as the 53-bit uniform
// u = ((wa >> 5) * 2^26 + (wb >> 6) + 0.5) * 2^-53 in (0, 1), and
// Exp = -mean_interval * eq_log(u) (include/eq_math.h, shared with the oracle).
#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/eq_math.h"
#include "../../include/eventq_b200.h"

namespace {

__device__ __forceinline__ void philox4x32_10(uint32_t ctr[4], uint32_t k0, uint32_t k1) {
  const uint32_t M0 = 0xD2511F53u, M1 = 0xCD9E8D57u, W0 = 0x9E3779B9u, W1 = 0xBB67AE85u;
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    const uint32_t lo0 = M0 * ctr[0], hi0 = __umulhi(M0, ctr[0]);
    const uint32_t lo1 = M1 * ctr[2], hi1 = __umulhi(M1, ctr[2]);
    const uint32_t n0 = hi1 ^ ctr[1] ^ k0, n2 = hi0 ^ ctr[3] ^ k1;
    ctr[0] = n0;
    ctr[1] = lo1;
    ctr[2] = n2;
    ctr[3] = lo0;
    k0 += W0;
    k1 += W1;
  }
}

__device__ __forceinline__ double u53(uint32_t a, uint32_t b) {
  return ((double)(a >> 5) * 67108864.0 + (double)(b >> 6) + 0.5) * (1.0 / 9007199254740992.0);
}

// The walk state of one neuron: current pulse [lo, hi) in steps and the next
// start time; draws come two per Philox call.
struct Walk {
  double t;       // start of the next pulse (physical time)
  int lo, hi;     // current pulse's active steps
  uint32_t call;  // next Philox call
  double spare;   // second exponential of the last call
  bool has_spare;
};

__device__ __forceinline__ double next_exp(Walk& w, uint32_t i, uint32_t b, uint32_t k0, uint32_t k1, double mean) {
  if (w.has_spare) {
    w.has_spare = false;
    return w.spare;
  }
  uint32_t c[4] = {w.call, i, b, 0x5d0f1eedu};
  philox4x32_10(c, k0, k1);
  w.call += 1;
  w.spare = -mean * eq_log(u53(c[2], c[3]));
  w.has_spare = true;
  return -mean * eq_log(u53(c[0], c[1]));
}

// One warp per (trial, 32-neuron mask word), lane = neuron within the word;
// a CTA of 32 warps covers 32 consecutive words and writes 32 steps at a time
// through a shared-memory tile as 128-byte row segments.  Pulses are generated
// kPulses at a time per lane, all lanes together (the per-pulse Philox + log
// would otherwise run one lane at a time inside the step loop), and consumed
// from a per-lane list as the steps advance.
constexpr int kTileSteps = 32;
constexpr int kPulses = 48;
__global__ void __launch_bounds__(1024) k_poisson_drive(int n, int B, int T, int words, double dt, double mean,
                                                        double dur, double t_total, uint32_t k0, uint32_t k1,
                                                        uint32_t* mask) {
  __shared__ uint32_t tile[kTileSteps][33];
  const int lane = threadIdx.x & 31, wp = threadIdx.x >> 5;
  const int wblocks = (words + 31) / 32;
  const int b = blockIdx.x / wblocks;
  const int wd0 = (blockIdx.x - b * wblocks) * 32;
  const int wd = wd0 + wp;
  const int i = wd * 32 + lane;
  const bool live = wd < words && i < n;
  Walk w;
  w.call = 0;
  w.has_spare = false;
  w.lo = w.hi = 0x7fffffff;
  w.t = live ? next_exp(w, (uint32_t)i, (uint32_t)b, k0, k1, mean) : t_total;
  int2 pl[kPulses];   // this lane's next pulses as active-step ranges
  int np = 0, pi = 0;
  auto refill = [&]() {   // up to kPulses more pulses (network.py:117-120, materialize :140-141)
    np = 0;
    pi = 0;
    while (np < kPulses && w.t < t_total) {
      const double s = w.t, e = s + dur;
      const int lo = (int)fmin(fmax(ceil(s / dt), 0.0), (double)T);
      const int hi = (int)fmin(fmax(ceil(e / dt), 0.0), (double)T);
      w.t = s + (dur + next_exp(w, (uint32_t)i, (uint32_t)b, k0, k1, mean));   // :118 t += dur + Exp
      if (hi > lo) pl[np++] = make_int2(lo, hi);   // pulses empty on the grid are never active
    }
  };
  refill();
  int lo = 0x7fffffff, hi = 0x7fffffff;
  if (np > 0) {
    lo = pl[0].x;
    hi = pl[0].y;
  }
  uint32_t* out = mask + (size_t)b * T * words;
  for (int m0 = 0; m0 < T; m0 += kTileSteps) {
    for (int mm = 0; mm < kTileSteps; ++mm) {
      const int m = m0 + mm;
      while (hi <= m) {                                    // next pulse of this lane
        if (++pi >= np) {
          if (w.t < t_total) refill();
          else np = 0;
          if (np == 0) {
            lo = hi = 0x7fffffff;
            break;
          }
        }
        lo = pl[pi].x;
        hi = pl[pi].y;
      }
      const bool on = live && lo <= m && m < hi;
      const unsigned bits = __ballot_sync(0xffffffffu, on);
      if (lane == 0) tile[mm][wp] = bits;
    }
    __syncthreads();
    const int mm = threadIdx.x >> 5, c = threadIdx.x & 31;
    if (m0 + mm < T && wd0 + c < words) out[(size_t)(m0 + mm) * words + wd0 + c] = tile[mm][c];
    __syncthreads();
  }
}

}  // namespace

extern "C" int eq_poisson_drive(int32_t n, int32_t n_trials, int32_t t_steps, double dt, double mean_interval,
                                double pulse_duration, uint64_t seed, uint32_t* mask_out, void* stream) {
  if (n < 1 || n_trials < 1 || t_steps < 1 || !(dt > 0.0) || !(mean_interval > 0.0) || !(pulse_duration >= 0.0) ||
      !mask_out)
    return EQ_ERR_CONFIGURATION;
  const int words = (n + 31) / 32;
  const long long grid = (long long)n_trials * ((words + 31) / 32);
  if (grid > 0x7fffffffLL) return EQ_ERR_CONFIGURATION;
  k_poisson_drive<<<(unsigned)grid, 1024, 0, (cudaStream_t)stream>>>(
      n, n_trials, t_steps, words, dt, mean_interval, pulse_duration, (double)t_steps * dt, (uint32_t)seed,
      (uint32_t)(seed >> 32), mask_out);
  return cudaGetLastError() == cudaSuccess ? EQ_OK : EQ_ERR_CUDA;
}
