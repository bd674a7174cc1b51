// eventq.cu — the C ABI (include/eventq_b200.h) over the sm_100a kernels.
//
// Host code only orchestrates: validation of the network on the device
// (reference checks of build_rsnn, network.py:213-268), buffer ownership, and
// one cooperative launch of a persistent kernel per eq_run / eq_backward.
#include <cuda_runtime.h>

#include <algorithm>
#include <array>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "eq_device.cuh"
#include "eq_ring.cuh"
#include "eq_bounded.cuh"
#include "eq_bq.cuh"
#include "eq_jvp.cuh"

#include <cub/cub.cuh>

using namespace eq;

namespace {

constexpr int kNT = 512;   // threads per CTA of the persistent kernels
constexpr int kErrWords = 8;  // device error word: [0] code, [1] step, [2] trial, [3] neuron, [4] step reached
constexpr int kU = 4;      // neurons per thread in flight per round
#ifndef EQ_SPLIT_F32
#define EQ_SPLIT_F32 320
#endif
#ifndef EQ_SPLIT_F32_HBM
#define EQ_SPLIT_F32_HBM 288
#endif
// forward event-side threads per CTA (fp32): 320 with the neuron state in shared
// memory and for the admission kinds, 288 for the ring with its state in HBM
// (the neuron side is heavier there): C3 x 24 fwd 32.62 -> 32.13 ms, C4 ring
// 76.10 at 288 vs 77.34 at 320 (profiles/r2bi_ab_fp32_split.txt)
constexpr int kSplitF = EQ_SPLIT_F32;
constexpr int kSplitFHbm = EQ_SPLIT_F32_HBM;
#ifndef EQ_SPLIT_B32
#define EQ_SPLIT_B32 352
#endif
constexpr int kSplitB = EQ_SPLIT_B32;  // reverse event-side threads per CTA (measured: 224..448, profiles/)
constexpr size_t kStateSmem = 72 * 1024;   // forward state in shared memory up to this size per CTA
// fp64 warp-group splits (event side / neuron side), measured per pass
#ifndef EQ_SPLIT_F64
#define EQ_SPLIT_F64 320   // fp64 forward event-side threads: 288 -> 320: fwd 76.5-77.1 -> 76.1-76.2 ms (profiles/r2bd_ab_fp64_split.txt)
#endif
#ifndef EQ_SPLIT_B64
#define EQ_SPLIT_B64 320   // 256 -> 288 with EV 2: fp64 bwd 59.6-61.1 -> 59.1 ms (profiles/r1h_ab_4.txt); 288 -> 320: 60.9 -> 60.2 ms (profiles/r2bf_ab_fp64_reverse_split.txt)
#endif
template <typename T> constexpr int split_f() { return sizeof(T) == 4 ? kSplitF : EQ_SPLIT_F64; }
template <typename T> constexpr int split_f_hbm() { return sizeof(T) == 4 ? kSplitFHbm : EQ_SPLIT_F64; }
template <typename T> constexpr int split_b() { return sizeof(T) == 4 ? kSplitB : EQ_SPLIT_B64; }


struct DeviceGuard {
  int prev = -1;
  explicit DeviceGuard(int dev) {
    cudaGetDevice(&prev);
    if (prev != dev) cudaSetDevice(dev);
  }
  ~DeviceGuard() {
    int cur = -1;
    cudaGetDevice(&cur);
    if (prev >= 0 && cur != prev) cudaSetDevice(prev);
  }
};

}  // namespace

struct eq_handle {
  eq_config cfg{};
  std::string err;
  int device = 0;
  int n_sm = 0;
  int G = 0;
  long long total = 0, per = 0;
  int horizon = 0, R = 0, frac_bits = 0;
  double scale = 1.0, inv_scale = 1.0;
  int64_t E = 0;
  const int64_t* rowptr = nullptr;
  const int32_t* col = nullptr;
  const void* w = nullptr;
  const void* d = nullptr;
  const uint32_t* mask = nullptr;
  const void* amp = nullptr;
  unsigned short* dcode = nullptr;   // per-edge delivery codes
  void* edges = nullptr;             // packed EdgeRec<T>[E] (snapshot of col/w/d at eq_set_network)
  bool net_set = false, drive_set = false;
  size_t tsize = 4;
  // forward state
  void* I = nullptr;
  void* V = nullptr;
  int32_t* refr = nullptr;
  long long* ring = nullptr;
  size_t ring_words = 0;
  bool ring_clean = false;   // false: the next reset clears the whole ring (fresh buffer, or a JVP run used it)
  // calendar (ring kind)
  long long* acc = nullptr;
  long long* bk = nullptr;
  int* bk_cnt = nullptr;
  long long cap_b = 0;
  long long cap_b_alloc = 0;   // cap_b the bucket storage was sized for
  int NB = 0;
  int* ring_dirty = nullptr;
  void* scratch = nullptr;
  void* log = nullptr;
  long long* log_r0 = nullptr;
  int* log_len = nullptr;
  long long log_cap = 0;
  long long log_used = 0;      // host copy of *log_count after the last forward launch
  int log_grows = 0;           // spike-log reallocations (eq_run resumed after each)
  unsigned long long* log_count = nullptr;
  long long* chunk_off = nullptr;
  int* chunk_cnt = nullptr;
  long long* step_start = nullptr;   // [t_cap + 1]
  int t_cap = 0;
  long long* counters = nullptr;
  int* err_dev = nullptr;
  unsigned* bar = nullptr;
  // reverse state
  void* lamV = nullptr;
  void* lamI = nullptr;
  void* lam = nullptr;
  void* lt_log = nullptr;
  double* gamp_bt = nullptr;
  // bounded kinds (fifo / heap / sorted)
  bool bounded = false;
  // lossy ring: run by the bounded kernel's step structure (an event may pop
  // one step after its emission), slots in `ring` as [B][lossy_slots][N]
  bool lossy = false;
  int lossy_slots = 0;         // physical slots: min(capacity, horizon) + 1
  long long lossy_cap = 0;     // the reference's capacity (aliasing modulus)
  int cap = 0;                 // physical events per queue
  long long cap_ref = 0;       // the reference's capacity (acceptance rule)
  long long* csc_off = nullptr;
  void* alist = nullptr;       // [2][B][E] arrival lists (Arrival<T>)
  int* acnt = nullptr;         // [2][B][N] arrivals per target
  void* q = nullptr;
  int4* meta = nullptr;
  bool staged = false;         // capacity <= kBqMaxCap: shared-memory staged queues (eq_bq.cuh)
  int C = 0;                   // their storage capacity
  unsigned* qkeys = nullptr;
  void* qpay = nullptr;
  int* qdue = nullptr;
  void* inbox = nullptr;       // [2][G][in_cap] owner inboxes
  int* in_cnt = nullptr;       // [2][G]
  long long in_cap = 0;        // max over CTAs of the in-degree sum of its queues (lossless bound)
  int* aoff = nullptr;         // [B*N]
  int* aidx = nullptr;         // [G][in_cap]
  int maxdeg = 1;               // largest CSR row (bounded kinds: event id = log position * maxdeg + row offset)
  // binaryheap / sortedarray by admission (eq_ring.cuh "admission"): the calendar
  // path plus one admission record per queue; `cal` = the calendar path runs
  bool adm = false;
  bool cal = false;
  void* adm_ctr = nullptr;      // aw [2][totp] int32, ac [2][totp] u16, aa [3][totp] u16
  long long totp = 0;
  int* fl = nullptr;            // [2][G][per]
  int* fl_cnt = nullptr;        // [2][G]
  int* lpos = nullptr;          // [3][total]
  int2* csc = nullptr;          // [E] {x, source} by target, ascending x
  unsigned long long csc_fp[2] = {0, 0};   // topology fingerprint the CSC was built for
  long long csc_E = -1;
  int2* slots = nullptr;        // [2][total][kAdmSlots]
  int adm_slots = kAdmSlots;    // eq_debug_set_admission_slots
  int* cring = nullptr;         // [B][R][N] counts of the DRAM ring rows
  unsigned* drop_bits = nullptr;
  long long drop_cap = 0;
  unsigned long long* tl_f = nullptr;   // debug timelines (EQ_TIMELINE=1)
  unsigned long long* tl_b = nullptr;
  int tl_steps = 0;
  int steps_done = 0;
  long long launches = 0;
  // partitioned network (eq_set_partition): CSR rows are all n_src sources,
  // columns the n_neurons owned targets; owned neuron j is source src_off + j
  int n_src = 0, src_off = 0;
  bool partitioned = false;
  int frac_safe = 0;                  // largest overflow-free fraction bits of this network
  void* imp = nullptr;                // imported spikes of all windows (SpikeRec)
  long long* imp_r0 = nullptr;
  int* imp_len = nullptr;
  void* imp_lt = nullptr;             // partial dL/dt_spk of each imported spike (reverse)
  long long imp_cap = 0, imp_n = 0;
  std::vector<std::array<long long, 4>> imp_blocks;   // {forward launch start step, first, count, fanned out}
  void* lt_rem = nullptr;             // [log_cap] other partitions' dL/dt_spk of own spikes
  // device-resident peer exchange (eq_set_peers): the partitions read each
  // other's spike logs and import-adjoint blocks directly (same GPU, or peers
  // with P2P access over NVLink); no host round trip per window
  bool peer_mode = false;
  int peer_me = -1;
  std::vector<eq_handle*> peers;
  long long* peer_blk = nullptr;      // [t_cap + 2][2] {first, count} of import block w
  long long* peer_count = nullptr;    // imports so far (device)
  // reverse pass in windows (eq_backward_begin / eq_backward_window)
  int bwd_cursor = -1;
  double* bw_gw = nullptr;
  double* bw_gd = nullptr;
  double* bw_gamp = nullptr;
  void* jvp_buf[24] = {};                         // eq_forward_jvp scratch
  void *ns_insum = nullptr, *ns_inocc = nullptr, *ns_indeg = nullptr, *ns_stats = nullptr;   // eq_set_network scratch
  std::vector<void*> owned;
  std::vector<std::pair<void*, size_t>> sizes;   // reusable buffers
};

namespace {

int fail(eq_handle* h, int code, const std::string& msg) {
  if (h) h->err = msg;
  return code;
}

int cuda_fail(eq_handle* h, cudaError_t e, const char* what) {
  return fail(h, EQ_ERR_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
}

#define EQ_CUDA(h, call)                                   \
  do {                                                     \
    cudaError_t _e = (call);                               \
    if (_e != cudaSuccess) return cuda_fail((h), _e, #call); \
  } while (0)

cudaError_t alloc(eq_handle* h, void** p, size_t bytes) {
  *p = nullptr;
  if (bytes == 0) bytes = 16;
  cudaError_t e = cudaMalloc(p, bytes);
  if (e == cudaSuccess) h->owned.push_back(*p);
  return e;
}

void release(eq_handle* h, void* p) {
  if (!p) return;
  cudaFree(p);
  h->owned.erase(std::remove(h->owned.begin(), h->owned.end(), p), h->owned.end());
  h->sizes.erase(std::remove_if(h->sizes.begin(), h->sizes.end(),
                                [p](const std::pair<void*, size_t>& e) { return e.first == p; }),
                 h->sizes.end());
}

// Keep *p if it already holds >= bytes (set_network is called every training
// step by the autograd shell; cudaMalloc/free per call would dominate).
cudaError_t ensure(eq_handle* h, void** p, size_t bytes) {
  if (*p) {
    for (auto& e : h->sizes)
      if (e.first == *p && e.second >= bytes) return cudaSuccess;
    release(h, *p);
    *p = nullptr;
  }
  cudaError_t e = alloc(h, p, bytes);
  if (e == cudaSuccess) h->sizes.push_back({*p, bytes});
  return e;
}

template <typename T>
constexpr int P_words() { return Prec<T>::kSlotWords; }

template <typename T>
StepConsts<T> consts(const eq_handle* h) {
  const eq_config& c = h->cfg;
  StepConsts<T> k;
  k.dt = (T)c.dt;
  k.tau_m = (T)c.tau_m;
  k.tau_s = (T)c.tau_syn;
  k.v_th = (T)c.v_th;
  k.v_reset = (T)c.v_reset;
  // computed in double with libm and rounded once, exactly as the reference
  // computes them (network.py:527-528, 183-185) and as the oracle does
  k.k_m = (T)std::exp(-c.dt / c.tau_m);
  k.k_s = (T)std::exp(-c.dt / c.tau_syn);
  k.cc = c.exact_delivery ? (T)(c.tau_syn / (c.tau_m - c.tau_syn)) : (T)0;
  k.cm = c.exact_delivery ? k.cc : (T)-1;
  k.inv_tau_m = (T)(1.0 / c.tau_m);
  k.inv_tau_s = (T)(1.0 / c.tau_syn);
  k.scale = (T)std::ldexp(1.0, h->frac_bits);
  k.inv_scale = (T)std::ldexp(1.0, -h->frac_bits);
  k.divN = FastDiv((unsigned)h->cfg.n_neurons);
  return k;
}

template <typename T>
NetView<T> netview(const eq_handle* h) {
  NetView<T> n;
  n.rowptr = h->rowptr;
  n.col = h->col;
  n.w = (const T*)h->w;
  n.d = (const T*)h->d;
  n.dcode = h->dcode;
  n.er = (const EdgeRec<T>*)h->edges;
  n.mask = h->mask;
  n.amp = (const T*)h->amp;
  n.words = (h->cfg.n_neurons + 31) / 32;
  n.t_mask = h->cfg.t_steps;
  return n;
}

// ------------------------------------------------------------ small kernels

// Network validation + statistics, one thread per source row.
// stats[0] = max ceil(d/dt); stats[1] = first bad edge (flat index) << 2 | code
// of that ConfigurationError; stats[4] = longest row; insum = fixed-point
// sum of |w| per target (2^-40 units; deterministic integer adds).
template <typename T>
__global__ void k_net_stats(int n_rows, int N, int src_off, const int64_t* rowptr, const int32_t* col, const T* w,
                            const T* d, T dt, int homogeneous_only, long long* insum, long long* stats,
                            long long* inocc, int* indeg) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n_rows) return;
  long long r0 = rowptr[i], r1 = rowptr[i + 1];
  int hmax = 1;
  T d0 = d[0];
  int prev = -1;
  for (long long x = r0; x < r1; ++x) {
    int j = col[x];
    int code = 0;
    if (j < 0 || j >= N || j + src_off == i || j <= prev) code = 1;
    else if (!(d[x] >= dt)) code = 2;
    else if (homogeneous_only && d[x] != d0) code = 3;
    if (code) {
      // smallest offending edge wins: reference loops i, j row-major (network.py:225-240)
      unsigned long long key = ((unsigned long long)x << 2) | (unsigned long long)code;
      atomicMin(reinterpret_cast<unsigned long long*>(stats + 1), key);
      return;
    }
    prev = j;
    int q = (int)ceil(d[x] / dt);
    hmax = q > hmax ? q : hmax;
    atomicAdd(reinterpret_cast<unsigned long long*>(inocc + j), (unsigned long long)(q + 1));
    atomicAdd(indeg + j, 1);
    atomicAdd(reinterpret_cast<unsigned long long*>(insum + j),
              (unsigned long long)__double2ll_rn(fabs((double)w[x]) * 1099511627776.0));
  }
  atomicMax(stats, (long long)hmax);
  atomicMax(stats + 4, (long long)(r1 - r0));
}

template <typename T>
__global__ void k_pack_edges(const int32_t* col, const T* w, const T* d, long long E, T dt, unsigned short* code,
                             EdgeRec<T>* out) {
  for (long long x = blockIdx.x * (long long)blockDim.x + threadIdx.x; x < E; x += (long long)gridDim.x * blockDim.x) {
    const unsigned short cd = delivery_code(d[x], dt);
    code[x] = cd;
    EdgeRec<T> e;
    e.col = col[x];
    e.w = w[x];
    e.d = d[x];
    e.code = cd;
    out[x] = e;
  }
}

// Topology fingerprint of a CSR column array: sum of (x+1)*col[x] and of
// col[x]*col[x] (wrapping): the admission kinds rebuild their CSC only when it
// changes (set_network runs every training step with new weights and delays).
__global__ void k_col_fingerprint(const int32_t* col, long long n, unsigned long long* out) {
  unsigned long long a = 0, b = 0;
  for (long long x = blockIdx.x * (long long)blockDim.x + threadIdx.x; x < n; x += (long long)gridDim.x * blockDim.x) {
    const unsigned long long c = (unsigned long long)(unsigned)col[x];
    a += (unsigned long long)(x + 1) * (c + 1);
    b += (c + 7) * (c + 7);
  }
  for (int off = 16; off; off >>= 1) {
    a += __shfl_xor_sync(0xffffffffu, a, off);
    b += __shfl_xor_sync(0xffffffffu, b, off);
  }
  if ((threadIdx.x & 31) == 0) {
    atomicAdd(out, a);
    atomicAdd(out + 1, b);
  }
}

template <typename E>
__global__ void k_max_ll(const E* a, long long n, long long* out) {
  long long best = 0;
  for (long long k = blockIdx.x * (long long)blockDim.x + threadIdx.x; k < n;
       k += (long long)gridDim.x * blockDim.x)
    best = a[k] > best ? a[k] : best;
  for (int off = 16; off; off >>= 1) {
    long long o = __shfl_xor_sync(0xffffffffu, best, off);
    best = o > best ? o : best;
  }
  if ((threadIdx.x & 31) == 0) atomicMax(out, best);
}

template <typename T>
__global__ void k_fill(T* p, long long n, T v) {
  for (long long k = blockIdx.x * (long long)blockDim.x + threadIdx.x; k < n;
       k += (long long)gridDim.x * blockDim.x)
    p[k] = v;
}

template <typename T>
__global__ void k_sum_trials(const double* bt, int B, int N, double* out) {
  int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= N) return;
  double s = 0.0;
  for (int b = 0; b < B; ++b) s += bt[(size_t)b * N + j];
  out[j] = s;
}

template <typename T>
__global__ void k_decode_spikes(const SpikeRec<T>* log, const long long* chunk_off, const int* chunk_cnt,
                                int n_chunks, int G, int N, int32_t* step, int32_t* trial,
                                int32_t* neuron, T* t) {
  int wid = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  int lane = threadIdx.x & 31;
  if (wid >= n_chunks) return;
  long long off = chunk_off[wid];
  int cnt = chunk_cnt[wid];
  int m = wid / G;
  for (int k = lane; k < cnt; k += 32) {
    SpikeRec<T> r = log[off + k];
    step[off + k] = m;
    trial[off + k] = r.idx / N;
    neuron[off + k] = r.idx % N;
    if (t) t[off + k] = r.t;
  }
}

// Calendar ring contents pending after a run at step `now`: acc[now&1] holds
// due `now`, acc[(now+1)&1] due now+1, the CTAs' buckets (now+h)%NB due now+h
// (h >= 2), plus flagged DRAM ring rows (bucket overflow).  out int64 [B*N][H][2].
template <typename T>
__global__ void k_pending_calendar(const long long* acc, const long long* bk,
                                   const int* bk_cnt, long long cap_b, int NB, int G, const long long* ring,
                                   const int* ring_dirty, int B, int R, int N, int H, int now, long long* out) {
  const int W = Prec<T>::kSlotWords;
  const long long total = (long long)B * N;
  const long long stride = (long long)gridDim.x * blockDim.x;
  const long long g0 = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  for (long long idx = g0; idx < total; idx += stride) {
    for (int h = 0; h < H; ++h) {
      long long qs = 0, qm = 0;
      if (h < 2) {
        const long long* a = acc + (size_t)((now + h) & 1) * total * W;
        if (W == 1) unpack2(a[idx], qs, qm);
        else { qs = a[2 * idx]; qm = a[2 * idx + 1]; }
      }
      const int row = (now + h) % R;
      if (ring_dirty[row]) {
        const int b = (int)(idx / N);
        const size_t so = ((size_t)b * R + row) * N + (idx - (long long)b * N);
        long long rs, rm;
        if (W == 1) unpack2(ring[so], rs, rm);
        else { rs = ring[2 * so]; rm = ring[2 * so + 1]; }
        qs += rs;
        qm += rm;
      }
      atomicAdd(reinterpret_cast<unsigned long long*>(out + (idx * H + h) * 2), (unsigned long long)qs);
      atomicAdd(reinterpret_cast<unsigned long long*>(out + (idx * H + h) * 2 + 1), (unsigned long long)qm);
    }
  }
  for (int cta = 0; cta < G; ++cta) {
    for (int h = 2; h < H; ++h) {
      const int bin = (now + h) % NB;
      long long n = bk_cnt[(size_t)cta * NB + bin];
      n = n < cap_b ? n : cap_b;
      const size_t base = ((size_t)cta * NB + bin) * cap_b;
      for (long long k = g0; k < n; k += stride) {
        const long long* ent = bk + (base + k) * bk_words<T>();
        const long long tg = ent[0] & (kNegEntry - 1);   // admission kinds: withdrawn events carry negated payloads
        long long qs, qm;
        const long long* pp = ent + 1;
        if (W == 1) unpack2(pp[0], qs, qm);
        else { qs = pp[0]; qm = pp[1]; }
        atomicAdd(reinterpret_cast<unsigned long long*>(out + (tg * H + h) * 2), (unsigned long long)qs);
        atomicAdd(reinterpret_cast<unsigned long long*>(out + (tg * H + h) * 2 + 1), (unsigned long long)qm);
      }
    }
  }
}

template <typename T>
__global__ void k_pending(const long long* ring, int B, int R, int N, int H, int now, long long* out) {
  long long total = (long long)B * N * H;
  for (long long k = blockIdx.x * (long long)blockDim.x + threadIdx.x; k < total;
       k += (long long)gridDim.x * blockDim.x) {
    int hh = (int)(k % H);
    long long bj = k / H;
    int j = (int)(bj % N);
    int b = (int)(bj / N);
    size_t so = ((size_t)b * R + (size_t)((now + hh) % R)) * N + j;
    long long qs, qm;
    if (Prec<T>::kSlotWords == 1) {
      unpack2(ring[so], qs, qm);
    } else {
      qs = ring[2 * so];
      qm = ring[2 * so + 1];
    }
    out[2 * k] = qs;
    out[2 * k + 1] = qm;
  }
}

// Reset of the ring kind's DRAM overflow rows: only rows a bucket overflow
// flagged hold anything (every popped row is cleared by its pop), so only those
// are zeroed — not the whole B x R x N ring (1.27 GB at C3 x 24).
// grid: x over the row's words, y = b * R + r.
__global__ void k_clear_dirty_rows(long long* ring, int* ring_dirty, int R, long long row_words) {
  const int r = blockIdx.y % R;
  if (ring_dirty[r] == 0) return;
  long long* row = ring + (size_t)blockIdx.y * row_words;
  for (long long k = blockIdx.x * (long long)blockDim.x + threadIdx.x; k < row_words;
       k += (long long)gridDim.x * blockDim.x)
    row[k] = 0;
}

// Same for the admission kinds' event counts of those rows ([B][R][N] int32).
__global__ void k_clear_dirty_rows_i32(int* cring, const int* ring_dirty, int R, long long row_words) {
  const int r = blockIdx.y % R;
  if (ring_dirty[r] == 0) return;
  int* row = cring + (size_t)blockIdx.y * row_words;
  for (long long k = blockIdx.x * (long long)blockDim.x + threadIdx.x; k < row_words;
       k += (long long)gridDim.x * blockDim.x)
    row[k] = 0;
}

// CSC of the admission kinds: source row of every CSR edge, then {x, source}
// in (target, x) order (a stable radix sort of the edge indices by target).
__global__ void k_row_src(const int64_t* rowptr, int n_src, int* src) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n_src; i += gridDim.x * blockDim.x)
    for (int64_t x = rowptr[i]; x < rowptr[i + 1]; ++x) src[x] = i;
}
__global__ void k_iota_i32(int* p, long long n) {
  for (long long k = blockIdx.x * (long long)blockDim.x + threadIdx.x; k < n; k += (long long)gridDim.x * blockDim.x)
    p[k] = (int)k;
}
__global__ void k_csc_pack(const int* xs, const int* src, long long n, int2* csc) {
  for (long long k = blockIdx.x * (long long)blockDim.x + threadIdx.x; k < n; k += (long long)gridDim.x * blockDim.x)
    csc[k] = make_int2(xs[k], src[xs[k]]);
}

// Lossy ring contents pending at step `now`: slot (now + h) % S holds the
// events popped at now + h for h < S - 1 (= min(capacity, horizon)); larger h
// alias to earlier steps and stay empty.  out int64 [B*N][H][2].
__global__ void k_pending_lossy(const long long* ring, int W, int S, int B, int N, int H, int now, long long* out) {
  const long long total = (long long)B * N;
  for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < total;
       idx += (long long)gridDim.x * blockDim.x) {
    const int b = (int)(idx / N), j = (int)(idx - (long long)b * N);
    for (int h = 0; h < H; ++h) {
      long long qs = 0, qm = 0;
      if (h < S - 1) {
        const long long* sl = ring + (((size_t)b * S + (size_t)((now + h) % S)) * N + j) * W;
        if (W == 1) unpack2(sl[0], qs, qm);
        else { qs = sl[0]; qm = sl[1]; }
      }
      out[(idx * H + h) * 2] = qs;
      out[(idx * H + h) * 2 + 1] = qm;
    }
  }
}

__global__ void k_meta_init(int4* meta, long long n) {
  for (long long k = blockIdx.x * (long long)blockDim.x + threadIdx.x; k < n; k += (long long)gridDim.x * blockDim.x)
    meta[k] = make_int4(0, 0, -1, 0x7fffffff);
}

template <typename T>
__global__ void k_pending_bounded(const QEv<T>* q, const int4* meta, int kind, int cap, long long total, int H,
                                  int now, long long* out) {
  for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < total;
       idx += (long long)gridDim.x * blockDim.x) {
    long long* o = out + idx * H * 2;
    for (int k = 0; k < 2 * H; ++k) o[k] = 0;
    const int4 mt = meta[idx];
    const QEv<T>* qq = q + idx * cap;
    for (int k = 0; k < mt.x; ++k) {
      int pos = k;
      if (kind != EQ_KIND_BINARYHEAP) {
        pos = mt.y + k;
        if (pos >= cap) pos -= cap;
      }
      const QEv<T> ev = qq[pos];
      const int h = ev.due - now;
      if (h >= 0 && h < H) {
        long long a = 0, b = 0;
        ev.add_to(a, b);
        o[2 * h] += a;
        o[2 * h + 1] += b;
      }
    }
  }
}

// ------------------------------------------------------------ spike exchange (partitioned networks)

// Wire record of one spike (eq_spike_f32 / eq_spike_f64 in the header).
template <typename T>
struct ExRec {
  int src, trial, step;
  T t;
};
static_assert(sizeof(ExRec<float>) == 16 && sizeof(ExRec<double>) == 24, "wire layout");

// Log records of steps [lo, hi) -> wire records with global source ids.
template <typename T>
__global__ void k_export(const SpikeRec<T>* log, const long long* step_start, int lo, int hi, int N, int src_off,
                         ExRec<T>* out) {
  const long long k0 = step_start[lo], n = step_start[hi] - k0;
  for (long long k = blockIdx.x * (long long)blockDim.x + threadIdx.x; k < n;
       k += (long long)gridDim.x * blockDim.x) {
    const long long pos = k0 + k;
    int a = lo, b = hi;                    // largest m in [lo, hi) with step_start[m] <= pos
    while (b - a > 1) {
      const int mid = (a + b) >> 1;
      if (step_start[mid] <= pos) a = mid;
      else b = mid;
    }
    const SpikeRec<T> r = log[pos];
    ExRec<T> e;
    e.trial = r.idx / N;
    e.src = src_off + (r.idx - e.trial * N);
    e.step = a;
    e.t = r.t;
    out[k] = e;
  }
}

// Wire records -> fan-out records of this partition: idx = trial base, a = emit
// step, CSR row of the (remote) source.
template <typename T>
__global__ void k_import(const ExRec<T>* in, long long n, const int64_t* rowptr, int n_src, int src_off, int n_own,
                         int B, int N, int now, SpikeRec<T>* imp, long long* r0, int* len, int* err) {
  for (long long k = blockIdx.x * (long long)blockDim.x + threadIdx.x; k < n;
       k += (long long)gridDim.x * blockDim.x) {
    const ExRec<T> e = in[k];
    const bool bad = e.src < 0 || e.src >= n_src || (e.src >= src_off && e.src < src_off + n_own) || e.trial < 0 ||
                     e.trial >= B || e.step < 0 || e.step >= now;
    if (bad) {
      raise_error(err, EQ_ERR_CONFIGURATION, e.step, e.trial, e.src);
      len[k] = 0;
      r0[k] = 0;
      SpikeRec<T> z{};
      imp[k] = z;
      continue;
    }
    SpikeRec<T> r{};
    r.idx = e.trial * N;
    r.t = e.t;
    r.a = (T)e.step;      // exact: steps < 2^24
    r.vh = (T)0;
    imp[k] = r;
    const long long a = rowptr[e.src];
    r0[k] = a;
    len[k] = (int)(rowptr[e.src + 1] - a);
  }
}

// ------------------------------------------------------------ peer exchange (device-resident)

constexpr int kMaxPeers = 16;
// What a partition's kernels read of every partition (its own entry included):
// spike log + step index (forward import), import adjoints + block index
// (reverse).  Device pointers; with several GPUs these are peer addresses
// reached over NVLink (cudaDeviceEnablePeerAccess in eq_set_peers).
struct PeerDesc {
  const void* log;               // SpikeRec<T>[log_cap]
  const long long* step_start;   // [t_cap + 1]
  const void* imp_lt;            // T[imp_cap]: partial dL/dt_spk of its imports
  const long long* blk;          // [t_cap + 2][2] {first, count} of its import block w
  int N, src_off;
};
struct PeerTable {
  PeerDesc d[kMaxPeers];
  int P, me;
};

// Import block of window w for partition `me`: the other partitions' spikes
// of steps [a_prev, a) read straight from their logs, in partition order then
// log order, appended at *count as fan-out records (idx = trial base, a = emit
// step, CSR row of the global source in this partition's CSR).
template <typename T>
__global__ void k_gather_peers(PeerTable tab, int a_prev, int a, int N_me, const int64_t* rowptr, SpikeRec<T>* imp,
                               long long* imp_r0, int* imp_len, const long long* count, long long cap, int* err) {
  const long long base = *count;
  long long off[kMaxPeers + 1];
  off[0] = 0;
  for (int q = 0; q < tab.P; ++q) {
    long long n = 0;
    if (q != tab.me) n = tab.d[q].step_start[a] - tab.d[q].step_start[a_prev];
    off[q + 1] = off[q] + n;
  }
  const long long total = off[tab.P];
  if (base + total > cap) {
    if (blockIdx.x == 0 && threadIdx.x == 0) raise_error(err, EQ_ERR_CAPACITY, a, -1, -1);
    return;
  }
  for (long long r = blockIdx.x * (long long)blockDim.x + threadIdx.x; r < total;
       r += (long long)gridDim.x * blockDim.x) {
    int q = 0;
    while (off[q + 1] <= r) ++q;
    const PeerDesc& d = tab.d[q];
    const long long pos = d.step_start[a_prev] + (r - off[q]);
    const SpikeRec<T> rec = static_cast<const SpikeRec<T>*>(d.log)[pos];
    int lo = a_prev, hi = a;                         // emit step: largest m with step_start[m] <= pos
    while (hi - lo > 1) {
      const int mid = (lo + hi) >> 1;
      if (d.step_start[mid] <= pos) lo = mid;
      else hi = mid;
    }
    const int trial = rec.idx / d.N;
    const int src = d.src_off + (rec.idx - trial * d.N);
    SpikeRec<T> o{};
    o.idx = trial * N_me;
    o.t = rec.t;
    o.a = (T)lo;                                     // exact: steps < 2^24
    imp[base + r] = o;
    const long long r0 = rowptr[src];
    imp_r0[base + r] = r0;
    imp_len[base + r] = (int)(rowptr[src + 1] - r0);
  }
}

__global__ void k_gather_commit(PeerTable tab, int a_prev, int a, long long* count, long long* blk) {
  long long total = 0;
  for (int q = 0; q < tab.P; ++q)
    if (q != tab.me) total += tab.d[q].step_start[a] - tab.d[q].step_start[a_prev];
  blk[0] = *count;
  blk[1] = total;
  *count += total;
}

// Before partition me's reverse window over steps [a, a_next): the other
// partitions' partial dL/dt_spk of its spikes of those steps, which each of
// them computed in import block w+1 (their imports of this window); summed in
// partition order into lt_rem (the order the host-routed exchange uses).
template <typename T>
__global__ void k_sum_peer_adjoints(PeerTable tab, int w, int a, int a_next, T* lt_rem) {
  const PeerDesc& mine = tab.d[tab.me];
  const long long k0 = mine.step_start[a], n = mine.step_start[a_next] - k0;
  for (long long k = blockIdx.x * (long long)blockDim.x + threadIdx.x; k < n;
       k += (long long)gridDim.x * blockDim.x) {
    T acc = (T)0;
    bool first = true;
    for (int p = 0; p < tab.P; ++p) {
      if (p == tab.me) continue;
      long long off = tab.d[p].blk[2 * (w + 1)];     // p's block w+1 holds the others' spikes of [a, a_next)
      for (int q = 0; q < tab.me; ++q)
        if (q != p) off += tab.d[q].step_start[a_next] - tab.d[q].step_start[a];
      const T v = static_cast<const T*>(tab.d[p].imp_lt)[off + k];
      acc = first ? v : acc + v;
      first = false;
    }
    lt_rem[k0 + k] = (T)0 + acc;
  }
}

template <typename T>
__global__ void k_add_lt(T* lt_rem, const long long* step_start, int lo, const T* vals, long long n) {
  const long long k0 = step_start[lo];
  for (long long k = blockIdx.x * (long long)blockDim.x + threadIdx.x; k < n;
       k += (long long)gridDim.x * blockDim.x)
    lt_rem[k0 + k] += vals[k];
}

// ------------------------------------------------------------ launches

// staged bounded-queue kernel: key staging of every warp
constexpr size_t bq_smem() { return (size_t)(kBqChunk + kBqPoolWords) * sizeof(unsigned); }

// reverse kernel dynamic smem: spiker bitmap + uint16 chunk position per owned neuron
size_t bwd_smem(long long per) {
  return (size_t)((per + 31) / 32) * sizeof(unsigned) + (size_t)((per + 1) / 2) * sizeof(unsigned);
}

// Wait for the stream and map the device error word to a status + message.
// `reached` (forward launches): the step the launch ended at (err[4]); the
// spike-log fill is cached in h->log_used on the same synchronisation.
int check_err(eq_handle* h, cudaStream_t s, int* reached = nullptr) {
  int e[kErrWords];
  unsigned long long used = 0;
  EQ_CUDA(h, cudaMemcpyAsync(e, h->err_dev, sizeof e, cudaMemcpyDeviceToHost, s));
  if (reached) EQ_CUDA(h, cudaMemcpyAsync(&used, h->log_count, sizeof used, cudaMemcpyDeviceToHost, s));
  EQ_CUDA(h, cudaStreamSynchronize(s));
  if (reached) {
    *reached = e[4];
    h->log_used = (long long)used;
  }
  if (e[0] == 0) return EQ_OK;
  char buf[256];
  switch (e[0]) {
    case EQ_ERR_GRAZING:
      snprintf(buf, sizeof buf, "grazing crossing at step %d (trial %d, neuron %d): slope below 1e-09",
               e[1], e[2], e[3]);
      break;
    case EQ_ERR_CAPACITY:
      snprintf(buf, sizeof buf, "spike log capacity %lld exceeded at step %d; raise eq_config.max_spikes",
               (long long)h->log_cap, e[1]);
      break;
    case EQ_ERR_CUDA:
      snprintf(buf, sizeof buf, "device watchdog: grid barrier timed out");
      break;
    case EQ_ERR_CAPABILITY:
      if (h->cfg.kind == EQ_KIND_FIFORING) {   // queues.py:220-224 (the step pair is not kept on the device)
        snprintf(buf, sizeof buf,
                 "fiforing supports homogeneous delays only: an event arrived after one due later "
                 "(enqueued at step %d, trial %d, neuron %d)", e[1], e[2], e[3]);
        break;
      }
      snprintf(buf, sizeof buf, "device error %d at step %d (trial %d, neuron %d)", e[0], e[1], e[2], e[3]);
      break;
    default:
      snprintf(buf, sizeof buf, "device error %d at step %d (trial %d, neuron %d)", e[0], e[1], e[2], e[3]);
  }
  return fail(h, e[0], buf);
}

bool getenv_flag(const char* name) {
  const char* v = getenv(name);
  return v && v[0] == '1';
}

std::array<long long, 4>* find_block(eq_handle* h, int start) {
  for (auto& b : h->imp_blocks)
    if (b[0] == start && b[2] > 0) return &b;
  return nullptr;
}

// Grow the spike log (and the per-record arrays, and the bounded kinds' drop
// bits, which are indexed by log position) to hold at least `need` records;
// the first log_used records are kept.
int grow_log(eq_handle* h, long long need, cudaStream_t s) {
  const long long ncap = std::max<long long>(need, 2 * h->log_cap);
  if (h->adm && ncap >= (1LL << 31))
    return fail(h, EQ_ERR_CAPACITY, "spike log beyond 2^31 records (admission kinds keep 32-bit log positions)");
  const size_t rec = h->cfg.precision == 32 ? sizeof(SpikeRec<float>) : sizeof(SpikeRec<double>);
  const long long used = h->log_used;
  void *lg = nullptr, *r0 = nullptr, *len = nullptr, *lt = nullptr, *ltr = nullptr;
  EQ_CUDA(h, alloc(h, &lg, (size_t)ncap * rec));
  EQ_CUDA(h, alloc(h, &r0, (size_t)ncap * sizeof(long long)));
  EQ_CUDA(h, alloc(h, &len, (size_t)ncap * sizeof(int)));
  EQ_CUDA(h, alloc(h, &lt, (size_t)ncap * h->tsize));
  EQ_CUDA(h, alloc(h, &ltr, (size_t)ncap * h->tsize));
  if (used > 0) {
    EQ_CUDA(h, cudaMemcpyAsync(lg, h->log, (size_t)used * rec, cudaMemcpyDeviceToDevice, s));
    EQ_CUDA(h, cudaMemcpyAsync(r0, h->log_r0, (size_t)used * sizeof(long long), cudaMemcpyDeviceToDevice, s));
    EQ_CUDA(h, cudaMemcpyAsync(len, h->log_len, (size_t)used * sizeof(int), cudaMemcpyDeviceToDevice, s));
  }
  if (h->bounded) {
    const long long ndrop = (ncap * h->maxdeg + 31) / 32 * 32;
    void* db = nullptr;
    EQ_CUDA(h, alloc(h, &db, (size_t)ndrop / 8));
    EQ_CUDA(h, cudaMemsetAsync(db, 0, (size_t)ndrop / 8, s));
    EQ_CUDA(h, cudaMemcpyAsync(db, h->drop_bits, (size_t)h->drop_cap / 8, cudaMemcpyDeviceToDevice, s));
    EQ_CUDA(h, cudaStreamSynchronize(s));
    release(h, h->drop_bits);
    h->drop_bits = (unsigned*)db;
    h->drop_cap = ndrop;
  }
  EQ_CUDA(h, cudaStreamSynchronize(s));
  release(h, h->log);
  release(h, h->log_r0);
  release(h, h->log_len);
  release(h, h->lt_log);
  release(h, h->lt_rem);
  h->log = lg;
  h->log_r0 = (long long*)r0;
  h->log_len = (int*)len;
  h->lt_log = lt;
  h->lt_rem = ltr;
  h->log_cap = ncap;
  h->log_grows += 1;
  return EQ_OK;
}

// Kernel arguments of a forward launch over steps [steps_done, steps_done + n_steps).
template <typename T>
FwdArgs<T> fwd_args(eq_handle* h, int n_steps, void* v_trace) {
  FwdArgs<T> A;
  A.N = h->cfg.n_neurons;
  A.B = h->cfg.n_trials;
  A.G = h->G;
  A.total = h->total;
  A.per = h->per;
  A.m0 = h->steps_done;
  A.m1 = h->steps_done + n_steps;
  A.R = h->R;
  A.kind = h->cfg.kind;
  A.refractory = h->cfg.refractory_steps;
  A.exact = h->cfg.exact_delivery;
  A.c = consts<T>(h);
  A.net = netview<T>(h);
  A.I = (T*)h->I;
  A.V = (T*)h->V;
  A.refr = h->refr;
  A.ring = h->ring;
  A.acc = h->acc;
  A.bk = h->bk;
  A.bk_cnt = h->bk_cnt;
  A.cap_b = h->cap_b;
  A.NB = h->NB;
  A.ring_dirty = h->ring_dirty;
  A.scratch = (SpikeRec<T>*)h->scratch;
  A.log = (SpikeRec<T>*)h->log;
  A.log_r0 = h->log_r0;
  A.log_len = h->log_len;
  A.log_cap = h->log_cap;
  A.log_count = h->log_count;
  A.chunk_off = h->chunk_off;
  A.chunk_cnt = h->chunk_cnt;
  A.step_start = h->step_start;
  A.counters = h->counters;
  A.v_trace = (T*)v_trace;
  A.src_off = h->src_off;
  A.smem_state = 0;
  A.imp = nullptr;
  A.imp_r0 = nullptr;
  A.imp_len = nullptr;
  A.imp_n = 0;
  A.imp_dev = nullptr;
  A.no_pause = 0;
  A.cal = h->cal;
  A.adm_cap = h->cap;
  A.totp = h->totp;
  A.aw = (int*)h->adm_ctr;
  A.ac = h->adm_ctr ? (unsigned short*)((int*)h->adm_ctr + 2 * h->totp) : nullptr;
  A.aa = h->adm_ctr ? A.ac + 2 * h->totp : nullptr;
  A.fl = h->fl;
  A.fl_cnt = h->fl_cnt;
  A.lpos = h->lpos;
  A.csc = h->csc;
  A.csc_off = h->csc_off;
  A.drop_bits = h->drop_bits;
  A.drop_cap = h->drop_cap;
  A.maxdeg = h->maxdeg;
  A.divPer = FastDiv((unsigned)h->per);
  A.cring = h->cring;
  A.slots = h->slots;
  A.adm_slots = h->adm_slots;
  A.tl = (h->tl_f && A.m1 <= h->tl_steps) ? h->tl_f : nullptr;
  A.err = h->err_dev;
  A.bar = h->bar;
  return A;
}

// One persistent launch over steps [steps_done, steps_done + n_steps); it may
// end early at a step boundary when the spike log could overflow (*reached).
template <typename T>
int launch_forward_once(eq_handle* h, int n_steps, void* v_trace, cudaStream_t s, int* reached) {
  FwdArgs<T> A = fwd_args<T>(h, n_steps, v_trace);
  std::array<long long, 4>* blk = find_block(h, h->steps_done);
  if (blk && !(*blk)[3]) {
    (*blk)[3] = 1;
    A.imp = (const SpikeRec<T>*)h->imp + (*blk)[1];
    A.imp_r0 = h->imp_r0 + (*blk)[1];
    A.imp_len = h->imp_len + (*blk)[1];
    A.imp_n = (*blk)[2];
  }
  if ((h->bounded && !h->adm) || h->lossy) {
    BndArgs<T> Bk;
    Bk.f = A;
    Bk.cap = h->lossy ? h->lossy_slots : h->cap;
    Bk.cap_ref = h->lossy ? (int)std::min<long long>(h->lossy_cap, 1LL << 30) : 0;
    Bk.csc_off = h->csc_off;
    Bk.E = h->E;
    Bk.alist = (Arrival<T>*)h->alist;
    Bk.acnt = h->acnt;
    Bk.q = (QEv<T>*)h->q;
    Bk.meta = h->meta;
    Bk.maxdeg = h->maxdeg;
    Bk.drop_bits = h->drop_bits;
    Bk.drop_cap = h->drop_cap;
    Bk.insert_first = h->steps_done;
    Bk.keys = h->qkeys;
    Bk.pay = h->qpay;
    Bk.C = h->C;
    Bk.qdue = h->qdue;
    Bk.inbox = h->inbox;
    Bk.in_cnt = h->in_cnt;
    Bk.in_cap = h->in_cap;
    Bk.aoff = h->aoff;
    Bk.aidx = h->aidx;
    Bk.divPer = FastDiv((unsigned)h->per);
    void* bargs[] = {&Bk};
    if (h->staged) {
      const void* kq = (const void*)k_forward_bq<T, kNT, kU>;
      EQ_CUDA(h, cudaFuncSetAttribute(kq, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bq_smem()));
      EQ_CUDA(h, cudaLaunchCooperativeKernel(kq, dim3(h->G), dim3(kNT), bargs, bq_smem(), s));
    } else {
      EQ_CUDA(h, cudaLaunchCooperativeKernel((const void*)k_forward_bounded<T, kNT, kU>, dim3(h->G), dim3(kNT),
                                             bargs, 0, s));
    }
  } else {
    void* args[] = {&A};
    if (A.imp_n > 0) {   // other partitions' spikes of the last window, due >= m0+1
      FwdArgs<T> Ai = A;
      Ai.tl = nullptr;
      k_import_fanout<T, kNT><<<h->G, kNT, 0, s>>>(Ai);
      h->launches += 1;
      if (n_steps == 0) return check_err(h, s);   // flush: deliver the imports, no step
    }
    const void* kf = h->adm ? (const void*)k_forward<T, kNT, kU, split_f<T>(), true>
                            : (const void*)k_forward<T, kNT, kU, split_f<T>()>;
    // fp32: I and V of each CTA's range in shared memory for the whole launch
    // when two CTAs per SM still fit (state 2 x per x 4 B next to ~39 KB static)
    const size_t st_bytes = (size_t)2 * h->per * sizeof(T);
    size_t dyn = 0;
    if (sizeof(T) == 4 && st_bytes <= kStateSmem && !getenv_flag("EQ_NO_SMEM_STATE")) {
      EQ_CUDA(h, cudaFuncSetAttribute(kf, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)st_bytes));
      int occ = 0;   // the cooperative grid must stay co-resident
      EQ_CUDA(h, cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kf, kNT, st_bytes));
      if ((long long)occ * h->n_sm >= h->G) dyn = st_bytes;
    }
    if (dyn == 0) {   // state in HBM: the ring's 288-thread event side; fp32 admission: one event in flight
      if (!h->adm) kf = (const void*)k_forward<T, kNT, kU, split_f_hbm<T>()>;
      else if (sizeof(T) == 4) kf = (const void*)k_forward<T, kNT, kU, split_f<T>(), true, 1>;
    }
    FwdArgs<T>* ap = &A;
    ap->smem_state = dyn > 0;
    EQ_CUDA(h, cudaLaunchCooperativeKernel(kf, dim3(h->G), dim3(kNT), args, dyn, s));
    if (h->adm) {   // reference-order fix-ups of the launch's last admissions (step reached: err[4])
      k_adm_fixup<T, kNT><<<h->G, kNT, 0, s>>>(A);
      h->launches += 1;
    }
  }
  h->launches += 1;
  return check_err(h, s, reached);
}

// eq_run's launches: as many persistent launches as the spike log needs (one
// unless it fills up; then it grows and the run resumes at the step reached).
template <typename T>
int launch_forward(eq_handle* h, int n_steps, void* v_trace, cudaStream_t s) {
  int done = 0;
  while (true) {
    if (n_steps > 0 && h->log_used + h->total > h->log_cap) {
      int rc = grow_log(h, h->log_used + 2 * h->total, s);
      if (rc) return rc;
    }
    if (done > 0) EQ_CUDA(h, cudaMemsetAsync(h->bar, 0, kBarWords * sizeof(unsigned), s));
    void* vt = v_trace ? (char*)v_trace + (size_t)done * h->total * h->tsize : nullptr;
    int reached = h->steps_done + (n_steps - done);
    int rc = launch_forward_once<T>(h, n_steps - done, vt, s, &reached);
    if (rc != EQ_OK) {
      if (rc == EQ_ERR_GRAZING) h->steps_done += n_steps - done;
      return rc;
    }
    if (n_steps == 0) return EQ_OK;
    if (reached <= h->steps_done || reached > h->steps_done + (n_steps - done))
      return fail(h, EQ_ERR_CUDA, "forward launch reported step " + std::to_string(reached));
    done += reached - h->steps_done;
    h->steps_done = reached;
    if (done == n_steps) return EQ_OK;
  }
}

template <typename T>
int backward_begin(eq_handle* h, const void* v_bar, const void* i_bar, double* gw, double* gd, double* gamp,
                   cudaStream_t s) {
  const long long total = h->total;
  EQ_CUDA(h, cudaMemcpyAsync(h->lamV, v_bar, total * sizeof(T), cudaMemcpyDeviceToDevice, s));
  if (i_bar) EQ_CUDA(h, cudaMemcpyAsync(h->lamI, i_bar, total * sizeof(T), cudaMemcpyDeviceToDevice, s));
  else EQ_CUDA(h, cudaMemsetAsync(h->lamI, 0, total * sizeof(T), s));
  // no clear of the reverse ring: R-fanout reads only rows of steps < m_run,
  // each written by R-neuron of its step earlier in the reverse sweep
  EQ_CUDA(h, cudaMemsetAsync(gw, 0, h->E * sizeof(double), s));
  EQ_CUDA(h, cudaMemsetAsync(gd, 0, h->E * sizeof(double), s));
  if (gamp) EQ_CUDA(h, cudaMemsetAsync(h->gamp_bt, 0, total * sizeof(double), s));
  if (h->partitioned) EQ_CUDA(h, cudaMemsetAsync(h->lt_rem, 0, (size_t)h->log_cap * sizeof(T), s));
  h->bwd_cursor = h->steps_done;
  h->bw_gw = gw;
  h->bw_gd = gd;
  h->bw_gamp = gamp;
  return EQ_OK;
}

// Reverse phases bwd_cursor-1 .. m_lo in one persistent launch.
template <typename T>
int launch_backward(eq_handle* h, int m_lo, cudaStream_t s, int peer_win = -1) {
  typedef typename Prec<T>::T2 T2;
  const int N = h->cfg.n_neurons, B = h->cfg.n_trials;
  EQ_CUDA(h, cudaMemsetAsync(h->bar, 0, kBarWords * sizeof(unsigned), s));
  BwdArgs<T> A;
  A.N = N;
  A.B = B;
  A.G = h->G;
  A.total = h->total;
  A.per = h->per;
  A.m_run = h->steps_done;
  A.m_hi = h->bwd_cursor;
  A.m_lo = m_lo;
  A.R = h->R;
  A.refractory = h->cfg.refractory_steps;
  A.c = consts<T>(h);
  A.net = netview<T>(h);
  A.lamV = (T*)h->lamV;
  A.lamI = (T*)h->lamI;
  A.lam = (T2*)h->lam;
  A.gw = h->bw_gw;
  A.gd = h->bw_gd;
  A.gamp_bt = h->bw_gamp ? h->gamp_bt : nullptr;
  A.log = (const SpikeRec<T>*)h->log;
  A.log_r0 = h->log_r0;
  A.log_len = h->log_len;
  A.lt_log = (T*)h->lt_log;
  A.chunk_off = h->chunk_off;
  A.chunk_cnt = h->chunk_cnt;
  A.step_start = h->step_start;
  A.maxdeg = h->maxdeg;
  A.drop_bits = h->bounded ? h->drop_bits : nullptr;
  A.exact = h->cfg.exact_delivery;
  A.lossy_cap = h->lossy ? (int)std::min<long long>(h->lossy_cap, 1LL << 30) : 0;
  A.serial = h->lossy && h->lossy_cap < h->horizon;   // aliasing can pop an event one step after emission
  A.no_events = h->cfg.kind == EQ_KIND_DONOTHING;
  A.lt_rem = h->partitioned ? (const T*)h->lt_rem : nullptr;
  A.imp = nullptr;
  A.imp_r0 = nullptr;
  A.imp_len = nullptr;
  A.imp_n = 0;
  A.imp_dev = nullptr;
  A.imp_lt = nullptr;
  if (peer_win > 0) {                                 // peer exchange: the block is on the device
    A.imp = (const SpikeRec<T>*)h->imp;
    A.imp_r0 = h->imp_r0;
    A.imp_len = h->imp_len;
    A.imp_lt = (T*)h->imp_lt;
    A.imp_dev = h->peer_blk + 2 * peer_win;
  } else if (std::array<long long, 4>* blk = find_block(h, m_lo)) {
    A.imp = (const SpikeRec<T>*)h->imp + (*blk)[1];
    A.imp_r0 = h->imp_r0 + (*blk)[1];
    A.imp_len = h->imp_len + (*blk)[1];
    A.imp_n = (*blk)[2];
    A.imp_lt = (T*)h->imp_lt + (*blk)[1];
  }
  A.tl = (h->tl_b && A.m_run <= h->tl_steps) ? h->tl_b : nullptr;
  A.err = h->err_dev;
  A.bar = h->bar;
  size_t smem = bwd_smem(h->per);
  void* args[] = {&A};
  const void* kb = (const void*)k_backward<T, kNT, kU, split_b<T>()>;
  // static + dynamic smem beyond 48 KB needs the opt-in (the static part alone is ~41 KB)
  EQ_CUDA(h, cudaFuncSetAttribute(kb, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  EQ_CUDA(h, cudaLaunchCooperativeKernel(kb, dim3(h->G), dim3(kNT), args, smem, s));
  h->launches += 1;
  if (A.imp_n > 0 || A.imp_dev) {   // partial dL/dt_spk of the imported spikes (reverse slots >= m_lo final)
    BwdArgs<T> Ai = A;
    Ai.tl = nullptr;
    k_import_rfanout<T, kNT><<<h->G, kNT, 0, s>>>(Ai);
    h->launches += 1;
  }
  h->bwd_cursor = m_lo;
  if (m_lo == 0 && h->bw_gamp) {
    k_sum_trials<T><<<(N + 255) / 256, 256, 0, s>>>(h->gamp_bt, B, N, h->bw_gamp);
    h->launches += 1;
  }
  if (peer_win >= 0) return EQ_OK;   // asynchronous windows: errors surface at eq_sync
  return check_err(h, s);
}

int setup_geometry(eq_handle* h) {
  // One persistent CTA set shared by forward and reverse (the reverse pass
  // finds a step's spikes through the forward's per-CTA chunks).
  int occ_f = 0, occ_b = 0;
  const void* kf;
  const void* kb;
  if (h->cfg.precision == 32) {
    kf = (const void*)k_forward<float, kNT, kU, kSplitF>;
    kb = (const void*)k_backward<float, kNT, kU, kSplitB>;
  } else {
    kf = (const void*)k_forward<double, kNT, kU, split_f<double>()>;
    kb = (const void*)k_backward<double, kNT, kU, split_b<double>()>;
  }
  EQ_CUDA(h, cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ_f, kf, kNT, 0));
  if (h->cfg.precision == 32) {   // the state-in-HBM split of the ring kernel too
    int occ_h = 0;
    EQ_CUDA(h, cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ_h, (const void*)k_forward<float, kNT, kU, kSplitFHbm>,
                                                             kNT, 0));
    occ_f = std::min(occ_f, occ_h);
  }
  {
    int occ_a = 0;
    const void* ka = h->cfg.precision == 32 ? (const void*)k_forward<float, kNT, kU, kSplitF, true>
                                            : (const void*)k_forward<double, kNT, kU, split_f<double>(), true>;
    EQ_CUDA(h, cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ_a, ka, kNT, 0));
    occ_f = std::min(occ_f, occ_a);
    const void* ka1 = h->cfg.precision == 32 ? (const void*)k_forward<float, kNT, kU, kSplitF, true, 1>
                                             : (const void*)k_forward<double, kNT, kU, split_f<double>(), true, 1>;
    EQ_CUDA(h, cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ_a, ka1, kNT, 0));
    occ_f = std::min(occ_f, occ_a);
  }
  {
    int occ_q = 0;
    const void* kq = h->cfg.precision == 32 ? (const void*)k_forward_bounded<float, kNT, kU>
                                            : (const void*)k_forward_bounded<double, kNT, kU>;
    EQ_CUDA(h, cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ_q, kq, kNT, 0));
    occ_f = std::min(occ_f, occ_q);
    const void* kb2 = h->cfg.precision == 32 ? (const void*)k_forward_bq<float, kNT, kU>
                                             : (const void*)k_forward_bq<double, kNT, kU>;
    EQ_CUDA(h, cudaFuncSetAttribute(kb2, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bq_smem()));
    EQ_CUDA(h, cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ_q, kb2, kNT, bq_smem()));
    occ_f = std::min(occ_f, occ_q);
  }
  int occ = std::max(1, occ_f);
  for (; occ >= 1; --occ) {
    long long G = (long long)h->n_sm * occ;
    long long per = (h->total + G - 1) / G;
    size_t smem = bwd_smem(per);
    if (smem > 160 * 1024) continue;
    EQ_CUDA(h, cudaFuncSetAttribute(kb, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    EQ_CUDA(h, cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ_b, kb, kNT, smem));
    if (occ_b >= occ) break;
  }
  if (occ < 1) return fail(h, EQ_ERR_CONFIGURATION, "problem too large for one persistent grid");
  h->G = h->n_sm * occ;
  if (h->cfg.max_ctas > 0 && h->cfg.max_ctas < h->G) h->G = h->cfg.max_ctas;
  // never more CTAs than there are neuron-trials to own
  if ((long long)h->G > h->total) h->G = (int)h->total;
  // ranges in whole warps so a warp's 32 neurons share one drive-mask word
  h->per = ((h->total + h->G - 1) / h->G + 31) / 32 * 32;
  h->G = (int)((h->total + h->per - 1) / h->per);
  return EQ_OK;
}

int ensure_chunks(eq_handle* h, int steps_needed) {
  if (steps_needed <= h->t_cap) return EQ_OK;
  int ncap = std::max(steps_needed, h->t_cap * 2);
  void *off = nullptr, *cnt = nullptr, *ss = nullptr;
  EQ_CUDA(h, alloc(h, &off, (size_t)ncap * h->G * sizeof(long long)));
  EQ_CUDA(h, alloc(h, &cnt, (size_t)ncap * h->G * sizeof(int)));
  EQ_CUDA(h, alloc(h, &ss, (size_t)(ncap + 1) * sizeof(long long)));
  EQ_CUDA(h, cudaMemset(ss, 0, (size_t)(ncap + 1) * sizeof(long long)));
  if (h->t_cap) {
    EQ_CUDA(h, cudaMemcpy(off, h->chunk_off, (size_t)h->t_cap * h->G * sizeof(long long), cudaMemcpyDeviceToDevice));
    EQ_CUDA(h, cudaMemcpy(cnt, h->chunk_cnt, (size_t)h->t_cap * h->G * sizeof(int), cudaMemcpyDeviceToDevice));
    EQ_CUDA(h, cudaMemcpy(ss, h->step_start, (size_t)(h->t_cap + 1) * sizeof(long long), cudaMemcpyDeviceToDevice));
  }
  release(h, h->chunk_off);
  release(h, h->chunk_cnt);
  release(h, h->step_start);
  h->chunk_off = (long long*)off;
  h->chunk_cnt = (int*)cnt;
  h->step_start = (long long*)ss;
  h->t_cap = ncap;
  return EQ_OK;
}

// Bounded kinds: in-edge ranks (stable CSC order via CUB radix sort), bitmap
// layout, queue storage.  Capacity: the reference's (`queue_capacity or
// horizon*(n-1)+1`, network.py:327); the physical array is min(that, the
// lossless bound max_j sum_{e->j}(ceil(d_e/dt)+1)), which cannot change any
// accept decision because occupancy never exceeds the bound.
int setup_bounded(eq_handle* h, const int* indeg, long long occ_bound, cudaStream_t s,
                  const unsigned long long* col_fp) {
  const eq_config& c = h->cfg;
  const int N = c.n_neurons, B = c.n_trials;
  const long long E = h->E;
  h->cap_ref = c.capacity > 0 ? c.capacity : (long long)h->horizon * (N - 1) + 1;
  long long cap = std::min<long long>(h->cap_ref, std::max<long long>(occ_bound, 1));
  if (cap > (1 << 20)) return fail(h, EQ_ERR_CONFIGURATION, "queue capacity too large; set eq_config.capacity");
  h->cap = (int)cap;
  if (E >= (1LL << 31)) return fail(h, EQ_ERR_CONFIGURATION, "bounded kinds support < 2^31 edges");
  if (h->adm) {
    // admission records (16-bit occupancy fields), fix-up lists, spike positions
    h->totp = (h->total + 7) / 8 * 8;
    EQ_CUDA(h, ensure(h, &h->adm_ctr, (size_t)h->totp * (2 * 4 + 2 * 2 + 3 * 2)));
    EQ_CUDA(h, ensure(h, (void**)&h->fl, (size_t)2 * h->G * h->per * sizeof(int)));
    EQ_CUDA(h, ensure(h, (void**)&h->fl_cnt, (size_t)2 * h->G * sizeof(int)));
    EQ_CUDA(h, ensure(h, (void**)&h->lpos, (size_t)3 * h->total * sizeof(int)));
    EQ_CUDA(h, ensure(h, (void**)&h->cring, (size_t)B * h->R * N * sizeof(int)));
    EQ_CUDA(h, ensure(h, (void**)&h->slots, (size_t)2 * h->total * kAdmSlots * sizeof(int2)));
    h->drop_cap = ((long long)h->log_cap * h->maxdeg + 31) / 32 * 32;
    EQ_CUDA(h, ensure(h, (void**)&h->drop_bits, (size_t)h->drop_cap / 8));
    // CSC: in-edge segments by exclusive scan of the in-degree, then the edge
    // indices stably sorted by target (ascending x within a target).  Only the
    // topology matters: unchanged (same edge count and column fingerprint, the
    // usual case of a training step with new weights and delays) -> kept.
    if (h->csc && h->csc_E == E && h->csc_fp[0] == col_fp[0] && h->csc_fp[1] == col_fp[1]) return EQ_OK;
    size_t tmp_bytes = 0;
    void* tmp = nullptr;
    EQ_CUDA(h, ensure(h, (void**)&h->csc_off, (size_t)(N + 1) * sizeof(long long)));
    EQ_CUDA(h, cub::DeviceScan::ExclusiveSum(nullptr, tmp_bytes, indeg, h->csc_off, N + 1, s));
    EQ_CUDA(h, alloc(h, &tmp, tmp_bytes));
    EQ_CUDA(h, cub::DeviceScan::ExclusiveSum(tmp, tmp_bytes, indeg, h->csc_off, N + 1, s));
    release(h, tmp);
    void *src = nullptr, *xin = nullptr, *xout = nullptr, *kout = nullptr;
    EQ_CUDA(h, alloc(h, &src, (size_t)E * sizeof(int)));
    EQ_CUDA(h, alloc(h, &xin, (size_t)E * sizeof(int)));
    EQ_CUDA(h, alloc(h, &xout, (size_t)E * sizeof(int)));
    EQ_CUDA(h, alloc(h, &kout, (size_t)E * sizeof(int)));
    k_row_src<<<(h->n_src + 255) / 256, 256, 0, s>>>(h->rowptr, h->n_src, (int*)src);
    k_iota_i32<<<1184, 256, 0, s>>>((int*)xin, E);
    int bits = 1;
    while ((1LL << bits) < N) ++bits;
    tmp_bytes = 0;
    EQ_CUDA(h, cub::DeviceRadixSort::SortPairs(nullptr, tmp_bytes, h->col, (int*)kout, (const int*)xin, (int*)xout,
                                               (int)E, 0, bits, s));
    EQ_CUDA(h, alloc(h, &tmp, tmp_bytes));
    EQ_CUDA(h, cub::DeviceRadixSort::SortPairs(tmp, tmp_bytes, h->col, (int*)kout, (const int*)xin, (int*)xout,
                                               (int)E, 0, bits, s));
    EQ_CUDA(h, ensure(h, (void**)&h->csc, (size_t)E * sizeof(int2)));
    k_csc_pack<<<1184, 256, 0, s>>>((const int*)xout, (const int*)src, E, h->csc);
    h->launches += 5;
    EQ_CUDA(h, cudaStreamSynchronize(s));
    release(h, tmp);
    release(h, src);
    release(h, xin);
    release(h, xout);
    release(h, kout);
    h->csc_E = E;
    h->csc_fp[0] = col_fp[0];
    h->csc_fp[1] = col_fp[1];
    return EQ_OK;
  }
  size_t qbytes = (size_t)B * N * h->cap * (c.precision == 32 ? sizeof(QEv<float>) : sizeof(QEv<double>));
  if (qbytes > ((size_t)96 << 30))
    return fail(h, EQ_ERR_CONFIGURATION, "queue storage " + std::to_string(qbytes >> 20) +
                                             " MiB exceeds 96 GiB; set eq_config.capacity");
  EQ_CUDA(h, ensure(h, (void**)&h->acnt, (size_t)2 * B * N * sizeof(int)));
  h->staged = c.staged_queues == 1 && h->cap <= kBqMaxCap;
  if (!h->staged) {
    // csc_off = exclusive scan of in-degree: target j's arrival list is its
    // in-edge segment [csc_off[j], csc_off[j+1]) (no step delivers more)
    size_t tmp_bytes = 0;
    void* tmp = nullptr;
    EQ_CUDA(h, ensure(h, (void**)&h->csc_off, (size_t)(N + 1) * sizeof(long long)));
    EQ_CUDA(h, cub::DeviceScan::ExclusiveSum(nullptr, tmp_bytes, indeg, h->csc_off, N + 1, s));
    EQ_CUDA(h, alloc(h, &tmp, tmp_bytes));
    EQ_CUDA(h, cub::DeviceScan::ExclusiveSum(tmp, tmp_bytes, indeg, h->csc_off, N + 1, s));
    release(h, tmp);
    h->launches += 1;
    EQ_CUDA(h, ensure(h, &h->alist, (size_t)2 * B * E * sizeof(Arrival<float>)));   // 32 bytes in both precisions
  } else {
    // owner inboxes: a step delivers at most one event per in-edge, so a CTA's
    // inbox needs the in-degree sum of its queues
    std::vector<int> deg(N);
    EQ_CUDA(h, cudaMemcpyAsync(deg.data(), indeg, (size_t)N * sizeof(int), cudaMemcpyDeviceToHost, s));
    EQ_CUDA(h, cudaStreamSynchronize(s));
    std::vector<long long> pre(N + 1, 0);
    for (int j = 0; j < N; ++j) pre[j + 1] = pre[j] + deg[j];
    auto upto = [&](long long idx) { return (idx / N) * pre[N] + pre[idx % N]; };   // sum over flat [0, idx)
    long long mx = 1;
    for (int cta = 0; cta < h->G; ++cta) {
      const long long a = (long long)cta * h->per, b = std::min<long long>(a + h->per, h->total);
      if (b > a) mx = std::max(mx, upto(b) - upto(a));
    }
    h->in_cap = mx;
    const size_t rec = c.precision == 32 ? sizeof(InArr<float>) : sizeof(InArr<double>);
    EQ_CUDA(h, ensure(h, &h->inbox, (size_t)2 * h->G * h->in_cap * rec));
    EQ_CUDA(h, ensure(h, (void**)&h->in_cnt, (size_t)2 * h->G * sizeof(int)));
    EQ_CUDA(h, ensure(h, (void**)&h->aoff, (size_t)B * N * sizeof(int)));
    EQ_CUDA(h, ensure(h, (void**)&h->aidx, (size_t)h->G * h->in_cap * sizeof(int)));
  }
  if (h->staged) {
    h->C = (h->cap + 3) / 4 * 4;
    const size_t pb = c.precision == 32 ? sizeof(long long) : sizeof(longlong2);
    EQ_CUDA(h, ensure(h, (void**)&h->qkeys, (size_t)B * N * h->C * sizeof(unsigned)));
    EQ_CUDA(h, ensure(h, &h->qpay, (size_t)B * N * h->C * pb));
    EQ_CUDA(h, ensure(h, (void**)&h->qdue, (size_t)B * N * sizeof(int)));
    // the step's popped sums, read by the ring kind's neuron pass
    EQ_CUDA(h, ensure(h, (void**)&h->acc, (size_t)2 * h->total * (c.precision == 32 ? 1 : 2) * sizeof(long long)));
  } else {
    EQ_CUDA(h, ensure(h, &h->q, qbytes));
  }
  EQ_CUDA(h, ensure(h, (void**)&h->meta, (size_t)B * N * sizeof(int4)));
  // one drop bit per possible event of a logged spike: grows with the log
  h->drop_cap = ((long long)h->log_cap * h->maxdeg + 31) / 32 * 32;
  EQ_CUDA(h, ensure(h, (void**)&h->drop_bits, (size_t)h->drop_cap / 8));
  return EQ_OK;
}

}  // namespace

extern "C" {

const char* eq_version(void) { return "eventq_b200 0.1.0 sm_100a"; }

const char* eq_last_error(const eq_handle* h) { return h ? h->err.c_str() : "null handle"; }

int eq_create(const eq_config* cfg, int device, eq_handle** out) {
  if (!cfg || !out) return EQ_ERR_CONFIGURATION;
  *out = nullptr;
  eq_handle* h = new eq_handle();
  h->cfg = *cfg;
  h->device = device;
  const eq_config& c = h->cfg;
  auto bad = [&](const std::string& m) {
    h->err = m;
    *out = h;
    return EQ_ERR_CONFIGURATION;
  };
  if (c.n_neurons < 2) return bad("a recurrent network needs n >= 2, got " + std::to_string(c.n_neurons));
  if (c.n_trials < 1) return bad("n_trials must be >= 1");
  if (c.t_steps < 1) return bad("t_steps must be >= 1, got " + std::to_string(c.t_steps));
  if (c.precision != 32 && c.precision != 64) return bad("precision must be 32 or 64");
  if (!(c.dt > 0.0)) return bad("dt must be positive");
  if (!(c.tau_m > 0.0)) return bad("tau_m must be positive, got " + std::to_string(c.tau_m));
  if (!(c.tau_syn > 0.0)) return bad("tau_syn must be positive, got " + std::to_string(c.tau_syn));
  if (!(c.v_th > c.v_reset)) return bad("threshold must sit above reset");
  if (c.kind != EQ_KIND_RING && c.kind != EQ_KIND_DONOTHING && c.kind != EQ_KIND_FIFORING &&
      c.kind != EQ_KIND_BINARYHEAP && c.kind != EQ_KIND_SORTEDARRAY && c.kind != EQ_KIND_LOSSYRING)
    return bad("unknown queue kind " + std::to_string(c.kind));
  if (c.capacity < 0) return bad("capacity must be >= 1, got " + std::to_string(c.capacity));
  if (c.max_ctas < 0) return bad("max_ctas must be >= 0");
  if (c.staged_queues < 0 || c.staged_queues > 2) return bad("staged_queues must be 0, 1 or 2");
  h->bounded = c.kind == EQ_KIND_FIFORING || c.kind == EQ_KIND_BINARYHEAP || c.kind == EQ_KIND_SORTEDARRAY;
  h->lossy = c.kind == EQ_KIND_LOSSYRING;
  if (c.exact_delivery && std::fabs(c.tau_m - c.tau_syn) < 1e-3 * c.tau_m)
    return bad("exact delivery splits the membrane/synapse eigenmodes and needs tau_m != tau_syn");
  h->total = (long long)c.n_neurons * c.n_trials;
  if (h->total >= (1LL << 31)) return bad("n_neurons * n_trials must be < 2^31");
  h->tsize = c.precision == 32 ? 4 : 8;
  DeviceGuard g(device);
  cudaDeviceProp prop;
  cudaError_t e = cudaGetDeviceProperties(&prop, device);
  if (e != cudaSuccess) {
    *out = h;
    return cuda_fail(h, e, "cudaGetDeviceProperties");
  }
  if (prop.major != 10) {
    *out = h;
    return fail(h, EQ_ERR_CUDA, "this build targets sm_100a (B200); device is sm_" +
                                    std::to_string(prop.major) + std::to_string(prop.minor));
  }
  h->n_sm = prop.multiProcessorCount;
  h->n_src = c.n_neurons;
  *out = h;
  int rc = setup_geometry(h);
  if (rc) return rc;
  const size_t T = h->tsize;
  EQ_CUDA(h, alloc(h, &h->I, h->total * T));
  EQ_CUDA(h, alloc(h, &h->V, h->total * T));
  EQ_CUDA(h, alloc(h, (void**)&h->refr, h->total * sizeof(int32_t)));
  EQ_CUDA(h, alloc(h, &h->lamV, h->total * T));
  EQ_CUDA(h, alloc(h, &h->lamI, h->total * T));
  EQ_CUDA(h, alloc(h, (void**)&h->gamp_bt, h->total * sizeof(double)));
  EQ_CUDA(h, alloc(h, (void**)&h->counters, (size_t)c.n_trials * 3 * sizeof(long long)));
  EQ_CUDA(h, alloc(h, (void**)&h->err_dev, kErrWords * sizeof(int)));
  EQ_CUDA(h, alloc(h, (void**)&h->bar, kBarWords * sizeof(unsigned)));
  EQ_CUDA(h, alloc(h, (void**)&h->log_count, sizeof(unsigned long long)));
  const size_t rec = c.precision == 32 ? sizeof(SpikeRec<float>) : sizeof(SpikeRec<double>);
  EQ_CUDA(h, alloc(h, &h->scratch, (size_t)h->G * h->per * rec));
  long long cap = c.max_spikes > 0 ? c.max_spikes
                                   : std::max<long long>(1LL << 20, h->total * (long long)c.t_steps / 32);
  h->log_cap = cap;
  EQ_CUDA(h, alloc(h, &h->log, (size_t)cap * rec));
  EQ_CUDA(h, alloc(h, (void**)&h->log_r0, (size_t)cap * sizeof(long long)));
  EQ_CUDA(h, alloc(h, (void**)&h->log_len, (size_t)cap * sizeof(int)));
  EQ_CUDA(h, alloc(h, &h->lt_log, (size_t)cap * T));
  EQ_CUDA(h, alloc(h, &h->lt_rem, (size_t)cap * T));
  rc = ensure_chunks(h, c.t_steps);
  if (rc) return rc;
  const char* tl = getenv("EQ_TIMELINE");
  if (tl && tl[0] == '1') {
    h->tl_steps = c.t_steps;
    size_t nb = (size_t)c.t_steps * h->G * 8 * sizeof(unsigned long long);
    EQ_CUDA(h, alloc(h, (void**)&h->tl_f, nb));
    EQ_CUDA(h, alloc(h, (void**)&h->tl_b, nb));
    EQ_CUDA(h, cudaMemset(h->tl_f, 0, nb));
    EQ_CUDA(h, cudaMemset(h->tl_b, 0, nb));
  }
  return EQ_OK;
}

int eq_destroy(eq_handle* h) {
  if (!h) return EQ_OK;
  {
    DeviceGuard g(h->device);
    for (void* p : h->owned) cudaFree(p);
  }
  delete h;
  return EQ_OK;
}

int eq_set_network(eq_handle* h, const int64_t* rowptr, const int32_t* col, const void* weight,
                   const void* delay, int64_t n_edges, void* stream) {
  if (!h) return EQ_ERR_CONFIGURATION;
  DeviceGuard g(h->device);
  cudaStream_t s = (cudaStream_t)stream;
  const eq_config& c = h->cfg;
  const int N = c.n_neurons;
  if (n_edges < 1) return fail(h, EQ_ERR_CONFIGURATION, "network has no edges");
  // validation scratch kept in the handle: the autograd shell calls this every
  // training step (RSNNFunction.forward), so no allocation happens per call
  EQ_CUDA(h, ensure(h, &h->ns_insum, (size_t)N * sizeof(long long)));
  EQ_CUDA(h, ensure(h, &h->ns_inocc, (size_t)N * sizeof(long long)));
  EQ_CUDA(h, ensure(h, &h->ns_indeg, (size_t)(N + 1) * sizeof(int)));   // +1: exclusive scan reads n+1
  EQ_CUDA(h, ensure(h, &h->ns_stats, 8 * sizeof(long long)));
  void *insum = h->ns_insum, *stats = h->ns_stats, *inocc = h->ns_inocc, *indeg = h->ns_indeg;
  long long init[8] = {1, -1LL, 0, 0, 1, 0, 0, 0};
  init[1] = (long long)~0ULL;
  EQ_CUDA(h, cudaMemsetAsync(insum, 0, (size_t)N * sizeof(long long), s));
  EQ_CUDA(h, cudaMemsetAsync(inocc, 0, (size_t)N * sizeof(long long), s));
  EQ_CUDA(h, cudaMemsetAsync(indeg, 0, (size_t)(N + 1) * sizeof(int), s));
  EQ_CUDA(h, cudaMemcpyAsync(stats, init, sizeof init, cudaMemcpyHostToDevice, s));
  int homog = c.kind == EQ_KIND_FIFORING;
  if (c.precision == 32)
    k_net_stats<float><<<(h->n_src + 127) / 128, 128, 0, s>>>(
        h->n_src, N, h->src_off, rowptr, col, (const float*)weight, (const float*)delay, (float)c.dt, homog,
        (long long*)insum, (long long*)stats, (long long*)inocc, (int*)indeg);
  else
    k_net_stats<double><<<(h->n_src + 127) / 128, 128, 0, s>>>(
        h->n_src, N, h->src_off, rowptr, col, (const double*)weight, (const double*)delay, c.dt, homog,
        (long long*)insum, (long long*)stats, (long long*)inocc, (int*)indeg);
  k_max_ll<<<256, 256, 0, s>>>((const long long*)insum, N, (long long*)stats + 2);
  k_max_ll<<<256, 256, 0, s>>>((const long long*)inocc, N, (long long*)stats + 3);
  k_max_ll<<<256, 256, 0, s>>>((const int*)indeg, N, (long long*)stats + 5);
  k_col_fingerprint<<<296, 256, 0, s>>>(col, n_edges, (unsigned long long*)stats + 6);
  h->launches += 5;
  long long st[8];
  EQ_CUDA(h, cudaMemcpyAsync(st, stats, sizeof st, cudaMemcpyDeviceToHost, s));
  EQ_CUDA(h, cudaStreamSynchronize(s));

  if ((unsigned long long)st[1] != ~0ULL) {
    unsigned long long key = (unsigned long long)st[1];
    long long x = (long long)(key >> 2);
    int code = (int)(key & 3);
    // locate the row of edge x on the host (validation path only)
    std::vector<int64_t> rp(h->n_src + 1);
    EQ_CUDA(h, cudaMemcpy(rp.data(), rowptr, (h->n_src + 1) * sizeof(int64_t), cudaMemcpyDeviceToHost));
    int i = (int)(std::upper_bound(rp.begin(), rp.end(), (int64_t)x) - rp.begin()) - 1;
    int j = -1;
    EQ_CUDA(h, cudaMemcpy(&j, col + x, sizeof(int), cudaMemcpyDeviceToHost));
    double dv = 0.0, d0 = 0.0;
    if (c.precision == 32) {
      float f, f0;
      EQ_CUDA(h, cudaMemcpy(&f, (const float*)delay + x, 4, cudaMemcpyDeviceToHost));
      EQ_CUDA(h, cudaMemcpy(&f0, delay, 4, cudaMemcpyDeviceToHost));
      dv = f;
      d0 = f0;
    } else {
      EQ_CUDA(h, cudaMemcpy(&dv, (const double*)delay + x, 8, cudaMemcpyDeviceToHost));
      EQ_CUDA(h, cudaMemcpy(&d0, delay, 8, cudaMemcpyDeviceToHost));
    }
    char buf[256];
    if (code == 1)
      snprintf(buf, sizeof buf, "CSR edge %lld (%d,%d): targets must be in [0,n), not the source, ascending",
               x, i, j);
    else if (code == 2)
      snprintf(buf, sizeof buf, "delay on edge (%d,%d) is %g, below one step (%g)", i, j, dv, c.dt);
    else
      snprintf(buf, sizeof buf,
               "fiforing supports homogeneous delays only, but edge (%d,%d) has %g while another edge has %g", i, j,
               dv, d0);
    return fail(h, EQ_ERR_CONFIGURATION, buf);
  }
  h->horizon = (int)st[0] + 1;           // network.py:188-198
  h->maxdeg = (int)std::max<long long>(1, st[4]);
  h->R = h->horizon + 1;                 // + one slot for in-phase pop/scatter overlap
  // fixed-point fraction bits: largest F with 4*max_in*2^F <= 2^(bits-2)
  double max_in = std::ldexp((double)st[2], -40);
  int bits = c.precision == 32 ? 32 : 64;
  if (max_in <= 0.0) {
    h->frac_bits = bits - 2;
  } else {
    int e;
    double m = std::frexp(4.0 * max_in, &e);
    int ceil_log2 = (m == 0.5) ? e - 1 : e;
    h->frac_bits = (bits - 2) - ceil_log2;
  }
  h->frac_safe = h->frac_bits;
  h->scale = std::ldexp(1.0, h->frac_bits);
  h->inv_scale = std::ldexp(1.0, -h->frac_bits);
  h->rowptr = rowptr;
  h->col = col;
  h->w = weight;
  h->d = delay;
  h->E = n_edges;
  if (h->horizon > 0x7ffe) return fail(h, EQ_ERR_CONFIGURATION, "delay horizon beyond 32766 steps");
  EQ_CUDA(h, ensure(h, (void**)&h->dcode, (size_t)n_edges * sizeof(unsigned short)));
  EQ_CUDA(h, ensure(h, &h->edges, (size_t)n_edges * (c.precision == 32 ? sizeof(EdgeRec<float>)
                                                                         : sizeof(EdgeRec<double>))));
  if (c.precision == 32)
    k_pack_edges<float><<<1184, 256, 0, s>>>(col, (const float*)weight, (const float*)delay, n_edges, (float)c.dt,
                                             h->dcode, (EdgeRec<float>*)h->edges);
  else
    k_pack_edges<double><<<1184, 256, 0, s>>>(col, (const double*)weight, (const double*)delay, n_edges, c.dt,
                                              h->dcode, (EdgeRec<double>*)h->edges);
  h->launches += 1;
  // heap / sorted run by admission on the calendar (eq_ring.cuh) unless the
  // queue structures are asked for (staged_queues 1 or 2) or the capacity
  // needs more than the record's 16-bit occupancy fields
  h->adm = false;
  // FIFO: with its homogeneous delay on the step grid every event of a step
  // has the same due step, so dues never decrease and the tail-key check
  // (queues.py:220-224) cannot fire: its accepted sets and pops are the heap's
  bool fifo_ok = c.kind != EQ_KIND_FIFORING;
  if (!fifo_ok && c.staged_queues == 0) {
    unsigned short code0 = 0x8000;
    EQ_CUDA(h, cudaMemcpyAsync(&code0, h->dcode, sizeof code0, cudaMemcpyDeviceToHost, s));
    EQ_CUDA(h, cudaStreamSynchronize(s));
    fifo_ok = (code0 & 0x8000) == 0;
  }
  if (h->bounded && fifo_ok && c.staged_queues == 0) {
    const long long cap_ref = c.capacity > 0 ? c.capacity : (long long)h->horizon * (N - 1) + 1;
    // 16-bit occupancy fields; 16-bit arrival counters (a step delivers at most
    // the in-degree to a queue)
    h->adm = std::min<long long>(cap_ref, std::max<long long>(st[3], 1)) < 32768 && st[5] < 65536;
  }
  h->cal = c.kind == EQ_KIND_RING || h->adm;
  // queue storage
  size_t words = h->cal ? (size_t)c.n_trials * h->R * N * (c.precision == 32 ? 1 : 2) : 1;
  if (h->lossy) {
    // LossyRingQueue capacity as the reference wires it (network.py:327):
    // queue_capacity or horizon*(n-1)+1; >= horizon never aliases
    h->lossy_cap = c.capacity > 0 ? c.capacity : (long long)h->horizon * (N - 1) + 1;
    h->lossy_slots = (int)std::min<long long>(h->lossy_cap, h->horizon) + 1;
    words = (size_t)c.n_trials * h->lossy_slots * N * (c.precision == 32 ? 1 : 2);
  }
  h->ring_words = words;
  {
    long long* before = h->ring;
    EQ_CUDA(h, ensure(h, (void**)&h->ring, words * sizeof(long long)));
    if (h->ring != before) h->ring_clean = false;
  }
  if (h->cal) {
    const int wd = c.precision == 32 ? 1 : 2;
    h->NB = h->R;
    if (h->NB > 512)
      return fail(h, EQ_ERR_CONFIGURATION, "ring horizon " + std::to_string(h->horizon) +
                                               " steps exceeds the calendar's 511");
    // per-CTA bucket capacity: events due at one step from one CTA's fan-out
    // share at a 1/64 spike rate (3.5x the BASELINE C3 rate); overflow spills
    // to the DRAM ring, so this only sizes the fast path
    long long avg_deg = std::max<long long>(1, n_edges / N);
    h->cap_b = std::max<long long>(256, (h->total * avg_deg / 64 + h->G - 1) / h->G);
    if (h->cap_b > (1LL << 30)) h->cap_b = 1LL << 30;
    h->cap_b_alloc = h->cap_b;
    EQ_CUDA(h, ensure(h, (void**)&h->acc, (size_t)2 * h->total * wd * sizeof(long long)));
    EQ_CUDA(h, ensure(h, (void**)&h->bk, (size_t)h->G * h->NB * h->cap_b * (wd == 1 ? 2 : 4) * sizeof(long long)));
    EQ_CUDA(h, ensure(h, (void**)&h->bk_cnt, (size_t)h->G * h->NB * sizeof(int)));
    EQ_CUDA(h, ensure(h, (void**)&h->ring_dirty, (size_t)h->R * sizeof(int)));
  }
  EQ_CUDA(h, ensure(h, &h->lam, (size_t)c.n_trials * h->R * N * 2 * h->tsize));
  if (h->bounded) {
    int rc = setup_bounded(h, (const int*)indeg, st[3], s, reinterpret_cast<const unsigned long long*>(st + 6));
    if (rc) return rc;
  }
  h->net_set = true;
  return eq_reset(h, stream);
}

int eq_set_drive(eq_handle* h, const uint32_t* mask, const void* amplitude, void* stream) {
  if (!h) return EQ_ERR_CONFIGURATION;
  (void)stream;
  h->mask = mask;
  h->amp = amplitude;
  h->drive_set = true;
  return EQ_OK;
}

int eq_reset(eq_handle* h, void* stream) {
  if (!h) return EQ_ERR_CONFIGURATION;
  if (!h->net_set) return fail(h, EQ_ERR_CONFIGURATION, "eq_set_network must come first");
  DeviceGuard g(h->device);
  cudaStream_t s = (cudaStream_t)stream;
  const size_t T = h->tsize;
  if (h->cal) {
    const int wd = h->cfg.precision == 32 ? 1 : 2;
    if (!h->ring_clean) {
      EQ_CUDA(h, cudaMemsetAsync(h->ring, 0, h->ring_words * sizeof(long long), s));
      if (h->adm) EQ_CUDA(h, cudaMemsetAsync(h->cring, 0, (size_t)h->total * h->R * sizeof(int), s));
      h->ring_clean = true;
    } else {
      const long long row_words = (long long)h->cfg.n_neurons * wd;
      k_clear_dirty_rows<<<dim3((unsigned)std::min<long long>((row_words + 255) / 256, 64),
                              (unsigned)(h->cfg.n_trials * h->R)), 256, 0, s>>>(h->ring, h->ring_dirty, h->R,
                                                                                row_words);
      h->launches += 1;
      if (h->adm) {
        k_clear_dirty_rows_i32<<<dim3((unsigned)std::min<long long>((h->cfg.n_neurons + 255) / 256, 64),
                                      (unsigned)(h->cfg.n_trials * h->R)), 256, 0, s>>>(h->cring, h->ring_dirty, h->R,
                                                                                        h->cfg.n_neurons);
        h->launches += 1;
      }
    }
    EQ_CUDA(h, cudaMemsetAsync(h->acc, 0, (size_t)2 * h->total * wd * sizeof(long long), s));
    EQ_CUDA(h, cudaMemsetAsync(h->bk_cnt, 0, (size_t)h->G * h->NB * sizeof(int), s));
    EQ_CUDA(h, cudaMemsetAsync(h->ring_dirty, 0, (size_t)h->R * sizeof(int), s));
  } else if (!h->ring_clean || h->lossy) {   // a lossy ring's pending events sit in its slots
    EQ_CUDA(h, cudaMemsetAsync(h->ring, 0, h->ring_words * sizeof(long long), s));
    h->ring_clean = true;
  }
  EQ_CUDA(h, cudaMemsetAsync(h->I, 0, h->total * T, s));
  if (h->cfg.precision == 32)
    k_fill<float><<<296, 256, 0, s>>>((float*)h->V, h->total, (float)h->cfg.v_reset);
  else
    k_fill<double><<<296, 256, 0, s>>>((double*)h->V, h->total, h->cfg.v_reset);
  h->launches += 1;
  EQ_CUDA(h, cudaMemsetAsync(h->refr, 0, h->total * sizeof(int32_t), s));
  EQ_CUDA(h, cudaMemsetAsync(h->counters, 0, (size_t)h->cfg.n_trials * 3 * sizeof(long long), s));
  EQ_CUDA(h, cudaMemsetAsync(h->err_dev, 0, kErrWords * sizeof(int), s));
  EQ_CUDA(h, cudaMemsetAsync(h->bar, 0, kBarWords * sizeof(unsigned), s));
  EQ_CUDA(h, cudaMemsetAsync(h->log_count, 0, sizeof(unsigned long long), s));
  EQ_CUDA(h, cudaMemsetAsync(h->step_start, 0, sizeof(long long), s));
  if (h->adm) {
    EQ_CUDA(h, cudaMemsetAsync(h->drop_bits, 0, (size_t)h->drop_cap / 8, s));
    EQ_CUDA(h, cudaMemsetAsync(h->adm_ctr, 0, (size_t)h->totp * (2 * 4 + 2 * 2 + 3 * 2), s));
    EQ_CUDA(h, cudaMemsetAsync(h->fl_cnt, 0, (size_t)2 * h->G * sizeof(int), s));
    EQ_CUDA(h, cudaMemsetAsync(h->lpos, 0xFF, (size_t)3 * h->total * sizeof(int), s));
  } else if (h->bounded) {
    const int B = h->cfg.n_trials, N = h->cfg.n_neurons;
    EQ_CUDA(h, cudaMemsetAsync(h->acnt, 0, (size_t)2 * B * N * sizeof(int), s));
    EQ_CUDA(h, cudaMemsetAsync(h->drop_bits, 0, (size_t)h->drop_cap / 8, s));
    if (h->staged) {
      k_meta_init_bq<<<592, 256, 0, s>>>(h->meta, h->qdue, (long long)B * N);
      EQ_CUDA(h, cudaMemsetAsync(h->in_cnt, 0, (size_t)2 * h->G * sizeof(int), s));
      EQ_CUDA(h, cudaMemsetAsync(h->acc, 0, (size_t)2 * h->total * (h->cfg.precision == 32 ? 1 : 2) *
                                                sizeof(long long), s));
    } else
      k_meta_init<<<592, 256, 0, s>>>(h->meta, (long long)B * N);
    h->launches += 1;
  }
  h->steps_done = 0;
  h->log_used = 0;
  h->imp_n = 0;
  h->imp_blocks.clear();
  h->bwd_cursor = -1;
  return EQ_OK;
}

int eq_run(eq_handle* h, int32_t n_steps, void* v_trace, void* stream) {
  if (!h) return EQ_ERR_CONFIGURATION;
  if (!h->net_set || !h->drive_set) return fail(h, EQ_ERR_CONFIGURATION, "network and drive must be set");
  if (n_steps < 0) return fail(h, EQ_ERR_CONFIGURATION, "n_steps must be >= 0");
  if (n_steps == 0) {   // partitioned: only fan out the spikes imported at this step
    std::array<long long, 4>* blk = find_block(h, h->steps_done);
    if (!blk || (*blk)[3]) return EQ_OK;
  }
  DeviceGuard g(h->device);
  int rc = ensure_chunks(h, h->steps_done + n_steps);
  if (rc) return rc;
  cudaStream_t s = (cudaStream_t)stream;
  EQ_CUDA(h, cudaMemsetAsync(h->bar, 0, kBarWords * sizeof(unsigned), s));
  // step_start[m0+1 .. m1]: sentinel -1 until the barrier after each phase publishes it
  if (n_steps > 0)
    EQ_CUDA(h, cudaMemsetAsync(h->step_start + h->steps_done + 1, 0xFF, (size_t)n_steps * sizeof(long long), s));
  if (h->cfg.precision == 32) return launch_forward<float>(h, n_steps, v_trace, s);
  return launch_forward<double>(h, n_steps, v_trace, s);
}

int eq_forward(eq_handle* h, void* v_out, void* i_out, void* v_trace, void* stream) {
  int rc = eq_reset(h, stream);
  if (rc) return rc;
  rc = eq_run(h, h->cfg.t_steps, v_trace, stream);
  if (rc) return rc;
  DeviceGuard g(h->device);
  cudaStream_t s = (cudaStream_t)stream;
  if (v_out) EQ_CUDA(h, cudaMemcpyAsync(v_out, h->V, h->total * h->tsize, cudaMemcpyDeviceToDevice, s));
  if (i_out) EQ_CUDA(h, cudaMemcpyAsync(i_out, h->I, h->total * h->tsize, cudaMemcpyDeviceToDevice, s));
  return EQ_OK;
}

int eq_forward_jvp(eq_handle* h, int32_t n_dir, const int32_t* dir_kind, const int64_t* dir_index, double* v_out,
                   double* v_tangent, void* stream) {
  if (!h) return EQ_ERR_CONFIGURATION;
  const eq_config& c = h->cfg;
  if (c.precision != 64 || c.kind != EQ_KIND_RING)
    return fail(h, EQ_ERR_CONFIGURATION, "forward-mode runs need precision 64 and the ring kind");
  if (h->partitioned) return fail(h, EQ_ERR_CONFIGURATION, "forward-mode runs on partitioned networks are not supported");
  if (!h->net_set || !h->drive_set) return fail(h, EQ_ERR_CONFIGURATION, "network and drive must be set");
  if (n_dir < 1 || !dir_kind || !dir_index || !v_tangent)
    return fail(h, EQ_ERR_CONFIGURATION, "need >= 1 direction and a tangent output");
  for (int d = 0; d < n_dir; ++d) {
    const long long lim = dir_kind[d] == 2 ? c.n_neurons : h->E;
    if (dir_kind[d] < 0 || dir_kind[d] > 2 || dir_index[d] < 0 || dir_index[d] >= lim)
      return fail(h, EQ_ERR_CONFIGURATION, "direction " + std::to_string(d) + " is not a weight/delay edge or a "
                                               "drive neuron");
  }
  DeviceGuard g(h->device);
  cudaStream_t s = (cudaStream_t)stream;
  int rc = eq_reset(h, stream);
  if (rc) return rc;
  const int N = c.n_neurons, B = c.n_trials, D = n_dir;
  const size_t td = (size_t)B * D * N;
  void *tI = nullptr, *tV = nullptr, *tslot = nullptr, *dk = nullptr, *di = nullptr, *sidx = nullptr, *st = nullptr,
       *std_ = nullptr, *sn = nullptr, *off = nullptr, *nev = nullptr, *mdev = nullptr, *pa = nullptr, *pv = nullptr,
       *pr = nullptr, *pku = nullptr, *pinfo = nullptr;
  // scratch kept in the handle between runs (grow-only, like the other buffers)
  const int cap = (int)std::min<long long>(h->total, 1 << 30);
  const std::vector<std::pair<void**, size_t>> list{
           {&tI, td * 8}, {&tV, td * 8}, {&tslot, td * h->R * 4 * 8}, {&dk, (size_t)D * 4}, {&di, (size_t)D * 8},
           {&sidx, (size_t)cap * 4}, {&st, (size_t)cap * 8}, {&std_, (size_t)cap * D * 8}, {&sn, 16},
           {&off, ((size_t)cap + 1) * 8}, {&nev, 16}, {&mdev, 16}, {&pa, (size_t)h->total * 8},
           {&pv, (size_t)h->total * 8}, {&pr, (size_t)h->total * 8}, {&pku, (size_t)h->total * 8},
           {&pinfo, (size_t)h->total * 8}};
  if (list.size() > sizeof(h->jvp_buf) / sizeof(void*)) return fail(h, EQ_ERR_CUDA, "jvp scratch table too small");
  for (const auto& pr : list) {
    void** slot = &h->jvp_buf[&pr - &*list.begin()];
    EQ_CUDA(h, ensure(h, slot, pr.second));
    *pr.first = *slot;
  }
  EQ_CUDA(h, cudaMemsetAsync(tI, 0, td * 8, s));
  EQ_CUDA(h, cudaMemsetAsync(tV, 0, td * 8, s));
  EQ_CUDA(h, cudaMemsetAsync(tslot, 0, td * h->R * 4 * 8, s));
  EQ_CUDA(h, cudaMemcpyAsync(dk, dir_kind, (size_t)D * 4, cudaMemcpyHostToDevice, s));
  EQ_CUDA(h, cudaMemcpyAsync(di, dir_index, (size_t)D * 8, cudaMemcpyHostToDevice, s));
  JvpArgs A;
  A.N = N;
  A.B = B;
  A.D = D;
  A.R = h->R;
  A.refractory = c.refractory_steps;
  A.exact = c.exact_delivery;
  A.total = h->total;
  A.c = consts<double>(h);
  A.net = netview<double>(h);
  A.I = (double*)h->I;
  A.V = (double*)h->V;
  A.refr = h->refr;
  A.ring = h->ring;
  A.tI = (double*)tI;
  A.tV = (double*)tV;
  A.tslot = (double*)tslot;
  A.dkind = (const int*)dk;
  A.dindex = (const long long*)di;
  A.spk_idx = (int*)sidx;
  A.spk_t = (double*)st;
  A.spk_tdot = (double*)std_;
  A.spk_n = (int*)sn;
  A.spk_cap = cap;
  A.counters = h->counters;
  A.err = h->err_dev;
  A.m_dev = (int*)mdev;
  A.pa = (double*)pa;
  A.pv = (double*)pv;
  A.pr = (double*)pr;
  A.pku = (double*)pku;
  A.pinfo = (int2*)pinfo;
  EQ_CUDA(h, cudaMemsetAsync(mdev, 0, 4, s));
  EQ_CUDA(h, cudaMemsetAsync(sn, 0, 4, s));
  const int ub = (int)((h->total + 255) / 256);
  const long long tb = (h->total * D + 255) / 256;
  if (tb > 0x7fffffffLL) return fail(h, EQ_ERR_CONFIGURATION, "too many directions x neuron-trials");
  auto step = [&](cudaStream_t q) {
    k_jvp_update<<<ub, 256, 0, q>>>(A);
    k_jvp_tangent<<<(unsigned)tb, 256, 0, q>>>(A);
    k_jvp_offsets<<<1, 1024, 0, q>>>(A, (long long*)off, (long long*)nev);
    k_jvp_fanout<<<1184, 256, 0, q>>>(A, (const long long*)nev, (const long long*)off);
    k_jvp_next<<<1, 1, 0, q>>>(A);
  };
  // a block of kGraphSteps steps captured once on a private stream and
  // replayed; the remainder launched directly; ordered with the caller's stream
  constexpr int kGraphSteps = 50;
  const int nblk = c.t_steps / kGraphSteps;
  cudaStream_t gs = nullptr;
  cudaEvent_t ev0 = nullptr, ev1 = nullptr;
  cudaGraph_t graph = nullptr;
  cudaGraphExec_t exec = nullptr;
  bool ok = nblk >= 2 && cudaStreamCreateWithFlags(&gs, cudaStreamNonBlocking) == cudaSuccess &&
            cudaEventCreateWithFlags(&ev0, cudaEventDisableTiming) == cudaSuccess &&
            cudaEventCreateWithFlags(&ev1, cudaEventDisableTiming) == cudaSuccess;
  if (ok) {
    ok = cudaStreamBeginCapture(gs, cudaStreamCaptureModeThreadLocal) == cudaSuccess;
    if (ok) {
      for (int k = 0; k < kGraphSteps; ++k) step(gs);
      ok = cudaStreamEndCapture(gs, &graph) == cudaSuccess &&
           cudaGraphInstantiate(&exec, graph, 0) == cudaSuccess;
    }
  }
  if (ok) {
    EQ_CUDA(h, cudaEventRecord(ev0, s));
    EQ_CUDA(h, cudaStreamWaitEvent(gs, ev0, 0));
    for (int k = 0; k < nblk; ++k) EQ_CUDA(h, cudaGraphLaunch(exec, gs));
    for (int m = nblk * kGraphSteps; m < c.t_steps; ++m) step(gs);
    EQ_CUDA(h, cudaEventRecord(ev1, gs));
    EQ_CUDA(h, cudaStreamWaitEvent(s, ev1, 0));
  } else {
    cudaGetLastError();
    for (int m = 0; m < c.t_steps; ++m) step(s);
  }
  h->launches += 5LL * c.t_steps;
  if (gs) cudaStreamSynchronize(gs);   // the graph and stream outlive their launches
  if (exec) cudaGraphExecDestroy(exec);
  if (graph) cudaGraphDestroy(graph);
  if (ev0) cudaEventDestroy(ev0);
  if (ev1) cudaEventDestroy(ev1);
  if (gs) cudaStreamDestroy(gs);
  EQ_CUDA(h, cudaGetLastError());
  if (v_out) EQ_CUDA(h, cudaMemcpyAsync(v_out, h->V, h->total * 8, cudaMemcpyDeviceToDevice, s));
  // [B][D][N] -> [D][B][N]
  for (int d = 0; d < D; ++d)
    for (int b = 0; b < B; ++b)
      EQ_CUDA(h, cudaMemcpyAsync(v_tangent + ((size_t)d * B + b) * N, (double*)tV + ((size_t)b * D + d) * N,
                                 (size_t)N * 8, cudaMemcpyDeviceToDevice, s));
  rc = check_err(h, s);
  h->steps_done = 0;   // the spike log / queues of eq_run are not populated by this path
  h->ring_clean = false;   // its pending events sit in unflagged ring rows
  return rc;
}

int eq_get_state(eq_handle* h, void* v_out, void* i_out, void* stream) {
  if (!h) return EQ_ERR_CONFIGURATION;
  DeviceGuard g(h->device);
  cudaStream_t s = (cudaStream_t)stream;
  if (v_out) EQ_CUDA(h, cudaMemcpyAsync(v_out, h->V, h->total * h->tsize, cudaMemcpyDeviceToDevice, s));
  if (i_out) EQ_CUDA(h, cudaMemcpyAsync(i_out, h->I, h->total * h->tsize, cudaMemcpyDeviceToDevice, s));
  return EQ_OK;
}

int eq_backward(eq_handle* h, const void* v_bar, const void* i_bar, double* grad_w, double* grad_d,
                double* grad_amp, void* stream) {
  if (!h) return EQ_ERR_CONFIGURATION;
  int rc = eq_backward_begin(h, v_bar, i_bar, grad_w, grad_d, grad_amp, stream);
  if (rc) return rc;
  return eq_backward_window(h, 0, stream);
}

int eq_backward_begin(eq_handle* h, const void* v_bar, const void* i_bar, double* grad_w, double* grad_d,
                      double* grad_amp, void* stream) {
  if (!h) return EQ_ERR_CONFIGURATION;
  if (h->steps_done < 1) return fail(h, EQ_ERR_CONFIGURATION, "backward needs a forward run first");
  if (!v_bar || !grad_w || !grad_d) return fail(h, EQ_ERR_CONFIGURATION, "v_bar, grad_w, grad_d are required");
  DeviceGuard g(h->device);
  cudaStream_t s = (cudaStream_t)stream;
  if (h->cfg.precision == 32) return backward_begin<float>(h, v_bar, i_bar, grad_w, grad_d, grad_amp, s);
  return backward_begin<double>(h, v_bar, i_bar, grad_w, grad_d, grad_amp, s);
}

int eq_backward_window(eq_handle* h, int32_t m_lo, void* stream) {
  if (!h) return EQ_ERR_CONFIGURATION;
  if (h->bwd_cursor < 0) return fail(h, EQ_ERR_CONFIGURATION, "eq_backward_begin must come first");
  if (m_lo < 0 || m_lo >= h->bwd_cursor)
    return fail(h, EQ_ERR_CONFIGURATION, "reverse window start " + std::to_string(m_lo) + " outside [0, " +
                                             std::to_string(h->bwd_cursor) + ")");
  DeviceGuard g(h->device);
  cudaStream_t s = (cudaStream_t)stream;
  if (h->cfg.precision == 32) return launch_backward<float>(h, m_lo, s);
  return launch_backward<double>(h, m_lo, s);
}

int eq_set_partition(eq_handle* h, int32_t n_global, int32_t src_offset) {
  if (!h) return EQ_ERR_CONFIGURATION;
  if (h->cfg.kind != EQ_KIND_RING)
    return fail(h, EQ_ERR_CONFIGURATION, "partitioned networks support the ring kind (bounded kinds insert in "
                                         "global source order, which needs the whole step's spikes)");
  if (src_offset < 0 || (long long)src_offset + h->cfg.n_neurons > n_global)
    return fail(h, EQ_ERR_CONFIGURATION, "partition [" + std::to_string(src_offset) + ", " +
                                             std::to_string((long long)src_offset + h->cfg.n_neurons) +
                                             ") outside the " + std::to_string(n_global) + "-neuron network");
  h->n_src = n_global;
  h->src_off = src_offset;
  h->partitioned = true;
  h->net_set = false;   // the CSR must be (re)validated with the new row count
  return EQ_OK;
}

int eq_set_frac_bits(eq_handle* h, int32_t frac_bits) {
  if (!h) return EQ_ERR_CONFIGURATION;
  if (!h->net_set) return fail(h, EQ_ERR_CONFIGURATION, "eq_set_network must come first");
  if (frac_bits < 0 || frac_bits > h->frac_safe)
    return fail(h, EQ_ERR_CONFIGURATION, "fraction bits " + std::to_string(frac_bits) + " outside [0, " +
                                             std::to_string(h->frac_safe) + "] (overflow-free bound)");
  h->frac_bits = frac_bits;
  h->scale = std::ldexp(1.0, frac_bits);
  h->inv_scale = std::ldexp(1.0, -frac_bits);
  return EQ_OK;
}

int eq_export_spikes(eq_handle* h, int32_t step_lo, int32_t step_hi, void* out, int64_t* n_out, void* stream) {
  if (!h) return EQ_ERR_CONFIGURATION;
  if (step_lo < 0 || step_hi < step_lo || step_hi > h->steps_done)
    return fail(h, EQ_ERR_CONFIGURATION, "export window [" + std::to_string(step_lo) + ", " +
                                             std::to_string(step_hi) + ") outside the run");
  DeviceGuard g(h->device);
  cudaStream_t s = (cudaStream_t)stream;
  long long ss[2];
  EQ_CUDA(h, cudaMemcpyAsync(&ss[0], h->step_start + step_lo, sizeof(long long), cudaMemcpyDeviceToHost, s));
  EQ_CUDA(h, cudaMemcpyAsync(&ss[1], h->step_start + step_hi, sizeof(long long), cudaMemcpyDeviceToHost, s));
  EQ_CUDA(h, cudaStreamSynchronize(s));
  const long long n = ss[1] - ss[0];
  if (n_out) *n_out = n;
  if (!out || n == 0) return EQ_OK;
  const int blocks = (int)std::min<long long>((n + 255) / 256, 4096);
  if (h->cfg.precision == 32)
    k_export<float><<<blocks, 256, 0, s>>>((const SpikeRec<float>*)h->log, h->step_start, step_lo, step_hi,
                                           h->cfg.n_neurons, h->src_off, (ExRec<float>*)out);
  else
    k_export<double><<<blocks, 256, 0, s>>>((const SpikeRec<double>*)h->log, h->step_start, step_lo, step_hi,
                                            h->cfg.n_neurons, h->src_off, (ExRec<double>*)out);
  h->launches += 1;
  EQ_CUDA(h, cudaGetLastError());
  return EQ_OK;
}

int eq_import_spikes(eq_handle* h, const void* recs, int64_t n, void* stream) {
  if (!h) return EQ_ERR_CONFIGURATION;
  if (!h->partitioned) return fail(h, EQ_ERR_CONFIGURATION, "eq_set_partition must come first");
  if (!h->net_set) return fail(h, EQ_ERR_CONFIGURATION, "eq_set_network must come first");
  if (n < 0 || (n > 0 && !recs)) return fail(h, EQ_ERR_CONFIGURATION, "bad import batch");
  if (find_block(h, h->steps_done))
    return fail(h, EQ_ERR_CONFIGURATION, "spikes already imported for the launch at step " +
                                             std::to_string(h->steps_done));
  if (n == 0) return EQ_OK;
  DeviceGuard g(h->device);
  cudaStream_t s = (cudaStream_t)stream;
  const size_t rec = h->cfg.precision == 32 ? sizeof(SpikeRec<float>) : sizeof(SpikeRec<double>);
  if (h->imp_n + n > h->imp_cap) {
    const long long ncap = std::max<long long>(h->imp_n + n, 2 * h->imp_cap);
    void *a = nullptr, *b = nullptr, *c = nullptr, *d = nullptr;
    EQ_CUDA(h, alloc(h, &a, (size_t)ncap * rec));
    EQ_CUDA(h, alloc(h, &b, (size_t)ncap * sizeof(long long)));
    EQ_CUDA(h, alloc(h, &c, (size_t)ncap * sizeof(int)));
    EQ_CUDA(h, alloc(h, &d, (size_t)ncap * h->tsize));
    if (h->imp_n) {
      EQ_CUDA(h, cudaMemcpyAsync(a, h->imp, (size_t)h->imp_n * rec, cudaMemcpyDeviceToDevice, s));
      EQ_CUDA(h, cudaMemcpyAsync(b, h->imp_r0, (size_t)h->imp_n * sizeof(long long), cudaMemcpyDeviceToDevice, s));
      EQ_CUDA(h, cudaMemcpyAsync(c, h->imp_len, (size_t)h->imp_n * sizeof(int), cudaMemcpyDeviceToDevice, s));
      EQ_CUDA(h, cudaStreamSynchronize(s));
    }
    release(h, h->imp);
    release(h, h->imp_r0);
    release(h, h->imp_len);
    release(h, h->imp_lt);
    h->imp = a;
    h->imp_r0 = (long long*)b;
    h->imp_len = (int*)c;
    h->imp_lt = d;
    h->imp_cap = ncap;
  }
  const long long k0 = h->imp_n;
  const int blocks = (int)std::min<long long>((n + 255) / 256, 4096);
  if (h->cfg.precision == 32)
    k_import<float><<<blocks, 256, 0, s>>>((const ExRec<float>*)recs, n, h->rowptr, h->n_src, h->src_off,
                                           h->cfg.n_neurons, h->cfg.n_trials, h->cfg.n_neurons, h->steps_done,
                                           (SpikeRec<float>*)h->imp + k0, h->imp_r0 + k0, h->imp_len + k0,
                                           h->err_dev);
  else
    k_import<double><<<blocks, 256, 0, s>>>((const ExRec<double>*)recs, n, h->rowptr, h->n_src, h->src_off,
                                            h->cfg.n_neurons, h->cfg.n_trials, h->cfg.n_neurons, h->steps_done,
                                            (SpikeRec<double>*)h->imp + k0, h->imp_r0 + k0, h->imp_len + k0,
                                            h->err_dev);
  h->launches += 1;
  EQ_CUDA(h, cudaGetLastError());
  int e[4];
  EQ_CUDA(h, cudaMemcpyAsync(e, h->err_dev, sizeof e, cudaMemcpyDeviceToHost, s));
  EQ_CUDA(h, cudaStreamSynchronize(s));
  if (e[0]) {
    EQ_CUDA(h, cudaMemsetAsync(h->err_dev, 0, kErrWords * sizeof(int), s));
    char buf[200];
    snprintf(buf, sizeof buf, "imported spike (source %d, trial %d, step %d) is not a remote spike of an "
                              "earlier step", e[3], e[2], e[1]);
    return fail(h, EQ_ERR_CONFIGURATION, buf);
  }
  h->imp_blocks.push_back({(long long)h->steps_done, k0, (long long)n, 0LL});
  h->imp_n += n;
  return EQ_OK;
}

int eq_get_import_adjoints(eq_handle* h, int32_t start_step, void* out, void* stream) {
  if (!h) return EQ_ERR_CONFIGURATION;
  std::array<long long, 4>* blk = find_block(h, start_step);
  if (!blk) return EQ_OK;
  if (h->bwd_cursor < 0 || h->bwd_cursor > start_step)
    return fail(h, EQ_ERR_CONFIGURATION, "the reverse pass has not reached step " + std::to_string(start_step));
  DeviceGuard g(h->device);
  EQ_CUDA(h, cudaMemcpyAsync(out, (char*)h->imp_lt + (*blk)[1] * h->tsize, (size_t)(*blk)[2] * h->tsize,
                             cudaMemcpyDeviceToDevice, (cudaStream_t)stream));
  return EQ_OK;
}

}  // extern "C"

namespace {
PeerTable peer_table(const eq_handle* h) {
  PeerTable t{};
  t.P = (int)h->peers.size();
  t.me = h->peer_me;
  for (int q = 0; q < t.P; ++q) {
    const eq_handle* p = h->peers[q];
    t.d[q].log = p->log;
    t.d[q].step_start = p->step_start;
    t.d[q].imp_lt = p->imp_lt;
    t.d[q].blk = p->peer_blk;
    t.d[q].N = p->cfg.n_neurons;
    t.d[q].src_off = p->src_off;
  }
  return t;
}
}  // namespace

extern "C" {

int eq_set_peers(eq_handle* h, int32_t n_parts, eq_handle* const* peers, int32_t me) {
  if (!h || !peers) return EQ_ERR_CONFIGURATION;
  if (n_parts < 2 || n_parts > kMaxPeers || me < 0 || me >= n_parts || peers[me] != h)
    return fail(h, EQ_ERR_CONFIGURATION, "peer table: 2.." + std::to_string(kMaxPeers) +
                                             " partitions, this handle at index `me`");
  if (!h->partitioned || !h->net_set) return fail(h, EQ_ERR_CONFIGURATION, "eq_set_partition and eq_set_network first");
  long long cap = 0;
  for (int q = 0; q < n_parts; ++q) {
    const eq_handle* p = peers[q];
    if (!p || !p->partitioned || !p->net_set || p->cfg.precision != h->cfg.precision ||
        p->cfg.n_trials != h->cfg.n_trials || p->n_src != h->n_src)
      return fail(h, EQ_ERR_CONFIGURATION, "peer " + std::to_string(q) + " is not a partition of the same network");
    if (q != me) cap += p->log_cap;
  }
  DeviceGuard g(h->device);
  for (int q = 0; q < n_parts; ++q) {   // other GPUs' memory over NVLink
    if (peers[q]->device == h->device) continue;
    cudaError_t e = cudaDeviceEnablePeerAccess(peers[q]->device, 0);
    if (e == cudaErrorPeerAccessAlreadyEnabled) cudaGetLastError();
    else if (e != cudaSuccess) return cuda_fail(h, e, "cudaDeviceEnablePeerAccess");
  }
  // imports can never exceed the other partitions' logs together
  const size_t rec = h->cfg.precision == 32 ? sizeof(SpikeRec<float>) : sizeof(SpikeRec<double>);
  if (cap + 1 > h->imp_cap) {
    release(h, h->imp);
    release(h, h->imp_r0);
    release(h, h->imp_len);
    release(h, h->imp_lt);
    EQ_CUDA(h, alloc(h, &h->imp, (size_t)(cap + 1) * rec));
    EQ_CUDA(h, alloc(h, (void**)&h->imp_r0, (size_t)(cap + 1) * sizeof(long long)));
    EQ_CUDA(h, alloc(h, (void**)&h->imp_len, (size_t)(cap + 1) * sizeof(int)));
    EQ_CUDA(h, alloc(h, &h->imp_lt, (size_t)(cap + 1) * h->tsize));
    h->imp_cap = cap + 1;
  }
  EQ_CUDA(h, ensure(h, (void**)&h->peer_blk, (size_t)(h->t_cap + 2) * 2 * sizeof(long long)));
  EQ_CUDA(h, ensure(h, (void**)&h->peer_count, sizeof(long long)));
  EQ_CUDA(h, cudaMemset(h->peer_blk, 0, (size_t)(h->t_cap + 2) * 2 * sizeof(long long)));
  EQ_CUDA(h, cudaMemset(h->peer_count, 0, sizeof(long long)));
  h->peers.assign(peers, peers + n_parts);
  h->peer_me = me;
  h->peer_mode = true;
  h->imp_n = 0;
  h->imp_blocks.clear();
  return EQ_OK;
}

int eq_run_window(eq_handle* h, int32_t w, int32_t a_prev, int32_t n_steps, void* stream) {
  if (!h) return EQ_ERR_CONFIGURATION;
  if (!h->peer_mode) return fail(h, EQ_ERR_CONFIGURATION, "eq_set_peers must come first");
  if (n_steps < 0 || w < 0 || w > h->t_cap + 1 || (w > 0 && (a_prev < 0 || a_prev >= h->steps_done)))
    return fail(h, EQ_ERR_CONFIGURATION, "bad window");
  if (h->steps_done + n_steps > h->t_cap)
    return fail(h, EQ_ERR_CONFIGURATION, "window beyond the run's t_steps");
  DeviceGuard g(h->device);
  cudaStream_t s = (cudaStream_t)stream;
  if (w == 0) EQ_CUDA(h, cudaMemsetAsync(h->peer_count, 0, sizeof(long long), s));
  const PeerTable tab = peer_table(h);
  const bool f32 = h->cfg.precision == 32;
  if (w > 0) {
    if (f32)
      k_gather_peers<float><<<h->G, 256, 0, s>>>(tab, a_prev, h->steps_done, h->cfg.n_neurons, h->rowptr,
                                                 (SpikeRec<float>*)h->imp, h->imp_r0, h->imp_len, h->peer_count,
                                                 h->imp_cap, h->err_dev);
    else
      k_gather_peers<double><<<h->G, 256, 0, s>>>(tab, a_prev, h->steps_done, h->cfg.n_neurons, h->rowptr,
                                                  (SpikeRec<double>*)h->imp, h->imp_r0, h->imp_len, h->peer_count,
                                                  h->imp_cap, h->err_dev);
    k_gather_commit<<<1, 1, 0, s>>>(tab, a_prev, h->steps_done, h->peer_count, h->peer_blk + 2 * w);
    h->launches += 2;
  }
  auto launch = [&](auto tag) -> int {
    typedef decltype(tag) T;
    FwdArgs<T> A = fwd_args<T>(h, n_steps, nullptr);
    A.no_pause = 1;
    if (w > 0) {
      A.imp = (const SpikeRec<T>*)h->imp;
      A.imp_r0 = h->imp_r0;
      A.imp_len = h->imp_len;
      A.imp_dev = h->peer_blk + 2 * w;
      FwdArgs<T> Ai = A;
      Ai.tl = nullptr;
      k_import_fanout<T, kNT><<<h->G, kNT, 0, s>>>(Ai);
      h->launches += 1;
    }
    if (n_steps == 0) return EQ_OK;
    EQ_CUDA(h, cudaMemsetAsync(h->bar, 0, kBarWords * sizeof(unsigned), s));
    EQ_CUDA(h, cudaMemsetAsync(h->step_start + h->steps_done + 1, 0xFF, (size_t)n_steps * sizeof(long long), s));
    void* args[] = {&A};
    const void* kf = (const void*)k_forward<T, kNT, kU, split_f_hbm<T>()>;   // state in HBM
    EQ_CUDA(h, cudaLaunchCooperativeKernel(kf, dim3(h->G), dim3(kNT), args, 0, s));
    h->launches += 1;
    h->steps_done += n_steps;
    return EQ_OK;
  };
  return f32 ? launch(float()) : launch(double());
}

int eq_backward_window_peer(eq_handle* h, int32_t w, int32_t m_lo, int32_t a_next, void* stream) {
  if (!h) return EQ_ERR_CONFIGURATION;
  if (!h->peer_mode) return fail(h, EQ_ERR_CONFIGURATION, "eq_set_peers must come first");
  if (h->bwd_cursor < 0) return fail(h, EQ_ERR_CONFIGURATION, "eq_backward_begin must come first");
  if (m_lo < 0 || m_lo >= h->bwd_cursor || a_next < m_lo || a_next > h->steps_done)
    return fail(h, EQ_ERR_CONFIGURATION, "bad reverse window");
  DeviceGuard g(h->device);
  cudaStream_t s = (cudaStream_t)stream;
  const PeerTable tab = peer_table(h);
  const bool f32 = h->cfg.precision == 32;
  if (a_next > m_lo && a_next < h->steps_done) {   // the others' partials of this window's spikes
    if (f32)
      k_sum_peer_adjoints<float><<<h->G, 256, 0, s>>>(tab, w, m_lo, a_next, (float*)h->lt_rem);
    else
      k_sum_peer_adjoints<double><<<h->G, 256, 0, s>>>(tab, w, m_lo, a_next, (double*)h->lt_rem);
    h->launches += 1;
  }
  return f32 ? launch_backward<float>(h, m_lo, s, w) : launch_backward<double>(h, m_lo, s, w);
}

int eq_sync(eq_handle* h, void* stream) {
  if (!h) return EQ_ERR_CONFIGURATION;
  DeviceGuard g(h->device);
  return check_err(h, (cudaStream_t)stream);
}

int eq_add_spike_adjoints(eq_handle* h, int32_t step_lo, const void* vals, int64_t n, void* stream) {
  if (!h) return EQ_ERR_CONFIGURATION;
  if (!h->partitioned) return fail(h, EQ_ERR_CONFIGURATION, "eq_set_partition must come first");
  if (step_lo < 0 || step_lo > h->steps_done) return fail(h, EQ_ERR_CONFIGURATION, "step outside the run");
  if (n <= 0) return EQ_OK;
  DeviceGuard g(h->device);
  cudaStream_t s = (cudaStream_t)stream;
  const int blocks = (int)std::min<long long>((n + 255) / 256, 4096);
  if (h->cfg.precision == 32)
    k_add_lt<float><<<blocks, 256, 0, s>>>((float*)h->lt_rem, h->step_start, step_lo, (const float*)vals, n);
  else
    k_add_lt<double><<<blocks, 256, 0, s>>>((double*)h->lt_rem, h->step_start, step_lo, (const double*)vals, n);
  h->launches += 1;
  EQ_CUDA(h, cudaGetLastError());
  return EQ_OK;
}

int eq_counters(eq_handle* h, int64_t* out, void* stream) {
  if (!h) return EQ_ERR_CONFIGURATION;
  DeviceGuard g(h->device);
  cudaStream_t s = (cudaStream_t)stream;
  EQ_CUDA(h, cudaMemcpyAsync(out, h->counters, (size_t)h->cfg.n_trials * 3 * sizeof(long long),
                             cudaMemcpyDeviceToHost, s));
  EQ_CUDA(h, cudaStreamSynchronize(s));
  return EQ_OK;
}

int64_t eq_spike_count(eq_handle* h, void* stream) {
  if (!h) return -1;
  DeviceGuard g(h->device);
  cudaStream_t s = (cudaStream_t)stream;
  unsigned long long n = 0;
  if (cudaMemcpyAsync(&n, h->log_count, sizeof n, cudaMemcpyDeviceToHost, s) != cudaSuccess) return -1;
  if (cudaStreamSynchronize(s) != cudaSuccess) return -1;
  return (int64_t)n;
}

int eq_get_spikes(eq_handle* h, int32_t* step, int32_t* trial, int32_t* neuron, void* t_spk, void* stream) {
  if (!h) return EQ_ERR_CONFIGURATION;
  DeviceGuard g(h->device);
  cudaStream_t s = (cudaStream_t)stream;
  int n_chunks = h->steps_done * h->G;
  if (n_chunks == 0) return EQ_OK;
  int blocks = (n_chunks * 32 + 255) / 256;
  if (h->cfg.precision == 32)
    k_decode_spikes<float><<<blocks, 256, 0, s>>>((const SpikeRec<float>*)h->log, h->chunk_off, h->chunk_cnt,
                                                   n_chunks, h->G, h->cfg.n_neurons, step, trial, neuron,
                                                   (float*)t_spk);
  else
    k_decode_spikes<double><<<blocks, 256, 0, s>>>((const SpikeRec<double>*)h->log, h->chunk_off, h->chunk_cnt,
                                                    n_chunks, h->G, h->cfg.n_neurons, step, trial, neuron,
                                                    (double*)t_spk);
  h->launches += 1;
  EQ_CUDA(h, cudaGetLastError());
  return EQ_OK;
}

int eq_get_pending(eq_handle* h, int64_t* host_out, void* stream) {
  if (!h) return EQ_ERR_CONFIGURATION;
  if (h->cfg.kind == EQ_KIND_DONOTHING) return fail(h, EQ_ERR_CONFIGURATION, "donothing holds no events");
  DeviceGuard g(h->device);
  cudaStream_t s = (cudaStream_t)stream;
  const int N = h->cfg.n_neurons, B = h->cfg.n_trials, H = h->horizon;
  size_t n = (size_t)B * N * H * 2;
  void* buf = nullptr;
  EQ_CUDA(h, alloc(h, &buf, n * sizeof(long long)));
  if (h->lossy) {
    k_pending_lossy<<<592, 256, 0, s>>>(h->ring, h->cfg.precision == 32 ? 1 : 2, h->lossy_slots, B, N, H,
                                        h->steps_done, (long long*)buf);
  } else if (h->bounded && h->staged) {
    if (h->cfg.precision == 32)
      k_pending_bq<float><<<592, 256, 0, s>>>(h->qkeys, (const long long*)h->qpay, h->meta, h->C,
                                               (long long)B * N, H, h->steps_done, (long long*)buf);
    else
      k_pending_bq<double><<<592, 256, 0, s>>>(h->qkeys, (const longlong2*)h->qpay, h->meta, h->C,
                                                (long long)B * N, H, h->steps_done, (long long*)buf);
  } else if (h->bounded && !h->adm) {
    if (h->cfg.precision == 32)
      k_pending_bounded<float><<<592, 256, 0, s>>>((const QEv<float>*)h->q, h->meta, h->cfg.kind, h->cap,
                                                    (long long)B * N, H, h->steps_done, (long long*)buf);
    else
      k_pending_bounded<double><<<592, 256, 0, s>>>((const QEv<double>*)h->q, h->meta, h->cfg.kind, h->cap,
                                                     (long long)B * N, H, h->steps_done, (long long*)buf);
  } else {
    EQ_CUDA(h, cudaMemsetAsync(buf, 0, n * sizeof(long long), s));
    if (h->cfg.precision == 32)
      k_pending_calendar<float><<<592, 256, 0, s>>>(h->acc, h->bk, h->bk_cnt, h->cap_b, h->NB, h->G,
                                                     h->ring,
                                                     h->ring_dirty, B, h->R, N, H, h->steps_done, (long long*)buf);
    else
      k_pending_calendar<double><<<592, 256, 0, s>>>(h->acc, h->bk, h->bk_cnt, h->cap_b, h->NB,
                                                      h->G, h->ring, h->ring_dirty, B, h->R, N, H, h->steps_done,
                                                      (long long*)buf);
  }
  h->launches += 1;
  EQ_CUDA(h, cudaMemcpyAsync(host_out, buf, n * sizeof(long long), cudaMemcpyDeviceToHost, s));
  EQ_CUDA(h, cudaStreamSynchronize(s));
  release(h, buf);
  return EQ_OK;
}

int eq_horizon(const eq_handle* h) { return h ? h->horizon : -1; }
int eq_frac_bits(const eq_handle* h) { return h ? h->frac_bits : -1; }
int eq_geometry(const eq_handle* h, int32_t* ctas, int32_t* threads) {
  if (!h) return EQ_ERR_CONFIGURATION;
  if (ctas) *ctas = h->G;
  if (threads) *threads = kNT;
  return EQ_OK;
}
int64_t eq_launch_count(const eq_handle* h) { return h ? h->launches : -1; }

int64_t eq_log_capacity(const eq_handle* h, int32_t* n_grows) {
  if (!h) return -1;
  if (n_grows) *n_grows = h->log_grows;
  return h->log_cap;
}

int eq_debug_set_bucket_capacity(eq_handle* h, int64_t cap) {
  if (!h) return EQ_ERR_CONFIGURATION;
  if (!h->cal || !h->net_set)
    return fail(h, EQ_ERR_CONFIGURATION, "bucket capacity: calendar kinds (ring, heap, sorted) after eq_set_network only");
  if (cap < 1 || cap > h->cap_b_alloc)
    return fail(h, EQ_ERR_CONFIGURATION, "bucket capacity outside [1, " + std::to_string(h->cap_b_alloc) + "]");
  h->cap_b = cap;
  return EQ_OK;
}

int eq_debug_set_admission_slots(eq_handle* h, int32_t k) {
  if (!h) return EQ_ERR_CONFIGURATION;
  if (k < 0 || k > kAdmSlots)
    return fail(h, EQ_ERR_CONFIGURATION, "admission slots outside [0, " + std::to_string(kAdmSlots) + "]");
  h->adm_slots = k;
  return EQ_OK;
}

/* Debug: per-step, per-CTA phase timestamps (ns) of the last forward (which=0)
 * or reverse (which=1) run, [t_steps][ctas][4]; needs EQ_TIMELINE=1 at create. */
int eq_debug_timeline(eq_handle* h, int which, uint64_t* host_out) {
  if (!h) return EQ_ERR_CONFIGURATION;
  unsigned long long* src = which ? h->tl_b : h->tl_f;
  if (!src) return fail(h, EQ_ERR_CONFIGURATION, "timeline disabled (set EQ_TIMELINE=1 before eq_create)");
  DeviceGuard g(h->device);
  EQ_CUDA(h, cudaDeviceSynchronize());
  EQ_CUDA(h, cudaMemcpy(host_out, src, (size_t)h->tl_steps * h->G * 8 * 8, cudaMemcpyDeviceToHost));
  return EQ_OK;
}

}  // extern "C"
