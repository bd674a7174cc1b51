// Random-gather microbenchmark: how fast can B200 serve N random 8-byte reads
// from a large array?  Mimics the reverse pass's reverse-slot gathers.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include <vector>

__global__ void k_gather(const float2* __restrict__ a, size_t n, const uint32_t* __restrict__ idx, int m,
                         float* out, int ev) {
  int tid = blockIdx.x * blockDim.x + threadIdx.x;
  int stride = gridDim.x * blockDim.x;
  float acc = 0.f;
  for (int i = tid; i < m; i += stride * 4) {
    float2 v[4];
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      int k = i + e * stride;
      v[e] = k < m ? a[idx[k] % n] : make_float2(0, 0);
    }
#pragma unroll
    for (int e = 0; e < 4; ++e) acc += v[e].x + v[e].y;
  }
  if (acc == 123.f) out[0] = acc;
}

// load-flavour variants of the same gather (mode 0 = plain ld.global)
template <int MODE>
__device__ __forceinline__ float2 ld_v(const float2* p) {
  float2 v;
  if (MODE == 0) {
    v = *p;
  } else if (MODE == 1) {
    v = __ldcg(p);
  } else if (MODE == 2) {
    v = __ldcs(p);
  } else if (MODE == 3) {
    asm volatile("ld.global.nc.L1::no_allocate.v2.f32 {%0, %1}, [%2];" : "=f"(v.x), "=f"(v.y) : "l"(p));
  } else if (MODE == 4) {
    asm volatile("ld.global.L1::no_allocate.v2.f32 {%0, %1}, [%2];" : "=f"(v.x), "=f"(v.y) : "l"(p));
  } else if (MODE == 5) {
    asm volatile("ld.global.cg.L2::64B.v2.f32 {%0, %1}, [%2];" : "=f"(v.x), "=f"(v.y) : "l"(p));
  } else {
    asm volatile("ld.relaxed.gpu.global.v2.f32 {%0, %1}, [%2];" : "=f"(v.x), "=f"(v.y) : "l"(p));
  }
  return v;
}

template <int MODE>
__global__ void k_gather_v(const float2* __restrict__ a, size_t n, const uint32_t* __restrict__ idx, int m,
                           float* out) {
  int tid = blockIdx.x * blockDim.x + threadIdx.x;
  int stride = gridDim.x * blockDim.x;
  float acc = 0.f;
  for (int i = tid; i < m; i += stride * 4) {
    float2 v[4];
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      int k = i + e * stride;
      v[e] = k < m ? ld_v<MODE>(a + idx[k] % n) : make_float2(0, 0);
    }
#pragma unroll
    for (int e = 0; e < 4; ++e) acc += v[e].x + v[e].y;
  }
  if (acc == 123.f) out[0] = acc;
}

__global__ void k_red(long long* a, size_t n, const uint32_t* __restrict__ idx, int m) {
  int tid = blockIdx.x * blockDim.x + threadIdx.x;
  int stride = gridDim.x * blockDim.x;
  for (int i = tid; i < m; i += stride) {
    asm volatile("red.relaxed.gpu.global.add.u64 [%0], %1;" ::"l"(a + (idx[i] % n)), "l"(1LL) : "memory");
  }
}

__global__ void k_init(uint32_t* idx, int m, uint32_t seed) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < m) {
    uint32_t x = i * 2654435761u + seed;
    x ^= x >> 16; x *= 0x7feb352d; x ^= x >> 15; x *= 0x846ca68b; x ^= x >> 16;
    idx[i] = x;
  }
}

int main(int argc, char** argv) {
  const int M = 711000;
  if (argc > 1 && argv[1][0] == 'r') {   // per-warp region size: a warp's 32 lanes fall in one region
    uint32_t* idx; cudaMalloc(&idx, M * 4);
    float* out; cudaMalloc(&out, 4);
    k_init<<<(M + 255) / 256, 256>>>(idx, M, 7);
    std::vector<uint32_t> h(M);
    cudaMemcpy(h.data(), idx, M * 4, cudaMemcpyDeviceToHost);
    const size_t n = (size_t)845 * (1 << 20) / 8;
    float2* a; cudaMalloc(&a, n * 8); cudaMemset(a, 0, n * 8);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    // the kernel's lane k of a warp is gather index i = tid + e*stride: consecutive k in one warp share tid/32
    const int stride = 592 * 256;
    for (size_t region : {(size_t)53 << 20, (size_t)8 << 20, (size_t)800 << 10, (size_t)64 << 10}) {
      const size_t rn = region / 8;
      std::vector<uint32_t> g(M);
      for (int k = 0; k < M; ++k) {
        const int tid = k % stride, e = k / stride;
        const uint32_t warp_key = (uint32_t)((tid / 32) * 7919u + e * 104729u);
        const size_t base = ((size_t)(warp_key * 2654435761u) % (n / rn)) * rn;
        g[k] = (uint32_t)(base + h[k] % rn);
      }
      uint32_t* gi; cudaMalloc(&gi, M * 4);
      cudaMemcpy(gi, g.data(), M * 4, cudaMemcpyHostToDevice);
      k_gather_v<0><<<592, 256>>>(a, n, gi, M, out);
      cudaEventRecord(e0);
      for (int r = 0; r < 20; ++r) k_gather_v<0><<<592, 256>>>(a, n, gi, M, out);
      cudaEventRecord(e1); cudaEventSynchronize(e1);
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      printf("845 MB, warp lanes within %8zu KB regions: %7.2f us per 711k\n", region >> 10, ms / 20 * 1e3);
      cudaFree(gi);
    }
    return 0;
  }
  if (argc > 1 && argv[1][0] == 's') {   // locality: 16 trial rings of 53 MB, gathers grouped by ring
    uint32_t* idx; cudaMalloc(&idx, M * 4);
    float* out; cudaMalloc(&out, 4);
    k_init<<<(M + 255) / 256, 256>>>(idx, M, 7);
    std::vector<uint32_t> h(M);
    cudaMemcpy(h.data(), idx, M * 4, cudaMemcpyDeviceToHost);
    const size_t n = (size_t)845 * (1 << 20) / 8, ring = n / 16;
    float2* a; cudaMalloc(&a, n * 8); cudaMemset(a, 0, n * 8);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    for (int groups : {1, 2, 4, 16}) {            // gathers ordered so `groups` consecutive chunks share a ring
      std::vector<uint32_t> g(M);
      for (int k = 0; k < M; ++k) {
        size_t chunk = (size_t)k * groups / M;      // which phase-slice of the gathers
        size_t r = groups == 1 ? (h[k] % 16) : (chunk * 16 / groups + h[k] % (16 / groups));
        g[k] = (uint32_t)(r * ring + (h[k] / 16) % ring);
      }
      uint32_t* gi; cudaMalloc(&gi, M * 4);
      cudaMemcpy(gi, g.data(), M * 4, cudaMemcpyHostToDevice);
      k_gather_v<0><<<592, 256>>>(a, n, gi, M, out);
      cudaEventRecord(e0);
      for (int r = 0; r < 20; ++r) k_gather_v<0><<<592, 256>>>(a, n, gi, M, out);
      cudaEventRecord(e1); cudaEventSynchronize(e1);
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      printf("845 MB, gathers in %2d slices over %2d rings each: %7.2f us per 711k\n", groups, 16 / groups,
             ms / 20 * 1e3);
      cudaFree(gi);
    }
    return 0;
  }
  if (argc > 1 && argv[1][0] == 'v') {   // load flavours at 845 MB
    uint32_t* idx; cudaMalloc(&idx, M * 4);
    float* out; cudaMalloc(&out, 4);
    k_init<<<(M + 255) / 256, 256>>>(idx, M, 7);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    size_t n = (size_t)845 * (1 << 20) / 8;
    float2* a; cudaMalloc(&a, n * 8); cudaMemset(a, 0, n * 8);
    void (*ks[])(const float2*, size_t, const uint32_t*, int, float*) = {
        k_gather_v<0>, k_gather_v<1>, k_gather_v<2>, k_gather_v<3>, k_gather_v<4>, k_gather_v<5>, k_gather_v<6>};
    const char* names[] = {"ld", "ld.cg", "ld.cs", "ld.nc.L1::no_allocate", "ld.L1::no_allocate", "ld.cg.L2::64B",
                           "ld.relaxed.gpu"};
    for (int k = 0; k < 7; ++k) {
      ks[k]<<<592, 256>>>(a, n, idx, M, out);
      cudaEventRecord(e0);
      for (int r = 0; r < 20; ++r) ks[k]<<<592, 256>>>(a, n, idx, M, out);
      cudaEventRecord(e1); cudaEventSynchronize(e1);
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      printf("845 MB %-24s: %7.2f us per 711k (%s)\n", names[k], ms / 20 * 1e3, cudaGetErrorString(cudaGetLastError()));
    }
    return 0;
  }
  if (argc > 1) {   // L2 fetch-granularity sweep at the C3 x 16 reverse-ring size
    uint32_t* idx; cudaMalloc(&idx, M * 4);
    float* out; cudaMalloc(&out, 4);
    k_init<<<(M + 255) / 256, 256>>>(idx, M, 7);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    size_t def = 0;
    cudaDeviceGetLimit(&def, cudaLimitMaxL2FetchGranularity);
    printf("default max L2 fetch granularity: %zu\n", def);
    for (size_t mb : {256, 845, 4096}) {
      size_t n = mb * (1 << 20) / 8;
      float2* a; cudaMalloc(&a, n * 8); cudaMemset(a, 0, n * 8);
      for (size_t g : {0, 32, 64, 128}) {
        cudaError_t e = cudaDeviceSetLimit(cudaLimitMaxL2FetchGranularity, g);
        size_t got = 0;
        cudaDeviceGetLimit(&got, cudaLimitMaxL2FetchGranularity);
        k_gather<<<592, 256>>>(a, n, idx, M, out, 4);
        cudaEventRecord(e0);
        for (int r = 0; r < 20; ++r) k_gather<<<592, 256>>>(a, n, idx, M, out, 4);
        cudaEventRecord(e1); cudaEventSynchronize(e1);
        float ms; cudaEventElapsedTime(&ms, e0, e1);
        long long* b = (long long*)a;
        k_red<<<592, 256>>>(b, n, idx, M);
        cudaEvent_t f0, f1; cudaEventCreate(&f0); cudaEventCreate(&f1);
        cudaEventRecord(f0);
        for (int r = 0; r < 20; ++r) k_red<<<592, 256>>>(b, n, idx, M);
        cudaEventRecord(f1); cudaEventSynchronize(f1);
        float ms2; cudaEventElapsedTime(&ms2, f0, f1);
        printf("%5zu MB  set %3zu (%s) got %3zu : gather %7.2f us  red %7.2f us per 711k\n", mb, g,
               cudaGetErrorString(e), got, ms / 20 * 1e3, ms2 / 20 * 1e3);
      }
      cudaFree(a);
    }
    return 0;
  }
  size_t sizes_mb[] = {16, 64, 128, 256, 845, 4096};
  uint32_t* idx; cudaMalloc(&idx, M * 4);
  float* out; cudaMalloc(&out, 4);
  k_init<<<(M + 255) / 256, 256>>>(idx, M, 7);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (size_t mb : sizes_mb) {
    size_t n = mb * (1 << 20) / 8;
    float2* a; cudaMalloc(&a, n * 8); cudaMemset(a, 0, n * 8);
    for (int threads : {256, 512}) for (int blocks : {296, 592}) {
      k_gather<<<blocks, threads>>>(a, n, idx, M, out, 4);
      cudaEventRecord(e0);
      for (int r = 0; r < 20; ++r) k_gather<<<blocks, threads>>>(a, n, idx, M, out, 4);
      cudaEventRecord(e1); cudaEventSynchronize(e1);
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      printf("gather %5zu MB  grid %4d x %3d : %7.2f us per 711k  (%.1f G/s)\n", mb, blocks, threads, ms / 20 * 1e3,
             M / (ms / 20 * 1e-3) / 1e9);
    }
    long long* b = (long long*)a;
    size_t nb = n;
    k_red<<<592, 256>>>(b, nb, idx, M);
    cudaEventRecord(e0);
    for (int r = 0; r < 20; ++r) k_red<<<592, 256>>>(b, nb, idx, M);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    printf("red    %5zu MB                   : %7.2f us per 711k  (%.1f G/s)\n", mb, ms / 20 * 1e3,
           M / (ms / 20 * 1e-3) / 1e9);
    cudaFree(a);
  }
  return 0;
}
