// Random-gather microbenchmark: how fast can B200 serve N random 8-byte reads
// from a large array?  Mimics the reverse pass's reverse-slot gathers.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

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

int main() {
  const int M = 711000;
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
