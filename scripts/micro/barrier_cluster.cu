// Grid barrier with a hardware cluster level, on B200: CTAs of a thread-block
// cluster sync with barrier.cluster (release/acquire at cluster scope), then
// one CTA per cluster arrives on the flip-bit word (eq_device.cuh grid_sync),
// so the single-address atomic serialises nclusters arrivals instead of G.
// Cooperative launch with a cluster dimension (cudaLaunchKernelEx).
#include <cooperative_groups.h>
#include <cstdio>
#include "../../paper_2512_05906_b200/csrc/eq_device.cuh"

using namespace eq;
namespace cg = cooperative_groups;

__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}

__device__ __forceinline__ void grid_sync_cluster(unsigned* bar, unsigned nclusters, unsigned crank, unsigned cid) {
  __syncthreads();
  cluster_sync_all();
  if (crank == 0 && threadIdx.x == 0) {
    const unsigned inc = cid == 0 ? 0x80000000u - (nclusters - 1) : 1u;
    const unsigned old = atom_add_acq_rel(bar, inc);
    if (((old ^ (old + inc)) & 0x80000000u) == 0)
      while (((ld_relaxed(bar) ^ old) & 0x80000000u) == 0) {
      }
    fence_acq_rel_gpu();
  }
  cluster_sync_all();
}

__global__ void __launch_bounds__(512, 2) k_bar_cluster(unsigned* bar, int iters) {
  unsigned crank, cnum, csize;
  asm("mov.u32 %0, %%cluster_ctarank;" : "=r"(crank));
  asm("mov.u32 %0, %%clusterid.x;" : "=r"(cnum));
  asm("mov.u32 %0, %%cluster_nctarank;" : "=r"(csize));
  const unsigned ncl = gridDim.x / csize;
  for (int i = 0; i < iters; ++i) grid_sync_cluster(bar, ncl, crank, cnum);
}

__global__ void __launch_bounds__(512, 2) k_bar_flat(unsigned* bar, int* err, int iters) {
  for (int i = 0; i < iters; ++i) grid_sync(bar, gridDim.x, err);
}

int main() {
  unsigned* bar;
  int* err;
  cudaMalloc(&bar, kBarWords * 4);
  cudaMalloc(&err, 16);
  const int iters = 2000;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int G = 296;
  {
    cudaMemset(bar, 0, kBarWords * 4);
    int it = iters;
    void* args[] = {&bar, &err, &it};
    cudaLaunchCooperativeKernel((const void*)k_bar_flat, G, 512, args, 0, 0);
    cudaEventRecord(e0);
    cudaLaunchCooperativeKernel((const void*)k_bar_flat, G, 512, args, 0, 0);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    printf("G=%d flat flip-bit grid_sync      %6.3f us per barrier (%s)\n", G, ms * 1e3 / iters,
           cudaGetErrorString(cudaGetLastError()));
  }
  for (int cs : {2, 4, 8}) {
    cudaMemset(bar, 0, kBarWords * 4);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(G);
    cfg.blockDim = dim3(512);
    cudaLaunchAttribute at[2];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = cs;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    at[1].id = cudaLaunchAttributeCooperative;
    at[1].val.cooperative = 1;
    cfg.attrs = at;
    cfg.numAttrs = 2;
    int it = iters;
    cudaError_t e = cudaLaunchKernelEx(&cfg, k_bar_cluster, bar, it);
    cudaDeviceSynchronize();
    cudaEventRecord(e0);
    e = cudaLaunchKernelEx(&cfg, k_bar_cluster, bar, it);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    int maxc = 0;
    cudaOccupancyMaxActiveClusters(&maxc, (void*)k_bar_cluster, &cfg);
    printf("G=%d cluster %d + flip-bit            %6.3f us per barrier (launch %s, last %s, max active clusters %d)\n",
           G, cs, ms * 1e3 / iters, cudaGetErrorString(e), cudaGetErrorString(cudaGetLastError()), maxc);
  }
  return 0;
}
