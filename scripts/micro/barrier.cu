// Grid-barrier latency on B200: 296 CTAs x 512 threads (the persistent
// kernels' geometry), 2000 barriers per launch, CUDA events.
#include <cooperative_groups.h>
#include <cstdio>
#include "../../paper_2512_05906_b200/csrc/eq_device.cuh"

using namespace eq;
namespace cg = cooperative_groups;

template <int MODE>
__global__ void __launch_bounds__(512, 2) k_bar(unsigned* bar, int* err, int iters, unsigned* single) {
  for (int i = 0; i < iters; ++i) {
    if (MODE == 0) {
      grid_sync(bar, gridDim.x, err);
    } else if (MODE == 1) {
      cg::this_grid().sync();
    } else {
      // single-level: one counter, generation release, pure spin
      __syncthreads();
      if (threadIdx.x == 0) {
        unsigned* cnt = single;
        unsigned* gen = single + 32;
        unsigned g = ld_relaxed(gen);
        if (atom_add_acq_rel(cnt, 1u) == gridDim.x - 1) {
          st_relaxed(cnt, 0u);
          st_release(gen, g + 1);
        } else {
          while (ld_relaxed(gen) == g) {
          }
        }
        fence_acq_rel_gpu();
      }
      __syncthreads();
    }
  }
}

int main() {
  unsigned *bar, *single;
  int* err;
  cudaMalloc(&bar, kBarWords * 4);
  cudaMalloc(&single, 64 * 4);
  cudaMalloc(&err, 16);
  const int iters = 2000;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  void (*ks[])(unsigned*, int*, int, unsigned*) = {k_bar<0>, k_bar<1>, k_bar<2>};
  const char* names[] = {"eq grid_sync (2-level)", "cg::grid.sync", "1-level spin"};
  for (int G : {148, 296}) {
    for (int k = 0; k < 3; ++k) {
      cudaMemset(bar, 0, kBarWords * 4);
      cudaMemset(single, 0, 64 * 4);
      cudaMemset(err, 0, 16);
      int it = iters;
      void* args[] = {&bar, &err, &it, &single};
      cudaLaunchCooperativeKernel((const void*)ks[k], G, 512, args, 0, 0);
      cudaEventRecord(e0);
      cudaLaunchCooperativeKernel((const void*)ks[k], G, 512, args, 0, 0);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      printf("G=%d %-24s %6.2f us per barrier (%s)\n", G, names[k], ms * 1e3 / iters,
             cudaGetErrorString(cudaGetLastError()));
    }
  }
  return 0;
}
