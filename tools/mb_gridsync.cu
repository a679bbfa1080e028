// Microbenchmark: cooperative-groups grid.sync cost on B200 (128 x 512 and 148 x 448 threads)
#include <cooperative_groups.h>
#include <cstdio>
namespace cg = cooperative_groups;
__global__ void k_sync(int iters, double* buf, int mode) {
  cg::grid_group g = cg::this_grid();
  double acc = 0;
  for (int i = 0; i < iters; ++i) {
    if (mode == 1) buf[(blockIdx.x * blockDim.x + threadIdx.x) * 4] = acc + i;   // a store before each sync
    if (mode == 2) acc += buf[((blockIdx.x + i) % gridDim.x) * blockDim.x * 4 + threadIdx.x * 4];
    g.sync();
  }
  if (acc == -1.0) buf[0] = acc;
}
int main() {
  double* buf; cudaMalloc(&buf, 148 * 1024 * 4 * 8);
  int cfg[][2] = {{128, 512}, {148, 448}, {148, 512}, {64, 1024}, {148, 256}};
  for (int mode = 0; mode < 3; ++mode)
    for (auto& c : cfg) {
      int iters = 2000;
      void* args[] = {&iters, &buf, &mode};
      cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
      cudaLaunchCooperativeKernel((void*)k_sync, c[0], c[1], args, 0, 0);
      cudaEventRecord(e0);
      cudaLaunchCooperativeKernel((void*)k_sync, c[0], c[1], args, 0, 0);
      cudaEventRecord(e1); cudaEventSynchronize(e1);
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      printf("mode %d grid %3d x %4d: %.3f us per grid.sync  (%s)\n", mode, c[0], c[1], ms * 1e3 / iters,
             cudaGetErrorString(cudaGetLastError()));
    }
}
