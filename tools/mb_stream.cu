// Microbenchmark: warp-per-subdomain streaming of 32x32 fp64 blocks (the PCG SpMV access pattern).
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k_stream(const double* __restrict__ B, double* out, int nsub, int nblk, int mode) {
  const int lane = threadIdx.x & 31, W = blockDim.x >> 5;
  const int gw = blockIdx.x * W + (threadIdx.x >> 5), TW = gridDim.x * W;
  double acc = 0.0;
  for (int E = gw; E < nsub; E += TW) {
    const double* P = B + (size_t)E * nblk * 1024;
    if (mode == 0) {
      for (int b = 0; b < nblk; ++b) {
        double buf[32];
#pragma unroll
        for (int k = 0; k < 32; ++k) buf[k] = __ldg(P + b * 1024 + k * 32 + lane);
#pragma unroll
        for (int k = 0; k < 32; ++k) acc += buf[k] * (k + 1);
      }
    } else {
      // all blocks' loads issued before use (nblk <= 3)
      double buf[96];
#pragma unroll
      for (int k = 0; k < 96; ++k) buf[k] = (k / 32 < nblk) ? __ldg(P + k * 32 + lane) : 0.0;
#pragma unroll
      for (int k = 0; k < 96; ++k) acc += buf[k] * (k + 1);
    }
  }
  if (acc == 12345.0) out[0] = acc;
}
int main() {
  const int nsub = 2048, nblk = 3;
  size_t n = (size_t)nsub * nblk * 1024;
  double *B, *out;
  cudaMalloc(&B, n * 8);
  cudaMalloc(&out, 8);
  cudaMemset(B, 0, n * 8);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0); cudaEventCreate(&e1);
  int cfg[][2] = {{128, 16}, {148, 14}, {296, 7}, {256, 8}, {512, 4}, {148, 16}};
  for (int mode = 0; mode < 2; ++mode)
    for (auto& c : cfg) {
      float best = 1e9;
      for (int r = 0; r < 20; ++r) {
        cudaEventRecord(e0);
        k_stream<<<c[0], c[1] * 32>>>(B, out, nsub, nblk, mode);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms; cudaEventElapsedTime(&ms, e0, e1);
        if (r > 2 && ms < best) best = ms;
      }
      printf("mode %d grid %4d x %2d warps: %7.2f us  %6.2f TB/s (L2-resident, %.1f MB)\n", mode, c[0], c[1],
             best * 1e3, n * 8 / (best * 1e-3) / 1e12, n * 8 / 1e6);
    }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
}
