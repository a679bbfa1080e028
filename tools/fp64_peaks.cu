// fp64 peak microbenchmarks for the roofline denominators (FFMA.F64 = DFMA and DMMA.8x8x4).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o fp64_peaks fp64_peaks.cu
#include <cstdio>
#include <cuda_runtime.h>

__global__ void dfma_kernel(double* out, int iters) {
  double a0 = threadIdx.x * 1e-9, a1 = a0 + 1, a2 = a0 + 2, a3 = a0 + 3;
  double a4 = a0 + 4, a5 = a0 + 5, a6 = a0 + 6, a7 = a0 + 7;
  const double b = 0.999999, c = 1e-7;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < 16; ++k) {
      a0 = fma(a0, b, c); a1 = fma(a1, b, c); a2 = fma(a2, b, c); a3 = fma(a3, b, c);
      a4 = fma(a4, b, c); a5 = fma(a5, b, c); a6 = fma(a6, b, c); a7 = fma(a7, b, c);
    }
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = a0 + a1 + a2 + a3 + a4 + a5 + a6 + a7;
}

__global__ void dmma_kernel(double* out, int iters) {
  double a = threadIdx.x * 1e-3, b = 1.0 - threadIdx.x * 1e-4;
  double c[4][2] = {};
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(c[k][0]), "+d"(c[k][1]) : "d"(a), "d"(b));
    }
  }
  double s = 0;
  for (int k = 0; k < 4; ++k) s += c[k][0] + c[k][1];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__global__ void copy_kernel(const double2* __restrict__ a, double2* __restrict__ b, size_t n) {
  size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x, st = (size_t)gridDim.x * blockDim.x;
  for (; i < n; i += st) b[i] = a[i];
}

int main() {
  int dev = 0, sms = 0, l2 = 0, smem = 0, clk = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaDeviceGetAttribute(&l2, cudaDevAttrL2CacheSize, dev);
  cudaDeviceGetAttribute(&smem, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, dev);
  double* out; cudaMalloc(&out, 148 * 64 * 1024 * sizeof(double));
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  float ms;
  // DFMA
  int iters = 4096, blocks = sms * 8, threads = 256;
  dfma_kernel<<<blocks, threads>>>(out, 16); cudaDeviceSynchronize();
  double best = 0;
  for (int r = 0; r < 5; ++r) {
    cudaEventRecord(e0); dfma_kernel<<<blocks, threads>>>(out, iters); cudaEventRecord(e1);
    cudaEventSynchronize(e1); cudaEventElapsedTime(&ms, e0, e1);
    double fl = 2.0 * 8 * 16 * (double)iters * blocks * threads;
    if (fl / ms / 1e9 > best) best = fl / ms / 1e9;
  }
  printf("{\"sms\": %d, \"l2_bytes\": %d, \"smem_optin\": %d, \"clock_khz\": %d,\n", sms, l2, smem, clk);
  printf(" \"dfma_tflops\": %.2f,\n", best);
  best = 0;
  for (int r = 0; r < 5; ++r) {
    cudaEventRecord(e0); dmma_kernel<<<blocks, threads>>>(out, iters); cudaEventRecord(e1);
    cudaEventSynchronize(e1); cudaEventElapsedTime(&ms, e0, e1);
    double fl = 2.0 * 8 * 8 * 4 * 4 * (double)iters * blocks * (threads / 32);
    if (fl / ms / 1e9 > best) best = fl / ms / 1e9;
  }
  printf(" \"dmma_tflops\": %.2f,\n", best);
  size_t n = (size_t)1 << 27;  // 2 GiB per buffer of double2
  double2 *a, *b; cudaMalloc(&a, n * 16); cudaMalloc(&b, n * 16);
  cudaMemset(a, 0, n * 16);
  best = 0;
  for (int r = 0; r < 6; ++r) {
    cudaEventRecord(e0); copy_kernel<<<sms * 8, 512>>>(a, b, n); cudaEventRecord(e1);
    cudaEventSynchronize(e1); cudaEventElapsedTime(&ms, e0, e1);
    double gbs = 2.0 * n * 16 / ms / 1e6;
    if (gbs > best) best = gbs;
  }
  printf(" \"copy_gbs\": %.1f,\n", best);
  // L2-resident copy: 32 MiB total
  size_t n2 = (size_t)1 << 20;
  best = 0;
  for (int r = 0; r < 20; ++r) {
    cudaEventRecord(e0);
    for (int k = 0; k < 10; ++k) copy_kernel<<<sms * 4, 512>>>(a, b, n2);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1); cudaEventElapsedTime(&ms, e0, e1);
    double gbs = 10 * 2.0 * n2 * 16 / ms / 1e6;
    if (gbs > best) best = gbs;
  }
  printf(" \"l2_copy_32MiB_gbs\": %.1f}\n", best);
  printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
