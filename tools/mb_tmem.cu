// Microbenchmark: tensor-memory (TMEM) load throughput vs shared memory on B200, as storage for an
// operator that stays on chip across the iterations of a solver.  One CTA per SM, W warps; warp w
// owns TMEM lanes 32 (w % 4) .. +31 and columns 128 (w / 4) .. +127 (two 32x32 fp64 blocks per warp).
// Reports bytes per SM-cycle for tcgen05.ld (x32 / x64 chunks) and for ld.shared.v2.f64.
#include <cstdio>
#include <cstdint>

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

#define LD32(taddr, v)                                                                                    \
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15," \
               "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];\n"                \
               : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]),      \
                 "=r"(v[7]), "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]),  \
                 "=r"(v[14]), "=r"(v[15]), "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]),            \
                 "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]), "=r"(v[24]), "=r"(v[25]),            \
                 "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])             \
               : "r"(taddr))
#define ST32(taddr, v)                                                                                    \
  asm volatile("tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15," \
               "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};\n" ::"r"(taddr),    \
               "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]),   \
               "r"(v[8]), "r"(v[9]), "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]),         \
               "r"(v[15]), "r"(v[16]), "r"(v[17]), "r"(v[18]), "r"(v[19]), "r"(v[20]), "r"(v[21]),       \
               "r"(v[22]), "r"(v[23]), "r"(v[24]), "r"(v[25]), "r"(v[26]), "r"(v[27]), "r"(v[28]),       \
               "r"(v[29]), "r"(v[30]), "r"(v[31]))

__global__ void k_tmem(int iters, double* out, unsigned long long* cyc) {
  __shared__ uint32_t tbase;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(smem_u32(&tbase)), "r"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
  const uint32_t taddr = tbase + ((uint32_t)(32 * (warp & 3)) << 16) + 128 * (warp >> 2);
  uint32_t v[32];
  for (int c = 0; c < 4; ++c) {
    for (int i = 0; i < 32; ++i) v[i] = __float_as_uint(1.0f + 1e-3f * (i + lane + c));
    ST32(taddr + 32 * c, v);
  }
  asm volatile("tcgen05.wait::st.sync.aligned;\n" ::: "memory");
  __syncthreads();
  float acc = 0.f;
  unsigned long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      LD32(taddr + 32 * c, v);
      asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
#pragma unroll
      for (int i = 0; i < 32; ++i) acc += __uint_as_float(v[i]);
    }
  }
  __syncthreads();
  unsigned long long t1 = clock64();
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tbase), "r"(512));
}

// same, with the 4 chunk loads issued before one wait (more loads in flight)
__global__ void k_tmem4(int iters, double* out, unsigned long long* cyc) {
  __shared__ uint32_t tbase;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(smem_u32(&tbase)), "r"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
  const uint32_t taddr = tbase + ((uint32_t)(32 * (warp & 3)) << 16) + 128 * (warp >> 2);
  uint32_t v[32], w[32];
  for (int c = 0; c < 4; ++c) {
    for (int i = 0; i < 32; ++i) v[i] = __float_as_uint(1.0f + 1e-3f * (i + lane + c));
    ST32(taddr + 32 * c, v);
  }
  asm volatile("tcgen05.wait::st.sync.aligned;\n" ::: "memory");
  __syncthreads();
  float acc = 0.f;
  unsigned long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int c = 0; c < 4; c += 2) {
      LD32(taddr + 32 * c, v);
      LD32(taddr + 32 * c + 32, w);
      asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
#pragma unroll
      for (int i = 0; i < 32; ++i) acc += __uint_as_float(v[i]) + __uint_as_float(w[i]);
    }
  }
  __syncthreads();
  unsigned long long t1 = clock64();
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tbase), "r"(512));
}

// shared memory: each warp reads its own 16 KB (two 32x32 fp64 blocks) per iteration, v2.f64 loads
__global__ void k_smem(int iters, double* out, unsigned long long* cyc) {
  extern __shared__ double sm[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  double* mine = sm + (size_t)warp * 2048;
  for (int i = lane; i < 2048; i += 32) mine[i] = 1.0 + 1e-3 * i;
  __syncthreads();
  double acc = 0.0;
  unsigned long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll 8
    for (int i = 0; i < 32; ++i) {
      const double2 x = reinterpret_cast<const double2*>(mine)[i * 32 + lane];
      acc += x.x + x.y;
    }
  }
  __syncthreads();
  unsigned long long t1 = clock64();
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}

int main() {
  double* out;
  unsigned long long* cyc;
  cudaMalloc(&out, 148 * 1024 * 8);
  cudaMallocManaged(&cyc, 148 * 8);
  const int iters = 2000;
  for (int W : {4, 8, 14, 16}) {
    for (int kind = 0; kind < 3; ++kind) {
      const size_t sm = kind == 2 ? (size_t)W * 2048 * 8 : 0;
      if (kind == 2) cudaFuncSetAttribute(k_smem, cudaFuncAttributeMaxDynamicSharedMemorySize, 232448);
      for (int rep = 0; rep < 2; ++rep) {
        if (kind == 0) k_tmem<<<148, 32 * W>>>(iters, out, cyc);
        else if (kind == 1) k_tmem4<<<148, 32 * W>>>(iters, out, cyc);
        else k_smem<<<148, 32 * W, sm>>>(iters, out, cyc);
      }
      cudaError_t e = cudaDeviceSynchronize();
      unsigned long long mx = 0;
      for (int b = 0; b < 148; ++b) mx = cyc[b] > mx ? cyc[b] : mx;
      const double bytes = (double)W * 16384.0 * iters;   // per SM
      printf("%-6s W=%2d: %8.1f B/SM-cycle  (%llu cycles, %s)\n", kind == 0 ? "tmem" : kind == 1 ? "tmem2" : "smem", W,
             bytes / mx, mx, cudaGetErrorString(e));
    }
  }
  return 0;
}
