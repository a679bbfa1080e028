// Microbenchmark: deterministic grid-wide reductions fused with a grid barrier (the PCG's three per
// iteration), 147 CTAs x 448 threads, each warp storing 256 B to global before every barrier.
//  mode 0: per-CTA partial -> __threadfence + atomicAdd counter -> spin (ld.acquire) -> __threadfence
//          -> warp 0 reads the G partials (k_pcg's grid_reduce)
//  mode 1: per-CTA partial published by a st.release into a 4-deep ring of slots pre-set to a NaN
//          sentinel; warp 0 polls the G slots with ld.acquire until none is the sentinel, sums them;
//          the slot of epoch e - 2 is reset to the sentinel when epoch e is written (no counter)
//  mode 2: as 1, relaxed polls + one fence.acq_rel after the last poll
//  mode 3/4: see reduce3
//  mode 5 (round 2): the whole grid is ONE thread-block cluster (G <= 16): barrier.cluster + partials
//          written into every CTA's shared memory over DSMEM (the k_pcg_tm launch for 17 <= n_s <= 224);
//          also run with the L2 reduction of mode 3 at the same grid size for comparison
#include <cooperative_groups.h>
#include <cstdint>
#include <cstdio>
namespace cg = cooperative_groups;

constexpr unsigned long long SENT = 0xFFFFFFFFFFFFFFFFull;

__device__ __forceinline__ unsigned ld_acq(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ unsigned long long ld_acq64(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ unsigned long long ld_rlx64(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_rel64(unsigned long long* p, unsigned long long v) {
  asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ double warp_sum(double v) {
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

__device__ double reduce0(double v, double* red, double* partials, unsigned* bar, unsigned& epoch, double* bc) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, W = blockDim.x >> 5, G = gridDim.x;
  if (lane == 0) red[warp] = v;
  __syncthreads();
  ++epoch;
  double* ps = partials + (size_t)(epoch & 3) * G;
  if (warp == 0) {
    if (lane == 0) {
      double t = 0.0;
      for (int w = 0; w < W; ++w) t += red[w];
      ps[blockIdx.x] = t;
      __threadfence();
      atomicAdd(bar, 1u);
      const unsigned target = epoch * (unsigned)G;
      while (ld_acq(bar) < target) {
      }
      __threadfence();
    }
    __syncwarp();
    double s = 0.0;
    for (int b = lane; b < G; b += 32) s += __ldcg(ps + b);
    s = warp_sum(s);
    if (lane == 0) *bc = s;
  }
  __syncthreads();
  return *bc;
}

// mode 3: red.release arrival (no fence, no return), ld.acquire spin on the counter
// mode 4: atom.acq_rel arrival; the last arriver releases a separate flag word that the others poll
template <int MODE>
__device__ double reduce3(double v, double* red, double* partials, unsigned* bar, unsigned& epoch, double* bc) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, W = blockDim.x >> 5, G = gridDim.x;
  if (lane == 0) red[warp] = v;
  __syncthreads();
  ++epoch;
  double* ps = partials + (size_t)(epoch & 3) * G;
  if (warp == 0) {
    if (lane == 0) {
      double t = 0.0;
      for (int w = 0; w < W; ++w) t += red[w];
      ps[blockIdx.x] = t;
      const unsigned target = epoch * (unsigned)G;
      if (MODE == 3) {
        asm volatile("red.release.gpu.global.add.u32 [%0], %1;" ::"l"(bar), "r"(1u) : "memory");
        while (ld_acq(bar) < target) {
        }
      } else {
        unsigned old;
        asm volatile("atom.acq_rel.gpu.global.add.u32 %0, [%1], %2;" : "=r"(old) : "l"(bar), "r"(1u) : "memory");
        if (old == target - 1) {
          asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(bar + 32), "r"(epoch) : "memory");
        } else {
          while (ld_acq(bar + 32) < epoch) {
          }
        }
      }
    }
    __syncwarp();
    double s = 0.0;
    for (int b = lane; b < G; b += 32) s += __ldcg(ps + b);
    s = warp_sum(s);
    if (lane == 0) *bc = s;
  }
  __syncthreads();
  return *bc;
}

template <int MODE>
__device__ double reduce1(double v, double* red, unsigned long long* slots, unsigned& epoch, double* bc) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, W = blockDim.x >> 5, G = gridDim.x;
  if (lane == 0) red[warp] = v;
  __syncthreads();
  ++epoch;
  unsigned long long* ps = slots + (size_t)(epoch & 3) * G;
  if (warp == 0) {
    if (lane == 0) {
      double t = 0.0;
      for (int w = 0; w < W; ++w) t += red[w];
      slots[(size_t)((epoch + 2) & 3) * G + blockIdx.x] = SENT;   // epoch - 2: read by everyone already
      st_rel64(ps + blockIdx.x, (unsigned long long)__double_as_longlong(t));
    }
    double s = 0.0;
    for (int b = lane; b < G; b += 32) {
      unsigned long long x;
      if (MODE == 1) {
        do { x = ld_acq64(ps + b); } while (x == SENT);
      } else {
        do { x = ld_rlx64(ps + b); } while (x == SENT);
      }
      s += __longlong_as_double((long long)x);
    }
    if (MODE == 2) asm volatile("fence.acq_rel.gpu;" ::: "memory");
    s = warp_sum(s);
    if (lane == 0) *bc = s;
  }
  __syncthreads();
  return *bc;
}

__device__ double reduce_cluster(double v, double* red, double (*cpart)[16], unsigned& epoch, double* bc) {
  cg::cluster_group cl = cg::this_cluster();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, W = blockDim.x >> 5;
  const int G = (int)cl.num_blocks(), me = (int)cl.block_rank();
  if (lane == 0) red[warp] = v;
  __syncthreads();
  ++epoch;
  if (warp == 0) {
    const double t = warp_sum(lane < W ? red[lane] : 0.0);
    if (lane < G) *cl.map_shared_rank(&cpart[epoch & 1][me], lane) = t;
  }
  cl.sync();
  if (warp == 0) {
    const double s = warp_sum(lane < G ? cpart[epoch & 1][lane] : 0.0);
    if (lane == 0) *bc = s;
  }
  __syncthreads();
  return *bc;
}

__global__ void __launch_bounds__(448, 1) k_bench_cluster(int iters, int mode, double* data, double* partials,
                                                          unsigned* bar, double* out) {
  __shared__ double red[16], bc[1], cpart[2][16];
  unsigned epoch = 0;
  const int gw = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5), lane = threadIdx.x & 31;
  double acc = 0.0;
  for (int i = 0; i < iters; ++i) {
    data[(size_t)gw * 32 + lane] = acc + i;
    const double nb = __ldcg(data + (size_t)((gw + 7) % (gridDim.x * (blockDim.x >> 5))) * 32 + lane);
    const double v = warp_sum(nb);
    acc += mode == 5 ? reduce_cluster(v, red, cpart, epoch, bc) : reduce3<3>(v, red, partials, bar, epoch, bc);
  }
  if (threadIdx.x == 0) out[blockIdx.x] = acc;
}

__global__ void __launch_bounds__(448, 1) k_bench(int iters, int mode, double* data, double* partials, unsigned* bar,
                                                  unsigned long long* slots, double* out) {
  __shared__ double red[16], bc[1];
  unsigned epoch = 0;
  const int gw = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5), lane = threadIdx.x & 31;
  double acc = 0.0;
  for (int i = 0; i < iters; ++i) {
    // a neighbour-exchange store and load, as in the PCG phases
    data[(size_t)gw * 32 + lane] = acc + i;
    const double nb = __ldcg(data + (size_t)((gw + 7) % (gridDim.x * (blockDim.x >> 5))) * 32 + lane);
    const double v = warp_sum(nb);
    if (mode == 0) acc += reduce0(v, red, partials, bar, epoch, bc);
    else if (mode == 1) acc += reduce1<1>(v, red, slots, epoch, bc);
    else if (mode == 2) acc += reduce1<2>(v, red, slots, epoch, bc);
    else if (mode == 3) acc += reduce3<3>(v, red, partials, bar, epoch, bc);
    else acc += reduce3<4>(v, red, partials, bar, epoch, bc);
  }
  if (threadIdx.x == 0) out[blockIdx.x] = acc;
}

int main() {
  const int G = 147, T = 448, iters = 3000;
  double *data, *partials, *out;
  unsigned* bar;
  unsigned long long* slots;
  cudaMalloc(&data, (size_t)G * 14 * 32 * 8);
  cudaMalloc(&partials, 4 * G * 8);
  cudaMalloc(&bar, 256);
  cudaMalloc(&slots, 4 * G * 8);
  cudaMalloc(&out, G * 8);
  for (int mode = 0; mode < 5; ++mode) {
    float best = 1e30f;
    double res[2];
    for (int rep = 0; rep < 3; ++rep) {
      cudaMemset(bar, 0, 256);
      cudaMemset(slots, 0xFF, 4 * G * 8);
      cudaMemset(data, 0, (size_t)G * 14 * 32 * 8);
      int it = iters, md = mode;
      void* args[] = {&it, &md, &data, &partials, &bar, &slots, &out};
      cudaEvent_t e0, e1;
      cudaEventCreate(&e0);
      cudaEventCreate(&e1);
      cudaEventRecord(e0);
      cudaError_t err = cudaLaunchCooperativeKernel((void*)k_bench, G, T, args, 0, 0);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      if (err != cudaSuccess) printf("launch: %s\n", cudaGetErrorString(err));
      best = ms < best ? ms : best;
      cudaMemcpy(res, out, 16, cudaMemcpyDeviceToHost);
    }
    printf("mode %d: %.3f us per exchange + reduction  (check %.6e %.6e)\n", mode, best * 1e3 / iters, res[0], res[1]);
  }
  // one cluster of 16 CTAs x 8 warps (the C3 launch shape): cluster barriers + DSMEM against the L2 reduction
  for (int mode = 5; mode >= 3; mode -= 2) {
    const int Gc = 16, Tc = 256;
    float best = 1e30f;
    for (int rep = 0; rep < 3; ++rep) {
      cudaMemset(bar, 0, 256);
      cudaMemset(data, 0, (size_t)G * 14 * 32 * 8);
      int it = iters, md = mode;
      void* args[] = {&it, &md, &data, &partials, &bar, &out};
      cudaLaunchConfig_t cfg = {};
      cfg.gridDim = dim3(Gc); cfg.blockDim = dim3(Tc);
      cudaLaunchAttribute at[1];
      at[0].id = cudaLaunchAttributeClusterDimension;
      at[0].val.clusterDim.x = Gc; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
      cfg.attrs = at; cfg.numAttrs = 1;
      cudaFuncSetAttribute(k_bench_cluster, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
      cudaEvent_t e0, e1;
      cudaEventCreate(&e0);
      cudaEventCreate(&e1);
      cudaEventRecord(e0);
      cudaError_t err = cudaLaunchKernelExC(&cfg, (void*)k_bench_cluster, args);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      if (err != cudaSuccess) printf("launch: %s\n", cudaGetErrorString(err));
      best = ms < best ? ms : best;
    }
    printf("16 CTAs x 8 warps, %s: %.3f us per exchange + reduction\n",
           mode == 5 ? "one cluster (barrier.cluster + DSMEM partials)" : "L2 reduction (mode 3)", best * 1e3 / iters);
  }
  return 0;
}
