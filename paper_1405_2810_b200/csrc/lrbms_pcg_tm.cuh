// lrbms_pcg_tm.cuh -- a3 (eq:reducedSystem): the deflated PCG of lrbms_pcg.cuh
// with the scaled reduced operator held ON CHIP for the whole solve.
//
// One cooperative persistent kernel, one CTA per SM, one warp per subdomain E (lane k <-> reduced
// coefficient k, N <= 32), so every per-subdomain vector (y, r, z, p, q) lives in registers and only
// the exchange with neighbouring subdomains goes through L2.  The scaled couplings
// Bh_{E,E+a} = L_E^-1 B_{E,E+a} L_{E+a}^-T (upper storage, 8 KB each) are loaded ONCE per solve:
//
//   tensor memory (TMEM, 256 KB per SM, 512 columns x 128 lanes): warp w may only address lane
//     quadrant q = w % 4, which holds 8 blocks (each lane keeps its 4 x 8 register tile of a block in
//     64 32-bit columns).  The m-th warp of the quadrant (m = w / 4) owns quadrant block slots
//     b = dim m + a; slots b < 8 are TMEM columns 64 b .. +63, read back with tcgen05.ld every
//     iteration (~300 B/SM-cycle measured, tools/mb_tmem.cu, vs ~127 B/cycle for shared memory);
//   the overflow slots b >= 8 (3D, more than two warps per quadrant) -> shared memory,
//     element-interleaved over lanes (bank-conflict free).  C5 (14 warps): 32 blocks in TMEM (all 512 columns), 10 in
//     shared memory;
//   deflation vectors Y_{E,F} (6 per subdomain) and the fp32 rows of the coarse inverse B_c^-1 of
//     the CTA's subdomains -> shared memory (C5: 221 KB in all).
//
// Iteration (3 grid barriers, each fused with its reduction, deterministic fixed-order sums):
//   A: p = z + beta p; q_own = p + sum_a U_a p_{E+a} (p_{E+a} rebuilt from the neighbour's published
//      z and previous p); U_a^T p_E -> T[E+a][a]; p.Bh p (symmetric form)              -> reduce
//   B: q = q_own + lower hand-overs; y += alpha p; r -= alpha q; r.r; deflation scatter -> reduce
//   C: g = Zh^T (I - Bh) r staged; e_E = (B_c^-1 g)_E; z = r + zh e_E; publish z; r.z  -> reduce
#pragma once
#include "lrbms_pcg.cuh"


namespace lrbms {

__device__ __forceinline__ uint32_t smem_addr_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void tm_cp16(void* dst, const void* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(smem_addr_u32(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void tm_cp8(void* dst, const void* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(smem_addr_u32(dst)), "l"(src) : "memory");
}

// 32 lanes x 32 consecutive 32-bit TMEM columns <-> 32 registers per lane
__device__ __forceinline__ void tm_ld32(uint32_t taddr, uint32_t (&v)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];\n"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
        "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]),
        "=r"(v[15]), "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]),
        "=r"(v[22]), "=r"(v[23]), "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]),
        "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
}
__device__ __forceinline__ void tm_st32(uint32_t taddr, const uint32_t (&v)[32]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,"
      "%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};\n" ::"r"(taddr),
      "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]), "r"(v[8]),
      "r"(v[9]), "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15]), "r"(v[16]),
      "r"(v[17]), "r"(v[18]), "r"(v[19]), "r"(v[20]), "r"(v[21]), "r"(v[22]), "r"(v[23]), "r"(v[24]),
      "r"(v[25]), "r"(v[26]), "r"(v[27]), "r"(v[28]), "r"(v[29]), "r"(v[30]), "r"(v[31]));
}

// Block tile of lane l = 4 a + b (see spmv_part): element k = 8 i + j is U[4a + i][b + 4j].
// Half h (0, 1) holds rows i = 2h, 2h + 1: 16 doubles = 32 TMEM columns.
//
// Accumulates pu[i] += sum_j U[.][.] vc[j] (rows) and pt[j] += sum_i U[.][.] vr[i] (columns).
template <bool ROWS = true, bool COLS = true>
__device__ __forceinline__ void tile_half(const double (&u)[16], int h, const double (&vr)[4], const double (&vc)[8],
                                          double (&pu)[4], double (&pt)[8]) {
#pragma unroll
  for (int ii = 0; ii < 2; ++ii)
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const double x = u[ii * 8 + j];
      if (ROWS) pu[2 * h + ii] = fma(x, vc[j], pu[2 * h + ii]);
      if (COLS) pt[j] = fma(x, vr[2 * h + ii], pt[j]);
    }
}

// 4-lane (rows) and 8-lane (columns) reduce-scatters of the tile partials: lane l ends with
// (U v)[l] in the return value and (U^T w)[l] in tcol.
__device__ __forceinline__ double tile_scatter(double (&pu)[4], double (&pt)[8], int lane, double& tcol) {
#pragma unroll
  for (int i = 0; i < 2; ++i) {
    const bool hi = lane & 2;
    const double send = hi ? pu[i] : pu[i + 2];
    const double keep = hi ? pu[i + 2] : pu[i];
    pu[i] = keep + __shfl_xor_sync(FULL, send, 2);
  }
  {
    const bool hi = lane & 1;
    const double send = hi ? pu[0] : pu[1];
    const double keep = hi ? pu[1] : pu[0];
    pu[0] = keep + __shfl_xor_sync(FULL, send, 1);
  }
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    const bool hi = lane & 16;
    const double send = hi ? pt[j] : pt[j + 4];
    const double keep = hi ? pt[j + 4] : pt[j];
    pt[j] = keep + __shfl_xor_sync(FULL, send, 16);
  }
#pragma unroll
  for (int j = 0; j < 2; ++j) {
    const bool hi = lane & 8;
    const double send = hi ? pt[j] : pt[j + 2];
    const double keep = hi ? pt[j + 2] : pt[j];
    pt[j] = keep + __shfl_xor_sync(FULL, send, 8);
  }
  {
    const bool hi = lane & 4;
    const double send = hi ? pt[0] : pt[1];
    const double keep = hi ? pt[1] : pt[0];
    pt[0] = keep + __shfl_xor_sync(FULL, send, 4);
  }
  tcol = pt[0];
  return pu[0];
}

__device__ __forceinline__ unsigned ld_relaxed_gpu(const unsigned* p) {
  unsigned v;
  asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

// Deterministic grid-wide sum fused with the grid barrier (as grid_reduce), arriving by a release
// reduction on the monotone counter instead of __threadfence + atomicAdd + __threadfence: one
// GPU-scope fence per CTA and barrier instead of two (tools/mb_gridreduce.cu: 2.84 vs 3.16 us).
__device__ __forceinline__ double grid_reduce_rel(double v, double* red16, double* partials, unsigned* bar,
                                                  unsigned& epoch, double* bc) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, W = blockDim.x >> 5, G = gridDim.x;
  if (lane == 0) red16[warp] = v;
  __syncthreads();
  ++epoch;
  double* ps = partials + (size_t)(epoch & 3) * G;
  if (warp == 0) {
    // the CTA's warp partials summed by a butterfly (bitwise identical in every lane, fixed order)
    // instead of one lane's W dependent shared-memory loads and adds
    const double t = warp_sum(lane < W ? red16[lane] : 0.0);
    if (lane == 0) {
      ps[blockIdx.x] = t;
      asm volatile("red.release.gpu.global.add.u32 [%0], %1;" ::"l"(bar), "r"(1u) : "memory");
      const unsigned target = epoch * (unsigned)G;
      while (ld_acquire_gpu(bar) < target) {
      }
    }
    __syncwarp();
    double sum = 0.0;
    for (int b = lane; b < G; b += 32) sum += __ldcg(ps + b);
    sum = warp_sum(sum);
    if (lane == 0) *bc = sum;
  }
  __syncthreads();
  return *bc;
}

// The on-chip PCG's grid synchronisations arrive on PCG_NBAR counters (128 bytes apart: different L2
// lines) instead of one, CTA b on counter b % PCG_NBAR, so that the 147 arrivals do not serialise on
// one address; lanes 0..PCG_NBAR-1 of warp 0 each acquire one counter.  Same epochs, same
// deterministic partial sums as grid_reduce_rel.
#ifndef PCG_NBAR
#define PCG_NBAR 8
#endif
constexpr int PCG_BAR_STRIDE = 32;   // unsigned words between counters
static_assert(PCG_NBAR >= 1 && PCG_NBAR <= 8, "the context's gbar buffer holds 8 counters (8 x 128 bytes)");
__device__ __forceinline__ void bar_arrive_wait_n(unsigned* bar, unsigned epoch) {
  const int lane = threadIdx.x & 31, G = gridDim.x;
  if (lane == 0)
    asm volatile("red.release.gpu.global.add.u32 [%0], %1;" ::"l"(bar + PCG_BAR_STRIDE * (blockIdx.x % PCG_NBAR)),
                 "r"(1u)
                 : "memory");
  if (lane < PCG_NBAR) {
    const unsigned cnt = (unsigned)((G - lane + PCG_NBAR - 1) / PCG_NBAR);   // CTAs b < G with b % NBAR == lane
    const unsigned target = epoch * cnt;
    const unsigned* ctr = bar + PCG_BAR_STRIDE * lane;
    while (ld_acquire_gpu(ctr) < target) {
    }
  }
  __syncwarp();
}
__device__ __forceinline__ double grid_reduce_n(double v, double* red16, double* partials, unsigned* bar,
                                               unsigned& epoch, double* bc) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, W = blockDim.x >> 5, G = gridDim.x;
  if (lane == 0) red16[warp] = v;
  __syncthreads();
  ++epoch;
  double* ps = partials + (size_t)(epoch & 3) * G;
  if (G == 1) {   // a single CTA (small configurations): the CTA barrier is the grid barrier
    if (warp == 0) {
      const double t = warp_sum(lane < W ? red16[lane] : 0.0);
      if (lane == 0) *bc = t;
    }
    __syncthreads();
    return *bc;
  }
  if (warp == 0) {
    const double t = warp_sum(lane < W ? red16[lane] : 0.0);
    if (lane == 0) ps[blockIdx.x] = t;
    bar_arrive_wait_n(bar, epoch);
    double sum = 0.0;
    for (int b = lane; b < G; b += 32) sum += __ldcg(ps + b);
    sum = warp_sum(sum);
    if (lane == 0) *bc = sum;
  }
  __syncthreads();
  return *bc;
}
__device__ __forceinline__ void grid_barrier_n(unsigned* bar, unsigned& epoch) {
  __syncthreads();
  ++epoch;
  if (gridDim.x == 1) return;   // a single CTA: global writes of the CTA are visible after the CTA barrier
  if ((threadIdx.x >> 5) == 0) bar_arrive_wait_n(bar, epoch);
  __syncthreads();
}

// Mid-size configurations (17 <= n_s <= 224: C3): the whole grid is ONE thread-block cluster of <= 16
// CTAs, so the grid synchronisations are hardware cluster barriers (barrier.cluster arrive.release /
// wait.acquire, which also order the CTAs' global-memory exchange at cluster scope) and the per-CTA
// partials of a reduction are written straight into every CTA's shared memory over DSMEM: no L2 round
// trip for the arrival, the spin or the partials.  Same fixed-order sums (a butterfly over the CTA
// ranks, bitwise identical in every CTA).
__device__ __forceinline__ double cluster_reduce(double v, double* red16, double (*cpart)[16], unsigned& epoch,
                                                 double* bc) {
  cg::cluster_group cl = cg::this_cluster();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, W = blockDim.x >> 5;
  const int G = (int)cl.num_blocks(), me = (int)cl.block_rank();
  if (lane == 0) red16[warp] = v;
  __syncthreads();
  ++epoch;
  if (warp == 0) {
    const double t = warp_sum(lane < W ? red16[lane] : 0.0);
    if (lane < G) *cl.map_shared_rank(&cpart[epoch & 1][me], lane) = t;
  }
  cl.sync();
  if (warp == 0) {
    const double sum = warp_sum(lane < G ? cpart[epoch & 1][lane] : 0.0);
    if (lane == 0) *bc = sum;
  }
  __syncthreads();
  return *bc;
}
__device__ __forceinline__ double sync_reduce(int cluster, double v, double* red16, double (*cpart)[16],
                                              double* partials, unsigned* bar, unsigned& epoch, double* bc) {
  return cluster ? cluster_reduce(v, red16, cpart, epoch, bc) : grid_reduce_n(v, red16, partials, bar, epoch, bc);
}
__device__ __forceinline__ void sync_barrier(int cluster, unsigned* bar, unsigned& epoch) {
  if (cluster) {
    ++epoch;
    cg::this_cluster().sync();
  } else {
    grid_barrier_n(bar, epoch);
  }
}

// Grid barrier without a reduction (release arrival on the same counter / epoch as grid_reduce_rel).
__device__ __forceinline__ void grid_barrier_rel(unsigned* bar, unsigned& epoch) {
  __syncthreads();
  ++epoch;
  if (threadIdx.x == 0) {
    asm volatile("red.release.gpu.global.add.u32 [%0], %1;" ::"l"(bar), "r"(1u) : "memory");
    const unsigned target = epoch * (unsigned)gridDim.x;
    while (ld_acquire_gpu(bar) < target) {
    }
  }
  __syncthreads();
}

// Multi-vector SpMV of the initial guess (replaces k_hist_spmv): V_j = W_j + sum_a U_a W_{E+a,j}
// (own part) and TH[j][E+a][a] = U_a^T W_{E,j} (hand-overs, added by k_hist_gram), warp per
// subdomain.  Each coupling block is read once into the 4 x 8 register tiling of the PCG SpMV and
// applied to all nh vectors; the vector operands come through L1 (read-only) instead of 2 x 32
// shuffles per block column, so the kernel is FMA-bound instead of shuffle-bound.
template <int NFIX>   // NFIX = 32: N known at compile time
__global__ void __launch_bounds__(128) k_hist_spmv_t(HistArgs A) {
  const Geo& g = A.g;
  const int N = NFIX ? NFIX : g.N, lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int E = blockIdx.x * 4 + warp;
  if (E >= g.n_s) return;
  const bool act = lane < N;
  const size_t R = (size_t)g.n_s * N;
  const int nh = A.nh;
  int C[3];
  sub_xyz(g, E, C);
  const int ra = (lane >> 2) * 4, cb = lane & 3;
  const double* Bd = A.blocks + (size_t)E * (1 + g.dim) * N * N;
  double v[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) v[j] = (j < nh && act) ? __ldg(A.W + j * R + E * N + lane) : 0.0;
  for (int a = 0; a < g.dim; ++a) {
    if (C[a] + 1 >= g.S[a]) continue;
    const int En = E + g.Estride[a];
    const double* U = Bd + (size_t)(1 + a) * N * N;
    double u[4][8];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int jj = 0; jj < 8; ++jj) {
        const int r = ra + i, c = cb + 4 * jj;
        u[i][jj] = (r < N && c < N) ? __ldg(U + r * N + c) : 0.0;
      }
#pragma unroll 1
    for (int j = 0; j < nh; ++j) {
      const double* wE = A.W + j * R + (size_t)E * N;
      const double* wN = A.W + j * R + (size_t)En * N;
      double vr[4], vc[8];
#pragma unroll
      for (int i = 0; i < 4; ++i) vr[i] = ra + i < N ? __ldg(wE + ra + i) : 0.0;
#pragma unroll
      for (int jj = 0; jj < 8; ++jj) vc[jj] = cb + 4 * jj < N ? __ldg(wN + cb + 4 * jj) : 0.0;
      double pu[4] = {0.0, 0.0, 0.0, 0.0}, pt[8] = {0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0};
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int jj = 0; jj < 8; ++jj) {
          pu[i] = fma(u[i][jj], vc[jj], pu[i]);
          pt[jj] = fma(u[i][jj], vr[i], pt[jj]);
        }
      double tc;
      const double tu = tile_scatter(pu, pt, lane, tc);
      // v[j] += tu (j is a runtime index: select)
#pragma unroll
      for (int q = 0; q < 8; ++q)
        if (q == j) v[q] += tu;
      if (act) A.TH[((size_t)j * g.n_s * 3 + (size_t)En * 3 + a) * N + lane] = tc;
    }
  }
#pragma unroll
  for (int j = 0; j < 8; ++j)
    if (j < nh && act) A.V[j * R + E * N + lane] = v[j];
}

// The nh x nh Galerkin system for the history weights from the sums of the k_hist_gram partials
// (every thread solves it redundantly; the same arithmetic as pcg_initial_guess).
__device__ __noinline__ void hist_weights(const PcgArgs& A, double* sh, double (&alpha_h)[8]) {
  const int nh = A.nh;
#pragma unroll
  for (int j = 0; j < 8; ++j) alpha_h[j] = 0.0;
  if (nh <= 0) return;
  // the 44 fixed-order sums of the Gram / rhs partials (formed by k_hist_sum before the launch)
  for (int q = threadIdx.x; q < 44; q += blockDim.x) sh[q] = A.gsum[q];
  __syncthreads();
  double G[8][8], rhs8[8];
  int q = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i)
#pragma unroll
    for (int j = i; j < 8; ++j) {
      const double v = (j < nh) ? sh[q] : 0.0;
      G[i][j] = v; G[j][i] = v;
      ++q;
    }
#pragma unroll
  for (int i = 0; i < 8; ++i) rhs8[i] = i < nh ? sh[36 + i] : 0.0;
  bool keep[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    keep[k] = k < nh && G[k][k] > 1e-12 * fabs(G[0][0]) && G[k][k] > 0.0;
    if (keep[k]) {
      const double piv = G[k][k];
#pragma unroll
      for (int i = k + 1; i < 8; ++i) {
        const double f = G[i][k] / piv;
#pragma unroll
        for (int j = k; j < 8; ++j) G[i][j] -= f * G[k][j];
        rhs8[i] -= f * rhs8[k];
      }
    }
  }
#pragma unroll
  for (int k = 7; k >= 0; --k) {
    if (k < nh && keep[k]) {
      double v = rhs8[k];
#pragma unroll
      for (int j = k + 1; j < 8; ++j) v -= G[k][j] * alpha_h[j];
      alpha_h[k] = v / G[k][k];
    }
  }
}

// the same, for one warp (k_pcg_tm: the CTA's warp 0)
__device__ __noinline__ void hist_weights_warp(const PcgArgs& A, double* sh, double (&alpha_h)[8]) {
  const int nh = A.nh;
#pragma unroll
  for (int j = 0; j < 8; ++j) alpha_h[j] = 0.0;
  if (nh <= 0) return;
  // the 44 fixed-order sums of the Gram / rhs partials (formed by k_hist_sum before the launch)
  for (int q = threadIdx.x & 31; q < 44; q += 32) sh[q] = A.gsum[q];
  __syncwarp();
  double G[8][8], rhs8[8];
  int q = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i)
#pragma unroll
    for (int j = i; j < 8; ++j) {
      const double v = (j < nh) ? sh[q] : 0.0;
      G[i][j] = v; G[j][i] = v;
      ++q;
    }
#pragma unroll
  for (int i = 0; i < 8; ++i) rhs8[i] = i < nh ? sh[36 + i] : 0.0;
  bool keep[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    keep[k] = k < nh && G[k][k] > 1e-12 * fabs(G[0][0]) && G[k][k] > 0.0;
    if (keep[k]) {
      const double piv = G[k][k];
#pragma unroll
      for (int i = k + 1; i < 8; ++i) {
        const double f = G[i][k] / piv;
#pragma unroll
        for (int j = k; j < 8; ++j) G[i][j] -= f * G[k][j];
        rhs8[i] -= f * rhs8[k];
      }
    }
  }
#pragma unroll
  for (int k = 7; k >= 0; --k) {
    if (k < nh && keep[k]) {
      double v = rhs8[k];
#pragma unroll
      for (int j = k + 1; j < 8; ++j) v -= G[k][j] * alpha_h[j];
      alpha_h[k] = v / G[k][k];
    }
  }
}

// TMEM block slots per lane quadrant (512 columns / 64 per block)
constexpr int TM_SLOTS = 8;
constexpr int TM_COLS = 512;
// blocks of warp w that do not fit its TMEM quadrant, and the first shared-memory slot of warp w
__host__ __device__ inline int tm_overflow(int w, int dim) {
  const int m = w >> 2, o = dim * m + dim - TM_SLOTS;
  return o < 0 ? 0 : (o > dim ? dim : o);
}
__host__ __device__ inline int tm_slot_base(int w, int dim) {
  int b = 0;
  for (int v = 0; v < w; ++v) b += tm_overflow(v, dim);
  return b;
}

// shared-memory layout of k_pcg_tm (dynamic part), in this order:
//   double ov[n_ov][32][32] (overflow coupling blocks, element k of lane l at [k][l])
//   double yd[W][6][32]     (deflation vectors, zero for missing sides / lanes >= N)
//   float  gs[n_pad]        (staged coarse vector)
//   float  bs[W][n_pad]     (rows of the coarse inverse)
//   float  cr[W][32]        (per-warp partials of the column-sliced coarse product)
struct TmLayout {
  size_t ov, yd, gs, bs, cr, total;
};
__host__ __device__ inline TmLayout tm_layout(int W, int dim, int n_pad) {
  TmLayout L;
  size_t o = 0;
  L.ov = o; o += (size_t)tm_slot_base(W, dim) * 1024 * 8;
  L.yd = o; o += (size_t)W * 6 * 32 * 8;
  L.gs = o; o += (size_t)n_pad * 4;
  L.bs = o; o += (size_t)W * n_pad * 4;
  L.cr = o; o += (size_t)W * 32 * 4;
  L.total = o;
  return L;
}

// debug per-CTA timeline (tstamp buffer, entries 4096 + 8 (it G + CTA) + k, it < 32); compiled only
// with -DLRBMS_DEBUG (tools/exp_timeline.py)
#ifdef LRBMS_DEBUG
#define TM_STAMP(k)                                                                            \
  do {                                                                                         \
    if (A.tstamp && threadIdx.x == 0 && it < 32)                                               \
      A.tstamp[4096 + 8 * ((size_t)it * gridDim.x + blockIdx.x) + (k)] = gtimer();             \
  } while (0)
// debug setup stamps (slots of "iteration 0": tstamp[4096 + 8 CTA + k])
#define TM_SSTAMP(k)                                                                           \
  do {                                                                                         \
    if (A.tstamp && threadIdx.x == 0) A.tstamp[4096 + 8 * (size_t)blockIdx.x + (k)] = gtimer();  \
  } while (0)
#else
#define TM_STAMP(k) do { } while (0)
#define TM_SSTAMP(k) do { } while (0)
#endif

// NFIX = 32: N known at compile time (the lane predicates fold away); MAXT: the block-size bound (448:
// 14 warps, 146 registers per thread; 512: 16 warps for the single-CTA launch of small configurations)
template <int NFIX, int MAXT = 448>
__global__ void __launch_bounds__(MAXT, 1) k_pcg_tm(PcgArgs A) {
  extern __shared__ __align__(16) unsigned char dsm[];
  __shared__ uint32_t tbase_s;
  __shared__ double red16[16];
  __shared__ double bc[4];
  __shared__ double sh46[46];
  __shared__ double cpart[2][16];   // cluster mode: the CTAs' partials of a reduction (written over DSMEM)
  const Geo& g = A.g;
  const int CL = A.cluster;
  const int N = NFIX ? NFIX : g.N, dim = g.dim;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, W = blockDim.x >> 5;
  const int E = blockIdx.x * W + warp;
  const bool own = E < g.n_s;
  const bool act = own && lane < N;
  const TmLayout L = tm_layout(W, dim, A.n_pad);
  double* ov = reinterpret_cast<double*>(dsm + L.ov) + (size_t)tm_slot_base(warp, dim) * 1024;
  const int a_ov = max(0, TM_SLOTS - dim * (warp >> 2));   // blocks a >= a_ov of this warp are in shared memory
  double* yd = reinterpret_cast<double*>(dsm + L.yd) + (size_t)warp * 6 * 32;
  float* gs = reinterpret_cast<float*>(dsm + L.gs);
  float* bs = reinterpret_cast<float*>(dsm + L.bs) + (size_t)warp * A.n_pad;
  const int n4 = A.n_pad >> 2;   // float4 chunks of a coarse row
  const int tm_ncols = TM_COLS;

  TM_SSTAMP(0);
  // ---- TMEM: allocate, then every warp writes its a = 0, 1 coupling tiles
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(smem_addr_u32(&tbase_s)),
                 "r"(tm_ncols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
  // TMEM address of block a of this warp: lane quadrant (warp % 4), columns 64 (dim (warp / 4) + a)
  const uint32_t tcol = tbase_s + ((uint32_t)(32 * (warp & 3)) << 16) + 64u * (uint32_t)(dim * (warp >> 2));

  int C[3] = {0, 0, 0};
  if (own) sub_xyz(g, E, C);
  bool up[3], lo[3];
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    up[a] = own && a < dim && C[a] + 1 < g.S[a];
    lo[a] = own && a < dim && C[a] > 0;
  }
  const int ra = (lane >> 2) * 4, cb = lane & 3;
  // Staging: the rows of the coarse inverse, the shared-memory coupling blocks and the deflation
  // vectors are copied with cp.async (no registers: they stream in the background) while the
  // TMEM-resident blocks go through registers and tcgen05.st.
  if (A.use_coarse) {
    const float4* src = reinterpret_cast<const float4*>(A.Binv + (size_t)(own ? E : 0) * A.n_pad);
    float4* dst = reinterpret_cast<float4*>(bs);
    for (int q = lane; q < (A.n_pad >> 2); q += 32) {
      if (own) tm_cp16(dst + q, src + q);
      else dst[q] = make_float4(0.f, 0.f, 0.f, 0.f);
    }
  }
#pragma unroll
  for (int s = 0; s < 6; ++s) {
    if (A.use_coarse == 2 && act && side_exists(g, C, s)) tm_cp8(yd + s * 32 + lane, A.Yd + ((size_t)E * 6 + s) * N + lane);
    else yd[s * 32 + lane] = 0.0;
  }
  {
    const double* Bd = A.blocks + (size_t)(own ? E : 0) * (1 + dim) * N * N;
    for (int a = a_ov; a < dim; ++a) {   // shared-memory blocks
      const double* U = Bd + (size_t)(1 + a) * N * N;
#pragma unroll
      for (int k = 0; k < 32; ++k) {
        const int i = k >> 3, j = k & 7, r = ra + i, c = cb + 4 * j;
        double* d = ov + (size_t)(a - a_ov) * 1024 + (size_t)k * 32 + lane;
        if (up[a] && r < N && c < N) tm_cp8(d, U + r * N + c);
        else *d = 0.0;
      }
    }
    asm volatile("cp.async.commit_group;\n" ::);
    for (int a = 0; a < min(dim, a_ov); ++a) {   // TMEM blocks
      if (!up[a]) continue;
      const double* U = Bd + (size_t)(1 + a) * N * N;
      double x[32];
#pragma unroll
      for (int k = 0; k < 32; ++k) {
        const int i = k >> 3, j = k & 7, r = ra + i, c = cb + 4 * j;
        x[k] = (r < N && c < N) ? __ldg(U + r * N + c) : 0.0;
      }
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        uint32_t v[32];
#pragma unroll
        for (int k = 0; k < 16; ++k) {
          v[2 * k] = (uint32_t)__double2loint(x[16 * h + k]);
          v[2 * k + 1] = (uint32_t)__double2hiint(x[16 * h + k]);
        }
        tm_st32(tcol + 64u * a + 32u * h, v);
      }
    }
    asm volatile("tcgen05.wait::st.sync.aligned;\n" ::: "memory");
    asm volatile("cp.async.wait_all;\n" ::: "memory");
  }
  const double zh = act ? A.zh[E * N + lane] : 0.0;
  TM_SSTAMP(1);
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");

  // coarse product e_E = (B_c^-1 gs)_E, the row of E in shared memory
  auto coarse_dot = [&]() -> float {
    const float4* g4 = reinterpret_cast<const float4*>(gs);
    const float4* b4 = reinterpret_cast<const float4*>(bs);
    float e0 = 0.f, e1 = 0.f;
#pragma unroll 4
    for (int F = lane; F < n4; F += 32) {
      const float4 b = b4[F], c = g4[F];
      e0 = fmaf(b.x, c.x, e0);
      e1 = fmaf(b.y, c.y, e1);
      e0 = fmaf(b.z, c.z, e0);
      e1 = fmaf(b.w, c.w, e1);
    }
    float e = e0 + e1;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) e += __shfl_xor_sync(FULL, e, o);
    return e;
  };
  auto coarse_gemv = [&]() -> float { return coarse_dot(); };
  auto stage_wc = [&]() {
    for (int i = threadIdx.x; i < A.n_pad; i += blockDim.x) gs[i] = i < g.n_s ? (float)__ldcg(A.wc + i) : 0.f;
    __syncthreads();
  };
  auto stage_g = [&]() {   // Zh^T (I - Bh) r = -(sum of the six neighbour contributions), fixed order
    const float* cw = A.cont_tm;   // [6][n_pad], coalesced float4 over F
    for (int q = threadIdx.x; q < (A.n_pad >> 2); q += blockDim.x) {
      float4 c[6];
#pragma unroll
      for (int sd = 0; sd < 6; ++sd) c[sd] = __ldcg(reinterpret_cast<const float4*>(cw + (size_t)sd * A.n_pad) + q);
      float4 v;
      v.x = -(((((c[0].x + c[1].x) + c[2].x) + c[3].x) + c[4].x) + c[5].x);
      v.y = -(((((c[0].y + c[1].y) + c[2].y) + c[3].y) + c[4].y) + c[5].y);
      v.z = -(((((c[0].z + c[1].z) + c[2].z) + c[3].z) + c[4].z) + c[5].z);
      v.w = -(((((c[0].w + c[1].w) + c[2].w) + c[3].w) + c[4].w) + c[5].w);
      reinterpret_cast<float4*>(gs)[q] = v;
    }
    __syncthreads();
  };
  // contributions Y_{E,F} . r_E to the coarse rhs of the neighbours F (as defl_scatter)
  auto scatter = [&](double rk) {
    double d[8];
#pragma unroll
    for (int s = 0; s < 6; ++s) d[s] = yd[s * 32 + lane] * rk;
    d[6] = d[7] = 0.0;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const bool hi = lane & 16;
      const double send = hi ? d[i] : d[i + 4];
      const double keep = hi ? d[i + 4] : d[i];
      d[i] = keep + __shfl_xor_sync(FULL, send, 16);
    }
#pragma unroll
    for (int i = 0; i < 2; ++i) {
      const bool hi = lane & 8;
      const double send = hi ? d[i] : d[i + 2];
      const double keep = hi ? d[i + 2] : d[i];
      d[i] = keep + __shfl_xor_sync(FULL, send, 8);
    }
    {
      const bool hi = lane & 4;
      const double send = hi ? d[0] : d[1];
      const double keep = hi ? d[1] : d[0];
      d[0] = keep + __shfl_xor_sync(FULL, send, 4);
    }
    d[0] += __shfl_xor_sync(FULL, d[0], 2);
    d[0] += __shfl_xor_sync(FULL, d[0], 1);
    const int s = lane >> 2;
    if (own && (lane & 3) == 0 && s < 6 && side_exists(g, C, s)) A.cont_tm[(size_t)s * A.n_pad + side_nb(g, E, s)] = (float)d[0];
  };

  unsigned epoch = 0;
  double* gparts = A.partials + 8 * (size_t)gridDim.x;

  // ---- initial guess: Galerkin combination of the history, y0 = W alpha, r0 = rb - V alpha
  double alpha_h[8];
  TM_SSTAMP(2);
  {   // one warp solves the 8 x 8 history system (every thread of the CTA doing it was 7-18 us of
      // fp64 divisions competing for the pipe), the weights go to the others through shared memory
    __shared__ double ah_s[8];
    if (warp == 0) {
      hist_weights_warp(A, sh46, alpha_h);
      if (lane < 8) ah_s[lane] = alpha_h[lane];
    }
    __syncthreads();
#pragma unroll
    for (int j = 0; j < 8; ++j) alpha_h[j] = ah_s[j];
  }
  TM_SSTAMP(3);
  const size_t R = (size_t)g.n_s * N;
  double y = 0.0, r = 0.0;
  double pbb = 0.0;
  if (own) {
    const double rbk = act ? A.rb[E * N + lane] : 0.0;
    r = rbk;
#pragma unroll
    for (int j = 0; j < 8; ++j)
      if (j < A.nh && act) {
        y += alpha_h[j] * A.W[j * R + E * N + lane];
        r -= alpha_h[j] * A.V[j * R + E * N + lane];
      }
    pbb = warp_sum(rbk * rbk);
    const double w = warp_sum(zh * r);
    if (lane == 0) A.wc[E] = w;
  }
  TM_SSTAMP(4);
  const double bb = sync_reduce(CL, pbb, red16, cpart, gparts, A.gbar, epoch, &bc[0]);
  TM_SSTAMP(5);
  const double tol2 = A.rtol * A.rtol * bb;
  double rr = 1.0;
  int it = 0;
  if (bb > 0.0) {
    if (A.use_coarse == 2) {
      // DEF starting vector (see k_pcg): y0 += Zh e0, e0 = B_c^-1 Zh^T r; r0 -= Bh Zh e0
      stage_wc();
      const float e = coarse_dot();
      if (own) {
        if (lane == 0) A.e0[E] = (double)e;
        y += zh * (double)e;
      }
      sync_barrier(CL, A.gbar, epoch);
      if (own) {
        double rk = r - zh * __ldcg(A.e0 + E);
#pragma unroll
        for (int s = 0; s < 6; ++s)
          if (act && side_exists(g, C, s)) rk -= yd[s * 32 + lane] * __ldcg(A.e0 + side_nb(g, E, s));
        r = act ? rk : 0.0;
      }
      scatter(r);
      sync_barrier(CL, A.gbar, epoch);
      stage_g();
    } else if (A.use_coarse == 1) {
      stage_wc();
    }
    double z = r;
    if (A.use_coarse) { const float ec = coarse_dot(); z = act ? r + zh * (double)ec : 0.0; }
    if (act) A.z[E * N + lane] = z;
    double rz = sync_reduce(CL, own ? warp_sum(z * r) : 0.0, red16, cpart, gparts, A.gbar, epoch, &bc[0]);
    TM_SSTAMP(6);
    double beta = 0.0, p = 0.0;
    for (it = (rz <= tol2) ? A.max_iters + 2 : 1; it <= A.max_iters; ++it) {
      double* pcur = (it & 1) ? A.pb1 : A.pb0;
      const double* pold = (it & 1) ? A.pb0 : A.pb1;
      const bool first = it == 1;
      // ---------------- A: p, q_own = (I + U) p, hand-overs, p.Bh p
      TM_STAMP(0);
      p = first ? z : z + beta * p;
      double qown = p, local = p * p;
      if (own) {
        if (act) pcur[E * N + lane] = p;
        double zn[3], pn[3];
#pragma unroll
        for (int a = 0; a < 3; ++a) {
          zn[a] = 0.0; pn[a] = 0.0;
          if (up[a] && act) {
            const int En = E + g.Estride[a];
            zn[a] = __ldcg(A.z + En * N + lane);
            if (!first) pn[a] = __ldcg(pold + En * N + lane);
          }
        }
        double vr[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) vr[i] = __shfl_sync(FULL, p, ra + i);
#pragma unroll
        for (int a = 0; a < 3; ++a) {
          if (!up[a]) continue;
          double pu[4] = {0.0, 0.0, 0.0, 0.0}, pt[8] = {0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0};
          double vc[8];
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            double u[16];
            if (a < a_ov) {
              uint32_t v[32];
              tm_ld32(tcol + 64u * a + 32u * h, v);
#pragma unroll
              for (int k = 0; k < 16; ++k) u[k] = __hiloint2double((int)v[2 * k + 1], (int)v[2 * k]);
            } else {
#pragma unroll
              for (int k = 0; k < 16; ++k) u[k] = ov[(size_t)(a - a_ov) * 1024 + (size_t)(16 * h + k) * 32 + lane];
            }
            // the column part first (own p only), so the neighbour loads of zn, pn are still in flight
            tile_half<false, true>(u, h, vr, vc, pu, pt);
            if (h == 0) {
              const double vN = first ? zn[a] : fma(beta, pn[a], zn[a]);
#pragma unroll
              for (int j = 0; j < 8; ++j) vc[j] = __shfl_sync(FULL, vN, cb + 4 * j);
            }
            tile_half<true, false>(u, h, vr, vc, pu, pt);
          }
          double tc;
          const double tu = tile_scatter(pu, pt, lane, tc);
          qown += tu;
          local = fma(2.0 * p, tu, local);
          if (act) A.T[((size_t)(E + g.Estride[a]) * 3 + a) * N + lane] = tc;
        }
      }
      LRBMS_TSTAMP(A.tstamp && blockIdx.x == 0 && threadIdx.x == 0 && it < 64, A.tstamp[4 * it + 0], gtimer());
      TM_STAMP(1);
      const double pq = sync_reduce(CL, own ? warp_sum(act ? local : 0.0) : 0.0, red16, cpart, gparts, A.gbar, epoch, &bc[0]);
      LRBMS_TSTAMP(A.tstamp && blockIdx.x == 0 && threadIdx.x == 0 && it < 64, A.tstamp[4 * it + 1], gtimer());
      if (!(pq > 0.0)) {
        if (blockIdx.x == 0 && threadIdx.x == 0) atomicOr(A.flags, FLAG_BREAKDOWN);
        break;
      }
      TM_STAMP(2);
      const double alpha = rz / pq;
      // ---------------- B: y, r, r.r, coarse rhs contributions
      double q = qown;
#pragma unroll
      for (int a = 0; a < 3; ++a)
        if (lo[a] && act) q += __ldcg(A.T + ((size_t)E * 3 + a) * N + lane);
      y = fma(alpha, p, y);
      r = act ? fma(-alpha, q, r) : 0.0;
      if (A.use_coarse == 2) {
        scatter(r);
      } else if (A.use_coarse == 1 && own) {
        const double w = warp_sum(zh * r);
        if (lane == 0) A.wc[E] = w;
      }
      TM_STAMP(3);
      sync_barrier(CL, A.gbar, epoch);
      LRBMS_TSTAMP(A.tstamp && blockIdx.x == 0 && threadIdx.x == 0 && it < 64, A.tstamp[4 * it + 2], gtimer());
      TM_STAMP(4);
      // ---------------- C: z = M^-1 r, r.z
      if (A.use_coarse == 2) stage_g();
      else if (A.use_coarse == 1) stage_wc();
      TM_STAMP(5);
      z = r;
      if (A.use_coarse) { const float ec = coarse_gemv(); z = act ? r + zh * (double)ec : 0.0; }
      if (act) A.z[E * N + lane] = z;
      TM_STAMP(6);
      const double rz_new = sync_reduce(CL, own ? warp_sum(z * r) : 0.0, red16, cpart, gparts, A.gbar, epoch, &bc[0]);
      LRBMS_TSTAMP(A.tstamp && blockIdx.x == 0 && threadIdx.x == 0 && it < 64, A.tstamp[4 * it + 3], gtimer());
      TM_STAMP(7);
      rr = rz_new;
      if (!(rz_new == rz_new)) break;   // NaN (flagged below)
      if (rz_new <= tol2) break;
      beta = rz_new / rz;
      rz = rz_new;
    }
    if (it == A.max_iters + 2) it = 0;
  } else {
    rr = 0.0;
  }
  TM_SSTAMP(7);
  // ---- back-transform c = L^-T y
  if (own) {
    const double* Li = A.Linv + (size_t)E * N * N;
    double xk = 0.0;
    for (int i = 0; i < N; ++i) {
      const double yi = __shfl_sync(FULL, y, i);
      if (act) xk += Li[i * N + lane] * yi;
    }
    if (act) {
      A.x[E * N + lane] = xk;
      A.hist_out[E * N + lane] = xk;
      A.y[E * N + lane] = y;
    }
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    A.iters[0] = it;
    A.iters[1] += min(it, A.max_iters);
    if (it > A.max_iters) atomicOr(A.flags, FLAG_NOCONV);
    if (!(rr == rr)) atomicOr(A.flags, FLAG_NAN);
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tbase_s), "r"(tm_ncols));
}

}  // namespace lrbms
