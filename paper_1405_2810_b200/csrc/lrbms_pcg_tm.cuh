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
//     element-interleaved over lanes (bank-conflict free).  C5 (14 warps): 46 blocks in TMEM, 10 in
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

#ifndef TM_SPIN
#define TM_SPIN 0     // grid reduction wait: 0 acquire spin on the counter, 1 relaxed + backoff, 2 last-arriver flag
#endif
#ifndef TM_NS
#define TM_NS 32      // backoff (ns) of the relaxed spins
#endif
#ifndef TM_NS_P2P
#define TM_NS_P2P 0   // backoff (ns) of the neighbour-flag spins
#endif

namespace lrbms {

__device__ __forceinline__ uint32_t smem_addr_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
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

// column part of tile_scatter only: (U^T w)[lane]
__device__ __forceinline__ double tile_scatter_cols(double (&pt)[8], int lane) {
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
  const bool hi = lane & 4;
  const double send = hi ? pt[0] : pt[1];
  const double keep = hi ? pt[1] : pt[0];
  return keep + __shfl_xor_sync(FULL, send, 4);
}
// row part only: (U v)[lane]
__device__ __forceinline__ double tile_scatter_rows(double (&pu)[4], int lane) {
#pragma unroll
  for (int i = 0; i < 2; ++i) {
    const bool hi = lane & 2;
    const double send = hi ? pu[i] : pu[i + 2];
    const double keep = hi ? pu[i + 2] : pu[i];
    pu[i] = keep + __shfl_xor_sync(FULL, send, 2);
  }
  const bool hi = lane & 1;
  const double send = hi ? pu[0] : pu[1];
  const double keep = hi ? pu[1] : pu[0];
  return keep + __shfl_xor_sync(FULL, send, 1);
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
__device__ __forceinline__ void st_release_u32(unsigned* p, unsigned v) {
  asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

// Two deterministic grid-wide sums fused with a grid barrier: per-CTA partials (warps in order) ->
// arrival by a release reduction on the monotone counter (no separate fence) -> acquire spin ->
// warp 0 sums the per-CTA partials in a fixed order -> shared broadcast.  Shares the counter and the
// epoch with grid_reduce; partial slots 16G + (epoch % 4) 2G.
__device__ __forceinline__ double grid_reduce2(double v0, double v1, double (*red)[16], double* partials, unsigned* bar,
                                               unsigned& epoch, double* bc, double& out1,
                                               unsigned long long* dbg = nullptr) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, W = blockDim.x >> 5, G = gridDim.x;
  if (lane == 0) {
    red[0][warp] = v0;
    red[1][warp] = v1;
  }
  __syncthreads();
  if (dbg && threadIdx.x == 0) dbg[0] = gtimer();
  ++epoch;
  double* ps = partials + 16 * (size_t)G + (size_t)(epoch & 3) * 2 * G;
  if (warp == 0) {
    if (lane == 0) {
      double t0 = 0.0, t1 = 0.0;
      for (int w = 0; w < W; ++w) {
        t0 += red[0][w];
        t1 += red[1][w];
      }
      ps[blockIdx.x] = t0;
      ps[G + blockIdx.x] = t1;
      const unsigned target = epoch * (unsigned)G;
#if TM_SPIN == 2
      // the last arriver releases a flag on another 128-byte line: the pollers do not contend with
      // the arrivals on the counter line
      unsigned old;
      asm volatile("atom.acq_rel.gpu.global.add.u32 %0, [%1], %2;" : "=r"(old) : "l"(bar), "r"(1u) : "memory");
      if (dbg) dbg[1] = gtimer();
      if (old == target - 1) {
        st_release_u32(bar + 32, epoch);
      } else {
        while (ld_relaxed_gpu(bar + 32) < epoch) __nanosleep(TM_NS);
        ld_acquire_gpu(bar + 32);
      }
#else
      asm volatile("red.release.gpu.global.add.u32 [%0], %1;" ::"l"(bar), "r"(1u) : "memory");
      if (dbg) dbg[1] = gtimer();
#if TM_SPIN == 1
      while (ld_relaxed_gpu(bar) < target) __nanosleep(TM_NS);
      ld_acquire_gpu(bar);
#else
      while (ld_acquire_gpu(bar) < target) {
      }
#endif
#endif
      if (dbg) dbg[2] = gtimer();
    }
    __syncwarp();
    double s0 = 0.0, s1 = 0.0;
    for (int b = lane; b < G; b += 32) {
      s0 += __ldcg(ps + b);
      s1 += __ldcg(ps + G + b);
    }
    s0 = warp_sum(s0);
    s1 = warp_sum(s1);
    if (lane == 0) {
      bc[0] = s0;
      bc[1] = s1;
    }
  }
  __syncthreads();
  out1 = bc[1];
  return bc[0];
}

// Sums of the k_hist_gram partials and the nh x nh Galerkin system for the history weights
// (every thread solves it redundantly; the same arithmetic as pcg_initial_guess).
__device__ __noinline__ void hist_weights(const PcgArgs& A, double* sh, double (&alpha_h)[8]) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int nh = A.nh;
#pragma unroll
  for (int j = 0; j < 8; ++j) alpha_h[j] = 0.0;
  if (nh <= 0) return;
  if (warp == 0) {
    for (int q = 0; q < 44; ++q) {
      double v = 0.0;
      for (int b = lane; b < A.ngram; b += 32) v += A.gpart[q * A.ngram + b];
      v = warp_sum(v);
      if (lane == 0) sh[q] = v;
    }
  }
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
//   float  yd[W][6][32]     (deflation vectors in fp32 for the coarse right-hand sides, which are
//                            fp32; zero for missing sides / lanes >= N)
//   float  gs[2][n_pad]     (staged coarse vectors g(w), g(r))
//   float  bs[W][n_pad]     (rows of the coarse inverse)
//   float  cr[W][64]        (per-warp partials of the column-sliced coarse products)
struct TmLayout {
  size_t ov, yd, gs, bs, cr, total;
};
__host__ __device__ inline TmLayout tm_layout(int W, int dim, int n_pad) {
  TmLayout L;
  size_t o = 0;
  L.ov = o; o += (size_t)tm_slot_base(W, dim) * 1024 * 8;
  L.yd = o; o += (size_t)W * 6 * 32 * 4;
  L.gs = o; o += 2 * (size_t)n_pad * 4;
  L.bs = o; o += (size_t)W * n_pad * 4;
  L.cr = o; o += (size_t)W * 64 * 4;   // coarse-product partials [W warps][2 x 32]
  L.total = o;
  return L;
}

// debug progress marker (tstamp buffer, entries 256 + CTA): last stage reached by each CTA
// debug per-CTA timeline (tstamp buffer, entries 4096 + 4 (it G + CTA) + k, it < 32)
#define TM_STAMP(k)                                                                            \
  do {                                                                                         \
    if (A.tstamp && threadIdx.x == 0 && it < 32)                                               \
      A.tstamp[4096 + 8 * ((size_t)it * gridDim.x + blockIdx.x) + (k)] = gtimer();             \
  } while (0)
// debug per-warp stamps (entries 65536 + 4 ((it G + CTA) 16 + warp) + k, it < 16)
#define TM_WSTAMP(k)                                                                           \
  do {                                                                                         \
    if (A.tstamp && lane == 0 && it < 16)                                                      \
      A.tstamp[65536 + 4 * (((size_t)it * gridDim.x + blockIdx.x) * 16 + warp) + (k)] = gtimer(); \
  } while (0)
#define TM_PROG(code)                                                                          \
  do {                                                                                         \
    if (A.tstamp && threadIdx.x == 0) {                                                        \
      reinterpret_cast<volatile unsigned long long*>(A.tstamp)[256 + blockIdx.x] = (code);     \
      __threadfence_system();                                                                  \
    }                                                                                          \
  } while (0)

__global__ void __launch_bounds__(448, 1) k_pcg_tm(PcgArgs A) {
  extern __shared__ __align__(16) unsigned char dsm[];
  __shared__ uint32_t tbase_s;
  __shared__ double red16[16];
  __shared__ double red32[2][16];
  __shared__ double bc[4];
  __shared__ double sh46[46];
  const Geo& g = A.g;
  const int N = g.N, dim = g.dim;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, W = blockDim.x >> 5;
  const int E = blockIdx.x * W + warp;
  const bool own = E < g.n_s;
  const bool act = own && lane < N;
  const TmLayout L = tm_layout(W, dim, A.n_pad);
  double* ov = reinterpret_cast<double*>(dsm + L.ov) + (size_t)tm_slot_base(warp, dim) * 1024;
  const int a_ov = max(0, TM_SLOTS - dim * (warp >> 2));   // blocks a >= a_ov of this warp are in shared memory
  float* yd = reinterpret_cast<float*>(dsm + L.yd) + (size_t)warp * 6 * 32;
  float* gs = reinterpret_cast<float*>(dsm + L.gs);   // g(w) in gs[0..n_pad), g(r) in gs[n_pad..2 n_pad)
  float* bs = reinterpret_cast<float*>(dsm + L.bs) + (size_t)warp * A.n_pad;
  float* bs0 = reinterpret_cast<float*>(dsm + L.bs);
  float* cr = reinterpret_cast<float*>(dsm + L.cr);
  const int n4 = A.n_pad >> 2;   // float4 chunks of a coarse row
  const int tm_ncols = TM_COLS;

  // ---- TMEM: allocate, then every warp writes its a = 0, 1 coupling tiles
  TM_PROG(1);
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

  TM_PROG(2);
  int C[3] = {0, 0, 0};
  if (own) sub_xyz(g, E, C);
  bool up[3], lo[3];
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    up[a] = own && a < dim && C[a] + 1 < g.S[a];
    lo[a] = own && a < dim && C[a] > 0;
  }
  const int ra = (lane >> 2) * 4, cb = lane & 3;
  {
    const double* Bd = A.blocks + (size_t)(own ? E : 0) * (1 + dim) * N * N;
#pragma unroll 1
    for (int a = 0; a < dim; ++a) {
      if (!up[a]) continue;
      const double* U = Bd + (size_t)(1 + a) * N * N;
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        uint32_t v[32];
#pragma unroll
        for (int ii = 0; ii < 2; ++ii)
#pragma unroll
          for (int j = 0; j < 8; ++j) {
            const int r = ra + 2 * h + ii, c = cb + 4 * j;
            const double x = (r < N && c < N) ? U[r * N + c] : 0.0;
            if (a < a_ov) {
              v[2 * (ii * 8 + j)] = (uint32_t)__double2loint(x);
              v[2 * (ii * 8 + j) + 1] = (uint32_t)__double2hiint(x);
            } else {
              ov[(size_t)(a - a_ov) * 1024 + (size_t)(16 * h + ii * 8 + j) * 32 + lane] = x;
            }
          }
        if (a < a_ov) tm_st32(tcol + 64u * a + 32u * h, v);
      }
    }
    asm volatile("tcgen05.wait::st.sync.aligned;\n" ::: "memory");
  }
#pragma unroll
  for (int s = 0; s < 6; ++s) {
    double v = 0.0;
    if (A.use_coarse == 2 && act && side_exists(g, C, s)) v = A.Yd[((size_t)E * 6 + s) * N + lane];
    yd[s * 32 + lane] = (float)v;
  }
  if (A.use_coarse) {
    const float4* src = reinterpret_cast<const float4*>(A.Binv + (size_t)(own ? E : 0) * A.n_pad);
    float4* dst = reinterpret_cast<float4*>(bs);
    for (int q = lane; q < (A.n_pad >> 2); q += 32) dst[q] = own ? __ldcs(src + q) : make_float4(0.f, 0.f, 0.f, 0.f);
  }
  const double zh = act ? A.zh[E * N + lane] : 0.0;
  TM_PROG(3);
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  TM_PROG(4);
  asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");

  // coarse product e_E = (B_c^-1 gs)_E, the row of E in shared memory
  auto coarse_dot = [&](const float* gsrc) -> float {
    const float4* g4 = reinterpret_cast<const float4*>(gsrc);
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
  // Both coarse products of the CTA's rows at once, sliced by COLUMNS: warp v takes a contiguous
  // slice of the float4 chunks of g(w), g(r) (gs[0..n_pad), gs[n_pad..2 n_pad)) and runs it against
  // all W rows, so every row and both vectors are read from shared memory once (128 KB per SM for
  // C5 instead of 448 KB with a row per warp).  Lane partials -> reduce-scatter (lane 2 j + v holds
  // row j, vector v) -> per-warp slots -> fixed-order sum over the warps.  Returns this warp's
  // (e_w, e_r) for its own row.
  auto coarse_gemv2 = [&](float& ew, float& er) {
    const int n4c = A.n_pad >> 2;
    const int q0 = (warp * n4c) / W, q1 = ((warp + 1) * n4c) / W;
    const float4* gw4 = reinterpret_cast<const float4*>(gs);
    const float4* gr4 = reinterpret_cast<const float4*>(gs + A.n_pad);
    float acc[32];
#pragma unroll
    for (int k = 0; k < 32; ++k) acc[k] = 0.f;
    for (int q = q0 + lane; q < q1; q += 32) {
      const float4 a = gw4[q], b = gr4[q];
#pragma unroll
      for (int j = 0; j < 16; ++j) {
        if (j < W) {
          const float4 m = reinterpret_cast<const float4*>(bs0 + (size_t)j * A.n_pad)[q];
          acc[2 * j] = fmaf(m.x, a.x, fmaf(m.y, a.y, fmaf(m.z, a.z, fmaf(m.w, a.w, acc[2 * j]))));
          acc[2 * j + 1] = fmaf(m.x, b.x, fmaf(m.y, b.y, fmaf(m.z, b.z, fmaf(m.w, b.w, acc[2 * j + 1]))));
        }
      }
    }
    // reduce-scatter of the 32 partials over the 32 lanes: lane l ends with the total of value l
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      const bool hi = lane & 16;
      const float send = hi ? acc[i] : acc[i + 16];
      const float keep = hi ? acc[i + 16] : acc[i];
      acc[i] = keep + __shfl_xor_sync(FULL, send, 16);
    }
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const bool hi = lane & 8;
      const float send = hi ? acc[i] : acc[i + 8];
      const float keep = hi ? acc[i + 8] : acc[i];
      acc[i] = keep + __shfl_xor_sync(FULL, send, 8);
    }
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const bool hi = lane & 4;
      const float send = hi ? acc[i] : acc[i + 4];
      const float keep = hi ? acc[i + 4] : acc[i];
      acc[i] = keep + __shfl_xor_sync(FULL, send, 4);
    }
#pragma unroll
    for (int i = 0; i < 2; ++i) {
      const bool hi = lane & 2;
      const float send = hi ? acc[i] : acc[i + 2];
      const float keep = hi ? acc[i + 2] : acc[i];
      acc[i] = keep + __shfl_xor_sync(FULL, send, 2);
    }
    {
      const bool hi = lane & 1;
      const float send = hi ? acc[0] : acc[1];
      const float keep = hi ? acc[1] : acc[0];
      acc[0] = keep + __shfl_xor_sync(FULL, send, 1);
    }
    // lane l holds value index v(l) = bit-reversed order of the halving steps: lane bits 4..0 select
    // halves 16, 8, 4, 2, 1 -> value index = lane (the "hi" half keeps the upper values)
    cr[warp * 64 + lane] = acc[0];
    __syncthreads();
    float tw = 0.f, tr = 0.f;
    for (int v = 0; v < W; ++v) {
      tw += cr[v * 64 + 2 * warp];
      tr += cr[v * 64 + 2 * warp + 1];
    }
    ew = tw;
    er = tr;
  };
  // stage Zh^T v (additive coarse level): nv vectors of n_pad doubles at wcb -> gs
  auto stage_wc = [&](const double* wcb, int nv) {
    for (int i = threadIdx.x; i < nv * A.n_pad; i += blockDim.x) {
      const int ii = i % A.n_pad;
      gs[i] = ii < g.n_s ? (float)__ldcg(wcb + i) : 0.f;
    }
    __syncthreads();
  };
  // stage Zh^T (I - Bh) v = -(sum of the six neighbour contributions), fixed order, from
  // contributions laid out [F][8] (slot s = side) -> gs
  auto stage_g8 = [&](const float* cb) {
    for (int F = threadIdx.x; F < A.n_pad; F += blockDim.x) {
      float v = 0.f;
      if (F < g.n_s) {
        const float4 c0 = __ldcg(reinterpret_cast<const float4*>(cb + (size_t)F * 8));
        const float2 c1 = __ldcg(reinterpret_cast<const float2*>(cb + (size_t)F * 8 + 4));
        v = -(((((c0.x + c0.y) + c0.z) + c0.w) + c1.x) + c1.y);
      }
      gs[F] = v;
    }
    __syncthreads();
  };
  // the same from side-major contributions [6][n_pad] (coalesced float4 over F) -> gs[0..n_pad),
  // together with a copy of the pre-summed vector gr[n_pad] -> gs[n_pad..2 n_pad)
  auto stage_g6 = [&](const float* cw, const float* gr) {
    const int n4 = A.n_pad >> 2;
    for (int q = threadIdx.x; q < 2 * n4; q += blockDim.x) {
      float4 v;
      if (q < n4) {
        float4 c[6];
#pragma unroll
        for (int sd = 0; sd < 6; ++sd) c[sd] = __ldcg(reinterpret_cast<const float4*>(cw + (size_t)sd * A.n_pad) + q);
        v.x = -(((((c[0].x + c[1].x) + c[2].x) + c[3].x) + c[4].x) + c[5].x);
        v.y = -(((((c[0].y + c[1].y) + c[2].y) + c[3].y) + c[4].y) + c[5].y);
        v.z = -(((((c[0].z + c[1].z) + c[2].z) + c[3].z) + c[4].z) + c[5].z);
        v.w = -(((((c[0].w + c[1].w) + c[2].w) + c[3].w) + c[4].w) + c[5].w);
      } else {
        v = __ldcg(reinterpret_cast<const float4*>(gr) + (q - n4));
      }
      reinterpret_cast<float4*>(gs)[q] = v;
    }
    __syncthreads();
  };
  // contributions Y_{E,F} . r_E to the coarse rhs of the neighbours F (as defl_scatter), stored at
  // cb[F sF + s ss] (s = the side of E that faces F)
  auto scatter = [&](double rk, float* cb, int sF, int ss) {
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
    if (own && (lane & 3) == 0 && s < 6 && side_exists(g, C, s)) cb[(size_t)side_nb(g, E, s) * sF + s * ss] = (float)d[0];
  };

  unsigned epoch = 0;
  double* gparts = A.partials + 8 * (size_t)gridDim.x;

  // ---- initial guess: Galerkin combination of the history, y0 = W alpha, r0 = rb - V alpha
  double alpha_h[8];
  hist_weights(A, sh46, alpha_h);
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
  TM_PROG(5);
  const double bb = grid_reduce(pbb, red16, gparts, A.gbar, epoch, &bc[0]);
  TM_PROG(6);
  const double tol2 = A.rtol * A.rtol * bb;
  double rr = 1.0;
  int it = 0;
  if (bb > 0.0) {
    if (A.use_coarse == 2) {
      // DEF starting vector (see k_pcg): y0 += Zh e0, e0 = B_c^-1 Zh^T r; r0 -= Bh Zh e0
      TM_PROG(60);
      stage_wc(A.wc, 1);
      TM_PROG(61);
      const float e = coarse_dot(gs);
      TM_PROG(62);
      if (own) {
        if (lane == 0) A.e0[E] = (double)e;
        y += zh * (double)e;
      }
      grid_reduce(0.0, red16, gparts, A.gbar, epoch, &bc[0]);
      TM_PROG(63);
      if (own) {
        double rk = r - zh * __ldcg(A.e0 + E);
#pragma unroll
        for (int s = 0; s < 6; ++s)
          if (act && side_exists(g, C, s)) rk -= A.Yd[((size_t)E * 6 + s) * N + lane] * __ldcg(A.e0 + side_nb(g, E, s));
        r = act ? rk : 0.0;
      }
      TM_PROG(64);
      scatter(r, A.cont, 8, 1);   // the k_pcg layout [F][8]: not touched by the iteration below
      TM_PROG(65);
      grid_reduce(0.0, red16, gparts, A.gbar, epoch, &bc[0]);
      TM_PROG(66);
      stage_g8(A.cont);
      TM_PROG(67);
    } else if (A.use_coarse == 1) {
      stage_wc(A.wc, 1);
    }
    // ---- PCG in the Chronopoulos-Gear form (one grid reduction of gamma = r.u and delta = w.u per
    // iteration, u = M^-1 r, w = Bh u, s = Bh p by recurrence) with point-to-point neighbour flags
    // instead of grid barriers for the SpMV exchange.  The coarse correction of u is carried by the
    // recurrences e_s = e_w + beta e_s, e_r -= alpha e_s of e = (B_c^-1 Zh^T (I - Bh) .)_E, linear in
    // its argument, so only e_w = (B_c^-1 g(w))_E is formed from gathered data each iteration.
    double e_r = 0.0, u = r;
    if (A.use_coarse) {
      const float ec = coarse_dot(gs);
      e_r = (double)ec;
      u = act ? r + zh * e_r : 0.0;
    }
    int nbu[3], nbl[3];
    unsigned upm = 0, lom = 0;
#pragma unroll
    for (int a = 0; a < 3; ++a) {
      nbu[a] = up[a] ? E + g.Estride[a] : 0;
      nbl[a] = lo[a] ? E - g.Estride[a] : 0;
      upm |= up[a] ? 1u << a : 0u;
      lom |= lo[a] ? 1u << a : 0u;
    }
    // lanes 0..2 wait for upper neighbour a = lane, lanes 3..5 for lower neighbour a = lane - 3
    const int my_nb = lane == 0 ? nbu[0] : lane == 1 ? nbu[1] : lane == 2 ? nbu[2] : lane == 3 ? nbl[0] : lane == 4 ? nbl[1] : nbl[2];
    const bool waits = lane < 3 ? ((upm >> lane) & 1u) : lane < 6 ? ((lom >> (lane - 3)) & 1u) : false;
    // one flag per subdomain ("u and the hand-overs of this iteration are published"), one 128-byte
    // line each so that pollers of one flag do not contend with the writers of others
    constexpr int FS = 32;
    unsigned* flag = A.pflags;
    double p = 0.0, sv = 0.0, e_s = 0.0, gamma_old = 1.0, alpha_old = 1.0, gamma = 0.0;
    int nit = 0;
    // one pass over the coupling tiles: rows (U v into pu) and/or columns (U^T vr into pt)
    auto load_half = [&](int a, int h, double (&ut)[16]) {
      if (a < a_ov) {
        uint32_t v[32];
        tm_ld32(tcol + 64u * a + 32u * h, v);
#pragma unroll
        for (int k = 0; k < 16; ++k) ut[k] = __hiloint2double((int)v[2 * k + 1], (int)v[2 * k]);
      } else {
#pragma unroll
        for (int k = 0; k < 16; ++k) ut[k] = ov[(size_t)(a - a_ov) * 1024 + (size_t)(16 * h + k) * 32 + lane];
      }
    };
    for (it = 1; it <= A.max_iters + 1; ++it) {
      // k_pcg_tm's region of cont: cont_r [n_pad][8] (single: consumed by the owners before the grid
      // reduction), then per parity cont_w [6][n_pad] and gr [n_pad]
      float* cont_r = A.cont_tm;
      float* cont_w = A.cont_tm + (size_t)A.n_pad * (8 + (it & 1) * 7);
      float* gr_it = cont_w + (size_t)A.n_pad * 6;
      double* wc_it = A.wc + (size_t)(it & 1) * 2 * A.n_pad;
      // ---------------- N: w = Bh u.  The hand-overs U_a^T u_E depend on u_E only: they are formed
      // first and published together with u_E under ONE release flag, so the SpMV needs a single
      // point-to-point exchange (the tiles are read twice, from TMEM / shared memory).
      double wv = 0.0;
      TM_STAMP(0);
      if (own) {
        double vr[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) vr[i] = __shfl_sync(FULL, u, ra + i);
        const double vz[8] = {0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0};
#pragma unroll
        for (int a = 0; a < 3; ++a) {
          if (!up[a]) continue;
          double pu[4], pt[8] = {0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0};
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            double ut[16];
            load_half(a, h, ut);
            tile_half<false, true>(ut, h, vr, vz, pu, pt);
          }
          const double tc = tile_scatter_cols(pt, lane);
          if (act) A.T[((size_t)nbu[a] * 3 + a) * N + lane] = tc;
        }
        TM_WSTAMP(0);
        if (act) A.z[E * N + lane] = u;
        if (A.use_coarse == 2) scatter(r, cont_r, 8, 1);   // coarse-rhs contributions of r, to the neighbours
        __syncwarp();
        if (lane == 0) st_release_u32(flag + FS * E, (unsigned)it);
        if (waits) {
          while (ld_relaxed_gpu(flag + FS * my_nb) < (unsigned)it) {
#if TM_NS_P2P > 0
            __nanosleep(TM_NS_P2P);
#endif
          }
          ld_acquire_gpu(flag + FS * my_nb);
        }
        __syncwarp();
        TM_WSTAMP(1);
        double un[3], tl[3];
#pragma unroll
        for (int a = 0; a < 3; ++a) {
          un[a] = (up[a] && act) ? __ldcg(A.z + nbu[a] * N + lane) : 0.0;
          tl[a] = (lo[a] && act) ? __ldcg(A.T + ((size_t)E * 3 + a) * N + lane) : 0.0;
        }
        if (A.use_coarse == 2) {   // g(r)_E = -(sum of the neighbours' contributions), fixed order
          const float cr = lane < 6 ? __ldcg(cont_r + (size_t)E * 8 + lane) : 0.f;
          float gsum = 0.f;
#pragma unroll
          for (int sd = 0; sd < 6; ++sd) gsum += __shfl_sync(FULL, cr, sd);
          if (lane == 0) gr_it[E] = -gsum;
        }
        const double v0[4] = {0.0, 0.0, 0.0, 0.0};
        wv = u;
#pragma unroll
        for (int a = 0; a < 3; ++a) {
          if (!up[a]) continue;
          double vc[8];
#pragma unroll
          for (int j = 0; j < 8; ++j) vc[j] = __shfl_sync(FULL, un[a], cb + 4 * j);
          double pu[4] = {0.0, 0.0, 0.0, 0.0}, pt[8];
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            double ut[16];
            load_half(a, h, ut);
            tile_half<true, false>(ut, h, v0, vc, pu, pt);
          }
          wv += tile_scatter_rows(pu, lane);
        }
        wv += (tl[0] + tl[1]) + tl[2];
        if (!act) wv = 0.0;
        TM_WSTAMP(2);
      }
      // coarse right-hand-side contributions of w, side-major (double-buffered with gr: a CTA may
      // start the next iteration while another still gathers this one).  e(r) is formed afresh
      // every iteration (g(r) pre-summed by the owners above) and only e(s) is carried by recurrence:
      // the fp32 rounding of the coarse products stays relative to the current residual.
      if (A.use_coarse == 2) {
        scatter(wv, cont_w, 1, A.n_pad);
      } else if (A.use_coarse == 1 && own) {
        const double wcW = warp_sum(zh * wv), wcR = warp_sum(zh * r);
        if (lane == 0) {
          wc_it[E] = wcW;
          wc_it[A.n_pad + E] = wcR;
        }
      }
      if (A.tstamp && blockIdx.x == 0 && threadIdx.x == 0 && it < 64) A.tstamp[4 * it + 0] = gtimer();
      TM_STAMP(1);
      double delta;
      gamma = grid_reduce2(own ? warp_sum(r * u) : 0.0, own ? warp_sum(wv * u) : 0.0, red32, A.partials, A.gbar,
                           epoch, &bc[0], delta,
                           (A.tstamp && it < 32) ? A.tstamp + 4096 + 8 * ((size_t)it * gridDim.x + blockIdx.x) + 4 : nullptr);
      if (A.tstamp && blockIdx.x == 0 && threadIdx.x == 0 && it < 64) A.tstamp[4 * it + 1] = gtimer();
      TM_STAMP(2);
      if (A.tstamp && blockIdx.x == 0 && threadIdx.x == 0 && it < 64) {
        reinterpret_cast<double*>(A.tstamp)[1024 + 2 * it] = gamma;
        reinterpret_cast<double*>(A.tstamp)[1024 + 2 * it + 1] = delta;
      }
      nit = it - 1;
      if (gamma <= tol2 || !(gamma == gamma) || it > A.max_iters) break;
      const double beta = it == 1 ? 0.0 : gamma / gamma_old;
      const double den = it == 1 ? delta : delta - beta * gamma / alpha_old;
      if (!(den > 0.0)) {
        if (blockIdx.x == 0 && threadIdx.x == 0) atomicOr(A.flags, FLAG_BREAKDOWN);
        break;
      }
      const double alpha = gamma / den;
      double e_w = 0.0, e_rf = 0.0;
      if (A.use_coarse) {
        if (A.use_coarse == 2) stage_g6(cont_w, gr_it);
        else stage_wc(wc_it, 2);
        float fw, fr;
        coarse_gemv2(fw, fr);
        e_w = (double)fw;
        e_rf = (double)fr;
      }
      if (A.tstamp && blockIdx.x == 0 && threadIdx.x == 0 && it < 64) A.tstamp[4 * it + 2] = gtimer();
      TM_STAMP(3);
      p = fma(beta, p, u);
      sv = fma(beta, sv, wv);
      y = fma(alpha, p, y);
      r = fma(-alpha, sv, r);
      e_s = fma(beta, e_s, e_w);
      e_r = fma(-alpha, e_s, e_rf);
      u = act ? (A.use_coarse ? fma(zh, e_r, r) : r) : 0.0;
      gamma_old = gamma;
      alpha_old = alpha;
      if (A.tstamp && blockIdx.x == 0 && threadIdx.x == 0 && it < 64) A.tstamp[4 * it + 3] = gtimer();
    }
    it = nit;
    rr = gamma;
  } else {
    rr = 0.0;
  }
  TM_PROG(7);
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
