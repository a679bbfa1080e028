// lrbms_pcg.cuh -- a3: the reduced solve B c = r (eq:reducedSystem) on the GPU.
//
// 1. k_block_chol (warp per subdomain): B_EE = L_E L_E^T (in-register Cholesky), L_E^-1, and the
//    transformed coarse vector zh_E = L_E^T zc_E.
// 2. k_transform_h (two warps per coupling block): Bh_{E,E'} = L_E^-1 B_{E,E'} L_E'^-T, in place.
//    The block-Jacobi-scaled system  Bh y = L^-1 r,  c = L^-T y  has an IDENTITY diagonal block:
//    the SpMV reads only the coupling blocks and the block-Jacobi preconditioner costs nothing.
// 3. k_pcg (the L2-streaming variant, onchip = 0; the default is k_pcg_tm, lrbms_pcg_tm.cuh):
//    one cooperative persistent kernel per solve, warp per subdomain (lane k <-> coefficient
//    k, N <= 32).  Preconditioned CG (Hestenes-Stiefel) on Bh with the coarse correction
//    M^-1 = I + Zh B_c^-1 Zh^T (B_c = Zh^T Bh Zh = Z^T B Z, the Galerkin operator on the subdomain
//    indicators, inverted every few steps), warm-started from the (extrapolated) previous solution,
//    iterated to ||rh||_2 <= rtol ||L^-1 b||_2 (exact-solve reading A17).
//
// SpMV with the upper block storage reads every coupling block ONCE per iteration: the warp of E
// loads U = Bh_{E,E+a} row by row (coalesced), forms U v_{E+a} for itself by a warp reduce-scatter
// and U^T v_E for E+a, which it hands over through T[E+a][a]; the owner adds it after the grid
// barrier that follows the SpMV anyway (p.q is formed symmetrically, p.Bp = sum_E p_E.p_E +
// 2 p_E.U p_{E+a}, so it needs no completed q).  3 grid barriers per iteration:
//   A: p = z + beta p_old (neighbours recomputed locally), q_partial, T, p.q     -> sync
//   B: alpha, y += alpha p, r -= alpha q, ||r||^2, Zh^T r                       -> sync
//   C: z = r + Zh B_c^-1 Zh^T r, r.z                                            -> sync
// Reductions are per-CTA in warp order, then every warp sums the per-CTA partials in a fixed
// order: all warps obtain bitwise-identical scalars, so the termination test is grid-uniform and
// runs are deterministic.  The coarse inverse is stored in fp32 (it only steers the iteration);
// every product with Bh, every vector update and every reduction is fp64.
#pragma once
#include "lrbms_kernels.cuh"

namespace lrbms {

struct PcgArgs {
  Geo g;
  const double* blocks;   // [n_s][1+dim][N][N]: L_E in slot 0, transformed couplings in 1..dim
  const double* Linv;     // [n_s][N][N] L_E^-1 (row-major)
  const double* rhs;      // [n_s][N] b
  const double* zh;       // [n_s][N] L_E^T zc_E
  const float* Binv;      // [n_pad][n_pad] coarse inverse (fp32)
  double* x;              // solution c (original variables)
  double* hist_out;       // slot receiving this solve's solution (history ring buffer)
  const double* W;        // [KH][n_s][N] transformed history L^T c^{n-j}
  const double* V;        // [KH][n_s][N] Bh W
  const double* rb;       // [n_s][N] L^-1 b
  const double* gpart;    // [44][ngram] Gram / rhs partials from k_hist_gram
  const double* gsum;     // [44] their sums (k_hist_sum), read by k_pcg_tm
  int ngram;
  double* y;              // transformed unknown L^T c
  double* r;
  double* z;
  double* pb0;            // search direction, double buffered
  double* pb1;
  double* qp;             // partial q
  double* T;              // [n_s][3][N] transposed contributions from lower neighbours
  double* wc;             // [n_s] coarse residual Zh^T r
  double* partials;       // [4][gridDim]
  int* iters;
  int* flags;
  double rtol;
  int max_iters;
  int n_pad;
  int use_coarse;         // 0: block Jacobi only; 1: additive coarse level; 2: A-DEF2 deflation
  int binv_smem;          // 1: the CTA's rows of Binv are staged in shared memory once per solve
  int nh;                 // number of history vectors (0..KH)
  unsigned long long* tstamp;  // optional phase timestamps (CTA 0, first iterations), or nullptr
  unsigned* gbar;         // grid-barrier arrival counter (zeroed before the launch)
  const double* Yd;       // [n_s][6][N] deflation vectors Y_{E,F} = Bh_{E,F} zh_F (k_transform), mode 2
  float* cont;            // [n_pad][8] contributions Y_{E,F}.r_E to the coarse rhs of F, by side
  double* e0;             // [n_pad] coarse correction of the starting vector
  float* cont_tm;         // k_pcg_tm coarse-rhs contributions, side-major [6][n_pad]
  int cluster;            // k_pcg_tm: 1 = the grid is ONE thread-block cluster (hardware cluster barriers, DSMEM partials)
};

__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}

// prefetch a contiguous range into L1 (cooperatively by the warp; 128-byte lines)
__device__ __forceinline__ void prefetch_l1(const void* p, int bytes, int lane) {
  const char* c = reinterpret_cast<const char*>(p);
  for (int o = lane * 128; o < bytes; o += 32 * 128) asm volatile("prefetch.global.L1 [%0];" ::"l"(c + o));
}

// lane l gets sum over lanes of w[l] (w[k] held by every lane): 31 shuffles (recursive halving)
__device__ __forceinline__ double reduce_scatter32(double (&w)[32], int lane) {
#pragma unroll
  for (int i = 0; i < 16; ++i) {
    const bool hi = lane & 16;
    const double send = hi ? w[i] : w[i + 16];
    const double keep = hi ? w[i + 16] : w[i];
    w[i] = keep + __shfl_xor_sync(FULL, send, 16);
  }
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const bool hi = lane & 8;
    const double send = hi ? w[i] : w[i + 8];
    const double keep = hi ? w[i + 8] : w[i];
    w[i] = keep + __shfl_xor_sync(FULL, send, 8);
  }
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const bool hi = lane & 4;
    const double send = hi ? w[i] : w[i + 4];
    const double keep = hi ? w[i + 4] : w[i];
    w[i] = keep + __shfl_xor_sync(FULL, send, 4);
  }
#pragma unroll
  for (int i = 0; i < 2; ++i) {
    const bool hi = lane & 2;
    const double send = hi ? w[i] : w[i + 2];
    const double keep = hi ? w[i + 2] : w[i];
    w[i] = keep + __shfl_xor_sync(FULL, send, 2);
  }
  {
    const bool hi = lane & 1;
    const double send = hi ? w[0] : w[1];
    const double keep = hi ? w[1] : w[0];
    w[0] = keep + __shfl_xor_sync(FULL, send, 1);
  }
  return w[0];
}

// Inputs of the Galerkin initial guess (below): the history ring buffer and its transformed copies.
struct HistArgs {
  Geo g;
  const double* blocks;   // scaled couplings in slots 1..dim
  const double* Linv;
  const double* rhs;
  const double* hist;     // [KH][R] ring buffer
  double* W;              // [KH][R]
  double* V;              // [KH][R]
  double* TH;             // [KH][n_s][3][N]
  double* rb;             // [R]  L^-1 b
  double* gpart;          // [44][gridDim] Gram / rhs partials
  int nh;
  int hslot[8];
  unsigned* gbar_reset;   // the PCG's grid-barrier counter, zeroed by k_block_chol (saves a memset per solve)
};

// ============================================================================ factorisation + transform

// Warp per subdomain.  Lane j holds column j of the (padded-to-32 with identity) block.
#ifndef CHOL_MINB
#define CHOL_MINB 4
#endif
template <int NFIX>   // NFIX = 32: N known at compile time
__global__ void __launch_bounds__(128, CHOL_MINB) k_block_chol(Geo g, double* __restrict__ blocks, double* __restrict__ Linv,
                                                      const double* __restrict__ zc, double* __restrict__ zh,
                                                      int* flags, double* __restrict__ Es, const HistArgs H) {
  // Lt[k][i] = L[i][k] (column k of L, published at step k by the lanes that hold it), rows padded
  // to 34 doubles so that row starts stay 16-byte aligned (vector broadcast loads); rinv[k] = 1/L[k][k]
  __shared__ __align__(16) double Lt[4][32 * 34];
  __shared__ double rinv[4][32];
  __shared__ double dg[4][32];
  __shared__ __align__(16) double xs[4][32 * 8];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  if (H.gbar_reset && blockIdx.x == 0 && threadIdx.x < 8) H.gbar_reset[32 * threadIdx.x] = 0u;   // k_pcg_tm's counters
  const int E = blockIdx.x * (blockDim.x >> 5) + w;
  if (E >= g.n_s) return;
  const int N = NFIX ? NFIX : g.N;
  double* Bd = blocks + (size_t)E * (1 + g.dim) * N * N;
  double m[32];
#pragma unroll
  for (int i = 0; i < 32; ++i) m[i] = (lane < N && i < N) ? Bd[i * N + lane] : (i == lane ? 1.0 : 0.0);
  bool bad = false;
  dg[w][lane] = lane < N ? Bd[lane * N + lane] : 1.0;   // original diagonal entries
  double* lt = Lt[w];
  // Right-looking Cholesky on the full symmetric trailing matrix: lane j's m[k] = M[k][j] = M[j][k],
  // so at step k lane j >= k holds L[j][k] L[k][k] and publishes L[j][k] to row k of Lt; the rank-1
  // update then reads column k back with broadcast loads, scaled by L[lane][k] on the trailing lanes
  // and by 0 on the finished ones (no per-entry selects).  Lanes < k publish values nobody reads.
  // A pivot below 1e-13 of its original diagonal entry means a numerically rank-deficient Phi_E.
#pragma unroll
  for (int k = 0; k < 32; ++k) {
    const double dkk = __shfl_sync(FULL, m[k], k);
    bad |= !(dkk > 1e-13 * dg[w][k]);
    const double rd = rsqrt(dkk);
    const double ljk = m[k] * rd;          // L[lane][k] for lane >= k
    lt[k * 34 + lane] = ljk;
    if (lane == 0) rinv[w][k] = rd;
    __syncwarp();
    const double lm = lane > k ? ljk : 0.0;
#pragma unroll
    for (int i = 0; i < 32; ++i)
      if (i > k) m[i] = fma(-lt[k * 34 + i], lm, m[i]);
  }
  if (bad && lane == 0) atomicOr(flags, FLAG_PIVOT);
  __syncwarp();
  // column lane of L: L[i][lane] = Lt[lane][i] for i >= lane
  const double zk = lane < N ? zc[E * N + lane] : 0.0;
  dg[w][lane] = zk;
  __syncwarp();
  double zhat = 0.0;   // (L^T zc)[lane] = sum_i L[i][lane] zc[i]
#pragma unroll
  for (int i = 0; i < 32; ++i) {
    m[i] = i >= lane ? lt[lane * 34 + i] : 0.0;
    zhat = fma(m[i], dg[w][i], zhat);
  }
  // L^-1 by column-oriented forward substitution, one column per lane: L x = e_lane; column k of L
  // is row k of Lt (vector broadcast loads)
  double x[32];
#pragma unroll
  for (int i = 0; i < 32; ++i) x[i] = i == lane ? 1.0 : 0.0;
#pragma unroll
  for (int k = 0; k < 32; ++k) {
    x[k] *= rinv[w][k];
#pragma unroll
    for (int i = 0; i < 32; ++i)
      if (i > k) x[i] = fma(-lt[k * 34 + i], x[k], x[i]);
  }
  if (lane < N) {
    double* Li = Linv + (size_t)E * N * N;
#pragma unroll
    for (int i = 0; i < 32; ++i)
      if (i < N) Li[i * N + lane] = x[i];
    zh[E * N + lane] = zhat;
  }
  // the initial guess's inputs (fused: L and L^-1 are at hand here)
  //   rb = L^-1 b: row lane of L^-1 from shared memory (x[] holds column lane), b broadcast;
  //   W_j = L^T c^{n-j}, j < nh: W_j[lane] = sum_i L[i][lane] c_j[i], c_j[i] broadcast as xs[i][j].
  const size_t R = (size_t)g.n_s * N;
  const bool act = lane < N;
  __syncwarp();   // every lane is done reading Lt
#pragma unroll
  for (int i = 0; i < 32; ++i) lt[i * 34 + lane] = x[i];
  dg[w][lane] = act ? H.rhs[E * N + lane] : 0.0;
#pragma unroll
  for (int j = 0; j < 8; ++j)
    xs[w][lane * 8 + j] = (j < H.nh && act) ? H.hist[(size_t)H.hslot[j] * R + E * N + lane] : 0.0;
  __syncwarp();
  double rbk = 0.0;
#pragma unroll
  for (int k = 0; k < 32; ++k) rbk = fma(lt[lane * 34 + k], dg[w][k], rbk);
  if (act) H.rb[E * N + lane] = rbk;
  if (H.nh > 0) {
    double wk[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) wk[j] = 0.0;
#pragma unroll
    for (int i = 0; i < 32; ++i)
#pragma unroll
      for (int j = 0; j < 8; ++j) wk[j] = fma(m[i], xs[w][i * 8 + j], wk[j]);
#pragma unroll
    for (int j = 0; j < 8; ++j)
      if (j < H.nh && act) H.W[j * R + E * N + lane] = wk[j];
  }
  if (Es) {   // coarse operator diagonal zc^T B_EE zc = |L^T zc|^2; the side slots are set by k_transform
    const double d = warp_sum(lane < N ? zhat * zhat : 0.0);
    if (lane < 8) Es[(size_t)E * 8 + lane] = lane == 0 ? d : 0.0;
  }
}

__device__ __forceinline__ void dmma_t(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}

// Bh_{E,E+a} = X_E U X_{E+a}^T (X = L^-1) in place, TWO warps per coupling block, each owning 16
// rows of Bh (both 32x32x32 products on DMMA with operand fragments read from L2, the intermediate
// T1 = X_E U re-laid out from the accumulator layout into A fragments by quad shuffles): rows of
// Bh = (X_E U) X_N^T depend only on the same rows of X_E U, so the halves are independent
// (128 registers, 16 warps per SM).  Y_{E,E+a} = Bh zh_{E+a}, Y_{E+a,E} = Bh^T zh_E and the coarse
// coupling zh_E . Y from the accumulator layout.  The column sums of
// Y_{E+a,E} and the coarse coupling combine the two halves through shared memory in a fixed order.
// CTA = 4 blocks x 2 halves.
#ifndef TRANSFORM_MINB
#define TRANSFORM_MINB 2
#endif
template <int NFIX>   // NFIX = 32: N known at compile time (no bounds predicates, constant strides)
__global__ void __launch_bounds__(256, TRANSFORM_MINB) k_transform_h(Geo g, double* __restrict__ blocks,
                                                    const double* __restrict__ Linv,
                                                    const double* __restrict__ zh, double* __restrict__ Yd,
                                                    double* __restrict__ Es) {
  __shared__ double colp[4][2][32];
  __shared__ double ecp[4][2];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int slot = warp >> 1, half = warp & 1;
  const int t = blockIdx.x * 4 + slot;
  bool live = t < g.n_s * g.dim;
  int E = 0, a = 0, En = 0;
  if (live) {
    E = t / g.dim;
    a = t - E * g.dim;
    int C[3];
    sub_xyz(g, E, C);
    live = C[a] + 1 < g.S[a];
    En = live ? E + g.Estride[a] : E;
  }
  const int N = NFIX ? NFIX : g.N, NN = N * N;
  const int fr = lane >> 2, q = lane & 3;
  double bh[2][4][2];
  if (live) {
    double* U = blocks + ((size_t)E * (1 + g.dim) + 1 + a) * NN;
    const double* XE = Linv + (size_t)E * NN;
    const double* XN = Linv + (size_t)En * NN;
    auto ld = [&](const double* M, int r, int c) -> double {
      return NFIX ? M[r * N + c] : ((r < N && c < N) ? M[r * N + c] : 0.0);
    };
    double t1[2][4][2];
#pragma unroll
    for (int ti = 0; ti < 2; ++ti)
#pragma unroll
      for (int tj = 0; tj < 4; ++tj) t1[ti][tj][0] = t1[ti][tj][1] = bh[ti][tj][0] = bh[ti][tj][1] = 0.0;
#pragma unroll
    for (int ks = 0; ks < 8; ++ks) {
      double af[2], bf[4];
#pragma unroll
      for (int ti = 0; ti < 2; ++ti) af[ti] = ld(XE, 16 * half + 8 * ti + fr, 4 * ks + q);
#pragma unroll
      for (int tj = 0; tj < 4; ++tj) bf[tj] = ld(U, 4 * ks + q, 8 * tj + fr);
#pragma unroll
      for (int ti = 0; ti < 2; ++ti)
#pragma unroll
        for (int tj = 0; tj < 4; ++tj) dmma_t(t1[ti][tj][0], t1[ti][tj][1], af[ti], bf[tj]);
    }
    const int src_lo = (lane & ~3) + (q >> 1), src_hi = (lane & ~3) + 2 + (q >> 1);
#pragma unroll
    for (int ks = 0; ks < 8; ++ks) {
      const int src = (ks & 1) ? src_hi : src_lo;
      double af[2], bf[4];
#pragma unroll
      for (int ti = 0; ti < 2; ++ti) {
        const double v0 = __shfl_sync(FULL, t1[ti][ks >> 1][0], src);
        const double v1 = __shfl_sync(FULL, t1[ti][ks >> 1][1], src);
        af[ti] = (q & 1) ? v1 : v0;
      }
#pragma unroll
      for (int tj = 0; tj < 4; ++tj) bf[tj] = ld(XN, 8 * tj + fr, 4 * ks + q);
#pragma unroll
      for (int ti = 0; ti < 2; ++ti)
#pragma unroll
        for (int tj = 0; tj < 4; ++tj) dmma_t(bh[ti][tj][0], bh[ti][tj][1], af[ti], bf[tj]);
    }
#pragma unroll
    for (int ti = 0; ti < 2; ++ti)
#pragma unroll
      for (int tj = 0; tj < 4; ++tj) {
        const int i = 16 * half + 8 * ti + fr, j = 8 * tj + 2 * q;
        if (i < N) {
          if (j < N) U[i * N + j] = bh[ti][tj][0];
          if (j + 1 < N) U[i * N + j + 1] = bh[ti][tj][1];
        }
      }
  }
  if (!Es && !Yd) return;   // uniform over the grid
  double o = 0.0;
  if (live) {
    const double* zN = zh + (size_t)En * N;
    const double* zE = zh + (size_t)E * N;
    // Y_{E,E+a}[i] for this half's rows (quad reduction), and its part of zh_E . Y
#pragma unroll
    for (int ti = 0; ti < 2; ++ti) {
      double v = 0.0;
#pragma unroll
      for (int tj = 0; tj < 4; ++tj) {
        const int j = 8 * tj + 2 * q;
        v = fma(bh[ti][tj][0], j < N ? zN[j] : 0.0, v);
        v = fma(bh[ti][tj][1], j + 1 < N ? zN[j + 1] : 0.0, v);
      }
      v += __shfl_xor_sync(FULL, v, 1);
      v += __shfl_xor_sync(FULL, v, 2);
      const int i = 16 * half + 8 * ti + fr;
      if (q == 0 && i < N) {
        if (Yd) Yd[((size_t)E * 6 + a) * N + i] = v;
        o = fma(v, zE[i], o);
      }
    }
    // this half's part of the column sums sum_i Bh[i][j] zh_E[i]
#pragma unroll
    for (int tj = 0; tj < 4; ++tj) {
      double v0 = 0.0, v1 = 0.0;
#pragma unroll
      for (int ti = 0; ti < 2; ++ti) {
        const int i = 16 * half + 8 * ti + fr;
        const double z = i < N ? zE[i] : 0.0;
        v0 = fma(bh[ti][tj][0], z, v0);
        v1 = fma(bh[ti][tj][1], z, v1);
      }
#pragma unroll
      for (int off = 4; off < 32; off <<= 1) {
        v0 += __shfl_xor_sync(FULL, v0, off);
        v1 += __shfl_xor_sync(FULL, v1, off);
      }
      if (fr == 0) {
        colp[slot][half][8 * tj + 2 * q] = v0;
        colp[slot][half][8 * tj + 2 * q + 1] = v1;
      }
    }
    o = warp_sum(o);
    if (lane == 0) ecp[slot][half] = o;
  }
  __syncthreads();
  if (live && half == 0) {
    if (Yd && lane < N) Yd[((size_t)En * 6 + 3 + a) * N + lane] = colp[slot][0][lane] + colp[slot][1][lane];
    if (Es && lane == 0) {
      const double e = ecp[slot][0] + ecp[slot][1];
      Es[(size_t)E * 8 + 1 + a] = e;
      Es[(size_t)En * 8 + 4 + a] = e;
    }
  }
}

// ============================================================================ PCG on the scaled system

// Part A of q = Bh v for subdomain E: returns lane's (v_E + sum_a U_a v_{E+a}); stores U_a^T v_E
// into T[E+a][a]; adds v_E.v_E + 2 v_E.(U_a v_{E+a}) (lane-local) to vbv.
//
// Register tiling of a 32 x 32 block: lane l = 4 a + b holds U[4a + i][b + 4j] (i < 4, j < 8): its
// four rows R(a) = {4a..4a+3} and eight columns C(b) = {b, b+4, .., b+28}.  U v is then a 4-lane
// reduce-scatter (rows) and U^T v an 8-lane one (columns), and both land on lane l = coefficient l:
// 10 fp64 shuffles per block instead of 63 for the row-per-load layout.  Every load instruction
// reads 8 rows x 32 contiguous bytes (full sectors).  sv is the warp's 2 x 32-double staging slot.
template <class VF>
__device__ __forceinline__ double spmv_part(const PcgArgs& A, int E, const int C[3], int lane, double vE,
                                            VF vload, double& vbv, double* sv) {
  const Geo& g = A.g;
  const int N = g.N, nb1 = 1 + g.dim;
  const double* Bd = A.blocks + (size_t)E * nb1 * N * N;
  const bool act = lane < N;
  const int ra = (lane >> 2) * 4, cb = lane & 3;
  double acc = vE;
  double local = vE * vE;
  sv[lane] = vE;
  __syncwarp();
  double vr[4];
#pragma unroll
  for (int i = 0; i < 4; ++i) vr[i] = sv[ra + i];
  for (int a = 0; a < g.dim; ++a) {
    if (C[a] + 1 >= g.S[a]) continue;
    const int En = E + g.Estride[a];
    const double vN = vload(En);
    const double* U = Bd + (size_t)(1 + a) * N * N;
    double u[4][8];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const int r = ra + i, c = cb + 4 * j;
        u[i][j] = (r < N && c < N) ? __ldg(U + r * N + c) : 0.0;
      }
    __syncwarp();
    sv[32 + lane] = vN;
    __syncwarp();
    double pu[4], pt[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) pt[j] = 0.0;
#pragma unroll
    for (int i = 0; i < 4; ++i) pu[i] = 0.0;
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const double vc = sv[32 + cb + 4 * j];
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        pu[i] = fma(u[i][j], vc, pu[i]);
        pt[j] = fma(u[i][j], vr[i], pt[j]);
      }
    }
    // rows: reduce-scatter over lane bits 1, 0 -> lane keeps row ra + cb = lane
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
    // columns: reduce-scatter over lane bits 4, 3, 2 -> lane keeps column cb + 4 (lane >> 2) = lane
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
    const double tU = pu[0];   // (U v_{E+a})[lane]
    acc += tU;
    local += 2.0 * vE * tU;
    if (act) A.T[((size_t)En * 3 + a) * N + lane] = pt[0];
  }
  __syncwarp();
  vbv += local;
  return acc;
}

__device__ __forceinline__ double lower_contrib(const PcgArgs& A, int E, const int C[3], int lane) {
  const Geo& g = A.g;
  double t = 0.0;
  if (lane < g.N)
    for (int a = 0; a < g.dim; ++a)
      if (C[a] > 0) t += A.T[((size_t)E * 3 + a) * g.N + lane];
  return t;
}

// e_E = (B_c^-1 g)_E for the staged coarse vector g (fp32: the coarse level only steers the
// iteration); warp-uniform result.
__device__ __forceinline__ float coarse_e(const PcgArgs& A, const float* wcv, const float* brow, int lane) {
  const float4* row = reinterpret_cast<const float4*>(brow);
  const float4* w4 = reinterpret_cast<const float4*>(wcv);
  const int n4 = A.n_pad >> 2;
  float e0 = 0.f, e1 = 0.f;
#pragma unroll 4
  for (int F = lane; F < n4; F += 32) {
    const float4 b0 = row[F], c0 = w4[F];
    e0 = fmaf(b0.x, c0.x, e0);
    e1 = fmaf(b0.y, c0.y, e1);
    e0 = fmaf(b0.z, c0.z, e0);
    e1 = fmaf(b0.w, c0.w, e1);
  }
  float e = e0 + e1;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) e += __shfl_xor_sync(FULL, e, o);
  return e;
}

// Two-level preconditioners on the scaled system (block-Jacobi part = I, Q = Zh B_c^-1 Zh^T):
//  mode 1, additive:  z = r + Q r                    (coarse rhs g = Zh^T r)
//  mode 2, A-DEF2:    z = P^T r + Q r,  P = I - Bh Q  (coarse rhs g = Zh^T (I - Bh) r)
// A-DEF2 needs a current B_c^-1 (kept current by a Newton-Schulz step per time step); its coarse
// rhs only involves the couplings (Bh_EE = I): g_F = -sum_{E nb F} Y_{E,F} . r_E (defl_scatter).
// In both, z_E = r_E + zh_E (B_c^-1 g)_E.
__device__ __forceinline__ double precond(const PcgArgs& A, const float* wcv, const float* brow, int E, int lane, double rk) {
  const int N = A.g.N;
  const float e = A.use_coarse ? coarse_e(A, wcv, brow, lane) : 0.f;
  return lane < N ? rk + A.zh[E * N + lane] * (double)e : 0.0;
}

// contributions Y_{E,F} . r_E of subdomain E to the coarse rhs of its neighbours F: cont[F][s]
// (slot s = the side of E that faces F: no slot has two writers).  One 8-value reduce-scatter
// (9 shuffles) instead of six warp sums.
__device__ __forceinline__ void defl_scatter(const PcgArgs& A, int E, const int C[3], int lane, double rk) {
  const Geo& g = A.g;
  const int N = g.N;
  double d[8];
#pragma unroll
  for (int s = 0; s < 6; ++s) d[s] = (lane < N && side_exists(g, C, s)) ? A.Yd[((size_t)E * 6 + s) * N + lane] * rk : 0.0;
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
  const int s = lane >> 2;   // lane holds the total of value index s (lane bits 4, 3, 2)
  if ((lane & 3) == 0 && s < 6 && side_exists(g, C, s)) A.cont[(size_t)side_nb(g, E, s) * 8 + s] = (float)d[0];
}

// per-CTA partial of a grid reduction: warps in order (deterministic).  red[slot][32] is only
// reused after the grid barrier that follows every call, so one CTA barrier suffices.
__device__ __forceinline__ void cta_partial(double v, double (*red)[32], double* partials, int slot) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, W = blockDim.x >> 5;
  if (lane == 0) red[slot][warp] = v;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int w = 0; w < W; ++w) t += red[slot][w];
    partials[slot * gridDim.x + blockIdx.x] = t;
  }
}
// like cta_partial, for the 44 Gram-matrix slots (own shared buffer, one barrier per slot)
__device__ __forceinline__ void cta_partial_n(double v, double (*red)[32], double* partials, int slot) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, W = blockDim.x >> 5;
  if (lane == 0) red[slot - 4][warp] = v;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int w = 0; w < W; ++w) t += red[slot - 4][w];
    partials[slot * gridDim.x + blockIdx.x] = t;
  }
}
// fixed-order total of the per-CTA partials, read by warp 0 only and broadcast through shared memory:
// 2048 warps hammering the same few L2 lines right after a grid barrier serialise at one L2 slice.
// bc is a per-call-site shared slot; every call site is followed by another CTA barrier before the
// same slot is written again.
__device__ __forceinline__ double grid_total_b(const double* partials, int slot, double* bc) {
  if ((threadIdx.x >> 5) == 0) {
    const int lane = threadIdx.x & 31, G = gridDim.x;
    double s = 0.0;
    for (int b = lane; b < G; b += 32) s += partials[slot * G + b];
    s = warp_sum(s);
    if (lane == 0) *bc = s;
  }
  __syncthreads();
  return *bc;
}

__device__ __forceinline__ unsigned ld_acquire_gpu(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
// Deterministic grid-wide sum fused with the grid barrier: per-CTA partial (warps in order) ->
// arrival on a monotone counter -> warp 0 sums the per-CTA partials in a fixed order -> shared
// broadcast.  Two CTA barriers per call instead of the four of cta_partial + grid.sync +
// grid_total_b.  Partials rotate over 4 slots (a slot is rewritten only 4 barriers later, after
// every CTA has read it); red16/bc are rewritten only after the first CTA barrier of the next call.
__device__ __forceinline__ double grid_reduce(double v, double* red16, double* partials, unsigned* bar,
                                              unsigned& epoch, double* bc) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, W = blockDim.x >> 5, G = gridDim.x;
  if (lane == 0) red16[warp] = v;
  __syncthreads();
  ++epoch;
  double* ps = partials + (size_t)(epoch & 3) * G;
  if (warp == 0) {
    if (lane == 0) {
      double t = 0.0;
      for (int w = 0; w < W; ++w) t += red16[w];
      ps[blockIdx.x] = t;
      __threadfence();
      atomicAdd(bar, 1u);
      const unsigned target = epoch * (unsigned)G;
      while (ld_acquire_gpu(bar) < target) {
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

__device__ __forceinline__ double grid_total(const double* partials, int slot) {
  const int lane = threadIdx.x & 31, G = gridDim.x;
  double s = 0.0;
  for (int b = lane; b < G; b += 32) s += partials[slot * G + b];
  return warp_sum(s);
}

// ============================================================================ initial guess (history)
// Galerkin projection of the new solution onto the span of the last nh solutions, in the scaled
// variables W_j = L^T c^{n-j}: minimise ||y - y*||_Bh over y0 = W alpha, (W^T Bh W) alpha = W^T rb.
// Three small kernels (W and rb; V = Bh W with one read of every coupling block; Gram partials)
// precede k_pcg, which solves the nh x nh system redundantly in every thread.


// complete V (lower hand-overs), Gram partials G_ij = W_i.V_j (i <= j) and g_i = W_i.rb per CTA
__global__ void __launch_bounds__(256) k_hist_gram(HistArgs A) {
  __shared__ double red[44][8];
  const Geo& g = A.g;
  const int N = g.N, lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int E = blockIdx.x * 8 + warp;
  const bool act = lane < N;
  const size_t R = (size_t)g.n_s * N;
  double gp[44];
#pragma unroll
  for (int q = 0; q < 44; ++q) gp[q] = 0.0;
  if (E < g.n_s) {
    int C[3];
    sub_xyz(g, E, C);
    double wv[8], vv[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      wv[j] = 0.0; vv[j] = 0.0;
      if (j < A.nh && act) {
        wv[j] = A.W[j * R + E * N + lane];
        double v = A.V[j * R + E * N + lane];
        for (int a = 0; a < g.dim; ++a)
          if (C[a] > 0) v += A.TH[((size_t)j * g.n_s * 3 + (size_t)E * 3 + a) * N + lane];
        vv[j] = v;
        A.V[j * R + E * N + lane] = v;
      }
    }
    const double rbk = act ? A.rb[E * N + lane] : 0.0;
    int q = 0;
#pragma unroll
    for (int i = 0; i < 8; ++i)
#pragma unroll
      for (int j = i; j < 8; ++j) {
        if (j < A.nh) gp[q] = warp_sum(wv[i] * vv[j]);
        ++q;
      }
#pragma unroll
    for (int i = 0; i < 8; ++i)
      if (i < A.nh) gp[36 + i] = warp_sum(wv[i] * rbk);
  }
  if (lane == 0) {
#pragma unroll
    for (int q = 0; q < 44; ++q) red[q][warp] = gp[q];
  }
  __syncthreads();
  if (threadIdx.x < 44) {
    double t = 0.0;
    for (int w = 0; w < 8; ++w) t += red[threadIdx.x][w];
    A.gpart[threadIdx.x * gridDim.x + blockIdx.x] = t;
  }
}

// the 44 fixed-order sums of the k_hist_gram partials, one warp per sum (for k_pcg_tm's setup)
__global__ void k_hist_sum(const double* __restrict__ gpart, int ngram, double* __restrict__ gsum) {
  const int q = blockIdx.x, lane = threadIdx.x;
  double v = 0.0;
  for (int b = lane; b < ngram; b += 32) v += gpart[(size_t)q * ngram + b];
  v = warp_sum(v);
  if (lane == 0) gsum[q] = v;
}

// Solve of one PCG run's setup (out of line: its register pressure stays out of the iteration
// loop): alpha from the Gram partials, y0 = W alpha, r0 = rb - V alpha, ||rb||^2, ||r0||^2, Zh^T r0.
__device__ __noinline__ void pcg_initial_guess(const PcgArgs& A, cg::grid_group& grid, double (*red)[32],
                                               double* sh, double& bb_out, double& rr_out) {
  const Geo& g = A.g;
  const int N = g.N;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, W = blockDim.x >> 5;
  const int TW = gridDim.x * W, gw = blockIdx.x * W + warp;
  const bool act = lane < N;
  const int nh = A.nh;
  const size_t R = (size_t)g.n_s * N;
  double alpha_h[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) alpha_h[j] = 0.0;
  if (nh > 0) {
    // fixed-order sums of the k_hist_gram partials by warp 0, broadcast through shared memory
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
  double pbb = 0.0, prr = 0.0;
  for (int E = gw; E < g.n_s; E += TW) {
    const double rbk = act ? A.rb[E * N + lane] : 0.0;
    double yk = 0.0, rk = rbk;
#pragma unroll
    for (int j = 0; j < 8; ++j)
      if (j < nh && act) {
        yk += alpha_h[j] * A.W[j * R + E * N + lane];
        rk -= alpha_h[j] * A.V[j * R + E * N + lane];
      }
    if (act) {
      A.y[E * N + lane] = yk;
      A.r[E * N + lane] = rk;
    }
    pbb += warp_sum(rbk * rbk);
    prr += warp_sum(rk * rk);
    const double w = warp_sum(act ? A.zh[E * N + lane] * rk : 0.0);
    if (lane == 0) A.wc[E] = w;
  }
  cta_partial(pbb, red, A.partials, 0);
  cta_partial(prr, red, A.partials, 1);
  grid.sync();
  bb_out = grid_total_b(A.partials, 0, &sh[44]);
  rr_out = grid_total_b(A.partials, 1, &sh[45]);
}

__global__ void __launch_bounds__(512, 1) k_pcg(PcgArgs A) {
  cg::grid_group grid = cg::this_grid();
  __shared__ double red[4][32];
  __shared__ double bc[4];
  __shared__ double sh46[46];
  __shared__ double vsm[16][64];   // per-warp SpMV staging (<= 16 warps)
  extern __shared__ float wcs[];
  const Geo& g = A.g;
  const int N = g.N;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int TW = gridDim.x * (blockDim.x >> 5), gw = blockIdx.x * (blockDim.x >> 5) + warp;
  const bool act = lane < N;
  const float* wcv = wcs;
  // rows of B_c^-1 of this CTA's subdomains (E = gw + j TW -> smem row j W + warp), staged once per
  // solve: the coarse product of every iteration then reads shared memory instead of 16.8 MB of L2
  float* bsm = wcs + A.n_pad;
  const int WPC = blockDim.x >> 5;
  if (A.use_coarse && A.binv_smem) {
    const int nrow = WPC * ((g.n_s + TW - 1) / TW);
    const int n4 = A.n_pad >> 2;
    for (int t = threadIdx.x; t < nrow * n4; t += blockDim.x) {
      const int rr = t / n4, F = t - rr * n4;
      const int E = blockIdx.x * WPC + (rr % WPC) + (rr / WPC) * TW;
      float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
      if (E < g.n_s) v = __ldcs(reinterpret_cast<const float4*>(A.Binv + (size_t)E * A.n_pad) + F);
      reinterpret_cast<float4*>(bsm)[t] = v;
    }
  }
  auto brow = [&](int E) -> const float* {
    return A.binv_smem ? bsm + (size_t)(((E - gw) / TW) * WPC + warp) * A.n_pad : A.Binv + (size_t)E * A.n_pad;
  };
  auto stage_wc = [&]() {   // Zh^T r -> shared memory (fp32, zero padded to n_pad)
    for (int i = threadIdx.x; i < A.n_pad; i += blockDim.x) wcs[i] = i < g.n_s ? (float)__ldcg(A.wc + i) : 0.f;
    __syncthreads();
  };
  auto stage_g = [&]() {    // Zh^T (I - Bh) r = -(sum of the six neighbour contributions), fixed order
    for (int i = threadIdx.x; i < A.n_pad; i += blockDim.x) {
      float v = 0.f;
      if (i < g.n_s) {
        const float4 u0 = __ldcg(reinterpret_cast<const float4*>(A.cont + (size_t)i * 8));
        const float4 u1 = __ldcg(reinterpret_cast<const float4*>(A.cont + (size_t)i * 8 + 4));
        v = -(((((u0.x + u0.y) + u0.z) + u0.w) + u1.x) + u1.y);
      }
      wcs[i] = v;
    }
    __syncthreads();
  };
  auto stage_coarse = [&]() {
    if (A.use_coarse == 1) stage_wc();
    else if (A.use_coarse == 2) stage_g();
  };

  double bb, rr;
  pcg_initial_guess(A, grid, red, sh46, bb, rr);
  __shared__ double red16[16];
  unsigned epoch = 0;
  double* gparts = A.partials + 8 * (size_t)gridDim.x;   // slots 8..11 (the setup uses 0..1)
  // stopping test on the preconditioned residual r.M^-1 r (an energy-norm error proxy that weights
  // the smooth, coarse-level residual components), relative to ||L^-1 b||^2 <= b.M^-1 b
  const double tol2 = A.rtol * A.rtol * bb;
  int it = 0;
  if (!(rr <= 0.0) && bb > 0.0) {
    double prz = 0.0;
    if (A.use_coarse == 2) {
      // DEF starting vector y0 = y + Zh e0, e0 = B_c^-1 Zh^T r, so that Zh^T r0 = 0 (up to the fp32
      // coarse inverse): r0 = r - Bh Zh e0 = r - zh_E e0_E - sum_F Y_{E,F} e0_F
      stage_wc();
      for (int E = gw; E < g.n_s; E += TW) {
        const float e = coarse_e(A, wcv, brow(E), lane);
        if (lane == 0) A.e0[E] = (double)e;
        if (act) A.y[E * N + lane] += A.zh[E * N + lane] * (double)e;
      }
      grid_reduce(0.0, red16, gparts, A.gbar, epoch, &bc[0]);
      for (int E = gw; E < g.n_s; E += TW) {
        int C[3];
        sub_xyz(g, E, C);
        double rk = 0.0;
        if (act) {
          rk = A.r[E * N + lane] - A.zh[E * N + lane] * __ldcg(A.e0 + E);
#pragma unroll
          for (int s = 0; s < 6; ++s)
            if (side_exists(g, C, s)) rk -= A.Yd[((size_t)E * 6 + s) * N + lane] * __ldcg(A.e0 + side_nb(g, E, s));
          A.r[E * N + lane] = rk;
        }
        defl_scatter(A, E, C, lane, rk);
      }
      grid_reduce(0.0, red16, gparts, A.gbar, epoch, &bc[0]);
    }
    stage_coarse();
    for (int E = gw; E < g.n_s; E += TW) {
      const double rk = act ? A.r[E * N + lane] : 0.0;
      const double zk = precond(A, wcv, brow(E), E, lane, rk);
      if (act) A.z[E * N + lane] = zk;
      prz += warp_sum(zk * rk);
    }
    double rz = grid_reduce(prz, red16, gparts, A.gbar, epoch, &bc[0]);
    double beta = 0.0;
    for (it = (rz <= tol2) ? A.max_iters + 2 : 1; it <= A.max_iters; ++it) {
      double* pcur = (it & 1) ? A.pb1 : A.pb0;
      const double* pold = (it & 1) ? A.pb0 : A.pb1;
      const bool first = it == 1;
      // A: p = z + beta p_old; q_partial = (I + U) p; T; p.Bh p
      double ppq = 0.0;
      for (int E = gw; E < g.n_s; E += TW) {
        int C[3];
        sub_xyz(g, E, C);
        auto pload = [&](int Ep) {
          if (!act) return 0.0;
          const double zz = A.z[Ep * N + lane];
          return first ? zz : zz + beta * pold[Ep * N + lane];
        };
        const double pE = pload(E);
        if (act) pcur[E * N + lane] = pE;
        double vbv = 0.0;
        const double q = spmv_part(A, E, C, lane, pE, pload, vbv, &vsm[warp][0]);
        if (act) A.qp[E * N + lane] = q;
        ppq += warp_sum(vbv);
      }
      LRBMS_TSTAMP(A.tstamp && blockIdx.x == 0 && threadIdx.x == 0 && it < 64, A.tstamp[4 * it + 0], gtimer());
      const double pq = grid_reduce(ppq, red16, gparts, A.gbar, epoch, &bc[0]);
      LRBMS_TSTAMP(A.tstamp && blockIdx.x == 0 && threadIdx.x == 0 && it < 64, A.tstamp[4 * it + 1], gtimer());
      if (!(pq > 0.0)) {
        if (blockIdx.x == 0 && threadIdx.x == 0) atomicOr(A.flags, FLAG_BREAKDOWN);
        break;
      }
      const double alpha = rz / pq;
      // B: y, r, ||r||^2, Zh^T r
      double prr = 0.0;
      for (int E = gw; E < g.n_s; E += TW) {
        int C[3];
        sub_xyz(g, E, C);
        double rk = 0.0;
        if (act) {
          const double q = A.qp[E * N + lane] + lower_contrib(A, E, C, lane);
          A.y[E * N + lane] += alpha * pcur[E * N + lane];
          rk = A.r[E * N + lane] - alpha * q;
          A.r[E * N + lane] = rk;
        }
        prr += warp_sum(rk * rk);
        if (A.use_coarse == 1) {
          const double w = warp_sum(act ? A.zh[E * N + lane] * rk : 0.0);
          if (lane == 0) A.wc[E] = w;
        } else if (A.use_coarse == 2) {
          defl_scatter(A, E, C, lane, rk);
        }
      }
      rr = grid_reduce(prr, red16, gparts, A.gbar, epoch, &bc[0]);
      LRBMS_TSTAMP(A.tstamp && blockIdx.x == 0 && threadIdx.x == 0 && it < 64, A.tstamp[4 * it + 2], gtimer());
      if (!(rr > 0.0)) break;   // exact solution (or NaN, flagged below)
      // C: z = M^-1 r, r.z
      double prz2 = 0.0;
      if (A.use_coarse && !A.binv_smem)
        for (int E = gw; E < g.n_s; E += TW) prefetch_l1(A.Binv + (size_t)E * A.n_pad, A.n_pad * 4, lane);
      stage_coarse();
      for (int E = gw; E < g.n_s; E += TW) {
        const double rk = act ? A.r[E * N + lane] : 0.0;
        const double zk = precond(A, wcv, brow(E), E, lane, rk);
        if (act) A.z[E * N + lane] = zk;
        prz2 += warp_sum(zk * rk);
      }
      const double rz_new = grid_reduce(prz2, red16, gparts, A.gbar, epoch, &bc[0]);
      LRBMS_TSTAMP(A.tstamp && blockIdx.x == 0 && threadIdx.x == 0 && it < 64, A.tstamp[4 * it + 3], gtimer());
      if (rz_new <= tol2) break;
      beta = rz_new / rz;
      rz = rz_new;
    }
    if (it == A.max_iters + 2) it = 0;   // converged at the initial guess
  }
  // ---- back-transform c = L^-T y (per subdomain; no barrier needed)
  for (int E = gw; E < g.n_s; E += TW) {
    const double yk = act ? A.y[E * N + lane] : 0.0;
    const double* Li = A.Linv + (size_t)E * N * N;
    double xk = 0.0;   // sum_i Linv[i][lane] y[i]
    for (int i = 0; i < N; ++i) {
      const double yi = __shfl_sync(FULL, yk, i);
      if (act) xk += Li[i * N + lane] * yi;
    }
    if (act) {
      A.x[E * N + lane] = xk;
      A.hist_out[E * N + lane] = xk;
    }
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    A.iters[0] = it;
    A.iters[1] += min(it, A.max_iters);
    if (it > A.max_iters) atomicOr(A.flags, FLAG_NOCONV);
    if (!(rr == rr)) atomicOr(A.flags, FLAG_NAN);
  }
}

// b = (float) a; with *bad set (a singular coarse matrix met a non-positive pivot) b = 0 instead: the
// coarse level is dropped and the solve continues as block Jacobi -- the same policy as k_coarse_gj32
__global__ void k_to_f32(const double* __restrict__ a, float* __restrict__ b, size_t n, const int* __restrict__ bad) {
  size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
  const size_t st = (size_t)gridDim.x * blockDim.x;
  const bool zero = bad && __ldcg(bad) != 0;
  for (; i < n; i += st) b[i] = zero ? 0.f : (float)a[i];
}

}  // namespace lrbms
