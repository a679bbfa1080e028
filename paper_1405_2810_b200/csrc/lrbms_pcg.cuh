// lrbms_pcg.cuh -- a3: the reduced solve B c = r (eq:reducedSystem) on the GPU.
//
// One cooperative persistent kernel per solve, warp per subdomain (lane k <-> coefficient k of
// c_E, N <= 32).  Two-level preconditioned CG (Hestenes-Stiefel), warm-started from the previous
// step, iterated to ||r||_2 <= rtol ||b||_2 (exact-solve reading A17):
//   M^-1 r = D^-1 r + Z B_c^-1 Z^T r,  D = blockdiag(B_EE),  Z_E = Phi_E 1_E (indicator coefficients).
// The preconditioner is stored in fp32 (it only steers the iteration; every product with B, every
// vector update and every reduction is fp64).
//
// SpMV with the upper block storage reads every coupling block ONCE per iteration: the warp of E
// loads U = B_{E,E+a} row by row (coalesced), forms U v_{E+a} for itself by a warp reduce-scatter
// and U^T v_E for E+a, which it hands over through T[E+a][a]; the owner adds it after the grid
// barrier that follows the SpMV anyway (p.q is formed symmetrically, p.Bp = sum_E p_E.D p_E +
// 2 p_E.U p_{E+a}, so it needs no completed q).  3 grid barriers per iteration:
//   A: p = z + beta p_old (neighbours recomputed locally), q_partial, T, p.q     -> sync
//   B: alpha, x += alpha p, r -= alpha q, ||r||^2, Z^T r                        -> sync
//   C: z = M^-1 r, r.z                                                          -> sync
// Reductions are per-CTA in warp order, then every warp sums the per-CTA partials in a fixed
// order: all warps obtain bitwise-identical scalars, so the termination test is grid-uniform and
// runs are deterministic.
#pragma once
#include "lrbms_kernels.cuh"

namespace lrbms {

struct PcgArgs {
  Geo g;
  const double* blocks;   // [n_s][1+dim][N][N]
  const double* rhs;      // [n_s][N]
  const double* zc;       // [n_s][N]
  const float* Binv;      // [n_pad][n_pad] coarse inverse (fp32)
  const float* DinvT;     // [n_s][N][N], DinvT[j][k] = (B_EE^-1)[k][j] (fp32)
  double* x;              // solution / warm start
  double* xprev;          // solution of the previous solve (for the extrapolated warm start)
  double* r;
  double* z;
  double* pb0;            // search direction, double buffered
  double* pb1;
  double* qp;             // partial q (diag + own upper blocks)
  double* T;              // [n_s][3][N] transposed contributions from lower neighbours
  double* wc;             // [n_s] coarse residual Z^T r
  double* partials;       // [4][gridDim]
  int* iters;
  int* flags;
  double rtol;
  int max_iters;
  int n_pad;
  int use_coarse;
  int extrap;             // 1: x0 = 2 c^n - c^{n-1} (linear extrapolation in time), 0: x0 = c^n
  int wc_smem;            // stage Z^T r in shared memory for the coarse product
  unsigned long long* tstamp;  // optional phase timestamps (CTA 0, first iterations), or nullptr
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

// Part A of y = B v for subdomain E: returns lane's (D v_E + sum_a U_a v_{E+a}); stores U_a^T v_E
// into T[E+a][a]; adds v_E.(D v_E) + 2 v_E.(U_a v_{E+a}) (lane-local) to vbv.
template <class VF>
__device__ __forceinline__ double spmv_part(const PcgArgs& A, int E, const int C[3], int lane, double vE,
                                            VF vload, double& vbv) {
  const Geo& g = A.g;
  const int N = g.N, nb1 = 1 + g.dim;
  const double* Bd = A.blocks + (size_t)E * nb1 * N * N;
  const bool act = lane < N;
  prefetch_l1(Bd, nb1 * N * N * 8, lane);   // the whole block row of E (diag + upper couplings) into L1
  double buf[32];
#pragma unroll
  for (int j = 0; j < 32; ++j) buf[j] = (j < N && act) ? __ldg(Bd + j * N + lane) : 0.0;
  double acc = 0.0;
#pragma unroll
  for (int j = 0; j < 32; ++j) acc += buf[j] * __shfl_sync(FULL, vE, j);
  double local = vE * acc;
  for (int a = 0; a < g.dim; ++a) {
    if (C[a] + 1 >= g.S[a]) continue;
    const int En = E + g.Estride[a];
    const double vN = vload(En);
    const double* U = Bd + (size_t)(1 + a) * N * N;
#pragma unroll
    for (int k = 0; k < 32; ++k) buf[k] = (k < N && act) ? __ldg(U + k * N + lane) : 0.0;
    double tT = 0.0;  // (U^T v_E)[lane] = sum_k U[k][lane] v_E[k]
#pragma unroll
    for (int k = 0; k < 32; ++k) tT += buf[k] * __shfl_sync(FULL, vE, k);
#pragma unroll
    for (int k = 0; k < 32; ++k) buf[k] *= vN;
    const double tU = reduce_scatter32(buf, lane);   // (U v_{E+a})[lane]
    acc += tU;
    local += 2.0 * vE * tU;
    if (act) A.T[((size_t)En * 3 + a) * N + lane] = tT;
  }
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

// z_E = D_E^-1 r_E + zc_E e_E with e_E = (B_c^-1 Z^T r)_E  (coarse product in fp32: preconditioner)
__device__ __forceinline__ double precond(const PcgArgs& A, const float* wcv, int E, int lane, double rk) {
  const int N = A.g.N;
  float e = 0.f;
  prefetch_l1(A.DinvT + (size_t)E * N * N, N * N * 4, lane);
  if (A.use_coarse) {
    const float4* row = reinterpret_cast<const float4*>(A.Binv + (size_t)E * A.n_pad);
    const float4* w4 = reinterpret_cast<const float4*>(wcv);
    const int n4 = A.n_pad >> 2;
    float e0 = 0.f, e1 = 0.f;
#pragma unroll 4
    for (int F = lane; F < n4; F += 32) {
      const float4 b0 = __ldg(row + F), c0 = w4[F];
      e0 = fmaf(b0.x, c0.x, e0);
      e1 = fmaf(b0.y, c0.y, e1);
      e0 = fmaf(b0.z, c0.z, e0);
      e1 = fmaf(b0.w, c0.w, e1);
    }
    e = e0 + e1;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) e += __shfl_xor_sync(FULL, e, o);
  }
  const float* Di = A.DinvT + (size_t)E * N * N;
  double acc = 0.0;
  const bool act = lane < N;
#pragma unroll 8
  for (int j = 0; j < N; ++j) {
    const float d = act ? __ldg(Di + j * N + lane) : 0.f;
    acc += (double)d * __shfl_sync(FULL, rk, j);
  }
  if (act) acc += A.zc[E * N + lane] * (double)e;
  return act ? acc : 0.0;
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
__device__ __forceinline__ double grid_total(const double* partials, int slot) {
  const int lane = threadIdx.x & 31, G = gridDim.x;
  double s = 0.0;
  for (int b = lane; b < G; b += 32) s += partials[slot * G + b];
  return warp_sum(s);
}

__global__ void __launch_bounds__(512, 1) k_pcg(PcgArgs A) {
  cg::grid_group grid = cg::this_grid();
  __shared__ double red[4][32];
  extern __shared__ float wcs[];
  const Geo& g = A.g;
  const int N = g.N;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int TW = gridDim.x * (blockDim.x >> 5), gw = blockIdx.x * (blockDim.x >> 5) + warp;
  const bool act = lane < N;
  const float* wcv = wcs;
  auto stage_wc = [&]() {   // Z^T r -> shared memory (fp32, zero padded to n_pad)
    if (A.use_coarse) {
      for (int i = threadIdx.x; i < A.n_pad; i += blockDim.x) wcs[i] = i < g.n_s ? (float)A.wc[i] : 0.f;
      __syncthreads();
    }
  };

  // ---- warm start: keep the history, optionally extrapolate linearly in time
  for (int E = gw; E < g.n_s; E += TW)
    if (act) {
      const double xn = A.x[E * N + lane], xp = A.xprev[E * N + lane];
      A.xprev[E * N + lane] = xn;
      if (A.extrap) A.x[E * N + lane] = 2.0 * xn - xp;
    }
  grid.sync();

  // ---- setup: r = b - B x, ||b||^2, ||r||^2, Z^T r, z = M^-1 r, r.z
  double dummy = 0.0;
  for (int E = gw; E < g.n_s; E += TW) {
    int C[3];
    sub_xyz(g, E, C);
    auto xload = [&](int Ep) { return act ? A.x[Ep * N + lane] : 0.0; };
    const double q = spmv_part(A, E, C, lane, xload(E), xload, dummy);
    if (act) A.qp[E * N + lane] = q;
  }
  grid.sync();
  double pbb = 0.0, prr = 0.0;
  for (int E = gw; E < g.n_s; E += TW) {
    int C[3];
    sub_xyz(g, E, C);
    const double bk = act ? A.rhs[E * N + lane] : 0.0;
    const double rk = act ? bk - (A.qp[E * N + lane] + lower_contrib(A, E, C, lane)) : 0.0;
    if (act) A.r[E * N + lane] = rk;
    pbb += warp_sum(bk * bk);
    prr += warp_sum(rk * rk);
    const double w = warp_sum(act ? A.zc[E * N + lane] * rk : 0.0);
    if (lane == 0) A.wc[E] = w;
  }
  cta_partial(pbb, red, A.partials, 0);
  cta_partial(prr, red, A.partials, 1);
  grid.sync();
  const double bb = grid_total(A.partials, 0);
  double rr = grid_total(A.partials, 1);
  const double tol2 = A.rtol * A.rtol * bb;
  int it = 0;
  if (!(rr <= tol2) && bb > 0.0) {
    double prz = 0.0;
    stage_wc();
    for (int E = gw; E < g.n_s; E += TW) {
      const double rk = act ? A.r[E * N + lane] : 0.0;
      const double zk = precond(A, wcv, E, lane, rk);
      if (act) A.z[E * N + lane] = zk;
      prz += warp_sum(zk * rk);
    }
    cta_partial(prz, red, A.partials, 2);
    grid.sync();
    double rz = grid_total(A.partials, 2);
    double beta = 0.0;
    for (it = 1; it <= A.max_iters; ++it) {
      double* pcur = (it & 1) ? A.pb1 : A.pb0;
      const double* pold = (it & 1) ? A.pb0 : A.pb1;
      const bool first = it == 1;
      // A: p = z + beta p_old; q_partial = (D + U) p; T; p.Bp
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
        const double q = spmv_part(A, E, C, lane, pE, pload, vbv);
        if (act) A.qp[E * N + lane] = q;
        ppq += warp_sum(vbv);
      }
      if (A.tstamp && blockIdx.x == 0 && threadIdx.x == 0 && it < 64) A.tstamp[4 * it + 0] = gtimer();
      cta_partial(ppq, red, A.partials, 3);
      grid.sync();
      if (A.tstamp && blockIdx.x == 0 && threadIdx.x == 0 && it < 64) A.tstamp[4 * it + 1] = gtimer();
      const double pq = grid_total(A.partials, 3);
      if (!(pq > 0.0)) {
        if (blockIdx.x == 0 && threadIdx.x == 0) atomicOr(A.flags, FLAG_BREAKDOWN);
        break;
      }
      const double alpha = rz / pq;
      // B: x, r, ||r||^2, Z^T r
      prr = 0.0;
      for (int E = gw; E < g.n_s; E += TW) {
        int C[3];
        sub_xyz(g, E, C);
        double rk = 0.0;
        if (act) {
          const double q = A.qp[E * N + lane] + lower_contrib(A, E, C, lane);
          A.x[E * N + lane] += alpha * pcur[E * N + lane];
          rk = A.r[E * N + lane] - alpha * q;
          A.r[E * N + lane] = rk;
        }
        prr += warp_sum(rk * rk);
        const double w = warp_sum(act ? A.zc[E * N + lane] * rk : 0.0);
        if (lane == 0) A.wc[E] = w;
      }
      cta_partial(prr, red, A.partials, 1);
      grid.sync();
      if (A.tstamp && blockIdx.x == 0 && threadIdx.x == 0 && it < 64) A.tstamp[4 * it + 2] = gtimer();
      rr = grid_total(A.partials, 1);
      if (rr <= tol2) break;
      // C: z = M^-1 r, r.z
      double prz2 = 0.0;
      if (A.use_coarse)
        for (int E = gw; E < g.n_s; E += TW) prefetch_l1(A.Binv + (size_t)E * A.n_pad, A.n_pad * 4, lane);
      stage_wc();
      for (int E = gw; E < g.n_s; E += TW) {
        const double rk = act ? A.r[E * N + lane] : 0.0;
        const double zk = precond(A, wcv, E, lane, rk);
        if (act) A.z[E * N + lane] = zk;
        prz2 += warp_sum(zk * rk);
      }
      cta_partial(prz2, red, A.partials, 2);
      grid.sync();
      if (A.tstamp && blockIdx.x == 0 && threadIdx.x == 0 && it < 64) A.tstamp[4 * it + 3] = gtimer();
      const double rz_new = grid_total(A.partials, 2);
      beta = rz_new / rz;
      rz = rz_new;
    }
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    A.iters[0] = it;
    A.iters[1] += min(it, A.max_iters);
    if (it > A.max_iters) atomicOr(A.flags, FLAG_NOCONV);
    if (!(rr == rr)) atomicOr(A.flags, FLAG_NAN);
  }
}

// In-register Gauss-Jordan inverse of the N x N diagonal block (padded to 32 with identity).
// Lane j holds column j.  No pivoting: B_EE is SPD, pivots are Schur-complement diagonals.
__global__ void __launch_bounds__(128) k_block_inverse(Geo g, const double* __restrict__ blocks,
                                                      float* __restrict__ DinvT, int* flags) {
  const int lane = threadIdx.x & 31;
  const int E = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (E >= g.n_s) return;
  const int N = g.N;
  const double* Bd = blocks + (size_t)E * (1 + g.dim) * N * N;
  double m[32];
#pragma unroll
  for (int i = 0; i < 32; ++i) m[i] = (lane < N && i < N) ? Bd[i * N + lane] : (i == lane ? 1.0 : 0.0);
  bool bad = false;
#pragma unroll
  for (int k = 0; k < 32; ++k) {
    double f[32];
#pragma unroll
    for (int i = 0; i < 32; ++i) f[i] = __shfl_sync(FULL, m[i], k);
    const double pk = f[k];
    bad |= !(pk > 0.0);
    const double rowk = ((lane == k) ? 1.0 : m[k]) / pk;
#pragma unroll
    for (int i = 0; i < 32; ++i)
      if (i != k) m[i] = ((lane == k) ? 0.0 : m[i]) - f[i] * rowk;
    m[k] = rowk;
  }
  if (bad && lane == 0) atomicOr(flags, FLAG_PIVOT);
  if (lane < N) {
    float* D = DinvT + (size_t)E * N * N;
#pragma unroll
    for (int i = 0; i < 32; ++i)
      if (i < N) D[lane * N + i] = (float)m[i];
  }
}

__global__ void k_to_f32(const double* __restrict__ a, float* __restrict__ b, size_t n) {
  size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
  const size_t st = (size_t)gridDim.x * blockDim.x;
  for (; i < n; i += st) b[i] = (float)a[i];
}

}  // namespace lrbms
