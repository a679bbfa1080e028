// lrbms_fine.cuh -- NEXT-2: the fine-scale reference scheme on the GPU.
//
//   alg:highDimTwoPhaseFlow at k = 0: per step the fine pressure system
//   A(lambda(s^n)) p = b(lambda(s^n)) of def:pressureDG (at k = 0 the operator of
//   eq:swipBilP reduces to A = sum_F w_F (e_a - e_b)(e_a - e_b)^T + sum_L g_L e_a e_a^T,
//   b = sum_L g_L p_L e_a with the face weights of reading R2), then the same fluxes, CFL step and
//   upwind transport as the reduced scheme (k_flux_cfl, k_transport).  This is the paper's
//   comparison run (the speed-up of P:1300-1302), i.e. the LRBMS step with Phi_E = I.
//
// Kernels:
//   k_fine_setup (CTA per subdomain, thread per cell): the static neighbour table (first call),
//     the + face weights w[a][i] = T_F (tau_a lambda_i + tau_b lambda_nb), the diagonal
//     d_i = sum of the weights of the faces of i + sum of its link weights, and b (links in the
//     subdomain's link order, by one thread: deterministic).
//   k_fine_coarse_stencil (CTA per subdomain): E = Z^T A Z on the subdomain indicators, inverted
//     each step by the reduced solver's Gauss-Jordan kernel (k_coarse_gj32, fp32).
//   k_fine_pcg (cooperative, grid-stride over cells): CG warm-started from the previous pressure,
//     preconditioned by M^-1 = D^-1 + Z E^-1 Z^T (Jacobi only when no coarse inverse is available);
//     the search direction p_new = z + beta p formed on the fly for the neighbours inside the SpMV
//     (double-buffered p); grid synchronisations per iteration: p.Ap, the coarse barrier (two-level
//     only), r.z; stop when r.M^-1 r <= rtol^2 b.D^-1 b.  Deterministic (fixed-order partials).
#pragma once
#include "lrbms_kernels.cuh"

namespace lrbms {

struct FineArgs {
  Geo g;
  Links L;
  const double2* fc;   // [n][3] static face coefficients (T tau_a, T tau_b) of the + face per axis
  const double* lam;   // [n] lambda_t(s^n)
  double* x;           // [n] pressure (warm start in, solution out): the context's p
  double* r;
  double* z;
  double* p0;          // search direction, double buffered
  double* p1;
  double* q;           // A p
  double* diag;        // [n]
  double* rhs;         // [n]
  double* w;           // [3][n] + face weight of cell i along axis a (0 without a + neighbour)
  unsigned short* nbr; // [n] neighbour code of cell i: bit d (side d = 2 a + (dir > 0)) = the neighbour
                       // exists, bit 6 + d = it lies in the adjacent subdomain; its index is then
                       // i + xoff[d], else i + ioff[d]
  int ioff[6], xoff[6];
  double* partials;    // [4][gridDim]
  unsigned* bar;       // grid-barrier counter (zeroed before the launch)
  int* iters;          // [0]: iterations of the last solve, [1]: running total
  int* flags;
  double rtol;
  int max_iters;
  int build_nbr;       // 1: k_fine_setup fills nbr (first call of a run)
  // two-level preconditioner M^-1 = D^-1 + Z E^-1 Z^T (Z = subdomain indicators, E = Z^T A Z)
  int coarse;          // 0: Jacobi only
  const float* Xc;     // [n_pad][n_pad] E^-1 (fp32: it only steers the iteration)
  double* wc;          // [n_s] Z^T r
  int n_pad;
  unsigned long long* dt_bits;   // the step's dt minimum (reset here, as k_recon does for the reduced step)
};

__global__ void __launch_bounds__(512) k_fine_setup(FineArgs A) {
  extern __shared__ double fsm[];
  double* dg = fsm;                // [n_loc] diagonal
  double* bl = fsm + A.g.n_loc;    // [n_loc] right-hand side
  const Geo& g = A.g;
  const int E = blockIdx.x, nl = g.n_loc;
  const size_t n = g.n;
  int C[3];
  sub_xyz(g, E, C);
  const size_t base = (size_t)E * nl;
  if (E == 0 && threadIdx.x == 0) *A.dt_bits = 0x7ff0000000000000ull;   // +inf
  for (int l = threadIdx.x; l < nl; l += blockDim.x) {
    int c[3];
    local_xyz(g, l, c);
    const size_t gl = base + l;
    const double ll = A.lam[gl];
    double d = 0.0;
    unsigned code = 0;
    for (int a = 0; a < 3; ++a)
      for (int t = 0; t < 2; ++t) {
        const int dir = t ? 1 : -1;
        const int nb = a < g.dim ? neighbour(g, E, C, l, c, a, dir) : -1;
        if (nb >= 0) {
          code |= 1u << (2 * a + t);
          if (c[a] + dir < 0 || c[a] + dir >= g.s[a]) code |= 1u << (6 + 2 * a + t);
        }
        if (nb < 0) {
          if (t) A.w[(size_t)a * n + gl] = 0.0;
          continue;
        }
        // the face between this cell and nb: T1 = the lower cell along a (eq:upwind orientation)
        const double wf = t ? face_w(A.fc[gl * 3 + a], ll, A.lam[nb]) : face_w(A.fc[(size_t)nb * 3 + a], A.lam[nb], ll);
        if (t) A.w[(size_t)a * n + gl] = wf;
        d += wf;
      }
    if (A.build_nbr) A.nbr[gl] = (unsigned short)code;
    dg[l] = d;
    bl[l] = 0.0;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int qi = A.L.sub_start[E]; qi < A.L.sub_start[E + 1]; ++qi) {
      const int l = A.L.local[qi];
      const double gL = A.L.gK[qi] * A.lam[base + l];
      dg[l] += gL;
      bl[l] += gL * A.L.p[qi];
    }
  }
  __syncthreads();
  for (int l = threadIdx.x; l < nl; l += blockDim.x) {
    A.diag[base + l] = dg[l];
    A.rhs[base + l] = bl[l];
  }
}

// E = Z^T A Z on the subdomain indicators, as the 7-point stencil Es[E][0..7] of the reduced
// solver's coarse level (0: diagonal, 1 + a: coupling to E + e_a, 4 + a: coupling to E - e_a):
// E_EE = sum over the cells of E of (d_i - the weights of their faces inside E), E_EE' = - the sum
// of the weights of the faces between E and E'.  CTA per subdomain, fixed-order block sums.
__global__ void __launch_bounds__(256) k_fine_coarse_stencil(FineArgs A, double* __restrict__ Es) {
  __shared__ double red[8][7];
  const Geo& g = A.g;
  const int E = blockIdx.x, nl = g.n_loc;
  const size_t n = g.n;
  double v[7];
#pragma unroll
  for (int k = 0; k < 7; ++k) v[k] = 0.0;
  for (int l = threadIdx.x; l < nl; l += blockDim.x) {
    const size_t i = (size_t)E * nl + l;
    const unsigned code = A.nbr[i];
    double dsum = A.diag[i];
#pragma unroll
    for (int d = 0; d < 6; ++d) {
      if (!((code >> d) & 1u)) continue;
      const int a = d >> 1;
      const bool cross = (code >> (6 + d)) & 1u;
      const size_t j = i + (cross ? A.xoff[d] : A.ioff[d]);
      const double wf = (d & 1) ? A.w[(size_t)a * n + i] : A.w[(size_t)a * n + j];
      if (cross) v[1 + ((d & 1) ? a : 3 + a)] -= wf;
      else dsum -= wf;
    }
    v[0] += dsum;
  }
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int k = 0; k < 7; ++k) {
    const double t = warp_sum(v[k]);
    if (lane == 0) red[warp][k] = t;
  }
  __syncthreads();
  if (threadIdx.x < 8) {
    double t = 0.0;
    if (threadIdx.x < 7)
      for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += red[w][threadIdx.x];
    Es[(size_t)E * 8 + threadIdx.x] = t;
  }
}

// fixed-order block sum (every thread gets the same value)
__device__ __forceinline__ double fine_block_sum(double v, double* sh) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  v = warp_sum(v);
  if (lane == 0) sh[warp] = v;
  __syncthreads();
  double t = 0.0;
  for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += sh[w];
  __syncthreads();
  return t;
}

// two-level part, CTA per subdomain: wc[E] = sum of r over E (r already updated), then after a grid
// barrier z = D^-1 r + e_E with e = E^-1 wc; returns this thread's part of r.z
__device__ __forceinline__ double fine_coarse_z(const FineArgs& A, double* sh, unsigned& epoch) {
  const Geo& g = A.g;
  const int nl = g.n_loc;
  for (int E = blockIdx.x; E < g.n_s; E += gridDim.x) {
    double ws = 0.0;
    for (int l = threadIdx.x; l < nl; l += blockDim.x) ws += A.r[(size_t)E * nl + l];
    ws = fine_block_sum(ws, sh);
    if (threadIdx.x == 0) A.wc[E] = ws;
  }
  grid_barrier_rel(A.bar, epoch);
  double prz = 0.0;
  for (int E = blockIdx.x; E < g.n_s; E += gridDim.x) {
    double ep = 0.0;
    const float* row = A.Xc + (size_t)E * A.n_pad;
    for (int F = threadIdx.x; F < g.n_s; F += blockDim.x) ep = fma((double)row[F], __ldcg(A.wc + F), ep);
    const double e = fine_block_sum(ep, sh);
    for (int l = threadIdx.x; l < nl; l += blockDim.x) {
      const size_t i = (size_t)E * nl + l;
      const double ri = A.r[i];
      const double zi = ri / A.diag[i] + e;
      A.z[i] = zi;
      prz = fma(ri, zi, prz);
    }
  }
  return prz;
}

// (A v)_i = d_i v_i - sum over the faces of i of w_F v_nb, with v_j = vz[j] + beta * vp[j] for
// every j (beta = 0, vp = nullptr: v = vz)
__device__ __forceinline__ double fine_apply(const FineArgs& A, size_t i, const double* vz, const double* vp,
                                             double beta, double vi) {
  const size_t n = A.g.n;
  double acc = A.diag[i] * vi;
  const unsigned code = A.nbr[i];
#pragma unroll
  for (int d = 0; d < 6; ++d) {
    if (!((code >> d) & 1u)) continue;
    const size_t j = i + (((code >> (6 + d)) & 1u) ? A.xoff[d] : A.ioff[d]);
    const double wf = (d & 1) ? A.w[(size_t)(d >> 1) * n + i] : A.w[(size_t)(d >> 1) * n + j];
    const double vj = vp ? fma(beta, vp[j], vz[j]) : vz[j];
    acc = fma(-wf, vj, acc);
  }
  return acc;
}

__global__ void __launch_bounds__(256) k_fine_pcg(FineArgs A) {
  __shared__ double red16[16];
  __shared__ double bc[1];
  unsigned epoch = 0;
  const size_t n = A.g.n;
  const size_t stride = (size_t)gridDim.x * blockDim.x;
  const size_t i0 = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  // r = b - A x, z = D^-1 r
  double prz = 0.0, pbb = 0.0;
  for (size_t i = i0; i < n; i += stride) {
    const double ri = A.rhs[i] - fine_apply(A, i, A.x, nullptr, 0.0, A.x[i]);
    const double zi = ri / A.diag[i];
    A.r[i] = ri;
    A.z[i] = zi;
    prz = fma(ri, zi, prz);
    pbb = fma(A.rhs[i], A.rhs[i] / A.diag[i], pbb);
  }
  __shared__ double shb[8];
  if (A.coarse) {   // r was written grid-stride: a barrier before the per-subdomain sums
    grid_barrier_rel(A.bar, epoch);
    prz = fine_coarse_z(A, shb, epoch);
  }
  double rz = grid_reduce_rel(warp_sum(prz), red16, A.partials, A.bar, epoch, &bc[0]);
  const double bb = grid_reduce_rel(warp_sum(pbb), red16, A.partials, A.bar, epoch, &bc[0]);
  const double tol2 = A.rtol * A.rtol * bb;
  double beta = 0.0;
  int it = 0;
  bool ok = true;
  while (rz > tol2 && it < A.max_iters) {
    // phase A: p_new = z + beta p (p = the previous direction, absent in the first iteration),
    // q = A p_new with the neighbours' p_new formed on the fly
    const double* pold = it == 0 ? nullptr : ((it & 1) ? A.p0 : A.p1);
    double* pnew = (it & 1) ? A.p1 : A.p0;
    double ppq = 0.0;
    for (size_t i = i0; i < n; i += stride) {
      const double pi = pold ? fma(beta, pold[i], A.z[i]) : A.z[i];
      const double qi = fine_apply(A, i, A.z, pold, beta, pi);
      pnew[i] = pi;
      A.q[i] = qi;
      ppq = fma(pi, qi, ppq);
    }
    const double pq = grid_reduce_rel(warp_sum(ppq), red16, A.partials, A.bar, epoch, &bc[0]);
    if (!(pq > 0.0)) {
      ok = false;
      break;
    }
    const double alpha = rz / pq;
    // phase B: x += alpha p, r -= alpha q, z = D^-1 r, r.z
    prz = 0.0;
    if (A.coarse) {   // x, r updated per subdomain, then the coarse correction (one more barrier)
      const int nl = A.g.n_loc;
      for (int E = blockIdx.x; E < A.g.n_s; E += gridDim.x)
        for (int l = threadIdx.x; l < nl; l += blockDim.x) {
          const size_t i = (size_t)E * nl + l;
          A.x[i] = fma(alpha, pnew[i], A.x[i]);
          A.r[i] = fma(-alpha, A.q[i], A.r[i]);
        }
      __syncthreads();
      prz = fine_coarse_z(A, shb, epoch);
    } else {
      for (size_t i = i0; i < n; i += stride) {
        A.x[i] = fma(alpha, pnew[i], A.x[i]);
        const double ri = fma(-alpha, A.q[i], A.r[i]);
        const double zi = ri / A.diag[i];
        A.r[i] = ri;
        A.z[i] = zi;
        prz = fma(ri, zi, prz);
      }
    }
    const double rz_new = grid_reduce_rel(warp_sum(prz), red16, A.partials, A.bar, epoch, &bc[0]);
    beta = rz_new / rz;
    rz = rz_new;
    ++it;
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    A.iters[0] = it;
    A.iters[1] += it;
    if (!ok) atomicOr(A.flags, FLAG_BREAKDOWN);
    else if (rz > tol2) atomicOr(A.flags, FLAG_NOCONV);
    if (!(rz == rz)) atomicOr(A.flags, FLAG_NAN);
  }
}

}  // namespace lrbms
