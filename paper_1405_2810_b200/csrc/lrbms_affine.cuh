// lrbms_affine.cuh -- NEXT-1: the paper's affine online variant of the reduced system (a2 replaced).
//
//   eq:parameterizedMob: lambda_alpha(s) ~ sum_q theta_q(s) lambda_{alpha,q}, with M
//       saturation-independent mobility profiles;
//   eq:leastSquaresFit: Theta(s) = argmin || lambda_t(s) - sum_q theta_q lambda_{t,q} ||_l2
//       over the fine degrees of freedom (k = 0: cells), solved through the normal equations
//       G theta = h, G_qr = <lambda_q, lambda_r> (formed once with the profiles), h_q = <lambda_t(s), lambda_q>;
//   eq:reducedSystem: (c + sum_q theta_q b_q) p_H = e + sum_q theta_q d_q, where b_q, d_q are
//       the projections of the operator / right-hand side of lambda_{t,q} (offline, by k_project), and
//       c = e = 0 under reading R2 (the k = 0 operator and its Dirichlet data are linear in lambda).
//
// Per step: k_theta_partials (one pass over lambda and the M profiles, fixed-order per-CTA partials),
// k_theta_solve (one warp: fixed-order sums, Cholesky of G with dropped pivots for dependent profiles
// -- the paper's first and last profiles are both constant fields -- and the substitutions), and
// k_affine_combine (blocks = sum_q theta_q b_q, r = sum_q theta_q d_q: a streaming pass over the M
// precomputed operators, HBM-bound).  Deterministic: no atomics.
#pragma once
#include "lrbms_kernels.cuh"

namespace lrbms {

constexpr int AFF_MAXM = 16;

// part[q][blockIdx] = sum over this CTA's cells of x_i * Y[q][i], q < M (grid-stride over cells)
__global__ void __launch_bounds__(256) k_theta_partials(const double* __restrict__ x, const double* __restrict__ Y,
                                                        int M, size_t n, double* __restrict__ part) {
  __shared__ double red[8][AFF_MAXM];
  double acc[AFF_MAXM];
#pragma unroll
  for (int q = 0; q < AFF_MAXM; ++q) acc[q] = 0.0;
  const size_t stride = (size_t)gridDim.x * blockDim.x;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += stride) {
    const double xi = x[i];
#pragma unroll
    for (int q = 0; q < AFF_MAXM; ++q)
      if (q < M) acc[q] = fma(xi, Y[(size_t)q * n + i], acc[q]);
  }
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int q = 0; q < AFF_MAXM; ++q) {
    if (q >= M) break;
    const double v = warp_sum(acc[q]);
    if (lane == 0) red[warp][q] = v;
  }
  __syncthreads();
  if (threadIdx.x < M) {
    double t = 0.0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += red[w][threadIdx.x];
    part[(size_t)threadIdx.x * gridDim.x + blockIdx.x] = t;
  }
}

// out[q] = sum_b part[q][b] in a fixed order (one warp; lane-strided, then a fixed shuffle tree)
__device__ __forceinline__ void sum_partials(const double* part, int G, int M, double* out) {
  const int lane = threadIdx.x & 31;
  for (int q = 0; q < M; ++q) {
    double v = 0.0;
    for (int b = lane; b < G; b += 32) v += part[(size_t)q * G + b];
    v = warp_sum(v);
    if (lane == 0) out[q] = v;
  }
}

// one warp: row r of the Gram matrix from the partials
__global__ void k_gram_row(const double* __restrict__ part, int G, int M, double* __restrict__ gram, int r) {
  sum_partials(part, G, M, gram + (size_t)r * M);
}

// one warp: h from the partials, then theta from G theta = h.  Cholesky in index order; a pivot
// below 1e-12 of its original diagonal entry marks a profile that depends on the previous ones: its
// column is dropped (theta_q = 0), which leaves the fitted mobility sum_q theta_q lambda_q -- the
// least-squares projection -- unchanged.
__global__ void k_theta_solve(const double* __restrict__ part, int G, int M, const double* __restrict__ gram,
                              double* __restrict__ theta) {
  __shared__ double h[AFF_MAXM];
  sum_partials(part, G, M, h);
  __syncwarp();
  if (threadIdx.x != 0) return;
  double L[AFF_MAXM][AFF_MAXM], y[AFF_MAXM], t[AFF_MAXM];
  bool keep[AFF_MAXM];
  for (int i = 0; i < M; ++i)
    for (int j = 0; j < M; ++j) L[i][j] = gram[(size_t)i * M + j];
  for (int k = 0; k < M; ++k) {
    double d = L[k][k];
    for (int j = 0; j < k; ++j)
      if (keep[j]) d -= L[k][j] * L[k][j];
    keep[k] = d > 1e-12 * gram[(size_t)k * M + k] && d > 0.0;
    const double lkk = keep[k] ? sqrt(d) : 0.0;
    for (int i = k + 1; i < M; ++i) {
      double v = L[i][k];
      for (int j = 0; j < k; ++j)
        if (keep[j]) v -= L[i][j] * L[k][j];
      L[i][k] = keep[k] ? v / lkk : 0.0;
    }
    L[k][k] = lkk;
  }
  for (int i = 0; i < M; ++i) {   // L y = h
    double v = h[i];
    for (int j = 0; j < i; ++j) v -= L[i][j] * y[j];
    y[i] = keep[i] ? v / L[i][i] : 0.0;
  }
  for (int i = M - 1; i >= 0; --i) {   // L^T t = y
    double v = y[i];
    for (int j = i + 1; j < M; ++j) v -= L[j][i] * t[j];
    t[i] = keep[i] ? v / L[i][i] : 0.0;
  }
  for (int q = 0; q < M; ++q) theta[q] = t[q];
}

// out[i] = sum_q theta_q X[q * qstride + i] for i < len (the reduced operator or right-hand side), 16-byte
// streaming loads -- one pass over the M precomputed operators.  qstride (elements between profiles)
// is even (profile_stride), so every profile starts 16-byte aligned whatever the parity of len.
__global__ void __launch_bounds__(256) k_affine_combine(const double* __restrict__ X, const double* __restrict__ theta,
                                                        int M, size_t len, size_t qstride, double* __restrict__ out) {
  double th[AFF_MAXM];
#pragma unroll
  for (int q = 0; q < AFF_MAXM; ++q) th[q] = q < M ? theta[q] : 0.0;
  const size_t stride = (size_t)gridDim.x * blockDim.x;
  const size_t h = len >> 1, h2 = qstride >> 1;
  const double2* X2 = reinterpret_cast<const double2*>(X);
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < h; i += stride) {
    double a0 = 0.0, a1 = 0.0;
#pragma unroll
    for (int q = 0; q < AFF_MAXM; ++q)
      if (q < M) {
        const double2 v = __ldcs(X2 + (size_t)q * h2 + i);
        a0 = fma(th[q], v.x, a0);
        a1 = fma(th[q], v.y, a1);
      }
    reinterpret_cast<double2*>(out)[i] = make_double2(a0, a1);
  }
  if ((len & 1) && blockIdx.x == 0 && threadIdx.x == 0) {
    double a = 0.0;
    for (int q = 0; q < M; ++q) a = fma(th[q], X[(size_t)q * qstride + len - 1], a);
    out[len - 1] = a;
  }
}

}  // namespace lrbms
