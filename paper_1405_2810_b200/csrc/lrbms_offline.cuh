// lrbms_offline.cuh -- NEXT-3: the offline basis recipe on the GPU (its host reference
// is offline/recipe.py, checked against it in tests/test_gpu_offline.py).
//
//   1. the fine pressure at s0 (def:pressureDG P:337-345, the NEXT-2 solver) and its fluxes, dt^0
//   2. time of flight, eq:timeOfFlight at k = 0: per cell
//        tau_i * sum_{F out} F  =  phi_i V_i  +  sum_{F in} |F| tau_up(F)      (tau_up = 0 on inflow links)
//      The paper solves it by flow-ordered back substitution; on the GPU the same system
//      is solved by in-place relaxation sweeps from tau = 0: a cell's value is final once its upwind
//      cells are, so the sweeps reach the exact fixed point of the lower-triangular system after at
//      most (longest flow path) sweeps, each evaluated in the order of the host sweep (-x, +x, -y, +y,
//      -z, +z).  Stagnant cells (no outflow) get the largest finite tau.
//   3. mobility profiles and the training mobilities lambda^(j) = sum_q mu_q lambda_{t,q}
//      (P:679-680), mu from the caller (seeded training set)
//   4. fine snapshots p(lambda^(j)) (the NEXT-2 solver, one solve per training parameter)
//   5. per subdomain: Y = (I - v0 v0^T) P|_E, its thin SVD by one-sided (Hestenes) Jacobi rotations on
//      the snapshot columns (accurate singular vectors down to eps ||Y||, which the Gram-matrix route
//      would lose), Phi_E = [v0, left singular vectors above the noise floor, graded monomials
//      orthogonalised against them up to N] (reading A32).
#pragma once
#include "lrbms_kernels.cuh"

namespace lrbms {

constexpr int OFF_MAXJ = 64;      // training parameters (2N, N <= 32)
constexpr int OFF_MAXM = 16;      // mobility profiles
constexpr int OFF_NMONO = 48;     // graded monomial exponents passed in

struct OffArgs {
  Geo g;
  Links L;
  const double2* fc;
  const double* p;        // fine pressure at s0 (internal order)
  const double* lam0;     // lambda_t(s0)
  const double* phiV;     // phi V or nullptr
  double* outs;           // [n] sum of outgoing fluxes
  double* inm;            // [6][n] inflow magnitude through side d (0 if none)
  double* tau;            // [n]
  int* changed;           // sweep flags
};

// per cell: the outflow sum (the host recipe's order: +a faces as T1, then -a faces as T2, then links)
// and the inflow magnitudes per side; CTA per subdomain (links by one thread, deterministic)
__global__ void __launch_bounds__(512) k_off_flux(OffArgs A) {
  const Geo& g = A.g;
  const int E = blockIdx.x, nl = g.n_loc;
  const size_t n = g.n, base = (size_t)E * nl;
  int C[3];
  sub_xyz(g, E, C);
  for (int l = threadIdx.x; l < nl; l += blockDim.x) {
    int c[3];
    local_xyz(g, l, c);
    const size_t gl = base + l;
    const double pl = A.p[gl], ll = A.lam0[gl];
    double Fp[3] = {0.0, 0.0, 0.0}, Fm[3] = {0.0, 0.0, 0.0};   // flux out through +a / -a
    for (int a = 0; a < g.dim; ++a) {
      const int up = neighbour(g, E, C, l, c, a, +1), dn = neighbour(g, E, C, l, c, a, -1);
      if (up >= 0) Fp[a] = face_w(A.fc[gl * 3 + a], ll, A.lam0[up]) * (pl - A.p[up]);
      if (dn >= 0) Fm[a] = -(face_w(A.fc[(size_t)dn * 3 + a], A.lam0[dn], ll) * (A.p[dn] - pl));
      A.inm[(size_t)(2 * a) * n + gl] = fmax(-Fm[a], 0.0);       // side -a
      A.inm[(size_t)(2 * a + 1) * n + gl] = fmax(-Fp[a], 0.0);   // side +a
    }
    for (int a = g.dim; a < 3; ++a) {
      A.inm[(size_t)(2 * a) * n + gl] = 0.0;
      A.inm[(size_t)(2 * a + 1) * n + gl] = 0.0;
    }
    double o = 0.0;
    for (int a = 0; a < g.dim; ++a) o += fmax(Fp[a], 0.0);
    for (int a = 0; a < g.dim; ++a) o += fmax(Fm[a], 0.0);
    A.outs[gl] = o;
    A.tau[gl] = 0.0;
  }
  __syncthreads();
  if (threadIdx.x == 0)
    for (int q = A.L.sub_start[E]; q < A.L.sub_start[E + 1]; ++q) {
      const size_t gl = base + A.L.local[q];
      const double F = A.L.gK[q] * A.lam0[gl] * (A.p[gl] - A.L.p[q]);
      A.outs[gl] += fmax(F, 0.0);   // inflow links carry tau_up = 0: no term
    }
}

// one in-place relaxation sweep of the time-of-flight system; *changed = 1 if any tau moved
__global__ void __launch_bounds__(256) k_off_tof_sweep(OffArgs A) {
  const Geo& g = A.g;
  const size_t n = g.n;
  bool ch = false;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    const double o = A.outs[i];
    if (!(o > 0.0)) continue;
    const int E = (int)(i / g.n_loc), l = (int)(i - (size_t)E * g.n_loc);
    int C[3], c[3];
    sub_xyz(g, E, C);
    local_xyz(g, l, c);
    double acc = A.phiV ? A.phiV[i] : g.vol;
    for (int a = 0; a < g.dim; ++a)
      for (int t = 0; t < 2; ++t) {
        const double m = A.inm[(size_t)(2 * a + t) * n + i];
        if (m > 0.0) {
          const int nb = neighbour(g, E, C, l, c, a, t ? 1 : -1);
          acc += m * __ldcg(A.tau + nb);
        }
      }
    const double tn = acc / o;
    if (tn != __ldcg(A.tau + i)) {
      __stcg(A.tau + i, tn);
      ch = true;
    }
  }
  if (__any_sync(FULL, ch) && (threadIdx.x & 31) == 0) *A.changed = 1;
}

// stagnant cells (no outflow) -> the largest finite tau; tmax = that maximum (one CTA)
__global__ void k_off_tof_max(OffArgs A, double* tmax) {
  __shared__ double red[32];
  const size_t n = A.g.n;
  double m = 0.0;
  for (size_t i = threadIdx.x; i < n; i += blockDim.x)
    if (A.outs[i] > 0.0) m = fmax(m, A.tau[i]);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) m = fmax(m, __shfl_xor_sync(FULL, m, o));
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = m;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t = fmax(t, red[w]);
    *tmax = t;
  }
}
__global__ void k_off_tof_fill(OffArgs A, const double* tmax) {
  const size_t n = A.g.n;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
    if (!(A.outs[i] > 0.0)) A.tau[i] = *tmax;
}

struct TrainArgs {
  size_t n;
  int M;
  double thr[OFF_MAXM];    // tau threshold of profile q (inj where tau <= thr), q = 2..M-1
  double mu[OFF_MAXM];     // the training parameter of this snapshot
  const double* tau;
  const double* s0;        // initial saturation (internal order)
  Flu f;
  double s_inj;
  double* lam;             // out: lambda^(j)
};

// lambda^(j)_i = sum_q mu_q (lambda_w,q + lambda_o,q)(i), q in order
__global__ void k_off_train_lambda(TrainArgs T) {
  double lw1, lo1;
  mobilities(T.f, T.s_inj, lw1, lo1);
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < T.n; i += (size_t)gridDim.x * blockDim.x) {
    double lw0, lo0;
    mobilities(T.f, T.s0[i], lw0, lo0);
    const double t = T.tau[i];
    double acc = 0.0;
    for (int q = 0; q < T.M; ++q) {
      const bool inj = q == T.M - 1 ? true : (q == 0 ? false : !(t > T.thr[q]));
      acc = fma(T.mu[q], inj ? lw1 + lo1 : lw0 + lo0, acc);
    }
    T.lam[i] = acc;
  }
}

struct PodArgs {
  Geo g;
  int J;                   // snapshots (columns)
  int N;
  double* P;               // [J][n] snapshots (internal order), Y_E columns in place, then unit U columns
  double* sigma;           // [n_s][J] singular values in decreasing order
  int* order;              // [n_s][J] column of the k-th largest singular value
  double* Phi;             // out [n_s][N][n_loc]
  int* kept;               // out [n_s]
  double eps_pca;
  const double* sref;      // largest singular value over all subdomains
  int nmono;
  int mexp[OFF_NMONO][3];  // graded monomial exponents (x, y, z)
};

__device__ __forceinline__ double blk_sum(double v, double* red) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  v = warp_sum(v);
  __syncthreads();
  if (lane == 0) red[warp] = v;
  __syncthreads();
  double t = 0.0;
  for (int w = 0; w < nw; ++w) t += red[w];
  return t;
}

// per subdomain (CTA of 512 threads): project out v0, one-sided Jacobi on the J columns (round-robin
// pairs, a warp per pair, fixed schedule: deterministic), singular values and their order
__global__ void __launch_bounds__(512) k_off_pod_svd(PodArgs A) {
  __shared__ double red[16];
  __shared__ int pairs[OFF_MAXJ];
  __shared__ int rot_any;
  const Geo& g = A.g;
  const int E = blockIdx.x, nl = g.n_loc, J = A.J, Jp = J + (J & 1);
  const size_t n = g.n, base = (size_t)E * nl;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const double v0 = 1.0 / sqrt((double)nl);
  // Y = (I - v0 v0^T) P|_E, column by column
  for (int j = 0; j < J; ++j) {
    double* y = A.P + (size_t)j * n + base;
    double s = 0.0;
    for (int l = threadIdx.x; l < nl; l += blockDim.x) s += v0 * y[l];
    s = blk_sum(s, red);
    for (int l = threadIdx.x; l < nl; l += blockDim.x) y[l] -= v0 * s;
  }
  __syncthreads();
  // ||Y||_F^2: pairs whose columns are both below the rounding level of Y are left alone
  double fro = 0.0;
  for (int j = 0; j < J; ++j) {
    const double* y = A.P + (size_t)j * n + base;
    for (int l = threadIdx.x; l < nl; l += blockDim.x) fro = fma(y[l], y[l], fro);
  }
  fro = blk_sum(fro, red);
  const double tiny = 1e-32 * fro;
  // round-robin tournament over Jp slots (slot J = a zero dummy column when J is odd)
  if (threadIdx.x < Jp) pairs[threadIdx.x] = threadIdx.x;
  __syncthreads();
  for (int sweep = 0; sweep < 40; ++sweep) {
    if (threadIdx.x == 0) rot_any = 0;
    __syncthreads();
    for (int round = 0; round < Jp - 1; ++round) {
      for (int pi = warp; pi < Jp / 2; pi += nw) {
        int a = pairs[pi], b = pairs[Jp - 1 - pi];
        if (a >= J || b >= J) continue;
        if (a > b) { const int t = a; a = b; b = t; }
        double* x = A.P + (size_t)a * n + base;
        double* y = A.P + (size_t)b * n + base;
        double xx = 0.0, yy = 0.0, xy = 0.0;
        for (int l = lane; l < nl; l += 32) {
          const double xv = __ldcg(x + l), yv = __ldcg(y + l);
          xx = fma(xv, xv, xx);
          yy = fma(yv, yv, yy);
          xy = fma(xv, yv, xy);
        }
        xx = warp_sum(xx); yy = warp_sum(yy); xy = warp_sum(xy);
        if (fabs(xy) > 1e-15 * sqrt(xx * yy) && xx > tiny && yy > tiny) {
          const double zeta = (yy - xx) / (2.0 * xy);
          const double t = (zeta >= 0.0 ? 1.0 : -1.0) / (fabs(zeta) + sqrt(1.0 + zeta * zeta));
          const double cs = 1.0 / sqrt(1.0 + t * t), sn = cs * t;
          for (int l = lane; l < nl; l += 32) {
            const double xv = __ldcg(x + l), yv = __ldcg(y + l);
            __stcg(x + l, cs * xv - sn * yv);
            __stcg(y + l, sn * xv + cs * yv);
          }
          if (lane == 0) rot_any = 1;
        }
      }
      __syncthreads();
      if (threadIdx.x == 0) {   // rotate the tournament: slot 0 fixed, the others shift by one
        const int last = pairs[Jp - 1];
        for (int k = Jp - 1; k > 1; --k) pairs[k] = pairs[k - 1];
        pairs[1] = last;
      }
      __threadfence_block();
      __syncthreads();
    }
    const int any = rot_any;
    __syncthreads();
    if (!any) break;
  }
  // singular values = column norms; order by decreasing value (ties by column index)
  double* sg = A.sigma + (size_t)E * J;
  for (int j = warp; j < J; j += nw) {
    const double* y = A.P + (size_t)j * n + base;
    double s = 0.0;
    for (int l = lane; l < nl; l += 32) { const double v = __ldcg(y + l); s = fma(v, v, s); }
    s = warp_sum(s);
    if (lane == 0) sg[j] = sqrt(s);
  }
  __syncthreads();
  if (threadIdx.x < J) {
    const double me = sg[threadIdx.x];
    int rank = 0;
    for (int k = 0; k < J; ++k) {
      const double o = sg[k];
      rank += (o > me) || (o == me && k < (int)threadIdx.x);
    }
    A.order[(size_t)E * J + rank] = threadIdx.x;
  }
}

__global__ void k_off_sigma_max(const double* sigma, size_t cnt, double* out) {
  __shared__ double red[32];
  double m = 0.0;
  for (size_t i = threadIdx.x; i < cnt; i += blockDim.x) m = fmax(m, sigma[i]);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) m = fmax(m, __shfl_xor_sync(FULL, m, o));
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = m;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t = fmax(t, red[w]);
    *out = t;
  }
}

// per subdomain: Phi_E = [v0, the kept left singular vectors in decreasing singular value, graded
// monomials], each candidate orthogonalised against the columns before it (classical Gram-Schmidt
// twice), normalised and signed so that its largest-magnitude entry is positive -- the host recipe's
// construction (offline/recipe.py pod_bases)
__global__ void __launch_bounds__(512) k_off_pod_assemble(PodArgs A) {
  extern __shared__ double osm[];   // [N][n_loc] the columns so far, then [n_loc] the candidate
  __shared__ double red[16];
  __shared__ double cf[32];
  __shared__ int arg_s;
  const Geo& g = A.g;
  const int E = blockIdx.x, nl = g.n_loc, N = A.N, J = A.J;
  const size_t n = g.n, base = (size_t)E * nl;
  double* Q = osm;
  double* v = osm + (size_t)N * nl;
  const double v0 = 1.0 / sqrt((double)nl);
  for (int l = threadIdx.x; l < nl; l += blockDim.x) Q[l] = v0;
  const double* sg = A.sigma + (size_t)E * J;
  const int* ord = A.order + (size_t)E * J;
  const double thr = A.eps_pca * *A.sref;
  int k = 0;
  while (k < N - 1 && k < J && sg[ord[k]] > thr) ++k;
  int cols = 1, cand = 0;
  const int ncand = k + A.nmono;
  __syncthreads();
  while (cols < N && cand < ncand) {
    const bool mode = cand < k;
    double nc2 = 0.0;
    for (int l = threadIdx.x; l < nl; l += blockDim.x) {
      double x;
      if (mode) {
        x = __ldcg(A.P + (size_t)ord[cand] * n + base + l);
      } else {
        const int* e = A.mexp[cand - k];
        int c[3];
        local_xyz(g, l, c);
        const double X = (2.0 * c[0] + 1.0) / g.s[0] - 1.0, Y = (2.0 * c[1] + 1.0) / g.s[1] - 1.0,
                     Z = (2.0 * c[2] + 1.0) / g.s[2] - 1.0;
        x = 1.0;
        for (int q = 0; q < e[0]; ++q) x *= X;
        for (int q = 0; q < e[1]; ++q) x *= Y;
        for (int q = 0; q < e[2]; ++q) x *= Z;
      }
      v[l] = x;
      nc2 = fma(x, x, nc2);
    }
    const double nc = sqrt(blk_sum(nc2, red));
    for (int pass = 0; pass < 2; ++pass) {   // v -= Q (Q^T v)
      __syncthreads();
      for (int m = 0; m < cols; ++m) {
        double d = 0.0;
        for (int l = threadIdx.x; l < nl; l += blockDim.x) d = fma(Q[(size_t)m * nl + l], v[l], d);
        d = blk_sum(d, red);
        if (threadIdx.x == 0) cf[m] = d;
      }
      __syncthreads();
      for (int l = threadIdx.x; l < nl; l += blockDim.x) {
        double x = v[l];
        for (int m = 0; m < cols; ++m) x -= Q[(size_t)m * nl + l] * cf[m];
        v[l] = x;
      }
    }
    __syncthreads();
    double nv2 = 0.0;
    for (int l = threadIdx.x; l < nl; l += blockDim.x) nv2 = fma(v[l], v[l], nv2);
    const double nv = sqrt(blk_sum(nv2, red));
    if (nv > (mode ? 0.5 : 1e-8) * nc) {
      // sign: the largest-magnitude entry positive (first index on ties)
      if (threadIdx.x == 0) {
        int am = 0;
        double best = -1.0;
        for (int l = 0; l < nl; ++l) {
          const double a = fabs(v[l]);
          if (a > best) { best = a; am = l; }
        }
        arg_s = am;
      }
      __syncthreads();
      const double sgn = v[arg_s] > 0.0 ? 1.0 : -1.0;
      for (int l = threadIdx.x; l < nl; l += blockDim.x) Q[(size_t)cols * nl + l] = sgn * (v[l] / nv);
      ++cols;
    }
    ++cand;
    __syncthreads();
  }
  for (int m = 0; m < N; ++m)
    for (int l = threadIdx.x; l < nl; l += blockDim.x) A.Phi[((size_t)E * N + m) * nl + l] = m < cols ? Q[(size_t)m * nl + l] : 0.0;
  if (threadIdx.x == 0) A.kept[E] = cols < N ? -1 : k;
}

}  // namespace lrbms
