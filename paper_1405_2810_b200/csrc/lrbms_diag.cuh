// lrbms_diag.cuh -- K6 diagnostics of the last step (SURVEY §2e K6, §5 metrics), off the timed path.
//
// On the state after a step (p^n of the step, lambda(s^n), f(s^n), s^n and s^{n+1} still in the
// double buffers): the water volume before and after (eq:saturationDG conserves it up to the link
// fluxes: pin P3), the saturation range, the relative mass loss of the reduced velocity
//   zeta(T) = |int_dT u.n dS| / max_{x in dT} |u(x)|            (reading A33)
// (its maximum and mean over the cells), the coarse conservation defect max_E |sum_{i in E} div_i|
// (0 when 1_E is in span Phi_E: P4), the water leaving through links, and the total link
// in- and outflow.  One CTA per subdomain writes fixed-order partials; k_diag_final reduces them in a
// fixed order (deterministic).
#pragma once
#include "lrbms_kernels.cuh"

namespace lrbms {

constexpr int DIAG_NP = 10;   // partials per subdomain

struct DiagArgs {
  Geo g;
  Flu f;
  Links L;
  const double* p;       // pressure of the last step (internal order)
  const double* lam;     // lambda_t(s^n)
  const double* fw;      // f_w(s^n)
  const double* s_prev;  // s^n
  const double* s;       // s^{n+1}
  const double* phiV;    // phi V or nullptr
  const double2* fc;
  double area[3];        // |F| of an interior face normal to axis a
  double* part;          // [n_s][DIAG_NP]
};

// block reduction in a fixed order: warp shuffles, then warp 0 over the warps in index order
template <typename Op>
__device__ __forceinline__ double block_reduce(double v, double* red, Op op) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = (blockDim.x + 31) >> 5;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = op(v, __shfl_xor_sync(FULL, v, o));
  __syncthreads();
  if (lane == 0) red[warp] = v;
  __syncthreads();
  double r = red[0];
  for (int w = 1; w < nw; ++w) r = op(r, red[w]);
  return r;
}

__global__ void __launch_bounds__(512) k_diag(DiagArgs A) {
  extern __shared__ double diag_sm[];   // [n_loc] net outflow, [n_loc] max |u.n|
  __shared__ double red[16];
  const Geo& g = A.g;
  const int E = blockIdx.x, nl = g.n_loc;
  double* net = diag_sm;
  double* umax = diag_sm + nl;
  int C[3];
  sub_xyz(g, E, C);
  const size_t base = (size_t)E * nl;
  for (int l = threadIdx.x; l < nl; l += blockDim.x) {
    int c[3];
    local_xyz(g, l, c);
    const double pl = A.p[base + l], ll = A.lam[base + l];
    double acc = 0.0, um = 0.0;
    for (int a = 0; a < g.dim; ++a)
      for (int dir = -1; dir <= 1; dir += 2) {
        const int nb = neighbour(g, E, C, l, c, a, dir);
        if (nb < 0) continue;
        const double F = dir > 0 ? face_w(A.fc[(base + l) * 3 + a], ll, A.lam[nb]) * (pl - A.p[nb])
                                 : -(face_w(A.fc[(size_t)nb * 3 + a], A.lam[nb], ll) * (A.p[nb] - pl));
        acc += F;
        um = fmax(um, fabs(F) / A.area[a]);
      }
    net[l] = acc;
    umax[l] = um;
  }
  __syncthreads();
  double w_out = 0.0, q_in = 0.0, q_out = 0.0;
  if (threadIdx.x == 0) {   // links in the subdomain's link order
    for (int q = A.L.sub_start[E]; q < A.L.sub_start[E + 1]; ++q) {
      const int l = A.L.local[q];
      const double F = A.L.gK[q] * A.lam[base + l] * (A.p[base + l] - A.L.p[q]);
      net[l] += F;
      w_out += F * (F >= 0.0 ? A.fw[base + l] : frac_flow(A.f, A.L.s_ext[q]));
      q_in += fmax(-F, 0.0);
      q_out += fmax(F, 0.0);
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) {   // the link faces' flux densities enter max |u|; a link face normal to axis
    // a has |F| = sqrt(geo2 V / 2) (geo2 = 2 |F| / h_a, V = |F| h_a)
    for (int q = A.L.sub_start[E]; q < A.L.sub_start[E + 1]; ++q) {
      const int l = A.L.local[q];
      const double F = A.L.gK[q] * A.lam[base + l] * (A.p[base + l] - A.L.p[q]);
      umax[l] = fmax(umax[l], fabs(F) / sqrt(0.5 * A.L.geo2[q] * g.vol));
    }
  }
  __syncthreads();
  double m0 = 0.0, m1 = 0.0, smin = INFINITY, smax = -INFINITY, zmax = 0.0, zsum = 0.0, dsum = 0.0;
  for (int l = threadIdx.x; l < nl; l += blockDim.x) {
    const double pv = A.phiV ? A.phiV[base + l] : g.vol;
    m0 += pv * A.s_prev[base + l];
    const double sn = A.s[base + l];
    m1 += pv * sn;
    smin = fmin(smin, sn);
    smax = fmax(smax, sn);
    const double z = umax[l] > 0.0 ? fabs(net[l]) / umax[l] : 0.0;
    zmax = fmax(zmax, z);
    zsum += z;
    dsum += net[l];
  }
  auto add = [](double a, double b) { return a + b; };
  auto mn = [](double a, double b) { return fmin(a, b); };
  auto mx = [](double a, double b) { return fmax(a, b); };
  const double r0 = block_reduce(m0, red, add), r1 = block_reduce(m1, red, add);
  const double r2 = block_reduce(smin, red, mn), r3 = block_reduce(smax, red, mx);
  const double r4 = block_reduce(zmax, red, mx), r5 = block_reduce(zsum, red, add);
  const double r6 = block_reduce(dsum, red, add);
  if (threadIdx.x == 0) {
    double* o = A.part + (size_t)E * DIAG_NP;
    o[0] = r0; o[1] = r1; o[2] = r2; o[3] = r3; o[4] = r4; o[5] = r5; o[6] = r6;
    o[7] = w_out; o[8] = q_in; o[9] = q_out;
  }
}

// out[0..9]: mass_prev, mass, s_min, s_max, zeta_max, zeta_sum, max_E |coarse defect|, water out,
// link inflow, link outflow.  One warp per quantity: lane-strided over the subdomains, then a fixed
// shuffle tree (deterministic; one thread walking all subdomains took 0.8 ms on C5).  Launch with
// 32 * DIAG_NP threads.
__global__ void k_diag_final(const double* __restrict__ part, int n_s, double* __restrict__ out) {
  const int k = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (blockIdx.x != 0 || k >= DIAG_NP) return;
  const bool is_min = k == 2, is_max = k == 3 || k == 4 || k == 6;
  double v = is_min ? INFINITY : (k == 3 ? -INFINITY : 0.0);
  for (int E = lane; E < n_s; E += 32) {
    double q = part[(size_t)E * DIAG_NP + k];
    if (k == 6) q = fabs(q);
    v = is_min ? fmin(v, q) : (is_max ? fmax(v, q) : v + q);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const double w = __shfl_xor_sync(FULL, v, o);
    v = is_min ? fmin(v, w) : (is_max ? fmax(v, w) : v + w);
  }
  if (lane == 0) out[k] = v;
}

}  // namespace lrbms
