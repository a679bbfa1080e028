// lrbms_transport.cuh -- a5 + a6 fused: face fluxes of the reconstructed pressure, the CFL step and
// the explicit upwind transport in ONE cooperative kernel.
//
//   a5  F_F = w_F(lambda(s^n)) (p_a - p_b), F_L = g_L (p_a - p_L)        eq:velocityDG P:366-377 (k = 0)
//       Q_i = max(sum out, sum in); dt = cfl min_i phi_i V_i / (f'_max Q_i)  reading R4
//   a6  s_i^{n+1} = s_i^n - dt / (phi_i V_i) sum_F F^out f(chi(s^n))        eq:saturationDG P:389-399,
//                                                                            eq:upwind P:400-417 (A5)
//       then lambda_t, f_w of s^{n+1}: a1 of the next step, formed once
//
// Each CTA walks its subdomains (grid-stride): phase 1 forms every cell's outward fractional-flow flux
// sum and flux bound Q from the neighbours' p, lambda, f_w (one thread per cell, the subdomain shape a
// compile-time constant where the configs allow it, so the neighbour index math is shifts and adds),
// keeps the sums in shared memory and folds the CTA's dt bound into the global minimum (atomicMin on
// the ordered bits: order-independent, deterministic); one grid barrier; phase 2 updates s of the
// same cells from shared memory.  The per-cell flux sums never go to HBM (they did between
// k_flux_cfl and k_transport), and the step's tail is one launch instead of two.
#pragma once
#include "lrbms_kernels.cuh"

namespace lrbms {

template <int S0, int S1, int S2>   // compile-time subdomain shape (sx, sy, sz), 0 = runtime
__global__ void __launch_bounds__(512) k_flux_transport(FluxArgs A, int kmax) {
  extern __shared__ double ft_sm[];   // [kmax][n_loc] flux sums of the CTA's subdomains, then [3][n_loc] scratch
  __shared__ double redmin[16];
  cg::grid_group grid = cg::this_grid();
  const Geo& g = A.g;
  const int s0 = S0 ? S0 : g.s[0], s1 = S1 ? S1 : g.s[1], s2 = S2 ? S2 : g.s[2];
  const int st1 = s0, st2 = s0 * s1, nl = s0 * s1 * s2;
  const int dim = S0 ? (S2 > 1 ? 3 : 2) : g.dim;
  const int tid = threadIdx.x, nt = blockDim.x, G = gridDim.x;
  double* netk = ft_sm;                                // [kmax][nl]
  double* opos = ft_sm + (size_t)kmax * nl;            // per-subdomain link scratch
  double* oneg = opos + nl;
  double* netl = oneg + nl;
  double mn = INFINITY;

  // ---- phase 1: fluxes, flux sums, Q, the CTA's dt bound.  32-bit cell indices (n < 2^31, checked at
  //      bind); the neighbour across a subdomain side is i +- xo[a]
  const int lst[3] = {1, st1, st2};
  const int sa[3] = {s0, s1, s2};
  int xo[3];
#pragma unroll
  for (int a = 0; a < 3; ++a) xo[a] = g.Estride[a] * nl - (sa[a] - 1) * lst[a];
  int k = 0;
  for (int E = blockIdx.x; E < g.n_s; E += G, ++k) {
    int C[3];
    sub_xyz(g, E, C);
    bool lo[3], hi[3];
#pragma unroll
    for (int a = 0; a < 3; ++a) {
      lo[a] = C[a] > 0;
      hi[a] = C[a] + 1 < g.S[a];
    }
    const int base = E * nl;
    const int q0 = A.L.sub_start[E], q1 = A.L.sub_start[E + 1];
    const bool links = q1 > q0;
    for (int l = tid; l < nl; l += nt) {
      const int c0 = l % s0, c1 = (l / s0) % s1, c2 = l / st2;
      const int cc[3] = {c0, c1, c2};
      const int gl = base + l;
      const double pl = A.p[gl], ll = A.lam[gl], fl = A.fw[gl];
      const double2* fco = A.fc + 3 * gl;
      double pos = 0.0, neg = 0.0, acc = 0.0;
#pragma unroll
      for (int a = 0; a < 3; ++a) {
        if (a >= dim) break;
        // -a face (this cell is T2; F = w (p_lower - p) leaves the lower cell), then the +a face (this
        // cell is T1): the order of k_flux_cfl, so the sums are bitwise those of the two-kernel path
        int nb = -1;
        if (cc[a] > 0) nb = gl - lst[a];
        else if (lo[a]) nb = gl - xo[a];
        if (nb >= 0) {
          const double F = face_w(A.fc[3 * nb + a], A.lam[nb], ll) * (A.p[nb] - pl);
          pos += fmax(-F, 0.0);
          neg += fmax(F, 0.0);
          acc += -(F * (F >= 0.0 ? A.fw[nb] : fl));
        }
        nb = -1;
        if (cc[a] + 1 < sa[a]) nb = gl + lst[a];
        else if (hi[a]) nb = gl + xo[a];
        if (nb >= 0) {
          const double F = face_w(fco[a], ll, A.lam[nb]) * (pl - A.p[nb]);
          pos += fmax(F, 0.0);
          neg += fmax(-F, 0.0);
          acc += F * (F >= 0.0 ? fl : A.fw[nb]);
          if (A.face_flux) {
            const int i = C[0] * s0 + c0, j = C[1] * s1 + c1, kk = C[2] * s2 + c2;
            A.face_flux[face_index(g, i, j, kk, a)] = F;
          }
        }
      }
      if (links) {
        opos[l] = pos;
        oneg[l] = neg;
        netl[l] = acc;
      } else {
        const double Q = fmax(pos, neg);
        if (Q > 0.0) mn = fmin(mn, A.cfl * (A.phiV ? A.phiV[gl] : g.vol) / (A.fpmax * Q));
        if (!(Q == Q)) atomicOr(A.flags, FLAG_NAN);
        netk[k * nl + l] = acc;
      }
    }
    if (links) {   // the subdomain's links in its link order (one thread: deterministic), then Q
      __syncthreads();
      if (tid == 0) {
        for (int q = q0; q < q1; ++q) {
          const int l = A.L.local[q];
          const double F = A.L.gK[q] * A.lam[base + l] * (A.p[base + l] - A.L.p[q]);
          opos[l] += fmax(F, 0.0);
          oneg[l] += fmax(-F, 0.0);
          netl[l] += F * (F >= 0.0 ? A.fw[base + l] : frac_flow(A.f, A.L.s_ext[q]));
          if (A.link_flux) A.link_flux[A.L.orig[q]] = F;
        }
      }
      __syncthreads();
      for (int l = tid; l < nl; l += nt) {
        const double Q = fmax(opos[l], oneg[l]);
        if (Q > 0.0) mn = fmin(mn, A.cfl * (A.phiV ? A.phiV[base + l] : g.vol) / (A.fpmax * Q));
        if (!(Q == Q)) atomicOr(A.flags, FLAG_NAN);
        netk[k * nl + l] = netl[l];
      }
      __syncthreads();   // opos/oneg/netl are reused by the next subdomain with links
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) mn = fmin(mn, __shfl_xor_sync(FULL, mn, o));
  if ((tid & 31) == 0) redmin[tid >> 5] = mn;
  __syncthreads();
  if (tid == 0) {
    double m = INFINITY;
    for (int w = 0; w < (nt >> 5); ++w) m = fmin(m, redmin[w]);
    if (m < INFINITY) atomicMin(A.dt_bits, (unsigned long long)__double_as_longlong(m));
  }
  grid.sync();

  // ---- phase 2: the upwind update of the same cells, and lambda, f_w of s^{n+1}
  double dt = A.dt_fixed;
  if (!(dt > 0.0)) dt = __longlong_as_double((long long)__ldcg(A.dt_bits));
  const double dtv = dt / g.vol;   // (dt / pv) with pv = V when phi = 1, hoisted: the same rounding
  k = 0;
  for (int E = blockIdx.x; E < g.n_s; E += G, ++k) {
    const int base = E * nl;
    for (int l = tid; l < nl; l += nt) {
      const int gl = base + l;
      const double sn = A.s[gl] - (A.phiV ? dt / A.phiV[gl] : dtv) * netk[k * nl + l];
      A.s_out[gl] = sn;
      double lw, lo;
      mobilities(A.f, sn, lw, lo);
      A.lam_out[gl] = lw + lo;
      A.fw_out[gl] = lw / (lw + lo);
      if (!(sn == sn)) atomicOr(A.flags, FLAG_NAN);
    }
  }
  if (blockIdx.x == 0 && tid == 0) {
    if (!(dt < INFINITY)) atomicOr(A.flags, FLAG_NOFLOW);
    *A.t_acc += dt;
    A.t_acc[1] = dt;
    if (A.dt_log) A.dt_log[A.step] = dt;
  }
}

}  // namespace lrbms
