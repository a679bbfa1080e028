// lrbms_k1.cuh -- NEXT-4: the LRBMS online step on the k = 1 SWIP-DG fine space with the
// RT0-flux P1 upwind transport and the Dedner limiter (PAPER.md eq:swipBilP P:295-303 with the penalty
// eq:penaltyParam P:305-310 and the Remark's lambda-free c_F / max(mu_w, mu_n) P:312-320; right-hand
// side P:324-333; eq:velocityDG P:366-377; eq:saturationDG P:389-399 with eq:upwind P:400-417; limiter
// P:419-469; def:coarseScalePressure P:621-631 on the P1 dofs).  Readings A4, A5, A25-A30: DESIGN.md 11.
//
// Dofs per cell T: the coefficients of psi_0 = 1 and psi_a = (x_a - b_{T,a}) / h_a (a = 1..dim), stored
// dof-major [nd][n] (nd = dim + 1) in the internal subdomain-major cell order.  Local bases
// Phi1[E][k][a n_loc + l] (ABI layout).  The reduced system has the block structure of the k = 0 one, so
// the reduced solve (a3: block Cholesky scaling, coarse level, deflated on-chip PCG) is reused unchanged.
//
// Kernels of one step:
//   k1_project   one CTA (8 warps, three per SM) per subdomain: Y = A_EE Phi1_E^T formed chunk by chunk (32 cells x
//                nd dofs) in shared memory from the face coefficients (a table per chunk), B_EE =
//                Phi1_E Y on the fp64 tensor cores (mma.sync m8n8k4 -> DMMA, a warp per 8 x 8 output
//                tile over the whole contraction: no cross-warp reduction, deterministic), then the
//                coupling blocks B_{E,E+e_a} from face chunks the same way, r_E from the links
//   (a3)         launch_solve of lrbms.cu
//   k1_recon     p1 = Phi1_E^T c_E
//   k1_flux      normal fluxes of eq:velocityDG on both faces of every axis per cell (each face with the
//                one expression both its cells evaluate), link fluxes, Q_i, the CFL minimum
//   k1_transport explicit Euler step of eq:saturationDG (two-point Gauss per direction, A30)
//   k1_limit     shock detector, flagging, gradient scales, eq:limiterMain; lambda of the new means
#pragma once
#include "lrbms_kernels.cuh"
#include "lrbms_project.cuh"

namespace lrbms {

constexpr int K1_CH = 32;                          // cells (or faces) per chunk of the projection
constexpr double K1_GP = 0.28867513459481287;      // two-point Gauss abscissa on [-1/2, 1/2] (A30)

struct K1Args {
  Geo g;
  Flu f;
  Links L;
  int nd, LDK, NP;
  double cpm;              // c_F / max(mu_w, mu_n)  (Remark P:316-320)
  double h[3], area[3], hF[3], inv_h2[3];
  double det_scale;        // 1 / (0.08 d sqrt(h_T) |T|)
  const int* l_axis;       // [n_links] (sorted link order) axis of the Dirichlet face
  const int* l_side;       // [n_links] -1: lower face of the cell, +1: upper face (A29)
  const double* l_c1;      // [n_links] sigma_F |F| / h_F with sigma_F = cpm K_cell
  const double* l_kl;      // [n_links] K_cell |F| / h_a
  const int* lfirst;       // [n] first link of the cell in the sorted order, -1: none
  const double* K;         // [n] permeability (internal order)
  const double* phiV;      // phi V or nullptr
  const double* Phi1;      // [n_s][N][nd n_loc]
  const double2* fk;       // [n][3]: (sigma_F |F| / h_F, kappa |F| / h_a) of the +a face, (0, 0): none
  const double* lam;       // [n] lambda_t(mean s^n)  (A25)
  double* lam_out;
  const double* s1;        // [nd][n] s^n
  double* sbar;            // [nd][n] after the transport, before the limiter
  double* s1_out;          // [nd][n] s^{n+1}
  double* p1;              // [nd][n]
  const double* c;         // [n_s][N]
  double* Fhi;             // [3][n] flux through the +a face of the cell, in the +a direction
  double* Flo;             // [3][n] flux through the -a face, in the +a direction
  double* Flink;           // [n_links] outward link fluxes (sorted order)
  double* blocks;
  double* rhs;
  unsigned long long* dt_bits;
  double* t_acc;
  double* dt_log;
  int* flags;
  int* nflag;              // number of cells the limiter flagged in the last step
  double cfl, fpmax, dt_fixed;
  int step, limiter;
};

// ------------------------------------------------------------------ static coefficients (set_basis)
__global__ void k1_face_coef(K1Args A, const double* __restrict__ K, double2* __restrict__ fk) {
  const Geo& g = A.g;
  const int idx = blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= g.n) return;
  const int E = idx / g.n_loc, l = idx % g.n_loc;
  int C[3], c[3];
  sub_xyz(g, E, C);
  local_xyz(g, l, c);
  for (int a = 0; a < 3; ++a) {
    double2 v = make_double2(0.0, 0.0);
    if (a < g.dim) {
      const int nb = neighbour(g, E, C, l, c, a, +1);
      if (nb >= 0) {
        const double Ka = K[idx], Kb = K[nb];
        const double sig = A.cpm * 2.0 * Ka * Kb / (Ka + Kb);
        const double kap = Ka * Kb / (Ka + Kb);   // omega_1 K_1 = omega_2 K_2 (A26)
        v = make_double2(sig / A.hF[a] * A.area[a], kap * A.area[a] / A.h[a]);
      }
    }
    fk[(size_t)idx * 3 + a] = v;
  }
}
__global__ void k1_link_coef(K1Args A, const double* __restrict__ K, double* __restrict__ c1, double* __restrict__ kl,
                             int* __restrict__ lfirst) {
  const Geo& g = A.g;
  const int E = blockIdx.x * blockDim.x + threadIdx.x;
  if (E >= g.n_s) return;
  const int q0 = A.L.sub_start[E], q1 = A.L.sub_start[E + 1];
  for (int q = q0; q < q1; ++q) {
    const int l = A.L.local[q], a = A.l_axis[q];
    const double Kc = K[(size_t)E * g.n_loc + l];
    c1[q] = A.cpm * Kc / A.hF[a] * A.area[a];
    kl[q] = Kc * A.area[a] / A.h[a];
    if (q == q0 || A.L.local[q - 1] != l) lfirst[(size_t)E * g.n_loc + l] = q;
  }
}
// coefficients of the subdomain indicator (mean dofs 1, slopes 0) in the local basis
__global__ void k1_indicator(Geo g, int nd, const double* __restrict__ Phi1, double* __restrict__ zc) {
  const int E = blockIdx.x;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  for (int k = warp; k < g.N; k += nw) {
    const double* row = Phi1 + ((size_t)E * g.N + k) * nd * g.n_loc;
    double acc = 0.0;
    for (int l = lane; l < g.n_loc; l += 32) acc += row[l];
    acc = warp_sum(acc);
    if (lane == 0) zc[E * g.N + k] = acc;
  }
}
__global__ void k1_mobility(K1Args A) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= A.g.n) return;
  A.lam_out[i] = total_mobility(A.f, A.s1[i]);
}

// ------------------------------------------------------------------ a2 on the P1 dofs
// One face of eq:swipBilP seen from cell `own` (dofs v) with the cell across it (dofs w, zero when the
// cell lies outside the subdomain: the diagonal block keeps the own-side terms only).  up: own is the
// lower cell T1 of the face.  Adds the face's rows of A v to y.
__device__ __forceinline__ void k1_face_rows(int nd, int ax, bool up, double c1, double ko, double kn,
                                             const double (&v)[4], const double (&w)[4], double (&y)[4]) {
  // [v] at the face centre and the flux mean, both oriented T1 -> T2
  const double j0 = up ? (v[0] + 0.5 * v[1 + ax] - w[0] + 0.5 * w[1 + ax])
                       : (w[0] + 0.5 * w[1 + ax] - v[0] + 0.5 * v[1 + ax]);
  const double DN = ko * v[1 + ax] + kn * w[1 + ax];
  const double G = c1 * j0 - DN;
  y[0] += up ? G : -G;
  y[1 + ax] += 0.5 * G - ko * j0;
  const double c2 = c1 * (1.0 / 12.0);
#pragma unroll
  for (int t = 0; t < 3; ++t)
    if (t != ax && 1 + t < nd) y[1 + t] += c2 * (v[1 + t] - w[1 + t]);
}

__global__ void __launch_bounds__(256, 3) k1_project(K1Args A) {
  extern __shared__ __align__(16) double sm[];
  const Geo& g = A.g;
  const int N = g.N, nl = g.n_loc, nd = A.nd, E = blockIdx.x, tid = threadIdx.x, nt = blockDim.x;
  const int lane = tid & 31, warp = tid >> 5;
  const int LDK = A.LDK, NP = A.NP, T = NP / 8, KD = nd * K1_CH;
  double* Ps = sm;                                  // [NP][LDK] Phi1 chunk (A operand)
  double* Ys = Ps + (size_t)NP * LDK;               // [NP][LDK] (A Phi1^T) chunk (B operand)
  double* tc1 = Ys + (size_t)NP * LDK;              // [CH][6]
  double* tko = tc1 + K1_CH * 6;
  double* tkn = tko + K1_CH * 6;
  double* tvol = tkn + K1_CH * 6;                   // [CH] lambda K |T|
  int* tnb = (int*)(tvol + K1_CH);                  // [CH][6] local neighbour, -1: outside E, -2: no face
  int* tl = tnb + K1_CH * 6;                        // [CH] first link of the cell / own face cell
  int* tl2 = tl + K1_CH;                            // [CH] neighbour face cell (couplings)
  int C[3];
  sub_xyz(g, E, C);
  const size_t base = (size_t)E * nl;
  const size_t rowlen = (size_t)nd * nl;
  const double* PE = A.Phi1 + (size_t)E * N * rowlen;
  const int lq0 = A.L.sub_start[E], lq1 = A.L.sub_start[E + 1];
  const int fr = lane >> 2, fc = lane & 3;
  double* BEE = A.blocks + (size_t)E * (1 + g.dim) * N * N;

  // ---- B_EE: chunks of K1_CH cells; warp w owns the upper tile pairs w and w + 8 (10 pairs, 8 warps)
  bool pair_live[2];
  int pti[2], ptj[2];
#pragma unroll
  for (int q = 0; q < 2; ++q) {
    const int pr = warp + 8 * q;
    pair_live[q] = pr < 10 && pair_tj(pr) < T;
    pti[q] = pair_ti(pr < 10 ? pr : 0);
    ptj[q] = pair_tj(pr < 10 ? pr : 0);
  }
  double acc[2][2] = {{0.0, 0.0}, {0.0, 0.0}};
  for (int l0 = 0; l0 < nl; l0 += K1_CH) {
    __syncthreads();
    for (int u = tid; u < K1_CH * 6; u += nt) {
      const int lc = u / 6, d = u - 6 * lc, a = d >> 1, up = d & 1, l = l0 + lc;
      int nbv = -2;
      double c1 = 0.0, ko = 0.0, kn = 0.0;
      if (a < g.dim && l < nl) {
        int c[3];
        local_xyz(g, l, c);
        const int nbg = neighbour(g, E, C, l, c, a, up ? +1 : -1);
        if (nbg >= 0) {
          const int nc = c[a] + (up ? 1 : -1);
          nbv = (nc >= 0 && nc < g.s[a]) ? (int)(nbg - base) : -1;
          const double2 k = A.fk[(up ? base + l : (size_t)nbg) * 3 + a];
          c1 = k.x;
          ko = k.y * A.lam[base + l];
          kn = k.y * A.lam[nbg];
        }
      }
      tnb[u] = nbv; tc1[u] = c1; tko[u] = ko; tkn[u] = kn;
    }
    for (int lc = tid; lc < K1_CH; lc += nt) {
      const int l = l0 + lc;
      tvol[lc] = l < nl ? A.lam[base + l] * A.K[base + l] * g.vol : 0.0;
      tl[lc] = l < nl ? A.lfirst[base + l] : -1;
    }
    __syncthreads();
    // pass A: the chunk's own dofs (coalesced) -> Ps
    for (int u = tid; u < NP * K1_CH; u += nt) {
      const int m = u / K1_CH, lc = u - m * K1_CH, l = l0 + lc;
      const bool live = m < N && l < nl;
      const double* pm = PE + (size_t)m * rowlen + l;
#pragma unroll
      for (int a = 0; a < 4; ++a)
        if (a < nd) Ps[(size_t)m * LDK + a * K1_CH + lc] = live ? pm[(size_t)a * nl] : 0.0;
    }
    __syncthreads();
    // pass B: the rows of A_EE Phi1^T; neighbours inside the chunk come from Ps, the others from L1/L2
    for (int u = tid; u < NP * K1_CH; u += nt) {
      const int m = u / K1_CH, lc = u - m * K1_CH, l = l0 + lc;
      double v[4] = {0.0, 0.0, 0.0, 0.0}, y[4] = {0.0, 0.0, 0.0, 0.0};
      if (m < N && l < nl) {
        const double* pm = PE + (size_t)m * rowlen;
        const double* ps = Ps + (size_t)m * LDK;
#pragma unroll
        for (int a = 0; a < 4; ++a)
          if (a < nd) v[a] = ps[a * K1_CH + lc];
#pragma unroll
        for (int d = 0; d < 6; ++d) {
          const int nbv = tnb[lc * 6 + d];
          if (nbv == -2) continue;
          double w[4] = {0.0, 0.0, 0.0, 0.0};
          if (nbv >= 0) {
            const int nc = nbv - l0;
            if (nc >= 0 && nc < K1_CH) {
#pragma unroll
              for (int a = 0; a < 4; ++a)
                if (a < nd) w[a] = ps[a * K1_CH + nc];
            } else {
#pragma unroll
              for (int a = 0; a < 4; ++a)
                if (a < nd) w[a] = pm[(size_t)a * nl + nbv];
            }
          }
          k1_face_rows(nd, d >> 1, d & 1, tc1[lc * 6 + d], tko[lc * 6 + d], tkn[lc * 6 + d], v, w, y);
        }
        const double vol = tvol[lc];
#pragma unroll
        for (int a = 1; a < 4; ++a)
          if (a < nd) y[a] += vol * A.inv_h2[a - 1] * v[a];
        // Dirichlet faces of the cell (links, A29): the one-sided face terms
        for (int q = tl[lc]; q >= 0 && q < lq1 && A.L.local[q] == l; ++q) {
          const int axq = A.l_axis[q];
          const double sg = (double)A.l_side[q], c1 = A.l_c1[q], kl = A.l_kl[q] * A.lam[base + l];
#pragma unroll
          for (int ax = 0; ax < 3; ++ax) {   // compile-time dof indices
            if (ax != axq) continue;
            const double j0 = v[0] + 0.5 * sg * v[1 + ax];
            const double DN = kl * sg * v[1 + ax];
            const double G = c1 * j0 - DN;
            y[0] += G;
            y[1 + ax] += 0.5 * sg * G - kl * sg * j0;
#pragma unroll
            for (int t = 0; t < 3; ++t)
              if (t != ax && 1 + t < nd) y[1 + t] += c1 * (1.0 / 12.0) * v[1 + t];
          }
        }
      }
#pragma unroll
      for (int a = 0; a < 4; ++a)
        if (a < nd) Ys[(size_t)m * LDK + a * K1_CH + lc] = y[a];
    }
    __syncthreads();
#pragma unroll
    for (int q = 0; q < 2; ++q)
      if (pair_live[q]) {
        const double* pa = Ps + (size_t)(8 * pti[q] + fr) * LDK + fc;
        const double* pb = Ys + (size_t)(8 * ptj[q] + fr) * LDK + fc;
        for (int ks = 0; ks < KD; ks += 4) dmma(acc[q][0], acc[q][1], pa[ks], pb[ks]);
      }
  }
#pragma unroll
  for (int q = 0; q < 2; ++q)
    if (pair_live[q]) {   // upper tile pairs, mirrored: B_EE exactly symmetric
#pragma unroll
      for (int hh = 0; hh < 2; ++hh) {
        const int cl = 2 * fc + hh, i = 8 * pti[q] + fr, j = 8 * ptj[q] + cl;
        const double val = acc[q][hh];
        if (i < N && j < N && (pti[q] < ptj[q] || fr <= cl)) {
          BEE[i * N + j] = val;
          BEE[j * N + i] = val;
        }
      }
    }

  // ---- r_E = Phi1_E b_E: b(w) = sum_{F in Gamma_D} int_F (sigma_F / h_F w - lambda K grad w . n) p_D
  if (tid < N) {
    const double* pm = PE + (size_t)tid * rowlen;
    double rr = 0.0;
    for (int q = lq0; q < lq1; ++q) {
      const int l = A.L.local[q], ax = A.l_axis[q];
      const double sg = (double)A.l_side[q], c1 = A.l_c1[q], kl = A.l_kl[q] * A.lam[base + l], pD = A.L.p[q];
      rr += pm[l] * (c1 * pD) + pm[(size_t)(1 + ax) * nl + l] * (0.5 * sg * c1 * pD - kl * sg * pD);
    }
    A.rhs[E * N + tid] = rr;
  }

  // ---- couplings B_{E,E+e_a}[i][j] = Phi1_E[i] . A_{E,E+a} Phi1_{E+a}[j]: chunks of K1_CH faces
  bool tile_live[2];
  int ti[2], tj[2];
#pragma unroll
  for (int q = 0; q < 2; ++q) {
    const int tt = warp + 8 * q;
    tile_live[q] = tt < T * T;
    ti[q] = tile_live[q] ? tt / T : 0;
    tj[q] = tile_live[q] ? tt - (tt / T) * T : 0;
  }
  for (int a = 0; a < g.dim; ++a) {
    double* BEN = BEE + (size_t)(1 + a) * N * N;
    if (C[a] + 1 >= g.S[a]) {
      for (int o = tid; o < N * N; o += nt) BEN[o] = 0.0;
      continue;
    }
    const int nf = g.nface[a];
    const size_t baseN = (size_t)(E + g.Estride[a]) * nl;
    const double* PN = A.Phi1 + (size_t)(E + g.Estride[a]) * N * rowlen;
    double cc[2][2] = {{0.0, 0.0}, {0.0, 0.0}};
    for (int f0 = 0; f0 < nf; f0 += K1_CH) {
      __syncthreads();
      for (int lc = tid; lc < K1_CH; lc += nt) {
        const int f = f0 + lc;
        int la = 0, lb = 0;
        double c1 = 0.0, ko = 0.0, kn = 0.0;
        if (f < nf) {
          la = face_cell(g, f, a, g.s[a] - 1);
          lb = face_cell(g, f, a, 0);
          const double2 k = A.fk[(base + la) * 3 + a];
          c1 = k.x;
          ko = k.y * A.lam[base + la];
          kn = k.y * A.lam[baseN + lb];
        }
        tl[lc] = la; tl2[lc] = lb; tc1[lc] = c1; tko[lc] = ko; tkn[lc] = kn;
      }
      __syncthreads();
      for (int u = tid; u < NP * K1_CH; u += nt) {
        const int m = u / K1_CH, lc = u - m * K1_CH, f = f0 + lc;
        double v[4] = {0.0, 0.0, 0.0, 0.0}, w[4] = {0.0, 0.0, 0.0, 0.0}, y[4] = {0.0, 0.0, 0.0, 0.0};
        if (m < N && f < nf) {
          const double* pm = PE + (size_t)m * rowlen + tl[lc];
          const double* pn = PN + (size_t)m * rowlen + tl2[lc];
#pragma unroll
          for (int q = 0; q < 4; ++q)
            if (q < nd) { v[q] = pm[(size_t)q * nl]; w[q] = pn[(size_t)q * nl]; }
          // rows of the own cell (T1) for a function supported on the upper cell (T2) only
          const double zero[4] = {0.0, 0.0, 0.0, 0.0};
          if (a == 0) k1_face_rows(nd, 0, true, tc1[lc], tko[lc], tkn[lc], zero, w, y);   // compile-time dof indices
          else if (a == 1) k1_face_rows(nd, 1, true, tc1[lc], tko[lc], tkn[lc], zero, w, y);
          else k1_face_rows(nd, 2, true, tc1[lc], tko[lc], tkn[lc], zero, w, y);
        }
#pragma unroll
        for (int q = 0; q < 4; ++q)
          if (q < nd) {
            Ps[(size_t)m * LDK + q * K1_CH + lc] = v[q];
            Ys[(size_t)m * LDK + q * K1_CH + lc] = y[q];
          }
      }
      __syncthreads();
#pragma unroll
      for (int q = 0; q < 2; ++q)
        if (tile_live[q]) {
          const double* pa = Ps + (size_t)(8 * ti[q] + fr) * LDK + fc;
          const double* pb = Ys + (size_t)(8 * tj[q] + fr) * LDK + fc;
          for (int ks = 0; ks < KD; ks += 4) dmma(cc[q][0], cc[q][1], pa[ks], pb[ks]);
        }
    }
#pragma unroll
    for (int q = 0; q < 2; ++q)
      if (tile_live[q]) {
        const int i = 8 * ti[q] + fr, j = 8 * tj[q] + 2 * fc;
        if (i < N && j < N) BEN[i * N + j] = cc[q][0];
        if (i < N && j + 1 < N) BEN[i * N + j + 1] = cc[q][1];
      }
  }
}

// ------------------------------------------------------------------ a4: p1 = Phi1_E^T c_E
__global__ void __launch_bounds__(256) k1_recon(K1Args A) {
  __shared__ double cs[32];
  const Geo& g = A.g;
  const int E = blockIdx.x, N = g.N, nl = g.n_loc, nd = A.nd;
  if (threadIdx.x < N) cs[threadIdx.x] = A.c[E * N + threadIdx.x];
  __syncthreads();
  const size_t rowlen = (size_t)nd * nl;
  const double* PE = A.Phi1 + (size_t)E * N * rowlen;
  for (int idx = threadIdx.x; idx < nd * nl; idx += blockDim.x) {
    double acc = 0.0;
    for (int k = 0; k < N; ++k) acc = fma(PE[(size_t)k * rowlen + idx], cs[k], acc);
    const int a = idx / nl, l = idx - a * nl;
    A.p1[(size_t)a * g.n + (size_t)E * nl + l] = acc;
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) *A.dt_bits = 0x7ff0000000000000ull;   // +inf: the CFL minimum
}

// ------------------------------------------------------------------ a5: eq:velocityDG normal fluxes
// flux through the face between ga (lower cell T1) and gb = ga + e_ax (T2), in the +ax direction:
// int_F -{lambda K grad p . n} + sigma_F / h_F [p]
__device__ __forceinline__ double k1_face_flux(const K1Args& A, size_t ga, size_t gb, int ax) {
  const size_t n = A.g.n;
  const double2 k = A.fk[ga * 3 + ax];
  const double pa0 = A.p1[ga], pax = A.p1[(size_t)(1 + ax) * n + ga];
  const double pb0 = A.p1[gb], pbx = A.p1[(size_t)(1 + ax) * n + gb];
  const double jump = pa0 + 0.5 * pax - pb0 + 0.5 * pbx;
  return k.x * jump - k.y * (A.lam[ga] * pax + A.lam[gb] * pbx);
}

__global__ void __launch_bounds__(256) k1_flux(K1Args A) {
  const Geo& g = A.g;
  const int E = blockIdx.x, nl = g.n_loc;
  __shared__ double redmin[8];
  int C[3];
  sub_xyz(g, E, C);
  const size_t base = (size_t)E * nl, n = g.n;
  const int q1 = A.L.sub_start[E + 1];
  double mn = INFINITY;
  for (int l = threadIdx.x; l < nl; l += blockDim.x) {
    int c[3];
    local_xyz(g, l, c);
    const size_t gi = base + l;
    double pos = 0.0, neg = 0.0;
    for (int a = 0; a < 3; ++a) {
      double fhi = 0.0, flo = 0.0;
      if (a < g.dim) {
        const int nu = neighbour(g, E, C, l, c, a, +1), nlw = neighbour(g, E, C, l, c, a, -1);
        if (nu >= 0) fhi = k1_face_flux(A, gi, (size_t)nu, a);
        if (nlw >= 0) flo = k1_face_flux(A, (size_t)nlw, gi, a);
      }
      A.Fhi[(size_t)a * n + gi] = fhi;
      A.Flo[(size_t)a * n + gi] = flo;
      pos += fmax(fhi, 0.0) + fmax(-flo, 0.0);
      neg += fmax(-fhi, 0.0) + fmax(flo, 0.0);
    }
    for (int q = A.lfirst[gi]; q >= 0 && q < q1 && A.L.local[q] == l; ++q) {
      const int ax = A.l_axis[q];
      const double sg = (double)A.l_side[q];
      const double p0 = A.p1[gi], px = A.p1[(size_t)(1 + ax) * n + gi];
      const double F = A.l_c1[q] * (p0 + 0.5 * sg * px - A.L.p[q]) - A.l_kl[q] * A.lam[gi] * sg * px;
      A.Flink[q] = F;
      if (sg > 0) A.Fhi[(size_t)ax * n + gi] = F;
      else A.Flo[(size_t)ax * n + gi] = -F;
      pos += fmax(F, 0.0);
      neg += fmax(-F, 0.0);
    }
    const double Q = fmax(pos, neg);
    if (Q > 0.0) {
      const double pv = A.phiV ? A.phiV[gi] : g.vol;
      mn = fmin(mn, A.cfl * pv / (A.fpmax * Q));
    }
    if (!(Q == Q)) atomicOr(A.flags, FLAG_NAN);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) mn = fmin(mn, __shfl_xor_sync(FULL, mn, o));
  if ((threadIdx.x & 31) == 0) redmin[threadIdx.x >> 5] = mn;
  __syncthreads();
  if (threadIdx.x == 0) {
    double m = INFINITY;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) m = fmin(m, redmin[w]);
    if (m < INFINITY) atomicMin(A.dt_bits, (unsigned long long)__double_as_longlong(m));
  }
}

// ------------------------------------------------------------------ a6: eq:saturationDG at k = 1
// value of the P1 function (dofs s) on the face of axis ax, side sd (+-1), at tangential offsets x
__device__ __forceinline__ double k1_trace(int nd, const double (&s)[4], int ax, double sd, const double (&x)[3]) {
  double v = s[0] + 0.5 * sd * s[1 + ax];
#pragma unroll
  for (int t = 0; t < 3; ++t)
    if (t != ax && 1 + t < nd) v += s[1 + t] * x[t];
  return v;
}
__device__ __forceinline__ void k1_load(const K1Args& A, const double* s1, size_t gi, double (&s)[4]) {
#pragma unroll
  for (int a = 0; a < 4; ++a) s[a] = a < A.nd ? s1[(size_t)a * A.g.n + gi] : 0.0;
}

__global__ void __launch_bounds__(256) k1_transport(K1Args A) {
  const Geo& g = A.g;
  const int E = blockIdx.x, nl = g.n_loc, nd = A.nd, dim = g.dim;
  double dt = A.dt_fixed;
  if (!(dt > 0.0)) dt = __longlong_as_double((long long)*((volatile unsigned long long*)A.dt_bits));
  int C[3];
  sub_xyz(g, E, C);
  const size_t base = (size_t)E * nl, n = g.n;
  const int q1 = A.L.sub_start[E + 1];
  const int ntp = dim == 3 ? 4 : 2;          // tangential Gauss points per face
  const double wf = 1.0 / ntp;
  for (int l = threadIdx.x; l < nl; l += blockDim.x) {
    int c[3];
    local_xyz(g, l, c);
    const size_t gi = base + l;
    double s[4], R[4] = {0.0, 0.0, 0.0, 0.0};
    k1_load(A, A.s1, gi, s);
    double Fl_[3], Fh_[3];
#pragma unroll
    for (int a = 0; a < 3; ++a) {
      Fl_[a] = a < dim ? A.Flo[(size_t)a * n + gi] : 0.0;
      Fh_[a] = a < dim ? A.Fhi[(size_t)a * n + gi] : 0.0;
    }
    // volume term: int_T u f(s) . grad psi_a, u_a linear in xi_a between the two face fluxes (RT0)
    const int nvp = 1 << dim;
    const double wv = g.vol / nvp;
    for (int q = 0; q < nvp; ++q) {
      double x[3] = {0.0, 0.0, 0.0};
      double sv = s[0];
#pragma unroll
      for (int d = 0; d < 3; ++d)
        if (d < dim) {
          x[d] = ((q >> (dim - 1 - d)) & 1) ? K1_GP : -K1_GP;
          sv += s[1 + d] * x[d];
        }
      const double fv = frac_flow(A.f, sv);
#pragma unroll
      for (int a = 0; a < 3; ++a)
        if (a < dim) {
          const double ua = (Fl_[a] * (0.5 - x[a]) + Fh_[a] * (0.5 + x[a])) / A.area[a];
          R[1 + a] += wv * ua * fv / A.h[a];
        }
    }
    // interior faces (axis and side unrolled: the dof arrays stay in registers)
#pragma unroll
    for (int a = 0; a < 3; ++a) {
      if (a >= dim) continue;
#pragma unroll
      for (int up = 0; up < 2; ++up) {
        const int nb = neighbour(g, E, C, l, c, a, up ? +1 : -1);
        if (nb < 0) continue;
        double w[4];
        k1_load(A, A.s1, (size_t)nb, w);
        const double F = up ? Fh_[a] : Fl_[a];
        for (int q = 0; q < ntp; ++q) {
          double x[3] = {0.0, 0.0, 0.0};
          int bit = ntp >> 1;
#pragma unroll
          for (int t = 0; t < 3; ++t)
            if (t != a && t < dim) {
              x[t] = (q & bit) ? K1_GP : -K1_GP;
              bit >>= 1;
            }
          // T1 = lower cell of the face: s_up = s|T1 if F >= 0 else s|T2 (eq:upwind)
          double su;
          if (up) su = F >= 0.0 ? k1_trace(nd, s, a, +1.0, x) : k1_trace(nd, w, a, -1.0, x);
          else su = F >= 0.0 ? k1_trace(nd, w, a, +1.0, x) : k1_trace(nd, s, a, -1.0, x);
          const double gq = F * wf * frac_flow(A.f, su);
          if (up) {
            R[0] -= gq;
            R[1 + a] -= 0.5 * gq;
#pragma unroll
            for (int t = 0; t < 3; ++t)
              if (t != a && t < dim) R[1 + t] -= gq * x[t];
          } else {
            R[0] += gq;
            R[1 + a] += -0.5 * gq;
#pragma unroll
            for (int t = 0; t < 3; ++t)
              if (t != a && t < dim) R[1 + t] += gq * x[t];
          }
        }
      }
    }
    // Dirichlet faces: n outward; chi = s_D on inflow (F < 0), the cell's trace on outflow
    for (int q = A.lfirst[gi]; q >= 0 && q < q1 && A.L.local[q] == l; ++q) {
      const int aq = A.l_axis[q];
      const double sg = (double)A.l_side[q], F = A.Flink[q];
#pragma unroll
      for (int a = 0; a < 3; ++a) {
        if (a != aq) continue;
        for (int k = 0; k < ntp; ++k) {
          double x[3] = {0.0, 0.0, 0.0};
          int bit = ntp >> 1;
#pragma unroll
          for (int t = 0; t < 3; ++t)
            if (t != a && t < dim) {
              x[t] = (k & bit) ? K1_GP : -K1_GP;
              bit >>= 1;
            }
          const double su = F >= 0.0 ? k1_trace(nd, s, a, sg, x) : A.L.s_ext[q];
          const double gq = F * wf * frac_flow(A.f, su);
          R[0] -= gq;
          R[1 + a] -= 0.5 * sg * gq;
#pragma unroll
          for (int t = 0; t < 3; ++t)
            if (t != a && t < dim) R[1 + t] -= gq * x[t];
        }
      }
    }
    const double pv = A.phiV ? A.phiV[gi] : g.vol;
    bool bad = false;
#pragma unroll
    for (int a = 0; a < 4; ++a)
      if (a < nd) {
        const double mass = a == 0 ? 1.0 : 1.0 / 12.0;
        const double v = s[a] + dt * R[a] / pv / mass;
        A.sbar[(size_t)a * n + gi] = v;
        bad |= !(v == v);
      }
    if (bad) atomicOr(A.flags, FLAG_NAN);
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    if (!(dt < INFINITY)) atomicOr(A.flags, FLAG_NOFLOW);
    *A.t_acc += dt;
    A.t_acc[1] = dt;
    if (A.dt_log) A.dt_log[A.step] = dt;
    *A.nflag = 0;
  }
}

// ------------------------------------------------------------------ limiter
__device__ __forceinline__ double k1_gradient_scale(double gr, double d) {   // m_i of P:449-456
  const bool big = fabs(gr) > 1e-8 && fabs(d) > 1e-8;
  if (gr * d < 0.0 && big) return 0.0;
  if (gr * d > 0.0 && fabs(gr) > fabs(d) && big) return d / gr;
  return 1.0;
}

__global__ void __launch_bounds__(256) k1_limit(K1Args A) {
  const Geo& g = A.g;
  const int E = blockIdx.x, nl = g.n_loc, nd = A.nd, dim = g.dim;
  int C[3];
  sub_xyz(g, E, C);
  const size_t base = (size_t)E * nl, n = g.n;
  const int q1 = A.L.sub_start[E + 1];
  int nfl = 0;
  for (int l = threadIdx.x; l < nl; l += blockDim.x) {
    int c[3];
    local_xyz(g, l, c);
    const size_t gi = base + l;
    double s[4];
    k1_load(A, A.sbar, gi, s);
    double mscale = 1.0;
    if (A.limiter) {
      // shock detector S(T): the jump integrals over the upstream faces (u . n_T < 0) (A27)
      double S = 0.0;
      double nbm[6], nbx[6];
      bool has[6];
#pragma unroll
      for (int a = 0; a < 3; ++a)
#pragma unroll
        for (int up = 0; up < 2; ++up) {
          const int d = 2 * a + up;
          has[d] = false;
          nbm[d] = nbx[d] = 0.0;
          if (a >= dim) continue;
          const int nb = neighbour(g, E, C, l, c, a, up ? +1 : -1);
          has[d] = nb >= 0;
          nbm[d] = nbx[d] = 0.0;
          if (!has[d]) continue;
          nbm[d] = A.sbar[(size_t)nb];
          nbx[d] = A.sbar[(size_t)(1 + a) * n + nb];
          const double F = up ? A.Fhi[(size_t)a * n + gi] : A.Flo[(size_t)a * n + gi];
          // inflow into this cell: through its upper face when F < 0, through its lower face when F > 0
          if (up ? (F < 0.0) : (F > 0.0)) {
            const double jump = up ? fabs((s[0] + 0.5 * s[1 + a]) - (nbm[d] - 0.5 * nbx[d]))
                                   : fabs((nbm[d] + 0.5 * nbx[d]) - (s[0] - 0.5 * s[1 + a]));
            S += A.area[a] * jump * A.det_scale;
          }
        }
      for (int q = A.lfirst[gi]; q >= 0 && q < q1 && A.L.local[q] == l; ++q)
        if (A.Flink[q] < 0.0) {
          const int a = A.l_axis[q];
          const double sg = (double)A.l_side[q];
          const double sl = a == 0 ? s[1] : (a == 1 ? s[2] : s[3]);
          S += A.area[a] * fabs(s[0] + 0.5 * sg * sl - A.L.s_ext[q]) * A.det_scale;
        }
      double spread = 0.0;
#pragma unroll
      for (int a = 1; a < 4; ++a)
        if (a < nd) spread += fabs(s[a]);
      spread *= 0.5;
      const bool flagged = S > 1.0 || s[0] - spread < 0.0 || s[0] + spread > 1.0;
      if (flagged) {
        ++nfl;
#pragma unroll
        for (int a = 0; a < 3; ++a)
#pragma unroll
          for (int up = 0; up < 2; ++up) {
            const int d = 2 * a + up;
            if (!has[d]) continue;
            const double gr = (up ? 1.0 : -1.0) * s[1 + a];
            mscale = fmin(mscale, k1_gradient_scale(gr, nbm[d] - s[0]));
          }
      }
    }
    A.s1_out[gi] = s[0];
#pragma unroll
    for (int a = 1; a < 4; ++a)
      if (a < nd) A.s1_out[(size_t)a * n + gi] = mscale * s[a];
    A.lam_out[gi] = total_mobility(A.f, s[0]);   // a1 of the next step (A25)
  }
  if (nfl) atomicAdd(A.nflag, nfl);
}

}  // namespace lrbms
