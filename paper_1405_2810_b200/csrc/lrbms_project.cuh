// lrbms_project.cuh -- a1 + a2: mobility, k = 0 SWIP operator and its Galerkin projection onto the
// local reduced bases (def:coarseScalePressure; readings R1-R3, R6).
//
// One CTA (8 warps) per subdomain E:
//   * Phi_E is staged in shared memory with cp.async (rows padded to LD = 4 mod 16 doubles, which
//     makes the m8n8k4 fragment loads bank-conflict free), overlapped with the mobility and face
//     weight evaluation (lambda(s) fused here, never stored);
//   * Y = A_EE Phi_E^T is formed chunk by chunk (64 local cells) by the 5/7-point stencil;
//   * B_EE = Phi_E Y^T on the fp64 tensor cores (mma.sync m8n8k4 f64 -> SASS DMMA), upper 8x8 tiles
//     only, K split over the 8 warps and reduced in a fixed warp order (deterministic), mirrored
//     so that B_EE is exactly symmetric;
//   * B_{E,E+e_a} = -(Phi_E,face diag(w)) Phi_{E+a},face^T, again with DMMA (K = face cells);
//   * r_E = Phi_E^T b_E from the links of E.
#pragma once
#include "lrbms_kernels.cuh"

namespace lrbms {

struct ProjArgs {
  Geo g;
  Flu f;
  Links L;
  const double* s;
  const double* K;
  const double* Phi;
  const double2* fc;   // [n][3] static face coefficients
  const double* lam;   // [n] lambda_t(s^n)
  double* blocks;
  double* rhs;
  int LD, nlp, NP, KC, LDY, nfmax, nfp, LDN;
  int ybuf;  // doubles reserved for the Y / neighbour-face / reduction buffer
};

__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}
__device__ __forceinline__ void cp_async8(void* dst, const void* src) {
  const unsigned d = (unsigned)__cvta_generic_to_shared(dst);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(d), "l"(src));
}
__device__ __forceinline__ void cp_async16(void* dst, const void* src) {
  const unsigned d = (unsigned)__cvta_generic_to_shared(dst);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(d), "l"(src));
}
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;\n" ::); }

// fixed enumeration of the upper 8x8 tile pairs (ti <= tj < 4)
__device__ __forceinline__ int pair_ti(int p) { return p < 4 ? 0 : p < 7 ? 1 : p < 9 ? 2 : 3; }
__device__ __forceinline__ int pair_tj(int p) {
  return p < 4 ? p : p < 7 ? p - 3 : p < 9 ? p - 5 : 3;
}

__global__ void __launch_bounds__(512) k_project(ProjArgs A) {
  extern __shared__ __align__(16) double sm[];
  const Geo& g = A.g;
  const int N = g.N, nl = g.n_loc, E = blockIdx.x, tid = threadIdx.x, nt = blockDim.x;
  const int lane = tid & 31, warp = tid >> 5, nwarp = nt >> 5;
  const int nb1 = 1 + g.dim, LD = A.LD, NP = A.NP, T = NP / 8;
  double* Phs = sm;                               // [NP][LD]
  double* Ys = Phs + (size_t)NP * LD;             // [NP][LDY] | [NP][LDN] | [8][64]
  double* lam = Ys + A.ybuf;                      // [nl]
  double* Kc = lam + nl;                          // [nl]
  double* diag = Kc + nl;                         // [nl]
  double* wp = diag + nl;                         // [3][nl]
  double* wi = wp + 3 * nl;                       // [3][nfmax]
  int* fcell = (int*)(wi + 3 * A.nfmax);          // [nfmax]
  int* nbm = fcell + A.nfmax;                     // [nl] in-subdomain neighbour bits (-x,+x,-y,+y,-z,+z)
  int C[3];
  sub_xyz(g, E, C);
  const size_t base = (size_t)E * nl;

  // 1. stage Phi_E asynchronously (zero padding rows/cols written with plain stores)
  const double* PhiE = A.Phi + (size_t)E * N * nl;
  if ((nl & 1) == 0) {
    const int h = nl >> 1;
    for (int k = warp; k < N; k += nwarp)
      for (int c2 = lane; c2 < h; c2 += 32)
        cp_async16(Phs + (size_t)k * LD + 2 * c2, PhiE + (size_t)k * nl + 2 * c2);
  } else {
    for (int k = warp; k < N; k += nwarp)
      for (int c1 = lane; c1 < nl; c1 += 32) cp_async8(Phs + (size_t)k * LD + c1, PhiE + (size_t)k * nl + c1);
  }
  asm volatile("cp.async.commit_group;\n" ::);
  for (int k = warp; k < NP; k += nwarp)
    for (int c1 = (k < N ? nl : 0) + lane; c1 < LD; c1 += 32) Phs[(size_t)k * LD + c1] = 0.0;

  // 2. a1: own mobilities
  for (int l = tid; l < nl; l += nt) lam[l] = A.lam[base + l];
  __syncthreads();
  // 3. face weights (R2) from the static coefficients: diag_l = sum over all faces of l; wp = weight
  //    to the +a neighbour in E; wi = weight across the +a subdomain side
  for (int l = tid; l < nl; l += nt) {
    int c[3];
    local_xyz(g, l, c);
    const double ll = lam[l];
    double d = 0.0;
    int m = 0;
    for (int a = 0; a < 3; ++a) wp[a * nl + l] = 0.0;
    for (int a = 0; a < g.dim; ++a) {
      if (c[a] > 0) m |= 1 << (2 * a);
      if (c[a] + 1 < g.s[a]) m |= 2 << (2 * a);
    }
    nbm[l] = m;
    for (int a = 0; a < g.dim; ++a) {
      const int st = g.lstride[a];
      // -a neighbour (the lower cell of that face owns its coefficients)
      if (c[a] > 0) {
        d += face_w(A.fc[(base + l - st) * 3 + a], lam[l - st], ll);
      } else if (C[a] > 0) {
        const int nb = neighbour(g, E, C, l, c, a, -1);
        d += face_w(A.fc[(size_t)nb * 3 + a], A.lam[nb], ll);
      }
      // +a neighbour
      if (c[a] + 1 < g.s[a]) {
        const double w = face_w(A.fc[(base + l) * 3 + a], ll, lam[l + st]);
        d += w;
        wp[a * nl + l] = w;
      } else if (C[a] + 1 < g.S[a]) {
        const int nb = neighbour(g, E, C, l, c, a, +1);
        const double w = face_w(A.fc[(base + l) * 3 + a], ll, A.lam[nb]);
        d += w;
        wi[a * A.nfmax + face_pos(g, c, a)] = w;
      }
    }
    diag[l] = d;
  }
  __syncthreads();
  if (tid == 0) {  // links of E (R6), sequential: deterministic
    for (int q = A.L.sub_start[E]; q < A.L.sub_start[E + 1]; ++q) {
      const int l = A.L.local[q];
      diag[l] += A.L.gK[q] * lam[l];
    }
  }
  cp_async_wait_all();
  __syncthreads();

  // 4. B_EE = Phi Y^T, Y = A_EE Phi^T in chunks of KC local cells; DMMA over upper tile pairs
  const int npairs = T * (T + 1) / 2;
  double acc[10][2];
#pragma unroll
  for (int p = 0; p < 10; ++p) acc[p][0] = acc[p][1] = 0.0;
  const int fr = lane >> 2, fc = lane & 3;
  for (int l0 = 0; l0 < A.nlp; l0 += A.KC) {
    const int kc = min(A.KC, A.nlp - l0);
    {  // thread <-> (cell ll of the chunk, row group jg): stencil set up once, then FMA-only rows
      const int ll = tid & 63, jg = tid >> 6, ngr = nt >> 6, l = l0 + ll;
      double wv[6] = {0, 0, 0, 0, 0, 0}, dd = 0.0;
      int off[6] = {0, 0, 0, 0, 0, 0};
      if (l < nl) {
        const int m = nbm[l];
        dd = diag[l];
#pragma unroll
        for (int a = 0; a < 3; ++a) {
          const int st = g.lstride[a];
          if (a < g.dim && (m & (1 << (2 * a)))) { wv[2 * a] = wp[a * nl + l - st]; off[2 * a] = -st; }
          if (a < g.dim && (m & (2 << (2 * a)))) { wv[2 * a + 1] = wp[a * nl + l]; off[2 * a + 1] = st; }
        }
      }
      const int lc = l < nl ? l : 0;
      for (int j = jg; j < NP; j += ngr) {
        const double* ph = Phs + (size_t)j * LD + lc;
        double y = dd * ph[0];
#pragma unroll
        for (int q = 0; q < 6; ++q) y -= wv[q] * ph[off[q]];
        Ys[(size_t)j * A.LDY + ll] = y;
      }
    }
    __syncthreads();
    for (int ks = warp; ks < kc / 4; ks += nwarp) {
      double af[4], bf[4];
#pragma unroll
      for (int t4 = 0; t4 < 4; ++t4) {
        af[t4] = t4 < T ? Phs[(size_t)(8 * t4 + fr) * LD + l0 + 4 * ks + fc] : 0.0;
        bf[t4] = t4 < T ? Ys[(size_t)(8 * t4 + fr) * A.LDY + 4 * ks + fc] : 0.0;
      }
#pragma unroll
      for (int p = 0; p < 10; ++p)
        if (p < 10 && pair_tj(p) < T) dmma(acc[p][0], acc[p][1], af[pair_ti(p)], bf[pair_tj(p)]);
    }
    __syncthreads();
  }
  // deterministic cross-warp reduction, one tile pair at a time; mirror for exact symmetry
  double* BEE = A.blocks + (size_t)E * nb1 * N * N;
  double* red = Ys;  // [nwarp][64]
#pragma unroll
  for (int p = 0; p < 10; ++p) {
    if (pair_tj(p) >= T) continue;
    red[warp * 64 + 2 * lane] = acc[p][0];
    red[warp * 64 + 2 * lane + 1] = acc[p][1];
    __syncthreads();
    if (tid < 64) {
      double v = 0.0;
      for (int w = 0; w < nwarp; ++w) v += red[w * 64 + tid];
      const int r = tid >> 3, cc = tid & 7, ti = pair_ti(p), tj = pair_tj(p);
      const int i = 8 * ti + r, j = 8 * tj + cc;
      if (i < N && j < N && (ti < tj || r <= cc)) {
        BEE[i * N + j] = v;
        BEE[j * N + i] = v;
      }
    }
    __syncthreads();
  }
  (void)npairs;

  // 5. r_E = Phi_E^T b_E, b = sum_L g_L p_L e_L
  if (tid < N) {
    double rr = 0.0;
    for (int q = A.L.sub_start[E]; q < A.L.sub_start[E + 1]; ++q) {
      const int l = A.L.local[q];
      rr += Phs[(size_t)tid * LD + l] * (A.L.gK[q] * lam[l] * A.L.p[q]);
    }
    A.rhs[E * N + tid] = rr;
  }

  // 6. coupling blocks B_{E,E+a}[i][j] = -sum_f w_f Phi_E[i][a_f] Phi_{E+a}[j][b_f]
  double* PhN = Ys;  // [NP][LDN]
  for (int a = 0; a < g.dim; ++a) {
    double* BEN = BEE + (size_t)(1 + a) * N * N;
    if (C[a] + 1 >= g.S[a]) {
      for (int t = tid; t < N * N; t += nt) BEN[t] = 0.0;
      continue;
    }
    const int En = E + g.Estride[a], nf = g.nface[a];
    const double* PhiN = A.Phi + (size_t)En * N * nl;
    for (int f = tid; f < nf; f += nt) fcell[f] = face_cell(g, f, a, g.s[a] - 1);
    __syncthreads();
    const int nshift = (g.s[a] - 1) * g.lstride[a];  // own +a side cell -> neighbour's -a side cell
    const double* wa = wi + a * A.nfmax;
    double* Af = Ys + (size_t)NP * A.LDN;           // [NP][LDN] own face rows scaled by w
    for (int k = warp; k < NP; k += nwarp)
      for (int f = lane; f < A.nfp; f += 32) {
        double* dst = PhN + (size_t)k * A.LDN + f;
        if (k < N && f < nf) cp_async8(dst, PhiN + (size_t)k * nl + fcell[f] - nshift);
        else *dst = 0.0;
        Af[(size_t)k * A.LDN + f] = f < nf ? Phs[(size_t)k * LD + fcell[f]] * wa[f] : 0.0;
      }
    asm volatile("cp.async.commit_group;\n" ::);
    cp_async_wait_all();
    __syncthreads();
    for (int t = warp; t < T * T; t += nwarp) {
      const int ti = t / T, tj = t - ti * T;
      double c0 = 0.0, c1 = 0.0;
      for (int ks = 0; ks < A.nfp / 4; ++ks) {
        const int f = 4 * ks + fc;
        const double av = Af[(size_t)(8 * ti + fr) * A.LDN + f];
        const double bv = PhN[(size_t)(8 * tj + fr) * A.LDN + f];
        dmma(c0, c1, av, bv);
      }
      const int i = 8 * ti + fr, j0 = 8 * tj + 2 * fc;
      if (i < N) {
        if (j0 < N) BEN[i * N + j0] = -c0;
        if (j0 + 1 < N) BEN[i * N + j0 + 1] = -c1;
      }
    }
    __syncthreads();
  }
}

}  // namespace lrbms
