// lrbms_project.cuh -- a1 + a2: mobility, k = 0 SWIP operator and its Galerkin projection onto the
// local reduced bases (def:coarseScalePressure; readings R1-R3, R6).
//
// One CTA (16 warps) per subdomain E:
//   * Phi_E and the three neighbour face slabs Phi_{E+e_a}|face are staged in shared memory with
//     cp.async at entry (rows padded to LD = 4 mod 16 doubles: conflict-free m8n8k4 fragment loads),
//     overlapped with the face-weight evaluation (lambda(s) read from the step-start array);
//   * B_EE = Phi_E A_EE Phi_E^T on the fp64 tensor cores (mma.sync m8n8k4 f64 -> SASS DMMA): every
//     warp owns a strided set of 4-cell k-steps and forms its B-operand fragments Y = A_EE Phi^T
//     directly in registers from the 5/7-point stencil (no Y buffer, no CTA barrier in the loop);
//     upper 8x8 tile pairs only, reduced over the warps in a fixed order (deterministic), mirrored so
//     that B_EE is exactly symmetric;
//   * B_{E,E+e_a} = -(Phi_E,face diag(w)) Phi_{E+a},face^T, again DMMA, from the staged slabs;
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
  int LD, nlp, NP, nfmax, nfp, LDN;
  int nwc;             // doubles of the per-cell weight table (>= 8 n_loc, >= 16 x 64 for the reduction)
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
  const int nb1 = 1 + g.dim, LD = A.LD, NP = A.NP, T = NP / 8, nfp = A.nfp, LDN = A.LDN;
  double* Phs = sm;                               // [NP][LD]
  double* Wc = Phs + (size_t)NP * LD;             // [nl][8] {diag, w-x, w+x, w-y, w+y, w-z, w+z, 0} | [16][64]
  double* PhN = Wc + A.nwc;                       // [3][NP][LDN] neighbour face slabs
  double* lam = PhN + (size_t)3 * NP * LDN;       // [nl] (rounded up to even)
  double* wi = lam + ((nl + 1) & ~1);             // [3][nfp] weights across the +a side
  int* fcell = (int*)(wi + 3 * nfp);              // [3][nfp] own local cell at face f of the +a side
  int C[3];
  sub_xyz(g, E, C);
  const size_t base = (size_t)E * nl;

  // 1. stage Phi_E and the neighbour face slabs asynchronously (padding with plain stores)
  const double* PhiE = A.Phi + (size_t)E * N * nl;
  if ((nl & 1) == 0) {
    const int h = nl >> 1;
    for (int t = tid; t < N * h; t += nt) {
      const int k = t / h, c2 = t - k * h;
      cp_async16(Phs + (size_t)k * LD + 2 * c2, PhiE + (size_t)k * nl + 2 * c2);
    }
  } else {
    for (int t = tid; t < N * nl; t += nt) {
      const int k = t / nl, c1 = t - k * nl;
      cp_async8(Phs + (size_t)k * LD + c1, PhiE + (size_t)k * nl + c1);
    }
  }
  for (int k = warp; k < NP; k += nwarp)
    for (int c1 = (k < N ? nl : 0) + lane; c1 < LD; c1 += 32) Phs[(size_t)k * LD + c1] = 0.0;
  for (int a = 0; a < 3; ++a) {
    const bool has = a < g.dim && C[a] + 1 < g.S[a];
    const int nf = a < g.dim ? g.nface[a] : 0;
    const double* PhiN = A.Phi + (size_t)(E + (has ? g.Estride[a] : 0)) * N * nl;
    double* dst = PhN + (size_t)a * NP * LDN;
    for (int t = tid; t < NP * LDN; t += nt) {
      const int k = t / LDN, f = t - k * LDN;
      if (has && k < N && f < nf) cp_async8(dst + t, PhiN + (size_t)k * nl + face_cell(g, f, a, 0));
      else dst[t] = 0.0;
    }
    for (int f = tid; f < nfp; f += nt) {
      fcell[a * nfp + f] = (f < nf) ? face_cell(g, f, a, g.s[a] - 1) : 0;
      wi[a * nfp + f] = 0.0;
    }
  }
  asm volatile("cp.async.commit_group;\n" ::);

  // 2. a1 + face weights (R2) from the static coefficients
  for (int l = tid; l < nl; l += nt) lam[l] = A.lam[base + l];
  __syncthreads();
  for (int l = tid; l < nl; l += nt) {
    int c[3];
    local_xyz(g, l, c);
    const double ll = lam[l];
    double d = 0.0, w[6] = {0, 0, 0, 0, 0, 0};
#pragma unroll
    for (int a = 0; a < 3; ++a) {
      if (a >= g.dim) break;
      const int st = g.lstride[a];
      if (c[a] > 0) {   // the lower cell of a face owns its coefficients
        w[2 * a] = face_w(A.fc[(base + l - st) * 3 + a], lam[l - st], ll);
        d += w[2 * a];
      } else if (C[a] > 0) {
        const int nb = neighbour(g, E, C, l, c, a, -1);
        d += face_w(A.fc[(size_t)nb * 3 + a], A.lam[nb], ll);
      }
      if (c[a] + 1 < g.s[a]) {
        w[2 * a + 1] = face_w(A.fc[(base + l) * 3 + a], ll, lam[l + st]);
        d += w[2 * a + 1];
      } else if (C[a] + 1 < g.S[a]) {
        const int nb = neighbour(g, E, C, l, c, a, +1);
        const double wv = face_w(A.fc[(base + l) * 3 + a], ll, A.lam[nb]);
        d += wv;
        wi[a * nfp + face_pos(g, c, a)] = wv;
      }
    }
    double2* wc2 = reinterpret_cast<double2*>(Wc + (size_t)l * 8);
    wc2[0] = make_double2(d, w[0]);
    wc2[1] = make_double2(w[1], w[2]);
    wc2[2] = make_double2(w[3], w[4]);
    wc2[3] = make_double2(w[5], 0.0);
  }
  __syncthreads();
  if (tid == 0) {  // links of E (R6), sequential: deterministic
    for (int q = A.L.sub_start[E]; q < A.L.sub_start[E + 1]; ++q) {
      const int l = A.L.local[q];
      Wc[(size_t)l * 8] += A.L.gK[q] * lam[l];
    }
  }
  asm volatile("cp.async.wait_all;\n" ::);
  __syncthreads();

  // 3. B_EE = Phi Y^T with Y = A_EE Phi^T formed in registers; warp-strided k-steps of 4 cells
  double acc[10][2];
#pragma unroll
  for (int p = 0; p < 10; ++p) acc[p][0] = acc[p][1] = 0.0;
  const int fr = lane >> 2, fc = lane & 3;
  const int st0 = g.lstride[0], st1 = g.lstride[1], st2 = g.lstride[2];
  for (int ks = warp; ks < A.nlp / 4; ks += nwarp) {
    const int l = 4 * ks + fc;
    double wv[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    if (l < nl) {
      const double2* wc2 = reinterpret_cast<const double2*>(Wc + (size_t)l * 8);
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const double2 v = wc2[q];
        wv[2 * q] = v.x;
        wv[2 * q + 1] = v.y;
      }
    }
    const int i1 = wv[1] != 0.0 ? l - st0 : l, i2 = wv[2] != 0.0 ? l + st0 : l;
    const int i3 = wv[3] != 0.0 ? l - st1 : l, i4 = wv[4] != 0.0 ? l + st1 : l;
    const int i5 = wv[5] != 0.0 ? l - st2 : l, i6 = wv[6] != 0.0 ? l + st2 : l;
    double af[4], bf[4];
#pragma unroll
    for (int t4 = 0; t4 < 4; ++t4) {
      af[t4] = bf[t4] = 0.0;
      if (t4 < T) {
        const double* ph = Phs + (size_t)(8 * t4 + fr) * LD;
        const double cv = ph[l];
        double y = wv[0] * cv;
        y = fma(-wv[1], ph[i1], y);
        y = fma(-wv[2], ph[i2], y);
        y = fma(-wv[3], ph[i3], y);
        y = fma(-wv[4], ph[i4], y);
        y = fma(-wv[5], ph[i5], y);
        y = fma(-wv[6], ph[i6], y);
        af[t4] = cv;
        bf[t4] = y;
      }
    }
#pragma unroll
    for (int p = 0; p < 10; ++p)
      if (pair_tj(p) < T) dmma(acc[p][0], acc[p][1], af[pair_ti(p)], bf[pair_tj(p)]);
  }
  // deterministic cross-warp reduction, one tile pair at a time; mirror for exact symmetry
  double* BEE = A.blocks + (size_t)E * nb1 * N * N;
  double* red = Wc;  // [nwarp][64]
  __syncthreads();   // every warp is done with the weight table
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

  // 4. r_E = Phi_E^T b_E, b = sum_L g_L p_L e_L
  if (tid < N) {
    double rr = 0.0;
    for (int q = A.L.sub_start[E]; q < A.L.sub_start[E + 1]; ++q) {
      const int l = A.L.local[q];
      rr += Phs[(size_t)tid * LD + l] * (A.L.gK[q] * lam[l] * A.L.p[q]);
    }
    A.rhs[E * N + tid] = rr;
  }

  // 5. coupling blocks B_{E,E+a}[i][j] = -sum_f w_f Phi_E[i][a_f] Phi_{E+a}[j][b_f], one tile per task
  for (int t = warp; t < g.dim * T * T; t += nwarp) {
    const int a = t / (T * T), tt = t - a * T * T, ti = tt / T, tj = tt - ti * T;
    double* BEN = BEE + (size_t)(1 + a) * N * N;
    const int i = 8 * ti + fr, j0 = 8 * tj + 2 * fc;
    double c0 = 0.0, c1 = 0.0;
    if (C[a] + 1 < g.S[a]) {
      const double* pn = PhN + (size_t)a * NP * LDN + (size_t)(8 * tj + fr) * LDN;
      const double* pe = Phs + (size_t)(8 * ti + fr) * LD;
      const int* fca = fcell + a * nfp;
      const double* wa = wi + a * nfp;
      for (int ks = 0; ks < nfp / 4; ++ks) {
        const int f = 4 * ks + fc;
        dmma(c0, c1, pe[fca[f]] * wa[f], pn[f]);
      }
    }
    if (i < N) {
      if (j0 < N) BEN[i * N + j0] = -c0;
      if (j0 + 1 < N) BEN[i * N + j0 + 1] = -c1;
    }
  }
}

}  // namespace lrbms
