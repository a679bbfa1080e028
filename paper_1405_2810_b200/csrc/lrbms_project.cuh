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
  int bulk;            // 1: n_loc and s_x even: Phi_E rows and the y/z face runs move in 16-byte granules
  unsigned long long* tstamp;   // optional phase timestamps of every 8th CTA (debug), or nullptr
};

__device__ __forceinline__ unsigned long long gtimer_p() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
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

// Local index helpers of a subdomain shape known at compile time (SX, SY, SZ > 0: the divisions and
// modulos fold to shifts and masks for 8 x 8 x 8) or at run time (0: read from g)
template <int SX, int SY, int SZ>
struct LShape {
  int sx, sy, sz, st1, st2;
  __device__ __forceinline__ explicit LShape(const Geo& g)
      : sx(SX ? SX : g.s[0]), sy(SY ? SY : g.s[1]), sz(SZ ? SZ : g.s[2]), st1(SX ? SX : g.s[0]),
        st2((SX ? SX : g.s[0]) * (SY ? SY : g.s[1])) {}
  __device__ __forceinline__ void xyz(int l, int c[3]) const {
    c[0] = l % sx;
    c[1] = (l / sx) % sy;
    c[2] = l / st2;
  }
  __device__ __forceinline__ int s(int a) const { return a == 0 ? sx : (a == 1 ? sy : sz); }
  __device__ __forceinline__ int stride(int a) const { return a == 0 ? 1 : (a == 1 ? st1 : st2); }
  __device__ __forceinline__ int nface(int a) const { return a == 0 ? sy * sz : (a == 1 ? sx * sz : sx * sy); }
  // internal index of the neighbour along axis a, direction dir (-1 outside the domain)
  __device__ __forceinline__ int nb(const Geo& g, int E, const int C[3], int l, const int c[3], int a, int dir) const {
    const int nc = c[a] + dir, sa = s(a), st = stride(a), nl = st2 * sz;
    if (nc >= 0 && nc < sa) return E * nl + l + dir * st;
    if (nc < 0) return C[a] == 0 ? -1 : (E - g.Estride[a]) * nl + l + (sa - 1) * st;
    return C[a] == g.S[a] - 1 ? -1 : (E + g.Estride[a]) * nl + l - (sa - 1) * st;
  }
  __device__ __forceinline__ int face_pos(const int c[3], int a) const {
    return a == 0 ? c[1] + sy * c[2] : (a == 1 ? c[0] + sx * c[2] : c[0] + sx * c[1]);
  }
  __device__ __forceinline__ int face_cell(int f, int a, int ca) const {
    if (a == 0) { const int y = f % sy, z = f / sy; return ca + sx * (y + sy * z); }
    if (a == 1) { const int x = f % sx, z = f / sx; return x + sx * (ca + sy * z); }
    const int x = f % sx, y = f / sx;
    return x + sx * (y + sy * ca);
  }
};

template <int NFIX, int SX, int SY, int SZ>   // compile-time N and subdomain shape (C5: 32; 8, 8, 8), 0 = runtime
__global__ void __launch_bounds__(512) k_project(ProjArgs A) {
  extern __shared__ __align__(16) double sm[];
  const Geo& g = A.g;
  constexpr int NLFIX = SX * SY * SZ;
  const LShape<SX, SY, SZ> S(g);
  const int N = NFIX ? NFIX : g.N, nl = NLFIX ? NLFIX : g.n_loc, E = blockIdx.x, tid = threadIdx.x, nt = blockDim.x;
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
  const int lq0 = A.L.sub_start[E], lq1 = A.L.sub_start[E + 1];   // link range of E, loaded at entry
  LRBMS_TSTAMP(A.tstamp && tid == 0 && (E & 7) == 0 && E < 8 * 256, A.tstamp[1024 + (E >> 3) * 8 + 0], gtimer_p());

  // 0. inputs of the face weights (a1 + R2) of the thread's first cell, loaded before the Phi staging
  //    floods the memory system with cp.async requests (the weights phase then no longer waits
  //    behind them)
  auto load_winputs = [&](int l, const int c[3], double& ll, double2 (&fp)[3], double2 (&fm)[3], double (&lp)[3],
                          double (&lm)[3], int (&wpos)[3]) {
    ll = A.lam[base + l];
#pragma unroll
    for (int a = 0; a < 3; ++a) {
      fp[a] = fm[a] = make_double2(0.0, 0.0);
      lp[a] = lm[a] = 0.0;
      wpos[a] = -1;
      if (a >= g.dim) continue;
      const int st = S.stride(a);
      if (c[a] + 1 < S.s(a)) {
        fp[a] = A.fc[(base + l) * 3 + a];
        lp[a] = A.lam[base + l + st];
      } else if (C[a] + 1 < g.S[a]) {
        const int nb = S.nb(g, E, C, l, c, a, +1);
        fp[a] = A.fc[(base + l) * 3 + a];
        lp[a] = A.lam[nb];
        wpos[a] = S.face_pos(c, a);
      }
      if (c[a] == 0 && C[a] > 0) {
        const int nb = S.nb(g, E, C, l, c, a, -1);
        fm[a] = A.fc[(size_t)nb * 3 + a];
        lm[a] = A.lam[nb];
      }
    }
  };
  double w_ll = 0.0, w_lp[3], w_lm[3];
  double2 w_fp[3], w_fm[3];
  int w_wpos[3];
  if (tid < nl) {
    int c0[3];
    S.xyz(tid, c0);
    load_winputs(tid, c0, w_ll, w_fp, w_fm, w_lp, w_lm, w_wpos);
  }

  // 1. stage Phi_E and the neighbour face slabs with cp.async (16-byte granules where the layout
  //    allows: Phi_E rows and the contiguous x-runs of the y/z faces; 8-byte gathers for x-faces)
  const double* PhiE = A.Phi + (size_t)E * N * nl;
  const bool v16 = A.bulk;   // n_loc and s_x even: 16-byte aligned rows and runs
  bool has[3];
#pragma unroll
  for (int a = 0; a < 3; ++a) has[a] = a < g.dim && C[a] + 1 < g.S[a];
  if (v16) {
    const int h = nl >> 1;
    for (int k = warp; k < N; k += nwarp)
      for (int c2 = lane; c2 < h; c2 += 32)
        cp_async16(Phs + (size_t)k * LD + 2 * c2, PhiE + (size_t)k * nl + 2 * c2);
  } else {
    for (int k = warp; k < N; k += nwarp)
      for (int c1 = lane; c1 < nl; c1 += 32) cp_async8(Phs + (size_t)k * LD + c1, PhiE + (size_t)k * nl + c1);
  }
  for (int a = 0; a < 3; ++a) {
    const int nf = a < g.dim ? S.nface(a) : 0;
    double* dst = PhN + (size_t)a * NP * LDN;
    if (has[a]) {
      const double* PhiN = A.Phi + (size_t)(E + g.Estride[a]) * N * nl;
      if (a > 0 && v16) {
        for (int k = warp; k < N; k += nwarp)
          for (int f2 = 2 * lane; f2 < nf; f2 += 64)
            cp_async16(dst + (size_t)k * LDN + f2, PhiN + (size_t)k * nl + S.face_cell(f2, a, 0));
      } else {
        for (int k = warp; k < N; k += nwarp)
          for (int f = lane; f < nf; f += 32)
            cp_async8(dst + (size_t)k * LDN + f, PhiN + (size_t)k * nl + S.face_cell(f, a, 0));
      }
    }
    for (int k = warp; k < NP; k += nwarp)
      for (int f = (has[a] && k < N ? nf : 0) + lane; f < LDN; f += 32) dst[(size_t)k * LDN + f] = 0.0;
    for (int f = tid; f < nfp; f += nt) {
      fcell[a * nfp + f] = (f < nf) ? S.face_cell(f, a, S.s(a) - 1) : 0;
      wi[a * nfp + f] = 0.0;
    }
  }
  asm volatile("cp.async.commit_group;\n" ::);
  for (int k = warp; k < NP; k += nwarp)
    for (int c1 = (k < N ? nl : 0) + lane; c1 < LD; c1 += 32) Phs[(size_t)k * LD + c1] = 0.0;
  LRBMS_TSTAMP(A.tstamp && tid == 0 && (E & 7) == 0 && E < 8 * 256, A.tstamp[1024 + (E >> 3) * 8 + 1], gtimer_p());

  // 2. a1 + face weights (R2) from the static coefficients.  Pass 1: every cell forms the weights of
  //    its +a faces (all loads issued up front) and of its -a faces across a subdomain side; the +a
  //    weight inside E is also the -a weight of the upper cell.  Pass 2: the diagonal.
  __syncthreads();   // wi / fcell initialised by the staging loop
  for (int l = tid; l < nl; l += nt) {
    int c[3];
    S.xyz(l, c);
    double ll;
    double2 fp[3], fm[3];
    double lp[3], lm[3];
    int wpos[3];
    if (l == tid) {   // the thread's first cell: inputs loaded before the Phi staging
      ll = w_ll;
#pragma unroll
      for (int a = 0; a < 3; ++a) {
        fp[a] = w_fp[a]; fm[a] = w_fm[a]; lp[a] = w_lp[a]; lm[a] = w_lm[a]; wpos[a] = w_wpos[a];
      }
    } else {
      load_winputs(l, c, ll, fp, fm, lp, lm, wpos);
    }
    lam[l] = ll;
    double dc = 0.0;
    double wl[3];
#pragma unroll
    for (int a = 0; a < 3; ++a) {
      const double wp = face_w(fp[a], ll, lp[a]);
      wl[a] = 0.0;
      if (a < g.dim) {
        if (wpos[a] >= 0) {
          wi[a * nfp + wpos[a]] = wp;
          dc += wp;
        } else if (c[a] + 1 < S.s(a)) {
          wl[a] = wp;
          Wc[(size_t)(l + S.stride(a)) * 8 + 1 + 2 * a] = wp;   // -a weight of the upper cell
        }
        dc += face_w(fm[a], lm[a], ll);
      }
    }
    // own slots only (the -a slots 1, 3, 5 belong to the lower cell inside E); slot 7 carries the
    // side-face weights to pass 2
    Wc[(size_t)l * 8 + 2] = wl[0];
    Wc[(size_t)l * 8 + 4] = wl[1];
    Wc[(size_t)l * 8 + 6] = wl[2];
    Wc[(size_t)l * 8 + 7] = dc;
  }
  __syncthreads();
  for (int l = tid; l < nl; l += nt) {
    int c[3];
    S.xyz(l, c);
    double* w = Wc + (size_t)l * 8;
    double d = w[7];
#pragma unroll
    for (int a = 0; a < 3; ++a) {
      if (a >= g.dim || c[a] == 0) w[1 + 2 * a] = 0.0;
      if (a < g.dim) d += w[1 + 2 * a] + w[2 + 2 * a];
    }
    w[0] = d;
    w[7] = 0.0;
  }
  __syncthreads();
  if (tid == 0) {  // links of E (R6), sequential: deterministic
    for (int q = lq0; q < lq1; ++q) {
      const int l = A.L.local[q];
      Wc[(size_t)l * 8] += A.L.gK[q] * lam[l];
    }
  }
  LRBMS_TSTAMP(A.tstamp && tid == 0 && (E & 7) == 0 && E < 8 * 256, A.tstamp[1024 + (E >> 3) * 8 + 2], gtimer_p());
  asm volatile("cp.async.wait_all;\n" ::);
  __syncthreads();
  LRBMS_TSTAMP(A.tstamp && tid == 0 && (E & 7) == 0 && E < 8 * 256, A.tstamp[1024 + (E >> 3) * 8 + 3], gtimer_p());

  // 3. B_EE = Phi Y^T with Y = A_EE Phi^T formed in registers; warp-strided k-steps of 4 cells
  double acc[10][2];
#pragma unroll
  for (int p = 0; p < 10; ++p) acc[p][0] = acc[p][1] = 0.0;
  const int fr = lane >> 2, fc = lane & 3;
  const int st0 = 1, st1 = S.st1, st2 = S.st2;
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
  LRBMS_TSTAMP(A.tstamp && tid == 0 && (E & 7) == 0 && E < 8 * 256, A.tstamp[1024 + (E >> 3) * 8 + 4], gtimer_p());
  double* BEE = A.blocks + (size_t)E * nb1 * N * N;

  // 4. r_E = Phi_E^T b_E, b = sum_L g_L p_L e_L
  if (tid < N) {
    double rr = 0.0;
    for (int q = lq0; q < lq1; ++q) {
      const int l = A.L.local[q];
      rr += Phs[(size_t)tid * LD + l] * (A.L.gK[q] * lam[l] * A.L.p[q]);
    }
    A.rhs[E * N + tid] = rr;
  }

  // 5. coupling blocks B_{E,E+a}[i][j] = -sum_f w_f Phi_E[i][a_f] Phi_{E+a}[j][b_f]; a warp owns a
  //    row of output tiles (a, ti) and its T accumulator chains share every A fragment (the gathered,
  //    weighted own-face row), so each k-step loads 1 + T fragments for T DMMAs
  const int ntask = g.dim * T;
  for (int t = warp; t < ntask; t += nwarp) {
    const int a = t / T, ti = t - a * T;
    const bool live = has[a];
    const double* pe = Phs + (size_t)(8 * ti + fr) * LD;
    const int* fca = fcell + a * nfp;
    const double* wa = wi + a * nfp;
    const double* pn = PhN + (size_t)a * NP * LDN + (size_t)fr * LDN;
    double cc[4][2];
#pragma unroll
    for (int tj = 0; tj < 4; ++tj) cc[tj][0] = cc[tj][1] = 0.0;
    if (live) {
      for (int ks = 0; ks < nfp / 4; ++ks) {
        const int f = 4 * ks + fc;
        const double av = pe[fca[f]] * wa[f];
#pragma unroll
        for (int tj = 0; tj < 4; ++tj)
          if (tj < T) dmma(cc[tj][0], cc[tj][1], av, pn[(size_t)8 * tj * LDN + f]);
      }
    }
    double* BEN = BEE + (size_t)(1 + a) * N * N;
    const int i = 8 * ti + fr;
#pragma unroll
    for (int tj = 0; tj < 4; ++tj) {
      const int j0 = 8 * tj + 2 * fc;
      if (tj < T && i < N) {
        if (j0 < N) BEN[i * N + j0] = -cc[tj][0];
        if (j0 + 1 < N) BEN[i * N + j0 + 1] = -cc[tj][1];
      }
    }
  }
  LRBMS_TSTAMP(A.tstamp && tid == 0 && (E & 7) == 0 && E < 8 * 256, A.tstamp[1024 + (E >> 3) * 8 + 5], gtimer_p());

  // 6. deterministic cross-warp reduction of B_EE (fixed warp order), mirrored for exact symmetry.
  //    All tile pairs at once through the (now free) Phi_E buffer when it is large enough.
  __syncthreads();   // all reads of Phs, Wc done
  if ((size_t)nwarp * 10 * 64 <= (size_t)NP * LD) {
    double* red = Phs;   // [nwarp][10 pairs][64]
#pragma unroll
    for (int p = 0; p < 10; ++p) {
      red[((size_t)warp * 10 + p) * 64 + 2 * lane] = acc[p][0];
      red[((size_t)warp * 10 + p) * 64 + 2 * lane + 1] = acc[p][1];
    }
    __syncthreads();
    for (int o = tid; o < 10 * 64; o += nt) {
      const int p = o >> 6, e = o & 63;
      const int ti = pair_ti(p), tj = pair_tj(p);
      if (tj >= T) continue;
      double v = 0.0;
      for (int w = 0; w < nwarp; ++w) v += red[(size_t)w * 10 * 64 + o];
      // fragment layout: element e = 2 lane + h holds row lane >> 2 = e >> 3, column 2 (lane & 3) + h = e & 7
      const int rr = e >> 3, cl = e & 7;
      const int i = 8 * ti + rr, j = 8 * tj + cl;
      if (i < N && j < N && (ti < tj || rr <= cl)) {
        BEE[i * N + j] = v;
        BEE[j * N + i] = v;
      }
    }
  } else {
    double* red = Wc;  // [nwarp][64]
#pragma unroll
    for (int p = 0; p < 10; ++p) {
      if (pair_tj(p) >= T) continue;
      red[warp * 64 + 2 * lane] = acc[p][0];
      red[warp * 64 + 2 * lane + 1] = acc[p][1];
      __syncthreads();
      if (tid < 64) {
        double v = 0.0;
        for (int w = 0; w < nwarp; ++w) v += red[w * 64 + tid];
        const int rr = tid >> 3, cl = tid & 7, ti = pair_ti(p), tj = pair_tj(p);
        const int i = 8 * ti + rr, j = 8 * tj + cl;
        if (i < N && j < N && (ti < tj || rr <= cl)) {
          BEE[i * N + j] = v;
          BEE[j * N + i] = v;
        }
      }
      __syncthreads();
    }
  }
#ifdef LRBMS_DEBUG
  if (A.tstamp) {
    __syncthreads();
    if (tid == 0 && (E & 7) == 0 && E < 8 * 256) A.tstamp[1024 + (E >> 3) * 8 + 6] = gtimer_p();
  }
#endif
}

}  // namespace lrbms
