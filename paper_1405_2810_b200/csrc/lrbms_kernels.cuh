// lrbms_kernels.cuh -- device kernels of the B200-native LRBMS online step (sm_100a, fp64).
//
// Internal layout: every per-cell field (s, p, K, phi V)
// is stored SUBDOMAIN-MAJOR: internal index g = E * n_loc + l, so that one subdomain's
// cells are one contiguous 4 KB (8x8x8) / 2 KB (16x16) run.  The local bases keep the
// ABI layout Phi[E][k][l] (basis function k contiguous over local cells): the
// reconstruction p_l = sum_k Phi[k][l] c_k then reads Phi fully coalesced.
//
// Paper references: PAPER.md line numbers (P:line); readings R1-R6/A1-A21: DESIGN.md.
#pragma once
#include <cooperative_groups.h>
#include <cstdint>

namespace lrbms {
namespace cg = cooperative_groups;

constexpr unsigned FULL = 0xffffffffu;

// Phase timestamps for the timeline tools (tools/exp_timeline.py, tools/exp_proj_phases.py): compiled
// only into a -DLRBMS_DEBUG build; the product build has no debug branches in its kernels.
#ifdef LRBMS_DEBUG
#define LRBMS_TSTAMP(cond, slot, val) \
  do {                                \
    if (cond) slot = val;             \
  } while (0)
#else
#define LRBMS_TSTAMP(cond, slot, val) \
  do {                                \
  } while (0)
#endif

struct Geo {
  int dim, nx, ny, nz;
  int s[3];        // subdomain size in cells per axis (sx, sy, sz)
  int S[3];        // number of subdomains per axis (Sx, Sy, Sz)
  int n_s, n_loc, N, n;
  int lstride[3];  // local strides 1, sx, sx*sy
  int Estride[3];  // subdomain strides 1, Sx, Sx*Sy
  int nface[3];    // fine faces on one subdomain side normal to axis a (= n_loc / s[a])
  double geo[3];   // |F|/d_F of an interior face normal to axis a (reading A3)
  double geo2[3];  // 2|F|/h_a of a link face normal to axis a (reading R6)
  double vol;      // cell volume
};

struct Flu {
  double mu_w, mu_o, swr, range, nw, no;
  double inv_range, inv_mu_w, inv_mu_o;   // reciprocals: no fp64 divisions in the per-cell kernels
  int kind;        // 1 = linear, 2 = quadratic Corey, 0 = general exponents
};

struct Links {     // sorted by (subdomain, local cell, original index)
  const int* sub_start;   // [n_s + 1]
  const int* local;       // [n_links] local cell l
  const int* orig;        // [n_links] index in the caller's link list
  const double* geo2;     // [n_links] 2|F|/h of the link face
  const double* gK;       // [n_links] 2|F|/h * K_cell (set with the medium): g_L = gK * lambda
  const double* p;        // [n_links] fixed pressure p_L
  const double* s_ext;    // [n_links] external saturation
};

// ------------------------------------------------------------------ a1: mobilities
// eq:brooksCorey P:183-186 with Corey k_r (R5), S_e clamped (A8); eq:frationalFlow P:203-206.
__device__ __forceinline__ void mobilities(const Flu& f, double s, double& lw, double& lo) {
  double se = (s - f.swr) * f.inv_range;
  se = fmin(fmax(se, 0.0), 1.0);
  double kw, ko;
  if (f.kind == 2) {
    kw = se * se;
    ko = (1.0 - se) * (1.0 - se);
  } else if (f.kind == 1) {
    kw = se;
    ko = 1.0 - se;
  } else {
    kw = pow(se, f.nw);
    ko = pow(1.0 - se, f.no);
  }
  lw = kw * f.inv_mu_w;
  lo = ko * f.inv_mu_o;
}
__device__ __forceinline__ double total_mobility(const Flu& f, double s) {
  double lw, lo;
  mobilities(f, s, lw, lo);
  return lw + lo;
}
__device__ __forceinline__ double frac_flow(const Flu& f, double s) {
  double lw, lo;
  mobilities(f, s, lw, lo);
  return lw / (lw + lo);
}

// ------------------------------------------------------------------ a2: face weights
// w_F = T_F (tau_a lambda_a + tau_b lambda_b), T_F = |F|/d_F * 2 K_a K_b/(K_a + K_b)
// (eq:penaltyParam P:305-307 with c_F = 1, weighted mean P:282-283; reading R2).
// Always called with (a, b) = (lower cell, upper cell) along the axis so that both cells
// of a face evaluate the bitwise-identical weight (exact flux antisymmetry).
__device__ __forceinline__ double face_weight(double geo, double Ka, double Kb, double la, double lb) {
  double T = geo * 2.0 * Ka * Kb / (Ka + Kb);
  double ta = Ka / (Ka + Kb);
  double tb = Kb / (Ka + Kb);
  return T * (ta * la + tb * lb);
}

// Static face coefficients (set with the medium): for the face between cell a (lower) and its +axis
// neighbour b, fc = (T_F tau_a, T_F tau_b), so w_F(lambda) = fc.x lambda_a + fc.y lambda_b.
// Both cells of a face read the same fc and evaluate the same expression: bitwise antisymmetric
// fluxes.  fc = (0, 0) where there is no +axis neighbour.
__device__ __forceinline__ double face_w(double2 fc, double la, double lb) { return fc.x * la + fc.y * lb; }

// ------------------------------------------------------------------ index helpers
__device__ __forceinline__ void local_xyz(const Geo& g, int l, int c[3]) {
  c[0] = l % g.s[0];
  int t = l / g.s[0];
  c[1] = t % g.s[1];
  c[2] = t / g.s[1];
}
__device__ __forceinline__ void sub_xyz(const Geo& g, int E, int C[3]) {
  C[0] = E % g.S[0];
  int t = E / g.S[0];
  C[1] = t % g.S[1];
  C[2] = t / g.S[1];
}
// internal index of the neighbour of local cell (c) of subdomain E (coords C) along axis a,
// direction dir = +-1; -1 outside the domain.
__device__ __forceinline__ int neighbour(const Geo& g, int E, const int C[3], int l, const int c[3],
                                         int a, int dir) {
  int nc = c[a] + dir;
  if (nc >= 0 && nc < g.s[a]) return E * g.n_loc + l + dir * g.lstride[a];
  if (nc < 0) {
    if (C[a] == 0) return -1;
    return (E - g.Estride[a]) * g.n_loc + l + (g.s[a] - 1) * g.lstride[a];
  }
  if (C[a] == g.S[a] - 1) return -1;
  return (E + g.Estride[a]) * g.n_loc + l - (g.s[a] - 1) * g.lstride[a];
}
// position of local cell c on the subdomain side normal to axis a
__device__ __forceinline__ int face_pos(const Geo& g, const int c[3], int a) {
  if (a == 0) return c[1] + g.s[1] * c[2];
  if (a == 1) return c[0] + g.s[0] * c[2];
  return c[0] + g.s[0] * c[1];
}
// local cell at position f on the side normal to axis a with coordinate ca along a
__device__ __forceinline__ int face_cell(const Geo& g, int f, int a, int ca) {
  if (a == 0) { int y = f % g.s[1], z = f / g.s[1]; return ca + g.s[0] * (y + g.s[1] * z); }
  if (a == 1) { int x = f % g.s[0], z = f / g.s[0]; return x + g.s[0] * (ca + g.s[1] * z); }
  int x = f % g.s[0], y = f / g.s[0];
  return x + g.s[0] * (y + g.s[1] * ca);
}

// sides s of subdomain E (coordinates C): s = a -> E + e_a, s = 3 + a -> E - e_a
__device__ __forceinline__ bool side_exists(const Geo& g, const int C[3], int s) {
  const int a = s < 3 ? s : s - 3;
  if (a >= g.dim) return false;
  return s < 3 ? C[a] + 1 < g.S[a] : C[a] > 0;
}
__device__ __forceinline__ int side_nb(const Geo& g, int E, int s) {
  return s < 3 ? E + g.Estride[s] : E - g.Estride[s - 3];
}

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(FULL, v, o);
  return v;
}

// error flag bits
enum : int { FLAG_PIVOT = 1, FLAG_NOCONV = 2, FLAG_NOFLOW = 4, FLAG_NAN = 8, FLAG_BREAKDOWN = 16 };
// words of the context's 16-int flag array: [0] the error bits above, [1] set_medium's phi check,
// [2] Newton-Schulz update skipped (guard tripped), [4..5] max |I - E X| of the step (ping-pong),
// [6] its maximum over the call
enum : int { FLAGW_NSTRIP = 2, FLAGW_NSMAX = 4 };
// Newton-Schulz safety net: when max_ij |(I - E X)_ij| reaches this (or is NaN) the update would not
// converge; the coarse inverse is dropped (X = 0: block Jacobi) until the next call rebuilds it
constexpr float NS_GUARD_MAX = 1.0f;

}  // namespace lrbms
