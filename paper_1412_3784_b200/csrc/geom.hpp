// geom.hpp -- host geometry (H0) of the cell-list path: lattice inverse,
// box heights, QR orientation, cell counts, stencil brackets, and the
// closed-form box evolution / remap policies.  Host C++ only, compiled with
// -ffp-contract=off so every expression is evaluated as written (the
// canonical fp64 arithmetic of DESIGN.md reading R16).  Independent of the
// oracle: it implements the same published definitions, nothing is shared.
#pragma once
#include <cmath>
#include <cstdint>
#include <cstring>

namespace nc {

// Row-major 3x3 helpers.  Columns of L are the box vectors (Eq. 1).
static inline double M(const double* A, int r, int c) { return A[3 * r + c]; }

// ---------------------------------------------------------------- inverse
// L^{-1} = adj(L)/det(L) with cofactors C_rc = L[r+1][c+1] L[r+2][c+2] -
// L[r+1][c+2] L[r+2][c+1] (indices mod 3) and det expanded along row 0 as
// (L00 C00 + L01 C01) + L02 C02 (R16).  Returns false unless det > 0 finite.
inline bool inverse3(const double* L, double* Li, double* det_out) {
  double C[3][3];
  for (int r = 0; r < 3; ++r)
    for (int c = 0; c < 3; ++c) {
      int r1 = (r + 1) % 3, r2 = (r + 2) % 3, c1 = (c + 1) % 3, c2 = (c + 2) % 3;
      C[r][c] = M(L, r1, c1) * M(L, r2, c2) - M(L, r1, c2) * M(L, r2, c1);
    }
  double det = (M(L, 0, 0) * C[0][0] + M(L, 0, 1) * C[0][1]) + M(L, 0, 2) * C[0][2];
  if (det_out) *det_out = det;
  if (!(det > 0.0) || !std::isfinite(det)) return false;
  for (int r = 0; r < 3; ++r)
    for (int c = 0; c < 3; ++c) Li[3 * r + c] = C[c][r] / det;
  return true;
}

static inline double len3(double x, double y, double z) { return std::sqrt((x * x + y * y) + z * z); }
static inline double dot3(const double* a, const double* b) { return (a[0] * b[0] + a[1] * b[1]) + a[2] * b[2]; }

// ---------------------------------------------------------------- QR
// Gram-Schmidt on the columns, r_kk > 0 (R8): the rotated box has
// one face in the xy plane and v1 on the x axis.
inline void qr3(const double* L, double* Q, double* R) {
  double v[3][3];
  for (int k = 0; k < 3; ++k)
    for (int r = 0; r < 3; ++r) v[k][r] = M(L, r, k);
  double r11 = len3(v[0][0], v[0][1], v[0][2]);
  double e1[3] = {v[0][0] / r11, v[0][1] / r11, v[0][2] / r11};
  double r12 = dot3(e1, v[1]);
  double u2[3] = {v[1][0] - r12 * e1[0], v[1][1] - r12 * e1[1], v[1][2] - r12 * e1[2]};
  double r22 = len3(u2[0], u2[1], u2[2]);
  double e2[3] = {u2[0] / r22, u2[1] / r22, u2[2] / r22};
  double e3[3] = {e1[1] * e2[2] - e1[2] * e2[1], e1[2] * e2[0] - e1[0] * e2[2], e1[0] * e2[1] - e1[1] * e2[0]};
  double r13 = dot3(e1, v[2]), r23 = dot3(e2, v[2]), r33 = dot3(e3, v[2]);
  for (int r = 0; r < 3; ++r) {
    Q[3 * r + 0] = e1[r];
    Q[3 * r + 1] = e2[r];
    Q[3 * r + 2] = e3[r];
  }
  const double Rv[9] = {r11, r12, r13, 0.0, r22, r23, 0.0, 0.0, r33};
  std::memcpy(R, Rv, sizeof Rv);
}

// Everything the kernels need about one box + variant + potential.  Passed
// to kernels BY VALUE (kernel-parameter constant bank).
struct Geom {
  double L[9], Li[9], Q[9], R[9];
  double det, h[3];
  int variant;      // 0 = DS, 1 = DO
  int dims[3];      // DS: c_k;  DO: l_k
  int64_t ncells;
  double w[3];      // DO widths r_kk/l_k
  double e[3];      // DO r_kk - l_k w_k (rounding residue, ~1e-16 r_kk)
  double d21, d31, d32;  // DO offsets in cell units r12/w1, r13/w1, r23/w2
  double cinv[3];   // DS 1/c_k (bracket arithmetic only)
  // potential
  double rc, rc2, eps, sig2, ushift;
  double band_lo, band_hi;  // canonical re-check band on r^2 (fp32 path)
  double rsplit2;           // fp32-mode pairs with r^2 >= rsplit2 (and below band_lo) use fp32 force math
  // fp32 copies for the fp32 kernels (constant-bank operands; set by the host with the above)
  float f_split2, f_lo, f_hi, f_sig2, f_c48, f_m24;
  // cell centre in the cell-local rotated frame (fp32 staging is centred on it), and the tensor-core
  // filter's superset bound on r^2 (kernels.cuh, mma_filter)
  double cc[3];
  float f_cc[3];
  float f_hmma;
  int dbg_drop;     // negative control (nc_debug): drop this many entries from every neighborhood
};

enum { GEOM_OK = 0, GEOM_BAD_BOX = 1, GEOM_DEGENERATE = 2 };

// Heights h_k = 1/||row_k(L^{-1})|| (R7); DS counts c_k =
// floor(h_k/d_cut); DO counts l_k = floor(r_kk/d_cut), widths
// w_k = r_kk/l_k.  Minimum grids of R9.
inline int make_geom(Geom& g, const double* L, int variant, double rc) {
  std::memcpy(g.L, L, sizeof(double) * 9);
  for (int k = 0; k < 9; ++k)
    if (!std::isfinite(L[k])) return GEOM_BAD_BOX;
  if (!inverse3(L, g.Li, &g.det)) return GEOM_BAD_BOX;
  for (int k = 0; k < 3; ++k) g.h[k] = 1.0 / len3(g.Li[3 * k], g.Li[3 * k + 1], g.Li[3 * k + 2]);
  qr3(L, g.Q, g.R);
  g.variant = variant;
  g.rc = rc;
  g.rc2 = rc * rc;
  if (variant == 0) {
    for (int k = 0; k < 3; ++k) {
      g.dims[k] = (int)std::floor(g.h[k] / rc);
      g.cinv[k] = 1.0 / (double)g.dims[k];
      g.w[k] = 0.0;
      g.e[k] = 0.0;
    }
    g.d21 = g.d31 = g.d32 = 0.0;
    if (g.dims[0] < 3 || g.dims[1] < 3 || g.dims[2] < 3) return GEOM_DEGENERATE;
  } else {
    for (int k = 0; k < 3; ++k) {
      double rkk = g.R[4 * k];
      g.dims[k] = (int)std::floor(rkk / rc);
      g.w[k] = rkk / (double)g.dims[k];
      g.e[k] = rkk - (double)g.dims[k] * g.w[k];
      g.cinv[k] = 0.0;
    }
    g.d21 = g.R[1] / g.w[0];
    g.d31 = g.R[2] / g.w[0];
    g.d32 = g.R[5] / g.w[1];
    if (g.dims[0] < 4 || g.dims[1] < 4 || g.dims[2] < 3) return GEOM_DEGENERATE;
  }
  g.ncells = (int64_t)g.dims[0] * g.dims[1] * g.dims[2];
  return GEOM_OK;
}

// ---------------------------------------------------------------- flows
inline bool is_diag(const double* A) {
  for (int r = 0; r < 3; ++r)
    for (int c = 0; c < 3; ++c)
      if (r != c && A[3 * r + c] != 0.0) return false;
  return true;
}

inline void matmul3(const double* A, const double* B, double* C) {
  double T[9];
  for (int r = 0; r < 3; ++r)
    for (int c = 0; c < 3; ++c) T[3 * r + c] = (M(A, r, 0) * M(B, 0, c) + M(A, r, 1) * M(B, 1, c)) + M(A, r, 2) * M(B, 2, c);
  std::memcpy(C, T, sizeof T);
}

// e^{A s}: diagonal -> exp per entry; nilpotent (A^2 = 0, e.g. the shear of
// Eq. 6) -> I + A s exactly; otherwise scaling-and-squaring Taylor.
inline void expm3(const double* A, double s, double* E) {
  if (is_diag(A)) {
    for (int k = 0; k < 9; ++k) E[k] = 0.0;
    for (int k = 0; k < 3; ++k) E[4 * k] = std::exp(A[4 * k] * s);
    return;
  }
  double A2[9];
  matmul3(A, A, A2);
  bool nil = true;
  for (int k = 0; k < 9; ++k) nil = nil && A2[k] == 0.0;
  if (nil) {
    for (int k = 0; k < 9; ++k) E[k] = A[k] * s + ((k % 4) == 0 ? 1.0 : 0.0);
    return;
  }
  double X[9], nrm = 0.0;
  for (int r = 0; r < 3; ++r) {
    double rs = std::fabs(A[3 * r] * s) + std::fabs(A[3 * r + 1] * s) + std::fabs(A[3 * r + 2] * s);
    nrm = rs > nrm ? rs : nrm;
  }
  int sq = nrm > 0 ? (int)std::ceil(std::log2(nrm)) + 4 : 0;
  if (sq < 0) sq = 0;
  double scale = std::ldexp(1.0, -sq);
  for (int k = 0; k < 9; ++k) X[k] = A[k] * s * scale;
  double term[9] = {1, 0, 0, 0, 1, 0, 0, 0, 1}, Ex[9] = {1, 0, 0, 0, 1, 0, 0, 0, 1};
  for (int j = 1; j < 30; ++j) {
    matmul3(term, X, term);
    for (int k = 0; k < 9; ++k) { term[k] /= j; Ex[k] += term[k]; }
  }
  for (int j = 0; j < sq; ++j) matmul3(Ex, Ex, Ex);
  std::memcpy(E, Ex, sizeof Ex);
}

// Remapped box L~_t for a policy (closed forms).
struct Policy {
  int kind;          // 0 none, 1 LE, 2 KR, 3 GKR, 4 lattice reduction (R30)
  double L0[9];
  double tstar;
  double om1[3], om2[3], beta[2], eps;
  double Lr[9], tr;  // kind 4: reduced basis Lr committed at time tr; L_t = e^{A (t - tr)} Lr
};

// Greedy pairwise Lagrange reduction of the columns of L (reading R30): sweep
// the ordered pairs (0,1),(0,2),(1,0),(1,2),(2,0),(2,1); mu = floor(v_i.v_j /
// v_j.v_j + 1/2); v_i <- v_i - mu v_j when |v_i - mu v_j|^2 < |v_i|^2 (1 - 1e-12);
// repeat until a sweep changes nothing.  Same lattice, det unchanged (unimodular
// column operations).  For shear it is the Lees-Edwards reset.
inline bool lattice_reduce(double* L) {
  static const int P[6][2] = {{0, 1}, {0, 2}, {1, 0}, {1, 2}, {2, 0}, {2, 1}};
  double v[3][3];
  for (int k = 0; k < 3; ++k)
    for (int r = 0; r < 3; ++r) v[k][r] = M(L, r, k);
  bool changed = false;
  for (int sweep = 0; sweep < 64; ++sweep) {
    bool step = false;
    for (int q = 0; q < 6; ++q) {
      const int i = P[q][0], j = P[q][1];
      const double mu = std::floor(dot3(v[i], v[j]) / dot3(v[j], v[j]) + 0.5);
      if (mu == 0.0) continue;
      const double w[3] = {v[i][0] - mu * v[j][0], v[i][1] - mu * v[j][1], v[i][2] - mu * v[j][2]};
      if (dot3(w, w) < dot3(v[i], v[i]) * (1.0 - 1e-12)) {
        v[i][0] = w[0]; v[i][1] = w[1]; v[i][2] = w[2];
        step = true;
      }
    }
    if (!step) break;
    changed = true;
  }
  for (int k = 0; k < 3; ++k)
    for (int r = 0; r < 3; ++r) L[3 * r + k] = v[k][r];
  return changed;
}

inline void box_at(const Policy& p, const double* A, double t, double* L) {
  if (p.kind == 1) {  // Lees-Edwards: tilt gamma0 + eps t kept in [-1/2, 1/2)
    double eps = A[1];
    double ay = p.L0[4];
    double g = p.L0[1] / ay + eps * t;
    g = g - std::floor(g + 0.5);
    std::memcpy(L, p.L0, sizeof(double) * 9);
    L[1] = g * ay;
    return;
  }
  if (p.kind == 2) {  // KR: e^{A (t mod t*)} L0 (Eq. 9)
    double tt = t - std::floor(t / p.tstar) * p.tstar;
    double E[9];
    expm3(A, tt, E);
    matmul3(E, p.L0, L);
    return;
  }
  if (p.kind == 4) {  // lattice reduction (R30), without committing (box_advance commits)
    double E[9];
    expm3(A, t - p.tr, E);
    matmul3(E, p.Lr, L);
    lattice_reduce(L);
    return;
  }
  if (p.kind == 3) {  // GKR, centered representative (R23)
    double f[2];
    for (int k = 0; k < 2; ++k) {
      double a = p.beta[k] * p.eps * t;
      f[k] = a - std::floor(a + 0.5);
    }
    double D[9] = {0, 0, 0, 0, 0, 0, 0, 0, 0};
    for (int k = 0; k < 3; ++k) D[4 * k] = std::exp(f[0] * p.om1[k] + f[1] * p.om2[k]);
    matmul3(D, p.L0, L);
    return;
  }
  double E[9];
  expm3(A, t, E);
  matmul3(E, p.L0, L);
}

// Box at t for the step loop: as box_at, and for kind 4 commits a reduction
// (Lr, tr) when one happens.
inline void box_advance(Policy& p, const double* A, double t, double* L) {
  if (p.kind != 4) {
    box_at(p, A, t, L);
    return;
  }
  double E[9];
  expm3(A, t - p.tr, E);
  matmul3(E, p.Lr, L);
  if (lattice_reduce(L)) {
    std::memcpy(p.Lr, L, sizeof(double) * 9);
    p.tr = t;
  }
}

}  // namespace nc
