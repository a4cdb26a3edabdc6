// TEST INFRASTRUCTURE ONLY (oracle).  Never linked into the product path.
//
// fp64 3x3 SVD and its reverse-mode rule.
//
// The reference computes the SVD with Eigen's JacobiSVD
// (/root/reference/proj/include/diffsim/svd3.hpp:8-22).  Eigen (3.x, version
// unpinned: the reference's CMakeLists.txt:12 only says
// find_package(Eigen3 REQUIRED)) is absent from this image, so this file
// restates the published one-sided (Hestenes) Jacobi SVD algorithm in plain
// C++.  Conventions follow the reference tape contract
// (tape.hpp:172-174): singular values descending and nonnegative, U and V
// orthogonal; V is made proper (det +1) so that for det(F) > 0 both U and V
// are rotations.
//
// svd3x3_adjoint restates the reference's reverse rule
// (svd3.hpp:27-63) with plain 3x3 loops, including the +-1e-9 clamp on the
// sigma-difference denominators (svd3.hpp:45-49).
#pragma once

#include <cmath>

namespace oracle {

inline void svd3x3_values(const double f[9], double u[9], double s[3], double vt[9]) {
  // g = F V, columns orthogonalised by plane rotations applied on the right.
  double g[3][3], v[3][3];
  for (int r = 0; r < 3; ++r)
    for (int c = 0; c < 3; ++c) {
      g[r][c] = f[3 * r + c];
      v[r][c] = (r == c) ? 1.0 : 0.0;
    }
  for (int sweep = 0; sweep < 60; ++sweep) {
    bool rotated = false;
    for (int p = 0; p < 2; ++p)
      for (int q = p + 1; q < 3; ++q) {
        double a = 0.0, b = 0.0, c = 0.0;
        for (int r = 0; r < 3; ++r) {
          a += g[r][p] * g[r][p];
          b += g[r][q] * g[r][q];
          c += g[r][p] * g[r][q];
        }
        if (c == 0.0 || std::fabs(c) <= 1e-17 * std::sqrt(a * b)) continue;
        rotated = true;
        const double zeta = (b - a) / (2.0 * c);
        const double t = (zeta >= 0.0 ? 1.0 : -1.0) / (std::fabs(zeta) + std::sqrt(1.0 + zeta * zeta));
        const double cs = 1.0 / std::sqrt(1.0 + t * t);
        const double sn = cs * t;
        for (int r = 0; r < 3; ++r) {
          const double gp = g[r][p], gq = g[r][q];
          g[r][p] = cs * gp - sn * gq;
          g[r][q] = sn * gp + cs * gq;
          const double vp = v[r][p], vq = v[r][q];
          v[r][p] = cs * vp - sn * vq;
          v[r][q] = sn * vp + cs * vq;
        }
      }
    if (!rotated) break;
  }
  double sig[3];
  for (int c = 0; c < 3; ++c)
    sig[c] = std::sqrt(g[0][c] * g[0][c] + g[1][c] * g[1][c] + g[2][c] * g[2][c]);
  // sort descending (selection; swap columns of g and v together)
  int order[3] = {0, 1, 2};
  for (int i = 0; i < 2; ++i)
    for (int j = i + 1; j < 3; ++j)
      if (sig[order[j]] > sig[order[i]]) {
        const int t = order[i];
        order[i] = order[j];
        order[j] = t;
      }
  double gs[3][3], vs[3][3], ss[3];
  for (int c = 0; c < 3; ++c) {
    ss[c] = sig[order[c]];
    for (int r = 0; r < 3; ++r) {
      gs[r][c] = g[r][order[c]];
      vs[r][c] = v[r][order[c]];
    }
  }
  // make V proper
  const double dv = vs[0][0] * (vs[1][1] * vs[2][2] - vs[1][2] * vs[2][1]) -
                    vs[0][1] * (vs[1][0] * vs[2][2] - vs[1][2] * vs[2][0]) +
                    vs[0][2] * (vs[1][0] * vs[2][1] - vs[1][1] * vs[2][0]);
  if (dv < 0.0)
    for (int r = 0; r < 3; ++r) {
      vs[r][2] = -vs[r][2];
      gs[r][2] = -gs[r][2];
    }
  // U columns = g / sigma, completing the basis for (near-)zero sigma
  double uc[3][3];
  for (int c = 0; c < 3; ++c) {
    if (ss[c] > 1e-300) {
      for (int r = 0; r < 3; ++r) uc[r][c] = gs[r][c] / ss[c];
    } else if (c == 2) {
      uc[0][2] = uc[1][0] * uc[2][1] - uc[2][0] * uc[1][1];
      uc[1][2] = uc[2][0] * uc[0][1] - uc[0][0] * uc[2][1];
      uc[2][2] = uc[0][0] * uc[1][1] - uc[1][0] * uc[0][1];
    } else {
      for (int r = 0; r < 3; ++r) uc[r][c] = (r == c) ? 1.0 : 0.0;
    }
  }
  for (int r = 0; r < 3; ++r)
    for (int c = 0; c < 3; ++c) {
      u[3 * r + c] = uc[r][c];
      vt[3 * r + c] = vs[c][r];
    }
  for (int i = 0; i < 3; ++i) s[i] = ss[i];
}

inline void svd3x3_adjoint(const double u[9], const double s[3], const double vt[9],
                           const double out_adj[21], double f_adj[9]) {
  // P = U^T dU, Q = V^T dV  (V = vt^T, dV = (d vt)^T)
  double P[3][3], Q[3][3];
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) {
      double p = 0.0, q = 0.0;
      for (int k = 0; k < 3; ++k) {
        p += u[3 * k + i] * out_adj[3 * k + j];
        // V(k, i) = vt(i, k); gV(k, j) = gvt(j, k)
        q += vt[3 * i + k] * out_adj[12 + 3 * j + k];
      }
      P[i][j] = p;
      Q[i][j] = q;
    }
  auto clamp_den = [](double d) {
    if (d >= 0.0 && d < 1e-9) return 1e-9;
    if (d < 0.0 && d > -1e-9) return -1e-9;
    return d;
  };
  double in[3][3] = {{0, 0, 0}, {0, 0, 0}, {0, 0, 0}};
  for (int i = 0; i < 3; ++i) in[i][i] = out_adj[9 + i];
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) {
      if (i == j) continue;
      const double fij = 1.0 / clamp_den(s[j] * s[j] - s[i] * s[i]);
      in[i][j] += fij * (P[i][j] - P[j][i]) * s[j];
      in[i][j] += s[i] * fij * (Q[i][j] - Q[j][i]);
    }
  // F_adj = U in V^T
  double t[3][3];
  for (int r = 0; r < 3; ++r)
    for (int c = 0; c < 3; ++c) {
      double a = 0.0;
      for (int k = 0; k < 3; ++k) a += u[3 * r + k] * in[k][c];
      t[r][c] = a;
    }
  for (int r = 0; r < 3; ++r)
    for (int c = 0; c < 3; ++c) {
      double a = 0.0;
      for (int k = 0; k < 3; ++k) a += t[r][k] * vt[3 * k + c];
      f_adj[3 * r + c] = a;
    }
}

}  // namespace oracle
