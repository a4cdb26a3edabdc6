// MLS-MPM physics: constitutive laws, SDF colliders, grid-node update, and
// the hand-written reverse-mode adjoint of each (replacing the reference's
// scalar tape, diffsim/tape.hpp:80-264).  Templated on the real type: fp32 on
// the device; fp64 in the host adjoint check (tests/native/adjoint_check.cpp).
//
// Forward semantics restate /root/reference/proj/include/diffsim/mpm.hpp:
//   stress_elastoplastic 165-198, stress_fluid 200-210, SdfCollider::query
//   86-131, grid_update 256-305; config-gap extensions per SURVEY.md 8(g)
//   (fixed-corotated, neo-Hookean + actuation, viscosity, cylinder, hollow
//   box, rotating colliders, sticky boundary) as in oracle/include/oracle/mpm.hpp.
// Adjoint branch semantics follow the tape: min/max/clamp take the active
// branch's subgradient and zero at ties; where() does not differentiate the
// predicate (tape.hpp:364-393).
#pragma once

#include "dm_math.cuh"

namespace dm {

enum : int { kFixedCorotated = 0, kNeoHookean = 1, kElastoplastic = 2, kFluid = 3 };
enum : int { kPlane = 0, kSphere = 1, kBox = 2, kCylinder = 3, kHollowBox = 4 };
enum : int { kSlip = 0, kSticky = 1 };
enum : int { kErrNone = 0, kErrP2GInterior = 1, kErrG2PInterior = 2, kErrDetF = 3 };

// Device-side material (derived constants precomputed on the host).
template <class R>
struct Law {
  int kind;
  R mu, lam, cy, visc, act_k;
  R mass, vol;
  R dmu_dE, dlam_dE;
};

template <class R>
struct Col {
  int kind;
  v3<R> c, vel, om, nrm;  // center, linear / angular velocity, plane normal or cylinder axis
  R radius, length, thickness;
  v3<R> half;
};

// ======================= constitutive laws =======================

// Hencky / von Mises return map quantities (mpm.hpp:165-188)
template <class R>
struct Hencky {
  Svd<R> sv;
  R eps[3], dev[3], m, N;  // log strain, deviator, mean, |dev| (+1e-30)
  bool yield;
  R k;                     // c_y / N (yield only)
  R epsp[3], sigp[3];      // projected log strain / singular values
};

template <class R>
DM_HD Hencky<R> hencky(const m3<R>& f, R cy) {
  Hencky<R> h;
  h.sv = svd3(f);
#pragma unroll
  for (int i = 0; i < 3; ++i) h.eps[i] = r_log(h.sv.s[i]);
  const R tr = h.eps[0] + h.eps[1] + h.eps[2];
  h.m = tr * R(1.0 / 3.0);
#pragma unroll
  for (int i = 0; i < 3; ++i) h.dev[i] = h.eps[i] - h.m;
  h.N = r_sqrt(h.dev[0] * h.dev[0] + h.dev[1] * h.dev[1] + h.dev[2] * h.dev[2] + R(1e-30));
  const R dgamma = h.N - cy;
  const R iN = R(1) / h.N;
  h.yield = dgamma > R(0);
  h.k = cy * iN;
  if (h.yield) {
    const R s = dgamma * iN;
#pragma unroll
    for (int i = 0; i < 3; ++i) {
      h.epsp[i] = h.eps[i] - h.dev[i] * s;
      h.sigp[i] = r_exp(h.epsp[i]);
    }
  } else {
#pragma unroll
    for (int i = 0; i < 3; ++i) {
      h.epsp[i] = h.eps[i];
      h.sigp[i] = h.sv.s[i];
    }
  }
  return h;
}

// First Piola stress for the P2G (mpm.hpp:212-217 extended).  For the
// elastoplastic law P is evaluated at the projected strain as the reference
// does (mpm.hpp:189-196).  *bad set when det F <= 0.
// memo (optional): receives the SVD / Hencky record of F for the SVD laws,
// which law_stress_vjp then reuses instead of decomposing F again.
template <class R>
DM_HD m3<R> law_stress(const Law<R>& L, const m3<R>& F, R act, bool* bad, Hencky<R>* memo = nullptr) {
  const R J = det(F);
  if (!(J > R(0))) *bad = true;
  switch (L.kind) {
    case kFixedCorotated: {
      const Svd<R> sv = svd3(F);
      if (memo) memo->sv = sv;
      const m3<R> Rot = mul_bt(sv.u, sv.v);
      return (F - Rot) * (R(2) * L.mu) + cofactor(F) * (L.lam * (J - R(1)));
    }
    case kNeoHookean: {
      const R alpha = R(1) + R(0.75) * L.mu / L.lam;
      const R ic = ddot(F, F);
      const R mt = L.mu * (R(1) - R(1) / (ic + R(1)));
      m3<R> P = F * mt + cofactor(F) * (L.lam * (J - alpha));
      const R ka = L.act_k * act;
      P(0, 0) += ka * F(0, 0);
      P(1, 0) += ka * F(1, 0);
      P(2, 0) += ka * F(2, 0);
      return P;
    }
    case kElastoplastic: {
      const Hencky<R> h = hencky(F, L.cy);
      if (memo) *memo = h;
      const R tr2 = h.epsp[0] + h.epsp[1] + h.epsp[2];
      R ps[3];
#pragma unroll
      for (int i = 0; i < 3; ++i) ps[i] = (R(2) * L.mu * h.epsp[i] + L.lam * tr2) / h.sigp[i];
      return usv(h.sv, ps[0], ps[1], ps[2]);
    }
    default:  // fluid
      return cofactor(F) * (L.lam * (J - R(1)));
  }
}

// G2P projection F' = proj(F_new) (mpm.hpp:341-344).
template <class R>
DM_HD m3<R> law_project(const Law<R>& L, const m3<R>& F, bool* bad) {
  if (L.kind == kElastoplastic) {
    if (!(det(F) > R(0))) *bad = true;
    const Hencky<R> h = hencky(F, L.cy);
    if (!h.yield) return F;
    return usv(h.sv, h.sigp[0], h.sigp[1], h.sigp[2]);
  }
  if (L.kind == kFluid) {
    const R J = det(F);
    if (!(J > R(0))) *bad = true;
    const R s = r_cbrt(J);
    return mdiag(s, s, s);
  }
  return F;
}

// ---- forward evaluation in deviation form ----
// The particle state stores D = F - I (fp32): a small strain keeps its
// relative precision (F itself would round it to 6e-8 absolute, i.e. 6 % of a
// 1e-6 strain; SURVEY 8(d)'s per-substep 1e-5 gate on a resting elastic body
// needs ~1e-7).  The forward stress and projection are evaluated from D:
//   * SVD laws (fixed-corotated, Hencky / von Mises): the SVD of F = I + D
//     from the symmetric eigenproblem of S = F^T F - I = D + D^T + D^T D
//     (fp32 Jacobi; S and its eigenvalues lambda_i = sigma_i^2 - 1 are
//     resolved relative to |D|, so eps_i = log1p(lambda_i) / 2 and
//     sigma_i - 1 = lambda_i / (1 + sigma_i) keep their precision) -- a
//     one-sided SVD of I + D rounds the singular values to 6e-8 absolute
//   * fluid: J - 1 = det(I + D) - 1 expanded in D (det1m), no cancellation
//   * neo-Hookean: P expanded around F = I (the two O(mu) terms cancel there)
// The adjoints linearise at F = I + D in fp32 (their terms do not cancel).

// det(I + D) - 1 = tr D + (principal 2x2 minors of D) + det D
template <class R>
DM_HD R det1m(const m3<R>& D) {
  const R m2 = (D(0, 0) * D(1, 1) - D(0, 1) * D(1, 0)) + (D(0, 0) * D(2, 2) - D(0, 2) * D(2, 0)) +
               (D(1, 1) * D(2, 2) - D(1, 2) * D(2, 1));
  return (D(0, 0) + D(1, 1) + D(2, 2)) + m2 + det(D);
}

template <class R>
DM_HD m3<R> eye_plus(const m3<R>& D) {
  m3<R> F = D;
  F(0, 0) += R(1);
  F(1, 1) += R(1);
  F(2, 2) += R(1);
  return F;
}

// SVD of F = I + D with lam_i = s_i^2 - 1 (Svd's s, u, v; v a rotation).
template <class R>
struct SvdD {
  Svd<R> sv;
  R lam[3];
};

template <class R>
DM_HD SvdD<R> svd3_dev(const m3<R>& D) {
  // S = D + D^T + D^T D (symmetric)
  R S[3][3];
#pragma unroll
  for (int i = 0; i < 3; ++i)
#pragma unroll
    for (int j = 0; j < 3; ++j) S[i][j] = D(i, j) + D(j, i) + (D(0, i) * D(0, j) + D(1, i) * D(1, j) + D(2, i) * D(2, j));
  m3<R> v = meye<R>();
  const int sweeps = sizeof(R) == 4 ? 8 : 16;
  for (int sw = 0; sw < sweeps; ++sw) {
    bool rot = false;
#pragma unroll
    for (int k = 0; k < 3; ++k) {
      const int p = k == 2 ? 1 : 0, q = k == 0 ? 1 : 2, r = 3 - p - q;
      const R apq = S[p][q];
      const R scale = r_abs(S[p][p]) + r_abs(S[q][q]);
      // converged at the rounding floor of the pair (fp32: 1e-7)
      if (!(r_abs(apq) > R(sizeof(R) == 4 ? 1e-7 : 1e-16) * scale + R(1e-35))) continue;
      rot = true;
      const R tau = (S[q][q] - S[p][p]) / (R(2) * apq);
      const R t = (tau >= R(0) ? R(1) : R(-1)) / (r_abs(tau) + r_sqrt(R(1) + tau * tau));
      const R c = R(1) / r_sqrt(R(1) + t * t), sn = t * c;
      S[p][p] -= t * apq;
      S[q][q] += t * apq;
      S[p][q] = S[q][p] = R(0);
      const R srp = S[r][p], srq = S[r][q];
      S[r][p] = S[p][r] = c * srp - sn * srq;
      S[r][q] = S[q][r] = sn * srp + c * srq;
#pragma unroll
      for (int i = 0; i < 3; ++i) {
        const R vp = v(i, p), vq = v(i, q);
        v(i, p) = c * vp - sn * vq;
        v(i, q) = sn * vp + c * vq;
      }
    }
    if (!rot) break;
  }
  if (det(v) < R(0)) {
#pragma unroll
    for (int i = 0; i < 3; ++i) v(i, 2) = -v(i, 2);
  }
  SvdD<R> o;
  o.sv.v = v;
#pragma unroll
  for (int c = 0; c < 3; ++c) {
    o.lam[c] = S[c][c];
    const R s = r_sqrt(R(1) + S[c][c]);
    o.sv.s[c] = s;
    const R inv = s > R(0) ? R(1) / s : R(0);
    // u_c = F v_c / s_c = (v_c + D v_c) / s_c
#pragma unroll
    for (int i = 0; i < 3; ++i) o.sv.u(i, c) = (v(i, c) + (D(i, 0) * v(0, c) + D(i, 1) * v(1, c) + D(i, 2) * v(2, c))) * inv;
  }
  return o;
}

// Hencky / von Mises record from the deviation-form SVD (hencky() with
// eps_i = log1p(lam_i) / 2).
template <class R>
DM_HD Hencky<R> hencky_dev(const SvdD<R>& sd, R cy) {
  Hencky<R> h;
  h.sv = sd.sv;
#pragma unroll
  for (int i = 0; i < 3; ++i) h.eps[i] = R(0.5) * r_log1p(sd.lam[i]);
  const R tr = h.eps[0] + h.eps[1] + h.eps[2];
  h.m = tr * R(1.0 / 3.0);
#pragma unroll
  for (int i = 0; i < 3; ++i) h.dev[i] = h.eps[i] - h.m;
  h.N = r_sqrt(h.dev[0] * h.dev[0] + h.dev[1] * h.dev[1] + h.dev[2] * h.dev[2] + R(1e-30));
  const R dgamma = h.N - cy;
  const R iN = R(1) / h.N;
  h.yield = dgamma > R(0);
  h.k = cy * iN;
  if (h.yield) {
    const R s = dgamma * iN;
#pragma unroll
    for (int i = 0; i < 3; ++i) {
      h.epsp[i] = h.eps[i] - h.dev[i] * s;
      h.sigp[i] = r_exp(h.epsp[i]);
    }
  } else {
#pragma unroll
    for (int i = 0; i < 3; ++i) {
      h.epsp[i] = h.eps[i];
      h.sigp[i] = h.sv.s[i];
    }
  }
  return h;
}

// First Piola stress from D = F - I (mpm.hpp:212-217 extended; same values as
// law_stress(I + D) up to rounding).
template <class R>
DM_HD m3<R> law_stress_fwd(const Law<R>& L, const m3<R>& D, R act, bool* bad) {
  const R jm1 = det1m(D);
  if (!(jm1 > R(-1))) *bad = true;
  switch (L.kind) {
    case kFixedCorotated: {
      // P = 2 mu (F - R) + lam (J - 1) cof F = U diag(2 mu (s_i - 1) + lam (J - 1) J / s_i) V^T
      const SvdD<R> sd = svd3_dev(D);
      const R J = R(1) + jm1;
      R ph[3];
#pragma unroll
      for (int i = 0; i < 3; ++i)
        ph[i] = R(2) * L.mu * (sd.lam[i] / (R(1) + sd.sv.s[i])) + L.lam * jm1 * J / sd.sv.s[i];
      return usv(sd.sv, ph[0], ph[1], ph[2]);
    }
    case kElastoplastic: {
      const Hencky<R> h = hencky_dev(svd3_dev(D), L.cy);
      const R tr2 = h.epsp[0] + h.epsp[1] + h.epsp[2];
      R ps[3];
#pragma unroll
      for (int i = 0; i < 3; ++i) ps[i] = (R(2) * L.mu * h.epsp[i] + L.lam * tr2) / h.sigp[i];
      return usv(h.sv, ps[0], ps[1], ps[2]);
    }
    case kNeoHookean: {
      // P = mu (1 - 1/(I_C+1)) F + lam (J - alpha) cof F, alpha = 1 + 3 mu / (4 lam), as
      // mu [ 3/4 (D + D^T - tr D I - cof D) + (I_C - 3) / (4 (I_C + 1)) F ] + lam (J - 1) cof F
      const m3<R> F = eye_plus(D);
      const R trD = D(0, 0) + D(1, 1) + D(2, 2);
      const R ic3 = R(2) * trD + ddot(D, D);  // I_C - 3
      const m3<R> cD = cofactor(D);
      m3<R> S = D + transpose(D) - cD;
      S(0, 0) -= trD;
      S(1, 1) -= trD;
      S(2, 2) -= trD;
      m3<R> P = S * (R(0.75) * L.mu) + F * (L.mu * ic3 / (R(4) * (ic3 + R(4)))) + cofactor(F) * (L.lam * jm1);
      const R ka = L.act_k * act;
      P(0, 0) += ka * F(0, 0);
      P(1, 0) += ka * F(1, 0);
      P(2, 0) += ka * F(2, 0);
      return P;
    }
    default:  // fluid
      return cofactor(eye_plus(D)) * (L.lam * jm1);
  }
}

// G2P projection (mpm.hpp:341-344) in deviation form: D' = proj(I + Dn) - I.
// tau (elastoplastic): also the Kirchhoff stress P F'^T of the projected F'
// = U diag(2 mu epsp + lam tr epsp) U^T -- the value the next P2G's
// stress_elastoplastic(F') has (F' is on or inside the yield surface, so its
// own return mapping is the identity), from this SVD instead of a new one.
template <class R>
DM_HD m3<R> law_project_fwd(const Law<R>& L, const m3<R>& Dn, bool* bad, m3<R>* tau = nullptr) {
  if (L.kind == kElastoplastic) {
    if (!(det1m(Dn) > R(-1))) *bad = true;
    const Hencky<R> h = hencky_dev(svd3_dev(Dn), L.cy);
    if (tau) {
      const R tr = h.epsp[0] + h.epsp[1] + h.epsp[2];
      *tau = udut(h.sv.u, R(2) * L.mu * h.epsp[0] + L.lam * tr, R(2) * L.mu * h.epsp[1] + L.lam * tr,
                  R(2) * L.mu * h.epsp[2] + L.lam * tr);
    }
    if (!h.yield) return Dn;
    // D' = U diag(sigma_p - 1) V^T + (U V^T - I)  (yielding: |strain| > c_y, no cancellation issue)
    m3<R> Dp = usv(h.sv, h.sigp[0] - R(1), h.sigp[1] - R(1), h.sigp[2] - R(1)) + mul_bt(h.sv.u, h.sv.v);
    Dp(0, 0) -= R(1);
    Dp(1, 1) -= R(1);
    Dp(2, 2) -= R(1);
    return Dp;
  }
  if (L.kind == kFluid) {
    // F' = J^(1/3) I  ->  D' = (J^(1/3) - 1) I = expm1(log1p(J - 1) / 3) I
    const R jm1 = det1m(Dn);
    if (!(jm1 > R(-1))) *bad = true;
    const R w = r_expm1(r_log1p(jm1) * R(1.0 / 3.0));
    return mdiag(w, w, w);
  }
  return Dn;  // fixed-corotated, neo-Hookean: no projection (the next P2G checks det F)
}

// ---- adjoints ----

// isotropic Hencky stress phi_i = (2 mu e_i + lam tr e) / s_i at singular
// values s (no projection): jd, divided differences for isotropic_vjp.
template <class R>
DM_HD m3<R> hencky_stress_vjp(const Svd<R>& sv, const R e[3], R mu, R lam, const m3<R>& Pbar, R* mubar,
                              R* lambar) {
  const R tr = e[0] + e[1] + e[2];
  const R is[3] = {R(1) / sv.s[0], R(1) / sv.s[1], R(1) / sv.s[2]};
  R phi[3], jd[3][3];
#pragma unroll
  for (int i = 0; i < 3; ++i) phi[i] = (R(2) * mu * e[i] + lam * tr) * is[i];
#pragma unroll
  for (int i = 0; i < 3; ++i)
#pragma unroll
    for (int j = 0; j < 3; ++j)
      jd[i][j] = ((i == j ? R(2) * mu : R(0)) + lam) * (is[j] * is[i]) - (i == j ? phi[i] * is[i] : R(0));
  auto dd = [&](int i, int j) {
    const R L = log_dd(sv.s[i], sv.s[j]);
    return (R(2) * mu * (sv.s[j] * L - e[j]) - lam * tr) * (is[i] * is[j]);
  };
  const m3<R> ghat = ut_m_v(sv, Pbar);
  if (mubar) {
    R mb = R(0), lb = R(0);
#pragma unroll
    for (int i = 0; i < 3; ++i) {
      mb += ghat(i, i) * R(2) * e[i] * is[i];
      lb += ghat(i, i) * tr * is[i];
    }
    *mubar += mb;
    *lambar += lb;
  }
  return isotropic_vjp(sv, ghat, phi, jd, dd(0, 1), dd(0, 2), dd(1, 2));
}

// Return-map projection adjoint: Fbar from F'bar for a yielding Hencky state.
template <class R>
DM_HD m3<R> hencky_project_vjp(const Hencky<R>& h, R mu, R cy, const m3<R>& Fpbar, R* mubar) {
  R jd[3][3];
  const R iN = R(1) / h.N, kn2 = h.k * iN * iN;
  const R is[3] = {R(1) / h.sv.s[0], R(1) / h.sv.s[1], R(1) / h.sv.s[2]};
#pragma unroll
  for (int i = 0; i < 3; ++i)
#pragma unroll
    for (int j = 0; j < 3; ++j) {
      const R de = R(1.0 / 3.0) + h.k * ((i == j ? R(1) : R(0)) - R(1.0 / 3.0)) - kn2 * h.dev[i] * h.dev[j];
      jd[i][j] = h.sigp[i] * de * is[j];
    }
  auto dd = [&](int i, int j) {
    const R L = log_dd(h.sv.s[i], h.sv.s[j]);
    const R z = h.k * L * (h.sv.s[i] - h.sv.s[j]);
    const R E = r_abs(z) < R(1e-4) ? R(1) + R(0.5) * z : r_expm1(z) / z;
    return h.sigp[j] * h.k * L * E;
  };
  const m3<R> ghat = ut_m_v(h.sv, Fpbar);
  if (mubar) {
    // c_y = sigma_y / (c mu): d c_y / d mu = -c_y / mu; d e'_i / d c_y = dev_i / N
    R s = R(0);
#pragma unroll
    for (int i = 0; i < 3; ++i) s += ghat(i, i) * h.sigp[i] * h.dev[i];
    *mubar += s * iN * (-cy / mu);
  }
  return isotropic_vjp(h.sv, ghat, h.sigp, jd, dd(0, 1), dd(0, 2), dd(1, 2));
}

// Fbar += (dP/dF)^T Pbar; also mu/lambda/actuation cotangents.
template <class R>
DM_HD void law_stress_vjp(const Law<R>& L, const m3<R>& F, R act, const m3<R>& Pbar, m3<R>& Fbar, R& mubar,
                          R& lambar, R& actbar, const Hencky<R>* memo = nullptr) {
  const R J = det(F);
  switch (L.kind) {
    case kFixedCorotated: {
      // P = 2 mu (F - R) + lam (J - 1) cof F ; self-adjoint Hessian
      const Svd<R> sv = memo ? memo->sv : svd3(F);
      const m3<R> Rot = mul_bt(sv.u, sv.v);
      const m3<R> ph = ut_m_v(sv, Pbar);
      // skew part: wr(i, j) = -wr(j, i) = (ph(i, j) - ph(j, i)) / (s_i + s_j)
      const R w01 = (ph(0, 1) - ph(1, 0)) / (sv.s[0] + sv.s[1]);
      const R w02 = (ph(0, 2) - ph(2, 0)) / (sv.s[0] + sv.s[2]);
      const R w12 = (ph(1, 2) - ph(2, 1)) / (sv.s[1] + sv.s[2]);
      m3<R> wr = mzero<R>();
      wr(0, 1) = w01;
      wr(1, 0) = -w01;
      wr(0, 2) = w02;
      wr(2, 0) = -w02;
      wr(1, 2) = w12;
      wr(2, 1) = -w12;
      const m3<R> dR = u_m_vt(sv, wr);
      const m3<R> cof = cofactor(F);
      Fbar += (Pbar - dR) * (R(2) * L.mu) + cof * (L.lam * ddot(cof, Pbar)) +
              cofactor_jvp(F, Pbar) * (L.lam * (J - R(1)));
      mubar += R(2) * ddot(Pbar, F - Rot);
      lambar += (J - R(1)) * ddot(Pbar, cof);
      return;
    }
    case kNeoHookean: {
      const R alpha = R(1) + R(0.75) * L.mu / L.lam;
      const R ic = ddot(F, F);
      const R ip = R(1) / (ic + R(1));
      const m3<R> cof = cofactor(F);
      m3<R> d = F * (L.mu * R(2) * ddot(F, Pbar) * ip * ip) + Pbar * (L.mu * (R(1) - ip)) +
                cof * (L.lam * ddot(cof, Pbar)) + cofactor_jvp(F, Pbar) * (L.lam * (J - alpha));
      const R ka = L.act_k * act;
      d(0, 0) += ka * Pbar(0, 0);
      d(1, 0) += ka * Pbar(1, 0);
      d(2, 0) += ka * Pbar(2, 0);
      Fbar += d;
      mubar += ddot(Pbar, F * (R(1) - ip) - cof * R(0.75));
      lambar += (J - R(1)) * ddot(Pbar, cof);
      actbar += L.act_k * (Pbar(0, 0) * F(0, 0) + Pbar(1, 0) * F(1, 0) + Pbar(2, 0) * F(2, 0));
      return;
    }
    case kElastoplastic: {
      const Hencky<R> h = memo ? *memo : hencky(F, L.cy);
      if (!h.yield) {
        Fbar += hencky_stress_vjp(h.sv, h.eps, L.mu, L.lam, Pbar, &mubar, &lambar);
      } else {
        Svd<R> svp = h.sv;
#pragma unroll
        for (int i = 0; i < 3; ++i) svp.s[i] = h.sigp[i];
        const m3<R> fpb = hencky_stress_vjp(svp, h.epsp, L.mu, L.lam, Pbar, &mubar, &lambar);
        Fbar += hencky_project_vjp(h, L.mu, L.cy, fpb, &mubar);
      }
      return;
    }
    default: {
      const m3<R> cof = cofactor(F);
      Fbar += cof * (L.lam * ddot(cof, Pbar)) + cofactor_jvp(F, Pbar) * (L.lam * (J - R(1)));
      lambar += (J - R(1)) * ddot(Pbar, cof);
      return;
    }
  }
}

// Fnew_bar from F'bar through the G2P projection.
template <class R>
DM_HD m3<R> law_project_vjp(const Law<R>& L, const m3<R>& Fnew, const m3<R>& Fpbar, R& mubar) {
  if (L.kind == kElastoplastic) {
    const Hencky<R> h = hencky(Fnew, L.cy);
    if (!h.yield) return Fpbar;
    return hencky_project_vjp(h, L.mu, L.cy, Fpbar, &mubar);
  }
  if (L.kind == kFluid) {
    const R J = det(Fnew);
    const R s = r_cbrt(J);
    const R tr = Fpbar(0, 0) + Fpbar(1, 1) + Fpbar(2, 2);
    return cofactor(Fnew) * (tr * s / (R(3) * J));
  }
  return Fpbar;
}

// ======================= SDF colliders =======================

template <class R>
struct BoxQ {
  R q[3], o[3], outside, d;
  bool out;
  v3<R> n;
  R sgn[3];
};

// Box SDF (mpm.hpp:98-128) from per-axis face offsets q (q_a = |rel_a| -
// half_a), o = max(q, 0) and the signs of rel, filled by each caller in one
// pass: a shared helper taking q[] / sg[] arrays, or a second pass over the
// record, quadrupled the grid adjoint's code (instruction-cache bound,
// measured: 2k -> 9k instructions).
#define DM_BOX_QUERY_BODY                                                              \
  b.outside = r_sqrt(b.o[0] * b.o[0] + b.o[1] * b.o[1] + b.o[2] * b.o[2] + R(1e-18)); \
  b.out = b.q[0] > R(0) || b.q[1] > R(0) || b.q[2] > R(0);                            \
  if (b.out) {                                                                        \
    b.d = b.outside - R(1e-9);                                                        \
    b.n = mk3(b.o[0] / b.outside, b.o[1] / b.outside, b.o[2] / b.outside);            \
  } else {                                                                            \
    b.d = r_min(r_max(b.q[0], r_max(b.q[1], b.q[2])), R(0));                          \
    b.n = zero3<R>();                                                                 \
    if (b.q[0] >= b.q[1] && b.q[0] >= b.q[2])                                         \
      b.n.x = R(1);                                                                   \
    else if (b.q[1] >= b.q[2])                                                        \
      b.n.y = R(1);                                                                   \
    else                                                                              \
      b.n.z = R(1);                                                                   \
  }                                                                                   \
  b.n = mk3(b.n.x * b.sgn[0], b.n.y * b.sgn[1], b.n.z * b.sgn[2])

template <class R>
DM_HD BoxQ<R> box_query(v3<R> rel, v3<R> half) {
  BoxQ<R> b;
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    b.q[a] = r_abs(rel[a]) - half[a];
    b.o[a] = r_max(b.q[a], R(0));
    b.sgn[a] = rel[a] < R(0) ? R(-1) : R(1);
  }
  DM_BOX_QUERY_BODY;
  return b;
}

// The open-top hollow box's cavity: a box open at the top (z extent shifted
// up by 1, rc = rel - e_z, hc = half + e_z); its z face offset
// |rel.z - 1| - (half.z + 1) = -(rel.z + half.z) for rel.z < 1 is taken
// directly (the shifted form rounds it to ~6e-8 in fp32, which
// exp(-alpha_c d) turns into ~6e-6 relative).
template <class R>
DM_HD BoxQ<R> cavity_query(v3<R> rel, v3<R> half) {
  BoxQ<R> b;
  b.q[0] = r_abs(rel.x) - half.x;
  b.q[1] = r_abs(rel.y) - half.y;
  b.q[2] = -(rel.z + half.z);
  b.o[0] = r_max(b.q[0], R(0));
  b.o[1] = r_max(b.q[1], R(0));
  b.o[2] = r_max(b.q[2], R(0));
  b.sgn[0] = rel.x < R(0) ? R(-1) : R(1);
  b.sgn[1] = rel.y < R(0) ? R(-1) : R(1);
  b.sgn[2] = R(-1);  // sign of rc.z (rel.z < 1 in the domain)
  DM_BOX_QUERY_BODY;
  return b;
}

// dbar, nbar -> rel_bar
template <class R>
DM_HD v3<R> box_query_vjp(const BoxQ<R>& b, v3<R> rel, R dbar, v3<R> nbar) {
  R qb[3] = {R(0), R(0), R(0)};
  if (b.out) {
    R ob[3];
    const R inv = R(1) / b.outside;
    const R ns = nbar.x * b.sgn[0] * b.o[0] + nbar.y * b.sgn[1] * b.o[1] + nbar.z * b.sgn[2] * b.o[2];
#pragma unroll
    for (int a = 0; a < 3; ++a) ob[a] = dbar * b.o[a] * inv + nbar[a] * b.sgn[a] * inv - b.o[a] * inv * inv * inv * ns;
#pragma unroll
    for (int a = 0; a < 3; ++a) qb[a] = b.q[a] > R(0) ? ob[a] : R(0);
  } else {
    const R M1 = r_max(b.q[1], b.q[2]);
    const R M = r_max(b.q[0], M1);
    if (M < R(0)) {
      if (b.q[0] > M1)
        qb[0] = dbar;
      else if (M1 > b.q[0]) {
        if (b.q[1] > b.q[2])
          qb[1] = dbar;
        else if (b.q[2] > b.q[1])
          qb[2] = dbar;
      }
    }
  }
  v3<R> rb;
#pragma unroll
  for (int a = 0; a < 3; ++a) rb[a] = qb[a] * (rel[a] > R(0) ? R(1) : (rel[a] < R(0) ? R(-1) : R(0)));
  return rb;
}

template <class R>
struct CylQ {
  v3<R> a, radial, er, eh;
  R h, rho, q0, q1, o0, o1, outside, d;
  bool out, radial_side;
  v3<R> n;
};

template <class R>
DM_HD CylQ<R> cyl_query(const Col<R>& col, v3<R> rel) {
  CylQ<R> c;
  c.a = col.nrm;
  c.h = dot(rel, c.a);
  c.radial = rel - c.a * c.h;
  c.rho = r_sqrt(dot(c.radial, c.radial) + R(1e-18));
  c.q0 = c.rho - col.radius;
  c.q1 = r_abs(c.h) - R(0.5) * col.length;
  c.o0 = r_max(c.q0, R(0));
  c.o1 = r_max(c.q1, R(0));
  c.outside = r_sqrt(c.o0 * c.o0 + c.o1 * c.o1 + R(1e-18));
  c.out = c.q0 > R(0) || c.q1 > R(0);
  c.er = c.radial * (R(1) / c.rho);
  c.eh = c.a * (c.h < R(0) ? R(-1) : R(1));
  c.radial_side = c.q0 >= c.q1;
  if (c.out) {
    c.d = c.outside - R(1e-9);
    c.n = c.er * (c.o0 / c.outside) + c.eh * (c.o1 / c.outside);
  } else {
    c.d = r_max(c.q0, c.q1);
    c.n = c.radial_side ? c.er : c.eh;
  }
  return c;
}

template <class R>
DM_HD v3<R> cyl_query_vjp(const CylQ<R>& c, R dbar, v3<R> nbar) {
  v3<R> erb = zero3<R>();
  R q0b = R(0), q1b = R(0);
  if (c.out) {
    const R inv = R(1) / c.outside;
    const R c0 = c.o0 * inv, c1 = c.o1 * inv;
    erb = nbar * c0;
    const R c0b = dot(nbar, c.er), c1b = dot(nbar, c.eh);
    R ob0 = c0b * inv, ob1 = c1b * inv;
    R outb = dbar - (c0b * c.o0 + c1b * c.o1) * inv * inv;
    ob0 += outb * c.o0 * inv;
    ob1 += outb * c.o1 * inv;
    q0b = c.q0 > R(0) ? ob0 : R(0);
    q1b = c.q1 > R(0) ? ob1 : R(0);
  } else {
    if (c.q0 > c.q1)
      q0b = dbar;
    else if (c.q1 > c.q0)
      q1b = dbar;
    if (c.radial_side) erb = nbar;
  }
  const R irho = R(1) / c.rho;
  v3<R> radb = (erb - c.er * dot(c.er, erb)) * irho;
  radb += c.radial * (q0b * irho);
  R hb = q1b * (c.h > R(0) ? R(1) : (c.h < R(0) ? R(-1) : R(0)));
  hb -= dot(c.a, radb);
  return radb + c.a * hb;
}

// Query: d, n at point p; relb(dbar, nbar) computed by collider_query_vjp.
// CK >= 0 fixes the collider kind at compile time (the switch folds: small
// code for single-kind batches); CK = -1 dispatches on col.kind.
template <class R, int CK = -1>
DM_HD void collider_query_body(const Col<R>& col, v3<R> rel, R& d, v3<R>& n) {
  switch (CK >= 0 ? CK : col.kind) {
    case kPlane:
      d = dot(rel, col.nrm);
      n = col.nrm;
      return;
    case kSphere: {
      const R r = r_sqrt(dot(rel, rel) + R(1e-18));
      d = r - col.radius;
      n = rel * (R(1) / r);
      return;
    }
    case kBox: {
      const BoxQ<R> b = box_query(rel, col.half);
      d = b.d;
      n = b.n;
      return;
    }
    case kCylinder: {
      const CylQ<R> c = cyl_query(col, rel);
      d = c.d;
      n = c.n;
      return;
    }
    default: {  // hollow open-top box
      const R th = col.thickness;
      const v3<R> ro = mk3(rel.x, rel.y, rel.z + R(0.5) * th);
      const v3<R> ho = mk3(col.half.x + th, col.half.y + th, col.half.z + R(0.5) * th);
      const BoxQ<R> bo = box_query(ro, ho);
      const BoxQ<R> bc = cavity_query(rel, col.half);
      if (bo.d >= -bc.d) {
        d = bo.d;
        n = bo.n;
      } else {
        d = -bc.d;
        n = -bc.n;
      }
      return;
    }
  }
}

// Out-of-line query (small code where several call sites or kinds meet:
// the adjoint kernels are instruction-cache bound); the forward node update
// with a compile-time kind inlines collider_query_body instead.
template <class R, int CK = -1>
DM_HD_NOINLINE void collider_query_r(const Col<R>& col, v3<R> rel, R& d, v3<R>& n) {
  collider_query_body<R, CK>(col, rel, d, n);
}

template <class R, int CK = -1>
DM_HD void collider_query(const Col<R>& col, v3<R> p, R& d, v3<R>& n) {
  collider_query_r<R, CK>(col, p - col.c, d, n);
}

// Returns pbar (gradient w.r.t. the query point; center gets -pbar).
template <class R, int CK = -1>
DM_HD_NOINLINE v3<R> collider_query_vjp(const Col<R>& col, v3<R> p, R dbar, v3<R> nbar) {
  const v3<R> rel = p - col.c;
  switch (CK >= 0 ? CK : col.kind) {
    case kPlane:
      return col.nrm * dbar;
    case kSphere: {
      const R r = r_sqrt(dot(rel, rel) + R(1e-18));
      const v3<R> n = rel * (R(1) / r);
      return n * dbar + (nbar - n * dot(n, nbar)) * (R(1) / r);
    }
    case kBox: {
      const BoxQ<R> b = box_query(rel, col.half);
      return box_query_vjp(b, rel, dbar, nbar);
    }
    case kCylinder: {
      const CylQ<R> c = cyl_query(col, rel);
      return cyl_query_vjp(c, dbar, nbar);
    }
    default: {
      const R th = col.thickness;
      const v3<R> ro = mk3(rel.x, rel.y, rel.z + R(0.5) * th);
      const v3<R> ho = mk3(col.half.x + th, col.half.y + th, col.half.z + R(0.5) * th);
      const v3<R> rc = mk3(rel.x, rel.y, rel.z - R(1));
      const v3<R> hc = mk3(col.half.x, col.half.y, col.half.z + R(1));
      const BoxQ<R> bo = box_query(ro, ho);
      const BoxQ<R> bc = cavity_query(rel, col.half);
      // one inlined vjp on the active branch (outer box, or the cavity with
      // negated cotangents) keeps the code compact
      const bool outer = bo.d >= -bc.d;
      const R sg = outer ? R(1) : R(-1);
      return box_query_vjp(outer ? bo : bc, outer ? ro : rc, sg * dbar, nbar * sg);
    }
  }
}

// Query record for a compile-time collider kind (CK >= 0): the node update
// adjoint queries the SDF once and reuses the record for the forward
// recompute, the coupling adjoint and the SDF adjoint (previously three
// queries per node).  Same arithmetic as collider_query /
// collider_query_vjp, so the results are bitwise unchanged.
template <class R>
struct ColRec {
  R d, sg, r;
  v3<R> n, rel;
  BoxQ<R> b;
  CylQ<R> cy;
};

template <class R, int CK>
DM_HD void collider_query_rec(const Col<R>& col, v3<R> p, ColRec<R>& q) {
  const v3<R> rel = p - col.c;
  if (CK == kPlane) {
    q.d = dot(rel, col.nrm);
    q.n = col.nrm;
  } else if (CK == kSphere) {
    q.r = r_sqrt(dot(rel, rel) + R(1e-18));
    q.d = q.r - col.radius;
    q.n = rel * (R(1) / q.r);
  } else if (CK == kBox) {
    q.b = box_query(rel, col.half);
    q.rel = rel;
    q.d = q.b.d;
    q.n = q.b.n;
  } else if (CK == kCylinder) {
    q.cy = cyl_query(col, rel);
    q.d = q.cy.d;
    q.n = q.cy.n;
  } else {  // hollow open-top box
    const R th = col.thickness;
    const v3<R> ro = mk3(rel.x, rel.y, rel.z + R(0.5) * th);
    const v3<R> ho = mk3(col.half.x + th, col.half.y + th, col.half.z + R(0.5) * th);
    const v3<R> rc = mk3(rel.x, rel.y, rel.z - R(1));
    const v3<R> hc = mk3(col.half.x, col.half.y, col.half.z + R(1));
    const BoxQ<R> bo = box_query(ro, ho);
    const BoxQ<R> bc = cavity_query(rel, col.half);
    const bool outer = bo.d >= -bc.d;
    q.b = outer ? bo : bc;
    q.rel = outer ? ro : rc;
    q.sg = outer ? R(1) : R(-1);
    q.d = outer ? bo.d : -bc.d;
    q.n = outer ? bo.n : -bc.n;
  }
}

template <class R, int CK>
DM_HD v3<R> collider_query_vjp_rec(const Col<R>& col, const ColRec<R>& q, R dbar, v3<R> nbar) {
  if (CK == kPlane) return col.nrm * dbar;
  if (CK == kSphere) return q.n * dbar + (nbar - q.n * dot(q.n, nbar)) * (R(1) / q.r);
  if (CK == kBox) return box_query_vjp(q.b, q.rel, dbar, nbar);
  if (CK == kCylinder) return cyl_query_vjp(q.cy, dbar, nbar);
  return box_query_vjp(q.b, q.rel, q.sg * dbar, nbar * q.sg);
}

// collide / collide_vjp on a query record (same arithmetic as below).
template <class R>
DM_HD v3<R> collide_rec(const Col<R>& col, R alpha_c, R mu_b, v3<R> node, v3<R> v, const ColRec<R>& q) {
  const R d = q.d;
  const v3<R> n = q.n;
  const R s = d < R(0) ? R(1) : r_exp(-alpha_c * r_max(d, R(0)));
  const v3<R> vcol = col.vel + cross(col.om, node - col.c);
  const v3<R> rel = v - vcol;
  const R vn = dot(rel, n);
  if (!(vn < R(0))) return v;
  const v3<R> tang = rel - n * vn;
  const R tnorm = r_sqrt(dot(tang, tang) + R(1e-18));
  const R keep = r_max(R(1) - mu_b * r_max(-vn, R(0)) / tnorm, R(0));
  const v3<R> vproj = vcol + tang * keep + n * r_max(vn, R(0));
  return v * (R(1) - s) + vproj * s;
}

// ======================= grid node update =======================

struct Coupling {
  float alpha_c, mu_b;
};

// One collider applied to node velocity v (mpm.hpp:275-294 + rotation).
template <class R, int CK = -1>
DM_HD v3<R> collide(const Col<R>& col, R alpha_c, R mu_b, v3<R> node, v3<R> v) {
  R d;
  v3<R> n;
  collider_query<R, CK>(col, node, d, n);
  const R s = d < R(0) ? R(1) : r_exp(-alpha_c * r_max(d, R(0)));
  const v3<R> vcol = col.vel + cross(col.om, node - col.c);
  const v3<R> rel = v - vcol;
  const R vn = dot(rel, n);
  if (!(vn < R(0))) return v;
  const v3<R> tang = rel - n * vn;
  const R tnorm = r_sqrt(dot(tang, tang) + R(1e-18));
  const R keep = r_max(R(1) - mu_b * r_max(-vn, R(0)) / tnorm, R(0));
  const v3<R> vproj = vcol + tang * keep + n * r_max(vn, R(0));
  return v * (R(1) - s) + vproj * s;
}

// Adjoint of collide: given vout_bar, returns v_bar and accumulates the
// collider's center / velocity / omega cotangents.
template <class R, int CK = -1>
DM_HD_NOINLINE v3<R> collide_vjp(const Col<R>& col, R alpha_c, R mu_b, v3<R> node, v3<R> v, v3<R> vb_out, v3<R>& cbar,
                        v3<R>& velbar, v3<R>& ombar) {
  R d;
  v3<R> n;
  collider_query<R, CK>(col, node, d, n);
  const v3<R> r = node - col.c;
  const v3<R> vcol = col.vel + cross(col.om, r);
  const v3<R> rel = v - vcol;
  const R vn = dot(rel, n);
  if (!(vn < R(0))) return vb_out;
  const R s = d < R(0) ? R(1) : r_exp(-alpha_c * r_max(d, R(0)));
  const v3<R> tang = rel - n * vn;
  const R tnorm = r_sqrt(dot(tang, tang) + R(1e-18));
  const R m = r_max(-vn, R(0));
  const R kk = R(1) - mu_b * m / tnorm;
  const R keep = r_max(kk, R(0));
  const v3<R> vproj = vcol + tang * keep + n * r_max(vn, R(0));
  // v' = v (1 - s) + vproj s
  v3<R> vb = vb_out * (R(1) - s);
  const R sb = dot(vproj - v, vb_out);
  const v3<R> vpb = vb_out * s;
  v3<R> vcolb = vpb;
  v3<R> tangb = vpb * keep;
  const R keepb = dot(tang, vpb);
  v3<R> nb = zero3<R>();  // n * max(vn, 0): vn < 0 here -> no contribution
  R vnb = R(0);
  if (kk > R(0)) {
    const R mb = -keepb * mu_b / tnorm;
    const R tnb = keepb * mu_b * m / (tnorm * tnorm);
    tangb += tang * (tnb / tnorm);
    if (-vn > R(0)) vnb -= mb;
  }
  // tang = rel - n vn
  v3<R> relb = tangb;
  nb -= tangb * vn;
  vnb -= dot(n, tangb);
  // vn = rel . n
  relb += n * vnb;
  nb += rel * vnb;
  // rel = v - vcol
  vb += relb;
  vcolb -= relb;
  // s = exp(-alpha max(d, 0)) for d >= 0
  R db = R(0);
  if (!(d < R(0)) && d > R(0)) db = -alpha_c * s * sb;
  // vcol = vel + om x r
  velbar += vcolb;
  ombar += cross(r, vcolb);
  const v3<R> rb = cross(vcolb, col.om);
  cbar -= rb;
  // query
  cbar -= collider_query_vjp<R, CK>(col, node, db, nb);
  return vb;
}

template <class R, int CK>
DM_HD v3<R> collide_vjp_rec(const Col<R>& col, R alpha_c, R mu_b, v3<R> node, v3<R> v, v3<R> vb_out, const ColRec<R>& q, v3<R>& cbar,
                        v3<R>& velbar, v3<R>& ombar) {
  const R d = q.d;
  const v3<R> n = q.n;
  const v3<R> r = node - col.c;
  const v3<R> vcol = col.vel + cross(col.om, r);
  const v3<R> rel = v - vcol;
  const R vn = dot(rel, n);
  if (!(vn < R(0))) return vb_out;
  const R s = d < R(0) ? R(1) : r_exp(-alpha_c * r_max(d, R(0)));
  const v3<R> tang = rel - n * vn;
  const R tnorm = r_sqrt(dot(tang, tang) + R(1e-18));
  const R m = r_max(-vn, R(0));
  const R kk = R(1) - mu_b * m / tnorm;
  const R keep = r_max(kk, R(0));
  const v3<R> vproj = vcol + tang * keep + n * r_max(vn, R(0));
  // v' = v (1 - s) + vproj s
  v3<R> vb = vb_out * (R(1) - s);
  const R sb = dot(vproj - v, vb_out);
  const v3<R> vpb = vb_out * s;
  v3<R> vcolb = vpb;
  v3<R> tangb = vpb * keep;
  const R keepb = dot(tang, vpb);
  v3<R> nb = zero3<R>();  // n * max(vn, 0): vn < 0 here -> no contribution
  R vnb = R(0);
  if (kk > R(0)) {
    const R mb = -keepb * mu_b / tnorm;
    const R tnb = keepb * mu_b * m / (tnorm * tnorm);
    tangb += tang * (tnb / tnorm);
    if (-vn > R(0)) vnb -= mb;
  }
  // tang = rel - n vn
  v3<R> relb = tangb;
  nb -= tangb * vn;
  vnb -= dot(n, tangb);
  // vn = rel . n
  relb += n * vnb;
  nb += rel * vnb;
  // rel = v - vcol
  vb += relb;
  vcolb -= relb;
  // s = exp(-alpha max(d, 0)) for d >= 0
  R db = R(0);
  if (!(d < R(0)) && d > R(0)) db = -alpha_c * s * sb;
  // vcol = vel + om x r
  velbar += vcolb;
  ombar += cross(r, vcolb);
  const v3<R> rb = cross(vcolb, col.om);
  cbar -= rb;
  // query
  cbar -= collider_query_vjp_rec<R, CK>(col, q, db, nb);
  return vb;
}

template <class R>
struct NodeCtx {
  int dims[3];
  R dx, dt;
  R dx_lo;  // fp32: dx - (float)dx, so node - center = i dx - c rounds once (node_rel)
  v3<R> gravity;
  int boundary;
  R alpha_c, mu_b;
};

// Domain boundary (mpm.hpp:296-302; sticky extension).  Returns the mask of
// components that were zeroed.
template <class R>
DM_HD int boundary_apply(const NodeCtx<R>& g, const int idx[3], v3<R>& v) {
  const int bound = 3;
  int mask = 0;
  if (g.boundary == kSticky) {
    bool band = false;
#pragma unroll
    for (int a = 0; a < 3; ++a) band = band || idx[a] < bound || idx[a] >= g.dims[a] - bound;
    if (band) {
      v = zero3<R>();
      mask = 7;
    }
    return mask;
  }
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    if ((idx[a] < bound && v[a] < R(0)) || (idx[a] >= g.dims[a] - bound && v[a] > R(0))) {
      v[a] = R(0);
      mask |= 1 << a;
    }
  }
  return mask;
}

// Forward node update; returns velocity.  mass <= 0 -> zero (mpm.hpp:265-268).
template <class R, int MAXC, int CK = -1>
DM_HD v3<R> node_update(const NodeCtx<R>& g, const Col<R>* cols, int ncol, const int idx[3], R mass, v3<R> mom) {
  if (!(mass > R(0))) return zero3<R>();
  const R inv = R(1) / mass;
  v3<R> v = mom * inv;
  v.x += g.dt * g.gravity.x;
  v.y += g.dt * g.gravity.y;
  v.z += g.dt * g.gravity.z;
  const v3<R> node = mk3(R(idx[0]) * g.dx, R(idx[1]) * g.dx, R(idx[2]) * g.dx);
  for (int c = 0; c < ncol && c < MAXC; ++c) v = collide<R, CK>(cols[c], g.alpha_c, g.mu_b, node, v);
  boundary_apply(g, idx, v);
  return v;
}

// ---- forward node update in a moving frame ----
// The forward transfers run relative to a per-env reference velocity vref
// (constant during the substep; k_bin: mean velocity of the env's first
// particles): P2G accumulates momentum relative to vref, the grid holds
// dv = v - vref and G2P adds vref back.  Galilean shifts commute with every
// step (momentum sums, gravity, the lab-frame collider and boundary
// projections, the B-spline's zero first moment), so the values are the
// reference's; fp32 then resolves velocity differences between nodes that
// are orders of magnitude below the common velocity (a settling body: C dx
// ~ 1e-3 |v| rounds to ~1e-4 relative in the lab frame, SURVEY 8(d)'s
// per-substep 1e-5 gate).  The adjoints linearise in the lab frame.

// node position minus c, i dx - c with one rounding (dx split in two words):
// the SDF distance feeds exp(-alpha_c d), which turns a 3e-8 position
// rounding into ~3e-6 relative at alpha_c = 100.
template <class R>
DM_HD v3<R> node_rel(const NodeCtx<R>& g, const int idx[3], v3<R> c) {
  v3<R> r;
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    const R i = R(idx[a]);
#ifdef __CUDA_ARCH__
    if constexpr (sizeof(R) == 4) {
      r[a] = fmaf(i, g.dx, fmaf(i, g.dx_lo, -c[a]));
      continue;
    }
#endif
    r[a] = i * g.dx + (i * g.dx_lo - c[a]);
  }
  return r;
}

// Increment of collide (mpm.hpp:275-294): v_out - v for lab velocity
// v = vref + dv.  For an approaching node (v_n < 0, max(v_n, 0) = 0):
// v_out - v = s (v_proj - v) = -s (n v_n + tang (1 - keep)).
template <class R, int CK = -1>
DM_HD v3<R> collide_delta(const Col<R>& col, R alpha_c, R mu_b, v3<R> node, v3<R> rel_c, v3<R> vref, v3<R> dv) {
  R d;
  v3<R> n;
  if constexpr (CK >= 0)
    collider_query_body<R, CK>(col, rel_c, d, n);
  else
    collider_query_r<R, CK>(col, rel_c, d, n);
  const R s = d < R(0) ? R(1) : r_exp(-alpha_c * r_max(d, R(0)));
  const v3<R> vcol = col.vel + cross(col.om, node - col.c);
  const v3<R> rel = (vref - vcol) + dv;
  const R vn = dot(rel, n);
  if (!(vn < R(0))) return zero3<R>();
  const v3<R> tang = rel - n * vn;
  const R tnorm = r_sqrt(dot(tang, tang) + R(1e-18));
  const R keep = r_max(R(1) - mu_b * r_max(-vn, R(0)) / tnorm, R(0));
  return (n * vn + tang * (R(1) - keep)) * (-s);
}

// node_update (mpm.hpp:256-305) from the momentum relative to vref
// (momr = mom - mass vref); returns dv = v_new - vref.
template <class R, int MAXC, int CK = -1>
DM_HD v3<R> node_update_rel(const NodeCtx<R>& g, const Col<R>* cols, int ncol, const int idx[3], R mass, v3<R> momr,
                            v3<R> vref) {
  if (!(mass > R(0))) return zero3<R>() - vref;  // v = 0 (mpm.hpp:265-268)
  const R inv = R(1) / mass;
  v3<R> dv = momr * inv;
  dv.x += g.dt * g.gravity.x;
  dv.y += g.dt * g.gravity.y;
  dv.z += g.dt * g.gravity.z;
  const v3<R> node = mk3(R(idx[0]) * g.dx, R(idx[1]) * g.dx, R(idx[2]) * g.dx);
  for (int c = 0; c < ncol && c < MAXC; ++c)
    dv += collide_delta<R, CK>(cols[c], g.alpha_c, g.mu_b, node, node_rel(g, idx, cols[c].c), vref, dv);
  // domain boundary on the lab-frame velocity (mpm.hpp:296-302)
  const int bound = 3;
  if (g.boundary == kSticky) {
    bool band = false;
#pragma unroll
    for (int a = 0; a < 3; ++a) band = band || idx[a] < bound || idx[a] >= g.dims[a] - bound;
    if (band) dv = zero3<R>() - vref;
    return dv;
  }
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    const R va = vref[a] + dv[a];
    if ((idx[a] < bound && va < R(0)) || (idx[a] >= g.dims[a] - bound && va > R(0))) dv[a] = -vref[a];
  }
  return dv;
}

// Node adjoint: from vbar_out to (mass_bar, mom_bar); collider cotangents
// accumulated into cgrad[c*9 + {0..8}] (center, velocity, omega).
template <class R, int MAXC, int CK = -1>
DM_HD void node_update_vjp(const NodeCtx<R>& g, const Col<R>* cols, int ncol, const int idx[3], R mass, v3<R> mom,
                           v3<R> vb, R& massb, v3<R>& momb, R* cgrad) {
  massb = R(0);
  momb = zero3<R>();
  if (!(mass > R(0))) return;
  const R inv = R(1) / mass;
  v3<R> v0 = mom * inv;
  v0.x += g.dt * g.gravity.x;
  v0.y += g.dt * g.gravity.y;
  v0.z += g.dt * g.gravity.z;
  const v3<R> node = mk3(R(idx[0]) * g.dx, R(idx[1]) * g.dx, R(idx[2]) * g.dx);
  if (CK >= 0 && MAXC == 1) {  // dispatched only for batches with exactly one collider
    // one compile-time collider: one SDF query per node (query record)
    ColRec<R> q;
    collider_query_rec<R, CK>(cols[0], node, q);
    v3<R> vfin = collide_rec(cols[0], g.alpha_c, g.mu_b, node, v0, q);
    const int mask = boundary_apply(g, idx, vfin);
#pragma unroll
    for (int a = 0; a < 3; ++a)
      if (mask & (1 << a)) vb[a] = R(0);
    v3<R> cb = zero3<R>(), velb = zero3<R>(), omb = zero3<R>();
    vb = collide_vjp_rec<R, CK>(cols[0], g.alpha_c, g.mu_b, node, v0, vb, q, cb, velb, omb);
    cgrad[0] += cb.x;
    cgrad[1] += cb.y;
    cgrad[2] += cb.z;
    cgrad[3] += velb.x;
    cgrad[4] += velb.y;
    cgrad[5] += velb.z;
    cgrad[6] += omb.x;
    cgrad[7] += omb.y;
    cgrad[8] += omb.z;
    momb = vb * inv;
    massb = -dot(vb, mom) * inv * inv;
    return;
  }
  v3<R> vs[MAXC + 1];
  vs[0] = v0;
  const int nc = ncol < MAXC ? ncol : MAXC;
  for (int c = 0; c < nc; ++c) vs[c + 1] = collide<R, CK>(cols[c], g.alpha_c, g.mu_b, node, vs[c]);
  v3<R> vfin = vs[nc];
  const int mask = boundary_apply(g, idx, vfin);
#pragma unroll
  for (int a = 0; a < 3; ++a)
    if (mask & (1 << a)) vb[a] = R(0);
  for (int c = nc - 1; c >= 0; --c) {
    v3<R> cb = zero3<R>(), velb = zero3<R>(), omb = zero3<R>();
    vb = collide_vjp<R, CK>(cols[c], g.alpha_c, g.mu_b, node, vs[c], vb, cb, velb, omb);
    R* o = cgrad + 9 * c;
    o[0] += cb.x;
    o[1] += cb.y;
    o[2] += cb.z;
    o[3] += velb.x;
    o[4] += velb.y;
    o[5] += velb.z;
    o[6] += omb.x;
    o[7] += omb.y;
    o[8] += omb.z;
  }
  momb = vb * inv;
  massb = -dot(vb, mom) * inv * inv;
}

// ======================= B-spline stencil =======================

template <class R>
DM_HD void bspline(R fx, R w[3]) {  // mpm.hpp:141-147
  w[0] = R(0.5) * (R(1.5) - fx) * (R(1.5) - fx);
  w[1] = R(0.75) - (fx - R(1)) * (fx - R(1));
  w[2] = R(0.5) * (fx - R(0.5)) * (fx - R(0.5));
}
template <class R>
DM_HD void bspline_d(R fx, R dw[3]) {
  dw[0] = fx - R(1.5);
  dw[1] = R(-2) * (fx - R(1));
  dw[2] = fx - R(0.5);
}

}  // namespace dm
