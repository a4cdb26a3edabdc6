// Per-particle MLS-MPM transfers (quadratic B-spline APIC) and their adjoints.
// Restates p2g (mpm.hpp:219-254) and g2p (mpm.hpp:307-346); node access goes
// through a functor so the same code serves the shared-memory tile kernels
// and the host fp64 adjoint check.
#pragma once

#include "dm_physics.cuh"

namespace dm {

// fp32 products/differences that must not be contracted into FMAs, so the
// stencil base (and therefore the bin key) is bit-reproducible on host and
// device (SURVEY.md 8(d) "Binning").
DM_HD float mul_rn(float a, float b) {
#ifdef __CUDA_ARCH__
  return __fmul_rn(a, b);
#else
  volatile float r = a * b;
  return r;
#endif
}
DM_HD float sub_rn(float a, float b) {
#ifdef __CUDA_ARCH__
  return __fsub_rn(a, b);
#else
  volatile float r = a - b;
  return r;
#endif
}

template <class R>
struct Stencil {
  int base[3];
  R fx[3];
  R w[3][3];   // w[axis][offset]
  R dw[3][3];  // d w / d fx
};

// Base cell + fractional offset.  fp32: gx = fl(x * inv_dx),
// base = floor(fl(gx - 0.5)), fx = fl(gx - base).  fp64 (host check): the
// reference's double division for base (mpm.hpp:153-154) and multiplication
// for fx (mpm.hpp:159).  Returns the first failing axis or -1.
// The interior test (1 <= base <= dims-4, mpm.hpp:155) is done on the float
// floor, before any integer conversion, so NaN/inf/huge positions are caught;
// a failing axis is clamped into range so every consumer stays in bounds
// while the error is reported.
DM_HD int stencil_base(const float x[3], float inv_dx, double dx, const int dims[3], int base[3], float fx[3]) {
  int bad = -1;
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    const float gx = mul_rn(x[a], inv_dx);
    const float b = floorf(sub_rn(gx, 0.5f));
    const bool ok = b >= 1.f && b <= static_cast<float>(dims[a] - 4);
    base[a] = ok ? static_cast<int>(b) : 1;
    fx[a] = ok ? sub_rn(gx, b) : 1.f;
    if (!ok && bad < 0) bad = a;
  }
  return bad;
}
DM_HD int stencil_base(const double x[3], double inv_dx, double dx, const int dims[3], int base[3], double fx[3]) {
  int bad = -1;
  for (int a = 0; a < 3; ++a) {
    const double b = floor(x[a] / dx - 0.5);
    const bool ok = b >= 1.0 && b <= static_cast<double>(dims[a] - 4);
    base[a] = ok ? static_cast<int>(b) : 1;
    fx[a] = ok ? x[a] * inv_dx - b : 1.0;
    if (!ok && bad < 0) bad = a;
  }
  return bad;
}

template <class R>
DM_HD int make_stencil(const R x[3], R inv_dx, double dx, const int dims[3], Stencil<R>& s) {
  const int bad = stencil_base(x, inv_dx, dx, dims, s.base, s.fx);
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    bspline(s.fx[a], s.w[a]);
    bspline_d(s.fx[a], s.dw[a]);
  }
  return bad;
}

template <class R>
struct TransferCtx {
  int dims[3];
  R dx, inv_dx, dt;
  double dx64;
};

// ---------------- P2G ----------------
// Affine momentum matrix A = -dt V0 4/dx^2 (P F^T + J eta (C + C^T)) + m C
// (mpm.hpp:236-239 + viscosity extension).  The node at offset o receives
//   mass: w_o m,   momentum: w_o (m v + A dpos_o),  dpos_o = (o - fx) dx
// written as w_o (q + Ad o) with q = m v - A fx dx and Ad = A dx.
// D = F - I (the stored deviation; law_stress_fwd).
template <class R>
DM_HD m3<R> p2g_affine(const Law<R>& L, const TransferCtx<R>& t, const m3<R>& D, const m3<R>& C, R act, bool* bad) {
  const m3<R> P = law_stress_fwd(L, D, act, bad);
  m3<R> tau = P + mul_bt(P, D);  // P F^T
  if (L.kind == kFluid && L.visc != R(0)) {
    const R jv = (R(1) + det1m(D)) * L.visc;
    tau += (C + transpose(C)) * jv;
  }
  const R kA = -t.dt * L.vol * R(4) * t.inv_dx * t.inv_dx;
  return tau * kA + C * L.mass;
}

// p2g_affine from a cached Kirchhoff stress tau = P F^T (elastoplastic: the
// G2P projection's value, no viscosity term).
template <class R>
DM_HD m3<R> p2g_affine_tau(const Law<R>& L, const TransferCtx<R>& t, const m3<R>& tau, const m3<R>& C) {
  const R kA = -t.dt * L.vol * R(4) * t.inv_dx * t.inv_dx;
  return tau * kA + C * L.mass;
}

template <class R>
DM_HD void p2g_payload(const m3<R>& A, R mass, v3<R> v, const Stencil<R>& s, R dx, v3<R>& q, m3<R>& Ad) {
  const v3<R> f = mk3(s.fx[0] * dx, s.fx[1] * dx, s.fx[2] * dx);
  q = v * mass - A * f;
  Ad = A * dx;
}

// ---------------- G2P ----------------
template <class R, class GetV>
DM_HD void g2p_gather(const Stencil<R>& s, R dx, GetV getv, v3<R>& vnew, m3<R>& B) {
  vnew = zero3<R>();
  B = mzero<R>();
#pragma unroll
  for (int i = 0; i < 3; ++i)
#pragma unroll
    for (int j = 0; j < 3; ++j)
#pragma unroll
      for (int k = 0; k < 3; ++k) {
        const R w = s.w[0][i] * s.w[1][j] * s.w[2][k];
        const v3<R> vw = getv(i, j, k) * w;
        const v3<R> dpos = mk3((R(i) - s.fx[0]) * dx, (R(j) - s.fx[1]) * dx, (R(k) - s.fx[2]) * dx);
        vnew += vw;
        B += outer(vw, dpos);
      }
}

// Forward G2P for one particle: returns new (x, v, C, F); *bad_adv when the
// advected particle leaves [1.5, dims-2.5] cells (mpm.hpp:335-340).
template <class R, class GetV>
DM_HD void g2p_particle(const Law<R>& L, const TransferCtx<R>& t, const Stencil<R>& s, GetV getv, v3<R>& x, v3<R>& v,
                        m3<R>& C, m3<R>& F, bool* bad_adv, bool* bad_det) {
  m3<R> B;
  g2p_gather(s, t.dx, getv, v, B);
  C = B * (R(4) * t.inv_dx * t.inv_dx);
  x.x += t.dt * v.x;
  x.y += t.dt * v.y;
  x.z += t.dt * v.z;
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    const R gx = x[a] / t.dx;
    if (!(gx >= R(1.5) && gx <= R(t.dims[a]) - R(2.5))) *bad_adv = true;  // NaN-safe
  }
  const m3<R> Fnew = (meye<R>() + C * t.dt) * F;
  F = law_project(L, Fnew, bad_det);
}

// Adjoint of g2p_particle.  Inputs: start-of-substep x (via stencil s), F;
// output cotangents xb', vb', Cb', Fb'.  Produces the particle-side partial
// cotangents (xb_part, Fb_part) and the node-scatter payload:
//   vbar_node(o) += w_o (gq + Bd o)   with gq = gbar - Bbar fx dx, Bd = Bbar dx.
template <class R, class GetV>
DM_HD void g2p_vjp(const Law<R>& L, const TransferCtx<R>& t, const Stencil<R>& s, GetV getv, const m3<R>& F,
                   v3<R> xb_o, v3<R> vb_o, const m3<R>& Cb_o, const m3<R>& Fb_o, v3<R>& xb_part, m3<R>& Fb_part,
                   v3<R>& gq, m3<R>& Bd, R& mubar) {
  // recompute forward
  v3<R> vnew;
  m3<R> B;
  g2p_gather(s, t.dx, getv, vnew, B);
  const R c4 = R(4) * t.inv_dx * t.inv_dx;
  const m3<R> Cn = B * c4;
  const m3<R> Ad = meye<R>() + Cn * t.dt;
  const m3<R> Fnew = Ad * F;
  const m3<R> Fnb = law_project_vjp(L, Fnew, Fb_o, mubar);
  // Fnew = (I + dt C) F
  const m3<R> Cb = Cb_o + mul_bt(Fnb, F) * t.dt;
  Fb_part = mul_at(Ad, Fnb);
  // x' = x + dt v' ;  C = c4 B
  const v3<R> gb = vb_o + xb_o * t.dt;
  const m3<R> Bb = Cb * c4;
  // per node: u = gb + Bb dpos; vbar_n += w u; wbar = v_n . u; dposbar = w Bb^T v_n
  R fxb[3] = {R(0), R(0), R(0)};
#pragma unroll
  for (int i = 0; i < 3; ++i)
#pragma unroll
    for (int j = 0; j < 3; ++j)
#pragma unroll
      for (int k = 0; k < 3; ++k) {
        const R w = s.w[0][i] * s.w[1][j] * s.w[2][k];
        const v3<R> vn = getv(i, j, k);
        const v3<R> dpos = mk3((R(i) - s.fx[0]) * t.dx, (R(j) - s.fx[1]) * t.dx, (R(k) - s.fx[2]) * t.dx);
        const v3<R> u = gb + Bb * dpos;
        const R wb = dot(vn, u);
        fxb[0] += wb * s.dw[0][i] * s.w[1][j] * s.w[2][k];
        fxb[1] += wb * s.w[0][i] * s.dw[1][j] * s.w[2][k];
        fxb[2] += wb * s.w[0][i] * s.w[1][j] * s.dw[2][k];
        const v3<R> dpb = tmul(Bb, vn) * w;
        fxb[0] -= t.dx * dpb.x;
        fxb[1] -= t.dx * dpb.y;
        fxb[2] -= t.dx * dpb.z;
      }
  xb_part = mk3(xb_o.x + fxb[0] * t.inv_dx, xb_o.y + fxb[1] * t.inv_dx, xb_o.z + fxb[2] * t.inv_dx);
  const v3<R> f = mk3(s.fx[0] * t.dx, s.fx[1] * t.dx, s.fx[2] * t.dx);
  gq = gb - Bb * f;
  Bd = Bb * t.dx;
}

// Adjoint of the P2G for one particle, given node cotangents (mass_bar,
// mom_bar) through getmb(i,j,k, mb, pb).  Adds into xb, vb, Fb, Cb, and the
// material / actuation cotangents.
template <class R, class GetMB>
DM_HD void p2g_vjp(const Law<R>& L, const TransferCtx<R>& t, const Stencil<R>& s, GetMB getmb, v3<R> v, const m3<R>& F,
                   const m3<R>& C, R act, v3<R>& xb, v3<R>& vb, m3<R>& Fb, m3<R>& Cb, R& mubar, R& lambar, R& actbar) {
  bool bad = false;
  const m3<R> P = law_stress(L, F, act, &bad);
  m3<R> tau = mul_bt(P, F);
  const bool visc = L.kind == kFluid && L.visc != R(0);
  const m3<R> Cs = C + transpose(C);
  const R J = det(F);
  if (visc) tau += Cs * (J * L.visc);
  const R kA = -t.dt * L.vol * R(4) * t.inv_dx * t.inv_dx;
  const m3<R> A = tau * kA + C * L.mass;
  const v3<R> mv = v * L.mass;
  R fxb[3] = {R(0), R(0), R(0)};
  v3<R> S = zero3<R>();
  m3<R> Ab = mzero<R>();
#pragma unroll
  for (int i = 0; i < 3; ++i)
#pragma unroll
    for (int j = 0; j < 3; ++j)
#pragma unroll
      for (int k = 0; k < 3; ++k) {
        const R w = s.w[0][i] * s.w[1][j] * s.w[2][k];
        R mb;
        v3<R> pb;
        getmb(i, j, k, mb, pb);
        const v3<R> dpos = mk3((R(i) - s.fx[0]) * t.dx, (R(j) - s.fx[1]) * t.dx, (R(k) - s.fx[2]) * t.dx);
        const v3<R> u = mv + A * dpos;
        const R wb = mb * L.mass + dot(pb, u);
        fxb[0] += wb * s.dw[0][i] * s.w[1][j] * s.w[2][k];
        fxb[1] += wb * s.w[0][i] * s.dw[1][j] * s.w[2][k];
        fxb[2] += wb * s.w[0][i] * s.w[1][j] * s.dw[2][k];
        const v3<R> ub = pb * w;
        S += ub;
        Ab += outer(ub, dpos);
        const v3<R> dpb = tmul(A, ub);
        fxb[0] -= t.dx * dpb.x;
        fxb[1] -= t.dx * dpb.y;
        fxb[2] -= t.dx * dpb.z;
      }
  xb += mk3(fxb[0] * t.inv_dx, fxb[1] * t.inv_dx, fxb[2] * t.inv_dx);
  vb += S * L.mass;
  Cb += Ab * L.mass;
  const m3<R> taub = Ab * kA;
  if (visc) {
    Cb += (taub + transpose(taub)) * (J * L.visc);
    Fb += cofactor(F) * (L.visc * ddot(Cs, taub));
  }
  // tau = P F^T
  const m3<R> Pb = taub * F;
  Fb += mul_at(taub, P);
  law_stress_vjp(L, F, act, Pb, Fb, mubar, lambar, actbar);
}


// ---------------- separable-stencil fast paths ----------------
// The quadratic B-spline weight factorises, w_ijk = wx_i wy_j wz_k, and every
// sum the transfers need is linear in the node offset o = (i,j,k):
//   sum_n w_n f_n (o_n - fx) dx = dx (M - (sum_n w_n f_n) fx^T),
//   M[:, c] = sum_n w_n f_n o_c = A_c[1] + 2 A_c[2]  with per-axis partial sums
// A_x[i] = sum_{jk} w f, A_y[j] = sum_{ik} w f, A_z[k] = sum_{ij} w f.
// This replaces the per-node outer products of the literal restatement
// (mpm.hpp:241-252, 321-331) by 9 FMAs per node.

// Factored over the separable weight (w_ijk = wij wz_k, wij = wx_i wy_j):
//   R_ij = sum_k wz_k v_ijk,  ax[i] = sum_j wij R_ij,  ay[j] = sum_i wij R_ij,
//   az[k] = wz_k sum_ij wij v_ijk     (~8 FMAs per node instead of 13)
//
// Centred on the stencil's middle node velocity v_c: B = sum w (v_n - v_c)
// (o - fx) dx (the v_c (sum w (o - fx)) dx term is zero -- the quadratic
// B-spline's first moment -- and is dropped) and v' = v_c + sum w (v_n - v_c).
// For a near-uniform grid velocity (a body at rest, free fall) the affine
// matrix is a small difference of O(|v|) sums: uncentred, fp32 rounding of
// those sums leaves ~1e-7 |v| / dx of noise in C, above the per-substep 1e-5
// gate when |C| dx << |v|.
template <class R, class GetV>
DM_HD void g2p_gather_sep(const Stencil<R>& s, R dx, GetV getv, v3<R>& vnew, m3<R>& B) {
  v3<R> ax[3], ay[3], az[3];
#pragma unroll
  for (int q = 0; q < 3; ++q) ax[q] = ay[q] = az[q] = zero3<R>();
  const v3<R> vc = getv(1, 1, 1);
#pragma unroll
  for (int i = 0; i < 3; ++i)
#pragma unroll
    for (int j = 0; j < 3; ++j) {
      const R wij = s.w[0][i] * s.w[1][j];
      v3<R> r = zero3<R>();
#pragma unroll
      for (int k = 0; k < 3; ++k) {
        const v3<R> g = getv(i, j, k) - vc;
        r += g * s.w[2][k];
        az[k] += g * wij;
      }
      ax[i] += r * wij;
      ay[j] += r * wij;
    }
#pragma unroll
  for (int k = 0; k < 3; ++k) az[k] = az[k] * s.w[2][k];
  const v3<R> dv = ax[0] + ax[1] + ax[2];
  vnew = vc + dv;
  const v3<R> mc[3] = {ax[1] + ax[2] * R(2), ay[1] + ay[2] * R(2), az[1] + az[2] * R(2)};
#pragma unroll
  for (int r = 0; r < 3; ++r)
#pragma unroll
    for (int c = 0; c < 3; ++c) B(r, c) = (mc[c][r] - dv[r] * s.fx[c]) * dx;
}

// Forward G2P in deviation form: D = F - I in, D' = proj(F_new) - I out, with
// F_new - I = D + dt C (I + D) (no rounding of F_new near I).  getv returns
// node velocities relative to vref (node_update_rel); v' = vref + gather.
template <class R, class GetV>
DM_HD void g2p_particle_sep(const Law<R>& L, const TransferCtx<R>& t, const Stencil<R>& s, GetV getv, v3<R>& x,
                            v3<R>& v, m3<R>& C, m3<R>& D, bool* bad_adv, bool* bad_det, v3<R> vref,
                            m3<R>* tau = nullptr) {
  m3<R> B;
  g2p_gather_sep(s, t.dx, getv, v, B);
  v = vref + v;
  C = B * (R(4) * t.inv_dx * t.inv_dx);
  x.x += t.dt * v.x;
  x.y += t.dt * v.y;
  x.z += t.dt * v.z;
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    const R gx = x[a] / t.dx;
    if (!(gx >= R(1.5) && gx <= R(t.dims[a]) - R(2.5))) *bad_adv = true;  // NaN-safe
  }
  const m3<R> Dn = D + (C + C * D) * t.dt;
  D = law_project_fwd(L, Dn, bad_det, tau);
}

// d/dfx of sum_n w_n h_n for a per-node scalar h_n, accumulated separably.
template <class R>
struct FxBar {
  R tx[3], ty[3], tz[3];
  DM_HD void zero() {
#pragma unroll
    for (int q = 0; q < 3; ++q) tx[q] = ty[q] = tz[q] = R(0);
  }
  DM_HD void add(const Stencil<R>& s, int i, int j, int k, R h) {
    tx[i] += h * s.w[1][j] * s.w[2][k];
    ty[j] += h * s.w[0][i] * s.w[2][k];
    tz[k] += h * s.w[0][i] * s.w[1][j];
  }
  DM_HD v3<R> result(const Stencil<R>& s) const {
    return mk3(s.dw[0][0] * tx[0] + s.dw[0][1] * tx[1] + s.dw[0][2] * tx[2],
               s.dw[1][0] * ty[0] + s.dw[1][1] * ty[1] + s.dw[1][2] * ty[2],
               s.dw[2][0] * tz[0] + s.dw[2][1] * tz[1] + s.dw[2][2] * tz[2]);
  }
};

// Adjoint of g2p_particle_sep (same contract as g2p_vjp).
template <class R, class GetV>
DM_HD void g2p_vjp_given(const Law<R>& L, const TransferCtx<R>& t, const Stencil<R>& s, GetV getv, const m3<R>& F,
                         v3<R> vnew, const m3<R>& Cn, v3<R> xb_o, v3<R> vb_o, const m3<R>& Cb_o, const m3<R>& Fb_o,
                         v3<R>& xb_part, m3<R>& Fb_part, v3<R>& gq, m3<R>& Bd, R& mubar, v3<R> vref);
template <class R, class GetV>
DM_HD void g2p_vjp_sep(const Law<R>& L, const TransferCtx<R>& t, const Stencil<R>& s, GetV getv, const m3<R>& F,
                       v3<R> xb_o, v3<R> vb_o, const m3<R>& Cb_o, const m3<R>& Fb_o, v3<R>& xb_part, m3<R>& Fb_part,
                       v3<R>& gq, m3<R>& Bd, R& mubar) {
  v3<R> vnew;
  m3<R> B;
  g2p_gather_sep(s, t.dx, getv, vnew, B);
  const m3<R> Cn = B * (R(4) * t.inv_dx * t.inv_dx);
  g2p_vjp_given(L, t, s, getv, F, vnew, Cn, xb_o, vb_o, Cb_o, Fb_o, xb_part, Fb_part, gq, Bd, mubar, zero3<R>());
}

// g2p_vjp_sep with the forward's G2P outputs (v', C' = the next state's v, C,
// bit-identical to a re-gather) supplied instead of recomputed.  getv may
// return node velocities relative to vref (node_update_rel): the weight
// derivatives of the quadratic B-spline sum to 0 and their first moment to 1,
// so vref's part of sum_n dw_n (v_n . u_n) is vref . bc_axis (9 FMAs instead
// of adding vref at all 27 nodes).
template <class R, class GetV>
DM_HD void g2p_vjp_given(const Law<R>& L, const TransferCtx<R>& t, const Stencil<R>& s, GetV getv, const m3<R>& F,
                         v3<R> vnew, const m3<R>& Cn, v3<R> xb_o, v3<R> vb_o, const m3<R>& Cb_o, const m3<R>& Fb_o,
                         v3<R>& xb_part, m3<R>& Fb_part, v3<R>& gq, m3<R>& Bd, R& mubar, v3<R> vref) {
  const R c4 = R(4) * t.inv_dx * t.inv_dx;
  const m3<R> Ad = meye<R>() + Cn * t.dt;
  const m3<R> Fnew = Ad * F;
  const m3<R> Fnb = law_project_vjp(L, Fnew, Fb_o, mubar);
  const m3<R> Cb = Cb_o + mul_bt(Fnb, F) * t.dt;
  Fb_part = mul_at(Ad, Fnb);
  const v3<R> gb = vb_o + xb_o * t.dt;
  const m3<R> Bb = Cb * c4;
  // u_n = gb + Bb (o - fx) dx = u0 + sum_c o_c bc
  const v3<R> f = mk3(s.fx[0] * t.dx, s.fx[1] * t.dx, s.fx[2] * t.dx);
  gq = gb - Bb * f;
  Bd = Bb * t.dx;
  const v3<R> bcx = mk3(Bd(0, 0), Bd(1, 0), Bd(2, 0));
  const v3<R> bcy = mk3(Bd(0, 1), Bd(1, 1), Bd(2, 1));
  const v3<R> bcz = mk3(Bd(0, 2), Bd(1, 2), Bd(2, 2));
  // sum_n h_n dw_n/dfx factored like the gather: H_ij = sum_k wz_k h_ijk
  FxBar<R> fb;
  fb.zero();
#pragma unroll
  for (int i = 0; i < 3; ++i) {
    const v3<R> ui = gq + bcx * R(i);
#pragma unroll
    for (int j = 0; j < 3; ++j) {
      const v3<R> uij = ui + bcy * R(j);
      const R wij = s.w[0][i] * s.w[1][j];
      R H = R(0);
#pragma unroll
      for (int k = 0; k < 3; ++k) {
        const v3<R> u = uij + bcz * R(k);
        const R h = dot(getv(i, j, k), u);
        H += h * s.w[2][k];
        fb.tz[k] += h * wij;
      }
      fb.tx[i] += H * s.w[1][j];
      fb.ty[j] += H * s.w[0][i];
    }
  }
  const v3<R> fxb = fb.result(s) + mk3(dot(vref, bcx), dot(vref, bcy), dot(vref, bcz)) - tmul(Bb, vnew) * t.dx;
  xb_part = mk3(xb_o.x + fxb.x * t.inv_dx, xb_o.y + fxb.y * t.inv_dx, xb_o.z + fxb.z * t.inv_dx);
}

// Adjoint of the P2G for one particle (same contract as p2g_vjp).
template <class R, class GetMB>
DM_HD void p2g_vjp_sep(const Law<R>& L, const TransferCtx<R>& t, const Stencil<R>& s, GetMB getmb, v3<R> v,
                       const m3<R>& F, const m3<R>& C, R act, v3<R>& xb, v3<R>& vb, m3<R>& Fb, m3<R>& Cb, R& mubar,
                       R& lambar, R& actbar) {
  bool bad = false;
  Hencky<R> memo;  // the SVD laws' decomposition of F, reused by law_stress_vjp
  const m3<R> P = law_stress(L, F, act, &bad, &memo);
  m3<R> tau = mul_bt(P, F);
  const bool visc = L.kind == kFluid && L.visc != R(0);
  const m3<R> Cs = C + transpose(C);
  const R J = det(F);
  if (visc) tau += Cs * (J * L.visc);
  const R kA = -t.dt * L.vol * R(4) * t.inv_dx * t.inv_dx;
  const m3<R> A = tau * kA + C * L.mass;
  // u_n = m v + A (o - fx) dx = q0 + sum_c o_c ac
  const v3<R> f = mk3(s.fx[0] * t.dx, s.fx[1] * t.dx, s.fx[2] * t.dx);
  const v3<R> q0 = v * L.mass - A * f;
  const v3<R> acx = mk3(A(0, 0) * t.dx, A(1, 0) * t.dx, A(2, 0) * t.dx);
  const v3<R> acy = mk3(A(0, 1) * t.dx, A(1, 1) * t.dx, A(2, 1) * t.dx);
  const v3<R> acz = mk3(A(0, 2) * t.dx, A(1, 2) * t.dx, A(2, 2) * t.dx);
  // separable factoring (w_ijk = wij wz_k): per (i, j) the k-sums
  // Rp = sum_k wz_k pb, H = sum_k wz_k h; per k the (i, j)-sums with wij
  v3<R> px[3], py[3], pz[3];
#pragma unroll
  for (int q = 0; q < 3; ++q) px[q] = py[q] = pz[q] = zero3<R>();
  FxBar<R> fb;
  fb.zero();
#pragma unroll
  for (int i = 0; i < 3; ++i) {
    const v3<R> ui = q0 + acx * R(i);
#pragma unroll
    for (int j = 0; j < 3; ++j) {
      const v3<R> uij = ui + acy * R(j);
      const R wij = s.w[0][i] * s.w[1][j];
      v3<R> Rp = zero3<R>();
      R H = R(0);
#pragma unroll
      for (int k = 0; k < 3; ++k) {
        const v3<R> u = uij + acz * R(k);
        R mb;
        v3<R> pb;
        getmb(i, j, k, mb, pb);
        Rp += pb * s.w[2][k];
        pz[k] += pb * wij;
        const R h = mb * L.mass + dot(pb, u);
        H += h * s.w[2][k];
        fb.tz[k] += h * wij;
      }
      px[i] += Rp * wij;
      py[j] += Rp * wij;
      fb.tx[i] += H * s.w[1][j];
      fb.ty[j] += H * s.w[0][i];
    }
  }
#pragma unroll
  for (int k = 0; k < 3; ++k) pz[k] = pz[k] * s.w[2][k];
  const v3<R> S = px[0] + px[1] + px[2];
  const v3<R> mc[3] = {px[1] + px[2] * R(2), py[1] + py[2] * R(2), pz[1] + pz[2] * R(2)};
  m3<R> Ab;
#pragma unroll
  for (int r = 0; r < 3; ++r)
#pragma unroll
    for (int c = 0; c < 3; ++c) Ab(r, c) = (mc[c][r] - S[r] * s.fx[c]) * t.dx;
  const v3<R> fxb = fb.result(s) - tmul(A, S) * t.dx;
  xb += mk3(fxb.x * t.inv_dx, fxb.y * t.inv_dx, fxb.z * t.inv_dx);
  vb += S * L.mass;
  Cb += Ab * L.mass;
  const m3<R> taub = Ab * kA;
  if (visc) {
    Cb += (taub + transpose(taub)) * (J * L.visc);
    Fb += cofactor(F) * (L.visc * ddot(Cs, taub));
  }
  const m3<R> Pb = taub * F;
  Fb += mul_at(taub, P);
  law_stress_vjp(L, F, act, Pb, Fb, mubar, lambar, actbar, &memo);
}

}  // namespace dm
