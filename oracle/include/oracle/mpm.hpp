// TEST INFRASTRUCTURE ONLY (oracle).  Never linked into the product path.
//
// CPU restatement of the reference's batched MLS-MPM substep
// (/root/reference/proj/include/diffsim/mpm.hpp), templated on the scalar so
// that the fp64 instantiation is the forward oracle and the instantiation on
// the reference's scalar tape (diffsim::Value, tape.hpp:17-27) is the
// gradient oracle.  Each function cites the reference lines it restates.
//
// Config-gap extensions are written in the same
// templated style so the reference tape differentiates them too:
//   * fixed-corotated law (cfg 1)            -- stress_fixed_corotated
//   * stable neo-Hookean + x-axis actuation  -- stress_neo_hookean, reusing the
//     energy of fem.hpp:111-142 (cfg 2)
//   * fluid viscosity tau = J eta (C + C^T)   -- p2g (cfg 4)
//   * capped cylinder and open-top hollow box SDFs, rotating colliders
//     (v_col = v + w x (p - c))               -- collider_query / grid_update
//   * sticky domain boundary (cfg 1)          -- grid_update
//   * material parameters (E) as scalars of type T, so dL/dE comes off the tape
//   * particle binning / stable sort (no reference function)
#pragma once

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <stdexcept>
#include <string>
#include <vector>

#include "oracle/linalg.hpp"
#include "oracle/svd3x3.hpp"

namespace oracle {

// ---- scalar primitives for double (tape overloads are found by ADL) ----
inline double exp(double a) { return std::exp(a); }
inline double log(double a) { return std::log(a); }
inline double sqrt(double a) { return std::sqrt(a); }
inline double abs(double a) { return std::fabs(a); }
inline double min(double a, double b) { return a < b ? a : b; }
inline double max(double a, double b) { return a > b ? a : b; }
inline double where(bool c, double a, double b) { return c ? a : b; }
inline double value_of(double a) { return a; }

inline void svd3(const M3<double>& f, M3<double>& u, V3<double>& s, M3<double>& vt) {
  double sv[3];
  svd3x3_values(f.m.data(), u.m.data(), sv, vt.m.data());
  s = {sv[0], sv[1], sv[2]};
}

// ---- descriptors ----

enum LawKind : int { kFixedCorotated = 0, kNeoHookean = 1, kElastoplastic = 2, kFluid = 3 };
enum ColliderKind : int { kPlane = 0, kSphere = 1, kBox = 2, kCylinder = 3, kHollowBox = 4 };
enum BoundaryKind : int { kSlip = 0, kSticky = 1 };

// Material.  Lame parameters follow MpmMaterial (mpm.hpp:33-40); E is a T so
// the tape can differentiate it (the reference keeps it double, mpm.hpp:23-41).
template <class T>
struct Material {
  int kind = kFixedCorotated;
  T youngs = T(1e4);
  double poisson = 0.3;
  double density = 1.0;
  double volume = 1e-6;       // particle rest volume V0
  double yield_stress = 1e3;  // elastoplastic
  int wide_yield = 0;         // mpm.hpp:29-31
  double viscosity = 0.0;     // fluid extension
  double act_strength = 0.0;  // neo-Hookean x-axis actuation strength
  double bulk = 0.0;          // fluid: lambda override when > 0
  double mass() const { return density * volume; }
  T lame_mu() const { return youngs * T(1.0 / (2.0 * (1.0 + poisson))); }
  T lame_lambda() const {
    if (kind == kFluid && bulk > 0.0) return T(bulk);
    return youngs * T(poisson / ((1.0 + poisson) * (1.0 - 2.0 * poisson)));
  }
};

template <class T>
struct Collider {
  int kind = kPlane;
  V3<T> center{T(0.0), T(0.0), T(0.0)};
  V3<T> velocity{T(0.0), T(0.0), T(0.0)};
  V3<T> omega{T(0.0), T(0.0), T(0.0)};
  V3<double> normal{0.0, 0.0, 1.0};  // plane normal / cylinder axis (unit)
  double radius = 0.1;               // sphere, cylinder
  V3<double> half{0.1, 0.1, 0.1};    // box; hollow box cavity half extents
  double length = 0.3;               // cylinder full length
  double thickness = 0.02;           // hollow box wall thickness
};

struct SimParams {
  int dims[3] = {32, 32, 32};
  double dx = 1.0 / 32.0;
  double dt = 1e-4;
  double gravity[3] = {0.0, 0.0, -9.8};
  int boundary = kSlip;
  double alpha_c = 100.0;  // CouplingParams, mpm.hpp:134-137
  double mu_b = 0.0;
  int node_index(int i, int j, int k) const { return (i * dims[1] + j) * dims[2] + k; }
  int node_count() const { return dims[0] * dims[1] * dims[2]; }
};

template <class T>
struct State {
  std::vector<V3<T>> x, v;
  std::vector<M3<T>> F, C;
  std::vector<int> material;  // index into the material table
  std::vector<int> group;     // actuation group (neo-Hookean)
  std::size_t size() const { return x.size(); }
};

template <class T>
struct Grid {
  std::vector<V3<T>> momentum, vel;
  std::vector<T> mass;
  void clear(const SimParams& sp) {
    const int n = sp.node_count();
    momentum.assign(n, V3<T>{T(0.0), T(0.0), T(0.0)});
    vel.assign(n, V3<T>{T(0.0), T(0.0), T(0.0)});
    mass.assign(n, T(0.0));
  }
};

// ---- transfers (mpm.hpp:141-161) ----

template <class T>
void bspline_weights(const T& fx, T w[3]) {  // mpm.hpp:141-147
  w[0] = T(0.5) * (T(1.5) - fx) * (T(1.5) - fx);
  w[1] = T(0.75) - (fx - T(1.0)) * (fx - T(1.0));
  w[2] = T(0.5) * (fx - T(0.5)) * (fx - T(0.5));
}

template <class T>
void stencil_base(const SimParams& sp, const V3<T>& x, std::size_t p, int base[3], V3<T>& fx) {
  // mpm.hpp:149-161: base by double division, fx by multiplication
  for (int a = 0; a < 3; ++a) {
    const double gx = value_of(x[a]) / sp.dx;
    base[a] = static_cast<int>(std::floor(gx - 0.5));
    if (base[a] < 1 || base[a] + 2 > sp.dims[a] - 2)
      throw std::runtime_error("mpm: particle " + std::to_string(p) +
                               " outside grid interior (axis " + std::to_string(a) + ")");
    fx[a] = x[a] * T(1.0 / sp.dx) - T(static_cast<double>(base[a]));
  }
}

// ---- constitutive laws: first Piola P and the projected F ----

// Gradient-oracle hook.  On the reference tape (oracle/src/ref_capi.cpp) the
// SVD laws can be recorded as isotropic matrix maps with their exact
// derivative instead of through Tape::svd3x3, whose adjoint clamps
// sigma_j^2 - sigma_i^2 to +-1e-9 (svd3.hpp:45-49) and drops the rotation
// terms at (near-)repeated singular values -- F = I, or the uniaxial strain of
// a resting body.  Returns false: the literal restatement below.
// kind: 0 fixed-corotated (fills p), 2 elastoplastic (fills p and f_proj).
template <class T>
inline bool iso_law(int kind, const M3<T>& f, const T& mu, const T& lam, const T& c_y, M3<T>& p, M3<T>& f_proj) {
  (void)kind, (void)f, (void)mu, (void)lam, (void)c_y, (void)p, (void)f_proj;
  return false;
}

// Extension (cfg 1): fixed-corotated, P = 2 mu (F - R) + lambda (J - 1) cof(F)
// with R = U V^T from the SVD (R is a rotation since det F > 0, tape.hpp:172).
template <class T>
M3<T> stress_fixed_corotated(const M3<T>& f, const T& mu, const T& lam) {
  const T j = det(f);
  if (value_of(j) <= 0.0) throw std::runtime_error("stress_fixed_corotated: det(F) <= 0");
  {
    M3<T> p, fp;
    if (iso_law(0, f, mu, lam, T(0.0), p, fp)) return p;
  }
  M3<T> u, vt;
  V3<T> s;
  svd3(f, u, s, vt);
  const M3<T> r = u * vt;
  return (f - r) * (T(2.0) * mu) + cofactor(f) * (lam * (j - T(1.0)));
}

// Extension (cfg 2): stable neo-Hookean of fem.hpp:124-142 with the rest-stable
// alpha = 1 + 3 mu / (4 lambda) (fem.hpp:29-31) and an x-axis actuation
// P_act = k a F e_x e_x^T (energy k a |F e_x|^2 / 2).
template <class T>
M3<T> stress_neo_hookean(const M3<T>& f, const T& mu, const T& lam, double k_act, const T& act) {
  const T j = det(f);
  if (value_of(j) <= 0.0) throw std::runtime_error("stress_neo_hookean: det(F) <= 0");
  const T alpha = T(1.0) + T(0.75) * mu / lam;
  T ic(0.0);
  for (int i = 0; i < 9; ++i) ic = ic + f.m[i] * f.m[i];
  const T mu_term = mu * (T(1.0) - T(1.0) / (ic + T(1.0)));
  const M3<T> cof = cofactor(f);
  M3<T> p;
  for (int i = 0; i < 9; ++i) p.m[i] = mu_term * f.m[i] + lam * (j - alpha) * cof.m[i];
  if (k_act != 0.0) {
    const T ka = T(k_act) * act;
    for (int r = 0; r < 3; ++r) p(r, 0) = p(r, 0) + ka * f(r, 0);
  }
  return p;
}

// mpm.hpp:165-198: Hencky strain, von Mises return mapping.  Returns P; writes
// the projected F.
template <class T>
M3<T> stress_elastoplastic(const M3<T>& f, const T& mu, const T& lam, const T& c_y, M3<T>& f_proj) {
  if (value_of(det(f)) <= 0.0) throw std::runtime_error("stress_elastoplastic: det(F) <= 0");
  {
    M3<T> p;
    if (iso_law(2, f, mu, lam, c_y, p, f_proj)) return p;
  }
  M3<T> u, vt;
  V3<T> sig;
  svd3(f, u, sig, vt);
  V3<T> eps{log(sig.x), log(sig.y), log(sig.z)};
  const T tr = eps.x + eps.y + eps.z;
  const T third = tr * T(1.0 / 3.0);
  const V3<T> dev{eps.x - third, eps.y - third, eps.z - third};
  const T dev_norm = sqrt(dot(dev, dev) + T(1e-30));
  const T dgamma = dev_norm - c_y;
  f_proj = f;
  if (value_of(dgamma) > 0.0) {
    const T s = dgamma / dev_norm;
    eps = eps - dev * s;
    const V3<T> sn{exp(eps.x), exp(eps.y), exp(eps.z)};
    f_proj = u * M3<T>::diag(sn.x, sn.y, sn.z) * vt;
    sig = sn;
  }
  const T tr2 = eps.x + eps.y + eps.z;
  const T two_mu = T(2.0) * mu;
  const V3<T> ps{(two_mu * eps.x + lam * tr2) / sig.x, (two_mu * eps.y + lam * tr2) / sig.y,
                 (two_mu * eps.z + lam * tr2) / sig.z};
  return u * M3<T>::diag(ps.x, ps.y, ps.z) * vt;
}

// mpm.hpp:200-210: P = lambda (J - 1) cof(F), F_proj = J^{1/3} I.
template <class T>
M3<T> stress_fluid(const M3<T>& f, const T& lam, M3<T>& f_proj) {
  const T j = det(f);
  if (value_of(j) <= 0.0) throw std::runtime_error("stress_fluid: det(F) <= 0");
  const M3<T> p = cofactor(f) * (lam * (j - T(1.0)));
  const T s = exp(log(j) * T(1.0 / 3.0));
  f_proj = M3<T>::diag(s, s, s);
  return p;
}

// material_stress (mpm.hpp:212-217) extended to four laws.
template <class T>
M3<T> material_stress(const M3<T>& f, const Material<T>& mat, const T& act, M3<T>& f_proj) {
  const T mu = mat.lame_mu(), lam = mat.lame_lambda();
  switch (mat.kind) {
    case kFixedCorotated:
      f_proj = f;
      return stress_fixed_corotated(f, mu, lam);
    case kNeoHookean:
      f_proj = f;
      return stress_neo_hookean(f, mu, lam, mat.act_strength, act);
    case kElastoplastic: {
      const T c_y = mat.wide_yield ? T(mat.yield_stress) / mu : T(mat.yield_stress) / (T(2.0) * mu);
      return stress_elastoplastic(f, mu, lam, c_y, f_proj);
    }
    case kFluid:
    default:
      return stress_fluid(f, lam, f_proj);
  }
}

// ---- colliders (mpm.hpp:86-131 plus extensions) ----

template <class T>
void box_query(const V3<T>& rel, const V3<double>& half, T& d, V3<T>& n) {
  // restates the solid-box branch of SdfCollider::query, mpm.hpp:98-128
  const T qx = abs(rel.x) - T(half.x);
  const T qy = abs(rel.y) - T(half.y);
  const T qz = abs(rel.z) - T(half.z);
  const T ox = max(qx, T(0.0)), oy = max(qy, T(0.0)), oz = max(qz, T(0.0));
  const T outside = sqrt(ox * ox + oy * oy + oz * oz + T(1e-18));
  const T inside = min(max(qx, max(qy, qz)), T(0.0));
  const bool is_out = value_of(qx) > 0.0 || value_of(qy) > 0.0 || value_of(qz) > 0.0;
  d = where(is_out, outside - T(1e-9), inside);
  n = {T(0.0), T(0.0), T(0.0)};
  if (is_out) {
    n = {ox / outside, oy / outside, oz / outside};
  } else {
    const double ax = value_of(qx), ay = value_of(qy), az = value_of(qz);
    if (ax >= ay && ax >= az)
      n.x = T(1.0);
    else if (ay >= az)
      n.y = T(1.0);
    else
      n.z = T(1.0);
  }
  if (value_of(rel.x) < 0.0) n.x = T(0.0) - n.x;
  if (value_of(rel.y) < 0.0) n.y = T(0.0) - n.y;
  if (value_of(rel.z) < 0.0) n.z = T(0.0) - n.z;
}

template <class T>
void collider_query(const Collider<T>& col, const V3<T>& p, T& d, V3<T>& n) {
  const V3<T> rel = p - col.center;
  switch (col.kind) {
    case kPlane: {  // mpm.hpp:90-93
      const V3<T> nn{T(col.normal.x), T(col.normal.y), T(col.normal.z)};
      d = dot(rel, nn);
      n = nn;
      return;
    }
    case kSphere: {  // mpm.hpp:94-97
      const T r = sqrt(dot(rel, rel) + T(1e-18));
      d = r - T(col.radius);
      n = rel * (T(1.0) / r);
      return;
    }
    case kBox:
      box_query(rel, col.half, d, n);
      return;
    case kCylinder: {  // extension: capped cylinder, axis col.normal
      const V3<T> a{T(col.normal.x), T(col.normal.y), T(col.normal.z)};
      const T h = dot(rel, a);
      const V3<T> radial = rel - a * h;
      const T rho = sqrt(dot(radial, radial) + T(1e-18));
      const T q0 = rho - T(col.radius);
      const T q1 = abs(h) - T(0.5 * col.length);
      const T o0 = max(q0, T(0.0)), o1 = max(q1, T(0.0));
      const T outside = sqrt(o0 * o0 + o1 * o1 + T(1e-18));
      const bool is_out = value_of(q0) > 0.0 || value_of(q1) > 0.0;
      const V3<T> er = radial * (T(1.0) / rho);
      const double hs = value_of(h) < 0.0 ? -1.0 : 1.0;
      const V3<T> eh{T(hs * col.normal.x), T(hs * col.normal.y), T(hs * col.normal.z)};
      d = where(is_out, outside - T(1e-9), max(q0, q1));
      if (is_out) {
        const T c0 = o0 / outside, c1 = o1 / outside;
        n = er * c0 + eh * c1;
      } else {
        n = value_of(q0) >= value_of(q1) ? er : eh;
      }
      return;
    }
    case kHollowBox:
    default: {  // extension: open-top container = outer box minus cavity
      const double th = col.thickness;
      const V3<double> h = col.half;
      const double lift = 1.0;  // cavity extended upward: open top
      const V3<T> rel_o{rel.x, rel.y, rel.z + T(0.5 * th)};
      const V3<double> half_o{h.x + th, h.y + th, h.z + 0.5 * th};
      const V3<T> rel_c{rel.x, rel.y, rel.z - T(lift)};
      const V3<double> half_c{h.x, h.y, h.z + lift};
      T d_o, d_c;
      V3<T> n_o, n_c;
      box_query(rel_o, half_o, d_o, n_o);
      box_query(rel_c, half_c, d_c, n_c);
      const T neg_dc = T(0.0) - d_c;
      const bool use_outer = value_of(d_o) >= value_of(neg_dc);
      d = where(use_outer, d_o, neg_dc);
      n = use_outer ? n_o : V3<T>{T(0.0) - n_c.x, T(0.0) - n_c.y, T(0.0) - n_c.z};
      return;
    }
  }
}

// ---- P2G (mpm.hpp:219-254) ----

template <class T>
void p2g(const SimParams& sp, const State<T>& st, Grid<T>& g, const std::vector<Material<T>>& mats,
         const std::vector<T>& act) {
  g.clear(sp);
  const double inv_dx = 1.0 / sp.dx;
  for (std::size_t p = 0; p < st.size(); ++p) {
    int base[3];
    V3<T> fx;
    stencil_base(sp, st.x[p], p, base, fx);
    T wx[3], wy[3], wz[3];
    bspline_weights(fx.x, wx);
    bspline_weights(fx.y, wy);
    bspline_weights(fx.z, wz);
    const Material<T>& mat = mats.at(st.material[p]);
    const T a = (mat.kind == kNeoHookean && mat.act_strength != 0.0 && !act.empty())
                    ? act.at(st.group[p])
                    : T(0.0);
    M3<T> fp;
    const M3<T> stress = material_stress(st.F[p], mat, a, fp);
    (void)fp;
    M3<T> tau = stress * st.F[p].transposed();
    if (mat.kind == kFluid && mat.viscosity != 0.0) {  // extension: tau_v = J eta (C + C^T)
      const T jv = det(st.F[p]) * T(mat.viscosity);
      tau = tau + (st.C[p] + st.C[p].transposed()) * jv;
    }
    const double mass = mat.mass();
    const M3<T> affine = tau * T(-sp.dt * mat.volume * 4.0 * inv_dx * inv_dx) + st.C[p] * T(mass);
    for (int i = 0; i < 3; ++i)
      for (int j = 0; j < 3; ++j)
        for (int k = 0; k < 3; ++k) {
          const T w = wx[i] * wy[j] * wz[k];
          const V3<T> dpos{(T(static_cast<double>(i)) - fx.x) * T(sp.dx),
                           (T(static_cast<double>(j)) - fx.y) * T(sp.dx),
                           (T(static_cast<double>(k)) - fx.z) * T(sp.dx)};
          const int n = sp.node_index(base[0] + i, base[1] + j, base[2] + k);
          g.mass[n] = g.mass[n] + w * T(mass);
          g.momentum[n] = g.momentum[n] + (st.v[p] * T(mass) + affine * dpos) * w;
        }
  }
}

// ---- grid update (mpm.hpp:256-305) ----

template <class T>
V3<T> collide(const SimParams& sp, const Collider<T>& col, const V3<T>& node, const V3<T>& v_in) {
  T d;
  V3<T> nrm;
  collider_query(col, node, d, nrm);
  const T s = where(value_of(d) < 0.0, T(1.0), exp(T(0.0) - T(sp.alpha_c) * max(d, T(0.0))));
  const V3<T> vcol = col.velocity + cross(col.omega, node - col.center);
  const V3<T> rel = v_in - vcol;
  const T vn = dot(rel, nrm);
  const V3<T> tang = rel - nrm * vn;
  const T tnorm = sqrt(dot(tang, tang) + T(1e-18));
  const T keep = max(T(1.0) - T(sp.mu_b) * max(T(0.0) - vn, T(0.0)) / tnorm, T(0.0));
  const V3<T> proj_rel = tang * keep + nrm * max(vn, T(0.0));
  const V3<T> v_proj = vcol + proj_rel;
  const bool approaching = value_of(vn) < 0.0;
  V3<T> v = v_in;
  for (int a = 0; a < 3; ++a) v[a] = where(approaching, v_in[a] * (T(1.0) - s) + v_proj[a] * s, v_in[a]);
  return v;
}

template <class T>
void grid_update(const SimParams& sp, Grid<T>& g, const std::vector<Collider<T>>& cols) {
  const int bound = 3;
  for (int i = 0; i < sp.dims[0]; ++i)
    for (int j = 0; j < sp.dims[1]; ++j)
      for (int k = 0; k < sp.dims[2]; ++k) {
        const int n = sp.node_index(i, j, k);
        if (value_of(g.mass[n]) <= 0.0) {
          g.vel[n] = V3<T>{T(0.0), T(0.0), T(0.0)};
          continue;
        }
        V3<T> v = g.momentum[n] * (T(1.0) / g.mass[n]);
        v.x = v.x + T(sp.dt * sp.gravity[0]);
        v.y = v.y + T(sp.dt * sp.gravity[1]);
        v.z = v.z + T(sp.dt * sp.gravity[2]);
        const V3<T> node{T(i * sp.dx), T(j * sp.dx), T(k * sp.dx)};
        for (const auto& col : cols) v = collide(sp, col, node, v);
        const int idx[3] = {i, j, k};
        for (int a = 0; a < 3; ++a) {
          const bool lo = idx[a] < bound, hi = idx[a] >= sp.dims[a] - bound;
          if (sp.boundary == kSticky) {
            if (lo || hi) v[a] = T(0.0);
          } else {  // slip: zero the outward component (mpm.hpp:296-302)
            if (lo && value_of(v[a]) < 0.0) v[a] = T(0.0);
            if (hi && value_of(v[a]) > 0.0) v[a] = T(0.0);
          }
        }
        if (sp.boundary == kSticky) {
          bool band = false;
          for (int a = 0; a < 3; ++a) band = band || idx[a] < bound || idx[a] >= sp.dims[a] - bound;
          if (band) v = V3<T>{T(0.0), T(0.0), T(0.0)};
        }
        g.vel[n] = v;
      }
}

// ---- G2P (mpm.hpp:307-346) ----

template <class T>
void g2p(const SimParams& sp, State<T>& st, const Grid<T>& g, const std::vector<Material<T>>& mats,
         const std::vector<T>& act) {
  const double inv_dx = 1.0 / sp.dx;
  for (std::size_t p = 0; p < st.size(); ++p) {
    int base[3];
    V3<T> fx;
    stencil_base(sp, st.x[p], p, base, fx);
    T wx[3], wy[3], wz[3];
    bspline_weights(fx.x, wx);
    bspline_weights(fx.y, wy);
    bspline_weights(fx.z, wz);
    V3<T> v{T(0.0), T(0.0), T(0.0)};
    M3<T> b = M3<T>::zero();
    for (int i = 0; i < 3; ++i)
      for (int j = 0; j < 3; ++j)
        for (int k = 0; k < 3; ++k) {
          const T w = wx[i] * wy[j] * wz[k];
          const V3<T> dpos{(T(static_cast<double>(i)) - fx.x) * T(sp.dx),
                           (T(static_cast<double>(j)) - fx.y) * T(sp.dx),
                           (T(static_cast<double>(k)) - fx.z) * T(sp.dx)};
          const int n = sp.node_index(base[0] + i, base[1] + j, base[2] + k);
          const V3<T> vw = g.vel[n] * w;
          v = v + vw;
          b = b + outer(vw, dpos);
        }
    st.v[p] = v;
    st.C[p] = b * T(4.0 * inv_dx * inv_dx);
    for (int a = 0; a < 3; ++a) st.x[p][a] = st.x[p][a] + T(sp.dt) * v[a];
    for (int a = 0; a < 3; ++a) {
      const double gx = value_of(st.x[p][a]) / sp.dx;
      if (gx < 1.5 || gx > sp.dims[a] - 2.5)
        throw std::runtime_error("g2p: particle " + std::to_string(p) + " advected outside grid interior");
    }
    const M3<T> fnew = (M3<T>::identity() + st.C[p] * T(sp.dt)) * st.F[p];
    const Material<T>& mat = mats.at(st.material[p]);
    const T a = (mat.kind == kNeoHookean && mat.act_strength != 0.0 && !act.empty()) ? act.at(st.group[p])
                                                                                    : T(0.0);
    M3<T> fp;
    (void)material_stress(fnew, mat, a, fp);
    st.F[p] = fp;
  }
}

// One substep = p2g, grid_update, g2p (mpm.hpp:362-366).
template <class T>
void substep(const SimParams& sp, State<T>& st, Grid<T>& g, const std::vector<Material<T>>& mats,
             const std::vector<Collider<T>>& cols, const std::vector<T>& act) {
  p2g(sp, st, g, mats, act);
  grid_update(sp, g, cols);
  g2p(sp, st, g, mats, act);
}

// ---- binning / stable sort (build-defined; SURVEY 8(a) a7, 8(d) "Binning") ----
// Key = (linear index of the 4x4x4-cell tile holding the particle's stencil
// base) * 64 + (linear index of the base cell inside the tile), computed with
// the same fp32 operations as the device:
//   gx = fl(x * inv_dx); base = floor(fl(gx - 0.5)); tile = base >> 2; cell = base & 3.
inline int tile_dim(int dim) { return (dim + 3) / 4; }

inline void bin_keys_f32(const SimParams& sp, const float* x /* N x 3 */, std::size_t n, int* keys) {
  const float inv_dx = static_cast<float>(1.0 / sp.dx);
  const int td[3] = {tile_dim(sp.dims[0]), tile_dim(sp.dims[1]), tile_dim(sp.dims[2])};
  for (std::size_t p = 0; p < n; ++p) {
    int t[3], c[3];
    for (int a = 0; a < 3; ++a) {
      volatile float gx = x[3 * p + a] * inv_dx;  // volatile: no contraction
      volatile float gm = gx - 0.5f;
      const float b = std::floor(static_cast<float>(gm));
      const bool ok = b >= 1.f && b <= static_cast<float>(sp.dims[a] - 4);
      const int base = ok ? static_cast<int>(b) : 1;  // outside: reported, binned as base 1 (device rule)
      t[a] = base >> 2;
      c[a] = base & 3;
    }
    keys[p] = ((t[0] * td[1] + t[1]) * td[2] + t[2]) * 64 + (c[0] * 4 + c[1]) * 4 + c[2];
  }
}

inline void stable_sort_perm(const int* keys, std::size_t n, int* perm) {
  std::vector<int> idx(n);
  for (std::size_t i = 0; i < n; ++i) idx[i] = static_cast<int>(i);
  std::stable_sort(idx.begin(), idx.end(), [&](int a, int b) { return keys[a] < keys[b]; });
  for (std::size_t i = 0; i < n; ++i) perm[i] = idx[i];
}

// ---- observables (tasks.hpp:286-304, 330-338, 554-570, 604-615) ----

template <class T>
V3<T> center_of_mass(const State<T>& st) {
  V3<T> m{T(0.0), T(0.0), T(0.0)};
  const double inv_n = 1.0 / static_cast<double>(st.size());
  for (const auto& x : st.x) m = m + x * T(inv_n);
  return m;
}

template <class T>
V3<T> position_variance(const State<T>& st, const V3<T>& mean) {
  V3<T> var{T(0.0), T(0.0), T(0.0)};
  const double inv_n = 1.0 / static_cast<double>(st.size());
  for (const auto& x : st.x)
    for (int a = 0; a < 3; ++a) {
      const T d = x[a] - mean[a];
      var[a] = var[a] + d * d * T(inv_n);
    }
  return var;
}

// smoothed fraction outside a square footprint (MiniFluidMove::step, tasks.hpp:606-614)
template <class T>
T spill_fraction(const State<T>& st, const T& cx, const T& cy, double half, double temp) {
  T spill(0.0);
  const double inv_n = 1.0 / static_cast<double>(st.size());
  for (const auto& x : st.x) {
    const T sd = max(abs(x.x - cx), abs(x.y - cy)) - T(half);
    spill = spill + T(inv_n) / (T(1.0) + exp(T(0.0) - sd * T(1.0 / temp)));
  }
  return spill;
}

// env.hpp:33-39
template <class T>
T reward_distance_tiered(const T& d, double threshold, double low_mult, double high_mult) {
  const T base = T(1.0) / ((T(1.0) + d) * (T(1.0) + d));
  return base * where(value_of(d) > threshold, T(low_mult), T(high_mult));
}

}  // namespace oracle
