// TEST INFRASTRUCTURE ONLY (oracle/_ref).  Built from the reference headers
// where they lie (/root/reference/proj/include, read-only, compiled
// unchanged) plus the Eigen-free shim in oracle/shim/.  Output goes only to
// oracle/_ref/.  Three roles:
//   1. ref_mpm_rollout: the reference's own mpm_step<double> (mpm.hpp:348-367)
//      on reference descriptors -- pins the restatement's forward.
//   2. ref_mpm_grad:    the reference's own mpm_step<Value> + Tape::backward
//      (tape.hpp:124-164) -- pins the restatement's gradient.
//   3. ref_rollout_grad: the restatement (oracle/mpm.hpp) instantiated on the
//      reference tape, with recompute-on-backward segments via
//      Tape::checkpoint (tape.hpp:181-255) as step_checkpointed does
//      (algo.hpp:79-104) -- the gradient oracle for every BASELINE config,
//      including the config-gap extensions.
#include <chrono>
#include <cstdio>
#include <cstring>
#include <exception>
#include <span>
#include <vector>

#include "diffsim/linalg.hpp"
#include "diffsim/rng.hpp"
#include "diffsim/mpm.hpp"
#include "diffsim/tape.hpp"
#include "diffsim/env.hpp"
#include "diffsim/tasks.hpp"

// tape overload of the restatement's SVD hook (mirrors linalg.hpp:173-194)
#include "oracle/linalg.hpp"
namespace oracle {
inline void svd3(const M3<diffsim::Value>& f, M3<diffsim::Value>& u, V3<diffsim::Value>& s,
                 M3<diffsim::Value>& vt);
// SVD-law adjoint of the gradient oracle: 1 = isotropic-map nodes (exact
// derivative, default), 0 = the reference's Tape::svd3x3 (clamped adjoint).
inline int g_svd_adjoint = 1;
inline bool iso_law(int kind, const M3<diffsim::Value>& f, const diffsim::Value& mu, const diffsim::Value& lam,
                    const diffsim::Value& c_y, M3<diffsim::Value>& p, M3<diffsim::Value>& f_proj);
}
#include "oracle/driver.hpp"

// ---- isotropic matrix maps on the reference tape ----
// Phi(F) = U diag(phi(sigma; prm)) V^T for F = U diag(sigma) V^T (det F > 0,
// phi symmetric-separable: phi_i = f(sigma_i; symmetric functions of sigma)).
// The forward derivative (dF^ = U^T dF V):
//   dPhi^_ii = sum_j dphi_i/dsigma_j dF^_jj
//   [dPhi^_ij, dPhi^_ji] = [[a, b], [b, a]] [dF^_ij, dF^_ji],  i != j,
//   a, b = (dd_ij +- (phi_i + phi_j) / (sigma_i + sigma_j)) / 2,
//   dd_ij = (phi_i - phi_j) / (sigma_i - sigma_j)  ->  dphi_i/dsigma_i - dphi_i/dsigma_j
// at coinciding singular values (the limit for symmetric-separable phi).
// Each output is recorded as one linear combination of the 9 entries of F and
// the law parameters (chains of two-parent Tape::record nodes), with the
// partials of phi from a scratch tape.  Pinned against central differences of
// the fp64 forward in tests/test_oracle.py.
namespace oracle {
namespace {
using diffsim::Tape;
using diffsim::Value;

template <class T>
void phi_fcr(const T s[3], const T prm[3], bool, T out[3]) {
  const T J = s[0] * s[1] * s[2];
  for (int i = 0; i < 3; ++i) out[i] = T(2.0) * prm[0] * (s[i] - T(1.0)) + prm[1] * (J - T(1.0)) * J / s[i];
}

// Hencky / von Mises (mpm.hpp:165-198): which = 0 -> P's singular values, 1 -> F_proj's
template <class T, int WHICH>
void phi_hencky(const T s[3], const T prm[3], bool yield, T out[3]) {
  T e[3] = {log(s[0]), log(s[1]), log(s[2])};
  const T third = (e[0] + e[1] + e[2]) * T(1.0 / 3.0);
  T dev[3] = {e[0] - third, e[1] - third, e[2] - third};
  T sp[3] = {s[0], s[1], s[2]};
  if (yield) {
    const T n = sqrt(dev[0] * dev[0] + dev[1] * dev[1] + dev[2] * dev[2] + T(1e-30));
    const T k = (n - prm[2]) / n;
    for (int i = 0; i < 3; ++i) {
      e[i] = e[i] - dev[i] * k;
      sp[i] = exp(e[i]);
    }
  }
  const T tr2 = e[0] + e[1] + e[2];
  for (int i = 0; i < 3; ++i) out[i] = WHICH == 0 ? (T(2.0) * prm[0] * e[i] + prm[1] * tr2) / sp[i] : sp[i];
}

Value linear_node(Tape* tape, double value, const Value* in, const double* d, int n) {
  Value acc;
  bool have = false;
  int first = -1;
  for (int i = 0; i < n; ++i) {
    if (in[i].id < 0 || d[i] == 0.0) continue;
    if (first < 0) {
      first = i;
      continue;
    }
    if (!have) {
      acc = tape->record(value, in[first], d[first], in[i], d[i]);
      have = true;
    } else {
      acc = tape->record(value, acc, 1.0, in[i], d[i]);
    }
  }
  if (have) return acc;
  if (first >= 0) return tape->record(value, in[first], d[first]);
  return Value(value);
}

template <class PhiD, class PhiV>
void iso_record(const M3<Value>& f, const Value prm[3], bool yield, PhiD phi_d, PhiV phi_v, M3<Value>& out) {
  Tape* tape = nullptr;
  for (const Value& e : f.m)
    if (e.tape) tape = e.tape;
  for (int m = 0; m < 3; ++m)
    if (prm[m].tape) tape = prm[m].tape;
  double fd[9], U[9], S[3], Vt[9], pd[3], phi[3];
  for (int i = 0; i < 9; ++i) fd[i] = f.m[i].v;
  for (int m = 0; m < 3; ++m) pd[m] = prm[m].v;
  svd3x3_values(fd, U, S, Vt);
  phi_d(S, pd, yield, phi);
  double J[3][3], K[3][3];  // dphi_i / dsigma_j, dphi_i / dprm_m
  for (int i = 0; i < 3; ++i) {
    Tape t;
    Value sv[3] = {t.var(S[0]), t.var(S[1]), t.var(S[2])};
    Value pv[3] = {t.var(pd[0]), t.var(pd[1]), t.var(pd[2])};
    Value o[3];
    phi_v(sv, pv, yield, o);
    if (o[i].is_const()) {
      for (int j = 0; j < 3; ++j) J[i][j] = K[i][j] = 0.0;
      continue;
    }
    t.backward(o[i]);
    for (int j = 0; j < 3; ++j) {
      J[i][j] = t.grad(sv[j]);
      K[i][j] = t.grad(pv[j]);
    }
  }
  double a[3][3] = {}, b[3][3] = {};
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) {
      if (i == j) continue;
      const double ds = S[i] - S[j];
      const double dd = std::fabs(ds) > 1e-8 * (S[i] + S[j]) ? (phi[i] - phi[j]) / ds : J[i][i] - J[i][j];
      const double sp = (phi[i] + phi[j]) / (S[i] + S[j]);
      a[i][j] = 0.5 * (dd + sp);
      b[i][j] = 0.5 * (dd - sp);
    }
  auto uvt = [&](const double D[3][3], double o[9]) {  // U D V^T
    for (int r = 0; r < 3; ++r)
      for (int c = 0; c < 3; ++c) {
        double acc = 0.0;
        for (int i = 0; i < 3; ++i)
          for (int j = 0; j < 3; ++j) acc += U[3 * r + i] * D[i][j] * Vt[3 * j + c];
        o[3 * r + c] = acc;
      }
  };
  double val[9], jac[9][12];  // output (r,c) x input (9 F entries, 3 parameters)
  {
    double D[3][3] = {{phi[0], 0, 0}, {0, phi[1], 0}, {0, 0, phi[2]}};
    uvt(D, val);
  }
  for (int kl = 0; kl < 9; ++kl) {
    const int k = kl / 3, l = kl % 3;
    double G[3][3], D[3][3], o[9];
    for (int i = 0; i < 3; ++i)
      for (int j = 0; j < 3; ++j) G[i][j] = U[3 * k + i] * Vt[3 * j + l];
    for (int i = 0; i < 3; ++i)
      for (int j = 0; j < 3; ++j)
        D[i][j] = i == j ? J[i][0] * G[0][0] + J[i][1] * G[1][1] + J[i][2] * G[2][2] : a[i][j] * G[i][j] + b[i][j] * G[j][i];
    uvt(D, o);
    for (int q = 0; q < 9; ++q) jac[q][kl] = o[q];
  }
  for (int m = 0; m < 3; ++m) {
    double D[3][3] = {{K[0][m], 0, 0}, {0, K[1][m], 0}, {0, 0, K[2][m]}}, o[9];
    uvt(D, o);
    for (int q = 0; q < 9; ++q) jac[q][9 + m] = o[q];
  }
  Value in[12];
  for (int i = 0; i < 9; ++i) in[i] = f.m[i];
  for (int m = 0; m < 3; ++m) in[9 + m] = prm[m];
  for (int q = 0; q < 9; ++q) out.m[q] = tape ? linear_node(tape, val[q], in, jac[q], 12) : Value(val[q]);
}
}  // namespace

inline bool iso_law(int kind, const M3<Value>& f, const Value& mu, const Value& lam, const Value& c_y, M3<Value>& p,
                    M3<Value>& f_proj) {
  if (g_svd_adjoint == 0) return false;
  const Value prm[3] = {mu, lam, c_y};
  if (kind == 0) {
    iso_record(f, prm, false, phi_fcr<double>, phi_fcr<Value>, p);
    return true;
  }
  // the yield decision on values, as the restatement's value_of branch (mpm.hpp:182)
  double fd[9], U[9], S[3], Vt[9];
  for (int i = 0; i < 9; ++i) fd[i] = f.m[i].v;
  svd3x3_values(fd, U, S, Vt);
  const double e[3] = {std::log(S[0]), std::log(S[1]), std::log(S[2])};
  const double th = (e[0] + e[1] + e[2]) / 3.0;
  const double dv[3] = {e[0] - th, e[1] - th, e[2] - th};
  const bool yield = std::sqrt(dv[0] * dv[0] + dv[1] * dv[1] + dv[2] * dv[2] + 1e-30) - c_y.v > 0.0;
  iso_record(f, prm, yield, phi_hencky<double, 0>, phi_hencky<Value, 0>, p);
  if (yield)
    iso_record(f, prm, yield, phi_hencky<double, 1>, phi_hencky<Value, 1>, f_proj);
  else
    f_proj = f;
  return true;
}
}  // namespace oracle

namespace oracle {
inline void svd3(const M3<diffsim::Value>& f, M3<diffsim::Value>& u, V3<diffsim::Value>& s,
                 M3<diffsim::Value>& vt) {
  using diffsim::Value;
  diffsim::Tape* tape = nullptr;
  for (const Value& e : f.m)
    if (e.tape) {
      tape = e.tape;
      break;
    }
  Value sv[3];
  if (!tape) {
    double fd[9], ud[9], sd[3], vd[9];
    for (int i = 0; i < 9; ++i) fd[i] = f.m[i].v;
    svd3x3_values(fd, ud, sd, vd);
    for (int i = 0; i < 9; ++i) {
      u.m[i] = Value(ud[i]);
      vt.m[i] = Value(vd[i]);
    }
    s = {Value(sd[0]), Value(sd[1]), Value(sd[2])};
    return;
  }
  tape->svd3x3(f.m.data(), u.m.data(), sv, vt.m.data());
  s = {sv[0], sv[1], sv[2]};
}
}  // namespace oracle

using diffsim::Tape;
using diffsim::Value;

namespace {

void put_err(const char* msg, char* err, int errlen) {
  if (err && errlen > 0) std::snprintf(err, static_cast<std::size_t>(errlen), "%s", msg);
}

// ---- reference descriptors (mpm.hpp:23-137) ----
diffsim::mpm::MpmMaterial ref_material(const OrMat& m) {
  diffsim::mpm::MpmMaterial o;
  o.density = m.density;
  o.youngs = m.youngs;
  o.poisson = m.poisson;
  o.yield_stress = m.yield_stress;
  o.kind = m.kind == 3 ? diffsim::mpm::MaterialKind::kFluid : diffsim::mpm::MaterialKind::kElastoplastic;
  o.wide_yield = m.wide_yield != 0;
  return o;
}

template <class T>
diffsim::mpm::SdfCollider<T> ref_collider(const OrCol& c) {
  diffsim::mpm::SdfCollider<T> o;
  using K = typename diffsim::mpm::SdfCollider<T>::Kind;
  o.kind = c.kind == 0 ? K::kPlane : (c.kind == 1 ? K::kSphere : K::kBox);
  o.center = {T(c.center[0]), T(c.center[1]), T(c.center[2])};
  o.velocity = {T(c.velocity[0]), T(c.velocity[1]), T(c.velocity[2])};
  o.normal = {c.normal[0], c.normal[1], c.normal[2]};
  o.radius = c.radius;
  o.half = {c.half[0], c.half[1], c.half[2]};
  return o;
}

template <class T>
diffsim::mpm::MpmState<T> ref_state(const OrMat* mats, int n, const double* x, const double* v,
                                    const double* F, const double* C, const int* material) {
  diffsim::mpm::MpmState<T> st;
  for (int p = 0; p < n; ++p) {
    st.x.push_back({T(x[3 * p]), T(x[3 * p + 1]), T(x[3 * p + 2])});
    st.v.push_back({T(v[3 * p]), T(v[3 * p + 1]), T(v[3 * p + 2])});
    diffsim::Mat3<T> f, c;
    for (int i = 0; i < 9; ++i) {
      f.m[i] = T(F[9 * p + i]);
      c.m[i] = T(C[9 * p + i]);
    }
    st.F.push_back(f);
    st.C.push_back(c);
    const OrMat& m = mats[material[p]];
    st.mass.push_back(m.density * m.volume);
    st.volume0.push_back(m.volume);
    st.material_id.push_back(material[p]);
  }
  return st;
}

}  // namespace

extern "C" {

// (1) reference forward: n_sub substeps of mpm_step<double>, colliders fixed.
int ref_mpm_rollout(const OrSim* sim, const OrMat* mats, int nmat, const OrCol* cols, int ncol, int n,
                    double* x, double* v, double* F, double* C, const int* material, int n_sub,
                    double* seconds, char* err, int errlen) {
  try {
    std::vector<diffsim::mpm::MpmMaterial> mt;
    for (int i = 0; i < nmat; ++i) mt.push_back(ref_material(mats[i]));
    std::vector<diffsim::mpm::SdfCollider<double>> cl;
    for (int c = 0; c < ncol; ++c) cl.push_back(ref_collider<double>(cols[c]));
    auto st = ref_state<double>(mats, n, x, v, F, C, material);
    diffsim::mpm::MpmGrid<double> grid;
    grid.dims = {sim->dims[0], sim->dims[1], sim->dims[2]};
    grid.dx = sim->dx;
    grid.clear();
    diffsim::mpm::CouplingParams cp;
    cp.alpha_c = sim->alpha_c;
    cp.mu_b = sim->mu_b;
    const auto t0 = std::chrono::steady_clock::now();
    diffsim::mpm::mpm_step(st, grid, mt, cl, cp, {sim->gravity[0], sim->gravity[1], sim->gravity[2]},
                           sim->dt, n_sub);
    const auto t1 = std::chrono::steady_clock::now();
    if (seconds) *seconds = std::chrono::duration<double>(t1 - t0).count();
    for (int p = 0; p < n; ++p) {
      for (int a = 0; a < 3; ++a) {
        x[3 * p + a] = st.x[p][a];
        v[3 * p + a] = st.v[p][a];
      }
      for (int i = 0; i < 9; ++i) {
        F[9 * p + i] = st.F[p].m[i];
        C[9 * p + i] = st.C[p].m[i];
      }
    }
    return 0;
  } catch (const std::exception& e) {
    put_err(e.what(), err, errlen);
    return 1;
  }
}

// (2) reference gradient of L = |com(x_final) - target|^2 w.r.t. the initial
// state, through mpm_step<Value>.  seg = 0: one tape; seg = k > 0: every k
// substeps run inside a Tape::checkpoint segment (restated step_checkpointed).
int ref_mpm_grad(const OrSim* sim, const OrMat* mats, int nmat, const OrCol* cols, int ncol, int n,
                 const double* x, const double* v, const double* F, const double* C, const int* material,
                 int n_sub, int seg, const double* target, double* loss_out, double* gx, double* gv,
                 double* gF, double* gC, double* seconds, char* err, int errlen) {
  try {
    std::vector<diffsim::mpm::MpmMaterial> mt;
    for (int i = 0; i < nmat; ++i) mt.push_back(ref_material(mats[i]));
    std::vector<diffsim::mpm::SdfCollider<Value>> cl;
    for (int c = 0; c < ncol; ++c) cl.push_back(ref_collider<Value>(cols[c]));
    diffsim::mpm::CouplingParams cp;
    cp.alpha_c = sim->alpha_c;
    cp.mu_b = sim->mu_b;
    const diffsim::Vec3<double> grav{sim->gravity[0], sim->gravity[1], sim->gravity[2]};
    const auto t0 = std::chrono::steady_clock::now();
    Tape tape;
    auto st = ref_state<Value>(mats, n, x, v, F, C, material);
    std::vector<Value> leaves;
    auto visit = [&](auto&& fn) {
      for (auto& p : st.x) { fn(p.x); fn(p.y); fn(p.z); }
      for (auto& p : st.v) { fn(p.x); fn(p.y); fn(p.z); }
      for (auto& m : st.F) for (int i = 0; i < 9; ++i) fn(m.m[i]);
      for (auto& m : st.C) for (int i = 0; i < 9; ++i) fn(m.m[i]);
    };
    visit([&](Value& val) { val = tape.var(val.v); leaves.push_back(val); });
    const auto shape = st;
    auto run = [&](diffsim::mpm::MpmState<Value>& s, int k) {
      diffsim::mpm::MpmGrid<Value> grid;
      grid.dims = {sim->dims[0], sim->dims[1], sim->dims[2]};
      grid.dx = sim->dx;
      grid.clear();
      diffsim::mpm::mpm_step(s, grid, mt, cl, cp, grav, sim->dt, k);
    };
    int done = 0;
    while (done < n_sub) {
      const int k = seg > 0 ? std::min(seg, n_sub - done) : n_sub - done;
      if (seg > 0) {
        std::vector<Value> in;
        visit([&](Value& val) { in.push_back(val); });
        auto outs = tape.checkpoint(
            [&, k](Tape&, std::span<const Value> vin) {
              auto s = shape;
              std::size_t i = 0;
              for (auto& p : s.x) { p.x = vin[i++]; p.y = vin[i++]; p.z = vin[i++]; }
              for (auto& p : s.v) { p.x = vin[i++]; p.y = vin[i++]; p.z = vin[i++]; }
              for (auto& m : s.F) for (int q = 0; q < 9; ++q) m.m[q] = vin[i++];
              for (auto& m : s.C) for (int q = 0; q < 9; ++q) m.m[q] = vin[i++];
              run(s, k);
              std::vector<Value> out;
              for (auto& p : s.x) { out.push_back(p.x); out.push_back(p.y); out.push_back(p.z); }
              for (auto& p : s.v) { out.push_back(p.x); out.push_back(p.y); out.push_back(p.z); }
              for (auto& m : s.F) for (int q = 0; q < 9; ++q) out.push_back(m.m[q]);
              for (auto& m : s.C) for (int q = 0; q < 9; ++q) out.push_back(m.m[q]);
              return out;
            },
            in);
        std::size_t i = 0;
        visit([&](Value& val) { val = outs[i++]; });
      } else {
        run(st, k);
      }
      done += k;
    }
    Value loss(0.0);
    for (int a = 0; a < 3; ++a) {
      Value com(0.0);
      for (const auto& p : st.x) com += p[a] * Value(1.0 / n);
      const Value d = com - Value(target[a]);
      loss += d * d;
    }
    tape.backward(loss);
    const auto t1 = std::chrono::steady_clock::now();
    if (seconds) *seconds = std::chrono::duration<double>(t1 - t0).count();
    if (loss_out) *loss_out = loss.v;
    std::size_t i = 0;
    for (int p = 0; p < n; ++p)
      for (int a = 0; a < 3; ++a) gx[3 * p + a] = tape.grad(leaves[i++]);
    for (int p = 0; p < n; ++p)
      for (int a = 0; a < 3; ++a) gv[3 * p + a] = tape.grad(leaves[i++]);
    for (int p = 0; p < n; ++p)
      for (int q = 0; q < 9; ++q) gF[9 * p + q] = tape.grad(leaves[i++]);
    for (int p = 0; p < n; ++p)
      for (int q = 0; q < 9; ++q) gC[9 * p + q] = tape.grad(leaves[i++]);
    return 0;
  } catch (const std::exception& e) {
    put_err(e.what(), err, errlen);
    return 1;
  }
}

// (3) restatement on the reference tape: loss + gradients for a rollout of
// n_ctrl control steps x n_sub substeps.  seg = checkpoint segment length in
// substeps (0: record everything on one tape).
int ref_rollout_grad(const OrSim* sim, const OrMat* mats, int nmat, const OrCol* cols, int ncol,
                     const double* cvo, const double* act, int nact, int n, const double* x,
                     const double* v, const double* F, const double* C, const int* material,
                     const int* group, int n_ctrl, int n_sub, const OrLoss* loss, int seg,
                     double* loss_out, double* obs, double* gx, double* gv, double* gF, double* gC,
                     double* gcvo, double* gact, double* gE, double* seconds, char* err, int errlen) {
  using namespace oracle;
  try {
    const SimParams sp = sim_from(*sim);
    const auto t0 = std::chrono::steady_clock::now();
    Tape tape;
    std::vector<double> st0;
    st0.reserve(24 * static_cast<std::size_t>(n));
    st0.insert(st0.end(), x, x + 3 * n);
    st0.insert(st0.end(), v, v + 3 * n);
    st0.insert(st0.end(), F, F + 9 * n);
    st0.insert(st0.end(), C, C + 9 * n);
    std::vector<Value> s_leaves, c_leaves, a_leaves, e_leaves;
    for (double val : st0) s_leaves.push_back(tape.var(val));
    for (int i = 0; i < n_ctrl * ncol * 9; ++i) c_leaves.push_back(tape.var(cvo[i]));
    for (int i = 0; i < n_ctrl * nact; ++i) a_leaves.push_back(tape.var(act[i]));
    for (int i = 0; i < nmat; ++i) e_leaves.push_back(tape.var(mats[i].youngs));
    const std::vector<int> mat_ids(material, material + n);
    std::vector<int> grp(n, 0);
    if (group) grp.assign(group, group + n);

    // substeps k from flattened (state, colliders, act, E) -> flattened state
    auto body = [&, n](std::span<const Value> in, int k) {
      const Value* s = in.data();
      State<Value> stt = state_from<Value>(n, s, s + 3 * n, s + 6 * n, s + 15 * n, mat_ids.data(), grp.data());
      const Value* cp = s + 24 * n;
      std::vector<Collider<Value>> cl;
      for (int c = 0; c < ncol; ++c) cl.push_back(collider_from<Value>(cols[c], cp + 9 * c));
      const Value* ap = cp + 9 * ncol;
      std::vector<Value> a(ap, ap + nact);
      const Value* ep = ap + nact;
      std::vector<Material<Value>> mt;
      for (int i = 0; i < nmat; ++i) mt.push_back(material_from<Value>(mats[i], ep[i]));
      Grid<Value> g;
      for (int q = 0; q < k; ++q) substep(sp, stt, g, mt, cl, a);
      std::vector<Value> out(24 * static_cast<std::size_t>(n));
      for (int p = 0; p < n; ++p) {
        for (int d = 0; d < 3; ++d) {
          out[3 * p + d] = stt.x[p][d];
          out[3 * n + 3 * p + d] = stt.v[p][d];
        }
        for (int q = 0; q < 9; ++q) {
          out[6 * n + 9 * p + q] = stt.F[p].m[q];
          out[15 * n + 9 * p + q] = stt.C[p].m[q];
        }
      }
      return out;
    };

    std::vector<Value> cur = s_leaves;
    Value total(0.0);
    for (int t = 0; t < n_ctrl; ++t) {
      std::vector<Value> extra;
      for (int i = 0; i < ncol * 9; ++i) extra.push_back(c_leaves[t * ncol * 9 + i]);
      for (int i = 0; i < nact; ++i) extra.push_back(a_leaves[t * nact + i]);
      for (int i = 0; i < nmat; ++i) extra.push_back(e_leaves[i]);
      int done = 0;
      while (done < n_sub) {
        const int k = seg > 0 ? std::min(seg, n_sub - done) : n_sub - done;
        std::vector<Value> in = cur;
        in.insert(in.end(), extra.begin(), extra.end());
        if (seg > 0) {
          auto outs = tape.checkpoint([&, k](Tape&, std::span<const Value> vin) { return body(vin, k); }, in);
          cur = outs;
        } else {
          cur = body(std::span<const Value>(in), k);
        }
        done += k;
      }
      // observables on the main tape
      State<Value> stt = state_from<Value>(n, cur.data(), cur.data() + 3 * n, cur.data() + 6 * n,
                                           cur.data() + 15 * n, mat_ids.data(), grp.data());
      Value o[kObsDim];
      if (ncol > 0) {
        const Collider<Value> c0 = collider_from<Value>(cols[0], &c_leaves[t * ncol * 9]);
        observe(stt, &c0, *loss, o);
      } else {
        observe<Value>(stt, nullptr, *loss, o);
      }
      if (obs)
        for (int i = 0; i < kObsDim; ++i) obs[t * kObsDim + i] = o[i].v;
      total = total + step_loss(*loss, o, t == n_ctrl - 1);
    }
    if (total.is_const()) throw std::runtime_error("ref_rollout_grad: loss does not depend on inputs");
    tape.backward(total);
    const auto t1 = std::chrono::steady_clock::now();
    if (seconds) *seconds = std::chrono::duration<double>(t1 - t0).count();
    if (loss_out) *loss_out = total.v;
    for (int i = 0; i < 3 * n; ++i) {
      gx[i] = tape.grad(s_leaves[i]);
      gv[i] = tape.grad(s_leaves[3 * n + i]);
    }
    for (int i = 0; i < 9 * n; ++i) {
      gF[i] = tape.grad(s_leaves[6 * n + i]);
      gC[i] = tape.grad(s_leaves[15 * n + i]);
    }
    if (gcvo)
      for (int i = 0; i < n_ctrl * ncol * 9; ++i) gcvo[i] = tape.grad(c_leaves[i]);
    if (gact)
      for (int i = 0; i < n_ctrl * nact; ++i) gact[i] = tape.grad(a_leaves[i]);
    if (gE)
      for (int i = 0; i < nmat; ++i) gE[i] = tape.grad(e_leaves[i]);
    return 0;
  } catch (const std::exception& e) {
    put_err(e.what(), err, errlen);
    return 1;
  }
}

// (4) the reference's own tasks (tasks.hpp) stepped as EnvBatch does
// (env.hpp:55-117: per-env RngStream(seed, env_offset + i), Task::reset,
// auto-reset at episode_len) with given actions [T][E][A]: rewards [T][E]
// and observations [T+1][E][obs_dim] (before each step and after the last;
// a reset env's next observation is of its reset state).  With w_r != NULL
// the same rollout is recorded on the reference tape, each step a
// recompute-on-backward segment (step_checkpointed restated, algo.hpp:79-104),
// and dact receives dL/dactions of L = sum w_r reward + sum w_o obs (rows
// t >= 1 of w_o; gradients do not cross a reset, algo.hpp:171-178).
}  // extern "C"
namespace {
template <class Task>
diffsim::Value task_step_checkpointed(Tape& tape, const Task& task, typename Task::template State<Value>& st,
                                      const std::vector<Value>& action) {
  const auto shape = diffsim::env::lower_state<Task>(st);
  std::vector<Value> inputs;
  Task::visit(st, [&](Value& v) { inputs.push_back(v); });
  const std::size_t n_state = inputs.size();
  inputs.insert(inputs.end(), action.begin(), action.end());
  auto outs = tape.checkpoint(
      [&task, shape, n_state](Tape&, std::span<const Value> in) {
        auto s = Task::template convert<Value, double>(shape);
        std::size_t i = 0;
        Task::visit(s, [&](Value& v) { v = in[i++]; });
        std::vector<Value> act(in.begin() + n_state, in.end());
        Value r = task.step(s, std::span<const Value>(act));
        std::vector<Value> out;
        Task::visit(s, [&](Value& v) { out.push_back(v); });
        out.push_back(r);
        return out;
      },
      inputs);
  std::size_t i = 0;
  Task::visit(st, [&](Value& v) { v = outs[i++]; });
  return outs.back();
}

template <class Task>
void task_rollout(const Task& task, int n_envs, unsigned long long seed, int env_offset, int T,
                  const double* actions, double* rewards, double* obs, const double* w_r, const double* w_o,
                  double* dact) {
  const int A = task.act_dim(), od = task.obs_dim(), L = task.episode_len();
  for (int i = 0; i < n_envs; ++i) {
    diffsim::RngStream rng(seed, static_cast<std::uint64_t>(env_offset + i));
    typename Task::template State<double> s;
    task.reset(s, rng);
    auto s0 = s;
    auto rng0 = rng;
    int cursor = 0;
    auto put_obs = [&](int t, const std::vector<double>& o) {
      for (int k = 0; k < od; ++k) obs[((std::size_t)t * n_envs + i) * od + k] = o[k];
    };
    put_obs(0, task.observe(s));
    for (int t = 0; t < T; ++t) {
      const double* a = actions + ((std::size_t)t * n_envs + i) * A;
      const double r = task.step(s, std::span<const double>(a, A));
      rewards[(std::size_t)t * n_envs + i] = r;
      if (++cursor >= L) {
        task.reset(s, rng);
        cursor = 0;
      }
      put_obs(t + 1, task.observe(s));
    }
    if (!w_r) continue;
    Tape tape;
    rng = rng0;
    auto st = diffsim::env::lift_state<Task>(tape, s0);
    cursor = 0;
    Value total(0.0);
    std::vector<std::vector<Value>> leaves(T);
    for (int t = 0; t < T; ++t) {
      const double* a = actions + ((std::size_t)t * n_envs + i) * A;
      for (int k = 0; k < A; ++k) leaves[t].push_back(tape.var(a[k]));
      const Value r = task_step_checkpointed(tape, task, st, leaves[t]);
      total = total + r * Value(w_r[(std::size_t)t * n_envs + i]);
      if (++cursor >= L) {  // reset: a fresh (constant-lifted) state
        auto lowered = diffsim::env::lower_state<Task>(st);
        task.reset(lowered, rng);
        st = diffsim::env::lift_state<Task>(tape, lowered);
        cursor = 0;
      } else if (w_o) {
        const auto o = task.observe(st);
        for (int k = 0; k < od; ++k) total = total + o[k] * Value(w_o[((std::size_t)(t + 1) * n_envs + i) * od + k]);
      }
    }
    if (!total.is_const()) tape.backward(total);
    for (int t = 0; t < T; ++t)
      for (int k = 0; k < A; ++k)
        dact[((std::size_t)t * n_envs + i) * A + k] = total.is_const() ? 0.0 : tape.grad(leaves[t][k]);
  }
}
}  // namespace
extern "C" {

// cfg: the DmTaskConfig fields as doubles in header order from grid_n:
// grid_n, ppc, dt, substeps, episode_len, cloud_k, container_half, fill,
// speed, start_x, start_y, target_x, target_y, spill_temp, block_size,
// block_height, roller_radius, roller_speed, h_flat, youngs, yield_stress.
int ref_task_rollout(int kind, const double* cfg, int n_envs, unsigned long long seed, int env_offset, int T,
                     const double* actions, double* rewards, double* obs, const double* w_r, const double* w_o,
                     double* dact, int* dims, char* err, int errlen) {
  try {
    if (kind == 0) {
      diffsim::tasks::MiniFluidMove::Config c;
      c.grid_n = (int)cfg[0];
      c.ppc = (int)cfg[1];
      c.dt = cfg[2];
      c.substeps = (int)cfg[3];
      c.episode_len = (int)cfg[4];
      c.cloud_k = (int)cfg[5];
      c.container_half = cfg[6];
      c.fill = cfg[7];
      c.speed = cfg[8];
      c.start_x = cfg[9];
      c.start_y = cfg[10];
      c.target_x = cfg[11];
      c.target_y = cfg[12];
      c.spill_temp = cfg[13];
      diffsim::tasks::MiniFluidMove task(c);
      if (dims) {
        dims[0] = task.obs_dim();
        dims[1] = task.act_dim();
      }
      if (T > 0) task_rollout(task, n_envs, seed, env_offset, T, actions, rewards, obs, w_r, w_o, dact);
    } else {
      diffsim::tasks::MiniRollFlat::Config c;
      c.grid_n = (int)cfg[0];
      c.ppc = (int)cfg[1];
      c.dt = cfg[2];
      c.substeps = (int)cfg[3];
      c.episode_len = (int)cfg[4];
      c.cloud_k = (int)cfg[5];
      c.block_size = cfg[14];
      c.block_height = cfg[15];
      c.roller_radius = cfg[16];
      c.roller_speed = cfg[17];
      c.h_flat = cfg[18];
      c.youngs = cfg[19];
      c.yield_stress = cfg[20];
      diffsim::tasks::MiniRollFlat task(c);
      if (dims) {
        dims[0] = task.obs_dim();
        dims[1] = task.act_dim();
      }
      if (T > 0) task_rollout(task, n_envs, seed, env_offset, T, actions, rewards, obs, w_r, w_o, dact);
    }
    return 0;
  } catch (const std::exception& e) {
    put_err(e.what(), err, errlen);
    return 1;
  }
}

// The reference samplers (mpm.hpp:371-423): kind 0 sample_box(a = org,
// b = size), 1 sample_cylinder(a = base_center, b = (radius, height, -)).
// x receives up to cap points; returns the count (or -1).
int ref_sample(int kind, const double* a, const double* b, double dx, int ppc, double* x, int cap, double* vol) {
  diffsim::mpm::MpmMaterial m;
  const auto st = kind == 0 ? diffsim::mpm::sample_box({a[0], a[1], a[2]}, {b[0], b[1], b[2]}, dx, ppc, m, 0)
                            : diffsim::mpm::sample_cylinder({a[0], a[1], a[2]}, b[0], b[1], dx, ppc, m, 0);
  const int n = static_cast<int>(st.size());
  if (n > cap) return -1;
  for (int p = 0; p < n; ++p)
    for (int k = 0; k < 3; ++k) x[3 * p + k] = st.x[p][k];
  if (vol) *vol = n ? st.volume0[0] : 0.0;
  return n;
}

// SVD-law adjoint of the gradient oracle (ref_rollout_grad): 1 isotropic-map
// nodes (exact), 0 the reference's Tape::svd3x3.  Returns the previous mode.
int ref_set_svd_adjoint(int mode) {
  const int old = oracle::g_svd_adjoint;
  oracle::g_svd_adjoint = mode;
  return old;
}

// reference RngStream draws (rng.hpp:11-55): kind 0 u64, 1 double, 2 normal
void ref_rng_draws(unsigned long long seed, unsigned long long stream, int n, int kind, double* out,
                   unsigned long long* out_u64) {
  diffsim::RngStream r(seed, stream);
  for (int i = 0; i < n; ++i) {
    if (kind == 0)
      out_u64[i] = r.next_u64();
    else if (kind == 1)
      out[i] = r.next_double();
    else
      out[i] = r.normal();
  }
}

}  // extern "C"
