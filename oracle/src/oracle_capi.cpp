// TEST INFRASTRUCTURE ONLY (oracle).  fp64 forward oracle, C ABI for ctypes.
// Standalone: includes only oracle/ headers, so it also builds without
// /root/reference present.  Only tests/, __graft_entry__.smoke() and
// bench.py's cpu_baseline leg may load it.
#include <cstdio>
#include <cstring>
#include <exception>
#include <vector>

#include "oracle/driver.hpp"

using namespace oracle;

namespace {
void put_err(const char* msg, char* err, int errlen) {
  if (err && errlen > 0) {
    std::snprintf(err, static_cast<std::size_t>(errlen), "%s", msg);
  }
}
}  // namespace

extern "C" {

// Runs n_ctrl control steps of n_sub substeps in place on an fp64 state.
//   cols:  ncol descriptors (geometry); cvo: [n_ctrl][ncol][9] center, vel, omega
//   act:   [n_ctrl][nact] actuation per group
//   obs:   [n_ctrl][7] (com, var, spill) after every control step (may be null)
//   loss_out: scalar loss per OrLoss (may be null)
int or_rollout(const OrSim* sim, const OrMat* mats, int nmat, const OrCol* cols, int ncol,
               const double* cvo, const double* act, int nact, int n, double* x, double* v,
               double* F, double* C, const int* material, const int* group, int n_ctrl, int n_sub,
               const OrLoss* loss, double* obs, double* loss_out, char* err, int errlen) {
  try {
    const SimParams sp = sim_from(*sim);
    std::vector<Material<double>> mt;
    for (int i = 0; i < nmat; ++i) mt.push_back(material_from<double>(mats[i], mats[i].youngs));
    State<double> st = state_from<double>(n, x, v, F, C, material, group);
    Grid<double> g;
    double total = 0.0;
    OrLoss no_loss{};
    no_loss.kind = 2;
    const OrLoss& ls = loss ? *loss : no_loss;
    for (int t = 0; t < n_ctrl; ++t) {
      std::vector<Collider<double>> cl;
      for (int c = 0; c < ncol; ++c) cl.push_back(collider_from<double>(cols[c], cvo + (t * ncol + c) * 9));
      std::vector<double> a;
      if (nact > 0) a.assign(act + t * nact, act + (t + 1) * nact);
      for (int s = 0; s < n_sub; ++s) substep(sp, st, g, mt, cl, a);
      double o[kObsDim];
      observe(st, ncol > 0 ? &cl[0] : nullptr, ls, o);
      if (obs) std::memcpy(obs + t * kObsDim, o, sizeof(o));
      total += step_loss(ls, o, t == n_ctrl - 1);
    }
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
    if (loss_out) *loss_out = total;
    return 0;
  } catch (const std::exception& e) {
    put_err(e.what(), err, errlen);
    return 1;
  }
}

// Dense grid after p2g (+ grid_update when do_update): mass[n], mom[n][3], vel[n][3].
int or_p2g_grid(const OrSim* sim, const OrMat* mats, int nmat, const OrCol* cols, int ncol,
                const double* cvo, const double* act, int n, const double* x, const double* v,
                const double* F, const double* C, const int* material, const int* group,
                double* mass, double* mom, double* vel, char* err, int errlen) {
  try {
    const SimParams sp = sim_from(*sim);
    std::vector<Material<double>> mt;
    for (int i = 0; i < nmat; ++i) mt.push_back(material_from<double>(mats[i], mats[i].youngs));
    State<double> st = state_from<double>(n, x, v, F, C, material, group);
    std::vector<Collider<double>> cl;
    for (int c = 0; c < ncol; ++c) cl.push_back(collider_from<double>(cols[c], cvo + c * 9));
    std::vector<double> a(act, act + (act ? 8 : 0));
    Grid<double> g;
    p2g(sp, st, g, mt, a);
    const int nn = sp.node_count();
    for (int i = 0; i < nn; ++i) {
      mass[i] = g.mass[i];
      for (int k = 0; k < 3; ++k) mom[3 * i + k] = g.momentum[i][k];
    }
    grid_update(sp, g, cl);
    for (int i = 0; i < nn; ++i)
      for (int k = 0; k < 3; ++k) vel[3 * i + k] = g.vel[i][k];
    return 0;
  } catch (const std::exception& e) {
    put_err(e.what(), err, errlen);
    return 1;
  }
}

// Law evaluation: P and projected F for nf matrices (row-major, 9 each).
int or_stress(const OrMat* mat, int nf, const double* F, double act, double* P, double* Fp, char* err,
              int errlen) {
  try {
    const Material<double> m = material_from<double>(*mat, mat->youngs);
    for (int i = 0; i < nf; ++i) {
      M3<double> f, fp;
      for (int k = 0; k < 9; ++k) f.m[k] = F[9 * i + k];
      const M3<double> p = material_stress(f, m, act, fp);
      for (int k = 0; k < 9; ++k) {
        P[9 * i + k] = p.m[k];
        Fp[9 * i + k] = fp.m[k];
      }
    }
    return 0;
  } catch (const std::exception& e) {
    put_err(e.what(), err, errlen);
    return 1;
  }
}

// SDF query for np points: d[np], n[np][3]
void or_collider_query(const OrCol* col, int np, const double* p, double* d, double* nrm) {
  const Collider<double> c = collider_from<double>(*col, col->center);  // center, velocity, omega contiguous
  for (int i = 0; i < np; ++i) {
    double dd;
    V3<double> nn;
    collider_query(c, V3<double>{p[3 * i], p[3 * i + 1], p[3 * i + 2]}, dd, nn);
    d[i] = dd;
    for (int a = 0; a < 3; ++a) nrm[3 * i + a] = nn[a];
  }
}

void or_svd3(const double* f, double* u, double* s, double* vt) { svd3x3_values(f, u, s, vt); }

void or_bin_keys(const OrSim* sim, const float* x, int n, int* keys) {
  bin_keys_f32(sim_from(*sim), x, static_cast<std::size_t>(n), keys);
}

void or_stable_sort(const int* keys, int n, int* perm) {
  stable_sort_perm(keys, static_cast<std::size_t>(n), perm);
}

}  // extern "C"
