// TEST INFRASTRUCTURE ONLY.  fp64 host instantiation of the device physics
// and transfer code (paper_2412_12089_b200/csrc/dm_*.cuh) on a dense grid,
// with the hand-written adjoint run in reverse over stored substep states.
// tests/test_adjoint_host.py compares it with the reference-tape gradient
// oracle (oracle/_ref/libref.so) so adjoint formulas are checked on CPU before
// they run on the GPU.  Never used by the product path.
#include <cmath>
#include <cstdio>
#include <cstring>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../oracle/include/oracle/capi_types.h"
#include "../../paper_2412_12089_b200/csrc/dm_transfer.cuh"

using namespace dm;
using R = double;
constexpr int MAXC = 4;

namespace {

struct Setup {
  NodeCtx<R> g;
  TransferCtx<R> t;
  std::vector<Law<R>> laws;
  int nn;
};

Setup make_setup(const OrSim* sim, const OrMat* mats, int nmat) {
  Setup s;
  for (int a = 0; a < 3; ++a) {
    s.g.dims[a] = sim->dims[a];
    s.t.dims[a] = sim->dims[a];
  }
  s.g.dx = sim->dx;
  s.g.dx_lo = 0.0;
  s.g.dt = sim->dt;
  s.g.gravity = mk3(sim->gravity[0], sim->gravity[1], sim->gravity[2]);
  s.g.boundary = sim->boundary;
  s.g.alpha_c = sim->alpha_c;
  s.g.mu_b = sim->mu_b;
  s.t.dx = sim->dx;
  s.t.inv_dx = 1.0 / sim->dx;
  s.t.dt = sim->dt;
  s.t.dx64 = sim->dx;
  for (int i = 0; i < nmat; ++i) {
    const OrMat& m = mats[i];
    Law<R> L{};
    L.kind = m.kind;
    const double nu = m.poisson;
    L.mu = m.youngs / (2.0 * (1.0 + nu));
    L.dmu_dE = 1.0 / (2.0 * (1.0 + nu));
    if (m.kind == 3 && m.bulk > 0.0) {
      L.lam = m.bulk;
      L.dlam_dE = 0.0;
    } else {
      L.lam = m.youngs * nu / ((1.0 + nu) * (1.0 - 2.0 * nu));
      L.dlam_dE = nu / ((1.0 + nu) * (1.0 - 2.0 * nu));
    }
    L.cy = m.wide_yield ? m.yield_stress / L.mu : m.yield_stress / (2.0 * L.mu);
    L.visc = m.viscosity;
    L.act_k = m.act_strength;
    L.mass = m.density * m.volume;
    L.vol = m.volume;
    s.laws.push_back(L);
  }
  s.nn = sim->dims[0] * sim->dims[1] * sim->dims[2];
  return s;
}

std::vector<Col<R>> make_cols(const OrCol* cols, int ncol, const double* cvo) {
  std::vector<Col<R>> out;
  for (int c = 0; c < ncol; ++c) {
    Col<R> k{};
    k.kind = cols[c].kind;
    const double* p = cvo + 9 * c;
    k.c = mk3(p[0], p[1], p[2]);
    k.vel = mk3(p[3], p[4], p[5]);
    k.om = mk3(p[6], p[7], p[8]);
    k.nrm = mk3(cols[c].normal[0], cols[c].normal[1], cols[c].normal[2]);
    k.radius = cols[c].radius;
    k.length = cols[c].length;
    k.thickness = cols[c].thickness;
    k.half = mk3(cols[c].half[0], cols[c].half[1], cols[c].half[2]);
    out.push_back(k);
  }
  return out;
}

struct St {
  std::vector<double> x, v, F, C;  // n*3, n*3, n*9, n*9
};

inline int nidx(const Setup& s, int i, int j, int k) { return (i * s.g.dims[1] + j) * s.g.dims[2] + k; }

void p2g(const Setup& s, const St& st, int n, const int* mat, const int* grp, const double* act,
         std::vector<double>& gm, std::vector<double>& gp) {
  gm.assign(s.nn, 0.0);
  gp.assign(3 * s.nn, 0.0);
  for (int p = 0; p < n; ++p) {
    Stencil<R> sc;
    if (make_stencil(&st.x[3 * p], s.t.inv_dx, s.t.dx64, s.t.dims, sc) >= 0)
      throw std::runtime_error("mpm: particle " + std::to_string(p) + " outside grid interior");
    const Law<R>& L = s.laws[mat[p]];
    m3<R> F, C;
    for (int i = 0; i < 9; ++i) {
      F.a[i] = st.F[9 * p + i];
      C.a[i] = st.C[9 * p + i];
    }
    bool bad = false;
    const R a = act ? act[grp[p]] : 0.0;
    const m3<R> A = p2g_affine(L, s.t, F - meye<R>(), C, a, &bad);  // the device's deviation form D = F - I
    v3<R> q;
    m3<R> Ad;
    p2g_payload(A, L.mass, mk3(st.v[3 * p], st.v[3 * p + 1], st.v[3 * p + 2]), sc, s.t.dx, q, Ad);
    for (int i = 0; i < 3; ++i)
      for (int j = 0; j < 3; ++j)
        for (int k = 0; k < 3; ++k) {
          const R w = sc.w[0][i] * sc.w[1][j] * sc.w[2][k];
          const int nd = nidx(s, sc.base[0] + i, sc.base[1] + j, sc.base[2] + k);
          gm[nd] += w * L.mass;
          const v3<R> mo = (q + Ad * mk3(R(i), R(j), R(k))) * w;
          gp[3 * nd] += mo.x;
          gp[3 * nd + 1] += mo.y;
          gp[3 * nd + 2] += mo.z;
        }
  }
}

void grid(const Setup& s, const std::vector<Col<R>>& cols, const std::vector<double>& gm,
          const std::vector<double>& gp, std::vector<double>& gv) {
  gv.assign(3 * s.nn, 0.0);
  for (int i = 0; i < s.g.dims[0]; ++i)
    for (int j = 0; j < s.g.dims[1]; ++j)
      for (int k = 0; k < s.g.dims[2]; ++k) {
        const int nd = nidx(s, i, j, k);
        const int idx[3] = {i, j, k};
        const v3<R> v = node_update<R, MAXC>(s.g, cols.data(), (int)cols.size(), idx, gm[nd],
                                             mk3(gp[3 * nd], gp[3 * nd + 1], gp[3 * nd + 2]));
        gv[3 * nd] = v.x;
        gv[3 * nd + 1] = v.y;
        gv[3 * nd + 2] = v.z;
      }
}

void substep(const Setup& s, St& st, int n, const int* mat, const int* grp, const double* act,
             const std::vector<Col<R>>& cols) {
  std::vector<double> gm, gp, gv;
  p2g(s, st, n, mat, grp, act, gm, gp);
  grid(s, cols, gm, gp, gv);
  for (int p = 0; p < n; ++p) {
    Stencil<R> sc;
    make_stencil(&st.x[3 * p], s.t.inv_dx, s.t.dx64, s.t.dims, sc);
    auto getv = [&](int i, int j, int k) {
      const int nd = nidx(s, sc.base[0] + i, sc.base[1] + j, sc.base[2] + k);
      return mk3(gv[3 * nd], gv[3 * nd + 1], gv[3 * nd + 2]);
    };
    v3<R> x = mk3(st.x[3 * p], st.x[3 * p + 1], st.x[3 * p + 2]), v;
    m3<R> F, C;
    for (int i = 0; i < 9; ++i) F.a[i] = st.F[9 * p + i];
    bool ba = false, bd = false;
    m3<R> D = F - meye<R>();
    g2p_particle_sep(s.laws[mat[p]], s.t, sc, getv, x, v, C, D, &ba, &bd, zero3<R>());
    F = D + meye<R>();
    if (ba) throw std::runtime_error("g2p: particle " + std::to_string(p) + " advected outside grid interior");
    for (int a = 0; a < 3; ++a) {
      st.x[3 * p + a] = x[a];
      st.v[3 * p + a] = v[a];
    }
    for (int i = 0; i < 9; ++i) {
      st.F[9 * p + i] = F.a[i];
      st.C[9 * p + i] = C.a[i];
    }
  }
}

void observe(const St& st, int n, const Col<R>* c0, double half, double temp, double* o) {
  double m[3] = {0, 0, 0}, var[3] = {0, 0, 0}, sp = 0.0;
  for (int p = 0; p < n; ++p)
    for (int a = 0; a < 3; ++a) m[a] += st.x[3 * p + a] / n;
  for (int p = 0; p < n; ++p)
    for (int a = 0; a < 3; ++a) {
      const double d = st.x[3 * p + a] - m[a];
      var[a] += d * d / n;
    }
  if (c0 && temp > 0.0)
    for (int p = 0; p < n; ++p) {
      const double sd = std::max(std::fabs(st.x[3 * p] - c0->c.x), std::fabs(st.x[3 * p + 1] - c0->c.y)) - half;
      sp += (1.0 / n) / (1.0 + std::exp(-sd / temp));
    }
  for (int a = 0; a < 3; ++a) {
    o[a] = m[a];
    o[3 + a] = var[a];
  }
  o[6] = sp;
}

// obs adjoint into xbar; returns collider-0 center cotangent (x, y)
void observe_vjp(const St& st, int n, const Col<R>* c0, double half, double temp, const double* ob, double* xb,
                 double* cb) {
  double m[3] = {0, 0, 0};
  for (int p = 0; p < n; ++p)
    for (int a = 0; a < 3; ++a) m[a] += st.x[3 * p + a] / n;
  for (int p = 0; p < n; ++p)
    for (int a = 0; a < 3; ++a) xb[3 * p + a] += ob[a] / n + ob[3 + a] * 2.0 * (st.x[3 * p + a] - m[a]) / n;
  if (c0 && temp > 0.0 && ob[6] != 0.0)
    for (int p = 0; p < n; ++p) {
      const double dx_ = st.x[3 * p] - c0->c.x, dy_ = st.x[3 * p + 1] - c0->c.y;
      const double ax = std::fabs(dx_), ay = std::fabs(dy_);
      const double sd = std::max(ax, ay) - half;
      const double sg = 1.0 / (1.0 + std::exp(-sd / temp));
      const double g = ob[6] / n * sg * (1.0 - sg) / temp;
      if (ax > ay) {
        const double sgn = dx_ > 0 ? 1.0 : (dx_ < 0 ? -1.0 : 0.0);
        xb[3 * p] += g * sgn;
        cb[0] -= g * sgn;
      } else if (ay > ax) {
        const double sgn = dy_ > 0 ? 1.0 : (dy_ < 0 ? -1.0 : 0.0);
        xb[3 * p + 1] += g * sgn;
        cb[1] -= g * sgn;
      }
    }
}

}  // namespace

extern "C" int hc_rollout(const OrSim* sim, const OrMat* mats, int nmat, const OrCol* ocols, int ncol,
                          const double* cvo, const double* act, int nact, int n, const double* x, const double* v,
                          const double* F, const double* C, const int* material, const int* group, int n_ctrl,
                          int n_sub, double spill_half, double spill_temp, double* obs, const double* dobs,
                          double* gx, double* gv, double* gF, double* gC, double* gcvo, double* gact, double* gE,
                          char* err, int errlen) {
  try {
    const Setup s = make_setup(sim, mats, nmat);
    std::vector<St> states;
    St st{std::vector<double>(x, x + 3 * n), std::vector<double>(v, v + 3 * n), std::vector<double>(F, F + 9 * n),
          std::vector<double>(C, C + 9 * n)};
    for (int t = 0; t < n_ctrl; ++t) {
      const auto cols = make_cols(ocols, ncol, cvo + t * ncol * 9);
      const double* a = nact ? act + t * nact : nullptr;
      for (int q = 0; q < n_sub; ++q) {
        states.push_back(st);
        substep(s, st, n, material, group, a, cols);
      }
      observe(st, n, ncol ? &cols[0] : nullptr, spill_half, spill_temp, obs + 7 * t);
    }
    states.push_back(st);
    if (!dobs) return 0;
    // ---- reverse ----
    St bar{std::vector<double>(3 * n, 0.0), std::vector<double>(3 * n, 0.0), std::vector<double>(9 * n, 0.0),
           std::vector<double>(9 * n, 0.0)};
    std::vector<double> gEl(nmat, 0.0);
    for (int i = 0; i < n_ctrl * ncol * 9; ++i) gcvo[i] = 0.0;
    for (int i = 0; i < n_ctrl * nact; ++i) gact[i] = 0.0;
    for (int t = n_ctrl - 1; t >= 0; --t) {
      const auto cols = make_cols(ocols, ncol, cvo + t * ncol * 9);
      const double* a = nact ? act + t * nact : nullptr;
      {
        double cb[2] = {0.0, 0.0};
        observe_vjp(states[(t + 1) * n_sub], n, ncol ? &cols[0] : nullptr, spill_half, spill_temp, dobs + 7 * t,
                    bar.x.data(), cb);
        if (ncol) {
          gcvo[t * ncol * 9 + 0] += cb[0];
          gcvo[t * ncol * 9 + 1] += cb[1];
        }
      }
      for (int q = n_sub - 1; q >= 0; --q) {
        const St& s0 = states[t * n_sub + q];
        std::vector<double> gm, gp, gvel;
        p2g(s, s0, n, material, group, a, gm, gp);
        grid(s, cols, gm, gp, gvel);
        // G2P adjoint: particle partials + vbar scatter
        std::vector<double> vbar(3 * s.nn, 0.0);
        std::vector<double> xpart(3 * n), Fpart(9 * n);
        std::vector<double> mub(nmat, 0.0), lamb(nmat, 0.0);
        for (int p = 0; p < n; ++p) {
          Stencil<R> sc;
          make_stencil(&s0.x[3 * p], s.t.inv_dx, s.t.dx64, s.t.dims, sc);
          auto getv = [&](int i, int j, int k) {
            const int nd = nidx(s, sc.base[0] + i, sc.base[1] + j, sc.base[2] + k);
            return mk3(gvel[3 * nd], gvel[3 * nd + 1], gvel[3 * nd + 2]);
          };
          m3<R> Fm, Cb, Fb;
          for (int i = 0; i < 9; ++i) {
            Fm.a[i] = s0.F[9 * p + i];
            Cb.a[i] = bar.C[9 * p + i];
            Fb.a[i] = bar.F[9 * p + i];
          }
          v3<R> xp, gq;
          m3<R> Fp, Bd;
          g2p_vjp_sep(s.laws[material[p]], s.t, sc, getv, Fm, mk3(bar.x[3 * p], bar.x[3 * p + 1], bar.x[3 * p + 2]),
                  mk3(bar.v[3 * p], bar.v[3 * p + 1], bar.v[3 * p + 2]), Cb, Fb, xp, Fp, gq, Bd, mub[material[p]]);
          for (int a2 = 0; a2 < 3; ++a2) xpart[3 * p + a2] = xp[a2];
          for (int i = 0; i < 9; ++i) Fpart[9 * p + i] = Fp.a[i];
          for (int i = 0; i < 3; ++i)
            for (int j = 0; j < 3; ++j)
              for (int k = 0; k < 3; ++k) {
                const R w = sc.w[0][i] * sc.w[1][j] * sc.w[2][k];
                const int nd = nidx(s, sc.base[0] + i, sc.base[1] + j, sc.base[2] + k);
                const v3<R> c = (gq + Bd * mk3(R(i), R(j), R(k))) * w;
                vbar[3 * nd] += c.x;
                vbar[3 * nd + 1] += c.y;
                vbar[3 * nd + 2] += c.z;
              }
        }
        // grid adjoint
        std::vector<double> mb(s.nn, 0.0), pb(3 * s.nn, 0.0);
        std::vector<double> cg(9 * MAXC, 0.0);
        for (int i = 0; i < s.g.dims[0]; ++i)
          for (int j = 0; j < s.g.dims[1]; ++j)
            for (int k = 0; k < s.g.dims[2]; ++k) {
              const int nd = nidx(s, i, j, k);
              const int idx[3] = {i, j, k};
              R mbar;
              v3<R> pbar;
              node_update_vjp<R, MAXC>(s.g, cols.data(), (int)cols.size(), idx, gm[nd],
                                       mk3(gp[3 * nd], gp[3 * nd + 1], gp[3 * nd + 2]),
                                       mk3(vbar[3 * nd], vbar[3 * nd + 1], vbar[3 * nd + 2]), mbar, pbar, cg.data());
              mb[nd] = mbar;
              pb[3 * nd] = pbar.x;
              pb[3 * nd + 1] = pbar.y;
              pb[3 * nd + 2] = pbar.z;
            }
        for (int c = 0; c < ncol; ++c)
          for (int i = 0; i < 9; ++i) gcvo[(t * ncol + c) * 9 + i] += cg[9 * c + i];
        // P2G adjoint
        St nb{std::vector<double>(3 * n), std::vector<double>(3 * n), std::vector<double>(9 * n),
              std::vector<double>(9 * n)};
        for (int p = 0; p < n; ++p) {
          Stencil<R> sc;
          make_stencil(&s0.x[3 * p], s.t.inv_dx, s.t.dx64, s.t.dims, sc);
          auto getmb = [&](int i, int j, int k, R& m_, v3<R>& p_) {
            const int nd = nidx(s, sc.base[0] + i, sc.base[1] + j, sc.base[2] + k);
            m_ = mb[nd];
            p_ = mk3(pb[3 * nd], pb[3 * nd + 1], pb[3 * nd + 2]);
          };
          m3<R> Fm, Cm, Fb, Cb = mzero<R>();
          for (int i = 0; i < 9; ++i) {
            Fm.a[i] = s0.F[9 * p + i];
            Cm.a[i] = s0.C[9 * p + i];
            Fb.a[i] = Fpart[9 * p + i];
          }
          v3<R> xb = mk3(xpart[3 * p], xpart[3 * p + 1], xpart[3 * p + 2]), vb = zero3<R>();
          R actb = 0.0;
          const R av = a ? a[group[p]] : 0.0;
          p2g_vjp_sep(s.laws[material[p]], s.t, sc, getmb, mk3(s0.v[3 * p], s0.v[3 * p + 1], s0.v[3 * p + 2]), Fm, Cm, av,
                  xb, vb, Fb, Cb, mub[material[p]], lamb[material[p]], actb);
          if (nact) gact[t * nact + group[p]] += actb;
          for (int a2 = 0; a2 < 3; ++a2) {
            nb.x[3 * p + a2] = xb[a2];
            nb.v[3 * p + a2] = vb[a2];
          }
          for (int i = 0; i < 9; ++i) {
            nb.F[9 * p + i] = Fb.a[i];
            nb.C[9 * p + i] = Cb.a[i];
          }
        }
        for (int m = 0; m < nmat; ++m) gEl[m] += mub[m] * s.laws[m].dmu_dE + lamb[m] * s.laws[m].dlam_dE;
        bar = nb;
      }
    }
    std::memcpy(gx, bar.x.data(), sizeof(double) * 3 * n);
    std::memcpy(gv, bar.v.data(), sizeof(double) * 3 * n);
    std::memcpy(gF, bar.F.data(), sizeof(double) * 9 * n);
    std::memcpy(gC, bar.C.data(), sizeof(double) * 9 * n);
    for (int m = 0; m < nmat; ++m) gE[m] = gEl[m];
    return 0;
  } catch (const std::exception& e) {
    std::snprintf(err, errlen, "%s", e.what());
    return 1;
  }
}
