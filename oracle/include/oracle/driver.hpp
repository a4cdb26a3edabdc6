// TEST INFRASTRUCTURE ONLY (oracle).  Never linked into the product path.
//
// Rollout driver shared by the fp64 oracle and the tape-gradient oracle:
// T control steps of S substeps each, colliders frozen at their per-step pose
// for all substeps of the step (the reference task semantics,
// tasks.hpp:311-316, 577-589), observables after every control step, and the
// scalar losses of SURVEY.md section 8(d).
#pragma once

#include <vector>

#include "oracle/capi_types.h"
#include "oracle/mpm.hpp"

namespace oracle {

inline SimParams sim_from(const OrSim& s) {
  SimParams sp;
  for (int a = 0; a < 3; ++a) {
    sp.dims[a] = s.dims[a];
    sp.gravity[a] = s.gravity[a];
  }
  sp.dx = s.dx;
  sp.dt = s.dt;
  sp.boundary = s.boundary;
  sp.alpha_c = s.alpha_c;
  sp.mu_b = s.mu_b;
  return sp;
}

template <class T>
Material<T> material_from(const OrMat& m, const T& youngs) {
  Material<T> o;
  o.kind = m.kind;
  o.youngs = youngs;
  o.poisson = m.poisson;
  o.density = m.density;
  o.volume = m.volume;
  o.yield_stress = m.yield_stress;
  o.wide_yield = m.wide_yield;
  o.viscosity = m.viscosity;
  o.act_strength = m.act_strength;
  o.bulk = m.bulk;
  return o;
}

// Collider whose center/velocity/omega are the given scalars (tape leaves or
// plain doubles).
template <class T>
Collider<T> collider_from(const OrCol& c, const T* cvo /* center3, vel3, omega3 */) {
  Collider<T> o;
  o.kind = c.kind;
  o.center = {cvo[0], cvo[1], cvo[2]};
  o.velocity = {cvo[3], cvo[4], cvo[5]};
  o.omega = {cvo[6], cvo[7], cvo[8]};
  o.normal = {c.normal[0], c.normal[1], c.normal[2]};
  o.radius = c.radius;
  o.half = {c.half[0], c.half[1], c.half[2]};
  o.length = c.length;
  o.thickness = c.thickness;
  return o;
}

template <class T>
State<T> state_from(int n, const T* x, const T* v, const T* F, const T* C, const int* material,
                    const int* group) {
  State<T> st;
  st.x.resize(n);
  st.v.resize(n);
  st.F.resize(n);
  st.C.resize(n);
  st.material.assign(material, material + n);
  if (group)
    st.group.assign(group, group + n);
  else
    st.group.assign(n, 0);
  for (int p = 0; p < n; ++p) {
    st.x[p] = {x[3 * p], x[3 * p + 1], x[3 * p + 2]};
    st.v[p] = {v[3 * p], v[3 * p + 1], v[3 * p + 2]};
    for (int i = 0; i < 9; ++i) {
      st.F[p].m[i] = F[9 * p + i];
      st.C[p].m[i] = C[9 * p + i];
    }
  }
  return st;
}

// Observables after a control step: com(3), var(3), spill(1).
constexpr int kObsDim = 7;

template <class T>
void observe(const State<T>& st, const Collider<T>* col0, const OrLoss& loss, T* obs) {
  const V3<T> com = center_of_mass(st);
  const V3<T> var = position_variance(st, com);
  for (int a = 0; a < 3; ++a) {
    obs[a] = com[a];
    obs[3 + a] = var[a];
  }
  if (col0 && loss.spill_temp > 0.0)
    obs[6] = spill_fraction(st, col0->center.x, col0->center.y, loss.spill_half, loss.spill_temp);
  else
    obs[6] = T(0.0);
}

// Per-step loss contribution (is_last marks the final control step).
template <class T>
T step_loss(const OrLoss& loss, const T* obs, bool is_last) {
  switch (loss.kind) {
    case 0: {
      if (!is_last) return T(0.0);
      T acc(0.0);
      for (int a = 0; a < 3; ++a) {
        const T d = obs[a] - T(loss.target[a]);
        acc = acc + d * d;
      }
      return acc;
    }
    case 1:
      return T(0.0) - obs[2];
    case 2:
      return obs[5];
    case 3:
    default: {
      T acc(0.0);
      for (int a = 0; a < 3; ++a) {
        const T d = obs[a] - T(loss.target[a]);
        acc = acc + d * d;
      }
      const T dist = sqrt(acc + T(1e-12));
      const T r = reward_distance_tiered(dist, loss.tier_threshold, loss.tier_low, loss.tier_high);
      return T(0.0) - (r - obs[6]);
    }
  }
}

}  // namespace oracle
