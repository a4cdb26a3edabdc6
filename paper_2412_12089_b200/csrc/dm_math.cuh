// Register-resident 3-vector / row-major 3x3 algebra for the MLS-MPM kernels.
//
// Templated on the real type so the same code is the fp32 device path and
// (compiled by g++ in fp64) the host adjoint check in tests/native.
// Conventions follow the reference algebra (diffsim/linalg.hpp:10-162):
// row-major 3x3, cofactor(A) = det(A) A^{-T}.
#pragma once

#include <cmath>

#ifdef __CUDACC__
#define DM_HD __host__ __device__ __forceinline__
// large, rarely-hot helpers kept out of line: one copy of the collider code
// instead of one per call site keeps the grid kernels inside the I-cache
#define DM_HD_NOINLINE __host__ __device__ __noinline__
#else
#define DM_HD inline
#define DM_HD_NOINLINE inline
#endif

namespace dm {

template <class R>
struct v3 {
  R x, y, z;
  DM_HD R& operator[](int i) { return i == 0 ? x : (i == 1 ? y : z); }
  DM_HD const R& operator[](int i) const { return i == 0 ? x : (i == 1 ? y : z); }
};

template <class R>
struct m3 {
  R a[9];
  DM_HD R& operator()(int r, int c) { return a[3 * r + c]; }
  DM_HD const R& operator()(int r, int c) const { return a[3 * r + c]; }
};

// ---- scalar helpers (IEEE functions; no fast-math) ----
DM_HD float r_sqrt(float a) { return sqrtf(a); }
DM_HD double r_sqrt(double a) { return sqrt(a); }
DM_HD float r_exp(float a) { return expf(a); }
DM_HD double r_exp(double a) { return exp(a); }
DM_HD float r_log(float a) { return logf(a); }
DM_HD double r_log(double a) { return log(a); }
DM_HD float r_log1p(float a) { return log1pf(a); }
DM_HD double r_log1p(double a) { return log1p(a); }
DM_HD float r_expm1(float a) { return expm1f(a); }
DM_HD double r_expm1(double a) { return expm1(a); }
DM_HD float r_abs(float a) { return fabsf(a); }
DM_HD double r_abs(double a) { return fabs(a); }
DM_HD float r_cbrt(float a) { return cbrtf(a); }
DM_HD double r_cbrt(double a) { return cbrt(a); }
template <class R> DM_HD R r_max(R a, R b) { return a > b ? a : b; }
template <class R> DM_HD R r_min(R a, R b) { return a < b ? a : b; }

// ---- vectors ----
template <class R> DM_HD v3<R> mk3(R x, R y, R z) { return v3<R>{x, y, z}; }
template <class R> DM_HD v3<R> zero3() { return v3<R>{R(0), R(0), R(0)}; }
template <class R> DM_HD v3<R> operator+(v3<R> a, v3<R> b) { return {a.x + b.x, a.y + b.y, a.z + b.z}; }
template <class R> DM_HD v3<R> operator-(v3<R> a, v3<R> b) { return {a.x - b.x, a.y - b.y, a.z - b.z}; }
template <class R> DM_HD v3<R> operator-(v3<R> a) { return {-a.x, -a.y, -a.z}; }
template <class R> DM_HD v3<R> operator*(v3<R> a, R s) { return {a.x * s, a.y * s, a.z * s}; }
template <class R> DM_HD v3<R>& operator+=(v3<R>& a, v3<R> b) {
  a.x += b.x;
  a.y += b.y;
  a.z += b.z;
  return a;
}
template <class R> DM_HD v3<R>& operator-=(v3<R>& a, v3<R> b) {
  a.x -= b.x;
  a.y -= b.y;
  a.z -= b.z;
  return a;
}
template <class R> DM_HD R dot(v3<R> a, v3<R> b) { return a.x * b.x + a.y * b.y + a.z * b.z; }
template <class R> DM_HD v3<R> cross(v3<R> a, v3<R> b) {
  return {a.y * b.z - a.z * b.y, a.z * b.x - a.x * b.z, a.x * b.y - a.y * b.x};
}

// ---- matrices ----
template <class R> DM_HD m3<R> mzero() {
  m3<R> o;
#pragma unroll
  for (int i = 0; i < 9; ++i) o.a[i] = R(0);
  return o;
}
template <class R> DM_HD m3<R> meye() {
  m3<R> o = mzero<R>();
  o.a[0] = o.a[4] = o.a[8] = R(1);
  return o;
}
template <class R> DM_HD m3<R> mdiag(R a, R b, R c) {
  m3<R> o = mzero<R>();
  o.a[0] = a;
  o.a[4] = b;
  o.a[8] = c;
  return o;
}
template <class R> DM_HD m3<R> operator+(const m3<R>& a, const m3<R>& b) {
  m3<R> o;
#pragma unroll
  for (int i = 0; i < 9; ++i) o.a[i] = a.a[i] + b.a[i];
  return o;
}
template <class R> DM_HD m3<R> operator-(const m3<R>& a, const m3<R>& b) {
  m3<R> o;
#pragma unroll
  for (int i = 0; i < 9; ++i) o.a[i] = a.a[i] - b.a[i];
  return o;
}
template <class R> DM_HD m3<R> operator*(const m3<R>& a, R s) {
  m3<R> o;
#pragma unroll
  for (int i = 0; i < 9; ++i) o.a[i] = a.a[i] * s;
  return o;
}
template <class R> DM_HD m3<R>& operator+=(m3<R>& a, const m3<R>& b) {
#pragma unroll
  for (int i = 0; i < 9; ++i) a.a[i] += b.a[i];
  return a;
}
template <class R> DM_HD m3<R> operator*(const m3<R>& a, const m3<R>& b) {
  m3<R> o;
#pragma unroll
  for (int r = 0; r < 3; ++r)
#pragma unroll
    for (int c = 0; c < 3; ++c) o(r, c) = a(r, 0) * b(0, c) + a(r, 1) * b(1, c) + a(r, 2) * b(2, c);
  return o;
}
template <class R> DM_HD v3<R> operator*(const m3<R>& a, v3<R> v) {
  return {a.a[0] * v.x + a.a[1] * v.y + a.a[2] * v.z, a.a[3] * v.x + a.a[4] * v.y + a.a[5] * v.z,
          a.a[6] * v.x + a.a[7] * v.y + a.a[8] * v.z};
}
// a^T v
template <class R> DM_HD v3<R> tmul(const m3<R>& a, v3<R> v) {
  return {a.a[0] * v.x + a.a[3] * v.y + a.a[6] * v.z, a.a[1] * v.x + a.a[4] * v.y + a.a[7] * v.z,
          a.a[2] * v.x + a.a[5] * v.y + a.a[8] * v.z};
}
template <class R> DM_HD m3<R> transpose(const m3<R>& a) {
  m3<R> o;
#pragma unroll
  for (int r = 0; r < 3; ++r)
#pragma unroll
    for (int c = 0; c < 3; ++c) o(r, c) = a(c, r);
  return o;
}
// a * b^T
template <class R> DM_HD m3<R> mul_bt(const m3<R>& a, const m3<R>& b) {
  m3<R> o;
#pragma unroll
  for (int r = 0; r < 3; ++r)
#pragma unroll
    for (int c = 0; c < 3; ++c) o(r, c) = a(r, 0) * b(c, 0) + a(r, 1) * b(c, 1) + a(r, 2) * b(c, 2);
  return o;
}
// a^T * b
template <class R> DM_HD m3<R> mul_at(const m3<R>& a, const m3<R>& b) {
  m3<R> o;
#pragma unroll
  for (int r = 0; r < 3; ++r)
#pragma unroll
    for (int c = 0; c < 3; ++c) o(r, c) = a(0, r) * b(0, c) + a(1, r) * b(1, c) + a(2, r) * b(2, c);
  return o;
}
template <class R> DM_HD R ddot(const m3<R>& a, const m3<R>& b) {
  R s = R(0);
#pragma unroll
  for (int i = 0; i < 9; ++i) s += a.a[i] * b.a[i];
  return s;
}
template <class R> DM_HD R det(const m3<R>& a) {
  return a(0, 0) * (a(1, 1) * a(2, 2) - a(1, 2) * a(2, 1)) - a(0, 1) * (a(1, 0) * a(2, 2) - a(1, 2) * a(2, 0)) +
         a(0, 2) * (a(1, 0) * a(2, 1) - a(1, 1) * a(2, 0));
}
template <class R> DM_HD m3<R> cofactor(const m3<R>& a) {
  m3<R> o;
  o(0, 0) = a(1, 1) * a(2, 2) - a(1, 2) * a(2, 1);
  o(0, 1) = a(1, 2) * a(2, 0) - a(1, 0) * a(2, 2);
  o(0, 2) = a(1, 0) * a(2, 1) - a(1, 1) * a(2, 0);
  o(1, 0) = a(0, 2) * a(2, 1) - a(0, 1) * a(2, 2);
  o(1, 1) = a(0, 0) * a(2, 2) - a(0, 2) * a(2, 0);
  o(1, 2) = a(0, 1) * a(2, 0) - a(0, 0) * a(2, 1);
  o(2, 0) = a(0, 1) * a(1, 2) - a(0, 2) * a(1, 1);
  o(2, 1) = a(0, 2) * a(1, 0) - a(0, 0) * a(1, 2);
  o(2, 2) = a(0, 0) * a(1, 1) - a(0, 1) * a(1, 0);
  return o;
}
// directional derivative of cofactor(a) along d (cofactor is quadratic)
template <class R> DM_HD m3<R> cofactor_jvp(const m3<R>& a, const m3<R>& d) {
  m3<R> o;
  o(0, 0) = d(1, 1) * a(2, 2) + a(1, 1) * d(2, 2) - d(1, 2) * a(2, 1) - a(1, 2) * d(2, 1);
  o(0, 1) = d(1, 2) * a(2, 0) + a(1, 2) * d(2, 0) - d(1, 0) * a(2, 2) - a(1, 0) * d(2, 2);
  o(0, 2) = d(1, 0) * a(2, 1) + a(1, 0) * d(2, 1) - d(1, 1) * a(2, 0) - a(1, 1) * d(2, 0);
  o(1, 0) = d(0, 2) * a(2, 1) + a(0, 2) * d(2, 1) - d(0, 1) * a(2, 2) - a(0, 1) * d(2, 2);
  o(1, 1) = d(0, 0) * a(2, 2) + a(0, 0) * d(2, 2) - d(0, 2) * a(2, 0) - a(0, 2) * d(2, 0);
  o(1, 2) = d(0, 1) * a(2, 0) + a(0, 1) * d(2, 0) - d(0, 0) * a(2, 1) - a(0, 0) * d(2, 1);
  o(2, 0) = d(0, 1) * a(1, 2) + a(0, 1) * d(1, 2) - d(0, 2) * a(1, 1) - a(0, 2) * d(1, 1);
  o(2, 1) = d(0, 2) * a(1, 0) + a(0, 2) * d(1, 0) - d(0, 0) * a(1, 2) - a(0, 0) * d(1, 2);
  o(2, 2) = d(0, 0) * a(1, 1) + a(0, 0) * d(1, 1) - d(0, 1) * a(1, 0) - a(0, 1) * d(1, 0);
  return o;
}
template <class R> DM_HD m3<R> outer(v3<R> a, v3<R> b) {
  m3<R> o;
#pragma unroll
  for (int r = 0; r < 3; ++r)
#pragma unroll
    for (int c = 0; c < 3; ++c) o(r, c) = a[r] * b[c];
  return o;
}

// ---- 3x3 SVD: one-sided (Hestenes) Jacobi on the columns of F ----
// F = U diag(s) V^T with V a rotation; for det F > 0, U is a rotation and
// s > 0.  Singular values are not sorted (no consumer needs an order).
template <class R>
struct Svd {
  m3<R> u, v;  // columns are singular vectors (v, not v^T)
  R s[3];
};

// Returns whether it rotated (a sweep without any rotation leaves g, v
// unchanged, so later sweeps would too: svd3 stops there, bit-identically).
template <class R>
DM_HD bool jacobi_rot(m3<R>& g, m3<R>& v, int p, int q) {
  const R a = g(0, p) * g(0, p) + g(1, p) * g(1, p) + g(2, p) * g(2, p);
  const R b = g(0, q) * g(0, q) + g(1, q) * g(1, q) + g(2, q) * g(2, q);
  const R c = g(0, p) * g(0, q) + g(1, p) * g(1, q) + g(2, p) * g(2, q);
  R cs, sn;
#ifdef __CUDA_ARCH__
  if constexpr (sizeof(R) == 4) {
    // fp32 on the device: the same rotation from MUFU rsqrt/rcp instead of
    // three IEEE sqrt and three IEEE divides; t = sgn(b-a) 2c / (|b-a| +
    // sqrt((b-a)^2 + 4c^2)) is the smaller root of t^2 + 2 zeta t - 1 = 0,
    // zeta = (b-a)/(2c).  Converged at |c| <= 1e-7 sqrt(ab) (tested
    // squared): the fp32 rounding floor of c; a 1e-8 threshold sits below
    // it and ran all 6 sweeps for ~70 % of near-rotation F (3-4 suffice,
    // singular values unchanged at the 4e-7 level).
    if (c * c <= 1e-14f * a * b) return false;
    const float d = b - a, s2 = d * d + 4.f * c * c;
    const float den = fabsf(d) + s2 * rsqrtf(s2);
    const float t = __fdividef(d >= 0.f ? 2.f * c : -2.f * c, den);
    const float q = 1.f + t * t;
    const float c0 = rsqrtf(q);
    cs = c0 * fmaf(-0.5f * q * c0, c0, 1.5f);  // one Newton step: V stays orthonormal to ~1 ulp
    sn = cs * t;
  } else
#endif
  {
    if (r_abs(c) <= R(1e-30) + R(sizeof(R) == 4 ? 1e-8 : 1e-17) * r_sqrt(a * b)) return false;
    const R zeta = (b - a) / (R(2) * c);
    const R t = (zeta >= R(0) ? R(1) : R(-1)) / (r_abs(zeta) + r_sqrt(R(1) + zeta * zeta));
    cs = R(1) / r_sqrt(R(1) + t * t);
    sn = cs * t;
  }
#pragma unroll
  for (int r = 0; r < 3; ++r) {
    const R gp = g(r, p), gq = g(r, q);
    g(r, p) = cs * gp - sn * gq;
    g(r, q) = sn * gp + cs * gq;
    const R vp = v(r, p), vq = v(r, q);
    v(r, p) = cs * vp - sn * vq;
    v(r, q) = sn * vp + cs * vq;
  }
  return true;
}

template <class R>
DM_HD Svd<R> svd3(const m3<R>& f) {
  m3<R> g = f, v = meye<R>();
  const int sweeps = sizeof(R) == 4 ? 6 : 12;
  for (int s = 0; s < sweeps; ++s) {
    bool rot = jacobi_rot(g, v, 0, 1);
    rot = jacobi_rot(g, v, 0, 2) || rot;
    rot = jacobi_rot(g, v, 1, 2) || rot;
    if (!rot) break;  // converged: the remaining sweeps would not change g or v
  }
  if (det(v) < R(0)) {
#pragma unroll
    for (int r = 0; r < 3; ++r) {
      v(r, 2) = -v(r, 2);
      g(r, 2) = -g(r, 2);
    }
  }
  Svd<R> o;
  o.v = v;
#pragma unroll
  for (int c = 0; c < 3; ++c) {
    const R n = r_sqrt(g(0, c) * g(0, c) + g(1, c) * g(1, c) + g(2, c) * g(2, c));
    o.s[c] = n;
    const R inv = n > R(0) ? R(1) / n : R(0);
#pragma unroll
    for (int r = 0; r < 3; ++r) o.u(r, c) = g(r, c) * inv;
  }
  return o;
}

// U diag(d) V^T
template <class R>
DM_HD m3<R> usv(const Svd<R>& sv, R d0, R d1, R d2) {
  m3<R> o;
#pragma unroll
  for (int r = 0; r < 3; ++r)
#pragma unroll
    for (int c = 0; c < 3; ++c)
      o(r, c) = sv.u(r, 0) * d0 * sv.v(c, 0) + sv.u(r, 1) * d1 * sv.v(c, 1) + sv.u(r, 2) * d2 * sv.v(c, 2);
  return o;
}
// U diag(d) U^T (symmetric; the 6 upper entries computed, mirrored)
template <class R>
DM_HD m3<R> udut(const m3<R>& u, R d0, R d1, R d2) {
  m3<R> o;
#pragma unroll
  for (int r = 0; r < 3; ++r)
#pragma unroll
    for (int c = r; c < 3; ++c) {
      o(r, c) = u(r, 0) * d0 * u(c, 0) + u(r, 1) * d1 * u(c, 1) + u(r, 2) * d2 * u(c, 2);
      o(c, r) = o(r, c);
    }
  return o;
}
// the symmetric matrix of 6 stored components (xx, xy, xz, yy, yz, zz)
template <class R>
DM_HD m3<R> sym6(const R* t) {
  m3<R> o;
  o(0, 0) = t[0];
  o(0, 1) = o(1, 0) = t[1];
  o(0, 2) = o(2, 0) = t[2];
  o(1, 1) = t[3];
  o(1, 2) = o(2, 1) = t[4];
  o(2, 2) = t[5];
  return o;
}
// U M V^T
template <class R>
DM_HD m3<R> u_m_vt(const Svd<R>& sv, const m3<R>& m) {
  return mul_bt(sv.u * m, sv.v);
}
// U^T M V
template <class R>
DM_HD m3<R> ut_m_v(const Svd<R>& sv, const m3<R>& m) {
  return mul_at(sv.u, m) * sv.v;
}

// Apply the Jacobian-transpose of an isotropic matrix map
//   Phi(F) = U diag(phi(s)) V^T
// to a cotangent Gbar (already rotated: Ghat = U^T Gbar V), given
//   jd[i][j] = d phi_i / d s_j  and the off-diagonal divided differences
//   dd[i][j] = (phi_i - phi_j) / (s_i - s_j) (symmetric), returns U D V^T.
// Off-diagonal blocks: a = (dd + (phi_i+phi_j)/(s_i+s_j))/2,
//                      b = (dd - (phi_i+phi_j)/(s_i+s_j))/2.
template <class R>
DM_HD m3<R> isotropic_vjp(const Svd<R>& sv, const m3<R>& ghat, const R phi[3], const R jd[3][3],
                          const R dd01, const R dd02, const R dd12) {
  m3<R> d;
#pragma unroll
  for (int i = 0; i < 3; ++i) d(i, i) = jd[0][i] * ghat(0, 0) + jd[1][i] * ghat(1, 1) + jd[2][i] * ghat(2, 2);
  const int P[3][2] = {{0, 1}, {0, 2}, {1, 2}};
  const R DD[3] = {dd01, dd02, dd12};
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    const int i = P[k][0], j = P[k][1];
    const R sp = (phi[i] + phi[j]) / (sv.s[i] + sv.s[j]);
    const R a = R(0.5) * (DD[k] + sp), b = R(0.5) * (DD[k] - sp);
    d(i, j) = a * ghat(i, j) + b * ghat(j, i);
    d(j, i) = a * ghat(j, i) + b * ghat(i, j);
  }
  return u_m_vt(sv, d);
}

// (ln si - ln sj) / (si - sj), stable as si -> sj
template <class R>
DM_HD R log_dd(R si, R sj) {
  const R del = si - sj;
  const R r = del / sj;
  if (r_abs(r) < R(sizeof(R) == 4 ? 2e-3 : 1e-6)) return (R(1) - r * (R(0.5) - r * (R(1) / R(3)))) / sj;
  return r_log1p(r) / del;
}

}  // namespace dm
