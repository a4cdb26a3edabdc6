// TEST INFRASTRUCTURE ONLY (oracle).  Never linked into the product path.
//
// 3-vector / row-major 3x3 algebra for the CPU restatement of the reference
// MLS-MPM path.  Follows the conventions of the reference algebra
// (/root/reference/proj/include/diffsim/linalg.hpp:10-162): row-major Mat3,
// det by first-row expansion (123-128), cofactor = det(A) A^{-T}
// (130-144), outer(a, b)_rc = a_r b_c (156-162).  Templated on the scalar so
// the same code runs in fp64 and on the reference's scalar tape.
#pragma once

#include <array>

namespace oracle {

template <class T>
struct V3 {
  T x{}, y{}, z{};
  T& operator[](int i) { return i == 0 ? x : (i == 1 ? y : z); }
  const T& operator[](int i) const { return i == 0 ? x : (i == 1 ? y : z); }
};

template <class T> V3<T> operator+(const V3<T>& a, const V3<T>& b) { return {a.x + b.x, a.y + b.y, a.z + b.z}; }
template <class T> V3<T> operator-(const V3<T>& a, const V3<T>& b) { return {a.x - b.x, a.y - b.y, a.z - b.z}; }
template <class T> V3<T> operator*(const V3<T>& a, const T& s) { return {a.x * s, a.y * s, a.z * s}; }
template <class T> T dot(const V3<T>& a, const V3<T>& b) { return a.x * b.x + a.y * b.y + a.z * b.z; }
template <class T> V3<T> cross(const V3<T>& a, const V3<T>& b) {
  return {a.y * b.z - a.z * b.y, a.z * b.x - a.x * b.z, a.x * b.y - a.y * b.x};
}

template <class T>
struct M3 {
  std::array<T, 9> m{};
  T& operator()(int r, int c) { return m[3 * r + c]; }
  const T& operator()(int r, int c) const { return m[3 * r + c]; }
  static M3 identity() {
    M3 o;
    o.m = {T(1.0), T(0.0), T(0.0), T(0.0), T(1.0), T(0.0), T(0.0), T(0.0), T(1.0)};
    return o;
  }
  static M3 zero() {
    M3 o;
    for (auto& e : o.m) e = T(0.0);
    return o;
  }
  static M3 diag(const T& a, const T& b, const T& c) {
    M3 o = zero();
    o(0, 0) = a;
    o(1, 1) = b;
    o(2, 2) = c;
    return o;
  }
  M3 transposed() const {
    M3 o;
    for (int r = 0; r < 3; ++r)
      for (int c = 0; c < 3; ++c) o(r, c) = (*this)(c, r);
    return o;
  }
};

template <class T> M3<T> operator+(const M3<T>& a, const M3<T>& b) {
  M3<T> o;
  for (int i = 0; i < 9; ++i) o.m[i] = a.m[i] + b.m[i];
  return o;
}
template <class T> M3<T> operator-(const M3<T>& a, const M3<T>& b) {
  M3<T> o;
  for (int i = 0; i < 9; ++i) o.m[i] = a.m[i] - b.m[i];
  return o;
}
template <class T> M3<T> operator*(const M3<T>& a, const T& s) {
  M3<T> o;
  for (int i = 0; i < 9; ++i) o.m[i] = a.m[i] * s;
  return o;
}
template <class T> M3<T> operator*(const M3<T>& a, const M3<T>& b) {
  M3<T> o;
  for (int r = 0; r < 3; ++r)
    for (int c = 0; c < 3; ++c)
      o(r, c) = a(r, 0) * b(0, c) + a(r, 1) * b(1, c) + a(r, 2) * b(2, c);
  return o;
}
template <class T> V3<T> operator*(const M3<T>& a, const V3<T>& v) {
  return {a.m[0] * v.x + a.m[1] * v.y + a.m[2] * v.z,
          a.m[3] * v.x + a.m[4] * v.y + a.m[5] * v.z,
          a.m[6] * v.x + a.m[7] * v.y + a.m[8] * v.z};
}
template <class T> T det(const M3<T>& a) {
  return a(0, 0) * (a(1, 1) * a(2, 2) - a(1, 2) * a(2, 1)) -
         a(0, 1) * (a(1, 0) * a(2, 2) - a(1, 2) * a(2, 0)) +
         a(0, 2) * (a(1, 0) * a(2, 1) - a(1, 1) * a(2, 0));
}
template <class T> M3<T> cofactor(const M3<T>& a) {
  M3<T> o;
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
template <class T> M3<T> outer(const V3<T>& a, const V3<T>& b) {
  M3<T> o;
  for (int r = 0; r < 3; ++r)
    for (int c = 0; c < 3; ++c) o(r, c) = a[r] * b[c];
  return o;
}

}  // namespace oracle
