// ORACLE — test infrastructure only (tests/, __graft_entry__.smoke(), bench.py cpu_baseline).
// Plain dense FP64 polynomial algebra used by the oracle's transcription of the paper.
// Shares no code with paper_2405_13409_b200/csrc (the CUDA path).
//
// Univariate p(v) = sum_i c[i] v^i (ascending powers).
// Bivariate  p(u,v) = sum_{i+j<=deg} c(i,j) u^i v^j, dense triangular grid
// ("dense coefficient grids"); the coefficient slices a_i(v) of u^i are the
// objects PAPER.md:587-595 (Sec. 5.1) feeds to the Bezout matrix.
#pragma once
#include <algorithm>
#include <cmath>
#include <vector>

namespace oracle {

struct Uni {
  std::vector<double> c;  // c[i] multiplies v^i
  Uni() : c(1, 0.0) {}
  explicit Uni(std::vector<double> cc) : c(std::move(cc)) { if (c.empty()) c.push_back(0.0); }
  int deg() const { return (int)c.size() - 1; }
  double operator()(double x) const {  // Horner
    double s = 0.0;
    for (int i = (int)c.size() - 1; i >= 0; --i) s = s * x + c[i];
    return s;
  }
  double maxabs() const {
    double m = 0.0;
    for (double x : c) m = std::max(m, std::fabs(x));
    return m;
  }
  // exact-zero trim of the leading coefficients ("exact-zero trim only")
  void trim() {
    while (c.size() > 1 && c.back() == 0.0) c.pop_back();
  }
};

inline Uni operator+(const Uni& a, const Uni& b) {
  Uni r(std::vector<double>(std::max(a.c.size(), b.c.size()), 0.0));
  for (size_t i = 0; i < a.c.size(); ++i) r.c[i] += a.c[i];
  for (size_t i = 0; i < b.c.size(); ++i) r.c[i] += b.c[i];
  return r;
}
inline Uni operator-(const Uni& a, const Uni& b) {
  Uni r(std::vector<double>(std::max(a.c.size(), b.c.size()), 0.0));
  for (size_t i = 0; i < a.c.size(); ++i) r.c[i] += a.c[i];
  for (size_t i = 0; i < b.c.size(); ++i) r.c[i] -= b.c[i];
  return r;
}
inline Uni operator*(const Uni& a, const Uni& b) {
  Uni r(std::vector<double>(a.c.size() + b.c.size() - 1, 0.0));
  for (size_t i = 0; i < a.c.size(); ++i)
    for (size_t j = 0; j < b.c.size(); ++j) r.c[i + j] += a.c[i] * b.c[j];
  return r;
}
inline Uni operator*(double s, const Uni& a) {
  Uni r = a;
  for (double& x : r.c) x *= s;
  return r;
}
inline Uni derivative(const Uni& p) {
  if (p.c.size() <= 1) return Uni();
  std::vector<double> d(p.c.size() - 1);
  for (size_t i = 1; i < p.c.size(); ++i) d[i - 1] = (double)i * p.c[i];
  return Uni(d);
}

struct Biv {
  int deg = 0;
  std::vector<double> c;  // (deg+1)*(deg+1) square storage, only i+j<=deg used
  Biv() : deg(0), c(1, 0.0) {}
  explicit Biv(int d) : deg(d), c((size_t)(d + 1) * (d + 1), 0.0) {}
  static Biv constant(double x) { Biv b(0); b.c[0] = x; return b; }
  // 1st-degree polynomial alpha + beta*u + gamma*v
  static Biv linear(double alpha, double beta, double gamma) {
    Biv b(1);
    b.at(0, 0) = alpha; b.at(1, 0) = beta; b.at(0, 1) = gamma;
    return b;
  }
  double& at(int i, int j) { return c[(size_t)i * (deg + 1) + j]; }
  double at(int i, int j) const { return c[(size_t)i * (deg + 1) + j]; }
  double operator()(double u, double v) const {  // plain monomial sum
    double s = 0.0;
    for (int i = 0; i <= deg; ++i) {
      double ui = std::pow(u, i);
      for (int j = 0; i + j <= deg; ++j) s += at(i, j) * ui * std::pow(v, j);
    }
    return s;
  }
  double maxabs() const {
    double m = 0.0;
    for (int i = 0; i <= deg; ++i)
      for (int j = 0; i + j <= deg; ++j) m = std::max(m, std::fabs(at(i, j)));
    return m;
  }
  // slice a_i(v): coefficient of u^i (Sec. 5.1)
  Uni slice(int i) const {
    if (i > deg) return Uni();
    std::vector<double> s(deg - i + 1);
    for (int j = 0; i + j <= deg; ++j) s[j] = at(i, j);
    return Uni(s);
  }
  // a(u, v*) as a polynomial in u
  Uni at_v(double v) const {
    std::vector<double> s(deg + 1, 0.0);
    for (int i = 0; i <= deg; ++i) {
      double acc = 0.0;
      for (int j = deg - i; j >= 0; --j) acc = acc * v + at(i, j);
      s[i] = acc;
    }
    return Uni(s);
  }
  double du(double u, double v) const {
    double s = 0.0;
    for (int i = 1; i <= deg; ++i)
      for (int j = 0; i + j <= deg; ++j) s += i * at(i, j) * std::pow(u, i - 1) * std::pow(v, j);
    return s;
  }
  double dv(double u, double v) const {
    double s = 0.0;
    for (int i = 0; i <= deg; ++i)
      for (int j = 1; i + j <= deg; ++j) s += j * at(i, j) * std::pow(u, i) * std::pow(v, j - 1);
    return s;
  }
};

inline Biv operator+(const Biv& a, const Biv& b) {
  Biv r(std::max(a.deg, b.deg));
  for (int i = 0; i <= a.deg; ++i) for (int j = 0; i + j <= a.deg; ++j) r.at(i, j) += a.at(i, j);
  for (int i = 0; i <= b.deg; ++i) for (int j = 0; i + j <= b.deg; ++j) r.at(i, j) += b.at(i, j);
  return r;
}
inline Biv operator-(const Biv& a, const Biv& b) {
  Biv r(std::max(a.deg, b.deg));
  for (int i = 0; i <= a.deg; ++i) for (int j = 0; i + j <= a.deg; ++j) r.at(i, j) += a.at(i, j);
  for (int i = 0; i <= b.deg; ++i) for (int j = 0; i + j <= b.deg; ++j) r.at(i, j) -= b.at(i, j);
  return r;
}
inline Biv operator*(const Biv& a, const Biv& b) {
  Biv r(a.deg + b.deg);
  for (int i = 0; i <= a.deg; ++i)
    for (int j = 0; i + j <= a.deg; ++j) {
      double x = a.at(i, j);
      if (x == 0.0) continue;
      for (int k = 0; k <= b.deg; ++k)
        for (int l = 0; k + l <= b.deg; ++l) r.at(i + k, j + l) += x * b.at(k, l);
    }
  return r;
}
inline Biv operator*(double s, const Biv& a) {
  Biv r = a;
  for (double& x : r.c) x *= s;
  return r;
}

// 3-vector of bivariate polynomials (SPEC.md:139 PolyVec3)
struct BVec3 {
  Biv x, y, z;
  static BVec3 constant(const double p[3]) { return {Biv::constant(p[0]), Biv::constant(p[1]), Biv::constant(p[2])}; }
  // p0 + u*e1 + v*e2  (Eq. 1 / Eq. 2 barycentric interpolation with u-coordinate u, v-coordinate v)
  static BVec3 affine(const double p0[3], const double e1[3], const double e2[3]) {
    return {Biv::linear(p0[0], e1[0], e2[0]), Biv::linear(p0[1], e1[1], e2[1]), Biv::linear(p0[2], e1[2], e2[2])};
  }
  void eval(double u, double v, double out[3]) const { out[0] = x(u, v); out[1] = y(u, v); out[2] = z(u, v); }
};
inline BVec3 operator+(const BVec3& a, const BVec3& b) { return {a.x + b.x, a.y + b.y, a.z + b.z}; }
inline BVec3 operator-(const BVec3& a, const BVec3& b) { return {a.x - b.x, a.y - b.y, a.z - b.z}; }
inline BVec3 operator*(const Biv& s, const BVec3& a) { return {s * a.x, s * a.y, s * a.z}; }
inline BVec3 operator*(double s, const BVec3& a) { return {s * a.x, s * a.y, s * a.z}; }
inline Biv dot(const BVec3& a, const BVec3& b) { return a.x * b.x + a.y * b.y + a.z * b.z; }
inline BVec3 cross(const BVec3& a, const BVec3& b) {
  return {a.y * b.z - a.z * b.y, a.z * b.x - a.x * b.z, a.x * b.y - a.y * b.x};
}
inline Biv dotc(const BVec3& a, const double b[3]) {  // a . constant vector
  return b[0] * a.x + b[1] * a.y + b[2] * a.z;
}

}  // namespace oracle
