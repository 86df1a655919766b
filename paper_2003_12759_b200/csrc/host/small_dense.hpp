// Small dense host kernels for the r x r reduced model of the IRKA loop
// (the reference takes these from Eigen: EigenSolver birka.cpp:94/114-123,
// FullPivLU birka.cpp:119/283). r <= 64 here, so these are O(r^3) host loops.
#pragma once

#include <cstdint>
#include <vector>

namespace mpg::host {

// column-major r x c
struct Mat {
  int rows = 0, cols = 0;
  std::vector<double> a;
  Mat() = default;
  Mat(int r, int c, double v = 0.0) : rows(r), cols(c), a(size_t(r) * size_t(c), v) {}
  double& operator()(int i, int j) { return a[size_t(i) + size_t(j) * size_t(rows)]; }
  double operator()(int i, int j) const { return a[size_t(i) + size_t(j) * size_t(rows)]; }
  static Mat eye(int n) { Mat m(n, n); for (int i = 0; i < n; ++i) m(i, i) = 1.0; return m; }
};
Mat mul(const Mat& x, const Mat& y);
Mat transpose(const Mat& x);
double fro(const Mat& x);

struct Eig { double re, im; };
// Eigenvalues (Hessenberg reduction + Francis double-shift QR); throws on failure.
std::vector<Eig> eigenvalues(const Mat& m);
std::vector<Eig> sorted_eigenvalues(const Mat& m);

// Real block form m = R blocks R^{-1}: units sorted by (re, -|im|); pairs as
// [[a, b], [-b, a]] with b > 0 (Eigen's pseudoEigenvalueMatrix convention).
struct Spectrum {
  Mat blocks, basis, basis_inv;
  std::vector<int> unit_start, unit_width;
};
bool real_spectrum(const Mat& m, Spectrum& out);

// Full-pivoting LU with Eigen's invertibility threshold (n * eps * max pivot).
struct LU {
  Mat lu;
  std::vector<int> p, q;
  int nonzero = 0;
  double maxpivot = 0.0;
  explicit LU(const Mat& a);
  bool invertible() const;
  Mat solve(const Mat& b) const;
};

// Cholesky of an SPD matrix (upper R with G = R^T R); false if not positive.
bool cholesky_upper(const Mat& g, Mat& r);
// Inverse of an upper-triangular matrix.
Mat upper_inverse(const Mat& r);
// Householder thin Q of a tall matrix (host fallback when CholQR2 fails).
Mat householder_q(const Mat& m);

}  // namespace mpg::host
