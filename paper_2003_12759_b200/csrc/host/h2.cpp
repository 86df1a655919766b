// H2 norm and expansion-point update for the AIRGA driver (proj/src/h2.cpp,
// proj/src/airga.cpp:319-384). The reference takes the eigenvectors from
// Eigen's EigenSolver; here they come from inverse iteration on each computed
// eigenvalue (complex LU with partial pivoting), start vectors orthogonalised
// within a cluster of equal eigenvalues, so a diagonalisable repeated
// eigenvalue (the block-diagonal error system of two equal models) still
// yields independent vectors. The H2 norm does not depend on the eigenvector
// normalisation.
#include "h2.hpp"

#include <algorithm>
#include <cmath>
#include <complex>
#include <limits>
#include <stdexcept>

namespace mpg::host {
namespace {

using cd = std::complex<double>;
using CMat = std::vector<cd>;  // column-major n x n

// LU with partial pivoting of a complex n x n matrix (in place); false if singular.
bool clu(CMat& a, int n, std::vector<int>& piv, double& maxpiv, double& minpiv) {
  piv.resize(size_t(n));
  maxpiv = 0.0;
  minpiv = std::numeric_limits<double>::infinity();
  for (int k = 0; k < n; ++k) {
    int p = k;
    double best = std::abs(a[size_t(k + k * n)]);
    for (int i = k + 1; i < n; ++i)
      if (std::abs(a[size_t(i + k * n)]) > best) {
        best = std::abs(a[size_t(i + k * n)]);
        p = i;
      }
    piv[size_t(k)] = p;
    maxpiv = std::max(maxpiv, best);
    minpiv = std::min(minpiv, best);
    if (best == 0.0) continue;
    if (p != k)
      for (int j = 0; j < n; ++j) std::swap(a[size_t(k + j * n)], a[size_t(p + j * n)]);
    for (int i = k + 1; i < n; ++i) {
      const cd f = a[size_t(i + k * n)] / a[size_t(k + k * n)];
      a[size_t(i + k * n)] = f;
      for (int j = k + 1; j < n; ++j) a[size_t(i + j * n)] -= f * a[size_t(k + j * n)];
    }
  }
  return minpiv > 0.0;
}

void csolve(const CMat& lu, int n, const std::vector<int>& piv, cd* b) {
  for (int k = 0; k < n; ++k)
    if (piv[size_t(k)] != k) std::swap(b[k], b[piv[size_t(k)]]);
  for (int i = 0; i < n; ++i)
    for (int j = 0; j < i; ++j) b[i] -= lu[size_t(i + j * n)] * b[j];
  for (int i = n - 1; i >= 0; --i) {
    for (int j = i + 1; j < n; ++j) b[i] -= lu[size_t(i + j * n)] * b[j];
    b[i] /= lu[size_t(i + i * n)];
  }
}

// Diagonal similarity scaling by powers of two (Parlett-Reinsch balancing, as
// LAPACK's dgebal): the companion matrices of stiff second-order models mix
// entries of 1 and 1e12, where the unbalanced QR iteration can stall.
Mat balanced(Mat a) {
  const int n = a.rows;
  bool done = false;
  while (!done) {
    done = true;
    for (int i = 0; i < n; ++i) {
      double c = 0.0, r = 0.0;
      for (int j = 0; j < n; ++j)
        if (j != i) {
          c += std::fabs(a(j, i));
          r += std::fabs(a(i, j));
        }
      if (c == 0.0 || r == 0.0) continue;
      double g = r / 2.0, f = 1.0;
      const double sum = c + r;
      while (c < g) {
        f *= 2.0;
        c *= 4.0;
      }
      g = r * 2.0;
      while (c > g) {
        f /= 2.0;
        c /= 4.0;
      }
      if ((c + r) / f < 0.95 * sum) {
        done = false;
        for (int j = 0; j < n; ++j) a(i, j) /= f;
        for (int j = 0; j < n; ++j) a(j, i) *= f;
      }
    }
  }
  return a;
}

}  // namespace

StateSpace second_order_to_state_space(const Mat& m, const Mat& d, const Mat& k, const Mat& f, const Mat& c) {
  const int r = m.rows;
  const LU mlu(m);
  const Mat mk = mlu.solve(k), md = mlu.solve(d), mf = mlu.solve(f);
  StateSpace ss;
  ss.a = Mat(2 * r, 2 * r);
  for (int i = 0; i < r; ++i) ss.a(i, r + i) = 1.0;
  for (int j = 0; j < r; ++j)
    for (int i = 0; i < r; ++i) {
      ss.a(r + i, j) = -mk(i, j);
      ss.a(r + i, r + j) = -md(i, j);
    }
  ss.b = Mat(2 * r, f.cols);
  for (int j = 0; j < f.cols; ++j)
    for (int i = 0; i < r; ++i) ss.b(r + i, j) = mf(i, j);
  ss.c = Mat(c.cols, 2 * r);
  for (int i = 0; i < c.cols; ++i)
    for (int j = 0; j < r; ++j) ss.c(i, j) = c(j, i);
  return ss;
}

double h2_norm(const StateSpace& sys) {
  const int ns = sys.a.rows;
  if (ns == 0) return 0.0;
  if (sys.a.cols != ns || sys.b.rows != ns || sys.c.cols != ns) throw std::invalid_argument("h2_norm: inconsistent dimensions");
  const double inf = std::numeric_limits<double>::infinity();
  std::vector<Eig> ev;
  try {
    ev = eigenvalues(balanced(sys.a));
  } catch (const std::exception&) {
    return inf;
  }
  std::vector<cd> lam(static_cast<size_t>(ns));
  double max_abs = 0.0;
  for (int i = 0; i < ns; ++i) {
    lam[size_t(i)] = cd(ev[size_t(i)].re, ev[size_t(i)].im);
    max_abs = std::max(max_abs, std::abs(lam[size_t(i)]));
  }
  for (int i = 0; i < ns; ++i)
    if (lam[size_t(i)].real() >= -1e-12 * std::max(max_abs, 1.0)) return inf;
  // eigenvectors by inverse iteration
  CMat X(static_cast<size_t>(ns) * static_cast<size_t>(ns));
  const double anorm = std::max(fro(sys.a), 1e-300);
  for (int i = 0; i < ns; ++i) {
    const cd mu = lam[size_t(i)] + cd(1e-10 * anorm, 1e-10 * anorm * 0.5);
    CMat a(static_cast<size_t>(ns) * static_cast<size_t>(ns));
    for (int q = 0; q < ns; ++q)
      for (int p = 0; p < ns; ++p) a[size_t(p + q * ns)] = cd(sys.a(p, q), 0.0) - (p == q ? mu : cd(0.0));
    std::vector<int> piv;
    double mx, mn;
    clu(a, ns, piv, mx, mn);
    for (int p = 0; p < ns; ++p)
      if (std::abs(a[size_t(p + p * ns)]) == 0.0) a[size_t(p + p * ns)] = cd(1e-300, 0.0);
    std::vector<cd> x(static_cast<size_t>(ns));
    for (int p = 0; p < ns; ++p) x[size_t(p)] = cd(p == i % ns ? 1.0 : 0.0, 0.0) + cd(1e-3 * double((p * 7 + 3) % 11), 0.0);
    // earlier vectors of the same eigenvalue cluster
    std::vector<int> cluster;
    for (int j = 0; j < i; ++j)
      if (std::abs(lam[size_t(j)] - lam[size_t(i)]) <= 1e-8 * std::max(1.0, std::abs(lam[size_t(i)]))) cluster.push_back(j);
    for (int it = 0; it < 3; ++it) {
      for (int j : cluster) {  // keep independent of the cluster's earlier vectors
        cd dot(0.0);
        for (int p = 0; p < ns; ++p) dot += std::conj(X[size_t(p + j * ns)]) * x[size_t(p)];
        for (int p = 0; p < ns; ++p) x[size_t(p)] -= dot * X[size_t(p + j * ns)];
      }
      csolve(a, ns, piv, x.data());
      double nrm = 0.0;
      for (const cd& v : x) nrm += std::norm(v);
      nrm = std::sqrt(nrm);
      if (!(nrm > 0.0) || !std::isfinite(nrm)) return inf;
      for (cd& v : x) v /= nrm;
    }
    for (int j : cluster) {
      cd dot(0.0);
      for (int p = 0; p < ns; ++p) dot += std::conj(X[size_t(p + j * ns)]) * x[size_t(p)];
      for (int p = 0; p < ns; ++p) x[size_t(p)] -= dot * X[size_t(p + j * ns)];
    }
    double nrm = 0.0;
    for (const cd& v : x) nrm += std::norm(v);
    nrm = std::sqrt(nrm);
    if (!(nrm > 0.0)) return inf;
    for (int p = 0; p < ns; ++p) X[size_t(p + i * ns)] = x[size_t(p)] / nrm;
  }
  // X^{-1} B
  CMat xl = X;
  std::vector<int> piv;
  double mx, mn;
  if (!clu(xl, ns, piv, mx, mn) || mn <= double(ns) * std::numeric_limits<double>::epsilon() * mx) return inf;
  const int m = sys.b.cols;
  std::vector<cd> xb(static_cast<size_t>(ns) * static_cast<size_t>(m));
  for (int j = 0; j < m; ++j) {
    for (int p = 0; p < ns; ++p) xb[size_t(p + j * ns)] = cd(sys.b(p, j), 0.0);
    csolve(xl, ns, piv, xb.data() + size_t(j) * size_t(ns));
  }
  // S_ij = -G_ij / (l_i + conj(l_j)), G = XB XB^H; trace(CX S CX^H)
  const int q = sys.c.rows;
  std::vector<cd> cx(static_cast<size_t>(q) * static_cast<size_t>(ns), cd(0.0));
  for (int j = 0; j < ns; ++j)
    for (int p = 0; p < ns; ++p)
      for (int o = 0; o < q; ++o) cx[size_t(o + j * q)] += sys.c(o, p) * X[size_t(p + j * ns)];
  double trace = 0.0;
  for (int i = 0; i < ns; ++i)
    for (int j = 0; j < ns; ++j) {
      cd g(0.0);
      for (int t = 0; t < m; ++t) g += xb[size_t(i + t * ns)] * std::conj(xb[size_t(j + t * ns)]);
      const cd s = -g / (lam[size_t(i)] + std::conj(lam[size_t(j)]));
      cd acc(0.0);
      for (int o = 0; o < q; ++o) acc += cx[size_t(o + i * q)] * std::conj(cx[size_t(o + j * q)]);
      trace += (s * acc).real();
    }
  return std::sqrt(std::max(trace, 0.0));
}

double h2_distance(const StateSpace& a, const StateSpace& b) {
  if (a.b.cols != b.b.cols || a.c.rows != b.c.rows) throw std::invalid_argument("h2_distance: input/output count mismatch");
  const int na = a.a.rows, nb = b.a.rows;
  StateSpace e;
  e.a = Mat(na + nb, na + nb);
  for (int j = 0; j < na; ++j)
    for (int i = 0; i < na; ++i) e.a(i, j) = a.a(i, j);
  for (int j = 0; j < nb; ++j)
    for (int i = 0; i < nb; ++i) e.a(na + i, na + j) = b.a(i, j);
  e.b = Mat(na + nb, a.b.cols);
  for (int j = 0; j < a.b.cols; ++j) {
    for (int i = 0; i < na; ++i) e.b(i, j) = a.b(i, j);
    for (int i = 0; i < nb; ++i) e.b(na + i, j) = b.b(i, j);
  }
  e.c = Mat(a.c.rows, na + nb);
  for (int o = 0; o < a.c.rows; ++o) {
    for (int i = 0; i < na; ++i) e.c(o, i) = a.c(o, i);
    for (int i = 0; i < nb; ++i) e.c(o, na + i) = -b.c(o, i);
  }
  return h2_norm(e);
}

std::vector<double> update_expansion_points(const Mat& m, const Mat& d, const Mat& k,
                                            const std::vector<double>& current) {
  const size_t want = current.size();
  if (want == 0) return {};
  const int r = m.rows;
  if (r == 0) return current;
  const Mat zero(r, 1);
  const StateSpace ss = second_order_to_state_space(m, d, k, zero, zero);
  std::vector<Eig> ev;
  try {
    ev = eigenvalues(balanced(ss.a));
  } catch (const std::exception&) {
    return current;
  }
  std::vector<size_t> order(ev.size());
  for (size_t i = 0; i < order.size(); ++i) order[i] = i;
  std::sort(order.begin(), order.end(), [&](size_t a, size_t b) {
    const double ra = std::fabs(ev[a].re), rb = std::fabs(ev[b].re);
    if (ra != rb) return ra < rb;
    return std::fabs(ev[a].im) > std::fabs(ev[b].im);
  });
  std::vector<double> next;
  double max_s = 0.0;
  for (size_t idx : order) {
    if (next.size() >= want) break;
    const double absl = std::hypot(ev[idx].re, ev[idx].im);
    double s = std::fabs(ev[idx].im);
    if (s <= 1e-12 * absl) s = absl;
    if (!(s > 0.0) || !std::isfinite(s)) continue;
    bool close = false;
    const double spacing = 1e-6 * std::max({max_s, s, 1.0});
    for (double have : next)
      if (std::fabs(have - s) <= spacing) {
        close = true;
        break;
      }
    if (close) continue;
    next.push_back(s);
    max_s = std::max(max_s, s);
  }
  for (double s : current) {
    if (next.size() >= want) break;
    bool close = false;
    for (double have : next)
      if (std::fabs(have - s) <= 1e-6 * std::max({max_s, s, 1.0})) {
        close = true;
        break;
      }
    if (!close) next.push_back(s);
  }
  std::sort(next.begin(), next.end());
  return next;
}

}  // namespace mpg::host
