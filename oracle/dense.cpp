// CPU ORACLE — test infrastructure only (see oracle.hpp).
//
// Small dense kernels that the reference takes from Eigen3 (un-vendored,
// version unpinned: `find_package(Eigen3 3.3 REQUIRED NO_MODULE)`,
// proj/CMakeLists.txt:12). Restated from Eigen's published algorithms:
//   ColPivHouseholderQR  — proj/src/spai.cpp:34 (least squares + rank flag)
//   FullPivLU            — proj/src/birka.cpp:119, :283 (inverse, isInvertible)
//   HouseholderQR        — proj/src/birka.cpp:125-128 (thin Q)
//   EigenSolver          — proj/src/birka.cpp:94, :114-123 (real block form)
#include <algorithm>
#include <cmath>
#include <complex>
#include <limits>

#include "oracle.hpp"

namespace oracle {

namespace {
constexpr double kEps = std::numeric_limits<double>::epsilon();

// Eigen makeHouseholderInPlace on x[0..m): returns tau, beta; x[1..m) <- essential.
void make_householder(double* x, index_t m, double& tau, double& beta) {
  double tail = 0.0;
  for (index_t i = 1; i < m; ++i) tail += x[i] * x[i];
  const double c0 = x[0];
  if (tail <= std::numeric_limits<double>::min()) {
    tau = 0.0;
    beta = c0;
    for (index_t i = 1; i < m; ++i) x[i] = 0.0;
    return;
  }
  beta = std::sqrt(c0 * c0 + tail);
  if (c0 >= 0.0) beta = -beta;
  for (index_t i = 1; i < m; ++i) x[i] /= (c0 - beta);
  tau = (beta - c0) / beta;
}

// Apply H = I - tau [1; v][1; v]^T from the left to column segment y[0..m).
void apply_householder(const double* v, index_t m, double tau, double* y) {
  if (tau == 0.0) return;
  double t = y[0];
  for (index_t i = 1; i < m; ++i) t += v[i] * y[i];
  y[0] -= tau * t;
  for (index_t i = 1; i < m; ++i) y[i] -= tau * v[i] * t;
}

double colnorm(const double* x, index_t m) {
  double s = 0.0;
  for (index_t i = 0; i < m; ++i) s += x[i] * x[i];
  return std::sqrt(s);
}
}  // namespace

Dense Dense::transpose() const {
  Dense t(cols, rows);
  for (index_t j = 0; j < cols; ++j)
    for (index_t i = 0; i < rows; ++i) t(j, i) = (*this)(i, j);
  return t;
}

double Dense::norm() const {
  double s = 0.0;
  for (double v : a) s += v * v;
  return std::sqrt(s);
}

Dense matmul(const Dense& x, const Dense& y) {
  if (x.cols != y.rows) throw std::invalid_argument("matmul: dimension mismatch");
  Dense z(x.rows, y.cols);
  for (index_t j = 0; j < y.cols; ++j)
    for (index_t k = 0; k < x.cols; ++k) {
      const double b = y(k, j);
      if (b == 0.0) continue;
      for (index_t i = 0; i < x.rows; ++i) z(i, j) += x(i, k) * b;
    }
  return z;
}

Dense operator-(const Dense& x, const Dense& y) {
  Dense z = x;
  for (size_t i = 0; i < z.a.size(); ++i) z.a[i] -= y.a[i];
  return z;
}

// ---- ColPivHouseholderQR ----------------------------------------------------
ColPivQR::ColPivQR(const Dense& a) : qr(a) {
  const index_t rows = a.rows, cols = a.cols, size = std::min(rows, cols);
  hcoeffs.assign(static_cast<size_t>(size), 0.0);
  std::vector<double> upd(static_cast<size_t>(cols)), direct(static_cast<size_t>(cols));
  std::vector<index_t> transp(static_cast<size_t>(size));
  double maxnorm = 0.0;
  for (index_t k = 0; k < cols; ++k) {
    direct[size_t(k)] = upd[size_t(k)] = colnorm(qr.col(k), rows);
    maxnorm = std::max(maxnorm, upd[size_t(k)]);
  }
  const double threshold_helper = (maxnorm * kEps) * (maxnorm * kEps) / double(rows);
  const double downdate = std::sqrt(kEps);
  nonzero_pivots = size;
  maxpivot = 0.0;
  for (index_t k = 0; k < size; ++k) {
    index_t best = k;
    for (index_t j = k + 1; j < cols; ++j)
      if (upd[size_t(j)] > upd[size_t(best)]) best = j;  // first maximum wins
    const double best_sq = upd[size_t(best)] * upd[size_t(best)];
    if (nonzero_pivots == size && best_sq < threshold_helper * double(rows - k)) nonzero_pivots = k;
    transp[size_t(k)] = best;
    if (best != k) {
      for (index_t i = 0; i < rows; ++i) std::swap(qr(i, k), qr(i, best));
      std::swap(upd[size_t(k)], upd[size_t(best)]);
      std::swap(direct[size_t(k)], direct[size_t(best)]);
    }
    double tau, beta;
    make_householder(qr.col(k) + k, rows - k, tau, beta);
    hcoeffs[size_t(k)] = tau;
    qr(k, k) = beta;
    maxpivot = std::max(maxpivot, std::abs(beta));
    for (index_t j = k + 1; j < cols; ++j) {
      // Eigen applies to the whole remaining block; a single row when rows-k == 1.
      if (rows - k == 1) {
        qr(k, j) *= (1.0 - tau);
      } else {
        apply_householder(qr.col(k) + k, rows - k, tau, qr.col(j) + k);
      }
    }
    for (index_t j = k + 1; j < cols; ++j) {
      if (upd[size_t(j)] == 0.0) continue;
      double t = std::abs(qr(k, j)) / upd[size_t(j)];
      t = (1.0 + t) * (1.0 - t);
      if (t < 0.0) t = 0.0;
      const double ratio = upd[size_t(j)] / direct[size_t(j)];
      const double t2 = t * ratio * ratio;
      if (t2 <= downdate) {
        direct[size_t(j)] = colnorm(qr.col(j) + k + 1, rows - k - 1);
        upd[size_t(j)] = direct[size_t(j)];
      } else {
        upd[size_t(j)] *= std::sqrt(t);
      }
    }
  }
  perm.resize(static_cast<size_t>(cols));
  for (index_t i = 0; i < cols; ++i) perm[size_t(i)] = i;
  for (index_t k = 0; k < size; ++k) std::swap(perm[size_t(k)], perm[size_t(transp[size_t(k)])]);
}

index_t ColPivQR::rank() const {
  const double thr = std::abs(maxpivot) * double(std::min(qr.rows, qr.cols)) * kEps;
  index_t r = 0;
  for (index_t i = 0; i < nonzero_pivots; ++i) r += std::abs(qr(i, i)) > thr;
  return r;
}

Vec ColPivQR::solve(const Vec& b) const {
  const index_t rows = qr.rows, cols = qr.cols;
  Vec x(static_cast<size_t>(cols), 0.0);
  const index_t nz = nonzero_pivots;
  if (nz == 0) return x;
  Vec c = b;
  for (index_t k = 0; k < nz; ++k) {
    if (rows - k == 1) {
      c[size_t(k)] *= (1.0 - hcoeffs[size_t(k)]);
    } else {
      apply_householder(qr.col(k) + k, rows - k, hcoeffs[size_t(k)], c.data() + k);
    }
  }
  for (index_t i = nz - 1; i >= 0; --i) {
    double acc = c[size_t(i)];
    for (index_t j = i + 1; j < nz; ++j) acc -= qr(i, j) * c[size_t(j)];
    c[size_t(i)] = acc / qr(i, i);
  }
  for (index_t i = 0; i < nz; ++i) x[size_t(perm[size_t(i)])] = c[size_t(i)];
  return x;
}

// ---- FullPivLU ---------------------------------------------------------------
FullPivLU::FullPivLU(const Dense& a) : lu(a) {
  const index_t n = a.rows;
  if (a.rows != a.cols) throw std::invalid_argument("FullPivLU: square matrices only");
  p.resize(static_cast<size_t>(n));
  q.resize(static_cast<size_t>(n));
  for (index_t i = 0; i < n; ++i) p[size_t(i)] = q[size_t(i)] = i;
  nonzero = n;
  maxpivot = 0.0;
  for (index_t k = 0; k < n; ++k) {
    index_t br = k, bc = k;
    double big = -1.0;
    for (index_t j = k; j < n; ++j)
      for (index_t i = k; i < n; ++i)
        if (std::abs(lu(i, j)) > big) { big = std::abs(lu(i, j)); br = i; bc = j; }
    if (big == 0.0) { nonzero = k; break; }
    maxpivot = std::max(maxpivot, big);
    if (br != k) { for (index_t j = 0; j < n; ++j) std::swap(lu(k, j), lu(br, j)); std::swap(p[size_t(k)], p[size_t(br)]); }
    if (bc != k) { for (index_t i = 0; i < n; ++i) std::swap(lu(i, k), lu(i, bc)); std::swap(q[size_t(k)], q[size_t(bc)]); }
    for (index_t i = k + 1; i < n; ++i) lu(i, k) /= lu(k, k);
    for (index_t j = k + 1; j < n; ++j)
      for (index_t i = k + 1; i < n; ++i) lu(i, j) -= lu(i, k) * lu(k, j);
  }
}

bool FullPivLU::invertible() const {
  const index_t n = lu.rows;
  const double thr = std::abs(maxpivot) * double(n) * kEps;
  index_t rank = 0;
  for (index_t i = 0; i < nonzero; ++i) rank += std::abs(lu(i, i)) > thr;
  return rank == n;
}

Dense FullPivLU::solve(const Dense& b) const {
  const index_t n = lu.rows;
  Dense x(n, b.cols);
  Vec c(static_cast<size_t>(n));
  for (index_t col = 0; col < b.cols; ++col) {
    for (index_t i = 0; i < n; ++i) c[size_t(i)] = b(p[size_t(i)], col);
    for (index_t i = 0; i < n; ++i)
      for (index_t j = 0; j < i; ++j) c[size_t(i)] -= lu(i, j) * c[size_t(j)];
    for (index_t i = n - 1; i >= 0; --i) {
      for (index_t j = i + 1; j < n; ++j) c[size_t(i)] -= lu(i, j) * c[size_t(j)];
      c[size_t(i)] /= lu(i, i);
    }
    for (index_t i = 0; i < n; ++i) x(q[size_t(i)], col) = c[size_t(i)];
  }
  return x;
}

Dense FullPivLU::inverse() const { return solve(Dense::identity(lu.rows)); }

// ---- thin Householder Q --------------------------------------------------------
Dense thin_q(const Dense& m) {
  Dense qr = m;
  const index_t rows = m.rows, cols = m.cols, size = std::min(rows, cols);
  Vec tau(static_cast<size_t>(size));
  for (index_t k = 0; k < size; ++k) {
    double t, beta;
    make_householder(qr.col(k) + k, rows - k, t, beta);
    tau[size_t(k)] = t;
    qr(k, k) = beta;
    for (index_t j = k + 1; j < cols; ++j) apply_householder(qr.col(k) + k, rows - k, t, qr.col(j) + k);
  }
  Dense q(rows, cols);
  for (index_t j = 0; j < cols; ++j) q(j, j) = 1.0;
  for (index_t k = size - 1; k >= 0; --k)
    for (index_t j = 0; j < cols; ++j) apply_householder(qr.col(k) + k, rows - k, tau[size_t(k)], q.col(j) + k);
  return q;
}

// ---- eigenvalues: Householder Hessenberg reduction + Francis double shift -----
namespace {
void hessenberg(Dense& a) {
  const index_t n = a.rows;
  Vec v(static_cast<size_t>(n));
  for (index_t k = 0; k + 2 < n; ++k) {
    const index_t m = n - k - 1;
    for (index_t i = 0; i < m; ++i) v[size_t(i)] = a(k + 1 + i, k);
    double tau, beta;
    make_householder(v.data(), m, tau, beta);
    if (tau == 0.0) continue;
    // A <- H A H, H acting on rows/cols k+1..n-1.
    for (index_t j = 0; j < n; ++j) {
      double t = a(k + 1, j);
      for (index_t i = 1; i < m; ++i) t += v[size_t(i)] * a(k + 1 + i, j);
      a(k + 1, j) -= tau * t;
      for (index_t i = 1; i < m; ++i) a(k + 1 + i, j) -= tau * v[size_t(i)] * t;
    }
    for (index_t i = 0; i < n; ++i) {
      double t = a(i, k + 1);
      for (index_t j = 1; j < m; ++j) t += v[size_t(j)] * a(i, k + 1 + j);
      a(i, k + 1) -= tau * t;
      for (index_t j = 1; j < m; ++j) a(i, k + 1 + j) -= tau * v[size_t(j)] * t;
    }
    for (index_t i = k + 2; i < n; ++i) a(i, k) = 0.0;
  }
}

inline double sign_of(double a, double b) { return b >= 0.0 ? std::abs(a) : -std::abs(a); }

bool hqr(Dense& a, Vec& wr, Vec& wi) {
  const index_t n = a.rows;
  wr.assign(static_cast<size_t>(n), 0.0);
  wi.assign(static_cast<size_t>(n), 0.0);
  double anorm = 0.0;
  for (index_t i = 0; i < n; ++i)
    for (index_t j = std::max<index_t>(i - 1, 0); j < n; ++j) anorm += std::abs(a(i, j));
  index_t nn = n - 1;
  double t = 0.0;
  double p = 0, q = 0, r = 0, s = 0, w = 0, x = 0, y = 0, z = 0;
  while (nn >= 0) {
    int its = 0;
    index_t l;
    do {
      for (l = nn; l >= 1; --l) {
        s = std::abs(a(l - 1, l - 1)) + std::abs(a(l, l));
        if (s == 0.0) s = anorm;
        if (std::abs(a(l, l - 1)) + s == s) { a(l, l - 1) = 0.0; break; }
      }
      x = a(nn, nn);
      if (l == nn) {
        wr[size_t(nn)] = x + t;
        wi[size_t(nn)] = 0.0;
        --nn;
      } else {
        y = a(nn - 1, nn - 1);
        w = a(nn, nn - 1) * a(nn - 1, nn);
        if (l == nn - 1) {
          p = 0.5 * (y - x);
          q = p * p + w;
          z = std::sqrt(std::abs(q));
          x += t;
          if (q >= 0.0) {
            z = p + sign_of(z, p);
            wr[size_t(nn - 1)] = wr[size_t(nn)] = x + z;
            if (z != 0.0) wr[size_t(nn)] = x - w / z;
            wi[size_t(nn - 1)] = wi[size_t(nn)] = 0.0;
          } else {
            wr[size_t(nn - 1)] = wr[size_t(nn)] = x + p;
            wi[size_t(nn - 1)] = -(wi[size_t(nn)] = z);
          }
          nn -= 2;
        } else {
          if (its == 60) return false;
          if (its == 10 || its == 20 || its == 40) {
            t += x;
            for (index_t i = 0; i <= nn; ++i) a(i, i) -= x;
            s = std::abs(a(nn, nn - 1)) + std::abs(a(nn - 1, nn - 2));
            y = x = 0.75 * s;
            w = -0.4375 * s * s;
          }
          ++its;
          index_t m;
          for (m = nn - 2; m >= l; --m) {
            z = a(m, m);
            r = x - z;
            s = y - z;
            p = (r * s - w) / a(m + 1, m) + a(m, m + 1);
            q = a(m + 1, m + 1) - z - r - s;
            r = a(m + 2, m + 1);
            s = std::abs(p) + std::abs(q) + std::abs(r);
            p /= s; q /= s; r /= s;
            if (m == l) break;
            const double u = std::abs(a(m, m - 1)) * (std::abs(q) + std::abs(r));
            const double v = std::abs(p) * (std::abs(a(m - 1, m - 1)) + std::abs(z) + std::abs(a(m + 1, m + 1)));
            if (u + v == v) break;
          }
          for (index_t i = m + 2; i <= nn; ++i) {
            a(i, i - 2) = 0.0;
            if (i != m + 2) a(i, i - 3) = 0.0;
          }
          for (index_t k = m; k <= nn - 1; ++k) {
            if (k != m) {
              p = a(k, k - 1);
              q = a(k + 1, k - 1);
              r = 0.0;
              if (k != nn - 1) r = a(k + 2, k - 1);
              if ((x = std::abs(p) + std::abs(q) + std::abs(r)) != 0.0) { p /= x; q /= x; r /= x; }
            }
            if ((s = sign_of(std::sqrt(p * p + q * q + r * r), p)) != 0.0) {
              if (k == m) {
                if (l != m) a(k, k - 1) = -a(k, k - 1);
              } else {
                a(k, k - 1) = -s * x;
              }
              p += s;
              x = p / s; y = q / s; z = r / s; q /= p; r /= p;
              for (index_t j = k; j <= nn; ++j) {
                p = a(k, j) + q * a(k + 1, j);
                if (k != nn - 1) { p += r * a(k + 2, j); a(k + 2, j) -= p * z; }
                a(k + 1, j) -= p * y;
                a(k, j) -= p * x;
              }
              const index_t mmin = nn < k + 3 ? nn : k + 3;
              for (index_t i = l; i <= mmin; ++i) {
                p = x * a(i, k) + y * a(i, k + 1);
                if (k != nn - 1) { p += z * a(i, k + 2); a(i, k + 2) -= p * r; }
                a(i, k + 1) -= p * q;
                a(i, k) -= p;
              }
            }
          }
        }
      }
    } while (l < nn - 1);
  }
  return true;
}

using cplx = std::complex<double>;

// Inverse iteration for an eigenvector of m at eigenvalue lam (complex arithmetic).
bool eigvec(const Dense& m, cplx lam, std::vector<cplx>& v) {
  const index_t n = m.rows;
  const double scale = std::max(m.norm(), 1e-300);
  const cplx mu = lam + cplx(scale * 1e-13, 0.0);
  std::vector<cplx> lu(static_cast<size_t>(n * n));
  for (index_t j = 0; j < n; ++j)
    for (index_t i = 0; i < n; ++i) lu[size_t(i + j * n)] = cplx(m(i, j), 0.0) - (i == j ? mu : cplx(0, 0));
  std::vector<index_t> piv(static_cast<size_t>(n));
  for (index_t k = 0; k < n; ++k) {
    index_t pr = k;
    for (index_t i = k + 1; i < n; ++i)
      if (std::abs(lu[size_t(i + k * n)]) > std::abs(lu[size_t(pr + k * n)])) pr = i;
    piv[size_t(k)] = pr;
    if (pr != k)
      for (index_t j = 0; j < n; ++j) std::swap(lu[size_t(k + j * n)], lu[size_t(pr + j * n)]);
    if (std::abs(lu[size_t(k + k * n)]) == 0.0) lu[size_t(k + k * n)] = cplx(scale * 1e-16, 0.0);
    for (index_t i = k + 1; i < n; ++i) {
      lu[size_t(i + k * n)] /= lu[size_t(k + k * n)];
      for (index_t j = k + 1; j < n; ++j) lu[size_t(i + j * n)] -= lu[size_t(i + k * n)] * lu[size_t(k + j * n)];
    }
  }
  v.assign(static_cast<size_t>(n), cplx(0, 0));
  for (index_t i = 0; i < n; ++i) v[size_t(i)] = cplx(1.0 + 0.1 * double(i % 7) + 0.01 * double(i), 0.0);
  for (int it = 0; it < 4; ++it) {
    for (index_t k = 0; k < n; ++k) std::swap(v[size_t(k)], v[size_t(piv[size_t(k)])]);
    for (index_t i = 0; i < n; ++i)
      for (index_t j = 0; j < i; ++j) v[size_t(i)] -= lu[size_t(i + j * n)] * v[size_t(j)];
    for (index_t i = n - 1; i >= 0; --i) {
      for (index_t j = i + 1; j < n; ++j) v[size_t(i)] -= lu[size_t(i + j * n)] * v[size_t(j)];
      v[size_t(i)] /= lu[size_t(i + i * n)];
    }
    double nrm = 0.0;
    for (const cplx& c : v) nrm += std::norm(c);
    nrm = std::sqrt(nrm);
    if (!(nrm > 0.0) || !std::isfinite(nrm)) return false;
    // Normalise the phase on the largest entry so the real form is stable.
    index_t big = 0;
    for (index_t i = 1; i < n; ++i)
      if (std::abs(v[size_t(i)]) > std::abs(v[size_t(big)])) big = i;
    const cplx ph = std::abs(v[size_t(big)]) > 0 ? std::conj(v[size_t(big)]) / std::abs(v[size_t(big)]) : cplx(1, 0);
    for (cplx& c : v) c = c * ph / nrm;
  }
  return true;
}
}  // namespace

std::vector<Complex> eigenvalues(const Dense& m) {
  Dense h = m;
  hessenberg(h);
  Vec wr, wi;
  if (!hqr(h, wr, wi)) throw SolverError("irka: eigenvalue computation on the reduced state matrix failed");
  std::vector<Complex> out(wr.size());
  for (size_t i = 0; i < wr.size(); ++i) out[i] = {wr[i], wi[i]};
  return out;
}

std::vector<Complex> sorted_eigenvalues(const Dense& m) {
  auto lam = eigenvalues(m);
  std::sort(lam.begin(), lam.end(), [](const Complex& a, const Complex& b) {
    if (a.re != b.re) return a.re < b.re;
    return a.im < b.im;
  });
  return lam;
}

bool real_spectrum(const Dense& m, RealSpectrum& out) {
  const index_t n = m.rows;
  std::vector<Complex> lam;
  try { lam = eigenvalues(m); } catch (const SolverError&) { return false; }
  struct Unit { double re, im; };
  std::vector<Unit> units;
  for (const Complex& c : lam) {
    if (c.im == 0.0) units.push_back({c.re, 0.0});
    else if (c.im > 0.0) units.push_back({c.re, c.im});
  }
  std::stable_sort(units.begin(), units.end(), [](const Unit& a, const Unit& b) {
    if (a.re != b.re) return a.re < b.re;
    return -a.im < -b.im;
  });
  out.blocks = Dense(n, n);
  out.basis = Dense(n, n);
  index_t col = 0;
  std::vector<cplx> v;
  for (const Unit& u : units) {
    if (col >= n) return false;
    if (!eigvec(m, cplx(u.re, u.im), v)) return false;
    if (u.im == 0.0) {
      out.blocks(col, col) = u.re;
      for (index_t i = 0; i < n; ++i) out.basis(i, col) = v[size_t(i)].real();
      col += 1;
    } else {
      if (col + 1 >= n) return false;
      out.blocks(col, col) = u.re;
      out.blocks(col, col + 1) = u.im;
      out.blocks(col + 1, col) = -u.im;
      out.blocks(col + 1, col + 1) = u.re;
      for (index_t i = 0; i < n; ++i) {
        out.basis(i, col) = v[size_t(i)].real();
        out.basis(i, col + 1) = v[size_t(i)].imag();
      }
      col += 2;
    }
  }
  if (col != n) return false;
  FullPivLU lu(out.basis);
  if (!lu.invertible()) return false;
  out.basis_inv = lu.inverse();
  return true;
}

}  // namespace oracle
