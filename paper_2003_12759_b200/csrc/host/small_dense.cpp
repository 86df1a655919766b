#include "small_dense.hpp"

#include <algorithm>
#include <cfloat>
#include <cmath>
#include <complex>
#include <stdexcept>

namespace mpg::host {

Mat mul(const Mat& x, const Mat& y) {
  if (x.cols != y.rows) throw std::invalid_argument("mul: dimension mismatch");
  Mat z(x.rows, y.cols);
  for (int j = 0; j < y.cols; ++j)
    for (int k = 0; k < x.cols; ++k) {
      const double b = y(k, j);
      for (int i = 0; i < x.rows; ++i) z(i, j) += x(i, k) * b;
    }
  return z;
}

Mat transpose(const Mat& x) {
  Mat t(x.cols, x.rows);
  for (int j = 0; j < x.cols; ++j)
    for (int i = 0; i < x.rows; ++i) t(j, i) = x(i, j);
  return t;
}

double fro(const Mat& x) {
  double s = 0.0;
  for (double v : x.a) s += v * v;
  return std::sqrt(s);
}

namespace {

void householder_vec(double* x, int m, double& tau, double& beta) {
  double tail = 0.0;
  for (int i = 1; i < m; ++i) tail += x[i] * x[i];
  const double c0 = x[0];
  if (tail <= DBL_MIN) {
    tau = 0.0;
    beta = c0;
    for (int i = 1; i < m; ++i) x[i] = 0.0;
    return;
  }
  beta = std::sqrt(c0 * c0 + tail);
  if (c0 >= 0.0) beta = -beta;
  for (int i = 1; i < m; ++i) x[i] /= (c0 - beta);
  tau = (beta - c0) / beta;
}

void reduce_hessenberg(Mat& a) {
  const int n = a.rows;
  std::vector<double> v(static_cast<size_t>(n));
  for (int k = 0; k + 2 < n; ++k) {
    const int m = n - k - 1;
    for (int i = 0; i < m; ++i) v[size_t(i)] = a(k + 1 + i, k);
    double tau, beta;
    householder_vec(v.data(), m, tau, beta);
    if (tau == 0.0) continue;
    for (int j = 0; j < n; ++j) {
      double t = a(k + 1, j);
      for (int i = 1; i < m; ++i) t += v[size_t(i)] * a(k + 1 + i, j);
      for (int i = 0; i < m; ++i) a(k + 1 + i, j) -= tau * (i == 0 ? 1.0 : v[size_t(i)]) * t;
    }
    for (int i = 0; i < n; ++i) {
      double t = a(i, k + 1);
      for (int j = 1; j < m; ++j) t += v[size_t(j)] * a(i, k + 1 + j);
      for (int j = 0; j < m; ++j) a(i, k + 1 + j) -= tau * (j == 0 ? 1.0 : v[size_t(j)]) * t;
    }
    for (int i = k + 2; i < n; ++i) a(i, k) = 0.0;
  }
}

double sgn(double a, double b) { return b >= 0.0 ? std::fabs(a) : -std::fabs(a); }

// Francis double-shift QR on an upper Hessenberg matrix (eigenvalues only).
bool francis(Mat& a, std::vector<double>& wr, std::vector<double>& wi) {
  const int n = a.rows;
  wr.assign(size_t(n), 0.0);
  wi.assign(size_t(n), 0.0);
  double norm = 0.0;
  for (int i = 0; i < n; ++i)
    for (int j = std::max(i - 1, 0); j < n; ++j) norm += std::fabs(a(i, j));
  int hi = n - 1;
  double shift_acc = 0.0;
  while (hi >= 0) {
    int iter = 0, lo;
    do {
      for (lo = hi; lo >= 1; --lo) {
        double s = std::fabs(a(lo - 1, lo - 1)) + std::fabs(a(lo, lo));
        if (s == 0.0) s = norm;
        if (std::fabs(a(lo, lo - 1)) + s == s) {
          a(lo, lo - 1) = 0.0;
          break;
        }
      }
      double x = a(hi, hi);
      if (lo == hi) {
        wr[size_t(hi)] = x + shift_acc;
        wi[size_t(hi)] = 0.0;
        --hi;
        continue;
      }
      double y = a(hi - 1, hi - 1);
      double w = a(hi, hi - 1) * a(hi - 1, hi);
      if (lo == hi - 1) {
        const double p = 0.5 * (y - x);
        const double q = p * p + w;
        double z = std::sqrt(std::fabs(q));
        x += shift_acc;
        if (q >= 0.0) {
          z = p + sgn(z, p);
          wr[size_t(hi - 1)] = wr[size_t(hi)] = x + z;
          if (z != 0.0) wr[size_t(hi)] = x - w / z;
          wi[size_t(hi - 1)] = wi[size_t(hi)] = 0.0;
        } else {
          wr[size_t(hi - 1)] = wr[size_t(hi)] = x + p;
          wi[size_t(hi - 1)] = -z;
          wi[size_t(hi)] = z;
        }
        hi -= 2;
        continue;
      }
      if (iter == 60) return false;
      if (iter == 10 || iter == 20 || iter == 40) {  // exceptional shifts
        shift_acc += x;
        for (int i = 0; i <= hi; ++i) a(i, i) -= x;
        const double s = std::fabs(a(hi, hi - 1)) + std::fabs(a(hi - 1, hi - 2));
        x = y = 0.75 * s;
        w = -0.4375 * s * s;
      }
      ++iter;
      int m;
      double p = 0, q = 0, r = 0, z = 0;
      for (m = hi - 2; m >= lo; --m) {
        z = a(m, m);
        r = x - z;
        const double s0 = y - z;
        p = (r * s0 - w) / a(m + 1, m) + a(m, m + 1);
        q = a(m + 1, m + 1) - z - r - s0;
        r = a(m + 2, m + 1);
        const double s = std::fabs(p) + std::fabs(q) + std::fabs(r);
        p /= s;
        q /= s;
        r /= s;
        if (m == lo) break;
        const double u = std::fabs(a(m, m - 1)) * (std::fabs(q) + std::fabs(r));
        const double v = std::fabs(p) * (std::fabs(a(m - 1, m - 1)) + std::fabs(z) + std::fabs(a(m + 1, m + 1)));
        if (u + v == v) break;
      }
      for (int i = m + 2; i <= hi; ++i) {
        a(i, i - 2) = 0.0;
        if (i != m + 2) a(i, i - 3) = 0.0;
      }
      for (int k = m; k <= hi - 1; ++k) {
        if (k != m) {
          p = a(k, k - 1);
          q = a(k + 1, k - 1);
          r = k != hi - 1 ? a(k + 2, k - 1) : 0.0;
          x = std::fabs(p) + std::fabs(q) + std::fabs(r);
          if (x != 0.0) {
            p /= x;
            q /= x;
            r /= x;
          }
        }
        const double s = sgn(std::sqrt(p * p + q * q + r * r), p);
        if (s == 0.0) continue;
        if (k == m) {
          if (lo != m) a(k, k - 1) = -a(k, k - 1);
        } else {
          a(k, k - 1) = -s * x;
        }
        p += s;
        x = p / s;
        y = q / s;
        z = r / s;
        q /= p;
        r /= p;
        for (int j = k; j <= hi; ++j) {
          double t = a(k, j) + q * a(k + 1, j);
          if (k != hi - 1) {
            t += r * a(k + 2, j);
            a(k + 2, j) -= t * z;
          }
          a(k + 1, j) -= t * y;
          a(k, j) -= t * x;
        }
        const int mmin = hi < k + 3 ? hi : k + 3;
        for (int i = lo; i <= mmin; ++i) {
          double t = x * a(i, k) + y * a(i, k + 1);
          if (k != hi - 1) {
            t += z * a(i, k + 2);
            a(i, k + 2) -= t * r;
          }
          a(i, k + 1) -= t * q;
          a(i, k) -= t;
        }
      }
    } while (hi >= 0 && lo < hi - 1);
  }
  return true;
}

using cd = std::complex<double>;

bool inverse_iteration(const Mat& m, cd lam, std::vector<cd>& v) {
  const int n = m.rows;
  const double scale = std::max(fro(m), 1e-300);
  const cd mu = lam + cd(scale * 1e-13, 0.0);
  std::vector<cd> lu(size_t(n) * size_t(n));
  for (int j = 0; j < n; ++j)
    for (int i = 0; i < n; ++i) lu[size_t(i + j * n)] = cd(m(i, j), 0.0) - (i == j ? mu : cd(0.0, 0.0));
  std::vector<int> piv(static_cast<size_t>(n));
  for (int k = 0; k < n; ++k) {
    int pr = k;
    for (int i = k + 1; i < n; ++i)
      if (std::abs(lu[size_t(i + k * n)]) > std::abs(lu[size_t(pr + k * n)])) pr = i;
    piv[size_t(k)] = pr;
    if (pr != k)
      for (int j = 0; j < n; ++j) std::swap(lu[size_t(k + j * n)], lu[size_t(pr + j * n)]);
    if (std::abs(lu[size_t(k + k * n)]) == 0.0) lu[size_t(k + k * n)] = cd(scale * 1e-16, 0.0);
    for (int i = k + 1; i < n; ++i) {
      lu[size_t(i + k * n)] /= lu[size_t(k + k * n)];
      for (int j = k + 1; j < n; ++j) lu[size_t(i + j * n)] -= lu[size_t(i + k * n)] * lu[size_t(k + j * n)];
    }
  }
  v.assign(size_t(n), cd(0.0, 0.0));
  for (int i = 0; i < n; ++i) v[size_t(i)] = cd(1.0 + 0.1 * double(i % 7) + 0.01 * double(i), 0.0);
  for (int it = 0; it < 4; ++it) {
    for (int k = 0; k < n; ++k) std::swap(v[size_t(k)], v[size_t(piv[size_t(k)])]);
    for (int i = 0; i < n; ++i)
      for (int j = 0; j < i; ++j) v[size_t(i)] -= lu[size_t(i + j * n)] * v[size_t(j)];
    for (int i = n - 1; i >= 0; --i) {
      for (int j = i + 1; j < n; ++j) v[size_t(i)] -= lu[size_t(i + j * n)] * v[size_t(j)];
      v[size_t(i)] /= lu[size_t(i + i * n)];
    }
    double nrm = 0.0;
    for (const cd& c : v) nrm += std::norm(c);
    nrm = std::sqrt(nrm);
    if (!(nrm > 0.0) || !std::isfinite(nrm)) return false;
    int big = 0;
    for (int i = 1; i < n; ++i)
      if (std::abs(v[size_t(i)]) > std::abs(v[size_t(big)])) big = i;
    const cd ph = std::conj(v[size_t(big)]) / std::abs(v[size_t(big)]);
    for (cd& c : v) c = c * ph / nrm;
  }
  return true;
}

}  // namespace

std::vector<Eig> eigenvalues(const Mat& m) {
  Mat h = m;
  reduce_hessenberg(h);
  std::vector<double> wr, wi;
  if (!francis(h, wr, wi)) throw std::runtime_error("eigenvalue computation on the reduced state matrix failed");
  std::vector<Eig> out(wr.size());
  for (size_t i = 0; i < wr.size(); ++i) out[i] = {wr[i], wi[i]};
  return out;
}

std::vector<Eig> sorted_eigenvalues(const Mat& m) {
  auto l = eigenvalues(m);
  std::sort(l.begin(), l.end(), [](const Eig& a, const Eig& b) { return a.re != b.re ? a.re < b.re : a.im < b.im; });
  return l;
}

bool real_spectrum(const Mat& m, Spectrum& out) {
  const int n = m.rows;
  std::vector<Eig> lam;
  try {
    lam = eigenvalues(m);
  } catch (const std::exception&) {
    return false;
  }
  std::vector<Eig> units;
  for (const Eig& e : lam)
    if (e.im >= 0.0) units.push_back(e);
  std::stable_sort(units.begin(), units.end(),
                   [](const Eig& a, const Eig& b) { return a.re != b.re ? a.re < b.re : -a.im < -b.im; });
  out.blocks = Mat(n, n);
  out.basis = Mat(n, n);
  out.unit_start.clear();
  out.unit_width.clear();
  int col = 0;
  std::vector<cd> v;
  for (const Eig& u : units) {
    const int w = u.im == 0.0 ? 1 : 2;
    if (col + w > n) return false;
    if (!inverse_iteration(m, cd(u.re, u.im), v)) return false;
    out.unit_start.push_back(col);
    out.unit_width.push_back(w);
    if (w == 1) {
      out.blocks(col, col) = u.re;
      for (int i = 0; i < n; ++i) out.basis(i, col) = v[size_t(i)].real();
    } else {
      out.blocks(col, col) = u.re;
      out.blocks(col, col + 1) = u.im;
      out.blocks(col + 1, col) = -u.im;
      out.blocks(col + 1, col + 1) = u.re;
      for (int i = 0; i < n; ++i) {
        out.basis(i, col) = v[size_t(i)].real();
        out.basis(i, col + 1) = v[size_t(i)].imag();
      }
    }
    col += w;
  }
  if (col != n) return false;
  LU lu(out.basis);
  if (!lu.invertible()) return false;
  out.basis_inv = lu.solve(Mat::eye(n));
  return true;
}

LU::LU(const Mat& a) : lu(a) {
  const int n = a.rows;
  if (a.rows != a.cols) throw std::invalid_argument("LU: square only");
  p.resize(size_t(n));
  q.resize(size_t(n));
  for (int i = 0; i < n; ++i) p[size_t(i)] = q[size_t(i)] = i;
  nonzero = n;
  for (int k = 0; k < n; ++k) {
    int br = k, bc = k;
    double big = -1.0;
    for (int j = k; j < n; ++j)
      for (int i = k; i < n; ++i)
        if (std::fabs(lu(i, j)) > big) {
          big = std::fabs(lu(i, j));
          br = i;
          bc = j;
        }
    if (big == 0.0) {
      nonzero = k;
      break;
    }
    maxpivot = std::max(maxpivot, big);
    if (br != k) {
      for (int j = 0; j < n; ++j) std::swap(lu(k, j), lu(br, j));
      std::swap(p[size_t(k)], p[size_t(br)]);
    }
    if (bc != k) {
      for (int i = 0; i < n; ++i) std::swap(lu(i, k), lu(i, bc));
      std::swap(q[size_t(k)], q[size_t(bc)]);
    }
    for (int i = k + 1; i < n; ++i) lu(i, k) /= lu(k, k);
    for (int j = k + 1; j < n; ++j)
      for (int i = k + 1; i < n; ++i) lu(i, j) -= lu(i, k) * lu(k, j);
  }
}

bool LU::invertible() const {
  const int n = lu.rows;
  const double thr = std::fabs(maxpivot) * double(n) * DBL_EPSILON;
  int rank = 0;
  for (int i = 0; i < nonzero; ++i) rank += std::fabs(lu(i, i)) > thr;
  return rank == n;
}

Mat LU::solve(const Mat& b) const {
  const int n = lu.rows;
  Mat x(n, b.cols);
  std::vector<double> c(static_cast<size_t>(n));
  for (int col = 0; col < b.cols; ++col) {
    for (int i = 0; i < n; ++i) c[size_t(i)] = b(p[size_t(i)], col);
    for (int i = 0; i < n; ++i)
      for (int j = 0; j < i; ++j) c[size_t(i)] -= lu(i, j) * c[size_t(j)];
    for (int i = n - 1; i >= 0; --i) {
      for (int j = i + 1; j < n; ++j) c[size_t(i)] -= lu(i, j) * c[size_t(j)];
      c[size_t(i)] /= lu(i, i);
    }
    for (int i = 0; i < n; ++i) x(q[size_t(i)], col) = c[size_t(i)];
  }
  return x;
}

bool cholesky_upper(const Mat& g, Mat& r) {
  const int n = g.rows;
  r = Mat(n, n);
  for (int j = 0; j < n; ++j) {
    double s = g(j, j);
    for (int k = 0; k < j; ++k) s -= r(k, j) * r(k, j);
    if (!(s > 0.0) || !std::isfinite(s)) return false;
    const double d = std::sqrt(s);
    r(j, j) = d;
    for (int i = j + 1; i < n; ++i) {
      double t = g(j, i);
      for (int k = 0; k < j; ++k) t -= r(k, j) * r(k, i);
      r(j, i) = t / d;
    }
  }
  return true;
}

Mat upper_inverse(const Mat& r) {
  const int n = r.rows;
  Mat x(n, n);
  for (int j = 0; j < n; ++j) {
    x(j, j) = 1.0 / r(j, j);
    for (int i = j - 1; i >= 0; --i) {
      double s = 0.0;
      for (int k = i + 1; k <= j; ++k) s += r(i, k) * x(k, j);
      x(i, j) = -s / r(i, i);
    }
  }
  return x;
}

Mat householder_q(const Mat& m) {
  Mat qr = m;
  const int rows = m.rows, cols = m.cols, size = std::min(rows, cols);
  std::vector<double> tau(static_cast<size_t>(size));
  for (int k = 0; k < size; ++k) {
    double t, beta;
    householder_vec(&qr(k, k), rows - k, t, beta);
    tau[size_t(k)] = t;
    qr(k, k) = beta;
    for (int j = k + 1; j < cols; ++j) {
      double s = qr(k, j);
      for (int i = k + 1; i < rows; ++i) s += qr(i, k) * qr(i, j);
      qr(k, j) -= t * s;
      for (int i = k + 1; i < rows; ++i) qr(i, j) -= t * qr(i, k) * s;
    }
  }
  Mat q(rows, cols);
  for (int j = 0; j < cols; ++j) q(j, j) = 1.0;
  for (int k = size - 1; k >= 0; --k)
    for (int j = 0; j < cols; ++j) {
      double s = q(k, j);
      for (int i = k + 1; i < rows; ++i) s += qr(i, k) * q(i, j);
      q(k, j) -= tau[size_t(k)] * s;
      for (int i = k + 1; i < rows; ++i) q(i, j) -= tau[size_t(k)] * qr(i, k) * s;
    }
  return q;
}

}  // namespace mpg::host
