// Seeded synthetic inputs (include/mpg_gen.h): test and bench fixtures, built
// into libmpggen.so and, for the CPU reference arm, into oracle/liboracle.so.
// Not part of the product library libmpg.so.
//
// BASELINE.json's five configs have no generator in the reference (SURVEY.md
// §0.5f); they are defined here once so the oracle and the GPU
// path see identical inputs. The reference's own test fixtures
// (proj/tests/support.hpp:18-49) and its bilinear toy model
// (proj/src/generator.cpp:141-179) are restated with the same libstdc++
// std::mt19937_64 + distribution calls so the draw streams match the
// reference bit for bit when built with this image's g++.
//
// Config streams use only the raw 64-bit engine output (u53 = top 53 bits,
// Box-Muller normals), which is implementation independent.
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <random>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../../include/mpg_gen.h"

namespace {

thread_local std::string g_gen_err;

struct Trip { int64_t r, c; double v; };

mpg_host_csr* alloc_csr(int64_t nr, int64_t nc, int64_t nnz) {
  auto* m = new mpg_host_csr;
  m->nrows = nr;
  m->ncols = nc;
  m->nnz = nnz;
  m->rowptr = new int64_t[size_t(nr) + 1];
  m->colind = new int64_t[size_t(std::max<int64_t>(nnz, 1))];
  m->val = new double[size_t(std::max<int64_t>(nnz, 1))];
  return m;
}

// Sorted row-major, duplicates summed, exact-zero sums kept
// (the ingestion rule of proj/src/sparse.cpp:80-115).
mpg_host_csr* from_trips(int64_t nr, int64_t nc, std::vector<Trip> t) {
  std::sort(t.begin(), t.end(), [](const Trip& a, const Trip& b) { return a.r != b.r ? a.r < b.r : a.c < b.c; });
  std::vector<int64_t> ci;
  std::vector<double> v;
  std::vector<int64_t> rp(size_t(nr) + 1, 0);
  size_t p = 0;
  while (p < t.size()) {
    const int64_t r = t[p].r, c = t[p].c;
    double s = 0.0;
    while (p < t.size() && t[p].r == r && t[p].c == c) s += t[p++].v;
    ci.push_back(c);
    v.push_back(s);
    ++rp[size_t(r) + 1];
  }
  for (int64_t i = 0; i < nr; ++i) rp[size_t(i) + 1] += rp[size_t(i)];
  mpg_host_csr* m = alloc_csr(nr, nc, int64_t(ci.size()));
  std::copy(rp.begin(), rp.end(), m->rowptr);
  std::copy(ci.begin(), ci.end(), m->colind);
  std::copy(v.begin(), v.end(), m->val);
  return m;
}

// Merge of two CSR matrices a*A + b*B, dropping exact zeros
// (proj/src/sparse.cpp:156-202).
mpg_host_csr* combine(double a, const mpg_host_csr* x, double b, const mpg_host_csr* y) {
  std::vector<Trip> t;
  for (int64_t i = 0; i < x->nrows; ++i)
    for (int64_t k = x->rowptr[i]; k < x->rowptr[i + 1]; ++k) t.push_back({i, x->colind[k], a * x->val[k]});
  for (int64_t i = 0; i < y->nrows; ++i)
    for (int64_t k = y->rowptr[i]; k < y->rowptr[i + 1]; ++k) t.push_back({i, y->colind[k], b * y->val[k]});
  std::stable_sort(t.begin(), t.end(), [](const Trip& p, const Trip& q) { return p.r != q.r ? p.r < q.r : p.c < q.c; });
  std::vector<Trip> out;
  size_t p = 0;
  while (p < t.size()) {
    const int64_t r = t[p].r, c = t[p].c;
    double s = 0.0;
    while (p < t.size() && t[p].r == r && t[p].c == c) s += t[p++].v;
    if (s != 0.0) out.push_back({r, c, s});
  }
  return from_trips(x->nrows, x->ncols, std::move(out));
}

// Raw-engine helpers for the config streams.
struct Stream {
  std::mt19937_64 rng;
  explicit Stream(uint64_t seed) : rng(seed) {}
  double u53() { return double(rng() >> 11) * 0x1.0p-53; }
  double uniform(double a, double b) { return a + (b - a) * u53(); }
  double normal() {
    const double u1 = 1.0 - u53(), u2 = u53();
    return std::sqrt(-2.0 * std::log(u1)) * std::cos(6.283185307179586476925 * u2);
  }
  double lognormal(double mu, double s) { return std::exp(mu + s * normal()); }
};

template <class F>
int gen_guard(F&& f) {
  try {
    f();
    return 0;
  } catch (const std::exception& e) {
    g_gen_err = e.what();
    return MPG_ERR_INVALID;
  }
}

// Structured 27-slot row layout for the Q1 hexahedral mesh: slot index
// (dk+1)*9 + (dj+1)*3 + (di+1); compressed to CSR dropping off-grid slots.
mpg_host_csr* compress27(int64_t N, const std::vector<double>& slots) {
  const int64_t n = N * N * N;
  int64_t nnz = 0;
  auto in = [N](int64_t a) { return a >= 0 && a < N; };
  const int64_t per = 3 * N - 2;
  nnz = per * per * per;
  mpg_host_csr* m = alloc_csr(n, n, nnz);
  int64_t p = 0;
  for (int64_t k = 0; k < N; ++k)
    for (int64_t j = 0; j < N; ++j)
      for (int64_t i = 0; i < N; ++i) {
        const int64_t row = i + N * (j + N * k);
        m->rowptr[row] = p;
        for (int dk = -1; dk <= 1; ++dk)
          for (int dj = -1; dj <= 1; ++dj)
            for (int di = -1; di <= 1; ++di) {
              if (!in(i + di) || !in(j + dj) || !in(k + dk)) continue;
              m->colind[p] = row + di + N * (dj + N * dk);
              m->val[p] = slots[size_t(row) * 27 + size_t((dk + 1) * 9 + (dj + 1) * 3 + (di + 1))];
              ++p;
            }
      }
  m->rowptr[n] = p;
  m->nnz = p;
  return m;
}

}  // namespace

extern "C" {

const char* mpg_gen_last_error(void) { return g_gen_err.c_str(); }

void mpg_gen_csr_free(mpg_host_csr* m) {
  if (!m) return;
  delete[] m->rowptr;
  delete[] m->colind;
  delete[] m->val;
  delete m;
}

void mpg_gen_system_free(mpg_host_system* s) {
  if (!s) return;
  mpg_gen_csr_free(s->a);
  mpg_gen_csr_free(s->e);
  delete[] s->e_diag;
  delete[] s->b;
  delete[] s->c;
  delete[] s->shifts;
  delete s;
}

// proj/tests/support.hpp:18-25 (column-major fill order j outer, i inner)
int mpg_gen_random_dense(int64_t r, int64_t c, uint64_t seed, double* out) {
  std::mt19937_64 rng(seed);
  std::uniform_real_distribution<double> u(-1.0, 1.0);
  for (int64_t j = 0; j < c; ++j)
    for (int64_t i = 0; i < r; ++i) out[i + j * r] = u(rng);
  return 0;
}

// proj/tests/support.hpp:37-49
int mpg_gen_random_sparse(int64_t r, int64_t c, double density, uint64_t seed, double diag_shift, mpg_host_csr** out) {
  return gen_guard([&] {
    std::mt19937_64 rng(seed);
    std::uniform_real_distribution<double> u(-1.0, 1.0);
    std::uniform_real_distribution<double> keep(0.0, 1.0);
    std::vector<Trip> t;
    for (int64_t i = 0; i < r; ++i)
      for (int64_t j = 0; j < c; ++j)
        if (keep(rng) < density) t.push_back({i, j, u(rng)});
    if (diag_shift != 0.0)
      for (int64_t i = 0; i < std::min(r, c); ++i) t.push_back({i, i, diag_shift});
    *out = from_trips(r, c, std::move(t));
  });
}

int mpg_gen_from_triplets(int64_t nr, int64_t nc, int64_t nnz, const int64_t* ri, const int64_t* ci, const double* v,
                          mpg_host_csr** out) {
  return gen_guard([&] {
    std::vector<Trip> t(static_cast<size_t>(nnz));
    for (int64_t k = 0; k < nnz; ++k) {
      if (ri[k] < 0 || ri[k] >= nr || ci[k] < 0 || ci[k] >= nc) throw std::invalid_argument("triplet index out of range");
      t[size_t(k)] = {ri[k], ci[k], v[k]};
    }
    *out = from_trips(nr, nc, std::move(t));
  });
}

// proj/src/generator.cpp:141-179 with the couplings' draws consumed but the
// couplings dropped (N = 0, the linear IRKA case of proj/tests/test_birka.cpp:51-75).
// f: n x m column-major, c: n x 1.
static int bilinear_toy_impl(int64_t n, int64_t m, uint64_t seed, mpg_host_csr** k_out, mpg_host_csr** n_out, double* f,
                             double* c) {
  return gen_guard([&] {
    if (n < 2) throw std::invalid_argument("generator: n must be at least 2");
    if (m < 1) throw std::invalid_argument("generator: at least one input is required");
    std::mt19937_64 rng(seed);
    std::uniform_real_distribution<double> sym(-1.0, 1.0);
    std::uniform_int_distribution<int64_t> node(0, n - 1);
    std::vector<Trip> st;
    for (int64_t i = 0; i < n; ++i) {
      st.push_back({i, i, 3.0});
      if (i + 1 < n) { st.push_back({i, i + 1, -1.0}); st.push_back({i + 1, i, -1.0}); }
    }
    mpg_host_csr* stencil = from_trips(n, n, std::move(st));
    std::vector<Trip> skew;
    for (int64_t p = 0; p < n / 2; ++p) {
      const int64_t i = node(rng);
      const int64_t j = node(rng);
      const double w = 0.1 * sym(rng);
      if (i == j) continue;
      skew.push_back({i, j, w});
    }
    mpg_host_csr* pert = from_trips(n, n, std::move(skew));
    *k_out = combine(-1.0, stencil, 1.0, pert);
    mpg_gen_csr_free(stencil);
    mpg_gen_csr_free(pert);
    for (int64_t j = 0; j < m; ++j) {
      std::vector<Trip> t;
      for (int64_t i = 0; i < n; ++i) {
        const int64_t col = node(rng);
        t.push_back({i, col, 0.05 * sym(rng)});
      }
      mpg_host_csr* nj = from_trips(n, n, std::move(t));
      if (n_out) n_out[j] = nj;
      else mpg_gen_csr_free(nj);
    }
    for (int64_t j = 0; j < m; ++j)
      for (int64_t i = 0; i < n; ++i) f[i + j * n] = sym(rng);
    for (int64_t i = 0; i < n; ++i) c[i] = sym(rng);
  });
}

// generate_bilinear_toy (proj/src/generator.cpp:141-179): K, F (n x m), C (n x 1);
// the couplings N_j (one per input) are drawn and returned by the _n variant.
int mpg_gen_bilinear_toy(int64_t n, int64_t m, uint64_t seed, mpg_host_csr** k_out, double* f, double* c) {
  return bilinear_toy_impl(n, m, seed, k_out, nullptr, f, c);
}
int mpg_gen_bilinear_toy_n(int64_t n, int64_t m, uint64_t seed, mpg_host_csr** k_out, mpg_host_csr** n_out, double* f,
                           double* c) {
  return bilinear_toy_impl(n, m, seed, k_out, n_out, f, c);
}

// generate_qb_toy (proj/src/generator.cpp:181-207): D = tridiag(-1, 4, -1),
// K = -tridiag(-1, 2.5, -1), N one entry per row (i, node, 0.05 sym), H two
// entries per row (a, b n + c, 0.1 sym) with draws in the reference's order
// (node, then sym; b, c, then sym); F = C = e_1 (returned by the caller).
int mpg_gen_qb_toy(int64_t n, uint64_t seed, mpg_host_csr** d, mpg_host_csr** k, mpg_host_csr** n_op,
                   mpg_host_csr** h) {
  return gen_guard([&] {
    if (n < 2) throw std::invalid_argument("generator: n must be at least 2");
    std::mt19937_64 rng(seed);
    std::uniform_real_distribution<double> sym(-1.0, 1.0);
    std::uniform_int_distribution<int64_t> node(0, n - 1);
    auto tridiag = [n](double off, double diag, double scale) {
      std::vector<Trip> t;
      for (int64_t i = 0; i < n; ++i) {
        t.push_back({i, i, scale * diag});
        if (i + 1 < n) {
          t.push_back({i, i + 1, scale * off});
          t.push_back({i + 1, i, scale * off});
        }
      }
      return from_trips(n, n, std::move(t));
    };
    *d = tridiag(-1.0, 4.0, 1.0);
    *k = tridiag(-1.0, 2.5, -1.0);
    std::vector<Trip> nt;
    for (int64_t i = 0; i < n; ++i) {
      const int64_t j = node(rng);
      nt.push_back({i, j, 0.05 * sym(rng)});
    }
    *n_op = from_trips(n, n, std::move(nt));
    std::vector<Trip> ht;
    for (int64_t a = 0; a < n; ++a)
      for (int e = 0; e < 2; ++e) {
        const int64_t b = node(rng);
        const int64_t c = node(rng);
        ht.push_back({a, b * n + c, 0.1 * sym(rng)});
      }
    *h = from_trips(n, n * n, std::move(ht));
  });
}

// generate_disc_brake_like (proj/src/generator.cpp:37-139), same draw order:
// per-node scales, then (m, k_g) per node, then the 5-point stiffness with its
// boundary anchors, the skew loop and the random skew pairs; K = K_E + K_R +
// omega^2 K_G (linear_combination, zeros dropped), D = alpha M + beta K (the
// caller forms it), F = C = e_1.
int mpg_gen_disc_brake(int64_t n, double omega, uint64_t seed, mpg_host_csr** m_out, mpg_host_csr** k_out) {
  return gen_guard([&] {
    if (n < 4) throw std::invalid_argument("generator: n must be at least 4");
    if (!std::isfinite(omega)) throw std::invalid_argument("generator: omega, alpha, beta must be finite");
    std::mt19937_64 rng(seed);
    std::uniform_real_distribution<double> u01(0.0, 1.0);
    const double kappa = 1e9;
    const int64_t g = int64_t(std::ceil(std::sqrt(double(n))));
    std::vector<double> scale(static_cast<size_t>(n));
    for (int64_t v = 0; v < n; ++v) scale[size_t(v)] = std::pow(10.0, 6.0 * u01(rng));
    std::vector<Trip> m_t, ke_t, kr_t, kg_t;
    for (int64_t v = 0; v < n; ++v) {
      const double sv = scale[size_t(v)];
      const double mv = sv * (1.0 + 0.2 * u01(rng));
      m_t.push_back({v, v, mv});
      const double gv = 1e3 * sv * (1.0 + 0.2 * u01(rng));
      kg_t.push_back({v, v, gv});
    }
    for (int64_t v = 0; v < n; ++v) {
      const double sv = scale[size_t(v)];
      const int64_t row = v / g, right = v + 1, down = v + g;
      const bool has_right = right < n && right / g == row;
      const bool has_down = down < n;
      if (has_right) {
        const double w = kappa * std::sqrt(sv * scale[size_t(right)]) * (1.0 + 0.5 * u01(rng));
        ke_t.push_back({v, v, w});
        ke_t.push_back({right, right, w});
        ke_t.push_back({v, right, -w});
        ke_t.push_back({right, v, -w});
      }
      if (has_down) {
        const double w = kappa * std::sqrt(sv * scale[size_t(down)]) * (1.0 + 0.5 * u01(rng));
        ke_t.push_back({v, v, w});
        ke_t.push_back({down, down, w});
        ke_t.push_back({v, down, -w});
        ke_t.push_back({down, v, -w});
      }
      int missing = 0;
      if (v % g == 0) ++missing;
      if (!has_right) ++missing;
      if (v < g) ++missing;
      if (!has_down) ++missing;
      for (int b = 0; b < missing; ++b) ke_t.push_back({v, v, kappa * sv * (1.0 + 0.5 * u01(rng))});
    }
    for (int64_t v = 0; v < n; ++v) {
      const int64_t nxt = (v + 1) % n;
      const double w = 16.0 * kappa * std::sqrt(scale[size_t(v)] * scale[size_t(nxt)]) * (1.0 + 0.5 * u01(rng));
      kr_t.push_back({v, nxt, w});
      kr_t.push_back({nxt, v, -w});
    }
    const int64_t pairs = std::max<int64_t>(1, n / 8);
    std::uniform_int_distribution<int64_t> node(0, n - 1);
    for (int64_t p = 0; p < pairs; ++p) {
      const int64_t u = node(rng);
      const int64_t v = node(rng);
      const double draw = 2.0 * u01(rng) - 1.0;
      if (u == v) continue;
      const double w = 0.3 * kappa * std::sqrt(scale[size_t(u)] * scale[size_t(v)]) * draw;
      kr_t.push_back({u, v, w});
      kr_t.push_back({v, u, -w});
    }
    *m_out = from_trips(n, n, std::move(m_t));
    mpg_host_csr* ke = from_trips(n, n, std::move(ke_t));
    mpg_host_csr* kr = from_trips(n, n, std::move(kr_t));
    mpg_host_csr* kg = from_trips(n, n, std::move(kg_t));
    mpg_host_csr* k1 = combine(1.0, ke, 1.0, kr);
    *k_out = combine(1.0, k1, omega * omega, kg);
    mpg_gen_csr_free(ke);
    mpg_gen_csr_free(kr);
    mpg_gen_csr_free(kg);
    mpg_gen_csr_free(k1);
  });
}

// C1: 2D cell-centred 5-point diffusion on an N x N grid.
int mpg_gen_grid2d(int64_t N, uint64_t seed, mpg_host_system** out) {
  return gen_guard([&] {
    if (N < 2) throw std::invalid_argument("grid2d: N must be at least 2");
    Stream s(seed);
    const int64_t n = N * N;
    const double h2 = 1.0 / (double(N) * double(N));
    std::vector<double> kap(static_cast<size_t>(n));
    for (int64_t p = 0; p < n; ++p) kap[size_t(p)] = s.lognormal(0.0, 0.5);
    auto* sys = new mpg_host_system{};
    sys->n = n;
    sys->a = alloc_csr(n, n, 5 * n - 4 * N);
    int64_t q = 0;
    for (int64_t j = 0; j < N; ++j)
      for (int64_t i = 0; i < N; ++i) {
        const int64_t p = i + N * j;
        sys->a->rowptr[p] = q;
        double diag = 0.0;
        auto face = [&](int64_t ii, int64_t jj) -> double {
          if (ii < 0 || jj < 0 || ii >= N || jj >= N) return 2.0 * kap[size_t(p)] / h2;  // Dirichlet face
          const double a = kap[size_t(p)], b = kap[size_t(ii + N * jj)];
          return 2.0 * a * b / (a + b) / h2;  // harmonic-mean conductance
        };
        const int64_t nb[4][2] = {{i, j - 1}, {i - 1, j}, {i + 1, j}, {i, j + 1}};  // ascending column order
        double off[4];
        for (int t = 0; t < 4; ++t) { off[t] = face(nb[t][0], nb[t][1]); diag += off[t]; }
        auto emit = [&](int64_t col, double v) { sys->a->colind[q] = col; sys->a->val[q] = v; ++q; };
        if (j > 0) emit(p - N, off[0]);
        if (i > 0) emit(p - 1, off[1]);
        emit(p, -diag);
        if (i + 1 < N) emit(p + 1, off[2]);
        if (j + 1 < N) emit(p + N, off[3]);
      }
    sys->a->rowptr[n] = q;
    sys->a->nnz = q;
    sys->e_diag = new double[size_t(n)];
    for (int64_t p = 0; p < n; ++p) sys->e_diag[p] = s.uniform(1.0, 2.0);
    sys->m = sys->q = 1;
    sys->b = new double[size_t(n)];
    sys->c = new double[size_t(n)];
    const double sc = 1.0 / std::sqrt(double(n));
    for (int64_t p = 0; p < n; ++p) sys->b[p] = s.normal() * sc;
    for (int64_t p = 0; p < n; ++p) sys->c[p] = s.normal() * sc;
    sys->r = 4;
    sys->shifts = new double[4];
    for (int t = 0; t < 4; ++t) sys->shifts[t] = std::pow(10.0, -2.0 + 3.0 * t / 3.0);
    *out = sys;
  });
}

// C2: 3D 7-point diffusion + first-order upwind convection, M^3 interior nodes.
int mpg_gen_convdiff3d(int64_t M, uint64_t seed, mpg_host_system** out) {
  return gen_guard([&] {
    if (M < 2) throw std::invalid_argument("convdiff3d: M must be at least 2");
    Stream s(seed);
    const int64_t n = M * M * M;
    const double h = 1.0 / double(M + 1), ih2 = 1.0 / (h * h);
    const double vx = 0.5 * ih2, vy = 0.3 * ih2, vz = 0.2 * ih2;  // v = (0.5,0.3,0.2)/h, upwind / h
    auto* sys = new mpg_host_system{};
    sys->n = n;
    sys->a = alloc_csr(n, n, 7 * n - 6 * M * M);
    int64_t q = 0;
    for (int64_t k = 0; k < M; ++k)
      for (int64_t j = 0; j < M; ++j)
        for (int64_t i = 0; i < M; ++i) {
          const int64_t p = i + M * (j + M * k);
          sys->a->rowptr[p] = q;
          auto emit = [&](int64_t col, double v) { sys->a->colind[q] = col; sys->a->val[q] = v; ++q; };
          if (k > 0) emit(p - M * M, ih2 + vz);
          if (j > 0) emit(p - M, ih2 + vy);
          if (i > 0) emit(p - 1, ih2 + vx);
          emit(p, -6.0 * ih2 - vx - vy - vz);
          if (i + 1 < M) emit(p + 1, ih2);
          if (j + 1 < M) emit(p + M, ih2);
          if (k + 1 < M) emit(p + M * M, ih2);
        }
    sys->a->rowptr[n] = q;
    sys->a->nnz = q;
    sys->e_diag = new double[size_t(n)];
    for (int64_t p = 0; p < n; ++p) sys->e_diag[p] = s.uniform(0.5, 1.5);
    sys->m = sys->q = 1;
    sys->b = new double[size_t(n)];
    sys->c = new double[size_t(n)];
    for (int64_t p = 0; p < n; ++p) sys->b[p] = s.normal();
    for (int64_t p = 0; p < n; ++p) sys->c[p] = s.normal();
    sys->r = 8;
    sys->shifts = new double[8];
    for (int t = 0; t < 8; ++t) sys->shifts[t] = std::pow(10.0, -3.0 + 5.0 * t / 7.0);
    *out = sys;
  });
}

// C3/C4: Q1 hexahedral FEM on N^3 nodes ((N-1)^3 elements of side h = 1/(N-1)),
// per-element conductivity lognormal(0,1); A = -(K + Robin term on the x = 1
// face), E = consistent mass (same 27-point pattern). mimo = 0: SISO with B =
// normalised x = 0 face indicator, C = average over the centred 10^3 block
// (clipped to the grid), r = 8, shifts logspace(1e-4, 1e1). mimo = 1: m = q = 4
// with N(0,1) columns drawn after the conductivities, r = 16.
int mpg_gen_fem3d(int64_t N, uint64_t seed, int mimo, mpg_host_system** out) {
  return gen_guard([&] {
    if (N < 3) throw std::invalid_argument("fem3d: N must be at least 3");
    Stream s(seed);
    const int64_t n = N * N * N, ne = N - 1;
    const double h = 1.0 / double(ne);
    const double m1[2][2] = {{1.0 / 3.0, 1.0 / 6.0}, {1.0 / 6.0, 1.0 / 3.0}};
    const double s1[2][2] = {{1.0, -1.0}, {-1.0, 1.0}};
    double ke[8][8], me[8][8], mf[4][4];
    for (int a = 0; a < 8; ++a)
      for (int b = 0; b < 8; ++b) {
        const int ax = a & 1, ay = (a >> 1) & 1, az = a >> 2, bx = b & 1, by = (b >> 1) & 1, bz = b >> 2;
        ke[a][b] = h * (s1[ax][bx] * m1[ay][by] * m1[az][bz] + m1[ax][bx] * s1[ay][by] * m1[az][bz] +
                        m1[ax][bx] * m1[ay][by] * s1[az][bz]);
        me[a][b] = h * h * h * m1[ax][bx] * m1[ay][by] * m1[az][bz];
      }
    for (int a = 0; a < 4; ++a)
      for (int b = 0; b < 4; ++b) mf[a][b] = h * h * m1[a & 1][b & 1] * m1[a >> 1][b >> 1];
    std::vector<double> kslot(size_t(n) * 27, 0.0), mslot(size_t(n) * 27, 0.0);
    auto slot = [&](int64_t i, int64_t j, int64_t k, int di, int dj, int dk) {
      return size_t(i + N * (j + N * k)) * 27 + size_t((dk + 1) * 9 + (dj + 1) * 3 + (di + 1));
    };
    for (int64_t ek = 0; ek < ne; ++ek)
      for (int64_t ej = 0; ej < ne; ++ej)
        for (int64_t ei = 0; ei < ne; ++ei) {
          const double kap = s.lognormal(0.0, 1.0);
          for (int a = 0; a < 8; ++a) {
            const int ax = a & 1, ay = (a >> 1) & 1, az = a >> 2;
            for (int b = 0; b < 8; ++b) {
              const int bx = b & 1, by = (b >> 1) & 1, bz = b >> 2;
              const size_t sl = slot(ei + ax, ej + ay, ek + az, bx - ax, by - ay, bz - az);
              kslot[sl] += kap * ke[a][b];
              mslot[sl] += me[a][b];
            }
          }
        }
    // Robin term (unit transfer coefficient) on the x = 1 face keeps A nonsingular.
    for (int64_t ek = 0; ek < ne; ++ek)
      for (int64_t ej = 0; ej < ne; ++ej)
        for (int a = 0; a < 4; ++a)
          for (int b = 0; b < 4; ++b) {
            const int ay = a & 1, az = a >> 1, by = b & 1, bz = b >> 1;
            kslot[slot(N - 1, ej + ay, ek + az, 0, by - ay, bz - az)] += mf[a][b];
          }
    for (double& v : kslot) v = -v;  // A = -K
    auto* sys = new mpg_host_system{};
    sys->n = n;
    sys->a = compress27(N, kslot);
    kslot.clear();
    kslot.shrink_to_fit();
    sys->e = compress27(N, mslot);
    if (!mimo) {
      sys->m = sys->q = 1;
      sys->b = new double[size_t(n)]();
      sys->c = new double[size_t(n)]();
      const double bv = 1.0 / double(N);  // N^2 face nodes, unit 2-norm
      for (int64_t k = 0; k < N; ++k)
        for (int64_t j = 0; j < N; ++j) sys->b[N * (j + N * k)] = bv;
      const int64_t w = std::min<int64_t>(10, N), lo = (N - w) / 2;
      const double cv = 1.0 / double(w * w * w);
      for (int64_t k = lo; k < lo + w; ++k)
        for (int64_t j = lo; j < lo + w; ++j)
          for (int64_t i = lo; i < lo + w; ++i) sys->c[i + N * (j + N * k)] = cv;
      sys->r = 8;
      sys->shifts = new double[8];
      for (int t = 0; t < 8; ++t) sys->shifts[t] = std::pow(10.0, -4.0 + 5.0 * t / 7.0);
    } else {
      sys->m = sys->q = 4;
      sys->b = new double[size_t(n) * 4];
      sys->c = new double[size_t(n) * 4];
      for (int64_t p = 0; p < n * 4; ++p) sys->b[p] = s.normal();
      for (int64_t p = 0; p < n * 4; ++p) sys->c[p] = s.normal();
      sys->r = 16;
      sys->shifts = new double[16];
      for (int t = 0; t < 16; ++t) sys->shifts[t] = std::pow(10.0, -4.0 + 5.0 * t / 15.0);
    }
    *out = sys;
  });
}

// C5: random sparse rows with Zipf(1.8) lengths on [3, 2000] (diagonal
// included), uniform off-diagonal columns, N(0,1) values, a_ii =
// -1.1 * sum |a_ij|; E = diag U[1,2]; b ~ N(0,1); 64 shifts logspace(1e-3, 1e3).
int mpg_gen_zipf(int64_t n, uint64_t seed, int64_t min_len, int64_t max_len, double expo, int nshifts,
                 mpg_host_system** out) {
  return gen_guard([&] {
    if (n < 2 || min_len < 1 || max_len < min_len) throw std::invalid_argument("zipf: bad parameters");
    const int64_t cap = std::min<int64_t>(max_len, n);
    Stream s(seed);
    std::vector<double> cdf(static_cast<size_t>(cap - min_len + 1));
    double acc = 0.0;
    for (int64_t k = min_len; k <= cap; ++k) { acc += std::pow(double(k), -expo); cdf[size_t(k - min_len)] = acc; }
    for (double& v : cdf) v /= acc;
    std::vector<int64_t> rp(size_t(n) + 1, 0);
    std::vector<int64_t> ci;
    std::vector<double> va;
    ci.reserve(size_t(n) * 30);
    va.reserve(size_t(n) * 30);
    std::vector<std::pair<int64_t, double>> row;
    for (int64_t i = 0; i < n; ++i) {
      const double u = s.u53();
      const int64_t len = min_len + int64_t(std::upper_bound(cdf.begin(), cdf.end(), u) - cdf.begin());
      row.clear();
      for (int64_t t = 0; t + 1 < std::min<int64_t>(len, cap); ++t) {
        int64_t c = int64_t(s.u53() * double(n - 1));
        if (c >= i) ++c;
        row.push_back({c, s.normal()});
      }
      std::sort(row.begin(), row.end(), [](const auto& a, const auto& b) { return a.first < b.first; });
      double absum = 0.0;
      for (const auto& e : row) absum += std::abs(e.second);
      bool diag_done = false;
      size_t p = 0;
      while (p < row.size() || !diag_done) {
        if (!diag_done && (p >= row.size() || row[p].first > i)) {
          ci.push_back(i);
          va.push_back(-1.1 * absum);
          diag_done = true;
          continue;
        }
        const int64_t c = row[p].first;
        double v = 0.0;
        while (p < row.size() && row[p].first == c) v += row[p++].second;
        ci.push_back(c);
        va.push_back(v);
      }
      rp[size_t(i) + 1] = int64_t(ci.size());
    }
    auto* sys = new mpg_host_system{};
    sys->n = n;
    sys->a = alloc_csr(n, n, int64_t(ci.size()));
    std::copy(rp.begin(), rp.end(), sys->a->rowptr);
    std::copy(ci.begin(), ci.end(), sys->a->colind);
    std::copy(va.begin(), va.end(), sys->a->val);
    sys->e_diag = new double[size_t(n)];
    for (int64_t p = 0; p < n; ++p) sys->e_diag[p] = s.uniform(1.0, 2.0);
    sys->m = sys->q = 1;
    sys->b = new double[size_t(n)];
    sys->c = new double[size_t(n)];
    for (int64_t p = 0; p < n; ++p) sys->b[p] = s.normal();
    for (int64_t p = 0; p < n; ++p) sys->c[p] = sys->b[p];
    sys->r = nshifts;
    sys->shifts = new double[size_t(nshifts)];
    for (int t = 0; t < nshifts; ++t)
      sys->shifts[t] = nshifts == 1 ? 1e-3 : std::pow(10.0, -3.0 + 6.0 * t / double(nshifts - 1));
    *out = sys;
  });
}

}  // extern "C"
