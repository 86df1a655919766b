// morprec_gpu.hpp — header-only C++ mirror of the reference's solve-path API
// (/root/reference/proj/include/morprec) over the C ABI in mpg.h.
//
// Same names and argument meaning as the reference; Eigen containers are
// replaced by std::vector<double> (column-major for matrices). Errors are the
// reference's own exception classes (proj/include/morprec/errors.hpp:12-28):
// MPG_ERR_INVALID -> std::invalid_argument, MPG_ERR_CONFIG ->
// morprec::ConfigError, MPG_ERR_SOLVER -> morprec::SolverError, MPG_ERR_IO ->
// morprec::IoError, so a reference caller's handlers (tools/main.cpp:476-491,
// exit codes 2/3/4) see the same types. GMRES non-convergence stays a report
// flag (gmres.hpp:41-48). Device failures (MPG_ERR_CUDA) are DeviceError, a
// std::runtime_error (exit code 1 there, like any other std::exception).
#pragma once

#include <cmath>
#include <cstdint>
#include <memory>
#include <new>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "mpg.h"

#if __has_include(<morprec/errors.hpp>)
// Built inside the reference tree (its include/ on the path): its classes.
#include <morprec/errors.hpp>
#else
// Standalone: the same three declarations as the reference's Eigen-free
// errors.hpp, so code written against morprec:: compiles unchanged.
namespace morprec {
class ConfigError : public std::runtime_error {
 public:
  using std::runtime_error::runtime_error;
};
class SolverError : public std::runtime_error {
 public:
  using std::runtime_error::runtime_error;
};
class IoError : public std::runtime_error {
 public:
  using std::runtime_error::runtime_error;
};
}  // namespace morprec
#endif

namespace morprec_gpu {

using morprec::ConfigError;
using morprec::IoError;
using morprec::SolverError;
class DeviceError : public std::runtime_error {
 public:
  using std::runtime_error::runtime_error;
};

inline void check(int status) {
  if (status == MPG_OK) return;
  const std::string msg = mpg_last_error();
  switch (status) {
    case MPG_ERR_INVALID: throw std::invalid_argument(msg);
    case MPG_ERR_CONFIG: throw ConfigError(msg);
    case MPG_ERR_SOLVER: throw SolverError(msg);
    case MPG_ERR_IO: throw IoError(msg);
    case MPG_ERR_NOMEM: throw std::bad_alloc();
    case MPG_ERR_CUDA: throw DeviceError(msg);
    default: throw std::logic_error(msg);
  }
}

using index_t = std::int64_t;

// SparseMatrix (sparse.hpp:33-101): immutable, copies share the device storage.
class SparseMatrix {
 public:
  SparseMatrix() = default;
  static SparseMatrix from_csr(index_t nrows, index_t ncols, const std::vector<index_t>& row_offsets,
                               const std::vector<index_t>& col_indices, const std::vector<double>& values,
                               int device = 0) {
    if (row_offsets.size() != static_cast<size_t>(nrows) + 1)
      throw std::invalid_argument("sparse: row_offsets length must be nrows + 1");
    if (col_indices.size() != values.size())
      throw std::invalid_argument("sparse: col_indices and values lengths differ");
    mpg_csr* h = nullptr;
    check(mpg_csr_create(device, nrows, ncols, row_offsets.data(), col_indices.data(), values.data(), &h));
    return SparseMatrix(h);
  }
  index_t rows() const { return info()[0]; }
  index_t cols() const { return info()[1]; }
  index_t nnz() const { return info()[2]; }
  std::vector<double> multiply(const std::vector<double>& x) const {
    if (static_cast<index_t>(x.size()) != cols()) throw std::invalid_argument("sparse multiply: dimension mismatch");
    std::vector<double> y(static_cast<size_t>(rows()));
    check(mpg_csr_multiply(h_.get(), x.data(), y.data()));
    return y;
  }
  std::vector<double> multiply_transpose(const std::vector<double>& x) const {
    if (static_cast<index_t>(x.size()) != rows())
      throw std::invalid_argument("sparse multiply_transpose: dimension mismatch");
    std::vector<double> y(static_cast<size_t>(cols()));
    check(mpg_csr_multiply_transpose(h_.get(), x.data(), y.data()));
    return y;
  }
  SparseMatrix transpose() const {
    mpg_csr* t = nullptr;
    check(mpg_csr_transpose(h_.get(), &t));
    return SparseMatrix(t);
  }
  double frobenius_norm() const { return mpg_csr_frobenius_norm(h_.get()); }
  const mpg_csr* handle() const { return h_.get(); }
  explicit SparseMatrix(mpg_csr* h) : h_(h, mpg_csr_destroy) {}

 private:
  std::vector<int64_t> info() const {
    std::vector<int64_t> v(3);
    check(mpg_csr_info(h_.get(), &v[0], &v[1], &v[2]));
    return v;
  }
  std::shared_ptr<mpg_csr> h_;
};

// sigma E - A formed on the fly (replaces linear_combination + matvec_operator
// for shifted pencils, qbihomm.cpp:164-171, and the N = 0 KroneckerOperator).
class ShiftedOperator {
 public:
  explicit ShiftedOperator(const SparseMatrix& a, const SparseMatrix* e = nullptr) {
    mpg_op* h = nullptr;
    check(mpg_op_create(a.handle(), e ? e->handle() : nullptr, &h));
    h_.reset(h, mpg_op_destroy);
  }
  index_t dim() const { return mpg_op_dim(h_.get()); }
  std::vector<double> apply(double sigma_re, double sigma_im, bool transpose, const std::vector<double>& x) const {
    std::vector<double> y(x.size());
    check(mpg_op_apply(h_.get(), sigma_re, sigma_im, transpose, x.data(), y.data()));
    return y;
  }
  SparseMatrix explicit_matrix(double sigma_re, double sigma_im = 0.0, bool transpose = false) const {
    mpg_csr* m = nullptr;
    check(mpg_op_explicit(h_.get(), sigma_re, sigma_im, transpose, &m));
    return SparseMatrix(m);
  }
  const mpg_op* handle() const { return h_.get(); }

 private:
  std::shared_ptr<mpg_op> h_;
};

struct GmresConfig {  // gmres.hpp:20-24
  double rel_tol = 1e-6;
  int max_iter = 1000;
  bool record_history = false;
  mpg_gmres_cfg c() const { return {rel_tol, max_iter, record_history ? 1 : 0}; }
};

struct GmresReport {  // gmres.hpp:26-34
  int iterations = 0;
  bool converged = false;
  bool breakdown = false;
  double rhs_norm = 0.0;
  double final_residual = 0.0;
  double solve_seconds = 0.0;
  std::vector<double> residual_history;
};

struct GmresResult {
  std::vector<double> x;
  GmresReport report;
};

struct SpaiConfig {  // spai.hpp:25-33 (pattern_kind 0 diagonal, 1 pattern of A)
  int pattern_kind = 1;
  double fill_tol = 1e-4;
  int max_fill_per_col = 50;
  int max_pattern_sweeps = 3;
  mpg_spai_cfg c() const { return {pattern_kind, 2, fill_tol, max_fill_per_col, max_pattern_sweeps, 1}; }
};

struct SpaiResult {  // spai.hpp:43-48
  SparseMatrix p;
  std::vector<double> column_residuals;
  index_t fallback_count = 0;
  double build_seconds = 0.0;
};

struct UpdateFactor {  // chain.hpp:33-42
  SparseMatrix q;
  double min_residual = 0.0, matrix_change = 0.0, build_seconds = 0.0;
  index_t fallback_count = 0;
};

inline SpaiResult spai_build(const SparseMatrix& a, const SpaiConfig& cfg = {}) {
  SpaiResult r;
  r.column_residuals.resize(static_cast<size_t>(a.rows()));
  mpg_csr* p = nullptr;
  int64_t fb = 0;
  const mpg_spai_cfg c = cfg.c();
  check(mpg_spai_build(a.handle(), &c, &p, r.column_residuals.data(), &fb, &r.build_seconds));
  r.p = SparseMatrix(p);
  r.fallback_count = fb;
  return r;
}

inline UpdateFactor update_build(const SparseMatrix& a_prev, const SparseMatrix& a_new, const SpaiConfig& cfg = {}) {
  UpdateFactor f;
  mpg_csr* q = nullptr;
  int64_t fb = 0;
  const mpg_spai_cfg c = cfg.c();
  check(mpg_update_build(a_prev.handle(), a_new.handle(), &c, &q, &f.min_residual, &f.matrix_change, &fb,
                         &f.build_seconds));
  f.q = SparseMatrix(q);
  f.fallback_count = fb;
  return f;
}

// PrecondChain (chain.hpp:55-77): immutable, extended() shares the prefix.
class PrecondChain {
 public:
  PrecondChain() = default;
  explicit PrecondChain(const SparseMatrix& base) {
    mpg_chain* h = nullptr;
    check(mpg_chain_create(base.handle(), &h));
    h_.reset(h, mpg_chain_destroy);
  }
  bool empty() const { return !h_; }
  int length() const { return h_ ? mpg_chain_length(h_.get()) : 0; }
  PrecondChain extended(const UpdateFactor& f) const {
    if (!h_) throw std::logic_error("chain: cannot extend an empty chain");
    mpg_chain* h = nullptr;
    check(mpg_chain_extend(h_.get(), f.q.handle(), &h));
    PrecondChain c;
    c.h_.reset(h, mpg_chain_destroy);
    return c;
  }
  std::vector<double> apply(const std::vector<double>& in) const {
    if (!h_) throw std::logic_error("chain: apply on an empty chain");
    std::vector<double> out(in.size());
    check(mpg_chain_apply(h_.get(), in.data(), out.data()));
    return out;
  }
  const mpg_chain* handle() const { return h_.get(); }

 private:
  std::shared_ptr<mpg_chain> h_;
};

inline double standard_residual(const SparseMatrix& a, const PrecondChain& p) {
  double r = 0.0;
  check(mpg_standard_residual(a.handle(), p.handle(), &r));
  return r;
}

namespace detail {
inline GmresResult finish(const mpg_gmres_report& rep, std::vector<double> x, std::vector<double> hist) {
  GmresResult r;
  r.x = std::move(x);
  r.report.iterations = rep.iterations;
  r.report.converged = rep.converged != 0;
  r.report.breakdown = rep.breakdown != 0;
  r.report.rhs_norm = rep.rhs_norm;
  r.report.final_residual = rep.final_residual;
  r.report.solve_seconds = rep.solve_seconds;
  hist.resize(static_cast<size_t>(rep.history_len));
  r.report.residual_history = std::move(hist);
  return r;
}
}  // namespace detail

// gmres_right_preconditioned (gmres.hpp:49-50) with matvec_operator(a) and
// chain.as_operator() (or identity_operator() for an empty chain).
inline GmresResult gmres_right_preconditioned(const SparseMatrix& a, const PrecondChain& p,
                                              const std::vector<double>& b, const GmresConfig& cfg = {}) {
  std::vector<double> x(b.size());
  std::vector<double> hist(cfg.record_history ? static_cast<size_t>(cfg.max_iter) + 2 : 0);
  mpg_gmres_report rep{};
  const mpg_gmres_cfg c = cfg.c();
  check(mpg_gmres_csr(a.handle(), p.handle(), b.data(), x.data(), &c, &rep, hist.empty() ? nullptr : hist.data()));
  return detail::finish(rep, std::move(x), std::move(hist));
}

// The same solve on (sigma E - A) or its test-side form without materialising it.
inline GmresResult gmres_shifted(const ShiftedOperator& op, double sigma_re, double sigma_im, bool transpose,
                                 const PrecondChain& p, const std::vector<double>& b, const GmresConfig& cfg = {}) {
  std::vector<double> x(b.size());
  std::vector<double> hist(cfg.record_history ? static_cast<size_t>(cfg.max_iter) + 2 : 0);
  mpg_gmres_report rep{};
  const mpg_gmres_cfg c = cfg.c();
  check(mpg_gmres_shifted(op.handle(), sigma_re, sigma_im, transpose, p.handle(), b.data(), x.data(), &c, &rep,
                          hist.empty() ? nullptr : hist.data()));
  return detail::finish(rep, std::move(x), std::move(hist));
}

enum class PrecondMode { None = MPG_PRECOND_NONE, FreshSpai = MPG_PRECOND_FRESH, ReuseChain = MPG_PRECOND_REUSE_CHAIN,
                         ReuseFrozen = MPG_PRECOND_REUSE_FROZEN };

struct BirkaConfig {  // birka.hpp:49-61 (N = 0)
  int r = 2;
  double tol = 1e-4;
  int max_sweeps = 50;
  std::uint64_t seed = 1;
  GmresConfig gmres{1e-10, 1000, false};
  SpaiConfig spai{};
  int max_chain_len = 16;
  index_t standard_residual_max_dim = 5000;
  bool mirror_unstable = false;  // extension
  index_t explicit_nnz_cap = 200000;  // coupled systems only (joint solves)
};

struct BirkaState {  // birka.hpp:35-47 with the descriptor E_r, A_r
  int order = 0;
  std::vector<double> kr, fr, cr, er, ar;  // column-major
  std::vector<std::vector<double>> nr;      // coupled systems: N_r[j], r x r each
  std::vector<double> lambda_re, lambda_im;
  int sweeps = 0;
};

struct ReductionReport {  // report.hpp:49-61
  std::vector<mpg_report_row> rows;
  bool converged = false;
  int sweeps = 0;
  std::string warnings;  // '\n'-separated
};

// birka_reduce (birka.hpp:78-80) for x' = A x + B u with E x' (E may be null).
inline std::pair<BirkaState, ReductionReport> birka_reduce(const ShiftedOperator& op, const std::vector<double>& b,
                                                           int m, const std::vector<double>& c, int q,
                                                           const BirkaConfig& cfg, PrecondMode mode,
                                                           const std::vector<double>* init_shifts = nullptr) {
  mpg_irka_cfg k{};
  k.r = cfg.r;
  k.tol = cfg.tol;
  k.max_sweeps = cfg.max_sweeps;
  k.decoupled = 1;
  k.seed = cfg.seed;
  k.gmres = cfg.gmres.c();
  k.spai = cfg.spai.c();
  k.max_chain_len = cfg.max_chain_len;
  k.explicit_nnz_cap = 0;
  k.standard_residual_max_dim = cfg.standard_residual_max_dim;
  k.mirror_unstable = cfg.mirror_unstable;
  BirkaState st;
  const size_t r = static_cast<size_t>(cfg.r);
  st.order = cfg.r;
  st.kr.resize(r * r);
  st.er.resize(r * r);
  st.ar.resize(r * r);
  st.fr.resize(r * static_cast<size_t>(m));
  st.cr.resize(r * static_cast<size_t>(q));
  st.lambda_re.resize(r);
  st.lambda_im.resize(r);
  ReductionReport rep;
  rep.rows.resize(2 * r * static_cast<size_t>(cfg.max_sweeps) + 8);
  int sweeps = 0, conv = 0, nrows = 0;
  check(mpg_irka_reduce(op.handle(), b.data(), m, c.data(), q, &k, static_cast<int>(mode),
                        init_shifts ? init_shifts->data() : nullptr, st.kr.data(), st.fr.data(), st.cr.data(),
                        st.er.data(), st.ar.data(), st.lambda_re.data(), st.lambda_im.data(), nullptr, nullptr, &sweeps,
                        &conv, rep.rows.data(), static_cast<int>(rep.rows.size()), &nrows));
  rep.rows.resize(static_cast<size_t>(std::min<int>(nrows, static_cast<int>(rep.rows.size()))));
  st.sweeps = rep.sweeps = sweeps;
  rep.converged = conv != 0;
  return {std::move(st), std::move(rep)};
}

// The same from an initial reduced state: the reference's `const BirkaState* init` (birka.hpp:78-80). Only
// init.kr / fr / cr are read; an empty part keeps the default seed's.
inline std::pair<BirkaState, ReductionReport> birka_reduce(const ShiftedOperator& op, const std::vector<double>& b,
                                                           int m, const std::vector<double>& c, int q,
                                                           const BirkaConfig& cfg, PrecondMode mode,
                                                           const BirkaState& init) {
  mpg_irka_cfg k{};
  k.r = cfg.r;
  k.tol = cfg.tol;
  k.max_sweeps = cfg.max_sweeps;
  k.decoupled = 1;
  k.seed = cfg.seed;
  k.gmres = cfg.gmres.c();
  k.spai = cfg.spai.c();
  k.max_chain_len = cfg.max_chain_len;
  k.explicit_nnz_cap = 0;
  k.standard_residual_max_dim = cfg.standard_residual_max_dim;
  k.mirror_unstable = cfg.mirror_unstable;
  const size_t r = static_cast<size_t>(cfg.r);
  auto part = [](const std::vector<double>& v, size_t want, const char* what) -> const double* {
    if (v.empty()) return nullptr;
    if (v.size() != want) throw std::invalid_argument(std::string("birka: initial state dimensions do not match the system (") + what + ")");
    return v.data();
  };
  const double* ikr = part(init.kr, r * r, "kr");
  const double* ifr = part(init.fr, r * static_cast<size_t>(m), "fr");
  const double* icr = part(init.cr, r * static_cast<size_t>(q), "cr");
  BirkaState st;
  st.order = cfg.r;
  st.kr.resize(r * r);
  st.er.resize(r * r);
  st.ar.resize(r * r);
  st.fr.resize(r * static_cast<size_t>(m));
  st.cr.resize(r * static_cast<size_t>(q));
  st.lambda_re.resize(r);
  st.lambda_im.resize(r);
  ReductionReport rep;
  rep.rows.resize(2 * r * static_cast<size_t>(cfg.max_sweeps) + 8);
  int sweeps = 0, conv = 0, nrows = 0;
  check(mpg_irka_reduce_from(op.handle(), b.data(), m, c.data(), q, &k, static_cast<int>(mode), ikr, ifr, icr,
                             st.kr.data(), st.fr.data(), st.cr.data(), st.er.data(), st.ar.data(),
                             st.lambda_re.data(), st.lambda_im.data(), &sweeps, &conv, rep.rows.data(),
                             static_cast<int>(rep.rows.size()), &nrows));
  rep.rows.resize(static_cast<size_t>(std::min<int>(nrows, static_cast<int>(rep.rows.size()))));
  st.sweeps = rep.sweeps = sweeps;
  rep.converged = conv != 0;
  return {std::move(st), std::move(rep)};
}

// birka_reduce (birka.hpp:78-80) for x' = K x + sum_j N_j x u_j + F u with couplings: joint n r solves
// per side on the assembled Kronecker operator (mpg_birka_reduce).
inline std::pair<BirkaState, ReductionReport> birka_reduce(const SparseMatrix& k,
                                                           const std::vector<const SparseMatrix*>& n_ops,
                                                           const std::vector<double>& f, int m,
                                                           const std::vector<double>& c, int q,
                                                           const BirkaConfig& cfg, PrecondMode mode) {
  if (static_cast<int>(n_ops.size()) != m) throw std::invalid_argument("birka: one N per input is required");
  mpg_irka_cfg kc{};
  kc.r = cfg.r;
  kc.tol = cfg.tol;
  kc.max_sweeps = cfg.max_sweeps;
  kc.seed = cfg.seed;
  kc.gmres = cfg.gmres.c();
  kc.spai = cfg.spai.c();
  kc.max_chain_len = cfg.max_chain_len;
  kc.explicit_nnz_cap = cfg.explicit_nnz_cap;
  kc.standard_residual_max_dim = cfg.standard_residual_max_dim;
  std::vector<const mpg_csr*> hs;
  for (const SparseMatrix* nj : n_ops) hs.push_back(nj->handle());
  const size_t r = static_cast<size_t>(cfg.r);
  BirkaState st;
  st.order = cfg.r;
  st.kr.resize(r * r);
  std::vector<double> nr(r * r * static_cast<size_t>(std::max(m, 1)));
  st.fr.resize(r * static_cast<size_t>(m));
  st.cr.resize(r * static_cast<size_t>(q));
  st.lambda_re.resize(r);
  st.lambda_im.resize(r);
  ReductionReport rep;
  rep.rows.resize(2 * static_cast<size_t>(cfg.max_sweeps) + 4);
  int sweeps = 0, conv = 0, nrows = 0;
  char* warn = nullptr;
  check(mpg_birka_reduce(k.handle(), hs.data(), f.data(), m, c.data(), q, &kc, static_cast<int>(mode), st.kr.data(),
                         nr.data(), st.fr.data(), st.cr.data(), st.lambda_re.data(), st.lambda_im.data(), nullptr,
                         nullptr, &sweeps, &conv, rep.rows.data(), static_cast<int>(rep.rows.size()), &nrows, &warn));
  if (warn) {
    rep.warnings = warn;
    mpg_buffer_free(warn);
  }
  for (int j = 0; j < m; ++j) st.nr.emplace_back(nr.begin() + j * r * r, nr.begin() + (j + 1) * r * r);
  rep.rows.resize(static_cast<size_t>(std::min<int>(nrows, static_cast<int>(rep.rows.size()))));
  st.sweeps = rep.sweeps = sweeps;
  rep.converged = conv != 0;
  return {std::move(st), std::move(rep)};
}

// ---- QB-IHOMM (qbihomm.hpp:15-71) ------------------------------------------------
// QbSystem with H given as triplets (row a, column b n + c, value).
struct QbSystem {
  SparseMatrix d, k, n_op;
  std::vector<index_t> h_rows, h_cols;
  std::vector<double> h_vals;
  std::vector<double> f, c;  // SISO
  index_t dim() const { return d.rows(); }
};

struct QbConfig {  // qbihomm.hpp:35-43
  std::vector<double> sigmas;
  int p_moments = 1, q_moments = 1;
  GmresConfig gmres{};
  SpaiConfig spai{};
  int max_chain_len = 16;
  index_t standard_residual_max_dim = 5000;
};

struct ReducedQb {  // qbihomm.hpp:45-52, column-major
  int order = 0;
  std::vector<double> d, k, n_op, h, f, c, basis;
};

// qbihomm_reduce (qbihomm.hpp:66-67): the moment solves run on the device.
inline std::pair<ReducedQb, ReductionReport> qbihomm_reduce(const QbSystem& sys, const QbConfig& cfg, PrecondMode mode) {
  const ShiftedOperator op(sys.k, &sys.d);
  mpg_qb_cfg q{};
  q.p_moments = cfg.p_moments;
  q.q_moments = cfg.q_moments;
  q.gmres = cfg.gmres.c();
  q.spai = cfg.spai.c();
  q.max_chain_len = cfg.max_chain_len;
  q.standard_residual_max_dim = cfg.standard_residual_max_dim;
  const size_t n = static_cast<size_t>(sys.dim());
  const size_t cap = std::max<size_t>(1, cfg.sigmas.size() * static_cast<size_t>(cfg.p_moments + 2 * cfg.q_moments + 2));
  ReducedQb red;
  std::vector<double> basis(n * cap), d(cap * cap), k(cap * cap), nn(cap * cap), h(cap * cap * cap), f(cap), c(cap);
  ReductionReport rep;
  rep.rows.resize(4 * std::max<size_t>(1, cfg.sigmas.size()));
  int order = 0, nrows = 0;
  check(mpg_qbihomm_reduce(op.handle(), sys.n_op.handle(), static_cast<int64_t>(sys.h_vals.size()), sys.h_rows.data(),
                           sys.h_cols.data(), sys.h_vals.data(), sys.f.data(), sys.c.data(),
                           static_cast<int>(cfg.sigmas.size()), cfg.sigmas.data(), &q, static_cast<int>(mode),
                           static_cast<int>(cap), &order, basis.data(), d.data(), k.data(), nn.data(), h.data(),
                           f.data(), c.data(), rep.rows.data(), static_cast<int>(rep.rows.size()), &nrows));
  const size_t r = static_cast<size_t>(order);
  red.order = order;
  red.d.assign(d.begin(), d.begin() + long(r * r));
  red.k.assign(k.begin(), k.begin() + long(r * r));
  red.n_op.assign(nn.begin(), nn.begin() + long(r * r));
  red.h.assign(h.begin(), h.begin() + long(r * r * r));
  red.f.assign(f.begin(), f.begin() + long(r));
  red.c.assign(c.begin(), c.begin() + long(r));
  red.basis.assign(basis.begin(), basis.begin() + long(n * r));
  rep.rows.resize(static_cast<size_t>(std::min<int>(nrows, static_cast<int>(rep.rows.size()))));
  rep.converged = true;
  rep.sweeps = 1;
  return {std::move(red), std::move(rep)};
}

}  // namespace morprec_gpu
