// CPU ORACLE — test infrastructure only (see oracle.hpp).
// Restates proj/src/airga.cpp:136-384 (airga_reduce, update_expansion_points)
// with the helpers it uses: OrthBasis::append_block (proj/src/orth.cpp:15-39),
// second_order_to_state_space / h2_norm / h2_distance (proj/src/h2.cpp:11-77)
// and h2_gap (airga.cpp:32-39).
//
// The dense kernels the reference takes from Eigen are restated without it:
// the largest singular value of a block (JacobiSVD at orth.cpp:21-22) as the
// square root of the largest eigenvalue of its Gram matrix; M^{-1} by
// FullPivLU (PartialPivLU at h2.cpp:15); the H2 norm -- the reference
// diagonalises A (EigenSolver + FullPivLU, h2.cpp:28-60) -- by the Lyapunov
// Gramian computed with the matrix sign function (Newton iteration with
// determinant scaling), the same quantity by an independent algorithm; the
// stability test (Re lambda >= -1e-12 max |lambda| gives infinity) and the
// eigenvalue ordering of update_expansion_points use the oracle's Francis QR
// eigenvalues.
#include <algorithm>
#include <cmath>
#include <limits>
#include <string>

#include "oracle.hpp"

namespace oracle {

namespace {

const double kInf = std::numeric_limits<double>::infinity();

std::string shortest_str(double v) {
  char buf[64];
  for (int p = 1; p <= 17; ++p) {
    std::snprintf(buf, sizeof buf, "%.*g", p, v);
    if (std::strtod(buf, nullptr) == v) break;
  }
  return buf;
}

Dense scaled(const Dense& x, double s) {
  Dense y = x;
  for (double& v : y.a) v *= s;
  return y;
}

Dense add(const Dense& x, const Dense& y) {
  Dense z = x;
  for (size_t i = 0; i < z.a.size(); ++i) z.a[i] += y.a[i];
  return z;
}

// orth.cpp:15-39: two-pass Gram-Schmidt of each incoming column, deflation
// below drop_tol times the block's leading singular value.
index_t append_block(std::vector<Vec>& store, index_t capacity, const Dense& block, double drop_tol = 1e-10) {
  if (block.cols == 0) return 0;
  const Dense g = matmul(block.transpose(), block);
  double lmax = 0.0;
  for (const Complex& l : eigenvalues(g)) lmax = std::max(lmax, l.re);
  const double scale = std::sqrt(std::max(lmax, 0.0));
  if (scale == 0.0) return 0;
  const double cutoff = drop_tol * scale;
  index_t kept = 0;
  const index_t n = block.rows;
  for (index_t c = 0; c < block.cols && index_t(store.size()) < capacity; ++c) {
    Vec w(block.col(c), block.col(c) + n);
    for (int pass = 0; pass < 2; ++pass)
      for (const Vec& q : store) {
        double d = 0.0;
        for (index_t i = 0; i < n; ++i) d += q[size_t(i)] * w[size_t(i)];
        for (index_t i = 0; i < n; ++i) w[size_t(i)] -= d * q[size_t(i)];
      }
    double nn = 0.0;
    for (double v : w) nn += v * v;
    nn = std::sqrt(nn);
    if (nn <= cutoff) continue;
    for (double& v : w) v /= nn;
    store.push_back(std::move(w));
    ++kept;
  }
  return kept;
}

Dense basis_matrix(const std::vector<Vec>& store, index_t n) {
  Dense v(n, index_t(store.size()));
  for (size_t j = 0; j < store.size(); ++j) std::copy(store[j].begin(), store[j].end(), v.col(index_t(j)));
  return v;
}

// h2.cpp:11-26
StateSpaceO second_order_ss(const Dense& m, const Dense& d, const Dense& k, const Dense& f, const Dense& c) {
  const index_t r = m.rows;
  FullPivLU mlu(m);
  const Dense mk = mlu.solve(k), md = mlu.solve(d), mf = mlu.solve(f);
  StateSpaceO ss;
  ss.a = Dense(2 * r, 2 * r);
  for (index_t i = 0; i < r; ++i) ss.a(i, r + i) = 1.0;
  for (index_t j = 0; j < r; ++j)
    for (index_t i = 0; i < r; ++i) {
      ss.a(r + i, j) = -mk(i, j);
      ss.a(r + i, r + j) = -md(i, j);
    }
  ss.b = Dense(2 * r, f.cols);
  for (index_t j = 0; j < f.cols; ++j)
    for (index_t i = 0; i < r; ++i) ss.b(r + i, j) = mf(i, j);
  ss.c = Dense(c.cols, 2 * r);
  for (index_t j = 0; j < r; ++j)
    for (index_t i = 0; i < c.cols; ++i) ss.c(i, j) = c(j, i);
  return ss;
}

}  // namespace

// h2.cpp:28-60: infinity when A is not stable; otherwise sqrt(trace(C P C^T))
// with A P + P A^T + B B^T = 0, P from the sign function of A: with
// A_0 = A, Q_0 = B B^T, A_{k+1} = (A_k/c + c A_k^{-1})/2,
// Q_{k+1} = (Q_k/c + c A_k^{-1} Q_k A_k^{-T})/2 (c = |det A_k|^{1/n}),
// A_k -> -I and Q_k -> 2 P.
double h2_norm_o(const StateSpaceO& sys) {
  const index_t ns = sys.a.rows;
  if (ns == 0) return 0.0;
  if (sys.a.cols != ns || sys.b.rows != ns || sys.c.cols != ns) throw std::invalid_argument("h2_norm: inconsistent dimensions");
  std::vector<Complex> lam;
  try {
    lam = eigenvalues(sys.a);
  } catch (const std::exception&) {
    return kInf;
  }
  double max_abs = 0.0;
  for (const Complex& l : lam) max_abs = std::max(max_abs, std::hypot(l.re, l.im));
  for (const Complex& l : lam)
    if (l.re >= -1e-12 * std::max(max_abs, 1.0)) return kInf;
  Dense a = sys.a;
  Dense q = matmul(sys.b, sys.b.transpose());
  for (int it = 0; it < 100; ++it) {
    FullPivLU lu(a);
    if (!lu.invertible()) return kInf;
    const Dense ai = lu.inverse();
    double logdet = 0.0;
    for (index_t i = 0; i < ns; ++i) logdet += std::log(std::fabs(lu.lu(i, i)));
    const double c = std::exp(logdet / double(ns));
    const Dense an = scaled(add(scaled(a, 1.0 / c), scaled(ai, c)), 0.5);
    const Dense qn = scaled(add(scaled(q, 1.0 / c), scaled(matmul(matmul(ai, q), ai.transpose()), c)), 0.5);
    double diff = 0.0, nrm = 0.0;
    for (size_t i = 0; i < an.a.size(); ++i) {
      diff += (an.a[i] - a.a[i]) * (an.a[i] - a.a[i]);
      nrm += an.a[i] * an.a[i];
    }
    a = an;
    q = qn;
    if (std::sqrt(diff) <= 1e-14 * std::sqrt(nrm)) break;
  }
  const Dense p = scaled(q, 0.5);
  const Dense cpc = matmul(matmul(sys.c, p), sys.c.transpose());
  double tr = 0.0;
  for (index_t i = 0; i < cpc.rows; ++i) tr += cpc(i, i);
  return std::sqrt(std::max(tr, 0.0));
}

// h2.cpp:62-77
double h2_distance_o(const StateSpaceO& a, const StateSpaceO& b) {
  if (a.b.cols != b.b.cols || a.c.rows != b.c.rows) throw std::invalid_argument("h2_distance: input/output count mismatch");
  const index_t na = a.a.rows, nb = b.a.rows;
  StateSpaceO e;
  e.a = Dense(na + nb, na + nb);
  for (index_t j = 0; j < na; ++j)
    for (index_t i = 0; i < na; ++i) e.a(i, j) = a.a(i, j);
  for (index_t j = 0; j < nb; ++j)
    for (index_t i = 0; i < nb; ++i) e.a(na + i, na + j) = b.a(i, j);
  e.b = Dense(na + nb, a.b.cols);
  for (index_t j = 0; j < a.b.cols; ++j) {
    for (index_t i = 0; i < na; ++i) e.b(i, j) = a.b(i, j);
    for (index_t i = 0; i < nb; ++i) e.b(na + i, j) = b.b(i, j);
  }
  e.c = Dense(a.c.rows, na + nb);
  for (index_t i = 0; i < a.c.rows; ++i) {
    for (index_t j = 0; j < na; ++j) e.c(i, j) = a.c(i, j);
    for (index_t j = 0; j < nb; ++j) e.c(i, na + j) = -b.c(i, j);
  }
  return h2_norm_o(e);
}

namespace {
// airga.cpp:32-39
double h2_gap(const StateSpaceO& prev, const StateSpaceO& next) {
  const double dist = h2_distance_o(prev, next);
  if (!std::isfinite(dist)) return kInf;
  const double scale = h2_norm_o(next);
  if (!std::isfinite(scale)) return kInf;
  return dist / std::max(1.0, scale);
}

struct SolveStats { int solves = 0; long iterations = 0; double seconds = 0.0; };

// airga.cpp:96-119
Dense solve_block(const LinearOp& a_op, const LinearOp& p_op, const Dense& rhs, const GmresConfig& gmres, double sign,
                  int sweep, int point, int moment, SolveStats& stats) {
  Dense x(rhs.rows, rhs.cols);
  for (index_t col = 0; col < rhs.cols; ++col) {
    Vec b(rhs.col(col), rhs.col(col) + rhs.rows);
    double bn = 0.0;
    for (double v : b) bn += v * v;
    if (bn == 0.0) continue;
    const GmresResult res = gmres_right_preconditioned(a_op, p_op, b, gmres);
    stats.iterations += res.report.iterations;
    stats.seconds += res.report.solve_seconds;
    ++stats.solves;
    if (!res.report.converged)
      throw SolverError("gmres did not converge (sweep " + std::to_string(sweep) + ", point " + std::to_string(point) +
                        ", moment " + std::to_string(moment) + ", column " + std::to_string(col) +
                        "; relative residual " +
                        shortest_str(res.report.final_residual / std::max(res.report.rhs_norm, 1e-300)) + " after " +
                        std::to_string(res.report.iterations) + " iterations)");
    for (index_t i = 0; i < rhs.rows; ++i) x(i, col) = sign * res.x[size_t(i)];
  }
  return x;
}

// airga.cpp:121-132
AirgaModel project(const Csr& m, const Csr& d, const Csr& k, const Dense& v, const Dense& f, const Dense& c) {
  AirgaModel red;
  const Dense vt = v.transpose();
  red.m = matmul(vt, m.multiply(v));
  red.d = matmul(vt, d.multiply(v));
  red.k = matmul(vt, k.multiply(v));
  red.f = matmul(vt, f);
  red.c = matmul(vt, c);
  red.basis = v;
  return red;
}

StateSpaceO to_ss(const AirgaModel& r) { return second_order_ss(r.m, r.d, r.k, r.f, r.c); }
}  // namespace

// airga.cpp:319-384
std::vector<double> update_expansion_points(const Dense& m, const Dense& d, const Dense& k,
                                            const std::vector<double>& current) {
  const size_t want = current.size();
  if (want == 0) return {};
  const index_t r = m.rows;
  if (r == 0) return current;
  const Dense zero(r, 1);
  const StateSpaceO ss = second_order_ss(m, d, k, zero, zero);
  std::vector<Complex> lam;
  try {
    lam = eigenvalues(ss.a);
  } catch (const std::exception&) {
    return current;
  }
  std::vector<size_t> order(lam.size());
  for (size_t i = 0; i < order.size(); ++i) order[i] = i;
  std::sort(order.begin(), order.end(), [&](size_t a, size_t b) {
    const double ra = std::fabs(lam[a].re), rb = std::fabs(lam[b].re);
    if (ra != rb) return ra < rb;
    return std::fabs(lam[a].im) > std::fabs(lam[b].im);
  });
  std::vector<double> next;
  double max_s = 0.0;
  for (size_t idx : order) {
    if (next.size() >= want) break;
    const Complex l = lam[idx];
    const double labs = std::hypot(l.re, l.im);
    double s = std::fabs(l.im);
    if (s <= 1e-12 * labs) s = labs;
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

// airga.cpp:136-317
AirgaResult airga_reduce(const Csr& m, const Csr& d, const Csr& k, const Dense& f, const Dense& c, double alpha,
                         double beta, const AirgaConfigO& cfg, PrecondMode mode) {
  const index_t n = m.nrows;
  std::vector<double> points = cfg.expansion_points;
  if (points.empty()) throw ConfigError("airga: at least one expansion point is required");
  std::sort(points.begin(), points.end());
  for (double s : points)
    if (!(s > 0.0) || !std::isfinite(s)) throw ConfigError("airga: expansion points must be positive and finite");
  if (std::adjacent_find(points.begin(), points.end()) != points.end())
    throw ConfigError("airga: expansion points must be distinct");
  const int ell = int(points.size());
  if (cfg.r_max < ell)
    throw ConfigError("airga: r_max (" + std::to_string(cfg.r_max) +
                      ") must be at least the number of expansion points (" + std::to_string(ell) + ")");
  if (cfg.max_outer < 1) throw ConfigError("airga: max_outer must be at least 1");
  if (cfg.max_chain_len < 1) throw ConfigError("airga: max_chain_len must be at least 1");

  AirgaResult out;
  ReductionReport& report = out.report;
  {  // :156-163
    const double dnorm = d.frobenius_norm();
    const double defect = Csr::linear_combination({{1.0, &d}, {-alpha, &m}, {-beta, &k}}).frobenius_norm();
    if (dnorm > 0.0 && defect > 1e-12 * dnorm)
      report.warnings.push_back("damping deviates from alpha*M + beta*K (relative defect " +
                                shortest_str(defect / dnorm) + "); reduction proceeds on D as given");
  }
  PrecondChain prev_first_chain;
  Csr prev_first_matrix;
  AirgaModel model;
  StateSpaceO prev_ss;
  bool have_prev = false, converged = false;
  int sweeps_done = 0;
  std::vector<double> final_points = points;

  for (int z = 1; z <= cfg.max_outer; ++z) {
    out.point_history.push_back(points);
    std::vector<Vec> store;
    std::vector<Csr> a_ops;
    for (double s : points) a_ops.push_back(shifted_operator2(m, d, k, s));
    std::vector<PrecondChain> chains(static_cast<size_t>(ell));
    std::vector<LinearOp> precs(static_cast<size_t>(ell));
    std::vector<Dense> blocks(static_cast<size_t>(ell));
    for (int i = 0; i < ell; ++i) {  // :196-259
      ReportRow row;
      row.sweep = z;
      row.point = i + 1;
      if (mode == PrecondMode::None) {
        precs[size_t(i)] = identity_operator();
        row.kind = PrecondKind::None;
      } else if (mode == PrecondMode::FreshSpai) {
        SpaiResult built = spai_build(a_ops[size_t(i)], cfg.spai);
        row.precond_build_seconds = built.build_seconds;
        chains[size_t(i)] = PrecondChain(std::move(built.p), built.build_seconds);
        precs[size_t(i)] = chains[size_t(i)].as_operator();
        row.kind = PrecondKind::Fresh;
      } else {
        const bool first_ever = z == 1 && i == 0;
        const PrecondChain* parent = i == 0 ? (z == 1 ? nullptr : &prev_first_chain) : &chains[size_t(i - 1)];
        if (first_ever || parent->length() + 1 > cfg.max_chain_len) {
          SpaiResult built = spai_build(a_ops[size_t(i)], cfg.spai);
          row.precond_build_seconds = built.build_seconds;
          chains[size_t(i)] = PrecondChain(std::move(built.p), built.build_seconds);
          row.kind = PrecondKind::Fresh;
        } else {
          const Csr& a_prev = i == 0 ? prev_first_matrix : a_ops[size_t(i - 1)];
          UpdateFactor f = update_build(a_prev, a_ops[size_t(i)], cfg.spai);
          row.kind = i == 0 ? PrecondKind::Vertical : PrecondKind::Horizontal;
          row.precond_build_seconds = f.build_seconds;
          row.min_residual = f.min_residual;
          row.matrix_change = f.matrix_change;
          chains[size_t(i)] = parent->extended(std::make_shared<const UpdateFactor>(std::move(f)));
        }
        precs[size_t(i)] = chains[size_t(i)].as_operator();
      }
      SolveStats st;
      blocks[size_t(i)] = solve_block(matvec_operator(a_ops[size_t(i)]), precs[size_t(i)], f, cfg.gmres, 1.0, z, i + 1, 0, st);
      row.solves = st.solves;
      row.gmres_iterations = st.iterations;
      row.gmres_seconds = st.seconds;
      if (mode != PrecondMode::None && n <= cfg.standard_residual_max_dim)
        row.standard_residual = standard_residual(a_ops[size_t(i)], chains[size_t(i)]);
      report.rows.push_back(row);
    }
    for (int i = 0; i < ell; ++i) append_block(store, cfg.r_max, blocks[size_t(i)]);
    AirgaModel red = project(m, d, k, basis_matrix(store, n), f, c);
    StateSpaceO red_ss = to_ss(red);
    std::vector<ReportRow> moment_rows(static_cast<size_t>(ell));
    for (int i = 0; i < ell; ++i) {
      moment_rows[size_t(i)].sweep = z;
      moment_rows[size_t(i)].point = i + 1;
      moment_rows[size_t(i)].kind = PrecondKind::ReusedSameMatrix;
    }
    for (int j = 1; index_t(store.size()) < cfg.r_max; ++j) {  // :270-291
      bool appended = false;
      for (int i = 0; i < ell && index_t(store.size()) < cfg.r_max; ++i) {
        const Dense rhs = m.multiply(blocks[size_t(i)]);
        SolveStats st;
        blocks[size_t(i)] =
            solve_block(matvec_operator(a_ops[size_t(i)]), precs[size_t(i)], rhs, cfg.gmres, -1.0, z, i + 1, j, st);
        moment_rows[size_t(i)].solves += st.solves;
        moment_rows[size_t(i)].gmres_iterations += st.iterations;
        moment_rows[size_t(i)].gmres_seconds += st.seconds;
        if (append_block(store, cfg.r_max, blocks[size_t(i)]) > 0) appended = true;
      }
      if (!appended) break;
      AirgaModel next = project(m, d, k, basis_matrix(store, n), f, c);
      StateSpaceO next_ss = to_ss(next);
      const double gap = h2_gap(red_ss, next_ss);
      red = std::move(next);
      red_ss = std::move(next_ss);
      if (gap <= cfg.inner_tol) break;
    }
    if (index_t(store.size()) >= cfg.r_max && cfg.r_max > ell)
      report.warnings.push_back("sweep " + std::to_string(z) + ": basis reached r_max before inner convergence");
    for (const ReportRow& r : moment_rows)
      if (r.solves > 0) report.rows.push_back(r);
    sweeps_done = z;
    model = std::move(red);
    final_points = points;
    if (have_prev && h2_gap(prev_ss, red_ss) <= cfg.outer_tol) {
      converged = true;
      break;
    }
    prev_ss = std::move(red_ss);
    have_prev = true;
    if (mode == PrecondMode::ReuseChain) {
      prev_first_chain = chains[0];
      prev_first_matrix = a_ops[0];
    }
    if (z < cfg.max_outer) points = update_expansion_points(model.m, model.d, model.k, points);
  }
  report.converged = converged;
  report.reduced_order = int(model.basis.cols);
  report.sweeps = sweeps_done;
  out.model = std::move(model);
  out.final_points = final_points;
  if (!converged) report.warnings.push_back("outer loop left unconverged after " + std::to_string(sweeps_done) + " sweeps");
  return out;
}

}  // namespace oracle
