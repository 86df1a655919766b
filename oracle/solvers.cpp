// CPU ORACLE — test infrastructure only (see oracle.hpp).
// Restates proj/src/gmres.cpp, proj/src/spai.cpp, proj/src/chain.cpp and
// proj/src/parallel.cpp.
#include <algorithm>
#include <chrono>
#include <cmath>
#include <exception>
#include <mutex>
#include <thread>

#include "oracle.hpp"

namespace oracle {

// ---- parallel_for (proj/src/parallel.cpp:13-46) -------------------------------
void parallel_for(index_t begin, index_t end, int threads, const std::function<void(index_t)>& fn) {
  const index_t count = end - begin;
  if (count <= 0) return;
  const index_t workers = std::clamp<index_t>(threads, 1, std::max<index_t>(count, 1));
  if (workers == 1) {
    for (index_t i = begin; i < end; ++i) fn(i);
    return;
  }
  std::exception_ptr first;
  std::mutex mu;
  std::vector<std::thread> pool;
  const index_t chunk = (count + workers - 1) / workers;
  for (index_t w = 0; w < workers; ++w) {
    const index_t lo = begin + w * chunk, hi = std::min(end, lo + chunk);
    if (lo >= hi) break;
    pool.emplace_back([&, lo, hi] {
      try {
        for (index_t i = lo; i < hi; ++i) fn(i);
      } catch (...) {
        std::scoped_lock l(mu);
        if (!first) first = std::current_exception();
      }
    });
  }
  for (auto& t : pool) t.join();
  if (first) std::rethrow_exception(first);
}

// ---- GMRES (proj/src/gmres.cpp:40-186) -----------------------------------------
LinearOp identity_operator() {
  return [](const Vec& in, Vec& out) { out = in; };
}
LinearOp matvec_operator(const Csr& a) {
  auto m = std::make_shared<const Csr>(a);
  return [m](const Vec& in, Vec& out) { m->multiply(in, out); };
}

namespace {
constexpr double REORTH_TOL = 1e-10;  // proj/src/gmres.cpp:14

double dot(const Vec& a, const Vec& b) {
  double s = 0.0;
  for (size_t i = 0; i < a.size(); ++i) s += a[i] * b[i];
  return s;
}
double nrm(const Vec& a) { return std::sqrt(dot(a, a)); }
void axpy(double alpha, const Vec& x, Vec& y) {
  for (size_t i = 0; i < x.size(); ++i) y[i] += alpha * x[i];
}

// proj/src/gmres.cpp:17-26
Vec back_substitute(const std::vector<Vec>& h, const Vec& g, int k) {
  Vec y(static_cast<size_t>(k));
  for (int i = k - 1; i >= 0; --i) {
    double acc = g[size_t(i)];
    for (int j = i + 1; j < k; ++j) acc -= h[size_t(j)][size_t(i)] * y[size_t(j)];
    y[size_t(i)] = acc / h[size_t(i)][size_t(i)];
  }
  return y;
}
}  // namespace

GmresResult gmres_right_preconditioned(const LinearOp& apply_a, const LinearOp& apply_p, const Vec& b,
                                       const GmresConfig& cfg) {
  const auto t0 = std::chrono::steady_clock::now();
  GmresResult res;
  GmresReport& rep = res.report;
  const double bnorm = nrm(b);
  rep.rhs_norm = bnorm;
  if (bnorm == 0.0) throw std::invalid_argument("gmres: zero right-hand side");
  const double target = cfg.rel_tol * bnorm;
  const size_t n = b.size();
  std::vector<Vec> basis;
  basis.push_back(b);
  for (double& v : basis[0]) v /= bnorm;
  std::vector<Vec> h_cols;
  Vec gc, gs;
  Vec g(static_cast<size_t>(cfg.max_iter) + 1, 0.0);
  g[0] = bnorm;
  if (cfg.record_history) rep.residual_history.push_back(bnorm);
  Vec pv(n), w(n), probe(n), residual(n);
  double estimate = bnorm, recheck_at = target;

  auto assemble_solution = [&](int k) {
    const Vec y = back_substitute(h_cols, g, k);
    Vec u(n, 0.0);
    for (int j = 0; j < k; ++j) axpy(y[size_t(j)], basis[size_t(j)], u);
    Vec x(n);
    apply_p(u, x);
    return x;
  };
  auto true_residual = [&](const Vec& x) {
    apply_a(x, probe);
    for (size_t i = 0; i < n; ++i) residual[i] = b[i] - probe[i];
    return nrm(residual);
  };
  auto seconds = [&] { return std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count(); };
  auto finish = [&](int k, bool guess) {
    if (k > 0) {
      res.x = assemble_solution(k);
      rep.final_residual = true_residual(res.x);
    } else {
      res.x.assign(n, 0.0);
      rep.final_residual = bnorm;
    }
    rep.converged = guess && rep.final_residual <= target;
    rep.solve_seconds = seconds();
    return res;
  };

  for (int k = 0; k < cfg.max_iter; ++k) {
    apply_p(basis[size_t(k)], pv);
    apply_a(pv, w);
    const double wnorm_pre = nrm(w);
    Vec h(static_cast<size_t>(k) + 2, 0.0);
    for (int i = 0; i <= k; ++i) {  // modified Gram-Schmidt, :101-105
      const double hi = dot(basis[size_t(i)], w);
      h[size_t(i)] = hi;
      axpy(-hi, basis[size_t(i)], w);
    }
    double wnorm = nrm(w);
    if (wnorm > 0.0) {  // measured second pass, :108-119
      Vec d(static_cast<size_t>(k) + 1);
      for (int i = 0; i <= k; ++i) d[size_t(i)] = dot(basis[size_t(i)], w);
      if (nrm(d) > REORTH_TOL * wnorm) {
        for (int i = 0; i <= k; ++i) {
          axpy(-d[size_t(i)], basis[size_t(i)], w);
          h[size_t(i)] += d[size_t(i)];
        }
        wnorm = nrm(w);
        ++rep.reorth_passes;
      }
    }
    const bool invariant = wnorm <= 1e-14 * std::max(wnorm_pre, 1e-300);
    h[size_t(k) + 1] = invariant ? 0.0 : wnorm;
    for (int i = 0; i < k; ++i) {
      const double t1 = gc[size_t(i)] * h[size_t(i)] + gs[size_t(i)] * h[size_t(i) + 1];
      const double t2 = -gs[size_t(i)] * h[size_t(i)] + gc[size_t(i)] * h[size_t(i) + 1];
      h[size_t(i)] = t1;
      h[size_t(i) + 1] = t2;
    }
    const double diag = h[size_t(k)], sub = h[size_t(k) + 1];
    if (diag == 0.0 && sub == 0.0) {
      rep.breakdown = true;
      rep.iterations = k;
      return finish(k, estimate <= target);
    }
    const double denom = std::hypot(diag, sub);
    const double c = diag / denom, s = sub / denom;
    gc.push_back(c);
    gs.push_back(s);
    h[size_t(k)] = denom;
    h.resize(static_cast<size_t>(k) + 1);
    h_cols.push_back(std::move(h));
    g[size_t(k) + 1] = -s * g[size_t(k)];
    g[size_t(k)] = c * g[size_t(k)];
    estimate = std::abs(g[size_t(k) + 1]);
    rep.iterations = k + 1;
    if (cfg.record_history) rep.residual_history.push_back(estimate);
    if (invariant) {
      rep.breakdown = estimate > target;
      return finish(k + 1, estimate <= target);
    }
    if (estimate <= recheck_at) {  // :166-180
      Vec x = assemble_solution(k + 1);
      const double tr = true_residual(x);
      if (tr <= target) {
        res.x = std::move(x);
        rep.final_residual = tr;
        rep.converged = true;
        rep.solve_seconds = seconds();
        return res;
      }
      recheck_at *= 0.25;
    }
    Vec next = w;
    for (double& v : next) v /= wnorm;
    basis.push_back(std::move(next));
  }
  return finish(rep.iterations, estimate <= target);
}

// ---- SPAI (proj/src/spai.cpp) --------------------------------------------------------
// proj/src/spai.cpp:16-41
PatternSolve solve_pattern(const Csr& a, const std::vector<index_t>& pattern, const index_t* rhs_rows,
                           const double* rhs_vals, size_t rhs_n) {
  Csr::ColumnSubmatrix sub = a.extract_column_submatrix(pattern);
  const auto& rows = sub.row_map;
  Vec local(rows.size(), 0.0);
  double outside_sq = 0.0;
  for (size_t k = 0; k < rhs_n; ++k) {
    const auto it = std::lower_bound(rows.begin(), rows.end(), rhs_rows[k]);
    if (it != rows.end() && *it == rhs_rows[k]) local[size_t(it - rows.begin())] = rhs_vals[k];
    else outside_sq += rhs_vals[k] * rhs_vals[k];
  }
  ColPivQR qr(sub.block);
  PatternSolve out;
  out.coeffs = qr.solve(local);
  out.rank_deficient = qr.rank() < index_t(pattern.size());
  double local_sq = 0.0;
  for (size_t i = 0; i < rows.size(); ++i) {
    double r = local[i];
    for (size_t c = 0; c < pattern.size(); ++c) r -= sub.block(index_t(i), index_t(c)) * out.coeffs[c];
    local_sq += r * r;
  }
  out.residual = std::sqrt(local_sq + outside_sq);
  return out;
}

// proj/src/spai.cpp:43-87
std::vector<index_t> initial_pattern(const Csr& a, index_t col, const SpaiConfig& cfg) {
  std::vector<index_t> pattern;
  if (cfg.pattern_kind == 0) {
    pattern.push_back(col);
  } else if (cfg.pattern_kind == 1) {
    for (index_t k = a.col_begin(col); k < a.col_end(col); ++k) pattern.push_back(a.srow[size_t(k)]);
  } else {
    std::vector<index_t> frontier{col};
    std::vector<char> seen(static_cast<size_t>(a.nrows), 0);
    for (int step = 0; step < std::max(cfg.power, 1); ++step) {
      std::vector<index_t> next;
      for (index_t j : frontier)
        for (index_t k = a.col_begin(j); k < a.col_end(j); ++k) {
          const index_t i = a.srow[size_t(k)];
          if (!seen[size_t(i)]) { seen[size_t(i)] = 1; next.push_back(i); }
        }
      pattern.insert(pattern.end(), next.begin(), next.end());
      frontier = std::move(next);
      if (frontier.empty()) break;
    }
  }
  pattern.push_back(col);
  std::sort(pattern.begin(), pattern.end());
  pattern.erase(std::unique(pattern.begin(), pattern.end()), pattern.end());
  if (int(pattern.size()) > cfg.max_fill_per_col) {
    std::vector<index_t> kept(pattern.begin(), pattern.begin() + cfg.max_fill_per_col);
    if (!std::binary_search(kept.begin(), kept.end(), col)) {
      kept.back() = col;
      std::sort(kept.begin(), kept.end());
    }
    pattern = std::move(kept);
  }
  return pattern;
}

// proj/src/spai.cpp:89-154
AdaptiveOutcome adaptive_column(const Csr& a, index_t col, const index_t* rhs_rows, const double* rhs_vals,
                                size_t rhs_n, const SpaiConfig& cfg) {
  AdaptiveOutcome out;
  out.pattern = initial_pattern(a, col, cfg);
  double rhs_norm = 0.0;
  for (size_t k = 0; k < rhs_n; ++k) rhs_norm += rhs_vals[k] * rhs_vals[k];
  rhs_norm = std::sqrt(rhs_norm);
  const double threshold = cfg.fill_tol * rhs_norm;
  PatternSolve solve = solve_pattern(a, out.pattern, rhs_rows, rhs_vals, rhs_n);
  for (int sweep = 0; sweep < cfg.max_pattern_sweeps; ++sweep) {
    if (solve.residual <= threshold) break;
    if (int(out.pattern.size()) >= cfg.max_fill_per_col) break;
    std::vector<index_t> touched(rhs_rows, rhs_rows + rhs_n);
    for (index_t j : out.pattern)
      for (index_t k = a.col_begin(j); k < a.col_end(j); ++k) touched.push_back(a.srow[size_t(k)]);
    std::sort(touched.begin(), touched.end());
    touched.erase(std::unique(touched.begin(), touched.end()), touched.end());
    Vec resid(touched.size(), 0.0);
    auto slot = [&](index_t row) { return size_t(std::lower_bound(touched.begin(), touched.end(), row) - touched.begin()); };
    for (size_t k = 0; k < rhs_n; ++k) resid[slot(rhs_rows[k])] += rhs_vals[k];
    for (size_t c = 0; c < out.pattern.size(); ++c)
      for (index_t k = a.col_begin(out.pattern[c]); k < a.col_end(out.pattern[c]); ++k)
        resid[slot(a.srow[size_t(k)])] -= solve.coeffs[c] * a.sval[size_t(k)];
    index_t best = -1;
    double best_mag = 0.0;
    for (size_t k = 0; k < touched.size(); ++k) {
      const index_t row = touched[k];
      const double mag = std::abs(resid[k]);
      if (mag <= best_mag) continue;
      if (row >= a.ncols) continue;
      if (std::binary_search(out.pattern.begin(), out.pattern.end(), row)) continue;
      if (a.col_begin(row) == a.col_end(row)) continue;
      best = row;
      best_mag = mag;
    }
    if (best < 0) break;
    out.pattern.insert(std::lower_bound(out.pattern.begin(), out.pattern.end(), best), best);
    solve = solve_pattern(a, out.pattern, rhs_rows, rhs_vals, rhs_n);
  }
  out.coeffs = std::move(solve.coeffs);
  out.residual = solve.residual;
  out.rank_deficient = solve.rank_deficient;
  return out;
}

// proj/src/spai.cpp:158-173
SpaiColumn spai_column_solve(const Csr& a, index_t col, std::vector<index_t> pattern) {
  if (col < 0 || col >= a.ncols) throw std::invalid_argument("spai_column_solve: column out of range");
  std::sort(pattern.begin(), pattern.end());
  const index_t unit_row = col;
  const double unit_val = 1.0;
  PatternSolve s = solve_pattern(a, pattern, &unit_row, &unit_val, 1);
  SpaiColumn out;
  out.rows = std::move(pattern);
  out.values = std::move(s.coeffs);
  out.residual = s.residual;
  out.rank_deficient = s.rank_deficient;
  return out;
}

// proj/src/spai.cpp:175-238
SpaiResult spai_build(const Csr& a, const SpaiConfig& cfg) {
  if (a.nrows != a.ncols) throw std::invalid_argument("spai_build: matrix must be square");
  if (cfg.fill_tol < 0.0 || cfg.max_fill_per_col < 1 || cfg.max_pattern_sweeps < 0)
    throw std::invalid_argument("spai_build: invalid configuration");
  const auto t0 = std::chrono::steady_clock::now();
  const index_t n = a.nrows;
  struct ColumnOut { std::vector<index_t> rows; Vec values; double residual = 0; bool fallback = false; };
  std::vector<ColumnOut> columns(static_cast<size_t>(n));
  parallel_for(0, n, cfg.threads, [&](index_t col) {
    const index_t unit_row = col;
    const double unit_val = 1.0;
    AdaptiveOutcome got = adaptive_column(a, col, &unit_row, &unit_val, 1, cfg);
    ColumnOut& slot = columns[size_t(col)];
    if (got.rank_deficient) {
      slot.fallback = true;
      double diag = 0.0;
      for (index_t k = a.col_begin(col); k < a.col_end(col); ++k)
        if (a.srow[size_t(k)] == col) diag = a.sval[size_t(k)];
      const double coeff = diag != 0.0 ? 1.0 / diag : 1.0;
      slot.rows = {col};
      slot.values = {coeff};
      double sq = 0.0;
      bool hit = false;
      for (index_t k = a.col_begin(col); k < a.col_end(col); ++k) {
        const index_t r = a.srow[size_t(k)];
        const double e = (r == col ? 1.0 : 0.0) - coeff * a.sval[size_t(k)];
        if (r == col) hit = true;
        sq += e * e;
      }
      if (!hit) sq += 1.0;
      slot.residual = std::sqrt(sq);
      return;
    }
    slot.rows = std::move(got.pattern);
    slot.values = std::move(got.coeffs);
    slot.residual = got.residual;
  });
  std::vector<Triplet> entries;
  SpaiResult result;
  result.column_residuals.resize(static_cast<size_t>(n));
  for (index_t col = 0; col < n; ++col) {
    const ColumnOut& s = columns[size_t(col)];
    for (size_t k = 0; k < s.rows.size(); ++k) entries.push_back({s.rows[k], col, s.values[k]});
    result.column_residuals[size_t(col)] = s.residual;
    if (s.fallback) ++result.fallback_count;
  }
  result.p = Csr::from_triplets(n, n, std::move(entries));
  result.build_seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  return result;
}

// ---- update factors (proj/src/chain.cpp:16-98) -------------------------------------
UpdateFactor update_build(const Csr& prev, const Csr& next, const SpaiConfig& cfg) {
  if (prev.nrows != next.nrows || prev.ncols != next.ncols) throw std::invalid_argument("update_build: shape mismatch");
  if (next.nrows != next.ncols) throw std::invalid_argument("update_build: matrices must be square");
  const auto t0 = std::chrono::steady_clock::now();
  const index_t n = next.nrows;
  struct ColumnOut { std::vector<index_t> rows; Vec values; double residual_sq = 0; bool fallback = false; };
  std::vector<ColumnOut> columns(static_cast<size_t>(n));
  parallel_for(0, n, cfg.threads, [&](index_t col) {
    const index_t* rr = prev.srow.data() + prev.col_begin(col);
    const double* rv = prev.sval.data() + prev.col_begin(col);
    const size_t rn = size_t(prev.col_end(col) - prev.col_begin(col));
    ColumnOut& slot = columns[size_t(col)];
    if (rn == 0) {
      slot.rows = {col};
      slot.values = {0.0};
      return;
    }
    AdaptiveOutcome got = adaptive_column(next, col, rr, rv, rn, cfg);
    if (got.rank_deficient) {
      slot.fallback = true;
      slot.rows = {col};
      slot.values = {1.0};
      double sq = 0.0;
      const index_t* nr = next.srow.data() + next.col_begin(col);
      const double* nv = next.sval.data() + next.col_begin(col);
      const size_t nn = size_t(next.col_end(col) - next.col_begin(col));
      size_t pa = 0, pb = 0;
      while (pa < rn || pb < nn) {
        if (pb >= nn || (pa < rn && rr[pa] < nr[pb])) { sq += rv[pa] * rv[pa]; ++pa; }
        else if (pa >= rn || nr[pb] < rr[pa]) { sq += nv[pb] * nv[pb]; ++pb; }
        else { const double e = rv[pa] - nv[pb]; sq += e * e; ++pa; ++pb; }
      }
      slot.residual_sq = sq;
      return;
    }
    slot.rows = std::move(got.pattern);
    slot.values = std::move(got.coeffs);
    slot.residual_sq = got.residual * got.residual;
  });
  std::vector<Triplet> entries;
  double total = 0.0;
  UpdateFactor f;
  for (index_t col = 0; col < n; ++col) {
    const ColumnOut& s = columns[size_t(col)];
    for (size_t k = 0; k < s.rows.size(); ++k) entries.push_back({s.rows[k], col, s.values[k]});
    total += s.residual_sq;
    if (s.fallback) ++f.fallback_count;
  }
  f.q = Csr::from_triplets(n, n, std::move(entries));
  f.min_residual = std::sqrt(total);
  f.matrix_change = frobenius_distance(prev, next);
  f.build_seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  return f;
}

// ---- PrecondChain (proj/src/chain.cpp:100-138) -------------------------------------
PrecondChain::PrecondChain(Csr base, double secs)
    : total_build_seconds(secs), base_(std::make_shared<const Csr>(std::move(base))) {
  if (base_->nrows != base_->ncols) throw std::invalid_argument("chain: base must be square");
}

PrecondChain PrecondChain::extended(std::shared_ptr<const UpdateFactor> f) const {
  if (empty()) throw std::logic_error("chain: cannot extend an empty chain");
  if (!f) throw std::invalid_argument("chain: null update factor");
  if (f->q.nrows != dim() || f->q.ncols != dim()) throw std::invalid_argument("chain: factor dimension mismatch");
  PrecondChain next = *this;
  next.updates_.push_back(std::move(f));
  next.total_build_seconds += next.updates_.back()->build_seconds;
  return next;
}

void PrecondChain::apply(const Vec& in, Vec& out) const {
  if (empty()) throw std::logic_error("chain: apply on an empty chain");
  base_->multiply(in, out);
  Vec tmp;
  for (const auto& f : updates_) {
    f->q.multiply(out, tmp);
    out.swap(tmp);
  }
}

LinearOp PrecondChain::as_operator() const {
  return [chain = *this](const Vec& in, Vec& out) { chain.apply(in, out); };
}

// proj/src/chain.cpp:140-157
double standard_residual(const Csr& a, const PrecondChain& p) {
  if (a.nrows != a.ncols || a.nrows != p.dim()) throw std::invalid_argument("standard_residual: dimension mismatch");
  const index_t n = a.nrows;
  if (n == 0) return 0.0;
  Vec e(static_cast<size_t>(n), 0.0), pe, ape;
  double sq = 0.0;
  for (index_t j = 0; j < n; ++j) {
    e[size_t(j)] = 1.0;
    p.apply(e, pe);
    a.multiply(pe, ape);
    ape[size_t(j)] -= 1.0;
    for (double v : ape) sq += v * v;
    e[size_t(j)] = 0.0;
  }
  return std::sqrt(sq) / std::sqrt(double(n));
}

}  // namespace oracle
