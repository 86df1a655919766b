// CPU ORACLE — test infrastructure only (see oracle.hpp).
// Restates proj/src/birka.cpp:41-310 for N = 0 (linear tangential IRKA),
// generalised to a mass matrix E (the reference has E = I; with e == nullptr
// this is the reference loop exactly), and proj/src/bench.cpp:159-249 (the
// shift-sweep benchmark) for the first-order pencil sigma E - A.
#include <algorithm>
#include <atomic>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <map>
#include <thread>
#include <cmath>
#include <random>
#include <string>

#include "oracle.hpp"

namespace oracle {

namespace {
std::string shortest(double v) {
  char buf[64];
  for (int p = 1; p <= 17; ++p) {
    std::snprintf(buf, sizeof buf, "%.*g", p, v);
    if (std::strtod(buf, nullptr) == v) break;
  }
  return buf;
}

Dense dense_of(const Csr& m, const Dense& x) { return m.multiply(x); }

struct SidePrecond {
  PrecondChain chain;
  Csr prev_explicit;
  bool degraded = false;
  int shape = 0;  // decoupled mode: unit width of the slot that owns the chain
};
}  // namespace

// proj/src/birka.cpp:41-89
IrkaState irka_default_seed(const LinearSystem& sys, int r, std::uint64_t seed) {
  const index_t n = sys.a.nrows;
  if (r < 1) throw ConfigError("birka: reduced order must be at least 1");
  if (index_t(r) > n) throw ConfigError("birka: reduced order exceeds the system dimension");
  std::mt19937_64 rng(seed);
  std::uniform_real_distribution<double> unit(-1.0, 1.0);
  Vec x(static_cast<size_t>(n));
  for (index_t i = 0; i < n; ++i) x[size_t(i)] = unit(rng);
  double radius = 0.0, xn = 0.0;
  for (double v : x) xn += v * v;
  xn = std::sqrt(xn);
  if (xn > 0.0) {
    for (double& v : x) v /= xn;
    for (int it = 0; it < 20; ++it) {
      const Vec y = sys.a.multiply(x);
      double ny = 0.0;
      for (double v : y) ny += v * v;
      ny = std::sqrt(ny);
      if (ny == 0.0) { radius = 0.0; break; }
      radius = ny;
      for (size_t i = 0; i < y.size(); ++i) x[i] = y[i] / ny;
    }
  }
  if (!(radius > 0.0) || !std::isfinite(radius)) radius = 1.0;
  IrkaState s;
  s.kr = Dense(r, r);
  for (int i = 0; i < r; ++i) {
    const double t = r == 1 ? 1.0 : double(i) / (r - 1);
    s.kr(i, i) = -radius * std::pow(10.0, -3.0 * (1.0 - t));
  }
  s.nr.assign(sys.n_ops.size(), Dense(r, r));  // birka.cpp:76
  s.fr = Dense(r, sys.b.cols);
  s.cr = Dense(r, sys.c.cols);
  for (Dense* m : {&s.fr, &s.cr})
    for (index_t j = 0; j < m->cols; ++j) {
      double nn = 0.0;
      for (int i = 0; i < r; ++i) { (*m)(i, j) = unit(rng); nn += (*m)(i, j) * (*m)(i, j); }
      nn = std::sqrt(nn);
      if (nn > 0.0)
        for (int i = 0; i < r; ++i) (*m)(i, j) /= nn;
    }
  return s;
}

// proj/src/birka.cpp:139-310
std::pair<IrkaState, ReductionReport> irka_reduce(const LinearSystem& sys, const IrkaConfig& cfg,
                                                  PrecondMode mode, const IrkaState* init) {
  const index_t n = sys.a.nrows;
  if (sys.a.ncols != n) throw ConfigError("irka: A must be square");
  if (sys.e && (sys.e->nrows != n || sys.e->ncols != n)) throw ConfigError("irka: E must be n x n");
  if (sys.b.rows != n || sys.b.cols < 1) throw ConfigError("irka: B must have n rows and at least one column");
  if (sys.c.rows != n || sys.c.cols < 1) throw ConfigError("irka: C must have n rows and at least one column");
  if (cfg.max_sweeps < 1) throw ConfigError("birka: max_sweeps must be at least 1");
  if (cfg.max_chain_len < 1) throw ConfigError("birka: max_chain_len must be at least 1");
  for (const Csr& nj : sys.n_ops)
    if (nj.nrows != n || nj.ncols != n) throw ConfigError("bilinear system: every N must be n x n");
  if (!sys.n_ops.empty() && index_t(sys.n_ops.size()) != sys.b.cols)
    throw ConfigError("bilinear system: one N per input is required");
  if (!sys.n_ops.empty() && sys.e) throw ConfigError("irka: couplings with a mass matrix are not supported");
  IrkaState state = init ? *init : irka_default_seed(sys, cfg.r, cfg.seed);
  if (state.nr.size() != sys.n_ops.size()) state.nr.assign(sys.n_ops.size(), Dense(state.kr.rows, state.kr.rows));
  const index_t r = state.kr.rows;
  if (r < 1 || r > n) throw ConfigError("birka: reduced order must be in [1, n]");
  if (state.fr.rows != r || state.fr.cols != sys.b.cols || state.cr.rows != r || state.cr.cols != sys.c.cols)
    throw ConfigError("birka: initial state dimensions do not match the system");

  const Csr at = sys.a.transpose();
  std::vector<Csr> nts;
  for (const Csr& nj : sys.n_ops) nts.push_back(nj.transpose());
  const bool coupled = !sys.n_ops.empty();
  std::shared_ptr<Csr> et;
  if (sys.e) et = std::make_shared<Csr>(sys.e->transpose());

  ReductionReport report;
  report.reduced_order = int(r);
  std::vector<SidePrecond> sides(2);
  std::vector<std::vector<SidePrecond>> unit_sides(2, std::vector<SidePrecond>(static_cast<size_t>(r)));
  std::map<std::pair<int, index_t>, PrecondChain> frozen;  // ReuseFrozen: (side, unit width) -> base
  const bool verbose = std::getenv("ORC_IRKA_VERBOSE") != nullptr;
  const auto t_start = std::chrono::steady_clock::now();
  std::mt19937_64 perturb_rng(cfg.seed ^ 0x9e3779b97f4a7c15ull);
  std::vector<Complex> lambda_prev = sorted_eigenvalues(state.kr);
  bool converged = false;
  int sweeps_done = 0;

  for (int z = 1; z <= cfg.max_sweeps && !converged; ++z) {
    RealSpectrum spec;
    if (!real_spectrum(state.kr, spec)) {  // :167-180
      std::uniform_real_distribution<double> unit(-1.0, 1.0);
      Dense nudged = state.kr;
      const double scale = 1e-8 * std::max(1.0, state.kr.norm());
      for (double& v : nudged.a) v += scale * unit(perturb_rng);
      if (!real_spectrum(nudged, spec))
        throw SolverError("birka: reduced state matrix is not diagonalizable (sweep " + std::to_string(z) +
                          "), even after perturbation");
      state.kr = nudged;
      lambda_prev = sorted_eigenvalues(state.kr);
    }
    // ReuseFrozen builds each (side, width) base at the first unit in the GPU
    // path's unit order, (Re lambda, -|Im lambda|) ascending before mirroring
    // (small_dense.cpp real_spectrum), so both build it at the same shift.
    std::map<index_t, std::pair<double, double>> frozen_key;  // first column -> sort key
    for (index_t cc = 0; cc < r;) {
      const index_t w = (cc + 1 < r && spec.blocks(cc, cc + 1) != 0.0) ? 2 : 1;
      frozen_key[cc] = {spec.blocks(cc, cc), w == 2 ? -std::fabs(spec.blocks(cc, cc + 1)) : 0.0};
      cc += w;
    }
    if (cfg.mirror_unstable) {
      // Standard IRKA safeguard (not in the reference): shifts sigma = -lambda of
      // unstable reduced poles are reflected, Re(lambda) -> -|Re(lambda)|.
      for (index_t i = 0; i < r; ++i)
        if (spec.blocks(i, i) > 0.0) spec.blocks(i, i) = -spec.blocks(i, i);
    }
    const Dense rinv_t = spec.basis_inv.transpose();
    const Dense f2 = matmul(state.fr.transpose(), rinv_t);  // m x r, :182
    const Dense c2 = matmul(state.cr.transpose(), spec.basis);  // q x r, :183
    KronOp ops[2] = {{spec.blocks, &sys.a, sys.e.get(), {}}, {spec.blocks, &at, et.get(), {}}};
    for (size_t j = 0; j < sys.n_ops.size(); ++j) {  // n2[j] = R^T nr[j] R^{-T} (birka.cpp:184-194)
      const Dense n2 = matmul(matmul(spec.basis.transpose(), state.nr[j]), rinv_t);
      ops[0].couplers.push_back({n2, &sys.n_ops[j]});
      ops[1].couplers.push_back({n2.transpose(), &nts[j]});
    }
    const Dense rhs_mats[2] = {matmul(sys.b, f2), matmul(sys.c, c2)};  // :199

    Dense bases[2];
    for (int side = 0; side < 2; ++side) {
      const Dense& rhs = rhs_mats[side];
      double bn = 0.0;
      for (double v : rhs.a) bn += v * v;
      if (bn == 0.0)
        throw SolverError(std::string("birka: zero right-hand side on the ") + (side == 0 ? "trial" : "test") +
                          " side (sweep " + std::to_string(z) + "); input/output maps must be nonzero");
      Dense xsol(n, r);
      // Units: one joint n*r solve (reference), or one solve per real shift /
      // conjugate-pair block (decoupled; same fixed point).
      std::vector<std::pair<index_t, index_t>> units;  // (first column, width)
      if (cfg.decoupled && !coupled) {
        for (index_t c = 0; c < r;) {
          const index_t w = (c + 1 < r && spec.blocks(c, c + 1) != 0.0) ? 2 : 1;
          units.push_back({c, w});
          c += w;
        }
      } else {
        units.push_back({0, r});
      }
      // Pass 1 (unit order, serial): preconditioners exactly as the reference
      // builds them. Pass 2: the solves, which are independent of each other
      // (SPEC.md:151-152), on cfg.unit_threads threads. Pass 3 (unit order):
      // report rows and the first failure, as the serial loop raises it.
      struct UnitJob {
        index_t c0 = 0, width = 0;
        KronOp op;
        LinearOp prec;
        Vec b, x;
        double ubn = 0.0;
        ReportRow row;
        GmresResult res;
      };
      std::vector<UnitJob> jobs(units.size());
      std::vector<size_t> p1order(units.size());
      for (size_t u = 0; u < units.size(); ++u) p1order[u] = u;
      if (mode == PrecondMode::ReuseFrozen)
        std::stable_sort(p1order.begin(), p1order.end(), [&](size_t x, size_t y) {
          return frozen_key[units[x].first] < frozen_key[units[y].first];
        });
      for (size_t uidx : p1order) {
        const auto [c0, width] = units[uidx];
        UnitJob job;
        job.c0 = c0;
        job.width = width;
        ReportRow& row = job.row;
        row.sweep = z;
        row.point = side + 1;
        row.kind = PrecondKind::None;
        Dense lam(width, width);
        for (index_t i = 0; i < width; ++i)
          for (index_t j = 0; j < width; ++j) lam(i, j) = spec.blocks(c0 + i, c0 + j);
        job.op = KronOp{lam, ops[side].a, ops[side].e, {}};
        const KronOp& op = job.op;
        if (coupled) job.op.couplers = ops[side].couplers;  // the joint solve (width = r)
        const bool dec = cfg.decoupled && !coupled;
        SidePrecond& sp = dec ? unit_sides[size_t(side)][size_t(c0)] : sides[size_t(side)];
        if (dec && sp.shape != width) {  // slot changed shape: restart its chain
          sp = SidePrecond{};
          sp.shape = int(width);
        }
        LinearOp prec = identity_operator();
        if (mode == PrecondMode::ReuseFrozen) {
          // GPU extension (irka.cu REUSE_FROZEN): one base per (side, width);
          // a pair unit with only a real base applies it to both halves.
          auto it = frozen.find({side, width});
          if (it == frozen.end() && width == 2 && frozen.count({side, 1})) {
            const PrecondChain base = frozen[{side, 1}];
            prec = [base](const Vec& in, Vec& out) {
              const size_t h = in.size() / 2;
              Vec lo(in.begin(), in.begin() + long(h)), hi(in.begin() + long(h), in.end()), ylo, yhi;
              base.apply(lo, ylo);
              base.apply(hi, yhi);
              out.assign(ylo.begin(), ylo.end());
              out.insert(out.end(), yhi.begin(), yhi.end());
            };
            row.kind = PrecondKind::ReusedSameMatrix;
          } else if (it == frozen.end()) {
            const Csr a_explicit = assemble_explicit(op, cfg.explicit_nnz_cap);
            SpaiResult built = spai_build(a_explicit, cfg.spai);
            row.precond_build_seconds = built.build_seconds;
            PrecondChain ch(std::move(built.p), built.build_seconds);
            frozen[{side, width}] = ch;
            prec = ch.as_operator();
            row.kind = PrecondKind::Fresh;
            if (a_explicit.nrows <= cfg.standard_residual_max_dim) row.standard_residual = standard_residual(a_explicit, ch);
          } else {
            prec = it->second.as_operator();
            row.kind = PrecondKind::ReusedSameMatrix;
          }
        } else {
          bool have_explicit = false;
          Csr a_explicit;
          if (mode != PrecondMode::None && !sp.degraded) {
            try {
              a_explicit = assemble_explicit(op, cfg.explicit_nnz_cap);
              have_explicit = true;
            } catch (const ConfigError& e) {
              sp.degraded = true;
              report.warnings.push_back(std::string(side == 0 ? "trial" : "test") +
                                        " side continues unpreconditioned: " + e.what());
            }
          }
          if (have_explicit) {
            if (mode == PrecondMode::FreshSpai ||
                (mode == PrecondMode::ReuseChain && (sp.chain.empty() || sp.chain.length() + 1 > cfg.max_chain_len))) {
              SpaiResult built = spai_build(a_explicit, cfg.spai);
              sp.chain = PrecondChain(std::move(built.p), built.build_seconds);
              row.kind = PrecondKind::Fresh;
              row.precond_build_seconds = built.build_seconds;
            } else {
              UpdateFactor f = update_build(sp.prev_explicit, a_explicit, cfg.spai);
              row.kind = PrecondKind::Vertical;
              row.precond_build_seconds = f.build_seconds;
              row.min_residual = f.min_residual;
              row.matrix_change = f.matrix_change;
              sp.chain = sp.chain.extended(std::make_shared<const UpdateFactor>(std::move(f)));
            }
            if (mode == PrecondMode::ReuseChain) sp.prev_explicit = a_explicit;
            prec = sp.chain.as_operator();
            if (a_explicit.nrows <= cfg.standard_residual_max_dim)
              row.standard_residual = standard_residual(a_explicit, sp.chain);
          }
        }
        job.prec = prec;
        job.b.assign(rhs.col(c0), rhs.col(c0) + n * width);
        for (double v : job.b) job.ubn += v * v;
        job.x.assign(static_cast<size_t>(n * width), 0.0);
        jobs[uidx] = std::move(job);
      }
      {
        std::atomic<size_t> next{0};
        auto worker = [&] {
          for (size_t i; (i = next.fetch_add(1)) < jobs.size();) {
            UnitJob& j = jobs[i];
            if (!(j.ubn > 0.0)) continue;
            const KronOp* opp = &j.op;
            const LinearOp a_op = [opp](const Vec& in, Vec& out) { opp->apply(in, out); };
            j.res = gmres_right_preconditioned(a_op, j.prec, j.b, cfg.gmres);
          }
        };
        const int nt = std::max(1, std::min<int>(cfg.unit_threads, int(jobs.size())));
        std::vector<std::thread> pool;
        for (int t = 1; t < nt; ++t) pool.emplace_back(worker);
        worker();
        for (auto& th : pool) th.join();
      }
      for (UnitJob& j : jobs) {
        ReportRow& row = j.row;
        if (j.ubn > 0.0) {
          row.solves = 1;
          row.gmres_iterations = j.res.report.iterations;
          row.gmres_seconds = j.res.report.solve_seconds;
          j.x = j.res.x;
        }
        report.rows.push_back(row);
        if (j.ubn > 0.0 && !j.res.report.converged)
          throw SolverError(std::string("birka: gmres did not converge on the ") + (side == 0 ? "trial" : "test") +
                            " side (sweep " + std::to_string(z) + "; relative residual " +
                            shortest(j.res.report.final_residual / std::max(j.res.report.rhs_norm, 1e-300)) +
                            " after " + std::to_string(j.res.report.iterations) + " iterations)");
        std::copy(j.x.begin(), j.x.end(), xsol.col(j.c0));
      }
      bases[side] = thin_q(xsol);  // :278
    }
    const Dense& v = bases[0];
    const Dense& w = bases[1];
    const Dense wt = w.transpose();
    // E_r = W^T E V, A_r = W^T A V; reference (E = I): W^T V and W^T K V.
    const Dense er = sys.e ? matmul(wt, dense_of(*sys.e, v)) : matmul(wt, v);
    const Dense ar = matmul(wt, dense_of(sys.a, v));
    FullPivLU lu(er);
    if (!lu.invertible())
      throw SolverError("birka: projection matrix (test basis^T trial basis) is singular at sweep " + std::to_string(z));
    state.er = er;
    state.ar = ar;
    state.kr = lu.solve(ar);
    for (size_t j = 0; j < sys.n_ops.size(); ++j) state.nr[j] = lu.solve(matmul(wt, dense_of(sys.n_ops[j], v)));
    state.fr = lu.solve(matmul(wt, sys.b));
    state.cr = matmul(v.transpose(), sys.c);
    state.v = v;
    state.w = w;
    sweeps_done = z;
    const std::vector<Complex> lambda_new = sorted_eigenvalues(state.kr);
    double num = 0.0, den = 0.0;
    for (size_t i = 0; i < lambda_new.size(); ++i) {
      const double dr = lambda_new[i].re - lambda_prev[i].re, di = lambda_new[i].im - lambda_prev[i].im;
      num += dr * dr + di * di;
      den += lambda_prev[i].re * lambda_prev[i].re + lambda_prev[i].im * lambda_prev[i].im;
    }
    if (std::sqrt(num) / std::max(std::sqrt(den), 1e-300) < cfg.tol) converged = true;
    if (verbose) {
      long its = 0;
      for (const ReportRow& rw : report.rows)
        if (rw.sweep == z) its += rw.gmres_iterations;
      const double el = std::chrono::duration<double>(std::chrono::steady_clock::now() - t_start).count();
      std::fprintf(stderr, "[oracle irka] sweep %d: shift change %.3e, %ld GMRES iterations, %.1f s\n", z,
                   std::sqrt(num) / std::max(std::sqrt(den), 1e-300), its, el);
      // the sweep's sorted reduced poles at full precision (long offline runs
      // are read back sweep by sweep from this log)
      for (size_t i = 0; i < lambda_new.size(); ++i)
        std::fprintf(stderr, "[oracle irka] sweep %d lambda %zu %.17g %.17g\n", z, i, lambda_new[i].re, lambda_new[i].im);
    }
    lambda_prev = lambda_new;
  }
  state.lambda = lambda_prev;
  state.sweeps = sweeps_done;
  report.converged = converged;
  report.sweeps = sweeps_done;
  if (!converged) report.warnings.push_back("fixed point left unconverged after " + std::to_string(sweeps_done) + " sweeps");
  return {std::move(state), std::move(report)};
}

// proj/src/bench.cpp:159-249, with shifted_operator(s) = s E - A
SweepResult run_spai_bench(const Csr& a, const Csr* e, const Vec& b, const std::vector<double>& points,
                           const SpaiConfig& spai, const GmresConfig& gmres, PrecondMode mode, int max_chain_len,
                           bool keep_solutions) {
  if (points.empty()) throw ConfigError("spai-bench: at least one point is required");
  for (double s : points)
    if (!(s > 0.0) || !std::isfinite(s)) throw ConfigError("spai-bench: points must be positive and finite");
  if (max_chain_len < 1) throw ConfigError("spai-bench: max_chain_len must be at least 1");
  double bn = 0.0;
  for (double v : b) bn += v * v;
  if (bn == 0.0) throw ConfigError("spai-bench: the first input column must be nonzero");
  const Csr ident = e ? Csr() : Csr::identity(a.nrows);
  const Csr* emat = e ? e : &ident;
  SweepResult result;
  PrecondChain chain;
  Csr prev;
  for (size_t i = 0; i < points.size(); ++i) {
    const Csr op = Csr::linear_combination({{points[i], emat}, {-1.0, &a}});
    ReportRow row;
    row.sweep = 1;
    row.point = int(i) + 1;
    LinearOp prec = identity_operator();
    if (mode == PrecondMode::FreshSpai || (mode == PrecondMode::ReuseChain && (i == 0 || chain.length() + 1 > max_chain_len))) {
      SpaiResult built = spai_build(op, spai);
      chain = PrecondChain(std::move(built.p), built.build_seconds);
      row.kind = PrecondKind::Fresh;
      row.precond_build_seconds = built.build_seconds;
      prec = chain.as_operator();
    } else if (mode == PrecondMode::ReuseChain) {
      UpdateFactor f = update_build(prev, op, spai);
      row.kind = PrecondKind::Horizontal;
      row.precond_build_seconds = f.build_seconds;
      row.min_residual = f.min_residual;
      row.matrix_change = f.matrix_change;
      chain = chain.extended(std::make_shared<const UpdateFactor>(std::move(f)));
      prec = chain.as_operator();
    }
    prev = op;
    if (mode != PrecondMode::None && a.nrows <= 5000) row.standard_residual = standard_residual(op, chain);
    GmresResult res = gmres_right_preconditioned(matvec_operator(op), prec, b, gmres);
    row.solves = 1;
    row.gmres_iterations = res.report.iterations;
    row.gmres_seconds = res.report.solve_seconds;
    result.report.rows.push_back(row);
    if (!res.report.converged) {
      ++result.failed_solves;
      result.report.warnings.push_back("solve at point " + std::to_string(i + 1) + " (s = " + shortest(points[i]) +
                                       ") did not converge: relative residual " +
                                       shortest(res.report.final_residual / std::max(res.report.rhs_norm, 1e-300)) +
                                       " after " + std::to_string(res.report.iterations) + " iterations");
    }
    if (keep_solutions) result.x.push_back(std::move(res.x));
  }
  result.report.converged = result.failed_solves == 0;
  result.report.sweeps = 1;
  return result;
}

}  // namespace oracle
