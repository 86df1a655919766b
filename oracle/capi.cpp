// CPU ORACLE — test infrastructure only (see oracle.hpp).
// Flat C entry points so tests/ and bench.py's CPU-baseline leg can drive
// the restatement through ctypes. Status codes match include/mpg.h.
#include <cstdlib>
#include <cstring>
#include <sstream>
#include <string>

#include "oracle.hpp"

using namespace oracle;

namespace {
thread_local std::string g_err;

struct orc_chain { PrecondChain chain; };

template <class F>
int guard(F&& f) {
  try {
    f();
    return 0;
  } catch (const std::invalid_argument& e) {
    g_err = e.what();
    return 1;
  } catch (const ConfigError& e) {
    g_err = e.what();
    return 2;
  } catch (const SolverError& e) {
    g_err = e.what();
    return 3;
  } catch (const IoError& e) {
    g_err = e.what();
    return 7;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 4;
  }
}
}  // namespace

extern "C" {

typedef struct { int pattern_kind, power; double fill_tol; int max_fill_per_col, max_pattern_sweeps, threads; } orc_spai_cfg;
typedef struct { double rel_tol; int max_iter, record_history; } orc_gmres_cfg;
typedef struct {
  int iterations, converged, breakdown, history_len;
  double rhs_norm, final_residual, solve_seconds;
  int reorth_passes;
} orc_gmres_report;
typedef struct {
  int r; double tol; int max_sweeps; int decoupled; unsigned long long seed;
  orc_gmres_cfg gmres; orc_spai_cfg spai; int max_chain_len; long long explicit_nnz_cap, standard_residual_max_dim;
  int mirror_unstable;
  int unit_threads;
} orc_irka_cfg;
typedef struct {
  int sweep, point, kind, solves; long long iterations;
  double build_seconds, gmres_seconds, min_residual, matrix_change, standard_residual;
} orc_report_row;

static SpaiConfig to_spai(const orc_spai_cfg* c) {
  SpaiConfig s;
  if (c) {
    s.pattern_kind = c->pattern_kind; s.power = c->power; s.fill_tol = c->fill_tol;
    s.max_fill_per_col = c->max_fill_per_col; s.max_pattern_sweeps = c->max_pattern_sweeps; s.threads = c->threads;
  }
  return s;
}
static GmresConfig to_gmres(const orc_gmres_cfg* c) {
  GmresConfig g;
  if (c) { g.rel_tol = c->rel_tol; g.max_iter = c->max_iter; g.record_history = c->record_history != 0; }
  return g;
}
static void fill_report(const GmresReport& r, orc_gmres_report* out, double* history) {
  if (!out) return;
  out->iterations = r.iterations; out->converged = r.converged; out->breakdown = r.breakdown;
  out->rhs_norm = r.rhs_norm; out->final_residual = r.final_residual; out->solve_seconds = r.solve_seconds;
  out->history_len = int(r.residual_history.size());
  out->reorth_passes = r.reorth_passes;
  if (history) std::memcpy(history, r.residual_history.data(), r.residual_history.size() * sizeof(double));
}
static int copy_rows(const ReductionReport& rep, orc_report_row* rows, int max_rows, int* nrows) {
  const int n = int(rep.rows.size());
  if (nrows) *nrows = n;
  for (int i = 0; i < n && i < max_rows && rows; ++i) {
    const ReportRow& r = rep.rows[size_t(i)];
    rows[i] = {r.sweep, r.point, int(r.kind), r.solves, (long long)r.gmres_iterations, r.precond_build_seconds,
               r.gmres_seconds, r.min_residual, r.matrix_change, r.standard_residual};
  }
  return 0;
}
static Dense dense_from(const double* p, long long rows, long long cols) {
  Dense d(rows, cols);
  if (p) std::memcpy(d.a.data(), p, size_t(rows * cols) * sizeof(double));
  return d;
}

const char* orc_last_error(void) { return g_err.c_str(); }

int orc_csr_from_csr(long long nr, long long nc, const long long* rp, const long long* ci, const double* v, Csr** out) {
  return guard([&] {
    const size_t nnz = size_t(rp[nr]);
    *out = new Csr(Csr::from_csr(nr, nc, std::vector<index_t>(rp, rp + nr + 1), std::vector<index_t>(ci, ci + nnz),
                                 std::vector<double>(v, v + nnz)));
  });
}
int orc_csr_from_triplets(long long nr, long long nc, long long nnz, const long long* ri, const long long* ci,
                          const double* v, Csr** out) {
  return guard([&] {
    std::vector<Triplet> t(static_cast<size_t>(nnz));
    for (long long k = 0; k < nnz; ++k) t[size_t(k)] = {ri[k], ci[k], v[k]};
    *out = new Csr(Csr::from_triplets(nr, nc, std::move(t)));
  });
}
void orc_csr_free(Csr* h) { delete h; }
void orc_csr_info(const Csr* h, long long* nr, long long* nc, long long* nnz) {
  *nr = h->nrows; *nc = h->ncols; *nnz = h->nnz();
}
void orc_csr_export(const Csr* h, long long* rp, long long* ci, double* v) {
  std::memcpy(rp, h->rowptr.data(), h->rowptr.size() * sizeof(long long));
  std::memcpy(ci, h->colind.data(), h->colind.size() * sizeof(long long));
  std::memcpy(v, h->val.data(), h->val.size() * sizeof(double));
}
int orc_csr_multiply(const Csr* h, long long nx, const double* x, double* y) {
  return guard([&] {
    Vec in(x, x + nx), out;
    h->multiply(in, out);
    std::memcpy(y, out.data(), out.size() * sizeof(double));
  });
}
int orc_csr_multiply_transpose(const Csr* h, long long nx, const double* x, double* y) {
  return guard([&] {
    Vec out = h->multiply_transpose(Vec(x, x + nx));
    std::memcpy(y, out.data(), out.size() * sizeof(double));
  });
}
int orc_csr_transpose(const Csr* h, Csr** out) {
  return guard([&] { *out = new Csr(h->transpose()); });
}
int orc_csr_linear_combination(int nterms, const double* coeffs, const Csr* const* mats, Csr** out) {
  return guard([&] {
    std::vector<std::pair<double, const Csr*>> t;
    for (int i = 0; i < nterms; ++i) t.push_back({coeffs[i], mats[i]});
    *out = new Csr(Csr::linear_combination(t));
  });
}
double orc_csr_frobenius_norm(const Csr* h) { return h->frobenius_norm(); }
int orc_csr_extract(const Csr* h, long long np, const long long* pattern, long long* nrows_out, long long* row_map,
                    double* block, long long cap_rows) {
  return guard([&] {
    auto sub = h->extract_column_submatrix(std::vector<index_t>(pattern, pattern + np));
    *nrows_out = index_t(sub.row_map.size());
    if (row_map && index_t(sub.row_map.size()) <= cap_rows) {
      std::memcpy(row_map, sub.row_map.data(), sub.row_map.size() * sizeof(long long));
      std::memcpy(block, sub.block.a.data(), sub.block.a.size() * sizeof(double));
    }
  });
}

int orc_spai_build(const Csr* a, const orc_spai_cfg* cfg, Csr** p, double* col_res, long long* fallback, double* secs) {
  return guard([&] {
    SpaiResult r = spai_build(*a, to_spai(cfg));
    if (col_res) std::memcpy(col_res, r.column_residuals.data(), r.column_residuals.size() * sizeof(double));
    if (fallback) *fallback = r.fallback_count;
    if (secs) *secs = r.build_seconds;
    *p = new Csr(std::move(r.p));
  });
}
int orc_spai_column_solve(const Csr* a, long long col, long long np, const long long* pattern, double* values,
                          double* residual, int* rank_def) {
  return guard([&] {
    SpaiColumn c = spai_column_solve(*a, col, std::vector<index_t>(pattern, pattern + np));
    std::memcpy(values, c.values.data(), c.values.size() * sizeof(double));
    *residual = c.residual;
    *rank_def = c.rank_deficient;
  });
}
int orc_update_build(const Csr* prev, const Csr* next, const orc_spai_cfg* cfg, Csr** q, double* min_res,
                     double* change, long long* fallback, double* secs) {
  return guard([&] {
    UpdateFactor f = update_build(*prev, *next, to_spai(cfg));
    *min_res = f.min_residual; *change = f.matrix_change;
    if (fallback) *fallback = f.fallback_count;
    if (secs) *secs = f.build_seconds;
    *q = new Csr(std::move(f.q));
  });
}

int orc_chain_create(const Csr* base, orc_chain** out) {
  return guard([&] { *out = new orc_chain{PrecondChain(*base)}; });
}
int orc_chain_extend(const orc_chain* c, const Csr* q, orc_chain** out) {
  return guard([&] {
    auto f = std::make_shared<UpdateFactor>();
    f->q = *q;
    *out = new orc_chain{c->chain.extended(f)};
  });
}
int orc_chain_length(const orc_chain* c) { return c->chain.length(); }
void orc_chain_free(orc_chain* c) { delete c; }
int orc_chain_apply(const orc_chain* c, long long n, const double* x, double* y) {
  return guard([&] {
    Vec out;
    c->chain.apply(Vec(x, x + n), out);
    std::memcpy(y, out.data(), out.size() * sizeof(double));
  });
}
int orc_standard_residual(const Csr* a, const orc_chain* c, double* out) {
  return guard([&] { *out = standard_residual(*a, c->chain); });
}

// GMRES with a plain CSR operator (matvec_operator) or the Kronecker / shifted
// operator -(Lambda (x) E) - (I (x) A); chain null means identity.
int orc_gmres_csr(const Csr* m, const orc_chain* c, long long n, const double* b, double* x, const orc_gmres_cfg* cfg,
                  orc_gmres_report* rep, double* history) {
  return guard([&] {
    GmresResult r = gmres_right_preconditioned(matvec_operator(*m), c ? c->chain.as_operator() : identity_operator(),
                                               Vec(b, b + n), to_gmres(cfg));
    std::memcpy(x, r.x.data(), r.x.size() * sizeof(double));
    fill_report(r.report, rep, history);
  });
}
int orc_gmres_kron(const double* lambda, int r, const Csr* a, const Csr* e, const orc_chain* c, const double* b,
                   double* x, const orc_gmres_cfg* cfg, orc_gmres_report* rep, double* history) {
  return guard([&] {
    KronOp op{dense_from(lambda, r, r), a, e, {}};
    const LinearOp aop = [&op](const Vec& in, Vec& out) { op.apply(in, out); };
    const long long n = a->nrows * r;
    GmresResult res = gmres_right_preconditioned(aop, c ? c->chain.as_operator() : identity_operator(),
                                                 Vec(b, b + n), to_gmres(cfg));
    std::memcpy(x, res.x.data(), res.x.size() * sizeof(double));
    fill_report(res.report, rep, history);
  });
}
int orc_kron_apply(const double* lambda, int r, const Csr* a, const Csr* e, const double* x, double* y) {
  return guard([&] {
    KronOp op{dense_from(lambda, r, r), a, e, {}};
    Vec out;
    op.apply(Vec(x, x + a->nrows * r), out);
    std::memcpy(y, out.data(), out.size() * sizeof(double));
  });
}
int orc_kron_assemble(const double* lambda, int r, const Csr* a, const Csr* e, long long cap, Csr** out) {
  return guard([&] {
    KronOp op{dense_from(lambda, r, r), a, e, {}};
    *out = new Csr(assemble_explicit(op, cap));
  });
}

int orc_real_spectrum(const double* m, int r, double* blocks, double* basis, double* basis_inv) {
  RealSpectrum s;
  if (!real_spectrum(dense_from(m, r, r), s)) return 3;
  std::memcpy(blocks, s.blocks.a.data(), size_t(r * r) * sizeof(double));
  std::memcpy(basis, s.basis.a.data(), size_t(r * r) * sizeof(double));
  std::memcpy(basis_inv, s.basis_inv.a.data(), size_t(r * r) * sizeof(double));
  return 0;
}
int orc_sorted_eigenvalues(const double* m, int r, double* re, double* im) {
  return guard([&] {
    auto l = sorted_eigenvalues(dense_from(m, r, r));
    for (int i = 0; i < r; ++i) { re[i] = l[size_t(i)].re; im[i] = l[size_t(i)].im; }
  });
}
int orc_colpiv_solve(const double* a, long long rows, long long cols, const double* b, double* x, long long* rank) {
  return guard([&] {
    ColPivQR qr(dense_from(a, rows, cols));
    Vec s = qr.solve(Vec(b, b + rows));
    std::memcpy(x, s.data(), s.size() * sizeof(double));
    *rank = qr.rank();
  });
}
int orc_thin_q(const double* a, long long rows, long long cols, double* q) {
  return guard([&] {
    Dense d = thin_q(dense_from(a, rows, cols));
    std::memcpy(q, d.a.data(), d.a.size() * sizeof(double));
  });
}

static LinearSystem make_sys(const Csr* a, const Csr* e, const double* b, int m, const double* c, int q) {
  LinearSystem sys;
  sys.a = *a;
  if (e) sys.e = std::make_shared<Csr>(*e);
  sys.b = dense_from(b, a->nrows, m);
  sys.c = dense_from(c, a->nrows, q);
  return sys;
}

int orc_irka_default_seed(const Csr* a, const Csr* e, const double* b, int m, const double* c, int q, int r,
                          unsigned long long seed, double* kr, double* fr, double* cr) {
  return guard([&] {
    IrkaState s = irka_default_seed(make_sys(a, e, b, m, c, q), r, seed);
    std::memcpy(kr, s.kr.a.data(), s.kr.a.size() * sizeof(double));
    std::memcpy(fr, s.fr.a.data(), s.fr.a.size() * sizeof(double));
    std::memcpy(cr, s.cr.a.data(), s.cr.a.size() * sizeof(double));
  });
}

// Outputs: kr, er, ar (r x r), fr (r x m), cr (r x q), lambda (r), v, w (n x r);
// any output pointer may be null.
int orc_irka_reduce(const Csr* a, const Csr* e, const double* b, int m, const double* c, int q,
                    const orc_irka_cfg* cfg, int mode, const double* init_kr, const double* init_fr,
                    const double* init_cr, double* kr, double* fr, double* cr, double* er, double* ar,
                    double* lam_re, double* lam_im, double* v, double* w, int* sweeps, int* converged,
                    orc_report_row* rows, int max_rows, int* nrows) {
  return guard([&] {
    LinearSystem sys = make_sys(a, e, b, m, c, q);
    IrkaConfig ic;
    ic.r = cfg->r; ic.tol = cfg->tol; ic.max_sweeps = cfg->max_sweeps; ic.seed = cfg->seed;
    ic.gmres = to_gmres(&cfg->gmres); ic.spai = to_spai(&cfg->spai); ic.max_chain_len = cfg->max_chain_len;
    ic.explicit_nnz_cap = cfg->explicit_nnz_cap; ic.standard_residual_max_dim = cfg->standard_residual_max_dim;
    ic.decoupled = cfg->decoupled != 0;
    ic.mirror_unstable = cfg->mirror_unstable != 0;
    ic.unit_threads = std::max(1, cfg->unit_threads);
    IrkaState init;
    const IrkaState* initp = nullptr;
    if (init_kr) {
      init = irka_default_seed(sys, ic.r, ic.seed);  // keeps the fr/cr stream
      init.kr = dense_from(init_kr, ic.r, ic.r);
      if (init_fr) init.fr = dense_from(init_fr, ic.r, m);
      if (init_cr) init.cr = dense_from(init_cr, ic.r, q);
      initp = &init;
    }
    auto [s, rep] = irka_reduce(sys, ic, PrecondMode(mode), initp);
    const size_t rr = size_t(s.kr.rows);
    if (kr) std::memcpy(kr, s.kr.a.data(), rr * rr * sizeof(double));
    if (er) std::memcpy(er, s.er.a.data(), rr * rr * sizeof(double));
    if (ar) std::memcpy(ar, s.ar.a.data(), rr * rr * sizeof(double));
    if (fr) std::memcpy(fr, s.fr.a.data(), s.fr.a.size() * sizeof(double));
    if (cr) std::memcpy(cr, s.cr.a.data(), s.cr.a.size() * sizeof(double));
    for (size_t i = 0; i < s.lambda.size(); ++i) {
      if (lam_re) lam_re[i] = s.lambda[i].re;
      if (lam_im) lam_im[i] = s.lambda[i].im;
    }
    if (v) std::memcpy(v, s.v.a.data(), s.v.a.size() * sizeof(double));
    if (w) std::memcpy(w, s.w.a.data(), s.w.a.size() * sizeof(double));
    *sweeps = s.sweeps;
    *converged = rep.converged;
    copy_rows(rep, rows, max_rows, nrows);
  });
}

int orc_spai_bench(const Csr* a, const Csr* e, const double* b, int npoints, const double* points,
                   const orc_spai_cfg* spai, const orc_gmres_cfg* gmres, int mode, int max_chain_len, double* x_out,
                   orc_report_row* rows, int max_rows, int* nrows, int* failed) {
  return guard([&] {
    SweepResult r = run_spai_bench(*a, e, Vec(b, b + a->nrows), std::vector<double>(points, points + npoints),
                                   to_spai(spai), to_gmres(gmres), PrecondMode(mode), max_chain_len, x_out != nullptr);
    if (x_out)
      for (size_t i = 0; i < r.x.size(); ++i) std::memcpy(x_out + i * size_t(a->nrows), r.x[i].data(), r.x[i].size() * sizeof(double));
    copy_rows(r.report, rows, max_rows, nrows);
    *failed = r.failed_solves;
  });
}

// QB-IHOMM (proj/src/qbihomm.cpp:144-208). Outputs for reduced order r <=
// max_order: basis (n x r), red_d/k/n (r x r), red_h (r x r^2), red_f/c (r).
int orc_qbihomm_reduce(const Csr* d, const Csr* k, const Csr* n_op, const Csr* h, const double* f, const double* c,
                       int npoints, const double* sigmas, int p_moments, int q_moments, const orc_gmres_cfg* gmres,
                       const orc_spai_cfg* spai, int max_chain_len, long long sr_max_dim, int mode, int max_order,
                       int* order, double* basis, double* red_d, double* red_k, double* red_n, double* red_h,
                       double* red_f, double* red_c, orc_report_row* rows, int max_rows, int* nrows) {
  return guard([&] {
    QbSystem sys;
    sys.d = *d; sys.k = *k; sys.n_op = *n_op; sys.h = *h;
    sys.f.assign(f, f + d->nrows);
    sys.c.assign(c, c + d->nrows);
    QbConfig cfg;
    cfg.sigmas.assign(sigmas, sigmas + npoints);
    cfg.p_moments = p_moments; cfg.q_moments = q_moments;
    cfg.gmres = to_gmres(gmres); cfg.spai = to_spai(spai);
    cfg.max_chain_len = max_chain_len; cfg.standard_residual_max_dim = sr_max_dim;
    auto [red, rep] = qbihomm_reduce(sys, cfg, PrecondMode(mode));
    const int r = int(red.d.rows);
    *order = r;
    if (r > max_order) throw std::invalid_argument("qbihomm: reduced order exceeds max_order");
    auto put = [](double* dst, const Dense& m) { if (dst) std::memcpy(dst, m.a.data(), m.a.size() * sizeof(double)); };
    put(basis, red.basis); put(red_d, red.d); put(red_k, red.k); put(red_n, red.n_op); put(red_h, red.h);
    put(red_f, red.f); put(red_c, red.c);
    copy_rows(rep, rows, max_rows, nrows);
  });
}

int orc_kron_compress_quadratic(const Csr* h, const double* u, long long n, long long r, double* out) {
  return guard([&] {
    const Dense m = kron_compress_quadratic(*h, dense_from(u, n, r));
    std::memcpy(out, m.a.data(), m.a.size() * sizeof(double));
  });
}

int orc_mm_read_buffer(const char* data, long long len, const char* origin, Csr** out) {
  return guard([&] {
    std::istringstream in(std::string(data, size_t(len)));
    *out = new Csr(read_matrix_market(in, origin));
  });
}
int orc_mm_read_file(const char* path, Csr** out) {
  return guard([&] { *out = new Csr(read_matrix_market_file(path)); });
}
int orc_mm_write_buffer(const Csr* a, char** out, long long* len) {
  return guard([&] {
    std::ostringstream os;
    write_matrix_market(os, *a);
    const std::string t = os.str();
    *out = static_cast<char*>(std::malloc(t.size() + 1));
    std::memcpy(*out, t.data(), t.size());
    (*out)[t.size()] = 0;
    *len = (long long)t.size();
  });
}
void orc_buffer_free(char* p) { std::free(p); }

int orc_transfer_function_error(const Csr* m, const Csr* d, const Csr* k, const double* f, int n_in, const double* c,
                                int n_out, const double* rm, const double* rd, const double* rk, const double* rf,
                                const double* rc, int r, const double* grid, int ngrid, const orc_gmres_cfg* gmres,
                                const orc_spai_cfg* spai, int mode, int max_chain_len, double* errors) {
  return guard([&] {
    const long long n = m->nrows;
    const auto e = transfer_function_error(*m, *d, *k, dense_from(f, n, n_in), dense_from(c, n, n_out),
                                           dense_from(rm, r, r), dense_from(rd, r, r), dense_from(rk, r, r),
                                           dense_from(rf, r, n_in), dense_from(rc, r, n_out),
                                           std::vector<double>(grid, grid + ngrid), to_gmres(gmres), to_spai(spai),
                                           PrecondMode(mode), max_chain_len);
    std::copy(e.begin(), e.end(), errors);
  });
}

// airga_reduce (proj/src/airga.cpp:136-317). Outputs the reduced pencil
// (order x order, column-major, capacity r_max), F_r (order x n_in), C_r
// (order x n_out), the final points and every sweep's points (sweeps x ell).
typedef struct {
  int r_max; double outer_tol, inner_tol; int max_outer; orc_gmres_cfg gmres; orc_spai_cfg spai; int max_chain_len;
  long long standard_residual_max_dim;
} orc_airga_cfg;

int orc_airga_reduce(const Csr* m, const Csr* d, const Csr* k, const double* f, int n_in, const double* c, int n_out,
                     double alpha, double beta, const double* points, int npoints, const orc_airga_cfg* cfg, int mode,
                     int* order, double* rm, double* rd, double* rk, double* rf, double* rc, double* final_points,
                     double* point_history, int* sweeps, int* converged, orc_report_row* rows, int max_rows,
                     int* nrows) {
  return guard([&] {
    const long long n = m->nrows;
    AirgaConfigO ac;
    ac.expansion_points.assign(points, points + npoints);
    ac.r_max = cfg->r_max; ac.outer_tol = cfg->outer_tol; ac.inner_tol = cfg->inner_tol; ac.max_outer = cfg->max_outer;
    ac.gmres = to_gmres(&cfg->gmres); ac.spai = to_spai(&cfg->spai); ac.max_chain_len = cfg->max_chain_len;
    ac.standard_residual_max_dim = cfg->standard_residual_max_dim;
    const AirgaResult res = airga_reduce(*m, *d, *k, dense_from(f, n, n_in), dense_from(c, n, n_out), alpha, beta, ac,
                                         PrecondMode(mode));
    const AirgaModel& md = res.model;
    *order = int(md.m.rows);
    auto put = [](double* dst, const Dense& x) { if (dst) std::memcpy(dst, x.a.data(), x.a.size() * sizeof(double)); };
    put(rm, md.m); put(rd, md.d); put(rk, md.k); put(rf, md.f); put(rc, md.c);
    if (final_points) std::copy(res.final_points.begin(), res.final_points.end(), final_points);
    if (point_history)
      for (size_t z = 0; z < res.point_history.size(); ++z)
        std::copy(res.point_history[z].begin(), res.point_history[z].end(), point_history + z * size_t(npoints));
    *sweeps = res.report.sweeps;
    *converged = res.report.converged;
    copy_rows(res.report, rows, max_rows, nrows);
  });
}

int orc_update_expansion_points(const double* m, const double* d, const double* k, int r, const double* cur, int npts,
                                double* out) {
  return guard([&] {
    const auto v = update_expansion_points(dense_from(m, r, r), dense_from(d, r, r), dense_from(k, r, r),
                                           std::vector<double>(cur, cur + npts));
    std::copy(v.begin(), v.end(), out);
  });
}

// H2 norm of (A, B, C) (h2.cpp:28-60), infinity when A is not stable.
int orc_h2_norm(const double* a, const double* b, const double* c, int ns, int ni, int no, double* out) {
  return guard([&] {
    StateSpaceO ss{dense_from(a, ns, ns), dense_from(b, ns, ni), dense_from(c, no, ns)};
    *out = h2_norm_o(ss);
  });
}

// BIRKA with couplings N_1..N_m (proj/src/birka.cpp:139-310): the joint n r
// solve per side; outputs kr (r x r), nr (m blocks of r x r), fr, cr, lambda,
// v, w (n x r), any output may be null.
int orc_birka_reduce(const Csr* a, const Csr* const* n_ops, const double* b, int m, const double* c, int q,
                     const orc_irka_cfg* cfg, int mode, double* kr, double* nr, double* fr, double* cr,
                     double* lam_re, double* lam_im, double* v, double* w, int* sweeps, int* converged,
                     orc_report_row* rows, int max_rows, int* nrows) {
  return guard([&] {
    LinearSystem sys = make_sys(a, nullptr, b, m, c, q);
    for (int j = 0; j < m; ++j) sys.n_ops.push_back(*n_ops[j]);
    IrkaConfig ic;
    ic.r = cfg->r; ic.tol = cfg->tol; ic.max_sweeps = cfg->max_sweeps; ic.seed = cfg->seed;
    ic.gmres = to_gmres(&cfg->gmres); ic.spai = to_spai(&cfg->spai); ic.max_chain_len = cfg->max_chain_len;
    ic.explicit_nnz_cap = cfg->explicit_nnz_cap; ic.standard_residual_max_dim = cfg->standard_residual_max_dim;
    ic.decoupled = false;
    auto [st, rep] = irka_reduce(sys, ic, PrecondMode(mode), nullptr);
    const size_t rr = size_t(st.kr.rows);
    if (kr) std::memcpy(kr, st.kr.a.data(), rr * rr * sizeof(double));
    if (nr)
      for (size_t j = 0; j < st.nr.size(); ++j) std::memcpy(nr + j * rr * rr, st.nr[j].a.data(), rr * rr * sizeof(double));
    if (fr) std::memcpy(fr, st.fr.a.data(), st.fr.a.size() * sizeof(double));
    if (cr) std::memcpy(cr, st.cr.a.data(), st.cr.a.size() * sizeof(double));
    for (size_t i = 0; i < st.lambda.size(); ++i) {
      if (lam_re) lam_re[i] = st.lambda[i].re;
      if (lam_im) lam_im[i] = st.lambda[i].im;
    }
    if (v) std::memcpy(v, st.v.a.data(), st.v.a.size() * sizeof(double));
    if (w) std::memcpy(w, st.w.a.data(), st.w.a.size() * sizeof(double));
    *sweeps = st.sweeps;
    *converged = rep.converged;
    copy_rows(rep, rows, max_rows, nrows);
  });
}

// Kronecker operator with couplers (kron.cpp:34-131): apply and explicit assembly.
int orc_kron_coupled(const double* lambda, int r, const Csr* a, int ncp, const double* smalls, const Csr* const* sparses,
                     const double* x, double* y, Csr** explicit_out) {
  return guard([&] {
    KronOp op{dense_from(lambda, r, r), a, nullptr, {}};
    for (int j = 0; j < ncp; ++j) op.couplers.push_back({dense_from(smalls + size_t(j) * r * r, r, r), sparses[j]});
    if (x && y) {
      Vec in(x, x + a->nrows * r), out;
      op.apply(in, out);
      std::copy(out.begin(), out.end(), y);
    }
    if (explicit_out) *explicit_out = new Csr(assemble_explicit(op, (index_t(1) << 40)));
  });
}

}  // extern "C"
