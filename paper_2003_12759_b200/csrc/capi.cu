// extern "C" entry points of libmpg.so (include/mpg.h): thin wrappers that
// translate the reference's exception classes into status codes.
#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <map>
#include <mutex>
#include <string>

#include "host/h2.hpp"
#include "host/mmio.hpp"
#include "irka.hpp"

using namespace mpg;

struct mpg_csr { CsrPtr p; };
struct mpg_op { OpPtr p; };
struct mpg_chain { ChainPtr p; };

namespace {
thread_local std::string g_err;

template <class F>
int guard(F&& f) {
  try {
    f();
    return MPG_OK;
  } catch (const std::invalid_argument& e) {
    g_err = e.what();
    return MPG_ERR_INVALID;
  } catch (const mpg::ConfigError& e) {
    g_err = e.what();
    return MPG_ERR_CONFIG;
  } catch (const mpg::SolverError& e) {
    g_err = e.what();
    return MPG_ERR_SOLVER;
  } catch (const mpg::CudaError& e) {
    g_err = e.what();
    return MPG_ERR_CUDA;
  } catch (const mpg::IoError& e) {
    g_err = e.what();
    return MPG_ERR_IO;
  } catch (const std::bad_alloc&) {
    g_err = "device or host allocation failed";
    return MPG_ERR_NOMEM;
  } catch (const std::exception& e) {
    g_err = e.what();
    return MPG_ERR_LOGIC;
  }
}

SpaiOptions to_spai(const mpg_spai_cfg* c) {
  SpaiOptions o;
  if (c) {
    o.pattern_kind = c->pattern_kind;
    o.power = c->power;
    o.fill_tol = c->fill_tol;
    o.max_fill_per_col = c->max_fill_per_col;
    o.max_pattern_sweeps = c->max_pattern_sweeps;
  }
  return o;
}

GmresOptions to_gmres(const mpg_gmres_cfg* c) {
  GmresOptions o;
  if (c) {
    o.rel_tol = c->rel_tol;
    o.max_iter = c->max_iter;
    o.record_history = c->record_history != 0;
  }
  return o;
}

void fill(const GmresOutcome& o, mpg_gmres_report* r, double* history) {
  if (r) {
    r->iterations = o.iterations;
    r->converged = o.converged;
    r->breakdown = o.breakdown;
    r->history_len = int(o.history.size());
    r->rhs_norm = o.rhs_norm;
    r->final_residual = o.final_residual;
    r->solve_seconds = o.solve_seconds;
    r->reorth_passes = o.reorth_passes;
  }
  if (history && !o.history.empty()) std::memcpy(history, o.history.data(), o.history.size() * sizeof(double));
}

// A plain operator M x wrapped as the shifted family with sigma = 0, ca = +1.
std::mutex g_plain_mu;
OpPtr plain_op(const CsrPtr& m) {
  std::scoped_lock l(g_plain_mu);
  static std::map<const DevCsr*, std::weak_ptr<ShiftedOp>> cache;
  auto it = cache.find(m.get());
  if (it != cache.end())
    if (auto sp = it->second.lock()) return sp;
  if (m->nrows != m->ncols) throw std::invalid_argument("gmres: operator must be square");
  OpPtr op = op_create(m, nullptr);
  cache[m.get()] = op;
  return op;
}
}  // namespace

extern "C" {

const char* mpg_last_error(void) { return g_err.c_str(); }

int mpg_device_count(int* count) {
  return guard([&] {
    if (cudaGetDeviceCount(count) != cudaSuccess) {
      cudaGetLastError();
      *count = 0;
    }
  });
}

int mpg_stream(int device, void** stream) {
  return guard([&] { *stream = ctx(device).stream; });
}

int mpg_synchronize(int device) {
  return guard([&] {
    DeviceGuard g(device);
    MPG_CUDA(cudaStreamSynchronize(ctx(device).stream));
  });
}

long long mpg_launch_count(void) { return g_launches.load(); }

}  // extern "C"

namespace mpg {
void profile_set(bool on);
void profile_reset();
void profile_read(int kind, long long* launches, double* ms, double* bytes);
}  // namespace mpg

extern "C" {

static const char* const kProfNames[PK_COUNT] = {"chain_spmv", "shifted_spmv", "gs_dot", "gs_update_probe",
                                                 "gs_update", "gs_probe", "gs_reorth", "control", "assembly"};

void mpg_profile_enable(int on) {
  mpg::profile_set(on != 0);
  if (on) mpg::profile_reset();
}

int mpg_profile_count(void) { return PK_COUNT; }

int mpg_profile_read(int kind, const char** name, long long* launches, double* ms, double* bytes) {
  if (kind < 0 || kind >= PK_COUNT) return MPG_ERR_INVALID;
  *name = kProfNames[kind];
  mpg::profile_read(kind, launches, ms, bytes);
  return MPG_OK;
}

int mpg_copy(void* dst, const void* src, int64_t bytes) {
  // cudaMemcpy from pageable host memory returns once the data is staged, before the DMA into device memory
  // has completed; the library reads the destination on its own (non-blocking) stream, so wait for the copy.
  return guard([&] {
    MPG_CUDA(cudaMemcpy(dst, src, size_t(bytes), cudaMemcpyDefault));
    MPG_CUDA(cudaDeviceSynchronize());
  });
}

// ---- matrices -------------------------------------------------------------------
int mpg_csr_create(int device, int64_t nrows, int64_t ncols, const int64_t* rowptr, const int64_t* colind,
                   const double* values, mpg_csr** out) {
  return guard([&] { *out = new mpg_csr{csr_from_host(device, nrows, ncols, rowptr, colind, values)}; });
}
void mpg_csr_destroy(mpg_csr* m) { delete m; }
int mpg_csr_info(const mpg_csr* m, int64_t* nr, int64_t* nc, int64_t* nnz) {
  return guard([&] {
    *nr = m->p->nrows;
    *nc = m->p->ncols;
    *nnz = m->p->nnz;
  });
}
int mpg_csr_download(const mpg_csr* m, int64_t* rowptr, int64_t* colind, double* values) {
  return guard([&] {
    const DevCsr& d = *m->p;
    auto& c = ctx(d.device);
    DeviceGuard g(d.device);
    std::vector<int> rp(size_t(d.nrows) + 1), ci(static_cast<size_t>(d.nnz));
    MPG_CUDA(cudaMemcpyAsync(rp.data(), d.rowptr.get(), rp.size() * 4, cudaMemcpyDeviceToHost, c.stream));
    if (d.nnz) {
      MPG_CUDA(cudaMemcpyAsync(ci.data(), d.colind.get(), ci.size() * 4, cudaMemcpyDeviceToHost, c.stream));
      MPG_CUDA(cudaMemcpyAsync(values, d.val.get(), size_t(d.nnz) * 8, cudaMemcpyDefault, c.stream));
    }
    MPG_CUDA(cudaStreamSynchronize(c.stream));
    for (size_t i = 0; i < rp.size(); ++i) rowptr[i] = rp[i];
    for (size_t i = 0; i < ci.size(); ++i) colind[i] = ci[i];
  });
}

static void spmv_any(const DevCsr& m, const double* x, double* y) {
  auto& c = ctx(m.device);
  DeviceGuard g(m.device);
  DBuf<double> dx(m.device, size_t(m.ncols) + 1), dy(m.device, size_t(m.nrows) + 1);
  copy_in(dx.get(), x, size_t(m.ncols), c.stream);
  launch_spmv(m, dx.get(), dy.get(), 1.0, c.stream);
  copy_out(y, dy.get(), size_t(m.nrows), c.stream);
  MPG_CUDA(cudaStreamSynchronize(c.stream));
}

int mpg_csr_multiply(const mpg_csr* m, const double* x, double* y) {
  return guard([&] { spmv_any(*m->p, x, y); });
}
int mpg_csr_multiply_transpose(const mpg_csr* m, const double* x, double* y) {
  return guard([&] { spmv_any(*csr_transpose_cached(m->p), x, y); });
}
int mpg_csr_transpose(const mpg_csr* m, mpg_csr** out) {
  return guard([&] { *out = new mpg_csr{csr_transpose(*m->p)}; });
}
double mpg_csr_frobenius_norm(const mpg_csr* m) {
  double r = 0.0;
  guard([&] {
    const DevCsr& d = *m->p;
    auto& c = ctx(d.device);
    DeviceGuard g(d.device);
    r = std::sqrt(device_norm2(d.device, d.val.get(), d.nnz, c.stream));
  });
  return r;
}

// ---- shifted operator -------------------------------------------------------------
int mpg_op_create(const mpg_csr* a, const mpg_csr* e, mpg_op** out) {
  return guard([&] { *out = new mpg_op{op_create(a->p, e ? e->p : nullptr)}; });
}
void mpg_op_destroy(mpg_op* op) { delete op; }
int64_t mpg_op_dim(const mpg_op* op) { return op->p->n; }
int mpg_op_apply(const mpg_op* op, double sre, double sim, int transpose, const double* x, double* y) {
  return guard([&] {
    const ShiftedOp& o = *op->p;
    auto& c = ctx(o.device);
    DeviceGuard g(o.device);
    const int64_t len = sim != 0.0 ? 2 * o.n : o.n;
    DBuf<double> dx(o.device, size_t(len) + 1), dy(o.device, size_t(len) + 1);
    copy_in(dx.get(), x, size_t(len), c.stream);
    launch_op(o, transpose != 0, sre, sim, -1.0, dx.get(), dy.get(), nullptr, 1.0, c.stream, nullptr);
    copy_out(y, dy.get(), size_t(len), c.stream);
    MPG_CUDA(cudaStreamSynchronize(c.stream));
  });
}
int mpg_op_explicit(const mpg_op* op, double sre, double sim, int transpose, mpg_csr** out) {
  return guard([&] { *out = new mpg_csr{op_explicit(*op->p, sre, sim, transpose != 0)}; });
}

// ---- preconditioner builds ------------------------------------------------------------
int mpg_spai_build(const mpg_csr* a, const mpg_spai_cfg* cfg, mpg_csr** p, double* column_residuals,
                   int64_t* fallback_count, double* build_seconds) {
  return guard([&] {
    SpaiOutcome o = spai_or_update(a->p, nullptr, to_spai(cfg), column_residuals != nullptr);
    if (column_residuals) std::memcpy(column_residuals, o.column_residuals.data(), o.column_residuals.size() * 8);
    if (fallback_count) *fallback_count = o.fallback_count;
    if (build_seconds) *build_seconds = o.build_seconds;
    *p = new mpg_csr{o.p};
  });
}

int mpg_update_build(const mpg_csr* a_prev, const mpg_csr* a_new, const mpg_spai_cfg* cfg, mpg_csr** q,
                     double* min_residual, double* matrix_change, int64_t* fallback_count, double* build_seconds) {
  return guard([&] {
    SpaiOutcome o = spai_or_update(a_new->p, a_prev->p, to_spai(cfg), false);
    if (min_residual) *min_residual = o.min_residual;
    if (matrix_change) *matrix_change = o.matrix_change;
    if (fallback_count) *fallback_count = o.fallback_count;
    if (build_seconds) *build_seconds = o.build_seconds;
    *q = new mpg_csr{o.p};
  });
}

int mpg_spai_column_solve(const mpg_csr* a, int64_t col, int64_t npattern, const int64_t* pattern, double* values,
                          double* residual, int* rank_deficient) {
  // Fixed-pattern solve (spai.cpp:158-173) through the same warp kernel.
  return guard([&] {
    std::vector<double> v;
    bool rd = false;
    spai_column_solve_dev(a->p, col, std::vector<int64_t>(pattern, pattern + std::max<int64_t>(npattern, 0)), v,
                          *residual, rd);
    std::memcpy(values, v.data(), v.size() * 8);
    *rank_deficient = rd;
  });
}

// ---- chains ---------------------------------------------------------------------------------
int mpg_chain_create(const mpg_csr* base, mpg_chain** out) {
  return guard([&] {
    if (base->p->nrows != base->p->ncols) throw std::invalid_argument("chain: base must be square");
    auto c = std::make_shared<Chain>();
    c->factors.push_back(base->p);
    *out = new mpg_chain{c};
  });
}
int mpg_chain_extend(const mpg_chain* chain, const mpg_csr* q, mpg_chain** out) {
  return guard([&] {
    if (!chain || !chain->p) throw std::logic_error("chain: cannot extend an empty chain");
    if (!q) throw std::invalid_argument("chain: null update factor");
    const int64_t d = chain->p->factors[0]->nrows;
    if (q->p->nrows != d || q->p->ncols != d) throw std::invalid_argument("chain: factor dimension mismatch");
    auto c = std::make_shared<Chain>(*chain->p);
    c->factors.push_back(q->p);
    *out = new mpg_chain{c};
  });
}
void mpg_chain_destroy(mpg_chain* chain) { delete chain; }
int mpg_chain_length(const mpg_chain* chain) { return chain->p->length(); }
const void* mpg_chain_factor_id(const mpg_chain* chain, int i) {
  if (i < 0 || i >= int(chain->p->factors.size())) return nullptr;
  return chain->p->factors[size_t(i)].get();
}
int mpg_chain_apply(const mpg_chain* chain, const double* x, double* y) {
  return guard([&] {
    const Chain& ch = *chain->p;
    const DevCsr& base = *ch.factors[0];
    auto& c = ctx(base.device);
    DeviceGuard g(base.device);
    const size_t n = size_t(base.nrows);
    DBuf<double> dx(base.device, n + 1), dy(base.device, n + 1), tmp(base.device, n + 1);
    copy_in(dx.get(), x, n, c.stream);
    launch_chain(ch, dx.get(), dy.get(), tmp.get(), c.stream);
    copy_out(y, dy.get(), n, c.stream);
    MPG_CUDA(cudaStreamSynchronize(c.stream));
  });
}

}  // extern "C"

namespace mpg {
double std_residual_public(const CsrPtr& m, const ChainPtr& ch);
void project_public(const ShiftedOp& op, const double* v_any, const double* w_any, int r, host::Mat& er, host::Mat& ar);
}

extern "C" {

int mpg_standard_residual(const mpg_csr* a, const mpg_chain* chain, double* out) {
  return guard([&] {
    if (a->p->nrows != a->p->ncols || a->p->nrows != chain->p->factors[0]->nrows)
      throw std::invalid_argument("standard_residual: dimension mismatch");
    *out = std_residual_public(a->p, chain->p);
  });
}

// ---- GMRES ------------------------------------------------------------------------------------
int mpg_gmres_csr(const mpg_csr* m, const mpg_chain* chain, const double* b, double* x, const mpg_gmres_cfg* cfg,
                  mpg_gmres_report* report, double* history) {
  return guard([&] {
    OpPtr op = plain_op(m->p);
    std::vector<SolveSpec> specs(1);
    specs[0].ca = 1.0;
    specs[0].chain = chain ? chain->p : nullptr;
    specs[0].b = b;
    specs[0].x = x;
    auto out = gmres_batch(*op, specs, to_gmres(cfg));
    fill(out[0], report, history);
  });
}

int mpg_gmres_shifted(const mpg_op* op, double sre, double sim, int transpose, const mpg_chain* chain, const double* b,
                      double* x, const mpg_gmres_cfg* cfg, mpg_gmres_report* report, double* history) {
  return guard([&] {
    std::vector<SolveSpec> specs(1);
    specs[0].sre = sre;
    specs[0].sim = sim;
    specs[0].transpose = transpose != 0;
    specs[0].chain = chain ? chain->p : nullptr;
    specs[0].b = b;
    specs[0].x = x;
    auto out = gmres_batch(*op->p, specs, to_gmres(cfg));
    fill(out[0], report, history);
  });
}

int mpg_gmres_batch(const mpg_op* op, int nsolves, const double* sre, const double* sim, const int* transpose,
                    const mpg_chain* const* chains, const double* const* b, double* const* x,
                    const mpg_gmres_cfg* cfg, mpg_gmres_report* reports) {
  return guard([&] {
    std::vector<SolveSpec> specs(size_t(std::max(nsolves, 0)));
    for (int i = 0; i < nsolves; ++i) {
      specs[size_t(i)].sre = sre[i];
      specs[size_t(i)].sim = sim ? sim[i] : 0.0;
      specs[size_t(i)].transpose = transpose ? transpose[i] != 0 : false;
      specs[size_t(i)].chain = chains && chains[i] ? chains[i]->p : nullptr;
      specs[size_t(i)].b = b[i];
      specs[size_t(i)].x = x[i];
    }
    auto out = gmres_batch(*op->p, specs, to_gmres(cfg));
    for (int i = 0; i < nsolves; ++i) fill(out[size_t(i)], reports ? reports + i : nullptr, nullptr);
  });
}

// ---- IRKA / sweep -------------------------------------------------------------------------------
static IrkaSettings to_irka(const mpg_irka_cfg* c, int mode, const double* init_shifts) {
  IrkaSettings s;
  s.r = c->r;
  s.tol = c->tol;
  s.max_sweeps = c->max_sweeps;
  s.seed = c->seed;
  s.gmres = to_gmres(&c->gmres);
  s.spai = to_spai(&c->spai);
  s.max_chain_len = c->max_chain_len;
  s.standard_residual_max_dim = c->standard_residual_max_dim;
  s.mode = mode;
  s.mirror_unstable = c->mirror_unstable != 0;
  if (init_shifts) s.init_shifts.assign(init_shifts, init_shifts + c->r);
  return s;
}

static void copy_rows(const std::vector<mpg_report_row>& rows, mpg_report_row* out, int max_rows, int* nrows) {
  if (nrows) *nrows = int(rows.size());
  for (size_t i = 0; out && i < rows.size() && int(i) < max_rows; ++i) out[i] = rows[i];
}

int mpg_irka_reduce(const mpg_op* op, const double* b, int m, const double* c, int q, const mpg_irka_cfg* cfg,
                    int mode, const double* init_shifts, double* kr, double* fr, double* cr, double* er, double* ar,
                    double* lam_re, double* lam_im, double* v, double* w, int* sweeps, int* converged,
                    mpg_report_row* rows, int max_rows, int* nrows) {
  return guard([&] {
    IrkaSettings s = to_irka(cfg, mode, init_shifts);
    s.want_vw = v || w;
    IrkaResult r = irka_run(*op->p, b, m, c, q, s, 0, 1, nullptr, nullptr);
    if (kr) std::memcpy(kr, r.kr.a.data(), r.kr.a.size() * 8);
    if (fr) std::memcpy(fr, r.fr.a.data(), r.fr.a.size() * 8);
    if (cr) std::memcpy(cr, r.cr.a.data(), r.cr.a.size() * 8);
    if (er) std::memcpy(er, r.er.a.data(), r.er.a.size() * 8);
    if (ar) std::memcpy(ar, r.ar.a.data(), r.ar.a.size() * 8);
    for (size_t i = 0; i < r.lambda.size(); ++i) {
      if (lam_re) lam_re[i] = r.lambda[i].re;
      if (lam_im) lam_im[i] = r.lambda[i].im;
    }
    if (v) std::memcpy(v, r.v.data(), r.v.size() * 8);
    if (w) std::memcpy(w, r.w.data(), r.w.size() * 8);
    if (sweeps) *sweeps = r.sweeps;
    if (converged) *converged = r.converged;
    copy_rows(r.rows, rows, max_rows, nrows);
  });
}

int mpg_irka_reduce_from(const mpg_op* op, const double* b, int m, const double* c, int q, const mpg_irka_cfg* cfg,
                         int mode, const double* init_kr, const double* init_fr, const double* init_cr, double* kr,
                         double* fr, double* cr, double* er, double* ar, double* lam_re, double* lam_im, int* sweeps,
                         int* converged, mpg_report_row* rows, int max_rows, int* nrows) {
  return guard([&] {
    if (!cfg || cfg->r < 1) throw ConfigError("birka: reduced order must be at least 1");
    IrkaSettings s = to_irka(cfg, mode, nullptr);
    const size_t r = size_t(cfg->r);
    if (init_kr) s.init_kr.assign(init_kr, init_kr + r * r);
    if (init_fr) s.init_fr.assign(init_fr, init_fr + r * size_t(std::max(m, 0)));
    if (init_cr) s.init_cr.assign(init_cr, init_cr + r * size_t(std::max(q, 0)));
    IrkaResult res = irka_run(*op->p, b, m, c, q, s, 0, 1, nullptr, nullptr);
    if (kr) std::memcpy(kr, res.kr.a.data(), res.kr.a.size() * 8);
    if (fr) std::memcpy(fr, res.fr.a.data(), res.fr.a.size() * 8);
    if (cr) std::memcpy(cr, res.cr.a.data(), res.cr.a.size() * 8);
    if (er) std::memcpy(er, res.er.a.data(), res.er.a.size() * 8);
    if (ar) std::memcpy(ar, res.ar.a.data(), res.ar.a.size() * 8);
    for (size_t i = 0; i < res.lambda.size(); ++i) {
      if (lam_re) lam_re[i] = res.lambda[i].re;
      if (lam_im) lam_im[i] = res.lambda[i].im;
    }
    if (sweeps) *sweeps = res.sweeps;
    if (converged) *converged = res.converged;
    copy_rows(res.rows, rows, max_rows, nrows);
  });
}

static int put_buffer(const std::string& text, char** out, int64_t* len);

int mpg_birka_reduce(const mpg_csr* k, const mpg_csr* const* n_ops, const double* b, int m, const double* c, int q,
                     const mpg_irka_cfg* cfg, int mode, double* kr, double* nr, double* fr, double* cr,
                     double* lam_re, double* lam_im, double* v, double* w, int* sweeps, int* converged,
                     mpg_report_row* rows, int max_rows, int* nrows, char** warnings) {
  return guard([&] {
    if (!k || (m > 0 && !n_ops)) throw ConfigError("birka: null operator");
    std::vector<CsrPtr> ns;
    for (int j = 0; j < m; ++j) {
      if (!n_ops[j]) throw ConfigError("birka: null coupling matrix");
      ns.push_back(n_ops[j]->p);
    }
    IrkaSettings s = to_irka(cfg, mode, nullptr);
    BirkaOutcome o = birka_coupled_run(k->p, ns, b, m, c, q, s, cfg->explicit_nnz_cap);
    if (kr) std::memcpy(kr, o.kr.a.data(), o.kr.a.size() * 8);
    for (size_t j = 0; nr && j < o.nr.size(); ++j)
      std::memcpy(nr + j * o.nr[j].a.size(), o.nr[j].a.data(), o.nr[j].a.size() * 8);
    if (fr) std::memcpy(fr, o.fr.a.data(), o.fr.a.size() * 8);
    if (cr) std::memcpy(cr, o.cr.a.data(), o.cr.a.size() * 8);
    for (size_t i = 0; i < o.lambda.size(); ++i) {
      if (lam_re) lam_re[i] = o.lambda[i].re;
      if (lam_im) lam_im[i] = o.lambda[i].im;
    }
    if (v) std::memcpy(v, o.v.data(), o.v.size() * 8);
    if (w) std::memcpy(w, o.w.data(), o.w.size() * 8);
    if (sweeps) *sweeps = o.sweeps;
    if (converged) *converged = o.converged;
    copy_rows(o.rows, rows, max_rows, nrows);
    if (warnings) {
      std::string t;
      for (const auto& wn : o.warnings) t += wn + "\n";
      int64_t len = 0;
      put_buffer(t, warnings, &len);
    }
  });
}

int mpg_irka_reduce_sharded(const mpg_op* op, const double* b, int m, const double* c, int q,
                            const mpg_irka_cfg* cfg, int mode, const double* init_shifts, int rank, int world,
                            mpg_allgather_fn allgather, void* actx, double* kr, double* fr, double* cr,
                            double* lam_re, double* lam_im, int* sweeps, int* converged, mpg_report_row* rows,
                            int max_rows, int* nrows) {
  return guard([&] {
    IrkaSettings s = to_irka(cfg, mode, init_shifts);
    IrkaResult r = irka_run(*op->p, b, m, c, q, s, rank, world, allgather, actx);
    if (kr) std::memcpy(kr, r.kr.a.data(), r.kr.a.size() * 8);
    if (fr) std::memcpy(fr, r.fr.a.data(), r.fr.a.size() * 8);
    if (cr) std::memcpy(cr, r.cr.a.data(), r.cr.a.size() * 8);
    for (size_t i = 0; i < r.lambda.size(); ++i) {
      if (lam_re) lam_re[i] = r.lambda[i].re;
      if (lam_im) lam_im[i] = r.lambda[i].im;
    }
    if (sweeps) *sweeps = r.sweeps;
    if (converged) *converged = r.converged;
    copy_rows(r.rows, rows, max_rows, nrows);
  });
}

int mpg_spai_bench(const mpg_op* op, const double* b, int npoints, const double* points, const mpg_spai_cfg* spai,
                   const mpg_gmres_cfg* gmres, int mode, int max_chain_len, double* x_out, mpg_report_row* rows,
                   int max_rows, int* nrows, int* failed) {
  return guard([&] {
    SweepOutcome o = sweep_run(*op->p, b, std::vector<double>(points, points + std::max(npoints, 0)), to_spai(spai),
                               to_gmres(gmres), mode, max_chain_len, x_out);
    copy_rows(o.rows, rows, max_rows, nrows);
    if (failed) *failed = o.failed;
  });
}

int mpg_qbihomm_reduce(const mpg_op* op, const mpg_csr* n_op, int64_t h_nnz, const int64_t* h_row,
                       const int64_t* h_col, const double* h_val, const double* f, const double* c, int npoints,
                       const double* sigmas, const mpg_qb_cfg* cfg, int mode, int max_order, int* order,
                       double* basis, double* red_d, double* red_k, double* red_n, double* red_h, double* red_f,
                       double* red_c, mpg_report_row* rows, int max_rows, int* nrows) {
  return guard([&] {
    if (!op || !n_op || !cfg || !f || !c || (npoints > 0 && !sigmas) || h_nnz < 0 || (h_nnz > 0 && !(h_row && h_col && h_val)))
      throw std::invalid_argument("qbihomm: null argument");
    const ShiftedOp& o = *op->p;
    const int64_t n = o.n;
    if (n_op->p->device != o.device) throw std::invalid_argument("qbihomm: N on a different device");
    // H: sorted by row, duplicates summed (SparseMatrix::from_triplets, sparse.cpp:80-115)
    struct E { int64_t r, col; double v; };
    std::vector<E> t(static_cast<size_t>(h_nnz));
    for (int64_t i = 0; i < h_nnz; ++i) {
      if (h_row[i] < 0 || h_row[i] >= n || h_col[i] < 0 || h_col[i] >= n * n)
        throw std::invalid_argument("qbihomm: H entry out of range (H is n x n^2)");
      t[size_t(i)] = {h_row[i], h_col[i], h_val[i]};
    }
    std::stable_sort(t.begin(), t.end(), [](const E& a, const E& b) { return a.r != b.r ? a.r < b.r : a.col < b.col; });
    std::vector<int> rp(size_t(n) + 1, 0), bc, cc;
    std::vector<double> hv;
    for (size_t p = 0; p < t.size();) {
      const int64_t r = t[p].r, col = t[p].col;
      double v = 0.0;
      while (p < t.size() && t[p].r == r && t[p].col == col) v += t[p++].v;
      bc.push_back(int(col / n));
      cc.push_back(int(col % n));
      hv.push_back(v);
      ++rp[size_t(r) + 1];
    }
    for (int64_t i = 0; i < n; ++i) rp[size_t(i) + 1] += rp[size_t(i)];
    DeviceGuard g(o.device);
    cudaStream_t s = ctx(o.device).stream;
    QbH h;
    h.n = n;
    h.nnz = int64_t(hv.size());
    h.rowptr = DBuf<int>(o.device, rp.size());
    h.bcol = DBuf<int>(o.device, std::max<size_t>(1, bc.size()));
    h.ccol = DBuf<int>(o.device, std::max<size_t>(1, cc.size()));
    h.val = DBuf<double>(o.device, std::max<size_t>(1, hv.size()));
    MPG_CUDA(cudaMemcpyAsync(h.rowptr.get(), rp.data(), rp.size() * sizeof(int), cudaMemcpyHostToDevice, s));
    if (!hv.empty()) {
      MPG_CUDA(cudaMemcpyAsync(h.bcol.get(), bc.data(), bc.size() * sizeof(int), cudaMemcpyHostToDevice, s));
      MPG_CUDA(cudaMemcpyAsync(h.ccol.get(), cc.data(), cc.size() * sizeof(int), cudaMemcpyHostToDevice, s));
      MPG_CUDA(cudaMemcpyAsync(h.val.get(), hv.data(), hv.size() * sizeof(double), cudaMemcpyHostToDevice, s));
    }
    QbSettings qs;
    qs.sigmas.assign(sigmas, sigmas + std::max(npoints, 0));
    qs.p_moments = cfg->p_moments;
    qs.q_moments = cfg->q_moments;
    qs.gmres = to_gmres(&cfg->gmres);
    qs.spai = to_spai(&cfg->spai);
    qs.max_chain_len = cfg->max_chain_len;
    qs.standard_residual_max_dim = cfg->standard_residual_max_dim;
    qs.mode = mode;
    QbOutcome r = qbihomm_run(o, *n_op->p, h, f, c, qs);
    if (order) *order = r.r;
    if (r.r > max_order) throw std::invalid_argument("qbihomm: reduced order exceeds max_order");
    auto put = [](double* dst, const host::Mat& m) { if (dst) std::memcpy(dst, m.a.data(), m.a.size() * sizeof(double)); };
    put(red_d, r.d); put(red_k, r.k); put(red_n, r.n_op); put(red_h, r.h); put(red_f, r.f); put(red_c, r.c);
    if (basis) {
      copy_out(basis, r.basis.get(), size_t(n) * size_t(r.r), s);
      MPG_CUDA(cudaStreamSynchronize(s));
    }
    copy_rows(r.rows, rows, max_rows, nrows);
  });
}

double mpg_shard_cost(int width, int last_iterations) { return shard_cost(width, last_iterations); }

int mpg_shard_plan(int nunits, const double* cost, const int* fixed, int world, int* owner) {
  return guard([&] {
    if (nunits < 0 || (nunits > 0 && (!cost || !owner))) throw std::invalid_argument("shard_plan: null argument");
    std::vector<double> c(cost, cost + nunits);
    std::vector<int> f = fixed ? std::vector<int>(fixed, fixed + nunits) : std::vector<int>(size_t(nunits), -1);
    const std::vector<int> o = shard_plan(c, f, world);
    std::copy(o.begin(), o.end(), owner);
  });
}

// ---- native NCCL exchange (comm.cu) -----------------------------------------
int mpg_comm_unique_id(char* id, int len) {
  return guard([&] {
    if (!id) throw std::invalid_argument("comm: null id buffer");
    comm_unique_id(id, len);
  });
}

int mpg_comm_create(int device, int rank, int world, const char* id, mpg_comm** out) {
  return guard([&] {
    if (!id || !out) throw std::invalid_argument("comm: null argument");
    *out = comm_create(device, rank, world, id);
  });
}

int mpg_comm_destroy(mpg_comm* comm) {
  return guard([&] { comm_destroy(comm); });
}

int mpg_comm_allgather(void* comm, const void* send, void* recv, int64_t bytes_per_rank) {
  return comm_allgather(static_cast<mpg_comm*>(comm), send, recv, bytes_per_rank);
}

int mpg_comm_stats(const mpg_comm* comm, long long* calls, double* bytes) {
  return guard([&] { comm_stats(comm, calls, bytes); });
}

int mpg_nccl_version(int* version) {
  return guard([&] {
    if (!version) throw std::invalid_argument("comm: null argument");
    *version = nccl_version();
  });
}

// ---- Matrix Market IO and the report CSV (host side) -------------------------
static mpg_host_csr* to_host_csr(mmio::Csr&& c) {
  auto* m = new mpg_host_csr;
  m->nrows = c.nrows;
  m->ncols = c.ncols;
  m->nnz = c.nnz;
  m->rowptr = c.rowptr.release();
  m->colind = c.colind ? c.colind.release() : new int64_t[1];
  m->val = c.val ? c.val.release() : new double[1];
  return m;
}

void mpg_host_csr_free(mpg_host_csr* m) {
  if (!m) return;
  delete[] m->rowptr;
  delete[] m->colind;
  delete[] m->val;
  delete m;
}

// SparseMatrix::from_triplets (sparse.cpp:80-115): rows by a stable counting
// sort, columns by a stable sort within each row, duplicates summed in input
// order (the reference's std::sort leaves that order unspecified).
int mpg_host_csr_from_triplets(int64_t nr, int64_t nc, int64_t nnz, const int64_t* ri, const int64_t* ci,
                               const double* v, mpg_host_csr** out) {
  return guard([&] {
    if (nr < 0 || nc < 0 || nnz < 0 || !out || (nnz > 0 && (!ri || !ci || !v)))
      throw std::invalid_argument("sparse: negative dimension or null triplets");
    for (int64_t k = 0; k < nnz; ++k)
      if (ri[k] < 0 || ri[k] >= nr || ci[k] < 0 || ci[k] >= nc)
        throw std::invalid_argument("sparse: triplet index out of range");
    std::vector<int64_t> start(size_t(nr) + 1, 0);
    std::vector<int64_t> order(static_cast<size_t>(nnz));
    for (int64_t k = 0; k < nnz; ++k) ++start[size_t(ri[k]) + 1];
    for (int64_t i = 0; i < nr; ++i) start[size_t(i) + 1] += start[size_t(i)];
    {
      std::vector<int64_t> fill(start.begin(), start.end() - 1);
      for (int64_t k = 0; k < nnz; ++k) order[size_t(fill[size_t(ri[k])]++)] = k;
    }
    mmio::Csr c;
    c.nrows = nr;
    c.ncols = nc;
    c.rowptr.reset(new int64_t[size_t(nr) + 1]);
    std::vector<int64_t> cols;
    std::vector<double> vals;
    cols.reserve(size_t(nnz));
    vals.reserve(size_t(nnz));
    c.rowptr[0] = 0;
    for (int64_t i = 0; i < nr; ++i) {
      auto b = order.begin() + start[size_t(i)], e = order.begin() + start[size_t(i) + 1];
      std::stable_sort(b, e, [&](int64_t x, int64_t y) { return ci[x] < ci[y]; });
      for (auto p = b; p != e;) {
        const int64_t col = ci[*p];
        double sum = 0.0;
        for (; p != e && ci[*p] == col; ++p) sum += v[*p];
        cols.push_back(col);
        vals.push_back(sum);
      }
      c.rowptr[size_t(i) + 1] = int64_t(cols.size());
    }
    c.nnz = int64_t(cols.size());
    c.colind.reset(new int64_t[std::max<size_t>(1, cols.size())]);
    c.val.reset(new double[std::max<size_t>(1, vals.size())]);
    std::copy(cols.begin(), cols.end(), c.colind.get());
    std::copy(vals.begin(), vals.end(), c.val.get());
    *out = to_host_csr(std::move(c));
  });
}

static mmio::Csr from_host_csr(const mpg_host_csr* a) {
  if (!a || a->nrows < 0 || a->ncols < 0 || (a->nrows > 0 && !a->rowptr)) throw std::invalid_argument("mmio: bad matrix");
  mmio::Csr c;
  c.nrows = a->nrows;
  c.ncols = a->ncols;
  c.nnz = a->rowptr[a->nrows];
  c.rowptr.reset(new int64_t[size_t(a->nrows) + 1]);
  std::copy(a->rowptr, a->rowptr + a->nrows + 1, c.rowptr.get());
  c.colind.reset(new int64_t[size_t(std::max<int64_t>(1, c.nnz))]);
  c.val.reset(new double[size_t(std::max<int64_t>(1, c.nnz))]);
  std::copy(a->colind, a->colind + c.nnz, c.colind.get());
  std::copy(a->val, a->val + c.nnz, c.val.get());
  return c;
}

static int put_buffer(const std::string& text, char** out, int64_t* len) {
  *out = static_cast<char*>(std::malloc(text.size() + 1));
  if (!*out) throw std::bad_alloc();
  std::memcpy(*out, text.data(), text.size());
  (*out)[text.size()] = '\0';
  *len = int64_t(text.size());
  return 0;
}

int mpg_mm_read_file(const char* path, int threads, mpg_host_csr** out) {
  return guard([&] {
    if (!path || !out) throw std::invalid_argument("mmio: null argument");
    *out = to_host_csr(mmio::read_file(path, threads));
  });
}

int mpg_mm_read_buffer(const char* data, int64_t len, const char* origin, int threads, mpg_host_csr** out) {
  return guard([&] {
    if ((!data && len > 0) || len < 0 || !out) throw std::invalid_argument("mmio: null argument");
    *out = to_host_csr(mmio::read(data, size_t(len), origin ? origin : "<stream>", threads));
  });
}

int mpg_mm_write_file(const char* path, const mpg_host_csr* a, int threads) {
  return guard([&] {
    if (!path) throw std::invalid_argument("mmio: null argument");
    mmio::write_file(path, mmio::write(from_host_csr(a), threads));
  });
}

int mpg_mm_write_buffer(const mpg_host_csr* a, int threads, char** out, int64_t* len) {
  return guard([&] {
    if (!out || !len) throw std::invalid_argument("mmio: null argument");
    put_buffer(mmio::write(from_host_csr(a), threads), out, len);
  });
}

int mpg_mm_write_dense_buffer(int64_t rows, int64_t cols, const double* colmajor, char** out, int64_t* len) {
  return guard([&] {
    if (rows < 0 || cols < 0 || (rows * cols > 0 && !colmajor) || !out || !len)
      throw std::invalid_argument("mmio: bad dense block");
    put_buffer(mmio::write_dense(rows, cols, colmajor), out, len);
  });
}

int mpg_report_csv(const mpg_report_row* rows, int nrows, char** out, int64_t* len) {
  return guard([&] {
    if ((nrows > 0 && !rows) || !out || !len) throw std::invalid_argument("report: null argument");
    put_buffer(mmio::report_csv(rows, nrows), out, len);
  });
}

void mpg_buffer_free(char* p) { std::free(p); }

int mpg_transfer_function_error(const mpg_csr* m, const mpg_csr* d, const mpg_csr* k, const double* f, int n_in,
                                const double* c, int n_out, const double* red_m, const double* red_d,
                                const double* red_k, const double* red_f, const double* red_c, int r,
                                const double* grid, int ngrid, const mpg_gmres_cfg* gmres, const mpg_spai_cfg* spai,
                                int mode, int max_chain_len, double* errors, long long* total_iterations) {
  return guard([&] {
    if (!m || !d || !k || !f || !c || !red_m || !red_d || !red_k || !red_f || !red_c || (ngrid > 0 && (!grid || !errors)) ||
        r < 1)
      throw std::invalid_argument("transfer_function_error: null argument");
    auto mat = [](const double* p, int rows, int cols) {
      host::Mat x(rows, cols);
      std::memcpy(x.a.data(), p, x.a.size() * sizeof(double));
      return x;
    };
    TfSettings ts;
    ts.gmres = to_gmres(gmres);
    ts.spai = to_spai(spai);
    ts.mode = mode;
    ts.max_chain_len = max_chain_len;
    const auto e = tf_error_run(m->p, d->p, k->p, f, n_in, c, n_out, mat(red_m, r, r), mat(red_d, r, r),
                                mat(red_k, r, r), mat(red_f, r, n_in), mat(red_c, r, n_out),
                                std::vector<double>(grid, grid + std::max(ngrid, 0)), ts, total_iterations);
    std::copy(e.begin(), e.end(), errors);
  });
}

int mpg_project(const mpg_op* op, const double* v, const double* w, int r, double* er, double* ar) {
  return guard([&] {
    if (!op || !v || !w) throw std::invalid_argument("project: null argument");
    host::Mat e, a;
    project_public(*op->p, v, w, r, e, a);
    if (er) std::memcpy(er, e.a.data(), e.a.size() * sizeof(double));
    if (ar) std::memcpy(ar, a.a.data(), a.a.size() * sizeof(double));
  });
}

int mpg_airga_reduce(const mpg_csr* m, const mpg_csr* d, const mpg_csr* k, const double* f, int n_in, const double* c,
                     int n_out, double alpha, double beta, const double* points, int npoints,
                     const mpg_airga_cfg* cfg, int mode, int* order, double* red_m, double* red_d, double* red_k,
                     double* red_f, double* red_c, double* basis, double* final_points, int* sweeps, int* converged,
                     mpg_report_row* rows, int max_rows, int* nrows, char** warnings) {
  return guard([&] {
    if (!m || !d || !k || !f || !c || !cfg || (npoints > 0 && !points)) throw std::invalid_argument("airga: null argument");
    AirgaSettings as;
    as.points.assign(points, points + std::max(npoints, 0));
    as.r_max = cfg->r_max;
    as.outer_tol = cfg->outer_tol;
    as.inner_tol = cfg->inner_tol;
    as.max_outer = cfg->max_outer;
    as.gmres = to_gmres(&cfg->gmres);
    as.spai = to_spai(&cfg->spai);
    as.max_chain_len = cfg->max_chain_len;
    as.standard_residual_max_dim = cfg->standard_residual_max_dim;
    as.mode = mode;
    as.alpha = alpha;
    as.beta = beta;
    AirgaOutcome o = airga_run(m->p, d->p, k->p, f, n_in, c, n_out, as);
    if (order) *order = o.r;
    auto put = [](double* dst, const host::Mat& x) { if (dst && !x.a.empty()) std::memcpy(dst, x.a.data(), x.a.size() * sizeof(double)); };
    put(red_m, o.m); put(red_d, o.d); put(red_k, o.k); put(red_f, o.f); put(red_c, o.c);
    if (basis && o.r > 0) {
      copy_out(basis, o.basis.get(), size_t(m->p->nrows) * size_t(o.r), ctx(m->p->device).stream);
      MPG_CUDA(cudaStreamSynchronize(ctx(m->p->device).stream));
    }
    if (final_points) std::copy(o.final_points.begin(), o.final_points.end(), final_points);
    if (sweeps) *sweeps = o.sweeps;
    if (converged) *converged = o.converged;
    copy_rows(o.rows, rows, max_rows, nrows);
    if (warnings) {
      std::string t;
      for (const auto& w : o.warnings) t += w + "\n";
      int64_t len = 0;
      put_buffer(t, warnings, &len);
    }
  });
}

int mpg_update_expansion_points(const double* m, const double* d, const double* k, int r, const double* current,
                                int ncurrent, double* next) {
  return guard([&] {
    auto mat = [r](const double* p) {
      host::Mat x(r, r);
      std::memcpy(x.a.data(), p, x.a.size() * sizeof(double));
      return x;
    };
    const auto nx = host::update_expansion_points(mat(m), mat(d), mat(k), std::vector<double>(current, current + ncurrent));
    std::copy(nx.begin(), nx.end(), next);
  });
}

int mpg_h2_norm(const double* a, const double* b, const double* c, int ns, int m, int q, double* out) {
  return guard([&] {
    host::StateSpace ss;
    ss.a = host::Mat(ns, ns);
    ss.b = host::Mat(ns, m);
    ss.c = host::Mat(q, ns);
    std::memcpy(ss.a.a.data(), a, ss.a.a.size() * sizeof(double));
    std::memcpy(ss.b.a.data(), b, ss.b.a.size() * sizeof(double));
    std::memcpy(ss.c.a.data(), c, ss.c.a.size() * sizeof(double));
    *out = host::h2_norm(ss);
  });
}

}  // extern "C"
