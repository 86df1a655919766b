// CPU ORACLE — test infrastructure only.
//
// A from-scratch C++ restatement of the reference `morprec` solve path
// (/root/reference/proj, which cannot be built here: Eigen3 and the vendored
// doctest/CLI11 headers are absent). Only tests/,
// __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference leg
// may load this code, and only as the checker or the timed CPU baseline.
// The product (paper_2003_12759_b200/) never links or calls it.
//
// Parity pinning: the restatement is checked against every known-answer and
// dense-oracle assertion of the reference's own tests (proj/tests/*.cpp),
// restated in tests/test_oracle_*.py. There are no golden files upstream.
//
// Every function cites the reference file:line it follows.
#pragma once

#include <cstdint>
#include <functional>
#include <iosfwd>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

namespace oracle {

using index_t = std::int64_t;
using Vec = std::vector<double>;

// ---- errors (proj/include/morprec/errors.hpp:12-28) -----------------------
struct ConfigError : std::runtime_error { using std::runtime_error::runtime_error; };
struct SolverError : std::runtime_error { using std::runtime_error::runtime_error; };
struct IoError : std::runtime_error { using std::runtime_error::runtime_error; };

// ---- small column-major dense matrix (stands in for Eigen::MatrixXd) ------
struct Dense {
  index_t rows = 0, cols = 0;
  std::vector<double> a;  // column-major
  Dense() = default;
  Dense(index_t r, index_t c, double v = 0.0) : rows(r), cols(c), a(size_t(r * c), v) {}
  double& operator()(index_t i, index_t j) { return a[size_t(i + j * rows)]; }
  double operator()(index_t i, index_t j) const { return a[size_t(i + j * rows)]; }
  double* col(index_t j) { return a.data() + j * rows; }
  const double* col(index_t j) const { return a.data() + j * rows; }
  static Dense identity(index_t n) { Dense d(n, n); for (index_t i = 0; i < n; ++i) d(i, i) = 1; return d; }
  Dense transpose() const;
  double norm() const;
};
Dense matmul(const Dense& x, const Dense& y);
Dense operator-(const Dense& x, const Dense& y);

// Eigen::ColPivHouseholderQR semantics (used at proj/src/spai.cpp:34).
struct ColPivQR {
  Dense qr;
  std::vector<double> hcoeffs;
  std::vector<index_t> perm;  // column permutation: x[perm[k]] <- z[k]
  index_t nonzero_pivots = 0;
  double maxpivot = 0.0;
  explicit ColPivQR(const Dense& a);
  index_t rank() const;
  Vec solve(const Vec& b) const;
};

// Eigen::FullPivLU semantics for small square systems (proj/src/birka.cpp:283).
struct FullPivLU {
  Dense lu;
  std::vector<index_t> p, q;  // row / column permutations
  index_t nonzero = 0;
  double maxpivot = 0.0;
  explicit FullPivLU(const Dense& a);
  bool invertible() const;
  Dense solve(const Dense& b) const;
  Dense inverse() const;
};

// Thin Householder Q (proj/src/birka.cpp:125-128).
Dense thin_q(const Dense& m);

struct Complex { double re, im; };
// Eigenvalues of a real square matrix (Hessenberg + Francis double shift).
std::vector<Complex> eigenvalues(const Dense& m);
// Eigenvalues sorted by (re, im) (proj/src/birka.cpp:93-104).
std::vector<Complex> sorted_eigenvalues(const Dense& m);
// Real block decomposition m = basis * blocks * basis^{-1}, 1x1 blocks for
// real eigenvalues and [[a, b], [-b, a]] (b > 0) for pairs, as Eigen's
// pseudoEigenvalueMatrix (proj/src/birka.cpp:114-123). Blocks are ordered by
// (re, im) of the eigenvalue with b >= 0, so that shift slots are stable.
struct RealSpectrum { Dense blocks, basis, basis_inv; };
bool real_spectrum(const Dense& m, RealSpectrum& out);

// ---- sparse CSR with CSC shadow (proj/src/sparse.cpp:12-46) ---------------
struct Triplet { index_t row, col; double value; };

class Csr {
 public:
  index_t nrows = 0, ncols = 0;
  std::vector<index_t> rowptr, colind;
  std::vector<double> val;
  std::vector<index_t> colptr, srow;  // shadow
  std::vector<double> sval;

  static Csr from_triplets(index_t nr, index_t nc, std::vector<Triplet> t);
  static Csr from_csr(index_t nr, index_t nc, std::vector<index_t> rp, std::vector<index_t> ci,
                      std::vector<double> v);
  static Csr identity(index_t n);
  static Csr diagonal(const Vec& d);
  static Csr zero(index_t nr, index_t nc);
  static Csr linear_combination(const std::vector<std::pair<double, const Csr*>>& terms);

  index_t nnz() const { return index_t(val.size()); }
  void multiply(const Vec& x, Vec& y) const;
  Vec multiply(const Vec& x) const { Vec y; multiply(x, y); return y; }
  Vec multiply_transpose(const Vec& x) const;
  Dense multiply(const Dense& x) const;
  Csr transpose() const;
  double frobenius_norm() const;
  Dense to_dense() const;
  struct ColumnSubmatrix { Dense block; std::vector<index_t> row_map; };
  ColumnSubmatrix extract_column_submatrix(const std::vector<index_t>& pattern) const;

  index_t col_begin(index_t j) const { return colptr[size_t(j)]; }
  index_t col_end(index_t j) const { return colptr[size_t(j) + 1]; }
  void build_shadow();
  void validate() const;
};
double frobenius_distance(const Csr& a, const Csr& b);

// ---- GMRES (proj/src/gmres.cpp:40-186) ------------------------------------
using LinearOp = std::function<void(const Vec&, Vec&)>;
LinearOp identity_operator();
LinearOp matvec_operator(const Csr& a);

struct GmresConfig { double rel_tol = 1e-6; int max_iter = 1000; bool record_history = false; };
struct GmresReport {
  int iterations = 0;
  bool converged = false, breakdown = false;
  double rhs_norm = 0, final_residual = 0, solve_seconds = 0;
  std::vector<double> residual_history;
  int reorth_passes = 0;
};
struct GmresResult { Vec x; GmresReport report; };
GmresResult gmres_right_preconditioned(const LinearOp& a, const LinearOp& p, const Vec& b,
                                       const GmresConfig& cfg);

// ---- SPAI (proj/src/spai.cpp) ---------------------------------------------
struct SpaiConfig {
  int pattern_kind = 1;  // 0 Diagonal, 1 PatternOfA, 2 PatternOfAPow
  int power = 2;
  double fill_tol = 1e-4;
  int max_fill_per_col = 50;
  int max_pattern_sweeps = 3;
  int threads = 1;
};
struct SpaiResult { Csr p; Vec column_residuals; index_t fallback_count = 0; double build_seconds = 0; };
struct PatternSolve { Vec coeffs; double residual = 0; bool rank_deficient = false; };
PatternSolve solve_pattern(const Csr& a, const std::vector<index_t>& pattern,
                           const index_t* rhs_rows, const double* rhs_vals, size_t rhs_n);
std::vector<index_t> initial_pattern(const Csr& a, index_t col, const SpaiConfig& cfg);
struct AdaptiveOutcome { std::vector<index_t> pattern; Vec coeffs; double residual = 0; bool rank_deficient = false; };
AdaptiveOutcome adaptive_column(const Csr& a, index_t col, const index_t* rhs_rows,
                                const double* rhs_vals, size_t rhs_n, const SpaiConfig& cfg);
SpaiResult spai_build(const Csr& a, const SpaiConfig& cfg);
struct SpaiColumn { std::vector<index_t> rows; Vec values; double residual = 0; bool rank_deficient = false; };
SpaiColumn spai_column_solve(const Csr& a, index_t col, std::vector<index_t> pattern);

void parallel_for(index_t begin, index_t end, int threads, const std::function<void(index_t)>& fn);

// ---- update factors and chains (proj/src/chain.cpp) -----------------------
struct UpdateFactor {
  Csr q;
  double min_residual = 0, matrix_change = 0, build_seconds = 0;
  index_t fallback_count = 0;
};
UpdateFactor update_build(const Csr& prev, const Csr& next, const SpaiConfig& cfg);

class PrecondChain {
 public:
  PrecondChain() = default;
  explicit PrecondChain(Csr base, double secs = 0.0);
  bool empty() const { return !base_ || base_->nrows == 0; }
  index_t dim() const { return base_ ? base_->nrows : 0; }
  int length() const { return int(updates_.size()); }
  PrecondChain extended(std::shared_ptr<const UpdateFactor> f) const;
  void apply(const Vec& in, Vec& out) const;
  LinearOp as_operator() const;
  const Csr& base() const { return *base_; }
  const std::vector<std::shared_ptr<const UpdateFactor>>& updates() const { return updates_; }
  double total_build_seconds = 0.0;
 private:
  std::shared_ptr<const Csr> base_;
  std::vector<std::shared_ptr<const UpdateFactor>> updates_;
};
double standard_residual(const Csr& a, const PrecondChain& p);

// ---- Kronecker operator, N = 0, generalised to a mass matrix --------------
// -(Lambda (x) E) - (I_r (x) A) acting on vec(X) (proj/src/kron.cpp:34-64
// with E = I). `e` null means the identity.
struct KronOp {
  Dense lambda;
  const Csr* a = nullptr;
  const Csr* e = nullptr;
  // bilinear couplers (kron.cpp:54-63): -(S^T (x) N) vec(X) = -vec(N X S)
  struct Coupler { Dense small; const Csr* sparse; };
  std::vector<Coupler> couplers;
  void apply(const Vec& in, Vec& out) const;
  index_t dim() const { return a->nrows * lambda.rows; }
};
Csr assemble_explicit(const KronOp& op, index_t max_nnz);

// ---- reports (proj/include/morprec/report.hpp:14-61) ----------------------
enum class PrecondKind { None = 0, Fresh = 1, Horizontal = 2, Vertical = 3, ReusedSameMatrix = 4 };
// ReuseFrozen (3) is the GPU path's extension for configs 2-4 ("built once at
// the first shift and reused"): one SPAI per (side, unit width), built at the
// first unit that needs it and applied unchanged afterwards.
enum class PrecondMode { None = 0, FreshSpai = 1, ReuseChain = 2, ReuseFrozen = 3 };
struct ReportRow {
  int sweep = 0, point = 0;
  PrecondKind kind = PrecondKind::None;
  int solves = 0;
  double precond_build_seconds = 0;
  long gmres_iterations = 0;
  double gmres_seconds = 0;
  double min_residual = 0.0 / 0.0, matrix_change = 0.0 / 0.0, standard_residual = 0.0 / 0.0;
};
struct ReductionReport {
  std::vector<ReportRow> rows;
  std::vector<std::string> warnings;
  bool converged = false;
  int reduced_order = 0, sweeps = 0;
};

// ---- IRKA (BIRKA with N = 0, proj/src/birka.cpp:139-310), E general -------
struct LinearSystem {
  Csr a;                   // n x n (reference K)
  std::vector<Csr> n_ops;  // bilinear couplings N_j (one per input), empty = linear
  std::shared_ptr<Csr> e;  // n x n mass, null = identity
  Dense b;                 // n x m (reference F)
  Dense c;                 // n x q (reference C)
};
struct IrkaConfig {
  int r = 2;
  double tol = 1e-4;
  int max_sweeps = 50;
  std::uint64_t seed = 1;
  GmresConfig gmres{1e-10, 1000, false};
  SpaiConfig spai{};
  int max_chain_len = 16;
  index_t explicit_nnz_cap = 200000;
  index_t standard_residual_max_dim = 5000;
  bool decoupled = false;  // one GMRES per shift unit instead of one joint n*r solve
  bool mirror_unstable = false;  // extension: reflect Re(lambda) > 0 before solving
  int unit_threads = 1;  // decoupled units solved concurrently (solves are independent)
};
struct IrkaState {
  Dense kr, fr, cr;        // reduced K = E_r^{-1} A_r, E_r^{-1} W^T B, V^T C
  std::vector<Dense> nr;   // reduced couplings E_r^{-1} W^T N_j V
  Dense er, ar;            // W^T E V, W^T A V
  std::vector<Complex> lambda;
  Dense v, w;
  int sweeps = 0;
};
IrkaState irka_default_seed(const LinearSystem& sys, int r, std::uint64_t seed);
std::pair<IrkaState, ReductionReport> irka_reduce(const LinearSystem& sys, const IrkaConfig& cfg,
                                                  PrecondMode mode, const IrkaState* init);

// ---- shift sweep (proj/src/bench.cpp:159-249) for sigma E - A -------------
struct SweepResult { ReductionReport report; int failed_solves = 0; std::vector<Vec> x; };
SweepResult run_spai_bench(const Csr& a, const Csr* e, const Vec& b, const std::vector<double>& points,
                           const SpaiConfig& spai, const GmresConfig& gmres, PrecondMode mode,
                           int max_chain_len, bool keep_solutions);

// ---- QB-IHOMM (proj/src/qbihomm.cpp, proj/src/orth.cpp) -------------------
struct QbSystem {
  Csr d, k, n_op;  // n x n
  Csr h;           // n x n^2, column b n + c
  Vec f, c;        // n (SISO)
  void validate() const;
};
struct QbConfig {
  std::vector<double> sigmas;
  int p_moments = 1, q_moments = 1;
  GmresConfig gmres{};
  SpaiConfig spai{};
  int max_chain_len = 16;
  index_t standard_residual_max_dim = 5000;
};
struct ReducedQb { Dense d, k, n_op, h, f, c, basis; };
struct OrthBasis {
  index_t dim = 0, capacity = 0;
  std::vector<Vec> cols;
  OrthBasis(index_t d, index_t cap) : dim(d), capacity(cap) {
    if (d <= 0 || cap <= 0) throw std::invalid_argument("orth: dimension and capacity must be positive");
  }
  bool append(const Vec& col, double drop_tol = 1e-10);
  Dense matrix() const;
};
Dense kron_compress_quadratic(const Csr& h, const Dense& u);
std::pair<ReducedQb, ReductionReport> qbihomm_reduce(const QbSystem& sys, const QbConfig& cfg, PrecondMode mode);

// ---- Matrix Market IO (proj/src/matrix_market.cpp) ------------------------
Csr read_matrix_market(std::istream& in, const std::string& origin);
Csr read_matrix_market_file(const std::string& path);
void write_matrix_market(std::ostream& out, const Csr& a);

// ---- AIRGA (proj/src/airga.cpp:136-384, h2.cpp, orth.cpp) -----------------
struct StateSpaceO { Dense a, b, c; };
double h2_norm_o(const StateSpaceO& sys);
double h2_distance_o(const StateSpaceO& a, const StateSpaceO& b);
struct AirgaConfigO {
  std::vector<double> expansion_points;
  int r_max = 20;
  double outer_tol = 1e-4, inner_tol = 1e-6;
  int max_outer = 20;
  GmresConfig gmres{};
  SpaiConfig spai{};
  int max_chain_len = 16;
  index_t standard_residual_max_dim = 5000;
};
struct AirgaModel { Dense m, d, k, f, c, basis; };
struct AirgaResult {
  AirgaModel model;
  ReductionReport report;
  std::vector<double> final_points;
  std::vector<std::vector<double>> point_history;  // the expansion points of every sweep
};
std::vector<double> update_expansion_points(const Dense& m, const Dense& d, const Dense& k,
                                            const std::vector<double>& current);
AirgaResult airga_reduce(const Csr& m, const Csr& d, const Csr& k, const Dense& f, const Dense& c, double alpha,
                         double beta, const AirgaConfigO& cfg, PrecondMode mode);

// ---- second-order transfer error (proj/src/airga.cpp:80-85, :386-447) -----
Csr shifted_operator2(const Csr& m, const Csr& d, const Csr& k, double s);
std::vector<double> transfer_function_error(const Csr& m, const Csr& d, const Csr& k, const Dense& f, const Dense& c,
                                            const Dense& rm, const Dense& rd, const Dense& rk, const Dense& rf,
                                            const Dense& rc, const std::vector<double>& grid, const GmresConfig& gmres,
                                            const SpaiConfig& spai, PrecondMode mode, int max_chain_len);

}  // namespace oracle
