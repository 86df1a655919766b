// IRKA and shift-sweep drivers (irka.cu).
#pragma once

#include <string>
#include <vector>

#include "host/small_dense.hpp"
#include "runtime.cuh"

namespace mpg {

struct IrkaSettings {
  int r = 2;
  double tol = 1e-4;
  int max_sweeps = 50;
  unsigned long long seed = 1;
  GmresOptions gmres{1e-10, 1000, false};
  SpaiOptions spai{};
  int max_chain_len = 16;
  long long standard_residual_max_dim = 5000;
  int mode = MPG_PRECOND_REUSE_CHAIN;
  std::vector<double> init_shifts;  // empty: default seed (power iteration)
  // Initial reduced state (birka_reduce's `const BirkaState* init`, birka.hpp:78-80),
  // column-major; each empty part keeps the default seed's. init_kr (r x r) wins over init_shifts.
  std::vector<double> init_kr, init_fr, init_cr;
  bool want_vw = false;
  bool mirror_unstable = false;
};

struct IrkaResult {
  host::Mat kr, fr, cr, er, ar;
  std::vector<host::Eig> lambda;
  std::vector<double> v, w;
  int sweeps = 0, reduced_order = 0;
  bool converged = false;
  long long total_iterations = 0, total_solves = 0;
  std::vector<mpg_report_row> rows;
};

// Owner map of the sharded IRKA: units placed longest-first (stable in unit
// order) on the least-loaded rank (lowest rank on ties); fixed[i] >= 0 pins a
// unit. shard_cost models a solve as w K (K + 40) from its slot's previous
// iteration count K (100 when unknown): the Gram-Schmidt work grows as K^2.
double shard_cost(int width, int last_iterations);
std::vector<int> shard_plan(const std::vector<double>& cost, const std::vector<int>& fixed, int world);

// Native NCCL exchange (comm.cu).
int comm_unique_id(char* out, int len);
mpg_comm* comm_create(int device, int rank, int world, const char* id_bytes);
void comm_destroy(mpg_comm* c);
int comm_allgather(mpg_comm* c, const void* send, void* recv, int64_t bytes);
void comm_stats(const mpg_comm* c, long long* calls, double* bytes);
int nccl_version();

IrkaResult irka_run(const ShiftedOp& op, const double* b_any, int m, const double* c_any, int q,
                    const IrkaSettings& cfg, int rank, int world, mpg_allgather_fn allgather, void* agctx);

struct SweepOutcome {
  std::vector<mpg_report_row> rows;
  int failed = 0;
  long long total_iterations = 0;
};
SweepOutcome sweep_run(const ShiftedOp& op, const double* b_any, const std::vector<double>& points,
                       const SpaiOptions& spai, const GmresOptions& gmres, int mode, int max_chain_len,
                       double* x_out);

}  // namespace mpg

namespace mpg {

// Quadratic term H (n x n^2, column b n + c) on the device, rows sorted.
struct QbH {
  int64_t n = 0, nnz = 0;
  DBuf<int> rowptr, bcol, ccol;
  DBuf<double> val;
};

struct QbSettings {
  std::vector<double> sigmas;
  int p_moments = 1, q_moments = 1;
  GmresOptions gmres{};
  SpaiOptions spai{};
  int max_chain_len = 16;
  long long standard_residual_max_dim = 5000;
  int mode = MPG_PRECOND_REUSE_CHAIN;
};

struct QbOutcome {
  int r = 0;
  host::Mat d, k, n_op, h, f, c;
  DBuf<double> basis;  // n x r, column-major, on the device
  std::vector<mpg_report_row> rows;
  long long total_iterations = 0, total_solves = 0;
};

// qbihomm_reduce (proj/src/qbihomm.cpp:144-208) on one device: op is the
// shifted family sigma E - A with A = K, E = D; n_op = N.
QbOutcome qbihomm_run(const ShiftedOp& op, const DevCsr& n_op, const QbH& h, const double* f_any, const double* c_any,
                      const QbSettings& cfg);

}  // namespace mpg

namespace mpg {

// transfer_function_error (proj/src/airga.cpp:386-447) for M x'' + D x' + K x
// = F u, y = C^T x, against a reduced model (r x r m, d, k; r x n_in f;
// r x n_out c). One shifted matrix s^2 M + s D + K per grid point, formed on
// the device from the merged pattern; preconditioner per mode (none, fresh,
// horizontal chain along the grid); NaN where a solve fails.
struct TfSettings {
  GmresOptions gmres{1e-10, 1000, false};
  SpaiOptions spai{};
  int mode = MPG_PRECOND_REUSE_CHAIN;
  int max_chain_len = 16;
};
std::vector<double> tf_error_run(const CsrPtr& m, const CsrPtr& d, const CsrPtr& k, const double* f_any, int n_in,
                                 const double* c_any, int n_out, const host::Mat& rm, const host::Mat& rd,
                                 const host::Mat& rk, const host::Mat& rf, const host::Mat& rc,
                                 const std::vector<double>& grid, const TfSettings& cfg, long long* total_iterations);

}  // namespace mpg

namespace mpg {

// airga_reduce (proj/src/airga.cpp:136-317) on one device.
struct AirgaSettings {
  std::vector<double> points;
  int r_max = 20;
  double outer_tol = 1e-4, inner_tol = 1e-6;
  int max_outer = 20;
  GmresOptions gmres{1e-6, 1000, false};
  SpaiOptions spai{};
  int max_chain_len = 16;
  long long standard_residual_max_dim = 5000;
  int mode = MPG_PRECOND_REUSE_CHAIN;
  double alpha = 0.0, beta = 0.0;
};
struct AirgaOutcome {
  int r = 0, sweeps = 0;
  bool converged = false;
  host::Mat m, d, k, f, c;
  DBuf<double> basis;  // n x r on the device
  std::vector<double> final_points;
  std::vector<mpg_report_row> rows;
  std::vector<std::string> warnings;
};
AirgaOutcome airga_run(const CsrPtr& m, const CsrPtr& d, const CsrPtr& k, const double* f_any, int n_in,
                       const double* c_any, int n_out, const AirgaSettings& cfg);

}  // namespace mpg

namespace mpg {

// birka_reduce with couplings N_1..N_m (proj/src/birka.cpp:139-310): per side
// one joint n r solve of the Kronecker operator -(Lambda (x) I) - (I (x) K) -
// sum_j (S_j^T (x) N_j), formed explicitly (kron.cpp:72-131) on the device
// and solved there; SPAI of that matrix unless it exceeds explicit_nnz_cap
// (then the side continues unpreconditioned, as the reference does).
struct BirkaOutcome {
  host::Mat kr, fr, cr;
  std::vector<host::Mat> nr;
  std::vector<host::Eig> lambda;
  std::vector<double> v, w;
  int sweeps = 0;
  bool converged = false;
  std::vector<mpg_report_row> rows;
  std::vector<std::string> warnings;
};
BirkaOutcome birka_coupled_run(const CsrPtr& k, const std::vector<CsrPtr>& n_ops, const double* b_any, int m,
                               const double* c_any, int q, const IrkaSettings& cfg, long long explicit_nnz_cap);

}  // namespace mpg
