// Drives the C++ mirror (include/morprec_gpu.hpp) the way a morprec user would:
// assemble a shifted 1D Laplacian, build a SPAI, solve with GMRES on the GPU,
// extend the chain with an update factor and solve the next shift.
// Exit code 0 on success. Built by tests/test_boundary.py, run by tests/test_gpu_cpp.py.
#include <cmath>
#include <cstdio>
#include <vector>

#include "morprec_gpu.hpp"

using namespace morprec_gpu;

static SparseMatrix lap1d(index_t n) {
  std::vector<index_t> rp{0}, ci;
  std::vector<double> v;
  for (index_t i = 0; i < n; ++i) {
    if (i > 0) { ci.push_back(i - 1); v.push_back(1.0); }
    ci.push_back(i); v.push_back(-2.0);
    if (i + 1 < n) { ci.push_back(i + 1); v.push_back(1.0); }
    rp.push_back(static_cast<index_t>(ci.size()));
  }
  return SparseMatrix::from_csr(n, n, rp, ci, v);
}

int main() {
  const index_t n = 500;
  SparseMatrix a = lap1d(n);  // A = -(Laplacian): sigma I - A is SPD for sigma > 0
  ShiftedOperator op(a);
  std::vector<double> b(static_cast<size_t>(n), 1.0);
  SparseMatrix m1 = op.explicit_matrix(0.5);
  SpaiResult p = spai_build(m1);
  PrecondChain chain(p.p);
  GmresConfig cfg{1e-10, 500, true};
  GmresResult r1 = gmres_shifted(op, 0.5, 0.0, false, chain, b, cfg);
  SparseMatrix m2 = op.explicit_matrix(0.7);
  UpdateFactor q = update_build(m1, m2);
  PrecondChain chain2 = chain.extended(q);
  GmresResult r2 = gmres_shifted(op, 0.7, 0.0, false, chain2, b, cfg);
  // true residual via the explicit matrix
  std::vector<double> ax = m2.multiply(r2.x);
  double res = 0.0, bn = 0.0;
  for (size_t i = 0; i < b.size(); ++i) { res += (b[i] - ax[i]) * (b[i] - ax[i]); bn += b[i] * b[i]; }
  std::printf("its %d %d chain %d rel %.3e hist %zu\n", r1.report.iterations, r2.report.iterations, chain2.length(),
              std::sqrt(res / bn), r1.report.residual_history.size());
  bool ok = r1.report.converged && r2.report.converged && chain2.length() == 1 && std::sqrt(res / bn) <= 1e-9 &&
            q.min_residual <= q.matrix_change;
  try {
    (void)gmres_right_preconditioned(a, PrecondChain(), std::vector<double>(static_cast<size_t>(n), 0.0));
    ok = false;  // zero rhs must throw std::invalid_argument
  } catch (const std::invalid_argument&) {
  }
  // bilinear system with one coupling N = 0.05 I (joint-solve birka_reduce)
  {
    const index_t nb = 60;
    SparseMatrix kb = lap1d(nb);
    std::vector<index_t> rp, ci;
    for (index_t i = 0; i <= nb; ++i) rp.push_back(i);
    for (index_t i = 0; i < nb; ++i) ci.push_back(i);
    SparseMatrix nm = SparseMatrix::from_csr(nb, nb, rp, ci, std::vector<double>(static_cast<size_t>(nb), 0.05));
    std::vector<double> fb(static_cast<size_t>(nb)), cb(static_cast<size_t>(nb));
    for (index_t i = 0; i < nb; ++i) { fb[size_t(i)] = 1.0; cb[size_t(i)] = double(i + 1) / double(nb); }
    BirkaConfig bc;
    bc.r = 2;
    bc.tol = 1e-8;
    bc.max_sweeps = 100;
    auto [st, rep] = birka_reduce(kb, {&nm}, fb, 1, cb, 1, bc, PrecondMode::ReuseChain);
    std::printf("birka sweeps %d conv %d lam %.6f %.6f\n", st.sweeps, int(rep.converged), st.lambda_re[0],
                st.lambda_re[1]);
    ok = ok && rep.converged && st.nr.size() == 1 && st.lambda_re[0] < 0 && st.lambda_re[1] < 0 &&
         rep.rows.size() == 2 * static_cast<size_t>(st.sweeps);
  }
  return ok ? 0 : 1;
}
