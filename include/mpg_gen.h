/* mpg_gen.h — seeded synthetic inputs (test / bench fixtures, NOT the product).
 *
 * Built from paper_2003_12759_b200/csrc/gen/generators.cpp into its own
 * library, libmpggen.so, used by the GPU arm of bench.py and the tests to
 * create inputs, and compiled a second time into oracle/liboracle.so so the
 * CPU reference arm maps nothing outside oracle/. The five BASELINE.json
 * configs have no generator in the reference; the
 * reference's test fixtures (proj/tests/support.hpp:18-49) and toy models
 * (proj/src/generator.cpp:37-207) are restated draw for draw.
 * Returned objects are freed with mpg_gen_csr_free / mpg_gen_system_free of
 * the same library. Status: 0 ok, nonzero error (mpg_gen_last_error). */
#ifndef MPG_GEN_H
#define MPG_GEN_H
#include "mpg.h"
#ifdef __cplusplus
extern "C" {
#endif

const char* mpg_gen_last_error(void);
void mpg_gen_csr_free(mpg_host_csr* m);
void mpg_gen_system_free(mpg_host_system* s);
int mpg_gen_random_dense(int64_t r, int64_t c, uint64_t seed, double* out);
int mpg_gen_random_sparse(int64_t r, int64_t c, double density, uint64_t seed, double diag_shift, mpg_host_csr** out);
/* test helper: the same ingestion rule as mpg_host_csr_from_triplets */
int mpg_gen_from_triplets(int64_t nr, int64_t nc, int64_t nnz, const int64_t* ri, const int64_t* ci, const double* v,
                          mpg_host_csr** out);
int mpg_gen_bilinear_toy(int64_t n, int64_t m, uint64_t seed, mpg_host_csr** k_out, double* f, double* c);
/* ... with the couplings N_1..N_m (n_out: m pointers). */
int mpg_gen_bilinear_toy_n(int64_t n, int64_t m, uint64_t seed, mpg_host_csr** k_out, mpg_host_csr** n_out, double* f,
                           double* c);
/* generate_disc_brake_like (proj/src/generator.cpp:37-139): M and K = K_E + K_R + omega^2 K_G; D = alpha M + beta K
 * and F = C = e_1 are formed by the caller. */
int mpg_gen_disc_brake(int64_t n, double omega, uint64_t seed, mpg_host_csr** m_out, mpg_host_csr** k_out);
/* generate_qb_toy (proj/src/generator.cpp:181-207): D, K, N (n x n), H (n x n^2, column b n + c); F = C = e_1. */
int mpg_gen_qb_toy(int64_t n, uint64_t seed, mpg_host_csr** d, mpg_host_csr** k, mpg_host_csr** n_op,
                   mpg_host_csr** h);
int mpg_gen_grid2d(int64_t N, uint64_t seed, mpg_host_system** out);
int mpg_gen_convdiff3d(int64_t M, uint64_t seed, mpg_host_system** out);
int mpg_gen_fem3d(int64_t N, uint64_t seed, int mimo, mpg_host_system** out);
int mpg_gen_zipf(int64_t n, uint64_t seed, int64_t min_len, int64_t max_len, double expo, int nshifts,
                 mpg_host_system** out);

#ifdef __cplusplus
}
#endif
#endif /* MPG_GEN_H */
