/*
 * aapdhg_oracle.h — TEST INFRASTRUCTURE ONLY.
 *
 * Plain-C restatement of the reference AA-PDHG / FAA-PDHG solve path
 * (proj/src/{sparse_linalg,pdhg_core,anderson,filtering,solver}.cpp), used
 * only by tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * reference legs as the CHECKER. The product path never links it.
 *
 * Pinned: bit-for-bit against the reference itself compiled into
 * oracle/_ref (tests/test_oracle_pin.py) and against the committed golden
 * fixtures generated from it (tests/golden/, tests/golden/make_golden.py).
 *
 * Same POD structs and error codes as the CUDA C-ABI (include/aapdhg_cuda.h)
 * so the parity tests drive both through one Python wrapper.
 */
#ifndef AAPDHG_ORACLE_H_
#define AAPDHG_ORACLE_H_

#include "aapdhg_cuda.h"

#ifdef __cplusplus
extern "C" {
#endif

int aapdhg_oracle_solve(const aapdhg_problem_view* prob,
                        const aapdhg_solve_params* prm, const double* x0,
                        const double* y0, aapdhg_solve_result* res,
                        double* x_out, double* y_out, double* lambda_out,
                        aapdhg_record_sink sink, void* ctx, char* err,
                        size_t errlen);
int aapdhg_oracle_select_step_sizes(const aapdhg_problem_view* prob,
                                    const aapdhg_solve_params* prm, double* tau,
                                    double* sigma, char* err, size_t errlen);
int aapdhg_oracle_power_norm(const aapdhg_problem_view* prob, int32_t max_iters,
                             double rel_tol, uint64_t seed, double* out,
                             int32_t* rounds);
/* Seeded start vector of the power iteration: mt19937_64(seed) through
 * libstdc++'s uniform_real_distribution(-1, 1) (sparse_linalg.cpp:102-105). */
void aapdhg_oracle_power_start(uint64_t seed, int64_t n, double* out);
int aapdhg_oracle_matvec(const aapdhg_problem_view* prob, const double* x,
                         double* out);
int aapdhg_oracle_matvec_transpose(const aapdhg_problem_view* prob,
                                   const double* y, double* out);
int aapdhg_oracle_pdhg_step(const aapdhg_problem_view* prob, double tau,
                            double sigma, const double* x, const double* y,
                            double* xn, double* yn);
int aapdhg_oracle_kkt_metrics(const aapdhg_problem_view* prob, const double* x,
                              const double* y, double* kkt, double* lambda);
int aapdhg_oracle_aa_apply(int32_t p, int64_t N, const double* du_cols,
                           const double* dg_cols, double beta,
                           const double* d_hat, double eta, const double* u,
                           const double* g, double* out);
int aapdhg_oracle_filtered_aa_apply(int32_t p, int64_t N, const double* e_cols,
                                    const double* f_cols, double c_s,
                                    double kappa_bar, double beta,
                                    const double* d_hat, const double* u,
                                    const double* g, double* out,
                                    int32_t* kept);
/* length_bounds (filtering.cpp:92-114) on f given as p column norms^2. */
void aapdhg_oracle_length_bounds(int32_t p, const double* fn_sq, double c_s,
                                 double* b);
int aapdhg_oracle_safeguard_pass(double g_norm, double g0_norm, uint64_t i,
                                 double d, double eps);

#ifdef __cplusplus
}
#endif

#endif
