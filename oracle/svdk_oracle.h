/*
 * svdk_oracle.h — CPU restatement of the reference svdkit hot path.
 *
 * TEST INFRASTRUCTURE ONLY. This library is the parity checker for the
 * B200 engine (libsvdk). Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load it. The product path
 * (paper_1906_12085_b200, libsvdk.so, libsvdkit.so) never links or calls it.
 *
 * Every function restates the reference algorithm in plain C, following the
 * same operation order so that, compiled with -ffp-contract=off, results are
 * bit-identical to the compiled reference (pinned by tests/test_oracle.py
 * against oracle/_ref and the golden vectors in tests/golden/).
 *
 * Matrices are column-major, leading dimension = rows (dense_matrix.hpp:41-46).
 * Return codes follow the engine's status convention (include/svdk.h):
 *   0 ok, 1 dimension, 2 param, 3 numerical (residual in *residual).
 */
#ifndef SVDK_ORACLE_H
#define SVDK_ORACLE_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum { ORC_OK = 0, ORC_E_DIM = 1, ORC_E_PARAM = 2, ORC_E_NUMERICAL = 3 };

/* kernels.cpp:348-379 */
int orc_gaussian_matrix(size_t rows, size_t cols, uint64_t seed, double* out);
/* kernels.cpp:14-45 ; c is m x l */
int orc_matmul(const double* a, size_t m, size_t n, const double* b, size_t l, double* c);
/* kernels.cpp:47-67 ; c is n x l */
int orc_matmul_tl(const double* a, size_t m, size_t n, const double* b, size_t l, double* c);
/* kernels.cpp:80-97 */
int orc_gram(const double* a, size_t m, size_t n, double* g);
/* kernels.cpp:99-105 */
double orc_frobenius_norm_sq(const double* a, size_t count);
/* kernels.cpp:111-224 ; q m x p, r p x p */
int orc_qr_thin(const double* h, size_t m, size_t p, double* q, double* r, size_t* rank);
/* kernels.cpp:241-346 ; w n, v n x n; on NUMERICAL *residual = off-norm */
int orc_eig_sym(const double* s, size_t n, int max_sweeps, double* w, double* v,
                double* residual, int* sweeps_done);
/* svd_methods.cpp:121-158 ; u m x n (first rank cols valid), sigma n, v n x n */
int orc_truncated_svd(const double* a, size_t m, size_t n, double* u, double* sigma,
                      double* v, size_t* rank);
/* svd_methods.cpp:160-170 ; u m x l, sigma l, v n x l */
int orc_randomized_pca(const double* a, size_t m, size_t n, size_t l, size_t q, uint64_t seed,
                       double* u, double* sigma, double* v, size_t* rank);
/* svd_methods.cpp:172-196 ; u m x w, sigma w, v n x w with w = min((i+1)l, n) upper bound */
int orc_krylov_svd(const double* a, size_t m, size_t n, size_t l, size_t iters, uint64_t seed,
                   double* u, double* sigma, double* v, size_t* rank);
/* pca.cpp:13-55 ; orientation 0 = ColumnsAreExamples, 1 = RowsAreExamples */
int orc_center(const double* a, size_t m, size_t n, int orientation, double* centered,
               double* mean);
/* pca.cpp:61-89 ; *k = 0 encodes nullopt */
int orc_select_components(const double* w, size_t count, double total, double threshold,
                          size_t* k);

#ifdef __cplusplus
}
#endif
#endif
