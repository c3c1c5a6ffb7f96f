/* TEST INFRASTRUCTURE ONLY — the CPU checker for the signature hot path.
 *
 * A plain-C restatement of the reference algorithm
 * (/root/reference/proj/include/sigkit/detail/sig_core.hpp and
 * proj/src/tensor_algebra.cpp, proj/src/oracle.cpp). It follows the
 * reference's floating-point operation order exactly, so with the same
 * compiler flags (no FMA contraction) it is bit-identical to the reference;
 * tests/test_oracle.py pins that against oracle/_ref and tests/golden/.
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg may
 * load this library. The product path (paper_2501_08455_b200/) never does.
 */
#ifndef SIG_ORACLE_H
#define SIG_ORACLE_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* sig_dim (tensor_algebra.cpp:10-20); returns 0 for d < 1 or N < 1. */
size_t sigo_sig_dim(int d, int N);

/* detail::sequential_forward<double/float> (sig_core.hpp:116-147).
 * paths (B,L,d) row-major -> out (B,D); stream_out (B,L-1,D) or NULL.
 * threads > 1 splits batch rows over pthreads (rows are independent,
 * SPEC.md:220-221). Returns L-1 (the fold-step counter). */
int64_t sigo_sequential_forward_f64(const double* paths, size_t B, size_t L, int d, int N,
                                    double* out, double* stream_out, int threads);
int64_t sigo_sequential_forward_f32(const float* paths, size_t B, size_t L, int d, int N,
                                    float* out, float* stream_out, int threads);

/* chen_product on flat signatures (tensor_algebra.cpp:80-102). */
void sigo_chen_product_f64(int d, int N, const double* a, const double* b, double* c);

/* restricted_exp flattened (tensor_algebra.cpp:63-78). */
void sigo_restricted_exp_f64(int d, int N, const double* v, double* out);

/* signature_bruteforce, weakly increasing tuples (oracle.cpp:28-96).
 * Returns 0, or 2 when L-1 > 8, N > 4 or d > 3 (OracleLimits, oracle.hpp:12-16). */
int sigo_bruteforce_f64(const double* path, size_t L, int d, int N, double* out);

#ifdef __cplusplus
}
#endif
#endif
