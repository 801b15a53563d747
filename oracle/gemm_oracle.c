/*
 * gemm_oracle.c -- CPU restatement of the reference's GEMM loop nests.
 *
 * TEST INFRASTRUCTURE ONLY.  This file is the parity checker and the CPU
 * baseline ("port") of the B200 library; only tests/, __graft_entry__.smoke()
 * and bench.py's cpu_baseline / --impl reference legs may load it.  The
 * product path (paper_1806_07060_b200) never links or calls it.
 *
 * Restates /root/reference/pkg/src/adaptgemm/kernels.py:
 *   oracle_reference  <- _kernel_reference   kernels.py:184-195
 *   oracle_direct     <- _kernel_direct      kernels.py:198-227
 *   oracle_tiled      <- _kernel_tiled       kernels.py:230-260
 *   oracle_pack       <- pack_padded         kernels.py:304-309
 *   oracle_indirect   <- _run_indirect       kernels.py:312-325
 * Every loop keeps the reference's float64 accumulation and summation order
 * and is compiled with -ffp-contract=off (numba/LLVM does not contract a
 * multiply and an add into an FMA without fastmath), so results are
 * bit-identical to the reference's numba kernels -- pinned against outputs
 * of the reference itself in tests/golden/.
 *
 * Parallelism (for the CPU baseline only): OpenMP over independent output
 * tiles (row block x column block); each output element is still computed
 * by one thread in the reference order, so threading never changes a bit.
 *
 * dtype: 0 float32, 1 float64.  Matrices are row-major with leading dims.
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define LOAD(p, dt, idx) ((dt) ? ((const double*)(p))[idx] : (double)((const float*)(p))[idx])
#define STORE(p, dt, idx, v)                                  \
    do {                                                      \
        if (dt) ((double*)(p))[idx] = (v);                    \
        else ((float*)(p))[idx] = (float)(v);                 \
    } while (0)

/* kernels.py:184-195 */
void oracle_reference(int64_t M, int64_t N, int64_t K, double alpha, double beta, int ta, int tb, int dt,
                      const void* A, int64_t lda, const void* B, int64_t ldb, const void* C, int64_t ldc,
                      void* out, int64_t ldo) {
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < M; ++i)
        for (int64_t j = 0; j < N; ++j) {
            double acc = 0.0;
            for (int64_t k = 0; k < K; ++k) {
                const double a = ta ? LOAD(A, dt, k * lda + i) : LOAD(A, dt, i * lda + k);
                const double b = tb ? LOAD(B, dt, j * ldb + k) : LOAD(B, dt, k * ldb + j);
                acc += a * b;
            }
            STORE(out, dt, i * ldo + j, alpha * acc + beta * LOAD(C, dt, i * ldc + j));
        }
}

static int64_t imin(int64_t a, int64_t b) { return a < b ? a : b; }

/* kernels.py:198-227: blocked bm x bn x bk, tm x tn micro tiles, unpadded
 * operands; per element the k order is 0..K-1 (block by block). */
void oracle_direct(int64_t M, int64_t N, int64_t K, double alpha, double beta, int ta, int tb, int dt,
                   const void* A, int64_t lda, const void* B, int64_t ldb, const void* C, int64_t ldc,
                   void* out, int64_t ldo, int bm, int bn, int bk, int tm, int tn) {
    const int64_t nbm = (M + bm - 1) / bm, nbn = (N + bn - 1) / bn;
#pragma omp parallel
    {
        double* acc = (double*)malloc(sizeof(double) * (size_t)bm * bn);
#pragma omp for schedule(dynamic)
        for (int64_t t = 0; t < nbm * nbn; ++t) {
            const int64_t ii = (t / nbn) * bm, ih = imin(ii + bm, M);
            {
                const int64_t jj = (t % nbn) * bn;
                const int64_t jh = imin(jj + bn, N);
                for (int64_t i = 0; i < ih - ii; ++i)
                    for (int64_t j = 0; j < jh - jj; ++j) acc[i * bn + j] = 0.0;
                for (int64_t kk = 0; kk < K; kk += bk) {
                    const int64_t kh = imin(kk + bk, K);
                    for (int64_t i0 = ii; i0 < ih; i0 += tm) {
                        const int64_t i1 = imin(i0 + tm, ih);
                        for (int64_t j0 = jj; j0 < jh; j0 += tn) {
                            const int64_t j1 = imin(j0 + tn, jh);
                            for (int64_t k = kk; k < kh; ++k)
                                for (int64_t i = i0; i < i1; ++i) {
                                    const double a = ta ? LOAD(A, dt, k * lda + i) : LOAD(A, dt, i * lda + k);
                                    for (int64_t j = j0; j < j1; ++j) {
                                        const double b = tb ? LOAD(B, dt, j * ldb + k) : LOAD(B, dt, k * ldb + j);
                                        acc[(i - ii) * bn + (j - jj)] += a * b;
                                    }
                                }
                        }
                    }
                }
                for (int64_t i = ii; i < ih; ++i)
                    for (int64_t j = jj; j < jh; ++j)
                        STORE(out, dt, i * ldo + j,
                              alpha * acc[(i - ii) * bn + (j - jj)] + beta * LOAD(C, dt, i * ldc + j));
            }
        }
        free(acc);
    }
}

/* kernels.py:230-260: exact tile multiples; uk == 2 adds a0*b0 + a1*b1 as
 * one pairwise term per accumulator update. */
void oracle_tiled(int64_t Mp, int64_t Np, int64_t Kp, double alpha, double beta, int dt, const void* Ap,
                  const void* Bp, const void* Cp, void* outp, int bm, int bn, int bk, int tm, int tn, int uk) {
    const int64_t nbm = Mp / bm, nbn = Np / bn;
#pragma omp parallel
    {
        double* acc = (double*)malloc(sizeof(double) * (size_t)bm * bn);
#pragma omp for schedule(dynamic)
        for (int64_t t = 0; t < nbm * nbn; ++t) {
            const int64_t ii = (t / nbn) * bm;
            {
                const int64_t jj = (t % nbn) * bn;
                for (int64_t i = 0; i < (int64_t)bm * bn; ++i) acc[i] = 0.0;
                for (int64_t kk = 0; kk < Kp; kk += bk)
                    for (int64_t i0 = ii; i0 < ii + bm; i0 += tm)
                        for (int64_t j0 = jj; j0 < jj + bn; j0 += tn) {
                            if (uk == 2) {
                                for (int64_t k = kk; k < kk + bk; k += 2)
                                    for (int64_t i = i0; i < i0 + tm; ++i) {
                                        const double a0 = LOAD(Ap, dt, i * Kp + k);
                                        const double a1 = LOAD(Ap, dt, i * Kp + k + 1);
                                        for (int64_t j = j0; j < j0 + tn; ++j)
                                            acc[(i - ii) * bn + (j - jj)] +=
                                                a0 * LOAD(Bp, dt, k * Np + j) + a1 * LOAD(Bp, dt, (k + 1) * Np + j);
                                    }
                            } else {
                                for (int64_t k = kk; k < kk + bk; ++k)
                                    for (int64_t i = i0; i < i0 + tm; ++i) {
                                        const double a = LOAD(Ap, dt, i * Kp + k);
                                        for (int64_t j = j0; j < j0 + tn; ++j)
                                            acc[(i - ii) * bn + (j - jj)] += a * LOAD(Bp, dt, k * Np + j);
                                    }
                            }
                        }
                for (int64_t i = 0; i < bm; ++i)
                    for (int64_t j = 0; j < bn; ++j)
                        STORE(outp, dt, (ii + i) * Np + jj + j,
                              alpha * acc[i * bn + j] + beta * LOAD(Cp, dt, (ii + i) * Np + jj + j));
            }
        }
        free(acc);
    }
}

/* kernels.py:304-309: zeros(pad_rows, pad_cols) with op(X) in the corner */
void oracle_pack(int dt, const void* X, int64_t ldx, int64_t rows, int64_t cols, int transpose, void* dst,
                 int64_t pad_rows, int64_t pad_cols) {
    const size_t es = dt ? 8 : 4;
    memset(dst, 0, es * (size_t)pad_rows * (size_t)pad_cols);
    for (int64_t r = 0; r < rows; ++r)
        for (int64_t c = 0; c < cols; ++c)
            STORE(dst, dt, r * pad_cols + c, transpose ? LOAD(X, dt, c * ldx + r) : LOAD(X, dt, r * ldx + c));
}

static int64_t round_up(int64_t x, int64_t s) { return (x + s - 1) / s * s; }

/* kernels.py:312-325: pack, tiled core, unpad; C is only read if beta != 0 */
int oracle_indirect(int64_t M, int64_t N, int64_t K, double alpha, double beta, int ta, int tb, int dt,
                    const void* A, int64_t lda, const void* B, int64_t ldb, const void* C, int64_t ldc, void* out,
                    int64_t ldo, int bm, int bn, int bk, int tm, int tn, int uk) {
    const int64_t Mp = round_up(M, bm), Np = round_up(N, bn), Kp = round_up(K, bk);
    const size_t es = dt ? 8 : 4;
    void* Ap = malloc(es * (size_t)Mp * Kp);
    void* Bp = malloc(es * (size_t)Kp * Np);
    void* Cp = malloc(es * (size_t)Mp * Np);
    void* outp = malloc(es * (size_t)Mp * Np);
    if (!Ap || !Bp || !Cp || !outp) {
        free(Ap); free(Bp); free(Cp); free(outp);
        return 1;
    }
    oracle_pack(dt, A, lda, M, K, ta, Ap, Mp, Kp);
    oracle_pack(dt, B, ldb, K, N, tb, Bp, Kp, Np);
    if (beta != 0.0) oracle_pack(dt, C, ldc, M, N, 0, Cp, Mp, Np);
    else memset(Cp, 0, es * (size_t)Mp * Np);
    oracle_tiled(Mp, Np, Kp, alpha, beta, dt, Ap, Bp, Cp, outp, bm, bn, bk, tm, tn, uk);
    for (int64_t i = 0; i < M; ++i) memcpy((char*)out + es * (size_t)(i * ldo), (char*)outp + es * (size_t)(i * Np), es * (size_t)N);
    free(Ap); free(Bp); free(Cp); free(outp);
    return 0;
}

int oracle_num_threads(void) {
#ifdef _OPENMP
    extern int omp_get_max_threads(void);
    return omp_get_max_threads();
#else
    return 1;
#endif
}

/* the CPU baseline uses every host thread, whatever OMP_NUM_THREADS a
   launcher (torchrun sets 1) left in the environment */
void oracle_set_threads(int n) {
#ifdef _OPENMP
    extern void omp_set_num_threads(int);
    if (n > 0) omp_set_num_threads(n);
#else
    (void)n;
#endif
}
