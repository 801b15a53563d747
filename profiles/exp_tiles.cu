// exp_tiles.cu -- candidate indirect-core tiles outside the shipped domains,
// timed by profiles/exp_tiles.py before they are added to a search space
// (measurement only, not product code).  Uses the product launcher as is.
#include <cstdint>
#include <string>

#include "../paper_1806_07060_b200/csrc/launch.cuh"
#include "../paper_1806_07060_b200/csrc/fp32_tma.cuh"

using namespace ag;

#define EXP_LIST(X)            \
    X(128, 128, 32, 8, 8, 1)   \
    X(128, 256, 16, 8, 16, 1)  \
    X(128, 256, 32, 8, 16, 1)  \
    X(256, 128, 16, 16, 8, 1)  \
    X(256, 128, 32, 16, 8, 1)  \
    X(128, 128, 32, 8, 16, 1)  \
    X(128, 128, 32, 16, 8, 1)  \
    X(128, 128, 16, 8, 16, 1)  \
    X(64, 256, 32, 8, 16, 1)

// uk = 0 rows: the pack-free in-place core (split-K family's loader) with one
// slice, i.e. the indirect family's math without the pack passes
#define INPLACE_LIST(X)       \
    X(32, 16, 32, 4, 2, 0)    \
    X(64, 16, 32, 4, 2, 0)    \
    X(128, 16, 32, 8, 2, 0)   \
    X(256, 16, 32, 8, 2, 0)   \
    X(128, 16, 64, 8, 2, 0)   \
    X(64, 16, 64, 4, 2, 0)    \
    X(128, 32, 32, 8, 4, 0)   \
    X(64, 32, 32, 4, 4, 0)    \
    X(32, 32, 32, 4, 4, 0)    \
    X(128, 128, 32, 8, 8, 0)  \
    X(64, 64, 16, 8, 8, 0)    \
    X(128, 128, 32, 8, 16, 0) \
    X(128, 256, 32, 8, 16, 0) \
    X(128, 128, 32, 16, 8, 0)

// uk = 9 rows: the TMA-fed core (fp32_tma.cuh), bk = 32
#define TMA_LIST(X)           \
    X(128, 128, 32, 8, 8, 9)  \
    X(64, 128, 32, 8, 8, 9)   \
    X(128, 64, 32, 8, 8, 9)   \
    X(64, 64, 32, 8, 8, 9)    \
    X(128, 256, 32, 8, 16, 9) \
    X(128, 128, 32, 8, 16, 9) \
    X(128, 128, 32, 16, 8, 9)

// ring-depth variants of the shipped big tiles: uk field = uk + 100 * stages
#define STAGE_LIST(X)              \
    X(64, 128, 32, 8, 8, 2, 2)     \
    X(64, 128, 32, 8, 8, 2, 3)     \
    X(64, 128, 32, 8, 8, 2, 4)     \
    X(64, 128, 32, 8, 8, 2, 5)     \
    X(128, 64, 32, 8, 8, 2, 3)     \
    X(64, 128, 16, 8, 8, 2, 4)     \
    X(64, 128, 16, 8, 8, 2, 6)     \
    X(128, 128, 16, 16, 8, 1, 2)   \
    X(128, 128, 16, 16, 8, 1, 3)   \
    X(128, 128, 16, 16, 8, 1, 4)   \
    X(128, 256, 32, 8, 16, 1, 2)   \
    X(128, 256, 32, 8, 16, 1, 3)   \
    X(128, 256, 16, 8, 16, 1, 3)   \
    X(128, 256, 16, 8, 16, 1, 5)

struct Exp { int bm, bn, bk, tm, tn, uk; LaunchFn fn; };
#define EXP_ENTRY(bm, bn, bk, tm, tn, uk) {bm, bn, bk, tm, tn, uk, &launch_indirect<float, bm, bn, bk, tm, tn, uk>},
#define INPLACE_ENTRY(bm, bn, bk, tm, tn, uk) {bm, bn, bk, tm, tn, uk, &launch_inplace<bm, bn, bk, tm, tn>},
#define TMA_ENTRY(bm, bn, bk, tm, tn, uk) {bm, bn, bk, tm, tn, uk, &f32tma::launch_tma<bm, bn, tm, tn>},
#define STAGE_ENTRY(bm, bn, bk, tm, tn, uk, st) \
    {bm, bn, bk, tm, tn, uk + 100 * st, &launch_indirect<float, bm, bn, bk, tm, tn, uk, false, st>},
static const Exp kExps[] = {EXP_LIST(EXP_ENTRY) INPLACE_LIST(INPLACE_ENTRY) TMA_LIST(TMA_ENTRY)
                                STAGE_LIST(STAGE_ENTRY)};

extern "C" int exp_count() { return (int)(sizeof(kExps) / sizeof(kExps[0])); }
extern "C" void exp_tile(int i, int* t) {
    const Exp& e = kExps[i];
    t[0] = e.bm; t[1] = e.bn; t[2] = e.bk; t[3] = e.tm; t[4] = e.tn; t[5] = e.uk;
}
extern "C" size_t exp_ws(int i, int64_t M, int64_t N, int64_t K, int splits) {
    const Exp& e = kExps[i];
    return indirect_workspace_bytes<float>(M, N, K, e.bm, e.bn, e.bk, splits);
}

// median-free best-of-reps device time (seconds) of one config, warm buffers
extern "C" int exp_time(int i, int64_t M, int64_t N, int64_t K, const float* A, const float* B, float* out,
                        void* ws, size_t ws_bytes, int reps, int splits, double* seconds) {
    const Exp& e = kExps[i];
    std::string err;
    GemmCall c{};
    c.M = M; c.N = N; c.K = K; c.alpha = 1.0; c.beta = 0.0; c.ta = 0; c.tb = 0; c.dtype = 0;
    c.A = A; c.lda = K; c.B = B; c.ldb = N; c.C = out; c.ldc = N; c.out = out; c.ldo = N;
    c.ws = ws; c.ws_bytes = ws_bytes; c.stream = 0; c.splits = splits; c.err = &err;
    c.bm = e.bm; c.bn = e.bn; c.bk = e.bk; c.tm = e.tm; c.tn = e.tn; c.uk = e.uk;
    int rc = e.fn(c);
    if (rc) return rc;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    double best = 1e30;
    for (int r = 0; r < reps; ++r) {
        cudaEventRecord(e0, 0);
        rc = e.fn(c);
        cudaEventRecord(e1, 0);
        cudaEventSynchronize(e1);
        float ms = 0.f;
        cudaEventElapsedTime(&ms, e0, e1);
        if (ms * 1e-3 < best) best = ms * 1e-3;
    }
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    *seconds = best;
    return rc ? rc : (cudaGetLastError() == cudaSuccess ? 0 : 3);
}
