// skinny_probe.cu -- times skinny_n / skinny_m candidates (csrc/skinny.cuh)
// against the shipped split-K picks on the DeepBench skinny shapes, with an
// L2 flush before every sample (bench.py's regime).  Measurement only.
#include <cstdint>
#include <string>

#include "../paper_1806_07060_b200/csrc/launch.cuh"
#include "../paper_1806_07060_b200/csrc/skinny.cuh"

using namespace ag;

struct Exp { int kind, a, b, c; LaunchFn fn; };  // kind 0: skinny_n<TM,BN,NW>, 1: skinny_m<BM,TN2,NW>
#define N_LIST(X) X(1, 16, 4) X(1, 16, 8) X(2, 16, 4) X(2, 16, 8) X(4, 16, 4) X(1, 32, 4) X(1, 32, 8) X(2, 32, 4) X(2, 32, 8) X(1, 64, 4) X(1, 64, 8) X(4, 32, 4) X(2, 64, 4)
#define M_LIST(X) X(40, 2, 4) X(40, 2, 8) X(48, 2, 4) X(24, 2, 4) X(16, 4, 4) X(32, 2, 4) X(16, 2, 4) X(8, 4, 4)
// kind 2: skinny_m<40, 2, NW> with the B granule ring varied: (QK k per granule, NBUF buffers)
#define M2_LIST(X) X(8, 4, 4) X(4, 4, 4) X(4, 8, 4) X(8, 2, 8) X(8, 4, 8) X(4, 8, 8)
#define N_ENTRY(a, b, c) {0, a, b, c, &skinny::launch_n<a, b, c>},
#define M_ENTRY(a, b, c) {1, a, b, c, &skinny::launch_m<a, b, c>},
#define M2_ENTRY(qk, nb, nw) {2, qk, nb, nw, &skinny::launch_m<40, 2, nw, qk, nb>},
static const Exp kExps[] = {N_LIST(N_ENTRY) M_LIST(M_ENTRY) M2_LIST(M2_ENTRY)};

extern "C" int exp_count() { return (int)(sizeof(kExps) / sizeof(kExps[0])); }
extern "C" void exp_info(int i, int* t) { t[0] = kExps[i].kind; t[1] = kExps[i].a; t[2] = kExps[i].b; t[3] = kExps[i].c; }

__global__ void read_kernel(const float4* __restrict__ p, size_t n, float* sink) {
    float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
        const float4 v = p[i];
        acc.x += v.x; acc.y += v.y; acc.z += v.z; acc.w += v.w;
    }
    if (acc.x + acc.y + acc.z + acc.w == 1234.5f) *sink = acc.x;
}

// mode 0: 256 MB write; 1: write then a 256 MB read (L2 ends up clean and
// cold); 2: nothing (warm)
static int g_mode = 0;
extern "C" void set_flush_mode(int m) { g_mode = m; }
static void do_flush(void* flush, size_t bytes, int r) {
    if (g_mode == 2) return;
    cudaMemsetAsync(flush, r & 0xff, bytes, 0);
    if (g_mode == 1) read_kernel<<<148 * 8, 256>>>((const float4*)flush, bytes / 16, (float*)flush);
}

// median of `reps` samples, each: flush, event, one call, event
extern "C" int exp_time(int i, int64_t M, int64_t N, int64_t K, const float* A, const float* B, float* out,
                        int splits, void* flush, size_t flush_bytes, int reps, double* seconds) {
    const Exp& e = kExps[i];
    std::string err;
    GemmCall c{};
    c.M = M; c.N = N; c.K = K; c.alpha = 1.0; c.beta = 0.0; c.ta = 0; c.tb = 0; c.dtype = 0;
    c.A = A; c.lda = K; c.B = B; c.ldb = N; c.C = out; c.ldc = N; c.out = out; c.ldo = N;
    c.stream = 0; c.splits = splits; c.err = &err;
    int rc = e.fn(c);
    if (rc) { fprintf(stderr, "exp %d: %s\n", i, err.c_str()); return rc; }
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    double s[64];
    reps = reps > 64 ? 64 : reps;
    for (int r = 0; r < reps; ++r) {
        do_flush(flush, flush_bytes, r);
        cudaEventRecord(e0, 0);
        rc |= e.fn(c);
        cudaEventRecord(e1, 0);
        cudaEventSynchronize(e1);
        float ms = 0.f;
        cudaEventElapsedTime(&ms, e0, e1);
        s[r] = ms * 1e-3;
    }
    for (int a = 0; a < reps; ++a)
        for (int b = a + 1; b < reps; ++b)
            if (s[b] < s[a]) { double t = s[a]; s[a] = s[b]; s[b] = t; }
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    *seconds = s[reps / 2];
    return rc ? rc : (cudaGetLastError() == cudaSuccess ? 0 : 3);
}

__global__ void empty_kernel() {}
extern "C" double empty_launch(void* flush, size_t flush_bytes, int reps) {
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    empty_kernel<<<148, 256>>>();  // module load outside the samples
    cudaDeviceSynchronize();
    double best = 1e9, sum = 0;
    for (int r = 0; r < reps; ++r) {
        do_flush(flush, flush_bytes, r);
        cudaEventRecord(e0, 0);
        empty_kernel<<<148, 256>>>();
        cudaEventRecord(e1, 0);
        cudaEventSynchronize(e1);
        float ms = 0.f;
        cudaEventElapsedTime(&ms, e0, e1);
        sum += ms;
        best = ms < best ? ms : best;
    }
    (void)sum;
    return best * 1e-3;
}
extern "C" void do_flush_ext(void* flush, size_t bytes, int r) { do_flush(flush, bytes, r); }

// ---- streaming-read floor: how long a pure read of `bytes` takes in the
// bench regime (flush, event, one kernel, event).  Each CTA reads one
// contiguous chunk with UNROLL independent 16-byte loads in flight per
// thread.  The floor any skinny GEMM over an operand of that size can reach.
template <int UNROLL>
__global__ void __launch_bounds__(256) chunk_read_kernel(const float4* __restrict__ p, size_t n, float* sink) {
    const size_t per = (n + gridDim.x - 1) / gridDim.x;
    const size_t b = blockIdx.x * per, e = min(n, b + per);
    float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
    for (size_t i = b + threadIdx.x; i < e; i += 256 * UNROLL) {
        float4 v[UNROLL];
#pragma unroll
        for (int u = 0; u < UNROLL; ++u) {
            const size_t j = i + (size_t)u * 256;
            v[u] = j < e ? __ldg(p + j) : make_float4(0.f, 0.f, 0.f, 0.f);
        }
#pragma unroll
        for (int u = 0; u < UNROLL; ++u) { acc.x += v[u].x; acc.y += v[u].y; acc.z += v[u].z; acc.w += v[u].w; }
    }
    if (acc.x + acc.y + acc.z + acc.w == 1234.5f) *sink = acc.x;
}

extern "C" double read_floor(const void* src, size_t bytes, int ctas, int unroll, void* flush, size_t flush_bytes,
                             int reps) {
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    auto go = [&]() {
        const float4* p = (const float4*)src;
        float* sink = (float*)flush;
        if (unroll == 4) chunk_read_kernel<4><<<ctas, 256>>>(p, bytes / 16, sink);
        else if (unroll == 8) chunk_read_kernel<8><<<ctas, 256>>>(p, bytes / 16, sink);
        else chunk_read_kernel<16><<<ctas, 256>>>(p, bytes / 16, sink);
    };
    go();
    cudaDeviceSynchronize();
    double s[64];
    reps = reps > 64 ? 64 : reps;
    for (int r = 0; r < reps; ++r) {
        do_flush(flush, flush_bytes, r);
        cudaEventRecord(e0, 0);
        go();
        cudaEventRecord(e1, 0);
        cudaEventSynchronize(e1);
        float ms = 0.f;
        cudaEventElapsedTime(&ms, e0, e1);
        s[r] = ms * 1e-3;
    }
    for (int a = 0; a < reps; ++a)
        for (int b = a + 1; b < reps; ++b)
            if (s[b] < s[a]) { double t = s[a]; s[a] = s[b]; s[b] = t; }
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    return s[reps / 2];
}
