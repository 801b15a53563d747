// kernels.cuh -- sm_100a CUDA kernels of the two GEMM families.
//
// Reference semantics (/root/reference/pkg/src/adaptgemm/kernels.py):
//   direct   (_kernel_direct, :198-227): one kernel over the caller's unpadded
//            operands; ragged tile edges and both transposes handled inside
//            the kernel; always reads C (beta * C even when beta == 0).
//   indirect (_run_indirect + pack_padded + _kernel_tiled, :230-260,
//            :304-325): O(n^2) helper passes copy op(A), op(B) into zero-padded
//            tile-multiple buffers, then a branch-free blocked core runs on
//            exact multiples; C is only read when beta != 0 (:318-321).
//
// B200 design (not a translation of the numba loop nests):
//   * block_m x block_n is the CTA tile, block_k the K depth of one shared
//     memory stage, tile_m x tile_n the per-thread register tile, unroll_k the
//     number of K steps whose fragments are loaded before the FMAs.
//   * FP32 runs on the CUDA cores (FFMA) with fp32 accumulation; operands are
//     staged global->shared with cp.async (16-byte, L1-bypassing, multi-stage
//     ring for the indirect core; 4/8-byte zero-filling predicated copies for
//     the direct family), register tiles read with 64/128-bit LDS in an
//     interleaved layout that is bank-conflict free.
//   * The indirect pack writes op(A)^T (K-major) so both operands stream as
//     contiguous rows; the padded output + unpad copy of the reference are
//     fused into a masked store epilogue (same values, two fewer passes).
//   * BM/BN/BK == 0 instantiations take the tile sizes at run time (used for
//     float64 and for legal configs outside the enumerated domains).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace ag {

typedef long long i64;

template <typename T> struct VecW;
template <> struct VecW<float> { static constexpr int W = 4; };
template <> struct VecW<double> { static constexpr int W = 2; };

// widest vector (elements) that divides n, bounded by 16 bytes
template <typename T, int n> struct FragW {
    static constexpr int W = (n % VecW<T>::W == 0) ? VecW<T>::W : ((n % 2 == 0 && VecW<T>::W >= 2) ? 2 : 1);
};

template <typename T, int W> struct alignas(sizeof(T) * W) Vec { T v[W]; };

__device__ __forceinline__ uint32_t smem_addr(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

// cp.async with zero fill: copies `pred ? BYTES : 0` bytes, zero-fills the rest
template <int BYTES>
__device__ __forceinline__ void cp_async(void* smem, const void* gmem, bool pred = true) {
    const uint32_t s = smem_addr(smem);
    const int src = pred ? BYTES : 0;
    if constexpr (BYTES == 16) {
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(s), "l"(gmem), "r"(src) : "memory");
    } else {
        asm volatile("cp.async.ca.shared.global [%0], [%1], %2, %3;\n" ::"r"(s), "l"(gmem), "n"(BYTES), "r"(src) : "memory");
    }
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory"); }

// programmatic dependent launch (launch.cuh launch_maybe_dependent): a helper
// pass lets the next kernel of its family path launch early; that kernel
// waits here before touching global memory.  Both are no-ops otherwise.
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory"); }
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;\n" ::: "memory"); }

__device__ __forceinline__ float fmadd(float a, float b, float c) { return __fmaf_rn(a, b, c); }
__device__ __forceinline__ double fmadd(double a, double b, double c) { return __fma_rn(a, b, c); }

// Packed fp32 pairs for the sm_100 paired FMA (fma.rn.f32x2 -> SASS FFMA2).
// One FFMA2 does two IEEE fp32 FMAs (each rounded once, exactly as two
// fma.rn.f32), so the per-element operation sequence -- and the result -- is
// unchanged.  With a scalar first operand ptxas emits the broadcast form
// `FFMA2 Rd, Ra.F32, Rb.F32x2, Rc.F32x2`: a register tile updated as
// acc[i][j:j+2] += a[i] * b[j:j+2] issues half the instructions of the
// scalar loop, and every pair operand spans both register banks, which
// removes the bank-conflict dispatch stalls of the 3-register FFMA.
typedef unsigned long long f32x2;
__device__ __forceinline__ f32x2 pack2(float lo, float hi) {
    f32x2 r;
    asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(lo), "f"(hi));
    return r;
}
__device__ __forceinline__ void unpack2(f32x2 v, float& lo, float& hi) {
    asm("mov.b64 {%0, %1}, %2;" : "=f"(lo), "=f"(hi) : "l"(v));
}
__device__ __forceinline__ void ffma2(f32x2& d, float a, f32x2 b) {
    asm("fma.rn.f32x2 %0, %1, %2, %0;" : "+l"(d) : "l"(pack2(a, a)), "l"(b));
}

// Register tile acc[TM][TN] += a[TM] (x) b[TN].  For fp32 with an even TN the
// tile is held as TM x TN/2 packed pairs and updated with FFMA2; otherwise
// scalar FMAs.  Same products, same per-element order either way.
template <typename T, int TM, int TN>
struct RegTile {
    static constexpr bool PAIRED = false;
    T acc[TM][TN];
    __device__ __forceinline__ void zero() {
#pragma unroll
        for (int i = 0; i < TM; ++i)
#pragma unroll
            for (int j = 0; j < TN; ++j) acc[i][j] = T(0);
    }
    __device__ __forceinline__ void fma(const T (&a)[TM], const T (&b)[TN]) {
#pragma unroll
        for (int i = 0; i < TM; ++i)
#pragma unroll
            for (int j = 0; j < TN; ++j) acc[i][j] = fmadd(a[i], b[j], acc[i][j]);
    }
    __device__ __forceinline__ void unpack(T (&out)[TM][TN]) const {
#pragma unroll
        for (int i = 0; i < TM; ++i)
#pragma unroll
            for (int j = 0; j < TN; ++j) out[i][j] = acc[i][j];
    }
};

template <int TM, int TN>
struct RegTilePaired {
    static constexpr bool PAIRED = true;
    f32x2 acc[TM][TN / 2];
    __device__ __forceinline__ void zero() {
#pragma unroll
        for (int i = 0; i < TM; ++i)
#pragma unroll
            for (int j = 0; j < TN / 2; ++j) acc[i][j] = 0ull;
    }
    __device__ __forceinline__ void fma(const float (&a)[TM], const float (&b)[TN]) {
        f32x2 bp[TN / 2];
#pragma unroll
        for (int j = 0; j < TN / 2; ++j) bp[j] = pack2(b[2 * j], b[2 * j + 1]);
#pragma unroll
        for (int i = 0; i < TM; ++i)
#pragma unroll
            for (int j = 0; j < TN / 2; ++j) ffma2(acc[i][j], a[i], bp[j]);
    }
    __device__ __forceinline__ void unpack(float (&out)[TM][TN]) const {
#pragma unroll
        for (int i = 0; i < TM; ++i)
#pragma unroll
            for (int j = 0; j < TN / 2; ++j) unpack2(acc[i][j], out[i][2 * j], out[i][2 * j + 1]);
    }
};

template <typename T, int TM, int TN, bool OK = (sizeof(T) == 4 && TN % 2 == 0)>
struct RegTileFor { typedef RegTile<T, TM, TN> type; };
template <int TM, int TN>
struct RegTileFor<float, TM, TN, true> { typedef RegTilePaired<TM, TN> type; };

// Interleaved register-tile layout: thread t (of TT along a dimension) owns
// elements g*TT*W + t*W + e for g < TILE/W, e < W.  Consecutive threads read
// consecutive W-vectors, so a warp's LDS.64/LDS.128 phases are conflict free.
template <int W>
__device__ __forceinline__ int tile_index(int i, int t, int TT) {
    return (i / W) * TT * W + t * W + (i % W);
}

template <typename T, int TILE, int W>
__device__ __forceinline__ void load_frag(T (&f)[TILE], const T* row, int t, int TT) {
#pragma unroll
    for (int g = 0; g < TILE / W; ++g) {
        const Vec<T, W> v = *reinterpret_cast<const Vec<T, W>*>(row + g * TT * W + t * W);
#pragma unroll
        for (int e = 0; e < W; ++e) f[g * W + e] = v.v[e];
    }
}

template <typename T>
struct DirectParams {
    int M, N, K;
    T alpha, beta;
    int ta, tb;
    const T* A; i64 lda;
    const T* B; i64 ldb;
    const T* C; i64 ldc;
    T* out; i64 ldo;
    int bm, bn, bk;  // run-time tile sizes when the template sizes are 0
};

template <typename T>
struct TiledParams {
    int Mp, Np, Kp, M, N;
    T alpha, beta;
    int use_c;    // beta != 0: read C (reference packs C only then)
    int vec_out;  // out/C rows are W-aligned: vector epilogue allowed
    const T* At; i64 lda;  // Kp x Mp, op(A)^T, K-major, zero padded
    const T* Bp; i64 ldb;  // Kp x Np, op(B), zero padded
    const T* C; i64 ldc;
    T* out; i64 ldo;
    int bm, bn, bk, uk;
    int tiles_m, tiles_n, group_m;  // 1-D grid, grouped ("swizzled") tile order
    int splits, kt_per_split;       // split-K: blockIdx.y is the K slice
    T* partial;                     // splits x Mp x Np fp partial sums (splits > 1)
    int cluster_red;                // in-place core: the slices of a tile are one cluster, reduced over DSMEM
};

// thread bound of a kernel instantiation: exact for fixed tiles; for the
// run-time-tile kernels sized so the register tile never spills
template <typename T, int BM, int BN, int TM, int TN>
__host__ __device__ constexpr int cta_threads_bound() {
    return (BM > 0 && BN > 0) ? (BM / TM) * (BN / TN)
         : ((int)(TM * TN * sizeof(T) / 4) >= 32 ? 256 : ((int)(TM * TN * sizeof(T) / 4) >= 16 ? 512 : 1024));
}

// shared-memory footprint helpers (host + device)
template <typename T>
__host__ __device__ constexpr int direct_pad() { return VecW<T>::W; }

template <typename T>
__host__ __device__ inline size_t direct_smem_bytes(int bm, int bn, int bk) {
    return (size_t)2 * bk * ((bm + direct_pad<T>()) + (bn + direct_pad<T>())) * sizeof(T);
}
template <typename T>
__host__ __device__ inline size_t tiled_smem_bytes(int bm, int bn, int bk, int stages) {
    return (size_t)stages * bk * (bm + bn) * sizeof(T);
}
// pipeline depth of the indirect core: deep rings for small stages, capped
// so that one CTA fits the 227 KB shared memory of an sm_100 SM
template <typename T>
__host__ __device__ constexpr int tiled_stages(int bm, int bn, int bk) {
    return (bm == 0) ? 2
         : ((size_t)4 * bk * (bm + bn) * sizeof(T) <= 96 * 1024 ? 4
         : ((size_t)3 * bk * (bm + bn) * sizeof(T) <= 200 * 1024 ? 3 : 2));
}

// ---------------------------------------------------------------------------
// direct family
// ---------------------------------------------------------------------------
template <typename T, int BM_, int BN_, int BK_, int TM, int TN>
__global__ void __launch_bounds__(cta_threads_bound<T, BM_, BN_, TM, TN>())
direct_gemm_kernel(const DirectParams<T> p) {
    constexpr int PAD = direct_pad<T>();
    constexpr int WA = FragW<T, TM>::W;
    constexpr int WB = FragW<T, TN>::W;
    const int BM = BM_ > 0 ? BM_ : p.bm;
    const int BN = BN_ > 0 ? BN_ : p.bn;
    const int BK = BK_ > 0 ? BK_ : p.bk;
    const int TX = BN / TN, TY = BM / TM, NT = TX * TY;
    const int LA = BM + PAD, LB = BN + PAD;

    extern __shared__ __align__(16) unsigned char smem_raw[];
    T* As = reinterpret_cast<T*>(smem_raw);
    T* Bs = As + 2 * BK * LA;

    const int tid = threadIdx.x;
    const int tx = tid % TX, ty = tid / TX;
    const int m0 = blockIdx.y * BM, n0 = blockIdx.x * BN;
    const int M = p.M, N = p.N, K = p.K;

    typename RegTileFor<T, TM, TN>::type rt;
    rt.zero();

    auto load_tile = [&](int kt, int s) {
        const int k0 = kt * BK;
        T* as = As + s * BK * LA;
        T* bs = Bs + s * BK * LB;
        if (!p.ta) {  // A is M x K: walk k fastest (contiguous in global)
            for (int e = tid; e < BM * BK; e += NT) {
                const int k = e % BK, i = e / BK;
                const int gm = m0 + i, gk = k0 + k;
                const bool ok = gm < M && gk < K;
                const T* src = ok ? p.A + (i64)gm * p.lda + gk : p.A;
                cp_async<sizeof(T)>(as + k * LA + i, src, ok);
            }
        } else {  // A stored K x M: walk m fastest
            for (int e = tid; e < BM * BK; e += NT) {
                const int i = e % BM, k = e / BM;
                const int gm = m0 + i, gk = k0 + k;
                const bool ok = gm < M && gk < K;
                const T* src = ok ? p.A + (i64)gk * p.lda + gm : p.A;
                cp_async<sizeof(T)>(as + k * LA + i, src, ok);
            }
        }
        if (!p.tb) {  // B is K x N
            for (int e = tid; e < BK * BN; e += NT) {
                const int n = e % BN, k = e / BN;
                const int gn = n0 + n, gk = k0 + k;
                const bool ok = gn < N && gk < K;
                const T* src = ok ? p.B + (i64)gk * p.ldb + gn : p.B;
                cp_async<sizeof(T)>(bs + k * LB + n, src, ok);
            }
        } else {  // B stored N x K
            for (int e = tid; e < BK * BN; e += NT) {
                const int k = e % BK, n = e / BK;
                const int gn = n0 + n, gk = k0 + k;
                const bool ok = gn < N && gk < K;
                const T* src = ok ? p.B + (i64)gn * p.ldb + gk : p.B;
                cp_async<sizeof(T)>(bs + k * LB + n, src, ok);
            }
        }
    };

    const int nk = (K + BK - 1) / BK;
    load_tile(0, 0);
    cp_async_commit();
    for (int kt = 0; kt < nk; ++kt) {
        if (kt + 1 < nk) load_tile(kt + 1, (kt + 1) & 1);
        cp_async_commit();
        cp_async_wait<1>();
        __syncthreads();
        const T* as = As + (kt & 1) * BK * LA;
        const T* bs = Bs + (kt & 1) * BK * LB;
#pragma unroll 4
        for (int k = 0; k < BK; ++k) {
            T a[TM], b[TN];
            load_frag<T, TM, WA>(a, as + k * LA, ty, TY);
            load_frag<T, TN, WB>(b, bs + k * LB, tx, TX);
            rt.fma(a, b);
        }
        __syncthreads();
    }
    T acc[TM][TN];
    rt.unpack(acc);

    // out = alpha * acc + beta * C, C always read (kernels.py:227)
#pragma unroll
    for (int i = 0; i < TM; ++i) {
        const int gm = m0 + tile_index<WA>(i, ty, TY);
        if (gm >= M) continue;
#pragma unroll
        for (int j = 0; j < TN; ++j) {
            const int gn = n0 + tile_index<WB>(j, tx, TX);
            if (gn < N) {
                const T c = p.C[(i64)gm * p.ldc + gn];
                p.out[(i64)gm * p.ldo + gn] = fmadd(p.alpha, acc[i][j], p.beta * c);
            }
        }
    }
}

// ---------------------------------------------------------------------------
// indirect family: unpredicated multi-stage core on packed operands
// ---------------------------------------------------------------------------
// AROW: A is read straight from the caller's row-major M x K operand (no
// transpose-pack) with 4-byte copies transposed into the K-major tile; the
// A tile rows are padded by 4 elements to spread the transposing writes
// over the banks.  Used by the split-K family when M and K are tile
// multiples -- skinny memory-bound shapes, where the pack would double the
// A traffic.
template <typename T, bool AROW>
__host__ __device__ constexpr int a_pad() { return AROW ? 4 : 0; }

template <typename T, int BM_, int BN_, int BK_, int TM, int TN, int UK, int STAGES, bool AROW = false>
__global__ void __launch_bounds__(cta_threads_bound<T, BM_, BN_, TM, TN>())
tiled_gemm_kernel(const TiledParams<T> p) {
    pdl_wait();     // behind this call's packs (dependent launch), else a no-op
    pdl_trigger();  // the split-K reduction may launch while the last wave runs
    constexpr bool FIXED = BM_ > 0 && BN_ > 0 && BK_ > 0;
    static_assert(!AROW || FIXED, "row-major A needs fixed tiles");
    constexpr int VL = FIXED ? VecW<T>::W : 1;  // elements per cp.async
    constexpr int WA = FragW<T, TM>::W;
    constexpr int WB = FragW<T, TN>::W;
    const int BM = FIXED ? BM_ : p.bm;
    const int BN = FIXED ? BN_ : p.bn;
    const int BK = FIXED ? BK_ : p.bk;
    const int TX = BN / TN, TY = BM / TM, NT = TX * TY;
    const int LA = BM + a_pad<T, AROW>();  // A tile row stride (elements)

    extern __shared__ __align__(16) unsigned char smem_raw[];
    T* As = reinterpret_cast<T*>(smem_raw);  // [STAGES][BK][LA]
    T* Bs = As + STAGES * BK * LA;            // [STAGES][BK][BN]

    const int tid = threadIdx.x;
    const int tx = tid % TX, ty = tid / TX;
    // grouped rasterisation: consecutive CTAs walk group_m row tiles of one
    // column band, so the band's B tiles and the group's A tiles stay in L2
    int tm_idx, tn_idx;
    {
        const int pid = blockIdx.x;
        const int per_group = p.group_m * p.tiles_n;
        const int first_m = (pid / per_group) * p.group_m;
        const int gsz = min(p.tiles_m - first_m, p.group_m);
        const int r = pid - (pid / per_group) * per_group;
        tm_idx = first_m + r % gsz;
        tn_idx = r / gsz;
    }
    const int m0 = tm_idx * BM, n0 = tn_idx * BN;

    typename RegTileFor<T, TM, TN>::type rt;
    rt.zero();

    // K-major packed A: row k of the tile is contiguous; row-major A (AROW):
    // row i of the tile is contiguous along k
    const T* gA = AROW ? p.At + (i64)m0 * p.lda : p.At + m0;
    const T* gB = p.Bp + n0;
    // fixed tiles: chunk loops with compile-time trip counts (fully unrolled,
    // predicated only when the chunk count is not a multiple of the CTA size)
    constexpr int NT_C = FIXED ? (BM_ / TM) * (BN_ / TN) : 1;
    constexpr int CA_C = FIXED ? BK_ * BM_ / VL : 0;
    constexpr int CB_C = FIXED ? BK_ * BN_ / VL : 0;
    constexpr int LA_C = BM_ + a_pad<T, AROW>();
    auto load_tile = [&](int kt, int s) {
        const int k0 = kt * BK;
        T* as = As + s * BK * LA;
        T* bs = Bs + s * BK * BN;
        if constexpr (FIXED && AROW) {
            // element copies, k fastest (coalesced rows), transposed into As[k][i]
            constexpr int EA = BK_ * BM_;
#pragma unroll
            for (int it = 0; it < (EA + NT_C - 1) / NT_C; ++it) {
                const int e = tid + it * NT_C;
                if (EA % NT_C == 0 || e < EA) {
                    const int k = e % BK_, i = e / BK_;
                    cp_async<sizeof(T)>(as + k * LA_C + i, gA + (i64)i * p.lda + k0 + k);
                }
            }
        }
        if constexpr (FIXED) {
            constexpr int ca = BM_ / VL, cb = BN_ / VL;
#pragma unroll
            for (int it = 0; it < (CA_C + NT_C - 1) / NT_C; ++it) {
                if constexpr (AROW) break;
                const int e = tid + it * NT_C;
                if (CA_C % NT_C == 0 || e < CA_C) {
                    const int k = e / ca, c = e - k * ca;
                    cp_async<VL * sizeof(T)>(as + k * BM_ + c * VL, gA + (i64)(k0 + k) * p.lda + c * VL);
                }
            }
#pragma unroll
            for (int it = 0; it < (CB_C + NT_C - 1) / NT_C; ++it) {
                const int e = tid + it * NT_C;
                if (CB_C % NT_C == 0 || e < CB_C) {
                    const int k = e / cb, c = e - k * cb;
                    cp_async<VL * sizeof(T)>(bs + k * BN_ + c * VL, gB + (i64)(k0 + k) * p.ldb + c * VL);
                }
            }
        } else {
            const int ca = BM / VL, cb = BN / VL;
            for (int e = tid; e < BK * ca; e += NT) {
                const int k = e / ca, c = e - k * ca;
                cp_async<VL * sizeof(T)>(as + k * BM + c * VL, gA + (i64)(k0 + k) * p.lda + c * VL);
            }
            for (int e = tid; e < BK * cb; e += NT) {
                const int k = e / cb, c = e - k * cb;
                cp_async<VL * sizeof(T)>(bs + k * BN + c * VL, gB + (i64)(k0 + k) * p.ldb + c * VL);
            }
        }
    };

    // this CTA's K range: all K tiles, or one split-K slice of them
    const int kt0 = blockIdx.y * p.kt_per_split;
    const int nk = min(p.Kp / BK - kt0, p.kt_per_split);
    gA += AROW ? (i64)kt0 * BK : (i64)kt0 * BK * p.lda;
    gB += (i64)kt0 * BK * p.ldb;
#pragma unroll
    for (int s = 0; s < STAGES - 1; ++s) {
        if (s < nk) load_tile(s, s);
        cp_async_commit();
    }
    const int uk = FIXED ? UK : p.uk;
    for (int kt = 0; kt < nk; ++kt) {
        cp_async_wait<STAGES - 2>();
        __syncthreads();
        {
            const int nt = kt + STAGES - 1;
            if (nt < nk) load_tile(nt, nt % STAGES);
            cp_async_commit();
        }
        const int s = kt % STAGES;
        const T* as = As + s * BK * LA;
        const T* bs = Bs + s * BK * BN;
        if (FIXED) {
#pragma unroll
            for (int k = 0; k < BK; k += UK) {
                T a[UK][TM], b[UK][TN];
#pragma unroll
                for (int u = 0; u < UK; ++u) {
                    load_frag<T, TM, WA>(a[u], as + (k + u) * LA_C, ty, TY);
                    load_frag<T, TN, WB>(b[u], bs + (k + u) * BN, tx, TX);
                }
#pragma unroll
                for (int u = 0; u < UK; ++u) rt.fma(a[u], b[u]);
            }
        } else {
            for (int k = 0; k < BK; k += uk) {
                for (int u = 0; u < uk; ++u) {
                    T a[TM], b[TN];
                    load_frag<T, TM, WA>(a, as + (k + u) * BM, ty, TY);
                    load_frag<T, TN, WB>(b, bs + (k + u) * BN, tx, TX);
                    rt.fma(a, b);
                }
            }
        }
    }
    cp_async_wait<0>();
    T acc[TM][TN];
    rt.unpack(acc);

    if (p.splits > 1) {
        // split-K: raw partial sums into this slice's padded Mp x Np slab;
        // splitk_reduce_kernel adds the slices in order (deterministic)
        T* slab = p.partial + (i64)blockIdx.y * p.Mp * p.Np;
#pragma unroll
        for (int i = 0; i < TM; ++i) {
            const int gm = m0 + tile_index<WA>(i, ty, TY);
#pragma unroll
            for (int g = 0; g < TN / WB; ++g) {
                const int gn = n0 + g * TX * WB + tx * WB;
                Vec<T, WB> o;
#pragma unroll
                for (int e = 0; e < WB; ++e) o.v[e] = acc[i][g * WB + e];
                *reinterpret_cast<Vec<T, WB>*>(slab + (i64)gm * p.Np + gn) = o;
            }
        }
        return;
    }

    // masked store epilogue (replaces outp + unpad copy, kernels.py:322-325)
    const bool full = (m0 + BM <= p.M) && (n0 + BN <= p.N);
    if (full && p.vec_out) {
#pragma unroll
        for (int i = 0; i < TM; ++i) {
            const int gm = m0 + tile_index<WA>(i, ty, TY);
#pragma unroll
            for (int g = 0; g < TN / WB; ++g) {
                const int gn = n0 + g * TX * WB + tx * WB;
                Vec<T, WB> o;
                if (p.use_c) {
                    const Vec<T, WB> c = *reinterpret_cast<const Vec<T, WB>*>(p.C + (i64)gm * p.ldc + gn);
#pragma unroll
                    for (int e = 0; e < WB; ++e) o.v[e] = fmadd(p.alpha, acc[i][g * WB + e], p.beta * c.v[e]);
                } else {
#pragma unroll
                    for (int e = 0; e < WB; ++e) o.v[e] = p.alpha * acc[i][g * WB + e];
                }
                *reinterpret_cast<Vec<T, WB>*>(p.out + (i64)gm * p.ldo + gn) = o;
            }
        }
    } else {
#pragma unroll
        for (int i = 0; i < TM; ++i) {
            const int gm = m0 + tile_index<WA>(i, ty, TY);
            if (gm >= p.M) continue;
#pragma unroll
            for (int j = 0; j < TN; ++j) {
                const int gn = n0 + tile_index<WB>(j, tx, TX);
                if (gn >= p.N) continue;
                T v = p.alpha * acc[i][j];
                if (p.use_c) v = fmadd(p.alpha, acc[i][j], p.beta * p.C[(i64)gm * p.ldc + gn]);
                p.out[(i64)gm * p.ldo + gn] = v;
            }
        }
    }
}

// ---------------------------------------------------------------------------
// in-place core (split-K family): no pack passes.  op(A) = the caller's
// row-major A and op(B) = the caller's row-major B are streamed with 16-byte
// cp.async straight from their own layouts, zero-filled past M, N and the
// slice's K end (K and N multiples of 4, 16-byte aligned rows; the launcher
// checks).  The A stage is row-major in shared memory ([BM][BK + 4], rows
// 16-byte aligned, an odd number of 16-byte chunks apart so a warp's
// LDS.128 over consecutive rows is conflict free); each thread reads 4 k
// of a row with one LDS.128 and applies them in k order, so every output
// element sees exactly the FMA sequence of the packed core: the zero fill is
// the pack's zero padding, and the result is bit-identical to it.  Thread
// rows are strided by TY (row r = i * TY + ty), B columns interleaved as in
// the packed core.
template <int BM, int BN, int BK, int TM, int TN, int STAGES>
__global__ void __launch_bounds__((BM / TM) * (BN / TN), ((BM / TM) * (BN / TN) >= 256 && TM * TN <= 64) ? 2 : 1)
inplace_gemm_kernel(const TiledParams<float> p, int K) {
    pdl_trigger();  // slab path: the reduction kernel may launch early
    static_assert(BK % 4 == 0 && BN % 4 == 0, "16-byte chunks");
    constexpr int TX = BN / TN, TY = BM / TM, NT = TX * TY;
    constexpr int LA = BK + 4;  // A stage row stride (floats): 16-byte aligned, odd in chunks when BK % 8 == 0
    constexpr int WB = FragW<float, TN>::W;
    constexpr int CA = BM * (BK / 4), CB = BK * (BN / 4);
    // k values per A fragment load: one LDS.128 per row per 4 k (2-k LDS.64
    // loads measured the same; the 8 x 8 tile fits 128 registers either way)
    constexpr int KV = 4;

    extern __shared__ __align__(16) unsigned char smem_raw[];
    float* As = reinterpret_cast<float*>(smem_raw);  // [STAGES][BM][LA]
    float* Bs = As + STAGES * BM * LA;                // [STAGES][BK][BN]

    const int tid = threadIdx.x;
    const int tx = tid % TX, ty = tid / TX;
    int tm_idx, tn_idx;
    {
        const int pid = blockIdx.x;
        const int per_group = p.group_m * p.tiles_n;
        const int first_m = (pid / per_group) * p.group_m;
        const int gsz = min(p.tiles_m - first_m, p.group_m);
        const int r = pid - (pid / per_group) * per_group;
        tm_idx = first_m + r % gsz;
        tn_idx = r / gsz;
    }
    const int m0 = tm_idx * BM, n0 = tn_idx * BN;
    const int kt0 = blockIdx.y * p.kt_per_split;
    const int k_begin = kt0 * BK;
    const int k_end = min(K, k_begin + p.kt_per_split * BK);
    const int nk = (k_end - k_begin + BK - 1) / BK;

    typename RegTileFor<float, TM, TN>::type rt;
    rt.zero();

    auto load_tile = [&](int kt, int s) {
        const int k0 = k_begin + kt * BK;
        float* as = As + s * BM * LA;
        float* bs = Bs + s * BK * BN;
#pragma unroll
        for (int it = 0; it < (CA + NT - 1) / NT; ++it) {
            const int e = tid + it * NT;
            if (CA % NT == 0 || e < CA) {
                const int i = e / (BK / 4), c = e - i * (BK / 4);
                const int gm = m0 + i, gk = k0 + 4 * c;
                const bool ok = gm < p.M && gk < k_end;
                cp_async<16>(as + i * LA + 4 * c, ok ? p.At + (i64)gm * p.lda + gk : p.At, ok);
            }
        }
#pragma unroll
        for (int it = 0; it < (CB + NT - 1) / NT; ++it) {
            const int e = tid + it * NT;
            if (CB % NT == 0 || e < CB) {
                const int k = e / (BN / 4), c = e - k * (BN / 4);
                const int gk = k0 + k, gn = n0 + 4 * c;
                const bool ok = gk < k_end && gn < p.N;
                cp_async<16>(bs + k * BN + 4 * c, ok ? p.Bp + (i64)gk * p.ldb + gn : p.Bp, ok);
            }
        }
    };

#pragma unroll
    for (int s = 0; s < STAGES - 1; ++s) {
        if (s < nk) load_tile(s, s);
        cp_async_commit();
    }
    for (int kt = 0; kt < nk; ++kt) {
        cp_async_wait<STAGES - 2>();
        __syncthreads();
        {
            const int nt = kt + STAGES - 1;
            if (nt < nk) load_tile(nt, nt % STAGES);
            cp_async_commit();
        }
        const int s = kt % STAGES;
        const float* as = As + s * BM * LA;
        const float* bs = Bs + s * BK * BN;
#pragma unroll
        for (int k4 = 0; k4 < BK; k4 += KV) {
            float av[TM][KV];
#pragma unroll
            for (int i = 0; i < TM; ++i) {
                const Vec<float, KV> v = *reinterpret_cast<const Vec<float, KV>*>(as + (i * TY + ty) * LA + k4);
#pragma unroll
                for (int e = 0; e < KV; ++e) av[i][e] = v.v[e];
            }
#pragma unroll
            for (int kk = 0; kk < KV; ++kk) {
                float a[TM], b[TN];
#pragma unroll
                for (int i = 0; i < TM; ++i) a[i] = av[i][kk];
                load_frag<float, TN, WB>(b, bs + (k4 + kk) * BN, tx, TX);
                rt.fma(a, b);
            }
        }
    }
    cp_async_wait<0>();
    float acc[TM][TN];
    rt.unpack(acc);

    if (p.splits > 1 && p.cluster_red) {
        // The splits slice-CTAs of this tile are one cluster (cluster dims
        // 1 x splits).  Each parks its partial tile in its own shared memory;
        // after a cluster barrier, CTA z sums its share of the tile's
        // elements over the slices in order 0..splits-1 through DSMEM --
        // the order of splitk_reduce_kernel, so the same bits, in one launch
        // with no partial slabs in HBM.
        __syncthreads();  // the stage ring is free: reuse it for the partial tile
        float* part = As;  // [BM][BN]
#pragma unroll
        for (int i = 0; i < TM; ++i) {
            const int r = i * TY + ty;
#pragma unroll
            for (int g = 0; g < TN / WB; ++g) {
                Vec<float, WB> o;
#pragma unroll
                for (int e = 0; e < WB; ++e) o.v[e] = acc[i][g * WB + e];
                *reinterpret_cast<Vec<float, WB>*>(part + r * BN + g * TX * WB + tx * WB) = o;
            }
        }
        asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;\n" ::: "memory");
        const int S = p.splits, z = blockIdx.y;
        constexpr int Q = BM * BN / 4;  // float4 chunks of the tile
        const int q0 = (int)((long long)Q * z / S), q1 = (int)((long long)Q * (z + 1) / S);
        const uint32_t local = smem_addr(part);
        for (int q = q0 + tid; q < q1; q += NT) {
            float4 sum;
            for (int src = 0; src < S; ++src) {
                uint32_t remote;
                asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(remote) : "r"(local + q * 16), "r"(src));
                float4 v;
                asm volatile("ld.shared::cluster.v4.f32 {%0, %1, %2, %3}, [%4];"
                             : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "r"(remote));
                if (src == 0) {
                    sum = v;
                } else {
                    sum.x += v.x; sum.y += v.y; sum.z += v.z; sum.w += v.w;
                }
            }
            const int r = (q * 4) / BN, c = (q * 4) % BN;
            const int gm = m0 + r;
            if (gm < p.M && p.vec_out && n0 + c + 4 <= p.N) {
                float4 o = make_float4(p.alpha * sum.x, p.alpha * sum.y, p.alpha * sum.z, p.alpha * sum.w);
                if (p.use_c) {
                    const float4 cc = *reinterpret_cast<const float4*>(p.C + (i64)gm * p.ldc + n0 + c);
                    o = make_float4(fmadd(p.alpha, sum.x, p.beta * cc.x), fmadd(p.alpha, sum.y, p.beta * cc.y),
                                    fmadd(p.alpha, sum.z, p.beta * cc.z), fmadd(p.alpha, sum.w, p.beta * cc.w));
                }
                *reinterpret_cast<float4*>(p.out + (i64)gm * p.ldo + n0 + c) = o;
            } else if (gm < p.M) {
                const float sv[4] = {sum.x, sum.y, sum.z, sum.w};
#pragma unroll
                for (int e = 0; e < 4; ++e) {
                    const int gn = n0 + c + e;
                    if (gn < p.N)
                        p.out[(i64)gm * p.ldo + gn] =
                            p.use_c ? fmadd(p.alpha, sv[e], p.beta * p.C[(i64)gm * p.ldc + gn]) : p.alpha * sv[e];
                }
            }
        }
        // no CTA may leave while a peer still reads its shared memory
        asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;\n" ::: "memory");
        return;
    }

    if (p.splits > 1) {  // raw partial sums into this slice's Mp x Np slab
        float* slab = p.partial + (i64)blockIdx.y * p.Mp * p.Np;
#pragma unroll
        for (int i = 0; i < TM; ++i) {
            const int gm = m0 + i * TY + ty;
#pragma unroll
            for (int g = 0; g < TN / WB; ++g) {
                const int gn = n0 + g * TX * WB + tx * WB;
                Vec<float, WB> o;
#pragma unroll
                for (int e = 0; e < WB; ++e) o.v[e] = acc[i][g * WB + e];
                *reinterpret_cast<Vec<float, WB>*>(slab + (i64)gm * p.Np + gn) = o;
            }
        }
        return;
    }
#pragma unroll
    for (int i = 0; i < TM; ++i) {
        const int gm = m0 + i * TY + ty;
        if (gm >= p.M) continue;
#pragma unroll
        for (int g = 0; g < TN / WB; ++g) {
            const int gn0 = n0 + g * TX * WB + tx * WB;
            if (p.vec_out && gn0 + WB <= p.N) {  // whole vector in range: one store
                Vec<float, WB> o;
                if (p.use_c) {
                    const Vec<float, WB> cc = *reinterpret_cast<const Vec<float, WB>*>(p.C + (i64)gm * p.ldc + gn0);
#pragma unroll
                    for (int e = 0; e < WB; ++e) o.v[e] = fmadd(p.alpha, acc[i][g * WB + e], p.beta * cc.v[e]);
                } else {
#pragma unroll
                    for (int e = 0; e < WB; ++e) o.v[e] = p.alpha * acc[i][g * WB + e];
                }
                *reinterpret_cast<Vec<float, WB>*>(p.out + (i64)gm * p.ldo + gn0) = o;
                continue;
            }
#pragma unroll
            for (int e = 0; e < WB; ++e) {
                const int gn = gn0 + e;
                if (gn >= p.N) continue;
                float v = p.alpha * acc[i][g * WB + e];
                if (p.use_c) v = fmadd(p.alpha, acc[i][g * WB + e], p.beta * p.C[(i64)gm * p.ldc + gn]);
                p.out[(i64)gm * p.ldo + gn] = v;
            }
        }
    }
}

// out = alpha * (sum over slices z = 0..splits-1, in order) + beta * C
// (C only when use_c): the fixed-order reduction of the split-K family
template <typename T>
__global__ void __launch_bounds__(256)
splitk_reduce_kernel(const T* __restrict__ partial, int splits, i64 slab, int Np, int M, int N, T alpha, T beta,
                     int use_c, const T* __restrict__ C, i64 ldc, T* __restrict__ out, i64 ldo) {
    pdl_wait();
    const i64 total = (i64)M * N;
    for (i64 idx = (i64)blockIdx.x * blockDim.x + threadIdx.x; idx < total; idx += (i64)gridDim.x * blockDim.x) {
        const int m = (int)(idx / N), n = (int)(idx - (i64)m * N);
        const T* src = partial + (i64)m * Np + n;
        T sum = src[0];
        for (int z = 1; z < splits; ++z) sum += src[z * slab];
        out[(i64)m * ldo + n] = use_c ? fmadd(alpha, sum, beta * C[(i64)m * ldc + n]) : alpha * sum;
    }
}

// ---------------------------------------------------------------------------
// helper passes and the parity oracle
// ---------------------------------------------------------------------------

// dst (dst_rows x dst_cols, ld_dst) = zero-padded L, where L (rows x cols) is
// src (ld_src) itself or, with `transpose`, src stored cols x rows.
// 32x32 tiles through shared memory keep both sides coalesced.
template <typename T>
__global__ void __launch_bounds__(256)
pack_pad_kernel(T* __restrict__ dst, i64 ld_dst, int dst_rows, int dst_cols,
                const T* __restrict__ src, i64 ld_src, int rows, int cols, int transpose) {
    pdl_trigger();
    __shared__ T tile[32][33];
    const int r0 = blockIdx.y * 32, c0 = blockIdx.x * 32;
    const int x = threadIdx.x, y = threadIdx.y;
    if (transpose) {
#pragma unroll
        for (int yy = y; yy < 32; yy += 8) {
            const int c = c0 + yy, r = r0 + x;  // src row c, col r (contiguous in r)
            tile[yy][x] = (r < rows && c < cols) ? src[(i64)c * ld_src + r] : T(0);
        }
        __syncthreads();
#pragma unroll
        for (int yy = y; yy < 32; yy += 8) {
            const int r = r0 + yy, c = c0 + x;
            if (r < dst_rows && c < dst_cols) dst[(i64)r * ld_dst + c] = tile[x][yy];
        }
    } else {
#pragma unroll
        for (int yy = y; yy < 32; yy += 8) {
            const int r = r0 + yy, c = c0 + x;
            if (r < dst_rows && c < dst_cols)
                dst[(i64)r * ld_dst + c] = (r < rows && c < cols) ? src[(i64)r * ld_src + c] : T(0);
        }
    }
}

// Non-transposing pack (dst = zero-padded copy of src): a flat grid-stride
// over the destination's 4-element quads, 4 quads per thread per step so 4
// loads are in flight; destination stores are 16-byte vectors (the packed
// buffers' rows are 16-byte multiples), source loads are vectors when the
// source rows allow it.  Replaces the 32 x 32 tile path for this case:
// 2048 x 8457 -> 2048 x 8576 went from 44.7 us (3.1 TB/s) to the copy rate.
template <typename T, bool SRC_VEC>
__global__ void __launch_bounds__(256)
pack_copy_kernel(T* __restrict__ dst, i64 ld_dst, int dst_rows, int dst_cols, const T* __restrict__ src,
                 i64 ld_src, int rows, int cols) {
    pdl_trigger();
    constexpr int W = VecW<T>::W;  // elements per 16 bytes
    const i64 qpr = dst_cols / W;
    const i64 total = (i64)dst_rows * qpr;
    const i64 stride = (i64)gridDim.x * blockDim.x;
    for (i64 q0 = (i64)blockIdx.x * blockDim.x + threadIdx.x; q0 < total; q0 += 4 * stride) {
        Vec<T, W> v[4];
        i64 r[4], c[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const i64 q = q0 + u * stride;
            r[u] = q / qpr;
            c[u] = (q - r[u] * qpr) * W;
            if (q >= total) continue;
            const T* sp = src + r[u] * ld_src + c[u];
            if (SRC_VEC && r[u] < rows && c[u] + W <= cols) {
                v[u] = *reinterpret_cast<const Vec<T, W>*>(sp);
            } else {
#pragma unroll
                for (int e = 0; e < W; ++e) v[u].v[e] = (r[u] < rows && c[u] + e < cols) ? __ldg(sp + e) : T(0);
            }
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            if (q0 + u * stride >= total) break;
            *reinterpret_cast<Vec<T, W>*>(dst + r[u] * ld_dst + c[u]) = v[u];
        }
    }
}

// Textbook (i, j, k) GEMM with float64 accumulation: every multiply and add
// separately rounded (no FMA contraction), k ascending, then
// alpha*acc + beta*C in float64 rounded once to T -- the same operation
// sequence as _kernel_reference (kernels.py:184-195), hence bit-identical.
template <typename T>
__global__ void __launch_bounds__(256)
reference_gemm_kernel(int M, int N, int K, double alpha, double beta, int ta, int tb,
                      const T* __restrict__ A, i64 lda, const T* __restrict__ B, i64 ldb,
                      const T* __restrict__ C, i64 ldc, T* __restrict__ out, i64 ldo) {
    const int j = blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= N) return;
    // rows strided over grid.y (<= 65535), so any M runs
    for (int i = blockIdx.y; i < M; i += gridDim.y) {
        double acc = 0.0;
        for (int k = 0; k < K; ++k) {
            const double a = (double)(ta ? A[(i64)k * lda + i] : A[(i64)i * lda + k]);
            const double b = (double)(tb ? B[(i64)j * ldb + k] : B[(i64)k * ldb + j]);
            acc = __dadd_rn(acc, __dmul_rn(a, b));
        }
        const double r = __dadd_rn(__dmul_rn(alpha, acc), __dmul_rn(beta, (double)C[(i64)i * ldc + j]));
        out[(i64)i * ldo + j] = (T)r;
    }
}

}  // namespace ag
