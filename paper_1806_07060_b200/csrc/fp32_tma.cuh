// fp32_tma.cuh -- the TMA-fed fp32 CUDA-core core (no pack passes).
//
// Same arithmetic as the packed indirect core (kernels.cuh tiled_gemm_kernel):
// a CTA tile BM x BN, K in steps of BK = 32, a TM x TN register tile per
// thread updated with FFMA2 in k order, the zero padding past M, N, K
// supplied by the TMA unit's out-of-bounds fill instead of a pack pass.  So
// every output element sees the same FMA sequence as the packed core and the
// result is bit-identical to it.
//
// Data movement, B200 style:
//   * op(A) = the caller's row-major A: TMA boxes of BM rows x 128 bytes of K
//     (SWIZZLE_128B: 16-byte chunk c of row r lands at c ^ (r & 7), so a
//     warp's LDS.128 over consecutive rows is conflict free);
//   * op(B) = the caller's row-major B: TMA boxes of 32 rows of k x BN
//     columns (no swizzle; fragment reads run along n);
//   * a STAGES-deep ring of full / empty mbarriers.  Thread 0 issues the TMA
//     for stage kt + STAGES - 1 once every warp has released that slot; the
//     other threads never touch a global address in the main loop (no
//     cp.async address math, no __syncthreads).
// Requirements (the launcher checks): no transposes, 16-byte aligned bases,
// K and N multiples of 4 (16-byte row strides for the TMA).
#pragma once
#include "kernels.cuh"
#include "launch.cuh"
#include "tc_kernels.cuh"

namespace ag {
namespace f32tma {

constexpr int BK = 32;  // one 128-byte swizzle row of A per k block

template <int BM, int BN>
constexpr size_t stage_bytes() {
    return (size_t)BM * BK * 4 + (size_t)BK * BN * 4;
}
template <int BM, int BN, int STAGES>
constexpr size_t smem_bytes() {
    return 1024 + STAGES * stage_bytes<BM, BN>() + 2 * STAGES * 8 + 64;
}
template <int BM, int BN>
constexpr int stages() {
    // 3-deep ring (2 CTAs of 128 x 128 per SM); 4 stages measured slower
    // (fewer resident CTAs), profiles/r01_exp_tiles_tma.jsonl
    return 3 * stage_bytes<BM, BN>() <= 110 * 1024 ? 3 : (2 * stage_bytes<BM, BN>() <= 200 * 1024 ? 2 : 1);
}

template <int BM, int BN, int TM, int TN, int STAGES>
__global__ void __launch_bounds__((BM / TM) * (BN / TN), ((BM / TM) * (BN / TN) >= 256 && TM * TN <= 64) ? 2 : 1)
tma_gemm_kernel(const __grid_constant__ CUtensorMap mapA, const __grid_constant__ CUtensorMap mapB,
                const TiledParams<float> p, int K) {
    constexpr int TX = BN / TN, TY = BM / TM, NT = TX * TY, NW = NT / 32;
    constexpr int WB = FragW<float, TN>::W;
    constexpr uint32_t A_BYTES = BM * BK * 4, B_BYTES = BK * BN * 4;
    constexpr int KV = TM * TN > 64 ? 2 : 4;
    static_assert(NT % 32 == 0, "whole warps");

    extern __shared__ uint8_t smem_raw[];
    // 1024-byte aligned (128-byte swizzle atoms); offset from the shared-window
    // address so the pointer stays in the shared space (LDS/STS, not generic)
    uint8_t* smem = smem_raw + ((1024u - (smem_addr(smem_raw) & 1023u)) & 1023u);
    uint8_t* sA = smem;                     // [STAGES][BM][128 B], 128-byte swizzle
    uint8_t* sB = smem + STAGES * A_BYTES;  // [STAGES][BK][BN] fp32
    uint64_t* full = reinterpret_cast<uint64_t*>(sB + STAGES * B_BYTES);
    uint64_t* empty = full + STAGES;

    const int tid = threadIdx.x, lane = tid & 31;
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
    const int nk = (K + BK - 1) / BK;

    if (tid == 0) {
        asm volatile("prefetch.tensormap [%0];\n" ::"l"(reinterpret_cast<uint64_t>(&mapA)) : "memory");
        asm volatile("prefetch.tensormap [%0];\n" ::"l"(reinterpret_cast<uint64_t>(&mapB)) : "memory");
        for (int s = 0; s < STAGES; ++s) {
            tc::mbar_init(&full[s], 1);
            tc::mbar_init(&empty[s], NW);
        }
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    }
    __syncthreads();

    auto issue = [&](int kt) {
        const int s = kt % STAGES;
        tc::mbar_expect_tx(&full[s], A_BYTES + B_BYTES);
        tc::tma_load_2d(sA + s * A_BYTES, &mapA, &full[s], kt * BK, m0);
        tc::tma_load_2d(sB + s * B_BYTES, &mapB, &full[s], n0, kt * BK);
    };
    if (tid == 0)
        for (int kt = 0; kt < STAGES - 1 && kt < nk; ++kt) issue(kt);

    typename RegTileFor<float, TM, TN>::type rt;
    rt.zero();
    for (int kt = 0; kt < nk; ++kt) {
        const int s = kt % STAGES;
        if (tid == 0) {  // refill the slot of block kt - 1 with block kt + STAGES - 1
            const int nt = kt + STAGES - 1;
            if (nt < nk) {
                if (nt >= STAGES) tc::mbar_wait(&empty[nt % STAGES], (uint32_t)((nt / STAGES - 1) & 1));
                issue(nt);
            }
        }
        tc::mbar_wait(&full[s], (uint32_t)((kt / STAGES) & 1));
        const uint8_t* as = sA + s * A_BYTES;
        const float* bs = reinterpret_cast<const float*>(sB + s * B_BYTES);
#pragma unroll
        for (int k0 = 0; k0 < BK; k0 += KV) {
            // KV consecutive k of each of the thread's rows: one LDS.128 (KV = 4)
            // or LDS.64 (KV = 2, wide register tiles) from the swizzled chunk
            float av[TM][KV];
#pragma unroll
            for (int i = 0; i < TM; ++i) {
                const int r = i * TY + ty;
                const Vec<float, KV> v = *reinterpret_cast<const Vec<float, KV>*>(
                    as + r * 128 + (((k0 >> 2) ^ (r & 7)) << 4) + (k0 & 3) * 4);
#pragma unroll
                for (int e = 0; e < KV; ++e) av[i][e] = v.v[e];
            }
#pragma unroll
            for (int kk = 0; kk < KV; ++kk) {
                float a[TM], b[TN];
#pragma unroll
                for (int i = 0; i < TM; ++i) a[i] = av[i][kk];
                load_frag<float, TN, WB>(b, bs + (k0 + kk) * BN, tx, TX);
                rt.fma(a, b);
            }
        }
        __syncwarp();
        if (lane == 0) tc::mbar_arrive(&empty[s]);
    }
    float acc[TM][TN];
    rt.unpack(acc);

#pragma unroll
    for (int i = 0; i < TM; ++i) {
        const int gm = m0 + i * TY + ty;
        if (gm >= p.M) continue;
#pragma unroll
        for (int g = 0; g < TN / WB; ++g) {
            const int gn0 = n0 + g * TX * WB + tx * WB;
            if (p.vec_out && gn0 + WB <= p.N) {
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

// fp32 row-major maps: A (M x K, box BK x BM, 128-byte swizzle), B (K x N, box BN x BK)
inline bool make_maps(CUtensorMap* mA, CUtensorMap* mB, const float* A, i64 lda, const float* B, i64 ldb, i64 M,
                      i64 N, i64 K, int bm, int bn) {
    auto fn = tc::encode_fn();
    if (!fn) return false;
    cuuint32_t estr[2] = {1, 1};
    cuuint64_t da[2] = {(cuuint64_t)K, (cuuint64_t)M}, sa[1] = {(cuuint64_t)(lda * 4)};
    cuuint32_t ba[2] = {(cuuint32_t)BK, (cuuint32_t)bm};
    cuuint64_t db[2] = {(cuuint64_t)N, (cuuint64_t)K}, sb[1] = {(cuuint64_t)(ldb * 4)};
    cuuint32_t bb[2] = {(cuuint32_t)bn, (cuuint32_t)BK};
    return fn(mA, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float*>(A), da, sa, ba, estr,
              CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
              CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS &&
           fn(mB, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float*>(B), db, sb, bb, estr,
              CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
              CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// whether the TMA core can take this call (row-major, 16-byte strides and bases)
inline bool eligible(const GemmCall& c) {
    return c.dtype == AG_F32 && !c.ta && !c.tb && c.K % 4 == 0 && c.N % 4 == 0 && c.lda % 4 == 0 &&
           c.ldb % 4 == 0 && aligned(c.A, 16) && aligned(c.B, 16);
}

template <int BM, int BN, int TM, int TN>
int launch_tma(const GemmCall& c) {
    static_assert(BM <= 256 && BN <= 256, "TMA box dimensions are at most 256");
    constexpr int STAGES = stages<BM, BN>();
    constexpr size_t smem = smem_bytes<BM, BN, STAGES>();
    static_assert(smem <= 227 * 1024, "stage ring exceeds shared memory");
    auto kernel = tma_gemm_kernel<BM, BN, TM, TN, STAGES>;
    static SmemGrant granted;
    if (ensure_smem(kernel, smem, granted) != cudaSuccess) return fail(c, AG_ERR_CUDA, "cudaFuncSetAttribute failed");
    const i64 M = c.M, N = c.N, K = c.K;
    const i64 tiles_m = (M + BM - 1) / BM, tiles_n = (N + BN - 1) / BN;
    if (tiles_m * tiles_n > 0x7fffffffLL || K > 0x7fffffffLL) return fail(c, AG_ERR_SHAPE, "problem too large");
    CUtensorMap mA, mB;
    if (!make_maps(&mA, &mB, static_cast<const float*>(c.A), c.lda, static_cast<const float*>(c.B), c.ldb, M, N, K,
                   BM, BN))
        return fail(c, AG_ERR_CUDA, "cuTensorMapEncodeTiled failed");
    TiledParams<float> p{};
    p.M = (int)M; p.N = (int)N;
    p.alpha = (float)c.alpha; p.beta = (float)c.beta;
    p.use_c = c.beta != 0.0;
    p.vec_out = (c.ldo % 4 == 0) && aligned(c.out, 16) && (!p.use_c || ((c.ldc % 4 == 0) && aligned(c.C, 16)));
    p.C = static_cast<const float*>(c.C); p.ldc = c.ldc;
    p.out = static_cast<float*>(c.out); p.ldo = c.ldo;
    p.tiles_m = (int)tiles_m; p.tiles_n = (int)tiles_n;
    p.group_m = group_rows(tiles_m, BM, round_up(K, BK), sizeof(float));
    p.splits = 1;
    kernel<<<(unsigned)(tiles_m * tiles_n), (BM / TM) * (BN / TN), smem, c.stream>>>(mA, mB, p, (int)K);
    return cudaGetLastError() == cudaSuccess ? AG_OK : fail(c, AG_ERR_CUDA, "TMA core launch failed");
}

}  // namespace f32tma
}  // namespace ag

namespace ag {
namespace f32tma {

// the "tma" family launcher: the TMA core when the operands allow it, else
// the packed core with the same tile (bk = 32, unroll 1) -- same bits
template <int BM, int BN, int TM, int TN>
int launch_tma_family(const GemmCall& c) {
    if (eligible(c)) return launch_tma<BM, BN, TM, TN>(c);
    return launch_indirect<float, BM, BN, BK, TM, TN, 1>(c);
}

}  // namespace f32tma
}  // namespace ag
