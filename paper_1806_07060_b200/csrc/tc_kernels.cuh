// tc_kernels.cuh -- the tensor-core families (B200 tc profile): tf32 and bf16.
//
// No reference analogue: the reference's two families are CUDA-core style
// loop nests (kernels.py:198-260).  These families serve the dense
// contraction on the 5th-generation tensor cores (BASELINE.json configs[4]).
// Operands are read where they lie, in either major: op(A) is K-major
// (MN-major when transA), op(B) is MN-major (K-major when transB); the
// tensor core takes both, so nothing is transposed or padded -- the TMA unit
// zero-fills boxes that run past M, N or K.  tf32 reads the caller's fp32
// matrices in place (the tensor core consumes the fp32 bits as tf32); bf16
// needs one streaming convert pass per operand (fp32 -> bf16, round to
// nearest even, layout kept), the helper pass of this family as the packs
// are the indirect family's (kernels.py:304-325).  The epilogue writes
// alpha * acc + beta * C, reading C only when beta != 0 (the indirect
// family's semantics, kernels.py:318-321).
//
// Core (tc_gemm_kernel): persistent, warp specialised, one CTA per SM.
//   warp 0 lane 0 : TMA producer -- cp.async.bulk.tensor 2D loads of the
//                   128 x BK A tile and BN x BK B tile (128-byte rows,
//                   SWIZZLE_128B) into a STAGES-deep ring guarded by
//                   full/empty mbarriers;
//   warp 1 lane 0 : MMA issuer -- tcgen05.mma.cta_group::1 (kind::tf32 or
//                   kind::f16), M = 128, N = BN, K = 8 / 16 per instruction,
//                   accumulating in TMEM; tcgen05.commit frees a smem stage
//                   and, after the last K block, publishes the accumulator;
//   warps 2..5    : epilogue -- tcgen05.ld 32x32b.x32 (one TMEM lane = one
//                   output row per thread), alpha/beta, masked stores.
// The accumulator is double buffered in TMEM (2 x BN fp32 columns) so the
// epilogue of tile i overlaps the main loop of tile i+1.
#pragma once
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>
#include <stdint.h>

#include <algorithm>
#include <cstring>
#include <atomic>
#include <mutex>

#include "kernels.cuh"
#include "launch.cuh"
#include "registry.h"

namespace ag {
namespace tc {

constexpr int KIND_TF32 = 0;
constexpr int KIND_BF16 = 1;
constexpr int KIND_TF32X3 = 2;  // fp32-accurate: 3 tf32 products over hi / lo operand parts
constexpr int BM = 128;          // UMMA M (cta_group::1): TMEM lane = output row
constexpr int ROW_BYTES = 128;   // one K block = one 128-byte swizzle row
constexpr int THREADS = 192;     // producer warp, MMA warp, 4 epilogue warps
constexpr int THREADS_X3 = 320;  // + 4 converter warps (tf32x3: the lo parts are made in shared memory)
constexpr int ACC_STAGES_MAX = 2;  // TMEM accumulator double buffer (when 2 buffers fit 512 columns)
constexpr int X3_CHUNK_BLOCKS = 8;  // 3xTF32: K blocks (8 x 32 = 256 k) per TMEM accumulation chunk

inline constexpr i64 round_up_i(i64 x, i64 s) { return (x + s - 1) / s * s; }

template <int KIND> struct Elem;
template <> struct Elem<KIND_TF32> {
    typedef float T;
    static constexpr int BK = ROW_BYTES / 4;  // 32 elements per K block
    static constexpr int UMMA_K = 8;
    static constexpr uint32_t FMT = 2;        // TF32
    static constexpr CUtensorMapDataType TMA = CU_TENSOR_MAP_DATA_TYPE_FLOAT32;
    static constexpr int PARTS = 1;           // operand parts staged per K block
};
template <> struct Elem<KIND_BF16> {
    typedef __nv_bfloat16 T;
    static constexpr int BK = ROW_BYTES / 2;  // 64 elements per K block
    static constexpr int UMMA_K = 16;
    static constexpr uint32_t FMT = 1;        // BF16
    static constexpr CUtensorMapDataType TMA = CU_TENSOR_MAP_DATA_TYPE_BFLOAT16;
    static constexpr int PARTS = 1;
};
// 3xTF32: x = hi + lo with hi = x with its low 13 mantissa bits cleared (the
// bits a tf32 MMA reads) and lo = x - hi (exact in fp32, |lo| < 2^-10 |x|).
// a.b ~ a_hi.b_hi + a_hi.b_lo + a_lo.b_hi: the dropped a_lo.b_lo and the
// tf32 truncation of the lo parts are below 2^-20 |a||b| per product, so the
// result meets the fp32 families' RF <= 1e-5 contract on the tensor pipe.
// A stage holds [hi | lo] of each operand: TMA lands the caller's fp32 tile
// (= hi as a tf32 MMA reads it), four converter warps write lo = x - hi next
// to it in shared memory (no HBM convert pass, half the L2 -> SM bytes of
// staging both parts), and the MMA issuer runs 3 tf32 MMAs per K step.
template <> struct Elem<KIND_TF32X3> : Elem<KIND_TF32> {
    static constexpr int PARTS = 2;
};
// 3xTF32 split: hi = the bits a tf32 MMA reads (low 13 mantissa bits
// cleared), lo = x - hi, exact in fp32
__host__ __device__ __forceinline__ float tf32_hi(float x) {
#ifdef __CUDA_ARCH__
    return __uint_as_float(__float_as_uint(x) & 0xFFFFE000u);
#else
    uint32_t u;
    std::memcpy(&u, &x, 4);
    u &= 0xFFFFE000u;
    std::memcpy(&x, &u, 4);
    return x;
#endif
}
__host__ __device__ __forceinline__ float tf32_lo(float x) { return x - tf32_hi(x); }
template <int KIND>
constexpr int kernel_threads() {
    return Elem<KIND>::PARTS == 2 ? THREADS_X3 : THREADS;
}

// ---------------------------------------------------------------- device PTX
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_addr(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_addr(bar)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(smem_addr(bar)) : "memory");
}
// wait until the phase with parity `parity` has completed
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    const uint32_t a = smem_addr(bar);
    uint32_t done = 0;
    do {
        asm volatile(
            "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
            : "=r"(done)
            : "r"(a), "r"(parity)
            : "memory");
    } while (!done);
}
__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, uint64_t* bar, int x, int y) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];\n" ::"r"(
            smem_addr(dst)),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_addr(bar)), "r"(x), "r"(y)
        : "memory");
}
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory"); }

// SWIZZLE_128B shared-memory matrix descriptors (sm_100 format: start
// address >> 4, LBO >> 4 at bit 16, SBO >> 4 at bit 32, version 1 at bit
// 46, layout type 2 = 128-byte swizzle at bit 61).
//  K-major  (a row of the tile = 128 bytes of K): SBO = 1024 B between
//           8-row groups; LBO unused.  One UMMA_K step = +32 bytes.
//  MN-major (a row of the tile = 128 bytes of M or N, one row per k):
//           SBO = 1024 B between 8-k groups, LBO = distance between the
//           128-byte MN chunks (BK * 128 B: each chunk is one TMA box of
//           BK rows).  One UMMA_K step = +UMMA_K * 128 bytes.
//           32-bit (tf32) MN-major operands use the 128-byte swizzle with
//           32-byte atoms instead (layout type 1, "128B_BASE32B": 32-byte
//           chunks XORed by k % 4, written by the TMA's SWIZZLE_128B_ATOM_32B
//           mode), so SBO = 512 B between 4-k groups.
__device__ __forceinline__ uint64_t sw128_desc(uint32_t saddr, uint32_t lbo_bytes = 16, uint32_t sbo_bytes = 1024,
                                               uint32_t layout = 2) {
    return (uint64_t)((saddr & 0x3FFFFu) >> 4) | ((uint64_t)(lbo_bytes >> 4) << 16) |
           ((uint64_t)(sbo_bytes >> 4) << 32) | ((uint64_t)1 << 46) | ((uint64_t)layout << 61);
}

// instruction descriptor: D f32, A/B format, A/B major (0 = K, 1 = MN),
// N >> 3, M >> 4 (M = 128 per CTA, 256 for a CTA pair)
template <int KIND>
__host__ __device__ constexpr uint32_t instr_desc(int m, int n, int a_mn, int b_mn) {
    return (1u << 4) | (Elem<KIND>::FMT << 7) | (Elem<KIND>::FMT << 10) | ((uint32_t)a_mn << 15) |
           ((uint32_t)b_mn << 16) | ((uint32_t)(n >> 3) << 17) | ((uint32_t)(m >> 4) << 24);
}

template <int KIND>
__device__ __forceinline__ void umma(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc, uint32_t acc) {
    if constexpr (KIND != KIND_BF16) {
        asm volatile(
            "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
            " tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem_d),
            "l"(adesc), "l"(bdesc), "r"(idesc), "r"(acc));
    } else {
        asm volatile(
            "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
            " tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem_d),
            "l"(adesc), "l"(bdesc), "r"(idesc), "r"(acc));
    }
}
__device__ __forceinline__ void umma_commit(uint64_t* bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(smem_addr(bar))
                 : "memory");
}

// 32 lanes x 32 consecutive fp32 columns: thread t gets row (lane base + t)
__device__ __forceinline__ void tmem_ld32(uint32_t taddr, uint32_t (&v)[32]) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, "
        "%15, %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31}, [%32];\n"
        : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
          "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15]),
          "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]),
          "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
        : "r"(taddr));
    asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
}

struct TcParams {
    int M, N, tiles_m, tiles_n, k_blocks, group_m;
    int a_mn, b_mn;   // operand majors: 0 = K-major, 1 = MN-major
    uint32_t idesc;
    float alpha, beta;
    int use_c, vec_out;
    const float* C;
    i64 ldc;
    float* out;
    i64 ldo;
};

// grouped rasterisation: `group_m` tile rows per group, column-major inside
__device__ __forceinline__ void tile_coords(const TcParams& p, int t, int& tm, int& tn) {
    const int per_group = p.group_m * p.tiles_n;
    const int g = t / per_group, r = t - g * per_group;
    const int first = g * p.group_m;
    const int gs = min(p.tiles_m - first, p.group_m);
    tm = first + r % gs;
    tn = r / gs;
}

// one accumulator buffer = ACC_PARTS x BN fp32 columns (3xTF32 keeps its two
// small products in a second accumulator); double buffered when two fit
template <int BN, int ACC_PARTS>
constexpr int acc_stages() {
    return 2 * ACC_PARTS * BN <= 512 ? ACC_STAGES_MAX : 1;
}
template <int BN, int ACC_PARTS = 1>
constexpr uint32_t tmem_cols() {
    constexpr int c = acc_stages<BN, ACC_PARTS>() * ACC_PARTS * BN;
    return c <= 32 ? 32 : c <= 64 ? 64 : c <= 128 ? 128 : c <= 256 ? 256 : 512;
}

// per-CTA shared memory: the stage ring (A: 128 rows, B: BN / CTAS rows of
// 128 bytes per stage) + alignment slack + barriers
// epilogue staging: one 32 x 32 fp32 block per epilogue warp, rows padded
// to 36 floats (144 bytes: 16-byte aligned rows, conflict-free STS.128 /
// LDS.128 phases)
constexpr int EPI_LD = 36;
constexpr size_t EPI_BYTES = 4 * 32 * EPI_LD * sizeof(float);

template <int BN, int STAGES, int CTAS, int PARTS = 1>
constexpr size_t smem_bytes() {
    return 1024 + (size_t)STAGES * PARTS * (BM + BN / CTAS) * ROW_BYTES + EPI_BYTES + 256;
}

__device__ __forceinline__ uint32_t cluster_rank() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;\n" : "=r"(r));
    return r;
}
__device__ __forceinline__ void cluster_sync() {
    asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;\n" ::: "memory");
}
// 2-CTA TMA: lands in this CTA's shared memory, completes the transaction
// on the leader CTA's barrier (shared::cluster address with the peer bit
// cleared)
__device__ __forceinline__ void tma_load_2d_pair(void* dst, const CUtensorMap* map, uint32_t leader_bar, int x,
                                                 int y) {
    asm volatile(
        "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, "
        "%4}], [%2];\n" ::"r"(smem_addr(dst)),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(leader_bar), "r"(x), "r"(y)
        : "memory");
}
template <int KIND>
__device__ __forceinline__ void umma_pair(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                          uint32_t acc) {
    if constexpr (KIND != KIND_BF16) {
        asm volatile(
            "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
            " tcgen05.mma.cta_group::2.kind::tf32 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem_d),
            "l"(adesc), "l"(bdesc), "r"(idesc), "r"(acc));
    } else {
        asm volatile(
            "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
            " tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem_d),
            "l"(adesc), "l"(bdesc), "r"(idesc), "r"(acc));
    }
}
// commit the pair's MMAs to the same barrier offset in both CTAs
__device__ __forceinline__ void umma_commit_pair(uint64_t* bar) {
    asm volatile(
        "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;\n" ::"r"(
            smem_addr(bar)),
        "h"((uint16_t)0x3)
        : "memory");
}
__device__ __forceinline__ void mbar_arrive_remote(uint64_t* bar, uint32_t cta) {
    uint32_t remote;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;\n" : "=r"(remote) : "r"(smem_addr(bar)), "r"(cta));
    asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];\n" ::"r"(remote) : "memory");
}

// CTAS = 1: one CTA per SM, UMMA M = 128.  CTAS = 2: a CTA pair on the two
// SMs of a TPC (cluster of 2) runs tcgen05.mma.cta_group::2 with M = 256:
// each CTA stages its own 128 rows of A and half of the BN columns of B,
// the leader CTA issues the MMAs for both, and each CTA's TMEM holds its
// 128 output rows.  Per SM this halves the B traffic of a 128 x BN tile.
template <int KIND, int BN, int STAGES, int CTAS>
__global__ void __launch_bounds__(kernel_threads<KIND>(), 1)
tc_gemm_kernel(const __grid_constant__ CUtensorMap mapA, const __grid_constant__ CUtensorMap mapB, TcParams p) {
    constexpr int BK = Elem<KIND>::BK;
    constexpr int PARTS = Elem<KIND>::PARTS;  // [hi | lo] per operand and stage for 3xTF32
    constexpr int BNC = BN / CTAS;  // B rows (N) staged by each CTA
    constexpr uint32_t A_BYTES = BM * ROW_BYTES, B_BYTES = BNC * ROW_BYTES;  // one part
    // TMA bytes per stage: the raw fp32 tiles; 3xTF32 lands them on each CTA's
    // own barrier (its converter warps wait there), the other kinds on the
    // leader's (the pair's MMA issuer waits there)
    constexpr uint32_t STAGE_TX = PARTS == 2 ? (A_BYTES + B_BYTES) : (A_BYTES + B_BYTES) * CTAS;
    // The tensor core's fp32 accumulation is not round-to-nearest: with exact
    // products (tf32-truncated inputs) its error grows linearly in K (RF
    // 6.0e-6 at K = 2560, 1.9e-5 at 8192, 7.7e-5 at 32768, against 0.9e-6 /
    // 1.6e-6 / 3.2e-6 for FFMA; profiles/r02_tc_accuracy.jsonl).  3xTF32
    // therefore accumulates in TMEM over chunks of KC K blocks only: each
    // chunk's accumulator is drained by the epilogue warps and added in IEEE
    // fp32 to a per-thread running sum (one output row per thread, BN <= 128
    // registers), while the MMA issuer fills the other TMEM buffer.
    constexpr int KC = PARTS == 2 ? X3_CHUNK_BLOCKS : 0;  // 0: the whole K range in TMEM
    static_assert(KC == 0 || BN <= 128, "3xTF32 keeps a BN-wide fp32 running sum per epilogue thread");
    constexpr int ACC_STAGES = acc_stages<BN, 1>();
    constexpr uint32_t ACC_COLS = (uint32_t)BN;
    constexpr uint32_t TMEM_COLS = tmem_cols<BN, 1>();
    constexpr int K_STEPS = BK / Elem<KIND>::UMMA_K;
    constexpr int CH = ROW_BYTES / (int)sizeof(typename Elem<KIND>::T);  // elements per 128-byte MN chunk
    constexpr uint32_t CHUNK_BYTES = BK * ROW_BYTES;                      // one MN chunk of one stage
    constexpr uint32_t MN_SBO = KIND != KIND_BF16 ? 512 : 1024;           // see sw128_desc
    constexpr uint32_t MN_LAYOUT = KIND != KIND_BF16 ? 1 : 2;
    static_assert(BN % 32 == 0 && BN >= 32 && BN <= 256, "UMMA N is 16..256; the epilogue drains 32 columns");
    static_assert(CTAS == 1 || CTAS == 2, "one CTA or a CTA pair");
    static_assert(BNC % CH == 0 || CTAS == 1, "pair tiles split B into whole 128-byte chunks");

    extern __shared__ uint8_t smem_raw[];
    // 1024-byte aligned (128-byte swizzle atoms); offset from the shared-window
    // address so the pointer stays in the shared space (LDS/STS, not generic)
    uint8_t* smem = smem_raw + ((1024u - (smem_addr(smem_raw) & 1023u)) & 1023u);
    uint8_t* sA = smem;                              // [STAGES][PARTS][A_BYTES]
    uint8_t* sB = smem + STAGES * PARTS * A_BYTES;   // [STAGES][PARTS][B_BYTES]
    float* sEpi = reinterpret_cast<float*>(sB + STAGES * PARTS * B_BYTES);
    uint64_t* full = reinterpret_cast<uint64_t*>(sB + STAGES * PARTS * B_BYTES + EPI_BYTES);
    uint64_t* empty = full + STAGES;
    uint64_t* tfull = empty + STAGES;
    uint64_t* tempty = tfull + ACC_STAGES;
    uint64_t* lo_full = tempty + ACC_STAGES;  // 3xTF32: lo parts of a stage written (converter warps, all CTAs)
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(lo_full + STAGES);

    const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
    const uint32_t rank = CTAS == 2 ? cluster_rank() : 0;
    const int unit = blockIdx.x / CTAS, units = gridDim.x / CTAS;  // one unit = one CTA or one pair
    if (warp == 0 && lane == 0) {
        asm volatile("prefetch.tensormap [%0];\n" ::"l"(reinterpret_cast<uint64_t>(&mapA)) : "memory");
        asm volatile("prefetch.tensormap [%0];\n" ::"l"(reinterpret_cast<uint64_t>(&mapB)) : "memory");
        for (int s = 0; s < STAGES; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], 1);
        }
        for (int a = 0; a < ACC_STAGES; ++a) {
            mbar_init(&tfull[a], 1);
            mbar_init(&tempty[a], 4 * CTAS);  // one arrival per epilogue warp of every CTA
        }
        if constexpr (PARTS == 2)
            for (int s = 0; s < STAGES; ++s) mbar_init(&lo_full[s], 4 * CTAS);  // one per converter warp and CTA
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    }
    if (warp == 1) {
        if constexpr (CTAS == 1) {
            asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(
                             smem_addr(tmem_slot)),
                         "n"(TMEM_COLS)
                         : "memory");
            asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n" ::: "memory");
        } else {
            asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(
                             smem_addr(tmem_slot)),
                         "n"(TMEM_COLS)
                         : "memory");
            asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;\n" ::: "memory");
        }
    }
    tc_fence_before();
    if constexpr (CTAS == 2) {
        cluster_sync();  // the peer's barriers are initialised before any remote arrive
    } else {
        __syncthreads();
    }
    tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;
    const int tiles = p.tiles_m * p.tiles_n;

    if (warp == 0) {
        if (lane == 0) {  // ---- TMA producer (every CTA stages its own share)
            // programmatic dependent launch: the setup above (barriers, TMEM,
            // tensormap prefetch) overlapped the staging convert's tail; no
            // operand byte is read before the upstream grid has completed.
            // Every other read / write of this kernel (C, out) happens after
            // the first full barrier, i.e. after this wait.
            asm volatile("griddepcontrol.wait;\n" ::: "memory");
            int stage = 0;
            uint32_t phase = 0;
            for (int t = unit; t < tiles; t += units) {
                int tm, tn;
                tile_coords(p, t, tm, tn);
                const int m0 = tm * BM * CTAS + (int)rank * BM, n0 = tn * BN + (int)rank * BNC;
                for (int kb = 0; kb < p.k_blocks; ++kb) {
                    mbar_wait(&empty[stage], phase ^ 1);
                    if constexpr (CTAS == 1 || PARTS == 2) {
                        mbar_expect_tx(&full[stage], STAGE_TX);
                    } else {
                        if (rank == 0) mbar_expect_tx(&full[stage], STAGE_TX);
                    }
                    // TMA loads the raw tiles (3xTF32: its lo parts are made in smem)
                    {
                        uint8_t* a = sA + stage * PARTS * A_BYTES;
                        uint8_t* b = sB + stage * PARTS * B_BYTES;
                        const CUtensorMap* ma = &mapA;
                        const CUtensorMap* mb = &mapB;
                        if constexpr (CTAS == 1 || PARTS == 2) {  // this CTA's own barrier
                            if (!p.a_mn) {
                                tma_load_2d(a, ma, &full[stage], kb * BK, m0);
                            } else {
#pragma unroll
                                for (int c = 0; c < BM / CH; ++c)
                                    tma_load_2d(a + c * CHUNK_BYTES, ma, &full[stage], m0 + c * CH, kb * BK);
                            }
                            if (!p.b_mn) {
                                tma_load_2d(b, mb, &full[stage], kb * BK, n0);
                            } else {
#pragma unroll
                                for (int c = 0; c < BNC / CH; ++c)
                                    tma_load_2d(b + c * CHUNK_BYTES, mb, &full[stage], n0 + c * CH, kb * BK);
                            }
                        } else {
                            const uint32_t bar = smem_addr(&full[stage]) & 0xFEFFFFFFu;  // leader's barrier
                            if (!p.a_mn) {
                                tma_load_2d_pair(a, ma, bar, kb * BK, m0);
                            } else {
#pragma unroll
                                for (int c = 0; c < BM / CH; ++c)
                                    tma_load_2d_pair(a + c * CHUNK_BYTES, ma, bar, m0 + c * CH, kb * BK);
                            }
                            if (!p.b_mn) {
                                tma_load_2d_pair(b, mb, bar, kb * BK, n0);
                            } else {
#pragma unroll
                                for (int c = 0; c < BNC / CH; ++c)
                                    tma_load_2d_pair(b + c * CHUNK_BYTES, mb, bar, n0 + c * CH, kb * BK);
                            }
                        }
                    }
                    if (++stage == STAGES) {
                        stage = 0;
                        phase ^= 1;
                    }
                }
            }
        }
    } else if (warp == 1) {
        if (lane == 0 && rank == 0) {  // ---- MMA issuer (the leader issues for the pair)
            int stage = 0, acc = 0;
            uint32_t phase = 0, acc_phase = 0;
            for (int t = unit; t < tiles; t += units) {
                uint32_t d = 0;
                for (int kb = 0; kb < p.k_blocks; ++kb) {
                    const int kc = KC ? kb % KC : kb;  // K block within the accumulation chunk
                    if (kc == 0) {  // a new chunk: publish the last one, take a free accumulator
                        if (kb > 0) {
                            if constexpr (CTAS == 1) {
                                umma_commit(&tfull[acc]);
                            } else {
                                umma_commit_pair(&tfull[acc]);
                            }
                            if (++acc == ACC_STAGES) {
                                acc = 0;
                                acc_phase ^= 1;
                            }
                        }
                        mbar_wait(&tempty[acc], acc_phase ^ 1);
                        tc_fence_after();
                        d = tmem_base + (uint32_t)acc * ACC_COLS;
                    }
                    if constexpr (PARTS == 2) {
                        mbar_wait(&lo_full[stage], phase);  // raw tiles landed and lo parts written, every CTA
                    } else {
                        mbar_wait(&full[stage], phase);
                    }
                    tc_fence_after();
                    const uint32_t a0 = smem_addr(sA + stage * PARTS * A_BYTES);
                    const uint32_t b0 = smem_addr(sB + stage * PARTS * B_BYTES);
                    auto adesc = [&](uint32_t base, int k) {
                        return p.a_mn ? sw128_desc(base + k * Elem<KIND>::UMMA_K * ROW_BYTES, CHUNK_BYTES, MN_SBO,
                                                   MN_LAYOUT)
                                      : sw128_desc(base + k * 32);
                    };
                    auto bdesc = [&](uint32_t base, int k) {
                        return p.b_mn ? sw128_desc(base + k * Elem<KIND>::UMMA_K * ROW_BYTES, CHUNK_BYTES, MN_SBO,
                                                   MN_LAYOUT)
                                      : sw128_desc(base + k * 32);
                    };
                    auto mma = [&](uint64_t ad, uint64_t bd, uint32_t accumulate) {
                        if constexpr (CTAS == 1) {
                            umma<KIND>(d, ad, bd, p.idesc, accumulate);
                        } else {
                            umma_pair<KIND>(d, ad, bd, p.idesc, accumulate);
                        }
                    };
#pragma unroll
                    for (int k = 0; k < K_STEPS; ++k) {
                        const uint64_t ad = adesc(a0, k), bd = bdesc(b0, k);
                        const uint32_t acc_on = (kc | k) != 0;
                        if constexpr (PARTS == 2) {  // small products first: a_lo.b_hi, a_hi.b_lo, a_hi.b_hi
                            mma(adesc(a0 + A_BYTES, k), bd, acc_on);
                            mma(ad, bdesc(b0 + B_BYTES, k), 1u);
                            mma(ad, bd, 1u);
                        } else {
                            mma(ad, bd, acc_on);
                        }
                    }
                    if constexpr (CTAS == 1) {
                        umma_commit(&empty[stage]);
                    } else {
                        umma_commit_pair(&empty[stage]);
                    }
                    if (++stage == STAGES) {
                        stage = 0;
                        phase ^= 1;
                    }
                }
                if constexpr (CTAS == 1) {
                    umma_commit(&tfull[acc]);
                } else {
                    umma_commit_pair(&tfull[acc]);
                }
                if (++acc == ACC_STAGES) {
                    acc = 0;
                    acc_phase ^= 1;
                }
            }
        }
    } else if (PARTS == 2 && warp >= 6) {  // ---- 3xTF32 converters: warps 6..9
        // lo = x - hi(x) for every element of this CTA's raw A and B tiles,
        // written at the same offset in the stage's lo part (the swizzle is a
        // function of the offset, so the layout carries over), then released
        // to the async proxy and counted on the leader's lo_full barrier
        const int ct = threadIdx.x - 6 * 32;  // 0..127
        int stage = 0;
        uint32_t phase = 0;
        const int iters = p.tiles_m * p.tiles_n;
        for (int t = unit; t < iters; t += units) {
            for (int kb = 0; kb < p.k_blocks; ++kb) {
                mbar_wait(&full[stage], phase);
                const uint4* ra = reinterpret_cast<const uint4*>(sA + stage * PARTS * A_BYTES);
                uint4* la = reinterpret_cast<uint4*>(sA + stage * PARTS * A_BYTES + A_BYTES);
#pragma unroll 4
                for (int i = ct; i < (int)(A_BYTES / 16); i += 128) {
                    const uint4 v = ra[i];
                    la[i] = make_uint4(__float_as_uint(tf32_lo(__uint_as_float(v.x))),
                                       __float_as_uint(tf32_lo(__uint_as_float(v.y))),
                                       __float_as_uint(tf32_lo(__uint_as_float(v.z))),
                                       __float_as_uint(tf32_lo(__uint_as_float(v.w))));
                }
                const uint4* rb = reinterpret_cast<const uint4*>(sB + stage * PARTS * B_BYTES);
                uint4* lb = reinterpret_cast<uint4*>(sB + stage * PARTS * B_BYTES + B_BYTES);
#pragma unroll 4
                for (int i = ct; i < (int)(B_BYTES / 16); i += 128) {
                    const uint4 v = rb[i];
                    lb[i] = make_uint4(__float_as_uint(tf32_lo(__uint_as_float(v.x))),
                                       __float_as_uint(tf32_lo(__uint_as_float(v.y))),
                                       __float_as_uint(tf32_lo(__uint_as_float(v.z))),
                                       __float_as_uint(tf32_lo(__uint_as_float(v.w))));
                }
                asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");  // generic writes -> tcgen05 reads
                __syncwarp();
                if (lane == 0) {
                    if (rank == 0) {
                        mbar_arrive(&lo_full[stage]);
                    } else {
                        mbar_arrive_remote(&lo_full[stage], 0);
                    }
                }
                if (++stage == STAGES) {
                    stage = 0;
                    phase ^= 1;
                }
            }
        }
    } else {  // ---- epilogue: warps 2..5 own TMEM lane quarters (warp % 4)
        // Each 32 x 32 block (32 TMEM lanes = output rows, 32 columns) goes
        // TMEM -> registers (one row per thread) -> this warp's smem block ->
        // registers (row-contiguous) -> global, so every store instruction
        // writes whole 128-byte row segments instead of 32 rows x 4/16 bytes.
        const int q = warp & 3;
        float* blk = sEpi + q * 32 * EPI_LD;
        int acc = 0;
        uint32_t acc_phase = 0;
        // release the TMEM buffer `acc` to the MMA issuer (every CTA's epilogue warps)
        auto release = [&]() {
            tc_fence_before();
            __syncwarp();
            if (lane == 0) {
                if (rank == 0) {
                    mbar_arrive(&tempty[acc]);
                } else {
                    mbar_arrive_remote(&tempty[acc], 0);
                }
            }
            if (++acc == ACC_STAGES) {
                acc = 0;
                acc_phase ^= 1;
            }
        };
        const uint32_t lane_base = tmem_base + ((uint32_t)(q * 32) << 16);
        for (int t = unit; t < tiles; t += units) {
            int tm, tn;
            tile_coords(p, t, tm, tn);
            const int row0 = tm * BM * CTAS + (int)rank * BM + q * 32;  // first row of this warp's block
            // 3xTF32: IEEE fp32 running sum of the chunk accumulators (this thread's row)
            float run[KC ? BN : 1];
            if constexpr (KC != 0) {
#pragma unroll
                for (int j = 0; j < BN; ++j) run[j] = 0.f;
                const int chunks = (p.k_blocks + KC - 1) / KC;
                for (int ch = 0; ch < chunks; ++ch) {
                    mbar_wait(&tfull[acc], acc_phase);
                    tc_fence_after();
#pragma unroll
                    for (int c0 = 0; c0 < BN; c0 += 32) {
                        uint32_t v[32];
                        tmem_ld32(lane_base + (uint32_t)acc * ACC_COLS + (uint32_t)c0, v);
#pragma unroll
                        for (int j = 0; j < 32; ++j) run[c0 + j] += __uint_as_float(v[j]);
                    }
                    release();
                }
            } else {
                mbar_wait(&tfull[acc], acc_phase);
                tc_fence_after();
            }
#pragma unroll
            for (int c0 = 0; c0 < BN; c0 += 32) {
                uint32_t v[32];
                if constexpr (KC != 0) {
#pragma unroll
                    for (int j = 0; j < 32; ++j) v[j] = __float_as_uint(run[c0 + j]);
                } else {
                    tmem_ld32(lane_base + (uint32_t)acc * ACC_COLS + (uint32_t)c0, v);
                }
                const int col0 = tn * BN + c0;
                if (row0 >= p.M || col0 >= p.N) continue;  // warp-uniform
#pragma unroll
                for (int j = 0; j < 32; j += 4)
                    *reinterpret_cast<float4*>(blk + lane * EPI_LD + j) =
                        make_float4(__uint_as_float(v[j]), __uint_as_float(v[j + 1]), __uint_as_float(v[j + 2]),
                                    __uint_as_float(v[j + 3]));
                __syncwarp();
                if (p.vec_out && col0 + 32 <= p.N) {
                    // 8 lanes per row, 4 rows per instruction, float4 each
                    const int cq = (lane & 7) * 4;
#pragma unroll
                    for (int rr = 0; rr < 32; rr += 4) {
                        const int r = rr + (lane >> 3);
                        const int row = row0 + r;
                        if (row < p.M) {
                            const float4 a = *reinterpret_cast<const float4*>(blk + r * EPI_LD + cq);
                            float4 o = make_float4(p.alpha * a.x, p.alpha * a.y, p.alpha * a.z, p.alpha * a.w);
                            if (p.use_c) {
                                const float4 cc = *reinterpret_cast<const float4*>(p.C + (i64)row * p.ldc + col0 + cq);
                                o.x += p.beta * cc.x;
                                o.y += p.beta * cc.y;
                                o.z += p.beta * cc.z;
                                o.w += p.beta * cc.w;
                            }
                            *reinterpret_cast<float4*>(p.out + (i64)row * p.ldo + col0 + cq) = o;
                        }
                    }
                } else {
                    // one row per instruction, lane = column
                    const int col = col0 + lane;
#pragma unroll 4
                    for (int r = 0; r < 32; ++r) {
                        const int row = row0 + r;
                        if (row < p.M && col < p.N) {
                            float o = p.alpha * blk[r * EPI_LD + lane];
                            if (p.use_c) o += p.beta * p.C[(i64)row * p.ldc + col];
                            p.out[(i64)row * p.ldo + col] = o;
                        }
                    }
                }
                __syncwarp();
            }
            if constexpr (KC == 0) release();
        }
    }
    tc_fence_before();
    if constexpr (CTAS == 2) {
        cluster_sync();
    } else {
        __syncthreads();
    }
    if (warp == 1) {
        tc_fence_after();
        if constexpr (CTAS == 1) {
            asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tmem_base), "n"(TMEM_COLS)
                         : "memory");
        } else {
            asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;\n" ::"r"(tmem_base), "n"(TMEM_COLS)
                         : "memory");
        }
    }
}

// helper pass (bf16 always; tf32 only when an operand's rows are not
// 16-byte aligned): dst (rows x cols, ld_dst) = src converted to the MMA
// element type, layout unchanged (no transpose: the core reads either
// major).  bf16 rounds to nearest even; the tf32 copy keeps the fp32 bits
// (the tensor core consumes them as tf32).  Four elements per thread,
// 16-byte loads when the source rows allow it.
__device__ __forceinline__ void store4(float* d, float a, float b, float c, float e, bool vec) {
    if (vec) {
        *reinterpret_cast<float4*>(d) = make_float4(a, b, c, e);
    } else {
        d[0] = a; d[1] = b; d[2] = c; d[3] = e;
    }
}
__device__ __forceinline__ void store4(__nv_bfloat16* d, float a, float b, float c, float e, bool vec) {
    const __nv_bfloat162 lo = __floats2bfloat162_rn(a, b), hi = __floats2bfloat162_rn(c, e);
    if (vec) {
        uint2 u;
        u.x = *reinterpret_cast<const uint32_t*>(&lo);
        u.y = *reinterpret_cast<const uint32_t*>(&hi);
        *reinterpret_cast<uint2*>(d) = u;
    } else {
        d[0] = lo.x; d[1] = lo.y; d[2] = hi.x; d[3] = hi.y;
    }
}
__device__ __forceinline__ void store1(float* d, float a) { *d = a; }
__device__ __forceinline__ void store1(__nv_bfloat16* d, float a) { *d = __float2bfloat16_rn(a); }

// One staging job: dst (rows x cols, ld_dst) = src converted to the MMA type.
template <typename D>
struct ConvertJob {
    D* dst;
    i64 ld_dst;
    const float* src;
    i64 ld_src;
    i64 rows, cols, quads;  // quads = rows * ceil(cols / 4); 0 = no job
    int vec;                // 16-byte source rows: one LDG.128 per quad
};
// every staging job of one call (up to hi / lo of A and B), one launch
template <typename D>
struct ConvertJobs {
    ConvertJob<D> j[4];
};



// Both operands' staging in ONE launch: a flat grid-stride over the
// (row, 4-column quad) space of job a then job b, 4 quads per thread per step
// so 4 loads are in flight.  (Separate row-per-block launches reached
// 5.3 TB/s on 7640 x 6966; one flat launch streams at the copy rate and
// pays one launch and one tail instead of two.)
template <typename D>
__device__ __forceinline__ void convert_quad(const ConvertJob<D>& j, i64 q) {
    const i64 qpr = (j.cols + 3) >> 2;
    const i64 r = q / qpr, c = (q - r * qpr) << 2;
    const float* sp = j.src + r * j.ld_src + c;
    D* dp = j.dst + r * j.ld_dst + c;
    if (c + 4 <= j.cols) {
        float4 v;
        if (j.vec) {
            v = __ldcs(reinterpret_cast<const float4*>(sp));
        } else {
            v = make_float4(__ldcs(sp), __ldcs(sp + 1), __ldcs(sp + 2), __ldcs(sp + 3));
        }
        store4(dp, v.x, v.y, v.z, v.w, true);
    } else {
        for (i64 k = c; k < j.cols; ++k) {
            const float x = j.src[r * j.ld_src + k];
            store1(j.dst + r * j.ld_dst + k, x);
        }
    }
}
template <typename D>
__global__ void __launch_bounds__(256)
tc_convert_kernel(const ConvertJobs<D> jobs) {
    // let the tc_gemm launch (programmatic dependent launch) start its setup
    asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory");
    const i64 q1 = jobs.j[0].quads, q2 = q1 + jobs.j[1].quads, q3 = q2 + jobs.j[2].quads;
    const i64 total = q3 + jobs.j[3].quads;
    const i64 stride = (i64)gridDim.x * blockDim.x;
    for (i64 q0 = (i64)blockIdx.x * blockDim.x + threadIdx.x; q0 < total; q0 += 4 * stride) {
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const i64 q = q0 + u * stride;
            if (q < q1) {
                convert_quad(jobs.j[0], q);
            } else if (q < q2) {
                convert_quad(jobs.j[1], q - q1);
            } else if (q < q3) {
                convert_quad(jobs.j[2], q - q2);
            } else if (q < total) {
                convert_quad(jobs.j[3], q - q3);
            }
        }
    }
}

// ------------------------------------------------------------------ host side
inline PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
    static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
    static std::once_flag once;
    std::call_once(once, [] {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
    });
    return fn;
}

inline int sm_count() { return device_sms(); }  // per device (launch.cuh)

// One operand as stored: `rows` x `cols` row-major with leading dimension
// `ld` (elements of the MMA type).  K-major when the contiguous dimension is
// K (box: 128 bytes of K x `box_rows` rows), MN-major when it is M or N
// (box: 128 bytes of MN x BK rows of k; the producer issues one box per
// 128-byte chunk).  Out-of-range boxes are zero-filled by the TMA unit, so
// no operand is padded to the tile.
template <int KIND>
inline bool make_map(CUtensorMap* map, const void* base, i64 rows, i64 cols, i64 ld, bool mn_major, int box_rows) {
    auto fn = encode_fn();
    if (!fn) return false;
    typedef typename Elem<KIND>::T T;
    constexpr int CH = ROW_BYTES / (int)sizeof(T);
    cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
    cuuint64_t strides[1] = {(cuuint64_t)(ld * (i64)sizeof(T))};
    cuuint32_t box[2] = {(cuuint32_t)CH, (cuuint32_t)(mn_major ? Elem<KIND>::BK : box_rows)};
    cuuint32_t estr[2] = {1, 1};
    // 32-bit MN-major tiles: 32-byte swizzle atoms (see sw128_desc)
    const CUtensorMapSwizzle swz =
        (KIND != KIND_BF16 && mn_major) ? CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B : CU_TENSOR_MAP_SWIZZLE_128B;
    CUresult r = fn(map, Elem<KIND>::TMA, 2, const_cast<void*>(base), dims, strides, box, estr,
                    CU_TENSOR_MAP_INTERLEAVE_NONE, swz, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                    CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return r == CUDA_SUCCESS;
}

// stored (rows, cols) of op(A) and op(B): A is M x K (K x M when transA),
// B is K x N (N x K when transB)
struct OperandLayout {
    i64 rows, cols;
};
inline OperandLayout layout_a(i64 M, i64 K, int ta) { return ta ? OperandLayout{K, M} : OperandLayout{M, K}; }
inline OperandLayout layout_b(i64 N, i64 K, int tb) { return tb ? OperandLayout{N, K} : OperandLayout{K, N}; }

// staged rows start on 128-byte boundaries, so every TMA box row is one
// whole L2 line (a 16-byte-aligned but line-straddling stride costs a
// second line per row)
template <int KIND>
inline i64 staged_ld(i64 cols) {
    return round_up_i(cols, ROW_BYTES / (i64)sizeof(typename Elem<KIND>::T));
}

// [A staging | B staging], each 1024-byte aligned: converted (bf16) or
// re-strided (tf32, only used when a row stride is not 16-byte aligned);
// 3xTF32 adds [A lo | B lo] after them
template <int KIND>
inline size_t staged_bytes(i64 rows, i64 cols) {
    return (size_t)round_up_i(rows * staged_ld<KIND>(cols) * (i64)sizeof(typename Elem<KIND>::T), 1024);
}
template <int KIND>
inline size_t workspace_bytes(i64 M, i64 N, i64 K, int ta, int tb) {
    // (3xTF32's lo parts are made in shared memory: its staging is tf32's)
    const OperandLayout a = layout_a(M, K, ta), b = layout_b(N, K, tb);
    return staged_bytes<KIND>(a.rows, a.cols) + staged_bytes<KIND>(b.rows, b.cols);
}

template <typename T>
inline int launch_converts(const ConvertJobs<T>& jobs, cudaStream_t stream) {
    const i64 total = jobs.j[0].quads + jobs.j[1].quads + jobs.j[2].quads + jobs.j[3].quads;
    if (total == 0) return AG_OK;
    const unsigned blocks = (unsigned)std::max<i64>(1, std::min<i64>((total + 1023) / 1024, (i64)sm_count() * 8));
    tc_convert_kernel<T><<<blocks, 256, 0, stream>>>(jobs);
    return cudaGetLastError() == cudaSuccess ? AG_OK : AG_ERR_CUDA;
}

inline int tc_fail(const GemmCall& c, int code, const char* msg) {
    if (c.err) *c.err = msg;
    return code;
}

// Stage one operand for the TMA: bf16 always converts into the workspace;
// tf32 reads the caller's fp32 matrix in place when its base and row stride
// are 16-byte aligned, else copies it to a re-strided buffer.  Returns the
// conversion job (quads = 0 when the operand is read in place).
template <int KIND>
inline ConvertJob<typename Elem<KIND>::T> plan_operand(const float* src, i64 ld_src, OperandLayout lay, void* ws,
                                                       const void** base, i64* ld) {
    typedef typename Elem<KIND>::T T;
    ConvertJob<T> j{};
    if (KIND != KIND_BF16 && ld_src % 4 == 0 && reinterpret_cast<uintptr_t>(src) % 16 == 0) {
        *base = src;
        *ld = ld_src;
        return j;
    }
    *ld = staged_ld<KIND>(lay.cols);
    *base = ws;
    j.dst = static_cast<T*>(ws);
    j.ld_dst = *ld;
    j.src = src;
    j.ld_src = ld_src;
    j.rows = lay.rows;
    j.cols = lay.cols;
    j.quads = lay.rows * ((lay.cols + 3) / 4);
    j.vec = (ld_src % 4 == 0) && (reinterpret_cast<uintptr_t>(src) % 16 == 0);
    return j;
}

// CTAS = 1: config bm = 128; CTAS = 2: bm = 256 on a CTA pair
template <int KIND, int BN, int STAGES, int CTAS = 1>
int launch_tc(const GemmCall& c) {
    typedef typename Elem<KIND>::T T;
    constexpr int BK = Elem<KIND>::BK;
    constexpr int TILE_M = BM * CTAS;
    if (c.dtype != AG_F32) return tc_fail(c, AG_ERR_CONFIG, "tensor-core families take float32 operands");
    const i64 M = c.M, N = c.N, K = c.K;
    const i64 tiles_m = (M + TILE_M - 1) / TILE_M, tiles_n = (N + BN - 1) / BN, k_blocks = (K + BK - 1) / BK;
    if (tiles_m * tiles_n > 0x7fffffffLL || k_blocks > 0x7fffffffLL)
        return tc_fail(c, AG_ERR_SHAPE, "problem too large for the tensor-core grid");
    const OperandLayout la = layout_a(M, K, c.ta), lb = layout_b(N, K, c.tb);
    const size_t need = workspace_bytes<KIND>(M, N, K, c.ta, c.tb);
    if (KIND == KIND_BF16 && (c.ws_bytes < need || c.ws == nullptr))
        return tc_fail(c, AG_ERR_SHAPE, "workspace too small for the tensor-core staging buffers");
    const size_t a_st = staged_bytes<KIND>(la.rows, la.cols);
    char* wsA = static_cast<char*>(c.ws);
    char* wsB = wsA ? wsA + a_st : nullptr;
    const void *baseA = nullptr, *baseB = nullptr;
    i64 ldA = 0, ldB = 0;
    ConvertJobs<T> jobs{};
    jobs.j[0] = plan_operand<KIND>(static_cast<const float*>(c.A), c.lda, la, wsA, &baseA, &ldA);
    jobs.j[1] = plan_operand<KIND>(static_cast<const float*>(c.B), c.ldb, lb, wsB, &baseB, &ldB);
    const bool staged = jobs.j[0].quads || jobs.j[1].quads || jobs.j[2].quads || jobs.j[3].quads;
    if (staged && (c.ws_bytes < need || c.ws == nullptr))
        return tc_fail(c, AG_ERR_SHAPE, "workspace too small for the tensor-core staging buffers");
    if (launch_converts<T>(jobs, c.stream) != AG_OK) return tc_fail(c, AG_ERR_CUDA, "staging of the operands failed");

    // A: K-major unless transA; B: MN-major unless transB.  Boxes are per
    // CTA: 128 rows of A, BN / CTAS rows of B.
    const int a_mn = c.ta ? 1 : 0, b_mn = c.tb ? 0 : 1;
    CUtensorMap mapA, mapB;
    if (!make_map<KIND>(&mapA, baseA, la.rows, la.cols, ldA, a_mn, BM) ||
        !make_map<KIND>(&mapB, baseB, lb.rows, lb.cols, ldB, b_mn, BN / CTAS))
        return tc_fail(c, AG_ERR_CUDA, "cuTensorMapEncodeTiled failed");

    TcParams p;
    p.M = (int)M;
    p.N = (int)N;
    p.tiles_m = (int)tiles_m;
    p.tiles_n = (int)tiles_n;
    p.k_blocks = (int)k_blocks;
    p.group_m = p.tiles_m < 8 ? p.tiles_m : 8;
    p.a_mn = a_mn;
    p.b_mn = b_mn;
    p.idesc = instr_desc<KIND>(TILE_M, BN, a_mn, b_mn);
    p.alpha = (float)c.alpha;
    p.beta = (float)c.beta;
    p.use_c = c.beta != 0.0;
    p.C = static_cast<const float*>(c.C);
    p.ldc = c.ldc;
    p.out = static_cast<float*>(c.out);
    p.ldo = c.ldo;
    p.vec_out = (c.ldo % 4 == 0) && (reinterpret_cast<uintptr_t>(c.out) % 16 == 0) &&
                (!p.use_c || ((c.ldc % 4 == 0) && (reinterpret_cast<uintptr_t>(c.C) % 16 == 0)));

    // >= 116 KB of shared memory keeps one CTA per SM, so a CTA never waits
    // on another CTA's TMEM allocation
    const size_t smem = std::max<size_t>(smem_bytes<BN, STAGES, CTAS, Elem<KIND>::PARTS>(), 116 * 1024);
    if (smem > 227 * 1024) return tc_fail(c, AG_ERR_CONFIG, "config exceeds 227 KB shared memory per CTA");
    auto kernel = tc_gemm_kernel<KIND, BN, STAGES, CTAS>;
    static SmemGrant granted;  // per device: the attribute applies to the current device only
    if (ensure_smem(kernel, smem, granted) != cudaSuccess)
        return tc_fail(c, AG_ERR_CUDA, "cudaFuncSetAttribute failed");
    // persistent: one CTA (pair) per SM (TPC), tiles strided over units
    const i64 units = std::min<i64>(tiles_m * tiles_n, sm_count() / CTAS);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)(units * CTAS));
    cfg.blockDim = dim3(kernel_threads<KIND>());
    cfg.dynamicSmemBytes = smem;
    cfg.stream = c.stream;
    cudaLaunchAttribute attr[2];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = CTAS;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    // dependent launch only behind this call's own staging convert: the
    // family path's first kernel never overlaps whatever the caller queued
    attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[1].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = staged ? 2 : 1;
    if (cudaLaunchKernelEx(&cfg, kernel, mapA, mapB, p) != cudaSuccess)
        return tc_fail(c, AG_ERR_CUDA, "tensor-core kernel launch failed");
    return cudaGetLastError() == cudaSuccess ? AG_OK : tc_fail(c, AG_ERR_CUDA, "tensor-core kernel launch failed");
}

}  // namespace tc
}  // namespace ag
