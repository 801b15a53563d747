// tc_kernels.cuh -- the tensor-core families (B200 tc profile): tf32 and bf16.
//
// No reference analogue: the reference's two families are CUDA-core style
// loop nests (kernels.py:198-260).  These families serve the dense
// contraction on the 5th-generation tensor cores (BASELINE.json configs[4])
// and follow the indirect family's structure (kernels.py:304-325): an O(n^2)
// helper pass packs op(A) and op(B)^T into zero-padded, K-major buffers in
// the MMA element type (tf32 = fp32 rounded to nearest, bf16 = round to
// nearest even), then an unpredicated core runs on exact tile multiples and
// a masked epilogue writes alpha * acc + beta * C (C read only when
// beta != 0, as the indirect family, kernels.py:318-321).
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
#include <atomic>
#include <mutex>

#include "kernels.cuh"
#include "registry.h"

namespace ag {
namespace tc {

constexpr int KIND_TF32 = 0;
constexpr int KIND_BF16 = 1;
constexpr int BM = 128;          // UMMA M (cta_group::1): TMEM lane = output row
constexpr int ROW_BYTES = 128;   // one K block = one 128-byte swizzle row
constexpr int THREADS = 192;     // producer warp, MMA warp, 4 epilogue warps
constexpr int ACC_STAGES = 2;    // TMEM accumulator double buffer

inline constexpr i64 round_up_i(i64 x, i64 s) { return (x + s - 1) / s * s; }

template <int KIND> struct Elem;
template <> struct Elem<KIND_TF32> {
    typedef float T;
    static constexpr int BK = ROW_BYTES / 4;  // 32 elements per K block
    static constexpr int UMMA_K = 8;
    static constexpr uint32_t FMT = 2;        // TF32
    static constexpr CUtensorMapDataType TMA = CU_TENSOR_MAP_DATA_TYPE_FLOAT32;
};
template <> struct Elem<KIND_BF16> {
    typedef __nv_bfloat16 T;
    static constexpr int BK = ROW_BYTES / 2;  // 64 elements per K block
    static constexpr int UMMA_K = 16;
    static constexpr uint32_t FMT = 1;        // BF16
    static constexpr CUtensorMapDataType TMA = CU_TENSOR_MAP_DATA_TYPE_BFLOAT16;
};

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

// K-major SWIZZLE_128B shared-memory matrix descriptor (sm_100 format):
// start address, LBO (unused for swizzled K-major), SBO = 1024 B between
// 8-row groups, version 1, layout type 2 (128B swizzle).
__device__ __forceinline__ uint64_t sw128_desc(uint32_t saddr) {
    return (uint64_t)((saddr & 0x3FFFFu) >> 4) | ((uint64_t)1 << 16) | ((uint64_t)(1024 >> 4) << 32) |
           ((uint64_t)1 << 46) | ((uint64_t)2 << 61);
}

// instruction descriptor: D f32, A/B format, both K-major, N >> 3, M >> 4
template <int KIND, int N>
__host__ __device__ constexpr uint32_t instr_desc() {
    return (1u << 4) | (Elem<KIND>::FMT << 7) | (Elem<KIND>::FMT << 10) | ((uint32_t)(N >> 3) << 17) |
           ((uint32_t)(BM >> 4) << 24);
}

template <int KIND>
__device__ __forceinline__ void umma(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc, uint32_t acc) {
    if constexpr (KIND == KIND_TF32) {
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

template <int BN>
constexpr uint32_t tmem_cols() {
    return (ACC_STAGES * BN) <= 32 ? 32 : (ACC_STAGES * BN) <= 64 ? 64 : (ACC_STAGES * BN) <= 128 ? 128
                                     : (ACC_STAGES * BN) <= 256 ? 256 : 512;
}

template <int BN, int STAGES>
constexpr size_t smem_bytes() {
    return 1024 /* alignment slack */ + (size_t)STAGES * (BM + BN) * ROW_BYTES + 256 /* barriers */;
}

template <int KIND, int BN, int STAGES>
__global__ void __launch_bounds__(THREADS, 1)
tc_gemm_kernel(const __grid_constant__ CUtensorMap mapA, const __grid_constant__ CUtensorMap mapB, TcParams p) {
    constexpr int BK = Elem<KIND>::BK;
    constexpr uint32_t A_BYTES = BM * ROW_BYTES, B_BYTES = BN * ROW_BYTES;
    constexpr uint32_t STAGE_TX = A_BYTES + B_BYTES;
    constexpr uint32_t TMEM_COLS = tmem_cols<BN>();
    constexpr uint32_t IDESC = instr_desc<KIND, BN>();
    constexpr int K_STEPS = BK / Elem<KIND>::UMMA_K;
    static_assert(BN % 16 == 0 && BN >= 16 && BN <= 256, "UMMA N for M=128 is 16..256 in steps of 16");
    static_assert(BN % 32 == 0, "epilogue drains 32 columns per tcgen05.ld");

    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~(uintptr_t)1023);
    uint8_t* sA = smem;
    uint8_t* sB = smem + STAGES * A_BYTES;
    uint64_t* full = reinterpret_cast<uint64_t*>(sB + STAGES * B_BYTES);
    uint64_t* empty = full + STAGES;
    uint64_t* tfull = empty + STAGES;
    uint64_t* tempty = tfull + ACC_STAGES;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + ACC_STAGES);

    const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
    if (warp == 0 && lane == 0) {
        asm volatile("prefetch.tensormap [%0];\n" ::"l"(reinterpret_cast<uint64_t>(&mapA)) : "memory");
        asm volatile("prefetch.tensormap [%0];\n" ::"l"(reinterpret_cast<uint64_t>(&mapB)) : "memory");
        for (int s = 0; s < STAGES; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], 1);
        }
        for (int a = 0; a < ACC_STAGES; ++a) {
            mbar_init(&tfull[a], 1);
            mbar_init(&tempty[a], 128);
        }
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    }
    if (warp == 1) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(smem_addr(tmem_slot)),
                     "n"(TMEM_COLS)
                     : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n" ::: "memory");
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;
    const int tiles = p.tiles_m * p.tiles_n;

    if (warp == 0) {
        if (lane == 0) {  // ---- TMA producer
            int stage = 0;
            uint32_t phase = 0;
            for (int t = blockIdx.x; t < tiles; t += gridDim.x) {
                int tm, tn;
                tile_coords(p, t, tm, tn);
                for (int kb = 0; kb < p.k_blocks; ++kb) {
                    mbar_wait(&empty[stage], phase ^ 1);
                    mbar_expect_tx(&full[stage], STAGE_TX);
                    tma_load_2d(sA + stage * A_BYTES, &mapA, &full[stage], kb * BK, tm * BM);
                    tma_load_2d(sB + stage * B_BYTES, &mapB, &full[stage], kb * BK, tn * BN);
                    if (++stage == STAGES) {
                        stage = 0;
                        phase ^= 1;
                    }
                }
            }
        }
    } else if (warp == 1) {
        if (lane == 0) {  // ---- MMA issuer
            int stage = 0, acc = 0;
            uint32_t phase = 0, acc_phase = 0;
            for (int t = blockIdx.x; t < tiles; t += gridDim.x) {
                mbar_wait(&tempty[acc], acc_phase ^ 1);
                tc_fence_after();
                const uint32_t d = tmem_base + (uint32_t)(acc * BN);
                for (int kb = 0; kb < p.k_blocks; ++kb) {
                    mbar_wait(&full[stage], phase);
                    tc_fence_after();
                    const uint32_t a0 = smem_addr(sA + stage * A_BYTES), b0 = smem_addr(sB + stage * B_BYTES);
#pragma unroll
                    for (int k = 0; k < K_STEPS; ++k)
                        umma<KIND>(d, sw128_desc(a0 + k * 32), sw128_desc(b0 + k * 32), IDESC, (kb | k) != 0);
                    umma_commit(&empty[stage]);
                    if (++stage == STAGES) {
                        stage = 0;
                        phase ^= 1;
                    }
                }
                umma_commit(&tfull[acc]);
                if (++acc == ACC_STAGES) {
                    acc = 0;
                    acc_phase ^= 1;
                }
            }
        }
    } else {  // ---- epilogue: warps 2..5 own TMEM lane quarters (warp % 4)
        const int q = warp & 3;
        const int row_in_tile = q * 32 + lane;
        int acc = 0;
        uint32_t acc_phase = 0;
        for (int t = blockIdx.x; t < tiles; t += gridDim.x) {
            int tm, tn;
            tile_coords(p, t, tm, tn);
            mbar_wait(&tfull[acc], acc_phase);
            tc_fence_after();
            const int row = tm * BM + row_in_tile;
            const bool row_ok = row < p.M;
            float* orow = p.out + (i64)row * p.ldo;
            const float* crow = p.C + (i64)row * p.ldc;
#pragma unroll 1
            for (int c0 = 0; c0 < BN; c0 += 32) {
                uint32_t v[32];
                tmem_ld32(tmem_base + ((uint32_t)(q * 32) << 16) + (uint32_t)(acc * BN + c0), v);
                const int col0 = tn * BN + c0;
                if (!row_ok || col0 >= p.N) continue;
                if (p.vec_out && col0 + 32 <= p.N) {
#pragma unroll
                    for (int j = 0; j < 32; j += 4) {
                        float4 r;
                        r.x = p.alpha * __uint_as_float(v[j]);
                        r.y = p.alpha * __uint_as_float(v[j + 1]);
                        r.z = p.alpha * __uint_as_float(v[j + 2]);
                        r.w = p.alpha * __uint_as_float(v[j + 3]);
                        if (p.use_c) {
                            const float4 cc = *reinterpret_cast<const float4*>(crow + col0 + j);
                            r.x += p.beta * cc.x;
                            r.y += p.beta * cc.y;
                            r.z += p.beta * cc.z;
                            r.w += p.beta * cc.w;
                        }
                        *reinterpret_cast<float4*>(orow + col0 + j) = r;
                    }
                } else {
#pragma unroll
                    for (int j = 0; j < 32; ++j) {
                        const int col = col0 + j;
                        if (col < p.N) {
                            float r = p.alpha * __uint_as_float(v[j]);
                            if (p.use_c) r += p.beta * crow[col];
                            orow[col] = r;
                        }
                    }
                }
            }
            tc_fence_before();
            mbar_arrive(&tempty[acc]);
            if (++acc == ACC_STAGES) {
                acc = 0;
                acc_phase ^= 1;
            }
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 1) {
        tc_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tmem_base), "n"(TMEM_COLS)
                     : "memory");
    }
}

// helper pass: dst (dst_rows x dst_cols, ld_dst) = zero-padded op(src)
// converted to the MMA element type; op = transpose when `transpose`
// (src then holds the cols x rows matrix).  32x32 tile through smem so
// both sides are coalesced.
__device__ __forceinline__ float to_elem(float x, float*) {
    uint32_t r;
    asm("cvt.rna.tf32.f32 %0, %1;\n" : "=r"(r) : "f"(x));
    return __uint_as_float(r);
}
__device__ __forceinline__ __nv_bfloat16 to_elem(float x, __nv_bfloat16*) { return __float2bfloat16_rn(x); }

template <typename D>
__global__ void __launch_bounds__(256)
tc_pack_kernel(D* __restrict__ dst, i64 ld_dst, int dst_rows, int dst_cols, const float* __restrict__ src,
               i64 ld_src, int rows, int cols, int transpose) {
    __shared__ float tile[32][33];
    const int r0 = blockIdx.y * 32, c0 = blockIdx.x * 32;
    const int x = threadIdx.x, y = threadIdx.y;
    if (transpose) {
#pragma unroll
        for (int yy = y; yy < 32; yy += 8) {
            const int c = c0 + yy, r = r0 + x;
            tile[yy][x] = (r < rows && c < cols) ? src[(i64)c * ld_src + r] : 0.0f;
        }
        __syncthreads();
#pragma unroll
        for (int yy = y; yy < 32; yy += 8) {
            const int r = r0 + yy, c = c0 + x;
            if (r < dst_rows && c < dst_cols) dst[(i64)r * ld_dst + c] = to_elem(tile[x][yy], (D*)nullptr);
        }
    } else {
#pragma unroll
        for (int yy = y; yy < 32; yy += 8) {
            const int r = r0 + yy, c = c0 + x;
            if (r < dst_rows && c < dst_cols)
                dst[(i64)r * ld_dst + c] =
                    to_elem((r < rows && c < cols) ? src[(i64)r * ld_src + c] : 0.0f, (D*)nullptr);
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

inline int sm_count() {
    static int n = 0;
    static std::once_flag once;
    std::call_once(once, [] {
        int dev = 0;
        cudaGetDevice(&dev);
        if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || n <= 0) n = 148;
    });
    return n;
}

// K-major (rows x cols) matrix with leading dimension `cols`, 128-byte boxes
template <int KIND>
inline bool make_map(CUtensorMap* map, const void* base, i64 rows, i64 cols, int box_rows) {
    auto fn = encode_fn();
    if (!fn) return false;
    typedef typename Elem<KIND>::T T;
    cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
    cuuint64_t strides[1] = {(cuuint64_t)(cols * (i64)sizeof(T))};
    cuuint32_t box[2] = {(cuuint32_t)Elem<KIND>::BK, (cuuint32_t)box_rows};
    cuuint32_t estr[2] = {1, 1};
    CUresult r = fn(map, Elem<KIND>::TMA, 2, const_cast<void*>(base), dims, strides, box, estr,
                    CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                    CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return r == CUDA_SUCCESS;
}

// [Ap (Mp x Kp) | Bp (Np x Kp)] in the element type, each 1024-byte aligned
template <int KIND>
inline size_t workspace_bytes(i64 M, i64 N, i64 K, int bn) {
    typedef typename Elem<KIND>::T T;
    const i64 Mp = round_up_i(M, BM), Np = round_up_i(N, bn), Kp = round_up_i(K, Elem<KIND>::BK);
    return (size_t)round_up_i(Mp * Kp * (i64)sizeof(T), 1024) + (size_t)round_up_i(Np * Kp * (i64)sizeof(T), 1024);
}

template <int KIND>
inline int launch_pack(typename Elem<KIND>::T* dst, i64 dst_rows, i64 dst_cols, const float* src, i64 ld_src,
                       i64 rows, i64 cols, int transpose, cudaStream_t stream) {
    dim3 grid((unsigned)((dst_cols + 31) / 32), (unsigned)((dst_rows + 31) / 32));
    if (grid.y > 65535u) return AG_ERR_SHAPE;
    tc_pack_kernel<typename Elem<KIND>::T><<<grid, dim3(32, 8), 0, stream>>>(
        dst, dst_cols, (int)dst_rows, (int)dst_cols, src, ld_src, (int)rows, (int)cols, transpose);
    return cudaGetLastError() == cudaSuccess ? AG_OK : AG_ERR_CUDA;
}

inline int tc_fail(const GemmCall& c, int code, const char* msg) {
    if (c.err) *c.err = msg;
    return code;
}

template <int KIND, int BN, int STAGES>
int launch_tc(const GemmCall& c) {
    typedef typename Elem<KIND>::T T;
    constexpr int BK = Elem<KIND>::BK;
    if (c.dtype != AG_F32) return tc_fail(c, AG_ERR_CONFIG, "tensor-core families take float32 operands");
    const i64 M = c.M, N = c.N, K = c.K;
    const i64 Mp = round_up_i(M, BM), Np = round_up_i(N, BN), Kp = round_up_i(K, BK);
    if (Mp > 0x7fffffffLL || Np > 0x7fffffffLL || Kp > 0x7fffffffLL)
        return tc_fail(c, AG_ERR_SHAPE, "dimension too large");
    const size_t need = workspace_bytes<KIND>(M, N, K, BN);
    if (c.ws_bytes < need || c.ws == nullptr)
        return tc_fail(c, AG_ERR_SHAPE, "workspace too small for the tensor-core pack buffers");
    T* Ap = static_cast<T*>(c.ws);
    T* Bp = reinterpret_cast<T*>(static_cast<char*>(c.ws) + round_up_i(Mp * Kp * (i64)sizeof(T), 1024));
    // op(A) -> Ap[m][k]; op(B)^T -> Bp[n][k]
    int r = launch_pack<KIND>(Ap, Mp, Kp, static_cast<const float*>(c.A), c.lda, M, K, c.ta ? 1 : 0, c.stream);
    if (r) return tc_fail(c, r, "pack of op(A) failed");
    r = launch_pack<KIND>(Bp, Np, Kp, static_cast<const float*>(c.B), c.ldb, N, K, c.tb ? 0 : 1, c.stream);
    if (r) return tc_fail(c, r, "pack of op(B) failed");

    CUtensorMap mapA, mapB;
    if (!make_map<KIND>(&mapA, Ap, Mp, Kp, BM) || !make_map<KIND>(&mapB, Bp, Np, Kp, BN))
        return tc_fail(c, AG_ERR_CUDA, "cuTensorMapEncodeTiled failed");

    TcParams p;
    p.M = (int)M;
    p.N = (int)N;
    p.tiles_m = (int)(Mp / BM);
    p.tiles_n = (int)(Np / BN);
    p.k_blocks = (int)(Kp / BK);
    p.group_m = p.tiles_m < 8 ? p.tiles_m : 8;
    p.alpha = (float)c.alpha;
    p.beta = (float)c.beta;
    p.use_c = c.beta != 0.0;
    p.C = static_cast<const float*>(c.C);
    p.ldc = c.ldc;
    p.out = static_cast<float*>(c.out);
    p.ldo = c.ldo;
    p.vec_out = (c.ldo % 4 == 0) && (reinterpret_cast<uintptr_t>(c.out) % 16 == 0) &&
                (!p.use_c || ((c.ldc % 4 == 0) && (reinterpret_cast<uintptr_t>(c.C) % 16 == 0)));
    const i64 tiles = (i64)p.tiles_m * p.tiles_n;
    if (tiles > 0x7fffffffLL) return tc_fail(c, AG_ERR_SHAPE, "too many tiles");

    // >= 116 KB of shared memory keeps one CTA per SM, so a CTA never waits
    // on another CTA's TMEM allocation
    const size_t smem = std::max<size_t>(smem_bytes<BN, STAGES>(), 116 * 1024);
    if (smem > 227 * 1024) return tc_fail(c, AG_ERR_CONFIG, "config exceeds 227 KB shared memory per CTA");
    auto kernel = tc_gemm_kernel<KIND, BN, STAGES>;
    static std::atomic<int> attr_done{0};
    if (!attr_done.load()) {
        if (cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess)
            return tc_fail(c, AG_ERR_CUDA, "cudaFuncSetAttribute failed");
        attr_done.store(1);
    }
    const unsigned grid = (unsigned)std::min<i64>(tiles, sm_count());
    kernel<<<grid, THREADS, smem, c.stream>>>(mapA, mapB, p);
    return cudaGetLastError() == cudaSuccess ? AG_OK : tc_fail(c, AG_ERR_CUDA, "tensor-core kernel launch failed");
}

}  // namespace tc
}  // namespace ag
