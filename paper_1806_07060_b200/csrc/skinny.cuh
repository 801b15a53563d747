// skinny.cuh -- the B200 "skinny" families: streaming fp32 CUDA-core kernels
// for GEMMs with one small output side.
//
//   skinny_n (N small, e.g. DeepBench 4096 x 16 x 4096): op(A) is the big
//     operand.  A lane owns TM output rows (row i * 32 + lane) and ALL bn
//     columns; per k it multiplies its rows' A values by the broadcast B row
//     B[k][0:bn] with FFMA2.  The CTA's NW warps split the CTA's K range
//     block by block (warp w takes K blocks w, w + NW, ...), each warp with
//     its own D-deep TMA ring (A box: bm rows x 128 bytes of K, 128-byte
//     swizzle; B box: 32 k x bn), so no warp ever waits on another inside the
//     main loop.  The warps' partial tiles are summed in shared memory in
//     warp order.
//   skinny_m (M small, e.g. DeepBench 35 x 8457 x 2560): op(B) is the big
//     operand.  A thread owns TN2 output columns (col n0 + j * NT + tid, so a
//     warp's B loads are 128-byte coalesced rows) and ALL bm rows; B streams
//     from global memory straight into registers (ld.global.nc, half a K
//     block ahead), the small A tile (bm x 32 k per block) is staged once per
//     CTA by TMA into a D-deep mbarrier ring and read as broadcast LDS.128.
//     B needs no alignment (N = 8457 works); A needs 16-byte rows.
//
// Both split K over `uk` CTAs that form one thread-block cluster (1 x uk):
// every CTA parks its partial tile in its own shared memory and, after a
// cluster barrier, CTA z reduces its 1/uk share of the tile over the slices
// in order 0..uk-1 through DSMEM and stores alpha * sum (+ beta * C).  One
// launch, no partial slabs in HBM, fixed summation order (bitwise
// repeatable).  Work per unit = 2MNK flops; algorithmic bytes = 4(MK + KN +
// MN); these shapes sit near the FFMA ridge (AI 8-17 FLOP/B), so the kernels
// are built to stream the big operand at HBM rate with 8+ warps per SM.
//
// Calls the kernels cannot take (transposes, unaligned rows for the TMA
// operands, float64) run the split-K family's run-time-tile path instead.
#pragma once
#include "kernels.cuh"
#include "launch.cuh"
#include "tc_kernels.cuh"

namespace ag {
namespace skinny {

constexpr int BK = 32;  // one 128-byte swizzle row of fp32 per K block

struct Params {
    int M, N, K;
    float alpha, beta;
    int use_c, vec_out;
    const float* B;
    i64 ldb;
    const float* C;
    i64 ldc;
    float* out;
    i64 ldo;
    int kb_per_slice;  // K blocks per slice (grid.y = slices)
    int tiles_m;       // grid.x = tiles_m * tiles_n
    int depth;         // skinny_n: TMA ring depth per warp (run time)
};

__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory"); }

__device__ __forceinline__ float ldg_stream(const float* p, bool ok) {
    float v = 0.f;
    if (ok) asm("ld.global.nc.L1::no_allocate.f32 %0, [%1];\n" : "=f"(v) : "l"(p));
    return v;
}

// Reduce the S partial tiles of a cluster (S = gridDim.y, cluster dims
// 1 x S) and store the output tile.  `part` is this CTA's partial tile,
// ROWS x COLS fp32 at row stride RS, complete and visible to the CTA.
template <int ROWS, int COLS, int RS, int NT>
__device__ __forceinline__ void reduce_store(const float* part, const Params& p, int m0, int n0) {
    static_assert(COLS % 4 == 0 && RS % 4 == 0, "float4 chunks");
    constexpr int QR = COLS / 4, Q = ROWS * QR;
    const int S = gridDim.y, tid = threadIdx.x;
    if (S > 1) tc::cluster_sync();
    const int z = S > 1 ? (int)blockIdx.y : 0;
    const int q0 = (int)((long long)Q * z / S), q1 = (int)((long long)Q * (z + 1) / S);
    const uint32_t local = smem_addr(part);
    for (int q = q0 + tid; q < q1; q += NT) {
        const int r = q / QR, c = (q - r * QR) * 4;
        const int off = (r * RS + c) * 4;
        float4 sum;
        if (S > 1) {
            for (int src = 0; src < S; ++src) {
                uint32_t remote;
                asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(remote) : "r"(local + off), "r"(src));
                float4 v;
                asm volatile("ld.shared::cluster.v4.f32 {%0, %1, %2, %3}, [%4];"
                             : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
                             : "r"(remote));
                if (src == 0) {
                    sum = v;
                } else {
                    sum.x += v.x; sum.y += v.y; sum.z += v.z; sum.w += v.w;
                }
            }
        } else {
            sum = *reinterpret_cast<const float4*>(part + r * RS + c);
        }
        const int gm = m0 + r, gn = n0 + c;
        if (gm >= p.M || gn >= p.N) continue;
        if (p.vec_out && gn + 4 <= p.N) {
            float4 o = make_float4(p.alpha * sum.x, p.alpha * sum.y, p.alpha * sum.z, p.alpha * sum.w);
            if (p.use_c) {
                const float4 cc = *reinterpret_cast<const float4*>(p.C + (i64)gm * p.ldc + gn);
                o = make_float4(fmadd(p.alpha, sum.x, p.beta * cc.x), fmadd(p.alpha, sum.y, p.beta * cc.y),
                                fmadd(p.alpha, sum.z, p.beta * cc.z), fmadd(p.alpha, sum.w, p.beta * cc.w));
            }
            *reinterpret_cast<float4*>(p.out + (i64)gm * p.ldo + gn) = o;
        } else {
            const float sv[4] = {sum.x, sum.y, sum.z, sum.w};
#pragma unroll
            for (int e = 0; e < 4; ++e) {
                if (gn + e >= p.N) break;
                const i64 o = (i64)gm * p.ldo + gn + e;
                p.out[o] = p.use_c ? fmadd(p.alpha, sv[e], p.beta * p.C[(i64)gm * p.ldc + gn + e]) : p.alpha * sv[e];
            }
        }
    }
    // no CTA may leave while a peer still reads its shared memory
    if (S > 1) tc::cluster_sync();
}

// ------------------------------------------------------------------ skinny_n
// bm = 32 * TM rows per CTA; the NW warps split the CTA's K range block by
// block (warp w takes blocks w, w + NW, ...), each with its own TMA ring, so
// no warp waits on another in the main loop.  The ring depth D is chosen at
// launch: every block of the warp when that fits (the whole slice is in
// flight from the first cycle), else as deep as the shared memory of one
// (grid <= #SMs) or two CTAs per SM allows.
template <int TM, int BN, int NW>
struct NShape {
    static constexpr int BM = 32 * TM, NT = NW * 32, RS = BN + 4;
    static constexpr uint32_t A_BYTES = BM * 128, B_BYTES = BK * BN * 4, STAGE = A_BYTES + B_BYTES;
    static constexpr size_t RED = (size_t)NW * BM * RS * 4;
    static constexpr size_t ring(int d) { return (size_t)NW * d * STAGE; }
    static constexpr size_t smem(int d) { return 1024 + (ring(d) > RED ? ring(d) : RED) + NW * d * 8 + 64; }
};

template <int TM, int BN, int NW>
__global__ void __launch_bounds__(NW * 32)
skinny_n_kernel(const __grid_constant__ CUtensorMap mapA, const __grid_constant__ CUtensorMap mapB, const Params p) {
    using S_ = NShape<TM, BN, NW>;
    constexpr int BM = S_::BM, NT = S_::NT, RS = S_::RS;
    constexpr uint32_t A_BYTES = S_::A_BYTES, B_BYTES = S_::B_BYTES;
    static_assert(BN % 4 == 0 && TM >= 1 && TM <= 8, "tile");
    const int D = p.depth;

    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = smem_raw + ((1024u - (smem_addr(smem_raw) & 1023u)) & 1023u);
    uint8_t* sA = smem;                                 // [NW][D][BM][128 B], 128-byte swizzle
    uint8_t* sB = smem + (size_t)NW * D * A_BYTES;      // [NW][D][BK][BN]
    const size_t ring = (size_t)NW * D * (A_BYTES + B_BYTES);
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + (ring > S_::RED ? ring : S_::RED));

    const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
    const int tile_m = blockIdx.x % p.tiles_m, tile_n = blockIdx.x / p.tiles_m;
    const int m0 = tile_m * BM, n0 = tile_n * BN;
    const int nkb = (p.K + BK - 1) / BK;
    const int kb0 = blockIdx.y * p.kb_per_slice;
    const int kb1 = min(nkb, kb0 + p.kb_per_slice);
    const int mine = (kb1 - kb0 > w) ? (kb1 - kb0 - w + NW - 1) / NW : 0;
    uint64_t* fw = full + w * D;
    if (tid == 0) {
        asm volatile("prefetch.tensormap [%0];\n" ::"l"(reinterpret_cast<uint64_t>(&mapA)) : "memory");
        asm volatile("prefetch.tensormap [%0];\n" ::"l"(reinterpret_cast<uint64_t>(&mapB)) : "memory");
        for (int s = 0; s < NW * D; ++s) tc::mbar_init(&full[s], 1);
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    }
    __syncthreads();

    auto issue = [&](int j) {
        const int s = j % D, kb = kb0 + w + j * NW;
        tc::mbar_expect_tx(&fw[s], A_BYTES + B_BYTES);
        tc::tma_load_2d(sA + (size_t)(w * D + s) * A_BYTES, &mapA, &fw[s], kb * BK, m0);
        tc::tma_load_2d(sB + (size_t)(w * D + s) * B_BYTES, &mapB, &fw[s], n0, kb * BK);
    };
    if (lane == 0)
        for (int j = 0; j < D && j < mine; ++j) issue(j);

    f32x2 acc[TM][BN / 2];
#pragma unroll
    for (int i = 0; i < TM; ++i)
#pragma unroll
        for (int j = 0; j < BN / 2; ++j) acc[i][j] = 0ull;

    for (int j = 0; j < mine; ++j) {
        const int s = j % D;
        tc::mbar_wait(&fw[s], (uint32_t)((j / D) & 1));
        const uint8_t* as = sA + (size_t)(w * D + s) * A_BYTES;
        const float* bs = reinterpret_cast<const float*>(sB + (size_t)(w * D + s) * B_BYTES);
#pragma unroll
        for (int k0 = 0; k0 < BK; k0 += 4) {
            float av[TM][4];
#pragma unroll
            for (int i = 0; i < TM; ++i) {
                const int r = i * 32 + lane;
                const float4 v = *reinterpret_cast<const float4*>(as + r * 128 + (((k0 >> 2) ^ (r & 7)) << 4));
                av[i][0] = v.x; av[i][1] = v.y; av[i][2] = v.z; av[i][3] = v.w;
            }
#pragma unroll
            for (int kk = 0; kk < 4; ++kk) {
                const float* brow = bs + (k0 + kk) * BN;
#pragma unroll
                for (int g = 0; g < BN / 4; ++g) {
                    const float4 b4 = *reinterpret_cast<const float4*>(brow + 4 * g);  // broadcast
                    const f32x2 b01 = pack2(b4.x, b4.y), b23 = pack2(b4.z, b4.w);
#pragma unroll
                    for (int i = 0; i < TM; ++i) {
                        ffma2(acc[i][2 * g], av[i][kk], b01);
                        ffma2(acc[i][2 * g + 1], av[i][kk], b23);
                    }
                }
            }
        }
        __syncwarp();
        if (lane == 0 && j + D < mine) {
            fence_proxy_async();  // the warp's generic reads of slot s precede the TMA overwrite
            issue(j + D);
        }
    }
    __syncthreads();  // every warp is done with the ring: reuse it for the partial tiles

    float* red = reinterpret_cast<float*>(smem);  // [NW][BM][RS]
#pragma unroll
    for (int i = 0; i < TM; ++i) {
        const int r = i * 32 + lane;
        float* dst = red + ((size_t)w * BM + r) * RS;
#pragma unroll
        for (int g = 0; g < BN / 4; ++g) {
            float4 o;
            unpack2(acc[i][2 * g], o.x, o.y);
            unpack2(acc[i][2 * g + 1], o.z, o.w);
            *reinterpret_cast<float4*>(dst + 4 * g) = o;
        }
    }
    __syncthreads();
    // the CTA's partial tile = the warps' tiles summed in warp order, into red[0]
    for (int q = tid; q < BM * BN / 4; q += NT) {
        const int r = q / (BN / 4), c = (q - r * (BN / 4)) * 4;
        float4 sum = *reinterpret_cast<const float4*>(red + r * RS + c);
#pragma unroll
        for (int ww = 1; ww < NW; ++ww) {
            const float4 v = *reinterpret_cast<const float4*>(red + ((size_t)ww * BM + r) * RS + c);
            sum.x += v.x; sum.y += v.y; sum.z += v.z; sum.w += v.w;
        }
        *reinterpret_cast<float4*>(red + r * RS + c) = sum;
    }
    __syncthreads();
    reduce_store<BM, BN, RS, NT>(red, p, m0, n0);
}

// ------------------------------------------------------------------ skinny_m
template <int BM, int TN2, int NW, int D>
struct MShape {
    static constexpr int NT = NW * 32, BNC = NT * TN2, RS = BNC;
    static constexpr uint32_t A_BYTES = BM * 128;
    static constexpr size_t RING = (size_t)D * A_BYTES;
    static constexpr size_t PART = (size_t)BM * RS * 4;
    static constexpr size_t SMEM = 1024 + (RING > PART ? RING : PART) + 2 * D * 8 + 64;
};

// B streams through registers in QK-k granules, NBUF granule buffers deep
// (NBUF - 1 granules in flight ahead of the FMAs; NBUF divides BK / QK so
// every buffer index is a compile-time constant).
template <int BM, int TN2, int NW, int D, int QK = 8, int NBUF = 2>
__global__ void __launch_bounds__(NW * 32, NW == 4 ? (NBUF > 2 ? 2 : 3) : 1)
skinny_m_kernel(const __grid_constant__ CUtensorMap mapA, const Params p) {
    using S_ = MShape<BM, TN2, NW, D>;
    constexpr int NT = S_::NT, BNC = S_::BNC, RS = S_::RS;
    static_assert((BK / QK) % NBUF == 0 && QK % 4 == 0, "granule ring");
    constexpr uint32_t A_BYTES = S_::A_BYTES;
    static_assert(BM % 4 == 0 && TN2 % 2 == 0, "tile");

    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = smem_raw + ((1024u - (smem_addr(smem_raw) & 1023u)) & 1023u);
    uint8_t* sA = smem;  // [D][BM][128 B], 128-byte swizzle
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + (S_::RING > S_::PART ? S_::RING : S_::PART));
    uint64_t* empty = full + D;

    const int tid = threadIdx.x, lane = tid & 31;
    const int tile_m = blockIdx.x % p.tiles_m, tile_n = blockIdx.x / p.tiles_m;
    const int m0 = tile_m * BM, n0 = tile_n * BNC;
    const int nkb = (p.K + BK - 1) / BK;
    const int kb0 = blockIdx.y * p.kb_per_slice;
    const int kb1 = min(nkb, kb0 + p.kb_per_slice);
    const int nk = max(kb1 - kb0, 0);
    if (tid == 0) {
        asm volatile("prefetch.tensormap [%0];\n" ::"l"(reinterpret_cast<uint64_t>(&mapA)) : "memory");
        for (int s = 0; s < D; ++s) {
            tc::mbar_init(&full[s], 1);
            tc::mbar_init(&empty[s], NW);
        }
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    }
    __syncthreads();
    auto issue = [&](int j) {
        const int s = j % D;
        tc::mbar_expect_tx(&full[s], A_BYTES);
        tc::tma_load_2d(sA + (size_t)s * A_BYTES, &mapA, &full[s], (kb0 + j) * BK, m0);
    };
    if (tid == 0)
        for (int j = 0; j < D - 1 && j < nk; ++j) issue(j);

    // the thread's columns and their in-range flags
    const float* bcol[TN2];
    bool cok[TN2];
#pragma unroll
    for (int c = 0; c < TN2; ++c) {
        const int gn = n0 + c * NT + tid;
        cok[c] = gn < p.N;
        bcol[c] = p.B + (cok[c] ? gn : 0);
    }
    // B granules (QK k x TN2) in registers, NBUF - 1 granules ahead
    float bq[NBUF][QK][TN2];
    auto load_q = [&](int q, float (&dst)[QK][TN2]) {  // granule q of this slice (4 per K block)
        const int kbase = kb0 * BK + q * QK;
#pragma unroll
        for (int kk = 0; kk < QK; ++kk) {
            const int k = kbase + kk;
            const bool kin = k < p.K;
#pragma unroll
            for (int c = 0; c < TN2; ++c) dst[kk][c] = ldg_stream(bcol[c] + (i64)k * p.ldb, kin && cok[c]);
        }
    };
    f32x2 acc[BM][TN2 / 2];
#pragma unroll
    for (int m = 0; m < BM; ++m)
#pragma unroll
        for (int c = 0; c < TN2 / 2; ++c) acc[m][c] = 0ull;

    constexpr int QPB = BK / QK;  // granules per K block
#pragma unroll
    for (int g = 0; g < NBUF - 1; ++g)
        if (g < QPB * nk) load_q(g, bq[g]);
    for (int j = 0; j < nk; ++j) {
        const int s = j % D;
        if (tid == 0) {  // refill the slot of block j - 1 with block j + D - 1
            const int nt = j + D - 1;
            if (nt < nk) {
                if (nt >= D) tc::mbar_wait(&empty[nt % D], (uint32_t)((nt / D - 1) & 1));
                issue(nt);
            }
        }
        tc::mbar_wait(&full[s], (uint32_t)((j / D) & 1));
        const uint8_t* as = sA + (size_t)s * A_BYTES;
#pragma unroll
        for (int h = 0; h < QPB; ++h) {
            const int qq = QPB * j + h;
            if (qq + NBUF - 1 < QPB * nk) load_q(qq + NBUF - 1, bq[(h + NBUF - 1) % NBUF]);
            const float(&b)[QK][TN2] = bq[h % NBUF];
#pragma unroll
            for (int k4 = 0; k4 < QK; k4 += 4) {
                f32x2 bp[4][TN2 / 2];
#pragma unroll
                for (int kk = 0; kk < 4; ++kk)
#pragma unroll
                    for (int c = 0; c < TN2 / 2; ++c) bp[kk][c] = pack2(b[k4 + kk][2 * c], b[k4 + kk][2 * c + 1]);
                const int chunk = (h * QK + k4) >> 2;
                // 4 rows at a time: 4 broadcast LDS.128, then 16 independent FFMA2 chains per k
#pragma unroll
                for (int m = 0; m < BM; m += 4) {
                    float av[4][4];
#pragma unroll
                    for (int mm = 0; mm < 4; ++mm) {
                        const float4 a4 =
                            *reinterpret_cast<const float4*>(as + (m + mm) * 128 + ((chunk ^ ((m + mm) & 7)) << 4));
                        av[mm][0] = a4.x; av[mm][1] = a4.y; av[mm][2] = a4.z; av[mm][3] = a4.w;
                    }
#pragma unroll
                    for (int kk = 0; kk < 4; ++kk)
#pragma unroll
                        for (int mm = 0; mm < 4; ++mm)
#pragma unroll
                            for (int c = 0; c < TN2 / 2; ++c) ffma2(acc[m + mm][c], av[mm][kk], bp[kk][c]);
                }
            }
        }
        __syncwarp();
        if (lane == 0) tc::mbar_arrive(&empty[s]);
    }
    __syncthreads();  // the ring is free: the partial tile overlays it

    float* part = reinterpret_cast<float*>(smem);  // [BM][RS]
#pragma unroll
    for (int m = 0; m < BM; ++m)
#pragma unroll
        for (int c = 0; c < TN2 / 2; ++c) {
            float lo, hi;
            unpack2(acc[m][c], lo, hi);
            part[m * RS + (2 * c) * NT + tid] = lo;
            part[m * RS + (2 * c + 1) * NT + tid] = hi;
        }
    __syncthreads();
    reduce_store<BM, BNC, RS, NT>(part, p, m0, n0);
}

// ------------------------------------------------------------------ launchers
inline bool make_map(CUtensorMap* m, const float* base, i64 rows, i64 cols, i64 ld, int box_cols, int box_rows,
                     bool swizzle) {
    auto fn = tc::encode_fn();
    if (!fn) return false;
    cuuint32_t estr[2] = {1, 1};
    cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows}, strides[1] = {(cuuint64_t)(ld * 4)};
    cuuint32_t box[2] = {(cuuint32_t)box_cols, (cuuint32_t)box_rows};
    return fn(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float*>(base), dims, strides, box, estr,
              CU_TENSOR_MAP_INTERLEAVE_NONE, swizzle ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_NONE,
              CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// the split-K family's run-time-tile path: the calls a skinny kernel cannot take
inline int fallback(const GemmCall& c) {
    GemmCall f = c;
    f.bm = 64; f.bn = 64; f.bk = 16; f.tm = 4; f.tn = 4; f.uk = 1;
    f.splits = c.splits;
    if (c.dtype == AG_F64) return launch_indirect<double, 0, 0, 0, 4, 4, 1>(f);
    return launch_indirect<float, 0, 0, 0, 4, 4, 1>(f);
}

inline Params base_params(const GemmCall& c) {
    Params p{};
    p.M = (int)c.M; p.N = (int)c.N; p.K = (int)c.K;
    p.alpha = (float)c.alpha; p.beta = (float)c.beta;
    p.use_c = c.beta != 0.0;
    p.vec_out = (c.ldo % 4 == 0) && aligned(c.out, 16) && (!p.use_c || ((c.ldc % 4 == 0) && aligned(c.C, 16)));
    p.B = static_cast<const float*>(c.B); p.ldb = c.ldb;
    p.C = static_cast<const float*>(c.C); p.ldc = c.ldc;
    p.out = static_cast<float*>(c.out); p.ldo = c.ldo;
    return p;
}

// grid (tiles, slices); the slices of a tile form one cluster (1 x slices;
// > 8 uses the non-portable cluster size)
// (`granted` / `np_ok`: the calling launcher's per-kernel, per-device state)
template <typename K, typename... Args>
int launch_sliced(const GemmCall& c, K kernel, SmemGrant& granted, PerDevice<int>& np_ok, size_t smem, int threads,
                  i64 tiles, int slices, Args... args) {
    if (ensure_smem(kernel, smem, granted) != cudaSuccess) return fail(c, AG_ERR_CUDA, "cudaFuncSetAttribute failed");
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)tiles, (unsigned)slices);
    cfg.blockDim = dim3(threads);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = c.stream;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = 1;
    attr[0].val.clusterDim.y = (unsigned)slices;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = slices > 1 ? 1 : 0;
    if (slices > 8) {
        if (!np_ok.here().load()) {
            if (cudaFuncSetAttribute(kernel, cudaFuncAttributeNonPortableClusterSizeAllowed, 1) != cudaSuccess)
                return fail(c, AG_ERR_CUDA, "non-portable cluster size not available");
            np_ok.here().store(1);
        }
    }
    if (cudaLaunchKernelEx(&cfg, kernel, args...) != cudaSuccess || cudaGetLastError() != cudaSuccess)
        return fail(c, AG_ERR_CUDA, "skinny kernel launch failed");
    return AG_OK;
}

inline int slices_for(i64 K, int want, int* kb_per) {
    const i64 nkb = (K + BK - 1) / BK;
    const int s = (int)std::max<i64>(1, std::min<i64>(want, nkb));
    *kb_per = (int)((nkb + s - 1) / s);
    return (int)((nkb + *kb_per - 1) / *kb_per);
}

// skinny_n:bm-bn-32-tm-nw-slices, bm = 32 tm
template <int TM, int BN, int NW>
int launch_n(const GemmCall& c) {
    using S_ = NShape<TM, BN, NW>;
    static_assert(S_::smem(2) <= 227 * 1024, "skinny_n ring exceeds shared memory");
    const bool ok = c.dtype == AG_F32 && !c.ta && !c.tb && c.K % 4 == 0 && c.N % 4 == 0 && c.lda % 4 == 0 &&
                    c.ldb % 4 == 0 && aligned(c.A, 16) && aligned(c.B, 16) && c.splits <= 16;
    if (!ok) return fallback(c);
    const i64 tiles_m = (c.M + S_::BM - 1) / S_::BM, tiles_n = (c.N + BN - 1) / BN;
    if (tiles_m * tiles_n > 0x7fffffffLL || c.K > 0x7fffffffLL) return fail(c, AG_ERR_SHAPE, "problem too large");
    Params p = base_params(c);
    const int slices = slices_for(c.K, c.splits, &p.kb_per_slice);
    p.tiles_m = (int)tiles_m;
    // ring depth: all of a warp's blocks if they fit, within one CTA per SM
    // when the grid is a single wave of one CTA per SM, else two
    const int per_warp = (p.kb_per_slice + NW - 1) / NW;
    const size_t budget = (tiles_m * tiles_n * slices <= device_sms() ? 220 : 110) * 1024;
    int depth = std::max(2, std::min(per_warp, 8));
    while (depth > 2 && S_::smem(depth) > budget) --depth;
    p.depth = depth;
    const size_t smem = S_::smem(depth);
    CUtensorMap mA, mB;
    if (!make_map(&mA, static_cast<const float*>(c.A), c.M, c.K, c.lda, BK, S_::BM, true) ||
        !make_map(&mB, static_cast<const float*>(c.B), c.K, c.N, c.ldb, BN, BK, false))
        return fail(c, AG_ERR_CUDA, "cuTensorMapEncodeTiled failed");
    static SmemGrant granted;
    static PerDevice<int> np_ok;
    return launch_sliced(c, skinny_n_kernel<TM, BN, NW>, granted, np_ok, smem, S_::NT, tiles_m * tiles_n, slices, mA,
                         mB, p);
}

// skinny_m:bm-bn-32-1-tn2-slices, bn = 32 nw tn2
template <int BM, int TN2, int NW, int QK = 8, int NBUF = 2>
int launch_m(const GemmCall& c) {
    constexpr int D = 4;
    using S_ = MShape<BM, TN2, NW, D>;
    static_assert(S_::SMEM <= 227 * 1024, "skinny_m partial tile exceeds shared memory");
    const bool ok = c.dtype == AG_F32 && !c.ta && !c.tb && c.K % 4 == 0 && c.lda % 4 == 0 && aligned(c.A, 16) &&
                    c.splits <= 16;
    if (!ok) return fallback(c);
    const i64 tiles_m = (c.M + BM - 1) / BM, tiles_n = (c.N + S_::BNC - 1) / S_::BNC;
    if (tiles_m * tiles_n > 0x7fffffffLL || c.K > 0x7fffffffLL) return fail(c, AG_ERR_SHAPE, "problem too large");
    Params p = base_params(c);
    const int slices = slices_for(c.K, c.splits, &p.kb_per_slice);
    p.tiles_m = (int)tiles_m;
    CUtensorMap mA;
    if (!make_map(&mA, static_cast<const float*>(c.A), c.M, c.K, c.lda, BK, BM, true))
        return fail(c, AG_ERR_CUDA, "cuTensorMapEncodeTiled failed");
    static SmemGrant granted;
    static PerDevice<int> np_ok;
    return launch_sliced(c, skinny_m_kernel<BM, TN2, NW, D, QK, NBUF>, granted, np_ok, S_::SMEM, S_::NT,
                         tiles_m * tiles_n,
                         slices, mA, p);
}

}  // namespace skinny
}  // namespace ag
