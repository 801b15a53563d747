// launch.cuh -- host-side launchers for one kernel instantiation.
//
// A launcher runs the complete family path of one config on one stream:
//   direct   : one predicated kernel on the caller's operands
//   indirect : [pack op(A)^T] [pack op(B)] tiled core (masked epilogue);
//              a pack is skipped when the operand already is a tile-multiple,
//              16-byte aligned matrix in the layout the core streams
//              (CLBlast-style "helpers only when needed").
#pragma once
#include <algorithm>
#include <atomic>
#include <cstdlib>
#include <cstdio>
#include <string>
#include <type_traits>
#include <utility>

#include "kernels.cuh"
#include "registry.h"

namespace ag {

inline i64 round_up(i64 x, i64 s) { return (x + s - 1) / s * s; }

// Per-device one-shot state.  Kernel attributes (cudaFuncSetAttribute) and
// device properties apply to the CURRENT device, so every cache below is
// indexed by it: one process may drive several GPUs.
constexpr int kMaxDevices = 64;
inline int current_device() {
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= kMaxDevices) dev = 0;
    return dev;
}
template <typename T>
struct PerDevice {
    std::atomic<T> v[kMaxDevices];
    PerDevice() {
        for (auto& x : v) x.store(T(0));
    }
    std::atomic<T>& here() { return v[current_device()]; }
};

// SM count of the current device (grid sizing)
inline int device_sms() {
    static PerDevice<int> cache;
    auto& slot = cache.here();
    int n = slot.load(std::memory_order_relaxed);
    if (n > 0) return n;
    if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, current_device()) != cudaSuccess || n <= 0) n = 148;
    slot.store(n);
    return n;
}

// raise the per-kernel dynamic shared-memory limit once per needed size and device
using SmemGrant = PerDevice<size_t>;
template <typename K>
inline cudaError_t ensure_smem(K kernel, size_t bytes, SmemGrant& grants) {
    if (bytes <= 48 * 1024) return cudaSuccess;
    std::atomic<size_t>& granted = grants.here();
    if (bytes <= granted.load(std::memory_order_relaxed)) return cudaSuccess;
    cudaError_t e = cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
    if (e == cudaSuccess) {
        size_t cur = granted.load();
        while (bytes > cur && !granted.compare_exchange_weak(cur, bytes)) {
        }
    }
    return e;
}

inline bool aligned(const void* p, size_t a) { return (reinterpret_cast<uintptr_t>(p) % a) == 0; }

// Launch `kernel` on `stream`, as a programmatic dependent launch when
// `dependent` (the previous kernel on the stream is this call's own helper
// pass, which triggers griddepcontrol.launch_dependents): the launch and CTA
// setup overlap that helper's tail, and the kernel's griddepcontrol.wait
// holds every global access until the helper has completed.  The first
// kernel of a family path is never dependent, so nothing overlaps work the
// caller queued before the call.
template <typename... KArgs, typename... Args>
inline cudaError_t launch_maybe_dependent(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem,
                                          cudaStream_t stream, bool dependent, Args&&... args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = stream;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = dependent ? 1 : 0;
    return cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...);
}

inline int fail(const GemmCall& c, int code, const std::string& msg) {
    if (c.err) *c.err = msg;
    return code;
}

template <typename T>
int launch_pack(T* dst, i64 ld_dst, i64 dst_rows, i64 dst_cols, const T* src, i64 ld_src,
                i64 rows, i64 cols, int transpose, cudaStream_t stream) {
    constexpr int W = VecW<T>::W;
    if (!transpose && dst_cols % W == 0 && ld_dst % W == 0 && aligned(dst, 16)) {
        const bool vec = ld_src % W == 0 && aligned(src, 16);
        const i64 total = dst_rows * (dst_cols / W);
        const int sms = device_sms();  // grid sizing only
        const unsigned blocks = (unsigned)std::max<i64>(1, std::min<i64>((total + 1023) / 1024, (i64)sms * 8));
        if (vec)
            pack_copy_kernel<T, true><<<blocks, 256, 0, stream>>>(dst, ld_dst, (int)dst_rows, (int)dst_cols, src,
                                                                  ld_src, (int)rows, (int)cols);
        else
            pack_copy_kernel<T, false><<<blocks, 256, 0, stream>>>(dst, ld_dst, (int)dst_rows, (int)dst_cols, src,
                                                                   ld_src, (int)rows, (int)cols);
        return cudaGetLastError() == cudaSuccess ? AG_OK : AG_ERR_CUDA;
    }
    dim3 grid((unsigned)((dst_cols + 31) / 32), (unsigned)((dst_rows + 31) / 32));
    if (grid.y > 65535u) return AG_ERR_SHAPE;
    pack_pad_kernel<T><<<grid, dim3(32, 8), 0, stream>>>(dst, ld_dst, (int)dst_rows, (int)dst_cols, src, ld_src,
                                                         (int)rows, (int)cols, transpose);
    return cudaGetLastError() == cudaSuccess ? AG_OK : AG_ERR_CUDA;
}

template <typename T, int BM, int BN, int BK, int TM, int TN>
int launch_direct(const GemmCall& c) {
    const int bm = BM ? BM : c.bm, bn = BN ? BN : c.bn, bk = BK ? BK : c.bk;
    const int threads = (bm / TM) * (bn / TN);
    if (threads > cta_threads_bound<T, BM, BN, TM, TN>())
        return fail(c, AG_ERR_CONFIG, "config needs more threads per CTA than its kernel supports");
    const size_t smem = direct_smem_bytes<T>(bm, bn, bk);
    if (smem > 227 * 1024) return fail(c, AG_ERR_CONFIG, "config exceeds 227 KB shared memory per CTA");
    auto kernel = direct_gemm_kernel<T, BM, BN, BK, TM, TN>;
    static SmemGrant granted;
    if (ensure_smem(kernel, smem, granted) != cudaSuccess) return fail(c, AG_ERR_CUDA, "cudaFuncSetAttribute failed");
    const i64 gy = (c.M + bm - 1) / bm, gx = (c.N + bn - 1) / bn;
    if (gy > 65535 || gx > 0x7fffffff) return fail(c, AG_ERR_SHAPE, "problem too large for the direct grid");
    DirectParams<T> p;
    p.M = (int)c.M; p.N = (int)c.N; p.K = (int)c.K;
    p.alpha = (T)c.alpha; p.beta = (T)c.beta;
    p.ta = c.ta; p.tb = c.tb;
    p.A = static_cast<const T*>(c.A); p.lda = c.lda;
    p.B = static_cast<const T*>(c.B); p.ldb = c.ldb;
    p.C = static_cast<const T*>(c.C); p.ldc = c.ldc;
    p.out = static_cast<T*>(c.out); p.ldo = c.ldo;
    p.bm = bm; p.bn = bn; p.bk = bk;
    kernel<<<dim3((unsigned)gx, (unsigned)gy), threads, smem, c.stream>>>(p);
    return cudaGetLastError() == cudaSuccess ? AG_OK : fail(c, AG_ERR_CUDA, "direct kernel launch failed");
}

// in-place core (split-K family) shared memory: A stage [bm][bk + 4], B stage [bk][bn]
constexpr size_t inplace_stage_bytes(int bm, int bn, int bk) { return (size_t)(bm * (bk + 4) + bk * bn) * 4; }
constexpr int inplace_stages(int bm, int bn, int bk) {
    return 4 * inplace_stage_bytes(bm, bn, bk) <= 96 * 1024 ? 4 : (3 * inplace_stage_bytes(bm, bn, bk) <= 200 * 1024 ? 3 : 2);
}
// the ring also holds one partial tile (bm x bn fp32) for the cluster reduction
constexpr size_t inplace_smem_bytes(int bm, int bn, int bk) {
    return inplace_stages(bm, bn, bk) * inplace_stage_bytes(bm, bn, bk) > (size_t)bm * bn * 4
               ? inplace_stages(bm, bn, bk) * inplace_stage_bytes(bm, bn, bk)
               : (size_t)bm * bn * 4;
}

// [At | Bp | split-K partial slabs], each 256-byte aligned
template <typename T>
size_t indirect_workspace_bytes(i64 M, i64 N, i64 K, int bm, int bn, int bk, int splits = 1) {
    const i64 Mp = round_up(M, bm), Np = round_up(N, bn), Kp = round_up(K, bk);
    size_t b = (size_t)round_up(Kp * Mp * (i64)sizeof(T), 256) + (size_t)round_up(Kp * Np * (i64)sizeof(T), 256);
    if (splits > 1) b += (size_t)round_up((i64)splits * Mp * Np * (i64)sizeof(T), 256);
    return b;
}

// L2-friendly tile grouping (CUTLASS-style swizzle): consecutive CTAs walk
// `group` row tiles of one column band, so op(B) is streamed from HBM once
// per group.  The group is as tall as ~32 MB of packed op(A) rows allows
// (>= 8 tiles), which keeps a group's A panel L2-resident (126 MB) while
// cutting the B re-reads: 5124 x 9124 x 2560 at 128 x 128 tiles goes from
// 5 B passes (group 8) to 2 (group 24).
inline int group_rows(i64 tiles_m, i64 bm, i64 Kp, size_t elem) {
    const i64 budget = 32LL << 20;
    i64 g = budget / std::max<i64>(1, bm * Kp * (i64)elem);
    g = std::max<i64>(g, 8);
    return (int)std::min<i64>(g, tiles_m);
}

// the split-K family's in-place path: in-place core over `splits` K slices
// into the partial slabs, then the fixed-order reduction (same slices, same
// order as the packed path, so the same bits)
template <int BM, int BN, int BK, int TM, int TN>
int launch_inplace(const GemmCall& c) {
    constexpr int STAGES = inplace_stages(BM, BN, BK);
    constexpr size_t smem = inplace_smem_bytes(BM, BN, BK);
    static_assert(smem <= 227 * 1024, "in-place stage ring exceeds shared memory");
    auto kernel = inplace_gemm_kernel<BM, BN, BK, TM, TN, STAGES>;
    static SmemGrant granted;
    if (ensure_smem(kernel, smem, granted) != cudaSuccess) return fail(c, AG_ERR_CUDA, "cudaFuncSetAttribute failed");
    const i64 M = c.M, N = c.N, K = c.K;
    const i64 Mp = round_up(M, BM), Np = round_up(N, BN), Kp = round_up(K, BK);
    if (Mp > 0x7fffffff || Np > 0x7fffffff || Kp > 0x7fffffff) return fail(c, AG_ERR_SHAPE, "dimension too large");
    const int splits = c.splits > 1 ? c.splits : 1;
    const size_t need = indirect_workspace_bytes<float>(M, N, K, BM, BN, BK, splits);
    if (c.ws_bytes < need || (need && c.ws == nullptr))
        return fail(c, AG_ERR_SHAPE, "workspace too small for the split-K partial slabs");
    const i64 tiles_m = Mp / BM, tiles_n = Np / BN, ktiles = Kp / BK;
    if (tiles_m * tiles_n > 0x7fffffffLL) return fail(c, AG_ERR_SHAPE, "too many tiles");
    const int kps = (int)((ktiles + splits - 1) / splits);
    const int used_splits = (int)((ktiles + kps - 1) / kps);
    TiledParams<float> p;
    p.Mp = (int)Mp; p.Np = (int)Np; p.Kp = (int)Kp; p.M = (int)M; p.N = (int)N;
    p.alpha = (float)c.alpha; p.beta = (float)c.beta;
    p.use_c = c.beta != 0.0;
    // 16-byte vector stores (and C loads) when out / C rows allow them
    p.vec_out = (c.ldo % 4 == 0) && aligned(c.out, 16) && (!p.use_c || ((c.ldc % 4 == 0) && aligned(c.C, 16)));
    p.At = static_cast<const float*>(c.A); p.lda = c.lda;
    p.Bp = static_cast<const float*>(c.B); p.ldb = c.ldb;
    p.C = static_cast<const float*>(c.C); p.ldc = c.ldc;
    p.out = static_cast<float*>(c.out); p.ldo = c.ldo;
    p.bm = BM; p.bn = BN; p.bk = BK; p.uk = 1;
    p.tiles_m = (int)tiles_m; p.tiles_n = (int)tiles_n; p.group_m = group_rows(tiles_m, BM, Kp, sizeof(float));
    p.splits = used_splits; p.kt_per_split = kps;
    p.partial = reinterpret_cast<float*>(static_cast<char*>(c.ws) + round_up(Kp * Mp * (i64)sizeof(float), 256) +
                                         round_up(Kp * Np * (i64)sizeof(float), 256));
    const dim3 grid((unsigned)(tiles_m * tiles_n), (unsigned)used_splits);
    // one launch: the slices of a tile form a cluster and reduce over DSMEM
    // (up to 16 slices: non-portable cluster sizes above 8); otherwise the
    // slab + splitk_reduce_kernel path, same summation order
    p.cluster_red = 0;
#ifdef AG_NO_CLUSTER_REDUCE  // measurement knob (profiles/exp_tiles.cu): slab + reduce kernel only
    if (false) {
#else
    // AG_SPLITK_REDUCE=slab (measurement knob, profiles/reduce_mode_probe.py):
    // the slab + splitk_reduce_kernel path even where a cluster fits
    static const bool force_slab = [] {
        const char* e = std::getenv("AG_SPLITK_REDUCE");
        return e && std::string(e) == "slab";
    }();
    // Clusters of up to 8 slices (the portable size).  More slices take the
    // slab path: a 16-CTA non-portable cluster must be co-resident in one
    // GPC.  Over the 1200 (DeepBench shape, config) calls with > 8 slices the
    // slab path is 1.12x faster (geomean; median 1.13x, p10 1.00x, min
    // 0.90x); with 2..8 slices the two are even (1.007x) and the single
    // launch is kept (profiles/r02_reduce_mode_probe.jsonl).
    if (used_splits > 1 && used_splits <= 8 && !force_slab) {
#endif
        static PerDevice<int> np_ok_dev;
        std::atomic<int>& np_ok = np_ok_dev.here();
        if (used_splits > 8 && !np_ok.load()) {
            if (cudaFuncSetAttribute(kernel, cudaFuncAttributeNonPortableClusterSizeAllowed, 1) == cudaSuccess)
                np_ok.store(1);
            else
                cudaGetLastError();
        }
        if (used_splits <= 8 || np_ok.load()) {
            p.cluster_red = 1;
            cudaLaunchConfig_t cfg = {};
            cfg.gridDim = grid;
            cfg.blockDim = dim3((BM / TM) * (BN / TN));
            cfg.dynamicSmemBytes = smem;
            cfg.stream = c.stream;
            cudaLaunchAttribute attr[1];
            attr[0].id = cudaLaunchAttributeClusterDimension;
            attr[0].val.clusterDim.x = 1;
            attr[0].val.clusterDim.y = (unsigned)used_splits;
            attr[0].val.clusterDim.z = 1;
            cfg.attrs = attr;
            cfg.numAttrs = 1;
            if (cudaLaunchKernelEx(&cfg, kernel, p, (int)K) == cudaSuccess) return AG_OK;
            cudaGetLastError();  // cluster shape not schedulable: fall back
            p.cluster_red = 0;
        }
    }
    kernel<<<grid, (BM / TM) * (BN / TN), smem, c.stream>>>(p, (int)K);
    if (cudaGetLastError() != cudaSuccess) return fail(c, AG_ERR_CUDA, "in-place kernel launch failed");
    if (used_splits > 1) {
        const i64 total = M * N;
        const unsigned blocks = (unsigned)std::min<i64>((total + 255) / 256, (i64)device_sms() * 16);
        const cudaError_t le = launch_maybe_dependent(
            splitk_reduce_kernel<float>, dim3(blocks), dim3(256), 0, c.stream, true, (const float*)p.partial,
            used_splits, (i64)(Mp * Np), (int)Np, (int)M, (int)N, p.alpha, p.beta, p.use_c, p.C, (i64)c.ldc, p.out,
            (i64)c.ldo);
        if (le != cudaSuccess || cudaGetLastError() != cudaSuccess)
            return fail(c, AG_ERR_CUDA, "split-K reduce launch failed");
    }
    return AG_OK;
}

// AROW_OK (split-K family launchers): when op(A) is the caller's row-major
// A and M, K are tile multiples, run the AROW core that reads A in place
// instead of transpose-packing it.
// STAGES_OVERRIDE (experiments only, profiles/exp_tiles.cu): the cp.async
// ring depth instead of tiled_stages' choice.
template <typename T, int BM, int BN, int BK, int TM, int TN, int UK, bool AROW_OK = false, int STAGES_OVERRIDE = 0>
int launch_indirect(const GemmCall& c) {
    constexpr bool FIXED = BM > 0 && BN > 0 && BK > 0;
    constexpr int STAGES = STAGES_OVERRIDE ? STAGES_OVERRIDE : tiled_stages<T>(BM, BN, BK);
    constexpr int STAGES_AROW = tiled_stages<T>(BM + a_pad<T, true>(), BN, BK);
    constexpr int VL = FIXED ? VecW<T>::W : 1;
    constexpr int WB = FragW<T, TN>::W;
    const int bm = FIXED ? BM : c.bm, bn = FIXED ? BN : c.bn, bk = FIXED ? BK : c.bk;
    const int uk = FIXED ? UK : c.uk;
    const int threads = (bm / TM) * (bn / TN);
    if (threads > cta_threads_bound<T, BM, BN, TM, TN>())
        return fail(c, AG_ERR_CONFIG, "config needs more threads per CTA than its kernel supports");
    if (bk % uk) return fail(c, AG_ERR_CONFIG, "block_k must be a multiple of unroll_k");
    const i64 M = c.M, N = c.N, K = c.K;
    // split-K family, row-major operands with 16-byte rows: the in-place
    // core streams both straight from the caller's layout (no packs).  For
    // N > 64 with M, K tile multiples the AROW core (row-major A read in
    // place by element copies, B packed) is kept: there the op(B) pack is
    // small and the AROW core's main loop is the faster one (measured over
    // the DeepBench / po2 sweeps); for narrow N its element copies of A are
    // load-issue bound and the in-place core wins.
    const bool arow_fit = !c.ta && M % bm == 0 && K % bk == 0;
    const bool inplace = FIXED && AROW_OK && std::is_same<T, float>::value && !c.ta && !c.tb && K % 4 == 0 &&
                         N % 4 == 0 && c.lda % 4 == 0 && c.ldb % 4 == 0 && aligned(c.A, 16) &&
                         aligned(c.B, 16) && (N <= 64 || !arow_fit);
    if constexpr (FIXED && AROW_OK && std::is_same<T, float>::value) {
        if (inplace) return launch_inplace<BM, BN, BK, TM, TN>(c);
    }
    const bool arow = FIXED && AROW_OK && !c.ta && M % bm == 0 && K % bk == 0;
    const size_t smem = arow ? tiled_smem_bytes<T>(bm + a_pad<T, true>(), bn, bk, STAGES_AROW)
                             : tiled_smem_bytes<T>(bm, bn, bk, STAGES);
    if (smem > 227 * 1024) return fail(c, AG_ERR_CONFIG, "config exceeds 227 KB shared memory per CTA");
    auto kernel = tiled_gemm_kernel<T, BM, BN, BK, TM, TN, UK, STAGES>;
    static SmemGrant granted;
    cudaError_t attr = cudaSuccess;
    if constexpr (AROW_OK && FIXED) {
        static SmemGrant granted_arow;
        attr = arow ? ensure_smem(tiled_gemm_kernel<T, BM, BN, BK, TM, TN, UK, STAGES_AROW, true>, smem, granted_arow)
                    : ensure_smem(kernel, smem, granted);
    } else {
        attr = ensure_smem(kernel, smem, granted);
    }
    if (attr != cudaSuccess) return fail(c, AG_ERR_CUDA, "cudaFuncSetAttribute failed");

    const i64 Mp = round_up(M, bm), Np = round_up(N, bn), Kp = round_up(K, bk);
    if (Mp > 0x7fffffff || Np > 0x7fffffff || Kp > 0x7fffffff) return fail(c, AG_ERR_SHAPE, "dimension too large");
    const int splits = c.splits > 1 ? c.splits : 1;
    const size_t need = indirect_workspace_bytes<T>(M, N, K, bm, bn, bk, splits);
    if (c.ws_bytes < need || (need && c.ws == nullptr))
        return fail(c, AG_ERR_SHAPE, "workspace too small for the indirect pack buffers");
    const i64 tiles_m = Mp / bm, tiles_n = Np / bn, ktiles = Kp / bk;
    if (tiles_m * tiles_n > 0x7fffffffLL) return fail(c, AG_ERR_SHAPE, "too many tiles");
    // split-K: equal K-tile slices; splits beyond the K tiles collapse
    const int kps = (int)((ktiles + splits - 1) / splits);
    const int used_splits = (int)((ktiles + kps - 1) / kps);
    const size_t va = VL * sizeof(T);

    // op(A)^T, K-major (Kp x Mp): A itself when transA and already padded
    const T* At;
    i64 lda_t;
    bool packed = false;  // a helper pass precedes the core on the stream
    T* wsA = static_cast<T*>(c.ws);
    T* wsB = reinterpret_cast<T*>(static_cast<char*>(c.ws) + round_up(Kp * Mp * (i64)sizeof(T), 256));
    if (arow) {  // row-major A read in place by the AROW core
        At = static_cast<const T*>(c.A);
        lda_t = c.lda;
    } else if (c.ta && M == Mp && K == Kp && c.lda % VL == 0 && aligned(c.A, va)) {
        At = static_cast<const T*>(c.A);
        lda_t = c.lda;
    } else {
        int r = launch_pack<T>(wsA, Mp, Kp, Mp, static_cast<const T*>(c.A), c.lda, K, M, c.ta ? 0 : 1, c.stream);
        if (r) return fail(c, r, "pack of op(A) failed");
        At = wsA;
        lda_t = Mp;
        packed = true;
    }
    const T* Bp;
    i64 ldb_p;
    if (!c.tb && N == Np && K == Kp && c.ldb % VL == 0 && aligned(c.B, va)) {
        Bp = static_cast<const T*>(c.B);
        ldb_p = c.ldb;
    } else {
        int r = launch_pack<T>(wsB, Np, Kp, Np, static_cast<const T*>(c.B), c.ldb, K, N, c.tb ? 1 : 0, c.stream);
        if (r) return fail(c, r, "pack of op(B) failed");
        Bp = wsB;
        ldb_p = Np;
        packed = true;
    }

    TiledParams<T> p;
    p.Mp = (int)Mp; p.Np = (int)Np; p.Kp = (int)Kp; p.M = (int)M; p.N = (int)N;
    p.alpha = (T)c.alpha; p.beta = (T)c.beta;
    p.use_c = c.beta != 0.0;
    const size_t wb = WB * sizeof(T);
    p.vec_out = (c.ldo % WB == 0) && aligned(c.out, wb) && (!p.use_c || ((c.ldc % WB == 0) && aligned(c.C, wb)));
    p.At = At; p.lda = lda_t;
    p.Bp = Bp; p.ldb = ldb_p;
    p.C = static_cast<const T*>(c.C); p.ldc = c.ldc;
    p.out = static_cast<T*>(c.out); p.ldo = c.ldo;
    p.bm = bm; p.bn = bn; p.bk = bk; p.uk = uk;
    p.tiles_m = (int)tiles_m; p.tiles_n = (int)tiles_n; p.group_m = group_rows(tiles_m, bm, Kp, sizeof(T));
    p.splits = used_splits; p.kt_per_split = kps; p.cluster_red = 0;
    p.partial = reinterpret_cast<T*>(static_cast<char*>(c.ws) + round_up(Kp * Mp * (i64)sizeof(T), 256) +
                                     round_up(Kp * Np * (i64)sizeof(T), 256));
    const dim3 grid((unsigned)(tiles_m * tiles_n), (unsigned)used_splits);
    bool launched = false;
    cudaError_t le = cudaSuccess;
    // The core is NOT a dependent launch behind its packs: launched early,
    // its CTAs became resident wherever the pack left room and a single-wave
    // grid ended up unevenly spread (1024^3 at 64 x 64 tiles: 39 -> 23
    // TFLOP/s, profiles/r01_pdl_probe.jsonl).  The small split-K reduction
    // behind it is.
    (void)packed;
    if constexpr (AROW_OK && FIXED) {
        if (arow) {
            le = launch_maybe_dependent(tiled_gemm_kernel<T, BM, BN, BK, TM, TN, UK, STAGES_AROW, true>, grid,
                                        dim3(threads), smem, c.stream, false, p);
            launched = true;
        }
    }
    if (!launched) le = launch_maybe_dependent(kernel, grid, dim3(threads), smem, c.stream, false, p);
    if (le != cudaSuccess || cudaGetLastError() != cudaSuccess)
        return fail(c, AG_ERR_CUDA, "indirect kernel launch failed");
    if (used_splits > 1) {
        const i64 total = M * N;
        const unsigned blocks = (unsigned)std::min<i64>((total + 255) / 256, (i64)device_sms() * 16);
        le = launch_maybe_dependent(splitk_reduce_kernel<T>, dim3(blocks), dim3(256), 0, c.stream, true,
                                    (const T*)p.partial, used_splits, (i64)(Mp * Np), (int)Np, (int)M, (int)N,
                                    p.alpha, p.beta, p.use_c, p.C, (i64)c.ldc, p.out, (i64)c.ldo);
        if (le != cudaSuccess || cudaGetLastError() != cudaSuccess)
            return fail(c, AG_ERR_CUDA, "split-K reduce launch failed");
    }
    return AG_OK;
}

}  // namespace ag
