/*
 * adaptgemm_b200.h -- C-ABI of the B200-native adaptive GEMM library.
 *
 * This is the drop-in boundary for the reference package `adaptgemm`
 * (arxiv 1806.07060 restated as a CPU toolkit, /root/reference/pkg).  The
 * reference has no FFI: its kernels are numba loop nests called in-process.
 * Each entry point below names the reference Python interface it replaces
 * (file:line under /root/reference/pkg/src/adaptgemm/); the Python package
 * `paper_1806_07060_b200` binds these symbols with ctypes and keeps the
 * reference's signatures, return values and exception types.
 *
 * Conventions
 *   - Matrices are row-major with a leading dimension (elements between rows),
 *     exactly the C-contiguous numpy layout the reference consumes.
 *   - All data pointers are CUDA device pointers; `stream` is a cudaStream_t
 *     (NULL = legacy default stream).
 *   - Return codes: AG_OK 0; AG_ERR_CONFIG 1 -> ConfigError;
 *     AG_ERR_SHAPE 2 -> ShapeError; AG_ERR_CUDA 3 -> MeasurementError /
 *     RuntimeError.  ag_last_error() returns a thread-local message for the
 *     last failing call on the calling thread.
 *   - Thread safety: every call is reentrant on disjoint buffers/streams; the
 *     only process-global state is the lazily built kernel registry
 *     (initialised once under a mutex) and compiled tree handles that the
 *     caller owns.
 */
#ifndef ADAPTGEMM_B200_H
#define ADAPTGEMM_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define AG_OK 0
#define AG_ERR_CONFIG 1
#define AG_ERR_SHAPE 2
#define AG_ERR_CUDA 3

/* KernelFamily (kernels.py:32-34).  Values 0/1 match the emitted C
 * dispatcher's `family` field (codegen.py:132).  2 is the B200-profile
 * split-K family: the indirect core over `uk` equal K slices (unroll_k
 * carries the slice count) plus a fixed-order reduction -- deterministic. */
#define AG_FAMILY_DIRECT 0
#define AG_FAMILY_INDIRECT 1
#define AG_FAMILY_SPLITK 2
/* 3, 4: the B200 tensor-core families (tcgen05.mma with TMEM accumulators,
 * TMA-fed): float32 operands packed to tf32 (round to nearest) or bf16
 * (round to nearest even), fp32 accumulation.  No reference analogue; they
 * enter only the "b200tc" search space (BASELINE.json configs[4]).
 * bm = 128 (UMMA M), bn = UMMA N, bk = one 128-byte K block (32 tf32 /
 * 64 bf16 elements), tm = shared-memory pipeline stages, tn = uk = 1. */
#define AG_FAMILY_TF32 3
#define AG_FAMILY_BF16 4
/* B200 profiles: the indirect core's tiles fed by TMA from row-major
 * operands (no pack passes; transposed / unaligned operands run the packed
 * core with the same tile and the same bits) */
#define AG_FAMILY_TMA 5
/* B200 profiles, the "skinny" families (csrc/skinny.cuh): streaming
 * kernels for one small output side, K split over `uk` CTAs of one cluster
 * (DSMEM reduction in a fixed order).
 *   skinny_n (N small): bm = 32 * tm rows per CTA, bn = N tile (16/32/64),
 *     bk = 32, tm = rows per thread, tn = warps splitting the CTA's K range,
 *     uk = K slices (CTAs per cluster).
 *   skinny_m (M small): bm = M tile (8..64), bn = CTA columns
 *     (= 32 * warps * tn), bk = 32, tm = 1, tn = columns per thread, uk =
 *     K slices. */
#define AG_FAMILY_SKINNY_N 6
#define AG_FAMILY_SKINNY_M 7
/* b200tc profile: fp32-accurate GEMM on the tensor pipe ("3xTF32").  Each
 * fp32 operand is split as x = hi + lo (hi = the bits a tf32 MMA reads,
 * lo = x - hi, made in shared memory by converter warps); a.b ~ a_hi.b_hi + a_hi.b_lo +
 * a_lo.b_hi as three tcgen05 kind::tf32 MMAs per K step into one TMEM
 * accumulator.  Meets the fp32 families' RF <= 1e-5 contract.  Tile fields
 * as the tf32 family (bm 128 / 256, bn, bk = 32, tm = stages). */
#define AG_FAMILY_TF32X3 8

/* element types accepted by gemm_execute (kernels.py:282-283) */
#define AG_F32 0
#define AG_F64 1

/* ProblemShape (kernels.py:37-61): C = alpha * op(A) @ op(B) + beta * C. */
typedef struct {
    int64_t m, n, k;
    double alpha, beta;
    int32_t trans_a, trans_b;
} ag_shape;

/* KernelConfig (kernels.py:85-119): family + (Mwg, Nwg, Kwg, Mwi, Nwi, Kwi).
 * Field order and meaning equal the emitted dispatcher struct
 * `gemm_config_t` (codegen.py:136-141). */
typedef struct {
    int32_t family;
    int32_t bm, bn, bk, tm, tn, uk;
} ag_config;

/* DeviceCaps (kernels.py:64-82) plus the B200 launch limit on threads per
 * CTA (max_threads; 1024 keeps the reference's legal space unchanged). */
typedef struct {
    int64_t tile_memory_cap;
    int64_t register_tile_cap_direct;
    int64_t register_tile_cap_indirect;
    int64_t element_size;
    int64_t max_threads;
} ag_caps;

/* ---------------------------------------------------------------- errors */
const char* ag_last_error(void);
const char* ag_version(void);

/* ------------------------------------------------------------ legality */
/* replaces kernels.is_legal (kernels.py:145-158); returns 1 legal, 0 not */
int ag_is_legal(const ag_config* config, const ag_caps* caps);

/* 1 if a compiled sm_100a kernel exists for (config, dtype), else 0 */
int ag_has_kernel(const ag_config* config, int dtype);

/* number of compiled kernel instantiations (all families / dtypes) */
int ag_num_kernels(void);

/* bytes of device workspace one gemm call needs (pack buffers of the
 * indirect family, kernels.py:304-322, and of the tensor-core families);
 * 0 for the direct family */
size_t ag_workspace_bytes(const ag_shape* shape, const ag_config* config, int dtype);

/* ------------------------------------------------------------ execution */
/* replaces kernels.gemm_execute (kernels.py:328-349) minus host timing:
 * runs the whole family path (indirect: pack/transpose-pad helpers + the
 * unpredicated tiled core with a masked store epilogue) on `stream`.
 * Legality is checked first (AG_ERR_CONFIG) then operands (AG_ERR_SHAPE),
 * the reference's error order. */
int ag_gemm(const ag_shape* shape, const ag_config* config, const ag_caps* caps, int dtype,
            const void* A, int64_t lda, const void* B, int64_t ldb,
            const void* C, int64_t ldc, void* out, int64_t ldo,
            void* workspace, size_t workspace_bytes, void* stream);

/* replaces kernels.gemm_execute (kernels.py:328-349) as the reference's
 * callers use it -- HOST operands in, HOST result out (numpy semantics) --
 * in one blocking call: H2D of op(A), op(B) (and C when the family reads
 * it), the family path, D2H of out.  The result is cut into `panels` row
 * panels (M >= N) or column panels (M < N), pipelined over three streams so
 * the PCIe copies of one panel overlap the kernels of the next; panels <= 0
 * picks 8 when the call moves >= 96 MB, 4 from 32 MB, else 1.  Each panel runs `config`
 * on a sub-problem with the same rows / columns and K order, so the result
 * equals ag_gemm's.  Host buffers should be pinned (pageable memory works
 * but its copies do not overlap).  `device_scratch` holds the staged
 * operands and the family workspace: ag_host_scratch_bytes(). */
size_t ag_host_scratch_bytes(const ag_shape* shape, const ag_config* config, int dtype, int panels);
int ag_gemm_host(const ag_shape* shape, const ag_config* config, const ag_caps* caps, int dtype,
                 const void* A, int64_t lda, const void* B, int64_t ldb,
                 const void* C, int64_t ldc, void* out, int64_t ldo,
                 void* device_scratch, size_t scratch_bytes, int panels, void* stream);

/* ag_gemm_host with options.  flags & AG_HOST_REGISTER: page-lock the
 * caller's host buffers (>= 1 MB) for the duration of the call, so pageable
 * numpy memory gets pinned-rate copies that overlap the kernels.
 * device_scratch == NULL: use the library's own grow-only scratch
 * (ag_device_scratch).  *kernel_seconds (if not NULL) receives the device
 * time of the family path (CUDA events around each panel's kernels, summed),
 * the reference's `seconds` without the copies. */
#define AG_HOST_REGISTER 1
/* flags & AG_HOST_STAGE: pageable host buffers cross through two
 * library-owned pinned rings (8 x 4 MB each per thread and device): a pool
 * of host copy workers fills / drains ring slots while the copy engines move
 * the neighbouring slots and the kernels run.  Pinned buffers are DMA'd
 * directly.  Takes precedence over AG_HOST_REGISTER for pageable buffers. */
#define AG_HOST_STAGE 2
int ag_gemm_host_ex(const ag_shape* shape, const ag_config* config, const ag_caps* caps, int dtype,
                    const void* A, int64_t lda, const void* B, int64_t ldb,
                    const void* C, int64_t ldc, void* out, int64_t ldo,
                    void* device_scratch, size_t scratch_bytes, int panels, int flags, void* stream,
                    double* kernel_seconds);

/* per-thread, per-device grow-only device buffer owned by the library
 * (cudaMalloc; NULL on failure).  Lets a caller without a device allocator
 * (the reference's numpy-only package) drive the host path. */
void* ag_device_scratch(size_t bytes);

/* Caching pinned host allocator for host-path RESULTS (the fresh numpy
 * output of gemm_execute(..., out=None), kernels.py:328-349): page-locked
 * (cudaHostAllocPortable) blocks in power-of-two size classes from 64 KB
 * to 2 MB and 2 MB multiples above, reused after ag_host_free, at most
 * AG_HOST_CACHE_BYTES (env, default 4 GiB) kept cached and at most
 * AG_HOST_PINNED_MAX_BYTES (default 16 GiB) owned in all.  A result written into such a block arrives by DMA with no
 * staging copy and no first-touch page faults.  NULL when pinning fails
 * (the caller then allocates pageable memory). */
void* ag_host_alloc(size_t bytes);
void ag_host_free(void* p);
size_t ag_host_cache_bytes(void); /* bytes cached (free) right now */

/* ag_gemm timed on the device: `warmup` untimed runs then `repeats` timed
 * samples (CUDA events on `stream`); each sample is the mean of `inner`
 * back-to-back runs replayed from one CUDA graph (inner <= 0: chosen so a
 * sample lasts >= ~50 us).  *median_s receives the median sample in seconds
 * (tuner.py:139-158 semantics with device time instead of perf_counter). */
int ag_gemm_timed(const ag_shape* shape, const ag_config* config, const ag_caps* caps, int dtype,
                  const void* A, int64_t lda, const void* B, int64_t ldb,
                  const void* C, int64_t ldc, void* out, int64_t ldo,
                  void* workspace, size_t workspace_bytes, void* stream,
                  int warmup, int repeats, int inner, double* median_s);

/* one exhaustive/random sweep of `n_configs` configs over one shape
 * (tuner._measure, tuner.py:139-158): elapsed_s[i] = median device seconds
 * of configs[i].  Stops at the first failing config and reports its index
 * through *failed_index (MeasurementError semantics, tuner.py:153-155). */
int ag_tune(const ag_shape* shape, const ag_config* configs, int n_configs,
            const ag_caps* caps, int dtype,
            const void* A, int64_t lda, const void* B, int64_t ldb,
            const void* C, int64_t ldc, void* out, int64_t ldo,
            void* workspace, size_t workspace_bytes, void* stream,
            int warmup, int repeats, double* elapsed_s, int* failed_index);

/* ag_tune with a choice of timing regime.  l2_flush = 0: ag_tune's warm,
 * graph-replayed back-to-back samples; l2_flush = 1: every sample is one
 * family path after a 256 MB write has evicted L2 (the regime bench.py
 * reports), so labels and the metric are measured the same way. */
int ag_tune_ex(const ag_shape* shape, const ag_config* configs, int n_configs,
               const ag_caps* caps, int dtype,
               const void* A, int64_t lda, const void* B, int64_t ldb,
               const void* C, int64_t ldc, void* out, int64_t ldo,
               void* workspace, size_t workspace_bytes, void* stream,
               int warmup, int repeats, int l2_flush, double* elapsed_s, int* failed_index);

/* replaces kernels.gemm_reference / _kernel_reference (kernels.py:184-195,
 * 294-301): textbook (i,j,k) GEMM, float64 accumulation in k order with
 * separately rounded multiply and add, one final rounding to dtype --
 * bit-identical to the reference oracle. */
int ag_gemm_reference(const ag_shape* shape, int dtype,
                      const void* A, int64_t lda, const void* B, int64_t ldb,
                      const void* C, int64_t ldc, void* out, int64_t ldo, void* stream);

/* replaces kernels.pack_padded (kernels.py:304-309): dst (pad_rows x
 * pad_cols, row-major, ld = pad_cols) = zero-padded op(src), op = transpose
 * if `transpose`; src holds a (rows x cols) logical matrix, stored
 * transposed (cols x rows) when `transpose` is set. */
int ag_pack_padded(int dtype, const void* src, int64_t ld_src, int64_t rows, int64_t cols,
                   int transpose, void* dst, int64_t pad_rows, int64_t pad_cols, void* stream);

/* FP32 FFMA throughput microbenchmark (the CUDA-core roofline
 * denominator): returns achieved TFLOP/s over a ~ms-long launch. */
int ag_ffma_peak(void* stream, double* tflops);

/* ------------------------------------------------------- decision tree */
/* CART training (model.train / best_split, model.py:136-232) in exact
 * 128-bit integer arithmetic.  Records: features[i*3 + f] (M,N,K as
 * int64), labels[i] class ids.  Output nodes in pre-order (left subtree
 * first): node_feature[j] = -1 for a leaf; node_threshold[j] the split
 * threshold; node_left/node_right child indices; node_class/node_count for
 * leaves.  Arrays must hold 2*n_records-1 entries.  max_height < 0 means
 * unbounded.  Returns node count through *n_nodes. */
int ag_tree_train(const int64_t* features, const int64_t* labels, int64_t n_records,
                  int64_t max_height, int64_t min_leaf,
                  int32_t* node_feature, double* node_threshold,
                  int32_t* node_left, int32_t* node_right,
                  int64_t* node_class, int64_t* node_count, int64_t* n_nodes);

/* best_split (model.py:136-185) on one sample set; returns 1 and
 * (feature, threshold, weighted gini) if a split exists, else 0. */
int ag_best_split(const int64_t* features, const int64_t* labels, int64_t n_records,
                  int64_t min_leaf, int32_t* feature, double* threshold, double* weighted);

/* Compiled dispatcher (replaces the emitted `select_gemm_config`,
 * codegen.py:136-150, and model.predict, model.py:235-241): the tree is
 * lowered to a branch-free form -- a per-feature threshold-bucket table
 * when it fits, else a fixed-trip predicated walk of the flattened node
 * array.  leaf_configs[j] is the config of node j when it is a leaf. */
typedef struct ag_selector ag_selector;
ag_selector* ag_selector_build(const int32_t* node_feature, const double* node_threshold,
                               const int32_t* node_left, const int32_t* node_right,
                               const int64_t* node_class, const ag_config* leaf_configs,
                               int64_t n_nodes, int64_t root);
/* as ag_selector_build with the lowering forced: kind 0 = bucket table
 * (NULL if the grid exceeds the table cap), 1 = predicated walk, -1 = auto */
ag_selector* ag_selector_build_kind(const int32_t* node_feature, const double* node_threshold,
                                    const int32_t* node_left, const int32_t* node_right,
                                    const int64_t* node_class, const ag_config* leaf_configs,
                                    int64_t n_nodes, int64_t root, int kind);
void ag_selector_free(ag_selector* sel);
/* 0 = bucket table, 1 = predicated walk */
int ag_selector_kind(const ag_selector* sel);
/* the selected leaf: its class id is returned, its config copied out
   (-1 and ag_last_error set for a null selector) */
int64_t ag_select(const ag_selector* sel, int64_t m, int64_t n, int64_t k, ag_config* out);
/* batched select; returns class ids for n_queries (m,n,k) triples */
int ag_select_many(const ag_selector* sel, const int64_t* mnk, int64_t n_queries,
                   int64_t* class_ids);
/* mean ns per select over `reps` calls on `mnk` (host steady_clock) */
double ag_select_bench_ns(const ag_selector* sel, int64_t m, int64_t n, int64_t k, int64_t reps);

/* dispatch_and_run (codegen.py:285-325) in one call: select, fall back to
 * *fallback when the pick is illegal under caps, run ag_gemm.  *selected
 * and *used_fallback report the choice. */
int ag_dispatch_gemm(const ag_selector* sel, const ag_config* fallback,
                     const ag_shape* shape, const ag_caps* caps, int dtype,
                     const void* A, int64_t lda, const void* B, int64_t ldb,
                     const void* C, int64_t ldc, void* out, int64_t ldo,
                     void* workspace, size_t workspace_bytes, void* stream,
                     ag_config* selected, int* used_fallback);

/* ag_dispatch_gemm over host operands: select (+ fallback), then
 * ag_gemm_host with the pick (scratch sized by ag_host_scratch_bytes for
 * the pick; the codegen.dispatch_and_run path of a numpy caller). */
int ag_dispatch_gemm_host(const ag_selector* sel, const ag_config* fallback,
                          const ag_shape* shape, const ag_caps* caps, int dtype,
                          const void* A, int64_t lda, const void* B, int64_t ldb,
                          const void* C, int64_t ldc, void* out, int64_t ldo,
                          void* device_scratch, size_t scratch_bytes, int panels, void* stream,
                          ag_config* selected, int* used_fallback);

/* ag_dispatch_gemm_host with ag_gemm_host_ex's flags and kernel time. */
int ag_dispatch_gemm_host_ex(const ag_selector* sel, const ag_config* fallback,
                             const ag_shape* shape, const ag_caps* caps, int dtype,
                             const void* A, int64_t lda, const void* B, int64_t ldb,
                             const void* C, int64_t ldc, void* out, int64_t ldo,
                             void* device_scratch, size_t scratch_bytes, int panels, int flags, void* stream,
                             ag_config* selected, int* used_fallback, double* kernel_seconds);

#ifdef __cplusplus
}
#endif
#endif /* ADAPTGEMM_B200_H */
