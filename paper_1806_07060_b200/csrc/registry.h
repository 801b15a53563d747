// registry.h -- one compiled launcher per (family, dtype, config) key.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <string>

#include "../../include/adaptgemm_b200.h"

namespace ag {

// everything one launch of one family path needs (host side)
struct GemmCall {
    int64_t M, N, K;
    double alpha, beta;
    int ta, tb;
    int dtype;
    const void* A; int64_t lda;
    const void* B; int64_t ldb;
    const void* C; int64_t ldc;
    void* out; int64_t ldo;
    void* ws; size_t ws_bytes;
    cudaStream_t stream;
    int bm, bn, bk, tm, tn, uk;  // run-time tile sizes (run-time-tile kernels)
    int splits;                  // split-K slices (splitk family); 1 otherwise
    std::string* err;
};

typedef int (*LaunchFn)(const GemmCall&);

struct KernelEntry {
    int family, dtype, bm, bn, bk, tm, tn, uk;
    LaunchFn fn;
};

// generated translation units each export one table
typedef const KernelEntry* (*EntryTableFn)(int* count);

}  // namespace ag
