/* adaptgemm dispatcher | tree sha256:7b72f4ccc6f0ec0b905210587222c2ffd18e03fdcd26abcecdc58d465eed4712 | provenance: workload dataset, model h1-L1, config 4976e415e379 | adaptgemm 0.1.0 */

typedef struct {
    int family; /* 0 = direct, 1 = indirect */
    int mwg, nwg, kwg, mwi, nwi, kwi;
} gemm_config_t;

static gemm_config_t select_gemm_config(long m, long n, long k) {
    if (m <= 12.0) {
        return (gemm_config_t){0, 32, 16, 16, 2, 4, 1};
    } else {
        return (gemm_config_t){0, 32, 32, 16, 2, 4, 1};
    }
}
