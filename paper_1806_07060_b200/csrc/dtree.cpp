// dtree.cpp -- CART training in exact integer arithmetic and the compiled
// branch-free dispatcher (host side of include/adaptgemm_b200.h).
//
// Training restates model.best_split / model.train
// (/root/reference/pkg/src/adaptgemm/model.py:136-232):
//   * candidates are midpoints between consecutive distinct sorted values of
//     a feature; both children must keep >= min_leaf samples;
//   * scores sum(c_L^2)/n_L + sum(c_R^2)/n_R are compared by
//     cross-multiplication in 128-bit integers (the reference relies on
//     Python's unbounded ints; n^5/16 overflows int64 beyond ~10.8k rows);
//   * a candidate must strictly beat the parent, and a later candidate must
//     strictly beat the best so far: ties keep the lowest feature, then the
//     lowest threshold;
//   * leaves take the majority label, ties to the smallest label;
//   * nodes are numbered in pre-order with the left subtree first.
//
// The selector lowers a trained tree to branch-free code: a per-feature
// threshold-bucket table (three branchless binary searches + one load) when
// the bucket grid is small, else a fixed-trip walk of the flattened node
// array whose child step is a select, not a branch.
#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <limits>
#include <string>
#include <vector>

#include "adaptgemm_b200.h"

typedef __int128 i128;

namespace {

struct Rec {
    int64_t f[3];
    int32_t lab;  // dense label index (order-preserving)
};

struct Split {
    int feature;
    double threshold;
    double weighted;
};

double midpoint(int64_t a, int64_t b) {
    // Python: (a + b) / 2 on ints is the correctly rounded exact quotient;
    // scaling by 1/2 commutes with rounding, so round(a+b) / 2 matches.
    return (double)((i128)a + (i128)b) / 2.0;
}

bool best_split(const std::vector<Rec>& recs, const std::vector<int32_t>& idx, int64_t min_leaf, int n_labels,
                Split* out) {
    const int64_t n = (int64_t)idx.size();
    if (n < 2 * min_leaf || n < 2) return false;
    std::vector<int64_t> parent(n_labels, 0);
    int distinct = 0;
    for (int32_t i : idx)
        if (parent[recs[i].lab]++ == 0) ++distinct;
    if (distinct == 1) return false;
    i128 parent_sq = 0;
    for (int64_t c : parent) parent_sq += (i128)c * c;

    bool found = false;
    i128 best_num = 0, best_den = 1;
    int best_f = -1;
    double best_thr = 0.0;
    std::vector<int32_t> ord(idx);
    std::vector<int64_t> left(n_labels), right(n_labels);
    for (int f = 0; f < 3; ++f) {
        std::sort(ord.begin(), ord.end(), [&](int32_t a, int32_t b) {
            if (recs[a].f[f] != recs[b].f[f]) return recs[a].f[f] < recs[b].f[f];
            return recs[a].lab < recs[b].lab;
        });
        std::fill(left.begin(), left.end(), 0);
        right = parent;
        i128 sq_l = 0, sq_r = parent_sq;
        for (int64_t pos = 0; pos < n - 1; ++pos) {
            const Rec& r = recs[ord[pos]];
            const int lab = r.lab;
            sq_l += 2 * (i128)left[lab] + 1;
            left[lab] += 1;
            sq_r -= 2 * (i128)right[lab] - 1;
            right[lab] -= 1;
            const int64_t value = r.f[f];
            const int64_t next_value = recs[ord[pos + 1]].f[f];
            if (value == next_value) continue;
            const int64_t n_l = pos + 1, n_r = n - n_l;
            if (n_l < min_leaf || n_r < min_leaf) continue;
            const i128 num = sq_l * n_r + sq_r * n_l;
            const i128 den = (i128)n_l * n_r;
            if (num * n <= parent_sq * den) continue;  // not strictly better than the parent
            if (!found || num * best_den > best_num * den) {
                found = true;
                best_num = num;
                best_den = den;
                best_f = f;
                best_thr = midpoint(value, next_value);
            }
        }
    }
    if (!found) return false;
    out->feature = best_f;
    out->threshold = best_thr;
    out->weighted = 1.0 - ((double)best_num / (double)best_den) / (double)n;
    return true;
}

int32_t majority(const std::vector<Rec>& recs, const std::vector<int32_t>& idx, int n_labels) {
    std::vector<int64_t> cnt(n_labels, 0);
    for (int32_t i : idx) cnt[recs[i].lab]++;
    int32_t best = 0;
    for (int32_t l = 1; l < n_labels; ++l)
        if (cnt[l] > cnt[best]) best = l;  // strict: ties keep the smallest label
    return best;
}

// compress arbitrary int64 labels to order-preserving dense indices
std::vector<int64_t> compress(const int64_t* labels, int64_t n, std::vector<Rec>& recs, const int64_t* features) {
    std::vector<int64_t> uniq(labels, labels + n);
    std::sort(uniq.begin(), uniq.end());
    uniq.erase(std::unique(uniq.begin(), uniq.end()), uniq.end());
    recs.resize(n);
    for (int64_t i = 0; i < n; ++i) {
        for (int f = 0; f < 3; ++f) recs[i].f[f] = features[i * 3 + f];
        recs[i].lab = (int32_t)(std::lower_bound(uniq.begin(), uniq.end(), labels[i]) - uniq.begin());
    }
    return uniq;
}

}  // namespace

struct ag_selector {
    int kind;  // 0 bucket table, 1 predicated walk
    // flattened nodes (walk + leaf payloads)
    std::vector<int32_t> feat, left, right;
    std::vector<double> thr;
    std::vector<int64_t> cls;
    std::vector<ag_config> cfg;
    int64_t root = 0;
    int height = 0;
    // bucket table
    std::vector<double> cut[3];  // sorted unique thresholds, +inf padded to 2^s
    int half[3] = {0, 0, 0};     // first search step (= size / 2)
    int64_t dim[3] = {1, 1, 1};  // buckets per feature (= #thresholds + 1)
    std::vector<int32_t> table;  // leaf node per (b0, b1, b2)
};

namespace {

inline int bucket(const std::vector<double>& cut, int half, int64_t x) {
    // count of thresholds t < x, i.e. x's bucket; branchless lower_bound
    const double xd = (double)x;
    int base = 0;
    for (int h = half; h >= 1; h >>= 1) base += (cut[base + h - 1] < xd) ? h : 0;
    return base;
}

inline int64_t walk(const ag_selector* s, int64_t m, int64_t n, int64_t k) {
    const int64_t x[3] = {m, n, k};
    int64_t i = s->root;
    for (int d = 0; d < s->height; ++d) {
        const double v = (double)x[s->feat[i]];
        i = (v <= s->thr[i]) ? s->left[i] : s->right[i];  // leaves loop onto themselves
    }
    return i;
}

inline int64_t leaf_of(const ag_selector* s, int64_t m, int64_t n, int64_t k) {
    if (s->kind == 0) {
        const int b0 = bucket(s->cut[0], s->half[0], m);
        const int b1 = bucket(s->cut[1], s->half[1], n);
        const int b2 = bucket(s->cut[2], s->half[2], k);
        return s->table[((int64_t)b0 * s->dim[1] + b1) * s->dim[2] + b2];
    }
    return walk(s, m, n, k);
}

const int64_t kTableCap = 1 << 18;  // 1 MB of int32 leaf ids

}  // namespace

namespace ag {
int set_last_error(int code, const std::string& msg);
std::string config_string(const ag_config& c);
}  // namespace ag

extern "C" {

int ag_best_split(const int64_t* features, const int64_t* labels, int64_t n_records, int64_t min_leaf,
                  int32_t* feature, double* threshold, double* weighted) {
    if (n_records <= 0) return 0;
    std::vector<Rec> recs;
    std::vector<int64_t> uniq = compress(labels, n_records, recs, features);
    std::vector<int32_t> idx(n_records);
    for (int64_t i = 0; i < n_records; ++i) idx[i] = (int32_t)i;
    Split s;
    if (!best_split(recs, idx, min_leaf, (int)uniq.size(), &s)) return 0;
    *feature = s.feature;
    *threshold = s.threshold;
    *weighted = s.weighted;
    return 1;
}

int ag_tree_train(const int64_t* features, const int64_t* labels, int64_t n_records, int64_t max_height,
                  int64_t min_leaf, int32_t* node_feature, double* node_threshold, int32_t* node_left,
                  int32_t* node_right, int64_t* node_class, int64_t* node_count, int64_t* n_nodes) {
    if (n_records <= 0 || n_records > (int64_t)1 << 30) return AG_ERR_SHAPE;
    std::vector<Rec> recs;
    std::vector<int64_t> uniq = compress(labels, n_records, recs, features);
    const int n_labels = (int)uniq.size();
    struct Item {
        std::vector<int32_t> idx;
        int64_t depth;
        int64_t parent;
        int side;  // 0 left, 1 right
    };
    std::vector<Item> stack;
    {
        Item root;
        root.idx.resize(n_records);
        for (int64_t i = 0; i < n_records; ++i) root.idx[i] = (int32_t)i;
        root.depth = 0;
        root.parent = -1;
        root.side = 0;
        stack.push_back(std::move(root));
    }
    int64_t count = 0;
    while (!stack.empty()) {
        Item it = std::move(stack.back());
        stack.pop_back();
        const int64_t id = count++;
        if (it.parent >= 0) (it.side == 0 ? node_left : node_right)[it.parent] = (int32_t)id;
        bool pure = true;
        for (int32_t i : it.idx)
            if (recs[i].lab != recs[it.idx[0]].lab) {
                pure = false;
                break;
            }
        Split s;
        bool chosen = false;
        if (!pure && (max_height < 0 || it.depth < max_height)) chosen = best_split(recs, it.idx, min_leaf, n_labels, &s);
        if (!chosen) {
            node_feature[id] = -1;
            node_threshold[id] = 0.0;
            node_left[id] = node_right[id] = -1;
            node_class[id] = uniq[majority(recs, it.idx, n_labels)];
            node_count[id] = (int64_t)it.idx.size();
            continue;
        }
        node_feature[id] = s.feature;
        node_threshold[id] = s.threshold;
        node_left[id] = node_right[id] = -1;
        node_class[id] = -1;
        node_count[id] = (int64_t)it.idx.size();
        Item l, r;
        for (int32_t i : it.idx) ((double)recs[i].f[s.feature] <= s.threshold ? l.idx : r.idx).push_back(i);
        l.depth = r.depth = it.depth + 1;
        l.parent = r.parent = id;
        l.side = 0;
        r.side = 1;
        stack.push_back(std::move(r));  // right pushed first: left is numbered first
        stack.push_back(std::move(l));
    }
    *n_nodes = count;
    return AG_OK;
}

ag_selector* ag_selector_build_kind(const int32_t* node_feature, const double* node_threshold,
                                    const int32_t* node_left, const int32_t* node_right, const int64_t* node_class,
                                    const ag_config* leaf_configs, int64_t n_nodes, int64_t root, int kind) {
    if (n_nodes <= 0 || root < 0 || root >= n_nodes) return nullptr;
    ag_selector* s = new ag_selector();
    s->root = root;
    s->feat.resize(n_nodes);
    s->left.resize(n_nodes);
    s->right.resize(n_nodes);
    s->thr.resize(n_nodes);
    s->cls.resize(n_nodes);
    s->cfg.resize(n_nodes);
    for (int64_t i = 0; i < n_nodes; ++i) {
        const bool leaf = node_feature[i] < 0;
        if (!leaf && (node_left[i] < 0 || node_left[i] >= n_nodes || node_right[i] < 0 || node_right[i] >= n_nodes ||
                      node_feature[i] > 2)) {
            delete s;
            return nullptr;
        }
        s->feat[i] = leaf ? 0 : node_feature[i];
        s->thr[i] = leaf ? 0.0 : node_threshold[i];
        s->left[i] = leaf ? (int32_t)i : node_left[i];
        s->right[i] = leaf ? (int32_t)i : node_right[i];
        s->cls[i] = leaf ? node_class[i] : -1;
        if (leaf && leaf_configs) s->cfg[i] = leaf_configs[i];
        else std::memset(&s->cfg[i], 0, sizeof(ag_config));
    }
    // height (longest root-to-leaf path); iterative DFS
    {
        std::vector<std::pair<int64_t, int>> st{{root, 0}};
        int64_t visited = 0;
        while (!st.empty()) {
            auto [i, d] = st.back();
            st.pop_back();
            if (++visited > n_nodes) {  // cycle guard
                delete s;
                return nullptr;
            }
            if (node_feature[i] < 0) {
                s->height = std::max(s->height, d);
            } else {
                st.push_back({s->left[i], d + 1});
                st.push_back({s->right[i], d + 1});
            }
        }
    }
    // bucket grid
    int64_t cells = 1;
    for (int f = 0; f < 3; ++f) {
        std::vector<double> c;
        for (int64_t i = 0; i < n_nodes; ++i)
            if (node_feature[i] == f) c.push_back(node_threshold[i]);
        std::sort(c.begin(), c.end());
        c.erase(std::unique(c.begin(), c.end()), c.end());
        s->dim[f] = (int64_t)c.size() + 1;
        int64_t p = 1;
        while (p < (int64_t)c.size() + 1) p <<= 1;
        s->half[f] = (int)(p / 2);
        c.resize(p, std::numeric_limits<double>::infinity());
        s->cut[f] = std::move(c);
        cells = (cells > kTableCap) ? cells : cells * s->dim[f];
    }
    const bool table_ok = cells <= kTableCap;
    s->kind = (kind == 1 || !table_ok) ? 1 : 0;
    if (kind == 0 && !table_ok) {
        delete s;
        return nullptr;
    }
    if (s->kind == 0) {
        // evaluate the tree once per bucket cell: x_f <= t_j  <=>  bucket_f <= j
        s->table.resize(cells);
        for (int64_t b0 = 0; b0 < s->dim[0]; ++b0)
            for (int64_t b1 = 0; b1 < s->dim[1]; ++b1)
                for (int64_t b2 = 0; b2 < s->dim[2]; ++b2) {
                    const int64_t b[3] = {b0, b1, b2};
                    int64_t i = root;
                    while (node_feature[i] >= 0) {
                        const int f = node_feature[i];
                        const auto& c = s->cut[f];
                        const int64_t j = std::lower_bound(c.begin(), c.end(), node_threshold[i]) - c.begin();
                        i = (b[f] <= j) ? node_left[i] : node_right[i];
                    }
                    s->table[(b0 * s->dim[1] + b1) * s->dim[2] + b2] = (int32_t)i;
                }
    }
    return s;
}

ag_selector* ag_selector_build(const int32_t* node_feature, const double* node_threshold, const int32_t* node_left,
                               const int32_t* node_right, const int64_t* node_class, const ag_config* leaf_configs,
                               int64_t n_nodes, int64_t root) {
    return ag_selector_build_kind(node_feature, node_threshold, node_left, node_right, node_class, leaf_configs,
                                  n_nodes, root, -1);
}

void ag_selector_free(ag_selector* s) { delete s; }

int ag_selector_kind(const ag_selector* s) { return s ? s->kind : -1; }

int64_t ag_select(const ag_selector* s, int64_t m, int64_t n, int64_t k, ag_config* out) {
    if (!s) return ag::set_last_error(AG_ERR_CONFIG, "null selector"), -1;
    const int64_t i = leaf_of(s, m, n, k);
    if (out) *out = s->cfg[i];
    return s->cls[i];
}

int ag_select_many(const ag_selector* s, const int64_t* mnk, int64_t n_queries, int64_t* class_ids) {
    if (!s) return ag::set_last_error(AG_ERR_CONFIG, "null selector");
    for (int64_t q = 0; q < n_queries; ++q) class_ids[q] = s->cls[leaf_of(s, mnk[3 * q], mnk[3 * q + 1], mnk[3 * q + 2])];
    return AG_OK;
}

double ag_select_bench_ns(const ag_selector* s, int64_t m, int64_t n, int64_t k, int64_t reps) {
    if (!s || reps <= 0) return -1.0;
    volatile int64_t sink = 0;
    volatile int64_t vm = m, vn = n, vk = k;  // defeat hoisting out of the loop
    const auto t0 = std::chrono::steady_clock::now();
    for (int64_t r = 0; r < reps; ++r) sink = sink + leaf_of(s, vm, vn, vk);
    const auto t1 = std::chrono::steady_clock::now();
    (void)sink;
    return std::chrono::duration<double, std::nano>(t1 - t0).count() / (double)reps;
}

}  // extern "C"

namespace {
// the tree's pick, or the fallback when the pick is illegal under `caps` or
// has no compiled kernel for `dtype` (codegen.py:312-322 legality fallback)
int pick_config(const ag_selector* sel, const ag_config* fallback, const ag_shape* shape, const ag_caps* caps,
                int dtype, ag_config* pick, int* fb) {
    if (!sel) return ag::set_last_error(AG_ERR_CONFIG, "null selector");
    if (!shape) return ag::set_last_error(AG_ERR_SHAPE, "null shape");
    *pick = sel->cfg[leaf_of(sel, shape->m, shape->n, shape->k)];
    *fb = 0;
    auto usable = [&](const ag_config* c) { return (!caps || ag_is_legal(c, caps)) && ag_has_kernel(c, dtype); };
    if (usable(pick)) return AG_OK;
    if (!fallback || !usable(fallback))
        return ag::set_last_error(AG_ERR_CONFIG, "selected config " + ag::config_string(*pick) +
                                                     " is not runnable and the fallback " +
                                                     (fallback ? ag::config_string(*fallback) : std::string("(none)")) +
                                                     " is not either");
    *pick = *fallback;
    *fb = 1;
    return AG_OK;
}
}  // namespace

extern "C" {

int ag_dispatch_gemm(const ag_selector* sel, const ag_config* fallback, const ag_shape* shape, const ag_caps* caps,
                     int dtype, const void* A, int64_t lda, const void* B, int64_t ldb, const void* C, int64_t ldc,
                     void* out, int64_t ldo, void* workspace, size_t workspace_bytes, void* stream,
                     ag_config* selected, int* used_fallback) {
    ag_config pick;
    int fb = 0;
    const int r = pick_config(sel, fallback, shape, caps, dtype, &pick, &fb);
    if (r) return r;
    if (selected) *selected = pick;
    if (used_fallback) *used_fallback = fb;
    return ag_gemm(shape, &pick, caps, dtype, A, lda, B, ldb, C, ldc, out, ldo, workspace, workspace_bytes, stream);
}

int ag_dispatch_gemm_host(const ag_selector* sel, const ag_config* fallback, const ag_shape* shape,
                          const ag_caps* caps, int dtype, const void* A, int64_t lda, const void* B, int64_t ldb,
                          const void* C, int64_t ldc, void* out, int64_t ldo, void* device_scratch,
                          size_t scratch_bytes, int panels, void* stream, ag_config* selected, int* used_fallback) {
    ag_config pick;
    int fb = 0;
    const int r = pick_config(sel, fallback, shape, caps, dtype, &pick, &fb);
    if (r) return r;
    if (selected) *selected = pick;
    if (used_fallback) *used_fallback = fb;
    return ag_gemm_host(shape, &pick, caps, dtype, A, lda, B, ldb, C, ldc, out, ldo, device_scratch, scratch_bytes,
                        panels, stream);
}

int ag_dispatch_gemm_host_ex(const ag_selector* sel, const ag_config* fallback, const ag_shape* shape,
                             const ag_caps* caps, int dtype, const void* A, int64_t lda, const void* B, int64_t ldb,
                             const void* C, int64_t ldc, void* out, int64_t ldo, void* device_scratch,
                             size_t scratch_bytes, int panels, int flags, void* stream, ag_config* selected,
                             int* used_fallback, double* kernel_seconds) {
    ag_config pick;
    int fb = 0;
    const int r = pick_config(sel, fallback, shape, caps, dtype, &pick, &fb);
    if (r) return r;
    if (selected) *selected = pick;
    if (used_fallback) *used_fallback = fb;
    return ag_gemm_host_ex(shape, &pick, caps, dtype, A, lda, B, ldb, C, ldc, out, ldo, device_scratch,
                           scratch_bytes, panels, flags, stream, kernel_seconds);
}

}  // extern "C"
