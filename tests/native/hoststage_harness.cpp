// hoststage_harness.cpp -- CPU-side checks of csrc/hoststage.h (no GPU):
// the copy-worker pool, the parallel pitched copy, and the slot chunking.
// Built and driven by tests/test_hoststage.py (g++, ctypes).
#include <cstdint>
#include <cstring>
#include <thread>
#include <vector>

#include "../../paper_1806_07060_b200/csrc/hoststage.h"

using namespace ag::hoststage;

extern "C" {

int hs_pool_threads() { return CopyPool::get().threads(); }

// dst (rows x width at dpitch) = src (rows x width at spitch), via copy_rows
void hs_copy_rows(char* dst, int64_t dpitch, const char* src, int64_t spitch, int64_t width, int64_t rows) {
    copy_rows(dst, dpitch, src, spitch, width, rows);
}

// the slot chunks of a block: writes up to cap (r0, nr, b0, nb) quadruples, returns the count
int hs_chunks(int64_t hpitch, int64_t dpitch, int64_t width, int64_t rows, int64_t* out, int cap) {
    Block b{nullptr, hpitch, nullptr, dpitch, width, rows};
    const std::vector<Chunk> cs = chunks_of(b);
    const int n = (int)cs.size();
    for (int i = 0; i < n && i < cap; ++i) {
        out[4 * i] = cs[i].r0;
        out[4 * i + 1] = cs[i].nr;
        out[4 * i + 2] = cs[i].b0;
        out[4 * i + 3] = cs[i].nb;
    }
    return n;
}

// several host threads running pool jobs at once: every item of every job
// runs exactly once; returns the number of mismatches
int hs_pool_stress(int callers, int jobs, int items) {
    std::vector<std::thread> ts;
    std::vector<int> bad(callers, 0);
    for (int c = 0; c < callers; ++c)
        ts.emplace_back([&, c] {
            for (int j = 0; j < jobs; ++j) {
                std::vector<std::atomic<int>> hit(items);
                for (auto& h : hit) h.store(0);
                CopyPool::get().run(items, [&](int i) { hit[i].fetch_add(1); });
                for (auto& h : hit) bad[c] += h.load() != 1;
            }
        });
    for (auto& t : ts) t.join();
    int total = 0;
    for (int b : bad) total += b;
    return total;
}

}  // extern "C"
