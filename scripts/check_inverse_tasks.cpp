// Host model of the persistent dataflow inverse's task list (csrc/inverse_tasks.hpp).
//
// Builds the list exactly as inverse_tasks_kernel lays it out (pairs of steps, segment-major over
// the matrices, matrices sorted by column-block count nt descending) and checks, for every
// combination of matrix sizes given:
//   * coverage: every panel (step k, column J) once; every tile (I, J) gets exactly one task per
//     step (a merged task counts for both of its steps); the tile value each task waits for is
//     produced by a task whose LAST step is exactly the one awaited (a merged task's intermediate
//     value is never observable);
//   * order: every wait of every task (the waits inverse_kernel performs) points to a task EARLIER
//     in the list.  CTAs take tasks in list order, so the earliest unfinished task always has its
//     producers finished: no deadlock;
//   * pair_counts agrees with what pair_emit writes.
// Build: g++ -O2 -std=c++17 -I paper_1811_12019_b200/csrc -I /usr/local/cuda/include
//        scripts/check_inverse_tasks.cpp -o /tmp/check_inverse_tasks
// Usage: check_inverse_tasks            (exhaustive: all sorted multisets of up to 3 sizes <= 12,
//                                        single sizes <= 40, and the stress mix)
//        check_inverse_tasks nt0 nt1 ... (one mix)
#include <algorithm>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <map>
#include <tuple>
#include <vector>

#include "inverse_tasks.hpp"

using namespace kfac_inv;

static int g_fail = 0;
static void CHECK(bool c, const char *fmt, ...) {
    if (c) return;
    if (g_fail < 20) {
        va_list ap;
        va_start(ap, fmt);
        std::fprintf(stderr, "FAIL: ");
        std::vfprintf(stderr, fmt, ap);
        std::fprintf(stderr, "\n");
        va_end(ap);
    }
    g_fail++;
}

static bool check_mix(std::vector<int> nt) {
    std::sort(nt.begin(), nt.end(), std::greater<int>());
    const int nm = (int)nt.size();
    const int steps = nt[0];
    const int npairs = (steps + 1) / 2;
    // lay out the list like inverse_launch + inverse_tasks_kernel
    std::vector<int4> list;
    for (int pr = 0; pr < npairs; pr++) {
        const int k = 2 * pr;
        const int base = (int)list.size();
        const int n = pair_tasks(nt.data(), nm, k);
        list.resize(base + n, make_int4(-1, -1, -1, -1));
        int tot[kSegs] = {0};
        std::vector<std::vector<int>> cnt(nm, std::vector<int>(kSegs));
        for (int m = 0; m < nm; m++) {
            pair_counts(nt[m], k, cnt[m].data());
            for (int q = 0; q < kSegs; q++) tot[q] += cnt[m][q];
        }
        for (int m = 0; m < nm; m++) {
            if (nt[m] <= k) continue;
            int cur[kSegs], end[kSegs], b = 0;
            for (int q = 0; q < kSegs; q++) {
                int pre = 0;
                for (int i = 0; i < m; i++) pre += cnt[i][q];
                cur[q] = b + pre;
                end[q] = cur[q] + cnt[m][q];
                b += tot[q];
            }
            pair_emit(nt[m], k, m, cur, list.data() + base);
            for (int q = 0; q < kSegs; q++) CHECK(cur[q] == end[q], "pair_counts != pair_emit (nt %d, k %d, seg %d)", nt[m], k, q);
        }
    }
    for (size_t g = 0; g < list.size(); g++) CHECK(list[g].x >= 0, "hole at %zu", g);
    if (g_fail) return false;

    // producers
    std::map<std::tuple<int, int, int>, int> panel;              // (m, k, J) -> index
    std::map<std::tuple<int, int, int, int>, int> tileval;       // (m, I, J, last step) -> index
    std::map<std::tuple<int, int, int, int>, int> tilestep;      // (m, I, J, step) -> count
    std::map<std::pair<int, int>, int> pivot;                    // (m, k) -> index producing P_k
    std::map<std::pair<int, int>, int> last_panel, last_tile;    // (m, k) -> max index of step k's panels / tiles
    std::map<std::pair<int, int>, int> npanel, ntile;            // (m, k) -> counts
    for (int m = 0; m < nm; m++) pivot[{m, 0}] = -1;            // pivot_kernel, before the launch
    for (int g = 0; g < (int)list.size(); g++) {
        const int4 t = list[g];
        const int k = t.x, m = t.z, I = t.w >> 16, J = t.w & 0xffff;
        if (t.y == 0 || t.y == 3) {  // a chain task (3) is panel (k, J) + update (k, J, J) + P_{k+1}
            CHECK(!panel.count({m, k, J}), "panel (%d,%d,%d) twice", m, k, J);
            panel[{m, k, J}] = g;
            last_panel[{m, k}] = std::max(last_panel.count({m, k}) ? last_panel[{m, k}] : -1, g);
            npanel[{m, k}]++;
            if (t.y == 3) CHECK(I == J && J == k + 1, "chain task at (%d,%d) step %d", I, J, k);
        }
        if (t.y != 0) {
            const int ns = t.y == 2 ? 2 : 1, last = k + ns - 1;
            CHECK(I <= J && J < nt[m], "bad tile (%d,%d) nt %d", I, J, nt[m]);
            if (ns == 2) CHECK(I != k && I != k + 1 && J != k && J != k + 1 && k + 1 < nt[m], "merged task on a pivot row/col");
            CHECK(!tileval.count({m, I, J, last}), "tile value (%d,%d,%d) step %d twice", m, I, J, last);
            tileval[{m, I, J, last}] = g;
            for (int s = k; s <= last; s++) {
                tilestep[{m, I, J, s}]++;
                last_tile[{m, s}] = std::max(last_tile.count({m, s}) ? last_tile[{m, s}] : -1, g);
                ntile[{m, s}]++;
            }
            if (I == last + 1 && J == last + 1) {
                CHECK(!pivot.count({m, last + 1}), "pivot %d twice", last + 1);
                pivot[{m, last + 1}] = g;
            }
        }
    }
    // coverage
    for (int m = 0; m < nm; m++) {
        const int n = nt[m], tiles = n * (n + 1) / 2;
        for (int k = 0; k < n; k++) {
            CHECK(npanel[{m, k}] == n, "m %d step %d: %d panels (want %d)", m, k, npanel[{m, k}], n);
            CHECK(ntile[{m, k}] == tiles, "m %d step %d: %d tile updates (want %d)", m, k, ntile[{m, k}], tiles);
            CHECK(pivot.count({m, k}), "m %d: P_%d never computed", m, k);
            for (int I = 0; I < n; I++)
                for (int J = I; J < n; J++) CHECK(tilestep[{m, I, J, k}] == 1, "tile (%d,%d,%d) step %d covered %d times", m, I, J, k, tilestep[{m, I, J, k}]);
        }
        for (int k = n; k < steps; k++) CHECK(!npanel.count({m, k}) && !ntile.count({m, k}), "m %d has tasks past its last step", m);
    }
    if (g_fail) return false;
    // waits (inverse_kernel), each must point earlier
    auto before = [&](int prod, int g, const char *what, int4 t) {
        CHECK(prod < g, "task %d {k %d kind %d m %d I %d J %d} waits on %s at %d (not earlier)", g, t.x, t.y, t.z, t.w >> 16, t.w & 0xffff, what, prod);
    };
    auto val = [&](int m, int I, int J, int s) -> int {  // the task whose last step is s
        auto it = tileval.find({m, std::min(I, J), std::max(I, J), s});
        CHECK(it != tileval.end(), "tile (%d,%d,%d): no task ends at step %d", m, I, J, s);
        return it == tileval.end() ? 1 << 30 : it->second;
    };
    for (int g = 0; g < (int)list.size(); g++) {
        const int4 t = list[g];
        const int k = t.x, m = t.z, I = t.w >> 16, J = t.w & 0xffff;
        if (t.y == 0 || t.y == 3) {
            if (k >= 1) {
                before(val(m, k, J, k - 1), g, "tile (K, J) of step k-1", t);
                before(pivot[{m, k}], g, "P_k", t);
                if (k >= 4) before(last_tile[{m, k - 4}], g, "step k-4's tiles (panel buffer k mod 4)", t);
            }
        }
        if (t.y != 0) {
            const int ns = t.y == 2 ? 2 : 1, last = k + ns - 1;
            // a chain task's own panel is done inside the task, before its update
            auto pan = [&](int s, int c) { return (t.y == 3 && s == k && c == J) ? -1 : panel[{m, s, c}]; };
            if (I != k) before(pan(last, I), g, "panel I of step last", t);
            if (J != k && J != I) before(pan(last, J), g, "panel J of step last", t);
            if (ns == 2) {  // step k's panels I, J: transitively via step k+1's (checked directly here)
                before(pan(k, I), g, "panel I of step k", t);
                before(pan(k, J), g, "panel J of step k", t);
            } else if (!(I == k || J == k)) {
                before(pan(k, I), g, "panel I", t);
            }
            if (I == k && J == k && k >= 1) before(pivot[{m, k}], g, "P_k", t);
            if (k >= 1) before(val(m, I, J, k - 1), g, "the tile's step k-1 value", t);
            if (I == last + 1 && J == last + 1 && last >= 1) before(last_panel[{m, last - 1}], g, "step last-1's panels (pivot slot)", t);
        }
    }
    return g_fail == 0;
}

int main(int argc, char **argv) {
    if (argc > 1) {
        std::vector<int> nt;
        for (int i = 1; i < argc; i++) nt.push_back(std::atoi(argv[i]));
        const bool ok = check_mix(nt);
        std::printf("%s\n", ok ? "OK" : "FAILED");
        return ok ? 0 : 1;
    }
    long mixes = 0;
    for (int a = 1; a <= 40; a++, mixes++)
        if (!check_mix({a})) return std::printf("FAILED at {%d}\n", a), 1;
    for (int a = 1; a <= 12; a++)
        for (int b = 1; b <= a; b++)
            for (int c = 0; c <= b; c++, mixes++) {
                std::vector<int> v{a, b};
                if (c) v.push_back(c);
                if (!check_mix(v)) return std::printf("FAILED at {%d,%d,%d}\n", a, b, c), 1;
            }
    // the stress config (tests/test_inverse_tasks.py also runs the RN50 mix from synth.shapes)
    mixes++;
    if (!check_mix({36, 4, 36, 4, 36, 4, 17, 8})) return std::printf("FAILED at stress\n"), 1;
    std::printf("OK (%ld mixes)\n", mixes);
    return 0;
}
