// Task list of the persistent dataflow inverse (inverse.cu): generator shared by the device
// (inverse_tasks_kernel) and the host (launch offsets; scripts/check_inverse_tasks.cpp, which
// verifies that every wait of every task points to an earlier task of the list).
#pragma once
#include <cuda_runtime.h>

namespace kfac_inv {

// ---- the task list.  Steps are processed in pairs (k, k+1), k even: the tiles away from block
// rows / columns k and k+1 ("bulk" tiles) get ONE merged task applying both steps' rank-128
// updates (one C read-modify-write for two steps), the tiles in rows / columns k, k+1 get
// individual tasks.  Records {k, kind, matrix, I << 16 | J}: kind 0 panel (k, J), 1 update of tile
// (I, J) at step k, 2 merged update of tile (I, J) for steps k and k+1, 3 the critical chain of
// step k in ONE task: panel (k, J = k+1), then the update of tile (J, J) at step k from that
// panel, then its inverse P_{k+1} (no stamp round trips or re-dispatch along the chain).
// CTAs take tasks in list order, so a task waits in the queue behind everything listed before
// it: the list of pair k (segment-major over the matrices, sorted by nt descending) puts the
// chain P_k -> chain(k) -> P_{k+1} -> chain(k+1) -> ... and the tasks it reads ahead of the bulk:
//   a   [k = 0] chain(0) and the other panels of step 0
//   b   look-ahead row / column k+1 at step k (pair 0 also: tile (2, 2) at step 0)
//   c   chain(k+1)
//   d   row / column k at step k (no work: the panels wrote them)
//   e   the other panels of step k+1
//   f   rows / columns k, k+1 at step k+1
//   g   merged tiles in rows / columns k+2, k+3, and tile (k+4, k+4)
//   h   chain(k+2); then what chain(k+3) reads: panel (k+2, k+4), tiles (k+3, k+4) and (k+4, k+4)
//       at step k+2 (in the next pair's b they would queue behind this pair's bulk tiles)
//   i   half of the other merged tiles                   j   the other panels of step k+2
//   k   the rest
// A matrix whose last step k is single (nt = k+1) puts all its step-k tiles in i.  Every task
// only waits for tasks earlier in the list (checked exhaustively against a host model,
// scripts/check_inverse_tasks.cpp).  (A software-pipelined variant -- a pair's far bulk tiles
// lagging behind the next pair's critical prefix -- measured slower: the prefix then queues
// behind the lagging bulk instead.)
constexpr int kSegs = 11;
enum { SA, SB, SC, SD, SE, SF, SG, SH, SI, SJ, SK };
__host__ __device__ inline void pair_counts(int nt, int k, int *c) {
    for (int q = 0; q < kSegs; q++) c[q] = 0;
    if (nt <= k) return;
    const bool full = nt > k + 1, nxt = nt > k + 3, d22 = nt > k + 2, f4 = nt > k + 4;
    if (k == 0) c[SA] = nt;
    if (!full) {
        c[SI] = nt * (nt + 1) / 2;
        return;
    }
    const int Bp = nt - 2, x = (nt > k + 2 ? 1 : 0) + (nt > k + 3 ? 1 : 0);
    const int la = Bp * (Bp + 1) / 2 - (Bp - x) * (Bp - x + 1) / 2 - (d22 ? 1 : 0) + (f4 ? 1 : 0);
    const int rest = (nt - 2) * (nt - 1) / 2 - la - (d22 ? 1 : 0);
    c[SB] = nt - 1 + ((k == 0 && d22) ? 1 : 0) - ((k >= 2 && d22) ? 1 : 0);
    c[SC] = d22 ? 1 : 0;
    c[SD] = nt - 1;
    c[SE] = nt - (d22 ? 1 : 0);
    c[SF] = 2 * nt - 1;
    c[SG] = la;
    c[SH] = (nxt ? 1 : 0) + (f4 ? 3 : 0);
    c[SI] = (rest + 1) / 2;
    c[SJ] = d22 ? nt - (nxt ? 1 : 0) - (f4 ? 1 : 0) : 0;
    c[SK] = rest - c[SI];
}
// write matrix m's tasks of pair k at the given per-segment cursors (each advanced)
__host__ __device__ inline void pair_emit(int nt, int k, int m, int *cur, int4 *out) {
    if (nt <= k) return;
    auto put = [&](int seg, int kk, int kind, int I, int J) { out[cur[seg]++] = make_int4(kk, kind, m, (I << 16) | J); };
    const bool full = nt > k + 1, nxt = nt > k + 3, d22 = nt > k + 2, f4 = nt > k + 4;
    const int L = k + 1;
    if (k == 0) {
        if (nt > 1) put(SA, 0, 3, 1, 1);  // chain(0): panel (0, 1) + tile (1, 1) + P_1
        for (int J = 0; J < nt; J++)
            if (!(nt > 1 && J == 1)) put(SA, 0, 0, 0, J);
    }
    if (!full) {
        for (int I = 0; I < nt; I++)
            for (int J = I; J < nt; J++) put(SI, k, 1, I, J);
        return;
    }
    for (int I = 0; I < L; I++) put(SB, k, 1, I, L);
    // (k+1, k+2) and (k+2, k+2) at step k feed chain(k+1): from pair 2 on, the previous pair's h
    for (int J = L + 1; J < nt; J++)
        if (!(k >= 2 && J == k + 2)) put(SB, k, 1, L, J);
    if (k == 0 && d22) put(SB, k, 1, k + 2, k + 2);
    if (d22) put(SC, k + 1, 3, k + 2, k + 2);  // chain(k+1)
    for (int I = 0; I < k; I++) put(SD, k, 1, I, k);
    for (int J = k; J < nt; J++)
        if (J != L) put(SD, k, 1, k, J);
    for (int J = 0; J < nt; J++)
        if (J != k + 2) put(SE, k + 1, 0, 0, J);
    int cnt[kSegs];
    pair_counts(nt, k, cnt);
    const int half = cnt[SI];
    int nrest = 0;
    for (int I = 0; I < nt; I++)
        for (int J = I; J < nt; J++) {
            if (I == k || I == L || J == k || J == L) {
                put(SF, k + 1, 1, I, J);
                continue;
            }
            if (I == k + 2 && J == k + 2) continue;  // single tasks (b / the previous pair's h) and chain(k+1)
            const bool la = I == k + 2 || I == k + 3 || J == k + 2 || J == k + 3 || (I == k + 4 && J == k + 4);
            if (la) put(SG, k, 2, I, J);
            else put(nrest++ < half ? SI : SK, k, 2, I, J);
        }
    if (nxt) put(SH, k + 2, 3, k + 3, k + 3);  // chain(k+2): panel (k+2, k+3) + tile (k+3, k+3) + P_{k+3}
    if (f4) {
        put(SH, k + 2, 0, 0, k + 4);
        put(SH, k + 2, 1, k + 3, k + 4);
        put(SH, k + 2, 1, k + 4, k + 4);
    }
    if (d22)
        for (int J = 0; J < nt; J++)
            if (!(nxt && J == k + 3) && !(f4 && J == k + 4)) put(SJ, k + 2, 0, 0, J);
}
// host: tasks of pair k over the sorted nt list
inline int pair_tasks(const int *nt, int nm, int k) {
    int c = 0, cnt[kSegs];
    for (int m = 0; m < nm; m++) {
        pair_counts(nt[m], k, cnt);
        for (int q = 0; q < kSegs; q++) c += cnt[q];
    }
    return c;
}


}  // namespace kfac_inv
