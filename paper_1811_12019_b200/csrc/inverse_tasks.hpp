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
// (I, J) at step k, 2 merged update of tile (I, J) for steps k and k+1.  The order of pair k
// (segment-major over the matrices, sorted by nt descending) follows the critical path
// P_k -> panel(k+1, K+2) -> tile (K+2, K+2) at step k+1 -> P_{k+2} -> ...:
//   a  [k = 0] step 0's panels (column 1 first) and the pivot tile (1, 1)
//   b  look-ahead row / column k+1 at step k, and tile (k+2, k+2) at step k
//   c  panel (k+1, k+2), then tile (k+2, k+2) at step k+1 (the fused pivot P_{k+2}: a single-step
//      task, so the critical chain P_k -> ... -> P_{k+2} carries one product per pivot, not two)
//   d  row / column k at step k (copies of P R)         e  the other panels of step k+1
//   f  rows / columns k, k+1 at step k+1                g  merged tiles in rows / columns k+2, k+3
//   h  panel (k+2, k+3) and update (k+2, k+3, k+3) (the next pair's pivot tile)
//   i  half of the other merged tiles                   j  the next pair's step-(k+2) panels
//   k  the rest
// A matrix whose last step k is single (nt = k+1) puts all its step-k tiles in i.  Every task
// only waits for tasks earlier in the list (checked exhaustively against a host model).
constexpr int kSegs = 11;
__host__ __device__ inline void pair_counts(int nt, int k, int *c) {
    for (int q = 0; q < kSegs; q++) c[q] = 0;
    if (nt <= k) return;
    const bool full = nt > k + 1, nxt = nt > k + 3, d22 = nt > k + 2;
    if (k == 0) c[0] = nt + (nt > 1 ? 1 : 0);
    if (!full) {
        c[8] = nt * (nt + 1) / 2;
        return;
    }
    const int Bp = nt - 2, x = (nt > k + 2 ? 1 : 0) + (nt > k + 3 ? 1 : 0);
    const int la = Bp * (Bp + 1) / 2 - (Bp - x) * (Bp - x + 1) / 2 - (d22 ? 1 : 0);
    const int rest = (nt - 2) * (nt - 1) / 2 - la - (d22 ? 1 : 0);
    c[1] = nt - 1 + (d22 ? 1 : 0);
    c[2] = d22 ? 2 : 0;
    c[3] = nt - 1;
    c[4] = nt - (d22 ? 1 : 0);
    c[5] = 2 * nt - 1;
    c[6] = la;
    c[7] = nxt ? 2 : 0;
    c[8] = (rest + 1) / 2;
    c[9] = d22 ? nt - (nxt ? 1 : 0) : 0;
    c[10] = rest - c[8];
}
// write matrix m's tasks of pair k at the given per-segment cursors (each advanced)
__host__ __device__ inline void pair_emit(int nt, int k, int m, int *cur, int4 *out) {
    if (nt <= k) return;
    auto put = [&](int seg, int kk, int kind, int I, int J) { out[cur[seg]++] = make_int4(kk, kind, m, (I << 16) | J); };
    const bool full = nt > k + 1, nxt = nt > k + 3, d22 = nt > k + 2;
    const int L = k + 1;
    if (k == 0) {
        if (nt > 1) put(0, 0, 0, 0, 1);
        for (int J = 0; J < nt; J++)
            if (!(nt > 1 && J == 1)) put(0, 0, 0, 0, J);
        if (nt > 1) put(0, 0, 1, 1, 1);
    }
    if (!full) {
        for (int I = 0; I < nt; I++)
            for (int J = I; J < nt; J++) put(8, k, 1, I, J);
        return;
    }
    for (int I = 0; I < L; I++) put(1, k, 1, I, L);
    for (int J = L + 1; J < nt; J++) put(1, k, 1, L, J);
    if (d22) put(1, k, 1, k + 2, k + 2);
    if (d22) {
        put(2, k + 1, 0, 0, k + 2);
        put(2, k + 1, 1, k + 2, k + 2);
    }
    for (int I = 0; I < k; I++) put(3, k, 1, I, k);
    for (int J = k; J < nt; J++)
        if (J != L) put(3, k, 1, k, J);
    for (int J = 0; J < nt; J++)
        if (J != k + 2) put(4, k + 1, 0, 0, J);
    int c5[kSegs];
    pair_counts(nt, k, c5);
    const int half = c5[8];
    int nrest = 0;
    for (int I = 0; I < nt; I++)
        for (int J = I; J < nt; J++) {
            const bool in_kl = I == k || I == L || J == k || J == L;
            if (in_kl) {
                put(5, k + 1, 1, I, J);
                continue;
            }
            if (I == k + 2 && J == k + 2) continue;  // in c
            const bool la = I == k + 2 || I == k + 3 || J == k + 2 || J == k + 3;
            if (la) put(6, k, 2, I, J);
            else put(nrest++ < half ? 8 : 10, k, 2, I, J);
        }
    if (nxt) {
        put(7, k + 2, 0, 0, k + 3);
        put(7, k + 2, 1, k + 3, k + 3);
    }
    if (d22)
        for (int J = 0; J < nt; J++)
            if (!(nxt && J == k + 3)) put(9, k + 2, 0, 0, J);
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
