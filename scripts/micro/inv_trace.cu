// Timeline of the persistent inverse on one n x n SPD matrix (build with -DINV_TRACE):
// inv_trace <n> > trace.txt   (one line per task: g k kind I J sm t0 t1 t2, ns)
#include <cstdio>
#include <cstdlib>
#include <vector>
#include "../../paper_1811_12019_b200/csrc/inverse.cu"
namespace kfac {
kfac_status set_error(kfac_status st, const std::string &m) { fprintf(stderr, "%s\n", m.c_str()); return st; }
std::atomic<int64_t> g_launches{0};
}
using namespace kfac;
int main(int argc, char **argv) {
    const int n = argc > 1 ? atoi(argv[1]) : 4608;
    // packed upper SPD: diagonally dominant random
    const int64_t np = (int64_t)n * (n + 1) / 2;
    std::vector<float> hp(np);
    srand(1);
    int64_t e = 0;
    for (int i = 0; i < n; i++)
        for (int j = i; j < n; j++) hp[e++] = (i == j) ? (float)n : (float)((rand() / (double)RAND_MAX - 0.5) * 0.5);
    float *dp, *dinv; double *work, *scratch; int *status; float *pi;
    cudaMalloc(&dp, np * 4); cudaMemcpy(dp, hp.data(), np * 4, cudaMemcpyHostToDevice);
    cudaMalloc(&dinv, (size_t)n * n * 4 * 2);
    cudaMalloc(&work, inverse_ws_doubles(n) * 8 * 2);
    cudaMalloc(&scratch, 1 << 20); cudaMalloc(&status, 8); cudaMalloc(&pi, 8);
    // pair: A = this matrix, G = a 128 x 128 identity-ish (same packed buffer prefix reused as n=128)
    std::vector<InvMat> mats(2);
    mats[0].packed = dp; mats[0].inv = dinv; mats[0].work = work; mats[0].panel = work + (int64_t)n * inverse_ld(n);
    mats[0].status = status; mats[0].n = n; mats[0].pair = 0; mats[0].is_A = 1;
    double *w2 = work + inverse_ws_doubles(n);
    mats[1].packed = dp; mats[1].inv = dinv + (size_t)n * n; mats[1].work = w2; mats[1].panel = w2 + (int64_t)128 * 128;
    mats[1].status = status + 1; mats[1].n = 128; mats[1].pair = 0; mats[1].is_A = 0;
    for (int r = 0; r < 3; r++) inverse_launch(mats, 1, 0.01f, scratch, pi, 0, 0);
    cudaDeviceSynchronize();
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    cudaEventRecord(e0);
    inverse_launch(mats, 1, 0.01f, scratch, pi, 0, 0);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    fprintf(stderr, "n=%d inverse %.3f ms (%s)\n", n, ms, cudaGetErrorString(cudaGetLastError()));
#ifdef INV_TRACE
    std::vector<TraceRec> tr(65536);
    cudaMemcpyFromSymbol(tr.data(), g_trace, sizeof(TraceRec) * 65536);
    for (auto &t : tr) if (t.t2) printf("%d %d %d %d %d %d %lld %lld %lld\n", t.g, t.k, t.kind, t.I, t.J, t.sm, t.t0, t.t1, t.t2);
#endif
    return 0;
}
