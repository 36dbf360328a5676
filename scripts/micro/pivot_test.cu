// Standalone check of inverse.cu's pivot_block on a 64x64 / 128x128 SPD block.
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <cmath>
#include "../../paper_1811_12019_b200/csrc/inverse.cu"
namespace kfac {
kfac_status set_error(kfac_status st, const std::string &) { return st; }
std::atomic<int64_t> g_launches{0};
}
using namespace kfac;

__global__ void __launch_bounds__(256, 1) tkernel(const double *Wsrc, double *W, int ld, int bk, double *P, int *st) {
    extern __shared__ double dyn[];
    // pivot_block writes -P back into W: every call starts from a fresh copy
    for (int e = threadIdx.x; e < ld * bk; e += blockDim.x) W[e] = Wsrc[e];
    __syncthreads();
    int f = pivot_block(W, ld, 0, bk, P, dyn);
    if (threadIdx.x == 0) *st = f;
}

int main(int argc, char **argv) {
    int n = argc > 1 ? atoi(argv[1]) : 64;
    std::vector<double> M(n * n), X(n * n);
    srand(1);
    for (int i = 0; i < n; i++)
        for (int j = 0; j < n; j++) X[i * n + j] = (rand() / (double)RAND_MAX) - 0.5;
    for (int i = 0; i < n; i++)
        for (int j = 0; j < n; j++) {
            double s = (i == j) ? n : 0;
            for (int k = 0; k < n; k++) s += X[i * n + k] * X[j * n + k];
            M[i * n + j] = s;
        }
    double *dW, *dWs, *dP; int *dst;
    cudaMalloc(&dW, n * n * 8); cudaMalloc(&dWs, n * n * 8); cudaMalloc(&dP, 128 * 128 * 8); cudaMalloc(&dst, 4);
    cudaMemcpy(dWs, M.data(), n * n * 8, cudaMemcpyHostToDevice);
    cudaFuncSetAttribute(tkernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kPivSmem);
    tkernel<<<1, 256, kPivSmem>>>(dWs, dW, n, n, dP, dst);
    cudaError_t e = cudaDeviceSynchronize();
    printf("n=%d kPivSmem=%d launch: %s\n", n, kPivSmem, cudaGetErrorString(e));
    if (e) return 1;
    std::vector<double> P(128 * 128); int st;
    cudaMemcpy(P.data(), dP, 128 * 128 * 8, cudaMemcpyDeviceToHost);
    cudaMemcpy(&st, dst, 4, cudaMemcpyDeviceToHost);
    double err = 0;
    for (int i = 0; i < n; i++)
        for (int j = 0; j < n; j++) {
            double s = 0;
            for (int k = 0; k < n; k++) s += M[i * n + k] * P[k * 128 + j];
            err = fmax(err, fabs(s - (i == j)));
        }
    printf("status %d  max|M P - I| = %.3e\n", st, err);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    cudaEventRecord(e0);
    for (int r = 0; r < 20; r++) tkernel<<<1, 256, kPivSmem>>>(dWs, dW, n, n, dP, dst);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    printf("pivot_block n=%d: %.1f us per call (incl. the W copy)\n", n, ms * 1e3 / 20);
#ifdef PIVOT_DBG
    long long c[64];
    cudaMemcpyFromSymbol(c, g_pclk, sizeof(c));
    for (int sb = 0; sb < 4; sb++)
        printf("sb %d: sweep %lld  O-copy %lld  W=QO %lld  update %lld\n", sb, c[1 + 4 * sb] - (sb ? c[4 * sb] : c[0]),
               c[2 + 4 * sb] - c[1 + 4 * sb], c[3 + 4 * sb] - c[2 + 4 * sb], c[4 + 4 * sb] - c[3 + 4 * sb]);
    printf("total %lld cycles\n", c[20] - c[0]);
#endif
    return 0;
}
