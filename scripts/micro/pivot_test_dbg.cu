// Standalone check of inverse.cu's pivot_block on a 64x64 / 128x128 SPD block.
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <cmath>
#define PIVOT_DBG 1
#include "../../paper_1811_12019_b200/csrc/inverse.cu"
namespace kfac {
kfac_status set_error(kfac_status st, const std::string &) { return st; }
std::atomic<int64_t> g_launches{0};
}
using namespace kfac;

__global__ void __launch_bounds__(256, 1) tkernel(const double *W, int ld, int bk, double *P, int *st) {
    extern __shared__ double dyn[];
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
    double *dW, *dP; int *dst;
    cudaMalloc(&dW, n * n * 8); cudaMalloc(&dP, 128 * 128 * 8); cudaMalloc(&dst, 4);
    cudaMemcpy(dW, M.data(), n * n * 8, cudaMemcpyHostToDevice);
    int dbg = argc > 2 ? atoi(argv[2]) : 0;
    cudaMemcpyToSymbol(g_pivot_dbg, &dbg, 4);
    cudaFuncSetAttribute(tkernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kPivSmem);
    tkernel<<<1, 256, kPivSmem>>>(dW, n, n, dP, dst);
    cudaError_t e = cudaDeviceSynchronize();
    printf("dbg=%d n=%d kPivSmem=%d launch: %s\n", dbg, n, kPivSmem, cudaGetErrorString(e));
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
    long long clk[64]; cudaMemcpyFromSymbol(clk, g_pclk, sizeof(clk));
    for (int k = 1; k <= 20; k++) if (clk[k]) printf("phase %2d: +%lld cycles\n", k, clk[k] - clk[0]);
    return 0;
}
