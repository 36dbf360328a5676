// In-situ-like tile products: distinct panels per tile (L2-resident) and C tile RMW from HBM.
#include <cstdio>
#include "../../paper_1811_12019_b200/csrc/inverse.cu"
namespace kfac {
kfac_status set_error(kfac_status st, const std::string &) { return st; }
std::atomic<int64_t> g_launches{0};
}
using namespace kfac;

template <int MODE>  // 0: same panels, no C; 1: distinct panels, no C; 2: distinct panels + C RMW
__global__ void __launch_bounds__(256, 1) bench(const double *R, const double *Wp, double *W, int n, int ntiles) {
    extern __shared__ double dyn[];
    const int nt = n / 128;
    for (int g = blockIdx.x; g < ntiles; g += gridDim.x) {
        __syncthreads();
        const int I = (g / nt) % nt, J = g % nt;
        const int i0 = MODE ? I * 128 : 0, j0 = MODE ? J * 128 : 0;
        double acc[8][8];
#pragma unroll
        for (int p = 0; p < 8; p++)
#pragma unroll
            for (int q = 0; q < 8; q++) acc[p][q] = 0.0;
        double *Cs = dyn + kTileSmem / 8;
        auto cslice = [&](int c, int nch) {
            if (MODE < 2) return;
            const int r0 = c * 128 / nch, r1 = (c + 1) * 128 / nch;
            for (int e = threadIdx.x; e < (r1 - r0) * 64; e += 256) {
                const int i = r0 + e / 64, j = (e % 64) * 2;
                cp_async16(Cs + i * SLD + j, W + (int64_t)(I * 128 + i) * n + J * 128 + j, true);
            }
        };
        tile_product(R + i0, n, 128, Wp + j0, n, 128, 128, acc, dyn, cslice);
        if (MODE == 2) {
#pragma unroll
            for (int p = 0; p < 8; p++)
#pragma unroll
                for (int q = 0; q < 8; q++) {
                    const int i = tile_row(p), j = tile_col(q);
                    W[(int64_t)(I * 128 + i) * n + J * 128 + j] = Cs[i * SLD + j] - acc[p][q];
                }
        } else {
            double s = 0;
#pragma unroll
            for (int p = 0; p < 8; p++)
#pragma unroll
                for (int q = 0; q < 8; q++) s += acc[p][q];
            if (s == 1.2345) W[0] = s;
        }
    }
}

int main() {
    const int n = 4608, ntiles = 148 * 6;
    double *R, *Wp, *W;
    cudaMalloc(&R, (size_t)128 * n * 8); cudaMalloc(&Wp, (size_t)128 * n * 8); cudaMalloc(&W, (size_t)n * n * 8);
    cudaMemset(R, 0, (size_t)128 * n * 8); cudaMemset(Wp, 0, (size_t)128 * n * 8); cudaMemset(W, 0, (size_t)n * n * 8);
    int smem = kTileSmem + 128 * SLD * 8;
    cudaFuncSetAttribute(bench<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaFuncSetAttribute(bench<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaFuncSetAttribute(bench<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    for (int mode = 0; mode < 3; mode++)
        for (int rep = 0; rep < 2; rep++) {
            cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
            cudaEventRecord(e0);
            if (mode == 0) bench<0><<<148, 256, smem>>>(R, Wp, W, n, ntiles);
            if (mode == 1) bench<1><<<148, 256, smem>>>(R, Wp, W, n, ntiles);
            if (mode == 2) bench<2><<<148, 256, smem>>>(R, Wp, W, n, ntiles);
            cudaEventRecord(e1); cudaEventSynchronize(e1);
            float ms; cudaEventElapsedTime(&ms, e0, e1);
            printf("mode %d: %.1f us per tile-wave, %.2f TFLOP/s (%s)\n", mode, ms * 1e3 / 6, 2.0 * 128 * 128 * 128 * ntiles / (ms / 1e3) / 1e12,
                   cudaGetErrorString(cudaGetLastError()));
        }
    return 0;
}
