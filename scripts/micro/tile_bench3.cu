// DMMA 128x128x128 tile product variants (distinct L2-resident panels per tile, no C):
//   v0: inverse.cu's tile_product (8 warps, 64x32 per warp, KC = 16)
//   v1: 16 warps (512 threads), 32x32 per warp (4x4 m8n8 blocks), KC = 16
//   v2: 8 warps, 64x32 per warp, KC = 32 (fewer barriers per tile)
#include <cstdio>
#include "../../paper_1811_12019_b200/csrc/inverse.cu"
namespace kfac {
kfac_status set_error(kfac_status st, const std::string &) { return st; }
std::atomic<int64_t> g_launches{0};
}
using namespace kfac;

template <int NW, int KCH>
__device__ __forceinline__ void tile_product_v(const double *__restrict__ A, int64_t lda, const double *__restrict__ Bm,
                                               int64_t ldb, double *smem, double (&acc)[(NW == 16) ? 4 : 8][(NW == 16) ? 8 : 8]) {
    constexpr int NT = NW * 32;
    constexpr int PR = NW == 16 ? 4 : 8;  // m8n8 row blocks per warp
    constexpr int QC = 4;                 // m8n8 column blocks per warp
    double *As = smem, *Bs = smem + 2 * KCH * SLD;
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int arow = (NW == 16 ? 32 * (w >> 2) : 64 * (w >> 2)) + (lane >> 2), bcol = 32 * (w & 3) + (lane >> 2);
    const int kl = lane & 3;
    constexpr int nchunks = 128 / KCH;
    auto load = [&](int c, int buf) {
        const int t0 = c * KCH;
        for (int e = threadIdx.x; e < KCH * B / 2; e += NT) {
            const int t = e >> 6, i = (e & 63) * 2;
            cp_async16(As + buf * KCH * SLD + t * SLD + i, A + (int64_t)(t0 + t) * lda + i, true);
            cp_async16(Bs + buf * KCH * SLD + t * SLD + i, Bm + (int64_t)(t0 + t) * ldb + i, true);
        }
        cp_async_commit();
    };
    load(0, 0);
    for (int c = 0; c < nchunks; c++) {
        const int buf = c & 1;
        if (c + 1 < nchunks) {
            load(c + 1, buf ^ 1);
            cp_async_wait_1();
        } else {
            cp_async_wait_0();
        }
        __syncthreads();
        const double *as = As + buf * KCH * SLD, *bs = Bs + buf * KCH * SLD;
#pragma unroll
        for (int kk = 0; kk < KCH / 4; kk++) {
            const int t = kk * 4 + kl;
            double a[PR], b[QC];
#pragma unroll
            for (int p = 0; p < PR; p++) a[p] = as[t * SLD + arow + 8 * p];
#pragma unroll
            for (int q = 0; q < QC; q++) b[q] = bs[t * SLD + bcol + 8 * q];
#pragma unroll
            for (int p = 0; p < PR; p++)
#pragma unroll
                for (int q = 0; q < QC; q++) dmma(acc[p][2 * q], acc[p][2 * q + 1], a[p], b[q]);
        }
        __syncthreads();
    }
}

template <int V>
__global__ void __launch_bounds__(V == 1 ? 512 : 256, 1) bench(const double *R, const double *Wp, double *W, int n, int ntiles) {
    extern __shared__ double dyn[];
    const int nt = n / 128;
    for (int g = blockIdx.x; g < ntiles; g += gridDim.x) {
        __syncthreads();
        const int I = (g / nt) % nt, J = g % nt;
        double s = 0;
        if (V == 0) {
            double acc[8][8];
#pragma unroll
            for (int p = 0; p < 8; p++)
#pragma unroll
                for (int q = 0; q < 8; q++) acc[p][q] = 0.0;
            tile_product(R + I * 128, n, 128, Wp + J * 128, n, 128, 128, acc, dyn);
#pragma unroll
            for (int p = 0; p < 8; p++)
#pragma unroll
                for (int q = 0; q < 8; q++) s += acc[p][q];
        } else if (V == 1) {
            double acc[4][8];
#pragma unroll
            for (int p = 0; p < 4; p++)
#pragma unroll
                for (int q = 0; q < 8; q++) acc[p][q] = 0.0;
            tile_product_v<16, 16>(R + I * 128, n, Wp + J * 128, n, dyn, acc);
#pragma unroll
            for (int p = 0; p < 4; p++)
#pragma unroll
                for (int q = 0; q < 8; q++) s += acc[p][q];
        } else {
            double acc[8][8];
#pragma unroll
            for (int p = 0; p < 8; p++)
#pragma unroll
                for (int q = 0; q < 8; q++) acc[p][q] = 0.0;
            tile_product_v<8, 32>(R + I * 128, n, Wp + J * 128, n, dyn, acc);
#pragma unroll
            for (int p = 0; p < 8; p++)
#pragma unroll
                for (int q = 0; q < 8; q++) s += acc[p][q];
        }
        if (s == 1.2345) W[0] = s;
    }
}

int main() {
    const int n = 4608, ntiles = 148 * 6;
    double *R, *Wp, *W;
    cudaMalloc(&R, (size_t)128 * n * 8); cudaMalloc(&Wp, (size_t)128 * n * 8); cudaMalloc(&W, 8);
    cudaMemset(R, 0, (size_t)128 * n * 8); cudaMemset(Wp, 0, (size_t)128 * n * 8);
    const int smem16 = 2 * 2 * 16 * SLD * 8 + 64, smem32 = 2 * 2 * 32 * SLD * 8 + 64;
    cudaFuncSetAttribute(bench<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem16);
    cudaFuncSetAttribute(bench<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem16);
    cudaFuncSetAttribute(bench<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem32);
    for (int v = 0; v < 3; v++)
        for (int rep = 0; rep < 2; rep++) {
            cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
            cudaEventRecord(e0);
            if (v == 0) bench<0><<<148, 256, smem16>>>(R, Wp, W, n, ntiles);
            if (v == 1) bench<1><<<148, 512, smem16>>>(R, Wp, W, n, ntiles);
            if (v == 2) bench<2><<<148, 256, smem32>>>(R, Wp, W, n, ntiles);
            cudaEventRecord(e1); cudaEventSynchronize(e1);
            float ms; cudaEventElapsedTime(&ms, e0, e1);
            printf("v%d: %.1f us per tile-wave, %.2f TFLOP/s (%s)\n", v, ms * 1e3 / 6,
                   2.0 * 128 * 128 * 128 * ntiles / (ms / 1e3) / 1e12, cudaGetErrorString(cudaGetLastError()));
        }
    return 0;
}
