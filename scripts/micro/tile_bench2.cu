// In-situ-like tile products: distinct panels per tile (L2-resident) and C tile RMW from HBM.
#include <cstdio>
#include "../../paper_1811_12019_b200/csrc/inverse.cu"
namespace kfac {
kfac_status set_error(kfac_status st, const std::string &) { return st; }
std::atomic<int64_t> g_launches{0};
}
using namespace kfac;

template <int MODE>  // 0: same panels, no C; 1: distinct panels, no C; 2: distinct panels + C RMW; 3: 2 + paired stores
__global__ void __launch_bounds__(256, 1) bench(const double *R, const double *Wp, double *W, int n, int ntiles) {
    extern __shared__ double dyn[];
    const int nt = n / 128;
    for (int g = blockIdx.x; g < ntiles; g += gridDim.x) {
        if (MODE == 6 && threadIdx.x < 128) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
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
            if (MODE < 2 || MODE == 5) return;
            const int r0 = c * 128 / nch, r1 = (c + 1) * 128 / nch;
            for (int e = threadIdx.x; e < (r1 - r0) * 64; e += 256) {
                const int i = r0 + e / 64, j = (e % 64) * 2;
                cp_async16(Cs + i * SLD + j, W + (int64_t)(I * 128 + i) * n + J * 128 + j, true);
            }
        };
        tile_product(R + i0, n, 128, Wp + j0, n, 128, 128, acc, dyn, cslice);
        if (MODE == 6) {  // C - acc in place, async bulk row stores
#pragma unroll
            for (int p = 0; p < 8; p++)
#pragma unroll
                for (int q = 0; q < 8; q += 2) {
                    double2 *c = reinterpret_cast<double2 *>(Cs + tile_row(p) * SLD + tile_col(q));
                    const double2 v = *c;
                    *c = make_double2(v.x - acc[p][q], v.y - acc[p][q + 1]);
                }
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            __syncthreads();
            if (threadIdx.x < 128) {
                asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(W + (int64_t)(I * 128 + threadIdx.x) * n + J * 128),
                             "r"((uint32_t)__cvta_generic_to_shared(Cs + threadIdx.x * SLD)), "r"(1024) : "memory");
                asm volatile("cp.async.bulk.commit_group;" ::: "memory");
            }
        } else if (MODE == 4) {  // C loaded, result not stored
            double sacc = 0;
#pragma unroll
            for (int p = 0; p < 8; p++)
#pragma unroll
                for (int q = 0; q < 8; q++) sacc += Cs[tile_row(p) * SLD + tile_col(q)] - acc[p][q];
            if (sacc == 1.2345) W[0] = sacc;
        } else if (MODE == 5) {  // stored (paired), C not loaded
#pragma unroll
            for (int p = 0; p < 8; p++)
#pragma unroll
                for (int q = 0; q < 8; q += 2) {
                    const int i = tile_row(p), j = tile_col(q);
                    *reinterpret_cast<double2 *>(W + (int64_t)(I * 128 + i) * n + J * 128 + j) = make_double2(-acc[p][q], -acc[p][q + 1]);
                }
        } else if (MODE == 3) {
#pragma unroll
            for (int p = 0; p < 8; p++)
#pragma unroll
                for (int q = 0; q < 8; q += 2) {
                    const int i = tile_row(p), j = tile_col(q);
                    const double2 c = *reinterpret_cast<const double2 *>(Cs + i * SLD + j);
                    *reinterpret_cast<double2 *>(W + (int64_t)(I * 128 + i) * n + J * 128 + j) =
                        make_double2(c.x - acc[p][q], c.y - acc[p][q + 1]);
                }
        } else if (MODE == 2) {
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
    cudaFuncSetAttribute(bench<3>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaFuncSetAttribute(bench<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaFuncSetAttribute(bench<5>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaFuncSetAttribute(bench<6>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    for (int mode = 2; mode < 7; mode++)
        for (int rep = 0; rep < 2; rep++) {
            cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
            cudaEventRecord(e0);
            if (mode == 0) bench<0><<<148, 256, smem>>>(R, Wp, W, n, ntiles);
            if (mode == 1) bench<1><<<148, 256, smem>>>(R, Wp, W, n, ntiles);
            if (mode == 2) bench<2><<<148, 256, smem>>>(R, Wp, W, n, ntiles);
            if (mode == 3) bench<3><<<148, 256, smem>>>(R, Wp, W, n, ntiles);
            if (mode == 4) bench<4><<<148, 256, smem>>>(R, Wp, W, n, ntiles);
            if (mode == 5) bench<5><<<148, 256, smem>>>(R, Wp, W, n, ntiles);
            if (mode == 6) bench<6><<<148, 256, smem>>>(R, Wp, W, n, ntiles);
            cudaEventRecord(e1); cudaEventSynchronize(e1);
            float ms; cudaEventElapsedTime(&ms, e0, e1);
            printf("mode %d: %.1f us per tile-wave, %.2f TFLOP/s (%s)\n", mode, ms * 1e3 / 6, 2.0 * 128 * 128 * 128 * ntiles / (ms / 1e3) / 1e12,
                   cudaGetErrorString(cudaGetLastError()));
        }
    return 0;
}
