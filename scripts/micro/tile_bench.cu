// fp64 128x128x128 tile-product throughput: inverse.cu's tile_product vs variants.
#include <cstdio>
#include <cstdlib>
#include <vector>
#include "../../paper_1811_12019_b200/csrc/inverse.cu"
namespace kfac {
kfac_status set_error(kfac_status st, const std::string &) { return st; }
std::atomic<int64_t> g_launches{0};
}
using namespace kfac;

// variant: thread owns rows 4*ty+{0..3} and 64+4*ty+{0..3} (LDS.128 fragments), register double-buffered
__device__ __forceinline__ void tile_product_v1(const double *__restrict__ A, int64_t lda, const double *__restrict__ Bm,
                                                int64_t ldb, int kt, double (&acc)[8][8], double *smem) {
    constexpr int LDP = B + 4;  // padded row (doubles)
    double *As = smem, *Bs = smem + 2 * KC * LDP;
    const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
    const int nchunks = (kt + KC - 1) / KC;
    auto load = [&](int c, int buf) {
        const int t0 = c * KC;
        for (int e = threadIdx.x; e < KC * B / 2; e += 256) {
            const int t = e >> 6, i = (e & 63) * 2;
            cp_async16(As + buf * KC * LDP + t * LDP + i, A + (int64_t)(t0 + t) * lda + i, true);
            cp_async16(Bs + buf * KC * LDP + t * LDP + i, Bm + (int64_t)(t0 + t) * ldb + i, true);
        }
        cp_async_commit();
    };
    load(0, 0);
    for (int c = 0; c < nchunks; c++) {
        const int buf = c & 1;
        if (c + 1 < nchunks) { load(c + 1, buf ^ 1); cp_async_wait_1(); } else { cp_async_wait_0(); }
        __syncthreads();
        const double *as = As + buf * KC * LDP, *bs = Bs + buf * KC * LDP;
#pragma unroll 2
        for (int t = 0; t < KC; t++) {
            double a[8], b[8];
            const double2 *ap = reinterpret_cast<const double2 *>(as + t * LDP);
            const double2 *bp = reinterpret_cast<const double2 *>(bs + t * LDP);
            double2 a0 = ap[ty * 2], a1 = ap[ty * 2 + 1], a2 = ap[32 + ty * 2], a3 = ap[32 + ty * 2 + 1];
            double2 b0 = bp[tx * 2], b1 = bp[tx * 2 + 1], b2 = bp[32 + tx * 2], b3 = bp[32 + tx * 2 + 1];
            a[0] = a0.x; a[1] = a0.y; a[2] = a1.x; a[3] = a1.y; a[4] = a2.x; a[5] = a2.y; a[6] = a3.x; a[7] = a3.y;
            b[0] = b0.x; b[1] = b0.y; b[2] = b1.x; b[3] = b1.y; b[4] = b2.x; b[5] = b2.y; b[6] = b3.x; b[7] = b3.y;
#pragma unroll
            for (int p = 0; p < 8; p++)
#pragma unroll
                for (int q = 0; q < 8; q++) acc[p][q] = fma(a[p], b[q], acc[p][q]);
        }
        __syncthreads();
    }
}

template <int V>
__global__ void __launch_bounds__(256, 1) bench(const double *A, const double *Bm, double *C, int ld, int reps) {
    extern __shared__ double dyn[];
    double acc[8][8];
#pragma unroll
    for (int p = 0; p < 8; p++)
#pragma unroll
        for (int q = 0; q < 8; q++) acc[p][q] = 0.0;
    const double *a = A + blockIdx.x * 128, *b = Bm + blockIdx.x * 128;
    for (int r = 0; r < reps; r++) {
        if (V == 0) tile_product(a, ld, 128, b, ld, 128, 128, acc, dyn);
        else tile_product_v1(a, ld, b, ld, 128, acc, dyn);
    }
    double s = 0;
#pragma unroll
    for (int p = 0; p < 8; p++)
#pragma unroll
        for (int q = 0; q < 8; q++) s += acc[p][q];
    C[blockIdx.x * 256 + threadIdx.x] = s;
}

int main() {
    const int nblk = 148, ld = 128 * nblk, reps = 50;
    double *A, *Bm, *C;
    cudaMalloc(&A, (size_t)128 * ld * 8); cudaMalloc(&Bm, (size_t)128 * ld * 8); cudaMalloc(&C, nblk * 256 * 8);
    cudaMemset(A, 0, (size_t)128 * ld * 8); cudaMemset(Bm, 0, (size_t)128 * ld * 8);
    int smem0 = kTileSmem, smem1 = 2 * 2 * KC * (B + 4) * 8;
    cudaFuncSetAttribute(bench<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem0);
    cudaFuncSetAttribute(bench<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem1);
    for (int v = 0; v < 2; v++) {
        for (int rep = 0; rep < 2; rep++) {
            cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
            cudaEventRecord(e0);
            if (v == 0) bench<0><<<nblk, 256, smem0>>>(A, Bm, C, ld, reps);
            else bench<1><<<nblk, 256, smem1>>>(A, Bm, C, ld, reps);
            cudaEventRecord(e1); cudaEventSynchronize(e1);
            float ms; cudaEventElapsedTime(&ms, e0, e1);
            double fl = 2.0 * 128 * 128 * 128 * reps * nblk;
            printf("variant %d: %.2f TFLOP/s (%s)\n", v, fl / (ms / 1e3) / 1e12, cudaGetErrorString(cudaGetLastError()));
        }
    }
    return 0;
}
