// Microbenchmark: TMA (cp.async.bulk.tensor.2d) streaming throughput into a smem ring,
// one elected thread issuing, consumer thread releasing immediately.  One CTA per SM.
#include <cstdio>
#include <cstdint>
#include <cuda.h>
#include <cuda_runtime.h>
#include "../../paper_1811_12019_b200/csrc/sm100.cuh"
using namespace kfac;

__global__ void __launch_bounds__(64, 1) tma_bench(const __grid_constant__ CUtensorMap map, int rows_total, int box_rows,
                                                   int boxes_per_stage, int stages, int iters, int C) {
    extern __shared__ uint8_t raw[];
    uint8_t *smem = (uint8_t *)(((uintptr_t)raw + 1023) & ~uintptr_t(1023));
    __shared__ uint64_t full[16], empty[16];
    const int warp = threadIdx.x / 32, lane = threadIdx.x & 31;
    if (threadIdx.x == 0) {
        for (int s = 0; s < stages; s++) { mbar_init(&full[s], 1); mbar_init(&empty[s], 1); }
        fence_barrier_init();
    }
    __syncthreads();
    const uint32_t box_bytes = box_rows * 128;
    const uint32_t stage_bytes = box_bytes * boxes_per_stage;
    const int nrowblk = rows_total / box_rows;
    if (warp == 0 && lane == 0) {
        uint32_t st = 0, ph = 0;
        for (int it = 0; it < iters; it++) {
            mbar_wait(&empty[st], ph ^ 1);
            mbar_arrive_expect_tx(&full[st], stage_bytes);
            for (int b = 0; b < boxes_per_stage; b++) {
                int rb = (blockIdx.x * 7 + it * 3 + b * 13) % nrowblk;
                int cb = (b % (C / 64)) * 64;
                tma_load_2d(smem + st * stage_bytes + b * box_bytes, &map, &full[st], cb, rb * box_rows);
            }
            if (++st == stages) { st = 0; ph ^= 1; }
        }
    } else if (warp == 1 && lane == 0) {
        uint32_t st = 0, ph = 0;
        for (int it = 0; it < iters; it++) {
            mbar_wait(&full[st], ph);
            mbar_arrive(&empty[st]);
            if (++st == stages) { st = 0; ph ^= 1; }
        }
    }
    __syncthreads();
}

typedef CUresult (*PFN)(CUtensorMap *, CUtensorMapDataType, cuuint32_t, void *, const cuuint64_t *, const cuuint64_t *,
                        const cuuint32_t *, const cuuint32_t *, CUtensorMapInterleave, CUtensorMapSwizzle,
                        CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

int main() {
    void *fn; cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
    PFN enc = (PFN)fn;
    const int rows = 1 << 16;
    for (int C : {64, 512}) {
        void *buf; cudaMalloc(&buf, (size_t)rows * C * 2);
        cudaMemset(buf, 0, (size_t)rows * C * 2);
        for (int box_rows : {64, 128, 256}) {
            for (int promo : {0, 2}) {
                CUtensorMap m;
                cuuint64_t dims[2] = {(cuuint64_t)C, (cuuint64_t)rows};
                cuuint64_t strides[1] = {(cuuint64_t)C * 2};
                cuuint32_t box[2] = {64, (cuuint32_t)box_rows};
                cuuint32_t es[2] = {1, 1};
                enc(&m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, buf, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                    CU_TENSOR_MAP_SWIZZLE_128B, promo ? CU_TENSOR_MAP_L2_PROMOTION_L2_256B : CU_TENSOR_MAP_L2_PROMOTION_NONE,
                    CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
                for (int bps : {1, 4}) {
                    for (int stages : {4, 8}) {
                        int stage_bytes = box_rows * 128 * bps;
                        int smem = stage_bytes * stages + 1024;
                        if (smem > 220 * 1024) continue;
                        cudaFuncSetAttribute(tma_bench, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
                        int iters = 4000 * 64 / (box_rows * bps);
                        tma_bench<<<148, 64, smem>>>(m, rows, box_rows, bps, stages, 10, C);
                        cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
                        cudaEventRecord(e0);
                        tma_bench<<<148, 64, smem>>>(m, rows, box_rows, bps, stages, iters, C);
                        cudaEventRecord(e1); cudaEventSynchronize(e1);
                        float ms; cudaEventElapsedTime(&ms, e0, e1);
                        double bytes = 148.0 * iters * stage_bytes;
                        printf("C=%4d box_rows=%3d promo=%d boxes/stage=%d stages=%d inflight=%6d B: %7.1f GB/s (%5.1f B/clk/SM) %s\n",
                               C, box_rows, promo, bps, stages, stage_bytes * stages, bytes / (ms / 1e3) / 1e9,
                               bytes / (ms / 1e3) / 148 / 1.9e9, cudaGetErrorString(cudaGetLastError()));
                    }
                }
            }
        }
        cudaFree(buf);
    }
    return 0;
}
