// TMA throughput: (a) boxes issued by 1 thread vs by 4 warps; (b) 3-D box {64 ch, R rows, nblk channel blocks}.
#include <cstdio>
#include <cstdint>
#include <cuda.h>
#include <cuda_runtime.h>
#include "../../paper_1811_12019_b200/csrc/sm100.cuh"
using namespace kfac;

__device__ __forceinline__ void tma3(void *dst, const CUtensorMap *m, uint64_t *bar, int c0, int c1, int c2) {
    asm volatile("cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5}], [%2];"
                 ::"r"(smem_u32(dst)), "l"((uint64_t)m), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "r"(c2) : "memory");
}

// mode 0: one thread issues `bps` 2-D boxes; mode 1: warps 0..bps-1 lane 0 each issue one 2-D box;
// mode 2: one thread issues one 3-D box of nblk channel blocks
__global__ void __launch_bounds__(160, 1) bench(const __grid_constant__ CUtensorMap m2, const __grid_constant__ CUtensorMap m3,
                                                int rows_total, int R, int bps, int stages, int iters, int mode) {
    extern __shared__ uint8_t raw[];
    uint8_t *smem = (uint8_t *)(((uintptr_t)raw + 1023) & ~uintptr_t(1023));
    __shared__ uint64_t full[16], empty[16];
    const int warp = threadIdx.x / 32, lane = threadIdx.x & 31;
    if (threadIdx.x == 0) {
        for (int s = 0; s < stages; s++) { mbar_init(&full[s], mode == 1 ? bps : 1); mbar_init(&empty[s], mode == 1 ? bps : 1); }
        fence_barrier_init();
    }
    __syncthreads();
    const uint32_t box_bytes = R * 128;
    const uint32_t stage_bytes = box_bytes * bps;
    const int nrb = rows_total / R;
    const bool issuer = (mode == 1) ? (warp < bps && lane == 0) : (warp == 0 && lane == 0);
    if (issuer) {
        uint32_t st = 0, ph = 0;
        for (int it = 0; it < iters; it++) {
            mbar_wait(&empty[st], ph ^ 1);
            int rb = (blockIdx.x * 7 + it * 3) % nrb;
            if (mode == 0) {
                mbar_arrive_expect_tx(&full[st], stage_bytes);
                for (int b = 0; b < bps; b++) tma_load_2d(smem + st * stage_bytes + b * box_bytes, &m2, &full[st], (b % 8) * 64, rb * R);
            } else if (mode == 1) {
                mbar_arrive_expect_tx(&full[st], box_bytes);
                tma_load_2d(smem + st * stage_bytes + warp * box_bytes, &m2, &full[st], (warp % 8) * 64, rb * R);
            } else {
                mbar_arrive_expect_tx(&full[st], stage_bytes);
                tma3(smem + st * stage_bytes, &m3, &full[st], 0, rb * R, 0);
            }
            if (++st == stages) { st = 0; ph ^= 1; }
        }
    }
    if (warp == 4 && lane == 0) {
        uint32_t st = 0, ph = 0;
        for (int it = 0; it < iters; it++) {
            mbar_wait(&full[st], ph);
            for (int k = 0; k < (mode == 1 ? bps : 1); k++) mbar_arrive(&empty[st]);
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
    const int rows = 1 << 15, C = 512;
    void *buf; cudaMalloc(&buf, (size_t)rows * C * 2); cudaMemset(buf, 0, (size_t)rows * C * 2);
    for (int R : {64, 128}) {
        for (int bps : {2, 4}) {
            CUtensorMap m2, m3;
            cuuint64_t d2[2] = {(cuuint64_t)C, (cuuint64_t)rows}; cuuint64_t s2[1] = {(cuuint64_t)C * 2};
            cuuint32_t b2[2] = {64, (cuuint32_t)R}; cuuint32_t e2[2] = {1, 1};
            enc(&m2, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, buf, d2, s2, b2, e2, CU_TENSOR_MAP_INTERLEAVE_NONE,
                CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
            cuuint64_t d3[3] = {64, (cuuint64_t)rows, (cuuint64_t)(C / 64)}; cuuint64_t s3[2] = {(cuuint64_t)C * 2, 128};
            cuuint32_t b3[3] = {64, (cuuint32_t)R, (cuuint32_t)bps}; cuuint32_t e3[3] = {1, 1, 1};
            CUresult r3 = enc(&m3, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, buf, d3, s3, b3, e3, CU_TENSOR_MAP_INTERLEAVE_NONE,
                              CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
            for (int mode = 0; mode < 3; mode++) {
                int stages = 4;
                int stage_bytes = R * 128 * bps;
                int smem = stage_bytes * stages + 1024;
                if (smem > 220 * 1024) continue;
                cudaFuncSetAttribute(bench, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
                int iters = 3000 * 64 / (R * bps) * 4;
                bench<<<148, 160, smem>>>(m2, m3, rows, R, bps, stages, 10, mode);
                cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
                cudaEventRecord(e0);
                bench<<<148, 160, smem>>>(m2, m3, rows, R, bps, stages, iters, mode);
                cudaEventRecord(e1); cudaEventSynchronize(e1);
                float ms; cudaEventElapsedTime(&ms, e0, e1);
                double bytes = 148.0 * iters * stage_bytes;
                printf("R=%3d boxes/stage=%d mode=%d (%s) enc3=%d: %7.1f GB/s (%5.1f B/clk/SM) %s\n", R, bps, mode,
                       mode == 0 ? "1 thread" : mode == 1 ? "1 warp per box" : "3-D box", (int)r3,
                       bytes / (ms / 1e3) / 1e9, bytes / (ms / 1e3) / 148 / 1.9e9, cudaGetErrorString(cudaGetLastError()));
            }
        }
    }
    return 0;
}
