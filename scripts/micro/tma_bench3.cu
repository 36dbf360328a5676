// TMA throughput of the factor kernel's box shapes (L2-resident NHWC activations, all SMs).
// A producer ring of `stages` stages x `bps` boxes; `nis` issuer warps (lane 0 each) issue the
// boxes of a stage round-robin, one consumer thread frees stages as soon as they land.
// Box kinds: 2-D {64 ch, 64 rows}; 4-D {64 ch, W cols, BH rows, 1 image} at a filter-tap
// offset (dw, dh) in {-1,0,1} (dw = -1 puts one column out of bounds -> zero fill).
#include <cstdio>
#include <cstdint>
#include <cuda.h>
#include <cuda_runtime.h>
#include "../../paper_1811_12019_b200/csrc/sm100.cuh"
using namespace kfac;

struct Cfg {
    int kind;  // 0: 2-D {64, BH rows}; 1: 4-D {64, BW, BH, 1}; 2: 3-D {64, BH rows, S slots}; 3: 5-D {64, BW, BH, 1, S}
    int W, H, N, C, BW, BH, taps_oob, S;
};

__global__ void __launch_bounds__(288, 1) bench(const __grid_constant__ CUtensorMap m, Cfg c, int bps, int stages,
                                                int nis, int iters, uint32_t box_bytes, long long *out) {
    extern __shared__ uint8_t raw[];
    uint8_t *smem = (uint8_t *)(((uintptr_t)raw + 1023) & ~uintptr_t(1023));
    __shared__ uint64_t full[8], empty[8];
    const int warp = threadIdx.x / 32, lane = threadIdx.x & 31;
    if (threadIdx.x == 0) {
        for (int s = 0; s < stages; s++) {
            mbar_init(&full[s], nis < 0 ? -nis : nis);
            mbar_init(&empty[s], 1);
        }
        fence_barrier_init();
    }
    __syncthreads();
    const uint32_t slot = (box_bytes + 1023) / 1024 * 1024, stage_bytes = slot * bps;
    long long t0 = clock64();
    const bool lanes_mode = nis < 0;  // -k: lanes 0..k-1 of warp 1 issue
    const int nisa = lanes_mode ? -nis : nis;
    if (lanes_mode ? (warp == 1 && lane < nisa) : (warp >= 1 && warp <= nis && lane == 0)) {
        const int w = lanes_mode ? lane : warp - 1;
        nis = nisa;
        uint32_t st = 0, ph = 0;
        for (int it = 0; it < iters; it++) {
            mbar_wait(&empty[st], ph ^ 1);
            uint32_t bytes = 0;
            for (int b = w; b < bps; b += nis) bytes += box_bytes;
            mbar_arrive_expect_tx(&full[st], bytes);
            const int chunk = (c.taps_oob & 2) ? it : blockIdx.x * 131 + it;  // taps_oob bit 1: all CTAs read the same rows
            for (int b = w; b < bps; b += nis) {
                uint8_t *dst = smem + st * stage_bytes + b * slot;
                if (c.kind == 0) {
                    const int rows = c.N * c.H * c.W;
                    tma_load_2d(dst, &m, &full[st], (b % (c.C / 64)) * 64, (chunk * c.BH) % (rows - c.BH));
                } else if (c.kind == 2) {
                    const int rows = c.N * c.H * c.W;
                    asm volatile("cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5}], [%2];"
                                 ::"r"(smem_u32(dst)), "l"((uint64_t)&m), "r"(smem_u32(&full[st])), "r"(0), "r"((chunk * c.BH) % (rows - c.BH)), "r"(0) : "memory");
                } else if (c.kind == 3) {
                    const int tap = (chunk + b) % 9;
                    const int dh = (c.taps_oob & 1) ? tap / 3 - 1 : 0, dw = (c.taps_oob & 1) ? tap % 3 - 1 : 0;
                    const int rpi = c.H / c.BH;
                    const int n = (chunk / rpi) % c.N, oh0 = (chunk % rpi) * c.BH;
                    asm volatile("cp.async.bulk.tensor.5d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5, %6, %7}], [%2];"
                                 ::"r"(smem_u32(dst)), "l"((uint64_t)&m), "r"(smem_u32(&full[st])), "r"(0), "r"(dw), "r"(oh0 + dh), "r"(n), "r"(0) : "memory");
                } else {
                    const int tap = (chunk + b) % 9;
                    const int dh = (c.taps_oob & 1) ? tap / 3 - 1 : 0, dw = (c.taps_oob & 1) ? tap % 3 - 1 : 0;
                    const int rpi = c.H / c.BH;
                    const int n = (chunk / rpi) % c.N, oh0 = (chunk % rpi) * c.BH;
                    tma_load_4d(dst, &m, &full[st], (b % (c.C / 64)) * 64, dw, oh0 + dh, n);
                }
            }
            if (++st == stages) { st = 0; ph ^= 1; }
        }
    }
    if (warp == 0 && lane == 0) {
        uint32_t st = 0, ph = 0;
        for (int it = 0; it < iters; it++) {
            mbar_wait(&full[st], ph);
            mbar_arrive(&empty[st]);
            if (++st == stages) { st = 0; ph ^= 1; }
        }
        if (blockIdx.x == 0) out[0] = clock64() - t0;
    }
    __syncthreads();
}

typedef CUresult (*PFN)(CUtensorMap *, CUtensorMapDataType, cuuint32_t, void *, const cuuint64_t *, const cuuint64_t *,
                        const cuuint32_t *, const cuuint32_t *, CUtensorMapInterleave, CUtensorMapSwizzle,
                        CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

int main() {
    void *fn;
    cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
    PFN enc = (PFN)fn;
    long long *dout;
    cudaMalloc(&dout, 8);
    Cfg cfgs[] = {
        {0, 56, 56, 32, 256, 64, 64, 0, 1},    // 2-D 64 rows x 128 B
        {0, 56, 56, 32, 256, 64, 128, 0, 1},   // 2-D 128 rows
        {0, 56, 56, 32, 256, 64, 256, 0, 1},   // 2-D 256 rows
        {2, 56, 56, 32, 256, 64, 64, 0, 4},    // 3-D 64 rows x 4 channel slots
        {1, 56, 56, 32, 64, 56, 1, 1, 1},      // 4-D one output row, 3x3 taps (OOB edges)
        {1, 56, 56, 32, 64, 56, 2, 1, 1},      // 4-D two output rows
        {3, 28, 28, 32, 256, 28, 2, 1, 4},     // 5-D two rows of 28 x 4 channel slots
        {1, 7, 7, 32, 512, 7, 7, 1, 1},        // 4-D 7x7 image
        {3, 7, 7, 32, 512, 7, 7, 1, 4},        // 5-D 7x7 image x 4 slots
        {2, 56, 56, 32, 256, 64, 64, 2, 4},    // 3-D 64 rows x 4 slots, all CTAs on the same rows
        {3, 28, 28, 32, 256, 28, 2, 3, 4},     // 5-D, all CTAs on the same rows
    };
    for (const Cfg &c : cfgs) {
        const size_t bytes = (size_t)c.N * c.H * c.W * c.C * 2;
        void *buf;
        cudaMalloc(&buf, bytes);
        cudaMemset(buf, 0, bytes);
        CUtensorMap m;
        CUresult r;
        uint32_t box_bytes;
        if (c.kind == 0) {
            cuuint64_t d[2] = {(cuuint64_t)c.C, (cuuint64_t)c.N * c.H * c.W};
            cuuint64_t s[1] = {(cuuint64_t)c.C * 2};
            cuuint32_t b[2] = {64, (cuuint32_t)c.BH}, e[2] = {1, 1};
            r = enc(&m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, buf, d, s, b, e, CU_TENSOR_MAP_INTERLEAVE_NONE,
                    CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
            box_bytes = c.BH * 128;
        } else if (c.kind == 2) {
            cuuint64_t d[3] = {64, (cuuint64_t)c.N * c.H * c.W, (cuuint64_t)c.C / 64};
            cuuint64_t s[2] = {(cuuint64_t)c.C * 2, 128};
            cuuint32_t b[3] = {64, (cuuint32_t)c.BH, (cuuint32_t)c.S}, e[3] = {1, 1, 1};
            r = enc(&m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, buf, d, s, b, e, CU_TENSOR_MAP_INTERLEAVE_NONE,
                    CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
            box_bytes = c.BH * 128 * c.S;
        } else if (c.kind == 3) {
            cuuint64_t d[5] = {64, (cuuint64_t)c.W, (cuuint64_t)c.H, (cuuint64_t)c.N, (cuuint64_t)c.C / 64};
            cuuint64_t s[4] = {(cuuint64_t)c.C * 2, (cuuint64_t)c.C * 2 * c.W, (cuuint64_t)c.C * 2 * c.W * c.H, 128};
            cuuint32_t b[5] = {64, (cuuint32_t)c.BW, (cuuint32_t)c.BH, 1, (cuuint32_t)c.S}, e[5] = {1, 1, 1, 1, 1};
            r = enc(&m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 5, buf, d, s, b, e, CU_TENSOR_MAP_INTERLEAVE_NONE,
                    CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
            box_bytes = c.BW * c.BH * 128 * c.S;
        } else {
            cuuint64_t d[4] = {(cuuint64_t)c.C, (cuuint64_t)c.W, (cuuint64_t)c.H, (cuuint64_t)c.N};
            cuuint64_t s[3] = {(cuuint64_t)c.C * 2, (cuuint64_t)c.C * 2 * c.W, (cuuint64_t)c.C * 2 * c.W * c.H};
            cuuint32_t b[4] = {64, (cuuint32_t)c.BW, (cuuint32_t)c.BH, 1}, e[4] = {1, 1, 1, 1};
            r = enc(&m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, buf, d, s, b, e, CU_TENSOR_MAP_INTERLEAVE_NONE,
                    CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
            box_bytes = c.BW * c.BH * 128;
        }
        // smem dst slots are 8 KB apart (64 rows) like the factor kernel
        const uint32_t slot = (box_bytes + 1023) / 1024 * 1024;
        for (int nis : {1, 4, 8, -4}) {
            for (int stages : {2}) {
                const int bps = c.S > 1 || box_bytes > 8192 ? 2 : 6;
                const int smem = slot * bps * stages + 1024;
                if (smem > 227 * 1024) continue;
                cudaFuncSetAttribute(bench, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
                const int iters = 4000;
                bench<<<148, 288, smem>>>(m, c, bps, stages, nis, 50, box_bytes, dout);
                cudaEvent_t e0, e1;
                cudaEventCreate(&e0);
                cudaEventCreate(&e1);
                cudaEventRecord(e0);
                bench<<<148, 288, smem>>>(m, c, bps, stages, nis, iters, box_bytes, dout);
                cudaEventRecord(e1);
                cudaEventSynchronize(e1);
                float ms;
                cudaEventElapsedTime(&ms, e0, e1);
                long long cyc;
                cudaMemcpy(&cyc, dout, 8, cudaMemcpyDeviceToHost);
                const double tot = 148.0 * iters * bps * box_bytes;
                printf("kind=%d C=%3d box %2dx%dx%d (%5u B) issuers=%d stages=%d enc=%d: %8.1f GB/s  %5.1f B/clk/SM  "
                       "(%.0f clk/stage) %s\n",
                       c.kind, c.C, c.kind % 2 ? c.BW : c.BH, c.kind % 2 ? c.BH : 1, c.S, box_bytes, nis, stages, (int)r,
                       tot / (ms / 1e3) / 1e9, (double)iters * bps * box_bytes / cyc, (double)cyc / iters,
                       cudaGetErrorString(cudaGetLastError()));
            }
        }
        cudaFree(buf);
    }
    return 0;
}
