// The factor kernel's MMA issue loop in isolation: a ring of `stages` smem stages (no TMA; a
// producer thread re-arms each stage as soon as it is freed), per chunk `ks` K=16 steps of
// two M=128 x N=256 MMAs (two TMEM accumulators sharing B), one commit per chunk.
// Variants: fence (tcgen05.fence::after_thread_sync after each full wait), one accumulator only.
#include <cstdio>
#include <cstdint>
#include "../../paper_1811_12019_b200/csrc/sm100.cuh"
using namespace kfac;

__global__ void __launch_bounds__(128, 1) loop_bench(int chunks, int stages, int ks, int two, int fence, int self, int n1, long long *out) {
    extern __shared__ uint8_t raw[];
    uint8_t *smem = (uint8_t *)(((uintptr_t)raw + 1023) & ~uintptr_t(1023));
    __shared__ uint64_t full[4], empty[4];
    __shared__ uint32_t tslot;
    const int warp = threadIdx.x / 32, lane = threadIdx.x & 31;
    for (int i = threadIdx.x; i < stages * 65536 / 4; i += blockDim.x) ((uint32_t *)smem)[i] = 0x3c003c00u;
    if (threadIdx.x == 0) {
        for (int s = 0; s < stages; s++) { mbar_init(&full[s], 1); mbar_init(&empty[s], 1); }
        fence_barrier_init();
    }
    if (warp == 0) tmem_alloc(&tslot, 512);
    fence_proxy_async_smem();
    tc_fence_before(); __syncthreads(); tc_fence_after();
    const uint32_t tmem = tslot;
    long long t0 = clock64();
    if (warp == 1 && lane == 0 && !self) {
        uint32_t st = 0, ph = 0;
        for (int c = 0; c < chunks; c++) {
            mbar_wait(&empty[st], ph ^ 1);
            mbar_arrive(&full[st]);
            if (++st == stages) { st = 0; ph ^= 1; }
        }
    }
    if (warp == 0 && lane == 0) {
        const uint32_t idesc = idesc_f16(1, 128, 256, 1, 1);
        const uint32_t idesc1 = idesc_f16(1, 128, n1, 1, 1);
        uint32_t st = 0, ph = 0;
        for (int c = 0; c < chunks; c++) {
            if (self) mbar_wait(&empty[st], ph ^ 1);  // one hop: wait for this stage's previous commit
            else mbar_wait(&full[st], ph);
            tc_fence_after();
            const uint32_t a = smem_u32(smem + st * 65536), b = a + 32768;
            if (fence == 2) {  // descriptors advanced by adding the K-step offset (addr >> 4) to the 64-bit word
                const uint64_t da = umma_desc(a, 8192, 1024, UMMA_SW128), db = umma_desc(b, 8192, 1024, UMMA_SW128);
                const uint64_t da1 = umma_desc(a + 16384, 8192, 1024, UMMA_SW128);
#pragma unroll 4
                for (int k = 0; k < ks; k++) {
                    const uint32_t acc = (c | k) ? 1u : 0u;
                    const uint64_t kk = (uint64_t)((k & 3) * 2048 >> 4);
                    mma_f16_ss(tmem, da + kk, db + kk, idesc, acc);
                    if (two) mma_f16_ss(tmem + 256, da1 + kk, db + kk, idesc1, acc);
                }
            } else
            for (int k = 0; k < ks; k++) {
                const uint32_t acc = (c | k) ? 1u : 0u;
                mma_f16_ss(tmem, umma_desc(a + (k & 3) * 2048, 8192, 1024, UMMA_SW128),
                           umma_desc(b + (k & 3) * 2048, 8192, 1024, UMMA_SW128), idesc, acc);
                if (two)
                    mma_f16_ss(tmem + 256, umma_desc(a + 16384 + (k & 3) * 2048, 8192, 1024, UMMA_SW128),
                               umma_desc(b + (k & 3) * 2048, 8192, 1024, UMMA_SW128), idesc1, acc);
            }
            mma_commit(&empty[st]);
            if (++st == stages) { st = 0; ph ^= 1; }
        }
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        // wait for the last commit: re-arm trick -- the producer already consumed all empties except the tail
        if (blockIdx.x == 0) out[0] = clock64() - t0;
    }
    tc_fence_before(); __syncthreads();
    if (warp == 0) { tc_fence_after(); tmem_dealloc(tmem, 512); }
}

int main() {
    long long *d;
    cudaMalloc(&d, 8);
    const int smem = 3 * 65536 + 1024;
    cudaFuncSetAttribute(loop_bench, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    struct V { int stages, ks, two, fence, self, n1; const char *name; } vs[] = {
        {3, 4, 1, 1, 0, 256, "4 ks, 2 acc (256+256)"},
        {3, 4, 1, 2, 0, 256, "4 ks, 2 acc (256+256) desc+="},
        {3, 4, 1, 1, 0, 128, "4 ks, 2 acc (256+128) diag"},
        {3, 4, 1, 2, 0, 128, "4 ks, 2 acc (256+128) diag desc+="},
        {3, 8, 1, 2, 0, 128, "8 ks, 2 acc (256+128) diag desc+="},
        {3, 4, 0, 1, 0, 256, "4 ks, 1 acc"},
        {3, 4, 0, 2, 0, 256, "4 ks, 1 acc desc+="},
        {3, 16, 0, 2, 0, 256, "16 ks, 1 acc desc+="},
        {3, 4, 1, 2, 0, 64, "4 ks, 2 acc (256+64) desc+="},
        {3, 2, 1, 2, 0, 256, "2 ks, 2 acc desc+="},
    };
    for (auto &v : vs) {
        const int chunks = 4000;
        loop_bench<<<148, 128, smem>>>(100, v.stages, v.ks, v.two, v.fence, v.self, v.n1, d);
        cudaEvent_t e0, e1;
        cudaEventCreate(&e0); cudaEventCreate(&e1);
        cudaEventRecord(e0);
        loop_bench<<<148, 128, smem>>>(chunks, v.stages, v.ks, v.two, v.fence, v.self, v.n1, d);
        cudaEventRecord(e1); cudaEventSynchronize(e1);
        float ms; cudaEventElapsedTime(&ms, e0, e1);
        long long cyc; cudaMemcpy(&cyc, d, 8, cudaMemcpyDeviceToHost);
        const double ideal = (double)v.ks * (128 + (v.two ? v.n1 / 2 : 0));
        const double flops = 2.0 * 128 * 16 * v.ks * (256 + (v.two ? v.n1 : 0)) * chunks * (double)148;
        printf("%-40s %7.1f clk/chunk (ideal %4.0f)  %7.1f TFLOP/s  %s\n", v.name, (double)cyc / chunks, ideal,
               flops / (ms / 1e3) / 1e12, cudaGetErrorString(cudaGetLastError()));
    }
    return 0;
}
