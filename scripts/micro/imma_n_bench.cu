// Throughput of tcgen05.mma kind::i8 (M = 128, K = 32, cta_group::1) as a function of N: one CTA per
// SM issues R back-to-back MMAs from shared memory (zeros) into TMEM; cycles per MMA and MACs/clk.
#include <cstdio>
#include <cstdint>
#include "../../paper_1811_12019_b200/csrc/sm100.cuh"
using namespace kfac;
__device__ __forceinline__ void mma_i8(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
    asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\ttcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}"
                 ::"r"(d), "l"(a), "l"(b), "r"(idesc), "r"(acc) : "memory");
}
__global__ void bench(int N, int R, long long *out) {
    extern __shared__ __align__(1024) uint8_t sm[];
    __shared__ uint32_t slot;
    __shared__ uint64_t bar;
    for (int i = threadIdx.x; i < 128 * 128 + 256 * 128; i += blockDim.x) sm[i] = 0;
    if (threadIdx.x == 0) { mbar_init(&bar, 1); fence_barrier_init(); }
    if (threadIdx.x < 32) tmem_alloc(&slot, 512);
    fence_proxy_async_smem();
    tc_fence_before(); __syncthreads(); tc_fence_after();
    const uint32_t idesc = (2u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
    if (threadIdx.x == 0) {
        const uint64_t da = umma_desc(smem_u32(sm), 16, 1024, UMMA_SW128), db = umma_desc(smem_u32(sm + 128 * 128), 16, 1024, UMMA_SW128);
        long long t0 = clock64();
        for (int r = 0; r < R; r++) mma_i8(slot, da + ((r & 3) * 2), db + ((r & 3) * 2), idesc, r > 0);
        mma_commit(&bar);
        mbar_wait(&bar, 0);
        long long t1 = clock64();
        out[blockIdx.x] = t1 - t0;
    }
    tc_fence_before(); __syncthreads();
    if (threadIdx.x < 32) { tc_fence_after(); tmem_dealloc(slot, 512); }
}
int main() {
    long long *d; cudaMalloc(&d, 148 * 8);
    cudaFuncSetAttribute(bench, cudaFuncAttributeMaxDynamicSharedMemorySize, 128 * 128 + 256 * 128 + 1024);
    for (int N : {16, 32, 48, 64, 96, 128, 160, 192, 256}) {
        const int R = 4096;
        bench<<<148, 128, 128 * 128 + 256 * 128 + 1024>>>(N, R, d);
        bench<<<148, 128, 128 * 128 + 256 * 128 + 1024>>>(N, R, d);
        long long h[148]; cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
        double c = 0; for (int i = 0; i < 148; i++) c += h[i]; c /= 148;
        printf("N=%3d: %.1f cycles/MMA, %.0f MACs/clk/SM (err %s)\n", N, c / R, 128.0 * N * 32 * R / c,
               cudaGetErrorString(cudaGetLastError()));
    }
    return 0;
}
