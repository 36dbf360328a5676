// Microbenchmark: tcgen05.mma kind::f16 issue rate for M=128, N in {128,256},
// operands MN- or K-major (SW128), smem-resident (no TMA).  One CTA per SM.
#include <cstdio>
#include <cstdint>
#include "../../paper_1811_12019_b200/csrc/sm100.cuh"
using namespace kfac;

template <int N, int AMN, int BMN>
__global__ void __launch_bounds__(128, 1) mma_bench(int iters, long long *cycles) {
    extern __shared__ uint8_t raw[];
    uint8_t *smem = (uint8_t *)(((uintptr_t)raw + 1023) & ~uintptr_t(1023));
    __shared__ uint64_t bar;
    __shared__ uint32_t tslot;
    const int warp = threadIdx.x / 32;
    for (int i = threadIdx.x; i < (128 + N) * 64 * 2 / 4; i += blockDim.x) ((uint32_t *)smem)[i] = 0x3c003c00u;
    if (threadIdx.x == 0) { mbar_init(&bar, 1); fence_barrier_init(); }
    if (warp == 0) tmem_alloc(&tslot, 512);
    fence_proxy_async_smem();
    tc_fence_before(); __syncthreads(); tc_fence_after();
    uint32_t tmem = tslot;
    if (threadIdx.x == 0) {
        const uint32_t a = smem_u32(smem), b = a + 128 * 64 * 2;
        const uint32_t idesc = idesc_f16(1, 128, N, AMN, BMN);
        long long t0 = clock64();
        for (int it = 0; it < iters; it++) {
            for (int k = 0; k < 4; k++) {
                uint64_t ad, bd;
                // MN-major SW128: 64-elem atoms along MN at LBO = 8 KB (64 rows x 128 B), K groups at SBO = 1 KB
                // K-major SW128: rows of 64 K-elems (128 B); 8-row groups at SBO = 1 KB; K=16 step = 32 B
                if (AMN) ad = umma_desc(a + k * 2048, 8192, 1024, UMMA_SW128);
                else ad = umma_desc(a + k * 32, 16, 1024, UMMA_SW128);
                if (BMN) bd = umma_desc(b + k * 2048, 8192, 1024, UMMA_SW128);
                else bd = umma_desc(b + k * 32, 16, 1024, UMMA_SW128);
                mma_f16_ss(tmem, ad, bd, idesc, (it | k) ? 1u : 0u);
            }
        }
        mma_commit(&bar);
        mbar_wait(&bar, 0);
        long long t1 = clock64();
        if (blockIdx.x == 0) cycles[0] = t1 - t0;
    }
    tc_fence_before(); __syncthreads();
    if (warp == 0) { tc_fence_after(); tmem_dealloc(tmem, 512); }
}

template <int N, int AMN, int BMN>
void run(const char *name) {
    long long *d; cudaMalloc(&d, 8);
    int smem = 1024 + (128 + N) * 64 * 2;
    cudaFuncSetAttribute(mma_bench<N, AMN, BMN>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    int iters = 2000;
    mma_bench<N, AMN, BMN><<<148, 128, smem>>>(iters, d);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    cudaEventRecord(e0);
    mma_bench<N, AMN, BMN><<<148, 128, smem>>>(iters, d);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    long long c; cudaMemcpy(&c, d, 8, cudaMemcpyDeviceToHost);
    double flops = 2.0 * 128 * N * 64 * iters * 148;
    printf("%-28s cycles/MMA(K16) %7.1f  (floor %d)  %7.1f TFLOP/s  err=%s\n", name, (double)c / (iters * 4),
           128 * N / 256, flops / (ms / 1e3) / 1e12, cudaGetErrorString(cudaGetLastError()));
    cudaFree(d);
}

int main() {
    run<128, 1, 1>("N128 A:MN B:MN");
    run<256, 1, 1>("N256 A:MN B:MN");
    run<128, 0, 0>("N128 A:K  B:K");
    run<256, 0, 0>("N256 A:K  B:K");
    run<256, 0, 1>("N256 A:K  B:MN");
    run<256, 1, 0>("N256 A:MN B:K");
    return 0;
}
