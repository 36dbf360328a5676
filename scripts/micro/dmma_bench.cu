// fp64 tensor-core (mma.sync.m8n8k4.f64, DMMA) throughput vs DFMA on B200.
#include <cstdio>
__global__ void dmma_kernel(double *out, int iters) {
    double a = threadIdx.x * 1e-3, b = 1.0 + threadIdx.x * 1e-4;
    double c[8][2];
#pragma unroll
    for (int i = 0; i < 8; i++) c[i][0] = c[i][1] = 0.0;
    for (int it = 0; it < iters; it++) {
#pragma unroll
        for (int i = 0; i < 8; i++)
            asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                         : "+d"(c[i][0]), "+d"(c[i][1]) : "d"(a), "d"(b));
    }
    double s = 0;
#pragma unroll
    for (int i = 0; i < 8; i++) s += c[i][0] + c[i][1];
    if (s == 1234.5) out[0] = s;
}
int main() {
    double *d; cudaMalloc(&d, 64);
    int blocks = 148 * 4, threads = 256, iters = 20000;
    dmma_kernel<<<blocks, threads>>>(d, 100);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    cudaEventRecord(e0);
    dmma_kernel<<<blocks, threads>>>(d, iters);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double flops = 2.0 * 8 * 8 * 4 * 8 * (double)iters * blocks * (threads / 32);
    printf("DMMA m8n8k4: %.2f TFLOP/s (%s)\n", flops / (ms / 1e3) / 1e12, cudaGetErrorString(cudaGetLastError()));
    return 0;
}
