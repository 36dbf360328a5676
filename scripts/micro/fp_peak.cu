// Measured FMA peaks: fp64 DFMA and fp32 FFMA, all SMs, independent chains.
#include <cstdio>
template <typename T>
__global__ void fma_kernel(T *out, int iters, T a, T b) {
    T x[16];
#pragma unroll
    for (int i = 0; i < 16; i++) x[i] = (T)(threadIdx.x + i);
    for (int it = 0; it < iters; it++) {
#pragma unroll
        for (int i = 0; i < 16; i++) x[i] = x[i] * a + b;
    }
    T s = 0;
#pragma unroll
    for (int i = 0; i < 16; i++) s += x[i];
    if (s == (T)1234.5) out[0] = s;
}
template <typename T>
void run(const char *name) {
    T *d; cudaMalloc(&d, 64);
    int blocks = 148 * 8, threads = 256, iters = 20000;
    fma_kernel<T><<<blocks, threads>>>(d, 100, (T)0.999, (T)0.001);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    cudaEventRecord(e0);
    fma_kernel<T><<<blocks, threads>>>(d, iters, (T)0.999, (T)0.001);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double flops = 2.0 * 16 * iters * (double)blocks * threads;
    printf("%s: %.2f TFLOP/s\n", name, flops / (ms / 1e3) / 1e12);
}
int main() { run<double>("fp64 DFMA"); run<float>("fp32 FFMA"); run<double>("fp64 DFMA"); return 0; }
