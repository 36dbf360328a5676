// fp64 tensor-core shapes on B200: m8n8k4 vs m16n8k4 / m16n8k8 / m16n8k16 (register operands),
// 2 warps per SMSP (the inverse tile kernel's occupancy) and 8 warps per SMSP.
#include <cstdio>
template <int SHAPE>
__global__ void k(double *out, int iters) {
    double a[8], b[4], c[8][4];
#pragma unroll
    for (int i = 0; i < 8; i++) a[i] = threadIdx.x * 1e-3 + i;
#pragma unroll
    for (int i = 0; i < 4; i++) b[i] = 1.0 + threadIdx.x * 1e-4 + i;
#pragma unroll
    for (int i = 0; i < 8; i++)
#pragma unroll
        for (int j = 0; j < 4; j++) c[i][j] = 0.0;
    for (int it = 0; it < iters; it++) {
#pragma unroll
        for (int i = 0; i < 8; i++) {
            if (SHAPE == 0)
                asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                             : "+d"(c[i][0]), "+d"(c[i][1]) : "d"(a[0]), "d"(b[0]));
            else if (SHAPE == 1)
                asm volatile("mma.sync.aligned.m16n8k4.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5}, {%6}, {%0,%1,%2,%3};"
                             : "+d"(c[i][0]), "+d"(c[i][1]), "+d"(c[i][2]), "+d"(c[i][3]) : "d"(a[0]), "d"(a[1]), "d"(b[0]));
            else if (SHAPE == 2)
                asm volatile("mma.sync.aligned.m16n8k8.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
                             : "+d"(c[i][0]), "+d"(c[i][1]), "+d"(c[i][2]), "+d"(c[i][3])
                             : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(b[0]), "d"(b[1]));
            else
                asm volatile("mma.sync.aligned.m16n8k16.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7,%8,%9,%10,%11}, {%12,%13,%14,%15}, {%0,%1,%2,%3};"
                             : "+d"(c[i][0]), "+d"(c[i][1]), "+d"(c[i][2]), "+d"(c[i][3])
                             : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(a[4]), "d"(a[5]), "d"(a[6]), "d"(a[7]),
                               "d"(b[0]), "d"(b[1]), "d"(b[2]), "d"(b[3]));
        }
    }
    double s = 0;
#pragma unroll
    for (int i = 0; i < 8; i++)
#pragma unroll
        for (int j = 0; j < 4; j++) s += c[i][j];
    if (s == 1234.5) out[0] = s;
}
template <int SHAPE>
void run(const char *name, int wps) {
    double *d; cudaMalloc(&d, 64);
    const int threads = wps * 4 * 32, blocks = 148, iters = 4000;
    k<SHAPE><<<blocks, threads>>>(d, 10);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    cudaEventRecord(e0);
    k<SHAPE><<<blocks, threads>>>(d, iters);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    const double fl[4] = {8 * 8 * 4, 16 * 8 * 4, 16 * 8 * 8, 16 * 8 * 16};
    double flops = 2.0 * fl[SHAPE] * 8 * (double)iters * blocks * (threads / 32);
    printf("%-10s %d warps/SMSP: %.2f TFLOP/s (%s)\n", name, wps, flops / (ms / 1e3) / 1e12, cudaGetErrorString(cudaGetLastError()));
}
int main() {
    for (int w : {2, 8}) {
        run<0>("m8n8k4", w);
        run<1>("m16n8k4", w);
        run<2>("m16n8k8", w);
        run<3>("m16n8k16", w);
    }
    return 0;
}
