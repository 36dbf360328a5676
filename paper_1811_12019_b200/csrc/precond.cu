// precond.cu -- stage 5 of distributed K-FAC (PAPER.md P:264-282 Eqs. K-FAC
// update): the preconditioned gradient of every owned layer
//     𝒢 = G_d^-1 * dW * A_d^-1        (row-major vec, reading R-14)
// as two grouped fp32 GEMM launches over all owned layers:
//     T = dW * A_d^-1   then   𝒢 = G_d^-1 * T.
// fp32 FFMA arithmetic (single-pass bf16/TF32 misses the
// 2e-3 bound on activation-consistent gradients); 128x128 output tiles,
// 256 threads x (8x8) register tiles, double-buffered shared memory.
#include <algorithm>
#include <cstring>

#include "kfac_internal.hpp"

namespace kfac {

constexpr int kMaxGemm = 128;
constexpr int GBM = 128, GBN = 128, GBK = 8;

struct GemmDesc {
    const float *A;  // [M, K] row-major
    const float *B;  // [K, N] row-major
    float *C;        // [M, N] row-major
    int32_t M, N, K, tile_begin, tiles_n;
};
struct GemmParams {
    int32_t ng, total;
    GemmDesc g[kMaxGemm];
};

__global__ void __launch_bounds__(256) sgemm_grouped_kernel(const __grid_constant__ GemmParams P) {
    int tile = blockIdx.x, gi = 0;
    while (gi + 1 < P.ng && P.g[gi + 1].tile_begin <= tile) gi++;
    const GemmDesc &g = P.g[gi];
    const int local = tile - g.tile_begin;
    const int m0 = (local / g.tiles_n) * GBM, n0 = (local % g.tiles_n) * GBN;
    if (m0 >= g.M) return;
    __shared__ float As[2][GBK][GBM];  // transposed A tile: As[k][m]
    __shared__ float Bs[2][GBK][GBN];
    const int tid = threadIdx.x;
    const int tx = tid & 15, ty = tid >> 4;
    // loaders: A tile 128x8 -> each thread 4 elements (rows tid/2, k 4*(tid&1)..+3)
    const int a_r = tid >> 1, a_k = (tid & 1) * 4;
    // B tile 8x128 -> each thread 4 elements (k = tid/32, n = 4*(tid%32)..+3)
    const int b_k = tid >> 5, b_n = (tid & 31) * 4;
    float acc[8][8];
#pragma unroll
    for (int i = 0; i < 8; i++)
#pragma unroll
        for (int j = 0; j < 8; j++) acc[i][j] = 0.f;
    const int ktiles = (g.K + GBK - 1) / GBK;
    float ra[4], rb[4];
    auto load = [&](int kt) {
        const int k0 = kt * GBK;
#pragma unroll
        for (int e = 0; e < 4; e++) {
            int r = m0 + a_r, k = k0 + a_k + e;
            ra[e] = (r < g.M && k < g.K) ? __ldg(g.A + (int64_t)r * g.K + k) : 0.f;
            int kk = k0 + b_k, c = n0 + b_n + e;
            rb[e] = (kk < g.K && c < g.N) ? __ldg(g.B + (int64_t)kk * g.N + c) : 0.f;
        }
    };
    auto store = [&](int buf) {
#pragma unroll
        for (int e = 0; e < 4; e++) {
            As[buf][a_k + e][a_r] = ra[e];
            Bs[buf][b_k][b_n + e] = rb[e];
        }
    };
    load(0);
    store(0);
    __syncthreads();
    for (int kt = 0; kt < ktiles; kt++) {
        const int buf = kt & 1;
        if (kt + 1 < ktiles) load(kt + 1);
#pragma unroll
        for (int k = 0; k < GBK; k++) {
            float a[8], b[8];
#pragma unroll
            for (int i = 0; i < 4; i++) {
                a[i] = As[buf][k][ty * 4 + i];
                a[i + 4] = As[buf][k][64 + ty * 4 + i];
                b[i] = Bs[buf][k][tx * 4 + i];
                b[i + 4] = Bs[buf][k][64 + tx * 4 + i];
            }
#pragma unroll
            for (int i = 0; i < 8; i++)
#pragma unroll
                for (int j = 0; j < 8; j++) acc[i][j] = fmaf(a[i], b[j], acc[i][j]);
        }
        if (kt + 1 < ktiles) {
            store(buf ^ 1);
        }
        __syncthreads();
    }
#pragma unroll
    for (int i = 0; i < 8; i++) {
        const int r = m0 + (i < 4 ? ty * 4 + i : 64 + ty * 4 + (i - 4));
        if (r >= g.M) continue;
#pragma unroll
        for (int j = 0; j < 8; j++) {
            const int c = n0 + (j < 4 ? tx * 4 + j : 64 + tx * 4 + (j - 4));
            if (c < g.N) g.C[(int64_t)r * g.N + c] = acc[i][j];
        }
    }
}

static kfac_status gemm_grouped(const std::vector<GemmDesc> &gs, cudaStream_t st) {
    for (size_t b = 0; b < gs.size(); b += kMaxGemm) {
        GemmParams P;
        memset(&P, 0, sizeof(P));
        int tiles = 0;
        P.ng = (int)std::min<size_t>(kMaxGemm, gs.size() - b);
        for (int i = 0; i < P.ng; i++) {
            GemmDesc d = gs[b + i];
            d.tiles_n = (d.N + GBN - 1) / GBN;
            d.tile_begin = tiles;
            tiles += ((d.M + GBM - 1) / GBM) * d.tiles_n;
            P.g[i] = d;
        }
        P.total = tiles;
        if (!tiles) continue;
        sgemm_grouped_kernel<<<tiles, 256, 0, st>>>(P);
        KFAC_LAUNCHED();
        KFAC_CUDA_TRY(cudaGetLastError());
    }
    return KFAC_OK;
}

kfac_status precond_launch(const std::vector<PrecJob> &jobs, cudaStream_t st) {
    std::vector<GemmDesc> g1, g2;
    for (const PrecJob &j : jobs) {
        GemmDesc a{};
        a.A = j.dW;
        a.B = j.Ainv;
        a.C = j.tmp;
        a.M = j.dG;
        a.N = j.dA;
        a.K = j.dA;
        g1.push_back(a);
        GemmDesc b{};
        b.A = j.Ginv;
        b.B = j.tmp;
        b.C = j.out;
        b.M = j.dG;
        b.N = j.dA;
        b.K = j.dG;
        g2.push_back(b);
    }
    kfac_status s = gemm_grouped(g1, st);
    if (s) return s;
    return gemm_grouped(g2, st);
}

}  // namespace kfac
