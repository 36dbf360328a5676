// bn.cu -- the Fisher of the Batch Normalization layers (NEXT-2; PAPER.md P:493-494,
// P:665-668 "we do not factorize the FIM for the Batch Normalization layers"
// diagonal approximation; reading R-22).
//
// A BN layer y = gamma * xhat + beta has 2C parameters.  Its empirical Fisher is
//   F = (1/N) sum_s S_s S_s^T,   S_s = [sum_p gy_s,p * xhat_s,p ; sum_p gy_s,p]  (2C, scale first)
// over the N samples s and the H*W pixels p.  F has rank <= N (32 per GPU), so the full-mode
// preconditioner never forms the 2C x 2C matrix: by the Woodbury identity
//   (F + lambda I)^-1 v = (v - S^T (lambda N I + S S^T)^-1 S v) / lambda,
// an N x N fp64 Cholesky solve per layer.  This is the same vector the paper's explicit
// (F + gamma_BN I)^-1 gives (exact up to rounding), at O(N^2 C) instead of O(C^3) work and with
// N x 2C instead of 2C(2C+1)/2 values to keep.
//   bn_grads_kernel    S from xhat, gy (NHWC half): one block per (layer, sample, 64-channel
//                      chunk), 8 warps over the pixels, fp32 accumulation, fixed-order combine.
//                      HBM-bound: 4 B per (pixel, channel) read.
//   bn_precond_kernel  one CTA per layer: diag mode grad_i / (F_ii + lambda); full mode the
//                      Woodbury solve above, fp64 throughout.
#include <cmath>

#include <cuda_fp16.h>

#include "kfac_internal.hpp"

namespace kfac {

namespace {

constexpr int kBnMax = 128;     // BN layers per grouped launch
constexpr int kBnChunk = 64;    // channels per bn_grads block (32 lanes x bf16x2)
constexpr int kBnCols = 128;    // S columns staged per chunk in bn_precond_kernel
constexpr int kBnThreads = 256;

struct BnGradParams {
    const uint32_t *x[kBnMax];  // xhat, NHWC, viewed as channel pairs
    const uint32_t *g[kBnMax];  // gy
    float *S[kBnMax];           // [n][2C]
    int32_t c[kBnMax], hw[kBnMax];
    int32_t first[kBnMax + 1];  // first block of layer l
    int32_t nl, n, fp16;
};

struct BnPrecParams {
    const float *S[kBnMax];
    const float *grad[kBnMax];
    float *out[kBnMax];
    int32_t c[kBnMax];
    int32_t nl, n, full;
    double lambda;
};

__device__ __forceinline__ float2 h2f(uint32_t v, int fp16) {
    if (fp16) {
        const __half2 h = *reinterpret_cast<const __half2 *>(&v);
        return __half22float2(h);
    }
    return make_float2(__uint_as_float(v << 16), __uint_as_float(v & 0xffff0000u));
}

__global__ void __launch_bounds__(kBnThreads) bn_grads_kernel(const __grid_constant__ BnGradParams P) {
    __shared__ float red[8][2][2 * 32];
    int l = 0, hi = P.nl - 1;
    while (l < hi) {
        const int mid = (l + hi + 1) >> 1;
        if (P.first[mid] <= (int)blockIdx.x) l = mid;
        else hi = mid - 1;
    }
    const int C = P.c[l], hw = P.hw[l], nchunk = (C + kBnChunk - 1) / kBnChunk;
    const int b = blockIdx.x - P.first[l];
    const int s = b / nchunk, c0 = (b % nchunk) * kBnChunk;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int cp = c0 / 2 + lane;  // channel pair index
    const bool ok = 2 * cp < C;
    const int64_t rowp = C / 2;  // pairs per pixel
    const uint32_t *xs = P.x[l] + (int64_t)s * hw * rowp + cp, *gs = P.g[l] + (int64_t)s * hw * rowp + cp;
    float sg0 = 0.f, sg1 = 0.f, sb0 = 0.f, sb1 = 0.f;
    if (ok) {
#pragma unroll 4
        for (int p = warp; p < hw; p += 8) {
            const float2 xv = h2f(__ldcs(xs + (int64_t)p * rowp), P.fp16);
            const float2 gv = h2f(__ldcs(gs + (int64_t)p * rowp), P.fp16);
            sg0 = fmaf(gv.x, xv.x, sg0);
            sg1 = fmaf(gv.y, xv.y, sg1);
            sb0 += gv.x;
            sb1 += gv.y;
        }
    }
    red[warp][0][2 * lane] = sg0;
    red[warp][0][2 * lane + 1] = sg1;
    red[warp][1][2 * lane] = sb0;
    red[warp][1][2 * lane + 1] = sb1;
    __syncthreads();
    if (threadIdx.x < 128) {  // 64 channels x {scale, shift}, warps combined in order
        const int which = threadIdx.x >> 6, j = threadIdx.x & 63, c = c0 + j;
        if (c < C) {
            float v = 0.f;
#pragma unroll
            for (int w = 0; w < 8; w++) v += red[w][which][j];
            P.S[l][(int64_t)s * 2 * C + which * C + c] = v;
        }
    }
}

__global__ void __launch_bounds__(kBnThreads) bn_precond_kernel(const __grid_constant__ BnPrecParams P) {
    extern __shared__ double bsm[];
    const int l = blockIdx.x, C2 = 2 * P.c[l], n = P.n, tid = threadIdx.x;
    const float *S = P.S[l], *v = P.grad[l];
    float *out = P.out[l];
    const double lam = P.lambda;
    if (!P.full) {  // diagonal Fisher
        for (int i = tid; i < C2; i += kBnThreads) {
            double f = 0.0;
            for (int s = 0; s < n; s++) {
                const double x = S[(int64_t)s * C2 + i];
                f += x * x;
            }
            out[i] = (float)((double)v[i] / (f / n + lam));
        }
        return;
    }
    // full Fisher via Woodbury: K = S S^T + lambda n I (n x n), u = S v, K y = u, out = (v - S^T y) / lambda
    double *K = bsm;                                      // [n][n]
    double *u = K + n * n;                                // [n]
    float *St = reinterpret_cast<float *>(u + n);         // [n][kBnCols + 1] staged S columns
    float *vs = St + n * (kBnCols + 1);                   // [kBnCols]
    const int npair = n * (n + 1) / 2;
    double kacc[(kBnMax * (kBnMax + 1) / 2 + kBnThreads - 1) / kBnThreads];
    constexpr int kPer = (kBnMax * (kBnMax + 1) / 2 + kBnThreads - 1) / kBnThreads;
#pragma unroll
    for (int q = 0; q < kPer; q++) kacc[q] = 0.0;
    double uacc = 0.0;
    for (int j0 = 0; j0 < C2; j0 += kBnCols) {
        const int nc = min(kBnCols, C2 - j0);
        __syncthreads();
        for (int e = tid; e < n * kBnCols; e += kBnThreads) {
            const int a = e / kBnCols, j = e % kBnCols;
            St[a * (kBnCols + 1) + j] = j < nc ? S[(int64_t)a * C2 + j0 + j] : 0.f;
        }
        for (int j = tid; j < kBnCols; j += kBnThreads) vs[j] = j < nc ? v[j0 + j] : 0.f;
        __syncthreads();
#pragma unroll
        for (int q = 0; q < kPer; q++) {
            const int pr = tid + q * kBnThreads;
            if (pr < npair) {
                int a = (int)((sqrtf(8.f * pr + 1.f) - 1.f) * 0.5f);  // pr -> (a, b), b <= a (row-major lower)
                while (a * (a + 1) / 2 > pr) a--;
                while ((a + 1) * (a + 2) / 2 <= pr) a++;
                const int bb = pr - a * (a + 1) / 2;
                const float *ra = St + a * (kBnCols + 1), *rb = St + bb * (kBnCols + 1);
                double acc = kacc[q];
                for (int j = 0; j < kBnCols; j++) acc += (double)ra[j] * rb[j];
                kacc[q] = acc;
            }
        }
        if (tid < n) {
            const float *ra = St + tid * (kBnCols + 1);
            for (int j = 0; j < kBnCols; j++) uacc += (double)ra[j] * vs[j];
        }
    }
#pragma unroll
    for (int q = 0; q < kPer; q++) {
        const int pr = tid + q * kBnThreads;
        if (pr < npair) {
            int a = (int)((sqrtf(8.f * pr + 1.f) - 1.f) * 0.5f);
            while (a * (a + 1) / 2 > pr) a--;
            while ((a + 1) * (a + 2) / 2 <= pr) a++;
            const int bb = pr - a * (a + 1) / 2;
            const double kv = kacc[q] + (a == bb ? lam * n : 0.0);
            K[a * n + bb] = kv;
            K[bb * n + a] = kv;
        }
    }
    if (tid < n) u[tid] = uacc;
    __syncthreads();
    // Cholesky K = L L^T in place (lower), right-looking, one column per step
    for (int k = 0; k < n; k++) {
        if (tid == 0) K[k * n + k] = sqrt(K[k * n + k]);
        __syncthreads();
        const double d = K[k * n + k];
        for (int i = k + 1 + tid; i < n; i += kBnThreads) K[i * n + k] /= d;
        __syncthreads();
        for (int e = tid; e < (n - k - 1) * (n - k - 1); e += kBnThreads) {
            const int i = k + 1 + e / (n - k - 1), j = k + 1 + e % (n - k - 1);
            if (j <= i) K[i * n + j] -= K[i * n + k] * K[j * n + k];
        }
        __syncthreads();
    }
    if (tid == 0) {  // L z = u, L^T y = z (y in u)
        for (int i = 0; i < n; i++) {
            double t = u[i];
            for (int j = 0; j < i; j++) t -= K[i * n + j] * u[j];
            u[i] = t / K[i * n + i];
        }
        for (int i = n - 1; i >= 0; i--) {
            double t = u[i];
            for (int j = i + 1; j < n; j++) t -= K[j * n + i] * u[j];
            u[i] = t / K[i * n + i];
        }
    }
    __syncthreads();
    for (int i = tid; i < C2; i += kBnThreads) {
        double t = v[i];
        for (int a = 0; a < n; a++) t -= (double)S[(int64_t)a * C2 + i] * u[a];
        out[i] = (float)(t / lam);
    }
}

}  // namespace

int64_t bn_precond_smem(int n) {
    return (int64_t)n * n * 8 + (int64_t)n * 8 + (int64_t)n * (kBnCols + 1) * 4 + kBnCols * 4;
}

kfac_status bn_grads_launch(const std::vector<BnJob> &jobs, int n, int fp16, cudaStream_t st) {
    for (size_t j0 = 0; j0 < jobs.size(); j0 += kBnMax) {
        static BnGradParams P;
        P.nl = (int)std::min<size_t>(kBnMax, jobs.size() - j0);
        P.n = n;
        P.fp16 = fp16;
        int32_t nb = 0;
        for (int k = 0; k < P.nl; k++) {
            const BnJob &b = jobs[j0 + k];
            P.x[k] = static_cast<const uint32_t *>(b.xhat);
            P.g[k] = static_cast<const uint32_t *>(b.gy);
            P.S[k] = b.S;
            P.c[k] = b.c;
            P.hw[k] = b.hw;
            P.first[k] = nb;
            nb += n * ((b.c + kBnChunk - 1) / kBnChunk);
        }
        P.first[P.nl] = nb;
        bn_grads_kernel<<<nb, kBnThreads, 0, st>>>(P);
        KFAC_LAUNCHED();
        KFAC_CUDA_TRY(cudaGetLastError());
    }
    return KFAC_OK;
}

kfac_status bn_precond_launch(const std::vector<BnJob> &jobs, int n, int full, double lambda, cudaStream_t st) {
    const int64_t smem = full ? bn_precond_smem(n) : 0;
    if (full) KFAC_CUDA_TRY(cudaFuncSetAttribute(bn_precond_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    for (size_t j0 = 0; j0 < jobs.size(); j0 += kBnMax) {
        static BnPrecParams P;
        P.nl = (int)std::min<size_t>(kBnMax, jobs.size() - j0);
        P.n = n;
        P.full = full;
        P.lambda = lambda;
        for (int k = 0; k < P.nl; k++) {
            const BnJob &b = jobs[j0 + k];
            P.S[k] = b.S;
            P.grad[k] = b.grad;
            P.out[k] = b.out;
            P.c[k] = b.c;
        }
        bn_precond_kernel<<<P.nl, kBnThreads, smem, st>>>(P);
        KFAC_LAUNCHED();
        KFAC_CUDA_TRY(cudaGetLastError());
    }
    return KFAC_OK;
}

}  // namespace kfac
