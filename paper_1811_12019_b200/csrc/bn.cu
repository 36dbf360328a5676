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
//   bn_grads_kernel    S from xhat, gy (NHWC half): one block per (layer, sample, 256-channel
//                      chunk), 16-byte loads (8 channels per lane; a warp spans 256 / C pixels
//                      when C < 256), 8 warps over the pixels, fp32 accumulation, fixed-order
//                      combine; a 4-byte channel-pair path covers other even C.
//                      HBM-bound: 4 B per (pixel, channel) read.
//   bn_diag_kernel     diag mode: grad_i / (F_ii + lambda).
//   bn_gram_kernel     full mode: partial K = S S^T and u = S v over 64-column work items (all layers
//                      in one launch, S staged as fp64 in shared memory).
//   bn_solve_kernel    full mode, one CTA per layer: fixed-order sum of the partials, K + lambda N I,
//                      fp64 Cholesky solve for y;
//   bn_out_kernel      out = (v - S^T y) / lambda, column-parallel.
#include <cmath>

#include <cuda_fp16.h>

#include "kfac_internal.hpp"

namespace kfac {

namespace {

constexpr int kBnMax = 128;     // BN layers per grouped launch
constexpr int kBnChunk = 64;    // channels per bn_grads block (32 lanes x bf16x2)
constexpr int kGramCols = 64;   // S columns per Gram work item (staged as fp64 in shared memory)
constexpr int kBnThreads = 256;

struct BnGradParams {
    const uint32_t *x[kBnMax];  // xhat, NHWC, viewed as channel pairs
    const uint32_t *g[kBnMax];  // gy
    float *S[kBnMax];           // [n][2C]
    int32_t c[kBnMax], hw[kBnMax], vec[kBnMax];  // vec: the 16-byte path
    int32_t first[kBnMax + 1];  // first block of layer l
    int32_t nl, n, fp16;
};

struct BnPrecParams {
    const float *S[kBnMax];
    const float *grad[kBnMax];
    float *out[kBnMax];
    int32_t c[kBnMax];
    int32_t item0[kBnMax + 1];  // first Gram work item of layer l (full mode)
    int32_t nl, n;
    double lambda;
    double *ws;  // Gram partials: per item n(n+1)/2 + n doubles
    double *y;   // [nl][n] solved y of each layer (after the partials in the workspace)
    double *kglob;  // [nl][n][n] K in the workspace when n > kBnSmemSamples, else null
};

__device__ __forceinline__ float2 h2f(uint32_t v, int fp16) {
    if (fp16) {
        const __half2 h = *reinterpret_cast<const __half2 *>(&v);
        return __half22float2(h);
    }
    return make_float2(__uint_as_float(v << 16), __uint_as_float(v & 0xffff0000u));
}

// 4-byte path (any even C): lanes on channel pairs, 64 channels per block
__device__ __forceinline__ void grads_pairs(const BnGradParams &P, int l, int b, float *smem) {
    float (*red)[2][2 * 32] = reinterpret_cast<float (*)[2][2 * 32]>(smem);
    const int C = P.c[l], hw = P.hw[l], nchunk = (C + kBnChunk - 1) / kBnChunk;
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

// 16-byte path (C % 8 == 0 with C/8 dividing 32 or a multiple of 32; 16-byte aligned rows): a lane
// loads 8 channels of one pixel per access; for C < 256 a warp covers 256 / C pixels per step.
// Per lane 8 x {scale, shift} fp32 accumulators; lanes sharing an octet are combined by
// shuffles, the 8 warps in order through shared memory.
__device__ __forceinline__ void grads_octets(const BnGradParams &P, int l, int b, float *smem) {
    float (*red)[32][16] = reinterpret_cast<float (*)[32][16]>(smem);
    const int C = P.c[l], hw = P.hw[l], oct = C / 8;
    const int nchunk = oct >= 32 ? oct / 32 : 1, lpp = oct >= 32 ? 32 : oct, ppw = 32 / lpp;
    const int s = b / nchunk, ch = b % nchunk;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int o = ch * 32 + lane % lpp, q = lane / lpp;
    const uint4 *xs = reinterpret_cast<const uint4 *>(P.x[l]) + (int64_t)s * hw * oct + o;
    const uint4 *gs = reinterpret_cast<const uint4 *>(P.g[l]) + (int64_t)s * hw * oct + o;
    float sg[8], sb[8];
#pragma unroll
    for (int e = 0; e < 8; e++) sg[e] = sb[e] = 0.f;
#pragma unroll 2
    for (int p = warp * ppw + q; p < hw; p += 8 * ppw) {
        const uint4 xv = __ldcs(xs + (int64_t)p * oct), gv = __ldcs(gs + (int64_t)p * oct);
        const uint32_t xw[4] = {xv.x, xv.y, xv.z, xv.w}, gw[4] = {gv.x, gv.y, gv.z, gv.w};
#pragma unroll
        for (int k = 0; k < 4; k++) {
            const float2 xf = h2f(xw[k], P.fp16), gf = h2f(gw[k], P.fp16);
            sg[2 * k] = fmaf(gf.x, xf.x, sg[2 * k]);
            sg[2 * k + 1] = fmaf(gf.y, xf.y, sg[2 * k + 1]);
            sb[2 * k] += gf.x;
            sb[2 * k + 1] += gf.y;
        }
    }
    for (int off = lpp; off < 32; off <<= 1)  // lanes o, o + lpp, ... hold the same octet
#pragma unroll
        for (int e = 0; e < 8; e++) {
            sg[e] += __shfl_xor_sync(0xffffffffu, sg[e], off);
            sb[e] += __shfl_xor_sync(0xffffffffu, sb[e], off);
        }
    if (q == 0)
#pragma unroll
        for (int e = 0; e < 8; e++) {
            red[warp][lane][e] = sg[e];
            red[warp][lane][8 + e] = sb[e];
        }
    __syncthreads();
    // item t < 16 * lpp: octet lane t / 16, element t % 16 (scale e < 8, shift e >= 8)
    for (int t = threadIdx.x; t < 16 * lpp; t += kBnThreads) {
        const int ol = t / 16, e = t % 16;
        float v = 0.f;
#pragma unroll
        for (int w = 0; w < 8; w++) v += red[w][ol][e];
        const int c = (ch * 32 + ol) * 8 + (e & 7);
        P.S[l][(int64_t)s * 2 * C + (e >> 3) * C + c] = v;
    }
}

__global__ void __launch_bounds__(kBnThreads) bn_grads_kernel(const __grid_constant__ BnGradParams P) {
    __shared__ __align__(16) float smem[8 * 32 * 16];
    int l = 0, hi = P.nl - 1;
    while (l < hi) {
        const int mid = (l + hi + 1) >> 1;
        if (P.first[mid] <= (int)blockIdx.x) l = mid;
        else hi = mid - 1;
    }
    const int b = blockIdx.x - P.first[l];
    if (P.vec[l]) grads_octets(P, l, b, smem);
    else grads_pairs(P, l, b, smem);
}

// pair index pr -> (a, b), b <= a, row-major lower triangle
__device__ __forceinline__ void pair_ab(int pr, int &a, int &b) {
    a = (int)((sqrtf(8.f * pr + 1.f) - 1.f) * 0.5f);
    while (a * (a + 1) / 2 > pr) a--;
    while ((a + 1) * (a + 2) / 2 <= pr) a++;
    b = pr - a * (a + 1) / 2;
}

// diagonal Fisher: out_i = grad_i / ((1/n) sum_s S_si^2 + lambda); grid (layer, 256 columns)
__global__ void __launch_bounds__(kBnThreads) bn_diag_kernel(const __grid_constant__ BnPrecParams P) {
    const int l = blockIdx.y, C2 = 2 * P.c[l], n = P.n;
    const int i = blockIdx.x * kBnThreads + threadIdx.x;
    if (i >= C2) return;
    const float *S = P.S[l];
    double f = 0.0;
    for (int s = 0; s < n; s++) {
        const double x = S[(int64_t)s * C2 + i];
        f += x * x;
    }
    P.out[l][i] = (float)((double)P.grad[l][i] / (f / n + P.lambda));
}

// full Fisher, phase 1: partial Gram K_ab = sum_j S_aj S_bj (lower triangle) and u_a = sum_j S_aj v_j over
// one work item = (layer, kGramCols columns), S staged as fp64 in shared memory (conversion once per
// element); every item writes its own partial (fixed-order combine in bn_solve_kernel)
__global__ void __launch_bounds__(kBnThreads) bn_gram_kernel(const __grid_constant__ BnPrecParams P) {
    extern __shared__ double gsm[];
    int l = 0, hi = P.nl - 1;
    while (l < hi) {
        const int mid = (l + hi + 1) >> 1;
        if (P.item0[mid] <= (int)blockIdx.x) l = mid;
        else hi = mid - 1;
    }
    const int C2 = 2 * P.c[l], n = P.n, tid = threadIdx.x, npair = n * (n + 1) / 2;
    const int j0 = (blockIdx.x - P.item0[l]) * kGramCols, nc = min(kGramCols, C2 - j0);
    const float *S = P.S[l], *v = P.grad[l];
    double *St = gsm;                     // [n][kGramCols + 1]
    double *vs = St + n * (kGramCols + 1);  // [kGramCols]
    for (int e = tid; e < n * kGramCols; e += kBnThreads) {
        const int a = e / kGramCols, j = e % kGramCols;
        St[a * (kGramCols + 1) + j] = j < nc ? (double)S[(int64_t)a * C2 + j0 + j] : 0.0;
    }
    for (int j = tid; j < kGramCols; j += kBnThreads) vs[j] = j < nc ? (double)v[j0 + j] : 0.0;
    __syncthreads();
    double *part = P.ws + (int64_t)blockIdx.x * (npair + n);
    for (int pr = tid; pr < npair; pr += kBnThreads) {
        int a, bb;
        pair_ab(pr, a, bb);
        const double *ra = St + a * (kGramCols + 1), *rb = St + bb * (kGramCols + 1);
        double acc0 = 0.0, acc1 = 0.0;
#pragma unroll 4
        for (int j = 0; j < kGramCols; j += 2) {
            acc0 = fma(ra[j], rb[j], acc0);
            acc1 = fma(ra[j + 1], rb[j + 1], acc1);
        }
        part[pr] = acc0 + acc1;
    }
    for (int a = tid; a < n; a += kBnThreads) {
        const double *ra = St + a * (kGramCols + 1);
        double acc = 0.0;
        for (int j = 0; j < kGramCols; j++) acc = fma(ra[j], vs[j], acc);
        part[npair + a] = acc;
    }
}

// full Fisher, phase 2 (one CTA per layer): K = sum of the partials + lambda n I, u likewise; fp64
// Cholesky K = L L^T and the two triangular solves in shared memory; out = (v - S^T y) / lambda
__global__ void __launch_bounds__(kBnThreads) bn_solve_kernel(const __grid_constant__ BnPrecParams P) {
    extern __shared__ double bsm[];
    const int l = blockIdx.x, n = P.n, tid = threadIdx.x, npair = n * (n + 1) / 2;
    const double lam = P.lambda;
    // K [n][n] in shared memory, or (n > kBnSmemSamples) in this layer's workspace slot
    double *K = P.kglob ? P.kglob + (int64_t)l * n * n : bsm;
    double *u = P.kglob ? bsm : K + n * n;  // [n]
    const int it0 = P.item0[l], nit = P.item0[l + 1] - it0;
    for (int q = tid; q < npair + n; q += kBnThreads) {
        double acc = 0.0;
#pragma unroll 8
        for (int it = 0; it < nit; it++) acc += P.ws[(int64_t)(it0 + it) * (npair + n) + q];
        if (q < npair) {
            int a, bb;
            pair_ab(q, a, bb);
            if (a == bb) acc += lam * n;
            K[a * n + bb] = acc;
            K[bb * n + a] = acc;
        } else {
            u[q - npair] = acc;
        }
    }
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
    if (tid < 32) {  // L z = u, then L^T y = z (y in u): warp 0, column-oriented, lanes over rows
        for (int i = 0; i < n; i++) {
            const double zi = u[i] / K[i * n + i];
            __syncwarp();
            if (tid == 0) u[i] = zi;
            for (int j = i + 1 + tid; j < n; j += 32) u[j] -= K[j * n + i] * zi;
            __syncwarp();
        }
        for (int i = n - 1; i >= 0; i--) {
            const double yi = u[i] / K[i * n + i];
            __syncwarp();
            if (tid == 0) u[i] = yi;
            for (int j = tid; j < i; j += 32) u[j] -= K[i * n + j] * yi;
            __syncwarp();
        }
    }
    __syncthreads();
    if (tid < n) P.y[l * n + tid] = u[tid];  // bn_out_kernel finishes the layer column-parallel
}

// full Fisher, phase 3: out = (v - S^T y) / lambda, grid (256-column blocks, layer)
__global__ void __launch_bounds__(kBnThreads) bn_out_kernel(const __grid_constant__ BnPrecParams P) {
    __shared__ double ys[kBnMaxSamples];
    const int l = blockIdx.y, C2 = 2 * P.c[l], n = P.n;
    for (int a = threadIdx.x; a < n; a += kBnThreads) ys[a] = P.y[l * n + a];
    __syncthreads();
    const int i = blockIdx.x * kBnThreads + threadIdx.x;
    if (i >= C2) return;
    const float *S = P.S[l];
    double t = P.grad[l][i];
#pragma unroll 8
    for (int a = 0; a < n; a++) t -= (double)__ldg(S + (int64_t)a * C2 + i) * ys[a];
    P.out[l][i] = (float)(t / P.lambda);
}

}  // namespace

static int64_t gram_items(int c) { return (2 * (int64_t)c + kGramCols - 1) / kGramCols; }

// K in shared memory up to this many samples; past it (up to kBnMaxSamples) each layer's K lives in
// the workspace (L2-resident: n = 256 is 512 KB per layer)
constexpr int kBnSmemSamples = 128;

int64_t bn_ws_bytes(const std::vector<int> &cs, int n) {
    int64_t items = 0;
    for (int c : cs) items += gram_items(c);
    const int64_t kglob = n > kBnSmemSamples ? (int64_t)cs.size() * n * n * 8 : 0;
    return items * ((int64_t)n * (n + 1) / 2 + n) * 8 + kglob + (int64_t)cs.size() * n * 8;
}

kfac_status bn_grads_launch(const std::vector<BnJob> &jobs, int n, int fp16, cudaStream_t st) {
    for (size_t j0 = 0; j0 < jobs.size(); j0 += kBnMax) {
        thread_local BnGradParams P;  // host staging (per thread: calls may come from several threads)
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
            const int oct = b.c / 8;
            const bool aligned = ((reinterpret_cast<uintptr_t>(b.xhat) | reinterpret_cast<uintptr_t>(b.gy)) & 15) == 0;
            P.vec[k] = aligned && b.c % 8 == 0 && (oct >= 32 ? oct % 32 == 0 : 32 % oct == 0);
            nb += n * (P.vec[k] ? (oct >= 32 ? oct / 32 : 1) : (b.c + kBnChunk - 1) / kBnChunk);
        }
        P.first[P.nl] = nb;
        bn_grads_kernel<<<nb, kBnThreads, 0, st>>>(P);
        KFAC_LAUNCHED();
        KFAC_CUDA_TRY(cudaGetLastError());
    }
    return KFAC_OK;
}

kfac_status bn_precond_launch(const std::vector<BnJob> &jobs, int n, int full, double lambda, double *ws,
                              int64_t ws_bytes, cudaStream_t st) {
    const int64_t gsmem = (int64_t)n * (kGramCols + 1) * 8 + kGramCols * 8;
    const int64_t ssmem = (n > kBnSmemSamples ? 0 : (int64_t)n * n * 8) + (int64_t)n * 8;
    if (full) {
        KFAC_CUDA_TRY(cudaFuncSetAttribute(bn_gram_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)gsmem));
        KFAC_CUDA_TRY(cudaFuncSetAttribute(bn_solve_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)ssmem));
    }
    for (size_t j0 = 0; j0 < jobs.size(); j0 += kBnMax) {
        thread_local BnPrecParams P;
        P.nl = (int)std::min<size_t>(kBnMax, jobs.size() - j0);
        P.n = n;
        P.lambda = lambda;
        P.ws = ws;
        int32_t items = 0, cmax = 0;
        std::vector<int> cs;
        for (int k = 0; k < P.nl; k++) {
            const BnJob &b = jobs[j0 + k];
            P.S[k] = b.S;
            P.grad[k] = b.grad;
            P.out[k] = b.out;
            P.c[k] = b.c;
            P.item0[k] = items;
            items += (int32_t)gram_items(b.c);
            cmax = std::max(cmax, b.c);
            cs.push_back(b.c);
        }
        P.item0[P.nl] = items;
        if (!full) {
            bn_diag_kernel<<<dim3((2 * cmax + kBnThreads - 1) / kBnThreads, P.nl), kBnThreads, 0, st>>>(P);
            KFAC_LAUNCHED();
            KFAC_CUDA_TRY(cudaGetLastError());
            continue;
        }
        if (!ws || bn_ws_bytes(cs, n) > ws_bytes)
            return set_error(KFAC_ERR_ARG, "kfac_bn_precondition: full mode needs kfac_bn_ws_bytes of workspace");
        P.y = ws + (bn_ws_bytes(cs, n) / 8 - (int64_t)P.nl * n);
        P.kglob = n > kBnSmemSamples ? P.y - (int64_t)P.nl * n * n : nullptr;
        bn_gram_kernel<<<items, kBnThreads, gsmem, st>>>(P);
        KFAC_LAUNCHED();
        KFAC_CUDA_TRY(cudaGetLastError());
        bn_solve_kernel<<<P.nl, kBnThreads, ssmem, st>>>(P);
        KFAC_LAUNCHED();
        KFAC_CUDA_TRY(cudaGetLastError());
        bn_out_kernel<<<dim3((2 * cmax + kBnThreads - 1) / kBnThreads, P.nl), kBnThreads, 0, st>>>(P);
        KFAC_LAUNCHED();
        KFAC_CUDA_TRY(cudaGetLastError());
    }
    return KFAC_OK;
}

}  // namespace kfac
