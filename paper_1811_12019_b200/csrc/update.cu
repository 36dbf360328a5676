// update.cu -- the update that follows the AllGather (NEXT-3):
//
//   w^(t+1) = w^(t) - eta * Gpre^(t) + m * (w^(t) - w^(t-1))
//   W      <- sqrt(2 d_out) * W / (||W||_F + eps)                    (Normalizing Weights)
//
// for every layer, with Gpre read from the gathered buffer at the plan's ag_off and the
// bias column (last, R-5) excluded from the rescale (R-21).  HBM-bound elementwise work:
//   update_step_kernel   reads w, w_prev, Gpre; writes w_prev <- w and w <- Eq. paramupdate;
//                        per-block fp64 sum of squares of the non-bias entries (workspace)
//   update_scale_kernel  (rescale only) each block sums its layer's partials in a fixed order
//                        and scales its own range of W (re-read mostly from L2).
// Algorithmic bytes: 20 per weight (three fp32 reads, two fp32 writes).
#include <cmath>

#include "kfac_internal.hpp"

namespace kfac {

namespace {

constexpr int kUpdThreads = 256;
constexpr int64_t kUpdChunk = 8192;  // weights per block
constexpr int kUpdMaxLayers = 160;

struct UpdParams {
    float *w[kUpdMaxLayers];
    float *w_prev[kUpdMaxLayers];
    const float *g[kUpdMaxLayers];
    int64_t count[kUpdMaxLayers];  // dG * dA
    int32_t cols[kUpdMaxLayers];   // dA
    int32_t dout[kUpdMaxLayers];   // dG
    int32_t bias[kUpdMaxLayers];
    int32_t first[kUpdMaxLayers + 1];
    int32_t nlayers;
    float lr, mom, eps;
    int32_t rescale;
    double *part;  // [total blocks]
};

__device__ __forceinline__ int find_layer(const UpdParams &P, int b) {
    int lo = 0, hi = P.nlayers - 1;
    while (lo < hi) {
        const int mid = (lo + hi + 1) >> 1;
        if (P.first[mid] <= b) lo = mid;
        else hi = mid - 1;
    }
    return lo;
}

__device__ __forceinline__ double block_sum(double v, double *sh) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = v;
    __syncthreads();
    double r = 0.0;
    if (threadIdx.x == 0)
        for (int i = 0; i < kUpdThreads / 32; i++) r += sh[i];
    return r;
}

__device__ __forceinline__ float upd1(float w, float wp, float g, float lr, float mom) {
    return w - lr * g + mom * (w - wp);
}

__global__ void __launch_bounds__(kUpdThreads) update_step_kernel(const __grid_constant__ UpdParams P) {
    __shared__ double sh[kUpdThreads / 32];
    const int l = find_layer(P, blockIdx.x);
    const int64_t lo = (int64_t)(blockIdx.x - P.first[l]) * kUpdChunk;
    const int64_t hi = min(lo + kUpdChunk, P.count[l]);
    float *w = P.w[l], *wp = P.w_prev[l];
    const float *g = P.g[l];
    const int cols = P.cols[l];
    const bool bias = P.bias[l] != 0;
    double ss = 0.0;
    const bool vec = ((reinterpret_cast<uintptr_t>(w) | reinterpret_cast<uintptr_t>(wp) |
                       reinterpret_cast<uintptr_t>(g)) & 15) == 0;
    int64_t done = lo;
    if (vec) {
        const int64_t nv = (hi - lo) / 4;
        float4 *w4 = reinterpret_cast<float4 *>(w + lo), *p4 = reinterpret_cast<float4 *>(wp + lo);
        const float4 *g4 = reinterpret_cast<const float4 *>(g + lo);
        for (int64_t i = threadIdx.x; i < nv; i += kUpdThreads) {
            // w_prev and P are touched once: streamed (evict-first), so the fresh w that
            // update_scale_kernel re-reads has the best chance to stay in L2
            const float4 a = w4[i], b = __ldcs(p4 + i), c = __ldcs(g4 + i);
            float4 r;
            r.x = upd1(a.x, b.x, c.x, P.lr, P.mom);
            r.y = upd1(a.y, b.y, c.y, P.lr, P.mom);
            r.z = upd1(a.z, b.z, c.z, P.lr, P.mom);
            r.w = upd1(a.w, b.w, c.w, P.lr, P.mom);
            __stcs(p4 + i, a);
            w4[i] = r;
            if (P.rescale) {
                const float v[4] = {r.x, r.y, r.z, r.w};
                const int e0 = (int)(lo + 4 * i);  // a layer has < 2^31 weights
#pragma unroll
                for (int q = 0; q < 4; q++)
                    if (!bias || (e0 + q) % cols != cols - 1) ss += (double)v[q] * v[q];
            }
        }
        done = lo + nv * 4;
    }
    for (int64_t e = done + threadIdx.x; e < hi; e += kUpdThreads) {
        const float a = w[e];
        const float r = upd1(a, wp[e], g[e], P.lr, P.mom);
        wp[e] = a;
        w[e] = r;
        if (P.rescale && (!bias || (int)e % cols != cols - 1)) ss += (double)r * r;
    }
    if (P.rescale) {
        const double t = block_sum(ss, sh);
        if (threadIdx.x == 0) P.part[blockIdx.x] = t;
    }
}

__global__ void __launch_bounds__(kUpdThreads) update_scale_kernel(const __grid_constant__ UpdParams P) {
    __shared__ double sh[kUpdThreads / 32];
    __shared__ float s_scale;
    const int l = find_layer(P, blockIdx.x);
    const int b0 = P.first[l], nb = P.first[l + 1] - b0;
    double v = 0.0;
    for (int i = threadIdx.x; i < nb; i += kUpdThreads) v += P.part[b0 + i];  // fixed order per thread
    const double t = block_sum(v, sh);
    if (threadIdx.x == 0) s_scale = (float)(sqrt(2.0 * P.dout[l]) / (sqrt(t) + (double)P.eps));
    __syncthreads();
    const float sc = s_scale;
    const int64_t lo = (int64_t)(blockIdx.x - b0) * kUpdChunk;
    const int64_t hi = min(lo + kUpdChunk, P.count[l]);
    float *w = P.w[l];
    const int cols = P.cols[l];
    const bool bias = P.bias[l] != 0;
    if (!bias && (reinterpret_cast<uintptr_t>(w) & 15) == 0) {  // no bias column: float4 sweep
        float4 *w4 = reinterpret_cast<float4 *>(w + lo);
        const int64_t nv = (hi - lo) / 4;
        for (int64_t i = threadIdx.x; i < nv; i += kUpdThreads) {
            float4 a = w4[i];
            a.x *= sc;
            a.y *= sc;
            a.z *= sc;
            a.w *= sc;
            w4[i] = a;
        }
        for (int64_t e = lo + nv * 4 + threadIdx.x; e < hi; e += kUpdThreads) w[e] *= sc;
        return;
    }
    for (int64_t e = lo + threadIdx.x; e < hi; e += kUpdThreads)
        if (!bias || (int)e % cols != cols - 1) w[e] *= sc;
}

}  // namespace

kfac_status update_launch(const std::vector<UpdJob> &jobs, float lr, float mom, int rescale, float eps, double *ws,
                          int64_t ws_bytes, cudaStream_t st) {
    for (size_t j0 = 0; j0 < jobs.size(); j0 += kUpdMaxLayers) {
        thread_local UpdParams P;  // host staging of the parameter block, per calling thread
        P.nlayers = (int)std::min<size_t>(kUpdMaxLayers, jobs.size() - j0);
        int32_t nb = 0;
        for (int k = 0; k < P.nlayers; k++) {
            const UpdJob &u = jobs[j0 + k];
            P.w[k] = u.w;
            P.w_prev[k] = u.w_prev;
            P.g[k] = u.g;
            P.count[k] = (int64_t)u.dG * u.dA;
            P.cols[k] = u.dA;
            P.dout[k] = u.dG;
            P.bias[k] = u.bias;
            P.first[k] = nb;
            nb += (int32_t)((P.count[k] + kUpdChunk - 1) / kUpdChunk);
        }
        P.first[P.nlayers] = nb;
        P.lr = lr;
        P.mom = mom;
        P.eps = eps;
        P.rescale = rescale;
        P.part = ws;
        if (rescale && (int64_t)nb * 8 > ws_bytes)
            return set_error(KFAC_ERR_STATE, "kfac_update: workspace too small for the norm partials");
        update_step_kernel<<<nb, kUpdThreads, 0, st>>>(P);
        KFAC_LAUNCHED();
        KFAC_CUDA_TRY(cudaGetLastError());
        if (rescale) {
            update_scale_kernel<<<nb, kUpdThreads, 0, st>>>(P);
            KFAC_LAUNCHED();
            KFAC_CUDA_TRY(cudaGetLastError());
        }
    }
    return KFAC_OK;
}

}  // namespace kfac
