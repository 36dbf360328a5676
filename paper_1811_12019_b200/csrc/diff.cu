// diff.cu -- the Kronecker-factor change rate of the stale-Fisher study
// (NEXT-1):
//
//     Diff^(t) = ||X^(t) - X^(t-1)||_F / ||X^(t-1)||_F
//
// for every owned A and G factor, read from two packed-upper recv chunks.
// For a symmetric X stored as its packed upper triangle p,
//     ||X||_F^2 = 2 * sum_k p_k^2 - sum_i X_ii^2,
// so the kernel streams each packed segment once (coalesced float4 loads of
// both chunks, fp64 squares) and gathers the n diagonal entries in a separate
// block per matrix.  HBM-bound: 8 B of algorithmic traffic per packed element
// (4 B from each chunk).  Block partials land in the workspace and a second
// launch combines them in a fixed order (run-to-run bit-reproducible).
#include <cmath>

#include "kfac_internal.hpp"

namespace kfac {

namespace {

constexpr int kDiffThreads = 256;
constexpr int64_t kDiffChunk = 32768;  // packed elements per range block (128 KB of each input)
constexpr int kDiffMaxMats = 256;

struct DiffParams {
    const float *cur[kDiffMaxMats];
    const float *prev[kDiffMaxMats];
    double *out[kDiffMaxMats];
    int64_t len[kDiffMaxMats];   // packed length n(n+1)/2
    int32_t n[kDiffMaxMats];
    int32_t first[kDiffMaxMats + 1];  // first block of matrix m: range blocks, then its diagonal block
    int32_t nmats;
    double2 *part;  // [total blocks] (sum (c-p)^2, sum p^2)
};

__device__ __forceinline__ double2 block_sum2(double a, double b, double2 *sh) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        a += __shfl_xor_sync(0xffffffffu, a, o);
        b += __shfl_xor_sync(0xffffffffu, b, o);
    }
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (lane == 0) sh[w] = make_double2(a, b);
    __syncthreads();
    double2 r = make_double2(0.0, 0.0);
    if (threadIdx.x == 0)
        for (int i = 0; i < kDiffThreads / 32; i++) {
            r.x += sh[i].x;
            r.y += sh[i].y;
        }
    return r;
}

__global__ void __launch_bounds__(kDiffThreads) diff_partial_kernel(const __grid_constant__ DiffParams P) {
    __shared__ double2 sh[kDiffThreads / 32];
    // grid-stride over the work items (one resident wave, no wave-quantisation tail); each item
    // still writes its own partial, so the combine order does not depend on the grid
    for (int b = blockIdx.x; b < P.first[P.nmats]; b += gridDim.x) {
        int m = 0, hi_m = P.nmats - 1;  // binary search: the last matrix whose first block <= b
        while (m < hi_m) {
            const int mid = (m + hi_m + 1) >> 1;
            if (P.first[mid] <= b) m = mid;
            else hi_m = mid - 1;
        }
        const float *cur = P.cur[m], *prev = P.prev[m];
        double num = 0.0, den = 0.0;
        const int nrange = P.first[m + 1] - P.first[m] - 1;
        const int rb = b - P.first[m];
        if (rb < nrange) {  // packed range [lo, hi)
            const int64_t lo = (int64_t)rb * kDiffChunk;
            const int64_t hi = min(lo + kDiffChunk, P.len[m]);
            // segments start 16-element aligned in the recv chunk, and so does lo
            const int64_t nv = (hi - lo) / 4;
            const float4 *c4 = reinterpret_cast<const float4 *>(cur + lo);
            const float4 *p4 = reinterpret_cast<const float4 *>(prev + lo);
#pragma unroll 4
            for (int64_t i = threadIdx.x; i < nv; i += kDiffThreads) {
                const float4 c = __ldcs(c4 + i), p = __ldcs(p4 + i);  // streamed once: evict-first
                const double d0 = (double)c.x - p.x, d1 = (double)c.y - p.y, d2 = (double)c.z - p.z,
                             d3 = (double)c.w - p.w;
                num += d0 * d0 + d1 * d1 + d2 * d2 + d3 * d3;
                den += (double)p.x * p.x + (double)p.y * p.y + (double)p.z * p.z + (double)p.w * p.w;
            }
            for (int64_t i = lo + nv * 4 + threadIdx.x; i < hi; i += kDiffThreads) {
                const double d = (double)cur[i] - prev[i];
                num += d * d;
                den += (double)prev[i] * prev[i];
            }
        } else {  // the diagonal: X_ii at i*n - i(i-1)/2
            const int64_t n = P.n[m];
            for (int64_t i = threadIdx.x; i < n; i += kDiffThreads) {
                const int64_t k = i * n - i * (i - 1) / 2;
                const double d = (double)cur[k] - prev[k];
                num += d * d;
                den += (double)prev[k] * prev[k];
            }
        }
        const double2 r = block_sum2(num, den, sh);
        if (threadIdx.x == 0) P.part[b] = r;
        __syncthreads();  // sh is reused by the next item
    }
}

// one warp per matrix: ||.||_F^2 = 2 * (range sum) - (diagonal sum), fixed-order combine
__global__ void diff_final_kernel(const __grid_constant__ DiffParams P) {
    const int m = blockIdx.x * (blockDim.x / 32) + (threadIdx.x >> 5);
    const int lane = threadIdx.x & 31;
    if (m >= P.nmats) return;
    const int b0 = P.first[m], diag = P.first[m + 1] - 1;
    double num = 0.0, den = 0.0;
    for (int b = b0 + lane; b < diag; b += 32) {
        num += P.part[b].x;
        den += P.part[b].y;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        num += __shfl_xor_sync(0xffffffffu, num, o);
        den += __shfl_xor_sync(0xffffffffu, den, o);
    }
    if (lane == 0) {
        const double2 dg = P.part[diag];
        const double fn = 2.0 * num - dg.x, fd = 2.0 * den - dg.y;
        *P.out[m] = fd > 0.0 ? sqrt(fmax(fn, 0.0) / fd) : __longlong_as_double(0x7ff8000000000000LL);  // NaN: missing
    }
}

}  // namespace

kfac_status diff_launch(const std::vector<DiffMat> &mats, double *ws, int64_t ws_bytes, cudaStream_t st) {
    for (size_t b0 = 0; b0 < mats.size(); b0 += kDiffMaxMats) {
        thread_local DiffParams P;  // host staging of the (large) parameter block, per calling thread
        P.nmats = (int)std::min<size_t>(kDiffMaxMats, mats.size() - b0);
        int32_t nb = 0;
        for (int k = 0; k < P.nmats; k++) {
            const DiffMat &d = mats[b0 + k];
            if ((reinterpret_cast<uintptr_t>(d.cur) | reinterpret_cast<uintptr_t>(d.prev)) & 15)
                return set_error(KFAC_ERR_ARG, "kfac_factor_diff: factor segments must be 16-byte aligned");
            P.cur[k] = d.cur;
            P.prev[k] = d.prev;
            P.out[k] = d.out;
            P.n[k] = d.n;
            P.len[k] = packed_len(d.n);
            P.first[k] = nb;
            nb += (int32_t)((P.len[k] + kDiffChunk - 1) / kDiffChunk) + 1;
        }
        P.first[P.nmats] = nb;
        if ((int64_t)nb * (int64_t)sizeof(double2) > ws_bytes)
            return set_error(KFAC_ERR_STATE, "kfac_factor_diff: workspace too small for the block partials");
        P.part = reinterpret_cast<double2 *>(ws);
        int sms = 0, per = 0;
        KFAC_TRY(dev_sm_count(&sms));
        KFAC_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, diff_partial_kernel, kDiffThreads, 0));
        const int grid = sms * std::max(per, 1);
        diff_partial_kernel<<<std::min(nb, grid), kDiffThreads, 0, st>>>(P);
        KFAC_LAUNCHED();
        KFAC_CUDA_TRY(cudaGetLastError());
        diff_final_kernel<<<(P.nmats + 7) / 8, 256, 0, st>>>(P);
        KFAC_LAUNCHED();
        KFAC_CUDA_TRY(cudaGetLastError());
    }
    return KFAC_OK;
}

}  // namespace kfac
