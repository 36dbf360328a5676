// inverse.cu -- stage 4 of distributed K-FAC: factored
// Tikhonov damping (reading R-1) and the inverses A_d^-1, G_d^-1
// of every owned layer (P:247-260 Eq. inv_fim), batched over all owned
// matrices in every launch.
//
// Arithmetic: fp64 (reading R-12: fp32 Cholesky misses the 1e-5 bound on the
// rank-deficient ReLU factors of the paper's workload, kappa ~ 1e3..1e4).
//
// Algorithm: block symmetric Gauss-Jordan ("sweep") on the upper triangle,
// block size b = kPanel = 64.  For pivot block K of M (symmetric, upper
// storage), with P = M_KK^-1 and R = M_K,: the current block row:
//     M_IJ <- M_IJ - R_I^T (P R_J)     I, J != K
//     M_KJ <- P R_J                     J != K
//     M_KK <- -P
// After sweeping every block, M holds -M^-1.  The sweep pivots are the LDL^T
// pivots, so a non-positive pivot at index j means M is not positive
// definite; its index (+1) is reported like the oracle's Cholesky status.
// Each step is three grouped launches (pivot inverse, panel, rank-b update);
// all n^3 flops are in the update, which touches only upper tiles.
#include <algorithm>
#include <cmath>
#include <cstring>

#include "kfac_internal.hpp"

namespace kfac {

constexpr int kMaxMats = 128;
constexpr int B = kPanel;  // 64
constexpr int kPanelSmem = 2 * B * (B + 1) * 8;
constexpr int kUpdateSmem = 2 * B * B * 8;

struct MatDesc {
    const float *packed;
    float *inv;
    double *work;
    double *panel;  // [2][B][n]: R then Wp = P R ; plus P (B*B) after them
    int32_t *status;
    int32_t n, pair, is_A, tile_begin;
};
struct InvParams {
    int32_t nm, total_tiles, k, pad;
    double gamma;
    double *pair_scratch;  // [npairs][4]: pi, dA, dG
    float *pi_out;
    MatDesc m[kMaxMats];
};

__device__ __forceinline__ int64_t poff(int64_t i, int64_t j, int64_t n) {  // packed upper (i <= j)
    return i * n - i * (i - 1) / 2 + (j - i);
}

// ---- prologue: traces -> pi and the damping of each (A, G) pair
__global__ void damp_trace_kernel(const __grid_constant__ InvParams P) {
    // one block per matrix; pair scratch written by the A matrix after both traces are known:
    // we compute both traces in the block of the A matrix (the G matrix block does nothing)
    const MatDesc &ma = P.m[blockIdx.x];
    if (!ma.is_A) return;
    const MatDesc *mg = nullptr;
    for (int k = 0; k < P.nm; k++)
        if (P.m[k].pair == ma.pair && !P.m[k].is_A) mg = &P.m[k];
    __shared__ double red[2][256];
    double ta = 0.0, tg = 0.0;
    for (int i = threadIdx.x; i < ma.n; i += blockDim.x) ta += (double)ma.packed[poff(i, i, ma.n)];
    for (int i = threadIdx.x; i < mg->n; i += blockDim.x) tg += (double)mg->packed[poff(i, i, mg->n)];
    red[0][threadIdx.x] = ta;
    red[1][threadIdx.x] = tg;
    __syncthreads();
    for (int s = blockDim.x / 2; s > 0; s >>= 1) {
        if (threadIdx.x < s) {
            red[0][threadIdx.x] += red[0][threadIdx.x + s];
            red[1][threadIdx.x] += red[1][threadIdx.x + s];
        }
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        ta = red[0][0];
        tg = red[1][0];
        double pi = 1.0;
        if (ta != 0.0 && tg != 0.0) pi = sqrt((ta / ma.n) / (tg / mg->n));
        double sg = sqrt(P.gamma);
        P.pair_scratch[4 * ma.pair + 0] = pi;
        P.pair_scratch[4 * ma.pair + 1] = pi * sg;  // added to A's diagonal
        P.pair_scratch[4 * ma.pair + 2] = sg / pi;  // added to G's diagonal
        if (P.pi_out) P.pi_out[ma.pair] = (float)pi;
        *ma.status = 0;
        *mg->status = 0;
    }
}

// packed fp32 -> fp64 working matrix (upper triangle), damped diagonal
__global__ void unpack_damp_kernel(const __grid_constant__ InvParams P) {
    const MatDesc &m = P.m[blockIdx.y];
    const int64_t n = m.n;
    const double add = P.pair_scratch[4 * m.pair + (m.is_A ? 1 : 2)];
    for (int64_t i = blockIdx.x; i < n; i += gridDim.x) {
        const float *src = m.packed + poff(i, i, n);
        double *dst = m.work + i * n;
        for (int64_t j = i + threadIdx.x; j < n; j += blockDim.x) {
            double v = (double)src[j - i];
            if (j == i) v += add;
            dst[j] = v;
        }
    }
}

// ---- step 1: P = M_KK^-1 by a scalar sweep in shared memory (one block per matrix)
__global__ void __launch_bounds__(256) pivot_kernel(const __grid_constant__ InvParams P) {
    const MatDesc &m = P.m[blockIdx.x];
    const int n = m.n, k0 = P.k * B;
    if (k0 >= n) return;
    if (*m.status != 0) return;  // an earlier pivot already failed
    const int bk = min(B, n - k0);
    __shared__ double S[B][B + 1];
    __shared__ double col[B], row[B];
    __shared__ int fail;
    if (threadIdx.x == 0) fail = 0;
    for (int e = threadIdx.x; e < bk * bk; e += blockDim.x) {
        int i = e / bk, j = e % bk;
        int a = min(i, j), b = max(i, j);
        S[i][j] = m.work[(int64_t)(k0 + a) * n + (k0 + b)];
    }
    __syncthreads();
    for (int t = 0; t < bk; t++) {
        const double d = S[t][t];
        if (!(d > 0.0)) {
            if (threadIdx.x == 0) fail = k0 + t + 1;
            break;
        }
        for (int e = threadIdx.x; e < bk; e += blockDim.x) {
            col[e] = S[e][t];
            row[e] = S[t][e];
        }
        __syncthreads();
        const double inv = 1.0 / d;
        for (int e = threadIdx.x; e < bk * bk; e += blockDim.x) {
            int i = e / bk, j = e % bk;
            double v;
            if (i == t && j == t) v = -inv;
            else if (i == t) v = row[j] * inv;
            else if (j == t) v = col[i] * inv;
            else v = S[i][j] - col[i] * row[j] * inv;
            S[i][j] = v;
        }
        __syncthreads();
    }
    __syncthreads();
    if (fail) {
        if (threadIdx.x == 0) *m.status = fail;
        return;
    }
    // P = -S  stored after the two panels
    double *Pm = m.panel + 2 * (int64_t)B * n;
    for (int e = threadIdx.x; e < bk * bk; e += blockDim.x) Pm[e] = -S[e / bk][e % bk];
}

// ---- step 2: R = block row K (from upper storage), Wp = P R   (64-column blocks)
__global__ void __launch_bounds__(256) panel_kernel(const __grid_constant__ InvParams P) {
    const MatDesc &m = P.m[blockIdx.y];
    const int n = m.n, k0 = P.k * B;
    if (k0 >= n || *m.status != 0) return;
    const int bk = min(B, n - k0);
    const int j0 = blockIdx.x * B;
    if (j0 >= n) return;
    const int bj = min(B, n - j0);
    extern __shared__ double dyn[];
    double (*Ps)[B + 1] = reinterpret_cast<double (*)[B + 1]>(dyn);
    double (*Rs)[B + 1] = reinterpret_cast<double (*)[B + 1]>(dyn + B * (B + 1));
    const double *Pm = m.panel + 2 * (int64_t)B * n;
    for (int e = threadIdx.x; e < bk * bk; e += blockDim.x) Ps[e / bk][e % bk] = Pm[e];
    for (int e = threadIdx.x; e < bk * bj; e += blockDim.x) {
        int i = e / bj, j = e % bj;
        int gi = k0 + i, gj = j0 + j;
        double v = (gi <= gj) ? m.work[(int64_t)gi * n + gj] : m.work[(int64_t)gj * n + gi];
        Rs[i][j] = v;
    }
    __syncthreads();
    double *R = m.panel, *Wp = m.panel + (int64_t)B * n;
    for (int e = threadIdx.x; e < bk * bj; e += blockDim.x) {
        int i = e / bj, j = e % bj;
        double s = 0.0;
        for (int t = 0; t < bk; t++) s += Ps[i][t] * Rs[t][j];
        R[(int64_t)i * n + j0 + j] = Rs[i][j];
        Wp[(int64_t)i * n + j0 + j] = s;
    }
}

// ---- step 3: rank-b update of every upper tile (I, J)
__global__ void __launch_bounds__(256) update_kernel(const __grid_constant__ InvParams P) {
    int tile = blockIdx.x, mi = 0;
    while (mi + 1 < P.nm && P.m[mi + 1].tile_begin <= tile) mi++;
    const MatDesc &m = P.m[mi];
    const int n = m.n, k0 = P.k * B;
    if (k0 >= n || *m.status != 0) return;
    const int nt = (n + B - 1) / B, K = P.k;
    int t = tile - m.tile_begin, I = 0;
    if (t >= nt * (nt + 1) / 2) return;
    while (t >= nt - I) {
        t -= nt - I;
        I++;
    }
    const int J = I + t;
    const int bk = min(B, n - k0);
    const int i0 = I * B, j0 = J * B;
    const int bi = min(B, n - i0), bj = min(B, n - j0);
    const double *R = m.panel, *Wp = m.panel + (int64_t)B * n;
    double *W = m.work;
    if (I == K && J == K) {
        const double *Pm = m.panel + 2 * (int64_t)B * n;
        for (int e = threadIdx.x; e < bk * bk; e += blockDim.x) {
            int i = e / bk, j = e % bk;
            if (j >= i) W[(int64_t)(k0 + i) * n + k0 + j] = -Pm[e];
        }
        return;
    }
    if (I == K) {  // M_KJ <- Wp_J
        for (int e = threadIdx.x; e < bk * bj; e += blockDim.x) {
            int i = e / bj, j = e % bj;
            W[(int64_t)(k0 + i) * n + j0 + j] = Wp[(int64_t)i * n + j0 + j];
        }
        return;
    }
    if (J == K) {  // M_IK <- Wp_I^T
        for (int e = threadIdx.x; e < bi * bk; e += blockDim.x) {
            int i = e / bk, j = e % bk;
            W[(int64_t)(i0 + i) * n + k0 + j] = Wp[(int64_t)j * n + i0 + i];
        }
        return;
    }
    // M_IJ -= R_I^T Wp_J  : 64x64 tile, 256 threads x (4x4)
    extern __shared__ double dyn[];
    double (*Rs)[B] = reinterpret_cast<double (*)[B]>(dyn);          // Rs[k][i] = R[k][i0+i]
    double (*Ws)[B] = reinterpret_cast<double (*)[B]>(dyn + B * B);  // Ws[k][j] = Wp[k][j0+j]
    for (int e = threadIdx.x; e < B * B; e += blockDim.x) {
        int k = e / B, c = e % B;
        Rs[k][c] = (k < bk && c < bi) ? R[(int64_t)k * n + i0 + c] : 0.0;
        Ws[k][c] = (k < bk && c < bj) ? Wp[(int64_t)k * n + j0 + c] : 0.0;
    }
    __syncthreads();
    const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
    double acc[4][4];
#pragma unroll
    for (int a = 0; a < 4; a++)
#pragma unroll
        for (int b = 0; b < 4; b++) acc[a][b] = 0.0;
    for (int k = 0; k < bk; k++) {
        double r[4], w[4];
#pragma unroll
        for (int a = 0; a < 4; a++) r[a] = Rs[k][ty * 4 + a];
#pragma unroll
        for (int b = 0; b < 4; b++) w[b] = Ws[k][tx * 4 + b];
#pragma unroll
        for (int a = 0; a < 4; a++)
#pragma unroll
            for (int b = 0; b < 4; b++) acc[a][b] = fma(r[a], w[b], acc[a][b]);
    }
#pragma unroll
    for (int a = 0; a < 4; a++) {
        int i = ty * 4 + a;
        if (i >= bi) continue;
#pragma unroll
        for (int b = 0; b < 4; b++) {
            int j = tx * 4 + b;
            if (j >= bj) continue;
            if (I == J && j < i) continue;  // diagonal tile: upper part only
            double *p = W + (int64_t)(i0 + i) * n + j0 + j;
            *p = *p - acc[a][b];
        }
    }
}

// ---- epilogue: inv = -M (symmetric, full fp32)
__global__ void finalize_kernel(const __grid_constant__ InvParams P) {
    const MatDesc &m = P.m[blockIdx.y];
    const int64_t n = m.n;
    for (int64_t i = blockIdx.x; i < n; i += gridDim.x)
        for (int64_t j = threadIdx.x; j < n; j += blockDim.x) {
            double v = (i <= j) ? m.work[i * n + j] : m.work[j * n + i];
            m.inv[i * n + j] = (float)(-v);
        }
}

kfac_status inverse_launch(const std::vector<InvMat> &mats, int npairs, float gamma, double *pair_scratch,
                           float *pi_out, cudaStream_t st) {
    if (mats.empty()) return KFAC_OK;
    if ((int)mats.size() > kMaxMats) return set_error(KFAC_ERR_UNSUPPORTED, "too many owned matrices for one launch");
    static bool attr = false;
    if (!attr) {
        KFAC_CUDA_TRY(cudaFuncSetAttribute(panel_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kPanelSmem));
        KFAC_CUDA_TRY(cudaFuncSetAttribute(update_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kUpdateSmem));
        attr = true;
    }
    InvParams P;
    memset(&P, 0, sizeof(P));
    P.nm = (int)mats.size();
    P.gamma = (double)gamma;
    P.pair_scratch = pair_scratch;
    P.pi_out = pi_out;
    int maxn = 0;
    for (size_t i = 0; i < mats.size(); i++) {
        MatDesc &d = P.m[i];
        d.packed = mats[i].packed;
        d.inv = mats[i].inv;
        d.work = mats[i].work;
        d.panel = mats[i].panel;
        d.status = mats[i].status;
        d.n = mats[i].n;
        d.pair = mats[i].pair;
        d.is_A = mats[i].is_A;
        maxn = std::max(maxn, d.n);
    }
    (void)npairs;
    damp_trace_kernel<<<P.nm, 256, 0, st>>>(P);
    KFAC_LAUNCHED();
    KFAC_CUDA_TRY(cudaGetLastError());
    unpack_damp_kernel<<<dim3(std::min(maxn, 1024), P.nm), 256, 0, st>>>(P);
    KFAC_LAUNCHED();
    KFAC_CUDA_TRY(cudaGetLastError());
    const int steps = (maxn + B - 1) / B;
    for (int k = 0; k < steps; k++) {
        // active matrices only (n > k*B), with their upper-tile prefix
        InvParams Q;
        memset(&Q, 0, offsetof(InvParams, m));
        Q.gamma = P.gamma;
        Q.k = k;
        int nm = 0, tiles = 0, maxcols = 0;
        for (int i = 0; i < P.nm; i++) {
            if (P.m[i].n <= k * B) continue;
            Q.m[nm] = P.m[i];
            Q.m[nm].tile_begin = tiles;
            int nt = (P.m[i].n + B - 1) / B;
            tiles += nt * (nt + 1) / 2;
            maxcols = std::max(maxcols, nt);
            nm++;
        }
        Q.nm = nm;
        Q.total_tiles = tiles;
        pivot_kernel<<<nm, 256, 0, st>>>(Q);
        KFAC_LAUNCHED();
        KFAC_CUDA_TRY(cudaGetLastError());
        panel_kernel<<<dim3(maxcols, nm), 256, kPanelSmem, st>>>(Q);
        KFAC_LAUNCHED();
        KFAC_CUDA_TRY(cudaGetLastError());
        update_kernel<<<tiles, 256, kUpdateSmem, st>>>(Q);
        KFAC_LAUNCHED();
        KFAC_CUDA_TRY(cudaGetLastError());
    }
    finalize_kernel<<<dim3(std::min(maxn, 2048), P.nm), 256, 0, st>>>(P);
    KFAC_LAUNCHED();
    KFAC_CUDA_TRY(cudaGetLastError());
    return KFAC_OK;
}

}  // namespace kfac
