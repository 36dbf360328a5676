// inverse.cu -- stage 4 of distributed K-FAC: factored
// Tikhonov damping (reading R-1) and the inverses A_d^-1, G_d^-1
// of every owned layer (P:247-260 Eq. inv_fim), batched over all owned
// matrices in every launch.
//
// Arithmetic: fp64 (reading R-12: fp32 Cholesky misses the 1e-5 bound on the
// rank-deficient ReLU factors of the paper's workload, kappa ~ 1e3..1e4).
//
// Algorithm: block symmetric Gauss-Jordan ("sweep") on the upper triangle,
// block size B = 128.  For pivot block K of M (symmetric, upper storage),
// with P = M_KK^-1 and R = M_K,: the current block row:
//     M_IJ <- M_IJ - R_I^T (P R_J)     I, J != K
//     M_KJ <- P R_J                     J != K
//     M_KK <- -P
// After sweeping every block, M holds -M^-1.  The sweep pivots are the LDL^T
// pivots, so a non-positive pivot at index j means M is not positive
// definite; its index (+1) is reported like the oracle's Cholesky status.
// Per step: pivot (one CTA per matrix, in-smem scalar sweep of the 128x128
// block), panel (P R as 128x128x128 tile products), update (rank-128 update
// of every upper tile) -- all n^3 flops are in the tile products, which run
// as fp64 DFMA tiles of 128x128 with 8x8 register blocking.
#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>

#include "kfac_internal.hpp"

namespace kfac {

constexpr int kMaxMats = 128;
constexpr int B = kPanel;     // 128
constexpr int KC = 16;        // K rows per smem chunk of the tile product
constexpr int kPivSmem = (B * (B + 1) + 2 * 32 * (B + 4) + 32 * 32) * 8 + 64;
constexpr int kTileSmem = 2 * 2 * KC * (B + 4) * 8;  // double-buffered A/B chunks (padded rows): 66 KB
constexpr int kUpdSmem = kPivSmem > kTileSmem + B * (B + 4) * 8 ? kPivSmem : kTileSmem + B * (B + 4) * 8;
constexpr int kPanelSmem = B * (B + 1) * 8 > kTileSmem ? B * (B + 1) * 8 : kTileSmem;

struct MatDesc {
    const float *packed;
    float *inv;
    double *work;
    double *panel;  // [R: B x ld][Wp: B x ld][P_even: B x B][P_odd: B x B]
    int32_t *status;
    int32_t n, ld, pair, is_A, tile_begin, col_begin, piv_idx, pad_;
};
struct InvParams {
    int32_t nm, total_tiles, k, total_cols, fuse, npiv;
    double gamma;
    double *pair_scratch;  // [npairs][4]: pi, dA, dG
    int *counter;          // this step's tile counter (zeroed per inverse call)
    float *pi_out;
    MatDesc m[kMaxMats];
};

__device__ __forceinline__ int64_t poff(int64_t i, int64_t j, int64_t n) {  // packed upper (i <= j)
    return i * n - i * (i - 1) / 2 + (j - i);
}

// DMMA (mma.sync m8n8k4 f64) 128 x 128 tile fragment mapping: warp w owns rows
// 64*(w>>2) + [0, 64) and columns 32*(w&3) + [0, 32) as 8 x 4 m8n8 blocks.
constexpr int SLD = B + 4;
__device__ __forceinline__ int tile_row(int p) {
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    return 64 * (w >> 2) + 8 * p + (lane >> 2);
}
__device__ __forceinline__ int tile_col(int q) {
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    return 32 * (w & 3) + 8 * (q >> 1) + 2 * (lane & 3) + (q & 1);
}
__device__ __forceinline__ void dmma(double &c0, double &c1, double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                 : "+d"(c0), "+d"(c1)
                 : "d"(a), "d"(b));
}

// ---- prologue: traces -> pi and the damping of each (A, G) pair
__global__ void damp_trace_kernel(const __grid_constant__ InvParams P) {
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
        double *dst = m.work + i * m.ld;
        for (int64_t j = i + threadIdx.x; j < n; j += blockDim.x) {
            double v = (double)src[j - i];
            if (j == i) v += add;
            dst[j] = v;
        }
    }
}

// ---- P = M_KK^-1 for the 128 x 128 diagonal block, in shared memory (full symmetric copy S).
// The block is itself swept in 4 sub-blocks of 32: the 32 x 32 sub-pivot is inverted by a
// scalar sweep in shared memory, then all 256 threads apply the rank-32 sweep update
//   S_IJ -= O_I^T W_J,  S_sJ = W_J,  S_Is = W_I^T,  S_ss = -Q   (O = old block row s, W = Q O).
// Returns 0 or the failing pivot index + 1 (the sweep pivots are the LDL^T pivots).
constexpr int S2 = 32;  // sub-pivot size

// scalar sweep of the 32 x 32 sub-pivot (smem, row-major, ping-pong buffers Q / Q2) by all 256
// threads (4 elements each), one barrier per pivot; the result -inv(sub-pivot) ends in Q (an even
// number of swaps).  Returns 0 or the failing pivot index + 1 (base-relative).
__device__ __forceinline__ int block_sweep32(double *Q, double *Q2, int base) {
    const int tid = threadIdx.x;
    double *src = Q, *dst = Q2;
    for (int t = 0; t < S2; t++) {
        const double d = src[t * S2 + t];
        if (!(d > 0.0)) return base + t + 1;  // uniform: every thread read the same d
        const double inv = __drcp_rn(d);
#pragma unroll
        for (int k = 0; k < 4; k++) {
            const int e = tid + 256 * k, l = e >> 5, j = e & 31;
            const double u = (l == t) ? -1.0 : src[l * S2 + t];
            const double v = (j == t) ? -inv : src[t * S2 + j] * inv;
            const double keep = (l == t || j == t) ? 0.0 : src[e];
            dst[e] = fma(-u, v, keep);
        }
        __syncthreads();
        double *tmp = src;
        src = dst;
        dst = tmp;
    }
    return 0;
}
static_assert(S2 % 2 == 0, "block_sweep32 leaves its result in Q after an even number of swaps");

#ifdef PIVOT_DBG
__device__ int g_pivot_dbg;
__device__ long long g_pclk[64];
#define PCLK(k) if (threadIdx.x == 0) g_pclk[k] = clock64();
#else
#define PCLK(k)
#endif
__device__ int pivot_block(const double *__restrict__ W, int64_t ld, int k0, int bk, double *__restrict__ Pout,
                           double *smem) {
    double(*S)[B + 1] = reinterpret_cast<double(*)[B + 1]>(smem);
    double *O = smem + B * (B + 1);       // [S2][SLD] old block row
    double *Wr = O + S2 * SLD;            // [S2][SLD] Q * O
    double *Q = Wr + S2 * SLD;            // [S2][S2] inverse of the sub-pivot
    int *fsh = reinterpret_cast<int *>(Q + S2 * S2);
    const int tid = threadIdx.x;
    for (int e = tid; e < B * B; e += blockDim.x) {
        const int i = e >> 7, j = e & (B - 1);
        double val = (i == j) ? 1.0 : 0.0;  // identity padding keeps the sweep well defined
        if (i < bk && j < bk) val = W[(int64_t)(k0 + min(i, j)) * ld + (k0 + max(i, j))];
        S[i][j] = val;
    }
    if (tid == 0) *fsh = 0;
    __syncthreads();
    PCLK(0)
    for (int sb = 0; sb < B / S2; sb++) {
        const int s0 = sb * S2;
        if (s0 >= bk) break;
        for (int e = tid; e < S2 * S2; e += blockDim.x) Q[e] = S[s0 + (e >> 5)][s0 + (e & 31)];
        __syncthreads();
        {
            const int f = block_sweep32(Q, Wr, k0 + s0);  // Q <- -inv(sub-pivot) (Wr: ping-pong scratch)
            if (f && tid == 0) *fsh = f;
            for (int e = tid; e < S2 * S2; e += blockDim.x) Q[e] = -Q[e];
        }
        PCLK(1 + 4 * sb)
        for (int e = tid; e < S2 * B; e += blockDim.x) O[(e >> 7) * SLD + (e & (B - 1))] = S[s0 + (e >> 7)][e & (B - 1)];
        __syncthreads();
        if (*fsh) break;
        PCLK(2 + 4 * sb)
#ifdef PIVOT_DBG
        if (g_pivot_dbg == 1 && sb >= 1) break;
#endif
        // W = Q O  (32 x 128): thread -> column j = tid & 127, rows a = (tid >> 7) + 2k (16 chains)
        {
            const int j = tid & (B - 1), a0 = tid >> 7;
            double w[S2 / 2];
#pragma unroll
            for (int k = 0; k < S2 / 2; k++) w[k] = 0.0;
            for (int b2 = 0; b2 < S2; b2++) {
                const double o = O[b2 * SLD + j];
#pragma unroll
                for (int k = 0; k < S2 / 2; k++) w[k] = fma(Q[(a0 + 2 * k) * S2 + b2], o, w[k]);
            }
#pragma unroll
            for (int k = 0; k < S2 / 2; k++) Wr[(a0 + 2 * k) * SLD + j] = w[k];
        }
        __syncthreads();
        PCLK(3 + 4 * sb)
#ifdef PIVOT_DBG
        if (g_pivot_dbg == 2 && sb >= 1) break;
#endif
        // rank-32 sweep update of every element on the fp64 tensor cores (DMMA); each thread then
        // writes only its own elements
        double acc[8][8];
#pragma unroll
        for (int p = 0; p < 8; p++)
#pragma unroll
            for (int q = 0; q < 8; q++) acc[p][q] = 0.0;
        {
            const int w = tid >> 5, lane = tid & 31;
            const int arow = 64 * (w >> 2) + (lane >> 2), bcol = 32 * (w & 3) + (lane >> 2), kl = lane & 3;
#pragma unroll
            for (int kk = 0; kk < S2 / 4; kk++) {
                const int t = kk * 4 + kl;
                double a[8], b[4];
#pragma unroll
                for (int p = 0; p < 8; p++) a[p] = O[t * SLD + arow + 8 * p];
#pragma unroll
                for (int q = 0; q < 4; q++) b[q] = Wr[t * SLD + bcol + 8 * q];
#pragma unroll
                for (int p = 0; p < 8; p++)
#pragma unroll
                    for (int q = 0; q < 4; q++) dmma(acc[p][2 * q], acc[p][2 * q + 1], a[p], b[q]);
            }
        }
#pragma unroll
        for (int p = 0; p < 8; p++) {
            const int i = tile_row(p);
            const bool is = (i >= s0 && i < s0 + S2);
#pragma unroll
            for (int q = 0; q < 8; q++) {
                const int j = tile_col(q);
                const bool js = (j >= s0 && j < s0 + S2);
                // clamped indices: every load is in range whatever the compiler speculates
                const int ii = min(max(i - s0, 0), S2 - 1), jj = min(max(j - s0, 0), S2 - 1);
                const double vq = Q[ii * S2 + jj], vwi = Wr[ii * SLD + j], vwj = Wr[jj * SLD + i];
                const double v = is ? (js ? -vq : vwi) : (js ? vwj : S[i][j] - acc[p][q]);
                S[i][j] = v;
            }
        }
        __syncthreads();
    }
    PCLK(20)
    const int fail = *fsh;
    if (fail) return fail;
    for (int e = tid; e < B * B; e += blockDim.x) {  // P = -S (zero outside bk)
        const int i = e >> 7, j = e & (B - 1);
        Pout[e] = (i < bk && j < bk) ? -S[i][j] : 0.0;
    }
    return 0;
}

__device__ __forceinline__ double *pivot_slot(const MatDesc &m, int k) {
    return m.panel + 2 * (int64_t)B * m.ld + (int64_t)(k & 1) * B * B;
}

// step 0 only: P_0 (later pivots are fused into the previous step's update kernel)
__global__ void __launch_bounds__(256, 1) pivot_kernel(const __grid_constant__ InvParams P) {
    const MatDesc &m = P.m[blockIdx.x];
    const int n = m.n, k0 = P.k * B;
    if (k0 >= n || *m.status != 0) return;
    extern __shared__ double dyn[];
    const int f = pivot_block(m.work, m.ld, k0, min(B, n - k0), pivot_slot(m, P.k), dyn);
    if (f && threadIdx.x == 0) *m.status = f;
}

__device__ __forceinline__ void cp_async16(void *dst, const void *src, bool ok) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"((uint32_t)__cvta_generic_to_shared(dst)),
                 "l"(src), "r"(ok ? 16 : 0)
                 : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_1() { asm volatile("cp.async.wait_group 1;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_0() { asm volatile("cp.async.wait_group 0;" ::: "memory"); }

// acc += sum_{t < kt} A[t][i] * Bm[t][j] for the 128 x 128 tile on the fp64 tensor cores
// (mma.sync m8n8k4 f64, DMMA: 256 FMAs per warp instruction).  Warp w owns rows
// 64*(w>>2) + [0, 64) and columns 32*(w&3) + [0, 32) as 8 x 4 m8n8 blocks; acc[p][q] is the
// element (tile_row(p), tile_col(q)) below.  A and Bm are row-major with 16-aligned leading
// dimensions; columns >= acols / bcols and rows >= kt read as zero.  Chunks of KC rows are
// double-buffered with cp.async; shared rows are padded to 132 doubles (conflict-free fragments).
struct NoExtra {
    __device__ __forceinline__ void operator()(int, int) const {}
};
template <typename Extra = NoExtra>
__device__ __forceinline__ void tile_product(const double *__restrict__ A, int64_t lda, int acols,
                                             const double *__restrict__ Bm, int64_t ldb, int bcols, int kt,
                                             double (&acc)[8][8], double *smem, Extra extra = Extra()) {
    double *As = smem, *Bs = smem + 2 * KC * SLD;
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int arow = 64 * (w >> 2) + (lane >> 2), bcol = 32 * (w & 3) + (lane >> 2), kl = lane & 3;
    const int nchunks = (kt + KC - 1) / KC;
    auto load = [&](int c, int buf) {
        const int t0 = c * KC;
        for (int e = threadIdx.x; e < KC * B / 2; e += 256) {  // pairs of doubles
            const int t = e >> 6, i = (e & 63) * 2;
            const bool okr = t0 + t < kt;
            const bool oka = okr && i < acols, okb = okr && i < bcols;
            cp_async16(As + buf * KC * SLD + t * SLD + i, oka ? A + (int64_t)(t0 + t) * lda + i : A, oka);
            cp_async16(Bs + buf * KC * SLD + t * SLD + i, okb ? Bm + (int64_t)(t0 + t) * ldb + i : Bm, okb);
        }
        extra(c, nchunks);  // e.g. a slice of the C tile, in the same cp.async group
        cp_async_commit();
    };
    load(0, 0);
    for (int c = 0; c < nchunks; c++) {
        const int buf = c & 1;
        if (c + 1 < nchunks) {
            load(c + 1, buf ^ 1);
            cp_async_wait_1();
        } else {
            cp_async_wait_0();
        }
        __syncthreads();
        const double *as = As + buf * KC * SLD, *bs = Bs + buf * KC * SLD;
#pragma unroll
        for (int kk = 0; kk < KC / 4; kk++) {
            const int t = kk * 4 + kl;
            double a[8], b[4];
#pragma unroll
            for (int p = 0; p < 8; p++) a[p] = as[t * SLD + arow + 8 * p];
#pragma unroll
            for (int q = 0; q < 4; q++) b[q] = bs[t * SLD + bcol + 8 * q];
#pragma unroll
            for (int p = 0; p < 8; p++)
#pragma unroll
                for (int q = 0; q < 4; q++) dmma(acc[p][2 * q], acc[p][2 * q + 1], a[p], b[q]);
        }
        __syncthreads();
    }
}

// ---- step 2: R_J = block row K (from upper storage), Wp_J = P R_J   (one CTA per 128-col block)
__global__ void __launch_bounds__(256, 1) panel_kernel(const __grid_constant__ InvParams P) {
    int cb = blockIdx.x, mi = 0;
    while (mi + 1 < P.nm && P.m[mi + 1].col_begin <= cb) mi++;
    const MatDesc &m = P.m[mi];
    const int n = m.n, k0 = P.k * B;
    const int64_t ld = m.ld;
    if (k0 >= n || *m.status != 0) return;
    const int J = cb - m.col_begin, K = P.k;
    const int j0 = J * B;
    if (j0 >= n) return;
    const int bk = min(B, n - k0), bj = min(B, n - j0);
    double *R = m.panel, *Wp = m.panel + (int64_t)B * ld;
    // R_J (rows t < bk, cols j < bj; zero up to the 16-aligned ld) staged through shared memory so
    // that both the read of W (upper storage, possibly transposed) and the write of R coalesce.
    extern __shared__ double dyn[];
    double(*T)[B + 1] = reinterpret_cast<double(*)[B + 1]>(dyn);
    const int bjp = min(B, (int)ld - j0);
    const bool trans = J < K;  // block row K left of the diagonal lives in column K of the upper storage
    const int r0 = trans ? j0 : k0, c0 = trans ? k0 : j0, nr = trans ? bj : bk, nc = trans ? bk : bj;
    for (int e = threadIdx.x; e < B * B; e += blockDim.x) {
        const int r = e >> 7, c = e & (B - 1);
        T[r][c] = (r < nr && c < nc && (J != K || c >= r)) ? m.work[(int64_t)(r0 + r) * ld + c0 + c] : 0.0;
    }
    __syncthreads();
    for (int e = threadIdx.x; e < bk * B; e += blockDim.x) {
        const int t = e >> 7, j = e & (B - 1);
        if (j >= bjp) continue;
        double v;
        if (trans) v = T[j][t];
        else if (J == K) v = (j >= t) ? T[t][j] : T[j][t];
        else v = T[t][j];
        R[(int64_t)t * ld + j0 + j] = v;
    }
    __threadfence_block();
    __syncthreads();
    double acc[8][8];
#pragma unroll
    for (int p = 0; p < 8; p++)
#pragma unroll
        for (int q = 0; q < 8; q++) acc[p][q] = 0.0;
    // Wp[i][j] = sum_t P[t][i] R[t][j]   (P symmetric, zero outside bk)
    tile_product(pivot_slot(m, P.k), B, bk, R + j0, ld, bj, bk, acc, dyn);
#pragma unroll
    for (int p = 0; p < 8; p++) {
        const int i = tile_row(p);
        if (i >= bk) continue;
#pragma unroll
        for (int q = 0; q < 8; q++) {
            const int j = tile_col(q);
            if (j < bjp) Wp[(int64_t)i * ld + j0 + j] = acc[p][q];
        }
    }
}

// ---- step 3: rank-B update of every upper tile (I, J); the CTA of tile (K+1, K+1) then
// inverts that block: the next step's pivot runs concurrently with this step's update.
// Global tile order: first every matrix's (K+1, K+1) tile (so the fused pivots start at once),
// then the remaining upper tiles matrix by matrix, row-major.  Persistent CTAs stride over it.
__device__ __forceinline__ void update_tile(const InvParams &P, int g, double *dyn, const int *sbeg,
                                            const int *spiv) {
    int mi = 0, t = 0;
    if (g < P.npiv) {
        while (spiv[mi] != g) mi++;
    } else {  // binary search of the (shared-memory copy of the) tile prefix
        int lo = 0, hi = P.nm - 1;
        while (lo < hi) {
            const int mid = (lo + hi + 1) >> 1;
            if (sbeg[mid] <= g) lo = mid; else hi = mid - 1;
        }
        mi = lo;
        t = g - sbeg[mi] + (spiv[mi] >= 0 ? 1 : 0);
    }
    const MatDesc &m = P.m[mi];
    const int n = m.n, k0 = P.k * B;
    const int64_t ld = m.ld;
    if (k0 >= n || *m.status != 0) return;
    const int nt = (n + B - 1) / B, K = P.k;
    const int ntiles = nt * (nt + 1) / 2;
    if (t >= ntiles) return;
    int I = 0, J = 0;
    if (K + 1 < nt) {
        const int dk = (K + 1) * nt - (K + 1) * K / 2;  // row-major index of (K+1, K+1)
        t = (t == 0) ? dk : (t <= dk ? t - 1 : t);
    }
    while (t >= nt - I) {
        t -= nt - I;
        I++;
    }
    J = I + t;
    const int bk = min(B, n - k0);
    const int i0 = I * B, j0 = J * B;
    const int bi = min(B, n - i0), bj = min(B, n - j0);
    const double *R = m.panel, *Wp = m.panel + (int64_t)B * ld;
    double *W = m.work;
    if (I == K && J == K) {
        const double *Pm = pivot_slot(m, K);
        for (int e = threadIdx.x; e < bk * bk; e += blockDim.x) {
            const int i = e / bk, j = e % bk;
            if (j >= i) W[(int64_t)(k0 + i) * ld + k0 + j] = -Pm[i * B + j];
        }
        return;
    }
    if (I == K) {  // M_KJ <- Wp_J
        for (int e = threadIdx.x; e < bk * bj; e += blockDim.x) {
            const int i = e / bj, j = e % bj;
            W[(int64_t)(k0 + i) * ld + j0 + j] = Wp[(int64_t)i * ld + j0 + j];
        }
        return;
    }
    if (J == K) {  // M_IK <- Wp_I^T
        for (int e = threadIdx.x; e < bi * bk; e += blockDim.x) {
            const int i = e / bk, j = e % bk;
            W[(int64_t)(i0 + i) * ld + k0 + j] = Wp[(int64_t)j * ld + i0 + i];
        }
        return;
    }
    double acc[8][8];
#pragma unroll
    for (int p = 0; p < 8; p++)
#pragma unroll
        for (int q = 0; q < 8; q++) acc[p][q] = 0.0;
    // the C tile M_IJ streams into shared memory in slices, one per K chunk of the product
    // (its HBM latency hides behind the tensor-core work instead of preceding it)
    double *Cs = dyn + kTileSmem / 8;
    auto cslice = [&](int c, int nch) {
        const int r0 = c * B / nch, r1 = (c + 1) * B / nch;  // rows of this slice
        for (int e = threadIdx.x; e < (r1 - r0) * (B / 2); e += 256) {
            const int i = r0 + e / (B / 2), j = (e % (B / 2)) * 2;
            const bool ok = i < bi && j < bj;
            cp_async16(Cs + i * SLD + j, ok ? W + (int64_t)(i0 + i) * ld + j0 + j : W, ok);
        }
    };
    // M_IJ -= R_I^T Wp_J : acc[i][j] = sum_t R[t][i0+i] Wp[t][j0+j]
    tile_product(R + i0, ld, bi, Wp + j0, ld, bj, bk, acc, dyn, cslice);
#pragma unroll
    for (int p = 0; p < 8; p++) {
        const int i = tile_row(p);
        if (i >= bi) continue;
#pragma unroll
        for (int q = 0; q < 8; q++) {
            const int j = tile_col(q);
            if (j >= bj || (I == J && j < i)) continue;
            W[(int64_t)(i0 + i) * ld + j0 + j] = Cs[i * SLD + j] - acc[p][q];  // padded rows: conflict-free
        }
    }
    if (P.fuse && I == K + 1 && J == K + 1) {  // fused next pivot: P_{K+1} = (updated M_{K+1,K+1})^-1
        __threadfence_block();
        __syncthreads();
        const int f = pivot_block(W, ld, i0, bi, pivot_slot(m, K + 1), dyn);
        if (f && threadIdx.x == 0) *m.status = f;
    }
}

// persistent CTAs take tiles from an atomic counter: the CTA that runs a fused pivot simply takes
// fewer tiles, so the pivot hides behind the other CTAs' updates
__global__ void __launch_bounds__(256, 1) update_kernel(const __grid_constant__ InvParams P) {
    extern __shared__ double dyn[];
    __shared__ int next;
    __shared__ int sbeg[kMaxMats], spiv[kMaxMats];  // decode tables (dynamic param indexing is slow)
    for (int i = threadIdx.x; i < P.nm; i += blockDim.x) {
        sbeg[i] = P.m[i].tile_begin;
        spiv[i] = P.m[i].piv_idx;
    }
    for (;;) {
        __syncthreads();  // the previous tile's epilogue / pivot is done with shared memory and `next`
        if (threadIdx.x == 0) next = atomicAdd(P.counter, 1);
        __syncthreads();
        const int g = next;
        if (g >= P.total_tiles) break;
        update_tile(P, g, dyn, sbeg, spiv);
    }
}

// ---- epilogue: inv = -M (symmetric, full fp32) from the upper storage, 32 x 32 tiles through
// shared memory so that the mirrored (lower) half is read and written coalesced
__global__ void __launch_bounds__(256) finalize_kernel(const __grid_constant__ InvParams P) {
    const MatDesc &m = P.m[blockIdx.y];
    const int n = m.n;
    const int64_t ld = m.ld;
    const int nt = (n + 31) / 32;
    __shared__ double T[32][33];
    const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
    for (int t = blockIdx.x; t < nt * nt; t += gridDim.x) {
        const int bi = t / nt, bj = t - bi * nt;
        const int si = min(bi, bj) * 32, sj = max(bi, bj) * 32;  // source tile in the upper storage
        __syncthreads();
        for (int r = ty; r < 32; r += 8) {
            const int i = si + r, j = sj + tx;
            T[r][tx] = (i < n && j < n) ? m.work[(int64_t)i * ld + j] : 0.0;
        }
        __syncthreads();
        for (int r = ty; r < 32; r += 8) {
            const int i = bi * 32 + r, j = bj * 32 + tx;
            if (i >= n || j >= n) continue;
            double v;
            if (bi < bj) v = T[r][tx];
            else if (bi > bj) v = T[tx][r];
            else v = (r <= tx) ? T[r][tx] : T[tx][r];
            m.inv[(int64_t)i * n + j] = (float)(-v);
        }
    }
}

static int g_inv_sms = 0;

int64_t inverse_ld(int n) { return (n + 15) / 16 * 16; }
int64_t inverse_ws_doubles(int n) {
    const int64_t ld = inverse_ld(n);
    return (n * ld + 2 * (int64_t)B * ld + 2 * (int64_t)B * B + 31) / 32 * 32;
}

kfac_status inverse_launch(const std::vector<InvMat> &mats, int npairs, float gamma, double *pair_scratch,
                           float *pi_out, cudaStream_t st) {
    if (mats.empty()) return KFAC_OK;
    if ((int)mats.size() > kMaxMats) return set_error(KFAC_ERR_UNSUPPORTED, "too many owned matrices for one launch");
    static bool attr = false;
    if (!g_inv_sms) {
        int dev = 0;
        KFAC_CUDA_TRY(cudaGetDevice(&dev));
        KFAC_CUDA_TRY(cudaDeviceGetAttribute(&g_inv_sms, cudaDevAttrMultiProcessorCount, dev));
    }
    if (!attr) {
        KFAC_CUDA_TRY(cudaFuncSetAttribute(pivot_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kPivSmem));
        KFAC_CUDA_TRY(cudaFuncSetAttribute(panel_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kPanelSmem));
        KFAC_CUDA_TRY(cudaFuncSetAttribute(update_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kUpdSmem));
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
        d.ld = (int)inverse_ld(d.n);
        d.pair = mats[i].pair;
        d.is_A = mats[i].is_A;
        maxn = std::max(maxn, d.n);
    }
    damp_trace_kernel<<<P.nm, 256, 0, st>>>(P);
    KFAC_LAUNCHED();
    KFAC_CUDA_TRY(cudaGetLastError());
    unpack_damp_kernel<<<dim3(std::min(maxn, 1024), P.nm), 256, 0, st>>>(P);
    KFAC_LAUNCHED();
    KFAC_CUDA_TRY(cudaGetLastError());
    const int steps = (maxn + B - 1) / B;
    const int fuse = getenv("KFAC_INV_NOFUSE") ? 0 : 1;
    // per-step tile counters live in the scratch after the pair data (plan reserves 1 KB)
    int *counters = reinterpret_cast<int *>(pair_scratch + ((4 * (int64_t)npairs + 15) / 16) * 16);
    if (steps > 256) return set_error(KFAC_ERR_UNSUPPORTED, "inverse: matrix too large for the step counters");
    KFAC_CUDA_TRY(cudaMemsetAsync(counters, 0, steps * sizeof(int), st));
    for (int k = 0; k < steps; k++) {
        // active matrices only (n > k*B), with their upper-tile and column-block prefixes
        InvParams Q;
        memset(&Q, 0, offsetof(InvParams, m));
        Q.gamma = P.gamma;
        Q.k = k;
        int nm = 0, tiles = 0, cols = 0, npiv = 0;
        for (int i = 0; i < P.nm; i++) {
            if (P.m[i].n <= k * B) continue;
            Q.m[nm] = P.m[i];
            const int nt = (P.m[i].n + B - 1) / B;
            Q.m[nm].piv_idx = (fuse && k + 1 < nt) ? npiv++ : -1;
            Q.m[nm].col_begin = cols;
            cols += nt;
            nm++;
        }
        tiles = npiv;
        for (int i = 0; i < nm; i++) {
            const int nt = (Q.m[i].n + B - 1) / B;
            Q.m[i].tile_begin = tiles;
            tiles += nt * (nt + 1) / 2 - (Q.m[i].piv_idx >= 0 ? 1 : 0);
        }
        Q.npiv = npiv;
        Q.counter = counters + k;
        Q.nm = nm;
        Q.total_tiles = tiles;
        Q.total_cols = cols;
        Q.fuse = fuse;
        if (k == 0 || !fuse) {
            pivot_kernel<<<nm, 256, kPivSmem, st>>>(Q);
            KFAC_LAUNCHED();
            KFAC_CUDA_TRY(cudaGetLastError());
        }
        panel_kernel<<<cols, 256, kPanelSmem, st>>>(Q);
        KFAC_LAUNCHED();
        KFAC_CUDA_TRY(cudaGetLastError());
        update_kernel<<<std::min(tiles, g_inv_sms), 256, kUpdSmem, st>>>(Q);
        KFAC_LAUNCHED();
        KFAC_CUDA_TRY(cudaGetLastError());
    }
    finalize_kernel<<<dim3(std::min(((maxn + 31) / 32) * ((maxn + 31) / 32), 1184), P.nm), 256, 0, st>>>(P);
    KFAC_LAUNCHED();
    KFAC_CUDA_TRY(cudaGetLastError());
    return KFAC_OK;
}

}  // namespace kfac
