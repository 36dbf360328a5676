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
#include <mutex>
#include <type_traits>
#include <cmath>
#include <cstdlib>
#include <cstring>

#include "kfac_internal.hpp"
#include "sm100.cuh"

namespace kfac {

// The persistent inverse kernel runs 8 worker warps (256 threads) and one producer warp (see OZ_*);
// worker-only code synchronises with WSYNC (named barrier 1, 256 threads), __syncthreads is for all.
constexpr int kWorkers = 256, kThreads = 288;
#define WSYNC() asm volatile("bar.sync 1, 256;" ::: "memory")

constexpr int kMaxMats = 128;
constexpr int kUnpRows = 8, kFinTiles = 4, kFinT = 64;  // finalize: 4 tile pairs of 64 x 64 per block
constexpr int kPanelBufs = 4;  // panel buffers per matrix (step mod 4)
constexpr int B = kPanel;     // 128
#ifndef KFAC_INV_KC  // experiment overrides (KFAC_NVCC_EXTRA)
#define KFAC_INV_KC 8
#endif
#ifndef KFAC_INV_STAGES
#define KFAC_INV_STAGES 4
#endif
constexpr int KC = KFAC_INV_KC;  // K rows per shared-memory ring stage of the tile product
constexpr int kStages = KFAC_INV_STAGES;  // ring depth
constexpr int kPivSmem = (B * (B + 1) + 2 * 32 * (B + 4) + 32 * 36 + 64) * 8 + 64;
constexpr int kTileSmem = kStages * 2 * KC * (B + 4) * 8;  // A/B chunk ring (padded rows): 66 KB
constexpr int kUpdSmemDmma = kPivSmem > kTileSmem + B * (B + 4) * 8 ? kPivSmem : kTileSmem + B * (B + 4) * 8;
constexpr int kUpdSmemOz = 2 * (5 * B * B) + 3 * (5 * 32 * B) + 4 * B * 4 + 1024;  // = kOzSmem (int8 updates)
constexpr int kUpdSmem = kUpdSmemDmma > kUpdSmemOz ? kUpdSmemDmma : kUpdSmemOz;
static_assert(kUpdSmem >= B * (B + 1) * 8 + kTileSmem, "panel staging + ring fit the update kernel's shared memory");

struct MatDesc {
    const float *packed;
    float *inv;
    double *work;
    double *panel;  // [R | Wp per step mod kPanelBufs: B x ld each][P_even | P_odd: B x B]
    int32_t *status;
    int32_t n, ld, pair, is_A;
    int32_t nt;          // column blocks
    int32_t col_begin;   // prefix of nt over the (nt-descending) matrix list: column / step flags
    int32_t tile_begin;  // prefix of nt (nt + 1) / 2: tile flags
    int32_t orig;        // index in the caller's matrix list (2 * pair + !is_A): report slot
    const CUtensorMap *tmaps;  // [3] in global memory: the digit tile sets as 4-D TMA maps (OZ_MAP_*)
    float *split;              // [2][n][round4(n)] tf32 hi / lo of the inverse for the precondition, or null
};
enum { OZ_MAP_A = 0, OZ_MAP_R5 = 1, OZ_MAP_R6 = 2 };  // boxes {128 B, 128 rows, 5 digits}, {., 32, 5}, {., 32, 6}
constexpr int kMaxSteps = 128;
struct InvParams {
    int32_t nm, steps, total_tasks, pad0_;
    double gamma;
    double *pair_scratch;  // [npairs][4]: pi, dA, dG
    float *pi_out;         // pi per pair (out; in for a G refresh: the cached pi of the last full refresh)
    int32_t g_only;        // G refresh: G matrices only, damped with the cached pi (R-20)
    int32_t prec_mode;     // inverse precision: KFAC_INV_AUTO / KFAC_INV_FP64 / KFAC_INV_INT8 (kfac.h)
    int32_t *ozflag;       // [nm] per matrix (launch order): 1 = int8-sliced updates, 0 = fp64 DMMA updates
    // dataflow state (zeroed per inverse call): one task counter, then per matrix / column / step
    // stamps and counters -- see inverse_kernel
    int *counter;
    int *pivflag;      // [nm]        k + 1 once P_k is in its slot
    int *colflag;      // [sum nt]    k + 1 once panel (R_J, Wp_J) of step k is written
    int *panels_done;  // [sum nt]    per (matrix, step): completed panel tasks
    int *tiles_done;   // [sum nt]    per (matrix, step): completed update tasks
    int *tileflag;     // [sum tiles] k + 1 once tile (I, J) holds its step-k value
    int4 *tasks;       // [total_tasks] task records (gen_step_tasks), built on the device per call
    int32_t step_begin[kMaxSteps + 1];  // first record of each pair's list (inverse_tasks.hpp)
    // flattened grids of the prologue / epilogue kernels: blocks [unp_begin[r], unp_begin[r+1]) unpack matrix r
    // (kUnpRows rows each), [fin_begin[r], fin_begin[r+1]) finalize it (kFinTiles 32 x 32 tile pairs each)
    int32_t unp_begin[kMaxMats + 1];
    int32_t fin_begin[kMaxMats + 1];
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

// ---- prologue: traces -> pi and the damping of each (A, G) pair, and the per-matrix
// precision of the sweep's updates (reading R-12): the a-priori condition bound
//     kappa(M_d) <= tr(M_d) / delta = (tr(M) + n delta) / delta,   delta = the damping added,
// picks int8-sliced updates (5 balanced 8-bit digits: measured error <= 3e-13 x bound on the
// workload's factors and on rank-deficient ReLU Grams, scripts/ozaki_proto.py) where
// bound <= kOzBound, i.e. a predicted error <= 1e-6 against the 1e-5 tolerance; the others keep
// fp64 DMMA updates.  Pair scratch (8 doubles per pair): pi, A's add,
// G's add, A's bound, G's bound, A's slices, G's slices (0 = fp64), spare.
constexpr double kOzBound = 3e6;
constexpr int kOzS = 5;  // 8-bit digits per operand of an int8-sliced update
__device__ double block_trace(const float *packed, int n, double *red) {
    double t = 0.0;
    for (int i = threadIdx.x; i < n; i += blockDim.x) t += (double)packed[poff(i, i, n)];
    red[threadIdx.x] = t;
    __syncthreads();
    for (int s = blockDim.x / 2; s > 0; s >>= 1) {
        if (threadIdx.x < s) red[threadIdx.x] += red[threadIdx.x + s];
        __syncthreads();
    }
    return red[0];
}
__device__ void decide_precision(const InvParams &P, int mi, double tr, double add) {
    const MatDesc &m = P.m[mi];
    const double bound = add > 0.0 ? (tr + m.n * add) / add : INFINITY;
    const int s = P.prec_mode == KFAC_INV_FP64 ? 0 : (P.prec_mode == KFAC_INV_INT8 ? kOzS : (bound <= kOzBound ? kOzS : 0));
    P.ozflag[mi] = s ? 1 : 0;
    P.pair_scratch[8 * m.pair + (m.is_A ? 3 : 4)] = bound;
    P.pair_scratch[8 * m.pair + (m.is_A ? 5 : 6)] = (double)s;
}
__global__ void damp_trace_kernel(const __grid_constant__ InvParams P) {
    const MatDesc &ma = P.m[blockIdx.x];
    __shared__ double red[256];
    if (!ma.is_A) {
        if (P.g_only) {  // G refresh: G_d = G + sqrt(gamma) / pi_cached I
            const double tg = block_trace(ma.packed, ma.n, red);
            if (threadIdx.x == 0) {
                const double pi = P.pi_out[ma.pair], sg = sqrt(P.gamma);
                P.pair_scratch[8 * ma.pair + 0] = pi;
                P.pair_scratch[8 * ma.pair + 2] = sg / pi;
                decide_precision(P, blockIdx.x, tg, sg / pi);
                *ma.status = 0;
            }
        }
        return;
    }
    int gi = -1;
    for (int k = 0; k < P.nm; k++)
        if (P.m[k].pair == ma.pair && !P.m[k].is_A) gi = k;
    const MatDesc &mg = P.m[gi];
    const double ta = block_trace(ma.packed, ma.n, red);
    __syncthreads();
    const double tg = block_trace(mg.packed, mg.n, red);
    if (threadIdx.x == 0) {
        double pi = 1.0;
        if (ta != 0.0 && tg != 0.0) pi = sqrt((ta / ma.n) / (tg / mg.n));
        double sg = sqrt(P.gamma);
        P.pair_scratch[8 * ma.pair + 0] = pi;
        P.pair_scratch[8 * ma.pair + 1] = pi * sg;  // added to A's diagonal
        P.pair_scratch[8 * ma.pair + 2] = sg / pi;  // added to G's diagonal
        if (P.pi_out) P.pi_out[ma.pair] = (float)pi;
        decide_precision(P, blockIdx.x, ta, pi * sg);
        decide_precision(P, gi, tg, sg / pi);
        *ma.status = 0;
        *mg.status = 0;
    }
}

// packed fp32 -> fp64 working matrix (upper triangle), damped diagonal
// the matrix a block of a flattened grid belongs to (prefix table, binary search; uniform per block)
__device__ __forceinline__ int flat_matrix(const int32_t *begin, int nm, int b) {
    int lo = 0, hi = nm - 1;
    while (lo < hi) {
        const int mid = (lo + hi + 1) >> 1;
        if (begin[mid] <= b) lo = mid;
        else hi = mid - 1;
    }
    return lo;
}
__global__ void unpack_damp_kernel(const __grid_constant__ InvParams P) {
    const int r = flat_matrix(P.unp_begin, P.nm, blockIdx.x);
    const MatDesc &m = P.m[r];
    const int64_t n = m.n;
    const double add = P.pair_scratch[8 * m.pair + (m.is_A ? 1 : 2)];
    const int64_t i0 = (int64_t)(blockIdx.x - P.unp_begin[r]) * kUnpRows;
    for (int64_t i = i0; i < min(n, i0 + kUnpRows); i++) {
        const float *src = m.packed + poff(i, i, n) - i;  // src[j] = packed (i, j)
        double *dst = m.work + i * m.ld;
        // 16-byte stores of element pairs (j even; the work rows are 128-byte aligned), an odd first
        // or last element alone
        const int64_t j0 = i + (i & 1);
        if (threadIdx.x == 0) {
            if (i & 1) dst[i] = (double)src[i] + add;
            if ((n - j0) & 1) dst[n - 1] = (double)src[n - 1] + (n - 1 == i ? add : 0.0);
        }
#pragma unroll 4
        for (int64_t j = j0 + 2 * threadIdx.x; j + 1 < n; j += 2 * blockDim.x) {
            double a = (double)src[j];
            if (j == i) a += add;
            *reinterpret_cast<double2 *>(dst + j) = make_double2(a, (double)src[j + 1]);
        }
    }
}

// ---- P = M_KK^-1 for the 128 x 128 diagonal block, in shared memory (full symmetric copy S).
// The block is itself swept in 4 sub-blocks of 32: the 32 x 32 sub-pivot is inverted by a
// scalar sweep in shared memory, then all 256 threads apply the rank-32 sweep update
//   S_IJ -= O_I^T W_J,  S_sJ = W_J,  S_Is = W_I^T,  S_ss = -Q   (O = old block row s, W = Q O).
// Returns 0 or the failing pivot index + 1 (the sweep pivots are the LDL^T pivots).
constexpr int S2 = 32;  // sub-pivot size
constexpr int S2_ = S2;
constexpr int QLD = S2 + 4;  // padded row stride of Q (conflict-free DMMA fragments)

// 1/d for a positive normal d: the hardware approximation refined by two Newton steps (error
// squared each time: full double precision up to the last bit or two; the sweep tolerates that,
// and it is off the IEEE-rounded __drcp_rn's longer software sequence on the sweep's serial chain)
__device__ __forceinline__ double rcp_fast(double d) {
    double r;
    asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(d));
    double e = fma(-d, r, 1.0);
    r = fma(r, e, r);
    e = fma(-d, r, 1.0);
    return fma(r, e, r);
}

// sweep of the 32 x 32 sub-pivot S[s0.., s0..] by all 8 warps with the block in registers: thread
// (w, lane) holds rows 4w..4w+3 of column `lane`.  The sweep keeps the block symmetric, so pivot
// row t equals column t: per pivot its owner warp publishes row t (ping-pong buffer), one barrier,
// then every thread updates its 4 elements.  Writes Q = inv(sub-pivot); returns 0 or the failing
// pivot index + 1 (uniform across the block).
__device__ __forceinline__ int block_sweep32(const double (*S)[B + 1], int s0, double *Q, double *rowbuf, int base) {
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    double x[4];
#pragma unroll
    for (int r = 0; r < 4; r++) {
        const int l = 4 * w + r;  // upper storage
        x[r] = S[s0 + min(l, lane)][s0 + max(l, lane)];
    }
    // unrolled by 4 only: the pivot runs once per step per matrix, and a fully unrolled body (32 copies)
    // misses the instruction cache on every call; t & 3 stays a compile-time index
#pragma unroll 4
    for (int t = 0; t < S2_; t++) {
        double *rb = rowbuf + (t & 1) * 32;
        if (w == (t >> 2)) rb[lane] = x[t & 3];
        WSYNC();
        const double d = rb[t];
        if (!(d > 0.0)) return base + t + 1;  // uniform: every thread read the same d
        const double inv = rcp_fast(d);
        const double vj = rb[lane] * inv;  // (t, lane) / d
#pragma unroll
        for (int r = 0; r < 4; r++) {
            const int l = 4 * w + r;
            const double c = rb[l];  // (l, t) = (t, l)
            if (l == t) x[r] = (lane == t) ? -inv : vj;
            else x[r] = (lane == t) ? c * inv : fma(-c, vj, x[r]);
        }
    }
#pragma unroll
    for (int r = 0; r < 4; r++) Q[(4 * w + r) * QLD + lane] = -x[r];
    return 0;
}

#ifdef PIVOT_DBG  // cycles per pivot phase, summed over every pivot (kfac_debug_pclk)
__device__ int g_pivot_dbg;
__device__ unsigned long long g_pacc[32];
#define PCLK(k)                                                                          \
    if (threadIdx.x == 0) {                                                              \
        const long long now_ = clock64();                                                \
        atomicAdd(&g_pacc[k], (unsigned long long)(now_ - pclk_last));                   \
        pclk_last = now_;                                                                \
    }
#else
#define PCLK(k)
#endif
// P = (S)^-1 into Pout (B x B, zero outside bk); -P also goes straight into the upper tile (K, K) of W,
// the value the sweep gives that tile at step K (no later task has to read the pivot slot for it)
__device__ __forceinline__ void pivot_write_w(const double (*S)[B + 1], double *__restrict__ W, int64_t ld, int k0, int bk) {
    for (int e = threadIdx.x; e < B * B; e += kWorkers) {  // W_KK = -P (upper storage)
        const int i = e >> 7, j = e & (B - 1);
        if (i < bk && j < bk && j >= i) W[(int64_t)(k0 + i) * ld + k0 + j] = S[i][j];
    }
}
__device__ int pivot_block(double *__restrict__ W, int64_t ld, int k0, int bk, double *__restrict__ Pout,
                           double *smem, bool preloaded = false, bool write_w = true) {
#ifdef PIVOT_DBG
    long long pclk_last = clock64();
#endif
    double(*S)[B + 1] = reinterpret_cast<double(*)[B + 1]>(smem);
    double *O = smem + B * (B + 1);       // [S2][SLD] old block row
    double *Wr = O + S2 * SLD;            // [S2][SLD] Q * O
    double *Q = Wr + S2 * SLD;            // [S2][QLD] inverse of the sub-pivot
    double *colbuf = Q + S2 * QLD;        // [2][32] sweep broadcast buffers (ping-pong)
    int *fsh = reinterpret_cast<int *>(colbuf + 64);
    const int tid = threadIdx.x;
    // only the upper triangle of S is ever read (min / max indexing below), so only it is loaded
    // (coalesced rows); identity padding beyond bk keeps the sweep well defined
    if (!preloaded)
        for (int e = tid; e < B * B; e += kWorkers) {
            const int i = e >> 7, j = e & (B - 1);
            if (j < i) continue;
            S[i][j] = (i < bk && j < bk) ? W[(int64_t)(k0 + i) * ld + (k0 + j)] : (i == j ? 1.0 : 0.0);
        }
    if (tid == 0) *fsh = 0;
    WSYNC();
    PCLK(0)
    for (int sb = 0; sb < B / S2; sb++) {
        const int s0 = sb * S2;
        if (s0 >= bk) break;
        {
            const int f = block_sweep32(S, s0, Q, colbuf, k0 + s0);  // Q = inv(sub-pivot)
            if (f) {
                if (tid == 0) *fsh = f;
                break;
            }
        }
        WSYNC();
        PCLK(1 + 4 * sb)
        for (int e = tid; e < S2 * B; e += kWorkers) {  // old block row s (upper storage)
            const int a = s0 + (e >> 7), c = e & (B - 1);
            O[(e >> 7) * SLD + c] = S[min(a, c)][max(a, c)];
        }
        WSYNC();
        if (*fsh) break;
        PCLK(2 + 4 * sb)
#ifdef PIVOT_DBG
        if (g_pivot_dbg == 1 && sb >= 1) break;
#endif
        // W = Q O  (32 x 128, K = 32) on the fp64 tensor cores: warp w owns columns 16w..16w+15,
        // all four 8-row blocks (m8n8k4: A frag Q[row][k], B frag O[k][col])
        {
            const int w = tid >> 5, lane = tid & 31, r8 = lane >> 2, k4 = lane & 3;
            double c[4][2][2];
#pragma unroll
            for (int i = 0; i < 4; i++)
#pragma unroll
                for (int j = 0; j < 2; j++) c[i][j][0] = c[i][j][1] = 0.0;
#pragma unroll
            for (int kk = 0; kk < S2 / 4; kk++) {
                double a[4], b[2];
#pragma unroll
                for (int i = 0; i < 4; i++) a[i] = Q[(8 * i + r8) * QLD + 4 * kk + k4];
#pragma unroll
                for (int j = 0; j < 2; j++) b[j] = O[(4 * kk + k4) * SLD + 16 * w + 8 * j + r8];
#pragma unroll
                for (int i = 0; i < 4; i++)
#pragma unroll
                    for (int j = 0; j < 2; j++) dmma(c[i][j][0], c[i][j][1], a[i], b[j]);
            }
#pragma unroll
            for (int i = 0; i < 4; i++)
#pragma unroll
                for (int j = 0; j < 2; j++)
                    *reinterpret_cast<double2 *>(Wr + (8 * i + r8) * SLD + 16 * w + 8 * j + 2 * k4) =
                        make_double2(c[i][j][0], c[i][j][1]);
        }
        WSYNC();
        PCLK(3 + 4 * sb)
#ifdef PIVOT_DBG
        if (g_pivot_dbg == 2 && sb >= 1) break;
#endif
        // rank-32 sweep update S -= O^T W of the upper triangle on the fp64 tensor cores (DMMA):
        // 8-row strips r and 15 - r (17 m8n8 blocks together) per warp, then the sub-block's rows
        // and columns get their sweep values: S_sJ = W_J, S_Is = W_I^T, S_ss = -Q
        {
            const int w = tid >> 5, lane = tid & 31, r8 = lane >> 2, k4 = lane & 3;
            const int nfirst = 16 - w;  // blocks of strip w (columns w..15); then strip 15-w
            double acc[17][2];
#pragma unroll
            for (int x = 0; x < 17; x++) acc[x][0] = acc[x][1] = 0.0;
#pragma unroll
            for (int kk = 0; kk < S2 / 4; kk++) {
                const int t = 4 * kk + k4;
                const double aA = O[t * SLD + 8 * w + r8], aB = O[t * SLD + 8 * (15 - w) + r8];
#pragma unroll
                for (int x = 0; x < 17; x++) {
                    const bool first = x < nfirst;
                    const int cb = first ? w + x : x - 1;
                    dmma(acc[x][0], acc[x][1], first ? aA : aB, Wr[t * SLD + 8 * cb + r8]);
                }
            }
#pragma unroll
            for (int x = 0; x < 17; x++) {
                const bool first = x < nfirst;
                const int i = 8 * (first ? w : 15 - w) + r8, j = 8 * (first ? w + x : x - 1) + 2 * k4;
                S[i][j] -= acc[x][0];
                S[i][j + 1] -= acc[x][1];
            }
        }
        WSYNC();
        for (int e = tid; e < S2 * B; e += kWorkers) {
            const int a = e >> 7, j = e & (B - 1);
            if (j >= s0 && j < s0 + S2) S[s0 + a][j] = -Q[a * QLD + (j - s0)];
            else if (j > s0) S[s0 + a][j] = Wr[a * SLD + j];  // right of the sub-block: its row band
            else S[j][s0 + a] = Wr[a * SLD + j];              // left: its column band (upper storage)
        }
        WSYNC();
        PCLK(4 + 4 * sb)
    }
    WSYNC();
    PCLK(20)
    const int fail = *fsh;
    if (fail) return fail;
    for (int e = tid; e < B * B; e += kWorkers) {  // P = -S (zero outside bk); W_KK = -P (upper)
        const int i = e >> 7, j = e & (B - 1);
        const bool in = i < bk && j < bk;
        if (Pout) Pout[e] = in ? -S[min(i, j)][max(i, j)] : 0.0;  // (int8 matrices: their panels read P's digits)
        if (write_w && in && j >= i) W[(int64_t)(k0 + i) * ld + k0 + j] = S[i][j];
    }
    PCLK(21)
    return 0;
}

__device__ __forceinline__ double *pivot_slot(const MatDesc &m, int k) {
    return m.panel + 2 * kPanelBufs * (int64_t)B * m.ld + (int64_t)(k & 1) * B * B;
}
// kPanelBufs R / P R panel buffers (step mod 4): a merged task reads steps k and k+1 while later
// steps' panels are written; with four, a panel's buffer wait (all updates of step k-4) points to
// the pair two pairs back, so chain tasks do not wait for the current bulk tiles
__device__ __forceinline__ double *panel_R(const MatDesc &m, int k) { return m.panel + (int64_t)(k % kPanelBufs) * 2 * B * m.ld; }
__device__ __forceinline__ double *panel_Wp(const MatDesc &m, int k) { return panel_R(m, k) + (int64_t)B * m.ld; }

__device__ __forceinline__ void cp_async16(void *dst, const void *src, bool ok) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"((uint32_t)__cvta_generic_to_shared(dst)),
                 "l"(src), "r"(ok ? 16 : 0)
                 : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_1() { asm volatile("cp.async.wait_group 1;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_0() { asm volatile("cp.async.wait_group 0;" ::: "memory"); }
// mbarrier + 1-D bulk copy (async proxy) for the C tile of an update
__device__ __forceinline__ uint32_t s2u(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void cbar_expect(uint64_t *bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(s2u(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void cbar_wait(uint64_t *bar, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "W_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra W_%=;\n\t}" ::"r"(s2u(bar)),
        "r"(parity)
        : "memory");
}
__device__ __forceinline__ void bulk_row(void *dst, const void *src, uint32_t bytes, uint64_t *bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(s2u(dst)),
                 "l"(src), "r"(bytes), "r"(s2u(bar))
                 : "memory");
}

// acc += sum_{t < kt} A[t][i] * Bm[t][j] for the 128 x 128 tile on the fp64 tensor cores
// (mma.sync m8n8k4 f64, DMMA: 256 FMAs per warp instruction).  Warp w owns rows
// 64*(w>>2) + [0, 64) and columns 32*(w&3) + [0, 32) as 8 x 4 m8n8 blocks; acc[p][q] is the
// element (tile_row(p), tile_col(q)) below.  A and Bm are row-major with 16-aligned leading
// dimensions; columns >= aw / bw and rows >= kt read as zero (cp.async zero fill).  Operand rows
// stream through a kStages-deep shared-memory ring of KC-row chunks: every thread copies its
// share of a chunk with 16-byte cp.async and signals the stage's `full` mbarrier on completion
// (cp.async.mbarrier.arrive.noinc); each warp releases a stage on its `empty` mbarrier once its
// fragments are loaded.  No CTA-wide barrier inside the product: warps drift up to a chunk
// apart, so their shared-load phases do not line up.  Two K segments (a merged two-step update)
// run as one chunk stream.  Shared rows are padded to 132 doubles (conflict-free fragments).
struct Seg {
    const double *A;
    int64_t lda;
    int aw;
    const double *Bm;
    int64_t ldb;
    int bw;
    int kt;
};
struct Ring {
    uint64_t *full, *empty;  // [kStages] each
    uint32_t g;              // chunks this CTA has streamed so far (uniform over the CTA)
};
// BSRC: 0 both operands through the ring; 1 / 2 the B operand is already resident in shared memory
// (Tb, row stride B+1: element (t, j) at Tb[t][j], or at Tb[j][t] for 2) and only A streams.
template <int BSRC = 0>
__device__ __forceinline__ void tile_product(const Seg &s0, const Seg &s1, double (&acc)[8][8], double *smem, Ring &ring,
                                             const double *Tb = nullptr) {
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int arow = 64 * (w >> 2) + (lane >> 2), bcol = 32 * (w & 3) + (lane >> 2), kl = lane & 3;
    const int n0 = (s0.kt + KC - 1) / KC, nch = n0 + (s1.kt + KC - 1) / KC;
    WSYNC();  // the caller's shared-memory use (staging, pivots, epilogues) is over
    auto produce = [&](int c) {  // every thread: its 16-byte pieces of chunk c
        const uint32_t G = ring.g + c, st = G % kStages;
        const bool first = c < n0;
        const double *A = first ? s0.A : s1.A, *Bm = first ? s0.Bm : s1.Bm;
        const int64_t lda = first ? s0.lda : s1.lda, ldb = first ? s0.ldb : s1.ldb;
        const int aw = first ? s0.aw : s1.aw, bw = first ? s0.bw : s1.bw;
        const int t0 = (first ? c : c - n0) * KC, kt = first ? s0.kt : s1.kt;
        if (G >= kStages) cbar_wait(ring.empty + st, ((G / kStages) + 1) & 1);  // chunk G - kStages consumed
        double *dst = smem + st * 2 * KC * SLD;
#pragma unroll
        for (int it = 0; it < (BSRC ? 1 : 2) * KC * B / 2 / 256; it++) {
            const int e = it * 256 + threadIdx.x, r = e >> 6, i = (e & 63) * 2;  // r < KC: A rows, else B
            const bool isA = r < KC;
            const int t = t0 + (isA ? r : r - KC);
            const bool ok = t < kt && i < (isA ? aw : bw);
            const double *src = isA ? A + (int64_t)t * lda + i : Bm + (int64_t)t * ldb + i;
            cp_async16(dst + r * SLD + i, ok ? src : A, ok);
        }
        asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(s2u(ring.full + st)) : "memory");
    };
    for (int c = 0; c < min(kStages - 1, nch); c++) produce(c);
    for (int c = 0; c < nch; c++) {
        const uint32_t G = ring.g + c, st = G % kStages;
        cbar_wait(ring.full + st, (G / kStages) & 1);
        const double *as = smem + st * 2 * KC * SLD, *bs = as + KC * SLD;
#pragma unroll
        for (int kk = 0; kk < KC / 4; kk++) {
            const int t = kk * 4 + kl;
            double a[8], b[4];
#pragma unroll
            for (int p = 0; p < 8; p++) a[p] = as[t * SLD + arow + 8 * p];
            const int tg = (c < n0 ? c : c - n0) * KC + t;  // K row within the segment (resident B)
#pragma unroll
            for (int q = 0; q < 4; q++)
                b[q] = BSRC == 0 ? bs[t * SLD + bcol + 8 * q]
                                 : (BSRC == 1 ? Tb[tg * (B + 1) + bcol + 8 * q] : Tb[(bcol + 8 * q) * (B + 1) + tg]);
#pragma unroll
            for (int p = 0; p < 8; p++)
#pragma unroll
                for (int q = 0; q < 4; q++) dmma(acc[p][2 * q], acc[p][2 * q + 1], a[p], b[q]);
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(ring.empty + st);
        if (c + kStages - 1 < nch) produce(c + kStages - 1);
    }
    ring.g += nch;
    WSYNC();  // every warp is done with the ring before the caller reuses the shared memory
}

__device__ __forceinline__ void cp_async8(void *dst, const void *src, bool ok) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;" ::"r"((uint32_t)__cvta_generic_to_shared(dst)), "l"(src),
                 "r"(ok ? 8 : 0)
                 : "memory");
}

#ifdef INV_TRACE  // experiment build only: per-task timeline
struct TraceRec { int g, k, kind, I, J, sm; long long t0, t1, t2, t3, t4, t5, t6, t7, t8; };
__device__ TraceRec g_trace[1 << 17];
__device__ long long g_trace_sub[1024][6];  // per CTA: [0, 1] end of the product / of the C-tile wait; [2..5] panel phases
__device__ __forceinline__ long long gtime() { long long t; asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t)); return t; }
#define TRACE(...) __VA_ARGS__
__device__ unsigned long long g_ozprof[8];  // cycles: ring wait, TE wait, A wait, TF wait, drain, issue, tasks
__device__ long long g_ozt[148][80];  // one merged task per CTA (the 20th): producer issue start/end, warp-1 TF done/drain done
__device__ int g_ozcnt[148];
#define OZPROF(i, t0) atomicAdd(&g_ozprof[i], (unsigned long long)(clock64() - (t0)))
#else
#define TRACE(...)
#endif
// ---- int8-sliced ("Ozaki") sweep updates on the tensor cores (tcgen05 kind::i8), the per-matrix
// fast path of reading R-12 (decide_precision).  Each column c of a step's panel block X (X = R_J
// or Wp_J, 128 rows t = the step's K index) is written with five balanced 8-bit digits
//     X[t][c] = 2^(e_c - 37) * sum_{s<5} q_s[t][c] 2^8(4-s),   q_s in [-128, 127] (|q_0| <= 33),
// e_c the column exponent (max_t |X[t][c]| < 2^e_c), |error| <= 2^(e_c - 38).  The update product
// R_I^T Wp_J then is 2^(e_i + f_j - 42) * sum_{d<5} 2^8(4-d) Acc_d with the exact int32 tensor-core
// sums Acc_d = sum_{s+u=d} q_s(R_I)^T q_u(Wp_J) (the 15 digit pairs of weight >= 2^-32 of the
// leading one), recombined exactly in int64 (|V| < 2^50) and scaled in fp64.  Measured on the
// workload's factors and rank-deficient ReLU Grams at kappa ~ 1e4: ~1e-8 relative error of the
// damped inverse (scripts/ozaki_proto.py), against 3e-8 for all-fp64 updates and the 1e-5 bound.
// Digit tiles are [128 columns][128 t] int8, K-major in the 128-byte swizzle, 16 KB each, written
// once per (step, column block) by the panel task; an update streams its B operand in column
// quarters (N = 32) through a 3-slot ring, and TMEM holds two quarter accumulator sets (5 x 32
// columns each) so that one quarter drains while the next one's 60 MMAs run.
constexpr int kOzSlice = B * B;       // bytes per int8 digit tile
constexpr int kOzQ = 32;              // columns per pass (MMA N)
constexpr int kOzQBytes = kOzQ * B;   // one digit tile's quarter (32 rows x 128 B)
constexpr int kOzD = 6;               // digits stored per column: x = 2^(e - 45) sum_{s<6} q_s 2^8(5-s)
constexpr int kOzBits = 45;
constexpr int kOzSet = kOzD * kOzSlice;            // one stored digit tile set (96 KB)
constexpr int kOzABytes = kOzS * kOzSlice;          // one step's A digits (80 KB)
constexpr int kOzRBytes = kOzS * kOzQBytes;         // one ring slot: a quarter of the 5 B tiles (20 KB)
constexpr int kOzSmem = 2 * kOzABytes + 3 * kOzRBytes + 4 * B * 4 + 1024;
static_assert(kOzS == 5, "the drain recombines exactly five diagonals");
static_assert(kOzSmem == kUpdSmemOz, "kUpdSmem accounts for the int8 pipeline");
static_assert(B * (B + 1) * 8 <= 133120 && kOzSet <= 133120, "the panel's T region holds R_J, P_k's digits and Wp_J");
static_assert(B * (B + 1) * 8 <= 2 * kOzABytes, "the product tile fits the A slots");
// instruction descriptor kind::i8: D s32, A and B s8, both K-major, M = 128, N = n
__host__ __device__ constexpr uint32_t idesc_i8(uint32_t n) {
    return (2u << 4) | (1u << 7) | (1u << 10) | ((n >> 3) << 17) | ((uint32_t)(B >> 4) << 24);
}

// per matrix, after the pivot slots: [step mod kPanelBufs][J][op: R_J, Wp_J] digit tile sets (6 x 16 KB),
// their column exponents [step mod kPanelBufs][op][n], and two pivot digit sets (P_k, k mod 2) + exponents
__device__ __forceinline__ uint8_t *oz_base(const MatDesc &m) {
    return reinterpret_cast<uint8_t *>(m.panel + 2 * kPanelBufs * (int64_t)B * m.ld + 2 * (int64_t)B * B);
}
__device__ __forceinline__ int oz_set(const MatDesc &m, int k, int J, int op) {
    return ((k % kPanelBufs) * m.nt + J) * 2 + op;
}
__device__ __forceinline__ uint8_t *oz_slices(const MatDesc &m, int k, int J, int op) {
    return oz_base(m) + (((int64_t)(k % kPanelBufs) * m.nt + J) * 2 + op) * kOzSet;
}
__device__ __forceinline__ int *oz_exps(const MatDesc &m, int k, int op) {
    return reinterpret_cast<int *>(oz_base(m) + (int64_t)kPanelBufs * m.nt * 2 * kOzSet) + ((int64_t)(k % kPanelBufs) * 2 + op) * m.nt * B;
}
__device__ __forceinline__ uint8_t *oz_pivdig(const MatDesc &m, int k) {
    return oz_base(m) + (int64_t)kPanelBufs * m.nt * 2 * kOzSet + (int64_t)kPanelBufs * 2 * m.nt * B * 4 + (k & 1) * (kOzSet + B * 4);
}
__device__ __forceinline__ int *oz_pivexp(const MatDesc &m, int k) { return reinterpret_cast<int *>(oz_pivdig(m, k) + kOzSet); }

// digits of the 128 x 128 block X -> dst (kOzD tiles) and the column exponents -> dexp[0..128) (and
// sexp, 128 ints of shared memory).  MODE 0: X[t][c] = T[t][c]; 1: T[c][t]; 2: the pivot,
// X = P = -S with S in upper storage, zero outside bk x bk.  All 256 threads.
template <int MODE>
__device__ __forceinline__ double oz_x(const double (*T)[B + 1], int t, int c, int bk) {
    if (MODE == 0) return T[t][c];
    if (MODE == 1) return T[c][t];
    if (MODE == 3) return (t < bk && c < bk) ? -T[t][c] : 0.0;  // the pivot after pivot_fill_lower
    return (t < bk && c < bk) ? -T[min(t, c)][max(t, c)] : 0.0;
}
#ifndef KFAC_OZ_SLICE_LANES
#define KFAC_OZ_SLICE_LANES 4  // measured per cut: 1 lane 8.0 us, 2 lanes 5.4 us, 4 lanes 5.2 us (RN50 panels)
#endif
// U = rint(x * sc) + 0x8080808080 without an fp64 -> int64 conversion: fma(x, sc, 1.5 * 2^52) rounds the
// exact product (|x sc| < 2^45) to an integer in one step (ties to even, like __double2ll_rn), and the
// bit pattern minus that of 1.5 * 2^52 is the integer
__device__ __forceinline__ long long oz_round_bias(double x, double sc) {
    return __double_as_longlong(fma(x, sc, 6755399441055744.0)) - (0x4338000000000000LL - 0x8080808080LL);
}
// the swept pivot block lives in upper storage; mirror it into the lower triangle so that its digit cut
// reads rows (MODE 3) instead of the min / max gather of MODE 2
__device__ __forceinline__ void pivot_fill_lower(double (*S)[B + 1]) {
    for (int e = threadIdx.x; e < B * B; e += kWorkers) {
        const int i = e >> 7, j = e & (B - 1);
        if (j < i) S[i][j] = S[j][i];
    }
}
template <int MODE>
__device__ void oz_slice(const double (*T)[B + 1], uint8_t *dst, int *dexp, int *sexp, int bk = B) {
    const int tid = threadIdx.x;
    {  // column maxima: two threads per column (half the rows each), 8 loads in flight
        const int c = tid & (B - 1), t0 = (tid >> 7) * (B / 2);
        double mx[8];
#pragma unroll
        for (int u = 0; u < 8; u++) mx[u] = 0.0;
#pragma unroll
        for (int t = 0; t < B / 2; t += 8)
#pragma unroll
            for (int u = 0; u < 8; u++) mx[u] = fmax(mx[u], fabs(oz_x<MODE>(T, t0 + t + u, c, bk)));
        const double m4 = fmax(fmax(fmax(mx[0], mx[1]), fmax(mx[2], mx[3])), fmax(fmax(mx[4], mx[5]), fmax(mx[6], mx[7])));
        double *red = reinterpret_cast<double *>(sexp + B);  // 128 doubles of scratch after the exponents
        if (tid >= B) red[c] = m4;
        WSYNC();
        if (tid < B) {
            const double m = fmax(m4, red[c]);
            int e = 0;
            if (m > 0.0) frexp(m, &e);
            e = max(e, -960);  // below: the digits (and the contribution) vanish
            sexp[c] = e;
            dexp[c] = e;
        }
    }
    WSYNC();
    // digits: U = Y + C with C = 0x80 in each of the five low bytes; the low bytes of U XOR 0x80 are the
    // balanced digits q_5..q_1 (q = u - 128), and U >> 40 is q_0 (|q_0| <= 33).  Four consecutive t are
    // transposed byte-wise (PRMT) into the digit planes.
    for (int it = tid; it < B * 8; it += 256) {
        // KFAC_OZ_SLICE_LANES consecutive lanes cut the consecutive 16-row chunks tc of one column, so a
        // warp's 16-byte stores cover 32 / LANES lines (LANES = 1: every lane its own column, 32 lines,
        // conflict-free shared reads; LANES = 2: 16 lines, still conflict-free for 8-byte reads)
        const int lane = it & 31, wi = it >> 5;  // warp item 0..31
        const int c = (KFAC_OZ_SLICE_LANES == 1) ? (it & (B - 1))
                                                 : (32 / KFAC_OZ_SLICE_LANES) * (wi % (B * KFAC_OZ_SLICE_LANES / 32)) +
                                                       lane % (32 / KFAC_OZ_SLICE_LANES);
        const int tc = (KFAC_OZ_SLICE_LANES == 1) ? (it >> 7)
                                                  : KFAC_OZ_SLICE_LANES * (wi / (B * KFAC_OZ_SLICE_LANES / 32)) +
                                                        lane / (32 / KFAC_OZ_SLICE_LANES);
        const double sc = __longlong_as_double((long long)(1023 + kOzBits - sexp[c]) << 52);
        uint32_t wd[kOzD][4];
#pragma unroll
        for (int g = 0; g < 4; g++) {
            uint32_t lo[4], hi[4];
#pragma unroll
            for (int u = 0; u < 4; u++) {
                const long long U = oz_round_bias(oz_x<MODE>(T, 16 * tc + 4 * g + u, c, bk), sc);
                lo[u] = (uint32_t)U ^ 0x80808080u;        // bytes: q_5, q_4, q_3, q_2
                hi[u] = (uint32_t)(U >> 32);              // byte 0: q_1 ^ 0x80, bits 8..: q_0
            }
            // 4 x 4 byte transpose of lo: plane 5 gets byte 0 of each, ... plane 2 byte 3
            const uint32_t a01 = __byte_perm(lo[0], lo[1], 0x5140), a23 = __byte_perm(lo[2], lo[3], 0x5140);
            const uint32_t b01 = __byte_perm(lo[0], lo[1], 0x7362), b23 = __byte_perm(lo[2], lo[3], 0x7362);
            wd[5][g] = __byte_perm(a01, a23, 0x5410);
            wd[4][g] = __byte_perm(a01, a23, 0x7632);
            wd[3][g] = __byte_perm(b01, b23, 0x5410);
            wd[2][g] = __byte_perm(b01, b23, 0x7632);
            const uint32_t h01 = __byte_perm(hi[0], hi[1], 0x5140), h23 = __byte_perm(hi[2], hi[3], 0x5140);
            wd[1][g] = __byte_perm(h01, h23, 0x5410) ^ 0x80808080u;
            wd[0][g] = __byte_perm(h01, h23, 0x7632);  // byte 1 of hi = q_0 (signed, |q_0| < 128)
        }
#pragma unroll
        for (int s = 0; s < kOzD; s++) {
            uint8_t *a = dst + s * kOzSlice + c * B + ((tc ^ (c & 7)) << 4);
            *reinterpret_cast<uint4 *>(a) = make_uint4(wd[s][0], wd[s][1], wd[s][2], wd[s][3]);
        }
    }
    asm volatile("fence.proxy.async;" ::: "memory");  // the digits are read back by bulk copies
}

// barriers of the int8 update pipeline (shared memory) and their phase bits (uniform per CTA)
enum { OZ_A = 0, OZ_R = 2, OZ_TF = 5, OZ_TE = 8, OZ_RD = 11, OZ_NBAR = 12 };
#ifndef KFAC_OZ_SETS
#define KFAC_OZ_SETS 2
#endif
constexpr int kOzSets = KFAC_OZ_SETS;  // TMEM accumulator sets of an update (3 x 5 x 32 columns); a panel uses 2 (2 x 6 x 32)
static_assert(kOzSets * kOzS * kOzQ + 3 * 64 <= 512 && 2 * kOzD * kOzQ + 2 * 64 <= 512,
              "accumulator sets + parked quarters fit TMEM (update: 3 quarters, panel: 2)");
// The persistent kernel runs 8 worker warps (256 threads: every task's arithmetic, epilogues, drains) and
// one producer warp (threads 256..287) whose lane 0 loads the int8 operands and issues the tensor-core
// MMAs of the int8 tasks, so that the MMAs of pass p run while the workers drain pass p-1.  Worker-only
// code synchronises with WSYNC (named barrier 1, 256 threads); __syncthreads is for all 288.

struct OzState {
    uint64_t *bar;  // [OZ_NBAR]: A digits per step (2), ring slots (3), TMEM full (3), TMEM empty (3), R_J digits out
    uint32_t ph;    // phase bit per barrier
    uint32_t tmem;  // 2 accumulator sets x (5 or 6) diagonals x 32 columns
    int *sexp;      // [128] shared: column exponents of the block being cut into digits
    int *eP;        // [128] shared: the pivot's row exponents (panel product)
};
__device__ __forceinline__ void oz_wait(OzState &o, int b) {
    cbar_wait(o.bar + b, (o.ph >> b) & 1);
    o.ph ^= 1u << b;
}

// 32 lanes x 8 columns of 32-bit
__device__ __forceinline__ void tmem_ld_x8(uint32_t taddr, uint32_t (&r)[8]) {
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
                 : "r"(taddr));
}
__device__ __forceinline__ void tmem_st_x32(uint32_t taddr, const uint32_t (&r)[32]) {
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], "
        "{%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,"
        "%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(taddr),
        "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]), "r"(r[9]),
        "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15]), "r"(r[16]), "r"(r[17]), "r"(r[18]),
        "r"(r[19]), "r"(r[20]), "r"(r[21]), "r"(r[22]), "r"(r[23]), "r"(r[24]), "r"(r[25]), "r"(r[26]), "r"(r[27]),
        "r"(r[28]), "r"(r[29]), "r"(r[30]), "r"(r[31])
        : "memory");
}
__device__ __forceinline__ void mma_i8(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}" ::"r"(d),
        "l"(a), "l"(b), "r"(idesc), "r"(acc)
        : "memory");
}
__device__ __forceinline__ void bulk_prefetch_l2(const void *src, uint32_t bytes) {
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(src), "r"(bytes) : "memory");
}
// L2 residency: the C tiles stream through once per two steps (evict first); the digit tiles are read
// by a whole step's tasks (evict last).  KFAC_OZ_HINTS=0 builds without hints (experiments).
#ifndef KFAC_OZ_HINTS
#define KFAC_OZ_HINTS 1
#endif
// C -= P through the L2: W_row += (-P)_row as one bulk reduce-add per row (fp64 adds performed at L2;
// W + (-P) is the same IEEE result as W - P).  Per-thread bulk groups: the issuing thread waits for
// the source reads before the staging is reused and for completion before the tile is released.
__device__ __forceinline__ void bulk_red_add_f64(double *dst, const void *src, uint32_t bytes) {
    asm volatile("cp.reduce.async.bulk.global.shared::cta.bulk_group.add.f64 [%0], [%1], %2;" ::"l"(dst), "r"(s2u(src)),
                 "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_read() { asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_all() {
    asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
    asm volatile("fence.proxy.async.global;" ::: "memory");  // the async-proxy writes before the generic release
}
#ifndef KFAC_OZ_BULK_RMW
#define KFAC_OZ_BULK_RMW 1
#endif
constexpr int kPn = B + 2;  // staging row stride of the bulk path (16-byte aligned rows)

__device__ __forceinline__ uint64_t pol_evict_first() {
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
    return p;
}
__device__ __forceinline__ uint64_t pol_evict_last() {
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
    return p;
}
__device__ __forceinline__ double ld_ef(const double *p, uint64_t pol) {
    double v;
    asm volatile("ld.global.L1::no_allocate.L2::cache_hint.f64 %0, [%1], %2;" : "=d"(v) : "l"(p), "l"(pol));
    return v;
}
__device__ __forceinline__ void st_ef(double *p, double v, uint64_t pol) {
    asm volatile("st.global.L1::no_allocate.L2::cache_hint.f64 [%0], %1, %2;" ::"l"(p), "d"(v), "l"(pol) : "memory");
}
__device__ __forceinline__ void bulk_row_hint(void *dst, const void *src, uint32_t bytes, uint64_t *bar, uint64_t pol) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(s2u(dst)),
                 "l"(src), "r"(bytes), "r"(s2u(bar)), "l"(pol)
                 : "memory");
}
// one thread: the 15 digit-pair products of one column quarter (K = 128 = 4 MMAs of K 32 each).
// The accumulator set is [diagonal d = 0..4][32 columns] and a ring slot holds the quarter tiles of
// B's digits u = 0..4 as consecutive 32-row blocks, so for A's digit s ONE MMA with B = rows
// [0, 32 (5 - s)) of the slot (N = 32 (5 - s)) adds q_s^T r_u into diagonal s + u for every u at
// once: 5 MMAs per K step, each A chunk read from shared memory once.
template <int ND>
__device__ __forceinline__ void oz_mma_pass(uint32_t tacc, uint32_t sa, uint32_t sb) {
    // descriptors from two bases: the start-address field is addr >> 4 (shared memory < 256 KB: no
    // carry out of the 14-bit field), so an operand offset is a constant add
    const uint64_t da = umma_desc(sa, 16, 1024, UMMA_SW128), db = umma_desc(sb, 16, 1024, UMMA_SW128);
#pragma unroll
    for (int s = 0; s < ND; s++)
#pragma unroll
        for (int kk = 0; kk < B / 32; kk++)
            mma_i8(tacc + kOzQ * s, da + (uint64_t)((s * kOzSlice + kk * 32) >> 4), db + (uint64_t)((kk * 32) >> 4),
                   idesc_i8(kOzQ * (ND - s)), (s > 0 || kk > 0) ? 1u : 0u);
}
// thread (warp w, lane): row 32 (w & 3) + lane, columns 16 (w >> 2) + [0, 16) of the quarter (eB: the
// quarter's 32 column exponents):
// acc += 2^(eA[row] + eB[col] - 42) * sum_d 2^8(4-d) Acc_d   (int64 exact, |V| < 2^50):
// x y = 2^(ea - 37) 2^(eb - 37) sum_{s,u} 2^8(8 - s - u) q_s r_u = 2^(ea + eb - 42) sum_d 2^8(4 - d) Acc_d
__device__ __forceinline__ void oz_drain(uint32_t tacc, double (&acc)[16], const int *eA, const int *eB) {
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t tb = tacc + ((uint32_t)(32 * (w & 3)) << 16) + 16 * (w >> 2);
    const int ea = eA[32 * (w & 3) + lane] - 42 + 1023;
    // all five diagonals' 16 columns in flight at once, one wait (a wait covers every earlier load)
    uint32_t a[kOzS][16];
#pragma unroll
    for (int d = 0; d < kOzS; d++) tmem_ld_32x32b_x16(tb + kOzQ * d, a[d]);
    tmem_ld_wait();
#pragma unroll
    for (int d = 0; d < kOzS; d++) tmem_regs_ready(a[d]);
#pragma unroll
    for (int c = 0; c < 16; c++) {
        const int v01 = (int)a[0][c] * 256 + (int)a[1][c];
        const long long V = ((long long)v01 * 256 + (int)a[2][c]) * 65536LL + ((long long)(int)a[3][c] * 256 + (int)a[4][c]);
        const double v = __longlong_as_double(V + 0x4338000000000000LL) - 6755399441055744.0;  // exact, |V| < 2^51
        const int ex = max(ea + eB[16 * (w >> 2) + c], 0);
        acc[c] = fma(v, __longlong_as_double((long long)ex << 52), acc[c]);
    }
}

// the panel product's drain (all six digits, the 21 pairs of weight >= 2^-40): per thread row t,
// columns 16 (w >> 2) + [0, 16) of the quarter; acc = 2^(eP[t] + eR[col] - 50) * sum_d 2^8(5-d) Acc_d,
// recombined as two exact halves (each |.| < 2^40) so that the fp64 conversion stays exact
__device__ __forceinline__ void oz_drain6(uint32_t tacc, double (&acc)[16], const int *eP, const int *eR) {
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t tb = tacc + ((uint32_t)(32 * (w & 3)) << 16) + 16 * (w >> 2);
    const int ea = eP[32 * (w & 3) + lane] - 50 + 1023;
#pragma unroll
    for (int h = 0; h < 2; h++) {
        uint32_t a[kOzD][8];
#pragma unroll
        for (int d = 0; d < kOzD; d++) tmem_ld_x8(tb + kOzQ * d + 8 * h, a[d]);
        tmem_ld_wait();
#pragma unroll
        for (int d = 0; d < kOzD; d++) tmem_regs_ready(a[d]);
#pragma unroll
        for (int c = 0; c < 8; c++) {
            const long long Vh = (long long)((int)a[0][c] * 256 + (int)a[1][c]) * 256 + (int)a[2][c];
            const long long Vl = (long long)((int)a[3][c] * 256 + (int)a[4][c]) * 256 + (int)a[5][c];
            const double vh = __longlong_as_double(Vh + 0x4338000000000000LL) - 6755399441055744.0;
            const double vl = __longlong_as_double(Vl + 0x4338000000000000LL) - 6755399441055744.0;
            const int ex = max(ea + eR[16 * (w >> 2) + 8 * h + c], 0);
            acc[8 * h + c] = fma(vh, 16777216.0, vl) * __longlong_as_double((long long)ex << 52);
        }
    }
}

// panel task (m, k, J) of an int8-sliced matrix: R_J staged and cut into digits (global, for the
// updates and for this product), Wp_J = P_k R_J from the pivot's digits on the tensor cores (4
// column-quarter passes, 21 digit pairs each, same pipeline as oz_update), then Wp_J's digits and
// the step-k value of tile (K, J).  Shared memory: T (R_J, then P_k's digits, then Wp_J) + a 3-slot
// ring of R_J's quarter digit tiles.
constexpr int kOzPRing = kOzD * kOzQBytes;  // 24 KB
constexpr int kOzPanelSmem = 133120 + 3 * kOzPRing + 1024;
static_assert(kOzPanelSmem <= kUpdSmem, "the int8 panel fits the update kernel's shared memory");
__device__ void oz_panel(const MatDesc &m, int k, int J, double *dyn, OzState &o, int *sexp, int *eP, const int *pivflag) {
    const int n = m.n, k0 = k * B, K = k;
    const int64_t ld = m.ld;
    const int j0 = J * B;
    const int bk = min(B, n - k0), bj = min(B, n - j0);
    uint8_t *sm = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(dyn) + 1023) & ~uintptr_t(1023));
    double(*T)[B + 1] = reinterpret_cast<double(*)[B + 1]>(sm);
    uint8_t *ring = sm + 133120;
    uint8_t *rdig = oz_slices(m, k, J, 0);
    if (threadIdx.x >= kWorkers) {  // ---- producer warp: after R_J's digits are out, P_k's digits into
        if (threadIdx.x != kWorkers) return;  // T, R_J's quarter tiles through the ring, 4 passes
        const uint32_t sA = smem_u32(sm), sR = smem_u32(ring);
        auto load_ring = [&](int q) {  // the quarter of R_J's 6 digit tiles: one TMA op (box {128, 32, 6})
            cbar_expect(o.bar + OZ_R + q % 3, kOzPRing);
            tma_load_4d(ring + (q % 3) * kOzPRing, m.tmaps + OZ_MAP_R6, o.bar + OZ_R + q % 3, 0, kOzQ * q, 0, oz_set(m, k, J, 0));
        };
        oz_wait(o, OZ_RD);  // the workers are done with T and R_J's digits are in global memory
        // P_k only now: R_J's staging and digits do not need it, so they overlap the pivot's tail
        // (the task waited for everything else at its start)
        if (k >= 1) {
            int v;
            for (;;) {
                asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(pivflag) : "memory");
                if (v >= k + 1) break;
                __nanosleep(64);
            }
        }
        asm volatile("fence.proxy.async;" ::: "memory");
        asm volatile("fence.proxy.tensormap::generic.acquire.gpu [%0], 128;" ::"l"(m.tmaps + OZ_MAP_R6) : "memory");
        cbar_expect(o.bar + OZ_A, kOzSet + B * 4);
        bulk_row(sm, oz_pivdig(m, k), kOzSet, o.bar + OZ_A);
        bulk_row(eP, oz_pivexp(m, k), B * 4, o.bar + OZ_A);
        for (int q = 0; q < 3; q++) load_ring(q);
        for (int p = 0; p < 4; p++) {
            oz_wait(o, OZ_TE + (p & 1));
            oz_wait(o, OZ_R + p % 3);
            if (p == 0) oz_wait(o, OZ_A);
            tc_fence_after();
            oz_mma_pass<kOzD>(o.tmem + (p & 1) * (kOzD * kOzQ), sA, sR + (p % 3) * kOzPRing);
            mma_commit(o.bar + OZ_TF + (p & 1));
        }
        return;
    }
    // ---- workers
    const int bjp = min(B, (int)ld - j0);
    const bool trans = J < K;
    const int r0 = trans ? j0 : k0, c0 = trans ? k0 : j0, nr = trans ? bj : bk, nc = trans ? bk : bj;
#pragma unroll 16
    for (int it = 0; it < B * B / 256; it++) {
        const int e = it * 256 + threadIdx.x, r = e >> 7, c = e & (B - 1);
        const bool ok = r < nr && c < nc;
        cp_async8(&T[r][c], ok ? m.work + (int64_t)(r0 + r) * ld + c0 + c : m.work, ok);
    }
    cp_async_commit();
    cp_async_wait_0();
    WSYNC();
    TRACE(if (threadIdx.x == 0) g_trace_sub[blockIdx.x][2] = gtime();)
    if (trans) oz_slice<1>(T, rdig, oz_exps(m, k, 0) + j0, sexp);
    else oz_slice<0>(T, rdig, oz_exps(m, k, 0) + j0, sexp);
    mbar_arrive(o.bar + OZ_RD);  // this worker's digit stores are proxy-fenced and it is done with T
    TRACE(if (threadIdx.x == 0) g_trace_sub[blockIdx.x][0] = gtime();)
    // quarters 0 and 1 of Wp_J are parked in TMEM beyond the two accumulator sets (2 words per value),
    // quarters 2 and 3 stay in registers
    double acc[4][16];
    const uint32_t tpark = o.tmem + ((uint32_t)(32 * ((threadIdx.x >> 5) & 3)) << 16) + 2 * kOzD * kOzQ + 32 * (threadIdx.x >> 7);
    auto iter = [&](auto pc) {
        constexpr int pd = decltype(pc)::value;
        if (pd == 0) oz_wait(o, OZ_A);  // P_k's exponents visible to every worker
        oz_wait(o, OZ_TF + (pd & 1));
        tc_fence_after();
        oz_drain6(o.tmem + (pd & 1) * (kOzD * kOzQ), acc[pd], eP, sexp + kOzQ * pd);
        if (pd < 2) {
            uint32_t rr[32];
#pragma unroll
            for (int c = 0; c < 16; c++) {
                rr[2 * c] = (uint32_t)__double2loint(acc[pd][c]);
                rr[2 * c + 1] = (uint32_t)__double2hiint(acc[pd][c]);
            }
            tmem_st_x32(tpark + 64 * pd, rr);
        }
        tc_fence_before();
        mbar_arrive(o.bar + OZ_TE + (pd & 1));
        if (pd == 0 && threadIdx.x == 0) {  // pass 0's MMAs are complete: its ring slot takes quarter 3
            cbar_expect(o.bar + OZ_R + 0, kOzPRing);
            tma_load_4d(ring, m.tmaps + OZ_MAP_R6, o.bar + OZ_R + 0, 0, kOzQ * 3, 0, oz_set(m, k, J, 0));
        }
    };
    iter(std::integral_constant<int, 0>());
    iter(std::integral_constant<int, 1>());
    iter(std::integral_constant<int, 2>());
    iter(std::integral_constant<int, 3>());
    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
    tc_fence_before();
    WSYNC();  // every MMA completed: P_k's digits in T are dead
    tc_fence_after();
    TRACE(if (threadIdx.x == 0) g_trace_sub[blockIdx.x][1] = gtime();)
    {
        const int w = threadIdx.x >> 5, lane = threadIdx.x & 31, t = 32 * (w & 3) + lane, cb = 16 * (w >> 2);
#pragma unroll
        for (int q = 0; q < 2; q++) {
            uint32_t rr[32];
            tmem_ld_32x32b_x32(tpark + 64 * q, rr);
            tmem_ld_wait();
            tmem_regs_ready(rr);
#pragma unroll
            for (int c = 0; c < 16; c++) T[t][32 * q + cb + c] = __hiloint2double((int)rr[2 * c + 1], (int)rr[2 * c]);
        }
#pragma unroll
        for (int q = 2; q < 4; q++)
#pragma unroll
            for (int c = 0; c < 16; c++) T[t][32 * q + cb + c] = acc[q][c];  // Wp_J (zero outside bk rows)
    }
    WSYNC();
    TRACE(if (threadIdx.x == 0) g_trace_sub[blockIdx.x][3] = gtime();)
    oz_slice<0>(T, oz_slices(m, k, J, 1), oz_exps(m, k, 1) + j0, sexp);  // Wp_J's digits
    TRACE(WSYNC(); if (threadIdx.x == 0) g_trace_sub[blockIdx.x][4] = gtime();)
    // the step-k value of tile (K, J), 16-byte stores (W rows and tile columns are 16-byte aligned)
    if (!trans) {
        for (int e = threadIdx.x; e < bk * (B / 2); e += 256) {
            const int t = e >> 6, j = 2 * (e & (B / 2 - 1));
            if (j < bjp)  // bjp is a multiple of 16
                *reinterpret_cast<double2 *>(m.work + (int64_t)(k0 + t) * ld + j0 + j) = make_double2(T[t][j], T[t][j + 1]);
        }
    } else {  // M_JK <- Wp_J^T: row j of tile (J, K), consecutive threads along t
        for (int e = threadIdx.x; e < bj * (B / 2); e += 256) {
            const int j = e >> 6, t = 2 * (e & (B / 2 - 1));
            double *dst = m.work + (int64_t)(j0 + j) * ld + k0 + t;
            if (t + 1 < bk) *reinterpret_cast<double2 *>(dst) = make_double2(T[t][j], T[t + 1][j]);
            else if (t < bk) *dst = T[t][j];
        }
    }
}

// pass order of an update task: quarter-major (both steps of quarter q, then quarter q+1), so that a
// quarter's product is final after its last step's pass and its C read-modify-write overlaps the
// following passes' MMAs
__host__ __device__ constexpr int oz_pass_q(int p, int ns) { return ns == 2 ? p >> 1 : p; }
__host__ __device__ constexpr int oz_pass_st(int p, int ns) { return ns == 2 ? p & 1 : 0; }

// update task (m, k, I, J) of an int8-sliced matrix, ns = 1 or 2 steps: 4 ns column-quarter passes
// (step st = p / 4, quarter q = p % 4, TMEM set p & 1, ring slot p % 3).  The producer thread (256)
// loads and issues; the workers drain pass p-1 while pass p runs, then take the product through
// shared memory to a coalesced C read-modify-write (the C tile was prefetched into L2 at the task
// start).  Same contract as update_task's DMMA path.
__device__ int oz_update(const InvParams &P, const MatDesc &m, int k, int ns, int I, int J, double *dyn, const int *pflag,
                         OzState &o, bool &deferred, int *pivf) {
    const int n = m.n, i0 = I * B, j0 = J * B, bi = min(B, n - i0);
    const int64_t ld = m.ld;
    double *W = m.work;
    const int last = k + ns - 1, Q = 4 * ns;
    uint8_t *sm = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(dyn) + 1023) & ~uintptr_t(1023));
    uint8_t *ring = sm + 2 * kOzABytes;
    int *eA = reinterpret_cast<int *>(ring + 3 * kOzRBytes), *eB = eA + 2 * B;  // [2 steps][128] each
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int jw = (int)min((int64_t)B, ld - j0);  // columns of the tile inside ld (a multiple of 16)
    if (threadIdx.x >= kWorkers) {  // ---- producer warp
        if (threadIdx.x != kWorkers) return 0;
        asm volatile("fence.proxy.async;" ::: "memory");  // the digits (generic stores of other CTAs, flags acquired)
        for (int t = 0; t < 2; t++)  // the maps were written by tmap_store_kernel (generic proxy)
            asm volatile("fence.proxy.tensormap::generic.acquire.gpu [%0], 128;" ::"l"(m.tmaps + t) : "memory");
        const uint32_t sA = smem_u32(sm), sR = smem_u32(ring);
        // one TMA op per operand load: the quarter of the 5 B digit tiles (box {128, 32, 5}) and the 5 A tiles
        auto load_ring = [&](int p) {  // the B digits of pass p into slot p % 3
            cbar_expect(o.bar + OZ_R + p % 3, kOzRBytes);
            tma_load_4d(ring + (p % 3) * kOzRBytes, m.tmaps + OZ_MAP_R5, o.bar + OZ_R + p % 3, 0, kOzQ * oz_pass_q(p, ns), 0,
                        oz_set(m, k + oz_pass_st(p, ns), J, 1));
        };
        // in the order the passes consume them: step st's A digits, then pass st's B quarter (pass 0
        // starts after 100 KB instead of waiting behind step 1's A as well)
        for (int st = 0; st < ns; st++) {
            cbar_expect(o.bar + OZ_A + st, kOzABytes + 2 * B * 4);
            tma_load_4d(sm + st * kOzABytes, m.tmaps + OZ_MAP_A, o.bar + OZ_A + st, 0, 0, 0, oz_set(m, k + st, I, 0));
            bulk_row(eA + st * B, oz_exps(m, k + st, 0) + i0, B * 4, o.bar + OZ_A + st);
            bulk_row(eB + st * B, oz_exps(m, k + st, 1) + j0, B * 4, o.bar + OZ_A + st);
            load_ring(st);
        }
        for (int p = ns; p < 3 && p < Q; p++) load_ring(p);
        TRACE(const bool rec = Q == 8 && g_ozcnt[blockIdx.x] == 20;)
        for (int p = 0; p < Q; p++) {
            const int st = oz_pass_st(p, ns);
            TRACE(if (rec) g_ozt[blockIdx.x][40 + p] = clock64();)
            oz_wait(o, OZ_TE + p % kOzSets);  // its TMEM set was drained (or never used: pre-armed)
            TRACE(if (rec) g_ozt[blockIdx.x][48 + p] = clock64();)
            oz_wait(o, OZ_R + p % 3);
            if (p < ns) oz_wait(o, OZ_A + st);  // the first pass of each step
            TRACE(if (p == 0) g_trace_sub[blockIdx.x][0] = gtime();)
            TRACE(if (rec) g_ozt[blockIdx.x][p] = clock64();)
            tc_fence_after();
            oz_mma_pass<kOzS>(o.tmem + (p % kOzSets) * (kOzS * kOzQ), sA + st * kOzABytes, sR + (p % 3) * kOzRBytes);
            mma_commit(o.bar + OZ_TF + p % kOzSets);
            TRACE(if (rec) g_ozt[blockIdx.x][8 + p] = clock64();)
        }
        return 0;
    }
    // ---- workers
    if (threadIdx.x < bi) bulk_prefetch_l2(W + (int64_t)(i0 + threadIdx.x) * ld + j0, jw * 8);
    // acc: the current quarter's product (fp64, this thread's 16 columns); a finished quarter is parked in
    // TMEM beyond the accumulator sets (2 words per value) so that only one quarter lives in registers
    double acc[16];
    const uint32_t tpark = o.tmem + ((uint32_t)(32 * (w & 3)) << 16) + kOzSets * kOzS * kOzQ + 32 * (w >> 2);
    TRACE(const bool wrec = Q == 8 && g_ozcnt[blockIdx.x] == 20;)
    // passes written out with a compile-time index (static register indices)
    auto iter = [&](auto pc) {
        constexpr int pd = decltype(pc)::value;
        if (pd < Q) {
            const int q = oz_pass_q(pd, ns), st = oz_pass_st(pd, ns);
            if (pd < ns) oz_wait(o, OZ_A + st);  // exponents visible to every worker
            if (st == 0) {
#pragma unroll
                for (int c = 0; c < 16; c++) acc[c] = 0.0;
            }
            oz_wait(o, OZ_TF + pd % kOzSets);
            TRACE(if (wrec && threadIdx.x == 32) g_ozt[blockIdx.x][16 + pd] = clock64();)
            tc_fence_after();
            oz_drain(o.tmem + (pd % kOzSets) * (kOzS * kOzQ), acc, eA + st * B, eB + st * B + kOzQ * q);
            tc_fence_before();
            mbar_arrive(o.bar + OZ_TE + pd % kOzSets);
            if (threadIdx.x == 0 && pd + 3 < Q) {  // the drained pass's MMAs are complete: its ring slot is free
                const int pn = pd + 3;
                cbar_expect(o.bar + OZ_R + pn % 3, kOzRBytes);
                tma_load_4d(ring + (pn % 3) * kOzRBytes, m.tmaps + OZ_MAP_R5, o.bar + OZ_R + pn % 3, 0, kOzQ * oz_pass_q(pn, ns),
                            0, oz_set(m, k + oz_pass_st(pn, ns), J, 1));
            }
            if (st == ns - 1 && q < 3) {  // quarter q is final: park it
                uint32_t rr[32];
#pragma unroll
                for (int c = 0; c < 16; c++) {
                    rr[2 * c] = (uint32_t)__double2loint(acc[c]);
                    rr[2 * c + 1] = (uint32_t)__double2hiint(acc[c]);
                }
                tmem_st_x32(tpark + 64 * q, rr);
            }
            TRACE(if (wrec && threadIdx.x == 32) g_ozt[blockIdx.x][24 + pd] = clock64();)
        }
    };
    iter(std::integral_constant<int, 0>());
    iter(std::integral_constant<int, 1>());
    iter(std::integral_constant<int, 2>());
    iter(std::integral_constant<int, 3>());
    iter(std::integral_constant<int, 4>());
    iter(std::integral_constant<int, 5>());
    iter(std::integral_constant<int, 6>());
    iter(std::integral_constant<int, 7>());
    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
    TRACE(WSYNC(); if (threadIdx.x == 0 && Q == 8) g_ozcnt[blockIdx.x]++;)
    // every MMA completed (all TMEM-full phases observed): the A slots are dead
    tc_fence_before();
    WSYNC();
    tc_fence_after();
    TRACE(if (threadIdx.x == 0) g_trace_sub[blockIdx.x][1] = gtime();)
    const bool piv = I == last + 1 && J == last + 1;
    if (KFAC_OZ_BULK_RMW && !piv) {
        // stage -P (rows 16-byte aligned) and hand the read-modify-write of C to the L2: warp 0's lanes
        // issue 4 row reductions each; the workers are free as soon as the staging is written
        double(*Pn)[kPn] = reinterpret_cast<double(*)[kPn]>(dyn);
        const int r = 32 * (w & 3) + lane, cb = 16 * (w >> 2);
#pragma unroll
        for (int q = 0; q < 3; q++) {
            uint32_t rr[32];
            tmem_ld_32x32b_x32(tpark + 64 * q, rr);
            tmem_ld_wait();
            tmem_regs_ready(rr);
#pragma unroll
            for (int c = 0; c < 16; c++) Pn[r][32 * q + cb + c] = -__hiloint2double((int)rr[2 * c + 1], (int)rr[2 * c]);
        }
#pragma unroll
        for (int c = 0; c < 16; c++) Pn[r][96 + cb + c] = -acc[c];
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // generic staging writes -> bulk reads
        WSYNC();
        if (w == 0) {
            for (int rr = lane; rr < bi; rr += 32) bulk_red_add_f64(W + (int64_t)(i0 + rr) * ld + j0, &Pn[rr][0], jw * 8);
            bulk_commit();
        }
        deferred = true;
        return 0;
    }
    double(*Pt)[B + 1] = reinterpret_cast<double(*)[B + 1]>(dyn);
    {
        const int r = 32 * (w & 3) + lane, cb = 16 * (w >> 2);
#pragma unroll
        for (int q = 0; q < 3; q++) {
            uint32_t rr[32];
            tmem_ld_32x32b_x32(tpark + 64 * q, rr);
            tmem_ld_wait();
            tmem_regs_ready(rr);
#pragma unroll
            for (int c = 0; c < 16; c++) Pt[r][32 * q + cb + c] = __hiloint2double((int)rr[2 * c + 1], (int)rr[2 * c]);
        }
#pragma unroll
        for (int c = 0; c < 16; c++) Pt[r][96 + cb + c] = acc[c];
    }
    WSYNC();
    // coalesced C read-modify-write: warp w takes rows w, w + 8, ...; lane l columns l + 32 i; 32 loads
    // of a lane in flight (L2 hits: the tile was prefetched at the task start)
#pragma unroll 1
    for (int half = 0; half < 2; half++) {
        double cv[B / 16][4];
#pragma unroll
        for (int i8 = 0; i8 < B / 16; i8++) {
            const int rr = w + 8 * (i8 + half * (B / 16));
            const double *crow = W + (int64_t)(i0 + rr) * ld + j0;
#pragma unroll
            for (int i = 0; i < 4; i++) {
                const int c = lane + 32 * i;
                cv[i8][i] = (rr < bi && c < jw) ? __ldcg(crow + c) : 0.0;
            }
        }
#pragma unroll
        for (int i8 = 0; i8 < B / 16; i8++) {
            const int rr = w + 8 * (i8 + half * (B / 16));
#pragma unroll
            for (int i = 0; i < 4; i++) {
                const int c = lane + 32 * i;
                const double v = cv[i8][i] - Pt[rr][c];
                if (piv) Pt[rr][c] = (rr < bi && c < bi) ? v : (rr == c ? 1.0 : 0.0);  // fused next pivot, in place
                else if (rr < bi && c < jw) W[(int64_t)(i0 + rr) * ld + j0 + c] = v;
            }
        }
    }
    if (piv) {
        WSYNC();
        TRACE(if (threadIdx.x == 0) g_trace_sub[blockIdx.x][2] = gtime();)
        if (last >= 1 && threadIdx.x == 0) {  // its slot held P_{last-1}: step last-1's panels must be done
            int vv;
            do {
                asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(vv) : "l"(pflag) : "memory");
                if (vv < m.nt) __nanosleep(128);
            } while (vv < m.nt);
        }
        WSYNC();
        TRACE(if (threadIdx.x == 0) g_trace_sub[blockIdx.x][1] = gtime();)
        // the panels read P's digits only (no fp64 pivot slot); W_KK is written after P's release
        const int f = pivot_block(W, ld, i0, bi, nullptr, dyn, true, false);
        TRACE(WSYNC(); if (threadIdx.x == 0) g_trace_sub[blockIdx.x][3] = gtime();)
        if (!f) {  // P_{last+1}'s digits (S = -P, upper storage) for the next step's panel products
            WSYNC();
            pivot_fill_lower(reinterpret_cast<double(*)[B + 1]>(dyn));
            WSYNC();
            oz_slice<3>(reinterpret_cast<const double(*)[B + 1]>(dyn), oz_pivdig(m, last + 1), oz_pivexp(m, last + 1), o.sexp, bi);
            // release P_{last+1} now: the next step's panels need only its digits (the task's end
            // repeats the same release after the tile stamp)
            __threadfence();
            WSYNC();
            if (threadIdx.x == 0) asm volatile("st.release.gpu.global.b32 [%0], %1;" ::"l"(pivf), "r"(last + 2) : "memory");
        }
        TRACE(WSYNC(); if (threadIdx.x == 0) g_trace_sub[blockIdx.x][4] = gtime();)
        pivot_write_w(reinterpret_cast<const double(*)[B + 1]>(dyn), W, ld, i0, bi);  // fenced by the task's end
        return f;
    }
    deferred = true;
    return 0;
}

// ---- panel task (m, k, J): R_J = block row K (from upper storage), Wp_J = P_k R_J.  The task also
// gives tile (K, J) its step-k value Wp_J (M_KJ <- Wp_J, or M_JK <- Wp_J^T left of the diagonal):
// nothing else reads that tile at step k, so the row / column K "copy" updates have no work left.
__device__ void panel_task(const MatDesc &m, int k, int J, double *dyn, Ring &ring, bool oz, OzState &ozs,
                           const int *pivflag) {
    if (oz) {
        oz_panel(m, k, J, dyn, ozs, ozs.sexp, ozs.eP, pivflag);
        return;
    }
    const int n = m.n, k0 = k * B, K = k;
    const int64_t ld = m.ld;
    const int j0 = J * B;
    const int bk = min(B, n - k0), bj = min(B, n - j0);
    double *R = panel_R(m, k), *Wp = panel_Wp(m, k);
    // R_J (rows t < bk, cols j < bj; zero up to the 16-aligned ld) staged through shared memory so
    // that both the read of W (upper storage, possibly transposed) and the write of R coalesce.
    // The tile comes in by 8-byte cp.async (all 64 loads of a thread in flight at once).
    double(*T)[B + 1] = reinterpret_cast<double(*)[B + 1]>(dyn);
    const int bjp = min(B, (int)ld - j0);
    const bool trans = J < K;  // block row K left of the diagonal lives in column K of the upper storage
    const int r0 = trans ? j0 : k0, c0 = trans ? k0 : j0, nr = trans ? bj : bk, nc = trans ? bk : bj;
#pragma unroll 16
    for (int it = 0; it < B * B / 256; it++) {
        const int e = it * 256 + threadIdx.x, r = e >> 7, c = e & (B - 1);
        const bool ok = r < nr && c < nc && (J != K || c >= r);
        cp_async8(&T[r][c], ok ? m.work + (int64_t)(r0 + r) * ld + c0 + c : m.work, ok);
    }
    cp_async_commit();
    cp_async_wait_0();
    WSYNC();
    for (int e = threadIdx.x; e < bk * B; e += 256) {
        const int t = e >> 7, j = e & (B - 1);
        if (j >= bjp) continue;
        double v;
        if (trans) v = T[j][t];
        else if (J == K) v = (j >= t) ? T[t][j] : T[j][t];
        else v = T[t][j];
        R[(int64_t)t * ld + j0 + j] = v;
    }
    double acc[8][8];
#pragma unroll
    for (int p = 0; p < 8; p++)
#pragma unroll
        for (int q = 0; q < 8; q++) acc[p][q] = 0.0;
    // Wp[i][j] = sum_t P[t][i] R[t][j]   (P symmetric, zero outside bk).  R is read straight from the
    // staged tile T (resident; zero outside the block), only P streams through the ring placed
    // after T -- the product does not wait for R's global write.
    const Seg seg{pivot_slot(m, k), B, B, nullptr, 0, 0, bk}, none{nullptr, 0, 0, nullptr, 0, 0, 0};
    if (trans) tile_product<2>(seg, none, acc, dyn + B * (B + 1), ring, &T[0][0]);
    else tile_product<1>(seg, none, acc, dyn + B * (B + 1), ring, &T[0][0]);
    WSYNC();  // the product's staging buffers are free: the result goes through T
#pragma unroll
    for (int p = 0; p < 8; p++)
#pragma unroll
        for (int q = 0; q < 8; q++) T[tile_row(p)][tile_col(q)] = acc[p][q];
    WSYNC();
    // Wp_J into the panel buffer (rows whole up to ld) and the step-k value of tile (K, J)
    for (int e = threadIdx.x; e < bk * B; e += 256) {
        const int t = e >> 7, j = e & (B - 1);
        if (j >= bjp) continue;
        const double v = T[t][j];
        Wp[(int64_t)t * ld + j0 + j] = v;
        if (!trans) m.work[(int64_t)(k0 + t) * ld + j0 + j] = v;
    }
    if (trans)  // M_JK <- Wp_J^T: row j of tile (J, K), consecutive threads along t
        for (int e = threadIdx.x; e < bj * B; e += 256) {
            const int j = e >> 7, t = e & (B - 1);
            if (t < bk) m.work[(int64_t)(j0 + j) * ld + k0 + t] = T[t][j];
        }
}

// ---- update task (m, k, I, J): rank-B sweep update of upper tile (I, J); the task of tile
// (K+1, K+1) then inverts that block (the next step's pivot).  Returns 0 or a pivot failure.
// nsteps = 1: the update of tile (I, J) at step k (incl. the copy tiles of row / column k);
// nsteps = 2: the merged update for steps k and k+1 (I, J not in {k, k+1}).
__device__ int update_task(const InvParams &P, const MatDesc &m, int k, int nsteps, int I, int J, double *dyn,
                           const int *pflag, uint64_t *cbar, uint32_t &cph, Ring &ring, bool &deferred, bool oz,
                           OzState &ozs, int *pivf) {
    const int n = m.n, k0 = k * B, K = k;
    const int64_t ld = m.ld;
    const int bk = min(B, n - k0);
    const int i0 = I * B, j0 = J * B;
    const int bi = min(B, n - i0), bj = min(B, n - j0);
    const double *R = panel_R(m, k), *Wp = panel_Wp(m, k);
    double *W = m.work;
    if (I == K && J == K) return 0;  // M_KK <- -P_K: written by the pivot itself (pivot_block)
    if (I == K || J == K) return 0;  // M_KJ <- Wp_J / M_IK <- Wp_I^T: written by the panel tasks
    if (oz) return oz_update(P, m, k, nsteps, I, J, dyn, pflag, ozs, deferred, pivf);
    double acc[8][8];
#pragma unroll
    for (int p = 0; p < 8; p++)
#pragma unroll
        for (int q = 0; q < 8; q++) acc[p][q] = 0.0;
    // the C tile M_IJ streams into shared memory in slices, one per K chunk of the product
    // (its HBM latency hides behind the tensor-core work instead of preceding it)
    // the C tile M_IJ comes in by one asynchronous bulk copy per row (async proxy, completion on an
    // mbarrier), issued before the product and awaited only at its end: it never stalls the
    // product's chunk pipeline.  Rows are copied whole up to the leading dimension (the padding
    // columns are never read).
    double *Cs = dyn + kTileSmem / 8;
    {
        const uint32_t rowb = (uint32_t)min((int64_t)B, ld - j0) * 8;
        if (threadIdx.x == 0) cbar_expect(cbar, rowb * bi);
        WSYNC();  // expect_tx before any complete_tx
        if (threadIdx.x < bi) bulk_row(Cs + threadIdx.x * SLD, W + (int64_t)(i0 + threadIdx.x) * ld + j0, rowb, cbar);
    }
    // M_IJ -= R_I^T Wp_J : acc[i][j] = sum_t R[t][i0+i] Wp[t][j0+j]   (for each step of the task)
    const int aw = min((int64_t)B, ld - i0), bw = min((int64_t)B, ld - j0);
    const Seg s0{R + i0, ld, aw, Wp + j0, ld, bw, bk};
    const Seg s1{panel_R(m, k + 1) + i0, ld, aw, panel_Wp(m, k + 1) + j0, ld, bw, nsteps == 2 ? min(B, n - k0 - B) : 0};
    tile_product(s0, s1, acc, dyn, ring);
    TRACE(if (threadIdx.x == 0) g_trace_sub[blockIdx.x][0] = gtime();)
    cbar_wait(cbar, cph);
    cph ^= 1;
    TRACE(if (threadIdx.x == 0) g_trace_sub[blockIdx.x][1] = gtime();)
    const int last = k + nsteps - 1;  // the step whose value the tile now holds
    if (I == last + 1 && J == last + 1) {
        // fused next pivot: P_{K+1} = (updated M_{K+1,K+1})^-1.  The updated tile goes straight into
        // the pivot's shared-memory copy: its global value is dead (the next step's (K,K) tile
        // overwrites it with -P and no panel reads the pivot column).
#pragma unroll
        for (int p = 0; p < 8; p++)
#pragma unroll
            for (int q = 0; q < 8; q++) acc[p][q] = Cs[tile_row(p) * SLD + tile_col(q)] - acc[p][q];
        WSYNC();  // Cs is read; the pivot's smem overlaps it
        double(*S)[B + 1] = reinterpret_cast<double(*)[B + 1]>(dyn);
#pragma unroll
        for (int p = 0; p < 8; p++) {
            const int i = tile_row(p);
#pragma unroll
            for (int q = 0; q < 8; q++) {
                const int j = tile_col(q);
                S[i][j] = (i < bi && j < bi) ? acc[p][q] : (i == j ? 1.0 : 0.0);
            }
        }
        WSYNC();
        // its slot held P_{last-1}: every step-(last-1) panel task must be done reading it
        if (last >= 1 && threadIdx.x == 0) {
            int v;
            do {
                asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(pflag) : "memory");
                if (v < m.nt) __nanosleep(128);
            } while (v < m.nt);
        }
        WSYNC();
        return pivot_block(W, ld, i0, bi, pivot_slot(m, last + 1), dyn, true);
    }
    // column pairs (16-byte stores); rows are written whole up to the leading dimension: the lower
    // half of a diagonal tile and the padding columns are never read (upper storage).  The task
    // does not wait for the stores: the kernel loop releases the tile's stamp at the start of the
    // CTA's next task (the drain overlaps the next task fetch).
#pragma unroll
    for (int p = 0; p < 8; p++) {
        const int i = tile_row(p);
        if (i >= bi) continue;
#pragma unroll
        for (int q = 0; q < 8; q += 2) {
            const int j = tile_col(q);
            if (j0 + j >= ld) continue;
            const double2 c = *reinterpret_cast<const double2 *>(Cs + i * SLD + j);
            *reinterpret_cast<double2 *>(W + (int64_t)(i0 + i) * ld + j0 + j) = make_double2(c.x - acc[p][q], c.y - acc[p][q + 1]);
        }
    }
    deferred = true;
    return 0;
}

__device__ __forceinline__ void wait_ge(const int *f, int target) {
    int v;
    for (;;) {
        asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(f) : "memory");
        if (v >= target) return;
        __nanosleep(200);
    }
}
__device__ __forceinline__ int upper_index(int I, int J, int nt) { return I * nt - I * (I - 1) / 2 + (J - I); }

// step 0 only: P_0 (later pivots are fused into the previous step's tile (K+1, K+1) update)
__global__ void __launch_bounds__(256, 1) pivot_kernel(const __grid_constant__ InvParams P) {
    const MatDesc &m = P.m[blockIdx.x];
    if (*m.status != 0) return;
    extern __shared__ double dyn[];
    const int f = pivot_block(m.work, m.ld, 0, min(B, m.n), P.ozflag[blockIdx.x] ? nullptr : pivot_slot(m, 0), dyn);
    if (f && threadIdx.x == 0) *m.status = f;
    if (!f && P.ozflag[blockIdx.x]) {  // P_0's digits for step 0's int8 panel products
        __shared__ __align__(16) int sexp[3 * B];
        WSYNC();
        pivot_fill_lower(reinterpret_cast<double(*)[B + 1]>(dyn));
        WSYNC();
        oz_slice<3>(reinterpret_cast<const double(*)[B + 1]>(dyn), oz_pivdig(m, 0), oz_pivexp(m, 0), sexp, min(B, m.n));
    }
}

#include "inverse_tasks.hpp"
using namespace kfac_inv;

// one thread per (pair, matrix): the matrix's cursor in each segment of the pair's list is the
// segment's start plus the counts of the matrices before it
__global__ void inverse_tasks_kernel(const __grid_constant__ InvParams P) {
    const int pr = blockIdx.x, m = blockIdx.y * blockDim.x + threadIdx.x;
    if (m >= P.nm) return;
    const int k = 2 * pr, nt = P.m[m].nt;
    if (nt <= k) return;
    int tot[kSegs], pre[kSegs], c[kSegs];
    for (int q = 0; q < kSegs; q++) tot[q] = pre[q] = 0;
    for (int i = 0; i < P.nm; i++) {
        pair_counts(P.m[i].nt, k, c);
        for (int q = 0; q < kSegs; q++) {
            tot[q] += c[q];
            if (i < m) pre[q] += c[q];
        }
    }
    int cur[kSegs], base = 0;
    for (int q = 0; q < kSegs; q++) {
        cur[q] = base + pre[q];
        base += tot[q];
    }
    pair_emit(nt, k, m, cur, P.tasks + P.step_begin[pr]);
}

// L2 prefetch (one warp) of what task t will read: t = the current task + gridDim.x, which some CTA
// takes about one task duration from now (tasks are handed out in order).  Stale lines are harmless
// (L2 is coherent: a later write of the producer updates them).
__device__ void prefetch_task(const InvParams &P, int t, int lane) {
    if (t >= P.total_tasks) return;
    const int4 task = P.tasks[t];
    const int k = task.x, I = task.w >> 16, J = task.w & 0xffff;
    const MatDesc &m = P.m[task.z];
    const int n = m.n;
    const int64_t ld = m.ld;
    if (task.y == 1 || task.y == 2) {
        if (!P.ozflag[task.z] || I == k || J == k) return;
        const int ns = task.y == 2 ? 2 : 1, i0 = I * B, j0 = J * B, bi = min(B, n - i0);
        const int jw = (int)min((int64_t)B, ld - j0);
        if (lane < 2 * ns) bulk_prefetch_l2(oz_slices(m, k + (lane >> 1), (lane & 1) ? J : I, lane & 1), kOzABytes);
        for (int r = lane; r < bi; r += 32) bulk_prefetch_l2(m.work + (int64_t)(i0 + r) * ld + j0, jw * 8);
    } else if (J != k) {  // panel: the staged block of row K (upper storage; transposed left of the diagonal)
        const int k0 = k * B, j0 = J * B, bk = min(B, n - k0), bj = min(B, n - j0);
        const bool trans = J < k;
        const int r0 = trans ? j0 : k0, c0 = trans ? k0 : j0, nr = trans ? bj : bk, nc = trans ? bk : bj;
        for (int r = lane; r < nr; r += 32) bulk_prefetch_l2(m.work + (int64_t)(r0 + r) * ld + c0, ((nc * 8 + 15) / 16) * 16);
    }
}

// ---- the whole sweep as ONE persistent launch: CTAs take tasks from an atomic counter in the
// order above, and each task waits on the stamps of the tasks it reads:
//   panel (m,k,J):   tile (K,J) of step k-1, P_k, and (buffer reuse) all of step k-2's updates
//   update (m,k,I,J): panels I and J of step k (P_k for the (K,K) tile) and its own step k-1 value;
//                    the fused pivot also waits for step k-1's panels (pivot slot reuse)
// Waits only point to earlier tasks, which are held by running CTAs: no deadlock.  Step k+1's
// panels and updates start while step k's tail is still running (look-ahead).
__global__ void __launch_bounds__(kThreads, 1) inverse_kernel(const __grid_constant__ InvParams P) {
    extern __shared__ double dyn[];
    __shared__ int next;
    __shared__ uint64_t cbar;  // C tile bulk loads of update tasks
    __shared__ uint64_t ring_full[kStages], ring_empty[kStages];
    __shared__ uint64_t ozbar[OZ_NBAR];  // int8-sliced updates: operand loads, TMEM full / empty
    __shared__ uint32_t tmem_slot;
    __shared__ __align__(16) int oz_sexp[3 * B], oz_eP[B];  // exponents + 128 doubles of reduction scratch
    uint32_t cph = 0;
    Ring ring{ring_full, ring_empty, 0};
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(s2u(&cbar)) : "memory");
        for (int st = 0; st < kStages; st++) {
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 256;" ::"r"(s2u(ring_full + st)) : "memory");
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 8;" ::"r"(s2u(ring_empty + st)) : "memory");
        }
        for (int b = 0; b < OZ_NBAR; b++) mbar_init(ozbar + b, ((b >= OZ_TE && b < OZ_TE + kOzSets) || b == OZ_RD) ? kWorkers : 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (threadIdx.x < 32) tmem_alloc(&tmem_slot, 512);  // one CTA per SM (shared memory): all of TMEM
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    OzState ozs{ozbar, 0u, tmem_slot, oz_sexp, oz_eP};
    const bool producer = threadIdx.x >= kWorkers;  // warp 8: int8 operand loads and MMA issue only
    if (!producer) {
        for (int b = 0; b < kOzSets; b++) mbar_arrive(ozbar + OZ_TE + b);  // the TMEM accumulator sets start empty
    }
    // deferred release of the previous update task (its tile stores may still be draining)
    bool pend = false, pend_two = false;
    int *pend_tile = nullptr, *pend_done = nullptr;
    int pend_val = 0;
    for (;;) {
        if (threadIdx.x < 32) {  // an update's bulk C reductions (warp 0): staging read before it is reused,
            bulk_wait_read();    // writes complete before the tile's release below
            if (pend) bulk_wait_all();
            __syncwarp();
        }
        asm volatile("fence.proxy.async;" ::: "memory");  // this task's generic accesses before the next one's bulk copies
        __syncthreads();  // the previous task is done with shared memory and `next`
        if (threadIdx.x == 0) {
            const int gn = atomicAdd(P.counter, 1);
            if (pend) {  // the previous update's stores precede this release (bar.sync + cumulative fence);
                         // done before any wait of the next task: the deadlock-freedom argument needs it
                __threadfence();
                asm volatile("st.release.gpu.global.b32 [%0], %1;" ::"l"(pend_tile), "r"(pend_val) : "memory");
                atomicAdd(pend_done, 1);
                if (pend_two) atomicAdd(pend_done + 1, 1);
            }
            next = gn;
        }
        pend = false;
        __syncthreads();
        const int g = next;
        if (g >= P.total_tasks) break;

        TRACE(long long tr0 = gtime(); long long tr1 = 0; int trI = -1, trJ = -1, trkind = 0;)
#ifdef KFAC_INV_PREFETCH  // experiment: L2 prefetch one round ahead (measured slower: 20.0 -> 24.5 us per merged task)
        if ((threadIdx.x >> 5) == 1) prefetch_task(P, g + gridDim.x, threadIdx.x & 31);
#endif
        const int4 task = P.tasks[g];
        const int k = task.x, mi = task.z, I = task.w >> 16, J = task.w & 0xffff;
        const MatDesc &m = P.m[mi];
        const int nt = m.nt;
        const bool oz = P.ozflag[mi] != 0;
        if (task.y == 0 || task.y == 3) {
            // ---------------- panel task (kind 0) / chain task (kind 3: panel (k, J = k+1), then the
            // update of tile (J, J) at step k and its inverse P_{k+1}, in one task)
            if (threadIdx.x < 32) {  // lanes poll one stamp each: one L2 round trip, not three
                const int lane = threadIdx.x;
                if (lane == 0 && k >= 1)
                    wait_ge(P.tileflag + m.tile_begin + (J >= k ? upper_index(k, J, nt) : upper_index(J, k, nt)), k);
                if (lane == 1 && k >= 1 && !oz) wait_ge(P.pivflag + mi, k + 1);  // int8 panels: inside, before P's digits
                if (lane == 2 && k >= kPanelBufs)  // its buffer's previous user: all updates of step k - kPanelBufs
                    wait_ge(P.tiles_done + m.col_begin + k - kPanelBufs, nt * (nt + 1) / 2);
                if (lane == 3 && task.y == 3 && k >= 1) wait_ge(P.tileflag + m.tile_begin + upper_index(J, J, nt), k);
                __syncwarp();  // orders the lanes' acquires before lane 0's status read
                if (lane == 0) next = *(volatile int *)m.status;  // one decision for the whole CTA
            }
            __syncthreads();
            TRACE(tr1 = gtime(); trJ = J; trkind = task.y == 3 ? 5 : 0;)
            const bool live = next == 0;
            if (live && J != k && (oz || !producer)) panel_task(m, k, J, dyn, ring, oz, ozs, P.pivflag + mi);  // R_K / P R_K are never read
            TRACE(if (task.y == 3 && threadIdx.x == 0) g_trace_sub[blockIdx.x][0] = gtime();)
            __threadfence();
            __syncthreads();
            if (threadIdx.x == 0) {
                asm volatile("st.release.gpu.global.b32 [%0], %1;" ::"l"(P.colflag + m.col_begin + J), "r"(k + 1) : "memory");
                atomicAdd(P.panels_done + m.col_begin + k, 1);
            }
            if (task.y == 3) {
                int f = 0;
                bool deferred = false;  // stays false: the pivot path writes W itself
                if (live && (oz || !producer))
                    f = update_task(P, m, k, 1, J, J, dyn, P.panels_done + m.col_begin + (k >= 1 ? k - 1 : 0), &cbar, cph,
                                    ring, deferred, oz, ozs, P.pivflag + mi);
                if (f && threadIdx.x == 0) *m.status = f;
                __threadfence();
                __syncthreads();
                if (threadIdx.x == 0) {
                    asm volatile("st.release.gpu.global.b32 [%0], %1;" ::"l"(P.tileflag + m.tile_begin + upper_index(J, J, nt)),
                                 "r"(k + 1)
                                 : "memory");
                    asm volatile("st.release.gpu.global.b32 [%0], %1;" ::"l"(P.pivflag + mi), "r"(k + 2) : "memory");
                    atomicAdd(P.tiles_done + m.col_begin + k, 1);
                }
            }
        } else {
            // ---------------- update task (kind 1) / merged update of steps k, k+1 (kind 2)
            const int ns = task.y == 2 ? 2 : 1, last = k + ns - 1;
            if (threadIdx.x < 32) {
                // panels of step `last` (for a merged task they complete after step k's, which
                // they depend on), P_k for the (K, K) copy, the tile's step k-1 value
                const int lane = threadIdx.x;
                if (lane == 0 && I != k) wait_ge(P.colflag + m.col_begin + I, last + 1);
                if (lane == 1 && J != k && J != I) wait_ge(P.colflag + m.col_begin + J, last + 1);
                if (lane == 2 && I == k && J == k && k >= 1) wait_ge(P.pivflag + mi, k + 1);
                if (lane == 3 && k >= 1) wait_ge(P.tileflag + m.tile_begin + upper_index(I, J, nt), k);
                __syncwarp();
                if (lane == 0) next = *(volatile int *)m.status;  // one decision for the whole CTA
            }
            __syncthreads();
            TRACE(tr1 = gtime(); trI = I; trJ = J; trkind = (I == last + 1 && J == last + 1) ? 2 : (ns == 2 ? 3 : ((I == k || J == k) ? 4 : 1));)
            int f = 0;
            bool deferred = false;
            if (next == 0 && (oz || !producer))
                f = update_task(P, m, k, ns, I, J, dyn, P.panels_done + m.col_begin + (last >= 1 ? last - 1 : 0), &cbar,
                                cph, ring, deferred, oz, ozs, P.pivflag + mi);
            if (deferred) {  // tile stores still draining: release at the next task's start
                pend = true;
                pend_tile = P.tileflag + m.tile_begin + upper_index(I, J, nt);
                pend_val = last + 1;
                pend_done = P.tiles_done + m.col_begin + k;
                pend_two = ns == 2;
                            }
            if (f && threadIdx.x == 0) *m.status = f;
            if (!deferred) __threadfence();
            __syncthreads();
            if (threadIdx.x == 0 && !deferred) {
                asm volatile("st.release.gpu.global.b32 [%0], %1;" ::"l"(P.tileflag + m.tile_begin + upper_index(I, J, nt)),
                             "r"(last + 1)
                             : "memory");
                if (I == last + 1 && J == last + 1)
                    asm volatile("st.release.gpu.global.b32 [%0], %1;" ::"l"(P.pivflag + mi), "r"(last + 2) : "memory");
                atomicAdd(P.tiles_done + m.col_begin + k, 1);
                if (ns == 2) atomicAdd(P.tiles_done + m.col_begin + k + 1, 1);
            }
        }
#ifdef INV_TRACE
        if (threadIdx.x == 0 && g < (1 << 17)) {
            int sm;
            asm volatile("mov.u32 %0, %%smid;" : "=r"(sm));
            g_trace[g] = TraceRec{g, k, trkind, trI, trJ, sm, tr0, tr1, gtime(), g_trace_sub[blockIdx.x][0], g_trace_sub[blockIdx.x][1],
                                  g_trace_sub[blockIdx.x][2], g_trace_sub[blockIdx.x][3], g_trace_sub[blockIdx.x][4],
                                  g_trace_sub[blockIdx.x][5]};
        }
#endif
    }
    tc_fence_before();
    __syncthreads();
    if (threadIdx.x < 32) {
        tc_fence_after();
        tmem_dealloc(tmem_slot, 512);
    }
}

// ---- epilogue: inv = -M (symmetric, full fp32) from the upper storage.  Each upper 64 x 64 tile is
// read once (coalesced, through shared memory) and written to both of its output blocks.
// the precondition's 3xTF32 operand (precond.cu split_kernel's format): hi = rn_tf32(v), lo = rn_tf32(v - hi),
// planes [2][n][kp], kp = n rounded up to 4 (the padding columns zero)
__device__ __forceinline__ float tf32_rn_inv(float x) {
    return __uint_as_float((__float_as_uint(x) + 0x1000u) & 0xFFFFE000u);
}
__device__ __forceinline__ void split_store(float *split, int n, int kp, int i, int j, float v) {
    const float hi = tf32_rn_inv(v);
    split[(int64_t)i * kp + j] = hi;
    split[(int64_t)n * kp + (int64_t)i * kp + j] = tf32_rn_inv(v - hi);
}
__global__ void __launch_bounds__(256) finalize_kernel(const __grid_constant__ InvParams P) {
    const int rm = flat_matrix(P.fin_begin, P.nm, blockIdx.x), bx = blockIdx.x - P.fin_begin[rm];
    const MatDesc &m = P.m[rm];
    const int n = m.n, kp = (n + 3) / 4 * 4;
    if (m.split && bx == 0 && kp > n)
        for (int i = threadIdx.x; i < n; i += blockDim.x)
            for (int j = n; j < kp; j++) m.split[(int64_t)i * kp + j] = m.split[(int64_t)n * kp + (int64_t)i * kp + j] = 0.f;
    const int64_t ld = m.ld;
    const int nt = (n + kFinT - 1) / kFinT, npairs = nt * (nt + 1) / 2;
    __shared__ double T[kFinT][kFinT + 1];
    const int tx = threadIdx.x & (kFinT - 1), ty = threadIdx.x / kFinT;  // 64 columns x 4 row groups
    constexpr int RG = 256 / kFinT;
    for (int t = bx * kFinTiles; t < min(npairs, (bx + 1) * kFinTiles); t++) {
        // tile t of the row-major upper tile order: row bi starts at S(bi) = bi nt - bi (bi - 1) / 2
        // (closed form + fix-up; a walk over the rows cost ~nt ALU steps per tile)
        const double b2 = 2.0 * nt + 1.0;
        int bi = (int)((b2 - sqrt(b2 * b2 - 8.0 * t)) * 0.5);
        bi = max(0, min(bi, nt - 1));
        while (bi > 0 && bi * nt - bi * (bi - 1) / 2 > t) bi--;
        while (bi + 1 < nt && (bi + 1) * nt - (bi + 1) * bi / 2 <= t) bi++;
        const int bj = bi + (t - (bi * nt - bi * (bi - 1) / 2));
        __syncthreads();
#pragma unroll
        for (int k = 0; k < kFinT / RG; k++) {  // 16 loads of a thread in flight
            const int r = ty + RG * k, i = bi * kFinT + r, j = bj * kFinT + tx;
            T[r][tx] = (i < n && j < n) ? m.work[(int64_t)i * ld + j] : 0.0;
        }
        __syncthreads();
        // writes: 16 threads x 4 consecutive columns per row (16-byte stores of the inverse when n is a
        // multiple of 4, and of both split planes: kp is), 16 rows per pass
        const int tq = threadIdx.x & 15, rq = threadIdx.x >> 4;
#pragma unroll 2
        for (int k = 0; k < kFinT / 16; k++) {
            const int r = rq + 16 * k;
#pragma unroll
            for (int side = 0; side < 2; side++) {
                if (side == 1 && bi == bj) break;
                // side 0: block (bi, bj), element (r, c); side 1: block (bj, bi), element (r, c) = -T[c][r]
                const int i = (side ? bj : bi) * kFinT + r, j = (side ? bi : bj) * kFinT + 4 * tq;
                if (i >= n || j >= n) continue;
                float v[4];
#pragma unroll
                for (int c = 0; c < 4; c++) {
                    const int cc = 4 * tq + c;
                    v[c] = (float)(-(side ? T[cc][r] : ((bi < bj || r <= cc) ? T[r][cc] : T[cc][r])));
                }
                float *dst = m.inv + (int64_t)i * n + j;
                if ((n & 3) == 0 && j + 3 < n) {
                    *reinterpret_cast<float4 *>(dst) = make_float4(v[0], v[1], v[2], v[3]);
                } else {
#pragma unroll
                    for (int c = 0; c < 4; c++)
                        if (j + c < n) dst[c] = v[c];
                }
                if (m.split) {
                    float hi[4], lo[4];
#pragma unroll
                    for (int c = 0; c < 4; c++) {
                        hi[c] = tf32_rn_inv(v[c]);
                        lo[c] = tf32_rn_inv(v[c] - hi[c]);
                        if (j + c >= n) hi[c] = lo[c] = 0.f;  // the padding columns (kp > n) stay zero
                    }
                    float *sh = m.split + (int64_t)i * kp + j, *sl = sh + (int64_t)n * kp;
                    if (j + 3 < kp) {  // kp is a multiple of 4 and j of 4: always true
                        *reinterpret_cast<float4 *>(sh) = make_float4(hi[0], hi[1], hi[2], hi[3]);
                        *reinterpret_cast<float4 *>(sl) = make_float4(lo[0], lo[1], lo[2], lo[3]);
                    }
                }
            }
        }
    }
}

#ifdef INV_TRACE
extern "C" __attribute__((visibility("default"))) int kfac_debug_ozt(void *host) {
    return (int)cudaMemcpyFromSymbol(host, g_ozt, sizeof(g_ozt));
}
extern "C" __attribute__((visibility("default"))) int kfac_debug_ozprof(void *host) {
    return (int)cudaMemcpyFromSymbol(host, g_ozprof, sizeof(g_ozprof));
}
extern "C" __attribute__((visibility("default"))) int kfac_debug_inverse_trace(void *host, int max) {
    const int n = max < (1 << 17) ? max : (1 << 17);
    return (int)cudaMemcpyFromSymbol(host, g_trace, sizeof(TraceRec) * n);
}
#endif

#ifdef PIVOT_DBG
extern "C" __attribute__((visibility("default"))) int kfac_debug_pclk(void *host) {
    return (int)cudaMemcpyFromSymbol(host, g_pacc, sizeof(g_pacc));
}
#endif
int64_t inverse_ld(int n) { return (n + 15) / 16 * 16; }
static int64_t pair_doubles(int npairs) { return ((8 * (int64_t)npairs + 15) / 16) * 16; }
static int64_t state_ints(int npairs, int64_t sum_nt, int64_t sum_tiles) {
    return 16 + 4 * (int64_t)npairs + 3 * sum_nt + sum_tiles;
}
static int64_t tasks_offset(int npairs, int64_t sum_nt, int64_t sum_tiles) {  // bytes
    return pair_doubles(npairs) * 8 + ((state_ints(npairs, sum_nt, sum_tiles) + 3) / 4) * 16;
}
static int64_t tmaps_offset(int npairs, int64_t sum_nt, int64_t sum_tiles, int64_t sum_tasks) {  // bytes, 128-aligned
    return (tasks_offset(npairs, sum_nt, sum_tiles) + sum_tasks * 16 + 127) / 128 * 128;
}
int64_t inverse_scratch_bytes(int npairs, int64_t sum_nt, int64_t sum_tiles, int64_t sum_tasks) {
    // pair data (8 doubles per pair) | counter + pivflag (2 npairs) + ozflag (2 npairs) | colflag,
    // panels_done, tiles_done (sum_nt each) | tileflag | task records (16 B each) | 3 TMA maps per matrix
    return tmaps_offset(npairs, sum_nt, sum_tiles, sum_tasks) + 2 * (int64_t)npairs * 3 * 128 + 256;
}
// tasks of one n x n matrix's sweep: nt panels + nt (nt + 1) / 2 tiles per step, nt steps
int64_t inverse_tasks(int n) {
    const int64_t nt = (n + B - 1) / B;
    return nt * (nt + nt * (nt + 1) / 2);
}
int64_t inverse_ws_doubles(int n) {
    // working matrix | fp64 R / Wp panels | pivot slots | int8 digit tiles | digit exponents
    const int64_t ld = inverse_ld(n), nt = (n + B - 1) / B;
    const int64_t oz = (kPanelBufs * nt * 2 * (int64_t)kOzSet + kPanelBufs * 2 * nt * B * 4 + 2 * (kOzSet + B * 4)) / 8;
    return (n * ld + 2 * kPanelBufs * (int64_t)B * ld + 2 * (int64_t)B * B + oz + 31) / 32 * 32;
}

// the digit tile maps of one inverse launch, written to global memory by a kernel (parameter space
// holds up to 32 KB); the TMA reads them through the tensormap proxy (released here, acquired by the
// producer before its first use)
constexpr int kMapChunk = 192;
struct alignas(64) MapChunk {
    int32_t n, pad[15];
    CUtensorMap maps[kMapChunk];
};
__global__ void tmap_store_kernel(const __grid_constant__ MapChunk C, CUtensorMap *dst) {
    const uint4 *src = reinterpret_cast<const uint4 *>(C.maps);
    uint4 *d = reinterpret_cast<uint4 *>(dst);
    for (int i = threadIdx.x; i < C.n * (int)(sizeof(CUtensorMap) / 16); i += blockDim.x) d[i] = src[i];
    __syncthreads();
    asm volatile("fence.proxy.tensormap::generic.release.gpu;" ::: "memory");
}

typedef CUresult (*PFN_invEncTiled)(CUtensorMap *, CUtensorMapDataType, cuuint32_t, void *, const cuuint64_t *,
                                    const cuuint64_t *, const cuuint32_t *, const cuuint32_t *, CUtensorMapInterleave,
                                    CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
static PFN_invEncTiled g_inv_enc = nullptr;
static std::mutex g_inv_enc_mu;
static kfac_status load_enc() {
    std::lock_guard<std::mutex> lock(g_inv_enc_mu);
    if (g_inv_enc) return KFAC_OK;
    cudaDriverEntryPointQueryResult q;
    void *f = nullptr;
    KFAC_CUDA_TRY(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q));
    if (!f) return set_error(KFAC_ERR_CUDA, "cuTensorMapEncodeTiled entry point unavailable");
    g_inv_enc = (PFN_invEncTiled)f;
    return KFAC_OK;
}

// one non-blocking side stream per device (created on first use)
static kfac_status side_stream(cudaStream_t *out) {
    static std::mutex mu;
    static cudaStream_t streams[64] = {};
    int dev = 0;
    KFAC_CUDA_TRY(cudaGetDevice(&dev));
    if (dev < 0 || dev >= 64) return set_error(KFAC_ERR_UNSUPPORTED, "inverse: device index >= 64");
    std::lock_guard<std::mutex> lock(mu);
    if (!streams[dev]) KFAC_CUDA_TRY(cudaStreamCreateWithFlags(&streams[dev], cudaStreamNonBlocking));
    *out = streams[dev];
    return KFAC_OK;
}

kfac_status inverse_launch(const std::vector<InvMat> &mats, int npairs, float gamma, double *pair_scratch,
                           float *pi_out, int g_only, int prec_mode, cudaStream_t st) {
    if (mats.empty()) return KFAC_OK;
    if ((int)mats.size() > kMaxMats) {
        // more than kMaxMats owned matrices (e.g. ResNet-101 on one GPU): several launches in stream
        // order, split at (A, G) pair boundaries (the damping couples a pair's traces); each launch
        // re-zeroes the dataflow state, which is sized for all matrices
        size_t b = 0;
        while (b < mats.size()) {
            size_t e = std::min(mats.size(), b + (size_t)kMaxMats);
            while (e < mats.size() && e > b + 1 && mats[e].pair == mats[e - 1].pair) e--;
            KFAC_TRY(inverse_launch(std::vector<InvMat>(mats.begin() + b, mats.begin() + e), npairs, gamma,
                                    pair_scratch, pi_out, g_only, prec_mode, st));
            b = e;
        }
        return KFAC_OK;
    }
    int sms = 0;
    KFAC_TRY(dev_sm_count(&sms));
    KFAC_TRY(dev_func_smem((const void *)pivot_kernel, kPivSmem));
    KFAC_TRY(dev_func_smem((const void *)inverse_kernel, kUpdSmem));
    InvParams P;
    memset(&P, 0, sizeof(P));
    P.nm = (int)mats.size();
    P.gamma = (double)gamma;
    P.pair_scratch = pair_scratch;
    P.pi_out = pi_out;
    P.g_only = g_only;
    P.prec_mode = prec_mode;
    // matrices by column blocks, descending: the matrices active at step k are a prefix
    std::vector<int> order(mats.size());
    for (size_t i = 0; i < mats.size(); i++) order[i] = (int)i;
    std::stable_sort(order.begin(), order.end(), [&](int a, int b) { return mats[a].n > mats[b].n; });
    int maxn = 0, sum_nt = 0, sum_tiles = 0;
    for (size_t r = 0; r < order.size(); r++) {
        const InvMat &src = mats[order[r]];
        MatDesc &d = P.m[r];
        d.packed = src.packed;
        d.inv = src.inv;
        d.work = src.work;
        d.panel = src.panel;
        d.status = src.status;
        d.n = src.n;
        d.ld = (int)inverse_ld(d.n);
        d.pair = src.pair;
        d.is_A = src.is_A;
        d.orig = order[r];
        d.split = src.split;
        d.nt = (d.n + B - 1) / B;
        d.col_begin = sum_nt;
        d.tile_begin = sum_tiles;
        sum_nt += d.nt;
        sum_tiles += d.nt * (d.nt + 1) / 2;
        maxn = std::max(maxn, d.n);
    }
    P.unp_begin[0] = P.fin_begin[0] = 0;
    for (int i = 0; i < P.nm; i++) {
        const int n = P.m[i].n, tf = (n + kFinT - 1) / kFinT;
        P.unp_begin[i + 1] = P.unp_begin[i] + (n + kUnpRows - 1) / kUnpRows;
        P.fin_begin[i + 1] = P.fin_begin[i] + (tf * (tf + 1) / 2 + kFinTiles - 1) / kFinTiles;
    }
    // the digit tile sets of every matrix as 4-D TMA maps (global memory, after the task records)
    int64_t sum_tasks_all = 0;
    for (int i = 0; i < P.nm; i++) sum_tasks_all += inverse_tasks(P.m[i].n);
    uint8_t *scratch0 = reinterpret_cast<uint8_t *>(pair_scratch);
    CUtensorMap *dmaps = reinterpret_cast<CUtensorMap *>(scratch0 + tmaps_offset(npairs, sum_nt, sum_tiles, sum_tasks_all));
    std::vector<CUtensorMap> hmaps(3 * (size_t)P.nm);
    KFAC_TRY(load_enc());
    for (int i = 0; i < P.nm; i++) {
        MatDesc &d = P.m[i];
        uint8_t *base = reinterpret_cast<uint8_t *>(d.panel + 2 * kPanelBufs * (int64_t)B * d.ld + 2 * (int64_t)B * B);
        const cuuint64_t dims[4] = {(cuuint64_t)B, (cuuint64_t)B, (cuuint64_t)kOzD, (cuuint64_t)kPanelBufs * d.nt * 2};
        const cuuint64_t strides[3] = {(cuuint64_t)B, (cuuint64_t)kOzSlice, (cuuint64_t)kOzSet};
        const cuuint32_t es[4] = {1, 1, 1, 1};
        const cuuint32_t boxes[3][4] = {{(cuuint32_t)B, (cuuint32_t)B, (cuuint32_t)kOzS, 1},
                                        {(cuuint32_t)B, (cuuint32_t)kOzQ, (cuuint32_t)kOzS, 1},
                                        {(cuuint32_t)B, (cuuint32_t)kOzQ, (cuuint32_t)kOzD, 1}};
        for (int t = 0; t < 3; t++) {
            const CUresult r = g_inv_enc(&hmaps[3 * i + t], CU_TENSOR_MAP_DATA_TYPE_UINT8, 4, base, dims, strides, boxes[t], es,
                                         CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                                         CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
            if (r != CUDA_SUCCESS) return set_error(KFAC_ERR_CUDA, "inverse: cuTensorMapEncodeTiled (digit tiles) failed");
        }
        d.tmaps = dmaps + 3 * i;
    }
    // stream-ordered upload through kernel parameters (no host synchronisation, unlike a pageable copy)
    for (size_t b = 0; b < hmaps.size(); b += kMapChunk) {
        MapChunk c;
        memset(&c, 0, sizeof(c));
        c.n = (int)std::min<size_t>(kMapChunk, hmaps.size() - b);
        memcpy(c.maps, hmaps.data() + b, c.n * sizeof(CUtensorMap));
        tmap_store_kernel<<<1, 256, 0, st>>>(c, dmaps + b);
        KFAC_LAUNCHED();
        KFAC_CUDA_TRY(cudaGetLastError());
    }
    const int steps = (maxn + B - 1) / B;
    if (steps > kMaxSteps) return set_error(KFAC_ERR_UNSUPPORTED, "inverse: matrix too large (more than 128 column blocks)");
    P.steps = steps;
    std::vector<int> ntl(P.nm);
    for (int i = 0; i < P.nm; i++) ntl[i] = P.m[i].nt;
    int task = 0;
    const int npairs_steps = (steps + 1) / 2;
    for (int pr = 0; pr < npairs_steps; pr++) {
        P.step_begin[pr] = task;
        task += pair_tasks(ntl.data(), P.nm, 2 * pr);
    }
    P.step_begin[npairs_steps] = task;
    P.total_tasks = task;
    // dataflow state after the pair data (inverse_scratch_bytes): zeroed once per call
    int *state = reinterpret_cast<int *>(pair_scratch + pair_doubles(npairs));
    P.counter = state;
    P.pivflag = state + 16;
    P.ozflag = P.pivflag + 2 * npairs;
    P.colflag = P.ozflag + 2 * npairs;
    P.panels_done = P.colflag + sum_nt;
    P.tiles_done = P.panels_done + sum_nt;
    P.tileflag = P.tiles_done + sum_nt;
    P.tasks = reinterpret_cast<int4 *>(reinterpret_cast<uint8_t *>(pair_scratch) + tasks_offset(npairs, sum_nt, sum_tiles));
    KFAC_CUDA_TRY(cudaMemsetAsync(state, 0, state_ints(npairs, sum_nt, sum_tiles) * sizeof(int), st));
    // the task list is data-independent: it is built on a side stream while damping, unpack and the
    // step-0 pivots run on `st`
    cudaStream_t side = nullptr;
    KFAC_TRY(side_stream(&side));
    cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
    KFAC_CUDA_TRY(cudaEventCreateWithFlags(&ev_fork, cudaEventDisableTiming));
    KFAC_CUDA_TRY(cudaEventCreateWithFlags(&ev_join, cudaEventDisableTiming));
    KFAC_CUDA_TRY(cudaEventRecord(ev_fork, st));
    KFAC_CUDA_TRY(cudaStreamWaitEvent(side, ev_fork, 0));
    inverse_tasks_kernel<<<dim3(npairs_steps, (P.nm + 31) / 32), 32, 0, side>>>(P);
    KFAC_LAUNCHED();
    KFAC_CUDA_TRY(cudaGetLastError());
    KFAC_CUDA_TRY(cudaEventRecord(ev_join, side));
    damp_trace_kernel<<<P.nm, 256, 0, st>>>(P);
    KFAC_LAUNCHED();
    KFAC_CUDA_TRY(cudaGetLastError());
    unpack_damp_kernel<<<P.unp_begin[P.nm], 256, 0, st>>>(P);
    KFAC_LAUNCHED();
    KFAC_CUDA_TRY(cudaGetLastError());
    pivot_kernel<<<P.nm, 256, kPivSmem, st>>>(P);
    KFAC_LAUNCHED();
    KFAC_CUDA_TRY(cudaGetLastError());
    KFAC_CUDA_TRY(cudaStreamWaitEvent(st, ev_join, 0));
    cudaEventDestroy(ev_fork);  // released once they complete
    cudaEventDestroy(ev_join);
    inverse_kernel<<<std::min(P.total_tasks, sms), kThreads, kUpdSmem, st>>>(P);
    KFAC_LAUNCHED();
    KFAC_CUDA_TRY(cudaGetLastError());
    finalize_kernel<<<P.fin_begin[P.nm], 256, 0, st>>>(P);
    KFAC_LAUNCHED();
    KFAC_CUDA_TRY(cudaGetLastError());
    return KFAC_OK;
}

}  // namespace kfac
