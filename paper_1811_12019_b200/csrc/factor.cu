// factor.cu -- stages 1-2 of distributed K-FAC (PAPER.md P:237-245 Eq. kf,
// P:313-318): the Kronecker factors
//     A = alpha * sum_rows ã ãᵀ   over im2col patches ã (+ bias coordinate 1)
//     G = alpha * sum_rows g gᵀ   over output-gradient pixels g
// as ONE grouped, persistent tcgen05 SYRK launch over every (layer, factor):
//
//   * operands are staged by TMA straight from the NHWC activation tensor:
//     2-D tiled boxes for G / 1x1 convs / FC, im2col boxes (cuTensorMapEncode-
//     Im2col) for k>1 or strided convs -- patch extraction is fused into the
//     shared-memory staging, no im2col matrix is materialised;
//     a gather producer (plain loads) covers the geometries TMA cannot
//     express (channel stride not a multiple of 16 B, e.g. the RGB stem);
//   * the MMA is tcgen05.mma kind::f16 (bf16/fp16 in, fp32 accumulate in
//     TMEM, "mixed precision"), M = N = 128, both operands
//     MN-major (the channel dimension is contiguous in NHWC; K = pixels);
//   * only upper tiles (ti <= tj) are computed and each output element is
//     written once, packed upper row-major, straight into the
//     ReduceScatter send buffer;
//   * large-K/small-d problems are split along K with a deterministic,
//     ordered fix-up (reading R-18).
//
// Warp roles (288 threads): warps 0-3 epilogue (TMEM -> smem -> packed
// global), warp 4 TMEM allocator + MMA issuer, warps 5-8 producers.
#include <cuda_bf16.h>
#include <cuda_fp16.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>

#include "kfac_internal.hpp"
#include "sm100.cuh"

namespace kfac {

constexpr int kStages = 4;
constexpr int kEpiThreads = 128;
constexpr int kMmaWarp = 4;
constexpr int kProdWarp0 = 5;
constexpr int kProdThreads = 128;
constexpr int kThreads = kEpiThreads + 32 + kProdThreads;  // 288
constexpr int kOpBytes = kTile * kBK * 2;                   // 16 KB per operand per stage
constexpr int kStageLd = kTile + 1;                         // staging row stride (floats)
constexpr int kTmemCols = 2 * kTile;                        // double-buffered accumulator
constexpr size_t kSmemOps = (size_t)kStages * 2 * kOpBytes;
constexpr size_t kSmemStage = (size_t)kTile * kStageLd * 4;
constexpr size_t kSmemBytes = 1024 + kSmemOps + kSmemStage + 256;

__device__ __forceinline__ float dec_half(uint16_t b, int fmt) {
    if (fmt == 1) return __half2float(__ushort_as_half(b));
    return __uint_as_float(((uint32_t)b) << 16);
}

struct ItemInfo {
    int p, ti, tj, split, tp, k0, k1;
};

__device__ __forceinline__ ItemInfo decode_item(const FactorParams &P, int item) {
    ItemInfo it;
    int p = 0;
    while (p + 1 < P.nprobs && P.probs[p + 1].item_begin <= item) p++;
    const FactorProb &pr = P.probs[p];
    int local = item - pr.item_begin;
    int T = pr.nt * (pr.nt + 1) / 2;
    // split-major: concurrently running CTAs share the same K rows (L2 reuse)
    it.split = local / T;
    it.tp = local % T;
    int ti = 0, rem = it.tp;
    while (rem >= pr.nt - ti) {
        rem -= pr.nt - ti;
        ti++;
    }
    it.p = p;
    it.ti = ti;
    it.tj = ti + rem;
    it.k0 = it.split * pr.chunks_per_split;
    it.k1 = min(pr.kchunks, it.k0 + pr.chunks_per_split);
    return it;
}

__device__ __forceinline__ uint32_t layout_of(int cb) {
    return cb == 64 ? UMMA_SW128 : (cb == 32 ? UMMA_SW64 : UMMA_SW32);
}

// gather one element of the operand: feature f (< d) of output row q (< rows)
__device__ __forceinline__ float gather_elem(const FactorProb &pr, int fmt, int64_t q, int f) {
    int hw = pr.ho * pr.wo;
    int64_t n = q / hw;
    int rem = (int)(q - n * hw);
    int oh = rem / pr.wo, ow = rem - oh * pr.wo;
    int kk = f / pr.c, c = f - kk * pr.c;
    int i = kk / pr.kw, j = kk - i * pr.kw;
    int h = oh * pr.sh - pr.ph + i, w = ow * pr.sw - pr.pw + j;
    if (h < 0 || h >= pr.h || w < 0 || w >= pr.w) return 0.f;
    return dec_half(__ldg(pr.src + (((n * pr.h + h) * pr.w + w) * pr.c + c)), fmt);
}

// fill one 128-feature x 64-row operand tile in the SW128 MN-major layout
__device__ __forceinline__ void gather_tile(const FactorProb &pr, int fmt, uint8_t *dst, int tile, int kc, int tid) {
    for (int u = tid; u < kBK * 16; u += kProdThreads) {
        int r = u >> 4, q = u & 15;  // row in chunk, 16-byte chunk along features
        int64_t row = (int64_t)kc * kBK + r;
        int f0 = tile * kTile + q * 8;
        uint32_t pk[4];
#pragma unroll
        for (int e = 0; e < 8; e += 2) {
            float v0 = 0.f, v1 = 0.f;
            if (row < pr.rows) {
                if (f0 + e < pr.d) v0 = gather_elem(pr, fmt, row, f0 + e);
                if (f0 + e + 1 < pr.d) v1 = gather_elem(pr, fmt, row, f0 + e + 1);
            }
            uint32_t lo, hi;
            if (fmt == 1) {
                lo = __half_as_ushort(__float2half_rn(v0));
                hi = __half_as_ushort(__float2half_rn(v1));
            } else {
                lo = __bfloat16_as_ushort(__float2bfloat16_rn(v0));
                hi = __bfloat16_as_ushort(__float2bfloat16_rn(v1));
            }
            pk[e / 2] = lo | (hi << 16);
        }
        int box = q >> 3, cq = q & 7;
        uint8_t *p = dst + box * (kBK * 128) + r * 128 + ((cq ^ (r & 7)) << 4);
        *reinterpret_cast<uint4 *>(p) = make_uint4(pk[0], pk[1], pk[2], pk[3]);
    }
}

__global__ void __launch_bounds__(kThreads, 1) factor_syrk_kernel(const __grid_constant__ FactorParams P) {
    extern __shared__ uint8_t smem_raw[];
    uint8_t *smem = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint8_t *ops = smem;
    float *stage_buf = reinterpret_cast<float *>(smem + kSmemOps);
    uint64_t *bars = reinterpret_cast<uint64_t *>(smem + kSmemOps + kSmemStage);
    uint64_t *full = bars, *empty = bars + kStages, *tfull = bars + 2 * kStages, *tempty = bars + 2 * kStages + 2;
    uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(bars + 2 * kStages + 4);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (threadIdx.x == 0) {
        for (int s = 0; s < kStages; s++) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], 1);
        }
        for (int b = 0; b < 2; b++) {
            mbar_init(&tfull[b], 1);
            mbar_init(&tempty[b], kEpiThreads);
        }
        fence_barrier_init();
    }
    if (warp == kMmaWarp) tmem_alloc(tmem_slot, kTmemCols);
    if (warp == kProdWarp0 && lane == 0) {
        for (int p = 0; p < P.nprobs; p++)
            if (P.probs[p].mode != MODE_GATHER) tma_prefetch(&P.probs[p].tmap);
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;
    const int fmt = P.ab_fmt == 1 ? 0 : 1;  // kind::f16 format code: 0 fp16, 1 bf16
    const int dec_fmt = P.ab_fmt;            // 0 bf16, 1 fp16 (kfac_dtype)

    if (warp >= kProdWarp0) {
        // ============================ producers ============================
        const int ptid = threadIdx.x - kProdWarp0 * 32;
        uint32_t stage = 0, phase = 0;
        for (int item = blockIdx.x; item < P.total_items; item += gridDim.x) {
            const ItemInfo it = decode_item(P, item);
            const FactorProb &pr = P.probs[it.p];
            const bool diag = it.ti == it.tj;
            if (pr.mode == MODE_GATHER) {
                for (int kc = it.k0; kc < it.k1; kc++) {
                    mbar_wait(&empty[stage], phase ^ 1);
                    uint8_t *a = ops + (size_t)stage * 2 * kOpBytes;
                    gather_tile(pr, dec_fmt, a, it.ti, kc, ptid);
                    if (!diag) gather_tile(pr, dec_fmt, a + kOpBytes, it.tj, kc, ptid);
                    fence_proxy_async_smem();
                    named_bar_sync(1, kProdThreads);
                    if (ptid == 0) mbar_arrive(&full[stage]);
                    if (++stage == kStages) {
                        stage = 0;
                        phase ^= 1;
                    }
                }
            } else {
                // one elected thread issues the TMA; the others only track the ring position
                const int cb = pr.cb, nbox = kTile / cb;
                const uint32_t box_bytes = kBK * cb * 2;
                for (int kc = it.k0; kc < it.k1; kc++) {
                    if (ptid != 0) {
                        if (++stage == kStages) {
                            stage = 0;
                            phase ^= 1;
                        }
                        continue;
                    }
                    mbar_wait(&empty[stage], phase ^ 1);
                    uint8_t *a = ops + (size_t)stage * 2 * kOpBytes;
                    uint32_t nb = 0;
                    for (int b = 0; b < nbox; b++) {
                        if (it.ti * kTile + b * cb < pr.d) nb++;
                        if (!diag && it.tj * kTile + b * cb < pr.d) nb++;
                    }
                    mbar_arrive_expect_tx(&full[stage], nb * box_bytes);
                    const int64_t q0 = (int64_t)kc * kBK;
                    int n0 = 0, bw = 0, bh = 0;
                    if (pr.mode == MODE_IM2COL) {
                        int hw = pr.ho * pr.wo;
                        n0 = (int)(q0 / hw);
                        int rem = (int)(q0 - (int64_t)n0 * hw);
                        int oh = rem / pr.wo, ow = rem - oh * pr.wo;
                        bw = ow * pr.sw - pr.pw;
                        bh = oh * pr.sh - pr.ph;
                    }
                    for (int op = 0; op < (diag ? 1 : 2); op++) {
                        const int tile = op == 0 ? it.ti : it.tj;
                        uint8_t *dst = a + op * kOpBytes;
                        for (int b = 0; b < nbox; b++) {
                            int f0 = tile * kTile + b * cb;
                            if (f0 >= pr.d) break;
                            if (pr.mode == MODE_TILED2D) {
                                tma_load_2d(dst + b * box_bytes, &pr.tmap, &full[stage], f0, (int32_t)q0);
                            } else {
                                int kk = f0 / pr.c, c0 = f0 - kk * pr.c;
                                int i = kk / pr.kw, j = kk - i * pr.kw;
                                tma_load_im2col_4d(dst + b * box_bytes, &pr.tmap, &full[stage], c0, bw, bh, n0,
                                                   (uint16_t)j, (uint16_t)i);
                            }
                        }
                    }
                    if (++stage == kStages) {
                        stage = 0;
                        phase ^= 1;
                    }
                }
            }
        }
    } else if (warp == kMmaWarp) {
        // ============================ MMA issuer ============================
        uint32_t stage = 0, phase = 0;
        uint32_t tph0 = 0, tph1 = 0;
        int buf = 0;
        for (int item = blockIdx.x; item < P.total_items; item += gridDim.x) {
            const ItemInfo it = decode_item(P, item);
            const FactorProb &pr = P.probs[it.p];
            const bool diag = it.ti == it.tj;
            const int cb = pr.cb;
            const uint32_t lbo = kBK * cb * 2, sbo = 8 * cb * 2, lay = layout_of(cb);
            const uint32_t kstep = 16 * cb * 2;  // bytes per K=16 slice
            const uint32_t idesc = idesc_f16(fmt, kTile, kTile, 1, 1);
            const uint32_t tacc = tmem_base + buf * kTile;
            if (lane == 0) {
                mbar_wait(&tempty[buf], (buf ? tph1 : tph0) ^ 1);
                tc_fence_after();
                for (int kc = it.k0; kc < it.k1; kc++) {
                    mbar_wait(&full[stage], phase);
                    tc_fence_after();
                    const uint32_t a_base = smem_u32(ops + (size_t)stage * 2 * kOpBytes);
                    const uint32_t b_base = diag ? a_base : a_base + kOpBytes;
#pragma unroll
                    for (int k = 0; k < kBK / 16; k++) {
                        uint64_t ad = umma_desc(a_base + k * kstep, lbo, sbo, lay);
                        uint64_t bd = umma_desc(b_base + k * kstep, lbo, sbo, lay);
                        mma_f16_ss(tacc, ad, bd, idesc, (kc > it.k0 || k > 0) ? 1u : 0u);
                    }
                    mma_commit(&empty[stage]);
                    if (++stage == kStages) {
                        stage = 0;
                        phase ^= 1;
                    }
                }
                mma_commit(&tfull[buf]);
            }
            __syncwarp();
            if (buf) tph1 ^= 1; else tph0 ^= 1;
            buf ^= 1;
        }
    } else {
        // ============================ epilogue ============================
        uint32_t tph0 = 0, tph1 = 0;
        int buf = 0;
        const int row = warp * 32 + lane;
        for (int item = blockIdx.x; item < P.total_items; item += gridDim.x) {
            const ItemInfo it = decode_item(P, item);
            const FactorProb &pr = P.probs[it.p];
            mbar_wait(&tfull[buf], buf ? tph1 : tph0);
            tc_fence_after();
            const uint32_t tacc = tmem_base + buf * kTile + ((uint32_t)(warp * 32) << 16);
#pragma unroll
            for (int c = 0; c < kTile / 32; c++) {
                uint32_t r[32];
                tmem_ld_32x32b_x32(tacc + c * 32, r);
                tmem_ld_wait();
#pragma unroll
                for (int i = 0; i < 32; i++) stage_buf[row * kStageLd + c * 32 + i] = __uint_as_float(r[i]);
            }
            tc_fence_before();
            mbar_arrive(&tempty[buf]);
            named_bar_sync(2, kEpiThreads);
            const int gi0 = it.ti * kTile, gj0 = it.tj * kTile;
            if (pr.splits == 1) {
                const int64_t dd = pr.d_out;
                const int jmax = min(kTile, pr.d - gj0);
                for (int r = warp; r < kTile; r += 4) {
                    const int gi = gi0 + r;
                    if (gi >= pr.d) break;
                    const int jlo = (it.ti == it.tj) ? r : 0;
                    float *orow = pr.out + ((int64_t)gi * dd - (int64_t)gi * (gi - 1) / 2 - gi);
                    for (int j = jlo + lane; j < jmax; j += 32) orow[gj0 + j] = pr.alpha * stage_buf[r * kStageLd + j];
                }
            } else {
                float *part = pr.partial + ((size_t)it.split * (pr.nt * (pr.nt + 1) / 2) + it.tp) * (kTile * kTile);
                for (int r = warp; r < kTile; r += 4)
                    for (int j = lane; j < kTile; j += 32) part[r * kTile + j] = stage_buf[r * kStageLd + j];
            }
            named_bar_sync(2, kEpiThreads);
            if (buf) tph1 ^= 1; else tph0 ^= 1;
            buf ^= 1;
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == kMmaWarp) {
        tc_fence_after();
        tmem_dealloc(tmem_base, kTmemCols);
    }
}

// ordered split-K fix-up: out = alpha * sum_{s=0..S-1} partial[s] (deterministic)
__global__ void __launch_bounds__(256) factor_fixup_kernel(const __grid_constant__ FactorParams P) {
    // blockIdx.x enumerates (problem with splits > 1, tile pair)
    int b = blockIdx.x, p = 0;
    for (; p < P.nprobs; p++) {
        const FactorProb &pr = P.probs[p];
        if (pr.splits <= 1) continue;
        int T = pr.nt * (pr.nt + 1) / 2;
        if (b < T) break;
        b -= T;
    }
    if (p >= P.nprobs) return;
    const FactorProb &pr = P.probs[p];
    const int T = pr.nt * (pr.nt + 1) / 2;
    int ti = 0, rem = b;
    while (rem >= pr.nt - ti) {
        rem -= pr.nt - ti;
        ti++;
    }
    const int tj = ti + rem;
    const int gi0 = ti * kTile, gj0 = tj * kTile;
    const int jmax = min(kTile, pr.d - gj0);
    const int64_t dd = pr.d_out;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    for (int r = warp; r < kTile; r += 8) {
        const int gi = gi0 + r;
        if (gi >= pr.d) break;
        const int jlo = (ti == tj) ? r : 0;
        float *orow = pr.out + ((int64_t)gi * dd - (int64_t)gi * (gi - 1) / 2 - gi);
        for (int j = jlo + lane; j < jmax; j += 32) {
            float s = 0.f;
            for (int sp = 0; sp < pr.splits; sp++)
                s += pr.partial[((size_t)sp * T + b) * (kTile * kTile) + r * kTile + j];
            orow[gj0 + j] = pr.alpha * s;
        }
    }
}

// bias row/column of A: A[f][dA-1] = alpha * sum_rows ã_f, A[dA-1][dA-1] = alpha * rows
// (the homogeneous coordinate, reading R-5); one thread per feature, fixed row order.
__global__ void __launch_bounds__(256) factor_bias_kernel(const __grid_constant__ FactorParams P) {
    const FactorProb &pr = P.probs[blockIdx.y];
    if (pr.d_out == pr.d) return;
    const int f = blockIdx.x * blockDim.x + threadIdx.x;
    const int dA = pr.d_out;
    if (f > pr.d) return;
    double s = 0.0;
    if (f == pr.d) {
        s = (double)pr.rows;
    } else {
        for (int64_t q = 0; q < pr.rows; q++) s += (double)gather_elem(pr, P.ab_fmt, q, f);
    }
    const int64_t off = (int64_t)f * dA - (int64_t)f * (f - 1) / 2 + (dA - 1 - f);
    pr.out[off] = (float)(pr.alpha * s);
}

// ---------------------------------------------------------------- host side
typedef CUresult (*PFN_encodeTiled)(CUtensorMap *, CUtensorMapDataType, cuuint32_t, void *, const cuuint64_t *,
                                    const cuuint64_t *, const cuuint32_t *, const cuuint32_t *, CUtensorMapInterleave,
                                    CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
typedef CUresult (*PFN_encodeIm2col)(CUtensorMap *, CUtensorMapDataType, cuuint32_t, void *, const cuuint64_t *,
                                     const cuuint64_t *, const int *, const int *, cuuint32_t, cuuint32_t,
                                     const cuuint32_t *, CUtensorMapInterleave, CUtensorMapSwizzle,
                                     CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static PFN_encodeTiled g_encTiled = nullptr;
static PFN_encodeIm2col g_encIm2col = nullptr;
static int g_driver = 0;

static kfac_status load_driver_fns() {
    if (g_encTiled && g_encIm2col) return KFAC_OK;
    cudaDriverEntryPointQueryResult q1, q2;
    void *f1 = nullptr, *f2 = nullptr;
    KFAC_CUDA_TRY(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f1, cudaEnableDefault, &q1));
    KFAC_CUDA_TRY(cudaGetDriverEntryPoint("cuTensorMapEncodeIm2col", &f2, cudaEnableDefault, &q2));
    if (!f1 || !f2) return set_error(KFAC_ERR_CUDA, "cuTensorMapEncode* entry points unavailable");
    g_encTiled = (PFN_encodeTiled)f1;
    g_encIm2col = (PFN_encodeIm2col)f2;
    cudaDriverGetVersion(&g_driver);
    return KFAC_OK;
}

static CUtensorMapSwizzle swz_of(int cb) {
    return cb == 64 ? CU_TENSOR_MAP_SWIZZLE_128B : (cb == 32 ? CU_TENSOR_MAP_SWIZZLE_64B : CU_TENSOR_MAP_SWIZZLE_32B);
}

static void small_tensor_fix(CUtensorMap *m, int64_t bytes) {
    // same driver workaround CUTLASS applies to descriptors of tensors < 128 KiB
    if (g_driver <= 13010 && bytes < 131072) reinterpret_cast<uint64_t *>(m)[1] &= ~(1ull << 21);
}

static bool force_gather() {
    const char *e = getenv("KFAC_FORCE_GATHER");
    return e && e[0] == '1';
}

// choose the staging mode of one factor problem and fill the TMA descriptor
static kfac_status setup_prob(const FactorJob &j, kfac_dtype dt, FactorProb *pr) {
    const Geom &g = j.g;
    memset(pr, 0, sizeof(*pr));
    pr->src = static_cast<const uint16_t *>(j.src);
    pr->out = j.out;
    pr->alpha = j.alpha;
    if (j.is_A) {
        pr->c = g.c_in;
        pr->h = g.h;
        pr->w = g.w;
        pr->kh = g.kh;
        pr->kw = g.kw;
        pr->sh = g.sh;
        pr->sw = g.sw;
        pr->ph = g.ph;
        pr->pw = g.pw;
        pr->ho = g.ho;
        pr->wo = g.wo;
        pr->d = g.dF;
        pr->d_out = g.dA;
    } else {  // G: a 1x1 "patch" over the gy pixels
        pr->c = g.c_out;
        pr->h = g.ho;
        pr->w = g.wo;
        pr->kh = pr->kw = pr->sh = pr->sw = 1;
        pr->ph = pr->pw = 0;
        pr->ho = g.ho;
        pr->wo = g.wo;
        pr->d = g.dG;
        pr->d_out = g.dG;
    }
    pr->rows = j.n * (int64_t)pr->ho * pr->wo;
    pr->nt = (pr->d + kTile - 1) / kTile;
    pr->kchunks = (int)((pr->rows + kBK - 1) / kBK);
    const int C = pr->c;
    const bool plain = (pr->kh == 1 && pr->kw == 1 && pr->sh == 1 && pr->sw == 1 && pr->ph == 0 && pr->pw == 0);
    const bool aligned16 = (C % 8) == 0 && (reinterpret_cast<uintptr_t>(j.src) % 16) == 0;
    int mode = MODE_GATHER, cb = 64;
    if (!force_gather() && aligned16) {
        if (plain) {
            mode = MODE_TILED2D;
            cb = C >= 64 ? 64 : (C > 16 ? (C > 32 ? 64 : 32) : 16);
        } else if (C % 16 == 0 && pr->pw <= 127 && pr->ph <= 127 && pr->kw <= 128 && pr->kh <= 128 && pr->sw <= 8 &&
                   pr->sh <= 8) {
            mode = MODE_IM2COL;
            cb = (C % 64 == 0) ? 64 : ((C % 32 == 0) ? 32 : 16);
        }
    }
    pr->mode = mode;
    pr->cb = cb;
    if (mode == MODE_GATHER) return KFAC_OK;
    kfac_status s = load_driver_fns();
    if (s) return s;
    const CUtensorMapDataType dty = dt == KFAC_FP16 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT16 : CU_TENSOR_MAP_DATA_TYPE_BFLOAT16;
    const int64_t bytes = pr->rows / ((int64_t)pr->ho * pr->wo) * pr->h * pr->w * (int64_t)C * 2;
    CUresult r;
    if (mode == MODE_TILED2D) {
        cuuint64_t dims[2] = {(cuuint64_t)C, (cuuint64_t)pr->rows};
        cuuint64_t strides[1] = {(cuuint64_t)C * 2};
        cuuint32_t box[2] = {(cuuint32_t)cb, (cuuint32_t)kBK};
        cuuint32_t es[2] = {1, 1};
        r = g_encTiled(&pr->tmap, dty, 2, const_cast<void *>(j.src), dims, strides, box, es,
                       CU_TENSOR_MAP_INTERLEAVE_NONE, swz_of(cb), CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                       CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    } else {
        const int64_t N = pr->rows / ((int64_t)pr->ho * pr->wo);
        cuuint64_t dims[4] = {(cuuint64_t)C, (cuuint64_t)pr->w, (cuuint64_t)pr->h, (cuuint64_t)N};
        cuuint64_t strides[3] = {(cuuint64_t)C * 2, (cuuint64_t)C * 2 * pr->w, (cuuint64_t)C * 2 * pr->w * pr->h};
        int lower[2] = {-pr->pw, -pr->ph};
        int upper[2] = {pr->pw - pr->kw + 1, pr->ph - pr->kh + 1};
        cuuint32_t es[4] = {1, (cuuint32_t)pr->sw, (cuuint32_t)pr->sh, 1};
        r = g_encIm2col(&pr->tmap, dty, 4, const_cast<void *>(j.src), dims, strides, lower, upper, (cuuint32_t)cb,
                        (cuuint32_t)kBK, es, CU_TENSOR_MAP_INTERLEAVE_NONE, swz_of(cb),
                        CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    }
    if (r != CUDA_SUCCESS) {
        char buf[160];
        snprintf(buf, sizeof buf, "cuTensorMapEncode%s failed (%d) for C=%d mode=%d", mode == MODE_TILED2D ? "Tiled" : "Im2col",
                 (int)r, C, mode);
        return set_error(KFAC_ERR_UNSUPPORTED, buf);
    }
    small_tensor_fix(&pr->tmap, bytes);
    return KFAC_OK;
}

static int g_num_sms = 0;

kfac_status factor_prepare(const std::vector<FactorJob> &jobs, kfac_dtype dt, void *ws, int64_t ws_cap,
                           bool dry_run, FactorLaunch *out) {
    out->params.clear();
    out->ws_bytes = 0;
    if (jobs.empty()) return KFAC_OK;
    int nsm = 148;
    if (!dry_run) {
        if (!g_num_sms) {
            int dev = 0;
            KFAC_CUDA_TRY(cudaGetDevice(&dev));
            KFAC_CUDA_TRY(cudaDeviceGetAttribute(&g_num_sms, cudaDevAttrMultiProcessorCount, dev));
        }
        nsm = g_num_sms;
    }
    // order problems by cost, heaviest first (static striding ~ LPT)
    std::vector<int> order(jobs.size());
    std::vector<double> cost(jobs.size());
    std::vector<int64_t> tiles(jobs.size()), kch(jobs.size());
    double total = 0;
    for (size_t i = 0; i < jobs.size(); i++) {
        const Geom &g = jobs[i].g;
        int d = jobs[i].is_A ? g.dF : g.dG;
        int64_t rows = jobs[i].n * (int64_t)g.ho * g.wo;
        int nt = (d + kTile - 1) / kTile;
        tiles[i] = (int64_t)nt * (nt + 1) / 2;
        kch[i] = (rows + kBK - 1) / kBK;
        cost[i] = (double)tiles[i] * kch[i];
        total += cost[i];
        order[i] = (int)i;
    }
    std::stable_sort(order.begin(), order.end(), [&](int a, int b) { return cost[a] > cost[b]; });
    const double target = std::max(32.0, total / (4.0 * 148));  // fixed: plan-time ws sizing must match
    int64_t ws_off = 0;
    for (size_t base = 0; base < order.size(); base += kMaxProbs) {
        FactorParams P;
        memset(&P, 0, sizeof(P));
        P.ab_fmt = (int)dt;
        int items = 0;
        size_t cnt = std::min((size_t)kMaxProbs, order.size() - base);
        for (size_t k = 0; k < cnt; k++) {
            const int i = order[base + k];
            FactorProb &pr = P.probs[k];
            if (!dry_run) {
                kfac_status s = setup_prob(jobs[i], dt, &pr);
                if (s) return s;
            } else {
                memset(&pr, 0, sizeof(pr));
                const Geom &g = jobs[i].g;
                pr.d = jobs[i].is_A ? g.dF : g.dG;
                pr.nt = (pr.d + kTile - 1) / kTile;
                pr.kchunks = (int)kch[i];
            }
            int S = (int)std::max<double>(1.0, std::min<double>((double)pr.kchunks, std::ceil((double)pr.kchunks / target)));
            pr.chunks_per_split = (pr.kchunks + S - 1) / S;
            S = (pr.kchunks + pr.chunks_per_split - 1) / pr.chunks_per_split;
            pr.splits = S;
            pr.item_begin = items;
            items += (int)(tiles[i] * S);
            if (S > 1) {
                pr.partial = reinterpret_cast<float *>(static_cast<uint8_t *>(ws) + ws_off);
                ws_off += (int64_t)tiles[i] * S * kTile * kTile * 4;
            }
        }
        P.nprobs = (int)cnt;
        P.total_items = items;
        out->params.push_back(P);
    }
    out->ws_bytes = ws_off;
    if (!dry_run && ws_off > ws_cap) return set_error(KFAC_ERR_ARG, "factor workspace too small");
    return KFAC_OK;
}

kfac_status factor_launch(const FactorLaunch &fl, const std::vector<FactorJob> &jobs, cudaStream_t st) {
    static bool attr_set = false;
    if (!attr_set) {
        KFAC_CUDA_TRY(cudaFuncSetAttribute(factor_syrk_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kSmemBytes));
        attr_set = true;
    }
    for (const FactorParams &P : fl.params) {
        if (P.total_items == 0) continue;
        int grid = std::min(P.total_items, g_num_sms ? g_num_sms : 148);
        factor_syrk_kernel<<<grid, kThreads, kSmemBytes, st>>>(P);
        KFAC_LAUNCHED();
        KFAC_CUDA_TRY(cudaGetLastError());
        int fix = 0, maxbias = 0;
        for (int p = 0; p < P.nprobs; p++) {
            const FactorProb &pr = P.probs[p];
            if (pr.splits > 1) fix += pr.nt * (pr.nt + 1) / 2;
            if (pr.d_out != pr.d) maxbias = std::max(maxbias, pr.d + 1);
        }
        if (fix) {
            factor_fixup_kernel<<<fix, 256, 0, st>>>(P);
            KFAC_LAUNCHED();
            KFAC_CUDA_TRY(cudaGetLastError());
        }
        if (maxbias) {
            dim3 g((maxbias + 255) / 256, P.nprobs);
            factor_bias_kernel<<<g, 256, 0, st>>>(P);
            KFAC_LAUNCHED();
            KFAC_CUDA_TRY(cudaGetLastError());
        }
    }
    (void)jobs;
    return KFAC_OK;
}

// ---------------------------------------------------------------- replicate (redundant owners)
struct ReplParams {
    int n;
    const float *src[64];
    float *dst[64];
    int64_t cnt[64];
};
__global__ void replicate_kernel(const __grid_constant__ ReplParams P) {
    const int k = blockIdx.y;
    const float *s = P.src[k];
    float *d = P.dst[k];
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < P.cnt[k]; i += (int64_t)gridDim.x * blockDim.x)
        d[i] = s[i];
}

kfac_status replicate_launch(const std::vector<std::pair<const float *, float *>> &sd, const std::vector<int64_t> &counts,
                             cudaStream_t st) {
    for (size_t b = 0; b < sd.size(); b += 64) {
        ReplParams P;
        P.n = (int)std::min<size_t>(64, sd.size() - b);
        for (int k = 0; k < P.n; k++) {
            P.src[k] = sd[b + k].first;
            P.dst[k] = sd[b + k].second;
            P.cnt[k] = counts[b + k];
        }
        replicate_kernel<<<dim3(256, P.n), 256, 0, st>>>(P);
        KFAC_LAUNCHED();
        KFAC_CUDA_TRY(cudaGetLastError());
    }
    return KFAC_OK;
}

}  // namespace kfac
