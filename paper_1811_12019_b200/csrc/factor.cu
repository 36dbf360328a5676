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
constexpr int kOpA = kTileM * kBK * 2;                      // 16 KB A operand per stage
constexpr int kOpB = kTileN * kBK * 2;                      // 32 KB B operand per stage
constexpr int kStageBytes = kOpA + kOpB;
constexpr int kQ = 32;                                      // epilogue column group (one tcgen05.ld x32)
constexpr int kStageLd = kQ + 1;                            // staging row stride (floats, conflict-free)
constexpr int kTmemCols = 2 * kTileN;                       // double-buffered 128 x 256 fp32 accumulator
constexpr size_t kSmemOps = (size_t)kStages * kStageBytes;
constexpr size_t kSmemStage = (size_t)kTileM * kStageLd * 4;
constexpr size_t kSmemHdr = (size_t)kMaxProbs * 24;         // per-problem decode table
constexpr size_t kSmemBytes = 1024 + kSmemOps + kSmemStage + kSmemHdr + 256;
static_assert(kSmemBytes <= 232448, "shared memory budget");

// zero rows for the K tail of short chunks, copied by the async proxy (cp.async.bulk)
__device__ __align__(128) uint4 g_zero_rows[kBK * 8];  // 64 rows x 128 B

__device__ __forceinline__ float dec_half(uint16_t b, int fmt) {
    if (fmt == 1) return __half2float(__ushort_as_half(b));
    return __uint_as_float(((uint32_t)b) << 16);
}

struct ItemInfo {
    int p, ti, tj, split, tp, k0, k1;
};

// tile pair tp -> (ti, tj): row tiles of 128, column tiles of 256, tj >= ti/2 (touches the upper triangle)
__device__ __forceinline__ void decode_pair(int tp, int ntm, int ntn, int &ti, int &tj) {
    int t = 0, rem = tp;
    while (rem >= ntn - t / 2) {
        rem -= ntn - t / 2;
        t++;
    }
    ti = t;
    tj = t / 2 + rem;
}

// per-problem decode fields, copied to shared memory once per CTA (dynamic indexing of the
// kernel-parameter array goes through the constant cache and is slow)
struct ProbHdr {
    int32_t item_begin, npairs, kchunks, cps;
    int16_t ntm, ntn;
    int32_t pad;
};
static_assert(sizeof(ProbHdr) == 24, "ProbHdr");

__device__ __forceinline__ ItemInfo decode_item(const ProbHdr *hdr, int nprobs, int item) {
    ItemInfo it;
    int lo = 0, hi = nprobs - 1;  // last problem with item_begin <= item
    while (lo < hi) {
        const int mid = (lo + hi + 1) >> 1;
        if (hdr[mid].item_begin <= item) lo = mid; else hi = mid - 1;
    }
    const ProbHdr h = hdr[lo];
    const int local = item - h.item_begin;
    // split-major: concurrently running CTAs share the same K rows (L2 reuse)
    it.split = local / h.npairs;
    it.tp = local - it.split * h.npairs;
    decode_pair(it.tp, h.ntm, h.ntn, it.ti, it.tj);
    it.p = lo;
    it.k0 = it.split * h.cps;
    it.k1 = min(h.kchunks, it.k0 + h.cps);
    return it;
}

// register copy of the fields a role needs for one work item
struct ProbRegs {
    int mode, d, d_out, cb, rpc, ksteps, bh, bn, rpi, c, h, w, ho, wo, kh, kw, sh, sw, ph, pw, splits, npairs;
    float alpha;
    float *out, *partial;
    const uint16_t *src;
    int64_t rows;
};
__device__ __forceinline__ ProbRegs load_prob(const FactorProb &g) {
    ProbRegs r;
    r.mode = g.mode; r.d = g.d; r.d_out = g.d_out; r.cb = g.cb; r.rpc = g.rpc; r.ksteps = g.ksteps;
    r.bh = g.bh; r.bn = g.bn; r.rpi = g.rpi; r.c = g.c; r.h = g.h; r.w = g.w; r.ho = g.ho; r.wo = g.wo;
    r.kh = g.kh; r.kw = g.kw; r.sh = g.sh; r.sw = g.sw; r.ph = g.ph; r.pw = g.pw; r.splits = g.splits;
    r.npairs = g.npairs; r.alpha = g.alpha; r.out = g.out; r.partial = g.partial; r.src = g.src; r.rows = g.rows;
    return r;
}

__device__ __forceinline__ uint32_t layout_of(int cb) {
    return cb == 64 ? UMMA_SW128 : (cb == 32 ? UMMA_SW64 : UMMA_SW32);
}

// gather one element: feature f (< d) of output row q (< rows)  [bias kernel]
__device__ __forceinline__ float gather_elem(const ProbRegs &pr, int fmt, int64_t q, int f) {
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

// gather producer: fill `nfeat` features (from f_base) x 64 rows in the SW128 MN-major layout
__device__ __forceinline__ void gather_tile(const ProbRegs &pr, int fmt, uint8_t *dst, int f_base, int nfeat,
                                            int kc, int tid) {
    const int nq = nfeat / 8;  // 16-byte chunks per row
    const int hw = pr.ho * pr.wo;
    for (int u = tid; u < kBK * nq; u += kProdThreads) {
        const int r = u / nq, q = u - r * nq;
        const int64_t row = (int64_t)kc * kBK + r;
        uint32_t pk[4] = {0u, 0u, 0u, 0u};
        int f = f_base + q * 8;
        if (row < pr.rows && f < pr.d) {
            const int64_t n = row / hw;
            const int rem = (int)(row - n * hw);
            const int oh = rem / pr.wo, ow = rem - oh * pr.wo;
            int kk = f / pr.c, c = f - kk * pr.c;
            int i = kk / pr.kw, j = kk - i * pr.kw;
            const uint16_t *base = pr.src + n * (int64_t)pr.h * pr.w * pr.c;
#pragma unroll
            for (int e = 0; e < 8; e++) {
                uint16_t v = 0;
                if (f + e < pr.d) {
                    const int h = oh * pr.sh - pr.ph + i, w = ow * pr.sw - pr.pw + j;
                    if (h >= 0 && h < pr.h && w >= 0 && w < pr.w) v = __ldg(base + ((int64_t)h * pr.w + w) * pr.c + c);
                }
                pk[e >> 1] |= (uint32_t)v << ((e & 1) * 16);
                if (++c == pr.c) {
                    c = 0;
                    if (++j == pr.kw) {
                        j = 0;
                        ++i;
                    }
                }
            }
        }
        (void)fmt;
        const int box = q >> 3, cq = q & 7;
        uint8_t *p = dst + box * (kBK * 128) + r * 128 + ((cq ^ (r & 7)) << 4);
        *reinterpret_cast<uint4 *>(p) = make_uint4(pk[0], pk[1], pk[2], pk[3]);
    }
}

// chunk -> (image, first output row) for MODE_TILED4D
__device__ __forceinline__ void chunk_origin(const ProbRegs &pr, int kc, int &n, int &oh0) {
    if (pr.bh < pr.ho) {
        n = kc / pr.rpi;
        oh0 = (kc - n * pr.rpi) * pr.bh;
    } else {
        n = kc * pr.bn;
        oh0 = 0;
    }
}

// The TMA boxes of one chunk: first the B operand (256 features at fb), then -- unless A is
// contained in B -- the A operand (128 features at fa); one box per cb-channel slot.  Issuer w
// (of kIssuers producer warps) issues boxes k = w, w + kIssuers, ...  Returns the bytes it
// asked for (for its expect_tx).
constexpr int kIssuers = 4;
__device__ __forceinline__ uint32_t issue_boxes(const ProbRegs &pr, const CUtensorMap *tmap, uint8_t *a, uint8_t *b,
                                                uint64_t *bar, int fa, int fb, bool a_in_b, int kc, int w, bool go) {
    const int cb = pr.cb;
    const uint32_t slot = kBK * cb * 2;
    const uint32_t box_bytes = (uint32_t)pr.rpc * cb * 2;
    int n = 0, oh0 = 0;
    if (pr.mode == MODE_TILED4D) chunk_origin(pr, kc, n, oh0);
    const int nbb = kTileN / cb, nba = a_in_b ? 0 : kTileM / cb;
    uint32_t bytes = 0;
    for (int k = w; k < nbb + nba; k += kIssuers) {
        const bool isB = k < nbb;
        const int slot_i = isB ? k : k - nbb;
        const int f0 = (isB ? fb : fa) + slot_i * cb;
        if (f0 >= pr.d) continue;
        bytes += box_bytes;
        if (!go) continue;
        uint8_t *dst = (isB ? b : a) + slot_i * slot;
        if (pr.mode == MODE_TILED2D) {
            tma_load_2d(dst, tmap, bar, f0, kc * kBK);
        } else {
            const int kk = f0 / pr.c, c0 = f0 - kk * pr.c;
            const int i = kk / pr.kw, j = kk - i * pr.kw;
            tma_load_4d(dst, tmap, bar, c0, j - pr.pw, oh0 * pr.sh - pr.ph + i, n);
        }
    }
    return bytes;
}

// zero rows [from, kBK) of every slot of one operand region (async proxy, completes on bar)
__device__ __forceinline__ uint32_t zero_tail(uint8_t *region, int nslots, int cb, int from, uint64_t *bar, bool go) {
    const uint32_t slot = kBK * cb * 2, bytes = (uint32_t)(kBK - from) * cb * 2;
    if (go)
        for (int s = 0; s < nslots; s++) bulk_load(region + s * slot + from * cb * 2, g_zero_rows, bytes, bar);
    return bytes * nslots;
}

__global__ void __launch_bounds__(kThreads, 1) factor_syrk_kernel(const __grid_constant__ FactorParams P) {
    extern __shared__ uint8_t smem_raw[];
    uint8_t *smem = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint8_t *ops = smem;
    float *stage_buf = reinterpret_cast<float *>(smem + kSmemOps);
    ProbHdr *hdr = reinterpret_cast<ProbHdr *>(smem + kSmemOps + kSmemStage);
    uint64_t *bars = reinterpret_cast<uint64_t *>(smem + kSmemOps + kSmemStage + kSmemHdr);
    uint64_t *full = bars, *empty = bars + kStages, *tfull = bars + 2 * kStages, *tempty = bars + 2 * kStages + 2;
    uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(bars + 2 * kStages + 4);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int nprobs = P.nprobs;
    for (int p = threadIdx.x; p < nprobs; p += blockDim.x) {
        ProbHdr h;
        h.item_begin = P.probs[p].item_begin;
        h.npairs = P.probs[p].npairs;
        h.kchunks = P.probs[p].kchunks;
        h.cps = P.probs[p].chunks_per_split;
        h.ntm = P.probs[p].ntm;
        h.ntn = P.probs[p].ntn;
        h.pad = 0;
        hdr[p] = h;
    }
    // operand stages start zeroed: the K tail rows of short chunks then stay zero until a
    // longer chunk dirties them (tracked by the issuer, re-zeroed with bulk copies)
    for (size_t i = threadIdx.x; i < kSmemOps / 16; i += blockDim.x)
        reinterpret_cast<uint4 *>(ops)[i] = make_uint4(0u, 0u, 0u, 0u);
    fence_proxy_async_smem();
    if (threadIdx.x == 0) {
        for (int s = 0; s < kStages; s++) {
            mbar_init(&full[s], kIssuers);
            mbar_init(&empty[s], 1);
        }
        for (int b = 0; b < 2; b++) {
            mbar_init(&tfull[b], 1);
            mbar_init(&tempty[b], kEpiThreads);
        }
        fence_barrier_init();
    }
    if (warp == kMmaWarp) tmem_alloc(tmem_slot, kTmemCols);
    if (warp == kProdWarp0) {
        for (int p = lane; p < nprobs; p += 32)
            if (P.probs[p].mode != MODE_GATHER) tma_prefetch(&P.probs[p].tmap);
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;
    const int mma_fmt = P.ab_fmt == 1 ? 0 : 1;  // kind::f16 A/B format: 0 fp16, 1 bf16
    const int dec_fmt = P.ab_fmt;                // kfac_dtype: 0 bf16, 1 fp16
    const int dbg = P.dbg;
    const int total = P.total_items;

    if (warp >= kProdWarp0) {
        // ============================ producers ============================
        // 4 warps; lane 0 of each issues a quarter of the TMA boxes of every stage (the TMA engine
        // overlaps boxes from different issuers); all 128 threads gather in MODE_GATHER.
        const int ptid = threadIdx.x - kProdWarp0 * 32;
        const int pw = warp - kProdWarp0;
        uint32_t stage = 0, phase = 0;
        int cleanA[kStages], cleanB[kStages];  // rows >= clean*[s] of that operand region are zero
#pragma unroll
        for (int s = 0; s < kStages; s++) cleanA[s] = cleanB[s] = 0;
        for (int item = blockIdx.x; item < total; item += gridDim.x) {
            const ItemInfo it = decode_item(hdr, nprobs, item);
            const ProbRegs pr = load_prob(P.probs[it.p]);
            const CUtensorMap *tmap = &P.probs[it.p].tmap;
            // A (128 features at ti*128) is contained in B (256 features at tj*256) when tj == ti/2
            const bool a_in_b = it.tj == it.ti / 2;
            const int fa = it.ti * kTileM, fb = it.tj * kTileN;
            const int written = pr.mode == MODE_TILED4D ? pr.rpc : kBK;   // rows each slot receives
            const int needed = pr.ksteps * 16;                              // rows the MMA reads
            for (int kc = it.k0; kc < it.k1; kc++) {
                uint8_t *a = ops + (size_t)stage * kStageBytes;
                uint8_t *b = a + kOpA;
                if (pr.mode == MODE_GATHER) {
                    mbar_wait(&empty[stage], phase ^ 1);
                    gather_tile(pr, dec_fmt, b, fb, kTileN, kc, ptid);
                    if (!a_in_b) gather_tile(pr, dec_fmt, a, fa, kTileM, kc, ptid);
                    fence_proxy_async_smem();
                    named_bar_sync(1, kProdThreads);
                    if (lane == 0) mbar_arrive(&full[stage]);
                } else if (lane == 0) {
                    mbar_wait(&empty[stage], phase ^ 1);
                    if (dbg >= 2) {  // debug: no TMA (measures the MMA pipeline alone)
                        mbar_arrive(&full[stage]);
                    } else {
                        uint32_t bytes = issue_boxes(pr, tmap, a, b, &full[stage], fa, fb, a_in_b, kc, pw, false);
                        const bool zb = pw == 0 && cleanB[stage] > written && needed > written;
                        const bool za = pw == 0 && !a_in_b && cleanA[stage] > written && needed > written;
                        if (zb) bytes += zero_tail(b, kTileN / pr.cb, pr.cb, written, &full[stage], false);
                        if (za) bytes += zero_tail(a, kTileM / pr.cb, pr.cb, written, &full[stage], false);
                        mbar_arrive_expect_tx(&full[stage], bytes);
                        issue_boxes(pr, tmap, a, b, &full[stage], fa, fb, a_in_b, kc, pw, true);
                        if (zb) zero_tail(b, kTileN / pr.cb, pr.cb, written, &full[stage], true);
                        if (za) zero_tail(a, kTileM / pr.cb, pr.cb, written, &full[stage], true);
                    }
                }
                // every producer thread tracks the same tail state (only issuer 0 acts on it)
                cleanB[stage] = (cleanB[stage] > written && needed > written) ? written : max(cleanB[stage], written);
                if (!a_in_b) cleanA[stage] = (cleanA[stage] > written && needed > written) ? written : max(cleanA[stage], written);
                if (pr.mode == MODE_GATHER) cleanA[stage] = cleanB[stage] = kBK;
                if (++stage == kStages) {
                    stage = 0;
                    phase ^= 1;
                }
            }
        }
    } else if (warp == kMmaWarp) {
        // ============================ MMA issuer ============================
        uint32_t stage = 0, phase = 0;
        uint32_t tph0 = 0, tph1 = 0;
        int buf = 0;
        const uint32_t idesc = idesc_f16(mma_fmt, kTileM, kTileN, 1, 1);
        for (int item = blockIdx.x; item < total; item += gridDim.x) {
            const ItemInfo it = decode_item(hdr, nprobs, item);
            const int cb = P.probs[it.p].cb, ksteps = P.probs[it.p].ksteps;
            const bool a_in_b = it.tj == it.ti / 2;
            const uint32_t slot = kBK * cb * 2;
            const uint32_t lbo = slot, sbo = 8 * cb * 2, lay = layout_of(cb);
            const uint32_t kstep = 16 * cb * 2;  // bytes per K=16 slice
            const uint32_t tacc = tmem_base + buf * kTileN;
            if (lane == 0) {
                mbar_wait(&tempty[buf], (buf ? tph1 : tph0) ^ 1);
                tc_fence_after();
                for (int kc = it.k0; kc < it.k1; kc++) {
                    mbar_wait(&full[stage], phase);
                    tc_fence_after();
                    const uint32_t b_base = smem_u32(ops + (size_t)stage * kStageBytes + kOpA);
                    const uint32_t a_base = a_in_b ? b_base + (it.ti & 1) * (kTileM / cb) * slot
                                                   : smem_u32(ops + (size_t)stage * kStageBytes);
                    if (dbg == 1 || dbg == 4) {  // debug: no MMA (measures the TMA pipeline alone)
                        mbar_arrive(&empty[stage]);
                    } else {
                        for (int k = 0; k < ksteps; k++) {
                            uint64_t ad = umma_desc(a_base + k * kstep, lbo, sbo, lay);
                            uint64_t bd = umma_desc(b_base + k * kstep, lbo, sbo, lay);
                            mma_f16_ss(tacc, ad, bd, idesc, (kc > it.k0 || k > 0) ? 1u : 0u);
                        }
                        mma_commit(&empty[stage]);
                    }
                    if (++stage == kStages) {
                        stage = 0;
                        phase ^= 1;
                    }
                }
                if (dbg == 1 || dbg == 4) mbar_arrive(&tfull[buf]);
                else mma_commit(&tfull[buf]);
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
        for (int item = blockIdx.x; item < total; item += gridDim.x) {
            const ItemInfo it = decode_item(hdr, nprobs, item);
            const ProbRegs pr = load_prob(P.probs[it.p]);
            mbar_wait(&tfull[buf], buf ? tph1 : tph0);
            tc_fence_after();
            const uint32_t tacc = tmem_base + buf * kTileN + ((uint32_t)(warp * 32) << 16);
            const int gi0 = it.ti * kTileM, gj0 = it.tj * kTileN;
            float *part = pr.splits > 1
                              ? pr.partial + ((size_t)it.split * pr.npairs + it.tp) * (size_t)(kTileM * kTileN)
                              : nullptr;
            const int64_t dd = pr.d_out;
            for (int q = 0; q < kTileN / kQ; q++) {
                const int gq = gj0 + q * kQ;
                const bool any = gq < pr.d && gq + kQ - 1 >= gi0;  // group has valid upper entries
                if (any) {
                    uint32_t r[32];
                    tmem_ld_32x32b_x32(tacc + q * kQ, r);
                    tmem_ld_wait();
#pragma unroll
                    for (int i = 0; i < 32; i++) stage_buf[row * kStageLd + i] = __uint_as_float(r[i]);
                }
                if (q == kTileN / kQ - 1) {
                    tc_fence_before();
                    mbar_arrive(&tempty[buf]);  // accumulator drained: the MMA may reuse it
                }
                if (any && dbg != 5) {
                    named_bar_sync(2, kEpiThreads);
                    if (part) {
                        for (int r = warp; r < kTileM; r += 4)
                            part[(size_t)r * kTileN + q * kQ + lane] = stage_buf[r * kStageLd + lane];
                    } else {
                        for (int r = warp; r < kTileM; r += 4) {
                            const int gi = gi0 + r;
                            if (gi >= pr.d) break;
                            const int j = lane;
                            if (gq + j >= gi && gq + j < pr.d) {
                                float *orow = pr.out + ((int64_t)gi * dd - (int64_t)gi * (gi - 1) / 2 - gi);
                                orow[gq + j] = pr.alpha * stage_buf[r * kStageLd + j];
                            }
                        }
                    }
                    named_bar_sync(2, kEpiThreads);
                }
            }
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

// ordered split-K fix-up: out = alpha * sum_{s=0..S-1} partial[s] (deterministic).
// One block per (tile pair, 8-row group); warp = row, lane = 8 columns; all S x 8 loads independent.
__global__ void __launch_bounds__(256) factor_fixup_kernel(const __grid_constant__ FactorParams P) {
    int b = blockIdx.x >> 4;
    const int rg = blockIdx.x & 15;
    int p = 0;
    for (; p < P.nprobs; p++) {
        const FactorProb &pr = P.probs[p];
        if (pr.splits <= 1) continue;
        if (b < pr.npairs) break;
        b -= pr.npairs;
    }
    if (p >= P.nprobs) return;
    const FactorProb &pr = P.probs[p];
    int ti, tj;
    decode_pair(b, pr.ntm, pr.ntn, ti, tj);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int r = rg * 8 + warp;
    const int gi = ti * kTileM + r, gj0 = tj * kTileN;
    if (gi >= pr.d) return;
    const int jlo = max(0, gi - gj0), jhi = min(kTileN, pr.d - gj0);
    if (jlo >= jhi) return;
    const size_t tile = (size_t)kTileM * kTileN, sstride = (size_t)pr.npairs * tile;
    const float *src = pr.partial + (size_t)b * tile + (size_t)r * kTileN + lane;
    float acc[8];
#pragma unroll
    for (int k = 0; k < 8; k++) acc[k] = 0.f;
    for (int sp = 0; sp < pr.splits; sp++) {
#pragma unroll
        for (int k = 0; k < 8; k++) acc[k] += __ldg(src + sp * sstride + 32 * k);
    }
    const int64_t dd = pr.d_out;
    float *orow = pr.out + ((int64_t)gi * dd - (int64_t)gi * (gi - 1) / 2 - gi) + gj0;
#pragma unroll
    for (int k = 0; k < 8; k++) {
        const int j = lane + 32 * k;
        if (j >= jlo && j < jhi) orow[j] = pr.alpha * acc[k];
    }
}

// materialise the im2col rows of problems with im2col_pre: col[q][f] = ã_f(q), zero for f >= d
__global__ void __launch_bounds__(256) im2col_kernel(const __grid_constant__ FactorParams P) {
    const ProbRegs pr = load_prob(P.probs[blockIdx.y]);
    if (!P.probs[blockIdx.y].im2col_pre) return;
    uint16_t *col = P.probs[blockIdx.y].col;
    const int cp = P.probs[blockIdx.y].cp, nq = cp / 8;
    const int hw = pr.ho * pr.wo;
    for (int64_t u = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; u < pr.rows * nq; u += (int64_t)gridDim.x * blockDim.x) {
        const int64_t row = u / nq;
        const int q = (int)(u - row * nq);
        const int64_t n = row / hw;
        const int rem = (int)(row - n * hw);
        const int oh = rem / pr.wo, ow = rem - oh * pr.wo;
        int f = q * 8;
        int kk = f / pr.c, c = f - kk * pr.c;
        int i = kk / pr.kw, j = kk - i * pr.kw;
        const uint16_t *base = pr.src + n * (int64_t)pr.h * pr.w * pr.c;
        uint32_t pk[4] = {0u, 0u, 0u, 0u};
#pragma unroll
        for (int e = 0; e < 8; e++) {
            uint16_t v = 0;
            if (f + e < pr.d) {
                const int h = oh * pr.sh - pr.ph + i, w = ow * pr.sw - pr.pw + j;
                if (h >= 0 && h < pr.h && w >= 0 && w < pr.w) v = __ldg(base + ((int64_t)h * pr.w + w) * pr.c + c);
            }
            pk[e >> 1] |= (uint32_t)v << ((e & 1) * 16);
            if (++c == pr.c) {
                c = 0;
                if (++j == pr.kw) {
                    j = 0;
                    ++i;
                }
            }
        }
        reinterpret_cast<uint4 *>(col)[u] = make_uint4(pk[0], pk[1], pk[2], pk[3]);
    }
}

// bias row/column of A: A[f][dA-1] = alpha * sum_rows ã_f, A[dA-1][dA-1] = alpha * rows
// (the homogeneous coordinate, reading R-5); one thread per feature, fixed row order.
__global__ void __launch_bounds__(256) factor_bias_kernel(const __grid_constant__ FactorParams P) {
    const ProbRegs pr = load_prob(P.probs[blockIdx.y]);
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


static PFN_encodeTiled g_encTiled = nullptr;
static int g_driver = 0;

static kfac_status load_driver_fns() {
    if (g_encTiled) return KFAC_OK;
    cudaDriverEntryPointQueryResult q1;
    void *f1 = nullptr;
    KFAC_CUDA_TRY(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f1, cudaEnableDefault, &q1));
    if (!f1) return set_error(KFAC_ERR_CUDA, "cuTensorMapEncodeTiled entry point unavailable");
    g_encTiled = (PFN_encodeTiled)f1;
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

// Geometry of one factor problem (no pointers): the mode the kernel will use, the
// chunking of K, the tile grid.  Shared by plan-time sizing and launch-time setup.
static void prob_geometry(const FactorJob &j, bool src_aligned, FactorProb *pr) {
    const Geom &g = j.g;
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
    pr->ntm = (pr->d + kTileM - 1) / kTileM;
    pr->ntn = (pr->d + kTileN - 1) / kTileN;
    pr->npairs = 0;
    for (int ti = 0; ti < pr->ntm; ti++) pr->npairs += pr->ntn - ti / 2;
    const int C = pr->c;
    const bool plain = (pr->kh == 1 && pr->kw == 1 && pr->sh == 1 && pr->sw == 1 && pr->ph == 0 && pr->pw == 0);
    const bool aligned16 = (C % 8) == 0 && src_aligned;
    int mode = MODE_GATHER, cb = 64;
    if (!force_gather() && aligned16) {
        if (plain) {
            mode = MODE_TILED2D;
            cb = C >= 64 ? 64 : (C > 16 ? (C > 32 ? 64 : 32) : 16);
        } else if (C % 16 == 0 && pr->wo <= kBK && (pr->wo - 1) * pr->sw + 1 <= 256 && pr->sw <= 8 && pr->sh <= 8) {
            mode = MODE_TILED4D;
            cb = (C % 64 == 0) ? 64 : ((C % 32 == 0) ? 32 : 16);
        }
    }
    pr->im2col_pre = 0;
    pr->cp = 0;
    if (mode == MODE_GATHER && !force_gather() && j.is_A && !plain && src_aligned) {
        // channel stride not a multiple of 16 B (e.g. the RGB stem): TMA cannot address the
        // pixels, so the patches are materialised once as [rows, cp] (cp = dF rounded to 8)
        // and staged by the 2-D TMA path
        pr->im2col_pre = 1;
        pr->cp = (int16_t)((pr->d + 7) / 8 * 8);
        mode = MODE_TILED2D;
        cb = pr->cp >= 64 ? 64 : (pr->cp > 16 ? (pr->cp > 32 ? 64 : 32) : 16);
    }
    pr->mode = mode;
    pr->cb = cb;
    pr->bh = pr->bn = 1;
    pr->rpi = 1;
    if (mode == MODE_TILED4D) {
        int bh = 1;
        for (int b = 1; b <= pr->ho; b++)
            if (pr->ho % b == 0 && b * pr->wo <= kBK) bh = b;
        pr->bh = bh;
        pr->rpi = pr->ho / bh;
        pr->bn = (bh == pr->ho) ? std::max(1, kBK / (pr->ho * pr->wo)) : 1;
        pr->rpc = pr->bn * bh * pr->wo;
        const int64_t N = j.n;
        pr->kchunks = bh < pr->ho ? (int)(N * pr->rpi) : (int)((N + pr->bn - 1) / pr->bn);
    } else {
        pr->rpc = kBK;
        pr->kchunks = (int)((pr->rows + kBK - 1) / kBK);
    }
    pr->ksteps = (pr->rpc + 15) / 16;
}

// pointers + TMA descriptor of one factor problem
static kfac_status setup_prob(const FactorJob &j, kfac_dtype dt, FactorProb *pr) {
    pr->src = static_cast<const uint16_t *>(j.src);
    pr->out = j.out;
    pr->alpha = j.alpha;
    if (pr->mode == MODE_GATHER) return KFAC_OK;
    kfac_status s = load_driver_fns();
    if (s) return s;
    const int C = pr->c, cb = pr->cb;
    const CUtensorMapDataType dty = dt == KFAC_FP16 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT16 : CU_TENSOR_MAP_DATA_TYPE_BFLOAT16;
    const int64_t N = pr->rows / ((int64_t)pr->ho * pr->wo);
    const int64_t bytes = N * pr->h * pr->w * (int64_t)C * 2;
    CUresult r;
    if (pr->mode == MODE_TILED2D) {
        const int64_t W = pr->im2col_pre ? pr->cp : C;
        void *base = pr->im2col_pre ? (void *)pr->col : const_cast<void *>(j.src);
        cuuint64_t dims[2] = {(cuuint64_t)W, (cuuint64_t)pr->rows};
        cuuint64_t strides[1] = {(cuuint64_t)W * 2};
        cuuint32_t box[2] = {(cuuint32_t)cb, (cuuint32_t)kBK};
        cuuint32_t es[2] = {1, 1};
        r = g_encTiled(&pr->tmap, dty, 2, base, dims, strides, box, es,
                       CU_TENSOR_MAP_INTERLEAVE_NONE, swz_of(cb), CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                       CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    } else {
        // 4-D tiled box: cb channels x Wo output columns x bh output rows x bn images of one filter
        // tap; the tap shifts the start coordinate, the conv stride is the traversal stride and the
        // zero padding is the TMA out-of-bounds fill.
        cuuint64_t dims[4] = {(cuuint64_t)C, (cuuint64_t)pr->w, (cuuint64_t)pr->h, (cuuint64_t)N};
        cuuint64_t strides[3] = {(cuuint64_t)C * 2, (cuuint64_t)C * 2 * pr->w, (cuuint64_t)C * 2 * pr->w * pr->h};
        cuuint32_t box[4] = {(cuuint32_t)cb, (cuuint32_t)((pr->wo - 1) * pr->sw + 1),
                             (cuuint32_t)((pr->bh - 1) * pr->sh + 1), (cuuint32_t)pr->bn};
        cuuint32_t es[4] = {1, (cuuint32_t)pr->sw, (cuuint32_t)pr->sh, 1};
        r = g_encTiled(&pr->tmap, dty, 4, const_cast<void *>(j.src), dims, strides, box, es,
                       CU_TENSOR_MAP_INTERLEAVE_NONE, swz_of(cb), CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                       CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    }
    if (r != CUDA_SUCCESS) {
        char buf[200];
        snprintf(buf, sizeof buf, "cuTensorMapEncodeTiled failed (%d) for C=%d mode=%d wo=%d bh=%d bn=%d", (int)r, C,
                 pr->mode, pr->wo, pr->bh, pr->bn);
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
    if (!dry_run && !g_num_sms) {
        int dev = 0;
        KFAC_CUDA_TRY(cudaGetDevice(&dev));
        KFAC_CUDA_TRY(cudaDeviceGetAttribute(&g_num_sms, cudaDevAttrMultiProcessorCount, dev));
    }
    const int nj = (int)jobs.size();
    std::vector<FactorProb> geo(nj);
    double total = 0;  // MMA K-steps over all tile pairs
    for (int i = 0; i < nj; i++) {
        memset(&geo[i], 0, sizeof(FactorProb));
        const bool aligned = dry_run || (reinterpret_cast<uintptr_t>(jobs[i].src) % 16) == 0;
        prob_geometry(jobs[i], aligned, &geo[i]);
        total += (double)geo[i].npairs * geo[i].kchunks * geo[i].ksteps;
    }
    // split K so that work items are ~1/3 of a CTA's fair share (static striding then balances)
    // -- fixed 148-SM target so that plan-time workspace sizing matches every launch
    const double target = std::max(64.0, total / (3.0 * 148));
    std::vector<int> splits(nj);
    std::vector<double> item_cost(nj);
    int64_t need = 0;
    for (int i = 0; i < nj; i++) {
        const FactorProb &g = geo[i];
        const double per_tile = (double)g.kchunks * g.ksteps;
        int S = (int)std::max(1.0, std::min<double>(g.kchunks, std::ceil(per_tile / target)));
        const int cps = (g.kchunks + S - 1) / S;
        S = (g.kchunks + cps - 1) / cps;
        splits[i] = S;
        item_cost[i] = (double)cps * g.ksteps;
        if (S > 1) need += (int64_t)g.npairs * S * kTileM * kTileN * 4;
    }
    int64_t col_need = 0;
    for (int i = 0; i < nj; i++)
        if (geo[i].im2col_pre) col_need += (geo[i].rows * geo[i].cp * 2 + 255) / 256 * 256;
    if (!dry_run && need + col_need > ws_cap) {  // not enough scratch (e.g. a fallback mode changed the chunking)
        for (int i = 0; i < nj; i++) splits[i] = 1, item_cost[i] = (double)geo[i].kchunks * geo[i].ksteps;
        need = 0;
    }
    if (!dry_run && col_need > ws_cap) return set_error(KFAC_ERR_ARG, "factor workspace too small for im2col staging");
    // heaviest items first
    std::vector<int> order(nj);
    for (int i = 0; i < nj; i++) order[i] = i;
    std::stable_sort(order.begin(), order.end(), [&](int a, int b) { return item_cost[a] > item_cost[b]; });
    int64_t ws_off = 0, col_off = 0;
    for (int base = 0; base < nj; base += kMaxProbs) {
        FactorParams P;
        memset(&P, 0, sizeof(P));
        P.ab_fmt = (int)dt;
        P.dbg = getenv("KFAC_DBG_MODE") ? atoi(getenv("KFAC_DBG_MODE")) : 0;
        int items = 0;
        const int cnt = std::min(kMaxProbs, nj - base);
        for (int k = 0; k < cnt; k++) {
            const int i = order[base + k];
            FactorProb &pr = P.probs[k];
            pr = geo[i];
            if (pr.im2col_pre) {
                pr.col = ws ? reinterpret_cast<uint16_t *>(static_cast<uint8_t *>(ws) + need + col_off) : nullptr;
                col_off += (pr.rows * pr.cp * 2 + 255) / 256 * 256;
            }
            if (!dry_run) {
                kfac_status s = setup_prob(jobs[i], dt, &pr);
                if (s) return s;
            }
            const int S = splits[i];
            pr.chunks_per_split = (pr.kchunks + S - 1) / S;
            pr.splits = S;
            pr.item_begin = items;
            items += pr.npairs * S;
            if (S > 1) {
                pr.partial = ws ? reinterpret_cast<float *>(static_cast<uint8_t *>(ws) + ws_off) : nullptr;
                ws_off += (int64_t)pr.npairs * S * kTileM * kTileN * 4;
            }
        }
        P.nprobs = cnt;
        P.total_items = items;
        if (!dry_run && getenv("KFAC_DEBUG")) {
            for (int k = 0; k < cnt; k++) {
                const FactorProb &pr = P.probs[k];
                fprintf(stderr,
                        "[kfac] factor prob %d: d=%d rows=%lld mode=%d cb=%d rpc=%d ksteps=%d bh=%d bn=%d pairs=%d "
                        "kchunks=%d splits=%d\n",
                        k, pr.d, (long long)pr.rows, pr.mode, pr.cb, pr.rpc, pr.ksteps, pr.bh, pr.bn, pr.npairs,
                        pr.kchunks, pr.splits);
            }
            fprintf(stderr, "[kfac] factor launch: %d problems, %d items, target %.0f k-steps/item\n", P.nprobs, items,
                    target);
        }
        out->params.push_back(P);
    }
    out->ws_bytes = need + col_need;
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
        bool pre = false;
        for (int p = 0; p < P.nprobs; p++) pre |= P.probs[p].im2col_pre != 0;
        if (pre) {
            im2col_kernel<<<dim3(2 * (g_num_sms ? g_num_sms : 148), P.nprobs), 256, 0, st>>>(P);
            KFAC_LAUNCHED();
            KFAC_CUDA_TRY(cudaGetLastError());
        }
        int grid = std::min(P.total_items, g_num_sms ? g_num_sms : 148);
        factor_syrk_kernel<<<grid, kThreads, kSmemBytes, st>>>(P);
        KFAC_LAUNCHED();
        KFAC_CUDA_TRY(cudaGetLastError());
        int fix = 0, maxbias = 0;
        for (int p = 0; p < P.nprobs; p++) {
            const FactorProb &pr = P.probs[p];
            if (pr.splits > 1) fix += pr.npairs;
            if (pr.d_out != pr.d) maxbias = std::max(maxbias, pr.d + 1);
        }
        if (fix && !getenv("KFAC_NO_FIXUP")) {
            factor_fixup_kernel<<<fix * 16, 256, 0, st>>>(P);
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
