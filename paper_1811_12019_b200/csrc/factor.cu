// factor.cu -- stages 1-2 of distributed K-FAC (PAPER.md P:237-245 Eq. kf,
// P:313-318): the Kronecker factors
//     A = alpha * sum_rows ã ãᵀ   over im2col patches ã (+ bias coordinate 1)
//     G = alpha * sum_rows g gᵀ   over output-gradient pixels g
// as ONE grouped, persistent tcgen05 SYRK launch over every (layer, factor):
//
//   * output tiles are 256 x 256 (upper tiles ti <= tj only): per 16-row K step
//     two tcgen05.mma kind::f16 M=128 x N=256 (bf16/fp16 in, fp32 accumulate in
//     TMEM, "mixed precision") share one B operand, so a stage of
//     64 pixel rows x (256 + 256) features feeds 2 x 128 x 256 x 64 MACs; on a
//     diagonal tile A == B (loaded once) and the lower half's MMA is N = 128;
//   * operands are staged by TMA straight from the NHWC activation tensor, in
//     slots of cb (64) channels, MN-major SW128, K = pixels.  One TMA box
//     carries S (up to 4) consecutive channel slots of one filter tap
//     (3-D map {cb, rows, C/cb} for G / 1x1 convs / FC, 5-D map
//     {cb, W, H, N, C/cb} for k>1 or strided convs): patch extraction is fused
//     into the shared-memory staging, no im2col matrix is materialised.  Every
//     chunk is exactly 64 pixel rows: the box width is the output width rounded
//     up to a power of two and the phantom columns are zero-filled by the TMA
//     out-of-bounds rule (one descriptor per distinct right edge, i.e. per
//     filter column), so the 16-row MMA steps never read past a slot;
//     a gather producer (plain loads) covers the geometries TMA cannot
//     express; the RGB stem (3 channels, 6 B pixels) is materialised once;
//   * each output element is written once, packed upper row-major
//     (P:407-411), straight into the ReduceScatter send buffer;
//   * large-K/small-d problems are split along K with a deterministic,
//     ordered fix-up (reading R-18).
//
// Warp roles (416 threads): warps 0-7 epilogue (TMEM -> smem -> packed
// global; warp w drains rows 32*(w%4).. of accumulator half w/4), warp 8 TMEM
// allocator + MMA issuer, warps 9-12 TMA producers (lane 0 issues).
#include <cuda_bf16.h>
#include <cuda_fp16.h>

#include <algorithm>
#include <mutex>
#include <cstdio>
#include <cstdlib>
#include <cstring>

#include "kfac_internal.hpp"
#include "sm100.cuh"

namespace kfac {

constexpr int kStages = 3;
constexpr int kHalf = 128;                                  // MMA M
constexpr int kEpiWarps = 8;
constexpr int kEpiThreads = kEpiWarps * 32;
constexpr int kMmaWarp = kEpiWarps;
constexpr int kProdWarp0 = kEpiWarps + 1;
#ifndef KFAC_PROD_WARPS
#define KFAC_PROD_WARPS 4
#endif
constexpr int kProdWarps = KFAC_PROD_WARPS;
constexpr int kProdThreads = kProdWarps * 32;
#ifndef KFAC_ISSUE_LANES
#define KFAC_ISSUE_LANES 1
#endif
constexpr int kIssueLanes = KFAC_ISSUE_LANES;                              // TMA-issuing lanes per producer warp
constexpr int kIssuers = kProdWarps * kIssueLanes;
constexpr int kThreads = kEpiThreads + 32 + kProdThreads;  // 416
constexpr int kOp = kTile * kBK * 2;                        // 32 KB operand (256 features x 64 rows)
constexpr int kStageBytes = 2 * kOp;
constexpr int kQ = 16;                                      // epilogue column group (one tcgen05.ld x16)
constexpr int kStageLd = 20;                                // staging row stride (floats; v4 stores conflict-free)
constexpr int kTmemCols = 2 * kTile;                        // two 128 x 256 fp32 accumulators
constexpr size_t kSmemOps = (size_t)kStages * kStageBytes;
constexpr size_t kSmemStage = (size_t)kEpiWarps * 32 * kStageLd * 4;
constexpr size_t kSmemHdr = (size_t)kMaxProbs * 24;         // per-problem decode table
constexpr int kQueue = 4;                                   // work-item queue depth (items the producers may run ahead)
constexpr int kConsumerWarps = kProdWarps + 1 + kEpiWarps;  // warps that read every queue entry
constexpr size_t kSmemBytes = 1024 + kSmemOps + kSmemStage + kSmemHdr + 512;
static_assert(kSmemBytes <= 232448, "shared memory budget");

__device__ __forceinline__ float dec_half(uint16_t b, int fmt) {
    if (fmt == 1) return __half2float(__ushort_as_half(b));
    return __uint_as_float(((uint32_t)b) << 16);
}

struct ItemInfo {
    int p, ti, tj, split, tp, k0, k1;
};

// tile pair tp -> (ti, tj), ti <= tj, row-major over the upper triangle of an nt x nt tile grid
__device__ __forceinline__ void decode_pair(int tp, int nt, int &ti, int &tj) {
    int t = 0, rem = tp;
    while (rem >= nt - t) {
        rem -= nt - t;
        t++;
    }
    ti = t;
    tj = t + rem;
}

// per-problem decode fields, copied to shared memory once per CTA (dynamic indexing of the
// kernel-parameter array goes through the constant cache and is slow)
struct ProbHdr {
    int32_t item_begin, npairs, kchunks, cps;
    int32_t nt, pad;
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
    decode_pair(it.tp, h.nt, it.ti, it.tj);
    it.p = lo;
    it.k0 = it.split * h.cps;
    it.k1 = min(h.kchunks, it.k0 + h.cps);
    return it;
}

// register copy of the fields a role needs for one work item
struct ProbRegs {
    int mode, d, d_out, cb, S, ksteps, bh, bn, rpi, c, h, w, ho, wo, kh, kw, sh, sw, ph, pw, splits, npairs, map0;
    uint64_t mapj;
    float alpha;
    float *out, *partial;
    const uint16_t *src;
    int64_t rows;
};
__device__ __forceinline__ ProbRegs load_prob(const FactorProb &g) {
    ProbRegs r;
    r.mode = g.mode; r.d = g.d; r.d_out = g.d_out; r.cb = g.cb; r.S = g.S; r.ksteps = g.ksteps;
    r.bh = g.bh; r.bn = g.bn; r.rpi = g.rpi; r.c = g.c; r.h = g.h; r.w = g.w; r.ho = g.ho; r.wo = g.wo;
    r.kh = g.kh; r.kw = g.kw; r.sh = g.sh; r.sw = g.sw; r.ph = g.ph; r.pw = g.pw; r.splits = g.splits;
    r.npairs = g.npairs; r.map0 = g.map0; r.mapj = g.mapj; r.alpha = g.alpha; r.out = g.out;
    r.partial = g.partial; r.src = g.src; r.rows = g.rows;
    return r;
}

__device__ __forceinline__ uint32_t layout_of(int cb) {
    return cb == 64 ? UMMA_SW128 : (cb == 32 ? UMMA_SW64 : UMMA_SW32);
}

// gather one element: feature f (< d) of output row q (< rows)  [bias kernel]
__device__ __forceinline__ float gather_elem(const ProbRegs &pr, int fmt, int q, int f) {
    int hw = pr.ho * pr.wo;
    int n = q / hw;
    int rem = q - n * hw;
    int oh = rem / pr.wo, ow = rem - oh * pr.wo;
    int kk = f / pr.c, c = f - kk * pr.c;
    int i = kk / pr.kw, j = kk - i * pr.kw;
    int h = oh * pr.sh - pr.ph + i, w = ow * pr.sw - pr.pw + j;
    if (h < 0 || h >= pr.h || w < 0 || w >= pr.w) return 0.f;
    return dec_half(__ldg(pr.src + (((int64_t)(n * pr.h + h) * pr.w + w) * pr.c + c)), fmt);
}

// gather producer: fill 256 features (from f_base) x 64 rows in the SW128 MN-major slot layout
// (cb = 64), zero outside the matrix
__device__ __forceinline__ void gather_tile(const ProbRegs &pr, uint8_t *dst, int f_base, int kc, int tid) {
    constexpr int nq = kTile / 8;  // 16-byte chunks per row
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
        const int box = q >> 3, cq = q & 7;
        uint8_t *p = dst + box * (kBK * 128) + r * 128 + ((cq ^ (r & 7)) << 4);
        *reinterpret_cast<uint4 *>(p) = make_uint4(pk[0], pk[1], pk[2], pk[3]);
    }
}

// The TMA boxes of one stage: operand B (256 features from fb), then -- off the diagonal --
// operand A (from fa); box b of an operand carries features [f_base + b*cb*S, +cb*S) = S channel
// slots of one filter tap.  Issuer w owns boxes k = w, w + kIssuers, ... of the stage; the
// chunk-independent part of each owned box (destination, descriptor, tap offsets, slot) is
// decoded once per work item, so the per-chunk issue loop is a handful of integer ops.
constexpr int kMaxOwned = 8;  // 2 operands x <= 16 boxes (cb * S >= 16) / kIssuers
static_assert(2 * kTile / 16 <= kMaxOwned * kIssuers, "owned box list");
struct OwnedBoxes {
    uint32_t dst[kMaxOwned];   // byte offset in the stage
    uint32_t tap[kMaxOwned];   // map index | (dw + 128) << 8 | (dh + 128) << 16 | slot << 24 (TILED4D)
    int n, bytes;
};
__device__ __forceinline__ void own_boxes(const ProbRegs &pr, int fa, int fb, bool diag, int w, OwnedBoxes &ob) {
    const int fpb = pr.cb * pr.S;
    const uint32_t box_bytes = (uint32_t)kBK * fpb * 2;  // S slots of kBK rows
    ob.n = 0;
    ob.bytes = 0;
    int k = 0;
    for (int op = 0; op < (diag ? 1 : 2); op++) {
        const int f_base = op == 0 ? fb : fa;
        const uint32_t base = (op == 0 && !diag) ? kOp : 0;  // diagonal: B (== A) from the stage start
        const int nbox = (min(kTile, pr.d - f_base) + fpb - 1) / fpb;
        for (int b = 0; b < nbox; b++, k++) {
            if (k % kIssuers != w || ob.n >= kMaxOwned) continue;
            const int f0 = f_base + b * fpb;
            uint32_t tap;
            if (pr.mode == MODE_TILED2D) {
                tap = (uint32_t)pr.map0 | ((uint32_t)(f0 / pr.cb) << 24);
            } else {
                const int kk = f0 / pr.c, c0 = f0 - kk * pr.c;
                const int i = kk / pr.kw, j = kk - i * pr.kw;
                const int mi = pr.map0 + (int)((pr.mapj >> (8 * j)) & 0xff);
                tap = (uint32_t)mi | ((uint32_t)(j - pr.pw + 128) << 8) | ((uint32_t)(i - pr.ph + 128) << 16) |
                      ((uint32_t)(c0 / pr.cb) << 24);
            }
            ob.dst[ob.n] = base + b * box_bytes;
            ob.tap[ob.n] = tap;
            ob.n++;
            ob.bytes += box_bytes;
        }
    }
}

// K units (64-row chunks) per pipeline stage: an off-diagonal tile loads A and B (512 features
// per unit, one unit fills a stage); a diagonal tile loads only B, so a stage holds 512 / (features
// loaded) units -- more MMA work per stage round trip (each commit -> empty -> refill round trip
// costs ~500 cycles of tensor-pipe time that only long enough stages hide).  Stage layout
// [unit][slot][64 rows][cb].
__device__ __forceinline__ int item_units(int mode, int fpb, int d, int tj, bool diag, int &unit_bytes) {
    const int fl = (min(kTile, d - tj * kTile) + fpb - 1) / fpb * fpb;  // B features loaded per unit
    unit_bytes = fl * kBK * 2;
    if (!diag || mode == MODE_GATHER) return 1;
    return min(8, 2 * kTile / fl);
}

// Work distribution: items are handed out in order (heaviest first) by a global atomic counter,
// one at a time, to whichever CTA asks -- a dynamic longest-processing-time schedule.  Producer
// warp 0 fetches item s on demand into a kQueue-deep shared-memory queue; every role reads the
// same sequence.  Without a counter the CTA takes items blockIdx.x + s * gridDim.x.
__device__ __forceinline__ int next_item(uint32_t s, const FactorParams &P, int *qitem, uint64_t *qfull,
                                         uint64_t *qempty, bool scheduler, int lane) {
    const int slot = (int)(s % kQueue);
    const uint32_t ph = (s / kQueue) & 1;
    if (scheduler && lane == 0) {
        mbar_wait(&qempty[slot], ph ^ 1);
        qitem[slot] = P.counter ? atomicAdd(P.counter, 1) : (int)(blockIdx.x + s * gridDim.x);
        mbar_arrive(&qfull[slot]);
    }
    mbar_wait(&qfull[slot], ph);
    const int item = qitem[slot];
    __syncwarp();
    if (lane == 0) mbar_arrive(&qempty[slot]);
    return item;
}

#ifndef KFAC_EPI_V4
#define KFAC_EPI_V4 1
#endif
#ifdef KFAC_FACTOR_PROF  // experiment build only: per-role cycle accounting printed by CTAs 0 and 100
#define FPROF(...) __VA_ARGS__
#else
#define FPROF(...)
#endif

__global__ void __launch_bounds__(kThreads, 1) factor_syrk_kernel(const __grid_constant__ FactorParams P) {
    FPROF(long long pf_start = clock64(); long long pf_a = 0, pf_b = 0, pf_c = 0, pf_i = 0, pf_q = 0, pf_e = 0; int pf_n = 0;)
    extern __shared__ uint8_t smem_raw[];
    uint8_t *smem = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint8_t *ops = smem;
    float *stage_buf = reinterpret_cast<float *>(smem + kSmemOps);
    ProbHdr *hdr = reinterpret_cast<ProbHdr *>(smem + kSmemOps + kSmemStage);
    uint64_t *bars = reinterpret_cast<uint64_t *>(smem + kSmemOps + kSmemStage + kSmemHdr);
    uint64_t *full = bars, *empty = bars + kStages, *tfull = bars + 2 * kStages, *tempty = bars + 2 * kStages + 1;
    uint64_t *qfull = bars + 2 * kStages + 3, *qempty = qfull + kQueue;
    int *qitem = reinterpret_cast<int *>(qempty + kQueue);
    uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(qitem + kQueue);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int nprobs = P.nprobs;
    for (int p = threadIdx.x; p < nprobs; p += blockDim.x) {
        ProbHdr h;
        h.item_begin = P.probs[p].item_begin;
        h.npairs = P.probs[p].npairs;
        h.kchunks = P.probs[p].kchunks;
        h.cps = P.probs[p].chunks_per_split;
        h.nt = P.probs[p].nt;
        h.pad = 0;
        hdr[p] = h;
    }
    if (threadIdx.x == 0) {
        for (int s = 0; s < kStages; s++) {
            mbar_init(&full[s], kIssuers);
            mbar_init(&empty[s], 1);
        }
        mbar_init(tfull, 1);
        mbar_init(&tempty[0], kEpiThreads / 2);
        mbar_init(&tempty[1], kEpiThreads / 2);
        for (int q = 0; q < kQueue; q++) {
            mbar_init(&qfull[q], 1);
            mbar_init(&qempty[q], kConsumerWarps);
        }
        fence_barrier_init();
    }
    if (warp == kMmaWarp) tmem_alloc(tmem_slot, kTmemCols);
    if (warp == kProdWarp0) {
        for (int m = lane; m < P.nmaps; m += 32) tma_prefetch(&P.maps[m]);
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;
    const int mma_fmt = P.ab_fmt == 1 ? 0 : 1;  // kind::f16 A/B format: 0 fp16, 1 bf16
    const int dbg = P.dbg;
    const bool no_mma = dbg == 1 || dbg == 4, no_tma = dbg >= 2, no_store = dbg == 5;
    const int total = P.total_items;

    if (warp >= kProdWarp0) {
        // ============================ producers ============================
        // lanes 0..kIssueLanes-1 of each warp issue a share of the TMA boxes of every stage (the
        // TMA engine overlaps boxes from different issuers); all 128 threads gather in MODE_GATHER.
        const int ptid = threadIdx.x - kProdWarp0 * 32;
        const int wid = (warp - kProdWarp0) * kIssueLanes + lane;
        const bool issuer = lane < kIssueLanes;
        uint32_t stage = 0, phase = 0;
        for (uint32_t s = 0;; s++) {
            const int item = next_item(s, P, qitem, qfull, qempty, warp == kProdWarp0, lane);
            if (item >= total) break;
            const ItemInfo it = decode_item(hdr, nprobs, item);
            const ProbRegs pr = load_prob(P.probs[it.p]);
            const bool diag = it.ti == it.tj;
            const int fa = it.ti * kTile, fb = it.tj * kTile;
            OwnedBoxes ob;
            if (pr.mode != MODE_GATHER && issuer) own_boxes(pr, fa, fb, diag, wid, ob);
            int ub;
            const int rf = item_units(pr.mode, pr.cb * pr.S, pr.d, it.tj, diag, ub);
            // TILED4D chunk origin (image n, first output row oh0), advanced incrementally
            int ig = it.k0 / pr.rpi, rg = it.k0 - ig * pr.rpi;
            for (int kc = it.k0; kc < it.k1;) {
                const int units = min(rf, it.k1 - kc);
                uint8_t *a = ops + (size_t)stage * kStageBytes;
                uint8_t *b = a + kOp;
                if (pr.mode == MODE_GATHER) {
                    mbar_wait(&empty[stage], phase ^ 1);
                    gather_tile(pr, diag ? a : b, fb, kc, ptid);  // diagonal: B (== A) at the stage start
                    if (!diag) gather_tile(pr, a, fa, kc, ptid);
                    fence_proxy_async_smem();
                    named_bar_sync(1, kProdThreads);
                    if (issuer) mbar_arrive(&full[stage]);
                } else if (issuer) {
                    FPROF(long long t0 = clock64();)
                    mbar_wait(&empty[stage], phase ^ 1);
                    FPROF(pf_a += clock64() - t0; pf_n++; t0 = clock64();)
                    if (no_tma) {
                        mbar_arrive(&full[stage]);
                    } else {
                        mbar_arrive_expect_tx(&full[stage], ob.bytes * units);
                        int ig2 = ig, rg2 = rg;
                        for (int u = 0; u < units; u++) {
                            const int n = ig2 * pr.bn, h0 = rg2 * pr.bh * pr.sh, k64 = (kc + u) * kBK;
                            uint8_t *ubase = a + u * ub;
#pragma unroll
                            for (int q = 0; q < kMaxOwned; q++) {
                                if (q < ob.n) {
                                    const uint32_t t = ob.tap[q];
                                    const CUtensorMap *m = &P.maps[t & 0xff];
                                    if (pr.mode == MODE_TILED2D)
                                        tma_load_3d(ubase + ob.dst[q], m, &full[stage], 0, k64, (int)(t >> 24));
                                    else
                                        tma_load_5d(ubase + ob.dst[q], m, &full[stage], 0, (int)((t >> 8) & 0xff) - 128,
                                                    h0 + (int)((t >> 16) & 0xff) - 128, n, (int)(t >> 24));
                                }
                            }
                            if (++rg2 == pr.rpi) {
                                rg2 = 0;
                                ig2++;
                            }
                        }
                    }
                    FPROF(pf_c += clock64() - t0;)
                }
                for (int u = 0; u < units; u++)
                    if (++rg == pr.rpi) {
                        rg = 0;
                        ig++;
                    }
                kc += units;
                // keep the non-issuing lanes in step with the issuers: an mbarrier parity wait
                // cannot tell phases apart that are two or more apart, so a lane that ran ahead
                // into a later gather item would see a stale "empty" phase as free
                __syncwarp();
                if (++stage == kStages) {
                    stage = 0;
                    phase ^= 1;
                }
            }
        }
    } else if (warp == kMmaWarp) {
        // ============================ MMA issuer ============================
        uint32_t stage = 0, phase = 0, tph = 0;
        for (uint32_t s = 0;; s++) {
            FPROF(long long tq = clock64();)
            const int item = next_item(s, P, qitem, qfull, qempty, false, lane);
            FPROF(pf_q += clock64() - tq; tq = clock64();)
            if (item >= total) break;
            const ItemInfo it = decode_item(hdr, nprobs, item);
            const int cb = P.probs[it.p].cb, ksteps = P.probs[it.p].ksteps, d = P.probs[it.p].d;
            const bool diag = it.ti == it.tj;
            const int nr = min(kTile, d - it.ti * kTile), nc = min(kTile, d - it.tj * kTile);
            const int n0 = (nc + 15) / 16 * 16;          // N of the upper-half MMA
            const bool h1 = nr > kHalf;                   // lower half has valid rows
            const int n1 = diag ? n0 - kHalf : n0;        // diagonal: only columns >= 128 reach the upper triangle
            const uint32_t slot = kBK * cb * 2;
            const uint32_t lbo = slot, sbo = 8 * cb * 2, lay = layout_of(cb);
            const uint32_t kstep = 16 * cb * 2;  // bytes per K=16 slice
            const uint32_t half_off = (kHalf / cb) * slot;  // features 128.. of an operand
            const uint32_t idesc0 = idesc_f16(mma_fmt, kHalf, n0, 1, 1);
            const uint32_t idesc1 = idesc_f16(mma_fmt, kHalf, h1 ? n1 : 16, 1, 1);
            const uint32_t t0 = tmem_base, t1 = tmem_base + kTile + (diag ? kHalf : 0);
            if (lane == 0) {
                FPROF(long long t00 = clock64();)
                mbar_wait(&tempty[0], tph ^ 1);
                mbar_wait(&tempty[1], tph ^ 1);
                FPROF(pf_b += clock64() - t00;)
                tc_fence_after();
                int ub;
                const int rf = item_units(P.probs[it.p].mode, cb * P.probs[it.p].S, d, it.tj, diag, ub);
                FPROF(long long tloop = clock64();)
                for (int kc = it.k0; kc < it.k1;) {
                    const int units = min(rf, it.k1 - kc);
                    FPROF(long long t1c = clock64();)
                    mbar_wait(&full[stage], phase);
                    FPROF(pf_a += clock64() - t1c; pf_n++; t1c = clock64();
                          pf_i += (long long)units * ksteps * (n0 / 2 + (h1 ? n1 / 2 : 0));)
                    tc_fence_after();
                    const uint32_t sbase = smem_u32(ops + (size_t)stage * kStageBytes);
                    if (no_mma) {
                        mbar_arrive(&empty[stage]);
                    } else {
                        for (int u = 0; u < units; u++) {
                            const uint32_t b_base = diag ? sbase + u * ub : sbase + kOp;
                            const uint32_t a_base = diag ? b_base : sbase;
                            const uint32_t b1_base = diag ? b_base + half_off : b_base;
                            for (int k = 0; k < ksteps; k++) {
                                const uint32_t acc = (kc > it.k0 || u > 0 || k > 0) ? 1u : 0u;
                                mma_f16_ss(t0, umma_desc(a_base + k * kstep, lbo, sbo, lay),
                                           umma_desc(b_base + k * kstep, lbo, sbo, lay), idesc0, acc);
                                if (h1)
                                    mma_f16_ss(t1, umma_desc(a_base + half_off + k * kstep, lbo, sbo, lay),
                                               umma_desc(b1_base + k * kstep, lbo, sbo, lay), idesc1, acc);
                            }
                        }
                        mma_commit(&empty[stage]);
                    }
                    FPROF(pf_c += clock64() - t1c;)
                    kc += units;
                    if (++stage == kStages) {
                        stage = 0;
                        phase ^= 1;
                    }
                }
                FPROF(pf_e += clock64() - tloop; long long tz = clock64();)
                if (no_mma) mbar_arrive(tfull);
                else mma_commit(tfull);
                FPROF(pf_q += clock64() - tz;)
            }
            __syncwarp();
            tph ^= 1;
        }
    } else {
        // ============================ epilogue ============================
        // warp w drains tile rows h*128 + 32*(w%4) + lane of accumulator half h = w/4 (a warp may
        // only address its own 32-lane quarter of TMEM), 16 columns at a time: TMEM -> registers
        // -> per-warp staging -> 2 rows x 64 B coalesced stores.
        const int h = warp >> 2, quarter = warp & 3;
        float *stg = stage_buf + warp * 32 * kStageLd;
        const int rbase = h * kHalf + quarter * 32;  // tile row of lane 0
        uint32_t tph = 0;
        for (uint32_t s = 0;; s++) {
            const int item = next_item(s, P, qitem, qfull, qempty, false, lane);
            if (item >= total) break;
            const ItemInfo it = decode_item(hdr, nprobs, item);
            const ProbRegs pr = load_prob(P.probs[it.p]);
            FPROF(long long t0 = clock64();)
            mbar_wait(tfull, tph);
            FPROF(pf_a += clock64() - t0; pf_n++; t0 = clock64();)
            tc_fence_after();
            const bool diag = it.ti == it.tj;
            const int nr = min(kTile, pr.d - it.ti * kTile), nc = min(kTile, pr.d - it.tj * kTile);
            const uint32_t tacc = tmem_base + ((uint32_t)(quarter * 32) << 16) + h * kTile;
            float *part = pr.splits > 1
                              ? pr.partial + ((size_t)it.split * pr.npairs + it.tp) * (size_t)(kTile * kTile)
                              : nullptr;
            const int64_t dd = pr.d_out;
            const int gi0 = it.ti * kTile + rbase, gj0 = it.tj * kTile;
            const int sub = lane >> 2, cq = (lane & 3) * 4, half = lane >> 4, cc = lane & 15;
            bool released = false;
            if (rbase < nr) {
                // the TMEM load of group c0 + kQ is in flight while group c0 is stored
                const int cbeg = diag ? (rbase & ~(kQ - 1)) : 0;
                uint32_t r[16];
                tmem_ld_32x32b_x16(tacc + cbeg, r);
                const int d = pr.d;
                const float alpha = pr.alpha;
                for (int c0 = cbeg; c0 < nc; c0 += kQ) {
                    tmem_ld_wait();
                    tmem_regs_ready(r);
                    float4 *srow = reinterpret_cast<float4 *>(stg + lane * kStageLd);
#pragma unroll
                    for (int m = 0; m < 4; m++)
                        srow[m] = make_float4(__uint_as_float(r[4 * m]), __uint_as_float(r[4 * m + 1]),
                                              __uint_as_float(r[4 * m + 2]), __uint_as_float(r[4 * m + 3]));
                    if (c0 + kQ < nc) {
                        tmem_ld_32x32b_x16(tacc + c0 + kQ, r);
                    } else {
                        tc_fence_before();
                        mbar_arrive(&tempty[h]);  // accumulator quarter drained: the MMA may reuse it
                        released = true;
                    }
                    __syncwarp();
                    if (!no_store) {
                        // lane -> (row sub + 8 it, columns cq .. cq+3) of the staged 32 x 16 block
                        if (part) {
#if KFAC_EPI_V4
                            float *dst = part + (size_t)(rbase + sub) * kTile + c0 + cq;
#pragma unroll
                            for (int it = 0; it < 4; it++)
                                *reinterpret_cast<float4 *>(dst + (size_t)it * 8 * kTile) =
                                    *reinterpret_cast<const float4 *>(stg + (it * 8 + sub) * kStageLd + cq);
#else
                            float *dst = part + (size_t)rbase * kTile + c0 + cc;
#pragma unroll 4
                            for (int rr = half; rr < 32; rr += 2) dst[(size_t)rr * kTile] = stg[rr * kStageLd + cc];
#endif
                        } else {
                            // packed upper row-major: (gi, gj) at gi*dd - gi*(gi-1)/2 + (gj - gi); lanes
                            // 0-15 / 16-31 write 64 contiguous bytes of rows rr / rr + 1
                            const int gj = gj0 + c0 + cc;
#pragma unroll 4
                            for (int rr = half; rr < 32; rr += 2) {
                                const int gi = gi0 + rr;
                                if (gj >= gi && gj < d && gi < d)
                                    pr.out[(int64_t)gi * dd - ((int64_t)gi * (gi - 1) >> 1) - gi + gj] =
                                        alpha * stg[rr * kStageLd + cc];
                            }
                        }
                    }
                    __syncwarp();
                }
            }
            if (!released) {
                tc_fence_before();
                mbar_arrive(&tempty[h]);
            }
            FPROF(pf_b += clock64() - t0;)
            tph ^= 1;
        }
    }
#ifdef KFAC_FACTOR_PROF
    if ((blockIdx.x == 0 || blockIdx.x == 100) && lane == 0 && (warp == 0 || warp == kMmaWarp || warp == kProdWarp0))
        printf("[fprof] cta %d warp %d: total %lld  waitA %lld waitB %lld body %lld ideal %lld q %lld pre %lld n %d\n",
               blockIdx.x, warp, clock64() - pf_start, pf_a, pf_b, pf_c, pf_i, pf_q, pf_e, pf_n);
#endif
    tc_fence_before();
    __syncthreads();
    if (warp == kMmaWarp) {
        tc_fence_after();
        tmem_dealloc(tmem_base, kTmemCols);
    }
}

// ordered split-K fix-up: out = alpha * sum_{s=0..S-1} partial[s] (deterministic).
// One block per (tile pair, 8-row group); warp = row, lane = 8 columns; all S x 8 loads independent.
constexpr int kFixRowGroups = kTile / 8;
// the blockIdx.x-th item of a list over the problems, item counts cnt[p] loaded in parallel into
// shared memory (a serial walk over the kernel-parameter array costs a constant-cache miss per problem)
__device__ __forceinline__ int locate(int *cnt, int nprobs, int &b) {
    __shared__ int res[2];
    __syncthreads();
    if (threadIdx.x == 0) {
        int p = 0;
        for (; p < nprobs; p++) {
            if (b < cnt[p]) break;
            b -= cnt[p];
        }
        res[0] = p;
        res[1] = b;
    }
    __syncthreads();
    b = res[1];
    return res[0];
}
__global__ void __launch_bounds__(256) factor_fixup_kernel(const __grid_constant__ FactorParams P) {
    __shared__ int cnt[kMaxProbs];
    for (int q = threadIdx.x; q < P.nprobs; q += blockDim.x) cnt[q] = P.probs[q].splits > 1 ? P.probs[q].npairs : 0;
    int b = blockIdx.x / kFixRowGroups;
    const int rg = blockIdx.x % kFixRowGroups;
    const int p = locate(cnt, P.nprobs, b);
    if (p >= P.nprobs) return;
    const FactorProb &pr = P.probs[p];
    int ti, tj;
    decode_pair(b, pr.nt, ti, tj);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int r = rg * 8 + warp;
    const int gi = ti * kTile + r, gj0 = tj * kTile;
    if (gi >= pr.d) return;
    const int jlo = max(0, gi - gj0), jhi = min(kTile, pr.d - gj0);
    if (jlo >= jhi) return;
    const size_t tile = (size_t)kTile * kTile, sstride = (size_t)pr.npairs * tile;
    const float *src = pr.partial + (size_t)b * tile + (size_t)r * kTile + lane;
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

// materialise the im2col rows of problems with im2col_pre: col[q][f] = ã_f(q), zero for f >= d.
// One warp per output pixel; lane k assembles features [8k, 8k+8) (feature f = (i*kw + j)*C + c,
// walked incrementally) and writes them as one 16-byte vector, so a warp writes its pixel's
// cp-element row contiguously.  32-bit index math only (rows < 2^31).
__global__ void __launch_bounds__(256) im2col_kernel(const __grid_constant__ FactorParams P) {
    __shared__ int cnt[kMaxProbs];  // blockIdx.y-th problem with materialised patches
    for (int q = threadIdx.x; q < P.nprobs; q += blockDim.x) cnt[q] = P.probs[q].im2col_pre ? 1 : 0;
    int b = blockIdx.y;
    const int p = locate(cnt, P.nprobs, b);
    if (p >= P.nprobs) return;
    const FactorProb &g = P.probs[p];
    const int C = g.c, kw = g.kw, nq = g.cp / 8, hw = g.ho * g.wo, d = g.d;
    const int lane = threadIdx.x & 31, wpb = blockDim.x >> 5;
    const int rows = (int)g.rows;
    // lane q's 8 features are the same for every pixel: decode them once
    // (tap row i, tap column j, offset (i*W + j)*C + c from the window corner; i = -1: zero)
    int ti[8], tj[8], toff[8];
    {
        const int f = lane * 8;
        int kk = f / C, c = f - kk * C;
        int i = kk / kw, j = kk - i * kw;
#pragma unroll
        for (int e = 0; e < 8; e++) {
            const bool ok = lane < nq && f + e < d;
            ti[e] = ok ? i : -1;
            tj[e] = j;
            toff[e] = (i * g.w + j) * C + c;
            if (++c == C) {
                c = 0;
                if (++j == kw) {
                    j = 0;
                    ++i;
                }
            }
        }
    }
    for (int row = blockIdx.x * wpb + (threadIdx.x >> 5); row < rows; row += gridDim.x * wpb) {
        const int n = row / hw;
        const int rem = row - n * hw;
        const int oh = rem / g.wo, ow = rem - oh * g.wo;
        const int h0 = oh * g.sh - g.ph, w0 = ow * g.sw - g.pw;
        const uint16_t *corner = g.src + ((int64_t)n * g.h * g.w + (int64_t)h0 * g.w + w0) * C;
        const bool inside = h0 >= 0 && h0 + g.kh <= g.h && w0 >= 0 && w0 + kw <= g.w;
        uint32_t pk[4] = {0u, 0u, 0u, 0u};
        if (inside) {  // warp-uniform: the whole window is inside the image
#pragma unroll
            for (int e = 0; e < 8; e++)
                if (ti[e] >= 0) pk[e >> 1] |= (uint32_t)__ldg(corner + toff[e]) << ((e & 1) * 16);
        } else {
#pragma unroll
            for (int e = 0; e < 8; e++) {
                const int h = h0 + ti[e], w = w0 + tj[e];
                if (ti[e] >= 0 && h >= 0 && h < g.h && w >= 0 && w < g.w)
                    pk[e >> 1] |= (uint32_t)__ldg(corner + toff[e]) << ((e & 1) * 16);
            }
        }
        if (lane < nq)
            reinterpret_cast<uint4 *>(g.col + (int64_t)row * g.cp)[lane] = make_uint4(pk[0], pk[1], pk[2], pk[3]);
    }
}

// bias row/column of A: A[f][dA-1] = alpha * sum_rows ã_f, A[dA-1][dA-1] = alpha * rows
// (the homogeneous coordinate, reading R-5).  Block = 32 features x 8 row-strided warps, fp64
// partial sums combined in a fixed order (deterministic).
__global__ void __launch_bounds__(256) factor_bias_kernel(const __grid_constant__ FactorParams P) {
    __shared__ int cnt[kMaxProbs];  // blockIdx.y-th problem with a bias coordinate
    __shared__ double part[8][33];
    for (int q = threadIdx.x; q < P.nprobs; q += blockDim.x) cnt[q] = P.probs[q].d_out != P.probs[q].d ? 1 : 0;
    int b = blockIdx.y;
    const int p = locate(cnt, P.nprobs, b);
    if (p >= P.nprobs) return;
    const ProbRegs pr = load_prob(P.probs[p]);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int f = blockIdx.x * 32 + lane;
    if (blockIdx.x * 32 > pr.d) return;
    const int dA = pr.d_out, rows = (int)pr.rows;
    double s = 0.0;
    if (f < pr.d)
        for (int q = warp; q < rows; q += 8) s += (double)gather_elem(pr, P.ab_fmt, q, f);
    part[warp][lane] = s;
    __syncthreads();
    if (warp == 0 && f <= pr.d) {
        double t = 0.0;
        for (int w = 0; w < 8; w++) t += part[w][lane];
        if (f == pr.d) t = (double)pr.rows;
        const int64_t off = (int64_t)f * dA - (int64_t)f * (f - 1) / 2 + (dA - 1 - f);
        pr.out[off] = (float)(pr.alpha * t);
    }
}

// ---------------------------------------------------------------- host side
typedef CUresult (*PFN_encodeTiled)(CUtensorMap *, CUtensorMapDataType, cuuint32_t, void *, const cuuint64_t *,
                                    const cuuint64_t *, const cuuint32_t *, const cuuint32_t *, CUtensorMapInterleave,
                                    CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);


static PFN_encodeTiled g_encTiled = nullptr;
static int g_driver = 0;

static std::mutex g_drv_mu;

static kfac_status load_driver_fns() {
    std::lock_guard<std::mutex> lock(g_drv_mu);
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

static int pow2ceil(int x) {
    int p = 1;
    while (p < x) p <<= 1;
    return p;
}

// right edge (exclusive) of the input columns filter column j may touch: output columns >= wo
// (the box's phantom columns) land at or beyond it and are zero-filled by TMA
static int tap_width(const FactorProb *pr, int j) {
    return std::min<int>(pr->w, (pr->wo - 1) * pr->sw - pr->pw + j + 1);
}

// Geometry of one factor problem (no pointers): the mode the kernel will use, the chunking of
// K, the tile grid, the descriptors it needs.  Shared by plan-time sizing and launch-time setup.
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
    pr->nt = (int16_t)((pr->d + kTile - 1) / kTile);
    pr->npairs = pr->nt * (pr->nt + 1) / 2;
    const int C = pr->c;
    const bool plain = (pr->kh == 1 && pr->kw == 1 && pr->sh == 1 && pr->sw == 1 && pr->ph == 0 && pr->pw == 0);
    const bool aligned16 = (C % 8) == 0 && src_aligned;
    int mode = MODE_GATHER, cb = 64;
    pr->wp = (int16_t)pow2ceil(pr->wo);
    pr->bh = pr->bn = 1;
    if (!force_gather() && aligned16) {
        if (plain) {
            mode = MODE_TILED2D;
            cb = C >= 64 ? 64 : (C > 16 ? (C > 32 ? 64 : 32) : 16);
            if (C > cb && C % cb) cb = (C % 32 == 0) ? 32 : 16;  // slots must tile the channels
            if (C > cb && C % cb) mode = MODE_GATHER, cb = 64;
        } else if (C % 16 == 0 && pr->wo <= kBK && pr->kw <= 8 && pr->sw <= 8 && pr->sh <= 8 &&
                   (pr->wp - 1) * pr->sw + 1 <= 256) {
            mode = MODE_TILED4D;
            cb = (C % 64 == 0) ? 64 : ((C % 32 == 0) ? 32 : 16);
            for (int jj = 0; jj < pr->kw; jj++)
                if (tap_width(pr, jj) < 1) mode = MODE_GATHER, cb = 64;  // a column of pure padding
        }
    }
    pr->im2col_pre = 0;
    pr->cp = 0;
    int Ceff = C;
    if (mode == MODE_GATHER && !force_gather() && j.is_A && !plain && src_aligned && (pr->d + 63) / 64 * 64 <= 256) {
        // channel stride not a multiple of 16 B (e.g. the RGB stem): TMA cannot address the
        // pixels, so the patches are materialised once as [rows, cp] (cp = dF rounded to 64)
        // and staged by the 2-D TMA path
        pr->im2col_pre = 1;
        pr->cp = (int16_t)((pr->d + 63) / 64 * 64);
        mode = MODE_TILED2D;
        cb = 64;
        Ceff = pr->cp;
    }
    pr->mode = (int8_t)mode;
    pr->cb = (int16_t)cb;
    // channel slots per box: consecutive slots of one tap (the box never straddles a tap)
    int S = 1;
    if (mode != MODE_GATHER)
        while (cb * S * 2 <= kTile && Ceff % (cb * S * 2) == 0) S *= 2;
    pr->S = (int16_t)S;
    pr->ksteps = kBK / 16;
    pr->nmaps = 0;
    pr->mapj = 0;
    if (mode == MODE_TILED4D) {
        // 64-row chunks: wp (pow2 >= wo) columns x bh rows (pow2 dividing ho) x bn images
        int bh = 1;
        while (pr->wp * bh * 2 <= kBK && pr->ho % (bh * 2) == 0) bh *= 2;
        pr->bh = (int16_t)bh;
        pr->bn = (int16_t)(kBK / (pr->wp * bh));
        pr->rpi = (int16_t)(pr->ho / bh);
        pr->kchunks = (int)((j.n + pr->bn - 1) / pr->bn) * pr->rpi;
        // one descriptor per distinct right edge
        int widths[8], nw = 0;
        for (int jj = 0; jj < pr->kw; jj++) {
            const int wj = tap_width(pr, jj);
            int m = 0;
            while (m < nw && widths[m] != wj) m++;
            if (m == nw) widths[nw++] = wj;
            pr->mapj |= (uint64_t)m << (8 * jj);
        }
        pr->nmaps = (int8_t)nw;
    } else {
        pr->rpi = 1;
        pr->kchunks = (int)((pr->rows + kBK - 1) / kBK);
        if (pr->kchunks == 1) pr->ksteps = (int16_t)((pr->rows + 15) / 16);  // e.g. FC at small batch
        pr->nmaps = mode == MODE_TILED2D ? 1 : 0;
    }
}

// pointers + TMA descriptors of one factor problem (written to maps[0 .. nmaps))
static kfac_status setup_prob(const FactorJob &j, kfac_dtype dt, FactorProb *pr, CUtensorMap *maps) {
    pr->src = static_cast<const uint16_t *>(j.src);
    pr->out = j.out;
    pr->alpha = j.alpha;
    if (pr->mode == MODE_GATHER) return KFAC_OK;
    kfac_status s = load_driver_fns();
    if (s) return s;
    const int cb = pr->cb, S = pr->S;
    const CUtensorMapDataType dty = dt == KFAC_FP16 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT16 : CU_TENSOR_MAP_DATA_TYPE_BFLOAT16;
    const int64_t N = pr->rows / ((int64_t)pr->ho * pr->wo);
    const int64_t bytes = N * pr->h * pr->w * (int64_t)pr->c * 2;
    CUresult r = CUDA_SUCCESS;
    if (pr->mode == MODE_TILED2D) {
        // {cb channels, rows, slot} over the [rows, C] matrix
        const int64_t W = pr->im2col_pre ? pr->cp : pr->c;
        void *base = pr->im2col_pre ? (void *)pr->col : const_cast<void *>(j.src);
        const bool one = W < cb;  // fewer channels than a slot: zero-filled to cb
        cuuint64_t dims[3] = {(cuuint64_t)(one ? W : cb), (cuuint64_t)pr->rows, (cuuint64_t)(one ? 1 : W / cb)};
        cuuint64_t strides[2] = {(cuuint64_t)W * 2, (cuuint64_t)(one ? W * 2 : cb * 2)};
        cuuint32_t box[3] = {(cuuint32_t)cb, (cuuint32_t)kBK, (cuuint32_t)S};
        cuuint32_t es[3] = {1, 1, 1};
        r = g_encTiled(&maps[0], dty, 3, base, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, swz_of(cb),
                       CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        small_tensor_fix(&maps[0], pr->im2col_pre ? pr->rows * W * 2 : bytes);
    } else {
        // {cb channels, W, H, N, slot}: the filter tap shifts the start coordinate, the conv
        // stride is the traversal stride, padding and phantom columns are the out-of-bounds fill
        const int C = pr->c;
        for (int m = 0; m < pr->nmaps && r == CUDA_SUCCESS; m++) {
            int wj = -1;
            for (int jj = 0; jj < pr->kw; jj++)
                if ((int)((pr->mapj >> (8 * jj)) & 0xff) == m) wj = tap_width(pr, jj);
            cuuint64_t dims[5] = {(cuuint64_t)cb, (cuuint64_t)wj, (cuuint64_t)pr->h, (cuuint64_t)N, (cuuint64_t)(C / cb)};
            cuuint64_t strides[4] = {(cuuint64_t)C * 2, (cuuint64_t)C * 2 * pr->w, (cuuint64_t)C * 2 * pr->w * pr->h,
                                     (cuuint64_t)cb * 2};
            cuuint32_t box[5] = {(cuuint32_t)cb, (cuuint32_t)((pr->wp - 1) * pr->sw + 1),
                                 (cuuint32_t)((pr->bh - 1) * pr->sh + 1), (cuuint32_t)pr->bn, (cuuint32_t)S};
            cuuint32_t es[5] = {1, (cuuint32_t)pr->sw, (cuuint32_t)pr->sh, 1, 1};
            r = g_encTiled(&maps[m], dty, 5, const_cast<void *>(j.src), dims, strides, box, es,
                           CU_TENSOR_MAP_INTERLEAVE_NONE, swz_of(cb), CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                           CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
            small_tensor_fix(&maps[m], bytes);
        }
    }
    if (r != CUDA_SUCCESS) {
        char buf[200];
        snprintf(buf, sizeof buf, "cuTensorMapEncodeTiled failed (%d) for C=%d mode=%d wo=%d bh=%d bn=%d S=%d", (int)r,
                 pr->c, pr->mode, pr->wo, pr->bh, pr->bn, S);
        return set_error(KFAC_ERR_UNSUPPORTED, buf);
    }
    return KFAC_OK;
}

kfac_status factor_prepare(const std::vector<FactorJob> &jobs, kfac_dtype dt, void *ws, int64_t ws_cap,
                           bool dry_run, FactorLaunch *out) {
    out->params.clear();
    out->ws_bytes = 0;
    if (jobs.empty()) return KFAC_OK;
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
        if (S > 1) need += (int64_t)g.npairs * S * kTile * kTile * 4;
    }
    int64_t col_need = 0;
    for (int i = 0; i < nj; i++)
        if (geo[i].im2col_pre) col_need += (geo[i].rows * geo[i].cp * 2 + 255) / 256 * 256;
    if (!dry_run && need + col_need > ws_cap) {  // not enough scratch (e.g. a fallback mode changed the chunking)
        for (int i = 0; i < nj; i++) splits[i] = 1, item_cost[i] = (double)geo[i].kchunks * geo[i].ksteps;
        need = 0;
    }
    if (!dry_run && col_need > ws_cap) return set_error(KFAC_ERR_ARG, "factor workspace too small for im2col staging");
    // the work-item counter lives after the partials and im2col staging (static striding without it)
    int32_t *counter = nullptr;
    if (ws && ws_cap >= need + col_need + 256)
        counter = reinterpret_cast<int32_t *>(static_cast<uint8_t *>(ws) + need + col_need);
    // heaviest items first
    std::vector<int> order(nj);
    for (int i = 0; i < nj; i++) order[i] = i;
    std::stable_sort(order.begin(), order.end(), [&](int a, int b) { return item_cost[a] > item_cost[b]; });
    int64_t ws_off = 0, col_off = 0;
#ifdef KFAC_DEBUG_KNOBS  // development switches (disable MMA / TMA / stores): never in a product build
    const int dbg = getenv("KFAC_DBG_MODE") ? atoi(getenv("KFAC_DBG_MODE")) : 0;
#else
    const int dbg = 0;
#endif
    for (int base = 0; base < nj;) {
        out->params.emplace_back();
        FactorParams &P = out->params.back();
        memset(&P, 0, sizeof(P));
        P.ab_fmt = (int)dt;
        P.dbg = dbg;
        P.counter = counter;
        int items = 0, cnt = 0, nmaps = 0;
        while (base + cnt < nj && cnt < kMaxProbs && nmaps + geo[order[base + cnt]].nmaps <= kMaxMaps) {
            const int i = order[base + cnt];
            FactorProb &pr = P.probs[cnt];
            pr = geo[i];
            pr.map0 = (int16_t)nmaps;
            if (pr.im2col_pre) {
                pr.col = ws ? reinterpret_cast<uint16_t *>(static_cast<uint8_t *>(ws) + need + col_off) : nullptr;
                col_off += (pr.rows * pr.cp * 2 + 255) / 256 * 256;
            }
            if (!dry_run) {
                kfac_status s = setup_prob(jobs[i], dt, &pr, &P.maps[nmaps]);
                if (s) return s;
            }
            nmaps += pr.nmaps;
            const int S = splits[i];
            pr.chunks_per_split = (pr.kchunks + S - 1) / S;
            pr.splits = S;
            pr.item_begin = items;
            items += pr.npairs * S;
            if (S > 1) {
                pr.partial = ws ? reinterpret_cast<float *>(static_cast<uint8_t *>(ws) + ws_off) : nullptr;
                ws_off += (int64_t)pr.npairs * S * kTile * kTile * 4;
            }
            cnt++;
        }
        P.nprobs = cnt;
        P.nmaps = nmaps;
        P.total_items = items;
#ifdef KFAC_DEBUG_KNOBS
        if (!dry_run && getenv("KFAC_DEBUG")) {
            for (int k = 0; k < cnt; k++) {
                const FactorProb &pr = P.probs[k];
                fprintf(stderr,
                        "[kfac] factor prob %d: d=%d rows=%lld mode=%d cb=%d S=%d ksteps=%d wp=%d bh=%d bn=%d pairs=%d "
                        "kchunks=%d splits=%d maps=%d\n",
                        k, pr.d, (long long)pr.rows, pr.mode, pr.cb, pr.S, pr.ksteps, pr.wp, pr.bh, pr.bn, pr.npairs,
                        pr.kchunks, pr.splits, pr.nmaps);
            }
            fprintf(stderr, "[kfac] factor launch: %d problems, %d descriptors, %d items, target %.0f k-steps/item\n",
                    P.nprobs, P.nmaps, items, target);
        }
#endif
        base += cnt;
    }
    out->ws_bytes = need + col_need + 256;
    return KFAC_OK;
}

kfac_status factor_launch(const FactorLaunch &fl, const std::vector<FactorJob> &jobs, cudaStream_t st) {
    int sms = 0;
    KFAC_TRY(dev_sm_count(&sms));
    KFAC_TRY(dev_func_smem((const void *)factor_syrk_kernel, (int)kSmemBytes));
    for (const FactorParams &P : fl.params) {
        if (P.total_items == 0) continue;
        int npre = 0;
        for (int p = 0; p < P.nprobs; p++) npre += P.probs[p].im2col_pre != 0;
        if (npre) {
            im2col_kernel<<<dim3(8 * sms, npre), 256, 0, st>>>(P);
            KFAC_LAUNCHED();
            KFAC_CUDA_TRY(cudaGetLastError());
        }
        int grid = std::min(P.total_items, sms);
        if (P.counter) KFAC_CUDA_TRY(cudaMemsetAsync(P.counter, 0, sizeof(int32_t), st));
        factor_syrk_kernel<<<grid, kThreads, kSmemBytes, st>>>(P);
        KFAC_LAUNCHED();
        KFAC_CUDA_TRY(cudaGetLastError());
        int fix = 0, maxbias = 0, nbias = 0;
        for (int p = 0; p < P.nprobs; p++) {
            const FactorProb &pr = P.probs[p];
            if (pr.splits > 1) fix += pr.npairs;
            if (pr.d_out != pr.d) maxbias = std::max(maxbias, pr.d + 1), nbias++;
        }
#ifdef KFAC_DEBUG_KNOBS
        if (getenv("KFAC_NO_FIXUP")) fix = 0;
#endif
        if (fix) {
            factor_fixup_kernel<<<fix * kFixRowGroups, 256, 0, st>>>(P);
            KFAC_LAUNCHED();
            KFAC_CUDA_TRY(cudaGetLastError());
        }
        if (maxbias) {
            dim3 g((maxbias + 31) / 32, nbias);
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
