// precond.cu -- stage 5 of distributed K-FAC (PAPER.md P:264-282 Eqs. K-FAC
// update): the preconditioned gradient of every owned layer
//     𝒢 = G_d^-1 * dW * A_d^-1        (row-major vec, reading R-14)
// as two grouped tcgen05 GEMM launches over all owned layers, both with
// K-major operands only (the inverses are symmetric):
//     T^T = A_d^-1 * dW^T      (A-op A_d^-1 [dA x dA], B-op dW [dG x dA])
//     𝒢   = G_d^-1 * T         (A-op G_d^-1 [dG x dG], B-op T^T [dA x dG])
// Precision: single-pass TF32 / bf16 miss the 2e-3 bound on
// activation-consistent gradients, so every product is a 3xTF32 split
//     a*b ~ hi(a)hi(b) + hi(a)lo(b) + lo(a)hi(b),  hi = rn_tf32(x), lo = rn_tf32(x - hi)
// on tcgen05.mma kind::tf32 with fp32 accumulation in TMEM (fp32-class error).  The tensor
// core's fp32 accumulation does not round to nearest, and over K = 4608 its error grows well
// past an fp32 GEMM's, so TMEM holds only 256-element K segments that the epilogue sums in
// registers with round-to-nearest adds.
// The operands are staged as [2][rows][K] (hi, lo) by a split kernel (the
// first GEMM's epilogue writes T^T already split); TMA loads 32-element K
// boxes (SW128, K-major) of hi and lo for both operands.
#include <algorithm>
#include <cstring>

#include "kfac_internal.hpp"
#include "sm100.cuh"

namespace kfac {

constexpr int GM = 128, GN = 128, GK = 32;  // tile M, N; K elements per stage (128 B rows)
constexpr int GStages = 3;
constexpr int GSeg = 8;                     // K chunks (256 elements) per TMEM accumulation segment
constexpr int GThreads = 192;               // warps 0-3 epilogue, 4 MMA, 5 TMA
constexpr int kMaxG = 96;
constexpr int GOp = GM * GK * 4;            // 16 KB per operand half per stage
constexpr int GStageBytes = 4 * GOp;        // A hi, A lo, B hi, B lo
constexpr int GLd = 33;                     // epilogue staging stride
constexpr size_t GSmem = 1024 + (size_t)GStages * GStageBytes + (size_t)GM * GLd * 4 + 256;

struct alignas(64) GemmProb {
    CUtensorMap tA;        // [2][M][Kp] fp32 (hi, lo)
    CUtensorMap tB;        // [2][N][Kp] fp32
    float *C;              // output, row-major ldc
    float *Clo;            // if non-null: write split output: C = hi copy, Clo = lo part
    int32_t M, N, K, ldc, tiles_n, item_begin, pad0, pad1;
};
struct GemmParams {
    int32_t np, total, dbg, pad;
    GemmProb p[kMaxG];
};

// round to the nearest tf32 value (ties away from zero); the result is exact in tf32, so the
// MMA's own operand truncation leaves it unchanged
__device__ __forceinline__ float tf32_rn(float x) {
    return __uint_as_float((__float_as_uint(x) + 0x1000u) & 0xFFFFE000u);
}

__device__ __forceinline__ void mma_tf32_ss(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                            uint32_t accumulate) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
        "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
        : "memory");
}

// idesc kind::tf32: D fp32 (1), A/B TF32 (2), both K-major
constexpr uint32_t kIdescTF32 = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(GN >> 3) << 17) | ((uint32_t)(GM >> 4) << 24);

__device__ __forceinline__ void gdecode(const GemmParams &P, int item, int &pi, int &m0, int &n0) {
    int p = 0;
    while (p + 1 < P.np && P.p[p + 1].item_begin <= item) p++;
    const int local = item - P.p[p].item_begin;
    pi = p;
    m0 = (local / P.p[p].tiles_n) * GM;
    n0 = (local % P.p[p].tiles_n) * GN;
}

__global__ void __launch_bounds__(GThreads, 1) gemm_3xtf32_kernel(const __grid_constant__ GemmParams P) {
    extern __shared__ uint8_t smem_raw[];
    uint8_t *smem = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    float *stage_buf = reinterpret_cast<float *>(smem + (size_t)GStages * GStageBytes);
    uint64_t *bars = reinterpret_cast<uint64_t *>(smem + (size_t)GStages * GStageBytes + (size_t)GM * GLd * 4);
    uint64_t *full = bars, *empty = bars + GStages, *tfull = bars + 2 * GStages, *tempty = bars + 2 * GStages + 2;
    uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(bars + 2 * GStages + 4);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (threadIdx.x == 0) {
        for (int s = 0; s < GStages; s++) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], 1);
        }
        for (int b = 0; b < 2; b++) {
            mbar_init(&tfull[b], 1);
            mbar_init(&tempty[b], 128);
        }
        fence_barrier_init();
    }
    if (warp == 4) tmem_alloc(tmem_slot, 2 * GN);
    if (warp == 5)
        for (int p = lane; p < P.np; p += 32) {
            tma_prefetch(&P.p[p].tA);
            tma_prefetch(&P.p[p].tB);
        }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;
    const int total = P.total;

    if (warp == 5) {
        if (lane == 0) {  // TMA producer
            uint32_t stage = 0, phase = 0;
            for (int item = blockIdx.x; item < total; item += gridDim.x) {
                int pi, m0, n0;
                gdecode(P, item, pi, m0, n0);
                const GemmProb &g = P.p[pi];
                const int kch = (g.K + GK - 1) / GK;
                for (int kc = 0; kc < kch; kc++) {
                    mbar_wait(&empty[stage], phase ^ 1);
                    uint8_t *s = smem + (size_t)stage * GStageBytes;
                    mbar_arrive_expect_tx(&full[stage], GStageBytes);
                    tma_load_3d(s, &g.tA, &full[stage], kc * GK, m0, 0);
                    tma_load_3d(s + GOp, &g.tA, &full[stage], kc * GK, m0, 1);
                    tma_load_3d(s + 2 * GOp, &g.tB, &full[stage], kc * GK, n0, 0);
                    tma_load_3d(s + 3 * GOp, &g.tB, &full[stage], kc * GK, n0, 1);
                    if (++stage == GStages) {
                        stage = 0;
                        phase ^= 1;
                    }
                }
            }
        }
    } else if (warp == 4) {
        // K is accumulated in TMEM segments of GSeg chunks; the epilogue adds each segment into
        // fp32 registers (round to nearest) while the MMAs of the next one run in the other buffer
        uint32_t stage = 0, phase = 0, tph = 0;
        int buf = 0;
        for (int item = blockIdx.x; item < total; item += gridDim.x) {
            int pi, m0, n0;
            gdecode(P, item, pi, m0, n0);
            const int kch = (P.p[pi].K + GK - 1) / GK;
            for (int k0 = 0; k0 < kch; k0 += GSeg) {
                const uint32_t tacc = tmem_base + buf * GN;
                if (lane == 0) {
                    mbar_wait(&tempty[buf], ((tph >> buf) & 1) ^ 1);
                    tc_fence_after();
                    for (int kc = k0; kc < kch && kc < k0 + GSeg; kc++) {
                        mbar_wait(&full[stage], phase);
                        tc_fence_after();
                        const uint32_t s = smem_u32(smem + (size_t)stage * GStageBytes);
                        const uint32_t ah = s, al = s + GOp, bh = s + 2 * GOp, bl = s + 3 * GOp;
#pragma unroll
                        for (int k = 0; k < GK / 8; k++) {  // K = 8 tf32 per MMA = 32 bytes within the SW128 atom
                            const uint32_t ko = k * 32;
                            const uint64_t dah = umma_desc(ah + ko, 16, 1024, UMMA_SW128);
                            const uint64_t dal = umma_desc(al + ko, 16, 1024, UMMA_SW128);
                            const uint64_t dbh = umma_desc(bh + ko, 16, 1024, UMMA_SW128);
                            const uint64_t dbl = umma_desc(bl + ko, 16, 1024, UMMA_SW128);
                            const uint32_t acc0 = (kc > k0 || k > 0) ? 1u : 0u;
                            mma_tf32_ss(tacc, dal, dbh, kIdescTF32, acc0);  // small terms first
                            mma_tf32_ss(tacc, dah, dbl, kIdescTF32, 1u);
                            mma_tf32_ss(tacc, dah, dbh, kIdescTF32, 1u);
                        }
                        mma_commit(&empty[stage]);
                        if (++stage == GStages) {
                            stage = 0;
                            phase ^= 1;
                        }
                    }
                    mma_commit(&tfull[buf]);
                }
                __syncwarp();
                tph ^= 1u << buf;
                buf ^= 1;
            }
        }
    } else {  // epilogue warps 0-3: thread = one output row, 128 fp32 register accumulators
        uint32_t tph = 0;
        int buf = 0;
        const int row = warp * 32 + lane;
        for (int item = blockIdx.x; item < total; item += gridDim.x) {
            int pi, m0, n0;
            gdecode(P, item, pi, m0, n0);
            const GemmProb &g = P.p[pi];
            float *C = g.C, *Clo = g.Clo;
            const int M = g.M, N = g.N, ldc = g.ldc;
            const int kch = (g.K + GK - 1) / GK;
            float acc[GN];
#pragma unroll
            for (int i = 0; i < GN; i++) acc[i] = 0.f;
            for (int k0 = 0; k0 < kch; k0 += GSeg) {
                mbar_wait(&tfull[buf], (tph >> buf) & 1);
                tc_fence_after();
                const uint32_t tacc = tmem_base + buf * GN + ((uint32_t)(warp * 32) << 16);
#pragma unroll
                for (int q = 0; q < GN / 32; q++) {
                    uint32_t r[32];
                    tmem_ld_32x32b_x32(tacc + q * 32, r);
                    tmem_ld_wait();
                    tmem_regs_ready(r);
#pragma unroll
                    for (int i = 0; i < 32; i++) acc[q * 32 + i] += __uint_as_float(r[i]);
                }
                tc_fence_before();
                mbar_arrive(&tempty[buf]);
                tph ^= 1u << buf;
                buf ^= 1;
            }
#pragma unroll
            for (int q = 0; q < GN / 32; q++) {
#pragma unroll
                for (int i = 0; i < 32; i++) stage_buf[row * GLd + i] = acc[q * 32 + i];
                named_bar_sync(2, 128);
                const int j = n0 + q * 32 + lane;
                for (int rr = warp; rr < GM; rr += 4) {
                    const int i = m0 + rr;
                    if (i >= M) break;
                    if (j < N) {
                        const float v = stage_buf[rr * GLd + lane];
                        if (Clo) {  // split output for the next product: hi = tf32(v), lo = tf32(v - hi)
                            const float hi = tf32_rn(v);
                            C[(int64_t)i * ldc + j] = hi;
                            Clo[(int64_t)i * ldc + j] = tf32_rn(v - hi);
                        } else {
                            C[(int64_t)i * ldc + j] = v;
                        }
                    } else if (Clo && j < ldc) {  // zero the K padding the next product reads
                        C[(int64_t)i * ldc + j] = 0.f;
                        Clo[(int64_t)i * ldc + j] = 0.f;
                    }
                }
                named_bar_sync(2, 128);
            }
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 4) {
        tc_fence_after();
        tmem_dealloc(tmem_base, 2 * GN);
    }
}

// split fp32 rows [rows][K] (row stride ld_src) into [2][rows][Kp]: hi = tf32(x), lo = tf32(x - hi)
struct SplitJob {
    const float *src;
    float *dst;
    int32_t rows, K, ld_src, Kp;
};
struct SplitParams {
    int32_t n, pad;
    SplitJob j[kMaxG];
};
__global__ void __launch_bounds__(256) split_kernel(const __grid_constant__ SplitParams P) {
    const SplitJob &J = P.j[blockIdx.y];
    const int64_t tot = (int64_t)J.rows * J.Kp;
    const int kq = J.Kp / 4;  // Kp is a multiple of 4: 16-byte hi / lo stores
    // one row per (block, warp-group) step: coalesced loads of the (unaligned) source row
    for (int r = blockIdx.x; r < J.rows; r += gridDim.x) {
        const float *src = J.src + (int64_t)r * J.ld_src;
        float4 *hi = reinterpret_cast<float4 *>(J.dst + (int64_t)r * J.Kp);
        float4 *lo = reinterpret_cast<float4 *>(J.dst + tot + (int64_t)r * J.Kp);
        for (int q = threadIdx.x; q < kq; q += blockDim.x) {
            float x[4], h[4], l[4];
#pragma unroll
            for (int e = 0; e < 4; e++) {
                const int k = 4 * q + e;
                x[e] = k < J.K ? __ldg(src + k) : 0.f;
                h[e] = tf32_rn(x[e]);
                l[e] = tf32_rn(x[e] - h[e]);  // |x - h - l| <= 2^-22 |x|
            }
            hi[q] = make_float4(h[0], h[1], h[2], h[3]);
            lo[q] = make_float4(l[0], l[1], l[2], l[3]);
        }
    }
}

// ---------------------------------------------------------------- host side
typedef CUresult (*PFN_encTiled)(CUtensorMap *, CUtensorMapDataType, cuuint32_t, void *, const cuuint64_t *,
                                 const cuuint64_t *, const cuuint32_t *, const cuuint32_t *, CUtensorMapInterleave,
                                 CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
static PFN_encTiled g_enc = nullptr;

static kfac_status split_map(CUtensorMap *m, float *base, int rows, int Kp) {
    if (!g_enc) {
        cudaDriverEntryPointQueryResult q;
        void *f = nullptr;
        KFAC_CUDA_TRY(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q));
        if (!f) return set_error(KFAC_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
        g_enc = (PFN_encTiled)f;
    }
    cuuint64_t dims[3] = {(cuuint64_t)Kp, (cuuint64_t)rows, 2};
    cuuint64_t strides[2] = {(cuuint64_t)Kp * 4, (cuuint64_t)Kp * 4 * rows};
    cuuint32_t box[3] = {GK, GM, 1};
    cuuint32_t es[3] = {1, 1, 1};
    CUresult r = g_enc(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, base, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                       CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) return set_error(KFAC_ERR_UNSUPPORTED, "cuTensorMapEncodeTiled (split operand) failed");
    return KFAC_OK;
}

static int64_t kpad(int k) { return (k + 3) / 4 * 4; }

int64_t precond_split_floats(int n) { return 2 * (int64_t)n * kpad(n); }

int64_t precond_ws_floats(int dG, int dA) {
    // A_d^-1 split, G_d^-1 split, dW split, T^T split (all [2][rows][Kp]) + output staging
    return 2 * ((int64_t)dA * kpad(dA) + (int64_t)dG * kpad(dG) + (int64_t)dG * kpad(dA) + (int64_t)dA * kpad(dG)) + 64;
}

static kfac_status launch_splits(const std::vector<SplitJob> &js, cudaStream_t st) {
    for (size_t b = 0; b < js.size(); b += kMaxG) {
        SplitParams P;
        memset(&P, 0, sizeof(P));
        P.n = (int)std::min<size_t>(kMaxG, js.size() - b);
        for (int i = 0; i < P.n; i++) P.j[i] = js[b + i];
        int maxrows = 1;
        for (int i = 0; i < P.n; i++) maxrows = std::max(maxrows, (int)P.j[i].rows);
        split_kernel<<<dim3(std::min(maxrows, 1024), P.n), 256, 0, st>>>(P);
        KFAC_LAUNCHED();
        KFAC_CUDA_TRY(cudaGetLastError());
    }
    return KFAC_OK;
}

static kfac_status launch_gemms(std::vector<GemmProb> &gs, cudaStream_t st) {
    int sms = 0;
    KFAC_TRY(dev_sm_count(&sms));
    KFAC_TRY(dev_func_smem((const void *)gemm_3xtf32_kernel, (int)GSmem));
    // heaviest problems first (static striding)
    std::stable_sort(gs.begin(), gs.end(), [](const GemmProb &a, const GemmProb &b) {
        return (int64_t)a.M * a.N * a.K > (int64_t)b.M * b.N * b.K;
    });
    for (size_t b = 0; b < gs.size(); b += kMaxG) {
        GemmParams P;
        memset(&P, 0, sizeof(P));
        P.np = (int)std::min<size_t>(kMaxG, gs.size() - b);
        int items = 0;
        for (int i = 0; i < P.np; i++) {
            P.p[i] = gs[b + i];
            P.p[i].tiles_n = (P.p[i].N + GN - 1) / GN;
            P.p[i].item_begin = items;
            items += ((P.p[i].M + GM - 1) / GM) * P.p[i].tiles_n;
        }
        P.total = items;
        if (!items) continue;
        gemm_3xtf32_kernel<<<std::min(items, sms), GThreads, GSmem, st>>>(P);
        KFAC_LAUNCHED();
        KFAC_CUDA_TRY(cudaGetLastError());
    }
    return KFAC_OK;
}

kfac_status precond_launch(const std::vector<PrecJob> &jobs, cudaStream_t st) {
    // workspace per job: [Ainv split][Ginv split][dW split][T^T split]
    std::vector<SplitJob> sj;
    std::vector<GemmProb> g1, g2;
    for (const PrecJob &j : jobs) {
        float *w = j.tmp;
        const int dA = j.dA, dG = j.dG;
        float *sA = j.sA ? j.sA : w;  // the inverses' split lives in inv_ws when the plan provides it
        w += 2 * (int64_t)dA * kpad(dA);
        float *sG = j.sG ? j.sG : w;
        w += 2 * (int64_t)dG * kpad(dG);
        float *sW = w;
        w += 2 * (int64_t)dG * kpad(dA);
        float *sT = w;
        if (j.resplit || !j.sA) sj.push_back({j.Ainv, sA, dA, dA, dA, (int32_t)kpad(dA)});
        if (j.resplitG || !j.sG) sj.push_back({j.Ginv, sG, dG, dG, dG, (int32_t)kpad(dG)});
        sj.push_back({j.dW, sW, dG, dA, dA, (int32_t)kpad(dA)});
        GemmProb a{};
        kfac_status s = split_map(&a.tA, sA, dA, (int)kpad(dA));
        if (s) return s;
        s = split_map(&a.tB, sW, dG, (int)kpad(dA));
        if (s) return s;
        a.M = dA;
        a.N = dG;
        a.K = dA;
        a.C = sT;  // T^T hi [dA][kpad(dG)], lo right after
        a.ldc = (int)kpad(dG);
        a.Clo = sT + (int64_t)dA * kpad(dG);
        g1.push_back(a);
        GemmProb b{};
        s = split_map(&b.tA, sG, dG, (int)kpad(dG));
        if (s) return s;
        s = split_map(&b.tB, sT, dA, (int)kpad(dG));
        if (s) return s;
        b.M = dG;
        b.N = dA;
        b.K = dG;
        b.C = j.out;
        b.ldc = dA;
        b.Clo = nullptr;
        g2.push_back(b);
    }
    kfac_status s = launch_splits(sj, st);
    if (s) return s;
    s = launch_gemms(g1, st);
    if (s) return s;
    return launch_gemms(g2, st);
}

}  // namespace kfac
