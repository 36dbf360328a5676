// kfac_internal.hpp -- shared host/device declarations of the K-FAC library
// (not part of the C-ABI; see include/kfac.h for the public contract).
#pragma once
#include <atomic>
#include <cstdint>
#include <string>
#include <vector>

#include <cuda.h>
#include <cuda_runtime.h>

#include "../../include/kfac.h"

namespace kfac {

// ---------------------------------------------------------------- errors
kfac_status set_error(kfac_status st, const std::string &msg);
extern std::atomic<int64_t> g_launches;  // kernels launched (kfac_launch_count)
#define KFAC_LAUNCHED() (::kfac::g_launches.fetch_add(1, std::memory_order_relaxed))
#define KFAC_CUDA_TRY(expr)                                                                     \
    do {                                                                                        \
        cudaError_t _e = (expr);                                                                \
        if (_e != cudaSuccess)                                                                  \
            return ::kfac::set_error(KFAC_ERR_CUDA, std::string(#expr) + ": " + cudaGetErrorString(_e)); \
    } while (0)

// per-device launch setup, thread-safe (a process may drive several GPUs from several threads):
// the current device's SM count, and the >48 KB dynamic shared memory opt-in of `func` on it
kfac_status dev_sm_count(int *sms);
kfac_status dev_func_smem(const void *func, int bytes);

#define KFAC_TRY(expr)                     \
    do {                                   \
        kfac_status _s = (expr);           \
        if (_s != KFAC_OK) return _s;      \
    } while (0)

inline int64_t packed_len(int64_t d) { return d * (d + 1) / 2; }
inline int64_t align16(int64_t v) { return (v + 15) / 16 * 16; }

struct Geom {  // derived geometry of one layer
    int c_in, c_out, kh, kw, sh, sw, ph, pw, h, w, ho, wo, bias, kind;
    int dF;  // c_in*kh*kw (patch features)
    int dA, dG;
};
kfac_status make_geom(const kfac_layer_desc &d, Geom *g);

// ---------------------------------------------------------------- factor kernel
constexpr int kMaxProbs = 112;   // factor problems per grouped launch
constexpr int kMaxMaps = 140;    // TMA descriptors per grouped launch
constexpr int kTile = 256;       // square output tile (two M = 128 halves x N = 256)
constexpr int kBK = 64;          // K rows (pixels) per pipeline stage

enum FactorMode : int32_t { MODE_TILED2D = 0, MODE_TILED4D = 1, MODE_GATHER = 2 };

struct alignas(64) FactorProb {  // 128 B
    const uint16_t *src;    // NHWC half input (MODE_GATHER, bias column sums, im2col staging)
    float *out;             // packed upper output, dimension d_out
    float *partial;         // split-K partial tiles (splits > 1)
    int64_t rows;           // K = n * ho * wo
    uint16_t *col;          // materialised im2col rows [rows, cp] (only when im2col_pre)
    uint64_t mapj;          // TILED4D: byte j = descriptor index (relative to map0) of filter column j
    float alpha;
    int32_t d, d_out, npairs, splits, kchunks, chunks_per_split, item_begin;
    int16_t nt, cb, S, map0;  // tiles per side, channels per slot, slots per TMA box, first descriptor
    int16_t ksteps, bh, bn, rpi;  // 16-row MMA steps per chunk; TILED4D rows / images per chunk, row groups
    int16_t c, h, w, ho, wo, cp, wp;  // cp: padded im2col width (im2col_pre); wp: box width (pow2 >= wo)
    int8_t mode, kh, kw, sh, sw, ph, pw, im2col_pre, nmaps;
};
static_assert(sizeof(FactorProb) == 128, "FactorProb layout");

struct FactorParams {  // kernel parameter block (< 32 KB)
    int32_t nprobs, total_items, ab_fmt, dbg, nmaps;
    int32_t pad0_;
    int32_t *counter;     // work-item counter in the workspace (zeroed before the launch); null: static striding
    int32_t pad_[8];
    FactorProb probs[kMaxProbs];
    CUtensorMap maps[kMaxMaps];
};
static_assert(sizeof(FactorParams) <= 32760, "kernel parameter space");

// one factor problem (a layer's A or G) as seen by the host planner
struct FactorJob {
    Geom g;
    bool is_A;            // A over im2col patches, else G over gy pixels
    const void *src;      // x or gy
    float *out;           // packed output (dimension dA or dG)
    float alpha;
    int64_t n;            // samples
};

// host planning of a list of jobs: item counts, splits, workspace bytes
struct FactorLaunch {
    std::vector<FactorParams> params;  // one per grouped launch (<= kMaxProbs problems)
    int64_t ws_bytes = 0;
};
kfac_status factor_prepare(const std::vector<FactorJob> &jobs, kfac_dtype dt, void *ws, int64_t ws_cap,
                           bool dry_run, FactorLaunch *out);
kfac_status factor_launch(const FactorLaunch &fl, const std::vector<FactorJob> &jobs, cudaStream_t st);

// ---------------------------------------------------------------- inverse / precondition
struct InvMat {        // one damped factor to invert
    const float *packed;  // packed upper fp32 (from rs_recv)
    float *inv;           // full fp32 output
    double *work;         // n*n fp64 working matrix
    double *panel;        // 8 * kPanel * ld + 2 * kPanel^2 fp64 (R, P R per step mod 4; two pivots)
    int32_t *status;      // device status word
    float *split;         // [2][n][round4(n)] tf32 hi / lo split of the inverse (the precondition's operand), or null
    int32_t n;
    int32_t pair;         // index of the (A, G) pair this matrix belongs to
    int32_t is_A;
};
struct PrecJob {
    const float *dW;      // [dG, dA]
    const float *Ainv;    // [dA, dA]
    const float *Ginv;    // [dG, dG]
    float *tmp;           // precond_ws_floats(dG, dA) scratch (3xTF32 split operands, T^T)
    float *out;           // [dG, dA]
    float *sA, *sG;       // persistent hi / lo split of A_d^-1, G_d^-1 (precond_split_floats each, in inv_ws)
    int32_t resplit;      // 1: split A_d^-1 into sA (full step); 0: reuse it (stale / G-refresh step, R-20)
    int32_t resplitG;     // 1: split G_d^-1 into sG (full / G-refresh step); 0: reuse it (stale step)
    int32_t dG, dA;
};
int64_t precond_split_floats(int n);  // [2][n][kpad(n)] hi / lo copy of one n x n inverse
kfac_status inverse_launch(const std::vector<InvMat> &mats, int npairs, float gamma, double *pair_scratch,
                           float *pi_out, int g_only, int prec_mode, cudaStream_t st);
kfac_status precond_launch(const std::vector<PrecJob> &jobs, cudaStream_t st);
struct DiffMat {          // one packed factor of the stale-Fisher change rate (diff.cu)
    const float *cur, *prev;  // packed upper, 16-byte aligned
    double *out;
    int32_t n;
};
struct WireSeg {            // one segment of the fp16 factor wire (wire.cu)
    int64_t src;              // float offset in the owner's chunk of rs_send / rs_recv
    int64_t dst;              // element offset in the owner's fp32 (kind 0) or fp16 (kind 1, 2) wire region
    int64_t len;              // elements
    int32_t kind;             // 0 dW (fp32), 1 A, 2 G (fp16 x scale)
    int32_t owner;
};
kfac_status wire_pack(const std::vector<WireSeg> &segs, const float *rs_send, int64_t rs_chunk, float *f32,
                      int64_t f32_stride, void *f16, int64_t f16_stride, float scale_A, float scale_G, cudaStream_t st);
kfac_status wire_unpack(const std::vector<WireSeg> &segs, const float *f32, const void *const *f16, int npeers,
                        float *rs_recv, float scale_A, float scale_G, cudaStream_t st);
struct UpdJob {            // one layer of the post-AllGather update (update.cu)
    float *w, *w_prev;        // [dG, dA] row-major fp32, caller-owned
    const float *g;           // preconditioned gradient in the AllGather buffer
    int32_t dG, dA, bias;
};
kfac_status update_launch(const std::vector<UpdJob> &jobs, float lr, float mom, int rescale, float eps, double *ws,
                          int64_t ws_bytes, cudaStream_t st);
struct BnJob {             // one Batch Normalization layer (bn.cu)
    const void *xhat, *gy;    // NHWC half [n, hw, c]
    float *S;                 // per-sample gradients [n][2c]
    const float *grad;        // [2c] (scale, shift)
    float *out;               // [2c]
    int32_t c, hw;
};
constexpr int kBnMaxSamples = 256;  // full-mode Woodbury solve: n x n fp64 K (8 ranks x 32 samples)
kfac_status bn_grads_launch(const std::vector<BnJob> &jobs, int n, int fp16, cudaStream_t st);
kfac_status bn_precond_launch(const std::vector<BnJob> &jobs, int n, int full, double lambda, double *ws,
                              int64_t ws_bytes, cudaStream_t st);
int64_t bn_ws_bytes(const std::vector<int> &cs, int n);  // full-mode Gram partials
kfac_status diff_launch(const std::vector<DiffMat> &mats, double *ws, int64_t ws_bytes, cudaStream_t st);
int64_t precond_ws_floats(int dG, int dA);  // split operands of one layer's two products
kfac_status replicate_launch(const std::vector<std::pair<const float *, float *>> &src_dst,
                             const std::vector<int64_t> &counts, cudaStream_t st);

constexpr int kPanel = 128;  // sweep block size of the inverse
constexpr int kMaxInverseDim = 128 * kPanel;  // 16384: the sweep's step table (kfac_plan_create rejects larger)
int64_t inverse_ws_doubles(int n);  // fp64 working matrix + panels of one n x n inverse
// pair data (pi, damping) + the dataflow state of the persistent sweep; over the owned matrices,
// sum_nt = sum of nt = ceil(n / kPanel), sum_tiles = sum of nt (nt + 1) / 2
int64_t inverse_scratch_bytes(int npairs, int64_t sum_nt, int64_t sum_tiles, int64_t sum_tasks);
int64_t inverse_tasks(int n);  // tasks of one matrix's sweep (sum_tasks = sum over owned matrices)

}  // namespace kfac
