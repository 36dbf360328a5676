/*
 * kfac.h -- C-ABI of the B200-native distributed K-FAC hot path
 * (Osawa et al., "Large-Scale Distributed Second-Order Optimization Using
 * Kronecker-Factored Approximate Curvature for Deep CNNs", arXiv 1811.12019).
 *
 * The calls follow the paper's statement of one K-FAC iteration (PAPER.md
 * §3.3, Fig. 1 and Algorithm 1), minus forward/backward and the
 * weight update:
 *
 *   stage 1-2  kfac_factor_A / kfac_factor_G / kfac_factor_all
 *              A_{l-1} = alpha * sum_rows a a^T over im2col patches (+bias 1),
 *              G_l     = alpha * sum_rows g g^T over output-gradient pixels
 *              (P:237-245 Eq. kf), written as the packed upper
 *              triangle (P:407-411 symmetry-aware communication).
 *   stage 3    kfac_reduce_scatter_factors: ReduceScatterV(mean) of
 *              (dW, A, G) to the layer owners (Alg. 1 line
 *              "Reduce+ScatterV").
 *   stage 4    kfac_damped_inverse: factored Tikhonov damping
 *              and the inverses A_d^-1, G_d^-1 (P:247-260 Eq. inv_fim).
 *   stage 5    kfac_precondition: G_d^-1 * dW * A_d^-1.
 *   stage 6    kfac_allgather_precond: AllGatherV of the preconditioned
 *              gradients.
 *
 * Conventions for every call
 *   - Pointers are CUDA device pointers unless marked "host".
 *   - `stream` is a cudaStream_t passed as void* (NULL = legacy default stream).
 *     Every call only ENQUEUES work on `stream`; none synchronises the device
 *     and none allocates device memory, except kfac_plan_create /
 *     kfac_comm_create (setup-time allocation of small metadata).
 *   - The caller owns every buffer.  The library owns only the opaque plan
 *     and communicator handles.
 *   - Errors are returned synchronously as kfac_status; kfac_last_error()
 *     gives a thread-local message.  Numeric failures found on the device
 *     (a non-positive pivot) are written to `dev_status`, never silently
 *     regularised (damping is the caller's gamma).
 *   - Calls on different streams / ranks may run concurrently; calls sharing
 *     a workspace must be stream-ordered.
 *
 * Data layouts
 *   x   layer input, NHWC [n, h_in, w_in, c_in] for conv2d, [n, c_in] for
 *       linear; bf16 or fp16.
 *   gy  gradient w.r.t. the layer output, NHWC [n, h_out, w_out, c_out]
 *       ([n, c_out] for linear); bf16 or fp16.
 *   dW  weight gradient [c_out, dA] row-major fp32, dA = c_in*kh*kw (+1 bias
 *       column, last); the patch feature order is (kh, kw, c), c fastest,
 *       i.e. channels-last weights (R-5, R-6).
 *   packed factor of dimension d: d(d+1)/2 fp32, upper triangle, row-major:
 *       element (i, j), j >= i, at i*d - i*(i-1)/2 + (j - i)  (R-10).
 *   inverse: full d x d fp32 row-major (symmetric).
 */
#ifndef KFAC_H
#define KFAC_H

#include <stdint.h>

#if defined(__GNUC__)
#define KFAC_API __attribute__((visibility("default")))
#else
#define KFAC_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
    KFAC_OK = 0,
    KFAC_ERR_ARG = 1,         /* bad argument: NULL pointer, n < 1, gamma <= 0, ... */
    KFAC_ERR_SHAPE = 2,       /* inconsistent shapes */
    KFAC_ERR_UNSUPPORTED = 3, /* geometry the kernels do not support */
    KFAC_ERR_CUDA = 4,        /* a CUDA runtime/driver call failed */
    KFAC_ERR_NCCL = 5,        /* an NCCL call failed */
    KFAC_ERR_NOT_PD = 6,      /* reserved: host-side report of a non-PD factor */
    KFAC_ERR_STATE = 7        /* plan/communicator mismatch, wrong world size, ... */
} kfac_status;

typedef enum { KFAC_BF16 = 0, KFAC_FP16 = 1 } kfac_dtype;

/* Layer ownership policy for the model-parallel stages (R-15).
 * ROUND_ROBIN: owner(l) = l mod world.  LPT: layers by descending stage-4/5
 * cost dA^3 + dG^3 + 2 dG^2 dA + 2 dG dA^2 (ties by index) to the least
 * loaded rank (ties by rank).  If world > L, rank r >= L also owns layer
 * r mod L redundantly ("some layers will be calculated
 * redundantly"; R-16).                                                      */
typedef enum { KFAC_OWN_ROUND_ROBIN = 0, KFAC_OWN_LPT = 1 } kfac_policy;

typedef struct {
    int32_t kind; /* 0 = conv2d, 1 = linear */
    int32_t c_in, c_out;
    int32_t kh, kw;             /* 1, 1 for linear */
    int32_t stride_h, stride_w; /* 1, 1 for linear */
    int32_t pad_h, pad_w;       /* 0, 0 for linear */
    int32_t h_in, w_in;         /* 1, 1 for linear */
    int32_t has_bias;           /* appends the homogeneous coordinate 1 to the patch */
} kfac_layer_desc;

typedef struct kfac_plan *kfac_plan_t;
typedef struct kfac_comm *kfac_comm_t;

/* Thread-local message describing the last non-OK status of this thread. */
KFAC_API const char *kfac_last_error(void);
/* Library version string, e.g. "kfac-b200 0.1 sm_100a". */
KFAC_API const char *kfac_version(void);
/* Instrumentation: number of CUDA kernels this library has launched in this
 * process so far (NCCL's own kernels are not counted).  Host-only, no sync. */
KFAC_API int64_t kfac_launch_count(void);

/* ------------------------------------------------------------------ plan
 * kfac_plan_create: ownership map + wire layout for L layers over `world`
 * ranks with `n_local` samples per rank.  host
 * `layers` is copied.  Rank r's ReduceScatter chunk lists its owned layers
 * in ascending order, each with the segments [dW (dG*dA), A packed, G
 * packed]; every segment starts on a 16-element (64 B) boundary and every
 * chunk is padded to rs_chunk = max chunk (NCCL has no V variant).  The
 * AllGather chunk of rank r holds the preconditioned gradient of each layer
 * whose PRIMARY owner is r, ascending, 16-aligned, padded to ag_chunk.
 * Limits: every factor dimension dA, dG <= 16384 (the inverse's step table);
 * any number of layers per rank (the inverse runs in launches of <= 64 owned
 * layers each, in stream order).
 * Errors: KFAC_ERR_ARG (NULL, L < 1, world < 1, n_local < 1, bad policy),
 * KFAC_ERR_SHAPE (a non-positive dimension, kind not 0/1),
 * KFAC_ERR_UNSUPPORTED (a factor dimension above 16384).                   */
KFAC_API kfac_status kfac_plan_create(const kfac_layer_desc *layers /* host [L] */, int32_t L, int32_t world,
                             int32_t n_local, kfac_policy policy, kfac_plan_t *out /* host */);

/* Host outputs (each may be NULL):
 *   owner[L]     primary owner of each layer
 *   seg_off[3L]  element offsets into the world*rs_chunk send buffer of the
 *                PRIMARY copy of (dW, A packed, G packed) of each layer
 *   rs_chunk     elements per rank of the ReduceScatter buffers
 *   ag_off[L]    element offset of each layer's preconditioned gradient in
 *                the world*ag_chunk AllGather buffer
 *   ag_chunk     elements per rank of the AllGather buffer
 *   ws_bytes     workspace bytes needed by any stage on any rank           */
KFAC_API kfac_status kfac_plan_query(kfac_plan_t plan, int32_t *owner, int64_t *seg_off, int64_t *rs_chunk,
                            int64_t *ag_off, int64_t *ag_chunk, int64_t *ws_bytes);

/* Layers owned by `rank` (primary and redundant), ascending.  Host outputs
 * (each may be NULL): n_owned; layers[n_owned]; local_off[3*n_owned] =
 * offsets of (dW, A, G) inside the rank's recv chunk; inv_off[2*n_owned] =
 * offsets (floats) of A_d^-1 and G_d^-1 inside inv_ws; inv_floats = size of
 * inv_ws in floats for this rank (the inverses, then the precondition's
 * cached 3xTF32 split of them).  A stale plan reports the same layout.      */
KFAC_API kfac_status kfac_plan_rank_layers(kfac_plan_t plan, int32_t rank, int32_t *n_owned, int32_t *layers,
                                  int64_t *local_off, int64_t *inv_off, int64_t *inv_floats);

KFAC_API void kfac_plan_destroy(kfac_plan_t plan);

/* ------------------------------------------------------------------ stale Fisher (NEXT-1)
 * The paper refreshes (A, G) only every interval^(e) iterations after the
 * first 500 and reuses the previous preconditioner in
 * between (reading R-20: the owner keeps its cached A_d^-1, G_d^-1 in inv_ws).
 *
 * kfac_plan_create_stale: a plan for the steps that reuse stale factors.  It
 * has the same owners, owned lists, AllGather layout, inverse layout
 * (inv_off, inv_floats) and ws_bytes as `full`, but every owned layer's
 * ReduceScatter segment list is [dW] only: seg_off / local_off of A and G are
 * -1 and rs_chunk shrinks to the gradient payload (a stale step moves
 * strictly fewer bytes in stage 3).  On a stale plan
 *   kfac_factor_all            launches no factor kernel; it only refreshes the
 *                              dW of redundant owner copies (xs, gys may be NULL);
 *   kfac_reduce_scatter_factors, kfac_precondition, kfac_allgather_precond
 *                              work unchanged (precondition reads the cached
 *                              inverses the last full step left in inv_ws);
 *   kfac_damped_inverse, kfac_factor_diff  return KFAC_ERR_STATE.
 * `full` must outlive nothing: the stale plan is independent (destroy both).
 * Errors: KFAC_ERR_ARG (NULL), KFAC_ERR_STATE (`full` is itself stale).       */
KFAC_API kfac_status kfac_plan_create_stale(kfac_plan_t full, kfac_plan_t *out /* host */);
/* 1 for a plan made by kfac_plan_create_stale, else 0. */
KFAC_API int32_t kfac_plan_is_stale(kfac_plan_t plan);

/* kfac_plan_create_grefresh: the plan of a step that refreshes G but keeps A stale (P:688-692,
 * "we can also consider refreshing A_{l-1} less frequently than G_l"; S:549 per-kind
 * intervals).  Same owners / inverse layout as `full`; each owned layer's segments are
 * [dW, G packed] (A's seg_off / local_off are -1).  On this plan
 *   kfac_factor_all       computes only the G factors (xs may be NULL);
 *   kfac_damped_inverse   inverts only G_d = G + sqrt(gamma)/pi I, with pi READ from pi_out
 *                         (the value the last full refresh wrote there, R-20); A_d^-1 in
 *                         inv_ws and dev_status[2k] are left as they are;
 *   kfac_precondition     re-splits G_d^-1 and reuses A_d^-1's cached split;
 *   kfac_factor_diff      returns KFAC_ERR_STATE.                                          */
KFAC_API kfac_status kfac_plan_create_grefresh(kfac_plan_t full, kfac_plan_t *out /* host */);
/* 0 full plan, 1 G-refresh plan, 2 stale plan, -1 NULL. */
KFAC_API int32_t kfac_plan_refresh_kind(kfac_plan_t plan);

/* Refresh schedules of the stale-Fisher runs (host-only, no device work). */
typedef enum {
    KFAC_REFRESH_RAMPUP = 0, /* interval^(e) = min(20, 5 floor(e/5) + 1) */
    KFAC_REFRESH_STEP13 = 1  /* interval^(e) = 1 if e < 13 else 20 */
} kfac_refresh_schedule;
/* interval^(e) of `schedule` for epoch e >= 0; -1 for a bad argument. */
KFAC_API int32_t kfac_refresh_interval(int32_t schedule, int32_t epoch);
/* Refresh decision of iteration t in epoch e: 1 if t < fresh_floor
 * (the paper's 500) or t mod interval == 0, else 0, where interval
 * is `interval` if > 0, else kfac_refresh_interval(schedule, epoch); -1 for a
 * bad argument (t < 0, unknown schedule).                                    */
KFAC_API int32_t kfac_refresh(int64_t t, int32_t epoch, int32_t schedule, int64_t fresh_floor, int32_t interval);

/* ------------------------------------------------------------------ comm
 * NCCL communicator over NVLink/NVSwitch (one process per GPU).  Rank 0 calls
 * kfac_comm_unique_id and broadcasts the 128 host bytes (e.g. with
 * torch.distributed); every rank then calls kfac_comm_create on its device.
 * Errors: KFAC_ERR_NCCL, KFAC_ERR_CUDA, KFAC_ERR_ARG.                       */
KFAC_API kfac_status kfac_comm_unique_id(uint8_t id[128] /* host */);
KFAC_API kfac_status kfac_comm_create(const uint8_t id[128] /* host */, int32_t rank, int32_t world, int32_t device,
                             kfac_comm_t *out /* host */);
KFAC_API void kfac_comm_destroy(kfac_comm_t comm);

/* ------------------------------------------------------------------ stage 1-2
 * kfac_factor_A: out_packed[dA(dA+1)/2] = alpha * sum over the n*h_out*w_out
 * patches ã of ã ã^T (patch extraction fused into the
 * kernel's shared-memory staging, zero padding, (kh,kw,c) order, bias 1
 * last).  Inputs are half precision, products are accumulated in fp32 on the
 * tensor cores.  alpha = 1/rows is the paper's mean (R-3).
 * `ws` is scratch of at least kfac_factor_ws_bytes(..., which=0) bytes (split-K
 * partials + the work-item counter of the dynamic tile schedule, zeroed by the
 * call on `stream`); it may be NULL (no split-K, static tile schedule).
 * Errors: KFAC_ERR_ARG, KFAC_ERR_UNSUPPORTED (e.g. dilation-like geometry the
 * descriptor cannot express), KFAC_ERR_CUDA.                                */
KFAC_API kfac_status kfac_factor_A(const kfac_layer_desc *layer /* host */, const void *x, kfac_dtype dtype, int32_t n,
                          float alpha, float *out_packed, void *ws, int64_t ws_bytes, void *stream);

/* kfac_factor_G: out_packed[dG(dG+1)/2] = alpha * sum over the n*h_out*w_out
 * pixels g = gy[pixel, :] of g g^T (the caller folds any per-sample
 * loss scale into gy or alpha, R-4).                                        */
KFAC_API kfac_status kfac_factor_G(const kfac_layer_desc *layer /* host */, const void *gy, kfac_dtype dtype, int32_t n,
                          float alpha, float *out_packed, void *ws, int64_t ws_bytes, void *stream);

/* Scratch bytes kfac_factor_A (which = 0) / kfac_factor_G (which = 1) need. */
KFAC_API kfac_status kfac_factor_ws_bytes(const kfac_layer_desc *layer /* host */, int32_t n, int32_t which,
                                 int64_t *bytes /* host */);

/* All factors of one rank in ONE grouped launch (plus a split-K fix-up):
 * A and G of every layer l are written packed into rs_send at every owner
 * copy of layer l (primary seg_off and redundant copies); the dW segment of
 * each redundant copy is refreshed from the primary copy (the caller writes
 * dW into the primary segments).  xs / gys: host arrays of L device
 * pointers; alphaA / alphaG: host arrays of L scales, or NULL for 1/rows.
 * ws: at least ws_bytes from kfac_plan_query.                               */
KFAC_API kfac_status kfac_factor_all(kfac_plan_t plan, const void *const *xs /* host [L] */,
                            const void *const *gys /* host [L] */, kfac_dtype dtype,
                            const float *alphaA /* host [L] or NULL */, const float *alphaG /* host [L] or NULL */,
                            float *rs_send /* [world*rs_chunk] */, void *ws, void *stream);

/* ------------------------------------------------------------------ stage 3
 * ReduceScatterV(mean): rs_recv[0:rs_chunk] of rank r = mean over ranks of
 * rs_send[r*rs_chunk : (r+1)*rs_chunk] (R-11).  One NCCL
 * ReduceScatter(ncclAvg) over the owner-major padded buffer.  comm may be NULL
 * only when world == 1 (then a device copy, or nothing if send == recv).   */
KFAC_API kfac_status kfac_reduce_scatter_factors(kfac_comm_t comm, kfac_plan_t plan, const float *rs_send,
                                        float *rs_recv, void *stream);

/* kfac_reduce_scatter_factors_ws: the same ReduceScatterV with a workspace `ws` (device, at least
 * ws_bytes from kfac_plan_query AFTER kfac_plan_set_wire), which an fp16-wire plan needs for its
 * staging (below); ws may be NULL for an fp32-wire plan.  kfac_reduce_scatter_factors is this call
 * with ws = NULL and returns KFAC_ERR_ARG on a plan whose wire needs staging.                       */
KFAC_API kfac_status kfac_reduce_scatter_factors_ws(kfac_comm_t comm, kfac_plan_t plan, const float *rs_send,
                                                    float *rs_recv, void *ws, void *stream);

/* Wire format of the factor segments in the ReduceScatterV (NEXT-4(ii); "half precision
 * floating point numbers for both computation [and communication]"; reading R-23):
 *   KFAC_WIRE_FP32  the packed A / G travel as the fp32 the factor kernels wrote (default);
 *   KFAC_WIRE_FP16  each rank's A (G) element x travels as binary16(x * scale_A (scale_G)), round to
 *                   nearest even; the fp16 words are gathered to the owner (grouped ncclSend /
 *                   ncclRecv, no arithmetic in flight), which writes their mean (fp32 sum in rank
 *                   order, / world) * 1/scale into rs_recv.  Halves the factor payload; dW always
 *                   travels in fp32 (ncclReduce / ReduceScatter avg as kfac_plan_set_rs_mode says).
 *                   The scales are powers of two chosen by the caller (like loss scaling) so that
 *                   every |x| * scale stays below 65504 (overflow gives inf, which the inverse reports
 *                   as a failed pivot) and above the fp16 subnormal range where accuracy matters.  At
 *                   world = 1 the round trip is still applied (the same rounding at every world size).
 * Changes ws_bytes (the staging: world x (fp32 dW region + fp16 factor region) for the send and one
 * fp32 + world fp16 regions for the receive); query the plan after this call.  Stale / G-refresh
 * plans take the wire of the plan they were made from.  Errors: KFAC_ERR_ARG (NULL plan, unknown
 * wire, a scale that is not a power of two in [2^-61, 2^59]), KFAC_ERR_UNSUPPORTED (fp16 wire with
 * more than 16 ranks).                                                                              */
typedef enum { KFAC_WIRE_FP32 = 0, KFAC_WIRE_FP16 = 1 } kfac_wire;
KFAC_API kfac_status kfac_plan_set_wire(kfac_plan_t plan, int32_t wire, float scale_A, float scale_G);

/* How kfac_reduce_scatter_factors moves the owner-major buffer:
 *   KFAC_RS_PADDED     one ncclReduceScatter(avg) of world x rs_chunk (every rank's chunk padded to the
 *                      largest; default);
 *   KFAC_RS_PER_OWNER  an ncclGroup of one ncclReduce(avg) per owner, rooted at it, over exactly the
 *                      floats its chunk uses (the ReduceScatterV of the paper: no padding; rs_recv
 *                      beyond the owner's payload is left untouched).
 * Same result on every element the layout uses.  Stale / G-refresh plans take the mode of the plan
 * they were made from.  Errors: KFAC_ERR_ARG.                                                      */
typedef enum { KFAC_RS_PADDED = 0, KFAC_RS_PER_OWNER = 1 } kfac_rs_mode;
KFAC_API kfac_status kfac_plan_set_rs_mode(kfac_plan_t plan, int32_t mode);

/* ------------------------------------------------------------------ stage 4
 * For every layer owned by `rank` (kfac_plan_rank_layers order, k-th layer):
 *   pi = sqrt((tr A / dA) / (tr G / dG)), pi = 1 if a trace is 0;
 *   A_d = A + pi*sqrt(gamma) I,  G_d = G + sqrt(gamma)/pi I   (R-1)
 * and writes A_d^-1, G_d^-1 (full fp32) at inv_off into inv_ws (R-12:
 * fp64-class arithmetic, see kfac_plan_set_inverse_precision).  dev_status[2k+0 / 2k+1] = 0 on success, else the failing
 * pivot index + 1 for A_d / G_d.  pi_out (device, may be NULL) receives pi per
 * owned layer.  Errors: KFAC_ERR_ARG (gamma <= 0, NULL), KFAC_ERR_STATE.    */
KFAC_API kfac_status kfac_damped_inverse(kfac_plan_t plan, int32_t rank, const float *rs_recv, float gamma, float *inv_ws,
                                int32_t *dev_status, float *pi_out, void *ws, void *stream);

/* Precision of the damped inverse's sweep updates (reading R-12).  The pivots,
 * panels P_k R_J and the working matrix are fp64 in every mode; what varies is the rank-128 update
 * M_IJ -= R_I^T (P_k R_J), > 90% of the flops:
 *   KFAC_INV_AUTO  per matrix, from the a-priori bound kappa(M_d) <= tr(M_d)/delta (delta = the
 *                  damping added): int8-sliced updates (each fp64 operand column as 5 balanced
 *                  8-bit digits under a power-of-two scale; exact int32 tensor-core sums of the
 *                  15 leading digit pairs, recombined exactly in int64 and scaled in fp64;
 *                  relative error <= ~3e-13 x bound on the paper's factors) where
 *                  bound <= 3e6, fp64 DMMA updates elsewhere (default);
 *   KFAC_INV_FP64  fp64 DMMA updates for every matrix;
 *   KFAC_INV_INT8  int8-sliced updates for every matrix (tests and experiments).
 * A stale / G-refresh plan takes the mode of the plan it was made from at creation.
 * Errors: KFAC_ERR_ARG (NULL plan, unknown mode).                                               */
typedef enum { KFAC_INV_AUTO = 0, KFAC_INV_FP64 = 1, KFAC_INV_INT8 = 2 } kfac_inv_precision;
KFAC_API kfac_status kfac_plan_set_inverse_precision(kfac_plan_t plan, int32_t mode);

/* After kfac_damped_inverse on `stream` with workspace `ws`: per owned matrix 2k+0 (A_d) / 2k+1
 * (G_d) of `rank`, the condition bound tr(M_d)/delta and the update precision it got (4 = int8
 * slices, 0 = fp64).  Host outputs of 2 x (owned layers) entries.  SYNCHRONISES `stream` (a
 * device-to-host copy of the pair data at the start of ws).  Errors: KFAC_ERR_ARG, KFAC_ERR_STATE
 * (stale plan, rank), KFAC_ERR_CUDA.  On a G-refresh plan the A entries are not meaningful.     */
KFAC_API kfac_status kfac_inverse_report(kfac_plan_t plan, int32_t rank, const void *ws, double *bound /* host */,
                                         int32_t *slices /* host */, void *stream);

/* Change rate of the Kronecker factors between two refreshes:
 * for the k-th layer owned by `rank` (kfac_plan_rank_layers order),
 *   diff[2k + 0] = ||A_cur - A_prev||_F / ||A_prev||_F,  diff[2k + 1] likewise for G,
 * Frobenius norms of the full symmetric matrices, computed in fp64 from the
 * packed segments of two recv chunks of the FULL plan (recv_cur = this
 * refresh's ReduceScatter output, recv_prev = the previous refresh's, kept by
 * the caller).  NaN where ||X_prev||_F = 0 ("recorded as missing").
 * diff: device fp64 [2 * n_owned].  ws: >= ws_bytes of the plan (block
 * partials).  Two launches, HBM-bound (reads both chunks' factor segments
 * once).  Errors: KFAC_ERR_ARG (NULL, a misaligned chunk), KFAC_ERR_STATE
 * (stale plan, rank out of range).                                          */
KFAC_API kfac_status kfac_factor_diff(kfac_plan_t plan, int32_t rank, const float *recv_cur, const float *recv_prev,
                             double *diff, void *ws, void *stream);

/* ------------------------------------------------------------------ stage 5
 * For every layer owned by `rank`: P = G_d^-1 * dW * A_d^-1, dW
 * read from rs_recv.  The primary owner writes P into ag_buf at ag_off[l]
 * (its own AllGather slot); a redundant owner writes into `ws`.  inv_ws is
 * read AND written: on a full plan the call stores the 3xTF32 hi / lo split of
 * each inverse after the inverses (the tail of inv_floats), and on a stale
 * plan it reuses that split instead of re-splitting (R-20), so a stale step
 * must follow a full-plan precondition on the same inv_ws.                  */
KFAC_API kfac_status kfac_precondition(kfac_plan_t plan, int32_t rank, const float *rs_recv, float *inv_ws,
                              float *ag_buf /* [world*ag_chunk] */, void *ws, void *stream);

/* ------------------------------------------------------------------ stage 6
 * In-place AllGatherV: afterwards every rank's ag_buf holds every layer's
 * preconditioned gradient at ag_off[l].  comm may be NULL when
 * world == 1 (no-op).                                                        */
KFAC_API kfac_status kfac_allgather_precond(kfac_comm_t comm, kfac_plan_t plan, float *ag_buf, void *stream);

/* ------------------------------------------------------------------ NEXT-3: the update
 * After the AllGather every rank applies, for every layer l (Eq. paramupdate):
 *   w_l <- w_l - lr * P_l + momentum * (w_l - w_prev_l),   w_prev_l <- (old) w_l
 * with P_l the preconditioned gradient at ag_off[l] in ag_buf, and then, if
 * rescale != 0, Normalizing Weights on the weight columns:
 *   W_l <- sqrt(2 dG) * W_l / (||W_l||_F + eps)     (the paper's eps = 1e-9)
 * where W_l is w_l without its bias column (the last column when has_bias;
 * reading R-21: the bias is updated but not rescaled).  w[l], w_prev[l]:
 * host arrays of L device pointers to [dG, dA] row-major fp32 (the layout of
 * dW, bias column last), updated in place; 16-byte alignment enables vector
 * access.  lr / momentum are this epoch's eta^(e), m^(e).
 * Arithmetic is fp32 per element, the norm is accumulated in fp64.
 * ws: >= ws_bytes of the plan.  One or two launches, HBM-bound (20 B per
 * weight).  Errors: KFAC_ERR_ARG (NULL, non-finite lr / momentum, eps < 0).   */
KFAC_API kfac_status kfac_update(kfac_plan_t plan, const float *ag_buf, float *const *w /* host [L] */,
                        float *const *w_prev /* host [L] */, float lr, float momentum, int32_t rescale, float eps,
                        void *ws, void *stream);

/* ------------------------------------------------------------------ NEXT-2: Batch Normalization Fisher
 * A BN layer y = gamma * xhat + beta has 2C parameters, ordered [gamma_1..gamma_C, beta_1..beta_C]
 * (reading R-22).  Its Fisher is not factored into A and G:
 *   F = (1/n) sum_s S_s S_s^T,  S_s = [sum_p gy_{s,p} * xhat_{s,p} ; sum_p gy_{s,p}]   (2C)
 * over the n samples s and hw pixels p; the paper damps it with gamma_BN = rho_BN * gamma
 * and also uses its diagonal ("approximate it with a diagonal matrix").
 *
 * kfac_bn_grads: S[l] ([n][2C] fp32, device) for nl BN layers in one launch, from xhat[l] and
 * gy[l] (NHWC half [n, hw[l], c[l]], the normalised BN input and the gradient w.r.t. the BN
 * output; the caller folds any per-sample loss scale into gy, R-4).  fp32 accumulation.
 * c, hw, xhat, gy, S: host arrays [nl].  Errors: KFAC_ERR_ARG (NULL, n < 1, dtype),
 * KFAC_ERR_SHAPE (c < 2, hw < 1), KFAC_ERR_UNSUPPORTED (odd c, xhat / gy not 4-byte aligned). */
KFAC_API kfac_status kfac_bn_grads(int32_t nl, const int32_t *c /* host [nl] */, const int32_t *hw /* host [nl] */,
                          const void *const *xhat /* host [nl] */, const void *const *gy /* host [nl] */,
                          kfac_dtype dtype, int32_t n, float *const *S /* host [nl] */, void *stream);

/* kfac_bn_precondition: out[l] = (F_l + gamma_bn I)^-1 grad[l] (full != 0) or
 * grad[l]_i / (F_l,ii + gamma_bn) (full == 0, the diagonal FIM), F_l from S[l] as above.
 * The full mode never forms F: F has rank <= n, and by the Woodbury identity
 *   (F + gamma_bn I)^-1 v = (v - S^T (gamma_bn n I + S S^T)^-1 S v) / gamma_bn,
 * i.e. a column-parallel fp64 Gram S S^T (all layers in one launch) and an n x n fp64
 * Cholesky solve per layer; n <= 256 (the samples of up to 8 ranks of 32 after an
 * all-gather of S; K sits in shared memory up to n = 128, in the workspace beyond).  grad / out: [2C] fp32 device (out may not alias grad).  ws: device
 * scratch of kfac_bn_ws_bytes (full mode; may be NULL for the diagonal mode).
 * Errors: KFAC_ERR_ARG (NULL, gamma_bn <= 0, n < 1, full mode without enough ws),
 * KFAC_ERR_SHAPE (c < 1), KFAC_ERR_UNSUPPORTED (full mode with n > 256).                */
KFAC_API kfac_status kfac_bn_precondition(int32_t nl, const int32_t *c /* host [nl] */, int32_t n,
                                 const float *const *S /* host [nl] */, const float *const *grad /* host [nl] */,
                                 float gamma_bn, int32_t full, float *const *out /* host [nl] */, void *ws,
                                 int64_t ws_bytes, void *stream);
/* Multi-GPU BN Fisher: every rank receives all ranks' per-sample gradients,
 * S_all[l] = [S_local[l] of rank 0; ...; of rank world-1] ([world * n_local][2C], the
 * samples of the global batch, so F over S_all is the mean of the ranks' F, P:319-321,
 * R-11), and grad[l] becomes the mean over ranks in place; then every rank runs
 * kfac_bn_precondition with n = world * n_local (BN work is tiny, so it is replicated
 * instead of owned, R-22).  One NCCL group of AllGathers / AllReduces over NVLink.
 * Errors: KFAC_ERR_ARG, KFAC_ERR_NCCL.                                              */
KFAC_API kfac_status kfac_bn_exchange(kfac_comm_t comm, int32_t nl, const int32_t *c /* host [nl] */, int32_t n_local,
                             const float *const *S_local /* host [nl] */, float *const *S_all /* host [nl] */,
                             float *const *grad /* host [nl] */, void *stream);
/* Workspace bytes kfac_bn_precondition's full mode needs for these layers and n. */
KFAC_API kfac_status kfac_bn_ws_bytes(int32_t nl, const int32_t *c /* host [nl] */, int32_t n,
                             int64_t *bytes /* host */);

#ifdef __cplusplus
}
#endif
#endif /* KFAC_H */
