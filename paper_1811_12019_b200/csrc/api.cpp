// api.cpp -- the C-ABI entry points of the K-FAC hot path (include/kfac.h):
// argument validation, marshalling into the grouped kernel launchers, and the
// NCCL collectives.  Every step of the path runs in this library's kernels or
// in NCCL; nothing here computes on the host.
#include <nvtx3/nvToolsExt.h>
#include <dlfcn.h>

#include <cmath>
#include <cstring>
#include <string>

#include <nccl.h>

#include "kfac_plan.hpp"

using namespace kfac;

// NVTX ranges around the stage entry points (SURVEY §5 tracing): header-only NVTX 3, a no-op unless a
// profiler injects its collector (nsys / ncu --nvtx)
struct NvtxRange {
    explicit NvtxRange(const char *name) { nvtxRangePushA(name); }
    ~NvtxRange() { nvtxRangePop(); }
    NvtxRange(const NvtxRange &) = delete;
    NvtxRange &operator=(const NvtxRange &) = delete;
};

struct kfac_comm {
    ncclComm_t comm = nullptr;
    int rank = 0, world = 1, device = 0;
};

#define KFAC_NCCL_TRY(expr)                                                                   \
    do {                                                                                      \
        ncclResult_t _r = (expr);                                                             \
        if (_r != ncclSuccess)                                                                \
            return set_error(KFAC_ERR_NCCL, std::string(#expr) + ": " + ncclGetErrorString(_r)); \
    } while (0)

// After enqueueing a collective: a communicator that has failed asynchronously (a peer died, a
// network / NVLink error) reports it here instead of hanging later (SURVEY §5 failure detection).
static kfac_status nccl_check_async(ncclComm_t comm) {
    ncclResult_t a = ncclSuccess;
    ncclResult_t r = ncclCommGetAsyncError(comm, &a);
    if (r != ncclSuccess) return set_error(KFAC_ERR_NCCL, std::string("ncclCommGetAsyncError: ") + ncclGetErrorString(r));
    if (a != ncclSuccess && a != ncclInProgress)
        return set_error(KFAC_ERR_NCCL, std::string("NCCL asynchronous error: ") + ncclGetErrorString(a));
    return KFAC_OK;
}

static cudaStream_t S(void *s) { return static_cast<cudaStream_t>(s); }

static kfac_status one_factor(const kfac_layer_desc *layer, const void *src, kfac_dtype dt, int32_t n, float alpha,
                              float *out, void *ws, int64_t ws_bytes, void *stream, bool is_A) {
    if (!layer || !src || !out) return set_error(KFAC_ERR_ARG, "kfac_factor: NULL argument");
    if (n < 1) return set_error(KFAC_ERR_ARG, "kfac_factor: n must be >= 1 (empty capture)");
    if (dt != KFAC_BF16 && dt != KFAC_FP16) return set_error(KFAC_ERR_ARG, "kfac_factor: dtype");
    FactorJob j{};
    kfac_status s = make_geom(*layer, &j.g);
    if (s) return s;
    j.is_A = is_A;
    j.src = src;
    j.out = out;
    j.alpha = alpha;
    j.n = n;
    std::vector<FactorJob> jobs{j};
    FactorLaunch fl;
    s = factor_prepare(jobs, dt, ws, ws ? ws_bytes : 0, false, &fl);
    if (s) return s;
    return factor_launch(fl, jobs, S(stream));
}

// Stale plan: no factor kernel; the dW segment of each redundant owner copy is
// refreshed from the primary copy, as kfac_factor_all does on a full step.
static kfac_status replicate_dw(kfac_plan *p, float *rs_send, void *stream) {
    std::vector<std::pair<const float *, float *>> sd;
    std::vector<int64_t> cnt;
    for (int r = 0; r < p->world; r++)
        for (size_t k = 0; k < p->owned[r].size(); k++) {
            const int l = p->owned[r][k];
            if (p->owner[l] == r) continue;
            sd.push_back({rs_send + p->seg_off[3 * l], rs_send + (int64_t)r * p->rs_chunk + p->local[r][k][0]});
            cnt.push_back((int64_t)p->geoms[l].dG * p->geoms[l].dA);
        }
    if (!sd.empty()) return replicate_launch(sd, cnt, S(stream));
    return KFAC_OK;
}

extern "C" {

kfac_status kfac_factor_A(const kfac_layer_desc *layer, const void *x, kfac_dtype dt, int32_t n, float alpha,
                          float *out_packed, void *ws, int64_t ws_bytes, void *stream) {
    return one_factor(layer, x, dt, n, alpha, out_packed, ws, ws_bytes, stream, true);
}

kfac_status kfac_factor_G(const kfac_layer_desc *layer, const void *gy, kfac_dtype dt, int32_t n, float alpha,
                          float *out_packed, void *ws, int64_t ws_bytes, void *stream) {
    return one_factor(layer, gy, dt, n, alpha, out_packed, ws, ws_bytes, stream, false);
}

kfac_status kfac_factor_ws_bytes(const kfac_layer_desc *layer, int32_t n, int32_t which, int64_t *bytes) {
    if (!layer || !bytes || n < 1 || (which != 0 && which != 1)) return set_error(KFAC_ERR_ARG, "kfac_factor_ws_bytes");
    FactorJob j{};
    kfac_status s = make_geom(*layer, &j.g);
    if (s) return s;
    j.is_A = which == 0;
    j.n = n;
    std::vector<FactorJob> jobs{j};
    FactorLaunch fl;
    s = factor_prepare(jobs, KFAC_BF16, nullptr, 0, true, &fl);
    if (s) return s;
    *bytes = fl.ws_bytes;
    return KFAC_OK;
}

kfac_status kfac_factor_all(kfac_plan_t p, const void *const *xs, const void *const *gys, kfac_dtype dt,
                            const float *alphaA, const float *alphaG, float *rs_send, void *ws, void *stream) {
    const NvtxRange nvtx_("kfac.factor_all");
    if (p && p->stale && rs_send) return replicate_dw(p, rs_send, stream);
    if (!p || (!xs && !p->g_only) || !gys || !rs_send) return set_error(KFAC_ERR_ARG, "kfac_factor_all: NULL argument");
    if (dt != KFAC_BF16 && dt != KFAC_FP16) return set_error(KFAC_ERR_ARG, "kfac_factor_all: dtype");
    if (p->factor_ws > 0 && !ws) return set_error(KFAC_ERR_ARG, "kfac_factor_all: workspace required");
    const int L = p->L;
    std::vector<float> aA(L), aG(L);
    for (int l = 0; l < L; l++) {
        const Geom &g = p->geoms[l];
        const double rows = (double)p->n_local * g.ho * g.wo;
        aA[l] = alphaA ? alphaA[l] : (float)(1.0 / rows);
        aG[l] = alphaG ? alphaG[l] : (float)(1.0 / rows);
        if ((!p->g_only && !xs[l]) || !gys[l]) return set_error(KFAC_ERR_ARG, "kfac_factor_all: NULL input pointer");
    }
    std::lock_guard<std::mutex> lock(p->c_mu);
    const std::vector<const void *> xv = p->g_only ? std::vector<const void *>(L, nullptr)
                                                   : std::vector<const void *>(xs, xs + L);
    const bool same = p->c_dt == (int)dt && p->c_send == rs_send && p->c_ws == ws && p->c_xs == xv &&
                      p->c_gys == std::vector<const void *>(gys, gys + L) && p->c_aA == aA && p->c_aG == aG;
    if (!same) {
        p->c_jobs.clear();
        for (int l = 0; l < L; l++) {
            FactorJob a{};
            a.g = p->geoms[l];
            a.n = p->n_local;
            a.is_A = true;
            a.src = p->g_only ? nullptr : xs[l];
            a.out = p->g_only ? nullptr : rs_send + p->seg_off[3 * l + 1];
            a.alpha = aA[l];
            if (!p->g_only) p->c_jobs.push_back(a);  // a G refresh keeps A stale
            FactorJob b = a;
            b.is_A = false;
            b.src = gys[l];
            b.out = rs_send + p->seg_off[3 * l + 2];
            b.alpha = aG[l];
            p->c_jobs.push_back(b);
        }
        kfac_status s = factor_prepare(p->c_jobs, dt, ws, p->ws_bytes, false, &p->c_fl);
        if (s) {
            p->c_dt = -1;
            return s;
        }
        p->c_dt = (int)dt;
        p->c_send = rs_send;
        p->c_ws = ws;
        p->c_xs = xv;
        p->c_gys.assign(gys, gys + L);
        p->c_aA = aA;
        p->c_aG = aG;
    }
    kfac_status s = factor_launch(p->c_fl, p->c_jobs, S(stream));
    if (s) return s;
    // redundant owners: copy the primary (dW, A, G) segments into their chunks
    std::vector<std::pair<const float *, float *>> sd;
    std::vector<int64_t> cnt;
    for (int r = 0; r < p->world; r++) {
        for (size_t k = 0; k < p->owned[r].size(); k++) {
            const int l = p->owned[r][k];
            if (p->owner[l] == r) continue;
            const Geom &g = p->geoms[l];
            const int64_t n3[3] = {(int64_t)g.dG * g.dA, packed_len(g.dA), packed_len(g.dG)};
            for (int s3 = 0; s3 < 3; s3++) {
                if (p->local[r][k][s3] < 0) continue;  // segment absent from this layout
                sd.push_back({rs_send + p->seg_off[3 * l + s3], rs_send + (int64_t)r * p->rs_chunk + p->local[r][k][s3]});
                cnt.push_back(n3[s3]);
            }
        }
    }
    if (!sd.empty()) return replicate_launch(sd, cnt, S(stream));
    return KFAC_OK;
}

// ------------------------------------------------------------------ stale Fisher (NEXT-1)
kfac_status kfac_factor_diff(kfac_plan_t p, int32_t rank, const float *recv_cur, const float *recv_prev, double *diff,
                             void *ws, void *stream) {
    const NvtxRange nvtx_("kfac.factor_diff");
    if (!p || !recv_cur || !recv_prev || !diff || !ws) return set_error(KFAC_ERR_ARG, "kfac_factor_diff: NULL argument");
    if (p->stale || p->g_only) return set_error(KFAC_ERR_STATE, "kfac_factor_diff: needs the full plan's recv chunks");
    if (rank < 0 || rank >= p->world) return set_error(KFAC_ERR_STATE, "kfac_factor_diff: rank out of range");
    const auto &ow = p->owned[rank];
    std::vector<DiffMat> mats;
    for (size_t k = 0; k < ow.size(); k++) {
        const Geom &g = p->geoms[ow[k]];
        for (int which = 0; which < 2; which++) {
            DiffMat m{};
            m.n = which == 0 ? g.dA : g.dG;
            m.cur = recv_cur + p->local[rank][k][1 + which];
            m.prev = recv_prev + p->local[rank][k][1 + which];
            m.out = diff + 2 * k + which;
            mats.push_back(m);
        }
    }
    if (mats.empty()) return KFAC_OK;
    return diff_launch(mats, static_cast<double *>(ws), p->ws_bytes, S(stream));
}

// ------------------------------------------------------------------ comm
kfac_status kfac_comm_unique_id(uint8_t id[128]) {
    if (!id) return set_error(KFAC_ERR_ARG, "kfac_comm_unique_id: NULL");
    static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId size");
    ncclUniqueId u;
    KFAC_NCCL_TRY(ncclGetUniqueId(&u));
    memcpy(id, &u, 128);
    return KFAC_OK;
}

kfac_status kfac_comm_create(const uint8_t id[128], int32_t rank, int32_t world, int32_t device, kfac_comm_t *out) {
    if (!id || !out || world < 1 || rank < 0 || rank >= world) return set_error(KFAC_ERR_ARG, "kfac_comm_create");
    KFAC_CUDA_TRY(cudaSetDevice(device));
    ncclUniqueId u;
    memcpy(&u, id, 128);
    kfac_comm *c = new kfac_comm();
    ncclResult_t r = ncclCommInitRank(&c->comm, world, u, rank);
    if (r != ncclSuccess) {
        delete c;
        return set_error(KFAC_ERR_NCCL, std::string("ncclCommInitRank: ") + ncclGetErrorString(r));
    }
    c->rank = rank;
    c->world = world;
    c->device = device;
    *out = c;
    return KFAC_OK;
}

void kfac_comm_destroy(kfac_comm_t c) {
    if (!c) return;
    if (c->comm) ncclCommDestroy(c->comm);
    delete c;
}

// ------------------------------------------------------------------ stage 3
// fp16 factor wire (NEXT-4(ii), R-23): pack -> NCCL (fp32 dW reduce, fp16 factor gather) -> unpack (wire.cu)
static kfac_status reduce_scatter_wire(kfac_comm_t c, kfac_plan_t p, const float *send, float *recv, void *ws,
                                       cudaStream_t st) {
    uint8_t *w = static_cast<uint8_t *>(ws);
    const int P = p->world, me = P == 1 ? 0 : c->rank;
    const int64_t c32 = p->wire_f32_chunk, c16 = p->wire_f16_chunk;
    float *s32 = reinterpret_cast<float *>(w + p->wire_off[0]);
    uint16_t *s16 = reinterpret_cast<uint16_t *>(w + p->wire_off[1]);
    float *r32 = P == 1 ? s32 : reinterpret_cast<float *>(w + p->wire_off[2]);
    uint16_t *r16 = reinterpret_cast<uint16_t *>(w + p->wire_off[3]);  // [P][c16]: the words from rank q at q * c16
    KFAC_TRY(wire_pack(p->wire_segs, send, p->rs_chunk, s32, c32, s16, c16, p->wire_scale[0], p->wire_scale[1], st));
    if (P > 1) {
        KFAC_NCCL_TRY(ncclGroupStart());
        ncclResult_t r = ncclSuccess;
        if (p->rs_mode == KFAC_RS_PER_OWNER) {
            for (int o = 0; o < P && r == ncclSuccess; o++)  // on an error, fall through to close the group
                if (p->wire_f32_used[o] > 0)
                    r = ncclReduce(s32 + (int64_t)o * c32, r32, (size_t)p->wire_f32_used[o], ncclFloat32, ncclAvg, o,
                                   c->comm, st);
        } else if (c32 > 0) {
            r = ncclReduceScatter(s32, r32, (size_t)c32, ncclFloat32, ncclAvg, c->comm, st);
        }
        for (int q = 0; q < P && r == ncclSuccess; q++) {  // gather: owner q's fp16 region of every rank to q
            if (q == me) continue;
            if (p->wire_f16_used[q] > 0) r = ncclSend(s16 + (int64_t)q * c16, (size_t)p->wire_f16_used[q], ncclFloat16, q, c->comm, st);
            if (r == ncclSuccess && p->wire_f16_used[me] > 0)
                r = ncclRecv(r16 + (int64_t)q * c16, (size_t)p->wire_f16_used[me], ncclFloat16, q, c->comm, st);
        }
        const ncclResult_t e = ncclGroupEnd();
        if (r != ncclSuccess) return set_error(KFAC_ERR_NCCL, std::string("wire collective: ") + ncclGetErrorString(r));
        if (e != ncclSuccess) return set_error(KFAC_ERR_NCCL, std::string("ncclGroupEnd: ") + ncclGetErrorString(e));
        KFAC_TRY(nccl_check_async(c->comm));
    }
    std::vector<const void *> src(P);
    for (int q = 0; q < P; q++) src[q] = q == me ? static_cast<const void *>(s16 + (int64_t)me * c16) : r16 + (int64_t)q * c16;
    const std::vector<WireSeg> mine(p->wire_segs.begin() + p->wire_seg_begin[me],
                                    p->wire_segs.begin() + p->wire_seg_begin[me + 1]);
    return wire_unpack(mine, r32, src.data(), P, recv, p->wire_scale[0], p->wire_scale[1], st);
}

kfac_status kfac_reduce_scatter_factors(kfac_comm_t c, kfac_plan_t p, const float *send, float *recv, void *stream) {
    return kfac_reduce_scatter_factors_ws(c, p, send, recv, nullptr, stream);
}

kfac_status kfac_reduce_scatter_factors_ws(kfac_comm_t c, kfac_plan_t p, const float *send, float *recv, void *ws,
                                           void *stream) {
    const NvtxRange nvtx_("kfac.reduce_scatter");
    if (!p || !send || !recv) return set_error(KFAC_ERR_ARG, "kfac_reduce_scatter_factors: NULL argument");
    if (p->world > 1 && (!c || c->world != p->world))
        return set_error(KFAC_ERR_STATE, "kfac_reduce_scatter_factors: comm/plan world mismatch");
    if (p->wire == KFAC_WIRE_FP16 && p->wire_f16_chunk > 0) {
        if (!ws) return set_error(KFAC_ERR_ARG, "kfac_reduce_scatter_factors: an fp16-wire plan needs ws (kfac_reduce_scatter_factors_ws)");
        return reduce_scatter_wire(c, p, send, recv, ws, S(stream));
    }
    if (p->world == 1) {
        if (send != recv)
            KFAC_CUDA_TRY(cudaMemcpyAsync(recv, send, p->rs_chunk * sizeof(float), cudaMemcpyDeviceToDevice, S(stream)));
        return KFAC_OK;
    }
    if (!c || c->world != p->world) return set_error(KFAC_ERR_STATE, "kfac_reduce_scatter_factors: comm/plan world mismatch");
    if (p->rs_mode == KFAC_RS_PER_OWNER) {
        // one ncclReduce(avg) per owner, rooted at it, over exactly its chunk's payload (no padding)
        KFAC_NCCL_TRY(ncclGroupStart());
        ncclResult_t r = ncclSuccess;
        for (int o = 0; o < p->world && r == ncclSuccess; o++)  // on an error, fall through to close the group
            if (p->rs_used[o] > 0)
                r = ncclReduce(send + (int64_t)o * p->rs_chunk, recv, (size_t)p->rs_used[o], ncclFloat32, ncclAvg, o, c->comm,
                               S(stream));
        const ncclResult_t e = ncclGroupEnd();
        if (r != ncclSuccess) return set_error(KFAC_ERR_NCCL, std::string("ncclReduce: ") + ncclGetErrorString(r));
        if (e != ncclSuccess) return set_error(KFAC_ERR_NCCL, std::string("ncclGroupEnd: ") + ncclGetErrorString(e));
    } else {
        KFAC_NCCL_TRY(ncclReduceScatter(send, recv, (size_t)p->rs_chunk, ncclFloat32, ncclAvg, c->comm, S(stream)));
    }
    KFAC_TRY(nccl_check_async(c->comm));
    return KFAC_OK;
}

// ------------------------------------------------------------------ stage 4
kfac_status kfac_damped_inverse(kfac_plan_t p, int32_t rank, const float *recv, float gamma, float *inv_ws,
                                int32_t *dev_status, float *pi_out, void *ws, void *stream) {
    const NvtxRange nvtx_("kfac.damped_inverse");
    if (!p || !recv || !inv_ws || !dev_status || !ws) return set_error(KFAC_ERR_ARG, "kfac_damped_inverse: NULL argument");
    if (p->stale) return set_error(KFAC_ERR_STATE, "kfac_damped_inverse: a stale plan carries no factors (reuse the cached inverses)");
    if (!(gamma > 0.f)) return set_error(KFAC_ERR_ARG, "kfac_damped_inverse: gamma must be > 0");
    if (rank < 0 || rank >= p->world) return set_error(KFAC_ERR_STATE, "kfac_damped_inverse: rank out of range");
    const auto &ow = p->owned[rank];
    uint8_t *w = static_cast<uint8_t *>(ws);
    double *pair_scratch = reinterpret_cast<double *>(w);
    int64_t sum_nt = 0, sum_tiles = 0, sum_tasks = 0;
    for (int l : ow)
        for (int n : {p->geoms[l].dA, p->geoms[l].dG}) {
            const int64_t nt = (n + kPanel - 1) / kPanel;
            sum_nt += nt;
            sum_tiles += nt * (nt + 1) / 2;
            sum_tasks += inverse_tasks(n);
        }
    int64_t off = align16(inverse_scratch_bytes((int)ow.size(), sum_nt, sum_tiles, sum_tasks));
    if (p->g_only && !pi_out)
        return set_error(KFAC_ERR_ARG, "kfac_damped_inverse: a G refresh reads the cached pi from pi_out");
    std::vector<InvMat> mats;
    for (size_t k = 0; k < ow.size(); k++) {
        const Geom &g = p->geoms[ow[k]];
        for (int which = p->g_only ? 1 : 0; which < 2; which++) {
            InvMat m{};
            m.n = which == 0 ? g.dA : g.dG;
            m.packed = recv + p->local[rank][k][1 + which];
            m.inv = inv_ws + p->inv_off[rank][2 * k + which];
            m.work = reinterpret_cast<double *>(w + off);
            const int64_t ld = (m.n + 15) / 16 * 16;
            m.panel = m.work + (int64_t)m.n * ld;
            off += inverse_ws_doubles(m.n) * 8;
            m.status = dev_status + 2 * k + which;
            m.split = inv_ws + p->split_off[rank][2 * k + which];  // the precondition's 3xTF32 operand, written here
            m.pair = (int)k;
            m.is_A = which == 0;
            mats.push_back(m);
        }
    }
    if (off > p->ws_bytes) return set_error(KFAC_ERR_STATE, "kfac_damped_inverse: workspace layout exceeds ws_bytes");
    return inverse_launch(mats, (int)ow.size(), gamma, pair_scratch, pi_out, p->g_only ? 1 : 0, p->inv_prec, S(stream));
}

kfac_status kfac_inverse_report(kfac_plan_t p, int32_t rank, const void *ws, double *bound, int32_t *slices, void *stream) {
    if (!p || !ws || !bound || !slices) return set_error(KFAC_ERR_ARG, "kfac_inverse_report: NULL argument");
    if (p->stale) return set_error(KFAC_ERR_STATE, "kfac_inverse_report: a stale plan runs no inverse");
    if (rank < 0 || rank >= p->world) return set_error(KFAC_ERR_STATE, "kfac_inverse_report: rank out of range");
    const size_t np = p->owned[rank].size();
    std::vector<double> h(8 * np);
    if (np) {
        KFAC_CUDA_TRY(cudaMemcpyAsync(h.data(), ws, h.size() * sizeof(double), cudaMemcpyDeviceToHost, S(stream)));
        KFAC_CUDA_TRY(cudaStreamSynchronize(S(stream)));
    }
    for (size_t k = 0; k < np; k++)
        for (int which = 0; which < 2; which++) {
            bound[2 * k + which] = h[8 * k + 3 + which];
            slices[2 * k + which] = (int32_t)h[8 * k + 5 + which];
        }
    return KFAC_OK;
}

// ------------------------------------------------------------------ stage 5
kfac_status kfac_precondition(kfac_plan_t p, int32_t rank, const float *recv, float *inv_ws, float *ag_buf,
                              void *ws, void *stream) {
    const NvtxRange nvtx_("kfac.precondition");
    if (!p || !recv || !inv_ws || !ag_buf || !ws) return set_error(KFAC_ERR_ARG, "kfac_precondition: NULL argument");
    if (rank < 0 || rank >= p->world) return set_error(KFAC_ERR_STATE, "kfac_precondition: rank out of range");
    const auto &ow = p->owned[rank];
    float *w = static_cast<float *>(ws);
    int64_t off = 0;
    std::vector<PrecJob> jobs;
    for (size_t k = 0; k < ow.size(); k++) {
        const int l = ow[k];
        const Geom &g = p->geoms[l];
        PrecJob j{};
        j.dG = g.dG;
        j.dA = g.dA;
        j.dW = recv + p->local[rank][k][0];
        j.Ainv = inv_ws + p->inv_off[rank][2 * k];
        j.Ginv = inv_ws + p->inv_off[rank][2 * k + 1];
        j.tmp = w + off;
        off += align16(precond_ws_floats(g.dG, g.dA));
        j.sA = inv_ws + p->split_off[rank][2 * k];
        j.sG = inv_ws + p->split_off[rank][2 * k + 1];
        j.resplit = 0;   // the inverses' tf32 hi / lo splits are written by kfac_damped_inverse (finalize_kernel)
        j.resplitG = 0;  // and cached in inv_ws for stale / G-refresh steps (R-20)
        if (p->owner[l] == rank) {
            j.out = ag_buf + p->ag_off[l];
        } else {
            j.out = w + off;
        }
        off += align16((int64_t)g.dG * g.dA);
        jobs.push_back(j);
    }
    if (off * 4 > p->ws_bytes) return set_error(KFAC_ERR_STATE, "kfac_precondition: workspace layout exceeds ws_bytes");
    return precond_launch(jobs, S(stream));
}

// ------------------------------------------------------------------ NEXT-3: the update after stage 6
kfac_status kfac_update(kfac_plan_t p, const float *ag_buf, float *const *w, float *const *w_prev, float lr,
                        float momentum, int32_t rescale, float eps, void *ws, void *stream) {
    const NvtxRange nvtx_("kfac.update");
    if (!p || !ag_buf || !w || !w_prev || !ws) return set_error(KFAC_ERR_ARG, "kfac_update: NULL argument");
    if (!(eps >= 0.f) || !std::isfinite(lr) || !std::isfinite(momentum))
        return set_error(KFAC_ERR_ARG, "kfac_update: lr, momentum finite and eps >= 0");
    std::vector<UpdJob> jobs;
    for (int l = 0; l < p->L; l++) {
        if (!w[l] || !w_prev[l]) return set_error(KFAC_ERR_ARG, "kfac_update: NULL layer pointer");
        const Geom &g = p->geoms[l];
        UpdJob u{};
        u.w = w[l];
        u.w_prev = w_prev[l];
        u.g = ag_buf + p->ag_off[l];
        u.dG = g.dG;
        u.dA = g.dA;
        u.bias = g.bias;
        jobs.push_back(u);
    }
    return update_launch(jobs, lr, momentum, rescale ? 1 : 0, eps, static_cast<double *>(ws), p->ws_bytes, S(stream));
}

// ------------------------------------------------------------------ NEXT-2: Batch Normalization Fisher
kfac_status kfac_bn_grads(int32_t nl, const int32_t *c, const int32_t *hw, const void *const *xhat,
                          const void *const *gy, kfac_dtype dt, int32_t n, float *const *Sv, void *stream) {
    const NvtxRange nvtx_("kfac.bn_grads");
    if (nl < 1 || !c || !hw || !xhat || !gy || !Sv) return set_error(KFAC_ERR_ARG, "kfac_bn_grads: NULL argument / nl < 1");
    if (n < 1) return set_error(KFAC_ERR_ARG, "kfac_bn_grads: n >= 1 (empty capture)");
    if (dt != KFAC_BF16 && dt != KFAC_FP16) return set_error(KFAC_ERR_ARG, "kfac_bn_grads: dtype");
    std::vector<BnJob> jobs;
    for (int l = 0; l < nl; l++) {
        if (!xhat[l] || !gy[l] || !Sv[l]) return set_error(KFAC_ERR_ARG, "kfac_bn_grads: NULL layer pointer");
        if (c[l] < 2 || hw[l] < 1) return set_error(KFAC_ERR_SHAPE, "kfac_bn_grads: c >= 2, hw >= 1");
        if ((c[l] & 1) || ((reinterpret_cast<uintptr_t>(xhat[l]) | reinterpret_cast<uintptr_t>(gy[l])) & 3))
            return set_error(KFAC_ERR_UNSUPPORTED, "kfac_bn_grads: c must be even and xhat / gy 4-byte aligned");
        BnJob b{};
        b.xhat = xhat[l];
        b.gy = gy[l];
        b.S = Sv[l];
        b.c = c[l];
        b.hw = hw[l];
        jobs.push_back(b);
    }
    return bn_grads_launch(jobs, n, dt == KFAC_FP16 ? 1 : 0, S(stream));
}

kfac_status kfac_bn_exchange(kfac_comm_t cm, int32_t nl, const int32_t *c, int32_t n_local, const float *const *S_local,
                             float *const *S_all, float *const *grad, void *stream) {
    const NvtxRange nvtx_("kfac.bn_exchange");
    if (!cm || nl < 1 || !c || !S_local || !S_all || !grad || n_local < 1)
        return set_error(KFAC_ERR_ARG, "kfac_bn_exchange: NULL argument / nl, n_local < 1");
    for (int l = 0; l < nl; l++)
        if (!S_local[l] || !S_all[l] || !grad[l] || c[l] < 1) return set_error(KFAC_ERR_ARG, "kfac_bn_exchange: layer argument");
    KFAC_NCCL_TRY(ncclGroupStart());
    ncclResult_t r = ncclSuccess;
    const char *what = "";
    for (int l = 0; l < nl && r == ncclSuccess; l++) {  // on an error, fall through to close the group
        const size_t cnt = (size_t)n_local * 2 * c[l];
        r = ncclAllGather(S_local[l], S_all[l], cnt, ncclFloat32, cm->comm, S(stream));
        what = "ncclAllGather";
        if (r == ncclSuccess) {
            r = ncclAllReduce(grad[l], grad[l], (size_t)2 * c[l], ncclFloat32, ncclAvg, cm->comm, S(stream));
            what = "ncclAllReduce";
        }
    }
    const ncclResult_t e = ncclGroupEnd();
    if (r != ncclSuccess) return set_error(KFAC_ERR_NCCL, std::string(what) + ": " + ncclGetErrorString(r));
    if (e != ncclSuccess) return set_error(KFAC_ERR_NCCL, std::string("ncclGroupEnd: ") + ncclGetErrorString(e));
    KFAC_TRY(nccl_check_async(cm->comm));
    return KFAC_OK;
}

kfac_status kfac_bn_ws_bytes(int32_t nl, const int32_t *c, int32_t n, int64_t *bytes) {
    if (nl < 1 || !c || !bytes || n < 1) return set_error(KFAC_ERR_ARG, "kfac_bn_ws_bytes");
    *bytes = bn_ws_bytes(std::vector<int>(c, c + nl), n);
    return KFAC_OK;
}

kfac_status kfac_bn_precondition(int32_t nl, const int32_t *c, int32_t n, const float *const *Sv,
                                 const float *const *grad, float gamma_bn, int32_t full, float *const *out,
                                 void *ws, int64_t ws_bytes, void *stream) {
    const NvtxRange nvtx_("kfac.bn_precondition");
    if (nl < 1 || !c || !Sv || !grad || !out) return set_error(KFAC_ERR_ARG, "kfac_bn_precondition: NULL argument / nl < 1");
    if (!(gamma_bn > 0.f)) return set_error(KFAC_ERR_ARG, "kfac_bn_precondition: gamma_bn must be > 0");
    if (n < 1) return set_error(KFAC_ERR_ARG, "kfac_bn_precondition: n >= 1");
    if (full && n > kBnMaxSamples)
        return set_error(KFAC_ERR_UNSUPPORTED, "kfac_bn_precondition: full mode supports n <= 256 samples");
    std::vector<BnJob> jobs;
    for (int l = 0; l < nl; l++) {
        if (!Sv[l] || !grad[l] || !out[l]) return set_error(KFAC_ERR_ARG, "kfac_bn_precondition: NULL layer pointer");
        if (c[l] < 1) return set_error(KFAC_ERR_SHAPE, "kfac_bn_precondition: c >= 1");
        BnJob b{};
        b.S = const_cast<float *>(Sv[l]);
        b.grad = grad[l];
        b.out = out[l];
        b.c = c[l];
        jobs.push_back(b);
    }
    return bn_precond_launch(jobs, n, full ? 1 : 0, (double)gamma_bn, static_cast<double *>(ws), ws_bytes, S(stream));
}

// ------------------------------------------------------------------ stage 6
kfac_status kfac_allgather_precond(kfac_comm_t c, kfac_plan_t p, float *ag_buf, void *stream) {
    const NvtxRange nvtx_("kfac.allgather");
    if (!p || !ag_buf) return set_error(KFAC_ERR_ARG, "kfac_allgather_precond: NULL argument");
    if (p->world == 1) return KFAC_OK;
    if (!c || c->world != p->world) return set_error(KFAC_ERR_STATE, "kfac_allgather_precond: comm/plan world mismatch");
    float *mine = ag_buf + (int64_t)c->rank * p->ag_chunk;
    KFAC_NCCL_TRY(ncclAllGather(mine, ag_buf, (size_t)p->ag_chunk, ncclFloat32, c->comm, S(stream)));
    KFAC_TRY(nccl_check_async(c->comm));
    return KFAC_OK;
}

}  // extern "C"
