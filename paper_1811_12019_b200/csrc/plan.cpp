// plan.cpp -- stage a0 of the K-FAC hot path: layer ownership and the
// owner-major wire layout of the ReduceScatterV / AllGatherV buffers
// ("multiple layers are handled by each GPU ...
// some layers will be calculated redundantly"; readings R-15, R-16).
// Host-only C++; the oracle carries its own independent implementation and
// tests/test_abi.py (test_plan_bit_exact_vs_oracle) compares the two bit-exactly.
#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstring>
#include <numeric>
#include <string>

#include <map>
#include <mutex>
#include <set>

#include "kfac_plan.hpp"

namespace kfac {

thread_local std::string g_last_error;
std::atomic<int64_t> g_launches{0};

kfac_status set_error(kfac_status st, const std::string &msg) {
    g_last_error = msg;
    return st;
}

// ---- per-device launch setup (the SM count and the shared memory opt-in are per device)
static std::mutex g_dev_mu;
static std::map<int, int> g_dev_sms;
static std::set<std::pair<int, const void *>> g_dev_attr;

kfac_status dev_sm_count(int *sms) {
    int dev = 0;
    KFAC_CUDA_TRY(cudaGetDevice(&dev));
    std::lock_guard<std::mutex> lock(g_dev_mu);
    auto it = g_dev_sms.find(dev);
    if (it == g_dev_sms.end()) {
        int v = 0;
        KFAC_CUDA_TRY(cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev));
        it = g_dev_sms.emplace(dev, v).first;
    }
    *sms = it->second;
    return KFAC_OK;
}

kfac_status dev_func_smem(const void *func, int bytes) {
    int dev = 0;
    KFAC_CUDA_TRY(cudaGetDevice(&dev));
    std::lock_guard<std::mutex> lock(g_dev_mu);
    if (g_dev_attr.count({dev, func})) return KFAC_OK;
    KFAC_CUDA_TRY(cudaFuncSetAttribute(func, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes));
    g_dev_attr.insert({dev, func});
    return KFAC_OK;
}

kfac_status make_geom(const kfac_layer_desc &d, Geom *g) {
    if (d.kind != 0 && d.kind != 1) return set_error(KFAC_ERR_SHAPE, "layer kind must be 0 (conv2d) or 1 (linear)");
    if (d.c_in < 1 || d.c_out < 1) return set_error(KFAC_ERR_SHAPE, "c_in, c_out must be >= 1");
    g->kind = d.kind;
    g->c_in = d.c_in;
    g->c_out = d.c_out;
    g->bias = d.has_bias ? 1 : 0;
    if (d.kind == 1) {
        g->kh = g->kw = g->sh = g->sw = 1;
        g->ph = g->pw = 0;
        g->h = g->w = g->ho = g->wo = 1;
    } else {
        if (d.kh < 1 || d.kw < 1 || d.stride_h < 1 || d.stride_w < 1 || d.pad_h < 0 || d.pad_w < 0 || d.h_in < 1 ||
            d.w_in < 1)
            return set_error(KFAC_ERR_SHAPE, "invalid conv2d geometry");
        g->kh = d.kh;
        g->kw = d.kw;
        g->sh = d.stride_h;
        g->sw = d.stride_w;
        g->ph = d.pad_h;
        g->pw = d.pad_w;
        g->h = d.h_in;
        g->w = d.w_in;
        g->ho = (d.h_in + 2 * d.pad_h - d.kh) / d.stride_h + 1;
        g->wo = (d.w_in + 2 * d.pad_w - d.kw) / d.stride_w + 1;
        if (g->ho < 1 || g->wo < 1) return set_error(KFAC_ERR_SHAPE, "empty conv2d output");
    }
    g->dF = g->c_in * g->kh * g->kw;
    g->dA = g->dF + g->bias;
    g->dG = g->c_out;
    return KFAC_OK;
}

static int64_t stage45_cost(const Geom &g) {
    const int64_t a = g.dA, b = g.dG;
    return a * a * a + b * b * b + 2 * b * b * a + 2 * b * a * a;
}

kfac_status plan_build(kfac_plan *p) {
    const int L = p->L, P = p->world;
    p->geoms.resize(L);
    for (int l = 0; l < L; l++) {
        kfac_status s = make_geom(p->layers[l], &p->geoms[l]);
        if (s) return s;
        if (p->geoms[l].dA > kMaxInverseDim || p->geoms[l].dG > kMaxInverseDim)
            return set_error(KFAC_ERR_UNSUPPORTED, "layer " + std::to_string(l) + ": a factor dimension exceeds " +
                                                       std::to_string(kMaxInverseDim) + " (inverse limit)");
    }
    // ownership
    p->owner.assign(L, 0);
    if (p->policy == KFAC_OWN_ROUND_ROBIN) {
        for (int l = 0; l < L; l++) p->owner[l] = l % P;
    } else {
        std::vector<int> order(L);
        std::iota(order.begin(), order.end(), 0);
        std::vector<int64_t> cost(L);
        for (int l = 0; l < L; l++) cost[l] = stage45_cost(p->geoms[l]);
        std::sort(order.begin(), order.end(), [&](int a, int b) {
            if (cost[a] != cost[b]) return cost[a] > cost[b];
            return a < b;
        });
        std::vector<int64_t> load(P, 0);
        for (int l : order) {
            int best = 0;
            for (int r = 1; r < P; r++)
                if (load[r] < load[best]) best = r;
            p->owner[l] = best;
            load[best] += cost[l];
        }
    }
    // owned lists (primary + the cyclic redundant copy when P > L)
    p->owned.assign(P, {});
    for (int r = 0; r < P; r++) {
        std::vector<int> v;
        for (int l = 0; l < L; l++)
            if (p->owner[l] == r) v.push_back(l);
        if (r >= L) {
            int extra = r % L;
            if (std::find(v.begin(), v.end(), extra) == v.end()) v.push_back(extra);
        }
        std::sort(v.begin(), v.end());
        p->owned[r] = v;
    }
    // RS layout
    p->local.assign(P, {});
    p->rs_used.assign(P, 0);
    int64_t maxc = 0;
    for (int r = 0; r < P; r++) {
        int64_t off = 0;
        for (int l : p->owned[r]) {
            const Geom &g = p->geoms[l];
            std::array<int64_t, 3> o;
            o[0] = off;
            off = align16(off + (int64_t)g.dG * g.dA);
            if (p->stale) {  // stale step: the owner reuses its cached inverses, only dW travels
                o[1] = o[2] = -1;
                p->local[r].push_back(o);
                continue;
            }
            if (p->g_only) {  // G refresh: A's cached inverse is reused, dW and G travel
                o[1] = -1;
                o[2] = off;
                off = align16(off + packed_len(g.dG));
                p->local[r].push_back(o);
                continue;
            }
            o[1] = off;
            off = align16(off + packed_len(g.dA));
            o[2] = off;
            off = align16(off + packed_len(g.dG));
            p->local[r].push_back(o);
        }
        maxc = std::max(maxc, off);
        p->rs_used[r] = off;
    }
    p->rs_chunk = maxc;
    p->seg_off.assign(3 * (size_t)L, 0);
    for (int l = 0; l < L; l++) {
        const int r = p->owner[l];
        const auto &ow = p->owned[r];
        const size_t k = std::find(ow.begin(), ow.end(), l) - ow.begin();
        for (int s = 0; s < 3; s++)
            p->seg_off[3 * l + s] = p->local[r][k][s] < 0 ? -1 : (int64_t)r * p->rs_chunk + p->local[r][k][s];
    }
    // AG layout (primary copies only)
    std::vector<int64_t> agl(L, 0);
    int64_t maxa = 0;
    for (int r = 0; r < P; r++) {
        int64_t off = 0;
        for (int l = 0; l < L; l++) {
            if (p->owner[l] != r) continue;
            agl[l] = off;
            off = align16(off + (int64_t)p->geoms[l].dG * p->geoms[l].dA);
        }
        maxa = std::max(maxa, off);
    }
    p->ag_chunk = maxa;
    p->ag_off.assign(L, 0);
    for (int l = 0; l < L; l++) p->ag_off[l] = (int64_t)p->owner[l] * p->ag_chunk + agl[l];
    // per-rank inverse layout and stage workspaces
    p->inv_off.assign(P, {});
    p->split_off.assign(P, {});
    p->inv_floats.assign(P, 0);
    int64_t ws = 0;
    for (int r = 0; r < P; r++) {
        int64_t off = 0, inv_ws = 0, prec_ws = 0, sum_nt = 0, sum_tiles = 0, sum_tasks = 0;
        for (int l : p->owned[r]) {
            const Geom &g = p->geoms[l];
            p->inv_off[r].push_back(off);
            off = align16(off + (int64_t)g.dA * g.dA);
            p->inv_off[r].push_back(off);
            off = align16(off + (int64_t)g.dG * g.dG);
            for (int n : {g.dA, g.dG}) {
                const int64_t nt = (n + kPanel - 1) / kPanel;
                inv_ws += inverse_ws_doubles(n) * 8;
                sum_nt += nt;
                sum_tiles += nt * (nt + 1) / 2;
                sum_tasks += inverse_tasks(n);
            }
            prec_ws += (align16(precond_ws_floats(g.dG, g.dA)) + align16((int64_t)g.dG * g.dA)) * 4;  // split operands + (redundant) output
        }
        // the inverses' 3xTF32 hi / lo split, written by a full step's precondition and reused by stale steps
        for (int l : p->owned[r]) {
            const Geom &g = p->geoms[l];
            p->split_off[r].push_back(off);
            off = align16(off + precond_split_floats(g.dA));
            p->split_off[r].push_back(off);
            off = align16(off + precond_split_floats(g.dG));
        }
        p->inv_floats[r] = off;
        inv_ws += align16(inverse_scratch_bytes((int)p->owned[r].size(), sum_nt, sum_tiles, sum_tasks));  // pair scratch, counters, flags
        ws = std::max(ws, std::max(inv_ws, prec_ws));
    }
    // factor stage: split-K partials of the grouped launch (same planner as the kernel)
    std::vector<FactorJob> jobs;
    for (int l = 0; l < L; l++) {
        FactorJob a{};
        a.g = p->geoms[l];
        a.is_A = true;
        a.n = p->n_local;
        jobs.push_back(a);
        FactorJob b = a;
        b.is_A = false;
        jobs.push_back(b);
    }
    FactorLaunch fl;
    kfac_status s = factor_prepare(jobs, KFAC_BF16, nullptr, 0, true, &fl);
    if (s) return s;
    p->factor_ws = fl.ws_bytes;
    ws = std::max(ws, fl.ws_bytes);
    p->ws_base = align16(ws) + 256;
    wire_build(p);
    return KFAC_OK;
}

void wire_build(kfac_plan *p) {
    const int P = p->world;
    p->wire_segs.clear();
    p->wire_seg_begin.assign(P + 1, 0);
    p->wire_f32_used.assign(P, 0);
    p->wire_f16_used.assign(P, 0);
    p->wire_f32_chunk = p->wire_f16_chunk = 0;
    p->ws_bytes = p->ws_base;
    if (p->wire != KFAC_WIRE_FP16) return;
    for (int r = 0; r < P; r++) {
        p->wire_seg_begin[r] = (int32_t)p->wire_segs.size();
        int64_t o32 = 0, o16 = 0;
        for (size_t k = 0; k < p->owned[r].size(); k++) {
            const Geom &g = p->geoms[p->owned[r][k]];
            const auto &loc = p->local[r][k];
            p->wire_segs.push_back(WireSeg{loc[0], o32, (int64_t)g.dG * g.dA, 0, r});
            o32 = align16(o32 + (int64_t)g.dG * g.dA);
            for (int which = 0; which < 2; which++) {
                if (loc[1 + which] < 0) continue;  // stale / G-refresh layouts
                const int64_t len = packed_len(which == 0 ? g.dA : g.dG);
                p->wire_segs.push_back(WireSeg{loc[1 + which], o16, len, 1 + which, r});
                o16 = align16(o16 + len);
            }
        }
        p->wire_f32_used[r] = o32;
        p->wire_f16_used[r] = o16;
        p->wire_f32_chunk = std::max(p->wire_f32_chunk, o32);
        p->wire_f16_chunk = std::max(p->wire_f16_chunk, o16);
    }
    p->wire_seg_begin[P] = (int32_t)p->wire_segs.size();
    auto a256 = [](int64_t v) { return (v + 255) / 256 * 256; };
    int64_t off = 0;
    p->wire_off[0] = off;
    off = a256(off + (int64_t)P * p->wire_f32_chunk * 4);
    p->wire_off[1] = off;
    off = a256(off + (int64_t)P * p->wire_f16_chunk * 2);
    p->wire_off[2] = off;
    off = a256(off + p->wire_f32_chunk * 4);
    p->wire_off[3] = off;  // the fp16 factor regions gathered from every rank
    off = a256(off + (int64_t)P * p->wire_f16_chunk * 2);
    if (p->wire_f16_chunk > 0) p->ws_bytes = std::max(p->ws_base, off + 256);
}

}  // namespace kfac

using namespace kfac;

extern "C" {

const char *kfac_last_error(void) { return g_last_error.c_str(); }
const char *kfac_version(void) { return "kfac-b200 0.1 sm_100a"; }
int64_t kfac_launch_count(void) { return g_launches.load(); }

kfac_status kfac_plan_create(const kfac_layer_desc *layers, int32_t L, int32_t world, int32_t n_local,
                             kfac_policy policy, kfac_plan_t *out) {
    if (!layers || !out) return set_error(KFAC_ERR_ARG, "kfac_plan_create: NULL argument");
    if (L < 1 || world < 1 || n_local < 1) return set_error(KFAC_ERR_ARG, "kfac_plan_create: L, world, n_local >= 1");
    if (policy != KFAC_OWN_ROUND_ROBIN && policy != KFAC_OWN_LPT)
        return set_error(KFAC_ERR_ARG, "kfac_plan_create: unknown policy");
    kfac_plan *p = new kfac_plan();
    p->layers.assign(layers, layers + L);
    p->L = L;
    p->world = world;
    p->n_local = n_local;
    p->policy = policy;
    kfac_status s = plan_build(p);
    if (s) {
        delete p;
        return s;
    }
    *out = p;
    return KFAC_OK;
}

kfac_status kfac_plan_create_stale(kfac_plan_t full, kfac_plan_t *out) {
    if (!full || !out) return set_error(KFAC_ERR_ARG, "kfac_plan_create_stale: NULL argument");
    if (full->stale || full->g_only) return set_error(KFAC_ERR_STATE, "kfac_plan_create_stale: plan is not a full plan");
    kfac_plan *p = new kfac_plan();
    p->layers = full->layers;
    p->L = full->L;
    p->world = full->world;
    p->n_local = full->n_local;
    p->policy = full->policy;
    p->rs_mode = full->rs_mode;
    p->inv_prec = full->inv_prec;
    p->wire = full->wire;
    p->wire_scale[0] = full->wire_scale[0];
    p->wire_scale[1] = full->wire_scale[1];
    p->stale = true;
    kfac_status s = plan_build(p);
    if (s) {
        delete p;
        return s;
    }
    *out = p;
    return KFAC_OK;
}

int32_t kfac_plan_is_stale(kfac_plan_t p) { return p && p->stale ? 1 : 0; }

kfac_status kfac_plan_create_grefresh(kfac_plan_t full, kfac_plan_t *out) {
    if (!full || !out) return set_error(KFAC_ERR_ARG, "kfac_plan_create_grefresh: NULL argument");
    if (full->stale || full->g_only) return set_error(KFAC_ERR_STATE, "kfac_plan_create_grefresh: plan is not a full plan");
    kfac_plan *p = new kfac_plan();
    p->layers = full->layers;
    p->L = full->L;
    p->world = full->world;
    p->n_local = full->n_local;
    p->policy = full->policy;
    p->rs_mode = full->rs_mode;
    p->inv_prec = full->inv_prec;
    p->wire = full->wire;
    p->wire_scale[0] = full->wire_scale[0];
    p->wire_scale[1] = full->wire_scale[1];
    p->g_only = true;
    kfac_status s = plan_build(p);
    if (s) {
        delete p;
        return s;
    }
    *out = p;
    return KFAC_OK;
}

kfac_status kfac_plan_set_rs_mode(kfac_plan_t p, int32_t mode) {
    if (!p) return set_error(KFAC_ERR_ARG, "kfac_plan_set_rs_mode: NULL plan");
    if (mode != KFAC_RS_PADDED && mode != KFAC_RS_PER_OWNER) return set_error(KFAC_ERR_ARG, "kfac_plan_set_rs_mode: bad mode");
    p->rs_mode = mode;
    return KFAC_OK;
}

kfac_status kfac_plan_set_wire(kfac_plan_t p, int32_t wire, float scale_A, float scale_G) {
    if (!p) return set_error(KFAC_ERR_ARG, "kfac_plan_set_wire: NULL plan");
    if (wire != KFAC_WIRE_FP32 && wire != KFAC_WIRE_FP16) return set_error(KFAC_ERR_ARG, "kfac_plan_set_wire: bad wire");
    if (wire == KFAC_WIRE_FP16 && p->world > 16) return set_error(KFAC_ERR_UNSUPPORTED, "kfac_plan_set_wire: fp16 wire up to 16 ranks");
    for (float s : {scale_A, scale_G}) {
        int e = 0;
        if (!(s > 0.f) || !std::isfinite(s) || std::frexp(s, &e) != 0.5f || e < -60 || e > 60)
            return set_error(KFAC_ERR_ARG, "kfac_plan_set_wire: scales must be powers of two in [2^-61, 2^59]");
    }
    p->wire = wire;
    p->wire_scale[0] = scale_A;
    p->wire_scale[1] = scale_G;
    wire_build(p);
    return KFAC_OK;
}

kfac_status kfac_plan_set_inverse_precision(kfac_plan_t p, int32_t mode) {
    if (!p) return set_error(KFAC_ERR_ARG, "kfac_plan_set_inverse_precision: NULL plan");
    if (mode < KFAC_INV_AUTO || mode > KFAC_INV_INT8) return set_error(KFAC_ERR_ARG, "kfac_plan_set_inverse_precision: bad mode");
    p->inv_prec = mode;
    return KFAC_OK;
}

int32_t kfac_plan_refresh_kind(kfac_plan_t p) { return !p ? -1 : p->stale ? 2 : p->g_only ? 1 : 0; }

int32_t kfac_refresh_interval(int32_t schedule, int32_t epoch) {
    if (epoch < 0) return -1;
    if (schedule == KFAC_REFRESH_RAMPUP) return std::min(20, 5 * (epoch / 5) + 1);
    if (schedule == KFAC_REFRESH_STEP13) return epoch < 13 ? 1 : 20;
    return -1;
}

int32_t kfac_refresh(int64_t t, int32_t epoch, int32_t schedule, int64_t fresh_floor, int32_t interval) {
    const int32_t iv = interval > 0 ? interval : kfac_refresh_interval(schedule, epoch);
    if (iv < 1 || t < 0) return -1;
    return (t < fresh_floor || t % iv == 0) ? 1 : 0;
}

kfac_status kfac_plan_query(kfac_plan_t p, int32_t *owner, int64_t *seg_off, int64_t *rs_chunk, int64_t *ag_off,
                            int64_t *ag_chunk, int64_t *ws_bytes) {
    if (!p) return set_error(KFAC_ERR_ARG, "kfac_plan_query: NULL plan");
    if (owner) std::copy(p->owner.begin(), p->owner.end(), owner);
    if (seg_off) std::copy(p->seg_off.begin(), p->seg_off.end(), seg_off);
    if (rs_chunk) *rs_chunk = p->rs_chunk;
    if (ag_off) std::copy(p->ag_off.begin(), p->ag_off.end(), ag_off);
    if (ag_chunk) *ag_chunk = p->ag_chunk;
    if (ws_bytes) *ws_bytes = p->ws_bytes;
    return KFAC_OK;
}

kfac_status kfac_plan_rank_layers(kfac_plan_t p, int32_t rank, int32_t *n_owned, int32_t *layers, int64_t *local_off,
                                  int64_t *inv_off, int64_t *inv_floats) {
    if (!p) return set_error(KFAC_ERR_ARG, "kfac_plan_rank_layers: NULL plan");
    if (rank < 0 || rank >= p->world) return set_error(KFAC_ERR_ARG, "kfac_plan_rank_layers: rank out of range");
    const auto &ow = p->owned[rank];
    if (n_owned) *n_owned = (int32_t)ow.size();
    for (size_t k = 0; k < ow.size(); k++) {
        if (layers) layers[k] = ow[k];
        if (local_off)
            for (int s = 0; s < 3; s++) local_off[3 * k + s] = p->local[rank][k][s];
        if (inv_off) {
            inv_off[2 * k] = p->inv_off[rank][2 * k];
            inv_off[2 * k + 1] = p->inv_off[rank][2 * k + 1];
        }
    }
    if (inv_floats) *inv_floats = p->inv_floats[rank];
    return KFAC_OK;
}

void kfac_plan_destroy(kfac_plan_t p) { delete p; }

}  // extern "C"
