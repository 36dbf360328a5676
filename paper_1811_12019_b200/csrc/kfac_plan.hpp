// kfac_plan.hpp -- the opaque plan / communicator objects behind the C-ABI.
#pragma once
#include <array>
#include <mutex>
#include <vector>

#include "kfac_internal.hpp"

struct kfac_plan {
    std::vector<kfac_layer_desc> layers;
    std::vector<kfac::Geom> geoms;
    int L = 0, world = 1, n_local = 1;
    kfac_policy policy = KFAC_OWN_ROUND_ROBIN;
    bool stale = false;   // stale-factor wire layout: dW segments only (R-20)
    bool g_only = false;  // G-refresh layout: dW and G segments (A kept stale, R-20)
    int inv_prec = KFAC_INV_AUTO;  // kfac_plan_set_inverse_precision
    int rs_mode = KFAC_RS_PADDED;  // kfac_plan_set_rs_mode
    std::vector<int64_t> rs_used;  // per rank: floats of its chunk the layout uses (<= rs_chunk)
    // fp16 factor wire (kfac_plan_set_wire; wire.cu): per owner a fp32 dW region and a fp16 factor region
    int wire = KFAC_WIRE_FP32;
    float wire_scale[2] = {1.f, 1.f};              // A, G (powers of two)
    std::vector<kfac::WireSeg> wire_segs;          // owner-major
    std::vector<int32_t> wire_seg_begin;           // per owner: first segment (world + 1 entries)
    std::vector<int64_t> wire_f32_used, wire_f16_used;  // per owner: elements of its regions in use
    int64_t wire_f32_chunk = 0, wire_f16_chunk = 0;     // region sizes per owner (max over owners)
    int64_t wire_off[4] = {0, 0, 0, 0};            // ws byte offsets: send fp32, send fp16, recv fp32, recv fp16
    int64_t ws_base = 0;                           // ws_bytes without the wire staging
    std::vector<int32_t> owner;
    std::vector<std::vector<int>> owned;                          // per rank, ascending
    std::vector<std::vector<std::array<int64_t, 3>>> local;       // per rank, per owned layer
    std::vector<int64_t> seg_off, ag_off;
    int64_t rs_chunk = 0, ag_chunk = 0, ws_bytes = 0, factor_ws = 0;
    std::vector<std::vector<int64_t>> inv_off;  // per rank: 2 per owned layer
    std::vector<std::vector<int64_t>> split_off;  // per rank: 2 per owned layer (3xTF32 split cache, after the inverses)
    std::vector<int64_t> inv_floats;
    // cached grouped factor launch (re-encoded when the pointers change); c_mu serialises
    // concurrent kfac_factor_all calls on one plan (the ABI allows calls from several threads)
    std::mutex c_mu;
    std::vector<const void *> c_xs, c_gys;
    std::vector<float> c_aA, c_aG;
    float *c_send = nullptr;
    void *c_ws = nullptr;
    int c_dt = -1;
    kfac::FactorLaunch c_fl;
    std::vector<kfac::FactorJob> c_jobs;
};

namespace kfac {
kfac_status plan_build(kfac_plan *p);
void wire_build(kfac_plan *p);  // the fp16 wire layout + staging (called by plan_build and kfac_plan_set_wire)
}
