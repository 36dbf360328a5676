// wire.cu -- the fp16 factor wire of the ReduceScatterV (NEXT-4(ii); "half precision
// floating point numbers for both computation [and communication]"; reading R-23).
//
// With a KFAC_WIRE_FP16 plan the owner-major fp32 send buffer is re-laid for the wire before the
// collective and back after it:
//
//   pack    rs_send (fp32, every owner's chunk) -> staging: per owner a dW region (fp32, copied) and a
//           factor region (the packed A / G segments as binary16 of x * scale, round to nearest even);
//   NCCL    Reduce(avg) per owner (or one ReduceScatter) of the fp32 dW regions; the fp16 factor
//           regions are GATHERED to their owner (grouped ncclSend / ncclRecv: the same bytes per rank
//           as a ring ReduceScatter, (P - 1) / P of the payload, but no fp16 arithmetic in flight);
//   unpack  the owner's regions -> rs_recv at the plan's offsets: dW copied, each factor element the
//           mean of its P fp16 wire words, summed in fp32 in rank order, / P, * 1/scale.
//
// Both passes are HBM-bound streaming copies: 4 B read + 2 B written per factor element (pack),
// 2P B + 4 B (unpack), 4 + 4 B per dW element.  Segments start on 16-element boundaries, so every
// thread moves 4 elements per access (16 B fp32 / 8 B fp16); only a segment's last group is ragged.
#include <cuda_fp16.h>

#include "kfac_internal.hpp"

namespace kfac {

namespace {

constexpr int kWireThreads = 256;
constexpr int64_t kWireTile = 4096;  // elements per tile (16 per thread)
constexpr int kWireMaxSegs = 240;

constexpr int kWirePeers = 16;  // ranks of an fp16 wire (the unpack sums one fp16 word per rank)

struct WireParams {
    const float *src_f32;    // pack: rs_send; unpack: received fp32 region
    const __half *src_f16[kWirePeers];  // unpack: the fp16 factor region received from each rank
    float *dst_f32;          // pack: fp32 send region; unpack: rs_recv
    __half *dst_f16;         // pack: fp16 send region
    int64_t send_stride;     // pack: floats per owner chunk of rs_send (rs_chunk)
    int64_t f32_stride;      // pack: elements per owner in the fp32 region
    int64_t f16_stride;      // pack: elements per owner in the fp16 region
    float scale[3];          // per kind: 1 (dW), scale_A, scale_G  (unpack: the reciprocals)
    int32_t nsegs, unpack, npeers;
    int32_t tile_begin[kWireMaxSegs + 1];
    WireSeg segs[kWireMaxSegs];
};

__device__ __forceinline__ void pack_group(const WireParams &P, const WireSeg &s, int64_t i, int64_t n) {
    const float *src = P.src_f32 + (int64_t)s.owner * P.send_stride + s.src + i;
    if (s.kind == 0) {
        float *dst = P.dst_f32 + (int64_t)s.owner * P.f32_stride + s.dst + i;
        if (n == 4) {
            *reinterpret_cast<float4 *>(dst) = __ldcs(reinterpret_cast<const float4 *>(src));
        } else {
            for (int j = 0; j < n; j++) dst[j] = src[j];
        }
        return;
    }
    const float sc = P.scale[s.kind];
    __half *dst = P.dst_f16 + (int64_t)s.owner * P.f16_stride + s.dst + i;
    if (n == 4) {
        const float4 v = __ldcs(reinterpret_cast<const float4 *>(src));
        __half2 lo = __floats2half2_rn(v.x * sc, v.y * sc), hi = __floats2half2_rn(v.z * sc, v.w * sc);
        uint2 u;
        u.x = *reinterpret_cast<uint32_t *>(&lo);
        u.y = *reinterpret_cast<uint32_t *>(&hi);
        *reinterpret_cast<uint2 *>(dst) = u;
    } else {
        for (int j = 0; j < n; j++) dst[j] = __float2half_rn(src[j] * sc);
    }
}

__device__ __forceinline__ void unpack_group(const WireParams &P, const WireSeg &s, int64_t i, int64_t n) {
    float *dst = P.dst_f32 + s.src + i;
    if (s.kind == 0) {
        const float *src = P.src_f32 + s.dst + i;
        if (n == 4) {
            *reinterpret_cast<float4 *>(dst) = *reinterpret_cast<const float4 *>(src);
        } else {
            for (int j = 0; j < n; j++) dst[j] = src[j];
        }
        return;
    }
    // the mean of the P wire words: fp32 sum in rank order (exact while the P values span < 2^13 in
    // magnitude), one division by P, then the exact power-of-two unscaling
    const float inv = P.scale[s.kind], np = (float)P.npeers;
    if (n == 4) {
        float4 a = make_float4(0.f, 0.f, 0.f, 0.f);
        for (int q = 0; q < P.npeers; q++) {
            const uint2 u = __ldcs(reinterpret_cast<const uint2 *>(P.src_f16[q] + s.dst + i));
            const float2 lo = __half22float2(*reinterpret_cast<const __half2 *>(&u.x));
            const float2 hi = __half22float2(*reinterpret_cast<const __half2 *>(&u.y));
            a.x += lo.x;
            a.y += lo.y;
            a.z += hi.x;
            a.w += hi.y;
        }
        *reinterpret_cast<float4 *>(dst) = make_float4(__fdiv_rn(a.x, np) * inv, __fdiv_rn(a.y, np) * inv,
                                                       __fdiv_rn(a.z, np) * inv, __fdiv_rn(a.w, np) * inv);
    } else {
        for (int j = 0; j < n; j++) {
            float a = 0.f;
            for (int q = 0; q < P.npeers; q++) a += __half2float(P.src_f16[q][s.dst + i + j]);
            dst[j] = __fdiv_rn(a, np) * inv;
        }
    }
}

__global__ void __launch_bounds__(kWireThreads) wire_kernel(const __grid_constant__ WireParams P) {
    const int total = P.tile_begin[P.nsegs];
    for (int t = blockIdx.x; t < total; t += gridDim.x) {
        int lo = 0, hi = P.nsegs - 1;  // the last segment whose first tile <= t
        while (lo < hi) {
            const int mid = (lo + hi + 1) >> 1;
            if (P.tile_begin[mid] <= t) lo = mid;
            else hi = mid - 1;
        }
        const WireSeg &s = P.segs[lo];
        const int64_t base = (int64_t)(t - P.tile_begin[lo]) * kWireTile;
        const int64_t end = min(s.len, base + kWireTile);
        for (int64_t i = base + 4 * (int64_t)threadIdx.x; i < end; i += 4 * kWireThreads) {
            const int64_t n = min((int64_t)4, end - i);
            if (P.unpack) unpack_group(P, s, i, n);
            else pack_group(P, s, i, n);
        }
    }
}

kfac_status wire_run(const std::vector<WireSeg> &segs, WireParams &P, cudaStream_t st) {
    int sms = 0;
    KFAC_TRY(dev_sm_count(&sms));
    for (size_t b = 0; b < segs.size(); b += kWireMaxSegs) {
        const int ns = (int)std::min<size_t>(kWireMaxSegs, segs.size() - b);
        P.nsegs = ns;
        int tiles = 0;
        for (int i = 0; i < ns; i++) {
            P.segs[i] = segs[b + i];
            P.tile_begin[i] = tiles;
            tiles += (int)((segs[b + i].len + kWireTile - 1) / kWireTile);
        }
        P.tile_begin[ns] = tiles;
        if (tiles == 0) continue;
        const int grid = std::min(tiles, sms * 8);
        wire_kernel<<<grid, kWireThreads, 0, st>>>(P);
        KFAC_LAUNCHED();
        KFAC_CUDA_TRY(cudaGetLastError());
    }
    return KFAC_OK;
}

}  // namespace

kfac_status wire_pack(const std::vector<WireSeg> &segs, const float *rs_send, int64_t rs_chunk, float *f32,
                      int64_t f32_stride, void *f16, int64_t f16_stride, float scale_A, float scale_G, cudaStream_t st) {
    WireParams P{};
    P.src_f32 = rs_send;
    P.dst_f32 = f32;
    P.dst_f16 = static_cast<__half *>(f16);
    P.send_stride = rs_chunk;
    P.f32_stride = f32_stride;
    P.f16_stride = f16_stride;
    P.scale[0] = 1.f;
    P.scale[1] = scale_A;
    P.scale[2] = scale_G;
    P.unpack = 0;
    return wire_run(segs, P, st);
}

kfac_status wire_unpack(const std::vector<WireSeg> &segs, const float *f32, const void *const *f16, int npeers,
                        float *rs_recv, float scale_A, float scale_G, cudaStream_t st) {
    if (npeers < 1 || npeers > kWirePeers) return set_error(KFAC_ERR_UNSUPPORTED, "fp16 wire: at most 16 ranks");
    WireParams P{};
    P.src_f32 = f32;
    for (int q = 0; q < npeers; q++) P.src_f16[q] = static_cast<const __half *>(f16[q]);
    P.npeers = npeers;
    P.dst_f32 = rs_recv;
    P.scale[0] = 1.f;
    P.scale[1] = 1.f / scale_A;  // exact: the scales are powers of two
    P.scale[2] = 1.f / scale_G;
    P.unpack = 1;
    return wire_run(segs, P, st);
}

}  // namespace kfac
