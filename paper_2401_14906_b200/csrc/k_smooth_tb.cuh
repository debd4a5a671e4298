// k_smooth_tb.cuh -- temporally blocked constrained smoothing (PAPER Eq. 1,
// P:64-69; double buffering P:94; smoothing cache P:154) for a whole volume.
//
// The per-iteration kernel streams every point's state from HBM once per
// iteration.  Here one persistent launch runs G consecutive Jacobi
// iterations as a WAVEFRONT over tiles of `tile` consecutive points: work
// item (t, u) = iteration t of tile u.  Points are k-major, so every stencil
// neighbour of tile u lies in a small tile range rng[u] (at most one voxel
// layer away, SV 8(e)); item (t, u) may run once every tile v in rng[u] has
// finished iteration t-1 (done[v] >= t).  By stencil symmetry the same wait
// also guarantees that nobody still reads the iteration t-2 values that
// (t, u) overwrites in the other ping-pong buffer.  Items are handed out in
// rounds r: round r holds (t, u) for u in block (r - 2t) of delta tiles, so
// every dependency of an item lies in one of the three previous rounds (the
// items of a round are independent; forward progress needs no co-residency).  The live window is about
// G x (one voxel layer of points), i.e. L2-resident, so HBM sees each
// point's state about once per G iterations.
//
// The per-point arithmetic is the one of k_smooth (bit-identical results):
// o' = clamp(o + lambda * (e + sum_j o_j - deg * o) * (1/deg), -d, d).
#pragma once
#include "k_smooth.cuh"

namespace psn {

constexpr uint32_t kTbTileMin = 256;   // smallest wavefront tile (sizes the schedule arrays)
constexpr uint32_t kTbSpinLimit = 1u << 26;

struct TbSched {                       // device-side schedule state (in the smoothing workspace)
    uint32_t counter;                  // next work item of the current launch
    uint32_t delta;                    // block width in tiles: > max tile distance of any neighbour
    uint32_t error;                    // a dependency wait timed out (schedule bug guard)
    uint32_t pad;
};

__device__ __forceinline__ float4 ldcg4(const float4 *p) {
    float4 v;
    asm volatile("ld.global.cg.v4.f32 {%0, %1, %2, %3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "l"(p));
    return v;
}

// Per tile: the range of tiles holding its points' stencil neighbours, and
// delta = 1 + max over tiles of that range's distance.
__global__ void __launch_bounds__(256) k_tile_ranges(const uint4 *nbr, const uint8_t *fmask, uint32_t n,
                                                     uint32_t tile, int2 *rng, TbSched *sch) {
    __shared__ uint32_t s_lo, s_hi;
    const uint32_t u = blockIdx.x;
    if (threadIdx.x == 0) { s_lo = 0xffffffffu; s_hi = 0u; }
    __syncthreads();
    const uint32_t p0 = u * tile, p1 = min(p0 + tile, n);
    uint32_t lo = 0xffffffffu, hi = 0u;
    for (uint32_t i = p0 + threadIdx.x; i < p1; i += blockDim.x) {
        const uint32_t f = fmask[i];
        const uint4 v = nbr_idx(nbr[i]);   // absent faces hold the point itself
        lo = min(lo, min(min(v.x, v.y), min(v.z, v.w)));
        hi = max(hi, max(max(v.x, v.y), max(v.z, v.w)));
        lo = min(lo, i - ((f >> 2) & 1u));
        hi = max(hi, i + ((f >> 3) & 1u));
    }
    lo = __reduce_min_sync(kFull, lo);
    hi = __reduce_max_sync(kFull, hi);
    if ((threadIdx.x & 31) == 0) { atomicMin(&s_lo, lo); atomicMax(&s_hi, hi); }
    __syncthreads();
    if (threadIdx.x == 0) {
        const uint32_t tlo = s_lo / tile, thi = s_hi / tile;
        rng[u] = make_int2((int)tlo, (int)thi);
        atomicMax(&sch->delta, max(u - tlo, thi - u) + 1u);
    }
}

struct TbArgs {
    float4 *buf[2];            // ping-pong index-space offsets (w unused)
    float *world;              // world output of the last iteration (float [n][3])
    const uint8_t *fmask;
    const uint4 *nbr;
    const float *points;       // fp32 voxel centres (anchors) for the world output
    const int2 *rng;
    uint32_t *done;            // per tile: iterations completed
    TbSched *sch;
    uint32_t n, U, tile;
    int32_t t0, G, T;          // this launch runs iterations [t0, t0 + G) of T
    float lambda;
    Constraint cons;
    double sp[3], org[3];
};

__global__ void __launch_bounds__(256, 4) k_smooth_tb(TbArgs a) {
    __shared__ uint32_t s_item;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const uint32_t delta = *reinterpret_cast<volatile uint32_t *>(&a.sch->delta);
    const uint32_t nb = (a.U + delta - 1) / delta;
    const uint64_t per_round = (uint64_t)a.G * delta;
    const uint64_t total = (uint64_t)(nb + 2 * (a.G - 1)) * per_round;
    for (;;) {
        if (threadIdx.x == 0) s_item = atomicAdd(&a.sch->counter, 1u);
        __syncthreads();
        const uint64_t item = s_item;
        __syncthreads();
        if (item >= total) break;
        const uint64_t r = item / per_round, rem = item % per_round;
        const uint32_t tl = (uint32_t)(rem / delta);
        if (r < 2u * tl) continue;
        const uint64_t b = r - 2u * tl;   // iteration t lags two blocks: all its dependencies are in earlier rounds
        if (b >= nb) continue;
        const uint32_t u = (uint32_t)(b * delta + rem % delta);
        if (u >= a.U) continue;
        const int32_t t = a.t0 + (int32_t)tl;
        // ---- wait until every tile holding a neighbour finished iteration t-1
        if (t > 0 && warp == 0) {
            const int2 rg = a.rng[u];
            for (int v = rg.x + lane; v <= rg.y; v += 32) {
                uint32_t spins = 0;
                while (ld_acquire(a.done + v) < (uint32_t)t) {
                    if (++spins > kTbSpinLimit) { atomicExch(&a.sch->error, 1u); break; }
                    __nanosleep(32);
                }
            }
            __threadfence();
        }
        __syncthreads();
        // ---- iteration t on the tile's points (64 per warp per round, two per lane)
        const float4 *__restrict__ src = t > 0 ? a.buf[t & 1] : nullptr;
        float4 *dst = a.buf[(t + 1) & 1];
        const bool last = (t == a.T - 1);
        const uint32_t p0 = u * a.tile, p1 = min(p0 + a.tile, a.n);
        for (uint32_t base = p0 + warp * 64; base < p1; base += 8 * 64) {
            uint32_t i[2], f[2];
            uint4 nbv[2];
            float4 o[2];
#pragma unroll
            for (int q = 0; q < 2; ++q) {
                i[q] = base + 32u * q + lane;
                const uint32_t ii = i[q] < p1 ? i[q] : p1 - 1u;
                f[q] = i[q] < p1 ? (uint32_t)__ldg(a.fmask + ii) : 0u;
                nbv[q] = nbr_idx(__ldg(a.nbr + ii));
                o[q] = src ? ldcg4(src + ii) : make_float4(0.f, 0.f, 0.f, 0.f);
            }
            float4 gth[2][4];
#pragma unroll
            for (int q = 0; q < 2; ++q) {
                if (src) {
                    gth[q][0] = ldcg4(src + nbv[q].x); gth[q][1] = ldcg4(src + nbv[q].y);
                    gth[q][2] = ldcg4(src + nbv[q].z); gth[q][3] = ldcg4(src + nbv[q].w);
                } else {
#pragma unroll
                    for (int c = 0; c < 4; ++c) gth[q][c] = make_float4(0.f, 0.f, 0.f, 0.f);
                }
            }
            float3 mxo[2], pxo[2];
#pragma unroll
            for (int q = 0; q < 2; ++q) {
                mxo[q].x = __shfl_up_sync(kFull, o[q].x, 1); mxo[q].y = __shfl_up_sync(kFull, o[q].y, 1);
                mxo[q].z = __shfl_up_sync(kFull, o[q].z, 1);
                pxo[q].x = __shfl_down_sync(kFull, o[q].x, 1); pxo[q].y = __shfl_down_sync(kFull, o[q].y, 1);
                pxo[q].z = __shfl_down_sync(kFull, o[q].z, 1);
            }
            {
                const float bx = __shfl_sync(kFull, o[1].x, 0), by = __shfl_sync(kFull, o[1].y, 0), bz = __shfl_sync(kFull, o[1].z, 0);
                const float ex = __shfl_sync(kFull, o[0].x, 31), ey = __shfl_sync(kFull, o[0].y, 31), ez = __shfl_sync(kFull, o[0].z, 31);
                if (lane == 31) pxo[0] = make_float3(bx, by, bz);
                if (lane == 0) mxo[1] = make_float3(ex, ey, ez);
            }
#pragma unroll
            for (int q = 0; q < 2; ++q) {
                if (i[q] >= p1) continue;
                const uint32_t fu = f[q];
                if (fu && src) {
                    if ((fu & 4u) && lane == 0 && q == 0) { const float4 v = ldcg4(src + i[q] - 1u); mxo[0] = make_float3(v.x, v.y, v.z); }
                    if ((fu & 8u) && ((lane == 31 && q == 1) || i[q] + 1u >= p1)) {
                        const float4 v = ldcg4(src + i[q] + 1u); pxo[q] = make_float3(v.x, v.y, v.z);
                    }
                }
                const float3 res = jacobi_update(fu, make_float3(o[q].x, o[q].y, o[q].z), mxo[q], pxo[q],
                                                 make_float3(gth[q][0].x, gth[q][0].y, gth[q][0].z),
                                                 make_float3(gth[q][1].x, gth[q][1].y, gth[q][1].z),
                                                 make_float3(gth[q][2].x, gth[q][2].y, gth[q][2].z),
                                                 make_float3(gth[q][3].x, gth[q][3].y, gth[q][3].z), a.lambda, a.cons);
                const uint32_t w = i[q];
                if (last) {
                    a.world[3u * w + 0u] = world_of(__ldg(a.points + 3u * w + 0u), res.x, a.org[0], a.sp[0]);
                    a.world[3u * w + 1u] = world_of(__ldg(a.points + 3u * w + 1u), res.y, a.org[1], a.sp[1]);
                    a.world[3u * w + 2u] = world_of(__ldg(a.points + 3u * w + 2u), res.z, a.org[2], a.sp[2]);
                } else {
                    dst[w] = make_float4(res.x, res.y, res.z, 0.f);
                }
            }
        }
        // ---- publish: iteration t of tile u is complete
        __syncthreads();
        if (threadIdx.x == 0) {
            __threadfence();
            st_release(a.done + u, (uint32_t)t + 1u);
        }
    }
}

}  // namespace psn
