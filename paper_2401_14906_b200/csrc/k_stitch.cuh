// k_stitch.cuh -- sub-volume blocks stitched into the whole-volume mesh (NEXT-4).
//
// the extraction leaves region boundaries open "so that the
// resulting distributed execution avoids introducing artificial partitions
// along adjacent sub-volume boundaries"; "PSN can be employed in this
// manner [sub-volumes of a larger input volume], with special attention placed
// on stitching output meshes together at subvolume boundaries".
//
// A block owns the voxel box [own_lo, own_hi) and is extracted as a standalone
// volume (origin 0, spacing 1) over its lattice box plus a one-voxel margin on
// every interior side.  Inside that box every owned voxel sees exactly the
// neighbours it has in the whole volume, so its point, face mask, stencil and
// quads come out right; only the ids are local.  Stitching renumbers them:
//
//   segment s = (global voxel row g = j + (N-1) k, x-block a), s = g * nx + a:
//   the owned voxels of one block in one voxel row.  Segments in s order are
//   the whole-volume id order (k-major rows, x within a row: reading Q4), so
//   the global id of a point is offP[s] + its rank in the segment, and the
//   quads / stencil entries of a segment are one contiguous range too.
//
// Local ids of one local voxel row are consecutive in x, and the x-owned voxels
// of a row lie between its margin voxels, so per local row the first / last
// x-owned point (and owned quad -- quads are voxel-major and their 3rd vertex is
// the owning voxel, reading Q6) bound the segment.  Stencils and quads only
// reference the +-1 neighbours, so a referenced point outside the block's x
// range is the last point of the left segment (offP[s] - 1) or the first of the
// right one (offP[s + 1]).  A stencil entry's voxel follows from its face (the
// entries are in face order -z,-y,-x,+x,+y,+z = ascending id); a quad vertex's
// from its local point.
//
// Local points are voxel centres fl32(idx + 0.5) (origin 0, spacing 1), which
// recover the local voxel index exactly (idx < 2^23); the stitched points are
// recomputed from the global index with the whole-volume origin and spacing
// (anchor_coord, C-3), so every output array is bit-identical to a
// whole-volume psn_extract.
#pragma once
#include <cstdint>
#include "k_emit.cuh"

namespace psn {

constexpr uint32_t kNone = 0xFFFFFFFFu;

struct StitchArgs {
    // local mesh (standalone extraction of the block's box)
    const float *lpts;
    const uint32_t *lquads, *lpairs, *lcsr, *lids;
    const uint8_t *lfm;
    int64_t nP, nQ;
    // local box
    int32_t bM, bN, bO;          // lattice dims of the box
    int32_t lo[3];               // box origin (global lattice index)
    int32_t own_lo[3], own_hi[3];
    int64_t N;                   // global lattice N
    int32_t xseg, nxseg;
    // per local voxel row tables (ws)
    uint32_t *pfirst, *plast, *qfirst, *qlast;
    // segments
    uint32_t *segP, *segQ, *segS;             // counts (stitch_count)
    const uint32_t *offP, *offQ, *offS;       // exclusive offsets (stitch_emit)
    // global mesh
    float *points;
    uint32_t *quads, *pairs, *csr, *ids;
    uint8_t *fm;
    const int64_t *totals;
    double org[3], sp[3];
};

struct LVox { int32_t i, j, k; };

__device__ __forceinline__ LVox lvox(const StitchArgs &a, uint32_t l) {
    const float *p = a.lpts + 3 * (size_t)l;
    return LVox{(int32_t)__ldg(p), (int32_t)__ldg(p + 1), (int32_t)__ldg(p + 2)};
}
__device__ __forceinline__ int32_t lrow(const StitchArgs &a, const LVox &v) { return v.j + (a.bN - 1) * v.k; }
__device__ __forceinline__ bool xown(const StitchArgs &a, const LVox &v) {
    const int32_t gi = v.i + a.lo[0];
    return gi >= a.own_lo[0] && gi < a.own_hi[0];
}
__device__ __forceinline__ bool owned(const StitchArgs &a, const LVox &v) {
    const int32_t gj = v.j + a.lo[1], gk = v.k + a.lo[2];
    return xown(a, v) && gj >= a.own_lo[1] && gj < a.own_hi[1] && gk >= a.own_lo[2] && gk < a.own_hi[2];
}
__device__ __forceinline__ int64_t seg_of(const StitchArgs &a, const LVox &v) {
    const int64_t g = (int64_t)(v.j + a.lo[1]) + (a.N - 1) * (int64_t)(v.k + a.lo[2]);
    return g * a.nxseg + a.xseg;
}

// First / last x-owned point of every local voxel row (one writer per entry: no atomics).  A warp
// takes 32 consecutive ids; the neighbours' voxels come by shuffle (one coalesced read per point).
template <bool QUADS>
__device__ __forceinline__ void mark_rows(const StitchArgs &a, int64_t n, uint32_t *first, uint32_t *last) {
    const int lane = threadIdx.x & 31;
    const int64_t nwarps = (int64_t)gridDim.x * (blockDim.x >> 5);
    for (int64_t base = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x - lane); base < n; base += nwarps * 32) {
        const int64_t t = base + lane;
        auto owner = [&](int64_t x) -> uint32_t {
            return QUADS ? __ldg(a.lquads + 4 * (size_t)x + 2) : (uint32_t)x;
        };
        LVox v{0, 0, -1};
        if (t < n) v = lvox(a, owner(t));
        const bool xo = t < n && xown(a, v);
        const int32_t r = t < n ? lrow(a, v) : -1;
        int32_t rp = __shfl_up_sync(kFull, r, 1), rn = __shfl_down_sync(kFull, r, 1);
        bool xp = __shfl_up_sync(kFull, xo, 1), xn = __shfl_down_sync(kFull, xo, 1);
        if (lane == 0) {
            rp = -1; xp = false;
            if (t > 0 && t < n) { const LVox u = lvox(a, owner(t - 1)); rp = lrow(a, u); xp = xown(a, u); }
        }
        if (lane == 31) {
            rn = -1; xn = false;
            if (t + 1 < n) { const LVox u = lvox(a, owner(t + 1)); rn = lrow(a, u); xn = xown(a, u); }
        }
        if (xo) {
            if (!(xp && rp == r)) first[r] = (uint32_t)t;
            if (!(xn && rn == r)) last[r] = (uint32_t)t;
        }
    }
}

__global__ void k_stitch_mark_points(StitchArgs a) { mark_rows<false>(a, a.nP, a.pfirst, a.plast); }

// First / last quad owned by an x-owned voxel of every local voxel row.
__global__ void k_stitch_mark_quads(StitchArgs a) { mark_rows<true>(a, a.nQ, a.qfirst, a.qlast); }

// Counts of the block's segments: one thread per owned voxel row (every owned segment written once).
__global__ void k_stitch_segments(StitchArgs a) {
    const int32_t ny = a.own_hi[1] - a.own_lo[1], nz = a.own_hi[2] - a.own_lo[2];
    const int64_t n = (int64_t)ny * nz;
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n; t += (int64_t)gridDim.x * blockDim.x) {
        LVox v;
        v.i = a.own_lo[0] - a.lo[0];
        v.j = (int32_t)(t % ny) + a.own_lo[1] - a.lo[1];
        v.k = (int32_t)(t / ny) + a.own_lo[2] - a.lo[2];
        const int32_t r = lrow(a, v);
        const int64_t s = seg_of(a, v);
        const uint32_t f = a.pfirst[r], e = a.plast[r], qf = a.qfirst[r], qe = a.qlast[r];
        a.segP[s] = f == kNone ? 0u : e - f + 1u;
        a.segS[s] = f == kNone ? 0u : __ldg(a.lcsr + e + 1) - __ldg(a.lcsr + f);
        a.segQ[s] = qf == kNone ? 0u : qe - qf + 1u;
    }
}

// Global id of local point m at local voxel v (owned by this block or by a neighbour through the margin).
__device__ __forceinline__ uint32_t remap_at(const StitchArgs &a, uint32_t m, const LVox &v) {
    const int64_t s = seg_of(a, v);
    const int32_t gi = v.i + a.lo[0];
    if (gi < a.own_lo[0]) return __ldg(a.offP + s) - 1u;   // last point of the left segment
    if (gi >= a.own_hi[0]) return __ldg(a.offP + s + 1);   // first point of the right segment
    return __ldg(a.offP + s) + (m - __ldg(a.pfirst + lrow(a, v)));
}
__device__ __forceinline__ uint32_t remap(const StitchArgs &a, uint32_t m) { return remap_at(a, m, lvox(a, m)); }

__global__ void k_stitch_points(StitchArgs a) {
    if (blockIdx.x == 0 && threadIdx.x == 0) a.csr[a.totals[0]] = (uint32_t)a.totals[2];   // CSR sentinel
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < a.nP; t += (int64_t)gridDim.x * blockDim.x) {
        const uint32_t l = (uint32_t)t;
        const LVox v = lvox(a, l);
        if (!owned(a, v)) continue;
        const int64_t s = seg_of(a, v);
        const uint32_t f = __ldg(a.pfirst + lrow(a, v));
        const uint32_t G = __ldg(a.offP + s) + (l - f);
        a.points[3 * (size_t)G + 0] = anchor_coord(a.org[0], a.sp[0], v.i + a.lo[0]);
        a.points[3 * (size_t)G + 1] = anchor_coord(a.org[1], a.sp[1], v.j + a.lo[1]);
        a.points[3 * (size_t)G + 2] = anchor_coord(a.org[2], a.sp[2], v.k + a.lo[2]);
        a.fm[G] = __ldg(a.lfm + l);
        const uint32_t c0 = __ldg(a.lcsr + l), c1 = __ldg(a.lcsr + l + 1);
        const uint32_t base = __ldg(a.offS + s) + (c0 - __ldg(a.lcsr + f));
        a.csr[G] = base;
        // stencil entries are in face order -z, -y, -x, +x, +y, +z over the set bits of the face mask
        // (= ascending id), so each neighbour's voxel is the owner's +- one step: no point gather
        uint32_t fmk = __ldg(a.lfm + l), e = c0;
        while (fmk) {
            const int f = __ffs(fmk) - 1;
            fmk &= fmk - 1u;
            LVox u = v;
            if (f == 0) --u.k; else if (f == 1) --u.j; else if (f == 2) --u.i;
            else if (f == 3) ++u.i; else if (f == 4) ++u.j; else ++u.k;
            a.ids[base + (e - c0)] = remap_at(a, __ldg(a.lids + e), u);
            ++e;
        }
    }
}

__global__ void k_stitch_quads(StitchArgs a) {
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < a.nQ; t += (int64_t)gridDim.x * blockDim.x) {
        const uint32_t q = (uint32_t)t;
        const uint4 lq = __ldg(reinterpret_cast<const uint4 *>(a.lquads) + q);
        const LVox v = lvox(a, lq.z);
        if (!owned(a, v)) continue;
        const int64_t s = seg_of(a, v);
        const uint32_t G = __ldg(a.offQ + s) + (q - __ldg(a.qfirst + lrow(a, v)));
        reinterpret_cast<uint4 *>(a.quads)[G] = make_uint4(remap(a, lq.x), remap(a, lq.y), remap(a, lq.z), remap(a, lq.w));
        reinterpret_cast<uint2 *>(a.pairs)[G] = __ldg(reinterpret_cast<const uint2 *>(a.lpairs) + q);
    }
}

// Exclusive scan of the three segment-count arrays (s order), two launches: per-tile sums, then
// each CTA adds the sums of the tiles before it and scans its own tile.  u64 sums; offsets are
// uint32 (the caller checks the totals against 2^32).
constexpr int kSegTile = 4096;
constexpr int kSegThreads = 512;

__global__ void k_seg_tile_sums(const uint32_t *cnt, int64_t nseg, unsigned long long *tsum) {
    const int arr = blockIdx.y;
    const uint32_t *c = cnt + (size_t)arr * nseg;
    const int64_t t0 = (int64_t)blockIdx.x * kSegTile;
    unsigned long long s = 0;
    for (int64_t i = t0 + threadIdx.x; i < min(t0 + kSegTile, nseg); i += blockDim.x) s += c[i];
    __shared__ unsigned long long red[kSegThreads / 32];
    for (int d = 16; d >= 1; d >>= 1) s += __shfl_down_sync(kFull, s, d);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
    __syncthreads();
    if (threadIdx.x == 0) {
        unsigned long long z = 0;
        for (int w = 0; w < kSegThreads / 32; ++w) z += red[w];
        tsum[(size_t)arr * gridDim.x + blockIdx.x] = z;
    }
}

__global__ void k_seg_scan(const uint32_t *cnt, uint32_t *off, int64_t nseg, const unsigned long long *tsum,
                           int64_t ntiles, int64_t *totals) {
    const int arr = blockIdx.y;
    const uint32_t *c = cnt + (size_t)arr * nseg;
    uint32_t *o = off + (size_t)arr * nseg;
    const unsigned long long *ts = tsum + (size_t)arr * ntiles;
    __shared__ unsigned long long red[kSegThreads / 32];
    __shared__ unsigned long long carry;
    // base of this tile = sum of the tile sums before it (and the grand total on CTA 0)
    const int64_t upto = blockIdx.x == 0 ? ntiles : blockIdx.x;
    unsigned long long s = 0;
    for (int64_t i = threadIdx.x; i < upto; i += blockDim.x) s += ts[i];
    for (int d = 16; d >= 1; d >>= 1) s += __shfl_down_sync(kFull, s, d);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
    __syncthreads();
    if (threadIdx.x == 0) {
        unsigned long long z = 0;
        for (int w = 0; w < kSegThreads / 32; ++w) z += red[w];
        if (blockIdx.x == 0) { totals[arr] = (int64_t)z; carry = 0; }
        else carry = z;
    }
    __syncthreads();
    // scan the tile in chunks of kSegThreads
    const int64_t t0 = (int64_t)blockIdx.x * kSegTile, t1 = min(t0 + kSegTile, nseg);
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    for (int64_t b = t0; b < t1; b += kSegThreads) {
        const int64_t i = b + threadIdx.x;
        const unsigned long long v = i < t1 ? c[i] : 0ull;
        unsigned long long x = v;
        for (int d = 1; d < 32; d <<= 1) {
            const unsigned long long y = __shfl_up_sync(kFull, x, d);
            if (lane >= d) x += y;
        }
        if (lane == 31) red[w] = x;
        __syncthreads();
        unsigned long long wbase = 0;
        for (int q = 0; q < w; ++q) wbase += red[q];
        if (i < t1) o[i] = (uint32_t)(carry + wbase + x - v);
        __syncthreads();
        if (threadIdx.x == kSegThreads - 1) carry += wbase + x;
        __syncthreads();
    }
}

}  // namespace psn
