// k_scan.cuh -- Pass 3 prefix sum ("the metadata is updated via a
// prefix sum operation ... memory is precisely allocated for the output").
//
// Single-pass exclusive scan of the per-voxel-row (P, Q, S) counts in k-major
// row order (reading Q4), with decoupled look-back across tiles: warp-level
// (shuffle) -> block-level (shared memory) -> inter-block (tile status words
// with release/acquire).  Tile ids are taken from an atomic counter so that a
// tile only ever waits on tiles already running (forward progress).
//
// Outputs: u32 exclusive offsets per row (relative to the first counted row
// for P -- the window index --, relative to the first own row for Q and S,
// which are zero in halo rows), and the u64 totals + halo point counts in the
// workspace header.
#pragma once
#include "psn_common.cuh"

namespace psn {

constexpr int kScanThreads = 256;
#ifndef PSN_SCAN_ITEMS
#define PSN_SCAN_ITEMS 4
#endif
constexpr int kScanItems = PSN_SCAN_ITEMS;
constexpr int kScanTile = kScanThreads * kScanItems;

struct TileStatus {           // 64 bytes per tile
    uint32_t flag;            // 0 = none, 1 = aggregate ready, 2 = inclusive prefix ready
    uint32_t pad;
    uint64_t agg[3];
    uint64_t inc[3];
};

struct ScanHeader {           // device-side header of the extraction workspace
    uint64_t total[3];        // P over all counted rows (window), Q, S
    uint64_t halo_lo, halo_hi;
    uint32_t tile_counter;
    uint32_t emit_status;     // 0 ok, 1 = emission skipped (capacity)
    uint64_t pad[2];
};

struct ScanArgs {
    const uint32_t *cntP, *cntQ, *cntS;
    const uint32_t *cntYZ;        // k_count3: y | z << 16 face counts per row (S completed below); NULL = S complete
    uint32_t *offP, *offQ, *offS;
    int64_t R;
    int64_t own_row0, own_row1;   // rows of own layers: [own_row0, own_row1)
    int64_t NV, kA, O;            // voxel rows per layer, first counted layer, lattice slices
    TileStatus *tiles;
    ScanHeader *hdr;
};

// Directed stencil entries of voxel row r.  k_count3 counts each shared face once, in the row
// that owns its lower side (-x, -y, -z of the voxel): the row's +y / +z faces are the -y faces of row
// j+1 and the -z faces of layer k+1, added here (own rows only; halo rows count points only).
// (j, k) of row r are passed in (callers step them incrementally: no 64-bit division per row).
__device__ __forceinline__ uint32_t row_stencil(const ScanArgs &a, int64_t r, int64_t j, int64_t k) {
    uint32_t s = a.cntS[r];
    if (a.cntYZ && r >= a.own_row0 && r < a.own_row1) {
        if (j + 1 < a.NV) s += a.cntYZ[r + 1] & 0xFFFFu;
        if (k + 3 <= a.O && r + a.NV < a.R) s += a.cntYZ[r + a.NV] >> 16;
    }
    return s;
}
__device__ __forceinline__ uint32_t row_stencil(const ScanArgs &a, int64_t r) {
    const int64_t q = r / a.NV;
    return row_stencil(a, r, r - q * a.NV, a.kA + q);
}

__device__ __forceinline__ void tile_publish(TileStatus *t, const uint64_t (&v)[3], uint32_t f) {
    if (f == 1) { t->agg[0] = v[0]; t->agg[1] = v[1]; t->agg[2] = v[2]; }
    else { t->inc[0] = v[0]; t->inc[1] = v[1]; t->inc[2] = v[2]; }
    st_release(&t->flag, f);   // release orders the value stores before the flag
}

__global__ void __launch_bounds__(kScanThreads) k_scan(ScanArgs a) {
    __shared__ uint32_t s_tile;
    __shared__ uint64_t s_warp[3][kScanThreads / 32];
    __shared__ uint64_t s_prefix[3];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    if (tid == 0) s_tile = atomicAdd(&a.hdr->tile_counter, 1u);
    __syncthreads();
    const int64_t tile = s_tile;
    const int64_t base = tile * kScanTile + (int64_t)tid * kScanItems;

    uint32_t v[3][kScanItems];
    uint64_t loc[3] = {0, 0, 0};
    int64_t jr = 0, kr = 0;   // (j, k) of row `base`, stepped per item
    if (a.cntYZ) { const int64_t q = base / a.NV; jr = base - q * a.NV; kr = a.kA + q; }
#pragma unroll
    for (int it = 0; it < kScanItems; ++it) {
        const int64_t r = base + it;
        const bool ok = r < a.R;
        v[0][it] = ok ? a.cntP[r] : 0u;
        v[1][it] = ok ? a.cntQ[r] : 0u;
        v[2][it] = ok ? row_stencil(a, r, jr, kr) : 0u;
        if (++jr == a.NV) { jr = 0; ++kr; }
#pragma unroll
        for (int c = 0; c < 3; ++c) loc[c] += v[c][it];
    }
    // warp inclusive scan of the thread totals
    uint64_t inc[3];
#pragma unroll
    for (int c = 0; c < 3; ++c) {
        uint64_t x = loc[c];
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
            uint64_t y = __shfl_up_sync(kFull, x, d);
            if (lane >= d) x += y;
        }
        inc[c] = x;
        if (lane == 31) s_warp[c][warp] = x;
    }
    __syncthreads();
    if (warp == 0) {
#pragma unroll
        for (int c = 0; c < 3; ++c) {
            uint64_t x = lane < kScanThreads / 32 ? s_warp[c][lane] : 0;
#pragma unroll
            for (int d = 1; d < 32; d <<= 1) {
                uint64_t y = __shfl_up_sync(kFull, x, d);
                if (lane >= d) x += y;
            }
            if (lane < kScanThreads / 32) s_warp[c][lane] = x;   // inclusive warp prefix
        }
    }
    __syncthreads();
    // decoupled look-back (warp 0)
    if (warp == 0) {
        uint64_t agg[3];
#pragma unroll
        for (int c = 0; c < 3; ++c) agg[c] = s_warp[c][kScanThreads / 32 - 1];
        uint64_t excl[3] = {0, 0, 0};
        TileStatus *me = a.tiles + tile;
        if (lane == 0) tile_publish(me, agg, tile == 0 ? 2u : 1u);
        if (tile > 0) {
            // walk back 32 tiles at a time
            int64_t look = tile - 1;
            bool done = false;
            while (!done) {
                const int64_t t = look - lane;
                uint32_t f = 2;   // tiles before 0 act as an inclusive zero
                if (t >= 0) {
                    do { f = ld_acquire(&a.tiles[t].flag); } while (f == 0);
                }
                const uint32_t inc_mask = __ballot_sync(kFull, f == 2);
                // lanes up to (and including) the first inclusive tile contribute
                const int stop = inc_mask ? __ffs(inc_mask) - 1 : 31;
                uint64_t part[3] = {0, 0, 0};
                if (lane <= stop && t >= 0) {
                    const uint64_t *src = (f == 2) ? a.tiles[t].inc : a.tiles[t].agg;
#pragma unroll
                    for (int c = 0; c < 3; ++c) part[c] = ld_relaxed64(src + c);
                }
#pragma unroll
                for (int c = 0; c < 3; ++c) {
                    uint64_t x = part[c];
#pragma unroll
                    for (int d = 16; d >= 1; d >>= 1) x += __shfl_xor_sync(kFull, x, d);
                    excl[c] += x;
                }
                if (inc_mask) done = true;
                else look -= 32;
            }
            if (lane == 0) {
                uint64_t incl[3];
#pragma unroll
                for (int c = 0; c < 3; ++c) incl[c] = excl[c] + agg[c];
                tile_publish(me, incl, 2u);
            }
        }
        if (lane == 0) {
#pragma unroll
            for (int c = 0; c < 3; ++c) s_prefix[c] = excl[c];
        }
    }
    __syncthreads();
    // per-row exclusive offsets
    uint64_t run[3];
#pragma unroll
    for (int c = 0; c < 3; ++c)
        run[c] = s_prefix[c] + (warp > 0 ? s_warp[c][warp - 1] : 0) + inc[c] - loc[c];
#pragma unroll
    for (int it = 0; it < kScanItems; ++it) {
        const int64_t r = base + it;
        if (r < a.R) {
            a.offP[r] = (uint32_t)run[0];
            a.offQ[r] = (uint32_t)run[1];
            a.offS[r] = (uint32_t)run[2];
            if (r == a.own_row0) a.hdr->halo_lo = run[0];
            if (r == a.own_row1) a.hdr->halo_hi = run[0];   // provisional: points before the hi halo
            if (r == a.R - 1) {
                a.hdr->total[0] = run[0] + v[0][it];
                a.hdr->total[1] = run[1] + v[1][it];
                a.hdr->total[2] = run[2] + v[2][it];
            }
        }
#pragma unroll
        for (int c = 0; c < 3; ++c) run[c] += v[c][it];
    }
}

}  // namespace psn
