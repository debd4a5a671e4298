// k_emit.cuh -- Pass 4 of PSN extraction on sm_100a.
//
// One warp per voxel row V_{j,k} (grid-stride).  The paper's 3x3 voxel-row
// iterator (Fig. 6) becomes prefix-popcounts over the natural-order
// point bit-planes written by k_count: the id of voxel i of row r' is
//     window_base + offP[r'] + popc(points of r' before i)
// computed per 32-voxel word with a warp scan.  Quads use rows (j-1,k-1),
// (j,k-1), (j-1,k); the stencil adds (j+1,k) and (j,k+1).
//
// Work is at POINT granularity: the row's points are compacted into a
// per-warp list and processed 32 at a time, one point per lane, so voxels
// without a point cost nothing ("rapidly skip data").  Each point reads
// its 8 corner labels, forms the 12 edge predicates, the face mask (c^f,
// P:118), its owned quads (open boundaries P:264) and writes them into
// the disjoint preallocated slots given by the scan -- no atomics.
#pragma once
#include "k_scan.cuh"
#include "k_smooth.cuh"
#include "psn_common.cuh"

namespace psn {

struct EmitArgs {
    const void *labels;
    int64_t M, N, O, z_lo;
    int64_t kA, kB, own_k0, own_k1, W32, R;
    const uint32_t *cntP, *offP, *offQ, *offS, *pmask;
    const uint16_t *ppre;      // per pmask word: points of the row before it (single x-tile rows)
    LabelSet ls;
    double sp[3], org[3];
    float *points;
    uint32_t *quads, *pairs, *csr_off, *csr_ids;
    uint8_t *fmask;
    int64_t cap_points, cap_quads, cap_stencil;
    uint32_t first_point, first_quad, first_stencil;
    const int64_t *first_dev;  // if non-NULL: the global first ids (point, quad, stencil) in device memory
    ScanHeader *hdr;
    uint2 *scache;             // if non-NULL (k_emit_band): packed smoothing cache of the own points
    int dual;                  // k_emit_band: both density variants launched, each returns unless selected
};

__device__ __forceinline__ float anchor_coord(double org, double sp, int64_t idx) {
    // C-3: fl32(origin + (idx + 0.5) * spacing), fp64 with no contraction
    return __double2float_rn(__dadd_rn(org, __dmul_rn(__dadd_rn((double)idx, 0.5), sp)));
}

template <typename T, bool ANZ>
__device__ __forceinline__ uint32_t code_at(const T *p, const LabelSet &ls) {
    uint32_t v = (uint32_t)__ldg(p);
    if (!ANZ && !ls.identity) v = in_L<T>(ls, v) ? v : ls.z;
    return v;
}

constexpr int kEmitWarps = 8;

// Warp-inclusive scan of three 10-bit counters packed in one word (the
// prefixes inside a 1024-voxel block never exceed 1023).
__device__ __forceinline__ uint32_t scan3(uint32_t x, int lane) {
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
        const uint32_t y = __shfl_up_sync(kFull, x, d);
        if (lane >= d) x += y;
    }
    return x;
}

template <typename T, bool ANZ>
__global__ void __launch_bounds__(256, 3) k_emit(EmitArgs a) {
    __shared__ uint32_t sbits[ANZ ? 1 : 2048];
    __shared__ uint16_t slist[kEmitWarps][1024];      // point x positions of the current 1024-voxel block
    __shared__ uint32_t sword[kEmitWarps][5][32];     // neighbour rows: mask word
    __shared__ uint32_t spre[kEmitWarps][5][32];      // neighbour rows: window index of the word's first point
    __shared__ uint32_t srun[kEmitWarps][5];          // neighbour rows: window index of the block's first point
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    LabelSet ls = a.ls;
    if (!ANZ && sizeof(T) < 4) {
        for (int t = threadIdx.x; t < (sizeof(T) == 1 ? 8 : 2048); t += blockDim.x) sbits[t] = a.ls.bits[t];
        ls.bits = sbits;
        __syncthreads();
    }
    // device-side capacity check (steady-state COUNT|EMIT path)
    if (a.first_dev) {   // device-side C1 (multi-GPU step without a host round trip)
        a.first_point = (uint32_t)a.first_dev[0]; a.first_quad = (uint32_t)a.first_dev[1];
        a.first_stencil = (uint32_t)a.first_dev[2];
    }
    const uint64_t totP = a.hdr->total[0], totQ = a.hdr->total[1], totS = a.hdr->total[2];
    const uint32_t halo_lo = (uint32_t)a.hdr->halo_lo;
    if (totP > (uint64_t)a.cap_points || totQ > (uint64_t)a.cap_quads || totS > (uint64_t)a.cap_stencil) {
        if (blockIdx.x == 0 && threadIdx.x == 0) a.hdr->emit_status = 1u;
        return;
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        const uint64_t before_hi = (a.kB > a.own_k1) ? a.hdr->halo_hi : totP;
        a.hdr->emit_status = 0u;
        a.csr_off[before_hi - halo_lo] = a.first_stencil + (uint32_t)totS;   // CSR sentinel entry
    }
    const uint32_t gid_base = a.first_point - halo_lo;   // global id of window index 0
    const uint32_t M = (uint32_t)a.M, N = (uint32_t)a.N, NV = N - 1, W32 = (uint32_t)a.W32;
    const uint32_t R = (uint32_t)a.R;
    const uint32_t kA = (uint32_t)a.kA, kB = (uint32_t)a.kB, own0 = (uint32_t)a.own_k0, own1 = (uint32_t)a.own_k1;
    const T *lab = reinterpret_cast<const T *>(a.labels);

    const uint32_t warps = gridDim.x * (blockDim.x >> 5);
    uint32_t rr = blockIdx.x * (blockDim.x >> 5) + warp;
    uint32_t cnt_next = rr < R ? __ldg(a.cntP + rr) : 0u;
    for (; rr < R; rr += warps) {
        // software pipelining: the next row's point count is in flight while this row is emitted
        const uint32_t cnt = cnt_next;
        cnt_next = (rr + warps < R) ? __ldg(a.cntP + rr + warps) : 0u;
        if (cnt == 0) continue;
        const uint32_t j = rr % NV, k = kA + rr / NV;
        const bool own = (k >= own0) && (k < own1);
        // neighbour rows (j-1,k-1), (j,k-1), (j-1,k), (j+1,k), (j,k+1); -1 = absent
        int32_t nbq = -1;
        if (lane < 5 && own) {
            const bool ok = lane == 0 ? (j >= 1 && k >= kA + 1) : lane == 1 ? (k >= kA + 1)
                          : lane == 2 ? (j >= 1) : lane == 3 ? (j + 1 <= N - 2) : (k + 1 < kB);
            const int32_t d = lane == 0 ? -(int32_t)NV - 1 : lane == 1 ? -(int32_t)NV : lane == 2 ? -1
                            : lane == 3 ? 1 : (int32_t)NV;
            if (ok) nbq = (int32_t)rr + d;
            srun[warp][lane] = ok ? __ldg(a.offP + nbq) : 0u;
        }
        const uint32_t offP = __ldg(a.offP + rr);
        const uint32_t qbase = own ? __ldg(a.offQ + rr) : 0u, sbase = own ? __ldg(a.offS + rr) : 0u;
        uint32_t run_o = 0, run_q = 0, run_s = 0;
        const size_t rowA = ((size_t)(k - (uint32_t)a.z_lo) * N + j) * M;
        const size_t rowB = rowA + M, rowC = rowA + (size_t)N * M, rowD = rowC + M;

        for (uint32_t w0 = 0; w0 < W32; w0 += 32) {
            const uint32_t w = w0 + lane;
            const bool wok = w < W32;
            const uint32_t om = wok ? __ldg(a.pmask + (size_t)rr * W32 + w) : 0u;
            // own points: exclusive scan of the word popcounts -> compact list
            const uint32_t oc = __popc(om);
            const uint32_t oi = scan3(oc, lane);
            const uint32_t blk_pts = __shfl_sync(kFull, oi, 31);
            // neighbour rows: per-word window index of the first point (two packed scans)
            uint32_t nm[5];
#pragma unroll
            for (int q = 0; q < 5; ++q) {
                const int32_t row = __shfl_sync(kFull, nbq, q);
                nm[q] = (row >= 0 && wok) ? __ldg(a.pmask + (size_t)row * W32 + w) : 0u;
            }
            __syncwarp();
            if (own) {
                const uint32_t c0 = __popc(nm[0]) | (__popc(nm[1]) << 10) | (__popc(nm[2]) << 20);
                const uint32_t c1 = __popc(nm[3]) | (__popc(nm[4]) << 10);
                // exclusive prefixes are <= 31*32 < 1024, so the packed fields never carry
                const uint32_t i0 = scan3(c0, lane) - c0, i1 = scan3(c1, lane) - c1;
                const uint32_t ex[5] = {i0 & 1023u, (i0 >> 10) & 1023u, (i0 >> 20) & 1023u, i1 & 1023u, (i1 >> 10) & 1023u};
                uint32_t tt[5];
#pragma unroll
                for (int q = 0; q < 5; ++q) tt[q] = __reduce_add_sync(kFull, (uint32_t)__popc(nm[q]));
#pragma unroll
                for (int q = 0; q < 5; ++q) {
                    sword[warp][q][lane] = nm[q];
                    spre[warp][q][lane] = srun[warp][q] + ex[q];
                }
                __syncwarp();
                if (lane < 5) srun[warp][lane] += lane == 0 ? tt[0] : lane == 1 ? tt[1] : lane == 2 ? tt[2] : lane == 3 ? tt[3] : tt[4];
            }
            if (blk_pts == 0) continue;
            {
                uint32_t pos = oi - oc, m = om;
                while (m) {
                    const int b = __ffs(m) - 1;
                    m &= m - 1;
                    slist[warp][pos++] = (uint16_t)(lane * 32 + b);
                }
            }
            __syncwarp();
            for (uint32_t base = 0; base < blk_pts; base += 32) {
                const uint32_t t = base + lane;
                const bool act = t < blk_pts;
                const uint32_t xb = act ? slist[warp][t] : 0u;          // position within the block
                const uint32_t i = w0 * 32 + xb;                         // voxel x
                const uint32_t wi = offP + run_o + t;                    // window index
                const uint32_t g = gid_base + wi;                        // global id
                uint32_t fm = 0, qb = 0;
                uint32_t cA = 0, cA1 = 0, cB = 0, cC = 0;
                if (act && own) {
                    const uint32_t A = code_at<T, ANZ>(lab + rowA + i, ls), A1 = code_at<T, ANZ>(lab + rowA + i + 1, ls);
                    const uint32_t B = code_at<T, ANZ>(lab + rowB + i, ls), B1 = code_at<T, ANZ>(lab + rowB + i + 1, ls);
                    const uint32_t C = code_at<T, ANZ>(lab + rowC + i, ls), C1 = code_at<T, ANZ>(lab + rowC + i + 1, ls);
                    const uint32_t D = code_at<T, ANZ>(lab + rowD + i, ls), D1 = code_at<T, ANZ>(lab + rowD + i + 1, ls);
                    const bool XA = A != A1, XB = B != B1, XC = C != C1, XD = D != D1;
                    const bool YAB = A != B, YA1 = A1 != B1, YCD = C != D, YC1 = C1 != D1;
                    const bool ZAC = A != C, ZA1 = A1 != C1, ZBD = B != D, ZB1 = B1 != D1;
                    fm |= ((XA | XB | YAB | YA1) && k >= 1) ? 1u : 0u;          // -z
                    fm |= ((XA | XC | ZAC | ZA1) && j >= 1) ? 2u : 0u;          // -y
                    fm |= ((YAB | YCD | ZAC | ZBD) && i >= 1) ? 4u : 0u;        // -x
                    fm |= ((YA1 | YC1 | ZA1 | ZB1) && i + 3 <= M) ? 8u : 0u;    // +x
                    fm |= ((XB | XD | ZBD | ZB1) && j + 3 <= N) ? 16u : 0u;     // +y
                    fm |= ((XC | XD | YCD | YC1) && k + 3 <= (uint32_t)a.O) ? 32u : 0u;   // +z
                    qb |= (XA && j >= 1 && k >= 1) ? 1u : 0u;
                    qb |= (YAB && i >= 1 && k >= 1) ? 2u : 0u;
                    qb |= (ZAC && i >= 1 && j >= 1) ? 4u : 0u;
                    cA = cls_of_code<T, ANZ>(ls, A); cA1 = cls_of_code<T, ANZ>(ls, A1);
                    cB = cls_of_code<T, ANZ>(ls, B); cC = cls_of_code<T, ANZ>(ls, C);
                }
                // warp exclusive scan of (quads << 16 | degree)
                const uint32_t packed = ((uint32_t)__popc(qb) << 16) | (uint32_t)__popc(fm);
                const uint32_t x = scan3(packed, lane);
                const uint32_t tot = __shfl_sync(kFull, x, 31);
                const uint32_t ex = x - packed;
                if (act) {
                    a.points[3 * (size_t)wi + 0] = anchor_coord(a.org[0], a.sp[0], i);
                    a.points[3 * (size_t)wi + 1] = anchor_coord(a.org[1], a.sp[1], j);
                    a.points[3 * (size_t)wi + 2] = anchor_coord(a.org[2], a.sp[2], k);
                    if (own) {
                        // ids of the neighbour-row voxels at x = i: window index of the word's first
                        // point + points below i in the word
                        const uint32_t wl = xb >> 5, below = (1u << (xb & 31)) - 1u;
                        auto gn = [&](int q) { return gid_base + spre[warp][q][wl] + __popc(sword[warp][q][wl] & below); };
                        const uint32_t o = wi - halo_lo;
                        uint32_t ss = sbase + run_s + (ex & 0xffffu);
                        a.fmask[o] = (uint8_t)fm;
                        a.csr_off[o] = a.first_stencil + ss;
                        if (fm & 1u) a.csr_ids[ss++] = gn(1);      // -z  (j, k-1)
                        if (fm & 2u) a.csr_ids[ss++] = gn(2);      // -y  (j-1, k)
                        if (fm & 4u) a.csr_ids[ss++] = g - 1u;     // -x
                        if (fm & 8u) a.csr_ids[ss++] = g + 1u;     // +x
                        if (fm & 16u) a.csr_ids[ss++] = gn(3);     // +y  (j+1, k)
                        if (fm & 32u) a.csr_ids[ss++] = gn(4);     // +z  (j, k+1)
                        uint32_t qs = qbase + run_q + (ex >> 16);
                        if (qb & 1u) {   // x-quad [(j-1,k-1), (j,k-1), (j,k), (j-1,k)]
                            *reinterpret_cast<uint4 *>(a.quads + 4 * (size_t)qs) = make_uint4(gn(0), gn(1), g, gn(2));
                            *reinterpret_cast<uint2 *>(a.pairs + 2 * (size_t)qs) = make_uint2(cA, cA1);
                            ++qs;
                        }
                        if (qb & 2u) {   // y-quad [(i-1,k-1), (i-1,k), (i,k), (i,k-1)] of row j
                            const uint32_t g1 = gn(1);
                            *reinterpret_cast<uint4 *>(a.quads + 4 * (size_t)qs) = make_uint4(g1 - 1u, g - 1u, g, g1);
                            *reinterpret_cast<uint2 *>(a.pairs + 2 * (size_t)qs) = make_uint2(cA, cB);
                            ++qs;
                        }
                        if (qb & 4u) {   // z-quad [(i-1,j-1), (i,j-1), (i,j), (i-1,j)] of layer k
                            const uint32_t g2 = gn(2);
                            *reinterpret_cast<uint4 *>(a.quads + 4 * (size_t)qs) = make_uint4(g2 - 1u, g2, g, g - 1u);
                            *reinterpret_cast<uint2 *>(a.pairs + 2 * (size_t)qs) = make_uint2(cA, cC);
                            ++qs;
                        }
                    }
                }
                run_q += tot >> 16;
                run_s += tot & 0xffffu;
            }
            run_o += blk_pts;
            __syncwarp();
        }
    }
}


// Pass 4 for rows that fit one k_count x-tile: k_count left, next to every
// point-plane word, the number of the row's points before it (ppre), so the id
// of voxel i of ANY row r' is  window_base + offP[r'] + ppre[r'][i/32] +
// popc(pmask[r'][i/32] & below(i))  -- one word lookup instead of a per-row
// scan.  Warp per voxel row; the row's points are listed by their running
// index (ppre + rank in the word) and processed one per lane.
template <typename T, bool ANZ>
__global__ void __launch_bounds__(256) k_emit_fast(EmitArgs a) {
    __shared__ uint32_t sbits[ANZ ? 1 : 2048];
    __shared__ uint16_t slist[kEmitWarps][1024];      // x of the block's points, by running index
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    LabelSet ls = a.ls;
    if (!ANZ && sizeof(T) < 4) {
        for (int t = threadIdx.x; t < (sizeof(T) == 1 ? 8 : 2048); t += blockDim.x) sbits[t] = a.ls.bits[t];
        ls.bits = sbits;
        __syncthreads();
    }
    if (a.first_dev) {   // device-side C1 (multi-GPU step without a host round trip)
        a.first_point = (uint32_t)a.first_dev[0]; a.first_quad = (uint32_t)a.first_dev[1];
        a.first_stencil = (uint32_t)a.first_dev[2];
    }
    const uint64_t totP = a.hdr->total[0], totQ = a.hdr->total[1], totS = a.hdr->total[2];
    const uint32_t halo_lo = (uint32_t)a.hdr->halo_lo;
    if (totP > (uint64_t)a.cap_points || totQ > (uint64_t)a.cap_quads || totS > (uint64_t)a.cap_stencil) {
        if (blockIdx.x == 0 && threadIdx.x == 0) a.hdr->emit_status = 1u;
        return;
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        const uint64_t before_hi = (a.kB > a.own_k1) ? a.hdr->halo_hi : totP;
        a.hdr->emit_status = 0u;
        a.csr_off[before_hi - halo_lo] = a.first_stencil + (uint32_t)totS;   // CSR sentinel entry
    }
    const uint32_t gid_base = a.first_point - halo_lo;
    const uint32_t M = (uint32_t)a.M, N = (uint32_t)a.N, NV = N - 1, W32 = (uint32_t)a.W32;
    const uint32_t R = (uint32_t)a.R;
    const uint32_t kA = (uint32_t)a.kA, kB = (uint32_t)a.kB, own0 = (uint32_t)a.own_k0, own1 = (uint32_t)a.own_k1;
    const T *lab = reinterpret_cast<const T *>(a.labels);

    const uint32_t warps = gridDim.x * (blockDim.x >> 5);
    uint32_t rr = blockIdx.x * (blockDim.x >> 5) + warp;
    // (j, k) of row rr, advanced incrementally (no division in the loop)
    uint32_t j = rr % NV, k = kA + rr / NV;
    const uint32_t dj = warps % NV, dk = warps / NV;
    uint32_t cnt_next = rr < R ? __ldg(a.cntP + rr) : 0u;
    for (; rr < R; rr += warps) {
        const uint32_t cnt = cnt_next;
        cnt_next = (rr + warps < R) ? __ldg(a.cntP + rr + warps) : 0u;
        const uint32_t jj = j, kk = k;
        j += dj; k += dk;
        if (j >= NV) { j -= NV; ++k; }
        if (cnt == 0) continue;
        const bool own = (kk >= own0) && (kk < own1);
        // neighbour rows (j-1,k-1), (j,k-1), (j-1,k), (j+1,k), (j,k+1): lane q holds row q and its offP
        int32_t nbq = -1;
        uint32_t nbo = 0;
        if (lane < 5 && own) {
            const bool ok = lane == 0 ? (jj >= 1 && kk >= kA + 1) : lane == 1 ? (kk >= kA + 1)
                          : lane == 2 ? (jj >= 1) : lane == 3 ? (jj + 1 <= N - 2) : (kk + 1 < kB);
            const int32_t d = lane == 0 ? -(int32_t)NV - 1 : lane == 1 ? -(int32_t)NV : lane == 2 ? -1
                            : lane == 3 ? 1 : (int32_t)NV;
            if (ok) { nbq = (int32_t)rr + d; nbo = __ldg(a.offP + nbq); }
        }
        const uint32_t offP = __ldg(a.offP + rr);
        const uint32_t qbase = own ? __ldg(a.offQ + rr) : 0u, sbase = own ? __ldg(a.offS + rr) : 0u;
        int32_t nrow[5];
        uint32_t noff[5];
#pragma unroll
        for (int q = 0; q < 5; ++q) { nrow[q] = __shfl_sync(kFull, nbq, q); noff[q] = __shfl_sync(kFull, nbo, q); }
        uint32_t run_q = 0, run_s = 0;
        const size_t rowA = ((size_t)(kk - (uint32_t)a.z_lo) * N + jj) * M;
        const size_t rowB = rowA + M, rowC = rowA + (size_t)N * M, rowD = rowC + M;

        for (uint32_t w0 = 0; w0 < W32; w0 += 32) {
            const uint32_t w = w0 + lane;
            const bool wok = w < W32;
            const uint32_t om = wok ? __ldg(a.pmask + (size_t)rr * W32 + w) : 0u;
            const uint32_t op = wok ? (uint32_t)__ldg(a.ppre + (size_t)rr * W32 + w) : 0u;
            const uint32_t blk_base = __shfl_sync(kFull, op, 0);
            const uint32_t blk_pts = __reduce_add_sync(kFull, (uint32_t)__popc(om));
            if (blk_pts == 0) continue;
            {
                uint32_t pos = op - blk_base, m = om;
                while (m) {
                    const int b = __ffs(m) - 1;
                    m &= m - 1;
                    slist[warp][pos++] = (uint16_t)(lane * 32 + b);
                }
            }
            __syncwarp();
            for (uint32_t base = 0; base < blk_pts; base += 32) {
                const uint32_t t = base + lane;
                const bool act = t < blk_pts;
                const uint32_t xb = act ? slist[warp][t] : 0u;
                const uint32_t i = w0 * 32 + xb;                 // voxel x
                const uint32_t wi = offP + blk_base + t;         // window index
                const uint32_t g = gid_base + wi;                // global id
                uint32_t fm = 0, qb = 0, cA = 0, cA1 = 0, cB = 0, cC = 0;
                uint32_t gn[5] = {0, 0, 0, 0, 0};
                if (act && own) {
                    const uint32_t A = code_at<T, ANZ>(lab + rowA + i, ls), A1 = code_at<T, ANZ>(lab + rowA + i + 1, ls);
                    const uint32_t B = code_at<T, ANZ>(lab + rowB + i, ls), B1 = code_at<T, ANZ>(lab + rowB + i + 1, ls);
                    const uint32_t C = code_at<T, ANZ>(lab + rowC + i, ls), C1 = code_at<T, ANZ>(lab + rowC + i + 1, ls);
                    const uint32_t D = code_at<T, ANZ>(lab + rowD + i, ls), D1 = code_at<T, ANZ>(lab + rowD + i + 1, ls);
                    // ids of the neighbour-row voxels at x = i (one word lookup each)
                    const uint32_t wl = i >> 5, below = (1u << (i & 31)) - 1u;
#pragma unroll
                    for (int q = 0; q < 5; ++q) {
                        if (nrow[q] >= 0) {
                            const size_t at = (size_t)nrow[q] * W32 + wl;
                            gn[q] = gid_base + noff[q] + __ldg(a.ppre + at) + __popc(__ldg(a.pmask + at) & below);
                        }
                    }
                    const bool XA = A != A1, XB = B != B1, XC = C != C1, XD = D != D1;
                    const bool YAB = A != B, YA1 = A1 != B1, YCD = C != D, YC1 = C1 != D1;
                    const bool ZAC = A != C, ZA1 = A1 != C1, ZBD = B != D, ZB1 = B1 != D1;
                    fm |= ((XA | XB | YAB | YA1) && kk >= 1) ? 1u : 0u;          // -z
                    fm |= ((XA | XC | ZAC | ZA1) && jj >= 1) ? 2u : 0u;          // -y
                    fm |= ((YAB | YCD | ZAC | ZBD) && i >= 1) ? 4u : 0u;         // -x
                    fm |= ((YA1 | YC1 | ZA1 | ZB1) && i + 3 <= M) ? 8u : 0u;     // +x
                    fm |= ((XB | XD | ZBD | ZB1) && jj + 3 <= N) ? 16u : 0u;     // +y
                    fm |= ((XC | XD | YCD | YC1) && kk + 3 <= (uint32_t)a.O) ? 32u : 0u;   // +z
                    qb |= (XA && jj >= 1 && kk >= 1) ? 1u : 0u;
                    qb |= (YAB && i >= 1 && kk >= 1) ? 2u : 0u;
                    qb |= (ZAC && i >= 1 && jj >= 1) ? 4u : 0u;
                    cA = cls_of_code<T, ANZ>(ls, A); cA1 = cls_of_code<T, ANZ>(ls, A1);
                    cB = cls_of_code<T, ANZ>(ls, B); cC = cls_of_code<T, ANZ>(ls, C);
                }
                const uint32_t packed = ((uint32_t)__popc(qb) << 16) | (uint32_t)__popc(fm);
                const uint32_t x = scan3(packed, lane);
                const uint32_t tot = __shfl_sync(kFull, x, 31);
                const uint32_t ex = x - packed;
                if (act) {
                    a.points[3 * (size_t)wi + 0] = anchor_coord(a.org[0], a.sp[0], i);
                    a.points[3 * (size_t)wi + 1] = anchor_coord(a.org[1], a.sp[1], jj);
                    a.points[3 * (size_t)wi + 2] = anchor_coord(a.org[2], a.sp[2], kk);
                    if (own) {
                        const uint32_t o = wi - halo_lo;
                        uint32_t ss = sbase + run_s + (ex & 0xffffu);
                        a.fmask[o] = (uint8_t)fm;
                        a.csr_off[o] = a.first_stencil + ss;
                        if (fm & 1u) a.csr_ids[ss++] = gn[1];      // -z  (j, k-1)
                        if (fm & 2u) a.csr_ids[ss++] = gn[2];      // -y  (j-1, k)
                        if (fm & 4u) a.csr_ids[ss++] = g - 1u;     // -x
                        if (fm & 8u) a.csr_ids[ss++] = g + 1u;     // +x
                        if (fm & 16u) a.csr_ids[ss++] = gn[3];     // +y  (j+1, k)
                        if (fm & 32u) a.csr_ids[ss++] = gn[4];     // +z  (j, k+1)
                        uint32_t qs = qbase + run_q + (ex >> 16);
                        if (qb & 1u) {   // x-quad [(j-1,k-1), (j,k-1), (j,k), (j-1,k)]
                            *reinterpret_cast<uint4 *>(a.quads + 4 * (size_t)qs) = make_uint4(gn[0], gn[1], g, gn[2]);
                            *reinterpret_cast<uint2 *>(a.pairs + 2 * (size_t)qs) = make_uint2(cA, cA1);
                            ++qs;
                        }
                        if (qb & 2u) {   // y-quad [(i-1,k-1), (i-1,k), (i,k), (i,k-1)] of row j
                            *reinterpret_cast<uint4 *>(a.quads + 4 * (size_t)qs) = make_uint4(gn[1] - 1u, g - 1u, g, gn[1]);
                            *reinterpret_cast<uint2 *>(a.pairs + 2 * (size_t)qs) = make_uint2(cA, cB);
                            ++qs;
                        }
                        if (qb & 4u) {   // z-quad [(i-1,j-1), (i,j-1), (i,j), (i-1,j)] of layer k
                            *reinterpret_cast<uint4 *>(a.quads + 4 * (size_t)qs) = make_uint4(gn[2] - 1u, gn[2], g, g - 1u);
                            *reinterpret_cast<uint2 *>(a.pairs + 2 * (size_t)qs) = make_uint2(cA, cC);
                            ++qs;
                        }
                    }
                }
                run_q += tot >> 16;
                run_s += tot & 0xffffu;
            }
            __syncwarp();
        }
    }
}
// Pass 4, band-staged (rows of <= 32 plane words).  A CTA emits BANDS of
// kBand consecutive voxel rows (k-major order, reading Q4).  For each band the
// point-plane words, per-word prefixes and offsets of every row an id lookup
// can touch -- rows rr0-1 .. rr0+kBand and the same rows one layer below /
// above (the paper's 3x3 row iterator) -- are three contiguous ranges
// of the workspace, staged in shared memory by TMA bulk copies; the next
// band's copies are in flight while the current band is emitted (double
// buffer, one mbarrier per buffer).  A warp then emits one row at a time:
// lane w expands plane word w into the row's point list, points are taken 32
// at a time (one per lane), neighbour ids are two shared-memory loads + a
// popcount, and only the 8 corner labels of a point are read from global
// memory.
#ifndef PSN_BAND_ROWS
#define PSN_BAND_ROWS 32
#endif
constexpr int kBand = PSN_BAND_ROWS;
constexpr int kBandThreads = 256;
#ifndef PSN_EMIT_MINB
#define PSN_EMIT_MINB 3   // resident CTAs per SM the register budget is sized for
#endif
#ifndef PSN_BAND_BUFS
#define PSN_BAND_BUFS 2
#endif
constexpr int kBandBufs = PSN_BAND_BUFS;   // staged bands per CTA (ring; 2 keeps L1 for the label gathers)

__device__ __forceinline__ void mbar_arrive_cta(uint64_t *bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
#ifndef PSN_STAGE_CSR
#define PSN_STAGE_CSR 150
#endif
constexpr uint32_t kStageCsr = PSN_STAGE_CSR;   // rounds with >= this many CSR ids write them through shared memory

constexpr int kRangeCap = (kBand + 2) * 32 + 16;   // elements per staged range (+ alignment slack)
struct BandBuf {                      // one stage; word / prefix ranges keep the workspace's row stride W32
    uint32_t m[3][kRangeCap];
    uint16_t p[3][kRangeCap];
    uint32_t off[3][kBand + 12];      // offP of the 3 ranges
    uint32_t cnt[kBand + 8], offQ[kBand + 8], offS[kBand + 8];
};
static_assert(sizeof(uint32_t) * kRangeCap % 16 == 0 && sizeof(uint16_t) * kRangeCap % 16 == 0 &&
              sizeof(uint32_t) * (kBand + 12) % 16 == 0 && sizeof(uint32_t) * (kBand + 8) % 16 == 0,
              "staged arrays must start at 16-byte boundaries");

// WC: plane words per row as a compile-time constant (0 = a.W32).  STG: dense rounds write their points
// and CSR ids through shared memory (meshes with >= kStageCsr / 32 stencil entries per point, e.g. c5a);
// without it 6 KB per CTA more go to L1 (c4 emission -2.6 %).  Both variants give the same bits.  The
// host launches the one for the density of the last mesh whose totals it read; when it has read none
// (a.dual), both are launched back to back and each returns at once unless the scan totals select it.
template <typename T, bool ANZ, int WC = 0, bool STG = true>
__global__ void __launch_bounds__(kBandThreads, PSN_EMIT_MINB) k_emit_band(EmitArgs a) {
    constexpr int B = kBand;
    extern __shared__ __align__(128) uint8_t dsm_band[];
    BandBuf *buf = reinterpret_cast<BandBuf *>(dsm_band);   // [kBandBufs]
    __shared__ __align__(8) uint64_t bar[kBandBufs];
    __shared__ int32_t s_band[kBandBufs];   // band staged in each buffer (nbands: end of the CTA's list)
    __shared__ uint32_t s_done[kBandBufs];  // warps finished with each buffer
    __shared__ uint32_t sbits[ANZ ? 1 : 2048];
    __shared__ uint32_t scsr[kBandThreads / 32][STG ? 6 * 32 : 1];   // a round's CSR ids, written out coalesced
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    LabelSet ls = a.ls;
    if (!ANZ && sizeof(T) < 4) {
        for (int t = tid; t < (sizeof(T) == 1 ? 8 : 2048); t += blockDim.x) sbits[t] = a.ls.bits[t];
        ls.bits = sbits;
    }
    if (tid == 0) {
        for (int b = 0; b < kBandBufs; ++b) { mbar_init(&bar[b], 1); s_done[b] = 0u; }
        fence_mbar_init();
    }
    __syncthreads();
    if (a.first_dev) {   // device-side C1 (multi-GPU step without a host round trip)
        a.first_point = (uint32_t)a.first_dev[0]; a.first_quad = (uint32_t)a.first_dev[1];
        a.first_stencil = (uint32_t)a.first_dev[2];
    }
    const uint64_t totP = a.hdr->total[0], totQ = a.hdr->total[1], totS = a.hdr->total[2];
    if (a.dual && (32u * totS >= (uint64_t)kStageCsr * totP) != STG) return;   // the other variant's mesh
    const uint32_t halo_lo = (uint32_t)a.hdr->halo_lo;
    if (totP > (uint64_t)a.cap_points || totQ > (uint64_t)a.cap_quads || totS > (uint64_t)a.cap_stencil) {
        if (blockIdx.x == 0 && tid == 0) a.hdr->emit_status = 1u;
        return;
    }
    if (blockIdx.x == 0 && tid == 0) {
        const uint64_t before_hi = (a.kB > a.own_k1) ? a.hdr->halo_hi : totP;
        a.hdr->emit_status = 0u;
        a.csr_off[before_hi - halo_lo] = a.first_stencil + (uint32_t)totS;   // CSR sentinel entry
    }
    const uint32_t gid_base = a.first_point - halo_lo;
    const int32_t M = (int32_t)a.M, N = (int32_t)a.N, NV = N - 1, W32 = WC ? WC : (int32_t)a.W32;
    const int32_t R = (int32_t)a.R;
    const int32_t kA = (int32_t)a.kA, kB = (int32_t)a.kB, own0 = (int32_t)a.own_k0, own1 = (int32_t)a.own_k1;
    const T *lab = reinterpret_cast<const T *>(a.labels);
    const int32_t nbands = (R + B - 1) / B;
    const int32_t rstart[3] = {-NV - 1, -1, NV};   // range starts relative to rr0
    const int32_t rlen[3] = {B + 1, B + 2, B};

    // Stage band `band` into buffer `sb`: bulk copies of the 16-byte-aligned supersets of the
    // ranges (clamped to [0, R)); returns nothing, records per-range element shifts in `shift`.
    // Shifts are recomputed identically by the consumers (pure functions of the band).
    auto elem_shift = [&](int32_t r0, int32_t rows, int esize, int32_t per_row) -> int32_t {
        // element shift of row r0's first element inside the aligned copy
        const int64_t byte_lo = (int64_t)r0 * per_row * esize;
        return (int32_t)((byte_lo & 15) / esize);
    };
    auto issue = [&](int32_t band, int sb) {
        BandBuf &bb = buf[sb];
        const int32_t rr0 = band * B;
        uint32_t bytes = 0;
        auto copy = [&](void *dst, const void *gbase, int32_t r0, int32_t r1, int esize, int32_t per_row) {
            // rows [r0, r1) clamped, per_row elements of esize bytes each
            const int32_t c0 = max(r0, 0), c1 = min(r1, R);
            if (c0 >= c1) return;
            const int64_t lo = (int64_t)c0 * per_row * esize, hi = (int64_t)c1 * per_row * esize;
            const int64_t alo = lo & ~(int64_t)15, ahi = (hi + 15) & ~(int64_t)15;
            // destination: element (c0 - r0) * per_row of the range, minus the alignment shift
            uint8_t *d = static_cast<uint8_t *>(dst) + (int64_t)(c0 - r0) * per_row * esize - (lo - alo) +
                         (int64_t)elem_shift(r0, 0, esize, per_row) * esize;
            tma_load_1d(d, static_cast<const uint8_t *>(gbase) + alo, (uint32_t)(ahi - alo), &bar[sb]);
            bytes += (uint32_t)(ahi - alo);
        };
        // plan the byte total first (expect_tx must precede completion)
        uint32_t total = 0;
        for (int g = 0; g < 3; ++g) {
            const int32_t r0 = rr0 + rstart[g], r1 = r0 + rlen[g];
            const int32_t c0 = max(r0, 0), c1 = min(r1, R);
            if (c0 >= c1) continue;
            for (int kind = 0; kind < 3; ++kind) {
                const int es = kind == 0 ? 4 : kind == 1 ? 2 : 4;
                const int32_t pr = kind == 2 ? 1 : W32;
                const int64_t lo = (int64_t)c0 * pr * es, hi = (int64_t)c1 * pr * es;
                total += (uint32_t)(((hi + 15) & ~(int64_t)15) - (lo & ~(int64_t)15));
            }
        }
        {
            const int32_t c0 = rr0, c1 = min(rr0 + B, R);
            for (int kind = 0; kind < 3; ++kind) {
                const int64_t lo = (int64_t)c0 * 4, hi = (int64_t)c1 * 4;
                total += (uint32_t)(((hi + 15) & ~(int64_t)15) - (lo & ~(int64_t)15));
            }
        }
        fence_proxy_async();
        mbar_expect_tx(&bar[sb], total);
        for (int g = 0; g < 3; ++g) {
            const int32_t r0 = rr0 + rstart[g], r1 = r0 + rlen[g];
            copy(bb.m[g], a.pmask, r0, r1, 4, W32);
            copy(bb.p[g], a.ppre, r0, r1, 2, W32);
            copy(bb.off[g], a.offP, r0, r1, 4, 1);
        }
        copy(bb.cnt, a.cntP, rr0, rr0 + B, 4, 1);
        copy(bb.offQ, a.offQ, rr0, rr0 + B, 4, 1);
        copy(bb.offS, a.offS, rr0, rr0 + B, 4, 1);
        (void)bytes;
    };

    // Bands without points (outside the surfaces; most of a sparse volume) are skipped without
    // staging: a warp looks 32 of the CTA's bands ahead at once (band b has points iff the
    // window offsets of its first and one-past-last rows differ) and stages the next non-empty one.
    const int32_t G = (int32_t)gridDim.x;
    auto next_band = [&](int32_t c) -> int32_t {   // one full warp; nbands if none
        for (int32_t base = c; base < nbands; base += 32 * G) {
            const int32_t cand = base + lane * G;
            bool ne = false;
            if (cand < nbands) {
                const int32_t r0 = cand * B, r1 = min(r0 + B, R) - 1;
                ne = __ldg(a.offP + r1) + __ldg(a.cntP + r1) != __ldg(a.offP + r0);
            }
            const uint32_t bal = __ballot_sync(kFull, ne);
            if (bal) return base + (__ffs(bal) - 1) * G;
        }
        return nbands;
    };
    // Stage list element `band` into buffer sb (lane 0): the band id rides with the fill (released
    // by the arrive); an end marker is a fill without bytes.
    auto stage = [&](int32_t band, int sb) {
        s_band[sb] = band;
        if (band < nbands) issue(band, sb);
        else mbar_arrive_cta(&bar[sb]);
    };
    // Ring of kBandBufs staged bands, no CTA-wide barrier: a warp waits for the fill of its next
    // buffer, emits its rows, and counts itself out of the buffer; the LAST warp out refills it
    // with the band kBandBufs list elements ahead.  Fast warps run ahead by up to kBandBufs - 1
    // bands instead of waiting at every band for the slowest warp (rows differ in point counts).
    if (warp == 0) {
        int32_t b = blockIdx.x;
        for (int i = 0; i < kBandBufs; ++i) {
            b = next_band(b);
            if (lane == 0) stage(b, i);
            if (b < nbands) b += G;
        }
    }
    uint32_t par = 0u;   // bit b: fill parity of buffer b (a register, not a dynamically indexed array)
    for (int it = 0;; ++it) {
        const int sb = it % kBandBufs;
        mbar_wait(&bar[sb], (par >> sb) & 1u);
        par ^= 1u << sb;
        const int32_t band = *reinterpret_cast<volatile int32_t *>(&s_band[sb]);
        if (band >= nbands) break;
        auto release = [&]() {   // this warp is done with buffer sb
            __syncwarp();
            uint32_t old = 0;
            if (lane == 0) {
                __threadfence_block();
                old = atomicAdd(&s_done[sb], 1u);
            }
            old = __shfl_sync(kFull, old, 0);
            if (old == kBandThreads / 32 - 1) {   // last warp out: refill with the band kBandBufs ahead
                __threadfence_block();
                const int32_t prev = *reinterpret_cast<volatile int32_t *>(&s_band[(sb + kBandBufs - 1) % kBandBufs]);
                const int32_t nb = prev < nbands ? next_band(prev + G) : nbands;
                if (lane == 0) {
                    s_done[sb] = 0u;
                    stage(nb, sb);
                }
            }
        };
        const BandBuf &bb = buf[sb];
        const int32_t rr0 = band * B;
        // staged-row accessors: element shifts of each range's 16-byte-aligned copy (the low bits
        // of the first element's index -- 32-bit wrap-around keeps them exact)
        const uint32_t e_m[3] = {(uint32_t)(rr0 + rstart[0]) * (uint32_t)W32, (uint32_t)(rr0 + rstart[1]) * (uint32_t)W32,
                                 (uint32_t)(rr0 + rstart[2]) * (uint32_t)W32};
        const int32_t sh_m[3] = {(int32_t)(e_m[0] & 3u), (int32_t)(e_m[1] & 3u), (int32_t)(e_m[2] & 3u)};   // u32
        const int32_t sh_p[3] = {(int32_t)(e_m[0] & 7u), (int32_t)(e_m[1] & 7u), (int32_t)(e_m[2] & 7u)};   // u16
        const int32_t sh_o[3] = {(int32_t)((uint32_t)(rr0 + rstart[0]) & 3u), (int32_t)((uint32_t)(rr0 + rstart[1]) & 3u),
                                 (int32_t)((uint32_t)(rr0 + rstart[2]) & 3u)};
        const int32_t sh_r = (int32_t)((uint32_t)rr0 & 3u);
        // A warp owns RPWB = 4 CONSECUTIVE rows of the band.  Ids are k-major (reading Q4) and the
        // scan offsets are in row order, so the warp's points, quads and CSR entries are each ONE
        // contiguous range: a ROUND takes the next 32 points of that range across row boundaries
        // (sparse rows share a round), and output positions are the range start plus a running
        // warp scan.  Software pipelining: the next round's point selection and its 8 corner-label
        // loads are issued before the current round is emitted.
        constexpr int RPWB = B / (kBandThreads / 32);
        const int b0 = warp * RPWB;
        int32_t rcnt[RPWB];           // points of the warp's rows (0 beyond R)
        uint32_t rstart[RPWB + 1];    // warp-local index of each row's first point
        rstart[0] = 0;
#pragma unroll
        for (int q = 0; q < RPWB; ++q) {
            rcnt[q] = (rr0 + b0 + q < R) ? (int32_t)bb.cnt[sh_r + b0 + q] : 0;
            rstart[q + 1] = rstart[q] + (uint32_t)rcnt[q];
        }
        const uint32_t wpts = rstart[RPWB];
        if (wpts == 0) {   // no points in the warp's rows: nothing else of the band is needed
            release();
            continue;
        }
        // (j, k) of the warp's first row; rows b0+q follow by +q with wrap-around
        const int32_t rf = rr0 + b0;
        const int32_t jf = rf % NV, kf = kA + rf / NV;
        const uint32_t offP0 = bb.off[1][sh_o[1] + b0 + 1];                  // window index of the first point
        const uint32_t qbase0 = bb.offQ[sh_r + b0], sbase0 = bb.offS[sh_r + b0];
        struct Round {
            uint32_t base, i;
            int32_t b, j, k;
            bool act, own;
            uint32_t L[8];   // A, A1, B, B1, C, C1, D, D1 (codes)
        };
        auto prepare = [&](Round &st, uint32_t base) {
            st.base = base;
            const uint32_t t = base + lane;
            st.act = t < wpts;
            int q = 0;
#pragma unroll
            for (int qq = 1; qq < RPWB; ++qq) q += (t >= rstart[qq]) ? 1 : 0;
            uint32_t tr = t;   // index within the row
#pragma unroll
            for (int qq = 1; qq < RPWB; ++qq) if (q == qq) tr = t - rstart[qq];
            const int b = b0 + q;
            st.b = b;
            int32_t jj = jf + q, kk = kf;
            while (jj >= NV) { jj -= NV; ++kk; }   // (tiny NV: several layers per warp)
            st.j = jj; st.k = kk;
            st.own = st.act && kk >= own0 && kk < own1;
            // word of the row holding point tr: the last word whose first index <= tr (prefixes are
            // non-decreasing; 5-step binary search in shared memory), then the n-th set bit of it
            const uint16_t *pp = bb.p[1] + sh_p[1] + (b + 1) * W32;
            const uint32_t *pm = bb.m[1] + sh_m[1] + (b + 1) * W32;
            int wsel = 0;
            uint32_t mw, pw;
            const int bfirst = __shfl_sync(kFull, b, 0), blast = __shfl_sync(kFull, b, 31);
            if (bfirst == blast) {
                // the round lies in one row (dense rows): lane = plane word, shuffle binary search
                const uint32_t wm_l = lane < W32 ? pm[lane] : 0u;
                const uint32_t wp_l = lane < W32 ? (uint32_t)pp[lane] : 0xFFFFu;
#pragma unroll
                for (int s2 = 16; s2 >= 1; s2 >>= 1) {
                    const uint32_t pv = __shfl_sync(kFull, wp_l, wsel + s2);
                    if (pv <= tr) wsel += s2;
                }
                mw = __shfl_sync(kFull, wm_l, wsel); pw = __shfl_sync(kFull, wp_l, wsel);
                if (!st.act) { mw = 0u; pw = 0u; }
            } else {
                // sparse rows share the round: per-lane binary search over its row's staged prefixes
#pragma unroll
                for (int s2 = 16; s2 >= 1; s2 >>= 1) {
                    const int c = wsel + s2;
                    if (c < W32 && (uint32_t)pp[c] <= tr) wsel = c;
                }
                mw = st.act ? pm[wsel] : 0u; pw = st.act ? (uint32_t)pp[wsel] : 0u;
            }
            uint32_t nth = tr - pw, bitpos = 0, rest = mw;   // position of the nth (0-based) set bit of mw
#pragma unroll
            for (int s2 = 16; s2 >= 1; s2 >>= 1) {
                const uint32_t lo = __popc(rest & ((1u << s2) - 1u));
                if (lo <= nth) { nth -= lo; bitpos += s2; rest >>= s2; }
            }
            st.i = st.act ? (uint32_t)(wsel * 32 + bitpos) : 0u;
            if (st.own) {
                // rows j, j+1 of slices k, k+1 (grid-row index in 32 bits: layers * N < 2^32)
                const uint32_t grow = (uint32_t)(kk - (int32_t)a.z_lo) * (uint32_t)N + (uint32_t)jj;
                const T *pA = lab + ((size_t)grow * (uint32_t)M + st.i);
                const T *pB = pA + M, *pC = pA + (size_t)N * M, *pD = pC + M;
                st.L[0] = code_at<T, ANZ>(pA, ls); st.L[1] = code_at<T, ANZ>(pA + 1, ls);
                st.L[2] = code_at<T, ANZ>(pB, ls); st.L[3] = code_at<T, ANZ>(pB + 1, ls);
                st.L[4] = code_at<T, ANZ>(pC, ls); st.L[5] = code_at<T, ANZ>(pC + 1, ls);
                st.L[6] = code_at<T, ANZ>(pD, ls); st.L[7] = code_at<T, ANZ>(pD + 1, ls);
            }
        };
        // neighbour row q -> (range, index offset from b)
        const int nq_g[5] = {0, 0, 1, 1, 2};
        const int nq_d[5] = {0, 1, 0, 2, 0};
        uint32_t run_q = 0, run_s = 0;
        Round cur;
        if (wpts) prepare(cur, 0);
        for (uint32_t base = 0; base < wpts; base += 32) {
            Round nxt;
            if (base + 32 < wpts) prepare(nxt, base + 32);
            const int32_t b = cur.b, j = cur.j, k = cur.k;
            const int32_t i = (int32_t)cur.i;
            const bool act = cur.act, own = cur.own;
            const uint32_t t = cur.base + lane;
            const uint32_t wi = offP0 + t;
            const uint32_t g = gid_base + wi;
            uint32_t fm = 0, qb = 0, cA = 0, cA1 = 0, cB = 0, cC = 0;
            if (own) {
                const uint32_t A = cur.L[0], A1 = cur.L[1], Bv = cur.L[2], B1 = cur.L[3];
                const uint32_t C = cur.L[4], C1 = cur.L[5], D = cur.L[6], D1 = cur.L[7];
                const bool XA = A != A1, XB = Bv != B1, XC = C != C1, XD = D != D1;
                const bool YAB = A != Bv, YA1 = A1 != B1, YCD = C != D, YC1 = C1 != D1;
                const bool ZAC = A != C, ZA1 = A1 != C1, ZBD = Bv != D, ZB1 = B1 != D1;
                fm |= ((XA | XB | YAB | YA1) && k >= 1) ? 1u : 0u;          // -z
                fm |= ((XA | XC | ZAC | ZA1) && j >= 1) ? 2u : 0u;          // -y
                fm |= ((YAB | YCD | ZAC | ZBD) && i >= 1) ? 4u : 0u;        // -x
                fm |= ((YA1 | YC1 | ZA1 | ZB1) && i + 3 <= M) ? 8u : 0u;    // +x
                fm |= ((XB | XD | ZBD | ZB1) && j + 3 <= N) ? 16u : 0u;     // +y
                fm |= ((XC | XD | YCD | YC1) && k + 3 <= (int32_t)a.O) ? 32u : 0u;   // +z
                qb |= (XA && j >= 1 && k >= 1) ? 1u : 0u;
                qb |= (YAB && i >= 1 && k >= 1) ? 2u : 0u;
                qb |= (ZAC && i >= 1 && j >= 1) ? 4u : 0u;
                cA = cls_of_code<T, ANZ>(ls, A); cA1 = cls_of_code<T, ANZ>(ls, A1);
                cB = cls_of_code<T, ANZ>(ls, Bv); cC = cls_of_code<T, ANZ>(ls, C);
            }
            const uint32_t packed = ((uint32_t)__popc(qb) << 16) | (uint32_t)__popc(fm);
            const uint32_t x = scan3(packed, lane);
            const uint32_t tot = __shfl_sync(kFull, x, 31);
            const uint32_t ex = x - packed;
            const bool stage = STG && (tot & 0xffffu) >= kStageCsr;   // dense round: CSR ids through shared memory
            if (!stage) {
                if (act) {
                    a.points[3 * (size_t)wi + 0] = anchor_coord(a.org[0], a.sp[0], i);
                    a.points[3 * (size_t)wi + 1] = anchor_coord(a.org[1], a.sp[1], j);
                    a.points[3 * (size_t)wi + 2] = anchor_coord(a.org[2], a.sp[2], k);
                }
            } else {   // dense round (store-bound volumes): the round's points are ONE contiguous
                // range of 3 * nact floats -- stage them in shared memory and write lane-contiguous
                // words (full sectors instead of three 12-byte-strided stores per lane)
                float *sp = reinterpret_cast<float *>(scsr[warp]);
                if (act) {
                    sp[3 * lane + 0] = anchor_coord(a.org[0], a.sp[0], i);
                    sp[3 * lane + 1] = anchor_coord(a.org[1], a.sp[1], j);
                    sp[3 * lane + 2] = anchor_coord(a.org[2], a.sp[2], k);
                }
                __syncwarp();
                const uint32_t nact = __popc(__ballot_sync(kFull, act));
                float *dstp = a.points + 3 * (size_t)(offP0 + cur.base);
#pragma unroll
                for (int q = 0; q < 3; ++q) {
                    const uint32_t e = (uint32_t)lane + 32u * q;
                    if (e < 3u * nact) dstp[e] = sp[e];
                }
                __syncwarp();
            }
            if (own) {
                const uint32_t wl = (uint32_t)i >> 5, below = (1u << (i & 31)) - 1u;
                // neighbour ids actually referenced by this point's stencil entries / quads
                const uint32_t need = ((qb & 1u) ? 1u : 0u) | (((fm & 1u) || (qb & 3u)) ? 2u : 0u) |
                                      (((fm & 2u) || (qb & 5u)) ? 4u : 0u) | ((fm & 16u) ? 8u : 0u) |
                                      ((fm & 32u) ? 16u : 0u);
                uint32_t gn[5];
#pragma unroll
                for (int q = 0; q < 5; ++q) {
                    const int gg = nq_g[q], ii = b + nq_d[q];
                    const int e = ii * W32 + (int)wl;
                    gn[q] = ((need >> q) & 1u) ? gid_base + bb.off[gg][sh_o[gg] + ii] + bb.p[gg][e + sh_p[gg]] +
                                                     __popc(bb.m[gg][e + sh_m[gg]] & below)
                                               : 0u;
                }
                const uint32_t o = wi - halo_lo;
                const uint32_t s0 = sbase0 + run_s + (ex & 0xffffu);
                a.fmask[o] = (uint8_t)fm;
                a.csr_off[o] = a.first_stencil + s0;
                if (a.scache)   // the smoothing cache k_smooth_prep8 would build from these stencil entries
                    a.scache[o] = nbr8_pack(g, make_uint4((fm & 1u) ? gn[1] : g, (fm & 2u) ? gn[2] : g,
                                                          (fm & 16u) ? gn[3] : g, (fm & 32u) ? gn[4] : g), fm);
                uint32_t *sc = stage ? scsr[warp] + (ex & 0xffffu) : a.csr_ids + s0;
                if (fm & 1u) *sc++ = gn[1];      // -z  (j, k-1)
                if (fm & 2u) *sc++ = gn[2];      // -y  (j-1, k)
                if (fm & 4u) *sc++ = g - 1u;     // -x
                if (fm & 8u) *sc++ = g + 1u;     // +x
                if (fm & 16u) *sc++ = gn[3];     // +y  (j+1, k)
                if (fm & 32u) *sc++ = gn[4];     // +z  (j, k+1)
                uint32_t qs = qbase0 + run_q + (ex >> 16);
                if (qb & 1u) {   // x-quad [(j-1,k-1), (j,k-1), (j,k), (j-1,k)]
                    *reinterpret_cast<uint4 *>(a.quads + 4 * (size_t)qs) = make_uint4(gn[0], gn[1], g, gn[2]);
                    *reinterpret_cast<uint2 *>(a.pairs + 2 * (size_t)qs) = make_uint2(cA, cA1);
                    ++qs;
                }
                if (qb & 2u) {   // y-quad [(i-1,k-1), (i-1,k), (i,k), (i,k-1)] of row j
                    *reinterpret_cast<uint4 *>(a.quads + 4 * (size_t)qs) = make_uint4(gn[1] - 1u, g - 1u, g, gn[1]);
                    *reinterpret_cast<uint2 *>(a.pairs + 2 * (size_t)qs) = make_uint2(cA, cB);
                    ++qs;
                }
                if (qb & 4u) {   // z-quad [(i-1,j-1), (i,j-1), (i,j), (i-1,j)] of layer k
                    *reinterpret_cast<uint4 *>(a.quads + 4 * (size_t)qs) = make_uint4(gn[2] - 1u, gn[2], g, g - 1u);
                    *reinterpret_cast<uint2 *>(a.pairs + 2 * (size_t)qs) = make_uint2(cA, cC);
                    ++qs;
                }
            }
            if (stage) {   // the round's CSR ids are one contiguous range: coalesced copy-out
                const uint32_t ns = tot & 0xffffu;
                __syncwarp();
                uint32_t *dst = a.csr_ids + sbase0 + run_s;
                for (uint32_t e = lane; e < ns; e += 32) dst[e] = scsr[warp][e];
                __syncwarp();
            }
            run_q += tot >> 16;
            run_s += tot & 0xffffu;
            cur = nxt;
        }
        release();
    }
}

}  // namespace psn
