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
    ScanHeader *hdr;
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

}  // namespace psn
