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

template <typename T, bool ANZ>
__global__ void __launch_bounds__(256) k_emit(EmitArgs a) {
    __shared__ uint32_t sbits[ANZ ? 1 : 2048];
    __shared__ uint16_t slist[kEmitWarps][1024];      // point x positions of the current 1024-voxel block
    __shared__ uint32_t sword[kEmitWarps][5][32];     // neighbour rows: mask word
    __shared__ uint32_t spre[kEmitWarps][5][32];      // neighbour rows: points before the word
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    LabelSet ls = a.ls;
    if (!ANZ && sizeof(T) < 4) {
        for (int t = threadIdx.x; t < (sizeof(T) == 1 ? 8 : 2048); t += blockDim.x) sbits[t] = a.ls.bits[t];
        ls.bits = sbits;
        __syncthreads();
    }
    // device-side capacity check (steady-state COUNT|EMIT path)
    const uint64_t totP = a.hdr->total[0], totQ = a.hdr->total[1], totS = a.hdr->total[2];
    const uint64_t halo_lo = a.hdr->halo_lo;
    if (totP > (uint64_t)a.cap_points || totQ > (uint64_t)a.cap_quads || totS > (uint64_t)a.cap_stencil) {
        if (blockIdx.x == 0 && threadIdx.x == 0) a.hdr->emit_status = 1u;
        return;
    }
    const uint64_t before_hi = (a.kB > a.own_k1) ? a.hdr->halo_hi : totP;
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        a.hdr->emit_status = 0u;
        a.csr_off[before_hi - halo_lo] = a.first_stencil + (uint32_t)totS;   // CSR sentinel entry
    }
    const uint32_t gid_base = a.first_point - (uint32_t)halo_lo;   // global id of window index 0
    const int64_t M = a.M, N = a.N, NV = N - 1, W32 = a.W32;
    const T *lab = reinterpret_cast<const T *>(a.labels);
    const uint32_t lt = (1u << lane) - 1u;

    const int64_t warps = (int64_t)gridDim.x * (blockDim.x >> 5);
    for (int64_t rr = blockIdx.x * (int64_t)(blockDim.x >> 5) + warp; rr < a.R; rr += warps) {
        if (__ldg(a.cntP + rr) == 0) continue;
        const int64_t j = rr % NV, k = a.kA + rr / NV;
        const bool own = (k >= a.own_k0) && (k < a.own_k1);
        int64_t nb[5];
        nb[0] = (own && j >= 1 && k - 1 >= a.kA) ? rr - NV - 1 : -1;   // (j-1,k-1)
        nb[1] = (own && k - 1 >= a.kA) ? rr - NV : -1;                  // (j,  k-1)
        nb[2] = (own && j >= 1) ? rr - 1 : -1;                           // (j-1,k)
        nb[3] = (own && j + 1 <= N - 2) ? rr + 1 : -1;                   // (j+1,k)
        nb[4] = (own && k + 1 < a.kB) ? rr + NV : -1;                    // (j,  k+1)
        const uint32_t offP = __ldg(a.offP + rr);
        uint32_t nbase[5];
#pragma unroll
        for (int q = 0; q < 5; ++q) nbase[q] = nb[q] >= 0 ? __ldg(a.offP + nb[q]) : 0u;
        const uint32_t qbase = own ? __ldg(a.offQ + rr) : 0u, sbase = own ? __ldg(a.offS + rr) : 0u;
        uint32_t run_o = 0, run_q = 0, run_s = 0;
        uint32_t run_n[5] = {0, 0, 0, 0, 0};
        const T *rowA = lab + ((k - a.z_lo) * N + j) * M;
        const T *rowB = rowA + M;
        const T *rowC = rowA + N * M;
        const T *rowD = rowC + M;

        for (int64_t w0 = 0; w0 < W32; w0 += 32) {
            const int64_t w = w0 + lane;
            const bool wok = w < W32;
            const uint32_t om = wok ? __ldg(a.pmask + rr * W32 + w) : 0u;
            // own points: exclusive scan of the word popcounts -> compact list
            const uint32_t oc = __popc(om);
            uint32_t oi = oc;
#pragma unroll
            for (int d = 1; d < 32; d <<= 1) { const uint32_t y = __shfl_up_sync(kFull, oi, d); if (lane >= d) oi += y; }
            const uint32_t blk_pts = __shfl_sync(kFull, oi, 31);
            if (blk_pts == 0) {
                if (own) {
#pragma unroll
                    for (int q = 0; q < 5; ++q) {
                        const uint32_t m = (nb[q] >= 0 && wok) ? __ldg(a.pmask + nb[q] * W32 + w) : 0u;
                        run_n[q] += __reduce_add_sync(kFull, __popc(m));
                    }
                }
                continue;
            }
            {
                uint32_t pos = oi - oc, m = om;
                while (m) {
                    const int b = __ffs(m) - 1;
                    m &= m - 1;
                    slist[warp][pos++] = (uint16_t)(lane * 32 + b);
                }
            }
            uint32_t blk_n[5] = {0, 0, 0, 0, 0};
            if (own) {
#pragma unroll
                for (int q = 0; q < 5; ++q) {
                    const uint32_t m = (nb[q] >= 0 && wok) ? __ldg(a.pmask + nb[q] * W32 + w) : 0u;
                    const uint32_t c = __popc(m);
                    uint32_t x = c;
#pragma unroll
                    for (int d = 1; d < 32; d <<= 1) { const uint32_t y = __shfl_up_sync(kFull, x, d); if (lane >= d) x += y; }
                    sword[warp][q][lane] = m;
                    spre[warp][q][lane] = run_n[q] + x - c;
                    blk_n[q] = __shfl_sync(kFull, x, 31);
                }
            }
            __syncwarp();
            for (uint32_t base = 0; base < blk_pts; base += 32) {
                const uint32_t t = base + lane;
                const bool act = t < blk_pts;
                const uint32_t xb = act ? slist[warp][t] : 0u;          // position within the block
                const int64_t i = w0 * 32 + xb;                          // voxel x
                const uint32_t n = run_o + t;                            // index of the point in the row
                const uint32_t wi = offP + n;                            // window index
                const uint32_t g = gid_base + wi;                        // global id
                uint32_t fm = 0, qb = 0, deg = 0;
                uint32_t cA = 0, cA1 = 0, cB = 0, cC = 0;
                uint32_t gn[5] = {0, 0, 0, 0, 0};
                if (act && own) {
                    const uint32_t A = code_at<T, ANZ>(rowA + i, ls), A1 = code_at<T, ANZ>(rowA + i + 1, ls);
                    const uint32_t B = code_at<T, ANZ>(rowB + i, ls), B1 = code_at<T, ANZ>(rowB + i + 1, ls);
                    const uint32_t C = code_at<T, ANZ>(rowC + i, ls), C1 = code_at<T, ANZ>(rowC + i + 1, ls);
                    const uint32_t D = code_at<T, ANZ>(rowD + i, ls), D1 = code_at<T, ANZ>(rowD + i + 1, ls);
                    const bool XA = A != A1, XB = B != B1, XC = C != C1, XD = D != D1;
                    const bool YAB = A != B, YA1 = A1 != B1, YCD = C != D, YC1 = C1 != D1;
                    const bool ZAC = A != C, ZA1 = A1 != C1, ZBD = B != D, ZB1 = B1 != D1;
                    fm |= ((XA | XB | YAB | YA1) && k >= 1) ? 1u : 0u;          // -z
                    fm |= ((XA | XC | ZAC | ZA1) && j >= 1) ? 2u : 0u;          // -y
                    fm |= ((YAB | YCD | ZAC | ZBD) && i >= 1) ? 4u : 0u;        // -x
                    fm |= ((YA1 | YC1 | ZA1 | ZB1) && i <= M - 3) ? 8u : 0u;    // +x
                    fm |= ((XB | XD | ZBD | ZB1) && j <= N - 3) ? 16u : 0u;     // +y
                    fm |= ((XC | XD | YCD | YC1) && k <= a.O - 3) ? 32u : 0u;   // +z
                    qb |= (XA && j >= 1 && k >= 1) ? 1u : 0u;
                    qb |= (YAB && i >= 1 && k >= 1) ? 2u : 0u;
                    qb |= (ZAC && i >= 1 && j >= 1) ? 4u : 0u;
                    deg = __popc(fm);
                    cA = cls_of_code<T, ANZ>(ls, A); cA1 = cls_of_code<T, ANZ>(ls, A1);
                    cB = cls_of_code<T, ANZ>(ls, B); cC = cls_of_code<T, ANZ>(ls, C);
                    const int wl = (int)(xb >> 5);
                    const uint32_t below = (1u << (xb & 31)) - 1u;
#pragma unroll
                    for (int q = 0; q < 5; ++q)
                        gn[q] = gid_base + nbase[q] + spre[warp][q][wl] + __popc(sword[warp][q][wl] & below);
                }
                // warp exclusive scan of (quads << 16 | degree)
                const uint32_t packed = ((uint32_t)__popc(qb) << 16) | deg;
                uint32_t x = packed;
#pragma unroll
                for (int d = 1; d < 32; d <<= 1) { const uint32_t y = __shfl_up_sync(kFull, x, d); if (lane >= d) x += y; }
                const uint32_t tot = __shfl_sync(kFull, x, 31);
                const uint32_t ex = x - packed;
                if (act) {
                    a.points[3 * (int64_t)wi + 0] = anchor_coord(a.org[0], a.sp[0], i);
                    a.points[3 * (int64_t)wi + 1] = anchor_coord(a.org[1], a.sp[1], j);
                    a.points[3 * (int64_t)wi + 2] = anchor_coord(a.org[2], a.sp[2], k);
                    if (own) {
                        const uint32_t o = wi - (uint32_t)halo_lo;
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
                            *reinterpret_cast<uint4 *>(a.quads + 4 * (int64_t)qs) = make_uint4(gn[0], gn[1], g, gn[2]);
                            *reinterpret_cast<uint2 *>(a.pairs + 2 * (int64_t)qs) = make_uint2(cA, cA1);
                            ++qs;
                        }
                        if (qb & 2u) {   // y-quad [(i-1,k-1), (i-1,k), (i,k), (i,k-1)] of row j
                            *reinterpret_cast<uint4 *>(a.quads + 4 * (int64_t)qs) = make_uint4(gn[1] - 1u, g - 1u, g, gn[1]);
                            *reinterpret_cast<uint2 *>(a.pairs + 2 * (int64_t)qs) = make_uint2(cA, cB);
                            ++qs;
                        }
                        if (qb & 4u) {   // z-quad [(i-1,j-1), (i,j-1), (i,j), (i-1,j)] of layer k
                            *reinterpret_cast<uint4 *>(a.quads + 4 * (int64_t)qs) = make_uint4(gn[2] - 1u, gn[2], g, g - 1u);
                            *reinterpret_cast<uint2 *>(a.pairs + 2 * (int64_t)qs) = make_uint2(cA, cC);
                            ++qs;
                        }
                    }
                }
                run_q += tot >> 16;
                run_s += tot & 0xffffu;
            }
            run_o += blk_pts;
#pragma unroll
            for (int q = 0; q < 5; ++q) run_n[q] += blk_n[q];
            __syncwarp();
        }
    }
}

}  // namespace psn
