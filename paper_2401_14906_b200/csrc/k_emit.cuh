// k_emit.cuh -- Pass 4 of PSN extraction on sm_100a.
//
// One warp per voxel row V_{j,k} (grid-stride), walking the row's 128-voxel
// chunks left to right.  The paper's 3x3 voxel-row iterator (Fig. 6)
// becomes a prefix-popc over the stored point bit-planes of the needed
// neighbour rows: every voxel's point id, and the ids of the neighbours its
// quads and stencil reference, are
//     window_base + offP[row'] + (points of row' before this chunk)
//                 + popc(planes of row' below this voxel inside the chunk).
// Quads use rows (j-1,k-1), (j,k-1), (j-1,k); the stencil adds (j+1,k) and
// (j,k+1).  Chunks with no point are skipped without touching the labels
// ("the trim interval plays an important role ... to rapidly skip data").
// All writes land in disjoint, preallocated slots given by the scan -- no
// atomics, no locks.
#pragma once
#include "k_scan.cuh"
#include "psn_common.cuh"

namespace psn {

struct EmitArgs {
    const void *labels;
    int64_t M, N, O, z_lo;
    int64_t kA, kB, own_k0, own_k1, W4, R;
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

__device__ __forceinline__ uint32_t popc4(uint4 m, uint32_t lt) {
    return __popc(m.x & lt) + __popc(m.y & lt) + __popc(m.z & lt) + __popc(m.w & lt);
}
__device__ __forceinline__ uint32_t bitp(uint4 m, int p, int lane) {
    uint32_t w = p == 0 ? m.x : p == 1 ? m.y : p == 2 ? m.z : m.w;
    return (w >> lane) & 1u;
}
__device__ __forceinline__ uint32_t popc_all(uint4 m) {
    return __popc(m.x) + __popc(m.y) + __popc(m.z) + __popc(m.w);
}
__device__ __forceinline__ uint4 ld_mask(const uint32_t *pm, int64_t row, int64_t W4, int64_t c) {
    if (row < 0) return make_uint4(0, 0, 0, 0);
    return __ldg(reinterpret_cast<const uint4 *>(pm + (row * W4 + c) * 4));
}

template <typename T, bool ANZ, bool VEC>
__global__ void __launch_bounds__(256) k_emit(EmitArgs a) {
    constexpr int NW = Pack<T>::NW;
    __shared__ uint32_t sbits[ANZ ? 1 : 2048];
    const int lane = threadIdx.x & 31;
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
    const int64_t M = a.M, N = a.N, NV = N - 1;
    const T *lab = reinterpret_cast<const T *>(a.labels);

    const int64_t warps = (int64_t)gridDim.x * (blockDim.x >> 5);
    for (int64_t rr = blockIdx.x * (int64_t)(blockDim.x >> 5) + (threadIdx.x >> 5); rr < a.R; rr += warps) {
        if (__ldg(a.cntP + rr) == 0) continue;
        const int64_t j = rr % NV, k = a.kA + rr / NV;
        const bool own = (k >= a.own_k0) && (k < a.own_k1);
        const int64_t n1 = (own && j >= 1 && k - 1 >= a.kA) ? rr - NV - 1 : -1;   // (j-1,k-1)
        const int64_t n2 = (own && k - 1 >= a.kA) ? rr - NV : -1;                  // (j,  k-1)
        const int64_t n3 = (own && j >= 1) ? rr - 1 : -1;                           // (j-1,k)
        const int64_t n4 = (own && j + 1 <= N - 2) ? rr + 1 : -1;                   // (j+1,k)
        const int64_t n5 = (own && k + 1 < a.kB) ? rr + NV : -1;                    // (j,  k+1)
        const uint32_t offP = __ldg(a.offP + rr);
        const uint32_t b1 = n1 >= 0 ? __ldg(a.offP + n1) : 0u, b2 = n2 >= 0 ? __ldg(a.offP + n2) : 0u;
        const uint32_t b3 = n3 >= 0 ? __ldg(a.offP + n3) : 0u, b4 = n4 >= 0 ? __ldg(a.offP + n4) : 0u;
        const uint32_t b5 = n5 >= 0 ? __ldg(a.offP + n5) : 0u;
        const uint32_t qbase = own ? __ldg(a.offQ + rr) : 0u, sbase = own ? __ldg(a.offS + rr) : 0u;
        uint32_t run_o = 0, run1 = 0, run2 = 0, run3 = 0, run4 = 0, run5 = 0, run_q = 0, run_s = 0;
        const T *rowA = lab + ((k - a.z_lo) * N + j) * M;
        const T *rowB = rowA + M;
        const T *rowC = rowA + N * M;
        const T *rowD = rowC + M;
        const uint32_t lt = (1u << lane) - 1u;

        for (int64_t c = 0; c < a.W4; ++c) {
            const uint4 po = ld_mask(a.pmask, rr, a.W4, c);
            const uint4 m1 = ld_mask(a.pmask, n1, a.W4, c), m2 = ld_mask(a.pmask, n2, a.W4, c);
            const uint4 m3 = ld_mask(a.pmask, n3, a.W4, c), m4 = ld_mask(a.pmask, n4, a.W4, c);
            const uint4 m5 = ld_mask(a.pmask, n5, a.W4, c);
            if (po.x | po.y | po.z | po.w) {
                const int64_t x0 = 128 * c + 4 * lane;
                uint32_t bits[4];
                uint32_t np = 0;
#pragma unroll
                for (int p = 0; p < 4; ++p) { bits[p] = bitp(po, p, lane); np += bits[p]; }
                const uint32_t pre_o = run_o + popc4(po, lt);
                if (!own) {
                    // halo layer: points only (window entries needed by smoothing / triangulation)
                    uint32_t acc = 0;
#pragma unroll
                    for (int p = 0; p < 4; ++p) {
                        if (!bits[p]) continue;
                        const uint32_t w = offP + pre_o + acc++;
                        a.points[3 * (int64_t)w + 0] = anchor_coord(a.org[0], a.sp[0], x0 + p);
                        a.points[3 * (int64_t)w + 1] = anchor_coord(a.org[1], a.sp[1], j);
                        a.points[3 * (int64_t)w + 2] = anchor_coord(a.org[2], a.sp[2], k);
                    }
                } else {
                    // labels of the voxel row's four grid rows (chunk + next element)
                    uint32_t A[NW], B[NW], C[NW], D[NW], hA[NW], hB[NW], hC[NW], hD[NW];
                    load_chunk<T, VEC>(rowA, x0, M, A);
                    load_chunk<T, VEC>(rowB, x0, M, B);
                    load_chunk<T, VEC>(rowC, x0, M, C);
                    load_chunk<T, VEC>(rowD, x0, M, D);
                    if (!ANZ) { remap<T>(ls, A); remap<T>(ls, B); remap<T>(ls, C); remap<T>(ls, D); }
                    uint32_t nA = __shfl_down_sync(kFull, A[0], 1), nB = __shfl_down_sync(kFull, B[0], 1);
                    uint32_t nC = __shfl_down_sync(kFull, C[0], 1), nD = __shfl_down_sync(kFull, D[0], 1);
                    if (lane == 31) {
                        nA = load_word<T, VEC>(rowA, x0 + 4, M); nB = load_word<T, VEC>(rowB, x0 + 4, M);
                        nC = load_word<T, VEC>(rowC, x0 + 4, M); nD = load_word<T, VEC>(rowD, x0 + 4, M);
                        if (!ANZ) { nA = remap1<T>(ls, nA); nB = remap1<T>(ls, nB); nC = remap1<T>(ls, nC); nD = remap1<T>(ls, nD); }
                    }
                    shift1<T>(A, nA, hA); shift1<T>(B, nB, hB); shift1<T>(C, nC, hC); shift1<T>(D, nD, hD);
                    uint32_t XA[NW], YAB[NW], ZAC[NW], Fmx[NW], Fpx[NW], Fmy[NW], Fpy[NW], Fmz[NW], Fpz[NW];
#pragma unroll
                    for (int q = 0; q < NW; ++q) {
                        XA[q] = neq<T>(A[q], hA[q]);
                        const uint32_t XB = neq<T>(B[q], hB[q]), XC = neq<T>(C[q], hC[q]), XD = neq<T>(D[q], hD[q]);
                        YAB[q] = neq<T>(A[q], B[q]);
                        const uint32_t YCD = neq<T>(C[q], D[q]);
                        ZAC[q] = neq<T>(A[q], C[q]);
                        const uint32_t ZBD = neq<T>(B[q], D[q]);
                        const uint32_t YABs = neq<T>(hA[q], hB[q]), YCDs = neq<T>(hC[q], hD[q]);
                        const uint32_t ZACs = neq<T>(hA[q], hC[q]), ZBDs = neq<T>(hB[q], hD[q]);
                        Fmx[q] = YAB[q] | YCD | ZAC[q] | ZBD;
                        Fpx[q] = YABs | YCDs | ZACs | ZBDs;
                        Fmy[q] = XA[q] | XC | ZAC[q] | ZACs;
                        Fpy[q] = XB | XD | ZBD | ZBDs;
                        Fmz[q] = XA[q] | XB | YAB[q] | YABs;
                        Fpz[q] = XC | XD | YCD | YCDs;
                    }
                    uint32_t fm[4], qb[4];
                    uint32_t nq = 0, ns = 0;
#pragma unroll
                    for (int p = 0; p < 4; ++p) {
                        const int64_t i = x0 + p;
                        uint32_t f = 0, qq = 0;
                        if (bits[p]) {
                            f |= (flag<T>(Fmz, p) && k >= 1) ? 1u : 0u;
                            f |= (flag<T>(Fmy, p) && j >= 1) ? 2u : 0u;
                            f |= (flag<T>(Fmx, p) && i >= 1) ? 4u : 0u;
                            f |= (flag<T>(Fpx, p) && i <= M - 3) ? 8u : 0u;
                            f |= (flag<T>(Fpy, p) && j <= N - 3) ? 16u : 0u;
                            f |= (flag<T>(Fpz, p) && k <= a.O - 3) ? 32u : 0u;
                            qq |= (flag<T>(XA, p) && j >= 1 && k >= 1) ? 1u : 0u;
                            qq |= (flag<T>(YAB, p) && i >= 1 && k >= 1) ? 2u : 0u;
                            qq |= (flag<T>(ZAC, p) && i >= 1 && j >= 1) ? 4u : 0u;
                        }
                        fm[p] = f; qb[p] = qq;
                        nq += __popc(qq); ns += __popc(f);
                    }
                    // warp exclusive scan of packed (points, quads, stencil entries)
                    const uint32_t packed = (np << 20) | (nq << 10) | ns;
                    uint32_t x = packed;
#pragma unroll
                    for (int d = 1; d < 32; d <<= 1) {
                        const uint32_t y = __shfl_up_sync(kFull, x, d);
                        if (lane >= d) x += y;
                    }
                    const uint32_t tot = __shfl_sync(kFull, x, 31);
                    const uint32_t ex = x - packed;
                    uint32_t qslot = qbase + run_q + ((ex >> 10) & 1023u);
                    uint32_t sslot = sbase + run_s + (ex & 1023u);
                    const uint32_t p1 = b1 + run1 + popc4(m1, lt), p2 = b2 + run2 + popc4(m2, lt);
                    const uint32_t p3 = b3 + run3 + popc4(m3, lt), p4 = b4 + run4 + popc4(m4, lt);
                    const uint32_t p5 = b5 + run5 + popc4(m5, lt);
                    uint32_t acc = 0, a1 = 0, a2 = 0, a3 = 0, a4 = 0, a5 = 0;
#pragma unroll
                    for (int p = 0; p < 4; ++p) {
                        if (bits[p]) {
                            const int64_t i = x0 + p;
                            const uint32_t w = offP + pre_o + acc;
                            const uint32_t g = gid_base + w;
                            const uint32_t g1 = gid_base + p1 + a1, g2 = gid_base + p2 + a2;
                            const uint32_t g3 = gid_base + p3 + a3, g4 = gid_base + p4 + a4;
                            const uint32_t g5 = gid_base + p5 + a5;
                            a.points[3 * (int64_t)w + 0] = anchor_coord(a.org[0], a.sp[0], i);
                            a.points[3 * (int64_t)w + 1] = anchor_coord(a.org[1], a.sp[1], j);
                            a.points[3 * (int64_t)w + 2] = anchor_coord(a.org[2], a.sp[2], k);
                            const uint32_t o = w - (uint32_t)halo_lo;
                            a.fmask[o] = (uint8_t)fm[p];
                            a.csr_off[o] = a.first_stencil + sslot;
                            const uint32_t f = fm[p];
                            if (f & 1u) a.csr_ids[sslot++] = g2;       // -z
                            if (f & 2u) a.csr_ids[sslot++] = g3;       // -y
                            if (f & 4u) a.csr_ids[sslot++] = g - 1u;   // -x
                            if (f & 8u) a.csr_ids[sslot++] = g + 1u;   // +x
                            if (f & 16u) a.csr_ids[sslot++] = g4;      // +y
                            if (f & 32u) a.csr_ids[sslot++] = g5;      // +z
                            const uint32_t cA = cls_of_code<T, ANZ>(ls, elem<T>(A, p));
                            if (qb[p] & 1u) {   // x-quad [(j-1,k-1), (j,k-1), (j,k), (j-1,k)]
                                *reinterpret_cast<uint4 *>(a.quads + 4 * (int64_t)qslot) = make_uint4(g1, g2, g, g3);
                                *reinterpret_cast<uint2 *>(a.pairs + 2 * (int64_t)qslot) =
                                    make_uint2(cA, cls_of_code<T, ANZ>(ls, elem<T>(hA, p)));
                                ++qslot;
                            }
                            if (qb[p] & 2u) {   // y-quad [(i-1,k-1), (i-1,k), (i,k), (i,k-1)] in row j
                                *reinterpret_cast<uint4 *>(a.quads + 4 * (int64_t)qslot) = make_uint4(g2 - 1u, g - 1u, g, g2);
                                *reinterpret_cast<uint2 *>(a.pairs + 2 * (int64_t)qslot) =
                                    make_uint2(cA, cls_of_code<T, ANZ>(ls, elem<T>(B, p)));
                                ++qslot;
                            }
                            if (qb[p] & 4u) {   // z-quad [(i-1,j-1), (i,j-1), (i,j), (i-1,j)] in layer k
                                *reinterpret_cast<uint4 *>(a.quads + 4 * (int64_t)qslot) = make_uint4(g3 - 1u, g3, g, g - 1u);
                                *reinterpret_cast<uint2 *>(a.pairs + 2 * (int64_t)qslot) =
                                    make_uint2(cA, cls_of_code<T, ANZ>(ls, elem<T>(C, p)));
                                ++qslot;
                            }
                            ++acc;
                        }
                        a1 += bitp(m1, p, lane); a2 += bitp(m2, p, lane); a3 += bitp(m3, p, lane);
                        a4 += bitp(m4, p, lane); a5 += bitp(m5, p, lane);
                    }
                    run_q += (tot >> 10) & 1023u;
                    run_s += tot & 1023u;
                }
            }
            run_o += popc_all(po);
            run1 += popc_all(m1); run2 += popc_all(m2); run3 += popc_all(m3);
            run4 += popc_all(m4); run5 += popc_all(m5);
        }
    }
}

}  // namespace psn
