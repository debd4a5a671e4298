// k_count.cuh -- Passes 1-3 (counting half) of PSN extraction on sm_100a.
//
// PAPER sec 2.3: Pass 1 classifies x-edges and trims rows, Pass 2
// classifies y/z-edges and adjusts the trim, Pass 3 combines
// them into the per-voxel edge case, point / quad / stencil counts per voxel
// row.  Here all three are one z-marching kernel:
//
//   CTA  = a block of TJ voxel rows (j0..j0+TJ-1) x up to 1024 x-positions,
//          marching over a z-chunk of voxel layers [kbeg, kend).
//   lane = a chunk of 4 lattice points (x0..x0+3) of the TJ+1 grid rows of
//          the current two lattice slices, kept in registers (packed words).
//
// Fast path (the GPU analogue of the paper's computational trimming):
// a lane's 4 voxels of a voxel row are uniform -- no edge, no point -- iff its
// four grid-row chunks are internally constant (x-equal incl. the next element)
// and equal to each other; a warp whose 32 lanes are all uniform skips the row
// with ~5 instructions.  Otherwise the slow path builds the 12 edge planes
// (X/Y/Z, SPREAD form), the six face planes (c^f) and the point plane
// (c^e != 0), and counts with popc.
//
// Outputs per voxel row r = j + (N-1)(k - kA): cntP/cntQ/cntS (halo layers
// count points only), the point trim [xL, xR) (P:124's final trim, in voxel
// units; [0,0) when empty) and the point bit-planes pmask[r][chunk][4]
// (de-interleaved: word p, bit l <-> voxel 128*chunk + 4*l + p).
#pragma once
#include "psn_common.cuh"

namespace psn {

struct CountArgs {
    const void *labels;
    int64_t M, N, O, z_lo;
    int64_t kA, kB;            // counted voxel layers (own plus halo)
    int64_t own_k0, own_k1;
    int64_t W4;                // 128-voxel chunks per row
    int64_t nXT, nJB, KZ;      // grid decomposition
    uint32_t *cntP, *cntQ, *cntS;
    int2 *trim;
    uint32_t *pmask;
    LabelSet ls;
    int multi_xt;              // several x-tiles per row: accumulate with global atomics
};

template <typename T, int TJ, bool ANZ, bool VEC>
__global__ void __launch_bounds__(256) k_count(CountArgs a) {
    constexpr int NW = Pack<T>::NW;
    constexpr uint32_t MSB = Pack<T>::MSB;
    __shared__ uint32_t sP[2][TJ], sQ[2][TJ], sS[2][TJ];
    __shared__ int sL[2][TJ], sR[2][TJ];
    __shared__ uint32_t sbits[ANZ ? 1 : 2048];

    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int64_t bid = blockIdx.x;
    const int64_t xt = bid % a.nXT;
    const int64_t jb = (bid / a.nXT) % a.nJB;
    const int64_t zc = bid / (a.nXT * a.nJB);
    const int64_t j0 = jb * TJ;
    const int64_t kbeg = a.kA + zc * a.KZ;
    const int64_t kend = min(kbeg + a.KZ, a.kB);
    const int64_t M = a.M, N = a.N;
    const int64_t x0 = xt * 1024 + 4 * (int64_t)threadIdx.x;
    const int64_t chunk = (xt * 1024 + 128 * (int64_t)warp) >> 7;
    const bool chunk_live = chunk < a.W4;

    LabelSet ls = a.ls;
    if (!ANZ && sizeof(T) < 4) {
        for (int t = threadIdx.x; t < (sizeof(T) == 1 ? 8 : 2048); t += blockDim.x) sbits[t] = a.ls.bits[t];
        ls.bits = sbits;
    }
    if (threadIdx.x < 2 * TJ) {
        int s = threadIdx.x / TJ, r = threadIdx.x % TJ;
        sP[s][r] = 0; sQ[s][r] = 0; sS[s][r] = 0; sL[s][r] = 0x7fffffff; sR[s][r] = -1;
    }
    __syncthreads();
    if (kbeg >= kend) return;

    // spread masks of this lane's 4 elements: voxel exists / has a -x / +x neighbour
    uint32_t mvox[NW], mi1[NW], miM3[NW];
#pragma unroll
    for (int q = 0; q < NW; ++q) { mvox[q] = 0; mi1[q] = 0; miM3[q] = 0; }
#pragma unroll
    for (int e = 0; e < 4; ++e) {
        const uint32_t bit = 1u << ((Pack<T>::EB * (e % Pack<T>::EPW) + Pack<T>::EB - 1) & 31);
        const int64_t i = x0 + e;
        if (i <= M - 2) mvox[e / Pack<T>::EPW] |= bit;
        if (i >= 1) mi1[e / Pack<T>::EPW] |= bit;
        if (i <= M - 3) miM3[e / Pack<T>::EPW] |= bit;
    }

    const T *lab = reinterpret_cast<const T *>(a.labels);
    uint32_t W0[TJ + 1][NW], H0[TJ + 1][NW], W1[TJ + 1][NW], H1[TJ + 1][NW];
    bool X0[TJ + 1], X1[TJ + 1];

    // Load the TJ+1 grid-row chunks of lattice slice k (plus the element after
    // each chunk), their one-element shift, and the x-uniform flag.
    auto load_slice = [&](uint32_t (&Wd)[TJ + 1][NW], uint32_t (&Hd)[TJ + 1][NW], bool (&Xd)[TJ + 1],
                          int64_t k) {
#pragma unroll
        for (int r = 0; r <= TJ; ++r) {
            const int64_t j = min(j0 + r, N - 1);
            const T *row = lab + ((k - a.z_lo) * N + j) * M;
            uint32_t w[NW];
            load_chunk<T, VEC>(row, x0, M, w);
            if (!ANZ) remap<T>(ls, w);
            uint32_t nxt = __shfl_down_sync(kFull, w[0], 1);
            if (lane == 31) {
                nxt = load_word<T, VEC>(row, x0 + 4, M);
                if (!ANZ) nxt = remap1<T>(ls, nxt);
            }
            uint32_t h[NW];
            shift1<T>(w, nxt, h);
            bool ex = true;
#pragma unroll
            for (int q = 0; q < NW; ++q) {
                Wd[r][q] = w[q]; Hd[r][q] = h[q];
                ex = ex && (w[q] == h[q]);
            }
            Xd[r] = ex;
        }
    };

    // Voxel layer k from slices k (lo) and k+1 (hi).
    auto process = [&](const uint32_t (&Wl)[TJ + 1][NW], const uint32_t (&Hl)[TJ + 1][NW], const bool (&Xl)[TJ + 1],
                       const uint32_t (&Wh)[TJ + 1][NW], const uint32_t (&Hh)[TJ + 1][NW], const bool (&Xh)[TJ + 1],
                       int64_t k, int slot) {
        const bool own = (k >= a.own_k0) && (k < a.own_k1);
#pragma unroll
        for (int r = 0; r < TJ; ++r) {
            const int64_t j = j0 + r;
            if (j > N - 2) break;
            bool uni = Xl[r] && Xl[r + 1] && Xh[r] && Xh[r + 1];
#pragma unroll
            for (int q = 0; q < NW; ++q)
                uni = uni && (Wl[r][q] == Wl[r + 1][q]) && (Wh[r][q] == Wh[r + 1][q]) && (Wl[r][q] == Wh[r][q]);
            const int64_t rr = j + (N - 1) * (k - a.kA);
            uint32_t *pm = a.pmask + (rr * a.W4 + chunk) * 4;
            if (__all_sync(kFull, uni)) {
                if (chunk_live && lane < 4) pm[lane] = 0u;
                continue;
            }
            uint32_t pt[NW];
            uint32_t cq = 0, cs = 0, cp = 0;
#pragma unroll
            for (int q = 0; q < NW; ++q) {
                const uint32_t A = Wl[r][q], B = Wl[r + 1][q], C = Wh[r][q], D = Wh[r + 1][q];
                const uint32_t hA = Hl[r][q], hB = Hl[r + 1][q], hC = Hh[r][q], hD = Hh[r + 1][q];
                const uint32_t XA = neq<T>(A, hA), XB = neq<T>(B, hB);
                const uint32_t XC = neq<T>(C, hC), XD = neq<T>(D, hD);
                const uint32_t YAB = neq<T>(A, B), YCD = neq<T>(C, D);
                const uint32_t ZAC = neq<T>(A, C), ZBD = neq<T>(B, D);
                const uint32_t YABs = neq<T>(hA, hB), YCDs = neq<T>(hC, hD);
                const uint32_t ZACs = neq<T>(hA, hC), ZBDs = neq<T>(hB, hD);
                const uint32_t Fmx = YAB | YCD | ZAC | ZBD;
                const uint32_t Fpx = YABs | YCDs | ZACs | ZBDs;
                const uint32_t Fmy = XA | XC | ZAC | ZACs;
                const uint32_t Fpy = XB | XD | ZBD | ZBDs;
                const uint32_t Fmz = XA | XB | YAB | YABs;
                const uint32_t Fpz = XC | XD | YCD | YCDs;
                pt[q] = (Fmx | Fpx | Fmy | Fpy | Fmz | Fpz) & mvox[q];
                cp += __popc(pt[q]);
                if (own) {
                    if (j >= 1 && k >= 1) cq += __popc(XA & mvox[q]);
                    if (k >= 1) cq += __popc(YAB & mvox[q] & mi1[q]);
                    if (j >= 1) cq += __popc(ZAC & mvox[q] & mi1[q]);
                    if (k >= 1) cs += __popc(Fmz & mvox[q]);
                    if (j >= 1) cs += __popc(Fmy & mvox[q]);
                    cs += __popc(Fmx & mvox[q] & mi1[q]);
                    cs += __popc(Fpx & miM3[q]);
                    if (j <= N - 3) cs += __popc(Fpy & mvox[q]);
                    if (k <= a.O - 3) cs += __popc(Fpz & mvox[q]);
                }
            }
            // point bit-planes (de-interleaved by element position)
            const uint32_t b0 = __ballot_sync(kFull, flag<T>(pt, 0));
            const uint32_t b1 = __ballot_sync(kFull, flag<T>(pt, 1));
            const uint32_t b2 = __ballot_sync(kFull, flag<T>(pt, 2));
            const uint32_t b3 = __ballot_sync(kFull, flag<T>(pt, 3));
            if (chunk_live && lane < 4) pm[lane] = lane == 0 ? b0 : lane == 1 ? b1 : lane == 2 ? b2 : b3;
            // trim: first / last point voxel of this lane
            int first = 0x7fffffff, last = -1;
#pragma unroll
            for (int e = 3; e >= 0; --e) if (flag<T>(pt, e)) first = (int)(x0 + e);
#pragma unroll
            for (int e = 0; e < 4; ++e) if (flag<T>(pt, e)) last = (int)(x0 + e);
            cp = __reduce_add_sync(kFull, cp);
            cq = __reduce_add_sync(kFull, cq);
            cs = __reduce_add_sync(kFull, cs);
            first = __reduce_min_sync(kFull, first);
            last = __reduce_max_sync(kFull, last);
            if (lane == 0 && cp) {
                atomicAdd(&sP[slot][r], cp);
                atomicAdd(&sQ[slot][r], cq);
                atomicAdd(&sS[slot][r], cs);
                atomicMin(&sL[slot][r], first);
                atomicMax(&sR[slot][r], last);
            }
        }
        __syncthreads();
        // flush this layer's TJ row counters (double-buffered slots: one barrier per layer)
        if (threadIdx.x < TJ) {
            const int r = threadIdx.x;
            const int64_t j = j0 + r;
            if (j <= N - 2) {
                const int64_t rr = j + (N - 1) * (k - a.kA);
                const uint32_t p = sP[slot][r];
                const int xl = p ? sL[slot][r] : 0, xr = p ? sR[slot][r] + 1 : 0;
                if (!a.multi_xt) {
                    a.cntP[rr] = p; a.cntQ[rr] = sQ[slot][r]; a.cntS[rr] = sS[slot][r];
                    a.trim[rr] = make_int2(xl, xr);
                } else if (p) {
                    atomicAdd(&a.cntP[rr], p); atomicAdd(&a.cntQ[rr], sQ[slot][r]);
                    atomicAdd(&a.cntS[rr], sS[slot][r]);
                    atomicMin(&a.trim[rr].x, xl); atomicMax(&a.trim[rr].y, xr);
                }
            }
            sP[slot][r] = 0; sQ[slot][r] = 0; sS[slot][r] = 0; sL[slot][r] = 0x7fffffff; sR[slot][r] = -1;
        }
    };

    load_slice(W0, H0, X0, kbeg);
    for (int64_t k = kbeg; k < kend; k += 2) {
        load_slice(W1, H1, X1, k + 1);
        process(W0, H0, X0, W1, H1, X1, k, 0);
        if (k + 1 >= kend) break;
        load_slice(W0, H0, X0, k + 2);
        process(W1, H1, X1, W0, H0, X0, k + 1, 1);
    }
}

// Multi-x-tile rows: empty rows keep the atomic-min sentinel; normalise to [0,0).
__global__ void k_trim_fix(int2 *trim, const uint32_t *cntP, int64_t R) {
    for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < R; r += (int64_t)gridDim.x * blockDim.x)
        if (cntP[r] == 0) trim[r] = make_int2(0, 0);
}

}  // namespace psn
