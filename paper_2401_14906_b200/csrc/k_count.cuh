// k_count.cuh -- Passes 1-3 (counting half) of PSN extraction on sm_100a.
//
// PAPER sec 2.3: Pass 1 classifies x-edges and trims rows, Pass 2
// classifies y/z-edges and adjusts the trim, Pass 3 combines
// them into the per-voxel edge case and the point / quad / stencil counts of
// each voxel row.  All three run in one z-marching kernel:
//
//   CTA   = TJ voxel rows (j0..j0+TJ-1) x up to 1024 x-positions, marching
//           over a z-chunk of voxel layers [kbeg, kend).
//   stage = the TJ+1 grid rows of one lattice slice, staged in shared memory
//           by the TMA engine (cp.async.bulk, one bulk copy per row) in a
//           4-deep ring completed on mbarriers, so HBM streams while the SMs
//           classify the previous slices.
//   lane  = a chunk of 4 consecutive x positions (packed words).
//
// Per layer each thread first runs the FAST test on its chunk for every row:
// the chunk's four grid rows are x-constant (incl. the next element) and equal
// to each other -> no intersected edge, no point (the GPU analogue of the
// paper's computational trimming: "rapidly skip portions of rows,
// entire rows, and even entire data slices").  The surviving (row, chunk)
// pairs are COMPACTED into a per-warp queue and processed with full lanes by
// the SWAR slow path, which builds the 12 edge planes (X/Y/Z), the six face
// planes (c^f), the point plane (c^e != 0) and counts with popc.
//
// Outputs per voxel row r = j + (N-1)(k - kA): cntP/cntQ/cntS (halo layers
// count points only), the point trim [xL, xR) (P:124's final trim in voxel
// units; [0,0) when empty) and the point bit-plane pmask[r][w] in natural
// order (bit b of word w <-> voxel 32w + b).
#pragma once
#include "psn_common.cuh"

namespace psn {

constexpr int kCountStages = 4;

struct CountArgs {
    const void *labels;
    int64_t M, N, O, z_lo;
    int64_t kA, kB;            // counted voxel layers (own plus halo)
    int64_t own_k0, own_k1;
    int64_t W32;               // 32-voxel words per row of pmask
    int64_t nXT, nJB, KZ;      // grid decomposition
    int64_t RB;                // bytes per staged row buffer (multiple of 16)
    uint32_t *cntP, *cntQ, *cntS;
    int2 *trim;
    uint32_t *pmask;
    LabelSet ls;
    int multi_xt;              // several x-tiles per row: accumulate with global atomics
    int tma;                   // rows are 16-byte aligned: stage with cp.async.bulk
};

template <typename T> constexpr int count_tj() { return sizeof(T) == 1 ? 16 : (sizeof(T) == 2 ? 8 : 4); }

template <typename T, int TJ, bool ANZ>
__global__ void __launch_bounds__(256) k_count(CountArgs a) {
    constexpr int NW = Pack<T>::NW, NS = kCountStages, EB = Pack<T>::EB, EPW = Pack<T>::EPW;
    constexpr int XT = 1024;                       // x positions per CTA
    constexpr int XPAD = 16 / (int)sizeof(T);      // extra elements staged (next element + 16-B rounding)
    extern __shared__ __align__(128) uint8_t dsm[];
    __shared__ __align__(8) uint64_t bars[NS];
    __shared__ uint32_t sP[2][TJ], sQ[2][TJ], sS[2][TJ];
    __shared__ int sL[2][TJ], sR[2][TJ];
    __shared__ uint32_t spm[2][TJ][32];
    __shared__ uint16_t squeue[2 * TJ * 256];   // CTA task queue of a 2-layer batch: (layer bit, row, chunk)
    __shared__ uint32_t sqn;
    __shared__ uint32_t sbits[ANZ ? 1 : 2048];

    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int64_t bid = blockIdx.x;
    const int64_t xt = bid % a.nXT;
    const int64_t jb = (bid / a.nXT) % a.nJB;
    const int64_t zc = bid / (a.nXT * a.nJB);
    const int64_t j0 = jb * TJ;
    const int64_t kbeg = a.kA + zc * a.KZ;
    const int64_t kend = min(kbeg + a.KZ, a.kB);
    const int64_t M = a.M, N = a.N;
    const int64_t x_t0 = xt * XT;
    const int64_t xlen = min((int64_t)(XT + XPAD), M - x_t0);   // staged elements per row
    const uint32_t copy_bytes = (uint32_t)(xlen * (int64_t)sizeof(T));
    const int64_t RB = a.RB;
    const int64_t stage_bytes = (TJ + 1) * RB;
    const int64_t x0 = x_t0 + 4 * (int64_t)tid;   // this thread's chunk
    const bool chunk_has_voxel = x0 <= M - 2;

    LabelSet ls = a.ls;
    if (!ANZ && sizeof(T) < 4) {
        for (int t = tid; t < (sizeof(T) == 1 ? 8 : 2048); t += blockDim.x) sbits[t] = a.ls.bits[t];
        ls.bits = sbits;
    }
    for (int t = tid; t < 2 * TJ; t += blockDim.x) {
        const int s = t / TJ, r = t % TJ;
        sP[s][r] = 0; sQ[s][r] = 0; sS[s][r] = 0; sL[s][r] = 0x7fffffff; sR[s][r] = -1;
    }
    for (int t = tid; t < 2 * TJ * 32; t += blockDim.x) (&spm[0][0][0])[t] = 0u;
    for (int64_t t = tid; t < NS * stage_bytes / 16; t += blockDim.x)
        reinterpret_cast<uint4 *>(dsm)[t] = make_uint4(0, 0, 0, 0);
    if (tid == 0) {
        for (int s = 0; s < NS; ++s) mbar_init(&bars[s], 1);
        fence_mbar_init();
    }
    __syncthreads();
    if (kbeg >= kend) return;
    const int64_t nsteps = kend - kbeg;           // voxel layers; slices kbeg..kend

    const T *lab = reinterpret_cast<const T *>(a.labels);
    auto row_src = [&](int64_t s, int g) -> const T * {
        const int64_t j = min(j0 + g, N - 1);
        return lab + ((s - a.z_lo) * N + j) * M + x_t0;
    };
    // Fill the stage of slice ordinal o (slice kbeg + o).  TMA: one elected
    // thread; fallback (rows not 16-B aligned): all threads copy.
    auto fill = [&](int64_t o) {
        const int st = (int)(o % NS);
        uint8_t *base = dsm + st * stage_bytes;
        if (a.tma) {
            if (tid == 0) {
                fence_proxy_async();   // prior generic reads of this stage precede the async-proxy writes
                mbar_expect_tx(&bars[st], copy_bytes * (TJ + 1));
#pragma unroll 1
                for (int g = 0; g <= TJ; ++g)
                    tma_load_1d(base + g * RB, row_src(kbeg + o, g), copy_bytes, &bars[st]);
            }
        } else {
            for (int64_t t = tid; t < (TJ + 1) * xlen; t += blockDim.x) {
                const int g = (int)(t / xlen);
                const int64_t x = t % xlen;
                reinterpret_cast<T *>(base + g * RB)[x] = row_src(kbeg + o, g)[x];
            }
        }
    };
    auto wait = [&](int64_t o) {
        if (a.tma) mbar_wait(&bars[o % NS], (uint32_t)((o / NS) & 1));
    };
    for (int64_t o = 0; o < NS && o <= nsteps; ++o) fill(o);
    if (!a.tma) __syncthreads();

    auto chunk_at = [&](int64_t o, int g, int64_t c, uint32_t (&w)[NW], uint32_t &nxt) {
        const uint8_t *p = dsm + (o % NS) * stage_bytes + g * RB + 4 * c * (int64_t)sizeof(T);
        if constexpr (NW == 1) { w[0] = *reinterpret_cast<const uint32_t *>(p); }
        else if constexpr (NW == 2) { uint2 v = *reinterpret_cast<const uint2 *>(p); w[0] = v.x; w[1] = v.y; }
        else { uint4 v = *reinterpret_cast<const uint4 *>(p); w[0] = v.x; w[1] = v.y; w[2] = v.z; w[3] = v.w; }
        nxt = *reinterpret_cast<const uint32_t *>(p + 4 * sizeof(T));
        if (!ANZ) { remap<T>(ls, w); nxt = remap1<T>(ls, nxt); }
    };

    // Per-slice flags of this thread's chunk: huM bit g = row g x-constant
    // (incl. the next element); eqYM bit g = rows g and g+1 equal.
    uint32_t Wa[TJ + 1][NW], Wb[TJ + 1][NW];
    uint32_t huA = 0, eqA = 0, huB = 0, eqB = 0;
    auto load_flags = [&](int64_t o, uint32_t (&W)[TJ + 1][NW], uint32_t &hu, uint32_t &eqy) {
        hu = 0; eqy = 0;
#pragma unroll
        for (int g = 0; g <= TJ; ++g) {
            uint32_t nxt, h[NW];
            chunk_at(o, g, tid, W[g], nxt);
            shift1<T>(W[g], nxt, h);
            bool e = true;
#pragma unroll
            for (int q = 0; q < NW; ++q) e = e && (W[g][q] == h[q]);
            hu |= (e ? 1u : 0u) << g;
        }
#pragma unroll
        for (int g = 0; g < TJ; ++g) {
            bool e = true;
#pragma unroll
            for (int q = 0; q < NW; ++q) e = e && (W[g][q] == W[g + 1][q]);
            eqy |= (e ? 1u : 0u) << g;
        }
    };

    const int64_t nrows = N - 1 - j0;   // voxel rows of this block (may be < TJ at the edge)
    const uint32_t rows_valid = (nrows >= TJ) ? ((1u << TJ) - 1u) : ((1u << (uint32_t)(nrows > 0 ? nrows : 0)) - 1u);

    // Slow path for one (row r, chunk c) task of voxel layer k (slices o, o+1).
    auto process_task = [&](int64_t o, int r, int c, int64_t k, bool own, int slot) {
        uint32_t A[NW], B[NW], C[NW], D[NW], hA[NW], hB[NW], hC[NW], hD[NW], n;
        chunk_at(o, r, c, A, n); shift1<T>(A, n, hA);
        chunk_at(o, r + 1, c, B, n); shift1<T>(B, n, hB);
        chunk_at(o + 1, r, c, C, n); shift1<T>(C, n, hC);
        chunk_at(o + 1, r + 1, c, D, n); shift1<T>(D, n, hD);
        const int64_t xc = x_t0 + 4 * (int64_t)c, j = j0 + r;
        uint32_t mvox[NW], mi1[NW], miM3[NW];
#pragma unroll
        for (int q = 0; q < NW; ++q) { mvox[q] = 0; mi1[q] = 0; miM3[q] = 0; }
#pragma unroll
        for (int e = 0; e < 4; ++e) {
            const uint32_t bit = 1u << ((EB * (e % EPW) + EB - 1) & 31);
            const int64_t i = xc + e;
            if (i <= M - 2) mvox[e / EPW] |= bit;
            if (i >= 1) mi1[e / EPW] |= bit;
            if (i <= M - 3) miM3[e / EPW] |= bit;
        }
        uint32_t pt[NW], cq = 0, cs = 0;
#pragma unroll
        for (int q = 0; q < NW; ++q) {
            const uint32_t XA = neq<T>(A[q], hA[q]), XB = neq<T>(B[q], hB[q]);
            const uint32_t XC = neq<T>(C[q], hC[q]), XD = neq<T>(D[q], hD[q]);
            const uint32_t YAB = neq<T>(A[q], B[q]), YCD = neq<T>(C[q], D[q]);
            const uint32_t ZAC = neq<T>(A[q], C[q]), ZBD = neq<T>(B[q], D[q]);
            const uint32_t YABs = neq<T>(hA[q], hB[q]), YCDs = neq<T>(hC[q], hD[q]);
            const uint32_t ZACs = neq<T>(hA[q], hC[q]), ZBDs = neq<T>(hB[q], hD[q]);
            const uint32_t Fmx = YAB | YCD | ZAC | ZBD;
            const uint32_t Fpx = YABs | YCDs | ZACs | ZBDs;
            const uint32_t Fmy = XA | XC | ZAC | ZACs;
            const uint32_t Fpy = XB | XD | ZBD | ZBDs;
            const uint32_t Fmz = XA | XB | YAB | YABs;
            const uint32_t Fpz = XC | XD | YCD | YCDs;
            pt[q] = (Fmx | Fpx | Fmy | Fpy | Fmz | Fpz) & mvox[q];
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
        uint32_t nib = 0;
#pragma unroll
        for (int e = 0; e < 4; ++e) nib |= flag<T>(pt, e) << e;
        if (nib) {
            atomicAdd(&sP[slot][r], (uint32_t)__popc(nib));
            atomicAdd(&sQ[slot][r], cq);
            atomicAdd(&sS[slot][r], cs);
            atomicOr(&spm[slot][r][c >> 3], nib << (4 * (c & 7)));
            atomicMin(&sL[slot][r], (int)(xc + __ffs(nib) - 1));
            atomicMax(&sR[slot][r], (int)(xc + 31 - __clz(nib)));
        }
    };

    // FAST test of one layer: every thread checks its chunk for the TJ rows and
    // appends the non-uniform (row, chunk) pairs to the CTA queue.
    auto fast = [&](int64_t o, const uint32_t (&Wl)[TJ + 1][NW], uint32_t hul, uint32_t eql,
                    const uint32_t (&Wh)[TJ + 1][NW], uint32_t huh, uint32_t eqh) {
        uint32_t eqz = 0;
#pragma unroll
        for (int r = 0; r < TJ; ++r) {
            bool e = true;
#pragma unroll
            for (int q = 0; q < NW; ++q) e = e && (Wl[r][q] == Wh[r][q]);
            eqz |= (e ? 1u : 0u) << r;
        }
        const uint32_t uni = hul & (hul >> 1) & huh & (huh >> 1) & eql & eqh & eqz;
        const uint32_t slow = chunk_has_voxel ? (~uni & rows_valid) : 0u;
        const uint32_t cnt = __popc(slow);
        uint32_t incl = cnt;
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
            const uint32_t y = __shfl_up_sync(kFull, incl, d);
            if (lane >= d) incl += y;
        }
        const uint32_t total = __shfl_sync(kFull, incl, 31);
        if (total) {
            uint32_t pos = 0;
            if (lane == 31) pos = atomicAdd(&sqn, total);
            pos = __shfl_sync(kFull, pos, 31) + incl - cnt;
            uint32_t m = slow;
            const uint32_t tag = (uint32_t)(o & 1) << 15 | (uint32_t)tid;
            while (m) {
                const int r = __ffs(m) - 1;
                m &= m - 1;
                squeue[pos++] = (uint16_t)(tag | (uint32_t)r << 8);
            }
        }
    };

    // SLOW phase of a batch of 1-2 layers [o0, o0+nb): all threads drain the
    // CTA queue with full lanes, then the layers' rows are flushed and their
    // lower slices released to the TMA producer.
    auto batch = [&](int64_t o0, int nb) {
        __syncthreads();
        const uint32_t nq = sqn;
        for (uint32_t t = tid; t < nq; t += blockDim.x) {
            const uint32_t task = squeue[t];
            const int ob = (int)(task >> 15);
            const int64_t o = o0 + ob;
            const int64_t k = kbeg + o;
            const bool own = (k >= a.own_k0) && (k < a.own_k1);
            process_task(o, (int)((task >> 8) & 0x7f), (int)(task & 0xff), k, own, (int)(o & 1));
        }
        __syncthreads();
        if (tid == 0) sqn = 0;
        for (int b = 0; b < nb; ++b) {
            const int64_t o = o0 + b;
            const int64_t k = kbeg + o;
            const int slot = (int)(o & 1);
            for (int t = tid; t < TJ * 32; t += blockDim.x) {
                const int r = t >> 5, w = t & 31;
                const int64_t gw = (x_t0 >> 5) + w;
                if (((rows_valid >> r) & 1u) && gw < a.W32) {
                    const int64_t rr = j0 + r + (N - 1) * (k - a.kA);
                    a.pmask[rr * a.W32 + gw] = spm[slot][r][w];
                }
                spm[slot][r][w] = 0u;
            }
            if (tid < TJ) {
                const int r = tid;
                if ((rows_valid >> r) & 1u) {
                    const int64_t rr = j0 + r + (N - 1) * (k - a.kA);
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
            // slice o is no longer read: refill its stage with slice o + NS
            if (o + NS <= nsteps) fill(o + NS);
        }
    };

    if (tid == 0) sqn = 0;
    __syncthreads();
    wait(0);
    load_flags(0, Wa, huA, eqA);
    for (int64_t o = 0; o < nsteps; o += 2) {
        wait(o + 1);
        load_flags(o + 1, Wb, huB, eqB);
        fast(o, Wa, huA, eqA, Wb, huB, eqB);
        const bool two = o + 1 < nsteps;
        if (two) {
            wait(o + 2);
            load_flags(o + 2, Wa, huA, eqA);
            fast(o + 1, Wb, huB, eqB, Wa, huA, eqA);
        }
        batch(o, two ? 2 : 1);
    }
}

// Multi-x-tile rows: empty rows keep the atomic-min sentinel; normalise to [0,0).
__global__ void k_trim_fix(int2 *trim, const uint32_t *cntP, int64_t R) {
    for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < R; r += (int64_t)gridDim.x * blockDim.x)
        if (cntP[r] == 0) trim[r] = make_int2(0, 0);
}

}  // namespace psn
