// k_count.cuh -- Passes 1-3 (counting half) of PSN extraction on sm_100a.
//
// PAPER sec 2.3: Pass 1 classifies x-edges and trims rows, Pass 2
// classifies y/z-edges and adjusts the trim, Pass 3 combines
// them into the per-voxel edge case and the point / quad / stencil counts of
// each voxel row.  All three run in one z-marching kernel:
//
//   CTA   = TJ voxel rows (j0..j0+TJ-1) x up to 256*E x-positions, marching
//           over a z-chunk of voxel layers [kbeg, kend).
//   stage = the TJ+1 grid rows of one lattice slice, staged in shared memory
//           by the TMA engine (cp.async.bulk, one bulk copy per row) in a
//           4-deep ring completed on mbarriers, so HBM streams while the SMs
//           classify the previous slices.
//   lane  = a 16-byte CHUNK of E = 16/sizeof(label) consecutive x positions.
//
// FAST test per (row, chunk): the chunk's four grid rows are x-constant
// (incl. the next element) and equal to each other -> no intersected edge, no
// point (the GPU analogue of the paper's computational trimming, P:121-124:
// "rapidly skip portions of rows, entire rows, and even entire data slices").
// It costs a few XOR/OR per 32-bit word, and one ballot per row hands the
// warp its non-uniform lanes.  Those (row, chunk) TASKS are COMPACTED into a
// CTA queue and drained every two layers with full lanes by the SWAR slow
// path, which builds the 12 edge planes (X/Y/Z), the six face planes (c^f,
// P:118), the point plane (c^e != 0) and counts with popc.
//
// Outputs per voxel row r = j + (N-1)(k - kA): cntP/cntQ/cntS (halo layers
// count points only), the point trim [xL, xR) (P:124's final trim in voxel
// units; [0,0) when empty), the point bit-plane pmask[r][w] in natural
// order (bit b of word w <-> voxel 32w + b) and ppre[r][w], the number of
// points of row r before word w inside the CTA's x-tile (the row iterator's
// running id, precomputed per word so Pass 4 needs no row scans).
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
    uint32_t *cntYZ;           // k_count3: per row y | z << 16 face counts (k_scan completes S with them)
    int2 *trim;
    uint32_t *pmask;
    uint16_t *ppre;            // per pmask word: points before it within the CTA's x-tile
    LabelSet ls;
    int multi_xt;              // several x-tiles per row: accumulate with global atomics
    int tma;                   // rows are 16-byte aligned: stage with cp.async.bulk
    int NS;                    // k_count3 ring slots
    int64_t stg_off, RB2;      // k_count3 rows of an odd 1/2-byte length: staging area (dynamic smem offset,
                               // bytes per staged row) for the TMA copy of each row's 16-byte-aligned superset
};

template <typename T> __host__ __device__ constexpr int count_tj() { return 4; }
template <typename T> __host__ __device__ constexpr int count_xt() { return 256 * Pack<T>::E; }   // x positions per CTA

template <typename T, int TJ, bool ANZ>
__global__ void __launch_bounds__(256) k_count(CountArgs a) {
    constexpr int NW = Pack<T>::NW, NS = kCountStages, EB = Pack<T>::EB, EPW = Pack<T>::EPW, E = Pack<T>::E;
    constexpr int XT = count_xt<T>();
    constexpr int XPAD = 16 / (int)sizeof(T);      // extra elements staged (next element + 16-B rounding)
    constexpr uint32_t CB = 16;                    // bytes per chunk
    constexpr int WPR = XT / 32;                   // pmask words per row per CTA
    extern __shared__ __align__(128) uint8_t dsm[];
    __shared__ __align__(8) uint64_t bars[NS];
    __shared__ uint32_t sP[2][TJ], sQ[2][TJ], sS[2][TJ];
    __shared__ int sL[2][TJ], sR[2][TJ];
    __shared__ uint32_t spm[2][TJ][WPR];
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
    const uint32_t RB = (uint32_t)a.RB;
    const uint32_t SB = (TJ + 1) * RB;                           // bytes per stage
    const uint32_t sbase = smem_u32(dsm);
    const int x0 = (int)(x_t0 + E * tid);                        // this thread's chunk
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
    for (int t = tid; t < 2 * TJ * WPR; t += blockDim.x) (&spm[0][0][0])[t] = 0u;
    for (uint32_t t = tid; t < NS * SB / 16; t += blockDim.x) reinterpret_cast<uint4 *>(dsm)[t] = make_uint4(0, 0, 0, 0);
    if (tid == 0) {
        for (int s = 0; s < NS; ++s) mbar_init(&bars[s], 1);
        fence_mbar_init();
        sqn = 0;
    }
    __syncthreads();
    if (kbeg >= kend) return;
    const int64_t nsteps = kend - kbeg;           // voxel layers; slices kbeg..kend

    const T *lab = reinterpret_cast<const T *>(a.labels);
    // Fill the stage of slice ordinal o (slice kbeg + o).  TMA: lanes 0..TJ of
    // warp 0 issue one bulk copy per row; fallback (rows not 16-B aligned):
    // all threads copy.  Must be called by the whole CTA.
    auto fill = [&](int64_t o) {
        const int st = (int)(o % NS);
        if (a.tma) {
            if (warp == 0) {
                if (lane == 0) mbar_expect_tx(&bars[st], copy_bytes * (TJ + 1));
                __syncwarp();
                if (lane <= TJ) {
                    fence_proxy_async();   // prior generic reads of this stage precede the async-proxy writes
                    const int64_t j = min(j0 + lane, N - 1);
                    const T *src = lab + ((kbeg + o - a.z_lo) * N + j) * M + x_t0;
                    tma_load_1d(dsm + st * SB + lane * RB, src, copy_bytes, &bars[st]);
                }
            }
        } else {
            for (int64_t t = tid; t < (TJ + 1) * xlen; t += blockDim.x) {
                const int g = (int)(t / xlen);
                const int64_t x = t % xlen;
                const int64_t j = min(j0 + g, N - 1);
                reinterpret_cast<T *>(dsm + st * SB + g * RB)[x] = lab[((kbeg + o - a.z_lo) * N + j) * M + x_t0 + x];
            }
        }
    };
    auto wait = [&](int64_t o) {
        if (a.tma) mbar_wait(&bars[o % NS], (uint32_t)((o / NS) & 1));
    };
    for (int64_t o = 0; o < NS && o <= nsteps; ++o) fill(o);
    if (!a.tma) __syncthreads();

    // shared address of chunk c of row g of the stage holding slice ordinal o
    auto saddr = [&](int64_t o, int g, int c) -> uint32_t {
        return sbase + (uint32_t)(o % NS) * SB + (uint32_t)g * RB + (uint32_t)c * CB;
    };
    auto chunk_at = [&](uint32_t addr, uint32_t (&w)[NW], uint32_t &nxt) {
        lds_chunk<T>(addr, w);
        nxt = lds32(addr + CB);
        if (!ANZ) { remap<T>(ls, w); nxt = remap1<T>(ls, nxt); }
    };

    const int nrows = (int)(N - 1 - j0);   // voxel rows of this block (may be < TJ at the edge)
    const uint32_t rows_valid = (nrows >= TJ) ? ((1u << TJ) - 1u) : ((1u << (nrows > 0 ? nrows : 0)) - 1u);

    // Slow path for one (row r, chunk c) task of voxel layer k (slices o, o+1).
    auto process_task = [&](int64_t o, int r, int c, int64_t k, bool own, int slot) {
        uint32_t A[NW], B[NW], C[NW], D[NW], hA[NW], hB[NW], hC[NW], hD[NW], n;
        chunk_at(saddr(o, r, c), A, n); shift1<T>(A, n, hA);
        chunk_at(saddr(o, r + 1, c), B, n); shift1<T>(B, n, hB);
        chunk_at(saddr(o + 1, r, c), C, n); shift1<T>(C, n, hC);
        chunk_at(saddr(o + 1, r + 1, c), D, n); shift1<T>(D, n, hD);
        const int xc = (int)x_t0 + E * c;
        const int64_t j = j0 + r;
        uint32_t mvox[NW], mi1[NW], miM3[NW];
#pragma unroll
        for (int q = 0; q < NW; ++q) { mvox[q] = 0; mi1[q] = 0; miM3[q] = 0; }
#pragma unroll
        for (int e = 0; e < E; ++e) {
            const uint32_t bit = 1u << ((EB * (e % EPW) + EB - 1) & 31);
            const int i = xc + e;
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
        uint32_t bits = 0;   // point bits of the chunk's E voxels
#pragma unroll
        for (int e = 0; e < E; ++e) bits |= flag<T>(pt, e) << e;
        if (bits) {
            const int wofs = (E * c) & 31;   // E divides 32: the chunk lies inside one pmask word
            atomicAdd(&sP[slot][r], (uint32_t)__popc(bits));
            atomicAdd(&sQ[slot][r], cq);
            atomicAdd(&sS[slot][r], cs);
            atomicOr(&spm[slot][r][(E * c) >> 5], bits << wofs);
            atomicMin(&sL[slot][r], xc + __ffs(bits) - 1);
            atomicMax(&sR[slot][r], xc + 31 - __clz(bits));
        }
    };

    // Per-slice row flags of this thread's chunk: rf[r] != 0 iff grid rows r and
    // r+1 of the slice are not both x-constant (incl. the next element) and
    // equal to each other.  slice_flags() computes the new slice's flags and,
    // against the previous slice's, appends the slow (row, chunk) tasks of
    // voxel layer o-1 to the CTA queue: one ballot per row gives the warp the
    // row's task lanes, one atomic per warp reserves the queue slots.
    uint32_t rfA[TJ], rfB[TJ];
    const uint32_t lt = (1u << lane) - 1u;
    auto slice_flags = [&](int64_t o, uint32_t (&rf)[TJ], const uint32_t (&rfl)[TJ], bool with_lo) {
        uint32_t Wp[NW], xdp = 0, b[TJ];
        uint32_t addr = saddr(o, 0, tid), addr_lo = saddr(o - 1, 0, tid);
#pragma unroll
        for (int g = 0; g <= TJ; ++g) {
            uint32_t W[NW], H[NW], nn;
            chunk_at(addr, W, nn);
            shift1<T>(W, nn, H);
            uint32_t xd = 0;
#pragma unroll
            for (int q = 0; q < NW; ++q) xd |= W[q] ^ H[q];
            if (g > 0) {
                uint32_t yd = 0;
#pragma unroll
                for (int q = 0; q < NW; ++q) yd |= Wp[q] ^ W[q];
                rf[g - 1] = xdp | xd | yd;
                if (with_lo) {
                    uint32_t Wo[NW];
                    lds_chunk<T>(addr_lo, Wo);
                    addr_lo += RB;
                    if (!ANZ) remap<T>(ls, Wo);
                    uint32_t zd = 0;
#pragma unroll
                    for (int q = 0; q < NW; ++q) zd |= Wo[q] ^ Wp[q];
                    const bool row_ok = ((rows_valid >> (g - 1)) & 1u) && chunk_has_voxel;
                    b[g - 1] = __ballot_sync(kFull, row_ok && (rfl[g - 1] | rf[g - 1] | zd) != 0u);
                }
            }
#pragma unroll
            for (int q = 0; q < NW; ++q) Wp[q] = W[q];
            xdp = xd;
            addr += RB;
        }
        if (!with_lo) return;
        uint32_t total = 0;
#pragma unroll
        for (int r = 0; r < TJ; ++r) total += __popc(b[r]);
        if (total == 0) return;
        uint32_t base = 0;
        if (lane == 0) base = atomicAdd(&sqn, total);
        base = __shfl_sync(kFull, base, 0);
        const uint32_t tag = (uint32_t)((o - 1) & 1) << 15 | (uint32_t)tid;
#pragma unroll
        for (int r = 0; r < TJ; ++r) {
            if ((b[r] >> lane) & 1u) squeue[base + __popc(b[r] & lt)] = (uint16_t)(tag | (uint32_t)r << 8);
            base += __popc(b[r]);
        }
    };

    // SLOW phase of a batch of 1-2 layers [o0, o0+nb): all threads drain the
    // CTA queue with full lanes, then the layers' rows are flushed and their
    // lower slices released to the TMA engine.
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
            const int64_t row0 = j0 + (N - 1) * (k - a.kA);
            uint32_t *pm0 = a.pmask + row0 * a.W32 + (x_t0 >> 5);
            uint16_t *pp0 = a.ppre + row0 * a.W32 + (x_t0 >> 5);
            const uint32_t W32 = (uint32_t)a.W32;
            const int64_t wrem = a.W32 - (x_t0 >> 5);
            const uint32_t wlim = wrem < WPR ? (uint32_t)wrem : (uint32_t)WPR;
            // point planes + per-word point prefix within this x-tile (one warp per row)
            constexpr int PPL = WPR / 32;   // words per lane
            for (int r = warp; r < TJ; r += (int)(blockDim.x >> 5)) {
                uint32_t wv[PPL], cnt = 0;
#pragma unroll
                for (int q = 0; q < PPL; ++q) { wv[q] = spm[slot][r][lane * PPL + q]; cnt += __popc(wv[q]); }
                uint32_t incl = cnt;
#pragma unroll
                for (int d = 1; d < 32; d <<= 1) {
                    const uint32_t y = __shfl_up_sync(kFull, incl, d);
                    if (lane >= d) incl += y;
                }
                uint32_t pre = incl - cnt;
                const bool rv = (rows_valid >> r) & 1u;
#pragma unroll
                for (int q = 0; q < PPL; ++q) {
                    const uint32_t w = (uint32_t)(lane * PPL + q);
                    if (rv && w < wlim) { pm0[r * W32 + w] = wv[q]; pp0[r * W32 + w] = (uint16_t)pre; }
                    pre += __popc(wv[q]);
                    spm[slot][r][w] = 0u;
                }
            }
            if (tid < TJ) {
                const int r = tid;
                if ((rows_valid >> r) & 1u) {
                    const int64_t rr = row0 + r;
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

    wait(0);
    slice_flags(0, rfA, rfB, false);
    for (int64_t o = 0; o < nsteps; o += 2) {
        wait(o + 1);
        slice_flags(o + 1, rfB, rfA, true);
        const bool two = o + 1 < nsteps;
        if (two) {
            wait(o + 2);
            slice_flags(o + 2, rfA, rfB, true);
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
