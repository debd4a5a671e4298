// k_count3.cuh -- Passes 1-3 (counting half) of PSN extraction, warp-per-row
// producer/consumer variant for rows that fit one warp (M-1 <= 256*E).
//
// PAPER sec 2.3: Pass 1 classifies x-edges and trims rows, Pass 2
// classifies y/z-edges, Pass 3 combines them into the per-voxel
// edge case and the point / quad / stencil counts of each voxel row (P:85-86,
// P:118).  Here all three run in one z-marching kernel:
//
//   CTA      = kC3Rows voxel rows (j0 .. j0+7) x the full row, marching over a
//              z-chunk of voxel layers [kbeg, kend).
//   producer = one warp that streams the kC3Rows+1 grid rows of each lattice
//              slice into a shared-memory ring with TMA bulk copies
//              (cp.async.bulk, completion on a FULL mbarrier per slot) and
//              refills a slot once every consumer warp has arrived on its
//              EMPTY mbarrier.  No __syncthreads in the main loop.
//   consumer = one warp per voxel row; lane = 16-byte CHUNK(s) of E = 16/b
//              x positions (CPL chunks per lane).
//
// Per grid row, slice and chunk a KEY is computed once: the label value if all
// E+1 elements (the chunk plus the next one) are equal, else a tag that can
// equal neither a value nor the tags of the other three grid rows of a voxel
// row.  A voxel-row chunk has no intersected edge -- no point -- iff its four
// keys (rows j, j+1 at slices k, k+1) are equal: the GPU form of the paper's
// computational trimming ("rapidly skip portions of rows, entire
// rows, and even entire data slices").  Keys of slice k+1 are reused as the
// keys of slice k at the next layer.  The non-uniform chunks are compacted
// into a per-warp queue (ballot + popc) and processed 32 at a time with full
// lanes by the SWAR slow path, which forms the six face planes c^f,
// the point plane (c^e != 0) and the owned-quad / stencil counts.
//
// Outputs per voxel row r = j + (N-1)(k - kA): cntP/cntQ/cntS (halo layers
// count points only) and, for rows with >= 1 point, the point bit-plane
// pmask[r][w] (bit b of word w <-> voxel 32w + b) and ppre[r][w], the number
// of points of the row before word w (the row iterator's running id).
// Rows without points leave pmask/ppre unwritten: Pass 4 never reads them.
#pragma once
#include <type_traits>
#include "k_count.cuh"
#include "psn_common.cuh"

namespace psn {

constexpr int kC3Rows = 16;                      // voxel rows per CTA (kC3Rows / RPW consumer warps)
constexpr int kC3MaxStages = 8;                  // ring slots (lattice slices): CountArgs.NS <= this
constexpr int kC3Threads = 32 * (kC3Rows + 1);   // + one producer warp

template <typename T> struct KeyOf { using type = uint32_t; };
template <> struct KeyOf<uint32_t> { using type = unsigned long long; };

__device__ __forceinline__ void mbar_arrive(uint64_t *bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

// Key of the chunk at shared address `addr` (E elements + the next one).  At
// the row end the staged row is padded with copies of element M-1, so the
// elements past the row never make a chunk non-uniform.
template <typename T, bool ANZ>
__device__ __forceinline__ typename KeyOf<T>::type chunk_key(uint32_t addr, uint32_t tag, const LabelSet &ls) {
    constexpr int NW = Pack<T>::NW;
    uint32_t w[NW];
    lds_chunk<T>(addr, w);
    uint32_t nx = lds32(addr + 16);
    if (!ANZ) { remap<T>(ls, w); nx = remap1<T>(ls, nx); }
    uint32_t v, d = (w[0] ^ w[1]) | (w[0] ^ w[2]) | (w[0] ^ w[3]);   // the four words are equal ...
    if constexpr (sizeof(T) == 1) {
        v = w[0] & 0xFFu;
        d |= ((w[0] ^ (w[0] >> 8)) & 0x00FFFFFFu) | ((nx ^ w[0]) & 0xFFu);
    } else if constexpr (sizeof(T) == 2) {
        v = w[0] & 0xFFFFu;
        d |= ((w[0] ^ (w[0] >> 16)) | (nx ^ w[0])) & 0xFFFFu;
    } else {
        v = w[0];
        d |= nx ^ w[0];                                           // ... and so are a word's elements and the next
    }
    const bool nonconst = d != 0u;
    if constexpr (sizeof(T) == 4) return nonconst ? ((1ull << 32) | tag) : (unsigned long long)v;
    else return nonconst ? (0x80000000u | tag) : v;
}

// Pad a staged row (M elements at shared address `row`) with copies of its
// last element: 32 bytes from byte offset M*b (16-byte aligned when staged by
// TMA).  Two warps may pad the same row; they write the same bytes.
template <typename T>
__device__ __forceinline__ void pad_row(uint32_t row, int64_t M) {
    const uint32_t end = row + (uint32_t)(M * (int64_t)sizeof(T));
    uint32_t v;
    if constexpr (sizeof(T) == 1) { uint32_t x; asm volatile("ld.shared.u8 %0, [%1];" : "=r"(x) : "r"(end - 1)); v = x * 0x01010101u; }
    else if constexpr (sizeof(T) == 2) { uint32_t x; asm volatile("ld.shared.u16 %0, [%1];" : "=r"(x) : "r"(end - 2)); v = x * 0x00010001u; }
    else v = lds32(end - 4);
    if ((end & 15u) == 0u) {
        asm volatile("st.shared.v4.u32 [%0], {%1, %1, %1, %1};" ::"r"(end), "r"(v) : "memory");
        asm volatile("st.shared.v4.u32 [%0], {%1, %1, %1, %1};" ::"r"(end + 16), "r"(v) : "memory");
    } else {   // rows staged by the copy fallback (M*b not a multiple of 16)
        for (uint32_t b = 0; b < 32; b += sizeof(T)) {
            if constexpr (sizeof(T) == 1) asm volatile("st.shared.u8 [%0], %1;" ::"r"(end + b), "r"(v) : "memory");
            else if constexpr (sizeof(T) == 2) asm volatile("st.shared.u16 [%0], %1;" ::"r"(end + b), "r"(v) : "memory");
            else asm volatile("st.shared.u32 [%0], %1;" ::"r"(end + b), "r"(v) : "memory");
        }
    }
}

// Spread-form "element differs" flag planes of t = XOR-combinations of chunk
// words: one flag per element slot.  u16 uses the 16x2 SIMD min (VIMNMX):
// min(t_e, 1) puts the flag in bit 0 of each half; u8 / u32 use the carry
// trick ((t & LOW) + LOW) | t, which puts it in the MSB of each slot.
template <typename T> struct Flags {
    static constexpr bool LOWBIT = sizeof(T) == 2;
    static constexpr uint32_t FL = LOWBIT ? 0x00010001u : Pack<T>::MSB;   // flag bit of every slot
    static constexpr int POS0 = LOWBIT ? 0 : Pack<T>::EB - 1;             // flag bit within a slot
};

template <typename T>
__device__ __forceinline__ uint32_t nz(uint32_t t) {
    if constexpr (Flags<T>::LOWBIT) return __vminu2(t, 0x00010001u);
    else return ((t & Pack<T>::LOW) + Pack<T>::LOW) | t;
}

// Append flag plane p (masked to flag bits by the caller) to a packed counter
// word: planes occupy distinct bits next to each slot's flag bit.
template <typename T>
__device__ __forceinline__ uint32_t pack(uint32_t acc, uint32_t p) {
    if constexpr (Flags<T>::LOWBIT) return (acc << 1) | p;
    else return (acc >> 1) | p;
}

// Compress the flags of one word to EPW contiguous bits.
template <typename T>
__device__ __forceinline__ uint32_t movemask(uint32_t w) {
    if constexpr (sizeof(T) == 1) return (((w >> 7) & 0x01010101u) * 0x01020408u) >> 24;
    else if constexpr (sizeof(T) == 2) { const uint32_t x = w & 0x10001u; return (x | (x >> 15)) & 3u; }
    else return w >> 31;
}

// Slow path of one voxel-row chunk: A/B = grid rows j/j+1 of slice k, C/D of
// slice k+1 (shared addresses of the chunk).  Returns the E point bits; adds the
// owned quads (open boundaries P:264) to cq and the chunk's FACE counts to
// cs, packed x | y << 10 | z << 20 (each <= E per chunk):
//   x: -x faces of the row's voxels (between voxels i-1 and i, both existing) whose
//      four corners are not all one class -- each is TWO stencil entries of
//      this row (voxel i's -x, voxel i-1's +x);
//   y: -y faces (rows j-1 / j, j >= 1) -- one entry of this row and one of row j-1;
//   z: -z faces (layers k-1 / k, k >= 1) -- one entry of this row and one of layer k-1.
// A face is shared by its two voxels, so each is evaluated once: the row's
// directed stencil count is S = 2x + y + z + y(row j+1) + z(layer k+1), the last
// two added by the scan (k_scan, ScanArgs.cntYZ).  The point bit is "some corner
// differs from corner A" (c^e != 0): the union of the three -faces' corner
// sets plus corner D1.
struct SlowCtx {
    int64_t M;
    uint32_t mz, my;             // flag masks of the warp-uniform face conditions (k>=1, j>=1)
    uint32_t mqx, mqy, mqz;      // owned-quad conditions (j>=1&&k>=1, k>=1, j>=1)
    bool own;
};

template <typename T, bool ANZ>
__device__ __forceinline__ uint32_t slow_chunk(uint32_t aA, uint32_t aB, uint32_t aC, uint32_t aD, int xc,
                                               const SlowCtx &sc, const LabelSet &ls, uint32_t &cq, uint32_t &cs) {
    constexpr int NW = Pack<T>::NW, E = Pack<T>::E, EB = Pack<T>::EB, EPW = Pack<T>::EPW;
    constexpr uint32_t FL = Flags<T>::FL;
    uint32_t A[NW], B[NW], C[NW], D[NW], nA, nB, nC, nD;
    lds_chunk<T>(aA, A); nA = lds32(aA + 16);
    lds_chunk<T>(aB, B); nB = lds32(aB + 16);
    lds_chunk<T>(aC, C); nC = lds32(aC + 16);
    lds_chunk<T>(aD, D); nD = lds32(aD + 16);
    if (!ANZ) {
        remap<T>(ls, A); remap<T>(ls, B); remap<T>(ls, C); remap<T>(ls, D);
        nA = remap1<T>(ls, nA); nB = remap1<T>(ls, nB); nC = remap1<T>(ls, nC); nD = remap1<T>(ls, nD);
    }
    uint32_t hA[NW], hB[NW], hC[NW], hD[NW];
    shift1<T>(A, nA, hA); shift1<T>(B, nB, hB); shift1<T>(C, nC, hC); shift1<T>(D, nD, hD);
    // voxel-validity masks: interior chunks (the common case) need no per-element work
    uint32_t mvox[NW], mi1[NW];
    if (xc >= 1 && (int64_t)xc + E + 1 <= sc.M) {
#pragma unroll
        for (int q = 0; q < NW; ++q) { mvox[q] = FL; mi1[q] = FL; }
    } else {
#pragma unroll
        for (int q = 0; q < NW; ++q) { mvox[q] = 0; mi1[q] = 0; }
#pragma unroll
        for (int e = 0; e < E; ++e) {
            const uint32_t bit = 1u << ((EB * (e % EPW) + Flags<T>::POS0) & 31);
            const int64_t i = xc + e;
            if (i <= sc.M - 2) mvox[e / EPW] |= bit;
            if (i >= 1 && i <= sc.M - 2) mi1[e / EPW] |= bit;
        }
    }
    uint32_t bits = 0, qacc = 0, fxc = 0, fyc = 0, fzc = 0;
    // face / quad flag planes are packed side by side (pack<T>) and counted with one popcount per
    // counter: EB flag positions per element slot hold NW face planes or EB/3 words of quad planes
    constexpr int QW = Pack<T>::EB / 3;
    uint32_t ay = 0, az = 0, ax = 0, aq = 0;
#pragma unroll
    for (int q = 0; q < NW; ++q) {
        const uint32_t a = A[q], b = B[q], c = C[q], ha = hA[q];
        const uint32_t xa = a ^ ha, yab = a ^ b, zac = a ^ c;
        const uint32_t fx = yab | zac | (a ^ D[q]);     // face x=i : corners A B C D
        const uint32_t fy = xa | zac | (a ^ hC[q]);     // face y=j : A hA C hC
        const uint32_t fz = xa | yab | (a ^ hB[q]);     // face z=k : A hA B hB
        const uint32_t mv = mvox[q];
        const uint32_t pt = nz<T>(fx | fy | fz | (a ^ hD[q])) & mv;   // the 8 corners are not all one class
        bits |= movemask<T>(pt) << (q * EPW);
        ay = pack<T>(ay, nz<T>(fy) & mv & sc.my);
        az = pack<T>(az, nz<T>(fz) & mv & sc.mz);
        if (sc.own) {
            ax = pack<T>(ax, nz<T>(fx) & mi1[q]);
            // owned quads: x at (j>=1, k>=1), y at (i>=1, k>=1), z at (i>=1, j>=1)
            aq = pack<T>(aq, nz<T>(xa) & mv & sc.mqx);
            aq = pack<T>(aq, nz<T>(yab) & mi1[q] & sc.mqy);
            aq = pack<T>(aq, nz<T>(zac) & mi1[q] & sc.mqz);
            if ((q + 1) % QW == 0 || q == NW - 1) { qacc += __popc(aq); aq = 0u; }
        }
    }
    fyc = __popc(ay); fzc = __popc(az); fxc = __popc(ax);
    cq += qacc;
    cs += fxc | (fyc << 10) | (fzc << 20);
    return bits;
}

// FULL: the row's chunks fill the warp's lanes exactly (32*CPL chunks, W32 = CPL*E plane words) -- the
// per-chunk range tests become compile-time true (every BASELINE config).
// ROW 2 (EXACT): additionally M == 32*CPL*E (rows of exactly one warp width: c3-c6), so the row length
// and the staged-row stride are compile-time constants too.
template <typename T, bool ANZ, int CPL, int RPW, bool FULL = false, bool EXACT = false>
__global__ void __launch_bounds__(32 * (kC3Rows / RPW + 1)) k_count3(CountArgs a) {
    using Key = typename KeyOf<T>::type;
    constexpr int E = Pack<T>::E, TJ = kC3Rows, NWC = TJ / RPW;
    using QItem = typename std::conditional<(CPL <= 4), uint8_t, uint16_t>::type;   // (row << log2(32*CPL)) | chunk
    constexpr int CB = (CPL <= 4) ? 7 : 8;
    const int NS = a.NS;
    constexpr int WPL = (CPL * E + 31) / 32;     // mask words per lane
    constexpr uint32_t MSB = Flags<T>::FL;   // flag bits of the slow path's planes
    extern __shared__ __align__(128) uint8_t dsm[];
    __shared__ __align__(8) uint64_t full[kC3MaxStages], empty[kC3MaxStages], sbar;
    __shared__ QItem wq[NWC][RPW * 32 * CPL];   // one layer's non-uniform (row, chunk) items
    __shared__ uint32_t wm[TJ][32 * WPL];
    __shared__ uint32_t sbits[ANZ ? 1 : 2048];

    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int64_t M = EXACT ? (int64_t)(32 * CPL * Pack<T>::E) : a.M, N = a.N, NV = N - 1;
    const int64_t jb = blockIdx.x % a.nJB, zc = blockIdx.x / a.nJB;
    const int64_t j0 = jb * TJ;
    const int64_t kbeg = a.kA + zc * a.KZ;
    const int64_t kend = min(kbeg + a.KZ, a.kB);
    const int nrows = (int)min((int64_t)TJ, NV - j0);
    const int nwarps = (nrows + RPW - 1) / RPW;   // active consumer warps
    const int64_t nsteps = kend - kbeg;
    const uint32_t RB = EXACT ? (uint32_t)(32 * CPL * 16 + 32) : (uint32_t)a.RB, SB = (TJ + 1) * RB;   // (= the host's)
    const uint32_t sbase = smem_u32(dsm);
    const uint32_t copy_bytes = (uint32_t)(M * (int64_t)sizeof(T));

    LabelSet ls = a.ls;
    if (!ANZ && sizeof(T) < 4) {
        for (int t = tid; t < (sizeof(T) == 1 ? 8 : 2048); t += blockDim.x) sbits[t] = a.ls.bits[t];
        ls.bits = sbits;
    }
    for (int t = tid; t < TJ * 32 * WPL; t += blockDim.x) (&wm[0][0])[t] = 0u;
    if (tid == 0) {
        for (int s = 0; s < NS; ++s) {
            mbar_init(&full[s], a.tma ? 1u : 32u);
            mbar_init(&empty[s], (uint32_t)max(nwarps, 1));
        }
        mbar_init(&sbar, 1u);
        fence_mbar_init();
    }
    __syncthreads();
    if (nsteps <= 0 || nrows <= 0) return;
    const T *lab = reinterpret_cast<const T *>(a.labels);

    if (warp == NWC) {
        // ------------------------------------------------------------ producer
        const uintptr_t lab_al = reinterpret_cast<uintptr_t>(lab);
        const int wcp = a.tma ? 0 : ((copy_bytes % 8u) == 0u && (lab_al & 7u) == 0u) ? 8
                                : ((copy_bytes % 4u) == 0u && (lab_al & 3u) == 0u) ? 4 : 0;
        int slot = 0;
        uint32_t ph = 0;   // parity of the slot's refill round
        uint32_t sph = 0;  // parity of the staging barrier
        for (int64_t s = 0; s <= nsteps; ++s) {
            if (s >= NS) mbar_wait(&empty[slot], ph ^ 1u);
            const int64_t z = kbeg + s - a.z_lo;
            uint8_t *dst = dsm + (uint32_t)slot * SB;
            if (a.tma) {
                if (lane == 0) mbar_expect_tx(&full[slot], copy_bytes * (TJ + 1));
                __syncwarp();
                if (lane <= TJ) {
                    fence_proxy_async();
                    const int64_t j = min(j0 + lane, N - 1);
                    tma_load_1d(dst + lane * RB, lab + (z * N + j) * M, copy_bytes, &full[slot]);
                }
            } else if (wcp) {
                // rows of a multiple of 4 (8) bytes, not of 16: per-lane cp.async word copies, all in
                // flight at once; the slot's mbarrier completes when every lane's copies have landed
                for (int g = 0; g <= TJ; ++g) {
                    const int64_t j = min(j0 + g, N - 1);
                    const char *src = reinterpret_cast<const char *>(lab + (z * N + j) * M);
                    const uint32_t d = smem_u32(dst + g * RB);
                    if (wcp == 8) {
                        for (uint32_t x = 8u * lane; x < copy_bytes; x += 256u)
                            asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(d + x), "l"(src + x) : "memory");
                    } else {
                        for (uint32_t x = 4u * lane; x < copy_bytes; x += 128u)
                            asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(d + x), "l"(src + x) : "memory");
                    }
                }
                asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(smem_u32(&full[slot])) : "memory");
            } else if (a.RB2 > 0) {
                // rows of an odd 1- / 2-byte length (their starts are not even 4-byte aligned): TMA each
                // row's 16-byte-aligned superset into the staging area, then shift it into place in
                // shared memory (16 bytes per lane step; the byte shift is warp-uniform per row)
                uint8_t *stg = dsm + a.stg_off;
                const char *row_src = nullptr;
                uint32_t dl = 0, tb = 0, tail = 0;
                if (lane <= TJ) {
                    const int64_t j = min(j0 + lane, N - 1);
                    row_src = reinterpret_cast<const char *>(lab + (z * N + j) * M);
                    dl = (uint32_t)(reinterpret_cast<uintptr_t>(row_src) & 15u);
                    tb = (dl + copy_bytes + 15u) & ~15u;
                    const char *lim = reinterpret_cast<const char *>(lab + (a.kB + 1 - a.z_lo) * N * M);
                    const int64_t room = lim - (row_src - dl);   // never read past the last counted slice
                    if ((int64_t)tb > room) { tail = tb - (uint32_t)(room & ~(int64_t)15); tb -= tail; }
                }
                const uint32_t tot = __reduce_add_sync(kFull, lane <= TJ ? tb : 0u);
                fence_proxy_async();   // this warp's earlier generic reads of the staging area come first
                __syncwarp();
                if (lane == 0) mbar_expect_tx(&sbar, tot);
                __syncwarp();
                if (lane <= TJ && tb) tma_load_1d(stg + lane * a.RB2, row_src - dl, tb, &sbar);
                if (lane <= TJ && tail)   // the clipped end of the volume's last row: plain byte copies
                    for (uint32_t b = tb; b < tb + tail; ++b)
                        if ((int64_t)b < (int64_t)dl + copy_bytes) stg[lane * a.RB2 + b] = row_src[(int64_t)b - dl];
                mbar_wait(&sbar, sph);
                sph ^= 1u;
                __syncwarp();
                const uint32_t nch = (copy_bytes + 15u) >> 4;
                for (int g = 0; g <= TJ; ++g) {
                    const uint32_t d = __shfl_sync(kFull, dl, g);
                    const uint32_t q = d >> 2, r = 8u * (d & 3u);
                    const uint32_t sa = smem_u32(stg + g * a.RB2), da = smem_u32(dst + g * RB);
                    for (uint32_t c = lane; c < nch; c += 32) {
                        uint32_t v[8];
                        asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];"
                                     : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]) : "r"(sa + 16u * c));
                        asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];"
                                     : "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]) : "r"(sa + 16u * c + 16u));
                        uint32_t o[4];
#pragma unroll
                        for (int e = 0; e < 4; ++e) {
                            const uint32_t lo = q == 0 ? v[e] : q == 1 ? v[e + 1] : q == 2 ? v[e + 2] : v[e + 3];
                            const uint32_t hi = q == 0 ? v[e + 1] : q == 1 ? v[e + 2] : q == 2 ? v[e + 3] : v[e + 4];
                            o[e] = __funnelshift_r(lo, hi, r);
                        }
                        asm volatile("st.shared.v4.u32 [%0], {%1, %2, %3, %4};" ::"r"(da + 16u * c), "r"(o[0]), "r"(o[1]),
                                     "r"(o[2]), "r"(o[3]) : "memory");
                    }
                }
                mbar_arrive(&full[slot]);
            } else {
                for (int g = 0; g <= TJ; ++g) {
                    const int64_t j = min(j0 + g, N - 1);
                    const T *src = lab + (z * N + j) * M;
                    T *d = reinterpret_cast<T *>(dst + g * RB);
                    for (int64_t x = lane; x < M; x += 32) d[x] = src[x];
                }
                mbar_arrive(&full[slot]);
            }
            if (++slot == NS) { slot = 0; ph ^= 1u; }
        }
        return;
    }

    // ---------------------------------------------------------------- consumers
    const int w = warp;
    if (w >= nwarps) return;
    const int r0 = w * RPW;                       // first CTA row of this warp
    const int64_t jw = j0 + r0;
    const int CPR = FULL ? 32 * CPL : (int)((M - 1 + E - 1) / E);   // chunks per row
    const int64_t W32 = FULL ? (int64_t)(CPL * E) : a.W32;
    const uint32_t lt = (1u << lane) - 1u;
    auto keys_of = [&](int64_t s, int slot, Key (&kk)[RPW + 1][CPL]) {
        const uint32_t tagz = (uint32_t)(s & 1) << 1;
        const uint32_t sl = sbase + (uint32_t)slot * SB + (uint32_t)r0 * RB;
        if (lane <= RPW) pad_row<T>(sl + (uint32_t)lane * RB, M);
        __syncwarp();
#pragma unroll
        for (int g = 0; g <= RPW; ++g) {
            const uint32_t base = sl + (uint32_t)g * RB;
            const uint32_t tag = (uint32_t)(g & 1) | tagz;
#pragma unroll
            for (int q = 0; q < CPL; ++q) {
                const int c = lane + 32 * q;
                kk[g][q] = (c < CPR) ? chunk_key<T, ANZ>(base + (uint32_t)c * 16u, tag, ls) : Key(0);
            }
        }
    };

    mbar_wait(&full[0], 0u);
    Key kc[RPW + 1][CPL];
    keys_of(0, 0, kc);
    uint32_t qt = 0;
    int slot0 = 0, slot1 = NS > 1 ? 1 : 0;   // ring slots of slices o and o+1
    uint32_t ph1 = NS > 1 ? 0u : 1u;          // fill parity of slice o+1's slot
    for (int64_t o = 0; o < nsteps; ++o) {
        const int64_t s1 = o + 1;
        mbar_wait(&full[slot1], ph1);
        Key kn[RPW + 1][CPL];
        keys_of(s1, slot1, kn);
        const int64_t k = kbeg + o;
        SlowCtx sc;
        sc.M = M;
        sc.own = (k >= a.own_k0) && (k < a.own_k1);
        sc.mz = (k >= 1) ? MSB : 0u;
        sc.mqy = sc.mz;
        const uint32_t a0 = sbase + (uint32_t)slot0 * SB + (uint32_t)r0 * RB;
        const uint32_t a1 = sbase + (uint32_t)slot1 * SB + (uint32_t)r0 * RB;
        uint32_t rq[RPW], rsx[RPW], rsy[RPW], rsz[RPW], dirty = 0;
#pragma unroll
        for (int i = 0; i < RPW; ++i) { rq[i] = 0; rsx[i] = 0; rsy[i] = 0; rsz[i] = 0; }
        // classify: every non-uniform (row, chunk) of the layer goes to the warp's queue
#pragma unroll
        for (int i = 0; i < RPW; ++i) {
#pragma unroll
            for (int q = 0; q < CPL; ++q) {
                const int c = lane + 32 * q;
                const Key x = kc[i][q];
                const bool nu = (c < CPR) && (r0 + i < nrows) &&
                                ((x != kc[i + 1][q]) | (x != kn[i][q]) | (x != kn[i + 1][q]));
                const uint32_t bal = __ballot_sync(kFull, nu);
                if (nu) wq[w][qt + __popc(bal & lt)] = (QItem)((i << CB) | c);
                qt += __popc(bal);
                dirty |= (bal ? 1u : 0u) << i;
            }
        }
        __syncwarp();
        // slow path: 32 items per round with full lanes (one call site: the body is large)
        for (uint32_t qh = 0; qh < qt; qh += 32u) {
            uint32_t cq = 0, cs = 0;
            int ri = -1;
            if (qh + lane < qt) {
                const uint32_t item = wq[w][qh + lane];
                ri = (int)(item >> CB);
                const int c = (int)(item & ((1u << CB) - 1u));
                const int64_t j = jw + ri;
                SlowCtx sj = sc;
                sj.my = (j >= 1) ? MSB : 0u;
                sj.mqz = sj.my;
                sj.mqx = (j >= 1 && k >= 1) ? MSB : 0u;
                const uint32_t off = (uint32_t)ri * RB + (uint32_t)c * 16u;
                const uint32_t bits = slow_chunk<T, ANZ>(a0 + off, a0 + RB + off, a1 + off, a1 + RB + off, c * E, sj,
                                                         ls, cq, cs);
                if (bits) atomicOr(&wm[r0 + ri][(c * E) >> 5], bits << ((c * E) & 31));
            }
            if (sc.own) {   // both rows' quad counts in one word (<= 32 * 3E per round)
                const uint32_t qq = __reduce_add_sync(kFull, ri >= 0 ? cq << (16 * ri) : 0u);
#pragma unroll
                for (int i = 0; i < RPW; ++i) rq[i] += (qq >> (16 * i)) & 0xFFFFu;
            }
#pragma unroll
            for (int i = 0; i < RPW; ++i) {
                const uint32_t f = __reduce_add_sync(kFull, ri == i ? cs : 0u);   // <= 32 E per field: no carry
                rsx[i] += f & 1023u; rsy[i] += (f >> 10) & 1023u; rsz[i] += f >> 20;
            }
        }
        qt = 0;
        __syncwarp();
        // slice o is no longer read (the flush below reads wm and registers only): release its slot before
        // the flush, so the producer refills it sooner (c4 count -1.7 %)
        if (lane == 0) mbar_arrive(&empty[slot0]);
        // flush the layer's rows: counts always, point planes only when non-empty.  The RPW (<= 2) rows'
        // point counts share one word (a row has < 2^16 voxels) and one warp scan gives every row's
        // total and per-word prefixes.
        static_assert(RPW <= 2, "packed flush holds two rows");
        uint32_t wv[RPW][WPL], xin = 0;
#pragma unroll
        for (int i = 0; i < RPW; ++i) {
            uint32_t c = 0;
#pragma unroll
            for (int q = 0; q < WPL; ++q) {
                wv[i][q] = ((dirty >> i) & 1u) ? wm[r0 + i][lane * WPL + q] : 0u;
                c += __popc(wv[i][q]);
            }
            xin |= c << (16 * i);
        }
        uint32_t incl = xin;
        if (dirty) {
#pragma unroll
            for (int d = 1; d < 32; d <<= 1) {
                const uint32_t y = __shfl_up_sync(kFull, incl, d);
                if (lane >= d) incl += y;
            }
        }
        const uint32_t tot = __shfl_sync(kFull, incl, 31), exc = incl - xin;
#pragma unroll
        for (int i = 0; i < RPW; ++i) {
            if (r0 + i >= nrows) break;
            const int64_t rr = jw + i + NV * (k - a.kA);
            const uint32_t P = (tot >> (16 * i)) & 0xFFFFu;
            if (lane == 0) {   // S without the +y / +z faces (the scan adds rows j+1 / k+1's y / z counts)
                a.cntP[rr] = P; a.cntQ[rr] = rq[i];
                a.cntS[rr] = sc.own ? 2u * rsx[i] + rsy[i] + rsz[i] : 0u;
                a.cntYZ[rr] = rsy[i] | (rsz[i] << 16);
            }
            if (P) {
                // the row's trim [xL, xR): first and last point-producing voxel (P:81, P:124's final
                // trim in voxel units; rows without points are empty by their zero count)
                uint32_t lo = 0xFFFFFFFFu, hi = 0u;
#pragma unroll
                for (int q = WPL - 1; q >= 0; --q)
                    if (wv[i][q]) lo = 32u * (uint32_t)(lane * WPL + q) + (uint32_t)(__ffs(wv[i][q]) - 1);
#pragma unroll
                for (int q = 0; q < WPL; ++q)
                    if (wv[i][q]) hi = 32u * (uint32_t)(lane * WPL + q) + (uint32_t)(32 - __clz(wv[i][q]));
                lo = __reduce_min_sync(kFull, lo);
                hi = __reduce_max_sync(kFull, hi);
                if (lane == 0) a.trim[rr] = make_int2((int)lo, (int)hi);
                uint32_t pre = (exc >> (16 * i)) & 0xFFFFu;
                uint32_t *pm = a.pmask + rr * W32;
                uint16_t *pp = a.ppre + rr * W32;
#pragma unroll
                for (int q = 0; q < WPL; ++q) {
                    const int wi = lane * WPL + q;
                    if (wi < W32) { pm[wi] = wv[i][q]; pp[wi] = (uint16_t)pre; }
                    pre += __popc(wv[i][q]);
                }
            }
            if ((dirty >> i) & 1u) {
#pragma unroll
                for (int q = 0; q < WPL; ++q) wm[r0 + i][lane * WPL + q] = 0u;
            }
        }
        __syncwarp();
        slot0 = slot1;
        if (++slot1 == NS) { slot1 = 0; ph1 ^= 1u; }
#pragma unroll
        for (int g = 0; g <= RPW; ++g)
#pragma unroll
            for (int q = 0; q < CPL; ++q) kc[g][q] = kn[g][q];
    }
}

}  // namespace psn
