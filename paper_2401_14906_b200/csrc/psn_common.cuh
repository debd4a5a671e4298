// psn_common.cuh -- device helpers shared by the PSN kernels (sm_100a).
//
// Data model: every lane owns a CHUNK of 4 consecutive
// lattice points of a grid row, held as NW packed 32-bit words
// (u8: 1 word, u16: 2 words, u32: 4 words).  A warp therefore covers 128
// consecutive x positions.  Per-element boolean planes are kept in SPREAD
// form: the most significant bit of each element slot is the flag, the other
// bits are don't-care until masked with Pack<T>::MSB.
//
// Edge predicate (reading Q1): I(a,b) = cls(a) != cls(b).  With
// all_nonzero (reading Q2) cls is injective on raw values, so I is a raw
// inequality; for a general label set L each raw value is first mapped to a
// CODE (v if v in L, else one fixed value z not in L), which is again
// injective on classes.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace psn {

constexpr uint32_t kFull = 0xffffffffu;
constexpr uint32_t kBackground = 0xFFFFFFFFu;

// A lane's CHUNK is 16 bytes of a grid row: E = 16/sizeof(T) consecutive
// elements in NW = 4 packed 32-bit words (EPW elements per word, EB bits each).
template <typename T> struct Pack;
template <> struct Pack<uint8_t> {
    static constexpr int NW = 4, EB = 8, EPW = 4, E = 16;
    static constexpr uint32_t LOW = 0x7F7F7F7Fu, MSB = 0x80808080u, EMASK = 0xFFu;
};
template <> struct Pack<uint16_t> {
    static constexpr int NW = 4, EB = 16, EPW = 2, E = 8;
    static constexpr uint32_t LOW = 0x7FFF7FFFu, MSB = 0x80008000u, EMASK = 0xFFFFu;
};
template <> struct Pack<uint32_t> {
    static constexpr int NW = 4, EB = 32, EPW = 1, E = 4;
    static constexpr uint32_t LOW = 0x7FFFFFFFu, MSB = 0x80000000u, EMASK = 0xFFFFFFFFu;
};

// Spread-form "elements differ": MSB of each element slot set iff a_e != b_e.
// ((t & LOW) + LOW) carries into the MSB iff the low bits are non-zero; OR t
// adds the MSB itself.  No carry crosses slots because LOW clears each MSB.
template <typename T>
__device__ __forceinline__ uint32_t neq(uint32_t a, uint32_t b) {
    uint32_t t = a ^ b;
    return ((t & Pack<T>::LOW) + Pack<T>::LOW) | t;
}

// Words of the chunk shifted by one element: element e of the result is
// element e+1 of the chunk; the last slot takes the first element of `nxt`.
template <typename T>
__device__ __forceinline__ void shift1(const uint32_t (&w)[Pack<T>::NW], uint32_t nxt,
                                       uint32_t (&h)[Pack<T>::NW]) {
    constexpr int NW = Pack<T>::NW;
#pragma unroll
    for (int q = 0; q < NW; ++q) {
        uint32_t hi = (q + 1 < NW) ? w[(q + 1) % NW] : nxt;
        h[q] = __funnelshift_rc(w[q], hi, Pack<T>::EB);
    }
}

// Flag bit of element e (0..E-1) of a spread plane.
template <typename T>
__device__ __forceinline__ uint32_t flag(const uint32_t (&p)[Pack<T>::NW], int e) {
    constexpr int EPW = Pack<T>::EPW, EB = Pack<T>::EB;
    return (p[e / EPW] >> (EB * (e % EPW) + EB - 1)) & 1u;
}

// Raw element e (0..E-1) of a packed chunk.
template <typename T>
__device__ __forceinline__ uint32_t elem(const uint32_t (&w)[Pack<T>::NW], int e) {
    constexpr int EPW = Pack<T>::EPW, EB = Pack<T>::EB;
    return (EB == 32) ? w[e] : ((w[e / EPW] >> (EB * (e % EPW))) & Pack<T>::EMASK);
}

// ---------------------------------------------------------------- classification
// General label sets (not all_nonzero): u8/u16 use a bitset of 2^bits in shared
// memory, u32 a sorted list in global memory.  code(v) = v if v in L else z.
struct LabelSet {
    const uint32_t *bits;   // bitset (u8/u16) -- shared memory copy
    const uint32_t *list;   // sorted unique values (u32)
    int64_t n_list;
    uint32_t z;             // a value not in L (code of every background value)
    int identity;           // every value of the dtype is in L: code(v) = v
};

__device__ __forceinline__ bool in_list(const uint32_t *__restrict__ L, int64_t n, uint32_t v) {
    int64_t lo = 0, hi = n;
    while (lo < hi) {
        int64_t mid = (lo + hi) >> 1;
        uint32_t x = __ldg(L + mid);
        if (x == v) return true;
        if (x < v) lo = mid + 1; else hi = mid;
    }
    return false;
}

template <typename T>
__device__ __forceinline__ bool in_L(const LabelSet &ls, uint32_t v) {
    if (sizeof(T) == 4) return in_list(ls.list, ls.n_list, v);
    return (ls.bits[v >> 5] >> (v & 31)) & 1u;
}

template <typename T>
__device__ __forceinline__ void remap(const LabelSet &ls, uint32_t (&w)[Pack<T>::NW]) {
    if (ls.identity) return;
    constexpr int NW = Pack<T>::NW, EPW = Pack<T>::EPW, EB = Pack<T>::EB;
#pragma unroll
    for (int q = 0; q < NW; ++q) {
        uint32_t out = 0;
#pragma unroll
        for (int e = 0; e < EPW; ++e) {
            uint32_t v = (EB == 32) ? w[q] : ((w[q] >> (EB * e)) & Pack<T>::EMASK);
            uint32_t c = in_L<T>(ls, v) ? v : ls.z;
            out |= (EB == 32) ? c : (c << (EB * e));
        }
        w[q] = out;
    }
}

// Remap the elements of one packed word (the `next` word loaded directly).
template <typename T>
__device__ __forceinline__ uint32_t remap1(const LabelSet &ls, uint32_t w) {
    if (ls.identity) return w;
    constexpr int EPW = Pack<T>::EPW, EB = Pack<T>::EB;
    uint32_t out = 0;
#pragma unroll
    for (int e = 0; e < EPW; ++e) {
        uint32_t v = (EB == 32) ? w : ((w >> (EB * e)) & Pack<T>::EMASK);
        uint32_t c = in_L<T>(ls, v) ? v : ls.z;
        out |= (EB == 32) ? c : (c << (EB * e));
    }
    return out;
}

// Class of a coded element for the two-tuple (reading Q3): background -> sentinel.
template <typename T, bool ANZ>
__device__ __forceinline__ uint32_t cls_of_code(const LabelSet &ls, uint32_t code) {
    if (ANZ) return code == 0 ? kBackground : code;
    if (ls.identity) return code;
    return code == ls.z ? kBackground : code;
}

// ---------------------------------------------------------------- memory-order helpers
__device__ __forceinline__ void st_release(uint32_t *p, uint32_t v) {
    asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ uint32_t ld_acquire(const uint32_t *p) {
    uint32_t v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
// System scope (peer GPUs over NVLink): the halo push of psn_smooth_step_peer.
__device__ __forceinline__ void st_release_sys64(uint64_t *p, uint64_t v) {
    asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ uint64_t ld_acquire_sys64(const uint64_t *p) {
    uint64_t v;
    asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ uint64_t globaltimer_ns() {
    uint64_t t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}
__device__ __forceinline__ uint64_t ld_relaxed64(const uint64_t *p) {
    uint64_t v;
    asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}

}  // namespace psn

// ---------------------------------------------------------------- TMA / mbarrier (sm_90+, used on sm_100a)
namespace psn {
__device__ __forceinline__ uint32_t smem_u32(const void *p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void fence_mbar_init() {
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void fence_proxy_async() {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t *bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
}
// 1-D bulk copy global -> shared (TMA engine), completing `bytes` on the mbarrier.
__device__ __forceinline__ void tma_load_1d(void *dst, const void *src, uint32_t bytes, uint64_t *bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred p;\n"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra WAIT_%=;\n}" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}
}  // namespace psn

// ---------------------------------------------------------------- 32-bit shared-memory loads
namespace psn {
__device__ __forceinline__ uint32_t lds32(uint32_t addr) {
    uint32_t v;
    asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(addr));
    return v;
}
__device__ __forceinline__ uint2 lds64(uint32_t addr) {
    uint2 v;
    asm volatile("ld.shared.v2.u32 {%0, %1}, [%2];" : "=r"(v.x), "=r"(v.y) : "r"(addr));
    return v;
}
__device__ __forceinline__ uint4 lds128(uint32_t addr) {
    uint4 v;
    asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "r"(addr));
    return v;
}
// The 4-element chunk (NW packed words) at shared address addr.
template <typename T>
__device__ __forceinline__ void lds_chunk(uint32_t addr, uint32_t (&w)[Pack<T>::NW]) {
    if constexpr (Pack<T>::NW == 1) { w[0] = lds32(addr); }
    else if constexpr (Pack<T>::NW == 2) { const uint2 v = lds64(addr); w[0] = v.x; w[1] = v.y; }
    else { const uint4 v = lds128(addr); w[0] = v.x; w[1] = v.y; w[2] = v.z; w[3] = v.w; }
}
}  // namespace psn
