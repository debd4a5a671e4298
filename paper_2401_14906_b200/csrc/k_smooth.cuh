// k_smooth.cuh -- constrained Laplacian smoothing (PAPER Eq. 1) with
// double buffering, and shortest-diagonal triangulation.
//
// Positions are fp32 INDEX-SPACE OFFSETS o from each point's exact voxel-centre
// anchor: the world difference p_j - p_i of face neighbours
// is s * (e_f + o_j - o_i) with e_f = +-1 along the face axis, and the box
// constraint (reading Q10) is |o_a| <= d.  So one Jacobi step is
//     o' = clamp(o + lambda * (1/N) * sum_f (e_f + o_j - o_i), -d, d)
// per axis, exactly Eq. 1 divided by s (box-mode Jacobi is per-axis affine
// equivariant, reading Q11).  The face of the n-th CSR entry is the n-th set
// bit of the 6-bit face mask (CSR order = face order, reading Q7).
// World output = fl32(anchor64 + s*o) with anchor64 recovered exactly from the
// fp32 voxel centre (idx = rint((p - origin)/s - 0.5)).
#pragma once
#include "psn_common.cuh"

namespace psn {

// Constraint on the total motion relative to the anchor (readings Q10 / Q26), in
// index-space offsets: box |o_a| <= d per axis; sphere |s (.) o| <= r = d * min(s) (world units).
struct Constraint {
    float d;             // box half-width, voxel units
    int sphere;          // 0 = box, 1 = sphere
    float r, r2;         // sphere radius (world units) and its square
    float sx, sy, sz;    // spacing (world units per voxel)
};

constexpr uint32_t kNbrIdx = 0x3FFFFFFFu;
__device__ __forceinline__ uint4 nbr_idx(uint4 v) {
    return make_uint4(v.x & kNbrIdx, v.y & kNbrIdx, v.z & kNbrIdx, v.w);
}
__device__ __forceinline__ uint32_t nbr_faces(uint4 v) {
    return (v.x >> 30) | ((v.y >> 30) << 2) | ((v.z >> 30) << 4);
}

__device__ __forceinline__ double anchor64_from(float p, double org, double sp) {
    const double idx = rint(__dsub_rn(__ddiv_rn(__dsub_rn((double)p, org), sp), 0.5));
    return __dadd_rn(org, __dmul_rn(__dadd_rn(idx, 0.5), sp));
}

__device__ __forceinline__ float world_of(float p, float o, double org, double sp) {
    return __double2float_rn(__dadd_rn(anchor64_from(p, org, sp), __dmul_rn(sp, (double)o)));
}

// One Jacobi update of Eq. 1 on index-space offsets (shared by k_smooth and
// k_smooth_tb, so both strategies are bit-identical).  f = face mask (bits
// -z,-y,-x,+x,+y,+z), o = own offset, mx/px = -x/+x neighbours, g0..g3 =
// -z,-y,+y,+z neighbours (values of absent faces are ignored).
//   s = e + sum_j o_j - deg * o          (e = sum of the face directions)
//   o' = constrain(o + lambda * s * (1/deg))           (readings Q8, Q9, Q10, Q26)
// Explicit _rn intrinsics: no FMA contraction, a fixed summation order.
__device__ __forceinline__ float jacobi_axis(float e, float o, float mx, float px, float g0, float g1, float g2,
                                             float g3, uint32_t f, float fd, float inv, float lambda, float d,
                                             bool box) {
    float acc = 0.f;
    if (f & 4u) acc = __fadd_rn(acc, mx);
    if (f & 8u) acc = __fadd_rn(acc, px);
    if (f & 1u) acc = __fadd_rn(acc, g0);
    if (f & 2u) acc = __fadd_rn(acc, g1);
    if (f & 16u) acc = __fadd_rn(acc, g2);
    if (f & 32u) acc = __fadd_rn(acc, g3);
    const float sum = __fadd_rn(__fadd_rn(e, acc), -__fmul_rn(fd, o));
    const float q = __fadd_rn(o, __fmul_rn(lambda, __fmul_rn(sum, inv)));
    return box ? fminf(fmaxf(q, -d), d) : q;
}

// Box-constraint update (the default path; same arithmetic as jacobi_update_t<false>).
__device__ __forceinline__ float jacobi_axis_box(float e, float o, float mx, float px, float g0, float g1, float g2,
                                             float g3, uint32_t f, float fd, float inv, float lambda, float d) {
    float acc = 0.f;
    if (f & 4u) acc = __fadd_rn(acc, mx);
    if (f & 8u) acc = __fadd_rn(acc, px);
    if (f & 1u) acc = __fadd_rn(acc, g0);
    if (f & 2u) acc = __fadd_rn(acc, g1);
    if (f & 16u) acc = __fadd_rn(acc, g2);
    if (f & 32u) acc = __fadd_rn(acc, g3);
    const float sum = __fadd_rn(__fadd_rn(e, acc), -__fmul_rn(fd, o));
    return fminf(fmaxf(__fadd_rn(o, __fmul_rn(lambda, __fmul_rn(sum, inv))), -d), d);
}

__device__ __forceinline__ float3 jacobi_update_box(uint32_t f, float3 o, float3 mx, float3 px, float3 g0, float3 g1,
                                                float3 g2, float3 g3, float lambda, float d) {
    if (!f) return o;
    const int deg = __popc(f);
    const float fd = (float)deg;
    const float inv = __frcp_rn(fd);   // correctly rounded 1/deg (== the constants 1, 1/2, 1/3, ... 1/6)
    const float ex = (float)((int)((f >> 3) & 1u) - (int)((f >> 2) & 1u));
    const float ey = (float)((int)((f >> 4) & 1u) - (int)((f >> 1) & 1u));
    const float ez = (float)((int)((f >> 5) & 1u) - (int)(f & 1u));
    return make_float3(jacobi_axis_box(ex, o.x, mx.x, px.x, g0.x, g1.x, g2.x, g3.x, f, fd, inv, lambda, d),
                       jacobi_axis_box(ey, o.y, mx.y, px.y, g0.y, g1.y, g2.y, g3.y, f, fd, inv, lambda, d),
                       jacobi_axis_box(ez, o.z, mx.z, px.z, g0.z, g1.z, g2.z, g3.z, f, fd, inv, lambda, d));
}

template <bool SPHERE>
__device__ __forceinline__ float3 jacobi_update_t(uint32_t f, float3 o, float3 mx, float3 px, float3 g0, float3 g1,
                                                  float3 g2, float3 g3, float lambda, const Constraint c) {
    if (!f) return o;
    const int deg = __popc(f);
    const float fd = (float)deg;
    const float inv = __frcp_rn(fd);   // correctly rounded 1/deg (== the constants 1, 1/2, 1/3, ... 1/6)
    const float ex = (float)((int)((f >> 3) & 1u) - (int)((f >> 2) & 1u));
    const float ey = (float)((int)((f >> 4) & 1u) - (int)((f >> 1) & 1u));
    const float ez = (float)((int)((f >> 5) & 1u) - (int)(f & 1u));
    constexpr bool box = !SPHERE;
    float3 q = make_float3(jacobi_axis(ex, o.x, mx.x, px.x, g0.x, g1.x, g2.x, g3.x, f, fd, inv, lambda, c.d, box),
                           jacobi_axis(ey, o.y, mx.y, px.y, g0.y, g1.y, g2.y, g3.y, f, fd, inv, lambda, c.d, box),
                           jacobi_axis(ez, o.z, mx.z, px.z, g0.z, g1.z, g2.z, g3.z, f, fd, inv, lambda, c.d, box));
    if (SPHERE) {   // radial projection onto the sphere of radius r about the anchor (reading Q26)
        const float wx = __fmul_rn(c.sx, q.x), wy = __fmul_rn(c.sy, q.y), wz = __fmul_rn(c.sz, q.z);
        const float n2 = __fadd_rn(__fadd_rn(__fmul_rn(wx, wx), __fmul_rn(wy, wy)), __fmul_rn(wz, wz));
        if (n2 > c.r2) {
            const float k = __fdiv_rn(c.r, __fsqrt_rn(n2));
            q = make_float3(__fmul_rn(q.x, k), __fmul_rn(q.y, k), __fmul_rn(q.z, k));
        }
    }
    return q;
}

__device__ __forceinline__ float3 jacobi_update(uint32_t f, float3 o, float3 mx, float3 px, float3 g0, float3 g1,
                                                float3 g2, float3 g3, float lambda, const Constraint c) {
    return c.sphere ? jacobi_update_t<true>(f, o, mx, px, g0, g1, g2, g3, lambda, c)
                    : jacobi_update_t<false>(f, o, mx, px, g0, g1, g2, g3, lambda, c);
}

// Smoothing cache: from the CSR stencil, a fixed-stride table of
// the -z,-y,+y,+z neighbour WINDOW indices of every own point (slots of absent
// faces hold the point itself); bits 30-31 of x, y, z carry the face mask
// (bits 0-1, 2-3, 4-5), readers mask indices with kNbrIdx.  The +-x neighbours need no table: ids are
// row-major, so they are w-1 / w+1 (reading Q4).  Built once per psn_smooth.
__global__ void __launch_bounds__(256) k_smooth_prep(const uint8_t *fmask, const uint32_t *csr_off,
                                                     const uint32_t *csr_ids, uint4 *nbr, int64_t n_own,
                                                     uint32_t halo_lo, uint32_t win_base, uint32_t first_stencil) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n_own; i += (int64_t)gridDim.x * blockDim.x) {
        const uint32_t f = fmask[i];
        const uint32_t w = halo_lo + (uint32_t)i;
        uint32_t s = csr_off[i] - first_stencil;
        uint4 v = make_uint4(w, w, w, w);
        if (f & 1u) v.x = csr_ids[s++] - win_base;    // -z
        if (f & 2u) v.y = csr_ids[s++] - win_base;    // -y
        if (f & 4u) ++s;                              // -x  (w - 1)
        if (f & 8u) ++s;                              // +x  (w + 1)
        if (f & 16u) v.z = csr_ids[s++] - win_base;   // +y
        if (f & 32u) v.w = csr_ids[s++] - win_base;   // +z
        // the face mask rides in the top two bits of x, y, z (window indices < 2^30, checked on the host)
        v.x |= (f & 3u) << 30; v.y |= ((f >> 2) & 3u) << 30; v.z |= ((f >> 4) & 3u) << 30;
        nbr[i] = v;
    }
}

// One Jacobi step on float4 offsets (x, y, z, unused): one 16-byte load per
// gathered neighbour instead of three scalar loads (the kernel is issue-bound,
// not DRAM-bound, so the extra 4 bytes per point cost less than the saved
// instructions).  Same arithmetic as k_smooth_tb (bit-identical).  Used by
// psn_smooth (whole volume, last step writes world coordinates) and by
// psn_smooth_step (slabs / shards: one step between halo exchanges).
// Peer (NVLink) halo push of one slab / shard step (SV 8(e) v2; psn_smooth_step_peer).
// side[0] = the lower neighbour (rank - 1), side[1] = the upper one (rank + 1).  Own
// window entries [src_begin, src_end) are ALSO stored into the neighbour's offset
// buffer `dst` (a peer pointer) at its window index dst_begin + (w - src_begin).
// Iteration g of every rank starts when both neighbours have finished g - 1
// (their signal words in this rank's memory, sig[0] from below, sig[1] from above,
// hold >= g) and ends, after every CTA has fenced its stores system-wide, with the
// last CTA writing g + 1 into the neighbours' signal words (release, system scope).
struct PeerSide {
    float4 *dst;               // the neighbour's buffer of this iteration's parity; NULL = no neighbour
    uint32_t src_begin, src_end, dst_begin;
    uint64_t *peer_sig;        // the neighbour's signal word for data from this rank
};
struct PeerArgs {
    PeerSide side[2];
    const uint64_t *sig;       // this rank's signal words [2] (written by the neighbours)
    unsigned long long *ctr;   // this rank's CTA completion counter (monotonic)
    unsigned long long ctr_last;   // counter value seen by the last CTA of this launch
    uint32_t *err;             // set on a wait timeout (a guard that must never trigger)
    uint64_t g;                // global iteration index of this step
};
constexpr uint64_t kPeerTimeoutNs = 5000000000ull;   // 5 s

struct SmoothV4 {
    const float4 *src;         // window offsets; NULL = all zero (first iteration)
    float4 *dst;
    float *world;              // if non-NULL: write AoS world coordinates here instead of dst
    const uint4 *nbr;          // smoothing cache (k_smooth_prep), or
    const uint2 *nbr8;         // its packed form (k_smooth_prep8) when the volume's rows / layers allow
    uint32_t *hi_out;          // split cache (k_smooth_split): first iteration writes the packed entry's hi word here
    const uint32_t *hi;        // ... which later iterations read (its lo word rides in the offsets' w slot)
    const uint8_t *fmask;      // k_smooth_first: the mesh's face masks / CSR stencil (the cache is built in-kernel)
    const uint32_t *csr_off, *csr_ids;
    uint32_t win_base, first_stencil;
    const float *points;
    uint32_t n_own, halo_lo;
    float lambda, d;
    double sp[3], org[3];
    Constraint cons;           // used by k_smooth_v4<..., SPHERE = true> only (reading Q26)
    PeerArgs peer;             // used by k_smooth_v4<..., PEER = true> only
};

// Packed smoothing cache, 8 bytes per point (k_smooth_prep8): the id DISTANCES
// to the -z, +z (21 bits each), -y, +y (10 bits each) neighbours -- 0 = no
// such face, the slot then names the point itself -- and the -x / +x face
// bits.  Ids are k-major (reading Q4), so a y neighbour is at most one row of
// cells away (<= M-1 ids) and a z neighbour at most one layer ((M-1)(N-1));
// the host selects this form when M-1 < 2^10 and (M-1)(N-1) < 2^21.
//   lo = dmz | dpz << 21            hi = dpz >> 11 | dmy << 10 | dpy << 20 | fx << 30
__device__ __forceinline__ uint2 nbr8_pack(uint32_t w, uint4 v, uint32_t f) {
    const uint32_t dmz = w - v.x, dmy = w - v.y, dpy = v.z - w, dpz = v.w - w;
    return make_uint2(dmz | (dpz << 21), (dpz >> 11) | (dmy << 10) | (dpy << 20) | (((f >> 2) & 3u) << 30));
}
__device__ __forceinline__ uint32_t nbr8_faces(uint2 e) {
    return ((e.x & 0x1FFFFFu) ? 1u : 0u) | ((e.y & (0x3FFu << 10)) ? 2u : 0u) | ((e.y >> 30) << 2) |
           ((e.y & (0x3FFu << 20)) ? 16u : 0u) | ((__funnelshift_r(e.x, e.y, 21) & 0x1FFFFFu) ? 32u : 0u);
}
__device__ __forceinline__ uint4 nbr8_idx(uint2 e, uint32_t w) {
    return make_uint4(w - (e.x & 0x1FFFFFu), w - ((e.y >> 10) & 0x3FFu), w + ((e.y >> 20) & 0x3FFu),
                      w + (__funnelshift_r(e.x, e.y, 21) & 0x1FFFFFu));
}

__global__ void __launch_bounds__(256) k_smooth_prep8(const uint8_t *fmask, const uint32_t *csr_off,
                                                      const uint32_t *csr_ids, uint2 *nbr8, int64_t n_own,
                                                      uint32_t halo_lo, uint32_t win_base, uint32_t first_stencil) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n_own; i += (int64_t)gridDim.x * blockDim.x) {
        const uint32_t f = fmask[i];
        const uint32_t w = halo_lo + (uint32_t)i;
        uint32_t s = csr_off[i] - first_stencil;
        uint4 v = make_uint4(w, w, w, w);
        if (f & 1u) v.x = csr_ids[s++] - win_base;    // -z
        if (f & 2u) v.y = csr_ids[s++] - win_base;    // -y
        if (f & 4u) ++s;                              // -x  (w - 1)
        if (f & 8u) ++s;                              // +x  (w + 1)
        if (f & 16u) v.z = csr_ids[s++] - win_base;   // +y
        if (f & 32u) v.w = csr_ids[s++] - win_base;   // +z
        nbr8[i] = nbr8_pack(w, v, f);
    }
}

// Streaming accesses of the per-iteration kernel: the packed smoothing cache is read once per iteration
// and never reused within it, the destination offsets are only read again by the next iteration (long
// after they left L2 on the large configs) -- keep both out of L1 so it serves the neighbour gathers.
// (Measured: c4 smoothing 8.01 -> 7.73 ms, c5a 12.26 -> 11.91 ms, c3 unchanged.)
__device__ __forceinline__ uint2 ld_stream_u2(const uint2 *p) {
    uint2 v;
    asm volatile("ld.global.nc.L1::no_allocate.v2.u32 {%0, %1}, [%2];" : "=r"(v.x), "=r"(v.y) : "l"(p));
    return v;
}
__device__ __forceinline__ void st_stream_f4(float4 *p, float4 v) {
    asm volatile("st.global.L1::no_allocate.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(p), "f"(v.x), "f"(v.y), "f"(v.z),
                 "f"(v.w) : "memory");
}

// Offset-buffer load: read-only path normally; for the peer step, whose halo entries are written by the
// neighbours over NVLink while the kernel runs (.nc data must stay unchanged for the kernel's lifetime),
// a coherent L2 load.
__device__ __forceinline__ uint32_t ld_stream_u32(const uint32_t *p) {
    uint32_t v;
    asm volatile("ld.global.nc.L1::no_allocate.u32 %0, [%1];" : "=r"(v) : "l"(p));
    return v;
}
__device__ __forceinline__ void st_stream_u32(uint32_t *p, uint32_t v) {
    asm volatile("st.global.L1::no_allocate.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

template <bool PEER>
__device__ __forceinline__ float4 ld_src(const float4 *p) {
    if constexpr (PEER) return __ldcg(p);
    else return __ldg(p);
}

// Peer step prologue: both neighbours finished iteration g - 1 (their halo pushes are here).
__device__ __forceinline__ void peer_wait(const SmoothV4 &a) {
    if (threadIdx.x == 0) {
        const uint64_t t0 = globaltimer_ns();
        for (int s = 0; s < 2; ++s) {
            if (!a.peer.side[s].dst) continue;
            while (ld_acquire_sys64(a.peer.sig + s) < a.peer.g) {
                if (globaltimer_ns() - t0 > kPeerTimeoutNs) {   // fail loudly: no smoothing on stale halos
                    atomicExch(a.peer.err, 1u);
                    __threadfence_system();
                    __trap();
                }
                __nanosleep(64);
            }
        }
    }
    __syncthreads();
}
// Peer step epilogue: this CTA's stores (local and peer) are visible system-wide; the last CTA signals.
__device__ __forceinline__ void peer_done(const SmoothV4 &a) {
    __threadfence_system();   // every thread fences its own stores
    __syncthreads();
    if (threadIdx.x == 0) {
        const unsigned long long old = atomicAdd(a.peer.ctr, 1ull);
        if (old == a.peer.ctr_last) {
            __threadfence_system();
            for (int s = 0; s < 2; ++s)
                if (a.peer.side[s].dst) st_release_sys64(a.peer.side[s].peer_sig, a.peer.g + 1);
        }
    }
}
// Boundary layers also go straight into the neighbours' halos (peer step).
__device__ __forceinline__ void peer_push(const SmoothV4 &a, uint32_t w, float4 r4) {
#pragma unroll
    for (int s = 0; s < 2; ++s) {
        const PeerSide &ps = a.peer.side[s];
        if (ps.dst && w >= ps.src_begin && w < ps.src_end) ps.dst[ps.dst_begin + (w - ps.src_begin)] = r4;
    }
}

template <bool PACKED, bool PREF = false, bool PEER = false, bool SPHERE = false>
__global__ void __launch_bounds__(256) k_smooth_v4(SmoothV4 a) {
    const int lane = threadIdx.x & 31;
    const uint32_t n = a.n_own;
    if constexpr (PEER) peer_wait(a);
    const float4 *__restrict__ src = a.src;
    const uint32_t stride = gridDim.x * blockDim.x;
    const uint32_t base0 = blockIdx.x * blockDim.x + (threadIdx.x & ~31u);
    // PREF: the next grid-stride step's cache entry is loaded one step ahead, so only the
    // neighbour gathers (not cache -> gathers) are on each step's critical path
    uint2 e_next = make_uint2(0u, 0u);
    if (PACKED && PREF && base0 < n) e_next = ld_stream_u2(a.nbr8 + min(base0 + lane, n - 1u));
    for (uint32_t base = base0; base < n; base += stride) {
        const uint32_t i = base + lane;
        const bool act = i < n;
        const uint32_t ii = act ? i : n - 1u;
        const uint32_t w = a.halo_lo + ii;
        uint32_t f, e_lo = 0u;
        uint4 nb;
        if constexpr (PACKED) {
            uint2 e;
            if constexpr (PREF) {
                e = e_next;
                if (base + stride < n) e_next = ld_stream_u2(a.nbr8 + min(base + stride + lane, n - 1u));
            } else {
                e = ld_stream_u2(a.nbr8 + ii);
            }
            f = act ? nbr8_faces(e) : 0u;
            nb = nbr8_idx(e, w);
            e_lo = e.x;
            if (a.hi_out && act) st_stream_u32(a.hi_out + ii, e.y);   // split cache (k_smooth_split)
        } else {
            const uint4 nbw = __ldg(a.nbr + ii);
            f = act ? nbr_faces(nbw) : 0u;
            nb = nbr_idx(nbw);
        }
        float4 o4 = make_float4(0.f, 0.f, 0.f, 0.f), h0 = o4, h1 = o4, h2 = o4, h3 = o4;
        if (src) {   // PEER: coherent (L2) loads -- neighbours store into the halo entries during the kernel
            o4 = ld_src<PEER>(src + w);
            h0 = ld_src<PEER>(src + nb.x); h1 = ld_src<PEER>(src + nb.y);
            h2 = ld_src<PEER>(src + nb.z); h3 = ld_src<PEER>(src + nb.w);
        }
        const float3 o = make_float3(o4.x, o4.y, o4.z);
        float3 mx, px;
        mx.x = __shfl_up_sync(kFull, o.x, 1); mx.y = __shfl_up_sync(kFull, o.y, 1); mx.z = __shfl_up_sync(kFull, o.z, 1);
        px.x = __shfl_down_sync(kFull, o.x, 1); px.y = __shfl_down_sync(kFull, o.y, 1); px.z = __shfl_down_sync(kFull, o.z, 1);
        if (!act) continue;
        if (src && f) {
            if ((f & 4u) && lane == 0) { const float4 v = ld_src<PEER>(src + w - 1u); mx = make_float3(v.x, v.y, v.z); }
            if ((f & 8u) && (lane == 31 || i + 1u >= n)) { const float4 v = ld_src<PEER>(src + w + 1u); px = make_float3(v.x, v.y, v.z); }
        }
        float3 r;
        if constexpr (SPHERE)   // sphere of radius d*min(s) about the anchor (reading Q26)
            r = jacobi_update_t<true>(f, o, mx, px, make_float3(h0.x, h0.y, h0.z), make_float3(h1.x, h1.y, h1.z),
                                      make_float3(h2.x, h2.y, h2.z), make_float3(h3.x, h3.y, h3.z), a.lambda, a.cons);
        else
            r = jacobi_update_box(f, o, mx, px, make_float3(h0.x, h0.y, h0.z), make_float3(h1.x, h1.y, h1.z),
                                  make_float3(h2.x, h2.y, h2.z), make_float3(h3.x, h3.y, h3.z), a.lambda, a.d);
        if (a.world) {
            a.world[3u * w + 0u] = world_of(__ldg(a.points + 3u * w + 0u), r.x, a.org[0], a.sp[0]);
            a.world[3u * w + 1u] = world_of(__ldg(a.points + 3u * w + 1u), r.y, a.org[1], a.sp[1]);
            a.world[3u * w + 2u] = world_of(__ldg(a.points + 3u * w + 2u), r.z, a.org[2], a.sp[2]);
        } else {
            const float4 r4 = make_float4(r.x, r.y, r.z, __uint_as_float(e_lo));   // w: split cache lo word
            st_stream_f4(a.dst + w, r4);
            if constexpr (PEER) peer_push(a, w, r4);
        }
    }
    if constexpr (PEER) peer_done(a);
}

// Split smoothing cache, iterations 2..T of psn_smooth (whole volume, packed cache): the offsets'
// unused w slot carries the lo word of the point's packed cache entry (written by the first
// iteration, k_smooth_v4 with hi_out, and copied forward by every store), the hi word is a 4-byte
// stream -- the point's own 16-byte offset load now brings half of its cache entry, so a step reads
// 16 + 4 instead of 16 + 8 bytes per point (VERDICT r1 "use the w slot for useful data").  Same
// update, same order: bit-identical to k_smooth_v4.  PREF loads the next grid-stride step's own
// offsets and hi word one step ahead, so the neighbour gathers are the only loads on a step's path.
template <bool PREF, bool SPHERE, bool PEER = false>
__global__ void __launch_bounds__(256) k_smooth_split(SmoothV4 a) {
    const int lane = threadIdx.x & 31;
    const uint32_t n = a.n_own;
    if constexpr (PEER) peer_wait(a);
    const float4 *__restrict__ src = a.src;
    const uint32_t stride = gridDim.x * blockDim.x;
    const uint32_t base0 = blockIdx.x * blockDim.x + (threadIdx.x & ~31u);
    float4 o_next = make_float4(0.f, 0.f, 0.f, 0.f);
    uint32_t h_next = 0u;
    if (PREF && base0 < n) {
        const uint32_t ii = min(base0 + lane, n - 1u);
        o_next = ld_src<PEER>(src + a.halo_lo + ii); h_next = ld_stream_u32(a.hi + ii);
    }
    for (uint32_t base = base0; base < n; base += stride) {
        const uint32_t i = base + lane;
        const bool act = i < n;
        const uint32_t ii = act ? i : n - 1u;
        const uint32_t w = a.halo_lo + ii;
        float4 o4;
        uint32_t hy;
        if constexpr (PREF) {
            o4 = o_next; hy = h_next;
            if (base + stride < n) {
                const uint32_t jn = min(base + stride + lane, n - 1u);
                o_next = ld_src<PEER>(src + a.halo_lo + jn); h_next = ld_stream_u32(a.hi + jn);
            }
        } else {
            o4 = ld_src<PEER>(src + w); hy = ld_stream_u32(a.hi + ii);
        }
        const uint2 e = make_uint2(__float_as_uint(o4.w), hy);
        const uint32_t f = act ? nbr8_faces(e) : 0u;
        const uint4 nb = nbr8_idx(e, w);
        const float4 h0 = ld_src<PEER>(src + nb.x), h1 = ld_src<PEER>(src + nb.y), h2 = ld_src<PEER>(src + nb.z),
                     h3 = ld_src<PEER>(src + nb.w);
        const float3 o = make_float3(o4.x, o4.y, o4.z);
        float3 mx, px;
        mx.x = __shfl_up_sync(kFull, o.x, 1); mx.y = __shfl_up_sync(kFull, o.y, 1); mx.z = __shfl_up_sync(kFull, o.z, 1);
        px.x = __shfl_down_sync(kFull, o.x, 1); px.y = __shfl_down_sync(kFull, o.y, 1); px.z = __shfl_down_sync(kFull, o.z, 1);
        if (!act) continue;
        if (f) {
            if ((f & 4u) && lane == 0) { const float4 v = ld_src<PEER>(src + w - 1u); mx = make_float3(v.x, v.y, v.z); }
            if ((f & 8u) && (lane == 31 || i + 1u >= n)) { const float4 v = ld_src<PEER>(src + w + 1u); px = make_float3(v.x, v.y, v.z); }
        }
        float3 r;
        if constexpr (SPHERE)
            r = jacobi_update_t<true>(f, o, mx, px, make_float3(h0.x, h0.y, h0.z), make_float3(h1.x, h1.y, h1.z),
                                      make_float3(h2.x, h2.y, h2.z), make_float3(h3.x, h3.y, h3.z), a.lambda, a.cons);
        else
            r = jacobi_update_box(f, o, mx, px, make_float3(h0.x, h0.y, h0.z), make_float3(h1.x, h1.y, h1.z),
                                  make_float3(h2.x, h2.y, h2.z), make_float3(h3.x, h3.y, h3.z), a.lambda, a.d);
        if (a.world) {
            a.world[3u * w + 0u] = world_of(__ldg(a.points + 3u * w + 0u), r.x, a.org[0], a.sp[0]);
            a.world[3u * w + 1u] = world_of(__ldg(a.points + 3u * w + 1u), r.y, a.org[1], a.sp[1]);
            a.world[3u * w + 2u] = world_of(__ldg(a.points + 3u * w + 2u), r.z, a.org[2], a.sp[2]);
        } else {
            const float4 r4 = make_float4(r.x, r.y, r.z, o4.w);
            st_stream_f4(a.dst + w, r4);
            if constexpr (PEER) peer_push(a, w, r4);
        }
    }
    if constexpr (PEER) peer_done(a);
}

// First Jacobi iteration of psn_smooth with the split cache, fused with the cache build (replaces
// k_smooth_prep8 + k_smooth_v4 for iteration 1): the packed entry is formed from the face mask and
// the CSR stencil exactly as k_smooth_prep8 forms it, its hi word is written to a.hi_out and its lo
// word rides in the w slot of the stored offsets.  All offsets are zero before the first iteration,
// so no neighbour is gathered (k_smooth_v4 with src = NULL computes the same update).
template <bool SPHERE>
__global__ void __launch_bounds__(256) k_smooth_first(SmoothV4 a) {
    const float3 z = make_float3(0.f, 0.f, 0.f);
    const uint32_t stride = gridDim.x * blockDim.x;
    uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    // face mask and CSR offset of the next grid-stride step loaded one step ahead: only the stencil-id
    // loads stay on a step's dependent chain (one resident wave of CTAs; c4 smoothing -1.0 %, c3 -1.4 %)
    uint32_t fm_n = 0u, so_n = 0u;
    if (i < a.n_own) { fm_n = a.fmask[i]; so_n = __ldg(a.csr_off + i); }
    for (; i < a.n_own; i += stride) {
        const uint32_t fm = fm_n;
        uint32_t s = so_n - a.first_stencil;
        if (i + stride < a.n_own) { fm_n = a.fmask[i + stride]; so_n = __ldg(a.csr_off + i + stride); }
        const uint32_t w = a.halo_lo + i;
        uint4 v = make_uint4(w, w, w, w);
        if (fm & 1u) v.x = __ldg(a.csr_ids + s++) - a.win_base;    // -z
        if (fm & 2u) v.y = __ldg(a.csr_ids + s++) - a.win_base;    // -y
        if (fm & 4u) ++s;                                          // -x  (w - 1)
        if (fm & 8u) ++s;                                          // +x  (w + 1)
        if (fm & 16u) v.z = __ldg(a.csr_ids + s++) - a.win_base;   // +y
        if (fm & 32u) v.w = __ldg(a.csr_ids + s++) - a.win_base;   // +z
        const uint2 e = nbr8_pack(w, v, fm);
        const uint32_t f = nbr8_faces(e);
        float3 r;
        if constexpr (SPHERE) r = jacobi_update_t<true>(f, z, z, z, z, z, z, z, a.lambda, a.cons);
        else r = jacobi_update_box(f, z, z, z, z, z, z, z, a.lambda, a.d);
        if (a.world) {
            a.world[3u * w + 0u] = world_of(__ldg(a.points + 3u * w + 0u), r.x, a.org[0], a.sp[0]);
            a.world[3u * w + 1u] = world_of(__ldg(a.points + 3u * w + 1u), r.y, a.org[1], a.sp[1]);
            a.world[3u * w + 2u] = world_of(__ldg(a.points + 3u * w + 2u), r.z, a.org[2], a.sp[2]);
        } else {
            st_stream_f4(a.dst + w, make_float4(r.x, r.y, r.z, __uint_as_float(e.x)));
            st_stream_u32(a.hi_out + i, e.y);
        }
    }
}

// Iterations 1 AND 2 of psn_smooth in one pass (split cache, whole volume).  Before iteration 1 every
// offset is zero, so a point's iteration-1 offset is a function of its face mask alone (Eq. 1 with all
// neighbour terms zero): the kernel tabulates it for the 64 masks with the same update code, then computes
// iteration 2 from the point's own and its six neighbours' face masks -- the values the stored-and-reloaded
// iteration-1 offsets would hold, bit for bit (fp32 stores and loads are exact) -- while building the split
// cache from the CSR stencil as k_smooth_first does.  One pass of 1 + 4 + 4S/P + ~4 (neighbour masks) bytes
// read and 20 written per point replaces k_smooth_first's pass plus one k_smooth_split pass.
template <bool SPHERE>
__global__ void __launch_bounds__(256) k_smooth_first2(SmoothV4 a) {
    __shared__ float3 tab[64];
    const float3 z = make_float3(0.f, 0.f, 0.f);
    for (int f = threadIdx.x; f < 64; f += blockDim.x) {
        if constexpr (SPHERE) tab[f] = jacobi_update_t<true>((uint32_t)f, z, z, z, z, z, z, z, a.lambda, a.cons);
        else tab[f] = jacobi_update_box((uint32_t)f, z, z, z, z, z, z, z, a.lambda, a.d);
    }
    __syncthreads();
    const int lane = threadIdx.x & 31;
    const uint32_t n = a.n_own;
    const uint32_t stride = gridDim.x * blockDim.x;
    uint32_t base = blockIdx.x * blockDim.x + (threadIdx.x & ~31u);
    // the next grid-stride step's face mask and CSR offset are loaded one step ahead (as k_smooth_first;
    // c4 -0.8 %, c3 -0.6 %, c6 -0.6 %)
    uint32_t fm_n = 0u, so_n = 0u;
    if (base < n) { const uint32_t j = min(base + lane, n - 1u); fm_n = a.fmask[j]; so_n = __ldg(a.csr_off + j); }
    for (; base < n; base += stride) {
        const uint32_t i = base + lane;
        const bool act = i < n;
        const uint32_t ii = act ? i : n - 1u;
        const uint32_t w = a.halo_lo + ii;   // whole volume: halo_lo = 0, window index = own index
        const uint32_t fm = fm_n;
        uint32_t s = so_n - a.first_stencil;
        if (base + stride < n) {
            const uint32_t j = min(base + stride + lane, n - 1u);
            fm_n = a.fmask[j]; so_n = __ldg(a.csr_off + j);
        }
        uint4 v = make_uint4(w, w, w, w);
        if (fm & 1u) v.x = __ldg(a.csr_ids + s++) - a.win_base;    // -z
        if (fm & 2u) v.y = __ldg(a.csr_ids + s++) - a.win_base;    // -y
        if (fm & 4u) ++s;                                          // -x  (w - 1)
        if (fm & 8u) ++s;                                          // +x  (w + 1)
        if (fm & 16u) v.z = __ldg(a.csr_ids + s++) - a.win_base;   // +y
        if (fm & 32u) v.w = __ldg(a.csr_ids + s++) - a.win_base;   // +z
        const uint2 e = nbr8_pack(w, v, fm);
        const uint32_t f = nbr8_faces(e);
        const float3 o = tab[f];
        float3 mx, px;
        mx.x = __shfl_up_sync(kFull, o.x, 1); mx.y = __shfl_up_sync(kFull, o.y, 1); mx.z = __shfl_up_sync(kFull, o.z, 1);
        px.x = __shfl_down_sync(kFull, o.x, 1); px.y = __shfl_down_sync(kFull, o.y, 1); px.z = __shfl_down_sync(kFull, o.z, 1);
        if (!act) continue;
        if ((f & 4u) && lane == 0) mx = tab[a.fmask[w - 1u - a.halo_lo]];
        if ((f & 8u) && (lane == 31 || i + 1u >= n)) px = tab[a.fmask[w + 1u - a.halo_lo]];
        const float3 g0 = tab[(f & 1u) ? a.fmask[v.x - a.halo_lo] : fm], g1 = tab[(f & 2u) ? a.fmask[v.y - a.halo_lo] : fm];
        const float3 g2 = tab[(f & 16u) ? a.fmask[v.z - a.halo_lo] : fm], g3 = tab[(f & 32u) ? a.fmask[v.w - a.halo_lo] : fm];
        float3 r;
        if constexpr (SPHERE) r = jacobi_update_t<true>(f, o, mx, px, g0, g1, g2, g3, a.lambda, a.cons);
        else r = jacobi_update_box(f, o, mx, px, g0, g1, g2, g3, a.lambda, a.d);
        if (a.world) {
            a.world[3u * w + 0u] = world_of(__ldg(a.points + 3u * w + 0u), r.x, a.org[0], a.sp[0]);
            a.world[3u * w + 1u] = world_of(__ldg(a.points + 3u * w + 1u), r.y, a.org[1], a.sp[1]);
            a.world[3u * w + 2u] = world_of(__ldg(a.points + 3u * w + 2u), r.z, a.org[2], a.sp[2]);
        } else {
            st_stream_f4(a.dst + w, make_float4(r.x, r.y, r.z, __uint_as_float(e.x)));
            st_stream_u32(a.hi_out + ii, e.y);
        }
    }
}

// World coordinates of window entries [w0, w1) from float4 offsets (NULL = anchors).
__global__ void __launch_bounds__(256) k_finalize(const float4 *offs, const float *points, float *out,
                                                  int64_t w0, int64_t w1, double sx, double sy, double sz,
                                                  double ox, double oy, double oz) {
    for (int64_t w = w0 + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; w < w1;
         w += (int64_t)gridDim.x * blockDim.x) {
        const float4 o = offs ? offs[w] : make_float4(0.f, 0.f, 0.f, 0.f);
        const float o0 = o.x, o1 = o.y, o2 = o.z;
        out[3 * w + 0] = world_of(points[3 * w + 0], o0, ox, sx);
        out[3 * w + 1] = world_of(points[3 * w + 1], o1, oy, sy);
        out[3 * w + 2] = world_of(points[3 * w + 2], o2, oz, sz);
    }
}

// Triangulation: quad q -> tris 2q, 2q+1; diagonal 0-2 -> (a,b,c),(a,c,d), 1-3 ->
// (a,b,d),(b,c,d).  Every quantity in fp64 from the fp32 points with explicit _rn operations
// in the oracle's order (C-8), so the choice is bit-identical to the host's:
//   1 shortest diagonal: |c-a|^2 <= |d-b|^2 (differences, squares, x+y+z; reading Q13)
//   2 minimum area:      |n(a,b,c)| + |n(a,c,d)| <= |n(a,b,d)| + |n(b,c,d)|      (reading Q27)
//   3 most co-planar:    cos(n(a,b,c), n(a,c,d)) >= cos(n(a,b,d), n(b,c,d))      (reading Q27)
// with n = cross product; ties -> 0-2; 0 = fixed 0-2 ("greedy").
struct D3 { double x, y, z; };
__device__ __forceinline__ D3 tri_normal(const float *p, const float *q, const float *r) {
    const double u0 = __dsub_rn((double)q[0], (double)p[0]), u1 = __dsub_rn((double)q[1], (double)p[1]),
                 u2 = __dsub_rn((double)q[2], (double)p[2]);
    const double v0 = __dsub_rn((double)r[0], (double)p[0]), v1 = __dsub_rn((double)r[1], (double)p[1]),
                 v2 = __dsub_rn((double)r[2], (double)p[2]);
    return D3{__dsub_rn(__dmul_rn(u1, v2), __dmul_rn(u2, v1)), __dsub_rn(__dmul_rn(u2, v0), __dmul_rn(u0, v2)),
              __dsub_rn(__dmul_rn(u0, v1), __dmul_rn(u1, v0))};
}
__device__ __forceinline__ double norm3(D3 n) {
    return __dsqrt_rn(__dadd_rn(__dadd_rn(__dmul_rn(n.x, n.x), __dmul_rn(n.y, n.y)), __dmul_rn(n.z, n.z)));
}
__device__ __forceinline__ double coplanarity(D3 n, D3 m) {
    const double den = __dmul_rn(norm3(n), norm3(m));
    if (den == 0.0) return 1.0;
    return __ddiv_rn(__dadd_rn(__dadd_rn(__dmul_rn(n.x, m.x), __dmul_rn(n.y, m.y)), __dmul_rn(n.z, m.z)), den);
}

__global__ void __launch_bounds__(256) k_triangulate(const uint32_t *quads, const float *points, uint32_t *tris,
                                                     int64_t nQ, uint32_t win_base, int strategy) {
    for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < nQ; q += (int64_t)gridDim.x * blockDim.x) {
        const uint4 v = __ldg(reinterpret_cast<const uint4 *>(quads) + q);
        bool d02 = true;
        if (strategy != 0) {
            const float *p0 = points + 3 * (int64_t)(v.x - win_base), *p1 = points + 3 * (int64_t)(v.y - win_base);
            const float *p2 = points + 3 * (int64_t)(v.z - win_base), *p3 = points + 3 * (int64_t)(v.w - win_base);
            if (strategy == 1) {
                double a0 = __dsub_rn((double)p2[0], (double)p0[0]), a1 = __dsub_rn((double)p2[1], (double)p0[1]);
                double a2 = __dsub_rn((double)p2[2], (double)p0[2]);
                double b0 = __dsub_rn((double)p3[0], (double)p1[0]), b1 = __dsub_rn((double)p3[1], (double)p1[1]);
                double b2 = __dsub_rn((double)p3[2], (double)p1[2]);
                const double da = __dadd_rn(__dadd_rn(__dmul_rn(a0, a0), __dmul_rn(a1, a1)), __dmul_rn(a2, a2));
                const double db = __dadd_rn(__dadd_rn(__dmul_rn(b0, b0), __dmul_rn(b1, b1)), __dmul_rn(b2, b2));
                d02 = da <= db;
            } else {
                const D3 n1 = tri_normal(p0, p1, p2), n2 = tri_normal(p0, p2, p3);
                const D3 m1 = tri_normal(p0, p1, p3), m2 = tri_normal(p1, p2, p3);
                if (strategy == 2) d02 = __dadd_rn(norm3(n1), norm3(n2)) <= __dadd_rn(norm3(m1), norm3(m2));
                else d02 = coplanarity(n1, n2) >= coplanarity(m1, m2);
            }
        }
        uint2 *t = reinterpret_cast<uint2 *>(tris + 6 * q);
        if (d02) { t[0] = make_uint2(v.x, v.y); t[1] = make_uint2(v.z, v.x); t[2] = make_uint2(v.z, v.w); }
        else     { t[0] = make_uint2(v.x, v.y); t[1] = make_uint2(v.w, v.y); t[2] = make_uint2(v.z, v.w); }
    }
}

}  // namespace psn
