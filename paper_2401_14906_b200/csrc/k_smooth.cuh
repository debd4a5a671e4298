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

struct SmoothArgs {
    const float *src;          // window offsets [n_window][3]; NULL = all zero
    float *dst;                // window offsets (own entries written)
    float *world;              // if non-NULL: write world coordinates here instead of dst
    const uint8_t *fmask;      // own points
    const uint4 *nbr;          // own points: window indices of the -z,-y,+y,+z neighbours (k_smooth_prep)
    const float *points;       // window anchors (fp32 voxel centres), for the world output
    int64_t n_own;
    uint32_t halo_lo;          // window index of the first own point
    float lambda, d;
    double sp[3], org[3];
};

__device__ __forceinline__ double anchor64_from(float p, double org, double sp) {
    const double idx = rint(__dsub_rn(__ddiv_rn(__dsub_rn((double)p, org), sp), 0.5));
    return __dadd_rn(org, __dmul_rn(__dadd_rn(idx, 0.5), sp));
}

__device__ __forceinline__ float world_of(float p, float o, double org, double sp) {
    return __double2float_rn(__dadd_rn(anchor64_from(p, org, sp), __dmul_rn(sp, (double)o)));
}

// Smoothing cache: from the CSR stencil, a fixed-stride table of
// the -z,-y,+y,+z neighbour WINDOW indices of every own point (slots of absent
// faces hold the point itself).  The +-x neighbours need no table: ids are
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
        nbr[i] = v;
    }
}

// One Jacobi step of Eq. 1 on index-space offsets (see header comment).
// Lanes hold consecutive points, so the +-x neighbours (w-1, w+1) come from
// the adjacent lanes by shuffle; the y/z neighbours are gathered through the
// smoothing cache.  sum_j (e_f + o_j - o_i) = e + sum_j o_j - deg * o_i.
__global__ void __launch_bounds__(256) k_smooth(SmoothArgs a) {
    const int lane = threadIdx.x & 31;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    // all lanes of a warp iterate together (shuffles below need full warps)
    for (int64_t base = (int64_t)blockIdx.x * blockDim.x + (threadIdx.x & ~31); base < a.n_own; base += stride) {
        const int64_t i = base + lane;
        const bool act = i < a.n_own;
        const uint32_t w = a.halo_lo + (uint32_t)(act ? i : a.n_own - 1);
        const uint32_t f = act ? a.fmask[i] : 0u;
        float ox = 0.f, oy = 0.f, oz = 0.f;
        uint4 nb = make_uint4(w, w, w, w);
        if (act) {
            if (a.src) { ox = a.src[3 * (size_t)w]; oy = a.src[3 * (size_t)w + 1]; oz = a.src[3 * (size_t)w + 2]; }
            if (f & 0x33u) nb = a.nbr[i];
        }
        // +-x neighbours from the adjacent lanes (lane 0 / 31 and the last point load)
        float mx = __shfl_up_sync(kFull, ox, 1), my = __shfl_up_sync(kFull, oy, 1), mz = __shfl_up_sync(kFull, oz, 1);
        float px = __shfl_down_sync(kFull, ox, 1), py = __shfl_down_sync(kFull, oy, 1), pz = __shfl_down_sync(kFull, oz, 1);
        if (!act) continue;
        const int deg = __popc(f);
        float nx = ox, ny = oy, nz = oz;
        if (deg) {
            float sx = (float)((int)((f >> 3) & 1u) - (int)((f >> 2) & 1u));
            float sy = (float)((int)((f >> 4) & 1u) - (int)((f >> 1) & 1u));
            float sz = (float)((int)((f >> 5) & 1u) - (int)(f & 1u));
            if (a.src) {
                float ax = 0.f, ay = 0.f, az = 0.f;
                if (f & 4u) {
                    if (lane == 0) { mx = a.src[3 * (size_t)(w - 1)]; my = a.src[3 * (size_t)(w - 1) + 1]; mz = a.src[3 * (size_t)(w - 1) + 2]; }
                    ax += mx; ay += my; az += mz;
                }
                if (f & 8u) {
                    if (lane == 31 || i + 1 >= a.n_own) { px = a.src[3 * (size_t)(w + 1)]; py = a.src[3 * (size_t)(w + 1) + 1]; pz = a.src[3 * (size_t)(w + 1) + 2]; }
                    ax += px; ay += py; az += pz;
                }
                if (f & 1u) { ax += a.src[3 * (size_t)nb.x]; ay += a.src[3 * (size_t)nb.x + 1]; az += a.src[3 * (size_t)nb.x + 2]; }
                if (f & 2u) { ax += a.src[3 * (size_t)nb.y]; ay += a.src[3 * (size_t)nb.y + 1]; az += a.src[3 * (size_t)nb.y + 2]; }
                if (f & 16u) { ax += a.src[3 * (size_t)nb.z]; ay += a.src[3 * (size_t)nb.z + 1]; az += a.src[3 * (size_t)nb.z + 2]; }
                if (f & 32u) { ax += a.src[3 * (size_t)nb.w]; ay += a.src[3 * (size_t)nb.w + 1]; az += a.src[3 * (size_t)nb.w + 2]; }
                const float fd = (float)deg;
                sx += ax - fd * ox; sy += ay - fd * oy; sz += az - fd * oz;
            }
            // m = sum / N (N <= 6: multiply by the fp32 reciprocal), q = o + lambda m, clamp (Q8, Q9)
            const float inv = deg == 1 ? 1.f : deg == 2 ? 0.5f : deg == 3 ? (1.f / 3.f) : deg == 4 ? 0.25f
                            : deg == 5 ? 0.2f : (1.f / 6.f);
            nx = fminf(fmaxf(__fadd_rn(ox, __fmul_rn(a.lambda, __fmul_rn(sx, inv))), -a.d), a.d);
            ny = fminf(fmaxf(__fadd_rn(oy, __fmul_rn(a.lambda, __fmul_rn(sy, inv))), -a.d), a.d);
            nz = fminf(fmaxf(__fadd_rn(oz, __fmul_rn(a.lambda, __fmul_rn(sz, inv))), -a.d), a.d);
        }
        if (a.world) {
            a.world[3 * (size_t)w + 0] = world_of(a.points[3 * (size_t)w + 0], nx, a.org[0], a.sp[0]);
            a.world[3 * (size_t)w + 1] = world_of(a.points[3 * (size_t)w + 1], ny, a.org[1], a.sp[1]);
            a.world[3 * (size_t)w + 2] = world_of(a.points[3 * (size_t)w + 2], nz, a.org[2], a.sp[2]);
        } else {
            a.dst[3 * (size_t)w + 0] = nx; a.dst[3 * (size_t)w + 1] = ny; a.dst[3 * (size_t)w + 2] = nz;
        }
    }
}

// World coordinates of window entries [w0, w1) from offsets (NULL = anchors).
__global__ void __launch_bounds__(256) k_finalize(const float *offs, const float *points, float *out,
                                                  int64_t w0, int64_t w1, double sx, double sy, double sz,
                                                  double ox, double oy, double oz) {
    for (int64_t w = w0 + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; w < w1;
         w += (int64_t)gridDim.x * blockDim.x) {
        const float o0 = offs ? offs[3 * w] : 0.f, o1 = offs ? offs[3 * w + 1] : 0.f, o2 = offs ? offs[3 * w + 2] : 0.f;
        out[3 * w + 0] = world_of(points[3 * w + 0], o0, ox, sx);
        out[3 * w + 1] = world_of(points[3 * w + 1], o1, oy, sy);
        out[3 * w + 2] = world_of(points[3 * w + 2], o2, oz, sz);
    }
}

// Triangulation: quad q -> tris 2q, 2q+1 (reading Q13 / C-8: diagonals from the
// fp32 points in fp64, differences, squares, sum x+y+z; ties -> 0-2).
__global__ void __launch_bounds__(256) k_triangulate(const uint32_t *quads, const float *points, uint32_t *tris,
                                                     int64_t nQ, uint32_t win_base, int shortest) {
    for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < nQ; q += (int64_t)gridDim.x * blockDim.x) {
        const uint4 v = __ldg(reinterpret_cast<const uint4 *>(quads) + q);
        bool d02 = true;
        if (shortest) {
            const float *p0 = points + 3 * (int64_t)(v.x - win_base), *p1 = points + 3 * (int64_t)(v.y - win_base);
            const float *p2 = points + 3 * (int64_t)(v.z - win_base), *p3 = points + 3 * (int64_t)(v.w - win_base);
            double a0 = __dsub_rn((double)p2[0], (double)p0[0]), a1 = __dsub_rn((double)p2[1], (double)p0[1]);
            double a2 = __dsub_rn((double)p2[2], (double)p0[2]);
            double b0 = __dsub_rn((double)p3[0], (double)p1[0]), b1 = __dsub_rn((double)p3[1], (double)p1[1]);
            double b2 = __dsub_rn((double)p3[2], (double)p1[2]);
            const double da = __dadd_rn(__dadd_rn(__dmul_rn(a0, a0), __dmul_rn(a1, a1)), __dmul_rn(a2, a2));
            const double db = __dadd_rn(__dadd_rn(__dmul_rn(b0, b0), __dmul_rn(b1, b1)), __dmul_rn(b2, b2));
            d02 = da <= db;
        }
        uint2 *t = reinterpret_cast<uint2 *>(tris + 6 * q);
        if (d02) { t[0] = make_uint2(v.x, v.y); t[1] = make_uint2(v.z, v.x); t[2] = make_uint2(v.z, v.w); }
        else     { t[0] = make_uint2(v.x, v.y); t[1] = make_uint2(v.w, v.y); t[2] = make_uint2(v.z, v.w); }
    }
}

}  // namespace psn
