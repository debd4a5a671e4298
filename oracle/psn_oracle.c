/*
 * psn_oracle.c -- plain, slow, single-threaded CPU SurfaceNets oracle.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and the
 * cpu_baseline / --impl reference legs of bench.py may load this library.
 * The product path (paper_2401_14906_b200/) never links, imports or calls it,
 * and this file shares no code, header, table or helper with it.
 *
 * What it computes is the plain definition of SurfaceNets as stated in
 * /root/reference/PAPER.md (cited "P:<line>"), with the readings listed in
 * DESIGN.md section 3 (Q1..Q24, mirroring SURVEY.md 8(c)):
 *
 *   - classification  cls(v) = v if v in L else B            P:53 (sec 2.1)
 *   - edge predicate   I(a,b) = cls(a) != cls(b)              P:58 (sec 2.2), reading Q1
 *   - a voxel emits one point at its centre iff any of its
 *     twelve edges is intersected
 *   - one quad per intersected lattice edge whose four sharing
 *     voxels exist (open boundaries)                           P:60, reading Q5
 *   - region-adjacency two-tuple per quad                      P:62, reading Q3/Q6
 *   - smoothing stencil: face neighbours whose shared face
 *     holds an intersected edge                                P:60, reading Q7
 *   - constrained Laplacian smoothing, Eq. 1, Jacobi           P:64-69, readings Q8-Q12
 *   - constraint box (per axis) or sphere at the voxel centre   P:69, readings Q10, Q26
 *   - triangulation: fixed, shorter diagonal, minimum area,
 *     most co-planar                                           P:97, readings Q13, Q27
 *
 * Nothing here is blocked, fused, trimmed, bit-sliced or scanned: every voxel
 * and every lattice edge is visited with the explicit edge lists below, in
 * row-major order (i fastest, then j, then k).  Extraction is exact integer
 * work (plus one fp64->fp32 rounding per point coordinate); smoothing runs in
 * fp64 in world coordinates.
 *
 * Build:  gcc -O2 -std=c99 -ffp-contract=off -fPIC -shared -o liboracle.so psn_oracle.c
 * (-ffp-contract=off: no FMA contraction, so every fp64 expression is the
 *  sequence of correctly rounded operations written here.)
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <math.h>

#define O_BACKGROUND 0xFFFFFFFFu  /* reading Q3: background sentinel in two-tuples */
#define O_NONE 0xFFFFFFFFu        /* "voxel has no point" in the id map */

/* ------------------------------------------------------------------------ */
/* Volume access                                                             */
/* ------------------------------------------------------------------------ */

typedef struct {
    const void *labels;   /* slices [z_lo, z_hi) of an M x N x O lattice, x fastest */
    int elem_bytes;       /* 1, 2 or 4 */
    int64_t M, N, O;      /* global lattice dims */
    int64_t z_lo, z_hi;
    const uint32_t *L;    /* selected labels, ascending, unique (unused if all_nonzero) */
    int64_t nL;
    int all_nonzero;      /* L = every non-zero value (reading Q2) */
} OVol;

/* raw scalar s_{i,j,k} */
static uint32_t o_raw(const OVol *v, int64_t i, int64_t j, int64_t k)
{
    int64_t idx = i + v->M * (j + v->N * (k - v->z_lo));
    if (v->elem_bytes == 1) return ((const uint8_t *)v->labels)[idx];
    if (v->elem_bytes == 2) return ((const uint16_t *)v->labels)[idx];
    return ((const uint32_t *)v->labels)[idx];
}

/* s in L ?   ("s_{i,j,k} in L ... background label B consisting of any s not in L") */
static int o_in_L(const OVol *v, uint32_t s)
{
    if (v->all_nonzero) return s != 0;
    /* plain binary search over the sorted label list */
    int64_t lo = 0, hi = v->nL;
    while (lo < hi) {
        int64_t mid = lo + (hi - lo) / 2;
        if (v->L[mid] == s) return 1;
        if (v->L[mid] < s) lo = mid + 1; else hi = mid;
    }
    return 0;
}

/* cls(s) = s if s in L else B  (reading Q1: classify first, then compare) */
static uint32_t o_cls(const OVol *v, int64_t i, int64_t j, int64_t k)
{
    uint32_t s = o_raw(v, i, j, k);
    return o_in_L(v, s) ? s : O_BACKGROUND;
}

/* Edge predicate: intersected iff s0 != s1 and not both background,
 * i.e. cls(s0) != cls(s1). */
static int o_I(uint32_t c0, uint32_t c1) { return c0 != c1; }

/* Lattice edges from point (i,j,k) towards +x / +y / +z (the voxel triad
 * edges of P:55).  Callers guarantee the far endpoint exists. */
static int o_X(const OVol *v, int64_t i, int64_t j, int64_t k)
{ return o_I(o_cls(v, i, j, k), o_cls(v, i + 1, j, k)); }
static int o_Y(const OVol *v, int64_t i, int64_t j, int64_t k)
{ return o_I(o_cls(v, i, j, k), o_cls(v, i, j + 1, k)); }
static int o_Z(const OVol *v, int64_t i, int64_t j, int64_t k)
{ return o_I(o_cls(v, i, j, k), o_cls(v, i, j, k + 1)); }

/* "If any of the cell's twelve edges is intersected, then a single
 * point is generated in the center of the voxel cell."  The twelve edges of
 * voxel (i,j,k): 4 x-edges, 4 y-edges, 4 z-edges. */
static int o_voxel_has_point(const OVol *v, int64_t i, int64_t j, int64_t k)
{
    return o_X(v, i, j, k)     || o_X(v, i, j + 1, k) ||
           o_X(v, i, j, k + 1) || o_X(v, i, j + 1, k + 1) ||
           o_Y(v, i, j, k)     || o_Y(v, i + 1, j, k) ||
           o_Y(v, i, j, k + 1) || o_Y(v, i + 1, j, k + 1) ||
           o_Z(v, i, j, k)     || o_Z(v, i + 1, j, k) ||
           o_Z(v, i, j + 1, k) || o_Z(v, i + 1, j + 1, k);
}

/* Faces in stencil order (reading Q7 / C-5): -z, -y, -x, +x, +y, +z. */
enum { F_MZ = 0, F_MY = 1, F_MX = 2, F_PX = 3, F_PY = 4, F_PZ = 5 };
static const int64_t F_DI[6] = { 0, 0, -1, 1, 0, 0 };
static const int64_t F_DJ[6] = { 0, -1, 0, 0, 1, 0 };
static const int64_t F_DK[6] = { -1, 0, 0, 0, 0, 1 };

/* The four edges bounding face f of voxel (i,j,k).  P:60: "for every
 * intersected edge, two voxel cell face neighbors are necessarily connected";
 * a face is selected iff one of its four edges is intersected. */
static int o_face(const OVol *v, int64_t i, int64_t j, int64_t k, int f)
{
    switch (f) {
    case F_MX: return o_Y(v, i, j, k) || o_Y(v, i, j, k + 1) || o_Z(v, i, j, k) || o_Z(v, i, j + 1, k);
    case F_PX: return o_Y(v, i + 1, j, k) || o_Y(v, i + 1, j, k + 1) || o_Z(v, i + 1, j, k) || o_Z(v, i + 1, j + 1, k);
    case F_MY: return o_X(v, i, j, k) || o_X(v, i, j, k + 1) || o_Z(v, i, j, k) || o_Z(v, i + 1, j, k);
    case F_PY: return o_X(v, i, j + 1, k) || o_X(v, i, j + 1, k + 1) || o_Z(v, i, j + 1, k) || o_Z(v, i + 1, j + 1, k);
    case F_MZ: return o_X(v, i, j, k) || o_X(v, i, j + 1, k) || o_Y(v, i, j, k) || o_Y(v, i + 1, j, k);
    case F_PZ: return o_X(v, i, j, k + 1) || o_X(v, i, j + 1, k + 1) || o_Y(v, i, j, k + 1) || o_Y(v, i + 1, j, k + 1);
    }
    return 0;
}

/* Is (i,j,k) a voxel of the M x N x O lattice?  (voxels: i<M-1, j<N-1, k<O-1) */
static int o_is_voxel(const OVol *v, int64_t i, int64_t j, int64_t k)
{
    return i >= 0 && j >= 0 && k >= 0 && i < v->M - 1 && j < v->N - 1 && k < v->O - 1;
}

/* Number of stencil entries of voxel (i,j,k): faces with an intersected edge
 * whose neighbour voxel exists. */
static int o_stencil_degree(const OVol *v, int64_t i, int64_t j, int64_t k)
{
    int d = 0;
    for (int f = 0; f < 6; ++f)
        if (o_face(v, i, j, k, f) && o_is_voxel(v, i + F_DI[f], j + F_DJ[f], k + F_DK[f])) ++d;
    return d;
}

/* Quads owned by voxel (i,j,k): one per intersected triad edge (x, y, z) whose
 * four sharing voxels exist (open boundaries P:264 / reading Q5). */
static int o_quad_x(const OVol *v, int64_t i, int64_t j, int64_t k) { return j >= 1 && k >= 1 && o_X(v, i, j, k); }
static int o_quad_y(const OVol *v, int64_t i, int64_t j, int64_t k) { return i >= 1 && k >= 1 && o_Y(v, i, j, k); }
static int o_quad_z(const OVol *v, int64_t i, int64_t j, int64_t k) { return i >= 1 && j >= 1 && o_Z(v, i, j, k); }

static int o_check_args(const OVol *v)
{
    if (v->M < 2 || v->N < 2 || v->O < 2) return -1;
    if (v->elem_bytes != 1 && v->elem_bytes != 2 && v->elem_bytes != 4) return -1;
    if (v->z_lo < 0 || v->z_hi > v->O || v->z_lo >= v->z_hi) return -1;
    if (!v->all_nonzero && v->nL > 0 && v->L == NULL) return -1;
    return 0;
}

/* ------------------------------------------------------------------------ */
/* Per-layer counts                                                          */
/* ------------------------------------------------------------------------ */

/* For every voxel layer k in [k0, k1): number of points, owned quads and
 * directed stencil entries ("the number of output points,
 * quadrilaterals, and smoothing stencil edges").  Needs slices [k0, k1].
 * Returns 0, or -1 on bad arguments. */
int oracle_layer_counts(const void *labels, int elem_bytes,
                        int64_t M, int64_t N, int64_t O, int64_t z_lo, int64_t z_hi,
                        const uint32_t *L, int64_t nL, int all_nonzero,
                        int64_t k0, int64_t k1,
                        int64_t *P_layer, int64_t *Q_layer, int64_t *S_layer)
{
    OVol v = { labels, elem_bytes, M, N, O, z_lo, z_hi, L, nL, all_nonzero };
    if (o_check_args(&v)) return -1;
    if (k0 < 0 || k1 > O - 1 || k0 > k1) return -1;
    if (k0 < k1 && (k0 < z_lo || k1 + 1 > z_hi)) return -1;
    for (int64_t k = k0; k < k1; ++k) {
        int64_t p = 0, q = 0, s = 0;
        for (int64_t j = 0; j < N - 1; ++j)
            for (int64_t i = 0; i < M - 1; ++i) {
                if (!o_voxel_has_point(&v, i, j, k)) continue;
                ++p;
                q += o_quad_x(&v, i, j, k) + o_quad_y(&v, i, j, k) + o_quad_z(&v, i, j, k);
                s += o_stencil_degree(&v, i, j, k);
            }
        if (P_layer) P_layer[k - k0] = p;
        if (Q_layer) Q_layer[k - k0] = q;
        if (S_layer) S_layer[k - k0] = s;
    }
    return 0;
}

/* ------------------------------------------------------------------------ */
/* Row trims (Pass 1 and Pass 2)                                             */
/* ------------------------------------------------------------------------ */

/* For every grid row E_{j,k} (j in [0,N), k in [k0,k1)), the computational
 * trim of PAPER sec 2.3:
 *   Pass 1: "the x-edges are classified ... and the trim positions
 *     xL and xR (first and last x-edge intersection)" -- xl1/xr1 = the
 *     tightest half-open interval [xL, xR) holding every i with X(i,j,k);
 *   Pass 2: "the y- and z-edges are classified ... and the trim
 *     positions adjusted" -- xl/xr = the tightest interval holding every i with
 *     X(i,j,k), Y(i,j,k) (if j+1 < N) or Z(i,j,k) (if k+1 < O).
 * An empty row gets [0, 0).  Arrays are [k1-k0][N], row r = j + N (k-k0).
 * Needs slices [k0, min(k1+1, O)).  Returns 0 or -1 on bad arguments. */
int oracle_row_trims(const void *labels, int elem_bytes,
                     int64_t M, int64_t N, int64_t O, int64_t z_lo, int64_t z_hi,
                     const uint32_t *L, int64_t nL, int all_nonzero,
                     int64_t k0, int64_t k1,
                     int64_t *xl1, int64_t *xr1, int64_t *xl, int64_t *xr)
{
    OVol v = { labels, elem_bytes, M, N, O, z_lo, z_hi, L, nL, all_nonzero };
    if (o_check_args(&v)) return -1;
    if (k0 < 0 || k1 > O || k0 > k1) return -1;
    if (k0 < k1 && (k0 < z_lo || (k1 < O ? k1 + 1 : O) > z_hi)) return -1;
    for (int64_t k = k0; k < k1; ++k)
        for (int64_t j = 0; j < N; ++j) {
            int64_t r = j + N * (k - k0);
            int64_t a1 = -1, b1 = -1, a = -1, b = -1;   /* first / last intersection, -1 = none */
            for (int64_t i = 0; i < M; ++i) {
                int x = i + 1 < M && o_X(&v, i, j, k);
                int y = j + 1 < N && o_Y(&v, i, j, k);
                int z = k + 1 < O && o_Z(&v, i, j, k);
                if (x) { if (a1 < 0) a1 = i; b1 = i; }
                if (x || y || z) { if (a < 0) a = i; b = i; }
            }
            xl1[r] = a1 < 0 ? 0 : a1; xr1[r] = a1 < 0 ? 0 : b1 + 1;
            xl[r] = a < 0 ? 0 : a;    xr[r] = a < 0 ? 0 : b + 1;
        }
    return 0;
}

/* ------------------------------------------------------------------------ */
/* Extraction                                                                */
/* ------------------------------------------------------------------------ */

/*
 * Extract the mesh owned by voxel layers [k0, k1) (k0 < k1 <= O-1).
 *
 * Input slices [z_lo, z_hi) must contain [max(k0-1,0), min(k1+1,O-1)] so that
 * the ids of the neighbouring layers k0-1 and k1 can be assigned.
 *
 * Point ids are global: the first point of layer k0 has id `point_base`;
 * ids increase in row-major voxel order (reading Q4), so layer k0-1's points
 * end at point_base-1 and layer k1's start right after layer k1-1's.
 * CSR offsets start at `stencil_base`.
 *
 * Outputs (caller-allocated, may all be NULL to only count):
 *   points     float[nP][3]   voxel centres, fl32(origin + (idx+0.5)*spacing) in fp64  (C-3)
 *   anchors    double[nP][3]  the same centres in fp64 (smoothing start, reading Q23)
 *   voxel_idx  int64[nP][3]   (i,j,k) of each point's voxel
 *   quads      uint32[nQ][4]  voxel-major, then x<y<z, winding C-4
 *   pairs      uint32[nQ][2]  (cls at edge origin, cls at far end)
 *   csr_off    uint32[nP+1]   stencil_base + running count
 *   csr_ids    uint32[nS]     neighbours in face order -z,-y,-x,+x,+y,+z
 *   face_mask  uint8[nP]      bit f set iff the CSR row holds the face-f neighbour
 * Capacities are checked; returns 0, -1 on bad args, -2 if a capacity is short
 * (counts are still returned).
 */
int oracle_extract(const void *labels, int elem_bytes,
                   int64_t M, int64_t N, int64_t O, int64_t z_lo, int64_t z_hi,
                   const uint32_t *L, int64_t nL, int all_nonzero,
                   const double *spacing, const double *origin,
                   int64_t k0, int64_t k1, int64_t point_base, int64_t stencil_base,
                   float *points, double *anchors, int64_t *voxel_idx,
                   uint32_t *quads, uint32_t *pairs,
                   uint32_t *csr_off, uint32_t *csr_ids, uint8_t *face_mask,
                   int64_t capP, int64_t capQ, int64_t capS,
                   int64_t *nP_out, int64_t *nQ_out, int64_t *nS_out)
{
    OVol v = { labels, elem_bytes, M, N, O, z_lo, z_hi, L, nL, all_nonzero };
    if (o_check_args(&v)) return -1;
    if (k0 < 0 || k1 > O - 1 || k0 >= k1) return -1;
    const int64_t ka = k0 > 0 ? k0 - 1 : 0;          /* first layer with ids */
    const int64_t kb = k1 < O - 1 ? k1 + 1 : O - 1;  /* one past last layer with ids */
    if (z_lo > ka || z_hi < kb + 1) return -1;

    const int64_t VX = M - 1, VY = N - 1;
    const int64_t layer = VX * VY;
    uint32_t *idmap = (uint32_t *)malloc((size_t)(layer * (kb - ka)) * sizeof(uint32_t));
    if (!idmap) return -3;

    /* Assign ids in row-major order.  Points of layer k0-1 precede point_base. */
    int64_t before = 0;
    if (ka < k0)
        for (int64_t j = 0; j < VY; ++j)
            for (int64_t i = 0; i < VX; ++i)
                if (o_voxel_has_point(&v, i, j, ka)) ++before;
    int64_t next = point_base - before;
    for (int64_t k = ka; k < kb; ++k)
        for (int64_t j = 0; j < VY; ++j)
            for (int64_t i = 0; i < VX; ++i) {
                uint32_t id = O_NONE;
                if (o_voxel_has_point(&v, i, j, k)) id = (uint32_t)(next++);
                idmap[(k - ka) * layer + j * VX + i] = id;
            }
#define ID(ii, jj, kk) idmap[((kk) - ka) * layer + (jj) * VX + (ii)]

    int64_t nP = 0, nQ = 0, nS = 0;
    int over = 0;
    if (csr_off) csr_off[0] = (uint32_t)stencil_base;   /* caller allocates capP + 1 entries */
    for (int64_t k = k0; k < k1; ++k)
        for (int64_t j = 0; j < VY; ++j)
            for (int64_t i = 0; i < VX; ++i) {
                uint32_t id = ID(i, j, k);
                if (id == O_NONE) continue;
                /* --- the point (C-3): voxel centre, fp64 then one rounding --- */
                if (nP < capP) {
                    int64_t idx[3] = { i, j, k };
                    for (int a = 0; a < 3; ++a) {
                        double c = origin[a] + ((double)idx[a] + 0.5) * spacing[a];
                        if (points) points[nP * 3 + a] = (float)c;
                        if (anchors) anchors[nP * 3 + a] = c;
                        if (voxel_idx) voxel_idx[nP * 3 + a] = idx[a];
                    }
                } else if (points || anchors || voxel_idx) over = 1;
                /* --- quads owned by this voxel, axes in the order x, y, z (C-4) --- */
                if (o_quad_x(&v, i, j, k)) {
                    if (nQ < capQ && quads) {
                        uint32_t *q = quads + nQ * 4;
                        q[0] = ID(i, j - 1, k - 1); q[1] = ID(i, j, k - 1);
                        q[2] = ID(i, j, k);         q[3] = ID(i, j - 1, k);
                        pairs[nQ * 2 + 0] = o_cls(&v, i, j, k);
                        pairs[nQ * 2 + 1] = o_cls(&v, i + 1, j, k);
                    } else if (quads && nQ >= capQ) over = 1;
                    ++nQ;
                }
                if (o_quad_y(&v, i, j, k)) {
                    if (nQ < capQ && quads) {
                        uint32_t *q = quads + nQ * 4;
                        q[0] = ID(i - 1, j, k - 1); q[1] = ID(i - 1, j, k);
                        q[2] = ID(i, j, k);         q[3] = ID(i, j, k - 1);
                        pairs[nQ * 2 + 0] = o_cls(&v, i, j, k);
                        pairs[nQ * 2 + 1] = o_cls(&v, i, j + 1, k);
                    } else if (quads && nQ >= capQ) over = 1;
                    ++nQ;
                }
                if (o_quad_z(&v, i, j, k)) {
                    if (nQ < capQ && quads) {
                        uint32_t *q = quads + nQ * 4;
                        q[0] = ID(i - 1, j - 1, k); q[1] = ID(i, j - 1, k);
                        q[2] = ID(i, j, k);         q[3] = ID(i - 1, j, k);
                        pairs[nQ * 2 + 0] = o_cls(&v, i, j, k);
                        pairs[nQ * 2 + 1] = o_cls(&v, i, j, k + 1);
                    } else if (quads && nQ >= capQ) over = 1;
                    ++nQ;
                }
                /* --- stencil row (C-5): faces in order -z,-y,-x,+x,+y,+z --- */
                uint8_t mask = 0;
                for (int f = 0; f < 6; ++f) {
                    int64_t ni = i + F_DI[f], nj = j + F_DJ[f], nk = k + F_DK[f];
                    if (!o_face(&v, i, j, k, f) || !o_is_voxel(&v, ni, nj, nk)) continue;
                    mask |= (uint8_t)(1u << f);
                    if (nS < capS && csr_ids) csr_ids[nS] = ID(ni, nj, nk);
                    else if (csr_ids && nS >= capS) over = 1;
                    ++nS;
                }
                if (nP < capP && face_mask) face_mask[nP] = mask;
                ++nP;
                if (csr_off && nP < capP + 1) csr_off[nP] = (uint32_t)(stencil_base + nS);
            }
#undef ID
    free(idmap);
    if (nP_out) *nP_out = nP;
    if (nQ_out) *nQ_out = nQ;
    if (nS_out) *nS_out = nS;
    return over ? -2 : 0;
}

/* ------------------------------------------------------------------------ */
/* Smoothing (Eq. 1), fp64, world coordinates                  */
/* ------------------------------------------------------------------------ */

/*
 * Jacobi constrained Laplacian smoothing.
 *   P^0 = anchors (exact fp64 voxel centres, reading Q23)
 *   for t = 1..T, for every point i with N = deg(i) > 0 and not frozen:
 *       m = (1/N) * sum_{j in stencil(i)} (P^{t-1}_j - P^{t-1}_i)     (Eq. 1, reading Q8)
 *       q = P^{t-1}_i + lambda * m
 *       shape 0 (box):    P^t_i = clamp(q, anchor_i - d*s, anchor_i + d*s) per axis
 *                         ("a fraction of the hexahedral voxel cell", readings Q9/Q10)
 *       shape 1 (sphere): r = d * min(s); if |q - anchor_i| > r then
 *                         P^t_i = anchor_i + (q - anchor_i) * (r / |q - anchor_i|), else q
 *                         ("a constraint sphere centered at the voxel center point",
 *                          reading Q26; the norm is sqrt(dx*dx + dy*dy + dz*dz) in that order)
 *   deg 0 or frozen: P^t_i = P^{t-1}_i.
 * csr_ids are global ids; local index = id - id_base.  `frozen` (may be NULL)
 * marks points held fixed (used only by windowed tests: errors entering from
 * frozen points move at most one stencil hop per iteration).
 * out: double[nP][3].
 */
int oracle_smooth(int64_t nP, const double *anchors, const uint32_t *csr_off,
                  const uint32_t *csr_ids, int64_t id_base, const uint8_t *frozen,
                  const double *spacing, int32_t T, double lambda, double d, int shape, double *out)
{
    if (nP < 0 || T < 0 || !(lambda >= 0.0 && lambda <= 1.0) || !(d >= 0.0)) return -1;
    if (shape != 0 && shape != 1) return -1;
    double smin = spacing[0];
    if (spacing[1] < smin) smin = spacing[1];
    if (spacing[2] < smin) smin = spacing[2];
    const double r = d * smin;   /* sphere radius, world units */
    double *cur = (double *)malloc((size_t)(nP > 0 ? nP : 1) * 3 * sizeof(double));
    double *nxt = (double *)malloc((size_t)(nP > 0 ? nP : 1) * 3 * sizeof(double));
    if (!cur || !nxt) { free(cur); free(nxt); return -3; }
    memcpy(cur, anchors, (size_t)nP * 3 * sizeof(double));
    const uint32_t off0 = nP > 0 ? csr_off[0] : 0;
    for (int32_t t = 0; t < T; ++t) {
        for (int64_t i = 0; i < nP; ++i) {
            uint32_t b = csr_off[i] - off0, e = csr_off[i + 1] - off0;
            int64_t N = (int64_t)e - (int64_t)b;
            if (N == 0 || (frozen && frozen[i])) {
                for (int a = 0; a < 3; ++a) nxt[i * 3 + a] = cur[i * 3 + a];
                continue;
            }
            double q[3];
            for (int a = 0; a < 3; ++a) {
                double sum = 0.0;
                for (uint32_t n = b; n < e; ++n) {
                    int64_t jdx = (int64_t)csr_ids[n] - id_base;
                    sum += cur[jdx * 3 + a] - cur[i * 3 + a];
                }
                double m = sum / (double)N;
                q[a] = cur[i * 3 + a] + lambda * m;
            }
            if (shape == 0) {
                for (int a = 0; a < 3; ++a) {
                    double lo = anchors[i * 3 + a] - d * spacing[a];
                    double hi = anchors[i * 3 + a] + d * spacing[a];
                    nxt[i * 3 + a] = q[a] < lo ? lo : (q[a] > hi ? hi : q[a]);
                }
            } else {
                double dx = q[0] - anchors[i * 3 + 0];
                double dy = q[1] - anchors[i * 3 + 1];
                double dz = q[2] - anchors[i * 3 + 2];
                double len = sqrt(dx * dx + dy * dy + dz * dz);
                if (len > r) {
                    double f = r / len;
                    nxt[i * 3 + 0] = anchors[i * 3 + 0] + dx * f;
                    nxt[i * 3 + 1] = anchors[i * 3 + 1] + dy * f;
                    nxt[i * 3 + 2] = anchors[i * 3 + 2] + dz * f;
                } else {
                    for (int a = 0; a < 3; ++a) nxt[i * 3 + a] = q[a];
                }
            }
        }
        double *tmp = cur; cur = nxt; nxt = tmp;   /* double buffering */
    }
    memcpy(out, cur, (size_t)nP * 3 * sizeof(double));
    free(cur); free(nxt);
    return 0;
}

/* ------------------------------------------------------------------------ */
/* Triangulation                                                      */
/* ------------------------------------------------------------------------ */

/* twice the area of triangle (p, q, r) = |(q - p) x (r - p)|, fp64 from fp32 points
 * (differences exact; products, differences, sum x+y+z, sqrt correctly rounded) */
static void tri_normal(const float *p, const float *q, const float *r, double n[3])
{
    double u0 = (double)q[0] - (double)p[0], u1 = (double)q[1] - (double)p[1], u2 = (double)q[2] - (double)p[2];
    double v0 = (double)r[0] - (double)p[0], v1 = (double)r[1] - (double)p[1], v2 = (double)r[2] - (double)p[2];
    n[0] = u1 * v2 - u2 * v1;
    n[1] = u2 * v0 - u0 * v2;
    n[2] = u0 * v1 - u1 * v0;
}

static double norm3(const double n[3]) { return sqrt(n[0] * n[0] + n[1] * n[1] + n[2] * n[2]); }

/* cosine of the angle between the two triangles' normals; 1 if either is degenerate */
static double coplanarity(const double n[3], const double m[3])
{
    double den = norm3(n) * norm3(m);
    if (den == 0.0) return 1.0;
    return (n[0] * m[0] + n[1] * m[1] + n[2] * m[2]) / den;
}

/*
 * Each quad (a,b,c,d) -> two triangles: diagonal 0-2 gives (a,b,c),(a,c,d),
 * diagonal 1-3 gives (a,b,d),(b,c,d); triangles 2q and 2q+1 come from quad q.
 * Quantities are computed in fp64 from the given fp32 points (reading Q13):
 *   strategy 0: fixed 0-2 ("greedy", reading Q13)
 *   strategy 1: shorter diagonal: |c-a|^2 <= |d-b|^2 (differences, squares,
 *               sum x+y+z)
 *   strategy 2: minimum area: |n(a,b,c)| + |n(a,c,d)| <= |n(a,b,d)| + |n(b,c,d)|
 *               (n = cross product, twice the triangle area; reading Q27)
 *   strategy 3: most co-planar: cos(n(a,b,c), n(a,c,d)) >= cos(n(a,b,d), n(b,c,d))
 *               (the smaller dihedral deviation; degenerate normals count as
 *               co-planar; reading Q27)
 * Ties go to 0-2.  point index = id - id_base.
 */
int oracle_triangulate(int64_t nQ, const uint32_t *quads, const float *points,
                       int64_t id_base, int strategy, uint32_t *tris)
{
    if (strategy < 0 || strategy > 3) return -1;
    for (int64_t q = 0; q < nQ; ++q) {
        const uint32_t *v = quads + q * 4;
        int diag02 = 1;
        const float *p0 = points + ((int64_t)v[0] - id_base) * 3;
        const float *p1 = points + ((int64_t)v[1] - id_base) * 3;
        const float *p2 = points + ((int64_t)v[2] - id_base) * 3;
        const float *p3 = points + ((int64_t)v[3] - id_base) * 3;
        if (strategy == 1) {
            double a0 = (double)p2[0] - (double)p0[0];
            double a1 = (double)p2[1] - (double)p0[1];
            double a2 = (double)p2[2] - (double)p0[2];
            double b0 = (double)p3[0] - (double)p1[0];
            double b1 = (double)p3[1] - (double)p1[1];
            double b2 = (double)p3[2] - (double)p1[2];
            double d02 = a0 * a0 + a1 * a1 + a2 * a2;
            double d13 = b0 * b0 + b1 * b1 + b2 * b2;
            diag02 = d02 <= d13;
        } else if (strategy >= 2) {
            double n1[3], n2[3], m1[3], m2[3];
            tri_normal(p0, p1, p2, n1);   /* (a,b,c) */
            tri_normal(p0, p2, p3, n2);   /* (a,c,d) */
            tri_normal(p0, p1, p3, m1);   /* (a,b,d) */
            tri_normal(p1, p2, p3, m2);   /* (b,c,d) */
            if (strategy == 2) diag02 = norm3(n1) + norm3(n2) <= norm3(m1) + norm3(m2);
            else diag02 = coplanarity(n1, n2) >= coplanarity(m1, m2);
        }
        uint32_t *t = tris + q * 6;
        if (diag02) { t[0] = v[0]; t[1] = v[1]; t[2] = v[2]; t[3] = v[0]; t[4] = v[2]; t[5] = v[3]; }
        else        { t[0] = v[0]; t[1] = v[1]; t[2] = v[3]; t[3] = v[1]; t[4] = v[2]; t[5] = v[3]; }
    }
    return 0;
}
