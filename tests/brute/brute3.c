/*
 * brute3.c -- exhaustive pin of the oracle over ALL 2^27 two-label 3x3x3
 * volumes (labels {0,1}, L = {1}) or a strided subset (argv[1] = stride).
 *
 * For every volume it calls oracle_extract() (oracle/psn_oracle.c) and checks
 * it against an independent formulation written here (corner / face based,
 * not the oracle's 12-edge lists):
 *   - P = #voxels whose 8 corners are not all equal
 *   - Q = #interior lattice edges with differing endpoints
 *   - S = 2 * #interior faces whose 4 corners are not all equal
 *   - every quad's 4 vertices are the 4 voxels around its edge, first vertex
 *     the smallest id, normal (q2-q0)x(q3-q1) along +axis, pair = (origin, far)
 *   - the stencil is symmetric and popcount(face mask) == degree
 * Prints "ok <volumes>" or the first failing volume.  Test infrastructure.
 */
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>

int oracle_extract(const void *labels, int elem_bytes,
                   int64_t M, int64_t N, int64_t O, int64_t z_lo, int64_t z_hi,
                   const uint32_t *L, int64_t nL, int all_nonzero,
                   const double *spacing, const double *origin,
                   int64_t k0, int64_t k1, int64_t point_base, int64_t stencil_base,
                   float *points, double *anchors, int64_t *voxel_idx,
                   uint32_t *quads, uint32_t *pairs,
                   uint32_t *csr_off, uint32_t *csr_ids, uint8_t *face_mask,
                   int64_t capP, int64_t capQ, int64_t capS,
                   int64_t *nP_out, int64_t *nQ_out, int64_t *nS_out);

#define V(i, j, k) lab[(i) + 3 * ((j) + 3 * (k))]

static int check(uint32_t bits)
{
    uint8_t lab[27];
    for (int t = 0; t < 27; ++t) lab[t] = (bits >> t) & 1u;
    const double sp[3] = { 1, 1, 1 }, org[3] = { 0, 0, 0 };
    float pts[8 * 3]; double anc[8 * 3]; int64_t vidx[8 * 3];
    uint32_t quads[6 * 4], pairs[6 * 2], off[9], ids[24];
    uint8_t fm[8];
    int64_t nP, nQ, nS;
    if (oracle_extract(lab, 1, 3, 3, 3, 0, 3, NULL, 0, 1, sp, org, 0, 2, 0, 0,
                       pts, anc, vidx, quads, pairs, off, ids, fm, 8, 6, 24, &nP, &nQ, &nS) != 0)
        return 1;
    /* independent counts */
    int P = 0, Q = 0, S = 0;
    int vid[2][2][2];
    for (int k = 0; k < 2; ++k) for (int j = 0; j < 2; ++j) for (int i = 0; i < 2; ++i) {
        int c = V(i, j, k), same = 1;
        for (int d = 1; d < 8; ++d) if (V(i + (d & 1), j + ((d >> 1) & 1), k + (d >> 2)) != c) same = 0;
        vid[k][j][i] = same ? -1 : P;
        if (!same) ++P;
    }
    /* interior edges of a 3^3 lattice: through the centre lines */
    for (int i = 0; i < 2; ++i) Q += V(i, 1, 1) != V(i + 1, 1, 1);
    for (int j = 0; j < 2; ++j) Q += V(1, j, 1) != V(1, j + 1, 1);
    for (int k = 0; k < 2; ++k) Q += V(1, 1, k) != V(1, 1, k + 1);
    /* interior faces: planes x=1, y=1, z=1, each split into 4 unit faces */
    for (int a = 0; a < 3; ++a)
        for (int u = 0; u < 2; ++u) for (int w = 0; w < 2; ++w) {
            int c[4], n = 0;
            for (int du = 0; du < 2; ++du) for (int dw = 0; dw < 2; ++dw) {
                int p[3]; p[a] = 1; p[(a + 1) % 3] = u + du; p[(a + 2) % 3] = w + dw;
                c[n++] = V(p[0], p[1], p[2]);
            }
            S += 2 * (c[1] != c[0] || c[2] != c[0] || c[3] != c[0]);
        }
    if (nP != P || nQ != Q || nS != S) return 2;
    /* quads: geometry, orientation, pairs */
    for (int q = 0; q < nQ; ++q) {
        const uint32_t *v = quads + 4 * q;
        int axis = -1;
        double c[4][3];
        for (int t = 0; t < 4; ++t) for (int a = 0; a < 3; ++a) c[t][a] = anc[v[t] * 3 + a];
        double e0[3], e1[3], n[3];
        for (int a = 0; a < 3; ++a) { e0[a] = c[2][a] - c[0][a]; e1[a] = c[3][a] - c[1][a]; }
        n[0] = e0[1] * e1[2] - e0[2] * e1[1];
        n[1] = e0[2] * e1[0] - e0[0] * e1[2];
        n[2] = e0[0] * e1[1] - e0[1] * e1[0];
        for (int a = 0; a < 3; ++a) if (n[a] > 0.5) axis = a;
        if (axis < 0) return 3;
        for (int a = 0; a < 3; ++a) if (a != axis && (n[a] > 1e-9 || n[a] < -1e-9)) return 4;
        /* the 4 vertex voxels share the lattice edge along `axis`: all have the
         * same coordinate along axis, and the other two coords cover {0,1}^2 */
        int ax0 = (int)vidx[v[0] * 3 + axis], seen = 0;
        for (int t = 0; t < 4; ++t) {
            if ((int)vidx[v[t] * 3 + axis] != ax0) return 5;
            int b = (int)vidx[v[t] * 3 + (axis + 1) % 3] + 2 * (int)vidx[v[t] * 3 + (axis + 2) % 3];
            seen |= 1 << b;
            if (v[t] < v[0]) return 6;
        }
        if (seen != 15) return 7;
        int o[3] = { 1, 1, 1 }; o[axis] = ax0;
        int f[3] = { 1, 1, 1 }; f[axis] = ax0 + 1;
        uint32_t co = V(o[0], o[1], o[2]) ? 1u : 0xFFFFFFFFu, cf = V(f[0], f[1], f[2]) ? 1u : 0xFFFFFFFFu;
        if (pairs[2 * q] != co || pairs[2 * q + 1] != cf || co == cf) return 8;
    }
    /* stencil symmetric, popcount(face mask) == degree */
    for (int p = 0; p < nP; ++p) {
        int deg = (int)(off[p + 1] - off[p]);
        if (__builtin_popcount(fm[p]) != deg) return 9;
        for (uint32_t e = off[p]; e < off[p + 1]; ++e) {
            uint32_t w = ids[e];
            int found = 0;
            for (uint32_t e2 = off[w]; e2 < off[w + 1]; ++e2) if (ids[e2] == (uint32_t)p) found = 1;
            if (!found) return 10;
        }
    }
    (void)vid;
    return 0;
}

int main(int argc, char **argv)
{
    uint32_t stride = argc > 1 ? (uint32_t)strtoul(argv[1], NULL, 10) : 1u;
    if (stride == 0) stride = 1;
    long long n = 0;
    int bad = 0; uint32_t badv = 0, badc = 0;
#pragma omp parallel for schedule(dynamic, 65536) reduction(+:n)
    for (long long b = 0; b < (1LL << 27); b += stride) {
        int r = check((uint32_t)b);
        ++n;
        if (r) {
#pragma omp critical
            { if (!bad) { bad = 1; badv = (uint32_t)b; badc = (uint32_t)r; } }
        }
    }
    if (bad) { printf("FAIL volume=0x%07x code=%u\n", badv, badc); return 1; }
    printf("ok %lld\n", n);
    return 0;
}
