/*
 * psn_gen.cu -- seeded synthetic label-volume generator (CPU + GPU), see psn_gen.h.
 *
 * Recipe: SURVEY.md 8(d) "Generator recipe" (every choice there that resolves
 * BASELINE.json wording is restated in DESIGN.md section 5).  Input generation
 * only -- no SurfaceNets arithmetic lives here.
 *
 * Build (both paths in one library):
 *   nvcc -O2 -gencode arch=compute_100a,code=sm_100a --fmad=false
 *        -Xcompiler -fPIC,-ffp-contract=off -shared -o libpsngen.so psn_gen.cu
 */
#include "psn_gen.h"
#include <cuda_runtime.h>
#include <math.h>
#include <string.h>

#define GAMMA64 0x9E3779B97F4A7C15ull

/* ---------------------------------------------------------------- SplitMix64 */
__host__ __device__ static inline uint64_t sm_mix(uint64_t z)
{
    z ^= z >> 30; z *= 0xBF58476D1CE4E5B9ull;
    z ^= z >> 27; z *= 0x94D049BB133111EBull;
    z ^= z >> 31;
    return z;
}

extern "C" uint64_t psn_gen_splitmix_next(uint64_t *state)
{
    *state += GAMMA64;
    return sm_mix(*state);
}

static double u01(uint64_t *st) { return (double)(psn_gen_splitmix_next(st) >> 11) * 0x1.0p-53; }
static double unif(uint64_t *st, double a, double b) { return a + (b - a) * u01(st); }
static double logunif(uint64_t *st, double a, double b)
{
    double u = u01(st);
    return exp(log(a) + u * (log(b) - log(a)));
}

/* --------------------------------------------------------- per-voxel labels */
/* Pure function of (i,j,k) and the shape list.  fp64 in index units, no FMA
 * (host: -ffp-contract=off; device: --fmad=false), inclusive (<=) membership,
 * painter's order (the last containing shape wins). */

__host__ __device__ static inline int in_sphere(double x, double y, double z, const double *e)
{
    double dx = x - e[0], dy = y - e[1], dz = z - e[2];
    return dx * dx + dy * dy + dz * dz <= e[3] * e[3];
}

__host__ __device__ static inline int in_ellipsoid(double x, double y, double z, const double *e)
{
    double dx = x - e[0], dy = y - e[1], dz = z - e[2];
    /* bounding-box prefilter is part of the definition (identical on both sides) */
    if (fabs(dx) > e[3] || fabs(dy) > e[4] || fabs(dz) > e[5]) return 0;
    double tx = dx / e[3], ty = dy / e[4], tz = dz / e[5];
    return tx * tx + ty * ty + tz * tz <= 1.0;
}

__host__ __device__ static inline uint32_t voronoi(double x, double y, double z, const psn_gen_spec *s)
{
    double best = 1e300;
    int arg = 0;
    for (int n = 0; n < s->n_seeds; ++n) {
        double dx = x - s->seeds[n][0], dy = y - s->seeds[n][1], dz = z - s->seeds[n][2];
        double d = dx * dx + dy * dy + dz * dz;
        if (d < best) { best = d; arg = n; }   /* strict <: ties -> lowest index */
    }
    return (uint32_t)arg;
}

__host__ __device__ static inline int in_c4_ball(double x, double y, double z)
{
    double dx = x - 511.5, dy = y - 511.5, dz = z - 511.5;
    return dx * dx + dy * dy + dz * dz <= 491.52 * 491.52;
}

__host__ __device__ static inline int in_c3_body(double x, double y)
{
    double tx = (x - 255.5) / 230.4, ty = (y - 255.5) / 230.4;
    return tx * tx + ty * ty <= 1.0;
}

__host__ __device__ static uint32_t psn_gen_voxel(const psn_gen_spec *s, int64_t i, int64_t j, int64_t k)
{
    const double x = (double)i, y = (double)j, z = (double)k;
    uint32_t lab = 0;
    switch (s->kind) {
    case PSN_GEN_C1:
    case PSN_GEN_C5B:
    case PSN_GEN_SPHERES:
    case PSN_GEN_C6:
        for (int n = 0; n < s->n_ell; ++n)
            if (in_sphere(x, y, z, s->ell[n])) lab = s->ell_label[n];
        break;
    case PSN_GEN_C2: {
        double dx = (x - 127.5) / 115.2, dy = (y - 127.5) / 102.4, dz = (z - 127.5) / 89.6;
        if (dx * dx + dy * dy + dz * dz <= 1.0) lab = 1 + voronoi(x, y, z, s);
        break;
    }
    case PSN_GEN_C3:
        if (in_c3_body(x, y)) {
            lab = 1;
            for (int n = 0; n < s->n_ell; ++n)
                if (in_ellipsoid(x, y, z, s->ell[n])) lab = s->ell_label[n];
        }
        break;
    case PSN_GEN_C4:
        if (in_c4_ball(x, y, z)) {
            lab = 1 + voronoi(x, y, z, s);
            for (int n = 0; n < s->n_ell; ++n)
                if (in_ellipsoid(x, y, z, s->ell[n])) lab = s->ell_label[n];
        }
        break;
    case PSN_GEN_C5A: {
        uint64_t idx = (uint64_t)i + (uint64_t)s->dims[0] * ((uint64_t)j + (uint64_t)s->dims[1] * (uint64_t)k);
        lab = (uint32_t)(sm_mix(s->seed + GAMMA64 * (idx + 1)) >> 62);  /* (idx+1)-th SplitMix64 output */
        break;
    }
    }
    return lab;
}

/* ------------------------------------------------------------ shape drawing */
extern "C" int psn_gen_config(int kind, uint64_t seed, psn_gen_spec *s)
{
    if (kind == PSN_GEN_SPHERES) {
        if (s->n_ell < 0 || s->n_ell > PSN_GEN_MAX_ELL) return -1;
        if (s->dims[0] < 2 || s->dims[1] < 2 || s->dims[2] < 2) return -1;
        int n = s->n_ell, eb = s->elem_bytes;
        int64_t d[3] = { s->dims[0], s->dims[1], s->dims[2] };
        memset(s, 0, sizeof(*s));
        s->kind = kind; s->elem_bytes = eb; s->seed = seed; s->n_ell = n;
        for (int a = 0; a < 3; ++a) { s->dims[a] = d[a]; s->spacing[a] = 1.0; }
        uint64_t st = seed;
        double m = (double)(d[0] < d[1] ? (d[0] < d[2] ? d[0] : d[2]) : (d[1] < d[2] ? d[1] : d[2]));
        uint32_t maxlab = eb == 1 ? 255u : (eb == 2 ? 65535u : 0xFFFFFFFEu);
        for (int e = 0; e < n; ++e) {
            double r = unif(&st, 0.5, 0.5 + 0.25 * m);
            s->ell[e][0] = unif(&st, -1.0, (double)d[0]);
            s->ell[e][1] = unif(&st, -1.0, (double)d[1]);
            s->ell[e][2] = unif(&st, -1.0, (double)d[2]);
            s->ell[e][3] = s->ell[e][4] = s->ell[e][5] = r;
            s->ell_label[e] = (uint32_t)(1 + (e % maxlab));
        }
        return 0;
    }
    memset(s, 0, sizeof(*s));
    s->kind = kind;
    s->seed = seed;
    s->spacing[0] = s->spacing[1] = s->spacing[2] = 1.0;
    uint64_t st = seed;
    switch (kind) {
    case PSN_GEN_C1:
        s->elem_bytes = 2; s->dims[0] = s->dims[1] = s->dims[2] = 32;
        s->n_ell = 3;
        for (int n = 0; n < 3; ++n) {
            double r = unif(&st, 5.0, 9.0);
            for (int a = 0; a < 3; ++a) s->ell[n][a] = unif(&st, r + 1.0, 30.0 - r);
            s->ell[n][3] = s->ell[n][4] = s->ell[n][5] = r;
            s->ell_label[n] = (uint32_t)(n + 1);
        }
        return 0;
    case PSN_GEN_C2:
        s->elem_bytes = 1; s->dims[0] = s->dims[1] = s->dims[2] = 256;
        s->n_seeds = 20;
        for (int n = 0; n < 20; ++n)
            for (int a = 0; a < 3; ++a) s->seeds[n][a] = unif(&st, 0.0, 256.0);
        return 0;
    case PSN_GEN_C3:
        s->elem_bytes = 2; s->dims[0] = 512; s->dims[1] = 512; s->dims[2] = 600;
        s->spacing[0] = 0.8; s->spacing[1] = 0.8; s->spacing[2] = 1.5;
        s->n_ell = 100;
        for (int n = 0; n < 100; ++n) {
            double x, y; int tries = 0;
            do { x = unif(&st, 0.0, 512.0); y = unif(&st, 0.0, 512.0); ++tries; } while (!in_c3_body(x, y));
            if (n == 0) s->tries_first = tries;
            s->ell[n][0] = x; s->ell[n][1] = y; s->ell[n][2] = unif(&st, 0.0, 600.0);
            for (int a = 0; a < 3; ++a) s->ell[n][3 + a] = logunif(&st, 5.0, 60.0);
            s->ell_label[n] = (uint32_t)(n + 2);
        }
        return 0;
    case PSN_GEN_C4:
        s->elem_bytes = 2; s->dims[0] = s->dims[1] = s->dims[2] = 1024;
        s->n_seeds = 200;
        for (int n = 0; n < 200; ++n) {
            double x, y, z; int tries = 0;
            do { x = unif(&st, 0.0, 1024.0); y = unif(&st, 0.0, 1024.0); z = unif(&st, 0.0, 1024.0); ++tries; }
            while (!in_c4_ball(x, y, z));
            if (n == 0) s->tries_first = tries;
            s->seeds[n][0] = x; s->seeds[n][1] = y; s->seeds[n][2] = z;
        }
        s->n_ell = 300;
        for (int n = 0; n < 300; ++n) {
            double x, y, z;
            do { x = unif(&st, 0.0, 1024.0); y = unif(&st, 0.0, 1024.0); z = unif(&st, 0.0, 1024.0); }
            while (!in_c4_ball(x, y, z));
            s->ell[n][0] = x; s->ell[n][1] = y; s->ell[n][2] = z;
            for (int a = 0; a < 3; ++a) s->ell[n][3 + a] = logunif(&st, 5.0, 60.0);
            s->ell_label[n] = (uint32_t)(1 + (int)floor(200.0 * u01(&st)));
        }
        return 0;
    case PSN_GEN_C5A:
        s->elem_bytes = 1; s->dims[0] = s->dims[1] = s->dims[2] = 512;
        return 0;
    case PSN_GEN_C6:
        /* PAPER Table 1 "Synthetic" (5.21 M points, 10.55 M triangles): 128 labels as
         * overlapping spheres in painter's order, radius U[rmin, rmax) calibrated so that the quad
         * count is ~5.28 M, centres uniform in the volume (spheres may be clipped by its faces) */
        s->elem_bytes = 2; s->dims[0] = s->dims[1] = s->dims[2] = 512;
        s->n_ell = 128;
        for (int n = 0; n < 128; ++n) {
            double r = unif(&st, 48.0, 84.0);
            for (int a = 0; a < 3; ++a) s->ell[n][a] = unif(&st, 0.0, 511.0);
            s->ell[n][3] = s->ell[n][4] = s->ell[n][5] = r;
            s->ell_label[n] = (uint32_t)(n + 1);
        }
        return 0;
    case PSN_GEN_C5B:
        s->elem_bytes = 1; s->dims[0] = s->dims[1] = s->dims[2] = 512;
        s->n_ell = 1;
        s->ell[0][0] = s->ell[0][1] = s->ell[0][2] = 255.5;
        s->ell[0][3] = s->ell[0][4] = s->ell[0][5] = 16.0;
        s->ell_label[0] = 1;
        return 0;
    }
    return -1;
}

static int spec_ok(const psn_gen_spec *s, int64_t z_lo, int64_t z_hi)
{
    if (!s) return 0;
    if (s->elem_bytes != 1 && s->elem_bytes != 2 && s->elem_bytes != 4) return 0;
    if (z_lo < 0 || z_hi > s->dims[2] || z_lo > z_hi) return 0;
    return 1;
}

static inline void store(void *out, int eb, int64_t idx, uint32_t v)
{
    if (eb == 1) ((uint8_t *)out)[idx] = (uint8_t)v;
    else if (eb == 2) ((uint16_t *)out)[idx] = (uint16_t)v;
    else ((uint32_t *)out)[idx] = v;
}

extern "C" int psn_gen_host(const psn_gen_spec *s, int64_t z_lo, int64_t z_hi, void *out)
{
    if (!spec_ok(s, z_lo, z_hi) || !out) return -1;
    const int64_t M = s->dims[0], N = s->dims[1];
    for (int64_t k = z_lo; k < z_hi; ++k)
        for (int64_t j = 0; j < N; ++j)
            for (int64_t i = 0; i < M; ++i)
                store(out, s->elem_bytes, i + M * (j + N * (k - z_lo)), psn_gen_voxel(s, i, j, k));
    return 0;
}

/* ------------------------------------------------------------------ GPU path */
__constant__ psn_gen_spec c_spec;

template <typename T>
__global__ void __launch_bounds__(256) k_gen(int64_t z_lo, int64_t z_hi, T *out)
{
    const int64_t M = c_spec.dims[0], N = c_spec.dims[1];
    const int64_t total = M * N * (z_hi - z_lo);
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total;
         t += (int64_t)gridDim.x * blockDim.x) {
        int64_t i = t % M, r = t / M;
        int64_t j = r % N, k = r / N + z_lo;
        out[t] = (T)psn_gen_voxel(&c_spec, i, j, k);
    }
}

extern "C" int psn_gen_device(const psn_gen_spec *s, int64_t z_lo, int64_t z_hi, void *out, void *stream)
{
    if (!spec_ok(s, z_lo, z_hi) || !out) return -1;
    cudaStream_t st = (cudaStream_t)stream;
    cudaError_t e = cudaMemcpyToSymbolAsync(c_spec, s, sizeof(*s), 0, cudaMemcpyHostToDevice, st);
    if (e != cudaSuccess) return (int)e;
    int64_t total = s->dims[0] * s->dims[1] * (z_hi - z_lo);
    if (total == 0) return 0;
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    int64_t blocks = (total + 255) / 256;
    if (blocks > (int64_t)sms * 64) blocks = (int64_t)sms * 64;
    if (s->elem_bytes == 1) k_gen<uint8_t><<<(unsigned)blocks, 256, 0, st>>>(z_lo, z_hi, (uint8_t *)out);
    else if (s->elem_bytes == 2) k_gen<uint16_t><<<(unsigned)blocks, 256, 0, st>>>(z_lo, z_hi, (uint16_t *)out);
    else k_gen<uint32_t><<<(unsigned)blocks, 256, 0, st>>>(z_lo, z_hi, (uint32_t *)out);
    e = cudaGetLastError();
    if (e != cudaSuccess) return (int)e;
    /* the constant-memory spec must outlive the launch: synchronise the copy */
    e = cudaStreamSynchronize(st);
    return (int)e;
}
