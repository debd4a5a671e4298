/*
 * psn_gen.h -- seeded synthetic label-volume generator (SURVEY.md 8(d) recipe).
 *
 * This module is INPUT GENERATION ONLY.  It holds none of the SurfaceNets
 * arithmetic: it produces label volumes shaped like the paper's workloads
 * (stood in for by BASELINE.json configs c1-c5), which the
 * CUDA path and the oracle then both consume byte for byte.
 *
 * Every per-voxel label is a pure function of (i,j,k) and a shape list drawn
 * once on the host with SplitMix64, so any z-slab can be generated alone and
 * the GPU and CPU generators agree bit for bit (fp64 membership tests with no
 * FMA contraction, in the operation order written in psn_gen_voxel()).
 */
#ifndef PSN_GEN_H
#define PSN_GEN_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum {
    PSN_GEN_C1 = 1,       /* 32^3 u16, 3 spheres                                  */
    PSN_GEN_C2 = 2,       /* 256^3 u8, 20-seed Voronoi clipped to an ellipsoid      */
    PSN_GEN_C3 = 3,       /* 512x512x600 u16 torso: cylinder + 100 ellipsoids       */
    PSN_GEN_C4 = 4,       /* 1024^3 u16 atlas: 200-seed Voronoi in a ball + 300 inclusions */
    PSN_GEN_C5A = 5,      /* 512^3 u8 iid {0,1,2,3}                                 */
    PSN_GEN_C5B = 6,      /* 512^3 u8 single sphere r=16 at the centre              */
    PSN_GEN_SPHERES = 7,  /* generic: n random spheres in a box (custom dims, used by tests) */
    PSN_GEN_C6 = 8        /* 512^3 u16 "Synthetic"-like: 128 overlapping spheres (NEXT-1)  */
};

#define PSN_GEN_MAX_SEEDS 256
#define PSN_GEN_MAX_ELL 320

typedef struct {
    int32_t kind;
    int32_t elem_bytes;          /* 1, 2, 4 */
    int64_t dims[3];             /* M, N, O */
    double spacing[3];
    uint64_t seed;
    int32_t n_seeds;             /* Voronoi seeds */
    int32_t n_ell;               /* spheres / ellipsoids */
    double seeds[PSN_GEN_MAX_SEEDS][3];
    double ell[PSN_GEN_MAX_ELL][6];   /* cx, cy, cz, ax, ay, az (spheres: ax=ay=az=r) */
    uint32_t ell_label[PSN_GEN_MAX_ELL];
    int32_t tries_first;         /* rejection tries of the first drawn shape (test vector) */
} psn_gen_spec;

/* Draw the shape list of a config on the host.  For PSN_GEN_SPHERES, dims /
 * elem_bytes / n_ell / seed are taken from *spec on input.  Returns 0 or -1. */
int psn_gen_config(int kind, uint64_t seed, psn_gen_spec *spec);

/* CPU: write lattice slices [z_lo, z_hi) (x fastest) into out.  0 or -1. */
int psn_gen_host(const psn_gen_spec *spec, int64_t z_lo, int64_t z_hi, void *out);

/* GPU: same bytes into device memory `out` on `stream` (a cudaStream_t).
 * Returns 0 or a CUDA error code. */
int psn_gen_device(const psn_gen_spec *spec, int64_t z_lo, int64_t z_hi, void *out, void *stream);

/* SplitMix64 helpers exported for the test vectors. */
uint64_t psn_gen_splitmix_next(uint64_t *state);

#ifdef __cplusplus
}
#endif
#endif
