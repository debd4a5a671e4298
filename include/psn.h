/*
 * psn.h -- C ABI of the B200-native Parallel SurfaceNets hot path.
 *
 * Library: paper_2401_14906_b200/libpsn.so (sm_100a CUDA kernels + this ABI).
 * Every entry point follows the paper's statement of the problem
 * (/root/reference/PAPER.md, cited "P:<line>"):
 *   input  = a label volume with spacing/origin, a label set L
 *            whose complement is background B, an iteration count, a
 *            relaxation factor lambda and a constraint distance;
 *   output = points, quads, region-adjacency two-tuples, smoothing stencils
 *             and optionally triangles.
 *
 * Conventions (all calls):
 *   - Plain pointers and sizes only; no exceptions cross the ABI.  Every call
 *     returns a psn_status; psn_last_error(ctx) gives a text message.
 *   - Device pointers are caller-owned (the library never allocates device
 *     memory).  Work is enqueued on the caller's CUDA stream `stream`
 *     (a cudaStream_t passed as void*); calls are stream-ordered and never
 *     synchronise the device, except where stated (PSN_COUNT reads 3 totals).
 *   - Arguments are validated before any launch; on an error nothing is launched.
 *   - Outputs are bit-identical across runs, launch configurations and rank
 *     counts (after rank-order concatenation): no atomics on output values.
 *   - Label volumes are x-fastest: idx = i + M*(j + N*(k - z_lo)).
 *   - Ids are uint32 (reading Q20); totals >= 2^32 give PSN_ERR_OVERFLOW.
 *   - Background in two-tuples is PSN_BACKGROUND (reading Q3).
 */
#ifndef PSN_H
#define PSN_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define PSN_BACKGROUND 0xFFFFFFFFu

typedef enum {
    PSN_OK = 0,
    PSN_ERR_ARG = 1,        /* bad argument: null pointer, dims < 2, spacing <= 0, lambda not in [0,1], d < 0, T < 0, bad slab bounds */
    PSN_ERR_LABELS = 2,     /* empty label set without all_nonzero, or PSN_BACKGROUND in the set */
    PSN_ERR_OVERFLOW = 3,   /* P, Q or S would reach 2^32: totals are still reported */
    PSN_ERR_CAPACITY = 4,   /* output capacities too small: totals reported, nothing emitted */
    PSN_ERR_STATE = 5,      /* PSN_EMIT without a matching PSN_COUNT on this workspace */
    PSN_ERR_CUDA = 6        /* a CUDA runtime error (message in psn_last_error) */
} psn_status;

typedef enum { PSN_U8 = 1, PSN_U16 = 2, PSN_U32 = 4 } psn_dtype;

typedef enum {
    PSN_TRI_FIXED_02 = 0,       /* "greedy": always diagonal 0-2 (reading Q13) */
    PSN_TRI_SHORTEST = 1,       /* shorter diagonal, ties -> 0-2 */
    PSN_TRI_MIN_AREA = 2,       /* minimum summed triangle area (reading Q27) */
    PSN_TRI_MOST_COPLANAR = 3   /* most co-planar triangle pair (reading Q27) */
} psn_tri;

enum { PSN_COUNT = 1, PSN_EMIT = 2, PSN_DEVICE = 4 };

typedef struct psn_ctx psn_ctx;   /* opaque HOST object: device id, SM count, last error */

/*
 * Label volume (device memory, caller-owned).  One process may hold a z-slab
 * of the global volume (multi-GPU): lattice slices [z_lo, z_hi)
 * are present in `labels`, and this call owns voxel layers [own_k0, own_k1).
 * Required: z_lo <= max(own_k0-1, 0) and z_hi >= min(own_k1+1, O-1) + 1,
 * i.e. a one-slice halo on each interior side.  Single GPU: z_lo=0, z_hi=O,
 * own_k0=0, own_k1=O-1.
 */
typedef struct {
    const void *labels;
    psn_dtype dtype;
    int64_t dims[3];        /* GLOBAL lattice points M, N, O; each >= 2 */
    double spacing[3];      /* world units per lattice step, > 0 */
    double origin[3];       /* world position of lattice point (0,0,0) */
    int64_t z_lo, z_hi;
    int64_t own_k0, own_k1;
} psn_volume;

/*
 * Selected label set L (HOST memory).  all_nonzero != 0 selects every
 * non-zero value (reading Q2) and ignores `values`.  Otherwise values need
 * not be sorted or unique; values that cannot occur in the dtype are ignored.
 */
typedef struct {
    const uint32_t *values;
    int64_t count;
    int all_nonzero;
} psn_labels;

/*
 * Extracted mesh (device arrays, caller-owned).  Point-indexed arrays use a
 * WINDOW index  w = id - (first_point - halo_lo_points):
 *   points          float[halo_lo + P + halo_hi][3]  voxel centres
 *                   fl32(origin + (idx + 0.5) * spacing) computed in fp64 (C-3);
 *                   includes the points of the halo layers own_k0-1 / own_k1
 *                   (needed by smoothing and triangulation on a slab)
 *   face_masks      uint8[P]      own points: bit f set iff stencil holds face f
 *                                 (f = -z,-y,-x,+x,+y,+z)
 *   stencil_offsets uint32[P+1]   own points: CSR row starts (global, start at first_stencil)
 *   stencil_ids     uint32[S]     neighbour point ids, face order = ascending id
 *   quads           uint32[Q][4]  point ids, voxel-major then x<y<z (reading Q4/Q6)
 *   pairs           uint32[Q][2]  (cls at edge origin, cls at far end)
 * Capacities cap_* count elements of the leading dimension (points: window
 * entries).  n_* / halo_* are written by PSN_COUNT; first_* are inputs to
 * PSN_EMIT (global offsets from the cross-rank exclusive scan, 0 on one GPU).
 */
typedef struct {
    float *points;
    uint32_t *quads;
    uint32_t *pairs;
    uint32_t *stencil_offsets;
    uint32_t *stencil_ids;
    uint8_t *face_masks;
    int64_t cap_points, cap_quads, cap_stencil;
    int64_t n_points, n_quads, n_stencil;        /* out: this call's own totals */
    int64_t halo_lo_points, halo_hi_points;      /* out: points in layers own_k0-1 / own_k1 */
    int64_t first_point, first_quad, first_stencil;  /* in (EMIT) */
    /* optional: uint32[cap_points][2] packed smoothing cache of the own points (see
     * psn_smooth_prepare).  When non-NULL, PSN_EMIT writes it alongside the
     * stencils if the volume allows the packed form and the band-staged
     * emission runs, and sets smooth_cache_valid = 1 (else 0); psn_smooth then
     * skips building the cache (saves reading the CSR back). */
    uint32_t *smooth_cache;
    int64_t smooth_cache_valid;                  /* out (EMIT) */
    /* optional (PSN_DEVICE emission): DEVICE int64[3] = first_point, first_quad, first_stencil,
     * read by the emission kernel instead of first_* -- the cross-rank exclusive scan (C1) can then
     * stay on the device (e.g. an NCCL all-gather of psn_extract_totals' output + a prefix sum). */
    const int64_t *first_dev;
} psn_mesh;

psn_status psn_ctx_create(int device, psn_ctx **out);
void psn_ctx_destroy(psn_ctx *ctx);
const char *psn_last_error(const psn_ctx *ctx);
const char *psn_status_string(psn_status s);

/* Bytes of device workspace psn_extract needs for this volume (row counts,
 * offsets, trims, point bit-planes, scan tile status, label bitset). */
psn_status psn_extract_workspace(const psn_volume *vol, size_t *bytes);

/*
 * Surface extraction (PAPER sec 2.3, Passes 1-4).
 *   phase & PSN_COUNT: Passes 1-3 -- per voxel row point/quad/stencil counts
 *       and point bit-planes (k_count3, or the x-tiled k_count for wide rows;
 *       psn_ctx_set_counting), then the row-wise exclusive scan (k_scan).  Reads 3 totals back (one stream synchronisation) into
 *       mesh->n_points/n_quads/n_stencil/halo_*.  PSN_ERR_OVERFLOW if any total
 *       reaches 2^32.
 *   phase == PSN_EMIT: Pass 4 (k_emit_band / k_emit_fast / k_emit,
 *       psn_ctx_set_emission) into the caller's arrays, using the
 *       scan kept in `ws` by the preceding PSN_COUNT.  Capacities are checked on
 *       the host against the counted totals (PSN_ERR_CAPACITY, nothing launched).
 *   phase == PSN_COUNT|PSN_EMIT: fully stream-ordered, no host sync: the emit
 *       kernel reads the device totals and writes nothing if they exceed the
 *       capacities; the totals are NOT written back to *mesh (call
 *       psn_mesh_totals later to read them and the device status word).
 *   PSN_DEVICE (with PSN_COUNT and / or PSN_EMIT): no host round trip -- COUNT leaves the
 *       totals on the device (psn_extract_totals copies them to a device buffer; *mesh is not
 *       updated), EMIT skips the host capacity check (the kernel checks the device totals against
 *       the capacities, as in the fused call) and takes mesh->first_dev if set.  The multi-GPU
 *       steady state: COUNT|DEVICE -> totals -> all-gather + prefix sum on the device -> EMIT|DEVICE.
 * ws must stay untouched between COUNT and EMIT.
 */
psn_status psn_extract(psn_ctx *ctx, const psn_volume *vol, const psn_labels *labels,
                       psn_mesh *mesh, unsigned phase, void *ws, size_t ws_bytes, void *stream);

/* Stream-ordered copy of this call's totals from ws into DEVICE int64 out[5] = own points,
 * quads, stencil entries, halo-lo points, halo-hi points (what PSN_COUNT writes into *mesh on the
 * host).  For the PSN_DEVICE path; no synchronisation. */
psn_status psn_extract_totals(psn_ctx *ctx, const psn_volume *vol, const void *ws, size_t ws_bytes, int64_t *out,
                              void *stream);

/* Synchronising read of the totals and capacity status left in ws by the
 * last psn_extract (for the PSN_COUNT|PSN_EMIT path).  Returns
 * PSN_ERR_CAPACITY if that emission was skipped. */
psn_status psn_mesh_totals(psn_ctx *ctx, const psn_volume *vol, psn_mesh *mesh,
                           const void *ws, size_t ws_bytes, void *stream);

/* Workspace of the smoothing calls: the smoothing cache (the
 * extracted mesh is kept so re-smoothing skips re-extraction) -- a fixed-stride
 * uint32[P][4] table of each own point's -z,-y,+y,+z neighbour window indices
 * -- followed by two [n_window] index-space offset buffers (double buffering,
 * P:94) and the wavefront schedule (tile ranges, per-tile progress). */
psn_status psn_smooth_workspace(const psn_mesh *mesh, size_t *bytes);

/* Build the smoothing cache of `mesh` into ws (psn_smooth does this itself;
 * slab users call it once before their psn_smooth_step loop).  `vol` (dims)
 * selects the cache form: the packed 8-byte one (id distances to the y/z
 * neighbours) when M-1 < 2^10 and (M-1)(N-1) < 2^21, else 16 bytes per
 * point.  psn_smooth_step must be given the
 * same volume.  PSN_ERR_ARG: NULL volume / mesh arrays, workspace too small. */
psn_status psn_smooth_prepare(psn_ctx *ctx, const psn_volume *vol, const psn_mesh *mesh, void *ws, size_t ws_bytes,
                              void *stream);

/*
 * Constrained Laplacian smoothing (Eq. 1) with double buffering
 * (P:94): builds the smoothing cache, runs `iterations` Jacobi steps on the
 * caller's stream, and writes world coordinates of every own point to out[w][3]:
 *   per own point with N = deg > 0:  o' = clamp(o + lambda * mean_j(p_j - p_i)/s, -d, +d)
 * computed on fp32 index-space offsets o from the exact voxel-centre anchor;
 * out = fl32(anchor64 + s * o).  iterations = 0 or lambda = 0 gives the anchors.
 * Single GPU / whole volume only (halo layers empty); a slab uses
 * psn_smooth_prepare + psn_smooth_step with a halo exchange between steps.
 * constraint_distance d is in voxel units (box half-width d*s per axis,
 * readings Q9/Q10).
 */
psn_status psn_smooth(psn_ctx *ctx, const psn_volume *vol, const psn_mesh *mesh, float *out,
                      int32_t iterations, float relaxation, float constraint_distance,
                      void *ws, size_t ws_bytes, void *stream);

/*
 * One Jacobi iteration over the own points of a slab: reads the window offset
 * buffer src[n_window][4] (float4 entries x, y, z, unused; 16-byte aligned;
 * halo entries must hold the neighbours' current values), writes the own
 * entries of dst (same layout; w written as 0).  ws must hold the smoothing
 * cache built by psn_smooth_prepare for the same `vol`.  src == NULL means
 * "all offsets zero" (first iteration from the anchors).  Same kernel and
 * bits as psn_smooth's per-iteration path (box or sphere constraint, as set
 * on the context).  PSN_ERR_ARG for NULL dst / vol, misaligned buffers or a
 * workspace too small.
 */
psn_status psn_smooth_step(psn_ctx *ctx, const psn_volume *vol, const psn_mesh *mesh, const void *ws, size_t ws_bytes,
                           const float *src, float *dst, float relaxation, float constraint_distance, void *stream);

/*
 * Per voxel row plan of the last PSN_COUNT on `ws` (Passes 1-3): for
 * every counted voxel row r = j + (N-1)(k - kA) (kA = own_k0 - 1 if own_k0 > 0,
 * else own_k0; layers [kA, kB) include the halo layers), copies into caller
 * device buffers (stream-ordered, no sync):
 *   counts  uint32[3][R]  points, owned quads, directed stencil entries of the
 *                         row (halo layers: points only) -- what Pass 4 emits
 *                         per row ("planned == emitted");
 *   trims   int32[R][2]   the row's computational trim [xL, xR) in voxel units
 *                         (P:81): the first and one past the last
 *                         point-producing voxel; [0, 0) for rows without points.
 * Either pointer may be NULL.  *rows (if non-NULL) receives R.  PSN_ERR_STATE
 * if ws holds no COUNT of this volume; PSN_ERR_ARG for bad arguments.
 */
psn_status psn_extract_rows(psn_ctx *ctx, const psn_volume *vol, const void *ws, size_t ws_bytes,
                            uint32_t *counts, int32_t *trims, int64_t *rows, void *stream);

/* Smoothing strategy of psn_smooth (whole volume):
 *   PSN_SMOOTH_PER_ITERATION (default): one launch per Jacobi iteration.
 *   PSN_SMOOTH_WAVEFRONT: G iterations per persistent launch, scheduled as a
 *     wavefront over tiles of consecutive points so each tile's state stays
 *     L2-resident across iterations (iterations_per_launch G, 0 = chosen
 *     from the L2 size; points_per_tile a multiple of 256, 0 = 1024).
 *     Bit-identical to the default; measured slower on B200. */
enum { PSN_SMOOTH_WAVEFRONT = 0, PSN_SMOOTH_PER_ITERATION = 1 };
psn_status psn_ctx_set_smoothing(psn_ctx *ctx, int mode, int32_t iterations_per_launch, int32_t points_per_tile);

/* Counting kernel of psn_extract(PSN_COUNT) (Passes 1-3):
 *   PSN_COUNT_AUTO (default): the warp-per-row producer/consumer kernel
 *     (k_count3) when a voxel row fits one warp (M-1 <= 256*16/b, b = label
 *     bytes; u32: M-1 <= 512), else the x-tiled kernel (k_count).
 *   PSN_COUNT_XTILE: always the x-tiled kernel.
 * Both produce identical counts and point planes (tested). */
enum { PSN_COUNT_AUTO = 0, PSN_COUNT_XTILE = 1 };
psn_status psn_ctx_set_counting(psn_ctx *ctx, int mode);

/* Constraint on the total motion of a point relative to its voxel centre
 * used by psn_smooth, psn_smooth_step and psn_smooth_step_peer:
 *   PSN_CONSTRAINT_BOX (default): |p - anchor|_a <= d * s_a per axis (reading Q10);
 *   PSN_CONSTRAINT_SPHERE: |p - anchor| <= d * min(s), radial projection after
 *     the lambda step ("a constraint sphere centered at the voxel center
 *     point", reading Q26). */
enum { PSN_CONSTRAINT_BOX = 0, PSN_CONSTRAINT_SPHERE = 1 };
psn_status psn_ctx_set_constraint(psn_ctx *ctx, int shape);

/* Emission kernel of psn_extract(PSN_EMIT) (Pass 4):
 *   PSN_EMIT_AUTO (default): band-staged k_emit_band (TMA-staged point planes,
 *     4 rows per warp) when a row has <= 32 point-plane words (M <= 1025);
 *   PSN_EMIT_SCAN: the general k_emit (per-row packed prefix scans, any width).
 * Wider rows always use the row-prefix / scan kernels.  All produce identical
 * outputs (tested).  (Mode 1, the former row-pipelined kernel, was removed:
 * PSN_ERR_ARG.) */
enum { PSN_EMIT_AUTO = 0, PSN_EMIT_SCAN = 2 };
psn_status psn_ctx_set_emission(psn_ctx *ctx, int mode);

/* Synchronising check of the last psn_smooth on ws: PSN_ERR_CUDA if a
 * wavefront dependency wait timed out (a guard that must never trigger). */
psn_status psn_smooth_status(psn_ctx *ctx, const psn_mesh *mesh, const void *ws, size_t ws_bytes, void *stream);

/* World coordinates out[w][3] of window entries [w0, w1) from float4 offsets
 * offsets[n_window][4] as psn_smooth_step writes them (NULL = anchors). */
psn_status psn_smooth_finalize(psn_ctx *ctx, const psn_volume *vol, const psn_mesh *mesh,
                               const float *offsets, int64_t w0, int64_t w1, float *out, void *stream);

/*
 * Triangulation: quad q -> triangles 2q, 2q+1; tris uint32[2Q][3];
 * the two-tuple of triangle t is pairs[t/2].  `points` is window-indexed
 * (as psn_mesh.points), typically the smoothed output of psn_smooth.
 */
psn_status psn_triangulate(psn_ctx *ctx, const psn_mesh *mesh, const float *points, psn_tri tri,
                           uint32_t *tris, void *stream);

/* Per-pass timing (bench.py's per_pass object): with events != NULL (4 cudaEvent_t
 * created on the context's device, passed as void*), every later psn_extract
 * records events[0] before the counting pass (incl. its header reset), [1]
 * between counting and the scan, [2] between the scan and the emission, [3]
 * after the emission (a COUNT-only call records [0..2], an EMIT-only call [3]);
 * stream-ordered, no synchronisation.  events == NULL stops the recording. */
psn_status psn_ctx_set_pass_events(psn_ctx *ctx, void *const *events);

/* Smoothing timing (bench.py's roofline): with events != NULL (2 cudaEvent_t of the context's device),
 * every later per-iteration psn_smooth records events[0] after its cache preparation (before the
 * first Jacobi launch) and events[1] after the last one: (events[1] - events[0]) / iterations is the
 * mean k_smooth_v4 launch time.  NULL stops the recording. */
psn_status psn_ctx_set_smooth_events(psn_ctx *ctx, void *const *events);

/* Number of kernel launches the last call on this ctx enqueued (bench.py's gpu_launches). */
int64_t psn_launch_count(const psn_ctx *ctx);

/* ------------------------------------------------------------------------
 * Peer (NVLink) halo exchange for the slab / shard smoothing loop (SURVEY
 * 8(e) v2; sub-volumes with open boundaries exchange the
 * boundary layer every Jacobi step).  Instead of a collective after each
 * psn_smooth_step, psn_smooth_step_peer's kernel stores the boundary layers
 * it computes straight into the neighbours' offset buffers (peer pointers,
 * CUDA IPC over NVLink) and signals them; a step starts once both neighbours
 * have finished the previous one.  One launch per iteration, no host sync.
 * ------------------------------------------------------------------------ */

/* CUDA IPC handle of the device allocation holding `dev_ptr` (+ the offset of
 * dev_ptr inside it), to be sent to the peer processes (host bytes).
 * PSN_ERR_CUDA if the memory cannot be exported (e.g. not from cudaMalloc). */
typedef struct { unsigned char handle[64]; uint64_t offset; } psn_ipc_handle;
psn_status psn_ipc_export(psn_ctx *ctx, const void *dev_ptr, psn_ipc_handle *out);
/* Map a peer process's exported allocation into this process (peer access
 * enabled for the context's device); *dev_ptr = mapped base + offset.
 * Release with psn_ipc_close(mapped pointer). */
psn_status psn_ipc_open(psn_ctx *ctx, const psn_ipc_handle *h, void **dev_ptr);
psn_status psn_ipc_close(psn_ctx *ctx, void *dev_ptr);

typedef struct {
    float *dst[2];              /* the neighbour's float4 [W'][4] offset buffers by parity (peer
                                   pointers); dst[0] == NULL: no neighbour on this side */
    int64_t src_begin, src_end; /* own window entries pushed (inside the own range) */
    int64_t dst_begin;          /* the neighbour's window index receiving src_begin */
    uint64_t *peer_sig;         /* the neighbour's signal word for this rank's pushes */
} psn_peer_side;

typedef struct {
    psn_peer_side side[2];      /* [0] = lower neighbour (rank - 1), [1] = upper (rank + 1) */
    uint64_t *sig;              /* this rank's signal words [2] (device; [0] written by the lower,
                                   [1] by the upper neighbour; zeroed once before the first step) */
    uint64_t *ctr;              /* this rank's CTA completion counter (device, zeroed once) */
    uint32_t *err;              /* timeout flag (device, zeroed once): a wait > 5 s sets it */
    uint64_t ctr_base;          /* in/out: CTAs counted on ctr so far (advanced by each call) */
    uint64_t iteration;         /* in/out: global iteration index (advanced by each call) */
} psn_peer;

/* psn_smooth_step plus the peer push: writes dst (own entries) and, for own
 * window entries [side.src_begin, side.src_end), the neighbour's buffer
 * side.dst[parity] at side.dst_begin + (w - src_begin).  Every rank calls it
 * once per iteration with the same `parity` (the caller's dst buffer index).
 * Ranks without points still call it (the step only waits and signals).
 * PSN_ERR_ARG for the conditions of psn_smooth_step, a NULL peer / sig / ctr /
 * err, or a non-empty push range outside the own entries.  A neighbour wait
 * longer than 5 s sets *err and traps the kernel (the stream then reports a
 * launch failure) instead of smoothing on with stale halos. */
psn_status psn_smooth_step_peer(psn_ctx *ctx, const psn_volume *vol, const psn_mesh *mesh, const void *ws,
                                size_t ws_bytes, const float *src, float *dst, int parity, float relaxation,
                                float constraint_distance, psn_peer *peer, void *stream);

/* `iterations` peer steps from the anchors in one call (no per-step host
 * round trip): with g = peer->iteration on entry, step t uses parity
 * p = (g+t)&1, reads buf[p^1] (nothing at t = 0) and writes buf[p] -- the loop
 * every rank would otherwise run around psn_smooth_step_peer.  The result is in
 * buf[(peer->iteration - 1) & 1] (peer->iteration as updated by the call).
 * Continuing the parity across calls keeps a later run's first push out of
 * the buffer a neighbour's previous run ended in.  With the packed cache and
 * iterations > 1 the run uses the split cache (as psn_smooth): step 0 writes
 * the hi words of the packed entries into the unused second half of the
 * cache region of `ws` (scratch of this call; the prepared cache itself is
 * not modified) and the lo words into the w slots of the offsets, steps
 * 1.. read them -- bit-identical to the 8-byte-cache steps. */
psn_status psn_smooth_run_peer(psn_ctx *ctx, const psn_volume *vol, const psn_mesh *mesh, const void *ws,
                               size_t ws_bytes, float *buf0, float *buf1, int32_t iterations, float relaxation,
                               float constraint_distance, psn_peer *peer, void *stream);

/* ------------------------------------------------------------------------
 * Sub-volume blocks stitched into the whole-volume mesh.
 * boundaries are left open "so that ... distributed execution
 * avoids introducing artificial partitions along adjacent sub-volume
 * boundaries"; sub-volumes of a larger input, "with special attention
 * placed on stitching output meshes together at subvolume boundaries".
 *
 * The voxels are cut into a grid of blocks along x, y and z (any cuts).  A
 * block owning voxels [own_lo, own_hi) is extracted as a STANDALONE volume
 * (psn_extract with origin 0, spacing 1, z_lo 0, all layers own) over its
 * lattice box [box_lo, box_hi) = own box plus a one-voxel margin on every
 * interior side (psn_block_box; a larger box is also valid).  Only that box needs to be in device memory
 * (psn_block_gather copies it from a host or device volume).  Stitching:
 *   1. every block:  psn_stitch_count  (its segments' point/quad/stencil counts)
 *   2. once:         psn_stitch_scan   (exclusive offsets of all segments)
 *   3. every block:  psn_stitch_emit   (owned points/quads/stencils, global ids)
 * A SEGMENT is the owned voxels of one block in one voxel row:
 *   s = (j + (N-1) k) * nxseg + xseg   (global voxel row, x-block index),
 * nseg = (N-1)(O-1) nxseg.  The stitched mesh (ids, order, every array) is
 * bit-identical to psn_extract over the whole volume with the same origin,
 * spacing and label set.
 * ------------------------------------------------------------------------ */
typedef struct {
    int64_t dims[3];              /* GLOBAL lattice points M, N, O */
    int64_t own_lo[3], own_hi[3]; /* owned voxel box [own_lo, own_hi), non-empty, inside [0, dims-1) */
    int64_t box_lo[3], box_hi[3]; /* lattice box of the block's standalone volume: contains the own box plus
                                     the one-voxel margin on interior sides (psn_block_box) */
    int64_t xseg, nxseg;          /* x-block index of the block, number of x-blocks */
} psn_block;

/* Host-only: box_lo = max(own_lo - 1, 0), box_hi = min(own_hi + 2, dims) per axis (the margin voxel on
 * each interior side needs one more lattice point).  With elem_bytes (1, 2 or 4; 0 = tight box) the x
 * range is then widened inside [0, M) to a multiple of 16 bytes when the volume is wide enough, so the
 * box rows are TMA-staged by k_count3 (voxels beyond the margin are extracted but never stitched: any
 * box containing the tight one is valid).  PSN_ERR_ARG for an empty or out-of-range own box, or an
 * x-block index that contradicts it (xseg > 0 iff own_lo[0] > 0, xseg < nxseg-1 iff own_hi[0] < M-1). */
psn_status psn_block_box(psn_block *blk, int elem_bytes);

/* Stream-ordered copy of lattice box [box_lo, box_hi) of an x-fastest global volume `src` (host --
 * pinned for an asynchronous copy -- or device memory, dims[3], element size by dtype) into the compact
 * device buffer dst[box z][box y][box x].  PSN_ERR_ARG for NULL pointers or a box outside dims. */
psn_status psn_block_gather(psn_ctx *ctx, const void *src, psn_dtype dtype, const psn_block *blk, void *dst,
                            void *stream);

/* Device scratch of psn_stitch_count / psn_stitch_emit for one block: uint32[4][(bN-1)(bO-1)] tables
 * (first / last owned-x point and quad of every local voxel row). */
psn_status psn_stitch_workspace(const psn_block *blk, size_t *bytes);

/* Step 1 for one block.  `local` = the block's standalone mesh (psn_extract of the box volume:
 * points, quads, pairs, stencil_offsets, stencil_ids, face_masks, n_points, n_quads).  Fills ws's
 * tables and, if seg != NULL, writes seg[0][s], seg[1][s], seg[2][s] = points, quads, stencil
 * entries of every segment this block owns (device uint32[3][nseg]; every segment is written by
 * exactly one block, so the array needs no clearing).  Re-run with seg == NULL to rebuild ws
 * before psn_stitch_emit if ws was not kept. */
psn_status psn_stitch_count(psn_ctx *ctx, const psn_block *blk, const psn_mesh *local, void *ws, size_t ws_bytes,
                            uint32_t *seg, void *stream);

/* Step 2: off[a][s] = exclusive prefix sum of seg[a][s] over s (a = points, quads, stencil entries;
 * device uint32[3][nseg] each), totals (device int64[3]) = the sums.  scratch: device bytes
 * >= psn_stitch_scan_workspace(nseg).  If host_totals != NULL the call synchronises the stream,
 * copies the totals there and returns PSN_ERR_OVERFLOW if one reaches 2^32. */
size_t psn_stitch_scan_workspace(int64_t nseg);
psn_status psn_stitch_scan(psn_ctx *ctx, int64_t nseg, const uint32_t *seg, uint32_t *off, int64_t *totals,
                           void *scratch, size_t scratch_bytes, int64_t *host_totals, void *stream);

/* Step 3 for one block: writes the block's owned points (recomputed from the global voxel index with
 * vol->origin / vol->spacing), face masks, stencil offsets and ids, quads and pairs into `global`
 * (capacities >= the totals; first_* and halo fields ignored: whole-volume ids) and the CSR sentinel
 * stencil_offsets[P] = S.  ws = this block's tables from psn_stitch_count; off / totals from
 * psn_stitch_scan.  vol: the global volume (dims must equal blk->dims; labels unused). */
psn_status psn_stitch_emit(psn_ctx *ctx, const psn_block *blk, const psn_volume *vol, const psn_mesh *local,
                           const void *ws, size_t ws_bytes, const uint32_t *off, const int64_t *totals,
                           psn_mesh *global, void *stream);

#ifdef __cplusplus
}
#endif
#endif /* PSN_H */
