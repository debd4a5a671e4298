// psn_api.cu -- host side of the C ABI declared in include/psn.h.
//
// Validation, workspace layout, label-set preparation and stream-ordered
// launches of the sm_100a kernels:
//   psn_extract(COUNT) -> k_count (Passes 1-3 counting) -> k_scan (Pass 3 prefix sum)
//   psn_extract(EMIT)  -> k_emit  (Pass 4)
//   psn_smooth         -> k_smooth x T (Eq. 1, double-buffered; last step fused with finalize)
//   psn_triangulate    -> k_triangulate
// The library never allocates device memory; every buffer is the caller's.
#include <cuda_runtime.h>

#include <algorithm>
#include <array>
#include <map>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <cstdlib>
#include <string>
#include <vector>

#include "psn.h"
#include "k_count.cuh"
#include "k_count3.cuh"
#include "k_emit.cuh"
#include "k_scan.cuh"
#include "k_smooth.cuh"
#include "k_smooth_tb.cuh"
#include "k_stitch.cuh"

using namespace psn;

struct psn_ctx {
    int device = 0;
    int sms = 148;
    std::string err;
    int64_t launches = 0;
    std::vector<uint32_t> label_host;     // bitset or sorted list kept alive for async copies
    // workspaces holding a valid COUNT result, with the volume signature they were counted for
    std::map<const void *, std::array<int64_t, 6>> counted;
    std::map<const void *, bool> yz_split;   // the COUNT on this workspace was k_count3 (S completed by the scan)
    int smooth_mode = PSN_SMOOTH_PER_ITERATION;   // psn_ctx_set_smoothing (measured faster)
    int32_t smooth_group = 0;                 // iterations per wavefront launch (0 = automatic)
    int32_t smooth_tile = 0;                  // points per wavefront tile (0 = automatic)
    int count_mode = PSN_COUNT_AUTO;          // psn_ctx_set_counting
    int emit_mode = PSN_EMIT_AUTO;            // psn_ctx_set_emission
    int emit_dense = -1;                      // stencil density of the last totals read back (k_emit_band STG); -1 unknown
    int constraint = PSN_CONSTRAINT_BOX;      // psn_ctx_set_constraint
    std::map<void *, void *> ipc_bases;       // psn_ipc_open: returned pointer -> mapped base
    cudaEvent_t pass_ev[4] = {nullptr, nullptr, nullptr, nullptr};   // psn_ctx_set_pass_events
    cudaEvent_t smooth_ev[2] = {nullptr, nullptr};                      // psn_ctx_set_smooth_events
};

namespace {

float __fmul_rn_host(float r) { volatile float x = r; return x * x; }   // one IEEE fp32 rounding

psn_status fail(psn_ctx *ctx, psn_status s, const char *fmt, ...) {
    if (ctx) {
        char buf[512];
        va_list ap;
        va_start(ap, fmt);
        vsnprintf(buf, sizeof(buf), fmt, ap);
        va_end(ap);
        ctx->err = buf;
    }
    return s;
}

psn_status cuda_check(psn_ctx *ctx, const char *where) {
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return fail(ctx, PSN_ERR_CUDA, "%s: %s", where, cudaGetErrorString(e));
    return PSN_OK;
}

constexpr size_t kAlign = 256;
size_t align_up(size_t x) { return (x + kAlign - 1) / kAlign * kAlign; }
size_t align16(size_t x) { return (x + 15) / 16 * 16; }

struct Layout {
    int64_t M, N, O, kA, kB, R, W32, nTiles;
    size_t hdr, tiles, cntP, cntQ, cntS, cntYZ, offP, offQ, offS, trim, pmask, ppre, labels, total;
};

constexpr int64_t kMaxList = 65536;   // u32 label-subset capacity in the workspace

psn_status layout(psn_ctx *ctx, const psn_volume *v, Layout *L) {
    if (!v) return fail(ctx, PSN_ERR_ARG, "volume is NULL");
    const int64_t M = v->dims[0], N = v->dims[1], O = v->dims[2];
    if (M < 2 || N < 2 || O < 2) return fail(ctx, PSN_ERR_ARG, "dims must be >= 2 (got %lld %lld %lld)",
                                             (long long)M, (long long)N, (long long)O);
    if (M > (1ll << 31) || N > (1ll << 31) || O > (1ll << 31)) return fail(ctx, PSN_ERR_ARG, "dims too large");
    if (v->dtype != PSN_U8 && v->dtype != PSN_U16 && v->dtype != PSN_U32)
        return fail(ctx, PSN_ERR_ARG, "dtype must be PSN_U8, PSN_U16 or PSN_U32");
    for (int a = 0; a < 3; ++a)
        if (!(v->spacing[a] > 0.0)) return fail(ctx, PSN_ERR_ARG, "spacing must be > 0");
    if (v->own_k0 < 0 || v->own_k1 > O - 1 || v->own_k0 >= v->own_k1)
        return fail(ctx, PSN_ERR_ARG, "need 0 <= own_k0 < own_k1 <= O-1");
    L->M = M; L->N = N; L->O = O;
    L->kA = v->own_k0 - (v->own_k0 > 0 ? 1 : 0);
    L->kB = v->own_k1 + (v->own_k1 < O - 1 ? 1 : 0);
    if (v->z_lo > L->kA || v->z_hi < L->kB + 1 || v->z_lo < 0 || v->z_hi > O)
        return fail(ctx, PSN_ERR_ARG, "slab slices [%lld,%lld) must contain [%lld,%lld] (one-slice halos)",
                    (long long)v->z_lo, (long long)v->z_hi, (long long)L->kA, (long long)L->kB);
    L->R = (N - 1) * (L->kB - L->kA);
    L->W32 = (M - 1 + 31) / 32;
    L->nTiles = (L->R + kScanTile - 1) / kScanTile;
    size_t off = 0;
    L->hdr = off; off += align_up(sizeof(ScanHeader));
    L->tiles = off; off += align_up(sizeof(TileStatus) * (size_t)L->nTiles);
    L->cntP = off; off += align_up(4 * (size_t)L->R);
    L->cntQ = off; off += align_up(4 * (size_t)L->R);
    L->cntS = off; off += align_up(4 * (size_t)L->R);
    L->cntYZ = off; off += align_up(4 * (size_t)L->R);
    L->offP = off; off += align_up(4 * (size_t)L->R);
    L->offQ = off; off += align_up(4 * (size_t)L->R);
    L->offS = off; off += align_up(4 * (size_t)L->R);
    L->trim = off; off += align_up(8 * (size_t)L->R);
    L->pmask = off; off += align_up(4 * (size_t)L->R * (size_t)L->W32);
    L->ppre = off; off += align_up(2 * (size_t)L->R * (size_t)L->W32);
    L->labels = off;
    off += align_up(v->dtype == PSN_U32 ? 4 * (size_t)kMaxList : 8192);
    L->total = off;
    return PSN_OK;
}

template <typename P> P *at(void *ws, size_t off) { return reinterpret_cast<P *>(static_cast<char *>(ws) + off); }

// Label set -> device LabelSet (bitset for u8/u16, sorted list for u32).
psn_status prepare_labels(psn_ctx *ctx, const psn_volume *v, const psn_labels *lab, void *ws, const Layout &L,
                          cudaStream_t st, LabelSet *out, bool *anz) {
    memset(out, 0, sizeof(*out));
    if (!lab) return fail(ctx, PSN_ERR_ARG, "labels is NULL");
    if (lab->all_nonzero) { *anz = true; return PSN_OK; }
    *anz = false;
    if (lab->count <= 0 || !lab->values) return fail(ctx, PSN_ERR_LABELS, "empty label set without all_nonzero");
    for (int64_t n = 0; n < lab->count; ++n)
        if (lab->values[n] == PSN_BACKGROUND) return fail(ctx, PSN_ERR_LABELS, "label set contains the background sentinel");
    uint32_t *dev = at<uint32_t>(ws, L.labels);
    if (v->dtype == PSN_U32) {
        std::vector<uint32_t> s(lab->values, lab->values + lab->count);
        std::sort(s.begin(), s.end());
        s.erase(std::unique(s.begin(), s.end()), s.end());
        if ((int64_t)s.size() > kMaxList) return fail(ctx, PSN_ERR_ARG, "u32 label subsets are limited to %lld values",
                                                      (long long)kMaxList);
        ctx->label_host = s;
        if (!s.empty() && cudaMemcpyAsync(dev, ctx->label_host.data(), 4 * s.size(), cudaMemcpyHostToDevice, st) != cudaSuccess)
            return cuda_check(ctx, "label upload");
        out->list = dev; out->n_list = (int64_t)s.size(); out->z = PSN_BACKGROUND; out->identity = 0;
        return PSN_OK;
    }
    const uint32_t nvals = v->dtype == PSN_U8 ? 256u : 65536u;
    ctx->label_host.assign(2048, 0u);
    for (int64_t n = 0; n < lab->count; ++n) {
        const uint32_t x = lab->values[n];
        if (x < nvals) ctx->label_host[x >> 5] |= 1u << (x & 31);   // values outside the dtype are ignored
    }
    uint32_t z = nvals;
    for (uint32_t x = 0; x < nvals; ++x)
        if (!((ctx->label_host[x >> 5] >> (x & 31)) & 1u)) { z = x; break; }
    if (cudaMemcpyAsync(dev, ctx->label_host.data(), 8192, cudaMemcpyHostToDevice, st) != cudaSuccess)
        return cuda_check(ctx, "label upload");
    out->bits = dev; out->z = z; out->identity = (z == nvals) ? 1 : 0;
    return PSN_OK;
}

__global__ void k_init_multixt(uint32_t *cp, uint32_t *cq, uint32_t *cs, int2 *trim, int64_t R) {
    for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < R; r += (int64_t)gridDim.x * blockDim.x) {
        cp[r] = 0; cq[r] = 0; cs[r] = 0; trim[r] = make_int2(0x7fffffff, 0);
    }
}

template <typename T, bool ANZ>
cudaError_t launch_count(const CountArgs &ca, int64_t blocks, int threads, size_t smem, cudaStream_t st) {
    constexpr int TJ = count_tj<T>();
    static size_t attr_set = 0;   // opt-in to > 48 KB dynamic shared memory (largest request so far)
    if (smem > attr_set) {
        cudaError_t e = cudaFuncSetAttribute(k_count<T, TJ, ANZ>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return e;
        attr_set = smem;
    }
    k_count<T, TJ, ANZ><<<(unsigned)blocks, threads, smem, st>>>(ca);
    return cudaGetLastError();
}

using V4Fn = void (*)(SmoothV4);
template <bool PK, bool PF, bool PE> V4Fn v4_sel(bool sphere) {
    return sphere ? k_smooth_v4<PK, PF, PE, true> : k_smooth_v4<PK, PF, PE, false>;
}

V4Fn split_sel(bool pref, bool sphere) {
    if (pref) return sphere ? k_smooth_split<true, true> : k_smooth_split<true, false>;
    return sphere ? k_smooth_split<false, true> : k_smooth_split<false, false>;
}

template <typename T, bool ANZ, int CPL, int RPW, bool FULL, bool EXACT>
cudaError_t launch_count3_f(const CountArgs &ca, int64_t blocks, size_t smem, cudaStream_t st) {
    static size_t attr_set = 0;
    if (smem > attr_set) {
        cudaError_t e = cudaFuncSetAttribute(k_count3<T, ANZ, CPL, RPW, FULL, EXACT>,
                                             cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return e;
        attr_set = smem;
    }
    k_count3<T, ANZ, CPL, RPW, FULL, EXACT><<<(unsigned)blocks, 32 * (kC3Rows / RPW + 1), smem, st>>>(ca);
    return cudaGetLastError();
}

template <typename T, bool ANZ, int CPL, int RPW>
cudaError_t launch_count3(const CountArgs &ca, int64_t blocks, size_t smem, cudaStream_t st) {
    constexpr int E = 16 / (int)sizeof(T);
    const int64_t chunks = (ca.M - 1 + E - 1) / E;
    // Exact-width rows (M == 32*CPL*E) get the fully constant row layout where it measured faster:
    // CPL <= 2 (c3 -4.6%, c5a -13%, c6 -5% count time); at CPL 4 (c4) it was +1.7%.
    if constexpr (CPL <= 2) {
        if (ca.M == 32 * CPL * E && ca.RB == 32 * CPL * 16 + 32)
            return launch_count3_f<T, ANZ, CPL, RPW, true, true>(ca, blocks, smem, st);
    }
    return chunks == 32 * CPL ? launch_count3_f<T, ANZ, CPL, RPW, true, false>(ca, blocks, smem, st)
                              : launch_count3_f<T, ANZ, CPL, RPW, false, false>(ca, blocks, smem, st);
}

template <typename T, bool ANZ, int RPW>
cudaError_t dispatch_count3_cpl(const CountArgs &ca, int cpl, int64_t blocks, size_t smem, cudaStream_t st) {
    switch (cpl) {
        case 1: return launch_count3<T, ANZ, 1, RPW>(ca, blocks, smem, st);
        case 2: return launch_count3<T, ANZ, 2, RPW>(ca, blocks, smem, st);
        case 4: return launch_count3<T, ANZ, 4, RPW>(ca, blocks, smem, st);
        default:
            if constexpr (sizeof(T) < 4) return launch_count3<T, ANZ, 8, RPW>(ca, blocks, smem, st);
            return cudaErrorInvalidValue;
    }
}

template <typename T>
cudaError_t dispatch_count3(const CountArgs &ca, bool anz, int cpl, int64_t blocks, size_t smem, cudaStream_t st) {
    constexpr int RPW = 2;   // voxel rows per consumer warp (measured: c3/c5b faster than 1, c4 equal; 4 slower)
    return anz ? dispatch_count3_cpl<T, true, RPW>(ca, cpl, blocks, smem, st)
               : dispatch_count3_cpl<T, false, RPW>(ca, cpl, blocks, smem, st);
}

template <typename T>
cudaError_t dispatch_count(const CountArgs &ca, bool anz, int64_t blocks, int threads, size_t smem, cudaStream_t st) {
    return anz ? launch_count<T, true>(ca, blocks, threads, smem, st) : launch_count<T, false>(ca, blocks, threads, smem, st);
}

template <typename T>
void dispatch_emit(const EmitArgs &ea, bool anz, bool fast, int64_t blocks, cudaStream_t st, int emit_mode, int dense) {
    if (fast && ea.W32 <= 32 && emit_mode == 0) {   // band-staged: shared-memory id lookups
        // the row-width classes of the common volumes (M <= 1025: 32 plane words; M <= 513: 16) get the word
        // count as a compile-time constant (c4 emission -6 %, c3 -7 %, c6 -7 %)
        // density variants (STG): the one the host's last read totals select, or both back to back (ea.dual:
        // each kernel checks the scan totals on entry and only the selected one does the work)
        const size_t sm = kBandBufs * sizeof(BandBuf);
        const bool sparse = ea.dual || dense == 0, dense_ = ea.dual || dense == 1;
        if (anz && ea.W32 == 32) {
            if (sparse) k_emit_band<T, true, 32, false><<<(unsigned)blocks, kBandThreads, sm, st>>>(ea);
            if (dense_) k_emit_band<T, true, 32, true><<<(unsigned)blocks, kBandThreads, sm, st>>>(ea);
        } else if (anz && ea.W32 == 16) {
            if (sparse) k_emit_band<T, true, 16, false><<<(unsigned)blocks, kBandThreads, sm, st>>>(ea);
            if (dense_) k_emit_band<T, true, 16, true><<<(unsigned)blocks, kBandThreads, sm, st>>>(ea);
        } else if (anz) {
            if (sparse) k_emit_band<T, true, 0, false><<<(unsigned)blocks, kBandThreads, sm, st>>>(ea);
            if (dense_) k_emit_band<T, true, 0, true><<<(unsigned)blocks, kBandThreads, sm, st>>>(ea);
        } else {
            if (sparse) k_emit_band<T, false, 0, false><<<(unsigned)blocks, kBandThreads, sm, st>>>(ea);
            if (dense_) k_emit_band<T, false, 0, true><<<(unsigned)blocks, kBandThreads, sm, st>>>(ea);
        }
    } else if (fast) {   // rows fit one k_count x-tile: per-word point prefixes are row prefixes
        if (anz) k_emit_fast<T, true><<<(unsigned)blocks, 256, 0, st>>>(ea);
        else k_emit_fast<T, false><<<(unsigned)blocks, 256, 0, st>>>(ea);
    } else {
        if (anz) k_emit<T, true><<<(unsigned)blocks, 256, 0, st>>>(ea);
        else k_emit<T, false><<<(unsigned)blocks, 256, 0, st>>>(ea);
    }
}

std::array<int64_t, 6> signature(const psn_volume *v) {
    return {v->dims[0], v->dims[1], v->dims[2], v->own_k0, v->own_k1, (int64_t)(intptr_t)v->labels};
}

psn_status read_totals(psn_ctx *ctx, const psn_volume *v, const Layout &L, const void *ws, psn_mesh *mesh,
                       cudaStream_t st, uint32_t *emit_status) {
    ScanHeader h;
    if (cudaMemcpyAsync(&h, static_cast<const char *>(ws) + L.hdr, sizeof(h), cudaMemcpyDeviceToHost, st) != cudaSuccess)
        return cuda_check(ctx, "totals read-back");
    if (cudaStreamSynchronize(st) != cudaSuccess) return cuda_check(ctx, "totals sync");
    const bool has_lo = L.kA < v->own_k0, has_hi = L.kB > v->own_k1;
    const uint64_t halo_lo = has_lo ? h.halo_lo : 0;
    const uint64_t before_hi = has_hi ? h.halo_hi : h.total[0];
    mesh->halo_lo_points = (int64_t)halo_lo;
    mesh->halo_hi_points = (int64_t)(h.total[0] - before_hi);
    mesh->n_points = (int64_t)(before_hi - halo_lo);
    mesh->n_quads = (int64_t)h.total[1];
    mesh->n_stencil = (int64_t)h.total[2];
    if (emit_status) *emit_status = h.emit_status;
    ctx->emit_dense = (32u * h.total[2] >= (uint64_t)kStageCsr * h.total[0]) ? 1 : 0;
    const uint64_t lim = 1ull << 32;
    if (h.total[0] >= lim || h.total[1] >= lim || h.total[2] >= lim)
        return fail(ctx, PSN_ERR_OVERFLOW, "output exceeds 32-bit ids: P=%llu Q=%llu S=%llu",
                    (unsigned long long)h.total[0], (unsigned long long)h.total[1], (unsigned long long)h.total[2]);
    return PSN_OK;
}

}  // namespace

extern "C" {

psn_status psn_ctx_create(int device, psn_ctx **out) {
    if (!out) return PSN_ERR_ARG;
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess || device < 0 || device >= n) {
        cudaGetLastError();
        *out = nullptr;
        return PSN_ERR_CUDA;
    }
    psn_ctx *c = new psn_ctx();
    c->device = device;
    cudaDeviceGetAttribute(&c->sms, cudaDevAttrMultiProcessorCount, device);
    *out = c;
    return PSN_OK;
}

void psn_ctx_destroy(psn_ctx *ctx) { delete ctx; }

const char *psn_last_error(const psn_ctx *ctx) { return ctx ? ctx->err.c_str() : "no context"; }

const char *psn_status_string(psn_status s) {
    switch (s) {
        case PSN_OK: return "PSN_OK";
        case PSN_ERR_ARG: return "PSN_ERR_ARG";
        case PSN_ERR_LABELS: return "PSN_ERR_LABELS";
        case PSN_ERR_OVERFLOW: return "PSN_ERR_OVERFLOW";
        case PSN_ERR_CAPACITY: return "PSN_ERR_CAPACITY";
        case PSN_ERR_STATE: return "PSN_ERR_STATE";
        case PSN_ERR_CUDA: return "PSN_ERR_CUDA";
    }
    return "unknown";
}

int64_t psn_launch_count(const psn_ctx *ctx) { return ctx ? ctx->launches : 0; }

psn_status psn_extract_workspace(const psn_volume *vol, size_t *bytes) {
    if (!bytes) return PSN_ERR_ARG;
    Layout L;
    psn_status s = layout(nullptr, vol, &L);
    if (s != PSN_OK) return s;
    *bytes = L.total;
    return PSN_OK;
}

namespace {
bool smooth_packed(const psn_ctx *, const psn_volume *vol);   // below, with the smoothing entry points
}

// Record a timing event on st; inside a stream capture as an external event node (the only kind a replayed
// graph records for cudaEventElapsedTime), outside one as a plain record.
static void record_event(cudaEvent_t ev, cudaStream_t st) {
    cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
    cudaStreamIsCapturing(st, &cs);
    if (cs == cudaStreamCaptureStatusActive) cudaEventRecordWithFlags(ev, st, cudaEventRecordExternal);
    else cudaEventRecord(ev, st);
}

static void pass_mark(const psn_ctx *ctx, int i, cudaStream_t st) {
    if (ctx->pass_ev[i]) record_event(ctx->pass_ev[i], st);
}

psn_status psn_ctx_set_smooth_events(psn_ctx *ctx, void *const *events) {
    if (!ctx) return PSN_ERR_ARG;
    for (int i = 0; i < 2; ++i) ctx->smooth_ev[i] = events ? static_cast<cudaEvent_t>(events[i]) : nullptr;
    return PSN_OK;
}

psn_status psn_ctx_set_pass_events(psn_ctx *ctx, void *const *events) {
    if (!ctx) return PSN_ERR_ARG;
    for (int i = 0; i < 4; ++i) ctx->pass_ev[i] = events ? static_cast<cudaEvent_t>(events[i]) : nullptr;
    return PSN_OK;
}

psn_status psn_extract(psn_ctx *ctx, const psn_volume *vol, const psn_labels *labels, psn_mesh *mesh,
                       unsigned phase, void *ws, size_t ws_bytes, void *stream) {
    if (!ctx) return PSN_ERR_ARG;
    ctx->launches = 0;
    Layout L;
    psn_status s = layout(ctx, vol, &L);
    if (s != PSN_OK) return s;
    if (!mesh) return fail(ctx, PSN_ERR_ARG, "mesh is NULL");
    if (!vol->labels) return fail(ctx, PSN_ERR_ARG, "labels pointer is NULL");
    if ((phase & 3u) == 0 || (phase & ~7u))
        return fail(ctx, PSN_ERR_ARG, "phase must be PSN_COUNT, PSN_EMIT or both (optionally | PSN_DEVICE)");
    const bool on_device = (phase & PSN_DEVICE) != 0;
    if (!ws || ws_bytes < L.total) return fail(ctx, PSN_ERR_ARG, "workspace too small: need %zu bytes", L.total);
    if (cudaSetDevice(ctx->device) != cudaSuccess) return cuda_check(ctx, "cudaSetDevice");
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    const int eb = (int)vol->dtype;
    LabelSet ls;
    bool anz = true;
    s = prepare_labels(ctx, vol, labels, ws, L, st, &ls, &anz);
    if (s != PSN_OK) return s;
    const void *slab0 = vol->labels;   // pointer to slice z_lo

    if (phase & PSN_COUNT) {
        pass_mark(ctx, 0, st);
        if (cudaMemsetAsync(at<char>(ws, L.hdr), 0, L.cntP - L.hdr, st) != cudaSuccess) return cuda_check(ctx, "memset");
        const int64_t E = 16 / eb;                            // elements per 16-byte lane chunk
        const int64_t chunks = (L.M - 1 + E - 1) / E;        // lane chunks per row
        const int64_t nLay = L.kB - L.kA;
        const int cpl_max = eb == 4 ? 4 : 8;
        int cpl = 1;
        while (cpl < cpl_max && 32 * cpl < chunks) cpl *= 2;
        const bool use3 = ctx->count_mode == PSN_COUNT_AUTO && chunks <= 32 * cpl;
        CountArgs ca{};
        ca.labels = slab0; ca.M = L.M; ca.N = L.N; ca.O = L.O; ca.z_lo = vol->z_lo;
        ca.kA = L.kA; ca.kB = L.kB; ca.own_k0 = vol->own_k0; ca.own_k1 = vol->own_k1; ca.W32 = L.W32;
        ca.cntP = at<uint32_t>(ws, L.cntP); ca.cntQ = at<uint32_t>(ws, L.cntQ); ca.cntS = at<uint32_t>(ws, L.cntS);
        ca.cntYZ = at<uint32_t>(ws, L.cntYZ);
        ca.trim = at<int2>(ws, L.trim); ca.pmask = at<uint32_t>(ws, L.pmask); ca.ppre = at<uint16_t>(ws, L.ppre);
        ca.ls = ls;
        ca.tma = ((L.M * eb) % 16 == 0) && ((reinterpret_cast<uintptr_t>(slab0) & 15u) == 0);
        cudaError_t ce;
        if (use3) {
            // warp-per-row producer/consumer kernel: 16 voxel rows per CTA, z-chunks sized for
            // ~8 waves of 2 CTAs per SM, each CTA marching >= 8 layers
            const int64_t nJB = (L.N - 1 + kC3Rows - 1) / kC3Rows;
            const int64_t target_ctas = (int64_t)ctx->sms * 2 * 8;
            int64_t nZC = std::max<int64_t>(1, (target_ctas + nJB - 1) / nJB);
            nZC = std::min(nZC, std::max<int64_t>(1, nLay / 8));   // >= 8 layers per CTA (c2: 16 -> 8 is -10 %)
            nZC = std::min(nZC, nLay);
            const int64_t KZ = (nLay + nZC - 1) / nZC;
            nZC = (nLay + KZ - 1) / KZ;
            const int64_t RB = (int64_t)align16((size_t)(L.M * eb)) + 32;   // row + 32-byte pad (pad_row)
            // ring depth: as many slices as keep 3 CTAs resident per SM (<= ~70 KB each), 3..8
            const int64_t SBy = (int64_t)(kC3Rows + 1) * RB;
            // (a general label set also keeps its 8 KB classification bitset in shared memory)
            // rows of an odd 1- / 2-byte length: a staging area for the aligned supersets (k_count3)
            const bool shift = !ca.tma && (L.M * eb) % 4 != 0 && (reinterpret_cast<uintptr_t>(slab0) & 15u) == 0;
            const int64_t RB2 = shift ? (int64_t)align16((size_t)(L.M * eb)) + 32 : 0;
            const int64_t stg = (int64_t)(kC3Rows + 1) * RB2;
            const int64_t budget = 108 * 1024 - ((!anz && eb < 4) ? 8 * 1024 : 0) - stg;
            int ns = (int)std::max<int64_t>(3, std::min<int64_t>(kC3MaxStages, budget / SBy));
            const size_t smem = (size_t)ns * (size_t)(kC3Rows + 1) * (size_t)RB + (size_t)stg;
            ca.NS = ns;
            ca.stg_off = (int64_t)ns * SBy; ca.RB2 = RB2;
            ca.nXT = 1; ca.nJB = nJB; ca.KZ = KZ; ca.RB = RB; ca.multi_xt = 0;
            const int64_t blocks = nJB * nZC;
            if (eb == 1) ce = dispatch_count3<uint8_t>(ca, anz, cpl, blocks, smem, st);
            else if (eb == 2) ce = dispatch_count3<uint16_t>(ca, anz, cpl, blocks, smem, st);
            else ce = dispatch_count3<uint32_t>(ca, anz, cpl, blocks, smem, st);
            if (ce != cudaSuccess) return fail(ctx, PSN_ERR_CUDA, "k_count3 launch: %s", cudaGetErrorString(ce));
            ++ctx->launches;
        } else {
            const int64_t nXT = (chunks + 255) / 256;             // 256 chunks (256*E x-positions) per CTA
            const int64_t WX = std::min<int64_t>((chunks + 31) / 32, 8);
            const int tj = eb == 1 ? count_tj<uint8_t>() : (eb == 2 ? count_tj<uint16_t>() : count_tj<uint32_t>());
            const int64_t nJB = (L.N - 1 + tj - 1) / tj;
            // z-chunks: ~8 waves of CTAs (4 resident per SM) so the last wave's tail is small,
            // while each CTA still marches >= 16 layers to amortise its TMA prologue
            const int64_t target_ctas = (int64_t)ctx->sms * 4 * 8;
            int64_t nZC = std::max<int64_t>(1, (target_ctas + nXT * nJB - 1) / (nXT * nJB));
            nZC = std::min(nZC, std::max<int64_t>(1, nLay / 16));
            nZC = std::min(nZC, nLay);
            const int64_t KZ = (nLay + nZC - 1) / nZC;
            nZC = (nLay + KZ - 1) / KZ;
            const int64_t xpad = 16 / eb;
            // every thread of the CTA reads its 16-byte chunk and the next word, so a staged row
            // spans the CTA's full width (zero-filled past the row end), plus the 16-byte pad
            const int64_t RB = (int64_t)align16((size_t)((32 * WX * E + xpad) * eb));
            const size_t smem = (size_t)kCountStages * (size_t)(tj + 1) * (size_t)RB;
            ca.nXT = nXT; ca.nJB = nJB; ca.KZ = KZ; ca.RB = RB;
            ca.multi_xt = nXT > 1 ? 1 : 0;
            const int64_t gridR = std::min<int64_t>((L.R + 255) / 256, (int64_t)ctx->sms * 8);
            if (ca.multi_xt) {
                k_init_multixt<<<(unsigned)gridR, 256, 0, st>>>(ca.cntP, ca.cntQ, ca.cntS, ca.trim, L.R);
                ++ctx->launches;
            }
            const int64_t blocks = nXT * nJB * nZC;
            const int threads = (int)(32 * WX);
            if (eb == 1) ce = dispatch_count<uint8_t>(ca, anz, blocks, threads, smem, st);
            else if (eb == 2) ce = dispatch_count<uint16_t>(ca, anz, blocks, threads, smem, st);
            else ce = dispatch_count<uint32_t>(ca, anz, blocks, threads, smem, st);
            if (ce != cudaSuccess) return fail(ctx, PSN_ERR_CUDA, "k_count launch: %s", cudaGetErrorString(ce));
            ++ctx->launches;
            if (ca.multi_xt) {
                k_trim_fix<<<(unsigned)gridR, 256, 0, st>>>(ca.trim, ca.cntP, L.R);
                ++ctx->launches;
            }
        }
        pass_mark(ctx, 1, st);
        ScanArgs sa;
        sa.cntP = ca.cntP; sa.cntQ = ca.cntQ; sa.cntS = ca.cntS;
        sa.cntYZ = use3 ? ca.cntYZ : nullptr;   // k_count3 counts shared faces once (row_stencil)
        sa.NV = L.N - 1; sa.kA = L.kA; sa.O = L.O;
        sa.offP = at<uint32_t>(ws, L.offP); sa.offQ = at<uint32_t>(ws, L.offQ); sa.offS = at<uint32_t>(ws, L.offS);
        sa.R = L.R;
        sa.own_row0 = (L.N - 1) * (vol->own_k0 - L.kA);
        sa.own_row1 = (L.N - 1) * (vol->own_k1 - L.kA);
        sa.tiles = at<TileStatus>(ws, L.tiles); sa.hdr = at<ScanHeader>(ws, L.hdr);
        k_scan<<<(unsigned)L.nTiles, kScanThreads, 0, st>>>(sa);
        ++ctx->launches;
        pass_mark(ctx, 2, st);
        if ((s = cuda_check(ctx, "count/scan launch")) != PSN_OK) return s;
        ctx->counted[ws] = signature(vol);
        ctx->yz_split[ws] = use3;
        if (!(phase & PSN_EMIT)) return on_device ? PSN_OK : read_totals(ctx, vol, L, ws, mesh, st, nullptr);
    } else {
        auto it = ctx->counted.find(ws);
        if (it == ctx->counted.end() || it->second != signature(vol))
            return fail(ctx, PSN_ERR_STATE, "PSN_EMIT needs a preceding PSN_COUNT of the same volume on this workspace");
        if (!on_device && (mesh->halo_lo_points + mesh->n_points + mesh->halo_hi_points > mesh->cap_points ||
                           mesh->n_quads > mesh->cap_quads || mesh->n_stencil > mesh->cap_stencil))
            return fail(ctx, PSN_ERR_CAPACITY, "capacity too small: need points %lld quads %lld stencil %lld",
                        (long long)(mesh->halo_lo_points + mesh->n_points + mesh->halo_hi_points),
                        (long long)mesh->n_quads, (long long)mesh->n_stencil);
    }
    // ---- EMIT
    if (!mesh->points || !mesh->quads || !mesh->pairs || !mesh->stencil_offsets || !mesh->stencil_ids || !mesh->face_masks)
        return fail(ctx, PSN_ERR_ARG, "mesh output pointers must be non-NULL");
    if ((reinterpret_cast<uintptr_t>(mesh->quads) & 15u) || (reinterpret_cast<uintptr_t>(mesh->pairs) & 7u))
        return fail(ctx, PSN_ERR_ARG, "quads must be 16-byte and pairs 8-byte aligned");
    EmitArgs ea;
    ea.labels = slab0; ea.M = L.M; ea.N = L.N; ea.O = L.O; ea.z_lo = vol->z_lo;
    ea.kA = L.kA; ea.kB = L.kB; ea.own_k0 = vol->own_k0; ea.own_k1 = vol->own_k1; ea.W32 = L.W32; ea.R = L.R;
    ea.cntP = at<uint32_t>(ws, L.cntP); ea.offP = at<uint32_t>(ws, L.offP);
    ea.offQ = at<uint32_t>(ws, L.offQ); ea.offS = at<uint32_t>(ws, L.offS); ea.pmask = at<uint32_t>(ws, L.pmask);
    ea.ppre = at<uint16_t>(ws, L.ppre);
    ea.ls = ls;
    for (int a = 0; a < 3; ++a) { ea.sp[a] = vol->spacing[a]; ea.org[a] = vol->origin[a]; }
    ea.points = mesh->points; ea.quads = mesh->quads; ea.pairs = mesh->pairs;
    ea.csr_off = mesh->stencil_offsets; ea.csr_ids = mesh->stencil_ids; ea.fmask = mesh->face_masks;
    ea.cap_points = mesh->cap_points; ea.cap_quads = mesh->cap_quads; ea.cap_stencil = mesh->cap_stencil;
    ea.first_point = (uint32_t)mesh->first_point; ea.first_quad = (uint32_t)mesh->first_quad;
    ea.first_stencil = (uint32_t)mesh->first_stencil;
    ea.first_dev = mesh->first_dev;
    ea.hdr = at<ScanHeader>(ws, L.hdr);
    ea.scache = nullptr;
    mesh->smooth_cache_valid = 0;
    int64_t blocks = std::max<int64_t>(1, std::min<int64_t>((L.R + 7) / 8, (int64_t)ctx->sms * 16));
    const int emode = ctx->emit_mode;
    if (L.W32 <= 32 && emode == 0) {   // k_emit_band: one resident wave of CTAs looping over bands
        if (mesh->smooth_cache && smooth_packed(ctx, vol)) {   // the packed smoothing cache rides along
            ea.scache = reinterpret_cast<uint2 *>(mesh->smooth_cache);
            mesh->smooth_cache_valid = 1;
        }
        int occ = 0;
        const void *fn = eb == 1 ? (anz ? (const void *)k_emit_band<uint8_t, true> : (const void *)k_emit_band<uint8_t, false>)
                       : eb == 2 ? (anz ? (const void *)k_emit_band<uint16_t, true> : (const void *)k_emit_band<uint16_t, false>)
                                 : (anz ? (const void *)k_emit_band<uint32_t, true> : (const void *)k_emit_band<uint32_t, false>);
        static bool attr = false;
        if (!attr) {
            for (const void *f : {(const void *)k_emit_band<uint8_t, true>, (const void *)k_emit_band<uint8_t, false>,
                                  (const void *)k_emit_band<uint16_t, true>, (const void *)k_emit_band<uint16_t, false>,
                                  (const void *)k_emit_band<uint32_t, true>, (const void *)k_emit_band<uint32_t, false>})
                cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)(kBandBufs * sizeof(BandBuf)));
            for (const void *f : {(const void *)k_emit_band<uint8_t, true, 32>, (const void *)k_emit_band<uint8_t, true, 16>,
                                  (const void *)k_emit_band<uint16_t, true, 32>, (const void *)k_emit_band<uint16_t, true, 16>,
                                  (const void *)k_emit_band<uint32_t, true, 32>, (const void *)k_emit_band<uint32_t, true, 16>})
                cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)(kBandBufs * sizeof(BandBuf)));
            for (const void *f : {(const void *)k_emit_band<uint8_t, true, 0, false>, (const void *)k_emit_band<uint8_t, false, 0, false>,
                                  (const void *)k_emit_band<uint16_t, true, 0, false>, (const void *)k_emit_band<uint16_t, false, 0, false>,
                                  (const void *)k_emit_band<uint32_t, true, 0, false>, (const void *)k_emit_band<uint32_t, false, 0, false>,
                                  (const void *)k_emit_band<uint8_t, true, 32, false>, (const void *)k_emit_band<uint8_t, true, 16, false>,
                                  (const void *)k_emit_band<uint16_t, true, 32, false>, (const void *)k_emit_band<uint16_t, true, 16, false>,
                                  (const void *)k_emit_band<uint32_t, true, 32, false>, (const void *)k_emit_band<uint32_t, true, 16, false>})
                cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)(kBandBufs * sizeof(BandBuf)));
            attr = true;
        }
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, fn, kBandThreads, kBandBufs * sizeof(BandBuf));
        blocks = std::max<int64_t>(1, std::min<int64_t>((L.R + kBand - 1) / kBand, (int64_t)ctx->sms * std::max(occ, 1)));
    }
    const bool fast = emode != PSN_EMIT_SCAN &&
                      (L.M - 1) <= (int64_t)(eb == 1 ? count_xt<uint8_t>() : eb == 2 ? count_xt<uint16_t>() : count_xt<uint32_t>());
    const bool band = fast && L.W32 <= 32 && emode == 0;
    const char *dv = getenv("PSN_EMIT_DENSE");   // test / A-B override: -1 both, 0 sparse, 1 dense variant
    const int dense = dv ? atoi(dv) : ctx->emit_dense;
    ea.dual = (band && dense < 0) ? 1 : 0;   // density unknown to the host: both variants
    if (eb == 1) dispatch_emit<uint8_t>(ea, anz, fast, blocks, st, emode, dense);
    else if (eb == 2) dispatch_emit<uint16_t>(ea, anz, fast, blocks, st, emode, dense);
    else dispatch_emit<uint32_t>(ea, anz, fast, blocks, st, emode, dense);
    ctx->launches += ea.dual ? 2 : 1;
    pass_mark(ctx, 3, st);
    return cuda_check(ctx, "emit launch");
}

namespace {
__global__ void k_rows_out(ScanArgs sa, const int2 *trim, uint32_t *counts, int2 *trims) {
    const int64_t R = sa.R;
    for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < R; r += (int64_t)gridDim.x * blockDim.x) {
        const uint32_t p = sa.cntP[r];
        if (counts) { counts[r] = p; counts[R + r] = sa.cntQ[r]; counts[2 * R + r] = row_stencil(sa, r); }
        if (trims) trims[r] = p ? trim[r] : make_int2(0, 0);
    }
}
}  // namespace

psn_status psn_extract_rows(psn_ctx *ctx, const psn_volume *vol, const void *ws, size_t ws_bytes, uint32_t *counts,
                            int32_t *trims, int64_t *rows, void *stream) {
    if (!ctx) return PSN_ERR_ARG;
    Layout L;
    psn_status s = layout(ctx, vol, &L);
    if (s != PSN_OK) return s;
    if (!ws || ws_bytes < L.total) return fail(ctx, PSN_ERR_ARG, "workspace too small: need %zu bytes", L.total);
    if ((reinterpret_cast<uintptr_t>(trims) & 7u)) return fail(ctx, PSN_ERR_ARG, "trims must be 8-byte aligned");
    auto it = ctx->counted.find(ws);
    if (it == ctx->counted.end() || it->second != signature(vol))
        return fail(ctx, PSN_ERR_STATE, "no PSN_COUNT of this volume on this workspace");
    if (rows) *rows = L.R;
    if (!counts && !trims) return PSN_OK;
    if (cudaSetDevice(ctx->device) != cudaSuccess) return cuda_check(ctx, "cudaSetDevice");
    const int64_t grid = std::max<int64_t>(1, std::min<int64_t>((L.R + 255) / 256, (int64_t)ctx->sms * 8));
    void *w = const_cast<void *>(ws);
    ScanArgs sa{};
    sa.cntP = at<uint32_t>(w, L.cntP); sa.cntQ = at<uint32_t>(w, L.cntQ); sa.cntS = at<uint32_t>(w, L.cntS);
    sa.cntYZ = ctx->yz_split[ws] ? at<uint32_t>(w, L.cntYZ) : nullptr;
    sa.R = L.R; sa.NV = L.N - 1; sa.kA = L.kA; sa.O = L.O;
    sa.own_row0 = (L.N - 1) * (vol->own_k0 - L.kA);
    sa.own_row1 = (L.N - 1) * (vol->own_k1 - L.kA);
    k_rows_out<<<(unsigned)grid, 256, 0, static_cast<cudaStream_t>(stream)>>>(sa, at<int2>(w, L.trim), counts,
                                                                             reinterpret_cast<int2 *>(trims));
    return cuda_check(ctx, "rows launch");
}

namespace {
__global__ void k_totals_out(const ScanHeader *h, int has_lo, int has_hi, int64_t *out) {
    if (threadIdx.x == 0 && blockIdx.x == 0) {
        const uint64_t lo = has_lo ? h->halo_lo : 0, before_hi = has_hi ? h->halo_hi : h->total[0];
        out[0] = (int64_t)(before_hi - lo); out[1] = (int64_t)h->total[1]; out[2] = (int64_t)h->total[2];
        out[3] = (int64_t)lo; out[4] = (int64_t)(h->total[0] - before_hi);
    }
}
}  // namespace

psn_status psn_extract_totals(psn_ctx *ctx, const psn_volume *vol, const void *ws, size_t ws_bytes, int64_t *out,
                              void *stream) {
    if (!ctx) return PSN_ERR_ARG;
    Layout L;
    psn_status s = layout(ctx, vol, &L);
    if (s != PSN_OK) return s;
    if (!ws || ws_bytes < L.total || !out) return fail(ctx, PSN_ERR_ARG, "bad workspace or output");
    if (cudaSetDevice(ctx->device) != cudaSuccess) return cuda_check(ctx, "cudaSetDevice");
    k_totals_out<<<1, 32, 0, static_cast<cudaStream_t>(stream)>>>(
        at<ScanHeader>(const_cast<void *>(ws), L.hdr), L.kA < vol->own_k0 ? 1 : 0, L.kB > vol->own_k1 ? 1 : 0, out);
    return cuda_check(ctx, "totals launch");
}

psn_status psn_mesh_totals(psn_ctx *ctx, const psn_volume *vol, psn_mesh *mesh, const void *ws, size_t ws_bytes,
                           void *stream) {
    if (!ctx) return PSN_ERR_ARG;
    Layout L;
    psn_status s = layout(ctx, vol, &L);
    if (s != PSN_OK) return s;
    if (!mesh || !ws || ws_bytes < L.total) return fail(ctx, PSN_ERR_ARG, "bad mesh or workspace");
    uint32_t es = 0;
    s = read_totals(ctx, vol, L, ws, mesh, static_cast<cudaStream_t>(stream), &es);
    if (s != PSN_OK) return s;
    if (es) return fail(ctx, PSN_ERR_CAPACITY, "emission skipped: capacities too small");
    return PSN_OK;
}

namespace {
struct SmoothLayout { size_t nbr, buf0, buf1, rng, done, sch, total; int64_t nw, U; };
// [nbr uint4 x P | buf0 float4 x W | buf1 float4 x W | rng int2 x U | done u32 x U | sched]
SmoothLayout smooth_layout(const psn_mesh *m) {
    SmoothLayout L;
    L.nw = m->halo_lo_points + m->n_points + m->halo_hi_points;
    L.U = (m->n_points + kTbTileMin - 1) / kTbTileMin;   // schedule arrays sized for the smallest tile
    L.nbr = 0;
    L.buf0 = align_up(16 * (size_t)std::max<int64_t>(m->n_points, 1));
    // offset buffers: float4 [W]
    const size_t bufb = 16 * (size_t)std::max<int64_t>(L.nw, 1);
    L.buf1 = L.buf0 + align_up(bufb);
    L.rng = L.buf1 + align_up(bufb);
    L.done = L.rng + align_up(8 * (size_t)std::max<int64_t>(L.U, 1));
    L.sch = L.done + align_up(4 * (size_t)std::max<int64_t>(L.U, 1));
    L.total = L.sch + align_up(sizeof(TbSched));
    return L;
}
}  // namespace

psn_status psn_smooth_workspace(const psn_mesh *mesh, size_t *bytes) {
    if (!bytes || !mesh || mesh->n_points < 0 || mesh->halo_lo_points < 0 || mesh->halo_hi_points < 0) return PSN_ERR_ARG;
    *bytes = smooth_layout(mesh).total;
    return PSN_OK;
}

namespace {
psn_status check_smooth_args(psn_ctx *ctx, const psn_mesh *mesh, float relaxation, float d) {
    if (!mesh) return fail(ctx, PSN_ERR_ARG, "mesh is NULL");
    if (mesh->halo_lo_points + mesh->n_points + mesh->halo_hi_points >= (1ll << 30))
        return fail(ctx, PSN_ERR_OVERFLOW, "smoothing supports windows of < 2^30 points");
    if (!(relaxation >= 0.f && relaxation <= 1.f)) return fail(ctx, PSN_ERR_ARG, "relaxation must be in [0,1]");
    if (!(d >= 0.f)) return fail(ctx, PSN_ERR_ARG, "constraint distance must be >= 0");
    if (mesh->n_points < 0 || mesh->halo_lo_points < 0 || mesh->halo_hi_points < 0)
        return fail(ctx, PSN_ERR_ARG, "negative point counts");
    if (mesh->n_points > 0 && (!mesh->face_masks || !mesh->stencil_offsets || (!mesh->stencil_ids && mesh->n_stencil > 0)))
        return fail(ctx, PSN_ERR_ARG, "mesh stencil arrays are NULL");
    return PSN_OK;
}

// Box constraint of half-width d (voxel units), or the sphere of radius d*min(s) (reading Q26).
Constraint make_constraint(int shape, float d, const double *sp) {
    Constraint c;
    c.d = d;
    c.sphere = shape == PSN_CONSTRAINT_SPHERE ? 1 : 0;
    c.sx = sp ? (float)sp[0] : 1.f; c.sy = sp ? (float)sp[1] : 1.f; c.sz = sp ? (float)sp[2] : 1.f;
    const double smin = sp ? std::min(sp[0], std::min(sp[1], sp[2])) : 1.0;
    c.r = (float)((double)d * smin);
    c.r2 = __fmul_rn_host(c.r);
    return c;
}

int64_t grid_for(psn_ctx *ctx, int64_t n) {
    return std::max<int64_t>(1, std::min<int64_t>((n + 255) / 256, (int64_t)ctx->sms * 16));
}

// Packed 8-byte smoothing cache (k_smooth_prep8) when the volume's rows / layers keep
// neighbour id distances within its fields: y < 2^10, z < 2^21.
bool smooth_packed(const psn_ctx *, const psn_volume *vol) {
    if (!vol || getenv("PSN_SMOOTH_NBR16")) return false;
    const int64_t Mc = vol->dims[0] - 1, Nc = vol->dims[1] - 1;
    return Mc < (1 << 10) && Mc * Nc < (1 << 21);
}

psn_status launch_prep8(psn_ctx *ctx, const psn_mesh *mesh, void *ws, cudaStream_t st) {
    if (mesh->n_points == 0) return PSN_OK;
    k_smooth_prep8<<<(unsigned)grid_for(ctx, mesh->n_points), 256, 0, st>>>(
        mesh->face_masks, mesh->stencil_offsets, mesh->stencil_ids, static_cast<uint2 *>(ws), mesh->n_points,
        (uint32_t)mesh->halo_lo_points, (uint32_t)(mesh->first_point - mesh->halo_lo_points),
        (uint32_t)mesh->first_stencil);
    ++ctx->launches;
    return cuda_check(ctx, "smooth prep launch");
}

SmoothV4 smooth_v4_args(const psn_ctx *ctx, const psn_volume *vol, const psn_mesh *mesh, const void *ws, float lambda,
                        float d) {
    SmoothV4 v;
    memset(&v, 0, sizeof(v));
    v.nbr = static_cast<const uint4 *>(ws); v.nbr8 = static_cast<const uint2 *>(ws); v.points = mesh->points;
    v.n_own = (uint32_t)mesh->n_points; v.halo_lo = (uint32_t)mesh->halo_lo_points;
    v.lambda = lambda; v.d = d;
    v.cons = make_constraint(ctx->constraint, d, vol->spacing);
    for (int c = 0; c < 3; ++c) { v.sp[c] = vol->spacing[c]; v.org[c] = vol->origin[c]; }
    return v;
}

// The k_smooth_v4 instantiation for (cache form, one-step-ahead cache loads, peer push, sphere).
V4Fn pick_v4(bool packed, bool pref, bool peer, bool sphere) {
    if (peer) return packed ? v4_sel<true, false, true>(sphere) : v4_sel<false, false, true>(sphere);
    if (packed) return pref ? v4_sel<true, true, false>(sphere) : v4_sel<true, false, false>(sphere);
    return v4_sel<false, false, false>(sphere);
}
int64_t v4_grid(psn_ctx *ctx, V4Fn kern, int64_t n) {
    int occ = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, 256, 0);
    return std::max<int64_t>(1, std::min<int64_t>((n + 255) / 256, (int64_t)ctx->sms * std::max(occ, 1)));
}

psn_status launch_prep(psn_ctx *ctx, const psn_mesh *mesh, void *ws, cudaStream_t st) {
    if (mesh->n_points == 0) return PSN_OK;
    k_smooth_prep<<<(unsigned)grid_for(ctx, mesh->n_points), 256, 0, st>>>(
        mesh->face_masks, mesh->stencil_offsets, mesh->stencil_ids, static_cast<uint4 *>(ws), mesh->n_points,
        (uint32_t)mesh->halo_lo_points, (uint32_t)(mesh->first_point - mesh->halo_lo_points),
        (uint32_t)mesh->first_stencil);
    ++ctx->launches;
    return cuda_check(ctx, "smooth prep launch");
}
}  // namespace

psn_status psn_smooth_prepare(psn_ctx *ctx, const psn_volume *vol, const psn_mesh *mesh, void *ws, size_t ws_bytes,
                              void *stream) {
    if (!ctx) return PSN_ERR_ARG;
    ctx->launches = 0;
    psn_status s = check_smooth_args(ctx, mesh, 0.f, 0.f);
    if (s != PSN_OK) return s;
    if (!vol) return fail(ctx, PSN_ERR_ARG, "volume is NULL");
    if (!ws || ws_bytes < smooth_layout(mesh).buf0) return fail(ctx, PSN_ERR_ARG, "smoothing workspace too small");
    if (cudaSetDevice(ctx->device) != cudaSuccess) return cuda_check(ctx, "cudaSetDevice");
    const cudaStream_t st = static_cast<cudaStream_t>(stream);
    return smooth_packed(ctx, vol) ? launch_prep8(ctx, mesh, ws, st) : launch_prep(ctx, mesh, ws, st);
}

psn_status psn_smooth(psn_ctx *ctx, const psn_volume *vol, const psn_mesh *mesh, float *out, int32_t iterations,
                      float relaxation, float constraint_distance, void *ws, size_t ws_bytes, void *stream) {
    if (!ctx) return PSN_ERR_ARG;
    ctx->launches = 0;
    psn_status s = check_smooth_args(ctx, mesh, relaxation, constraint_distance);
    if (s != PSN_OK) return s;
    if (!vol) return fail(ctx, PSN_ERR_ARG, "volume is NULL");
    if (iterations < 0) return fail(ctx, PSN_ERR_ARG, "iterations must be >= 0");
    if (mesh->halo_lo_points || mesh->halo_hi_points)
        return fail(ctx, PSN_ERR_ARG, "psn_smooth needs a whole volume; slabs use psn_smooth_step + halo exchange");
    const SmoothLayout SL = smooth_layout(mesh);
    if (!out || !mesh->points || !ws || ws_bytes < SL.total)
        return fail(ctx, PSN_ERR_ARG, "out/points NULL or workspace too small (need %zu)", SL.total);
    if (cudaSetDevice(ctx->device) != cudaSuccess) return cuda_check(ctx, "cudaSetDevice");
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    const int64_t nw = mesh->n_points;
    if (nw == 0) return PSN_OK;
    const int64_t g = grid_for(ctx, nw);
    if (iterations == 0 || relaxation == 0.f) {
        k_finalize<<<(unsigned)g, 256, 0, st>>>(nullptr, mesh->points, out, 0, nw, vol->spacing[0], vol->spacing[1],
                                               vol->spacing[2], vol->origin[0], vol->origin[1], vol->origin[2]);
        ++ctx->launches;
        return cuda_check(ctx, "finalize launch");
    }
    const Constraint cons = make_constraint(ctx->constraint, constraint_distance, vol->spacing);
    const bool packed = ctx->smooth_mode == PSN_SMOOTH_PER_ITERATION && smooth_packed(ctx, vol);
    // the packed cache written by the emission, if any, replaces the prep pass
    const bool cached = packed && mesh->smooth_cache && mesh->smooth_cache_valid;
    // split cache without an emitted cache: the first iteration builds it (k_smooth_first, no prep pass)
    const size_t hi_at = align_up(8 * (size_t)nw);
    const bool split = packed && iterations > 1 && hi_at + 4 * (size_t)nw <= SL.buf0 && !getenv("PSN_SMOOTH_NOSPLIT");
    const bool first = split && !cached && !getenv("PSN_SMOOTH_NOFIRST");
    if (!cached && !first && (s = packed ? launch_prep8(ctx, mesh, ws, st) : launch_prep(ctx, mesh, ws, st)) != PSN_OK)
        return s;
    if (ctx->smooth_mode == PSN_SMOOTH_PER_ITERATION) {
        // one launch per Jacobi iteration, offsets double-buffered in the two buffer slots
        SmoothV4 v = smooth_v4_args(ctx, vol, mesh, ws, relaxation, constraint_distance);
        if (cached) v.nbr8 = reinterpret_cast<const uint2 *>(mesh->smooth_cache);
        float4 *b4[2] = {at<float4>(ws, SL.buf0), at<float4>(ws, SL.buf1)};
        // one-step-ahead cache loads: measured faster up to tens of millions of points (c6
        // -8 %, c4 -3 %) and slower on c5a's 133 M (+8 %), where the step is closest to the
        // DRAM bound; chosen by size
        const bool pref = packed && nw < (1ll << 26);
        const V4Fn kern = pick_v4(packed, pref, false, cons.sphere != 0);
        const int64_t g4 = v4_grid(ctx, kern, nw);
        // split cache (k_smooth_split): iterations 2..T take the cache entry's lo word from the w slot of
        // the point's own offsets and its hi word from a 4-byte array in the cache region's second half
        // (free: the packed cache uses 8 of the 16 bytes per point the region holds)
        uint32_t *hi = split ? at<uint32_t>(ws, hi_at) : nullptr;
        const V4Fn kern2 = split ? split_sel(pref, cons.sphere != 0) : kern;
        const int64_t g42 = split ? v4_grid(ctx, kern2, nw) : g4;
        const float4 *s4 = nullptr;
        if (ctx->smooth_ev[0]) record_event(ctx->smooth_ev[0], st);
        int32_t t_begin = 0;
        if (first && !getenv("PSN_SMOOTH_NOFIRST2")) {   // iterations 1 and 2 in one pass (k_smooth_first2)
            const bool last = iterations == 2;
            v.src = nullptr; v.dst = last ? nullptr : b4[1]; v.world = last ? out : nullptr; v.hi_out = hi;
            v.fmask = mesh->face_masks; v.csr_off = mesh->stencil_offsets; v.csr_ids = mesh->stencil_ids;
            v.win_base = (uint32_t)(mesh->first_point - mesh->halo_lo_points);
            v.first_stencil = (uint32_t)mesh->first_stencil;
            const V4Fn f2 = cons.sphere ? k_smooth_first2<true> : k_smooth_first2<false>;
            f2<<<(unsigned)v4_grid(ctx, f2, nw), 256, 0, st>>>(v);
            ++ctx->launches;
            s4 = v.dst;
            t_begin = 2;
        }
        for (int32_t t = t_begin; t < iterations; ++t) {
            const bool last = (t == iterations - 1);
            v.src = s4; v.dst = last ? nullptr : b4[t & 1]; v.world = last ? out : nullptr;
            v.hi_out = (split && t == 0) ? hi : nullptr; v.hi = hi;
            if (t == 0 && first) {
                v.fmask = mesh->face_masks; v.csr_off = mesh->stencil_offsets; v.csr_ids = mesh->stencil_ids;
                v.win_base = (uint32_t)(mesh->first_point - mesh->halo_lo_points);
                v.first_stencil = (uint32_t)mesh->first_stencil;
                const int64_t gf = v4_grid(ctx, cons.sphere ? k_smooth_first<true> : k_smooth_first<false>, nw);
                if (cons.sphere) k_smooth_first<true><<<(unsigned)gf, 256, 0, st>>>(v);
                else k_smooth_first<false><<<(unsigned)gf, 256, 0, st>>>(v);
            } else if (t == 0) kern<<<(unsigned)g4, 256, 0, st>>>(v);
            else kern2<<<(unsigned)g42, 256, 0, st>>>(v);
            ++ctx->launches;
            s4 = v.dst;
        }
        if (ctx->smooth_ev[1]) record_event(ctx->smooth_ev[1], st);
        return cuda_check(ctx, "smooth launch");
    }
    // wavefront (temporally blocked) smoothing: G iterations per persistent launch
    TbSched *sch = at<TbSched>(ws, SL.sch);
    uint32_t *done = at<uint32_t>(ws, SL.done);
    int2 *rng = at<int2>(ws, SL.rng);
    const uint32_t tile = ctx->smooth_tile > 0 ? (uint32_t)ctx->smooth_tile : 1024u;
    const int64_t U = (nw + tile - 1) / tile;
    if (cudaMemsetAsync(sch, 0, sizeof(TbSched), st) != cudaSuccess ||
        cudaMemsetAsync(done, 0, 4 * (size_t)U, st) != cudaSuccess)
        return cuda_check(ctx, "smooth memset");
    k_tile_ranges<<<(unsigned)U, 256, 0, st>>>(static_cast<const uint4 *>(ws), mesh->face_masks, (uint32_t)nw, tile,
                                               rng, sch);
    ++ctx->launches;
    // iterations per launch: keep the live window (G x ~2 voxel layers of points x 49 B) well inside L2
    int32_t G = ctx->smooth_group;
    if (G <= 0) {
        const double layer_pts = (double)nw / (double)std::max<int64_t>(vol->dims[2] - 1, 1);
        // window ~ 2G blocks of (one layer ~ neighbour distance) points; ~40 MB of the 126 MB L2
        G = (int32_t)std::max(1.0, std::min((double)iterations, 40.0e6 / (4.0 * layer_pts * 49.0)));
    }
    TbArgs ta;
    memset(&ta, 0, sizeof(ta));
    ta.buf[0] = at<float4>(ws, SL.buf0); ta.buf[1] = at<float4>(ws, SL.buf1);
    ta.world = out; ta.fmask = mesh->face_masks; ta.nbr = static_cast<const uint4 *>(ws); ta.points = mesh->points;
    ta.rng = rng; ta.done = done; ta.sch = sch;
    ta.n = (uint32_t)nw; ta.U = (uint32_t)U; ta.tile = tile; ta.T = iterations;
    ta.lambda = relaxation; ta.cons = make_constraint(ctx->constraint, constraint_distance, vol->spacing);
    for (int c = 0; c < 3; ++c) { ta.sp[c] = vol->spacing[c]; ta.org[c] = vol->origin[c]; }
    const unsigned grid = (unsigned)std::max<int64_t>(1, std::min<int64_t>((int64_t)ctx->sms * 4, U * iterations));
    for (int32_t t0 = 0; t0 < iterations; t0 += G) {
        ta.t0 = t0; ta.G = std::min(G, iterations - t0);
        if (cudaMemsetAsync(&sch->counter, 0, sizeof(uint32_t), st) != cudaSuccess) return cuda_check(ctx, "smooth memset");
        k_smooth_tb<<<grid, 256, 0, st>>>(ta);
        ++ctx->launches;
    }
    return cuda_check(ctx, "smooth wavefront launch");
}

psn_status psn_smooth_status(psn_ctx *ctx, const psn_mesh *mesh, const void *ws, size_t ws_bytes, void *stream) {
    if (!ctx || !mesh || !ws) return PSN_ERR_ARG;
    const SmoothLayout SL = smooth_layout(mesh);
    if (ws_bytes < SL.total) return fail(ctx, PSN_ERR_ARG, "smoothing workspace too small");
    TbSched h;
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    if (cudaMemcpyAsync(&h, static_cast<const char *>(ws) + SL.sch, sizeof(h), cudaMemcpyDeviceToHost, st) != cudaSuccess ||
        cudaStreamSynchronize(st) != cudaSuccess)
        return cuda_check(ctx, "smooth status read-back");
    if (h.error) return fail(ctx, PSN_ERR_CUDA, "wavefront smoothing: a dependency wait timed out");
    return PSN_OK;
}

psn_status psn_ctx_set_constraint(psn_ctx *ctx, int shape) {
    if (!ctx || (shape != PSN_CONSTRAINT_BOX && shape != PSN_CONSTRAINT_SPHERE)) return PSN_ERR_ARG;
    ctx->constraint = shape;
    return PSN_OK;
}

psn_status psn_ctx_set_emission(psn_ctx *ctx, int mode) {
    if (!ctx || (mode != PSN_EMIT_AUTO && mode != PSN_EMIT_SCAN)) return PSN_ERR_ARG;
    ctx->emit_mode = mode;
    return PSN_OK;
}

psn_status psn_ctx_set_counting(psn_ctx *ctx, int mode) {
    if (!ctx || (mode != PSN_COUNT_AUTO && mode != PSN_COUNT_XTILE)) return PSN_ERR_ARG;
    ctx->count_mode = mode;
    return PSN_OK;
}

psn_status psn_ctx_set_smoothing(psn_ctx *ctx, int mode, int32_t iterations_per_launch, int32_t points_per_tile) {
    if (!ctx || (mode != PSN_SMOOTH_WAVEFRONT && mode != PSN_SMOOTH_PER_ITERATION) || iterations_per_launch < 0 ||
        points_per_tile < 0 || points_per_tile % (int32_t)kTbTileMin != 0)
        return PSN_ERR_ARG;
    ctx->smooth_mode = mode;
    ctx->smooth_group = iterations_per_launch;
    ctx->smooth_tile = points_per_tile;
    return PSN_OK;
}

psn_status psn_smooth_step(psn_ctx *ctx, const psn_volume *vol, const psn_mesh *mesh, const void *ws, size_t ws_bytes,
                           const float *src, float *dst, float relaxation, float constraint_distance, void *stream) {
    if (!ctx) return PSN_ERR_ARG;
    ctx->launches = 0;
    psn_status s = check_smooth_args(ctx, mesh, relaxation, constraint_distance);
    if (s != PSN_OK) return s;
    if (!dst || !vol) return fail(ctx, PSN_ERR_ARG, "dst / volume is NULL");
    if (!ws || ws_bytes < smooth_layout(mesh).buf0) return fail(ctx, PSN_ERR_ARG, "smoothing workspace too small");
    if ((reinterpret_cast<uintptr_t>(src) | reinterpret_cast<uintptr_t>(dst)) & 15u)
        return fail(ctx, PSN_ERR_ARG, "offset buffers must be 16-byte aligned (float4 entries)");
    if (mesh->n_points == 0) return PSN_OK;
    if (cudaSetDevice(ctx->device) != cudaSuccess) return cuda_check(ctx, "cudaSetDevice");
    SmoothV4 v = smooth_v4_args(ctx, vol, mesh, ws, relaxation, constraint_distance);
    v.src = reinterpret_cast<const float4 *>(src); v.dst = reinterpret_cast<float4 *>(dst); v.world = nullptr;
    const bool packed = smooth_packed(ctx, vol);   // the form psn_smooth_prepare built for this volume
    const V4Fn kern = pick_v4(packed, packed && mesh->n_points < (1ll << 26), false,
                              ctx->constraint == PSN_CONSTRAINT_SPHERE);
    kern<<<(unsigned)v4_grid(ctx, kern, mesh->n_points), 256, 0, static_cast<cudaStream_t>(stream)>>>(v);
    ++ctx->launches;
    return cuda_check(ctx, "smooth step launch");
}

namespace {
// split: 0 = k_smooth_v4 with the 8-byte cache, 1 = the same writing the split cache (first step of a run;
// hi -> its hi words), 2 = k_smooth_split reading it (later steps of the same psn_smooth_run_peer)
psn_status step_peer_impl(psn_ctx *ctx, const psn_volume *vol, const psn_mesh *mesh, const void *ws, size_t ws_bytes,
                          const float *src, float *dst, int parity, float relaxation, float constraint_distance,
                          psn_peer *peer, void *stream, int split, uint32_t *hi) {
    if (!ctx) return PSN_ERR_ARG;
    ctx->launches = 0;
    psn_status s = check_smooth_args(ctx, mesh, relaxation, constraint_distance);
    if (s != PSN_OK) return s;
    if (!dst || !vol || !peer || !peer->sig || !peer->ctr || !peer->err)
        return fail(ctx, PSN_ERR_ARG, "dst / volume / peer descriptor is NULL");
    if (parity != 0 && parity != 1) return fail(ctx, PSN_ERR_ARG, "parity must be 0 or 1");
    if (!ws || ws_bytes < smooth_layout(mesh).buf0) return fail(ctx, PSN_ERR_ARG, "smoothing workspace too small");
    if ((reinterpret_cast<uintptr_t>(src) | reinterpret_cast<uintptr_t>(dst)) & 15u)
        return fail(ctx, PSN_ERR_ARG, "offset buffers must be 16-byte aligned (float4 entries)");
    const int64_t own0 = mesh->halo_lo_points, own1 = own0 + mesh->n_points;
    SmoothV4 v = smooth_v4_args(ctx, vol, mesh, ws, relaxation, constraint_distance);
    v.src = reinterpret_cast<const float4 *>(src); v.dst = reinterpret_cast<float4 *>(dst); v.world = nullptr;
    for (int k = 0; k < 2; ++k) {
        const psn_peer_side &ps = peer->side[k];
        PeerSide &o = v.peer.side[k];
        if (!ps.dst[0]) continue;
        // an empty push range (a rank that only receives on this side, e.g. its first own layer holds no
        // points) may carry any indices; only a non-empty range must lie inside the own entries
        if (!ps.dst[1] || !ps.peer_sig || ps.src_begin > ps.src_end ||
            (ps.src_end > ps.src_begin && (ps.src_begin < own0 || ps.src_end > own1)) ||
            ps.dst_begin < 0 || ((reinterpret_cast<uintptr_t>(ps.dst[parity])) & 15u))
            return fail(ctx, PSN_ERR_ARG, "peer side %d: bad buffers or push range", k);
        o.dst = reinterpret_cast<float4 *>(ps.dst[parity]);
        o.src_begin = (uint32_t)ps.src_begin; o.src_end = (uint32_t)ps.src_end; o.dst_begin = (uint32_t)ps.dst_begin;
        o.peer_sig = ps.peer_sig;
    }
    if (cudaSetDevice(ctx->device) != cudaSuccess) return cuda_check(ctx, "cudaSetDevice");
    const bool sph = ctx->constraint == PSN_CONSTRAINT_SPHERE;
    const V4Fn kern = split == 2 ? (sph ? k_smooth_split<false, true, true> : k_smooth_split<false, false, true>)
                                 : pick_v4(smooth_packed(ctx, vol), false, true, sph);
    if (split == 1) v.hi_out = hi;
    if (split == 2) v.hi = hi;
    const int64_t g4 = v4_grid(ctx, kern, mesh->n_points);
    v.peer.sig = peer->sig; v.peer.ctr = reinterpret_cast<unsigned long long *>(peer->ctr); v.peer.err = peer->err;
    v.peer.ctr_last = (unsigned long long)(peer->ctr_base + (uint64_t)g4 - 1);
    v.peer.g = peer->iteration;
    kern<<<(unsigned)g4, 256, 0, static_cast<cudaStream_t>(stream)>>>(v);
    ++ctx->launches;
    if ((s = cuda_check(ctx, "smooth step (peer) launch")) != PSN_OK) return s;
    peer->ctr_base += (uint64_t)g4;
    peer->iteration += 1;
    return PSN_OK;
}
}  // namespace

psn_status psn_smooth_step_peer(psn_ctx *ctx, const psn_volume *vol, const psn_mesh *mesh, const void *ws,
                                size_t ws_bytes, const float *src, float *dst, int parity, float relaxation,
                                float constraint_distance, psn_peer *peer, void *stream) {
    // test hook (PSN_PEER_STEP_SPLIT): step with the split cache as psn_smooth_run_peer does (src = NULL writes
    // it, later steps read it), so single-process tests can interleave emulated ranks step by step
    int split = 0;
    uint32_t *hi = nullptr;
    if (getenv("PSN_PEER_STEP_SPLIT") && mesh && vol && smooth_packed(ctx, vol) && mesh->n_points > 0) {
        const size_t hi_at = align_up(8 * (size_t)mesh->n_points);
        if (hi_at + 4 * (size_t)mesh->n_points <= smooth_layout(mesh).buf0) {
            split = src ? 2 : 1;
            hi = reinterpret_cast<uint32_t *>(static_cast<char *>(const_cast<void *>(ws)) + hi_at);
        }
    }
    return step_peer_impl(ctx, vol, mesh, ws, ws_bytes, src, dst, parity, relaxation, constraint_distance, peer, stream,
                          split, hi);
}

psn_status psn_smooth_run_peer(psn_ctx *ctx, const psn_volume *vol, const psn_mesh *mesh, const void *ws,
                               size_t ws_bytes, float *buf0, float *buf1, int32_t iterations, float relaxation,
                               float constraint_distance, psn_peer *peer, void *stream) {
    if (!ctx) return PSN_ERR_ARG;
    if (iterations < 0) return fail(ctx, PSN_ERR_ARG, "iterations must be >= 0");
    if (!peer) return fail(ctx, PSN_ERR_ARG, "peer descriptor is NULL");
    int64_t launches = 0;
    float *buf[2] = {buf0, buf1};
    // buffer parity continues from the global iteration (not from 0 per call): the first step of a later
    // run then writes the buffer the neighbour's previous run did NOT end in (the one its finalize reads)
    const uint64_t g0 = peer->iteration;
    // split smoothing cache (as psn_smooth): the run's first step writes it, the later steps read it; its hi
    // words live in the second half of the cache region (the packed cache uses 8 of its 16 bytes per point)
    const int64_t n = mesh ? mesh->n_points : 0;
    const size_t hi_at = align_up(8 * (size_t)std::max<int64_t>(n, 0));
    const bool split = mesh && vol && smooth_packed(ctx, vol) && iterations > 1 && n > 0 &&
                       hi_at + 4 * (size_t)n <= smooth_layout(mesh).buf0 && !getenv("PSN_SMOOTH_NOSPLIT");
    uint32_t *hi = split ? reinterpret_cast<uint32_t *>(static_cast<char *>(const_cast<void *>(ws)) + hi_at) : nullptr;
    for (int32_t t = 0; t < iterations; ++t) {
        const int par = (int)((g0 + (uint64_t)t) & 1u);
        const psn_status s = step_peer_impl(ctx, vol, mesh, ws, ws_bytes, t ? buf[par ^ 1] : nullptr, buf[par], par,
                                            relaxation, constraint_distance, peer, stream, split ? (t ? 2 : 1) : 0, hi);
        if (s != PSN_OK) return s;
        launches += ctx->launches;
    }
    ctx->launches = launches;
    return PSN_OK;
}

psn_status psn_ipc_export(psn_ctx *ctx, const void *dev_ptr, psn_ipc_handle *out) {
    if (!ctx) return PSN_ERR_ARG;
    if (!dev_ptr || !out) return fail(ctx, PSN_ERR_ARG, "NULL argument");
    if (cudaSetDevice(ctx->device) != cudaSuccess) return cuda_check(ctx, "cudaSetDevice");
    // base of the cudaMalloc allocation holding dev_ptr (driver entry point, no libcuda link)
    typedef int (*GetRange)(unsigned long long *, size_t *, unsigned long long);
    static GetRange get_range = nullptr;
    if (!get_range) {
        void *fn = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuMemGetAddressRange", &fn, cudaEnableDefault, &q) != cudaSuccess || !fn)
            return fail(ctx, PSN_ERR_CUDA, "cuMemGetAddressRange entry point unavailable");
        get_range = reinterpret_cast<GetRange>(fn);
    }
    unsigned long long base = 0;
    size_t size = 0;
    if (get_range(&base, &size, (unsigned long long)(uintptr_t)dev_ptr) != 0)
        return fail(ctx, PSN_ERR_CUDA, "cuMemGetAddressRange failed");
    cudaIpcMemHandle_t h;
    if (cudaIpcGetMemHandle(&h, reinterpret_cast<void *>((uintptr_t)base)) != cudaSuccess)
        return cuda_check(ctx, "cudaIpcGetMemHandle");
    static_assert(sizeof(h) <= sizeof(out->handle), "IPC handle size");
    memset(out, 0, sizeof(*out));
    memcpy(out->handle, &h, sizeof(h));
    out->offset = (uint64_t)((uintptr_t)dev_ptr - (uintptr_t)base);
    return PSN_OK;
}

psn_status psn_ipc_open(psn_ctx *ctx, const psn_ipc_handle *hh, void **dev_ptr) {
    if (!ctx) return PSN_ERR_ARG;
    if (!hh || !dev_ptr) return fail(ctx, PSN_ERR_ARG, "NULL argument");
    if (cudaSetDevice(ctx->device) != cudaSuccess) return cuda_check(ctx, "cudaSetDevice");
    cudaIpcMemHandle_t h;
    memcpy(&h, hh->handle, sizeof(h));
    void *base = nullptr;
    if (cudaIpcOpenMemHandle(&base, h, cudaIpcMemLazyEnablePeerAccess) != cudaSuccess)
        return cuda_check(ctx, "cudaIpcOpenMemHandle");
    *dev_ptr = static_cast<char *>(base) + hh->offset;
    ctx->ipc_bases[*dev_ptr] = base;
    return PSN_OK;
}

psn_status psn_ipc_close(psn_ctx *ctx, void *dev_ptr) {
    if (!ctx) return PSN_ERR_ARG;
    auto it = ctx->ipc_bases.find(dev_ptr);
    if (it == ctx->ipc_bases.end()) return fail(ctx, PSN_ERR_ARG, "pointer was not opened by psn_ipc_open");
    if (cudaSetDevice(ctx->device) != cudaSuccess) return cuda_check(ctx, "cudaSetDevice");
    const cudaError_t e = cudaIpcCloseMemHandle(it->second);
    ctx->ipc_bases.erase(it);
    return e == cudaSuccess ? PSN_OK : cuda_check(ctx, "cudaIpcCloseMemHandle");
}

psn_status psn_smooth_finalize(psn_ctx *ctx, const psn_volume *vol, const psn_mesh *mesh, const float *offsets,
                               int64_t w0, int64_t w1, float *out, void *stream) {
    if (!ctx) return PSN_ERR_ARG;
    ctx->launches = 0;
    if (!vol || !mesh || !out || !mesh->points) return fail(ctx, PSN_ERR_ARG, "NULL argument");
    const int64_t nw = mesh->halo_lo_points + mesh->n_points + mesh->halo_hi_points;
    if (w0 < 0 || w1 > nw || w0 > w1) return fail(ctx, PSN_ERR_ARG, "window range out of bounds");
    if (w0 == w1) return PSN_OK;
    if (reinterpret_cast<uintptr_t>(offsets) & 15u) return fail(ctx, PSN_ERR_ARG, "offsets must be 16-byte aligned");
    if (cudaSetDevice(ctx->device) != cudaSuccess) return cuda_check(ctx, "cudaSetDevice");
    k_finalize<<<(unsigned)grid_for(ctx, w1 - w0), 256, 0, static_cast<cudaStream_t>(stream)>>>(
        reinterpret_cast<const float4 *>(offsets), mesh->points, out, w0, w1, vol->spacing[0], vol->spacing[1], vol->spacing[2], vol->origin[0],
        vol->origin[1], vol->origin[2]);
    ++ctx->launches;
    return cuda_check(ctx, "finalize launch");
}

psn_status psn_triangulate(psn_ctx *ctx, const psn_mesh *mesh, const float *points, psn_tri tri, uint32_t *tris,
                           void *stream) {
    if (!ctx) return PSN_ERR_ARG;
    ctx->launches = 0;
    if (!mesh || !tris || (mesh->n_quads > 0 && (!mesh->quads || !points)))
        return fail(ctx, PSN_ERR_ARG, "NULL argument");
    if (tri < PSN_TRI_FIXED_02 || tri > PSN_TRI_MOST_COPLANAR) return fail(ctx, PSN_ERR_ARG, "unknown triangulation");
    if ((reinterpret_cast<uintptr_t>(mesh->quads) & 15u) || (reinterpret_cast<uintptr_t>(tris) & 7u))
        return fail(ctx, PSN_ERR_ARG, "quads must be 16-byte and tris 8-byte aligned");
    if (mesh->n_quads == 0) return PSN_OK;
    if (cudaSetDevice(ctx->device) != cudaSuccess) return cuda_check(ctx, "cudaSetDevice");
    k_triangulate<<<(unsigned)grid_for(ctx, mesh->n_quads), 256, 0, static_cast<cudaStream_t>(stream)>>>(
        mesh->quads, points, tris, mesh->n_quads, (uint32_t)(mesh->first_point - mesh->halo_lo_points),
        (int)tri);
    ++ctx->launches;
    return cuda_check(ctx, "triangulate launch");
}


// ---------------------------------------------------------------- sub-volume blocks + stitching (NEXT-4)
namespace {
psn_status check_block(psn_ctx *ctx, const psn_block *b, bool need_box) {
    if (!b) return fail(ctx, PSN_ERR_ARG, "block is NULL");
    for (int a = 0; a < 3; ++a) {
        if (b->dims[a] < 2 || b->dims[a] > (1ll << 23)) return fail(ctx, PSN_ERR_ARG, "block dims out of range");
        if (b->own_lo[a] < 0 || b->own_hi[a] > b->dims[a] - 1 || b->own_lo[a] >= b->own_hi[a])
            return fail(ctx, PSN_ERR_ARG, "own box must be non-empty inside [0, dims-1)");
        if (need_box && (b->box_lo[a] < 0 || b->box_lo[a] > std::max<int64_t>(b->own_lo[a] - 1, 0) ||
                         b->box_hi[a] > b->dims[a] || b->box_hi[a] < std::min<int64_t>(b->own_hi[a] + 2, b->dims[a])))
            return fail(ctx, PSN_ERR_ARG, "box must contain the own box plus the one-voxel margin (psn_block_box)");
    }
    if (b->nxseg < 1 || b->xseg < 0 || b->xseg >= b->nxseg) return fail(ctx, PSN_ERR_ARG, "bad x-block index");
    if ((b->own_lo[0] > 0) != (b->xseg > 0) || (b->own_hi[0] < b->dims[0] - 1) != (b->xseg < b->nxseg - 1))
        return fail(ctx, PSN_ERR_ARG, "x-block index inconsistent with the own box");
    return PSN_OK;
}
int64_t block_rows(const psn_block *b) {
    return (b->box_hi[1] - b->box_lo[1] - 1) * (b->box_hi[2] - b->box_lo[2] - 1);
}
size_t stitch_ws_bytes(const psn_block *b) { return 4 * align_up(4 * (size_t)block_rows(b)); }

psn_status stitch_args(psn_ctx *ctx, const psn_block *b, const psn_mesh *local, void *ws, size_t ws_bytes,
                       StitchArgs *a) {
    psn_status s = check_block(ctx, b, true);
    if (s != PSN_OK) return s;
    if (!local || (local->n_points > 0 && (!local->points || !local->stencil_offsets || !local->face_masks ||
                                           (local->n_stencil > 0 && !local->stencil_ids))) ||
        (local->n_quads > 0 && (!local->quads || !local->pairs)) || !local->stencil_offsets)
        return fail(ctx, PSN_ERR_ARG, "local mesh arrays missing");
    if (local->halo_lo_points || local->halo_hi_points || local->first_point || local->first_stencil)
        return fail(ctx, PSN_ERR_ARG, "local mesh must be a standalone extraction (no halos, first ids 0)");
    if (!ws || ws_bytes < stitch_ws_bytes(b)) return fail(ctx, PSN_ERR_ARG, "stitch workspace too small");
    if ((reinterpret_cast<uintptr_t>(local->quads) & 15u) || (reinterpret_cast<uintptr_t>(local->pairs) & 7u))
        return fail(ctx, PSN_ERR_ARG, "quads must be 16-byte and pairs 8-byte aligned");
    *a = StitchArgs{};
    a->lpts = local->points; a->lquads = local->quads; a->lpairs = local->pairs;
    a->lcsr = local->stencil_offsets; a->lids = local->stencil_ids; a->lfm = local->face_masks;
    a->nP = local->n_points; a->nQ = local->n_quads;
    a->bM = (int32_t)(b->box_hi[0] - b->box_lo[0]); a->bN = (int32_t)(b->box_hi[1] - b->box_lo[1]);
    a->bO = (int32_t)(b->box_hi[2] - b->box_lo[2]);
    for (int d = 0; d < 3; ++d) {
        a->lo[d] = (int32_t)b->box_lo[d]; a->own_lo[d] = (int32_t)b->own_lo[d]; a->own_hi[d] = (int32_t)b->own_hi[d];
    }
    a->N = b->dims[1]; a->xseg = (int32_t)b->xseg; a->nxseg = (int32_t)b->nxseg;
    const size_t tb = align_up(4 * (size_t)block_rows(b));
    a->pfirst = at<uint32_t>(ws, 0); a->plast = at<uint32_t>(ws, tb);
    a->qfirst = at<uint32_t>(ws, 2 * tb); a->qlast = at<uint32_t>(ws, 3 * tb);
    return PSN_OK;
}
}  // namespace

psn_status psn_block_box(psn_block *blk, int elem_bytes) {
    psn_status s = check_block(nullptr, blk, false);
    if (s != PSN_OK) return s;
    if (elem_bytes != 0 && elem_bytes != 1 && elem_bytes != 2 && elem_bytes != 4) return PSN_ERR_ARG;
    for (int a = 0; a < 3; ++a) {
        blk->box_lo[a] = std::max<int64_t>(blk->own_lo[a] - 1, 0);
        blk->box_hi[a] = std::min<int64_t>(blk->own_hi[a] + 2, blk->dims[a]);
    }
    if (elem_bytes) {   // widen x (inside the volume) to rows of a multiple of 16 bytes: TMA-staged rows
        const int64_t q = 16 / elem_bytes;
        int64_t w = blk->box_hi[0] - blk->box_lo[0];
        const int64_t want = (w + q - 1) / q * q;
        if (want <= blk->dims[0]) {
            const int64_t grow_hi = std::min(want - w, blk->dims[0] - blk->box_hi[0]);
            blk->box_hi[0] += grow_hi;
            blk->box_lo[0] -= want - w - grow_hi;
        }
    }
    return PSN_OK;
}

psn_status psn_block_gather(psn_ctx *ctx, const void *src, psn_dtype dtype, const psn_block *blk, void *dst,
                            void *stream) {
    if (!ctx) return PSN_ERR_ARG;
    ctx->launches = 0;
    if (!src || !dst || !blk) return fail(ctx, PSN_ERR_ARG, "NULL argument");
    if (dtype != PSN_U8 && dtype != PSN_U16 && dtype != PSN_U32) return fail(ctx, PSN_ERR_ARG, "bad dtype");
    for (int a = 0; a < 3; ++a)
        if (blk->box_lo[a] < 0 || blk->box_hi[a] > blk->dims[a] || blk->box_lo[a] >= blk->box_hi[a])
            return fail(ctx, PSN_ERR_ARG, "box outside the volume");
    if (cudaSetDevice(ctx->device) != cudaSuccess) return cuda_check(ctx, "cudaSetDevice");
    const size_t b = (size_t)dtype;
    cudaMemcpy3DParms p{};
    p.srcPtr = make_cudaPitchedPtr(const_cast<void *>(src), (size_t)blk->dims[0] * b, (size_t)blk->dims[0],
                                   (size_t)blk->dims[1]);
    p.srcPos = make_cudaPos((size_t)blk->box_lo[0] * b, (size_t)blk->box_lo[1], (size_t)blk->box_lo[2]);
    const size_t bm = (size_t)(blk->box_hi[0] - blk->box_lo[0]);
    p.dstPtr = make_cudaPitchedPtr(dst, bm * b, bm, (size_t)(blk->box_hi[1] - blk->box_lo[1]));
    p.extent = make_cudaExtent(bm * b, (size_t)(blk->box_hi[1] - blk->box_lo[1]),
                               (size_t)(blk->box_hi[2] - blk->box_lo[2]));
    p.kind = cudaMemcpyDefault;
    if (cudaMemcpy3DAsync(&p, static_cast<cudaStream_t>(stream)) != cudaSuccess)
        return cuda_check(ctx, "cudaMemcpy3DAsync");
    return PSN_OK;
}

psn_status psn_stitch_workspace(const psn_block *blk, size_t *bytes) {
    if (!blk || !bytes) return PSN_ERR_ARG;
    psn_status s = check_block(nullptr, blk, true);
    if (s != PSN_OK) return s;
    *bytes = stitch_ws_bytes(blk);
    return PSN_OK;
}

psn_status psn_stitch_count(psn_ctx *ctx, const psn_block *blk, const psn_mesh *local, void *ws, size_t ws_bytes,
                            uint32_t *seg, void *stream) {
    if (!ctx) return PSN_ERR_ARG;
    ctx->launches = 0;
    StitchArgs a;
    psn_status s = stitch_args(ctx, blk, local, ws, ws_bytes, &a);
    if (s != PSN_OK) return s;
    if (cudaSetDevice(ctx->device) != cudaSuccess) return cuda_check(ctx, "cudaSetDevice");
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    if (cudaMemsetAsync(ws, 0xFF, stitch_ws_bytes(blk), st) != cudaSuccess) return cuda_check(ctx, "memset");
    if (a.nP > 0) { k_stitch_mark_points<<<(unsigned)grid_for(ctx, a.nP), 256, 0, st>>>(a); ++ctx->launches; }
    if (a.nQ > 0) { k_stitch_mark_quads<<<(unsigned)grid_for(ctx, a.nQ), 256, 0, st>>>(a); ++ctx->launches; }
    if (seg) {
        const int64_t nseg = (blk->dims[1] - 1) * (blk->dims[2] - 1) * blk->nxseg;
        a.segP = seg; a.segQ = seg + nseg; a.segS = seg + 2 * nseg;
        const int64_t rows = (blk->own_hi[1] - blk->own_lo[1]) * (blk->own_hi[2] - blk->own_lo[2]);
        k_stitch_segments<<<(unsigned)grid_for(ctx, rows), 256, 0, st>>>(a);
        ++ctx->launches;
    }
    return cuda_check(ctx, "stitch count launch");
}

size_t psn_stitch_scan_workspace(int64_t nseg) {
    const int64_t nt = std::max<int64_t>(1, (nseg + kSegTile - 1) / kSegTile);
    return 3 * (size_t)nt * sizeof(unsigned long long);
}

psn_status psn_stitch_scan(psn_ctx *ctx, int64_t nseg, const uint32_t *seg, uint32_t *off, int64_t *totals,
                           void *scratch, size_t scratch_bytes, int64_t *host_totals, void *stream) {
    if (!ctx) return PSN_ERR_ARG;
    ctx->launches = 0;
    if (nseg < 1 || nseg > (int64_t)1 << 40 || !seg || !off || !totals)
        return fail(ctx, PSN_ERR_ARG, "bad segment arrays");
    if (!scratch || scratch_bytes < psn_stitch_scan_workspace(nseg)) return fail(ctx, PSN_ERR_ARG, "scratch too small");
    const int64_t nt = (nseg + kSegTile - 1) / kSegTile;
    if (nt > 65535ll * 1024) return fail(ctx, PSN_ERR_ARG, "too many segments");
    if (cudaSetDevice(ctx->device) != cudaSuccess) return cuda_check(ctx, "cudaSetDevice");
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    auto *ts = static_cast<unsigned long long *>(scratch);
    k_seg_tile_sums<<<dim3((unsigned)nt, 3), kSegThreads, 0, st>>>(seg, nseg, ts);
    k_seg_scan<<<dim3((unsigned)nt, 3), kSegThreads, 0, st>>>(seg, off, nseg, ts, nt, totals);
    ctx->launches += 2;
    psn_status s = cuda_check(ctx, "stitch scan launch");
    if (s != PSN_OK || !host_totals) return s;
    if (cudaMemcpyAsync(host_totals, totals, 3 * sizeof(int64_t), cudaMemcpyDeviceToHost, st) != cudaSuccess ||
        cudaStreamSynchronize(st) != cudaSuccess)
        return cuda_check(ctx, "totals read-back");
    for (int a = 0; a < 3; ++a)
        if (host_totals[a] >= ((int64_t)1 << 32)) return fail(ctx, PSN_ERR_OVERFLOW, "stitched total reaches 2^32");
    return PSN_OK;
}

psn_status psn_stitch_emit(psn_ctx *ctx, const psn_block *blk, const psn_volume *vol, const psn_mesh *local,
                           const void *ws, size_t ws_bytes, const uint32_t *off, const int64_t *totals,
                           psn_mesh *global, void *stream) {
    if (!ctx) return PSN_ERR_ARG;
    ctx->launches = 0;
    StitchArgs a;
    psn_status s = stitch_args(ctx, blk, local, const_cast<void *>(ws), ws_bytes, &a);
    if (s != PSN_OK) return s;
    if (!vol || !off || !totals || !global) return fail(ctx, PSN_ERR_ARG, "NULL argument");
    for (int d = 0; d < 3; ++d)
        if (vol->dims[d] != blk->dims[d]) return fail(ctx, PSN_ERR_ARG, "volume dims differ from the block's");
    if (!global->points || !global->stencil_offsets || !global->face_masks || !global->stencil_ids ||
        !global->quads || !global->pairs)
        return fail(ctx, PSN_ERR_ARG, "global mesh arrays missing");
    if ((reinterpret_cast<uintptr_t>(global->quads) & 15u) || (reinterpret_cast<uintptr_t>(global->pairs) & 7u))
        return fail(ctx, PSN_ERR_ARG, "quads must be 16-byte and pairs 8-byte aligned");
    const int64_t nseg = (blk->dims[1] - 1) * (blk->dims[2] - 1) * blk->nxseg;
    a.offP = off; a.offQ = off + nseg; a.offS = off + 2 * nseg;
    a.points = global->points; a.quads = global->quads; a.pairs = global->pairs;
    a.csr = global->stencil_offsets; a.ids = global->stencil_ids; a.fm = global->face_masks;
    a.totals = totals;
    for (int d = 0; d < 3; ++d) { a.org[d] = vol->origin[d]; a.sp[d] = vol->spacing[d]; }
    if (cudaSetDevice(ctx->device) != cudaSuccess) return cuda_check(ctx, "cudaSetDevice");
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    k_stitch_points<<<(unsigned)grid_for(ctx, std::max<int64_t>(a.nP, 1)), 256, 0, st>>>(a);
    ++ctx->launches;
    if (a.nQ > 0) { k_stitch_quads<<<(unsigned)grid_for(ctx, a.nQ), 256, 0, st>>>(a); ++ctx->launches; }
    return cuda_check(ctx, "stitch emit launch");
}

}  // extern "C"
