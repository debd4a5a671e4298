// membench.cu -- read-bandwidth probes for the counting kernel's staging design
// (B200, sm_100a).  Not part of the library.
//
//   nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -o tools/membench tools/membench.cu
//   tools/membench [GiB]
//
// (a) plain vectorised LDG.128 read (grid-stride, XOR-reduced)
// (b) TMA bulk ring: CTA = R rows x RB bytes per stage, NS stages, one producer
//     warp issuing cp.async.bulk per row, consumers (W warps) only wait/release.
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <cuda_runtime.h>

__global__ void k_ldg(const uint4 *p, size_t n, uint32_t *out) {
    uint32_t acc = 0;
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
        uint4 v = __ldg(p + i);
        acc ^= v.x ^ v.y ^ v.z ^ v.w;
    }
    if (acc == 0x12345678u) out[0] = acc;
}

__device__ __forceinline__ uint32_t smem_u32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t *b, uint32_t c) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(c) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t *b, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t *b) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(b)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t *b, uint32_t par) {
    asm volatile("{\n\t.reg .pred p;\nW_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t@!p bra W_%=;\n}" ::"r"(
                     smem_u32(b)), "r"(par) : "memory");
}
__device__ __forceinline__ void tma1d(void *dst, const void *src, uint32_t bytes, uint64_t *bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     smem_u32(dst)), "l"(src), "r"(bytes), "r"(smem_u32(bar)) : "memory");
}

// rows of `rowbytes`, CTA handles R consecutive rows per stage; stage s = slice s of its column
__global__ void k_tma(const uint8_t *p, int64_t rows_per_slice, int64_t slices, int R, int NS, uint32_t rowbytes,
                      int64_t KZ, int W) {
    extern __shared__ __align__(128) uint8_t dsm[];
    __shared__ __align__(8) uint64_t full[16], empty[16];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int64_t nJB = (rows_per_slice + R - 1) / R;
    const int64_t jb = blockIdx.x % nJB, zc = blockIdx.x / nJB;
    const int64_t k0 = zc * KZ, k1 = min(k0 + KZ, slices);
    const int64_t n = k1 - k0;
    if (threadIdx.x == 0) {
        for (int s = 0; s < NS; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], W); }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    const uint32_t SB = R * rowbytes;
    if (warp == W) {
        for (int64_t s = 0; s < n; ++s) {
            const int slot = (int)(s % NS);
            if (s >= NS) mbar_wait(&empty[slot], (uint32_t)(((s / NS) - 1) & 1));
            if (lane == 0) mbar_expect_tx(&full[slot], rowbytes * R);
            __syncwarp();
            for (int g = lane; g < R; g += 32) {
                const int64_t j = min(jb * R + g, rows_per_slice - 1);
                tma1d(dsm + slot * SB + g * rowbytes, p + ((k0 + s) * rows_per_slice + j) * rowbytes, rowbytes, &full[slot]);
            }
        }
        return;
    }
    for (int64_t s = 0; s < n; ++s) {
        mbar_wait(&full[s % NS], (uint32_t)((s / NS) & 1));
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[s % NS]);
    }
}

int main(int argc, char **argv) {
    double gib = argc > 1 ? atof(argv[1]) : 2.0;
    size_t bytes = (size_t)(gib * (1ull << 30));
    uint8_t *p;
    uint32_t *out;
    cudaMalloc(&p, bytes);
    cudaMalloc(&out, 4);
    cudaMemset(p, 1, bytes);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    for (int bl : {2, 4, 8}) {
        float best = 1e9;
        for (int r = 0; r < 5; ++r) {
            cudaEventRecord(a);
            k_ldg<<<sms * bl, 512>>>((const uint4 *)p, bytes / 16, out);
            cudaEventRecord(b);
            cudaEventSynchronize(b);
            float ms;
            cudaEventElapsedTime(&ms, a, b);
            if (ms < best) best = ms;
        }
        printf("ldg128 blocks/SM=%d: %.3f ms  %.1f GB/s\n", bl, best, bytes / best / 1e6);
    }
    // c4-like: rows of 2048 B, 1024 rows per slice
    struct Cfg { uint32_t rowbytes; int R, NS, W; int64_t KZ; };
    Cfg cfgs[] = {{2048, 9, 4, 4, 56}, {2048, 9, 6, 4, 56}, {2048, 9, 8, 4, 56}, {2048, 17, 4, 8, 56},
                  {2048, 9, 4, 4, 128}, {2048, 9, 4, 4, 16}, {2048, 5, 8, 4, 56}, {512, 9, 4, 4, 17},
                  {512, 9, 8, 4, 32}, {512, 33, 4, 8, 32}};
    for (const Cfg &c : cfgs) {
        const int64_t rows_per_slice = 1024 * 2048 / c.rowbytes;   // 2 MiB slices
        const int64_t slices = bytes / (rows_per_slice * c.rowbytes);
        const int64_t nJB = (rows_per_slice + c.R - 1) / c.R;
        const int64_t nZC = (slices + c.KZ - 1) / c.KZ;
        const size_t smem = (size_t)c.NS * c.R * c.rowbytes;
        cudaFuncSetAttribute(k_tma, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        float best = 1e9;
        for (int r = 0; r < 5; ++r) {
            cudaEventRecord(a);
            k_tma<<<(unsigned)(nJB * nZC), 32 * (c.W + 1), smem>>>(p, rows_per_slice, slices, c.R, c.NS, c.rowbytes, c.KZ, c.W);
            cudaEventRecord(b);
            cudaEventSynchronize(b);
            float ms;
            cudaEventElapsedTime(&ms, a, b);
            if (ms < best) best = ms;
        }
        cudaError_t e = cudaGetLastError();
        int occ = 0;
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_tma, 32 * (c.W + 1), smem);
        printf("tma rowbytes=%u R=%d NS=%d W=%d KZ=%lld smem=%zuKB occ=%d: %.3f ms  %.1f GB/s %s\n", c.rowbytes, c.R, c.NS,
               c.W, (long long)c.KZ, smem / 1024, occ, best, (double)slices * rows_per_slice * c.rowbytes / best / 1e6,
               e == cudaSuccess ? "" : cudaGetErrorString(e));
    }
    return 0;
}
