// TMA load throughput on B200 for the skinny GEMM's weight stream: 148 CTAs,
// each streams its own [128 rows x K] slab of a row-major uint32 plane
// [N][ld] (K = 8192 -> ld = 256 words = 1 KB per row), through an 8-stage
// ring of 16 KB stages, one producer thread.  Modes:
//   0: 2-D tensor box 32 words x 128 rows (one 128-byte line per row)
//   1: 2-D tensor box 32 words x 32 rows, 4 per stage
//   2: 1-D cp.async.bulk of 128 B per row, 128 per stage (issued by 32 lanes)
//   3: 1-D cp.async.bulk of 16 contiguous rows' full K (16 KB) per stage
//   4: 2-D box 64 words x 64 rows (256 B per row)
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I paper_2604_03957_b200/csrc -lcuda \
//      -o tools/ubench/tma_ubench tools/ubench/tma_ubench.cu
#include <cstdio>
#include <cstdint>
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include "sm100.cuh"
using namespace bwta::sm100;

constexpr int STAGES = 8, STAGE = 16384;

__device__ __forceinline__ void bulk_g2s(uint32_t dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
                 "l"(src), "r"(bytes), "r"(smem_u32(bar))
                 : "memory");
}

__global__ void __launch_bounds__(64, 1) kern(const __grid_constant__ CUtensorMap m0, const __grid_constant__ CUtensorMap m1,
                                              const __grid_constant__ CUtensorMap m4, const __grid_constant__ CUtensorMap m8,
                                              const uint32_t* w, int ld, int mode,
                                              int slabs_per_cta, unsigned long long* out) {
    extern __shared__ __align__(1024) uint8_t raw[];
    uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(raw) + 1023) & ~uintptr_t(1023));
    __shared__ uint64_t full[STAGES], empty[STAGES];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (threadIdx.x == 0) {
        for (int s = 0; s < STAGES; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], 1); }
        fence_barrier_init();
    }
    __syncthreads();
    const int per_slab = 128 * ld * 4 / STAGE;  // stages per 128-row slab
    const int n = per_slab * slabs_per_cta;
    long long t0 = clock64();
    if (warp == 0) {
        for (int i = 0; i < n; ++i) {
            const int s = i % STAGES;
            const uint32_t ph = (i / STAGES) & 1;
            mbar_wait(&empty[s], ph ^ 1);
            const int slab = blockIdx.x * slabs_per_cta + i / per_slab, j = i % per_slab;
            uint8_t* dst = sm + s * STAGE;
            if (lane == 0) mbar_arrive_expect_tx(&full[s], STAGE);
            __syncwarp();
            if (mode == 0) {
                if (lane == 0) tma_load_4d(dst, &m0, &full[s], j * 32, slab * 128, 0, 0);
            } else if (mode == 1) {
                if (lane < 4) tma_load_4d(dst + lane * 4096, &m1, &full[s], j * 32, slab * 128 + lane * 32, 0, 0);
            } else if (mode == 2) {
                for (int r = lane; r < 128; r += 32)
                    bulk_g2s(smem_u32(dst + r * 128), w + size_t(slab * 128 + r) * ld + j * 32, 128, &full[s]);
            } else if (mode == 3) {
                if (lane == 0) bulk_g2s(smem_u32(dst), w + size_t(slab) * 128 * ld + size_t(j) * (STAGE / 4), STAGE, &full[s]);
            } else if (mode == 4) {
                if (lane == 0) tma_load_4d(dst, &m4, &full[s], (j % 4) * 64, slab * 128 + (j / 4) * 64, 0, 0);
            } else {  // mode 5: four 8-word x 128-row boxes (32 B per row, the tile kernel's 256-K slices)
                if (lane < 4) tma_load_4d(dst + lane * 4096, &m8, &full[s], (j * 4 + lane) * 8, slab * 128, 0, 0);
            }
        }
    } else if (lane == 0) {
        for (int i = 0; i < n; ++i) {
            const int s = i % STAGES;
            mbar_wait(&full[s], (i / STAGES) & 1);
            mbar_arrive(&empty[s]);
        }
    }
    __syncthreads();
    if (threadIdx.x == 0) out[blockIdx.x] = clock64() - t0;
}

__global__ void readflush(const uint4* p, size_t n, unsigned* sink) {
    uint4 acc = make_uint4(0, 0, 0, 0);
    for (size_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += size_t(gridDim.x) * blockDim.x) {
        const uint4 v = p[i];
        acc.x ^= v.x; acc.y ^= v.y; acc.z ^= v.z; acc.w ^= v.w;
    }
    if ((acc.x ^ acc.y ^ acc.z ^ acc.w) == 0x12345678u) *sink = 1;
}

int main() {
    const int K = 8192, ld = K / 32, slabs_per_cta = 2, grid = 148, N = 128 * slabs_per_cta * grid;
    uint32_t* w; cudaMalloc(&w, size_t(N) * ld * 4);
    cudaMemset(w, 0x5a, size_t(N) * ld * 4);
    unsigned long long* o; cudaMalloc(&o, 148 * 8);
    uint8_t* fl; cudaMalloc(&fl, 512 << 20);
    PFN_cuTensorMapEncodeTiled_v12000 enc;
    cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&enc, cudaEnableDefault, &q);
    CUtensorMap m[4];
    const uint32_t boxes[4][2] = {{32, 128}, {32, 32}, {64, 64}, {8, 128}};
    for (int i = 0; i < 4; ++i) {
        cuuint64_t d[4] = {cuuint64_t(ld), cuuint64_t(N), 1, 1};
        cuuint64_t st[3] = {cuuint64_t(ld) * 4, cuuint64_t(ld) * 4 * N, cuuint64_t(ld) * 4 * N};
        cuuint32_t b[4] = {boxes[i][0], boxes[i][1], 1, 1}, es[4] = {1, 1, 1, 1};
        CUresult r = enc(&m[i], CU_TENSOR_MAP_DATA_TYPE_UINT32, 4, w, d, st, b, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                         i >= 2 ? CU_TENSOR_MAP_SWIZZLE_NONE : CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                         CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        if (r != CUDA_SUCCESS) { printf("encode %d failed %d\n", i, r); return 1; }
    }
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, STAGES * STAGE + 1024);
    const char* names[6] = {"2D box 32w x 128r", "2D box 32w x 32r x4", "1D bulk 128 B x 128 rows", "1D bulk 16 KB contiguous", "2D box 64w x 64r", "2D box 8w x 128r x4"};
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    for (int carve = 0; carve <= 0; ++carve) {
    // carve = 1: the flush kernel asks for the max shared-memory carveout too,
    // so the SM need not reconfigure L1/smem between the two kernels
    cudaFuncSetAttribute(readflush, cudaFuncAttributePreferredSharedMemoryCarveout, carve ? 100 : -1);
    printf("flush kernel carveout %s\n", carve ? "max shared" : "default");
    for (int g : {1, 8, 148})
    for (int mode = 0; mode < 6; ++mode) {
        if (mode == 2) continue;
        for (int rep = 0; rep < 3; ++rep) {
            if (rep < 2) cudaMemset(fl, rep, 512 << 20);  // (dirty L2) ...
            readflush<<<592, 512>>>(reinterpret_cast<const uint4*>(fl), (512u << 20) / 16, reinterpret_cast<unsigned*>(o));  // ... evicted clean
            cudaEventRecord(e0);
            kern<<<g, 64, STAGES * STAGE + 1024>>>(m[0], m[1], m[2], m[3], w, ld, mode, slabs_per_cta, o);
            cudaEventRecord(e1);
            if (cudaDeviceSynchronize() != cudaSuccess) { printf("error %s\n", cudaGetErrorString(cudaGetLastError())); return 1; }
            float ms; cudaEventElapsedTime(&ms, e0, e1);
            unsigned long long h[148]; cudaMemcpy(h, o, sizeof(h), cudaMemcpyDeviceToHost);
            unsigned long long mx = 0; for (int i = 0; i < g; ++i) mx = h[i] > mx ? h[i] : mx;
            const double bytes = double(N) * ld * 4 * g / grid;
            if (rep == 2) printf("grid %3d %-28s %7.2f us  %6.0f GB/s  (max CTA %llu cycles = %.1f B/clk/SM, %.0f cyc/stage)\n", g, names[mode], ms * 1e3,
                                 bytes / (ms * 1e-3) / 1e9, mx, bytes / g / mx, double(mx) / (bytes / g / STAGE));
        }
    }
    }
    return 0;
}
