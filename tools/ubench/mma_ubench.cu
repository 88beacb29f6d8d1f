// tcgen05.mma.kind::i8 issue rate on B200: cycles per MMA (M x N x K=32)
// for cta_group::1 (M=128) and ::2 (M=256), N = 64..256, operands in smem
// (SW128 K-major), for three operand-value patterns (zeros, x64 BWTA codes,
// random bytes) -- is the rate proportional to N, and data dependent?
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I paper_2604_03957_b200/csrc \
//      -o tools/ubench/mma_ubench tools/ubench/mma_ubench.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include "sm100.cuh"
using namespace bwta::sm100;

template <int CG>
__global__ void __launch_bounds__(128, 1) kern(const uint8_t* src, int N, int iters, long long* out) {
    extern __shared__ uint8_t raw[];
    uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(raw) + 1023) & ~uintptr_t(1023));
    uint8_t* sA = sm;             // 128 rows x 128 B
    uint8_t* sB = sm + 16384;     // up to 256 rows x 128 B
    __shared__ uint64_t bar;
    __shared__ uint32_t tslot;
    const int rank = CG == 2 ? int(cluster_ctarank()) : 0;
    for (int i = threadIdx.x; i < (16384 + 32768) / 16; i += blockDim.x)
        reinterpret_cast<uint4*>(sm)[i] = reinterpret_cast<const uint4*>(src)[i];
    fence_proxy_async_smem();
    if (threadIdx.x == 0) { mbar_init(&bar, 1); fence_barrier_init(); }
    if (threadIdx.x < 32) { if (CG == 1) tmem_alloc(&tslot, 512); else tmem_alloc2(&tslot, 512); }
    tc_fence_before();
    if (CG == 2) cluster_sync(); else __syncthreads();
    tc_fence_after();
    const uint32_t tb = tslot;
    long long t0 = 0, t1 = 0;
    if (rank == 0 && threadIdx.x == 0) {
        const uint32_t idesc = idesc_i8(128 * CG, N);
        const uint32_t a0 = smem_u32(sA), b0 = smem_u32(sB);
        t0 = clock64();
        for (int it = 0; it < iters; ++it)
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                const uint64_t ad = smem_desc_sw128(a0 + 32 * k), bd = smem_desc_sw128(b0 + 32 * k);
                if (CG == 1) mma_i8(tb + (it & 1) * 256, ad, bd, idesc, 1);
                else mma_i8_cg2(tb + (it & 1) * 256, ad, bd, idesc, 1);
            }
        if (CG == 1) tc_commit(&bar); else tc_commit2_mc(&bar, 0x1);
        mbar_wait(&bar, 0);
        t1 = clock64();
        out[blockIdx.x] = (t1 - t0);
    }
    tc_fence_before();
    if (CG == 2) cluster_sync(); else __syncthreads();
    if (threadIdx.x < 32) { tc_fence_after(); if (CG == 1) tmem_dealloc(tb, 512); else tmem_dealloc2(tb, 512); }
}

int main() {
    const int bytes = 16384 + 32768;
    uint8_t* h = new uint8_t[bytes];
    uint8_t* d; cudaMalloc(&d, bytes);
    long long* o; cudaMalloc(&o, 1024 * 8);
    long long ho[1024];
    cudaFuncSetAttribute(kern<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
    cudaFuncSetAttribute(kern<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
    const char* pats[3] = {"zeros", "x64 codes", "random"};
    uint32_t seed = 1;
    for (int pat = 0; pat < 3; ++pat) {
        for (int i = 0; i < bytes; ++i) {
            seed = seed * 1664525u + 1013904223u;
            const uint32_t r = seed >> 24;
            h[i] = pat == 0 ? 0 : pat == 1 ? (r % 3 == 0 ? 0x40 : r % 3 == 1 ? 0xC0 : 0) : uint8_t(r);
        }
        cudaMemcpy(d, h, bytes, cudaMemcpyHostToDevice);
        for (int cg = 1; cg <= 2; ++cg)
            for (int n : {16, 32, 64, 128, 256}) {
                const int iters = 2000;
                for (int grid : {cg, 148}) {
                    cudaLaunchConfig_t cfg = {};
                    cfg.gridDim = dim3(grid); cfg.blockDim = dim3(128); cfg.dynamicSmemBytes = 64 * 1024;
                    cudaLaunchAttribute at[1];
                    at[0].id = cudaLaunchAttributeClusterDimension;
                    at[0].val.clusterDim.x = cg; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
                    cfg.attrs = at; cfg.numAttrs = 1;
                    cudaError_t e = cg == 1 ? cudaLaunchKernelEx(&cfg, kern<1>, (const uint8_t*)d, n, iters, o)
                                            : cudaLaunchKernelEx(&cfg, kern<2>, (const uint8_t*)d, n, iters, o);
                    if (e != cudaSuccess || cudaDeviceSynchronize() != cudaSuccess) {
                        printf("error %s\n", cudaGetErrorString(cudaGetLastError()));
                        return 1;
                    }
                    cudaMemcpy(ho, o, 8, cudaMemcpyDeviceToHost);
                    const double cyc = double(ho[0]) / (iters * 4);
                    const double macs = 128.0 * n * 32;  // per CTA per MMA
                    printf("%-9s cg%d N=%3d grid %3d: %6.1f cycles/MMA  %6.0f MAC/clk/SM\n", pats[pat], cg, n, grid, cyc,
                           macs / cyc);
                }
            }
    }
    return 0;
}
