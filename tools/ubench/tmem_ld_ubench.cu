// TMEM read bandwidth on B200: W warps per CTA (one CTA per SM) each repeatedly load 32 lanes x
// 32 columns (tcgen05.ld.32x32b.x32, 4 KB per warp) from TMEM, with or without .pack::16b, x16/x32
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I paper_2604_03957_b200/csrc -o /tmp/tmem_ld tools/ubench/tmem_ld_ubench.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include "sm100.cuh"
using namespace bwta::sm100;

__device__ __forceinline__ void ld_x32_pack(uint32_t taddr, uint32_t (&v)[16]) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.pack::16b.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
        : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]), "=r"(v[8]),
          "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
        : "r"(taddr));
}

__global__ void kern(int iters, int mode, long long* out, uint32_t* sink) {
    __shared__ uint32_t tslot;
    const int warp = threadIdx.x >> 5;
    if (warp == 0) tmem_alloc(&tslot, 512);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tb = tslot + (uint32_t((warp & 3) * 32) << 16) + uint32_t((warp >> 2) * 32 % 512);
    uint32_t acc = 0;
    __syncthreads();
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
        if (mode == 0) {
            uint32_t v[32];
            tmem_ld_32x32b_x32(tb, v);
            tmem_wait_ld();
#pragma unroll
            for (int i = 0; i < 32; ++i) acc += v[i];
        } else {
            uint32_t v[16];
            ld_x32_pack(tb, v);
            tmem_wait_ld();
#pragma unroll
            for (int i = 0; i < 16; ++i) acc += v[i];
        }
    }
    __syncthreads();
    long long t1 = clock64();
    if (threadIdx.x == 0) out[blockIdx.x] = t1 - t0;
    if (acc == 0x12345678) sink[0] = acc;
    tc_fence_before();
    __syncthreads();
    if (warp == 0) { tc_fence_after(); tmem_dealloc(tslot, 512); }
}

int main() {
    long long* d; uint32_t* s;
    cudaMalloc(&d, 148 * 8); cudaMalloc(&s, 4);
    for (int mode = 0; mode < 2; ++mode)
        for (int w : {4, 8, 16}) {
            const int iters = 2000;
            kern<<<148, 32 * w>>>(iters, mode, d, s);
            cudaDeviceSynchronize();
            long long h[148];
            cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
            double bytes = double(iters) * w * 4096;  // 32 lanes x 32 columns x 4 B per warp-load
            printf("mode %s warps %2d: %.1f B/clk/SM (TMEM bytes read %s)  err=%s\n", mode ? "pack16" : "x32   ", w,
                   bytes / double(h[0]), mode ? "assumed 4 KB" : "4 KB", cudaGetErrorString(cudaGetLastError()));
        }
    return 0;
}
