// tcgen05.mma.kind::mxf4 (block32, UE8M0 = 1.0) on B200: cycles per MMA
// (M=128 x N x K=64) with A from shared memory (SS) or from TMEM (TS), N =
// 16..256; and tcgen05.st.32x32b.x32 + wait::st cost per warp (4 / 8 warps).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I paper_2604_03957_b200/csrc \
//      -o tools/ubench/mxf4_ubench tools/ubench/mxf4_ubench.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include "sm100.cuh"
using namespace bwta::sm100;

__global__ void __launch_bounds__(256, 1) kern(int N, int ts, int iters, long long* out, int nacc) {
    extern __shared__ uint8_t raw[];
    uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(raw) + 1023) & ~uintptr_t(1023));
    uint8_t* sA = sm;             // 128 rows x 128 B
    uint8_t* sB = sm + 16384;     // up to 256 rows x 128 B
    __shared__ uint64_t bar;
    __shared__ uint32_t tslot;
    for (int i = threadIdx.x; i < (16384 + 32768) / 4; i += blockDim.x)
        reinterpret_cast<uint32_t*>(sm)[i] = 0x22222222u * ((i * 7) & 1);
    fence_proxy_async_smem();
    if (threadIdx.x == 0) { mbar_init(&bar, 1); fence_barrier_init(); }
    if (threadIdx.x < 32) tmem_alloc(&tslot, 512);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tb = tslot;
    const int warp = threadIdx.x >> 5;
    const int lane = threadIdx.x & 31;
    if (warp < 4) {  // scale factors (cols 480..495) and A codes (cols 256..287) in TMEM
        uint32_t v[16];
        for (int i = 0; i < 16; ++i) v[i] = 0x7F7F7F7Fu;
        tmem_st_32x32b_x16(tb + (uint32_t(warp * 32) << 16) + 480u, v);
        for (int i = 0; i < 16; ++i) v[i] = 0x22222222u;
        tmem_st_32x32b_x16(tb + (uint32_t(warp * 32) << 16) + 256u, v);
        tmem_st_32x32b_x16(tb + (uint32_t(warp * 32) << 16) + 272u, v);
        tmem_wait_st();
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    if (warp == 0 && nacc == 2) {  // whole warp runs the loop, elect.sync per MMA (CUTLASS style)
        const uint32_t idesc = (1u << 7) | (1u << 10) | (uint32_t(N >> 3) << 17) | (1u << 23) | (uint32_t(128 >> 4) << 24);
        const uint32_t a0 = smem_u32(sA), b0 = smem_u32(sB);
        long long t0 = clock64();
        for (int it = 0; it < iters; ++it)
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                const uint64_t bd = smem_desc_sw128(b0 + 32 * k);
                const uint32_t d = tb + (it & 1) * 64;
                uint32_t pred;
                asm volatile("{\n.reg .pred px;\nelect.sync _|px, 0xffffffff;\nselp.u32 %0, 1, 0, px;\n}" : "=r"(pred));
                if (pred) {
                    if (ts) mma_mxf4_ts(d, tb + 256 + 8 * k, bd, idesc, tb + 480, tb + 488, 1);
                    else mma_mxf4(d, smem_desc_sw128(a0 + 32 * k), bd, idesc, tb + 480, tb + 488, 1);
                }
                __syncwarp();
            }
        if (lane == 0) { tc_commit(&bar); }
        mbar_wait(&bar, 0);
        if (lane == 0) out[blockIdx.x * 4] = clock64() - t0;
    } else if (threadIdx.x == 0 && nacc >= 3) {  // nacc - 2 MMAs then one tcgen05.commit, repeated
        __shared__ uint64_t cb[8];
        for (int i = 0; i < 8; ++i) mbar_init(&cb[i], 1);
        fence_barrier_init();
        const uint32_t idesc = (1u << 7) | (1u << 10) | (uint32_t(N >> 3) << 17) | (1u << 23) | (uint32_t(128 >> 4) << 24);
        const uint32_t b0 = smem_u32(sB);
        const int per = nacc - 2;
        long long t0 = clock64();
        for (int it = 0; it < iters * 4 / per; ++it) {
            for (int k = 0; k < per; ++k)
                mma_mxf4_ts(tb + (it & 1) * 64, tb + 256 + 8 * (k & 3), smem_desc_sw128(b0 + 32 * (k & 3)), idesc, tb + 480, tb + 488, 1);
            tc_commit(&cb[it & 7]);
        }
        tc_commit(&bar);
        mbar_wait(&bar, 0);
        out[blockIdx.x * 4] = clock64() - t0;
    } else if (threadIdx.x == 0 && nacc == 1) {
        const uint32_t idesc = (1u << 7) | (1u << 10) | (uint32_t(N >> 3) << 17) | (1u << 23) | (uint32_t(128 >> 4) << 24);
        const uint32_t a0 = smem_u32(sA), b0 = smem_u32(sB);
        const uint32_t idesc8 = idesc_i8(128, N);
        long long t0 = clock64();
        for (int it = 0; it < iters; ++it)
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                const uint64_t bd = smem_desc_sw128(b0 + 32 * k);
                // nacc independent accumulators (N columns each) taken round-robin by the MMAs
                const uint32_t d = tb + (it & 1) * 64;
                if (ts >= 2) {  // kind::i8, K = 32 per MMA (32 bytes = 8 columns of A)
                    const uint32_t id8 = idesc8;
                    if (ts == 3) mma_i8_ts(d, tb + 256 + 8 * k, bd, id8, 1);
                    else mma_i8(d, smem_desc_sw128(a0 + 32 * k), bd, id8, 1);
                } else if (ts) mma_mxf4_ts(d, tb + 256 + 8 * k, bd, idesc, tb + 480, tb + 488, 1);
                else mma_mxf4(d, smem_desc_sw128(a0 + 32 * k), bd, idesc, tb + 480, tb + 488, 1);
            }
        tc_commit(&bar);
        mbar_wait(&bar, 0);
        out[blockIdx.x * 4] = clock64() - t0;
    }
    __syncthreads();
    // tcgen05.st throughput: every warp stores 32 columns x its 32 lanes, `iters` times
    {
        uint32_t v[32];
        for (int i = 0; i < 32; ++i) v[i] = threadIdx.x * i;
        const int nw = (ts & 1) ? 8 : 4;  // reuse ts to select 8 or 4 storing warps
        __syncthreads();
        long long t0 = clock64();
        if (warp < nw) {
            for (int it = 0; it < iters / 4; ++it) {
                tmem_st_32x32b_x32(tb + (uint32_t((warp & 3) * 32) << 16) + 64u + 32u * ((it + warp / 4) & 3), v);
                tmem_wait_st();
            }
        }
        __syncthreads();
        if (threadIdx.x == 0) out[blockIdx.x * 4 + 1] = clock64() - t0;
        t0 = clock64();
        if (warp < nw) {
            for (int it = 0; it < iters / 4; ++it)
                tmem_st_32x32b_x32(tb + (uint32_t((warp & 3) * 32) << 16) + 64u + 32u * ((it + warp / 4) & 3), v);
            tmem_wait_st();
        }
        __syncthreads();
        if (threadIdx.x == 0) out[blockIdx.x * 4 + 2] = clock64() - t0;
    }
    tc_fence_before();
    __syncthreads();
    if (threadIdx.x < 32) { tc_fence_after(); tmem_dealloc(tb, 512); }
}

int main() {
    long long* o; cudaMalloc(&o, 1024 * 8 * 4);
    long long ho[4];
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
    const int iters = 1000;
    for (int nacc : {1, 3, 4, 6})
    for (int ts = 0; ts <= (nacc >= 2 ? 1 : 3); ++ts)
        for (int n : {16, 32, 64, 128, 256}) {

            kern<<<148, 256, 64 * 1024>>>(n, ts, iters, o, nacc);
            if (cudaDeviceSynchronize() != cudaSuccess) { printf("error %s\n", cudaGetErrorString(cudaGetLastError())); return 1; }
            cudaMemcpy(ho, o, 32, cudaMemcpyDeviceToHost);
            if (nacc >= 3 && ts == 0) continue;
            printf(nacc >= 3 ? "commit every %d MMA: " : "mode %d ", nacc >= 3 ? nacc - 2 : nacc);
            printf("mxf4 %s N=%3d: %6.1f cycles/MMA (%6.0f MAC/clk)   | tcgen05.st.32x32b.x32 by %d warps: %6.1f cyc/st with wait each, %6.1f pipelined\n",
                   ts == 3 ? "i8 TS (A in TMEM)" : ts == 2 ? "i8 SS (A in smem)" : ts ? "TS (A in TMEM)" : "SS (A in smem)", n, double(ho[0]) / (iters * 4),
                   128.0 * n * (ts >= 2 ? 32 : 64) / (double(ho[0]) / (iters * 4)), (ts & 1) ? 8 : 4, double(ho[1]) / (iters / 4),
                   double(ho[2]) / (iters / 4));
        }
    return 0;
}
