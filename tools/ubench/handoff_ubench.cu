// mbarrier hand-off latency on B200: warp 0 signals barrier X (plain arrive, or tcgen05.commit with
// no MMA in flight, or a commit after one 128x128x64 mxf4 MMA), warp 1 waits X and arrives on Y,
// warp 0 waits Y: cycles per round trip (ping-pong), for hinted / un-hinted try_wait.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I paper_2604_03957_b200/csrc -o tools/ubench/handoff_ubench tools/ubench/handoff_ubench.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include "sm100.cuh"
using namespace bwta::sm100;

__device__ __forceinline__ void waitb(uint64_t* b, uint32_t ph, int hint) {
    if (hint) { while (!mbar_try_wait(b, ph)) {} }
    else { while (!mbar_try_wait_nh(b, ph)) {} }
}

__global__ void kern(int iters, int mode, int hint, long long* out) {
    extern __shared__ __align__(1024) uint8_t sm[];
    __shared__ uint64_t X, Y;
    __shared__ uint32_t tslot;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    for (int i = threadIdx.x; i < 32768 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(sm)[i] = 0;
    fence_proxy_async_smem();
    if (threadIdx.x == 0) { mbar_init(&X, 1); mbar_init(&Y, 1); fence_barrier_init(); }
    if (warp == 0) tmem_alloc(&tslot, 512);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tb = tslot;
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
        const uint32_t ph = it & 1;
        if (warp == 0) {
            if (lane == 0) {
                if (mode == 0) mbar_arrive(&X);
                else {
                    if (mode == 2) {
                        const uint32_t idesc = idesc_mxf4(128, 128);
                        mma_mxf4(tb, smem_desc_sw128(smem_u32(sm)), smem_desc_sw128(smem_u32(sm + 16384)), idesc, tb + 480, tb + 488, 0);
                    }
                    tc_commit(&X);
                }
            }
            __syncwarp();
            waitb(&Y, ph, hint);
        } else if (warp == 1) {
            waitb(&X, ph, hint);
            tc_fence_after();
            if (lane == 0) mbar_arrive(&Y);
            __syncwarp();
        }
    }
    long long t1 = clock64();
    if (threadIdx.x == 0) out[0] = (t1 - t0) / iters;
    tc_fence_before();
    __syncthreads();
    if (warp == 0) { tc_fence_after(); tmem_dealloc(tslot, 512); }
}

int main() {
    long long* d;
    cudaMalloc(&d, 8);
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 40000);
    const char* names[3] = {"mbarrier.arrive", "tcgen05.commit (no MMA)", "MMA 128x128x64 + commit"};
    for (int hint = 0; hint < 2; ++hint)
        for (int mode = 0; mode < 3; ++mode) {
            kern<<<1, 64, 40000>>>(1000, mode, hint, d);
            long long h;
            cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
            printf("%-26s %s try_wait: %lld cycles per round trip (%s)\n", names[mode], hint ? "hinted  " : "unhinted", h,
                   cudaGetErrorString(cudaGetLastError()));
        }
    return 0;
}
