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

// issue rate of the MMA thread: commits alone, or n MMAs (M=128, N, K=64 mxf4, A from smem or TMEM) + 1 commit
__global__ void issue_kern(int iters, int nmma, int N, int ts, long long* out) {
    extern __shared__ __align__(1024) uint8_t sm[];
    __shared__ uint64_t X;
    __shared__ uint32_t tslot;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    for (int i = threadIdx.x; i < 40000 / 4 - 16; i += blockDim.x) reinterpret_cast<uint32_t*>(sm)[i] = 0;
    fence_proxy_async_smem();
    if (threadIdx.x == 0) { mbar_init(&X, 1); fence_barrier_init(); }
    if (warp == 0) tmem_alloc(&tslot, 512);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tb = tslot;
    if (warp == 0 && lane == 0) {
        const uint32_t idesc = idesc_mxf4(128, N);
        long long t0 = clock64();
        for (int it = 0; it < iters; ++it) {
            for (int k = 0; k < nmma; ++k) {
                if (ts) mma_mxf4_ts(tb, tb + 256 + 8 * k, smem_desc_sw128(smem_u32(sm + 16384) + 32 * k), idesc, tb + 480, tb + 488, 1);
                else mma_mxf4(tb, smem_desc_sw128(smem_u32(sm) + 32 * k), smem_desc_sw128(smem_u32(sm + 16384) + 32 * k), idesc, tb + 480, tb + 488, 1);
            }
            tc_commit(&X);
        }
        long long t1 = clock64();
        mbar_wait(&X, (iters - 1) & 1);
        long long t2 = clock64();
        out[0] = (t1 - t0) / iters;
        out[1] = (t2 - t0) / iters;
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 0) { tc_fence_after(); tmem_dealloc(tslot, 512); }
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
    long long* d2;
    cudaMalloc(&d2, 16);
    cudaFuncSetAttribute(issue_kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 50000);
    for (int ts = 0; ts < 2; ++ts)
        for (int nmma : {0, 1, 2, 4})
            for (int N : {128, 192, 256}) {
                if (nmma == 0 && (N != 128 || ts)) continue;
                issue_kern<<<1, 64, 50000>>>(2000, nmma, N, ts, d2);
                long long h[2];
                cudaMemcpy(h, d2, 16, cudaMemcpyDeviceToHost);
                printf("issue: %d x MMA(128x%dx64, A %s) + commit: issue %lld cyc/iter, completion %lld cyc/iter (%s)\n",
                       nmma, N, ts ? "TMEM" : "smem", h[0], h[1], cudaGetErrorString(cudaGetLastError()));
            }
    return 0;
}
