// Cost of staging a 4 KB output chunk in shared memory and handing it to the
// async proxy: stmatrix / st.shared.v4 x8 per lane, fence.proxy.async, TMA-
// less (just the fence) -- cycles per chunk for 1..8 concurrent warps.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/fence_ubench tools/ubench/fence_ubench.cu
#include <cstdio>
#include <cstdint>
__device__ __forceinline__ uint32_t smem_u32(const void* p) { return uint32_t(__cvta_generic_to_shared(p)); }
template <int MODE>
__global__ void kern(unsigned long long* out, int iters) {
    __shared__ __align__(1024) uint8_t buf[8][4096];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t sb = smem_u32(buf[warp]);
    uint32_t r0 = lane, r1 = lane * 3, r2 = lane * 5, r3 = lane * 7;
    __syncthreads();
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
        for (int k = 0; k < 8; ++k) {
            if (MODE & 1) {
                const uint32_t a = sb + ((k * 4 + (lane >> 3)) & 31) * 128 + ((lane & 7) << 4);
                asm volatile("stmatrix.sync.aligned.m8n8.x4.shared.b16 [%0], {%1, %2, %3, %4};" ::"r"(a), "r"(r0),
                             "r"(r1), "r"(r2), "r"(r3) : "memory");
            } else {
                const uint32_t a = sb + lane * 128 + (((k ^ lane) & 7) << 4);
                asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(a), "r"(r0), "r"(r1), "r"(r2), "r"(r3)
                             : "memory");
            }
            r0 += 1; r1 += 2;
        }
        if (MODE & 2) asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        __syncwarp();
    }
    long long t1 = clock64();
    if (lane == 0) out[blockIdx.x * 16 + warp] = (t1 - t0) / iters;
    if (r0 == 12345) out[0] = r1 + r2 + r3;
}
int main() {
    unsigned long long* d; cudaMalloc(&d, 16 * 16 * 8);
    unsigned long long h[256];
    const char* names[4] = {"sts128 x8", "stmatrix.x4 x8", "sts128 x8 + fence", "stmatrix.x4 x8 + fence"};
    for (int mode = 0; mode < 4; ++mode)
        for (int warps : {1, 2, 4, 8}) {
            void (*k)(unsigned long long*, int) = mode == 0 ? kern<0> : mode == 1 ? kern<1> : mode == 2 ? kern<2> : kern<3>;
            k<<<1, warps * 32>>>(d, 1000);
            cudaDeviceSynchronize();
            cudaMemcpy(h, d, 16 * 8, cudaMemcpyDeviceToHost);
            printf("%-24s warps %2d: %llu cycles/chunk (warp 0)\n", names[mode], warps, h[0]);
        }
    return 0;
}
