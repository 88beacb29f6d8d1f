// Issue throughput of the epilogue's conversion: cvt.rn.f16x2.f32 (F2FP.PACK)
// vs FMUL, for 4..16 warps per SM (cycles per warp-instruction per SM).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/ubench/cvt_ubench tools/ubench/cvt_ubench.cu
#include <cstdio>
#include <cstdint>
#include <cuda_fp16.h>
template <int MODE>
__global__ void kern(float seed, uint32_t* out, long long* cyc, int iters) {
    float a[8];
    for (int i = 0; i < 8; ++i) a[i] = seed + threadIdx.x + i;
    uint32_t acc = 0;
    __syncthreads();
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            if (MODE == 0) {
                uint32_t r;
                asm volatile("cvt.rn.f16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(a[i]), "f"(a[(i + 1) & 7]));
                acc ^= r;
            } else {
                float r;
                asm volatile("mul.rn.f32 %0, %1, %2;" : "=f"(r) : "f"(a[i]), "f"(a[(i + 1) & 7]));
                acc ^= __float_as_uint(r);
            }
        }
    }
    __syncthreads();
    long long t1 = clock64();
    out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
    if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}
int main() {
    uint32_t* o; cudaMalloc(&o, 1 << 20);
    long long* c; cudaMalloc(&c, 8 * 148);
    long long h;
    for (int mode = 0; mode < 2; ++mode)
        for (int warps : {4, 8, 16}) {
            const int iters = 4096;
            if (mode == 0) kern<0><<<1, warps * 32>>>(1.0f, o, c, iters);
            else kern<1><<<1, warps * 32>>>(1.0f, o, c, iters);
            cudaDeviceSynchronize();
            cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
            const double instr = double(iters) * 8 * warps;  // warp-instructions (plus the xor)
            printf("%s warps %2d: %.3f cycles per warp-instr per SM (incl. 1 LOP each)\n", mode == 0 ? "F2FP.PACK" : "FMUL     ",
                   warps, double(h) / instr);
        }
    return 0;
}
