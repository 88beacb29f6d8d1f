// POPC vs LOP3 issue rate on B200 (thread-ops per clock per SM): 148 x 1024
// threads, 8 independent chains per thread.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/ubench/popc_ubench tools/ubench/popc_ubench.cu
#include <cstdio>
#include <cstdint>
template <int MODE>
__global__ void kern(uint32_t seed, int iters, uint32_t* out, long long* cyc) {
    uint32_t x[8], a[8];
    for (int i = 0; i < 8; ++i) { x[i] = seed * (threadIdx.x + 17 * i + 1); a[i] = 0; }
    __syncthreads();
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            if (MODE == 0) { a[i] += __popc(x[i]); x[i] ^= a[i]; }             // POPC + IADD + LOP
            else if (MODE == 1) { a[i] = (a[i] ^ x[i]) & (x[i] | 0x55u); x[i] += a[i]; }  // LOP3 + IADD
            else { a[i] += __popc(x[i]); x[i] += 0x9e3779b9u; }                 // POPC + 2 IADD
        }
    }
    long long t1 = clock64();
    uint32_t s = 0;
    for (int i = 0; i < 8; ++i) s ^= a[i] ^ x[i];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
    if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}
int main() {
    uint32_t* o; cudaMalloc(&o, 148 * 1024 * 4);
    long long* c; cudaMalloc(&c, 148 * 8);
    const int iters = 4096;
    for (int mode = 0; mode < 3; ++mode) {
        for (int rep = 0; rep < 2; ++rep) {
            if (mode == 0) kern<0><<<148, 1024>>>(7, iters, o, c);
            else if (mode == 1) kern<1><<<148, 1024>>>(7, iters, o, c);
            else kern<2><<<148, 1024>>>(7, iters, o, c);
        }
        cudaDeviceSynchronize();
        long long h; cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
        const double ops = 1024.0 * iters * 8;  // per SM: one POPC (mode 0/2) or one LOP3 (mode 1) per chain step
        printf("mode %d (%s): %.1f ops/clk/SM\n", mode, mode == 0 ? "POPC+IADD+LOP" : mode == 1 ? "LOP3+IADD" : "POPC+2 IADD", ops / h);
    }
    return 0;
}
