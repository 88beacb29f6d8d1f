// Microbenchmark: cycles per unpack of one A row (4 packed words -> 32 code
// words) per warp, for several instruction mixes.  ALU (LOP3/SHF) and FMA
// (IMAD) pipes each retire one warp instruction per 2 cycles per SMSP.
#include <cstdio>
#include <cstdint>
__device__ __forceinline__ uint32_t shr_fma(uint32_t x, int j) {  // x >> j on the FMA pipe
    if (j == 0) return x;
    return __umulhi(x, 1u << (32 - j));
}
__device__ __forceinline__ uint32_t shl_fma(uint32_t x, int k) {  // x << k as an IMAD (FMA pipe)
    uint32_t r;
    asm("mad.lo.u32 %0, %1, %2, 0;" : "=r"(r) : "r"(x), "r"(1u << k));
    return r;
}
template <int V> __device__ __forceinline__ uint32_t unpack_t(uint32_t s, uint32_t z, int j) {
    if (V == 4) {  // x64-scaled ternary: z -> bit 6, s -> bit 7 of each byte
        const uint32_t zz = j < 7 ? shl_fma(z, 6 - j) : (z >> 1);
        const uint32_t ss = shl_fma(s, 7 - j);
        return (zz & 0x40404040u) | (ss & 0x80808080u);
    }
    if (V == 5) {  // x64-scaled binary
        return (shl_fma(s, 7 - j) & 0x80808080u) | 0x40404040u;
    }
    if (V == 0) {  // current: SHF + LOP3 per plane, a&n, IMAD
        const uint32_t a = (s >> j) & 0x01010101u, n = (z >> j) & 0x01010101u;
        return n | ((a & n) * 0xfeu);
    } else if (V == 1) {  // shifts on the FMA pipe, canonical planes (no a & n)
        const uint32_t a = shr_fma(s, j) & 0x01010101u, n = shr_fma(z, j) & 0x01010101u;
        return a * 0xfeu + n;
    } else if (V == 2) {  // binary (one plane) current
        const uint32_t a = (s >> j) & 0x01010101u;
        return a * 0xfeu + 0x01010101u;
    } else {  // binary with FMA shift
        const uint32_t a = shr_fma(s, j) & 0x01010101u;
        return a * 0xfeu + 0x01010101u;
    }
}
template <int V>
__global__ void k_math(const uint32_t* in, uint32_t* out, long long* cyc, int iters) {
    uint32_t s[4], z[4];
    for (int i = 0; i < 4; ++i) { s[i] = in[threadIdx.x * 8 + i]; z[i] = in[threadIdx.x * 8 + 4 + i]; }
    uint32_t acc = 0;
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
        uint32_t o[32];
#pragma unroll
        for (int g = 0; g < 4; ++g)
#pragma unroll
            for (int j = 0; j < 8; ++j) o[8 * g + j] = unpack_t<V>(s[g], z[g], j);
        uint32_t x = 0;
#pragma unroll
        for (int i = 0; i < 32; i += 4) x += o[i] ^ o[i + 1] ^ o[i + 2] ^ o[i + 3];
        acc += x;
        s[it & 3] += acc;  // serialise iterations
    }
    long long t1 = clock64();
    out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
    if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}
__device__ __forceinline__ bool try_wait(uint64_t* bar, uint32_t parity, uint32_t hint) {
    uint32_t ok;
    asm volatile("{\n\t.reg .pred P;\n\tmbarrier.try_wait.parity.shared::cta.b64 P, [%1], %2, %3;\n\tselp.b32 %0, 1, 0, P;\n\t}"
                 : "=r"(ok) : "r"((uint32_t)__cvta_generic_to_shared(bar)), "r"(parity), "r"(hint) : "memory");
    return ok != 0;
}
// warps 0-3 unpack (variant 4), warps 4.. spin on a barrier that completes only at the end
__global__ void k_spin(const uint32_t* in, uint32_t* out, long long* cyc, int iters, uint32_t hint) {
    __shared__ uint64_t bar;
    __shared__ int done;
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"((uint32_t)__cvta_generic_to_shared(&bar)));
        done = 0;
    }
    __syncthreads();
    const int warp = threadIdx.x >> 5;
    if (warp < 4) {
        uint32_t s[4], z[4];
        for (int i = 0; i < 4; ++i) { s[i] = in[threadIdx.x * 8 + i]; z[i] = in[threadIdx.x * 8 + 4 + i]; }
        uint32_t acc = 0;
        long long t0 = clock64();
        for (int it = 0; it < iters; ++it) {
            uint32_t o[32];
#pragma unroll
            for (int g = 0; g < 4; ++g)
#pragma unroll
                for (int j = 0; j < 8; ++j) o[8 * g + j] = unpack_t<4>(s[g], z[g], j);
            uint32_t x = 0;
#pragma unroll
            for (int i = 0; i < 32; i += 4) x += o[i] ^ o[i + 1] ^ o[i + 2] ^ o[i + 3];
            acc += x;
            s[it & 3] += acc;
        }
        long long t1 = clock64();
        out[threadIdx.x] = acc;
        if (threadIdx.x == 0) cyc[0] = t1 - t0;
        __syncwarp();
        if (threadIdx.x == 0) {
            asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"((uint32_t)__cvta_generic_to_shared(&bar)) : "memory");
        }
    } else {
        while (!try_wait(&bar, 0, hint)) {}
    }
}
template <int V> void run(const char* name, uint32_t* in, uint32_t* out, long long* cyc) {
    const int iters = 1000;
    for (int warps : {1, 4}) {
        k_math<V><<<1, 32 * warps>>>(in, out, cyc, iters);
        cudaDeviceSynchronize();
        long long c; cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
        printf("%-28s warps %d: %6.1f cycles per row per warp\n", name, warps, double(c) / iters);
    }
}
int main() {
    uint32_t *in, *out; long long* cyc;
    cudaMalloc(&in, 1 << 20); cudaMalloc(&out, 1 << 20); cudaMalloc(&cyc, 8 * 1024);
    cudaMemset(in, 0x5a, 1 << 20);
    run<0>("ternary SHF+LOP3 (current)", in, out, cyc);
    run<1>("ternary IMAD.HI shifts", in, out, cyc);
    run<2>("binary SHF+LOP3 (current)", in, out, cyc);
    run<3>("binary IMAD.HI shift", in, out, cyc);
    run<4>("ternary x64 IMAD shl", in, out, cyc);
    run<5>("binary x64 IMAD shl", in, out, cyc);
    for (uint32_t hint : {0u, 1000u, 0x989680u}) {
        for (int spinners : {0, 4, 20}) {
            k_spin<<<1, 128 + 32 * spinners>>>(in, out, cyc, 1000, hint);
            cudaDeviceSynchronize();
            long long c; cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
            printf("ternary x64 with %2d spinning warps (hint %u): %6.1f cycles per row\n", spinners, hint, double(c) / 1000);
        }
    }
    return 0;
}
