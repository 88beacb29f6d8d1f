// peer.cu -- the cross-GPU completion barrier of the fused all-gather (bwta_gemm_peers).
//
// bwta_gemm_peers stores every output tile of rank r's N-shard into the Y^T buffer of each peer GPU
// directly from its epilogue (TMA stores through NVLink peer mappings), so the all-gather overlaps
// the GEMM tile by tile and needs no collective launch.  What remains is knowing when every
// peer's stores into this GPU's buffer have landed: this kernel, launched on the GEMM's stream
// after it (a normal launch, so it starts only once the GEMM has completed), reads this rank's
// barrier count c from device memory (so a CUDA graph replaying the step needs no new parameters),
// epoch = c + 1, and has thread t
//   1. st.release.sys flags[t][rank] = epoch  (signal peer t: "my stores to you are done" -- a
//      release at system scope, cumulative over every store of the preceding kernels, which
//      griddepcontrol.wait has made visible to this thread);
//   2. spin with ld.acquire.sys on flags[rank][t] until it reaches epoch (peer t's signal to us);
// then thread 0 stores the count epoch.
// After the kernel every peer's shard is visible to the work that follows on this stream.  A peer
// that never signals (a crashed rank) traps the kernel after 30 s instead of hanging the GPU.
#include "bwta_internal.h"

namespace bwta {
namespace {

struct BarrierArgs {
    uint32_t* flags[MAX_PEERS + 1];  // flags[r]: rank r's array of `world` epoch slots
    uint32_t* count;                 // this rank's barrier count (device, not shared)
    int world, rank;
};

__device__ __forceinline__ uint64_t globaltimer_ns() {
    uint64_t t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

__global__ void __launch_bounds__(32) peer_barrier_kernel(BarrierArgs a) {
    // launched with PDL: the next kernel may start its prologue now; its griddepcontrol.wait still
    // waits for this barrier to complete.  This kernel's own wait: the GEMM has completed and its
    // stores (incl. the peer stores) are performed.
    pdl_launch_dependents();
    pdl_wait();
    const int t = threadIdx.x;
    const uint32_t epoch = *reinterpret_cast<volatile uint32_t*>(a.count) + 1u;
    if (t < a.world) {
        asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(a.flags[t] + a.rank), "r"(epoch) : "memory");
        const uint32_t* mine = a.flags[a.rank] + t;
        const uint64_t t0 = globaltimer_ns();
        for (;;) {
            uint32_t v;
            asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(mine) : "memory");
            if (int32_t(v - epoch) >= 0) break;  // wrap-safe: epochs only grow
            if (globaltimer_ns() - t0 > 30ull * 1000000000ull) __trap();
            __nanosleep(256);
        }
    }
    __syncthreads();
    if (t == 0) *a.count = epoch;
}

}  // namespace

cudaError_t launch_peer_barrier(uint32_t* const* flags, int world, int rank, uint32_t* count, cudaStream_t s) {
    BarrierArgs a{};
    for (int r = 0; r < world; ++r) a.flags[r] = flags[r];
    a.count = count;
    a.world = world;
    a.rank = rank;
    return launch_pdl(peer_barrier_kernel, dim3(1), dim3(32), 0, s, 1, a);
}

}  // namespace bwta
