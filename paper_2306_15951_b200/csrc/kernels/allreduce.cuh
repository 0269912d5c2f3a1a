// allreduce.cuh -- KB-REDUCE-AR: the G_Z aggregation of Sk-dilated
// fused with the cross-GPU sum of the batch shards' partial dW (SURVEY §8
// a6 / f1), over peer memory (NVLink P2P stores), deterministic.
//
// The batch shard of rank r is the outermost segment of the paper's
// map-reduce over G_K = N*O_H*O_W; the whole reduction is one kernel:
//   phase 1 (reduce-scatter): every element i of dW is owned by rank
//     s = i / slice; rank r sums its G_Z partials of i in fixed order z =
//     0..gz-1 and stores the sum into slot r of owner s's receive buffer
//     (a P2P store when s != r);
//   cross-rank barrier 1 (release/acquire signal words, system scope);
//   phase 2 (all-gather): the owner sums its slice over the ranks in fixed
//     order q = 0..W-1 and stores the result into every rank's dW;
//   cross-rank barrier 2: when the kernel ends on any rank its dW is final.
// Every rank therefore holds the bit-identical sum ((part_0) + (part_1) + ...)
// with the same association on every run.  Traffic per rank equals a ring
// all-reduce's: 2 (W-1)/W |dW| over NVLink.
//
// Waits are bounded: a signal that never arrives (a peer that did not launch)
// sets *err and lets the kernel finish instead of hanging the GPU.
#pragma once
#include "ptx.cuh"

namespace cks {

constexpr int kArMaxRanks = 8;

struct ArParams {
    const float4* part;               // local partials [gz][nv] (gz = 1: the local dW)
    long long nv;                     // float4 elements of dW
    long long slice;                  // float4 elements per owner slice (ceil(nv / world))
    int gz, world, rank;
    float4* recv[kArMaxRanks];        // rank t's receive buffer [world][slice] (P2P-mapped)
    float4* out[kArMaxRanks];         // rank t's dW
    unsigned* flag[kArMaxRanks];      // rank t's signal words [2] (monotonic: epoch * world after phase k)
    unsigned* count;                  // this rank's words [3]: CTA arrival counters (zero on entry, left
                                      // zero) and the call sequence number (device-side, so a CUDA graph
                                      // replaying the call keeps counting)
    int* err;                         // set to 1 if a cross-rank wait timed out
};

__device__ __forceinline__ unsigned ld_acquire_sys(const unsigned* p) {
    unsigned v;
    asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void red_release_sys(unsigned* p, unsigned v) {
    asm volatile("red.release.sys.global.add.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

// All CTAs of this rank arrive; the last one signals every rank; then every CTA
// waits until all ranks signalled phase k of this epoch.
__device__ __forceinline__ void ar_barrier(const ArParams& p, int k, unsigned epoch) {
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence_system();  // this CTA's (remote) stores before the arrival
        const unsigned old = atomicAdd(&p.count[k], 1u);
        if (old == gridDim.x - 1) {
            p.count[k] = 0u;  // every CTA arrived: reset for the next call
            if (k == 1) p.count[2] = epoch;  // every CTA read the sequence number at its start (before barrier 0)
            __threadfence_system();
            for (int t = 0; t < p.world; ++t) red_release_sys(p.flag[t] + k, 1u);
        }
        const unsigned target = epoch * unsigned(p.world);
        long long spins = 0;
        while (ld_acquire_sys(p.flag[p.rank] + k) < target) {
            if (++spins > (1ll << 26)) {  // ~ seconds: a peer never arrived
                *p.err = 1;
                break;
            }
            __nanosleep(64);
        }
    }
    __syncwarp();
    __syncthreads();
}

// One rank's KB-REDUCE-AR (every CTA of the rank runs it; gridDim.x = the rank's CTAs).
__device__ __forceinline__ void ar_run(const ArParams& p) {
    __shared__ unsigned s_epoch;
    if (threadIdx.x == 0) s_epoch = *reinterpret_cast<volatile unsigned*>(p.count + 2) + 1u;  // this call's number
    __syncwarp();
    __syncthreads();
    const unsigned epoch = s_epoch;
    const long long stride = static_cast<long long>(gridDim.x) * blockDim.x;
    // phase 1: G_Z sums pushed to their owners (slot `rank` of the owner's receive buffer)
    for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < p.nv; i += stride) {
        float4 v = p.part[i];
        for (int z = 1; z < p.gz; ++z) {  // fixed order z = 0..gz-1
            const float4 w = p.part[z * p.nv + i];
            v.x += w.x;
            v.y += w.y;
            v.z += w.z;
            v.w += w.w;
        }
        const int s = int(i / p.slice);
        p.recv[s][p.rank * p.slice + (i - s * p.slice)] = v;
    }
    ar_barrier(p, 0, epoch);
    // phase 2: the owner sums its slice over the ranks (fixed order) and writes every rank's dW
    const long long lo = p.rank * p.slice;
    const long long len = min(p.slice, p.nv - lo);
    const float4* mine = p.recv[p.rank];
    for (long long j = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; j < len; j += stride) {
        float4 v = mine[j];
        for (int q = 1; q < p.world; ++q) {
            const float4 w = mine[q * p.slice + j];
            v.x += w.x;
            v.y += w.y;
            v.z += w.z;
            v.w += w.w;
        }
        for (int t = 0; t < p.world; ++t) p.out[t][lo + j] = v;
    }
    ar_barrier(p, 1, epoch);
}

__global__ void __launch_bounds__(256) reduce_allreduce_kernel(const __grid_constant__ ArParams p) {
    ptx::pdl_launch_dependents();
    ptx::pdl_wait();
    ar_run(p);
}

// Single-GPU emulation of `world` ranks: ONE cooperative launch, blockIdx.y = rank, so every
// CTA that spins at a cross-rank barrier is co-resident with the CTAs it waits for (separate
// launches that wait on one another are not guaranteed to run at the same time).
struct ArGroupParams {
    ArParams r[kArMaxRanks];
};
__global__ void __launch_bounds__(256) reduce_allreduce_emul_kernel(const __grid_constant__ ArGroupParams g) {
    ar_run(g.r[blockIdx.y]);
}

}  // namespace cks
