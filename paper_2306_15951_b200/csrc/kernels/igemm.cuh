// igemm.cuh -- KB-CONV / KB-KS: the trimmed-window implicit GEMM on
// tcgen05 tensor cores, shared by ConvV2 (Alg. 1) and the fused
// Stage2&3 of KS-deconv-V2 (Alg. 2/2B).
//
// One tile = 128 batch images x BN output channels at ONE output pixel
// (row rh, row rw of the per-axis plan tables).  All 128 GEMM rows of a tile
// therefore share one trimmed filter window [ts_h, te_h) x [ts_w, te_w) --
// the B200 analogue of P:156 "all threads in the same block have the same
// trimmed-filters ... no warp-divergence": padded zeros are never loaded or
// multiplied, and no bounds check exists in the K loop.
//
// GEMM view per tile: M = 128 images, N = BN channels, K = window taps x Ka
// channels, both operands K-major:
//   A[m][k] = act[n0+m, a0_h+ch, a0_w+cw, kc]   (TMA 4-D box (BK,1,1,128))
//   B[j][k] = filt[phase][nb*BN+j][ch*slot_stride+cw][kc]  (box (BK,1,BN,1))
//   out[n0+m, out_h, out_w, nb*BN+j] = D[m][j]  (fp32, overwritten)
// For ConvV2 act = X, filt = W (slot = fh*FW+fw), a0 = o*s - p (T1).  For
// KS-deconv act = dY, filt = the packed sub-filters C_{y,x} (Stage1), a0 =
// oh_s = u + a_y and out = u*sh + ih_s (T2): the epilogue IS Stage3's
// phase-strided composition ("Stage2 and Stage3 are fused").
//
// Warp roles (256 threads, 1 CTA/SM, persistent over tiles):
//   warp 0 lane 0  TMA producer  (smem ring of STAGES {A,B} slots, mbarriers)
//   warp 1 lane 0  MMA issuer    (tcgen05.mma into a double-buffered TMEM acc)
//   warp 2         TMEM allocator
//   warps 4..7     epilogue      (tcgen05.ld -> fp32 global stores)
#pragma once
#include "ptx.cuh"
#include "../../../include/cks.h"

namespace cks {

struct KAxis {
    int16_t a0[CKS_MAX_ROWS];   // A coordinate of tap 0
    int16_t out[CKS_MAX_ROWS];  // output coordinate
    uint8_t ts[CKS_MAX_ROWS];   // trimmed tap window [ts, te)
    uint8_t te[CKS_MAX_ROWS];
    uint8_t phase[CKS_MAX_ROWS];
};

struct IgemmParams {
    KAxis ah, aw;
    float* out;
    int rows_h, rows_w;
    int nblk, nbs;
    int kc_blocks;    // ceil(Ka / BK)
    int slot_stride;  // tap slot = ch * slot_stride + cw
    int phases_w;     // phase = phase_h * phases_w + phase_w
    int N;
    int out_H, out_W, out_C;
    long long num_tiles;
};

template <int BN, bool kTF32>
struct IgemmShape {
    static constexpr int EB = kTF32 ? 4 : 2;
    static constexpr int BK = 128 / EB;   // one 128-byte swizzle row of K
    static constexpr int UK = 32 / EB;    // K per tcgen05.mma
    static constexpr int A_BYTES = 128 * 128;
    static constexpr int B_BYTES = BN * 128;
    static constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
    static constexpr int STAGES = (200 * 1024 / STAGE_BYTES) > 8 ? 8 : (200 * 1024 / STAGE_BYTES);
    static constexpr int SMEM_BYTES = STAGES * STAGE_BYTES + 1024 + 256;
    static constexpr uint32_t TMEM_COLS = 2 * BN <= 32 ? 32 : 2 * BN <= 64 ? 64 : 2 * BN <= 128 ? 128 : 2 * BN <= 256 ? 256 : 512;
};

struct TileCoord {
    int nb, nblk, rh, rw;
};
__device__ __forceinline__ TileCoord decode_tile(long long t, const IgemmParams& p) {
    TileCoord c;
    c.nb = int(t % p.nbs);
    t /= p.nbs;
    c.nblk = int(t % p.nblk);
    t /= p.nblk;
    c.rw = int(t % p.rows_w);
    c.rh = int(t / p.rows_w);
    return c;
}

template <int BN, bool kTF32>
__global__ void __launch_bounds__(256, 1)
    igemm_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                 const __grid_constant__ IgemmParams p) {
    using S = IgemmShape<BN, kTF32>;
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + S::STAGES * S::STAGE_BYTES);
    uint64_t* empty = full + S::STAGES;
    uint64_t* tfull = empty + S::STAGES;
    uint64_t* tempty = tfull + 2;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);

    const uint32_t warp = ptx::warp_id(), lane = ptx::lane_id();
    if (warp == 0 && lane == 0) {
        ptx::prefetch_tmap(&tmA);
        ptx::prefetch_tmap(&tmB);
    }
    if (warp == 1 && lane == 0) {
        for (int i = 0; i < S::STAGES; ++i) {
            ptx::mbar_init(&full[i], 1);
            ptx::mbar_init(&empty[i], 1);
        }
        for (int i = 0; i < 2; ++i) {
            ptx::mbar_init(&tfull[i], 1);
            ptx::mbar_init(&tempty[i], 128);
        }
        ptx::fence_barrier_init();
    }
    if (warp == 2) ptx::tmem_alloc(tmem_slot, S::TMEM_COLS);
    ptx::tc_fence_before();
    __syncthreads();
    ptx::tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;

    if (warp == 0) {
        if (lane == 0) {
            // ---------------- TMA producer
            uint32_t stage = 0, phase = 0;
            for (long long t = blockIdx.x; t < p.num_tiles; t += gridDim.x) {
                const TileCoord c = decode_tile(t, p);
                const int chs = p.ah.ts[c.rh], che = p.ah.te[c.rh];
                const int cws = p.aw.ts[c.rw], cwe = p.aw.te[c.rw];
                const int a0h = p.ah.a0[c.rh], a0w = p.aw.a0[c.rw];
                const int ph = p.ah.phase[c.rh] * p.phases_w + p.aw.phase[c.rw];
                for (int ch = chs; ch < che; ++ch)
                    for (int cw = cws; cw < cwe; ++cw)
                        for (int kc = 0; kc < p.kc_blocks; ++kc) {
                            ptx::mbar_wait(&empty[stage], phase ^ 1);
                            ptx::mbar_arrive_expect_tx(&full[stage], S::STAGE_BYTES);
                            uint8_t* sa = smem + stage * S::STAGE_BYTES;
                            ptx::tma_load_4d(sa, &tmA, &full[stage], kc * S::BK, a0w + cw, a0h + ch, c.nblk * 128);
                            ptx::tma_load_4d(sa + S::A_BYTES, &tmB, &full[stage], kc * S::BK,
                                             ch * p.slot_stride + cw, c.nb * BN, ph);
                            if (++stage == S::STAGES) {
                                stage = 0;
                                phase ^= 1;
                            }
                        }
            }
        }
        __syncwarp();
    } else if (warp == 1) {
        if (lane == 0) {
            // ---------------- MMA issuer (single thread)
            constexpr uint32_t idesc = ptx::instr_desc(128, BN, kTF32, false, false);
            uint32_t stage = 0, phase = 0, acc = 0, acc_phase = 0;
            for (long long t = blockIdx.x; t < p.num_tiles; t += gridDim.x) {
                const TileCoord c = decode_tile(t, p);
                const int nsteps = (p.ah.te[c.rh] - p.ah.ts[c.rh]) * (p.aw.te[c.rw] - p.aw.ts[c.rw]) * p.kc_blocks;
                ptx::mbar_wait(&tempty[acc], acc_phase ^ 1);
                ptx::tc_fence_after();
                const uint32_t d = tmem_base + acc * BN;
                for (int k = 0; k < nsteps; ++k) {
                    ptx::mbar_wait(&full[stage], phase);
                    ptx::tc_fence_after();
                    const uint32_t a_addr = ptx::smem_u32(smem + stage * S::STAGE_BYTES);
                    const uint32_t b_addr = a_addr + S::A_BYTES;
#pragma unroll
                    for (int kk = 0; kk < S::BK / S::UK; ++kk) {
                        const uint64_t ad = ptx::smem_desc_sw128(a_addr + kk * 32, 16, 1024);
                        const uint64_t bd = ptx::smem_desc_sw128(b_addr + kk * 32, 16, 1024);
                        ptx::mma_ss<kTF32>(d, ad, bd, idesc, (k | kk) != 0);
                    }
                    ptx::mma_commit(&empty[stage]);  // frees the smem slot when these MMAs finish
                    if (++stage == S::STAGES) {
                        stage = 0;
                        phase ^= 1;
                    }
                }
                ptx::mma_commit(&tfull[acc]);  // accumulator ready (immediately if nsteps == 0)
                if (++acc == 2) {
                    acc = 0;
                    acc_phase ^= 1;
                }
            }
        }
        __syncwarp();
    } else if (warp >= 4) {
        // ---------------- epilogue: TMEM -> registers -> fp32 stores
        const uint32_t sub = warp & 3;  // TMEM sub-partition = lanes [32*sub, 32*sub+32)
        const int row = int(sub * 32 + lane);
        uint32_t acc = 0, acc_phase = 0;
        const bool vec4 = (p.out_C % 4) == 0;
        for (long long t = blockIdx.x; t < p.num_tiles; t += gridDim.x) {
            const TileCoord c = decode_tile(t, p);
            const bool empty_win = (p.ah.te[c.rh] <= p.ah.ts[c.rh]) || (p.aw.te[c.rw] <= p.aw.ts[c.rw]);
            ptx::mbar_wait(&tfull[acc], acc_phase);
            ptx::tc_fence_after();
            const int n = c.nblk * 128 + row;
            const int cbase = c.nb * BN;
            const int cvalid = min(BN, p.out_C - cbase);
            float* dst = nullptr;
            if (n < p.N)
                dst = p.out + ((static_cast<long long>(n) * p.out_H + p.ah.out[c.rh]) * p.out_W + p.aw.out[c.rw]) *
                                  p.out_C + cbase;
#pragma unroll 1
            for (int c0 = 0; c0 < BN; c0 += 32) {
                uint32_t r[32];
                ptx::tmem_ld32(tmem_base + ((sub * 32u) << 16) + acc * BN + c0, r);
                ptx::tmem_ld_wait();
                if (dst != nullptr && c0 < cvalid) {
                    if (empty_win) {
#pragma unroll
                        for (int j = 0; j < 32; ++j) r[j] = 0u;
                    }
                    if (vec4 && c0 + 32 <= cvalid) {
#pragma unroll
                        for (int j = 0; j < 32; j += 4)
                            *reinterpret_cast<float4*>(dst + c0 + j) =
                                make_float4(__uint_as_float(r[j]), __uint_as_float(r[j + 1]),
                                            __uint_as_float(r[j + 2]), __uint_as_float(r[j + 3]));
                    } else {
#pragma unroll
                        for (int j = 0; j < 32; ++j)
                            if (c0 + j < cvalid) dst[c0 + j] = __uint_as_float(r[j]);
                    }
                }
            }
            ptx::tc_fence_before();
            ptx::mbar_arrive(&tempty[acc]);
            if (++acc == 2) {
                acc = 0;
                acc_phase ^= 1;
            }
        }
    }
    __syncthreads();
    if (warp == 2) {
        ptx::tc_fence_after();
        ptx::tmem_dealloc(tmem_base, S::TMEM_COLS);
    }
}

}  // namespace cks
