// narrow.cuh -- KB-CONV-ROW / KB-WGRAD-ROW: ConvV2 forward and Sk-dilated
// weight gradient for narrow-channel layers (FW*C <= 64 bf16, the C = 3 input
// layers of all three workloads) on tcgen05 tensor cores.
//
// In NHWC the (fw, c) run of one filter row is CONTIGUOUS in X: for output
// column ow and filter row fh it is X[n][ih][(ow*sw - pw)*C + j], j = fw*C + c,
// j < FW*C.  So instead of one GEMM step per tap with a 3-of-64 used channel
// block (the generic path), a whole filter row is one K-block of JB = 16/32/64
// elements loaded by ONE TMA box element-addressed in the flattened (W*C) row;
// the w-direction padding is the box's out-of-bounds zero fill.  The row
// (h) direction keeps the paper's trimming: ConvV2 issues MMAs only for the
// valid filter rows [fh_s, fh_e) of each output row (T1, Alg. 1);
// Sk-dilated reads X with the leaping row ih = oh*sh + fh - ph (Fig. 7) and
// the out-of-range rows arrive as TMA zero fill (no DRAM traffic).
//
// TMA box origins must be 16-byte aligned in the innermost dimension, while
// the run starts at element (ow*sw - pw)*C.  With delta = that start mod 8
// elements, output columns fall into P = 8 / gcd(sw*C, 8) classes of equal
// delta; every CTA serves ONE class, loads the box from the aligned start
// (start - delta) and uses the filter row shifted right by delta (fwd), or
// drops the first delta rows of its result (wgrad).  JB covers delta + FW*C.
//
// KB-CONV-ROW  tile = one output pixel x 128 images x OC (<= 256):
//   D[n][oc] = sum_{fh valid} sum_j A_fh[n][j] * Wrow_fh[oc][j]
//   A: one box (JB, 128 images, FH rows) per tile, K-major (JB*2-byte rows);
//   B: all FH filter rows resident in shared memory for the whole kernel.
// KB-WGRAD-ROW tile = OC block x segment z of the G_Z map-reduce:
//   D[(fh, j)][oc] = sum_k X[n][oh*sh+fh-ph][(ow*sw-pw)*C + j] * dY[n][oh][ow][oc]
//   over k = (oh, ow, n) blocks of 64 images; both operands MN-major, M =
//   (fh, j) packed 128/JB filter rows per M-block.
#pragma once
#include "ptx.cuh"

namespace cks {

struct RowFwdParams {
    const uint16_t* w;  // W [OC][FH][FW*C] bf16 (dense, any alignment)
    float* y;           // Y [N][OH][OW][OC] fp32
    int N, H, W, C, OC, FH, FW, sh, sw, ph, pw, OH, OW;
    int nblk;           // ceil(N / 128)
    int P;              // column classes (gridDim.x is a multiple of P)
    int delta[8];       // per class: run start mod 8 (elements)
    int stages;         // A ring depth
    int tma_store;      // 1: epilogue via TMA store (OC % 32 == 0)
};

// Tiles of column class k = blockIdx.x % P, in the order (oh, ow, nb) with nb fastest.
struct RowClassIter {
    int k, owk, first, step, count;
    __device__ RowClassIter(int P, int OH, int OW, int nblk) {
        k = int(blockIdx.x) % P;
        owk = OW > k ? (OW - k + P - 1) / P : 0;
        first = int(blockIdx.x) / P;
        step = int(gridDim.x) / P;
        count = OH * owk * nblk;
    }
    __device__ void decode(int t, int P, int nblk, int& nb, int& oh, int& ow) const {
        nb = t % nblk;
        const int r = t / nblk;
        ow = k + P * (r % owk);
        oh = r / owk;
    }
};

template <int JB, int BN>
struct RowFwdShape {
    static constexpr int ROWB = JB * 2;                      // K bytes per row (swizzle width)
    static constexpr int TMEM_COLS = 2 * BN <= 32 ? 32 : (2 * BN <= 64 ? 64 : (2 * BN <= 128 ? 128 : (2 * BN <= 256 ? 256 : 512)));
    static constexpr int STAGING = 4 * 2 * 4096;             // 4 epilogue warps x 2 x (32 rows x 128 B)
};

__host__ __device__ constexpr int row_fwd_w_bytes(int JB, int BN, int FH) {
    return ((FH * BN * JB * 2) + 1023) / 1024 * 1024;
}
__host__ __device__ constexpr int row_fwd_stage_bytes(int JB, int FH) { return ((FH * 128 * JB * 2) + 1023) / 1024 * 1024; }

template <int JB, int BN>
__global__ void __launch_bounds__(256, 1)
    fwd_row_kernel(const __grid_constant__ CUtensorMap tmX, const __grid_constant__ CUtensorMap tmY,
                   const __grid_constant__ RowFwdParams p) {
    using S = RowFwdShape<JB, BN>;
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = smem_raw + ((1024u - (ptx::smem_u32(smem_raw) & 1023u)) & 1023u);
    const int wbytes = row_fwd_w_bytes(JB, BN, p.FH);
    const int sbytes = row_fwd_stage_bytes(JB, p.FH);
    uint8_t* wsm = smem;
    uint8_t* abuf = smem + wbytes;
    uint8_t* stg = abuf + p.stages * sbytes;
    uint64_t* full = reinterpret_cast<uint64_t*>(stg + S::STAGING);
    uint64_t* empty = full + 8;
    uint64_t* tfull = empty + 8;
    uint64_t* tempty = tfull + 2;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);

    ptx::pdl_launch_dependents();
    const uint32_t warp = ptx::warp_id(), lane = ptx::lane_id();
    if (warp == 0 && lane == 0) {
        ptx::prefetch_tmap(&tmX);
        if (p.tma_store) ptx::prefetch_tmap(&tmY);
    }
    if (warp == 1 && lane == 0) {
        for (int i = 0; i < p.stages; ++i) {
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
    ptx::pdl_wait();  // W and X may come from the previous kernel
    {   // all threads: gather the filter rows into the K-major swizzled B layout
        // (row r = fh*BN + oc, K = j), zero for oc >= OC and j >= FW*C
        const int jn = p.FW * p.C;
        const int dl = p.delta[int(blockIdx.x) % p.P];
        const int chunks = p.FH * BN * (JB / 8);
        for (int q = threadIdx.x; q < chunks; q += blockDim.x) {
            const int r = q / (JB / 8), c8 = q % (JB / 8);
            const int fh = r / BN, oc = r % BN;
            uint32_t v[4] = {0u, 0u, 0u, 0u};
            if (oc < p.OC) {
                const uint16_t* src = p.w + (static_cast<long long>(oc) * p.FH + fh) * jn;
#pragma unroll
                for (int e = 0; e < 8; ++e) {
                    const int j = c8 * 8 + e - dl;
                    const uint32_t x = (j >= 0 && j < jn) ? uint32_t(src[j]) : 0u;
                    v[e >> 1] |= x << (16 * (e & 1));
                }
            }
            const uint32_t off = ptx::swz(uint32_t(r * S::ROWB + c8 * 16), S::ROWB);
            *reinterpret_cast<uint4*>(wsm + off) = make_uint4(v[0], v[1], v[2], v[3]);
        }
        ptx::fence_proxy_async_smem();  // generic-proxy writes -> visible to tcgen05
    }
    ptx::tc_fence_before();
    __syncthreads();
    ptx::tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;

    if (warp == 0 || warp == 3) {
        // ---------------- TMA producers: warps 0 / 3 take alternate tiles
        const uint32_t mine = warp == 3 ? 1u : 0u;
        const RowClassIter it(p.P, p.OH, p.OW, p.nblk);
        const int dl = p.delta[it.k];
        uint32_t i = 0;
        for (int t = it.first; t < it.count; t += it.step, ++i) {
            if ((i & 1u) != mine) continue;
            int nb, oh, ow;
            it.decode(t, p.P, p.nblk, nb, oh, ow);
            const uint32_t s = i % uint32_t(p.stages), ph = (i / uint32_t(p.stages)) & 1u;
            ptx::mbar_wait(&empty[s], ph ^ 1u);
            if (ptx::elect_one()) {
                ptx::mbar_arrive_expect_tx(&full[s], uint32_t(p.FH * 128 * JB * 2));
                ptx::tma_load_4d(abuf + s * sbytes, &tmX, &full[s], (ow * p.sw - p.pw) * p.C - dl, nb * 128,
                                 oh * p.sh - p.ph, 0);
            }
            __syncwarp();
        }
    } else if (warp == 1) {
        // ---------------- MMA issuer: trimmed filter rows [fh_s, fh_e) (T1)
        constexpr uint32_t idesc = ptx::instr_desc(128, BN, false, false, false);
        const uint32_t a0 = ptx::smem_u32(abuf), w0 = ptx::smem_u32(wsm);
        const RowClassIter it(p.P, p.OH, p.OW, p.nblk);
        uint32_t i = 0;
        for (int t = it.first; t < it.count; t += it.step, ++i) {
            int nb, oh, ow;
            it.decode(t, p.P, p.nblk, nb, oh, ow);
            const int ih0 = oh * p.sh - p.ph;
            const int fs = max(-ih0, 0), fe = min(p.H - ih0, p.FH);
            const uint32_t s = i % uint32_t(p.stages), ph = (i / uint32_t(p.stages)) & 1u;
            const uint32_t acc = i & 1u, aph = (i >> 1) & 1u;
            ptx::mbar_wait(&tempty[acc], aph ^ 1u);
            ptx::mbar_wait(&full[s], ph);
            ptx::tc_fence_after();
            if (ptx::elect_one()) {
                const uint32_t d = tmem_base + acc * BN;
                for (int fh = fs; fh < fe; ++fh) {
                    const uint32_t sa = a0 + s * uint32_t(sbytes) + uint32_t(fh * 128 * S::ROWB);
                    const uint32_t sb = w0 + uint32_t(fh * BN * S::ROWB);
#pragma unroll
                    for (int k = 0; k < JB / 16; ++k)
                        ptx::mma_ss<false>(d, ptx::smem_desc_kmajor(sa + 32u * k, S::ROWB),
                                           ptx::smem_desc_kmajor(sb + 32u * k, S::ROWB), idesc,
                                           (fh > fs || k > 0) ? 1u : 0u);
                }
                ptx::mma_commit(&empty[s]);
                ptx::mma_commit(&tfull[acc]);
            }
            __syncwarp();
        }
    } else if (warp >= 4) {
        // ---------------- epilogue: TMEM -> registers -> (swizzled staging -> TMA store | direct stores)
        const uint32_t sub = warp & 3u;
        uint8_t* my = stg + sub * 2 * 4096;
        const RowClassIter it(p.P, p.OH, p.OW, p.nblk);
        uint32_t i = 0, q = 0;
        for (int t = it.first; t < it.count; t += it.step, ++i) {
            int nb, oh, ow;
            it.decode(t, p.P, p.nblk, nb, oh, ow);
            const uint32_t acc = i & 1u, aph = (i >> 1) & 1u;
            ptx::mbar_wait(&tfull[acc], aph);
            ptx::tc_fence_after();
            const int n = nb * 128 + int(sub * 32 + lane);
#pragma unroll 1
            for (int c0 = 0; c0 < BN; c0 += 32) {
                uint32_t r[32];
                ptx::tmem_ld32(tmem_base + ((sub * 32u) << 16) + acc * BN + c0, r);
                ptx::tmem_ld_wait();
                if (p.tma_store) {
                    if (c0 >= p.OC) continue;
                    uint8_t* buf = my + (q++ & 1u) * 4096;
                    if (ptx::elect_one()) ptx::bulk_wait_read1();  // buffer of chunk q-2 drained
                    __syncwarp();
#pragma unroll
                    for (int c = 0; c < 8; ++c)
                        *reinterpret_cast<uint4*>(buf + ptx::swz(lane * 128u + c * 16u, 128)) =
                            make_uint4(r[4 * c], r[4 * c + 1], r[4 * c + 2], r[4 * c + 3]);
                    ptx::fence_proxy_async_smem();
                    __syncwarp();
                    if (ptx::elect_one()) {
                        ptx::tma_store_4d(&tmY, buf, c0, ow, oh, nb * 128 + int(sub * 32));
                        ptx::bulk_commit();
                    }
                    __syncwarp();
                } else if (n < p.N) {
                    float* dst = p.y + ((static_cast<long long>(n) * p.OH + oh) * p.OW + ow) * p.OC;
#pragma unroll
                    for (int j = 0; j < 32; ++j)
                        if (c0 + j < p.OC) dst[c0 + j] = __uint_as_float(r[j]);
                }
            }
            ptx::tc_fence_before();
            ptx::mbar_arrive(&tempty[acc]);
        }
        if (p.tma_store && ptx::elect_one()) ptx::bulk_wait_read0();
        __syncwarp();
    }
    __syncthreads();
    if (warp == 2) {
        ptx::tc_fence_after();
        ptx::tmem_dealloc(tmem_base, S::TMEM_COLS);
    }
}

// ------------------------------------------------------------------ wgrad
struct RowWgradParams {
    float* out;  // dW [OC][FH][FW*C] (gz == 1) or partials [gz][OC][FH][FW*C]
    long long part_stride;
    int N, H, W, C, OC, FH, FW, sh, sw, ph, pw, OH, OW;
    int mb;       // M-blocks of 128 (fh, j) rows
    int nbs;      // OC blocks of BN
    int P;        // column classes
    int delta[8]; // per class: run start mod 8 (elements)
    int gzc;      // map-reduce segments per class; partial index = z * P + k
    int nblk64;   // ceil(N / 64)
    int num_tiles;  // nbs * P * gzc
    int stages;
    int a_bytes;  // mb * 128 * 64 * 2
};

// Tile t -> OC block nb, class k, segment z, and its k-block range [kb0, kb1)
// over the class's (oh, ow, 64-image) positions.
struct RowWTile {
    int nb, k, z, part, owk;
    uint32_t kb0, kb1;
    __device__ RowWTile(int t, const RowWgradParams& p) {
        nb = t % p.nbs;
        part = t / p.nbs;
        k = part % p.P;
        z = part / p.P;
        owk = p.OW > k ? (p.OW - k + p.P - 1) / p.P : 0;
        const uint32_t L = uint32_t(p.OH) * uint32_t(owk) * uint32_t(p.nblk64);
        kb0 = uint32_t(uint64_t(L) * uint32_t(z) / uint32_t(p.gzc));
        kb1 = uint32_t(uint64_t(L) * uint32_t(z + 1) / uint32_t(p.gzc));
    }
};

template <int JB, int BN>
__global__ void __launch_bounds__(256, 1)
    wgrad_row_kernel(const __grid_constant__ CUtensorMap tmX, const __grid_constant__ CUtensorMap tmDY,
                     const __grid_constant__ RowWgradParams p) {
    constexpr int ROWB = JB * 2;       // MN bytes per K row of A (one filter row)
    constexpr int R = 128 / JB;        // filter rows per M-block
    constexpr int B_BYTES = BN * 128;  // BN OC x 64 images bf16
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = smem_raw + ((1024u - (ptx::smem_u32(smem_raw) & 1023u)) & 1023u);
    const int stage_bytes = p.a_bytes + B_BYTES;
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + p.stages * stage_bytes);
    uint64_t* empty = full + 8;
    uint64_t* tfull = empty + 8;
    uint64_t* tempty = tfull + 1;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 1);
    const uint32_t tmem_cols = uint32_t(p.mb * BN) <= 64 ? 64u : (uint32_t(p.mb * BN) <= 128 ? 128u : (uint32_t(p.mb * BN) <= 256 ? 256u : 512u));

    ptx::pdl_launch_dependents();
    const uint32_t warp = ptx::warp_id(), lane = ptx::lane_id();
    if (warp == 0 && lane == 0) {
        ptx::prefetch_tmap(&tmX);
        ptx::prefetch_tmap(&tmDY);
    }
    if (warp == 1 && lane == 0) {
        for (int i = 0; i < p.stages; ++i) {
            ptx::mbar_init(&full[i], 2);
            ptx::mbar_init(&empty[i], 1);
        }
        ptx::mbar_init(tfull, 1);
        ptx::mbar_init(tempty, 128);
        ptx::fence_barrier_init();
    }
    if (warp == 2) ptx::tmem_alloc(tmem_slot, tmem_cols);
    ptx::tc_fence_before();
    __syncthreads();
    ptx::tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;
    ptx::pdl_wait();

    if (warp == 0 || warp == 3) {
        // ---------------- producers: warp 0 = X rows (A, leaping access), warp 3 = dY (B)
        const bool is_b = warp == 3;
        uint32_t stage = 0, phase = 0;
        for (int t = blockIdx.x; t < p.num_tiles; t += gridDim.x) {
            const RowWTile c(t, p);
            const int nb = c.nb, dl = p.delta[c.k];
            for (uint32_t kb = c.kb0; kb < c.kb1; ++kb) {
                const int n64 = int(kb % uint32_t(p.nblk64));
                const int pos = int(kb / uint32_t(p.nblk64));
                const int oh = pos / c.owk, ow = c.k + p.P * (pos % c.owk);
                ptx::mbar_wait(&empty[stage], phase ^ 1u);
                uint8_t* st = smem + stage * stage_bytes;
                if (ptx::elect_one()) {
                    if (!is_b) {
                        ptx::mbar_arrive_expect_tx(&full[stage], uint32_t(p.FH * 64 * ROWB));
                        ptx::tma_load_4d(st, &tmX, &full[stage], (ow * p.sw - p.pw) * p.C - dl, n64 * 64,
                                         oh * p.sh - p.ph, 0);
                    } else {
                        ptx::mbar_arrive_expect_tx(&full[stage], uint32_t(B_BYTES));
#pragma unroll
                        for (int j = 0; j < BN / 64; ++j)
                            ptx::tma_load_4d(st + p.a_bytes + j * 8192, &tmDY, &full[stage], nb * BN + j * 64, ow, oh,
                                             n64 * 64);
                    }
                }
                __syncwarp();
                if (++stage == uint32_t(p.stages)) {
                    stage = 0;
                    phase ^= 1u;
                }
            }
        }
    } else if (warp == 1) {
        // ---------------- MMA issuer
        constexpr uint32_t idesc = ptx::instr_desc(128, BN, false, true, true);
        uint32_t stage = 0, phase = 0, tph = 0;
        for (int t = blockIdx.x; t < p.num_tiles; t += gridDim.x) {
            const RowWTile c(t, p);
            const uint32_t kb0 = c.kb0, kb1 = c.kb1;
            ptx::mbar_wait(tempty, tph ^ 1u);
            ptx::tc_fence_after();
            for (uint32_t kb = kb0; kb < kb1; ++kb) {
                ptx::mbar_wait(&full[stage], phase);
                ptx::tc_fence_after();
                const uint32_t sa = ptx::smem_u32(smem + stage * stage_bytes);
                const uint32_t sb = sa + uint32_t(p.a_bytes);
                if (ptx::elect_one()) {
                    for (int m = 0; m < p.mb; ++m) {
#pragma unroll
                        for (int kk = 0; kk < 4; ++kk)  // 64 images = 4 x K16
                            ptx::mma_ss<false>(
                                tmem_base + uint32_t(m * BN),
                                ptx::smem_desc_mn(sa + uint32_t(m * R * 64 * ROWB + kk * 16 * ROWB), 64 * ROWB,
                                                  8 * ROWB, ROWB),
                                ptx::smem_desc_sw128(sb + uint32_t(kk * 2048), 8192, 1024), idesc,
                                (kb > kb0 || kk > 0) ? 1u : 0u);
                    }
                    ptx::mma_commit(&empty[stage]);
                }
                __syncwarp();
                if (++stage == uint32_t(p.stages)) {
                    stage = 0;
                    phase ^= 1u;
                }
            }
            if (ptx::elect_one()) ptx::mma_commit(tfull);
            __syncwarp();
            tph ^= 1u;
        }
    } else if (warp >= 4) {
        // ---------------- epilogue: row (fh, j) of M-block m -> dW[oc][fh][j]
        const uint32_t sub = warp & 3u;
        const int jn = p.FW * p.C;
        uint32_t tph = 0;
        for (int t = blockIdx.x; t < p.num_tiles; t += gridDim.x) {
            const RowWTile c(t, p);
            const int nb = c.nb;
            const uint32_t kb0 = c.kb0, kb1 = c.kb1;
            ptx::mbar_wait(tfull, tph);
            ptx::tc_fence_after();
            for (int m = 0; m < p.mb; ++m) {
                const int g = m * 128 + int(sub * 32 + lane);
                const int fh = g / JB, j = g % JB - p.delta[c.k];  // row j' of the shifted window
                const bool ok = fh < p.FH && j >= 0 && j < jn;
                float* dst = p.out + c.part * p.part_stride + static_cast<long long>(fh) * jn + j;
#pragma unroll 1
                for (int c0 = 0; c0 < BN; c0 += 32) {
                    uint32_t r[32];
                    ptx::tmem_ld32(tmem_base + ((sub * 32u) << 16) + uint32_t(m * BN + c0), r);
                    ptx::tmem_ld_wait();
                    if (ok) {
#pragma unroll
                        for (int q = 0; q < 32; ++q) {
                            const int oc = nb * BN + c0 + q;
                            if (oc < p.OC)
                                dst[static_cast<long long>(oc) * p.FH * jn] = kb1 > kb0 ? __uint_as_float(r[q]) : 0.f;
                        }
                    }
                }
            }
            ptx::tc_fence_before();
            ptx::mbar_arrive(tempty);
            tph ^= 1u;
        }
    }
    __syncthreads();
    if (warp == 2) {
        ptx::tc_fence_after();
        ptx::tmem_dealloc(tmem_base, tmem_cols);
    }
}

}  // namespace cks
