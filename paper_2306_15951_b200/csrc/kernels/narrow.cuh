// narrow.cuh -- KB-CONV-ROW / KB-WGRAD-ROW: ConvV2 forward and Sk-dilated
// weight gradient for narrow-channel layers (FW*C <= 64 bf16 / <= 32 fp32:
// the C = 3 input layers of all three workloads) on tcgen05 tensor cores,
// BF16 (kind::f16) or TF32 (kind::tf32, fp32 storage).
//
// In NHWC the (fw, c) run of one filter row is CONTIGUOUS in X: for output
// column ow and filter row fh it is X[n][ih][(ow*sw - pw)*C + j], j = fw*C + c,
// j < FW*C.  So instead of one GEMM step per tap with a 3-of-64 used channel
// block (the generic path), a whole filter row is one K-block of JB elements
// (ROWB = JB * element bytes = 32 / 64 / 128 B) loaded by ONE TMA box
// element-addressed in the flattened (W*C) row.
//
// Column classes.  TMA box origins must be 16-byte aligned in the innermost
// dimension, while the run of column ow starts at element start = (ow*sw -
// pw)*C.  Every output column belongs to one class c with a box origin
// start + off_c (off_c = -delta, delta = start mod (16 / eb), for interior
// columns; a border column, whose window overhangs the padding, is a class
// of its own: origin 0 on the left, rowlen - 32 B * m on the right).  Box element e holds run element j = off + e.  Each CTA
// serves one class; the host lists the classes (RowClass) with the K-chunk
// range [kc0, kc1) of the box row that holds valid elements.
//
// Trimming (Alg. 1 / Alg. 3B):
//   * ConvV2, h: only the valid filter rows of an output row are loaded and
//     multiplied (T1): one TMA box per valid X row, no zero fill.
//   * ConvV2, w: MMAs run over the K chunks [kc0, kc1) of the class only;
//     a left-border column's chunk grid starts at its first valid element,
//     a right-border column's ends at the last element of the X row, so no
//     issued chunk holds a padding position (cks_padding_macs: 0 unless a
//     window overhangs BOTH ends of a row narrower than the filter).
//   * Sk-dilated, h/w: the leaping rows ih = oh*sh + fh - ph outside X arrive
//     as TMA zero fill inside an M-block (M = 128 (fh, j) rows); an M-block
//     whose filter rows are all outside X for this oh is not issued.
//
// KB-CONV-ROW  tile = R consecutive output rows x one output column x 128
//   images x OC (<= 256): D_r[n][oc] = sum_{fh valid} sum_e A_ih[n][e] *
//   B_fh[oc][e], ih = (oh0 + r)*sh - ph + fh.  An X row is loaded ONCE per
//   tile and multiplied into every accumulator r that uses it (h reuse: a
//   7x7 s2 filter reads 13 rows for 4 outputs instead of 28).  B = the class's
//   filter rows, resident in shared memory (K-major, swizzled).
// KB-WGRAD-ROW tile = OC block x segment z of the G_Z map-reduce:
//   D[(fh, e)][oc] = sum_k X[n][oh*sh+fh-ph][origin + e] * dY[n][oh][ow][oc]
//   over k = (oh, ow, n) blocks of 64 images of ONE class; both operands
//   MN-major, M = (fh, e) packed 128/JB filter rows per M-block.  Every
//   segment writes a full partial dW (zeros where the class contributes
//   nothing); KB-REDUCE sums them in a fixed order.
#pragma once
#include "ptx.cuh"
#include "../cks_plan.h"

namespace cks {

struct RowClass {
    int16_t col0, cstep, ncols;  // output columns ow = col0 + cstep * i, i < ncols
    int16_t off;                 // box origin = (ow*sw - pw)*C + off; run element j = off + e
    int8_t kc0, kc1;             // ConvV2: 32-byte K chunks of the box row with valid elements
    int16_t base, cnt;           // ConvV2: CTA range; Sk-dilated: partial (segment) range
};

struct RowFwdParams {
    const void* w;  // W [OC][FH][FW*C] (bf16 or fp32, dense, any alignment)
    float* y;       // Y [N][OH][OW][OC] fp32
    int N, H, W, C, OC, FH, FW, sh, sw, ph, pw, OH, OW;
    int nblk;       // ceil(N / 128)
    int R;          // output rows per tile
    int ncls;
    RowClass cls[kRowClasses];
    int stages;     // A ring depth (one X row per stage)
    int tma_store;  // 1: epilogue via TMA store (OC % 32 == 0)
    // Row groups (small batches, N <= 64; kernel template RG): the M = 128 rows of a tile are
    // rg_pc columns of ONE class x rg images (row r = column r / rg, image r % rg), loaded by one
    // box of the class's own tensor map (RowXMaps: dims (W*C, N, class column, H), column stride
    // cstep * sw * C) -- every column of a class shares the box origin alignment and K chunks
    int rg, rg_shift, rg_pc;
};

// Per-class X tensor maps of the row-group ConvV2 (kernel parameter space, < 4 KB in total).
struct RowXMaps {
    CUtensorMap m[kRowClasses];
};

#ifndef CKS_ROW_EPI_BUFS
#define CKS_ROW_EPI_BUFS 2  // TMA-store staging buffers per epilogue warp (2 or 4)
#endif
template <int ROWB, int BN, bool TF>
struct RowFwdShape {
    static constexpr int EB = TF ? 4 : 2;
    static constexpr int JB = ROWB / EB;           // elements per box row
    static constexpr int STAGE = 128 * ROWB;       // one X row of 128 images
    // 4 epilogue warps x 2 x (32 rows x 128 B): two TMA stores in flight per warp
    // (four measured no faster on the stem: the stores are not what bounds it)
    static constexpr int EPI_BUFS = CKS_ROW_EPI_BUFS;
    static constexpr int STAGING = 4 * EPI_BUFS * 4096;
    static constexpr int RMAX = 256 / BN < 8 ? 256 / BN : 8;  // 2 x R x BN TMEM columns <= 512
};

__host__ __device__ constexpr int row_fwd_w_bytes(int ROWB, int BN, int FH) {
    return ((FH * BN * ROWB) + 1023) / 1024 * 1024;
}

__device__ __forceinline__ int row_class_of(const RowClass* cls, int ncls, int b) {
    int k = 0;
    while (k + 1 < ncls && b >= cls[k + 1].base) ++k;
    return k;
}

// Tile t of class k: (row block ob, column i, image block nb), nb fastest.  Row groups: (row
// block, column group g of rg_pc class columns starting at class column ci0), g fastest.
template <bool RG>
struct RowFwdTile {
    int nb, ow, oh0, rn;  // rn: rows in this block
    int ci0;              // row groups: first class column of the group
    __device__ RowFwdTile(int t, const RowClass& c, const RowFwdParams& p) {
        if (RG) {
            const int ng = (c.ncols + p.rg_pc - 1) / p.rg_pc;
            nb = 0;
            ci0 = (t % ng) * p.rg_pc;
            ow = c.col0 + c.cstep * ci0;
            oh0 = (t / ng) * p.R;
        } else {
            nb = t % p.nblk;
            const int r = t / p.nblk;
            ci0 = r % c.ncols;
            ow = c.col0 + c.cstep * ci0;
            oh0 = (r / c.ncols) * p.R;
        }
        rn = min(p.R, p.OH - oh0);
    }
};
template <bool RG>
__device__ __forceinline__ int row_fwd_ntiles(const RowClass& c, const RowFwdParams& p) {
    return ((p.OH + p.R - 1) / p.R) * (RG ? (c.ncols + p.rg_pc - 1) / p.rg_pc : c.ncols * p.nblk);
}

// Shared-memory row slot of filter row fh in KB-CONV-ROW's B operand: filter rows are grouped by
// fh mod sh, each group in DECREASING fh, so the filter rows fh, fh - sh, fh - 2 sh, ... that one X
// row meets in consecutive accumulators r, r + 1, ... are consecutive BN-row blocks -- one
// N-merged MMA (N = cnt * BN) serves them all.
__host__ __device__ __forceinline__ int row_fwd_slot(int fh, int FH, int sh) {
    const int c = fh % sh;
    const int base = c * (FH / sh) + min(c, FH % sh);  // filter rows with a smaller residue
    const int nc = (FH - c + sh - 1) / sh;              // filter rows with residue c
    return base + (nc - 1 - fh / sh);
}


template <int ROWB, int BN, bool TF, bool RG = false>
__global__ void __launch_bounds__(256, 1)
    fwd_row_kernel(const __grid_constant__ CUtensorMap tmX, const __grid_constant__ CUtensorMap tmY,
                   const __grid_constant__ RowFwdParams p, const __grid_constant__ RowXMaps xm) {
    using S = RowFwdShape<ROWB, BN, TF>;
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = smem_raw + ((1024u - (ptx::smem_u32(smem_raw) & 1023u)) & 1023u);
    const int wbytes = row_fwd_w_bytes(ROWB, BN, p.FH);
    uint8_t* wsm = smem;
    uint8_t* abuf = smem + wbytes;
    uint8_t* stg = abuf + p.stages * S::STAGE;
    uint64_t* full = reinterpret_cast<uint64_t*>(stg + S::STAGING);
    uint64_t* empty = full + 16;
    uint64_t* tfull = empty + 16;
    uint64_t* tempty = tfull + 2;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);
    // per-CTA tables (no runtime divisions by s_h in the issue loops): filter-row smem slots, and
    // for d = ih - (oh0*sh - ph) the accumulator range [r0, r1) that X row ih feeds ((r0 << 4) | r1)
    uint8_t* stab = reinterpret_cast<uint8_t*>(tmem_slot + 1);  // [32]
    uint8_t* rut = stab + 32;                                    // [128]
    constexpr uint32_t TMEM_COLS = 2 * S::RMAX * BN <= 64 ? 64 : (2 * S::RMAX * BN <= 128 ? 128 : (2 * S::RMAX * BN <= 256 ? 256 : 512));

    ptx::pdl_launch_dependents();
    const uint32_t warp = ptx::warp_id(), lane = ptx::lane_id();
    const int k = row_class_of(p.cls, p.ncls, int(blockIdx.x));
    const RowClass cl = p.cls[k];
    if (warp == 0 && lane == 0) {
        ptx::prefetch_tmap(&tmX);
        if (p.tma_store) ptx::prefetch_tmap(&tmY);
        if (RG) ptx::prefetch_tmap(&xm.m[k]);
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
    __syncwarp();  // reconverge the initialising lane's warp before the block barrier
    if (warp == 2) ptx::tmem_alloc(tmem_slot, TMEM_COLS);
    for (int i = threadIdx.x; i < 32 + 128; i += blockDim.x) {
        if (i < 32) {
            stab[i] = uint8_t(i < p.FH ? row_fwd_slot(i, p.FH, p.sh) : 0);
        } else {
            const int d = i - 32;
            const int r1 = min(15, d / p.sh + 1), lo = d - p.FH + 1;
            const int r0 = lo <= 0 ? 0 : min(15, (lo + p.sh - 1) / p.sh);
            rut[d] = uint8_t((r0 << 4) | r1);
        }
    }
    ptx::pdl_wait();  // W and X may come from the previous kernel
    {   // all threads: this class's filter rows in the K-major swizzled B layout,
        // row r = fh*BN + oc, K = box element e <-> run element off + e (zero outside [0, FW*C))
        constexpr int PER16 = 16 / S::EB;
        const int jn = p.FW * p.C;
        const int chunks = p.FH * BN * (ROWB / 16);
        for (int q = threadIdx.x; q < chunks; q += blockDim.x) {
            const int r = q / (ROWB / 16), c16 = q % (ROWB / 16);
            const int fh = r / BN, oc = r % BN;
            const int rs = row_fwd_slot(fh, p.FH, p.sh) * BN + oc;  // smem row of (fh, oc)
            uint32_t v[4] = {0u, 0u, 0u, 0u};
            if (oc < p.OC) {
#pragma unroll
                for (int e = 0; e < PER16; ++e) {
                    const int j = cl.off + c16 * PER16 + e;
                    if (j >= 0 && j < jn) {
                        const long long at = (static_cast<long long>(oc) * p.FH + fh) * jn + j;
                        if constexpr (TF)
                            v[e] = static_cast<const uint32_t*>(p.w)[at];
                        else
                            v[e >> 1] |= uint32_t(static_cast<const uint16_t*>(p.w)[at]) << (16 * (e & 1));
                    }
                }
            }
            const uint32_t off = ptx::swz(uint32_t(rs * ROWB + c16 * 16), ROWB);
            *reinterpret_cast<uint4*>(wsm + off) = make_uint4(v[0], v[1], v[2], v[3]);
        }
        ptx::fence_proxy_async_smem();  // generic-proxy writes -> visible to tcgen05
    }
    ptx::tc_fence_before();
    ptx::block_sync();
    ptx::tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;
    const int ci = int(blockIdx.x) - cl.base;
    const int ntiles = row_fwd_ntiles<RG>(cl, p);

    if (warp == 0) {
        // ---------------- TMA producer: one box per VALID X row of the tile (T1 trimming)
        uint32_t s = 0, ph = 0;
        for (int t = ci; t < ntiles; t += cl.cnt) {
            const RowFwdTile<RG> tl(t, cl, p);
            const int ih0 = tl.oh0 * p.sh - p.ph;
            const int rl = max(ih0, 0), rh = min(p.H, ih0 + p.sh * (tl.rn - 1) + p.FH);
            // box origin in the flattened (W*C) row; row groups: of class column 0 (the class map's
            // column coordinate adds ci0 * cstep * sw * C)
            const int origin = ((RG ? cl.col0 : tl.ow) * p.sw - p.pw) * p.C + cl.off;
            for (int ih = rl; ih < rh; ++ih) {
                const int ru = rut[ih - ih0];
                const int r0 = ru >> 4, r1 = min(tl.rn, ru & 15);
                if (r0 >= r1) continue;  // stride gap: no output uses this row
                ptx::mbar_wait(&empty[s], ph ^ 1u);
                if (ptx::elect_one()) {
                    ptx::mbar_arrive_expect_tx(&full[s], uint32_t(S::STAGE));
                    if (RG)  // rg_pc columns x rg images of the class (column stride in the class map)
                        ptx::tma_load_4d(abuf + s * S::STAGE, &xm.m[k], &full[s], origin, 0, tl.ci0, ih);
                    else
                        ptx::tma_load_4d(abuf + s * S::STAGE, &tmX, &full[s], origin, tl.nb * 128, ih, 0);
                }
                __syncwarp();
                if (++s == uint32_t(p.stages)) {
                    s = 0;
                    ph ^= 1u;
                }
            }
        }
    } else if (warp == 1) {
        // ---------------- MMA issuer: each loaded row into every accumulator that uses it,
        // K chunks [kc0, kc1) only
        constexpr uint32_t idesc0 = ptx::instr_desc(128, 0, TF, false, false);  // N set per MMA group
        const uint32_t a0 = ptx::smem_u32(abuf), w0 = ptx::smem_u32(wsm);
        const int nkc = cl.kc1 - cl.kc0;
        const uint64_t adesc0 = ptx::smem_desc_kmajor(a0 + 32u * uint32_t(cl.kc0), ROWB);
        const uint64_t bdesc0 = ptx::smem_desc_kmajor(w0 + 32u * uint32_t(cl.kc0), ROWB);
        uint32_t s = 0, ph = 0, i = 0;
        for (int t = ci; t < ntiles; t += cl.cnt, ++i) {
            const RowFwdTile<RG> tl(t, cl, p);
            const int ih0 = tl.oh0 * p.sh - p.ph;
            const int rl = max(ih0, 0), rh = min(p.H, ih0 + p.sh * (tl.rn - 1) + p.FH);
            const uint32_t acc = i & 1u, aph = (i >> 1) & 1u;
            ptx::mbar_wait(&tempty[acc], aph ^ 1u);
            ptx::tc_fence_after();
            const uint32_t dbase = tmem_base + acc * uint32_t(S::RMAX * BN);
            uint32_t started = 0;
            for (int ih = rl; ih < rh; ++ih) {
                const int ru = rut[ih - ih0];
                const int r0 = ru >> 4, r1 = min(tl.rn, ru & 15);
                if (r0 >= r1) continue;
                ptx::mbar_wait(&full[s], ph);
                ptx::tc_fence_after();
                if (ptx::elect_one()) {
                    // descriptors built once per stage / filter row and advanced by adds (the single
                    // issuing thread's scalar work per MMA bounds this kernel: ncu, TF32 stem)
                    const uint64_t ad = adesc0 + uint64_t((s * uint32_t(S::STAGE)) >> 4);
                    // accumulators [r0, r1) meet filter rows fh0, fh0 - sh, ...: consecutive B blocks
                    // (row_fwd_slot).  The started ones form a prefix (outputs start in row order):
                    // at most two N-merged MMA groups per K chunk, accumulate / overwrite.
                    const int slot0 = stab[ih - ih0 - r0 * p.sh];
                    int rsd = r0;
                    while (rsd < r1 && ((started >> rsd) & 1u)) ++rsd;
#pragma unroll
                    for (int grp = 0; grp < 2; ++grp) {
                        const int ga = grp == 0 ? r0 : rsd, gb = grp == 0 ? rsd : r1;
                        if (gb <= ga) continue;
                        const uint64_t bd = bdesc0 + uint64_t(uint32_t((slot0 + ga - r0) * BN * ROWB) >> 4);
                        const uint32_t d = dbase + uint32_t(ga * BN);
                        const uint32_t idesc = idesc0 | ((uint32_t((gb - ga) * BN) >> 3) << 17);
#pragma unroll
                        for (int k = 0; k < ROWB / 32; ++k)  // 32-byte K chunks [kc0, kc1) of the class
                            if (k < nkc)
                                ptx::mma_ss<TF>(d, ad + uint64_t(2 * k), bd + uint64_t(2 * k), idesc,
                                                (grp == 0 || k > 0) ? 1u : 0u);
                    }
                    ptx::mma_commit(&empty[s]);
                }
                __syncwarp();
                started |= ((1u << r1) - 1u) & ~((1u << r0) - 1u);
                if (++s == uint32_t(p.stages)) {
                    s = 0;
                    ph ^= 1u;
                }
            }
            if (ptx::elect_one()) ptx::mma_commit(&tfull[acc]);
            __syncwarp();
        }
    } else if (warp >= 4) {
        // ---------------- epilogue: TMEM -> registers -> (swizzled staging -> TMA store | direct stores)
        const uint32_t sub = warp & 3u;
        uint8_t* my = stg + sub * S::EPI_BUFS * 4096;
        uint32_t i = 0, q = 0;
        for (int t = ci; t < ntiles; t += cl.cnt, ++i) {
            const RowFwdTile<RG> tl(t, cl, p);
            const uint32_t acc = i & 1u, aph = (i >> 1) & 1u;
            ptx::mbar_wait(&tfull[acc], aph);
            ptx::tc_fence_after();
            // M row -> (column, image).  Row groups (rg >= 32): the warp's 32 rows are 32 images of
            // one class column; columns past the class's last are computed but never stored
            const int wci = RG ? tl.ci0 + (int(sub * 32) >> p.rg_shift) : tl.ci0;
            const bool wlive = !RG || wci < cl.ncols;
            const int wow = cl.col0 + cl.cstep * wci;
            const int n0 = RG ? (int(sub * 32) & (p.rg - 1)) : tl.nb * 128 + int(sub * 32);
            const int n = n0 + int(lane);
            for (int r = 0; r < tl.rn; ++r) {
                const int oh = tl.oh0 + r;
#pragma unroll 1
                for (int c0 = 0; c0 < BN; c0 += 32) {
                    if (c0 >= p.OC) break;
                    uint32_t v[32];
                    ptx::tmem_ld32(tmem_base + ((sub * 32u) << 16) + acc * uint32_t(S::RMAX * BN) + uint32_t(r * BN + c0), v);
                    ptx::tmem_ld_wait();
                    if (!wlive) continue;  // warp-uniform
                    if (p.tma_store) {
                        uint8_t* buf = my + (q++ & uint32_t(S::EPI_BUFS - 1)) * 4096;
                        if (ptx::elect_one()) {  // buffer of chunk q - EPI_BUFS drained
                            if constexpr (S::EPI_BUFS == 4)
                                ptx::bulk_wait_read3();
                            else
                                ptx::bulk_wait_read1();
                        }
                        __syncwarp();
#pragma unroll
                        for (int c = 0; c < 8; ++c)
                            *reinterpret_cast<uint4*>(buf + ptx::swz(lane * 128u + c * 16u, 128)) =
                                make_uint4(v[4 * c], v[4 * c + 1], v[4 * c + 2], v[4 * c + 3]);
                        ptx::fence_proxy_async_smem();
                        __syncwarp();
                        if (ptx::elect_one()) {
                            ptx::tma_store_4d(&tmY, buf, c0, wow, oh, n0);
                            ptx::bulk_commit();
                        }
                        __syncwarp();
                    } else if (n < p.N) {
                        float* dst = p.y + ((static_cast<long long>(n) * p.OH + oh) * p.OW + wow) * p.OC;
#pragma unroll
                        for (int j = 0; j < 32; ++j)
                            if (c0 + j < p.OC) dst[c0 + j] = __uint_as_float(v[j]);
                    }
                }
            }
            ptx::tc_fence_before();
            ptx::mbar_arrive(&tempty[acc]);
        }
        if (p.tma_store && ptx::elect_one()) ptx::bulk_wait_read0();
        __syncwarp();
    }
    ptx::block_sync();
    if (warp == 2) {
        ptx::tc_fence_after();
        ptx::tmem_dealloc(tmem_base, TMEM_COLS);
    }
}

// ------------------------------------------------------------------ wgrad
struct RowWgradParams {
    float* out;  // dW [OC][FH][FW*C] (one partial) or partials [gz][OC][FH][FW*C]
    long long part_stride;
    int N, H, W, C, OC, FH, FW, sh, sw, ph, pw, OH, OW;
    int mb;       // M-blocks of 128 (fh, e) rows
    int nbs;      // OC blocks of BN
    int ncls;
    RowClass cls[kRowClasses];  // base / cnt: partial (segment) range of the class
    int gz;       // total segments (partials)
    int nblk64;   // ceil(N / 64)
    int num_tiles;  // nbs * gz
    int stages;
    int a_bytes;  // A region: ((q - 1) * sh + mb * R) filter-row atoms of 64 images
    // q output rows per k-block (round 2): ONE X box of xrows = FH + sh * (q - 1) rows serves the
    // q rows' M-blocks (row oh0 + i starts at atom i * sh), so the X rows shared by neighbouring
    // output rows cross L2 -> SM once per k-block instead of once per output row
    int q, xrows;
    // Row groups (small batches, kernel template RG): a k-block is rg_pk class columns x rg images
    // (64 K rows, column-major), both operands from per-class maps (RowWXMaps) with a column dim
    int rg, rg_pk;
};

// Per-class X and dY tensor maps of the row-group Sk-dilated (kernel parameter space).
constexpr int kRowWgradRgClasses = 12;
struct RowWXMaps {
    CUtensorMap x[kRowWgradRgClasses], dy[kRowWgradRgClasses];
};
template <bool RG>
__device__ __forceinline__ int row_wgrad_cols(const RowClass& c, const RowWgradParams& p) {
    return RG ? (c.ncols + p.rg_pk - 1) / p.rg_pk : c.ncols;  // k-block column units of a class
}

// Tile t -> OC block nb, segment (partial) part of class k, its k-block range
// [kb0, kb1) over the class's (oh, column, 64-image) positions (row groups: column chunks).
template <bool RG>
struct RowWTile {
    int nb, k, part;
    uint32_t kb0, kb1;
    __device__ RowWTile(int t, const RowWgradParams& p) {
        nb = t % p.nbs;
        part = t / p.nbs;
        k = row_class_of(p.cls, p.ncls, part);
        const int z = part - p.cls[k].base, gzc = p.cls[k].cnt;
        const uint32_t L =
            uint32_t((p.OH + p.q - 1) / p.q) * uint32_t(row_wgrad_cols<RG>(p.cls[k], p)) * uint32_t(p.nblk64);
        kb0 = uint32_t(uint64_t(L) * uint32_t(z) / uint32_t(gzc));
        kb1 = uint32_t(uint64_t(L) * uint32_t(z + 1) / uint32_t(gzc));
    }
};

// M-blocks (R filter rows each) holding at least one filter row that is inside X for output row oh
__device__ __forceinline__ uint32_t row_wgrad_mmask(int oh, int R, const RowWgradParams& p) {
    const int ih0 = oh * p.sh - p.ph;
    const int fs = max(-ih0, 0), fe = min(p.H - ih0, p.FH);
    uint32_t m = 0;
    for (int b = 0; b < p.mb; ++b)
        if (b * R < fe && (b + 1) * R > fs) m |= 1u << b;
    return m;
}

template <int ROWB, int BN, bool TF, bool RG = false>
__global__ void __launch_bounds__(256, 1)
    wgrad_row_kernel(const __grid_constant__ CUtensorMap tmX, const __grid_constant__ CUtensorMap tmDY,
                     const __grid_constant__ RowWgradParams p, const __grid_constant__ RowWXMaps xm) {
    constexpr int EB = TF ? 4 : 2;
    constexpr int JB = ROWB / EB;       // MN elements per filter row of A
    constexpr int R = 128 / JB;         // filter rows per M-block
    constexpr int CH = 128 / EB;        // dY channels per 128-byte box
    constexpr int B_BYTES = BN * 64 * EB;  // BN OC x 64 images
    constexpr int UK = 32 / EB;         // images per MMA K step
    static_assert(!TF || ROWB == 128, "TF32 MN-major operands use the 128-byte (BASE32B) swizzle");
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = smem_raw + ((1024u - (ptx::smem_u32(smem_raw) & 1023u)) & 1023u);
    const int stage_bytes = p.a_bytes + p.q * B_BYTES;
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
    __syncwarp();  // reconverge the initialising lane's warp before the block barrier
    if (warp == 2) ptx::tmem_alloc(tmem_slot, tmem_cols);
    ptx::tc_fence_before();
    ptx::block_sync();
    ptx::tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;
    ptx::pdl_wait();

    if (warp == 0 || warp == 3) {
        // ---------------- producers: warp 0 = X rows (A, leaping access), warp 3 = dY (B)
        const bool is_b = warp == 3;
        const uint64_t pol = is_b ? ptx::l2_policy_evict_first() : ptx::l2_policy_evict_last();
        uint32_t stage = 0, phase = 0;
        for (int t = blockIdx.x; t < p.num_tiles; t += gridDim.x) {
            const RowWTile<RG> c(t, p);
            const RowClass cl = p.cls[c.k];
            for (uint32_t kb = c.kb0; kb < c.kb1; ++kb) {
                const int n64 = int(kb % uint32_t(p.nblk64));
                const int pos = int(kb / uint32_t(p.nblk64));
                const int cu = row_wgrad_cols<RG>(cl, p);
                const int ci0 = (pos % cu) * (RG ? p.rg_pk : 1);  // first class column of the k-block
                const int oh0 = (pos / cu) * p.q, ow = cl.col0 + cl.cstep * ci0;
                const int nq = min(p.q, p.OH - oh0);
                ptx::mbar_wait(&empty[stage], phase ^ 1u);
                uint8_t* st = smem + stage * stage_bytes;
                if (ptx::elect_one()) {
                    // X boxes overlap across neighbouring columns and rows (FW*C-wide runs at
                    // stride sw*C, FH rows at stride sh) and are re-read: keep them in L2 ahead of
                    // dY, which is read once (L2 eviction priorities)
                    if (!is_b) {
                        ptx::mbar_arrive_expect_tx(&full[stage], uint32_t(p.xrows * 64 * ROWB));
                        if (RG)  // rg_pk class columns x rg images (origin of class column 0 + column dim)
                            ptx::tma_load_4d_hint(st, &xm.x[c.k], &full[stage], (cl.col0 * p.sw - p.pw) * p.C + cl.off,
                                                  0, ci0, oh0 * p.sh - p.ph, pol);
                        else
                            ptx::tma_load_4d_hint(st, &tmX, &full[stage], (ow * p.sw - p.pw) * p.C + cl.off, n64 * 64,
                                                  oh0 * p.sh - p.ph, 0, pol);
                    } else {
                        ptx::mbar_arrive_expect_tx(&full[stage], uint32_t(nq * B_BYTES));
                        for (int i = 0; i < nq; ++i)
#pragma unroll
                            for (int j = 0; j < BN / CH; ++j) {
                                if (RG)
                                    ptx::tma_load_4d_hint(st + p.a_bytes + i * B_BYTES + j * 8192, &xm.dy[c.k],
                                                          &full[stage], c.nb * BN + j * CH, 0, ci0, oh0 + i, pol);
                                else
                                    ptx::tma_load_4d_hint(st + p.a_bytes + i * B_BYTES + j * 8192, &tmDY, &full[stage],
                                                          c.nb * BN + j * CH, ow, oh0 + i, n64 * 64, pol);
                            }
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
        constexpr uint32_t idesc = ptx::instr_desc(128, BN, TF, true, true);
        const uint32_t s0 = ptx::smem_u32(smem);
        const uint64_t adesc0 = TF ? ptx::smem_desc_mn_b32(s0, 64 * ROWB, 512) : ptx::smem_desc_mn(s0, 64 * ROWB, 8 * ROWB, ROWB);
        const uint64_t bdesc0 = TF ? ptx::smem_desc_mn_b32(s0, 8192, 512) : ptx::smem_desc_sw128(s0, 8192, 1024);
        uint32_t stage = 0, phase = 0, tph = 0;
        for (int t = blockIdx.x; t < p.num_tiles; t += gridDim.x) {
            const RowWTile<RG> c(t, p);
            const RowClass cl = p.cls[c.k];
            ptx::mbar_wait(tempty, tph ^ 1u);
            ptx::tc_fence_after();
            uint32_t started = 0;
            for (uint32_t kb = c.kb0; kb < c.kb1; ++kb) {
                const int oh0 = (int(kb / uint32_t(p.nblk64)) / row_wgrad_cols<RG>(cl, p)) * p.q;
                const int nq = min(p.q, p.OH - oh0);
                uint32_t mmq = 0;  // M-blocks issued in this k-block (any of its output rows)
                for (int i = 0; i < nq; ++i) mmq |= row_wgrad_mmask(oh0 + i, R, p);
                ptx::mbar_wait(&full[stage], phase);
                ptx::tc_fence_after();
                const uint32_t sa = ptx::smem_u32(smem + stage * stage_bytes);
                const uint32_t sb = sa + uint32_t(p.a_bytes);
                if (ptx::elect_one()) {
                    uint32_t st_loc = started;
                    for (int i = 0; i < nq; ++i) {
                        const uint32_t mm = row_wgrad_mmask(oh0 + i, R, p);
                        for (int m = 0; m < p.mb; ++m) {
                            if (!((mm >> m) & 1u)) continue;  // all filter rows of the block outside X
                            const uint32_t acc0 = (st_loc >> m) & 1u;
                            // output row oh0 + i: filter row fh = X box row i*sh + fh
                            // descriptors advanced by adds (start-address field, 16-byte units)
                            const uint64_t ad = adesc0 + uint64_t((sa - s0 + uint32_t((i * p.sh + m * R) * 64 * ROWB)) >> 4);
                            const uint64_t bd = bdesc0 + uint64_t((sb - s0 + uint32_t(i * B_BYTES)) >> 4);
#pragma unroll
                            for (int kk = 0; kk < 64 / UK; ++kk)
                                ptx::mma_ss<TF>(tmem_base + uint32_t(m * BN), ad + uint64_t((kk * UK * ROWB) >> 4),
                                                bd + uint64_t((kk * UK * 128) >> 4), idesc, (acc0 | uint32_t(kk)) != 0);
                        }
                        st_loc |= mm;
                    }
                    ptx::mma_commit(&empty[stage]);
                }
                __syncwarp();
                started |= mmq;
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
        // ---------------- epilogue: row (fh, e) of M-block m -> dW[oc][fh][off + e];
        // run elements outside the class's box window are written as 0 (full partial)
        const uint32_t sub = warp & 3u;
        const int jn = p.FW * p.C;
        uint32_t tph = 0;
        for (int t = blockIdx.x; t < p.num_tiles; t += gridDim.x) {
            const RowWTile<RG> c(t, p);
            const RowClass cl = p.cls[c.k];
            const int nb = c.nb;
            uint32_t started = 0;  // M-blocks that received an MMA (the same walk as the issuer)
            for (uint32_t kb = c.kb0; kb < c.kb1;) {
                const int pos = int(kb / uint32_t(p.nblk64));
                const int oh0 = (pos / row_wgrad_cols<RG>(cl, p)) * p.q;
                for (int i = 0; i < p.q && oh0 + i < p.OH; ++i) started |= row_wgrad_mmask(oh0 + i, R, p);
                kb = uint32_t(pos + 1) * uint32_t(p.nblk64);  // next position
            }
            ptx::mbar_wait(tfull, tph);
            ptx::tc_fence_after();
            float* part = p.out + c.part * p.part_stride;
            for (int m = 0; m < p.mb; ++m) {
                const int g = m * 128 + int(sub * 32 + lane);
                const int fh = g / JB, j = g % JB + cl.off;
                const bool ok = fh < p.FH && j >= 0 && j < jn;
                const bool live = (started >> m) & 1u;
                float* dst = part + static_cast<long long>(fh) * jn + j;
#pragma unroll 1
                for (int c0 = 0; c0 < BN; c0 += 32) {
                    uint32_t r[32];
                    ptx::tmem_ld32(tmem_base + ((sub * 32u) << 16) + uint32_t(m * BN + c0), r);
                    ptx::tmem_ld_wait();
                    if (ok) {
#pragma unroll
                        for (int q = 0; q < 32; ++q) {
                            const int oc = nb * BN + c0 + q;
                            if (oc < p.OC) dst[static_cast<long long>(oc) * p.FH * jn] = live ? __uint_as_float(r[q]) : 0.f;
                        }
                    }
                }
            }
            // run elements j outside [off, off + JB): no D row, the class contributes 0
            {
                const int jlo = max(cl.off, 0), jhi = min(cl.off + JB, jn);
                const int nz = jlo + (jn - jhi);
                const int ocn = min(BN, p.OC - nb * BN);
                for (int q = int(threadIdx.x) - 128; q < p.FH * nz * ocn; q += 128) {
                    const int oc = nb * BN + q / (p.FH * nz), rr = q % (p.FH * nz);
                    const int fh = rr / nz, jj = rr % nz;
                    const int j = jj < jlo ? jj : jhi + (jj - jlo);
                    part[(static_cast<long long>(oc) * p.FH + fh) * jn + j] = 0.f;
                }
            }
            ptx::tc_fence_before();
            ptx::mbar_arrive(tempty);
            tph ^= 1u;
        }
    }
    ptx::block_sync();
    if (warp == 2) {
        ptx::tc_fence_after();
        ptx::tmem_dealloc(tmem_base, tmem_cols);
    }
}

}  // namespace cks
