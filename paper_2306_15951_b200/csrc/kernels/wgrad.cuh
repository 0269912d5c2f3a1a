// wgrad.cuh -- KB-WGRAD: Sk-dilated-V2 weight gradient (Alg. 3/3B)
// on tcgen05 tensor cores with the G_Z map-reduce of P:210.
//
// Per filter tap (fh, fw) the weight gradient is a GEMM
//   dW[oc][ic] (tap) = sum_k dY[k][oc] * X[gather(k)][ic],
//   k = (oh, ow, n) over the TRIMMED range [oh_s, oh_e) x [ow_s, ow_e) x N
// (T3, reading c5) -- the filter dY is read densely (no inserted zeros) and
// X with LEAPING access ih = oh*sh + fh - ph, iw = ow*sw + fw - pw (P:196-206,
// Fig. 7).  In NHWC both operands have the reduction axis strided and the
// channel axis contiguous, so both are MN-major: a k-block is 64 images at
// one (oh, ow), loaded by TMA 4-D boxes (64 ch, 1, 1, 64 images) into the
// 128B-swizzled MN-major canonical layout (64-channel atoms, LBO = 8 KB
// between atoms, SBO = 1 KB between 8-row K groups).
//
// Tile = (tap, OC block of 128, IC block of BN, segment z of G_Z).  Segment z
// covers k-blocks [z*L/G_Z, (z+1)*L/G_Z) of the tap's L k-blocks; with G_Z > 1
// each segment writes fp32 partials that KB-REDUCE sums in a fixed order
// ("the results obtained from each segment are aggregated").
//
// Row tiles (MT = F_W taps per tile, narrow-IC layers): a tile is one filter
// ROW fh and all its F_W taps, each with its own TMEM accumulator; a k-block
// loads the dY block ONCE and the F_W leaping X columns iw = ow*sw + fw - pw,
// so the dY operand is shared by F_W MMAs (1/F_W of its L2->SM traffic).  The
// k range is the union of the taps' trimmed ow ranges; a tap whose ow is
// outside its own range [ow_s(fw), ow_e(fw)) (T3) neither loads nor multiplies
// (trimming stays exact).  Only the valid rows of the dY block (O_C channels)
// are loaded; accumulator rows >= O_C are never stored.
//
// Filter-row clusters (TC = F_H row tiles, round 2): the F_H row tiles of one
// segment form a thread-block cluster that walks the UNION of the filter rows'
// trimmed oh ranges in lockstep; cluster rank 0 loads each dY block once and
// multicasts it to the F_H CTAs (a filter row outside its own oh range neither
// loads X nor multiplies, so trimming stays exact), and every CTA's MMA commit
// releases the stage in all of them.  dY then crosses L2 -> SM once per
// segment instead of F_H times and the CTAs that share it stay in step (DRAM
// re-reads of dY / X between filter rows: ncu showed 2.7x the algorithmic
// bytes on the ResNet l1 layers without it).
//
// Position pairs (PP, round 2; F_W = 3, s_w = 1, O_C <= 64, I_C <= 64): the
// MMA's M = 128 holds the dY of TWO neighbouring output positions (ow, ow+1,
// 64 channels each) and each of the four X columns iw = ow - pw + j
// (j = 0..3) is ONE MMA: rows 0-63 accumulate tap j of position ow, rows
// 64-127 tap j-1 of position ow+1 -- every X column that both positions
// read is multiplied once, and no A row is idle (the plain row tile leaves
// the 64 upper M rows unused with O_C = 64).  Tap fw's sum is then
// D_fw[0:64] + D_{fw+1}[64:128]; the two halves are written as two G_Z
// partials (slots 2z, 2z+1) that KB-REDUCE adds in fixed order.  A column
// outside X is skipped for both halves (exact trimming).
#pragma once
#include "ptx.cuh"

namespace cks {

struct WgradParams {
    int16_t oh_s[32], oh_e[32], ow_s[32], ow_e[32];  // T3 per tap row / column
    // 3-D: T3 of the depth axis per filter depth, and the
    // row extents per depth slice of dY (OH) and X (H): rows are flattened
    // d * rows + h.  2-D: FD = 1, [od_s, od_e) = [0, 1), sd = 1, pd = 0.
    int16_t od_s[32], od_e[32];
    int FD, sd, pd, OHr, Hr;
    int ouw_s, ouw_e;       // row tiles: union of the taps' ow ranges
    float* out;             // dW (gz == 1) or partials [gz][OC][FH*FW][C]
    int FH, FW, sh, sw, ph, pw;
    int N, OC, C;
    int mblocks, nbs, gz, nblk64;  // nblk64: image blocks of KIMG (64 or 128) images
    long long num_tiles;
    long long part_stride;  // OC*FH*FW*C
    int zc;                 // cluster reduce: the gz segments of one tile are the gz CTAs of one cluster;
                            // partials staged in smem, summed in fixed order through DSMEM into dW
    int tc;                 // filter-row group size (F_H; 0/1 = off), row tiles only: the group's tiles walk
                            // the union oh range with identical segments (adjacent tiles)
    int tcmc;               // 1: the group is a cluster and rank 0 multicasts each dY block
    int pp;                 // position pairs (MT = 4 X columns per k-block of two positions)
    int Wx;                 // X width (position pairs: column range check)
    int ouh_s, ouh_e;       // filter-row clusters: union of the filter rows' oh ranges
    // Row groups (small batches): a k-block is rg_pk consecutive output positions x rg images
    // (position-major K rows; boxes over (C, N, W, H) maps); a tap multiplies only the K rows of
    // its valid positions.  rg = 0: k-blocks of KIMG images at one position (rg_pk = 1).
    int rg, rg_pk;
    int stag;  // filter-row groups, s_h = 1: staggered walk (the group shares X rows instead of dY rows)
};

// One TMA box = 128 B of channels x 64 images (64 bf16 / 32 fp32 channels):
// an MN-major swizzle atom column.  BF16: SWIZZLE_128B (16 B chunks, 8-row
// K groups, SBO 1 KB).  TF32: SWIZZLE_128B_BASE32B (32 B chunks, 4-row K
// groups, SBO 512 B) -- the MN-major layout tcgen05 kind::tf32 requires.
// A1: O_C <= 64 -- the stage holds only the dY atoms of 64 channels (one bf16
// atom, two tf32 atoms); the MMA's other 64 A rows read the stage's first X
// block (garbage rows of D, never stored), so the ring carries one more stage
// instead of zero-filled atoms.
template <int BN, bool kTF32 = false, int KIMG = 64, int MT = 1, bool A1 = false, bool PP = false>
struct WgradShape {
    static constexpr int EB = kTF32 ? 4 : 2;
    static constexpr int CH = 128 / EB;                 // channels per box
    static constexpr int ATOM = KIMG * 128;             // one box: 128 B of channels x KIMG images
    static constexpr int A_BYTES = (128 / CH) * ATOM;   // 128 OC x KIMG images
    static constexpr int B_BYTES = (BN / CH) * ATOM;    // BN IC x KIMG images
    static constexpr int UK = 32 / EB;                  // K (images) per MMA
    static constexpr int KSTEP = UK * 128;              // bytes per MMA K step
    // dY bytes reserved per stage (A1: 64 OC; position pairs: 64 OC of two positions = M 128)
    static constexpr int A_STAGE = PP ? 2 * (64 / CH) * ATOM : (A1 ? (64 / CH) * ATOM : A_BYTES);
    static constexpr int STAGE_BYTES = A_STAGE + MT * B_BYTES;
    static constexpr int STAGES = (200 * 1024 / STAGE_BYTES) > 8 ? 8 : (200 * 1024 / STAGE_BYTES);
    static constexpr int SMEM_BYTES = STAGES * STAGE_BYTES + 1024 + 256;
    // accumulator buffers: two (the epilogue of a tile overlaps the next tile's MMAs) when
    // they fit TMEM, else one (BN = 128 row tiles: long K loops, the epilogue is short)
    static constexpr int NACC = 2 * MT * BN <= 512 ? 2 : 1;
    static constexpr uint32_t TMEM_COLS = NACC * MT * BN <= 128 ? 128 : NACC * MT * BN <= 256 ? 256 : 512;
    static_assert(MT * BN <= 512, "the accumulators of MT taps must fit TMEM");
};

struct WTile {
    int nb, mb, z, fh, fw, fd;
    int kb0, kb1;  // k-block range of this segment
    int wn, hn;    // ow / oh extents (wn: k-block columns -- positions, pairs or position chunks)
    int wr;        // ow positions of the tile's (union) range
    int ohs, ows, ods;
};

template <int MT, bool RG = false>
__device__ __forceinline__ WTile wdecode(long long t64, const WgradParams& p) {
    WTile c;
    uint32_t t = uint32_t(t64);  // 32-bit decode (64-bit div/mod is slow)
    int tcr = 0;                 // filter-row cluster: rank = filter row (fastest)
    if (p.tc > 1) {
        tcr = int(t % uint32_t(p.tc));
        t /= uint32_t(p.tc);
    }
    if (p.zc) {  // segments fastest: the gz CTAs of a cluster share (tap, mb, nb)
        c.z = int(t % uint32_t(p.gz));
        t /= uint32_t(p.gz);
    }
    c.nb = int(t % uint32_t(p.nbs));
    t /= uint32_t(p.nbs);
    c.mb = int(t % uint32_t(p.mblocks));
    t /= uint32_t(p.mblocks);
    if (!p.zc) {
        c.z = int(t % uint32_t(p.gz));
        t /= uint32_t(p.gz);
    }
    const int tap = p.tc > 1 ? int(t) * p.tc + tcr : int(t);
    const int fdh = MT > 1 ? tap : tap / p.FW;  // filter (depth, row)
    c.fd = fdh / p.FH;
    c.fh = fdh - c.fd * p.FH;
    c.fw = MT > 1 ? 0 : tap % p.FW;
    // filter-row groups walk the union oh range in lockstep; staggered (s_h = 1): filter row fh
    // runs oh = t - fh at step t, so the group's CTAs read the SAME X row (ih = t - ph) together
    c.ohs = p.tc > 1 ? p.ouh_s - (p.stag ? c.fh : 0) : p.oh_s[c.fh];
    c.ods = p.od_s[c.fd];
    c.ows = MT > 1 ? p.ouw_s : p.ow_s[c.fw];
    const int hn = p.tc > 1 ? p.ouh_e - p.ouh_s + (p.stag ? p.tc - 1 : 0) : p.oh_e[c.fh] - c.ohs;
    const int wn = (MT > 1 ? p.ouw_e : p.ow_e[c.fw]) - c.ows;
    const int dn = p.od_e[c.fd] - c.ods;
    c.wn = p.pp ? wn / 2 : (RG ? (wn + p.rg_pk - 1) / p.rg_pk : wn);  // pairs (host: wn even) / chunks
    c.wr = wn;
    c.hn = hn;
    const uint32_t L = uint32_t(max(dn, 0)) * uint32_t(max(hn, 0)) * uint32_t(max(c.wn, 0)) * uint32_t(p.nblk64);
    c.kb0 = int(uint64_t(L) * uint32_t(c.z) / uint32_t(p.gz));
    c.kb1 = int(uint64_t(L) * uint32_t(c.z + 1) / uint32_t(p.gz));
    return c;
}

// row tiles: does tap fw see any k-block of the segment (else its partial is 0)?
template <bool RG>
__device__ __forceinline__ bool tap_has_work(const WTile& c, const WgradParams& p, int fw) {
    const int rpk = RG ? p.rg_pk : 1;  // positions per k-block
    if (c.kb1 <= c.kb0 || c.wn <= 0) return false;
    if (p.tc > 1) {  // union oh range: walk the segment's positions (this filter row's oh, the tap's ow)
        const int p0 = c.kb0 / p.nblk64, p1 = (c.kb1 - 1) / p.nblk64;
        for (int q = p0; q <= p1; ++q) {
            const int pq = q / c.wn;
            const int oh = c.ohs + (pq % c.hn), ow = c.ows + rpk * (q - pq * c.wn);
            if (oh >= p.oh_s[c.fh] && oh < p.oh_e[c.fh] && ow < p.ow_e[fw] && ow + rpk > p.ow_s[fw]) return true;
        }
        return false;
    }
    const int s = p.ow_s[fw] - c.ows, e = p.ow_e[fw] - c.ows;  // tap range, relative to the union start
    if (e <= s) return false;
    const int p0 = c.kb0 / p.nblk64, p1 = (c.kb1 - 1) / p.nblk64;
    if (p1 - p0 + 1 >= c.wn) return true;  // the segment covers every ow
    for (int q = p0; q <= p1; ++q) {
        const int w = (q % c.wn) * rpk;  // first position of the k-block (row groups: of the chunk)
        if (w < e && w + rpk > s) return true;
    }
    return false;
}

// position pairs: does X column j (iw = ow0 - pw + j) of any k-block of the segment lie in X?
__device__ __forceinline__ bool pp_col_has_work(const WTile& c, const WgradParams& p, int j) {
    if (c.kb1 <= c.kb0 || c.wn <= 0) return false;
    const int p0 = c.kb0 / p.nblk64, p1 = (c.kb1 - 1) / p.nblk64;
    for (int q = p0; q <= p1; ++q) {
        const int pq = q / c.wn;
        const int ow0 = c.ows + 2 * (q - pq * c.wn), oh = c.ohs + (pq % c.hn);
        const int iw = ow0 - p.pw + j;
        if (iw >= 0 && iw < p.Wx && (p.tc <= 1 || (oh >= p.oh_s[c.fh] && oh < p.oh_e[c.fh]))) return true;
    }
    return false;
}

template <int BN, bool kTF32 = false, int KIMG = 64, int MT = 1, bool A1 = false, bool PP = false, bool RG = false>
__global__ void __launch_bounds__(256, 1)
    wgrad_kernel(const __grid_constant__ CUtensorMap tmDY, const __grid_constant__ CUtensorMap tmX,
                 const __grid_constant__ WgradParams p) {
    using S = WgradShape<BN, kTF32, KIMG, MT, A1, PP>;
    static_assert(!(PP && RG), "position pairs and row groups exclude each other");
    // row groups (compile-time: the batch-as-K kernels keep their exact issue sequence)
    const int rpk = RG ? p.rg_pk : 1;
    static_assert(!PP || (MT == 4 && A1 && BN == 64), "position pairs: 4 X columns, 64 OC, 64 IC");
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = smem_raw + ((1024u - (ptx::smem_u32(smem_raw) & 1023u)) & 1023u);
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + S::STAGES * S::STAGE_BYTES);
    uint64_t* empty = full + S::STAGES;
    uint64_t* tfull = empty + S::STAGES;
    uint64_t* tempty = tfull + 2;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);

    ptx::pdl_launch_dependents();
    const uint32_t warp = ptx::warp_id(), lane = ptx::lane_id();
    if (warp == 0 && lane == 0) {
        ptx::prefetch_tmap(&tmDY);
        ptx::prefetch_tmap(&tmX);
    }
    if (warp == 1 && lane == 0) {
        for (int i = 0; i < S::STAGES; ++i) {
            ptx::mbar_init(&full[i], 2);  // A producer + B producer
            ptx::mbar_init(&empty[i], p.tcmc ? p.tc : 1);  // filter-row cluster: every CTA's MMA commit
        }
        for (int i = 0; i < 2; ++i) {
            ptx::mbar_init(&tfull[i], 1);
            ptx::mbar_init(&tempty[i], 128);
        }
        ptx::fence_barrier_init();
    }
    __syncwarp();  // reconverge the initialising lane's warp before the block barrier
    if (warp == 2) ptx::tmem_alloc(tmem_slot, S::TMEM_COLS);
    ptx::tc_fence_before();
    ptx::block_sync();
    if (p.tcmc) ptx::cluster_sync();  // peers' barriers exist before the first multicast / remote commit
    ptx::tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;
    const uint32_t tcrank = p.tc > 1 ? blockIdx.x % uint32_t(p.tc) : 0u;
    const uint16_t tcmask = uint16_t((1u << (p.tcmc ? p.tc : 1)) - 1u);
    ptx::pdl_wait();  // inputs of this op may come from the previous kernel

    if (warp == 0 || warp == 3) {
        // ---------------- TMA producers (whole warp walks the uniform schedule,
        // one elected lane issues): warp 0 loads dY (A, 2 OC chunks), warp 3
        // loads X (B, BN/64 IC chunks) with the leaping row ih = oh*sh + fh - ph
        const bool is_b = warp == 3;
        uint32_t stage = 0, phase = 0;
        for (long long t = blockIdx.x; t < p.num_tiles; t += gridDim.x) {
            const WTile c = wdecode<MT, RG>(t, p);
            for (int kb = c.kb0; kb < c.kb1; ++kb) {
                const int n64 = kb % p.nblk64;
                const int pos = kb / p.nblk64;
                const int pq = pos / c.wn;
                const int ow = c.ows + (PP ? 2 : rpk) * (pos - pq * c.wn);  // pairs / chunks: first position
                const int dq = pq / c.hn;
                const int oh = c.ohs + (pq - dq * c.hn), od = c.ods + dq;
                // filter-row clusters walk the union oh range: rows outside this filter row's own range
                const bool ohok = p.tc <= 1 || (oh >= p.oh_s[c.fh] && oh < p.oh_e[c.fh]);
                ptx::mbar_wait(&empty[stage], phase ^ 1);
                uint8_t* sa = smem + stage * S::STAGE_BYTES;
                if (ptx::elect_one()) {
                    if (PP && !is_b) {  // dY of positions ow, ow+1: 64 channels each (M rows 0-63, 64-127)
                        ptx::mbar_arrive_expect_tx(&full[stage], uint32_t(S::A_STAGE));
#pragma unroll
                        for (int q = 0; q < 2; ++q)
#pragma unroll
                            for (int j = 0; j < 64 / S::CH; ++j)
                                ptx::tma_load_4d(sa + (q * (64 / S::CH) + j) * S::ATOM, &tmDY, &full[stage], j * S::CH,
                                                 ow + q, od * p.OHr + oh, n64 * KIMG);
                    } else if (PP) {  // X columns iw = ow - pw + j, j = 0..3 (outside X: neither loaded nor used)
                        const int ih = (od * p.sd + c.fd - p.pd) * p.Hr + oh * p.sh + c.fh - p.ph;
                        uint32_t nv = 0;
#pragma unroll
                        for (int j = 0; j < 4; ++j) nv += (ohok && ow - p.pw + j >= 0 && ow - p.pw + j < p.Wx) ? 1u : 0u;
                        ptx::mbar_arrive_expect_tx(&full[stage], nv * S::B_BYTES);
#pragma unroll
                        for (int j = 0; j < 4; ++j) {
                            const int iw = ow - p.pw + j;
                            if (!ohok || iw < 0 || iw >= p.Wx) continue;
#pragma unroll
                            for (int jj = 0; jj < BN / S::CH; ++jj)
                                ptx::tma_load_4d(sa + S::A_STAGE + j * S::B_BYTES + jj * S::ATOM, &tmX, &full[stage],
                                                 c.nb * BN + jj * S::CH, iw, ih, n64 * KIMG);
                        }
                    } else if (!is_b) {
                        // only the atoms holding valid O_C rows (the rest of the MMA's M rows are never stored)
                        const int a_atoms = min(128 / S::CH, (p.OC - c.mb * 128 + S::CH - 1) / S::CH);
                        ptx::mbar_arrive_expect_tx(&full[stage], uint32_t(a_atoms * S::ATOM));
                        if (p.tcmc) {  // rank 0 loads the dY block once for the cluster (multicast)
                            if (tcrank == 0)
                                for (int j = 0; j < a_atoms; ++j)
                                    ptx::tma_load_4d_mc(sa + j * S::ATOM, &tmDY, &full[stage], c.mb * 128 + j * S::CH,
                                                        ow, od * p.OHr + oh, n64 * KIMG, tcmask);
                        } else if (RG) {  // rg_pk positions x rg images, (C, N, W, H) map
                            for (int j = 0; j < a_atoms; ++j)
                                ptx::tma_load_4d(sa + j * S::ATOM, &tmDY, &full[stage], c.mb * 128 + j * S::CH, 0, ow,
                                                 od * p.OHr + oh);
                        } else {
                            for (int j = 0; j < a_atoms; ++j)
                                ptx::tma_load_4d(sa + j * S::ATOM, &tmDY, &full[stage], c.mb * 128 + j * S::CH, ow,
                                                 od * p.OHr + oh, n64 * KIMG);
                        }
                    } else {
                        // leaping access (Fig. 7) on every axis: flattened X row of (id, ih)
                        const int ih = (od * p.sd + c.fd - p.pd) * p.Hr + oh * p.sh + c.fh - p.ph;
                        uint32_t nv = 0;
#pragma unroll
                        for (int f = 0; f < MT; ++f)
                            nv += (ohok && (MT == 1 || (ow < p.ow_e[f] && ow + rpk > p.ow_s[f]))) ? 1u : 0u;
                        ptx::mbar_arrive_expect_tx(&full[stage], nv * S::B_BYTES);
#pragma unroll
                        for (int f = 0; f < MT; ++f) {
                            // trimmed tap (row groups: no valid position in the chunk)
                            if (!ohok || (MT > 1 && !(ow < p.ow_e[f] && ow + rpk > p.ow_s[f]))) continue;
                            const int iw = ow * p.sw + (MT > 1 ? f : c.fw) - p.pw;
#pragma unroll
                            for (int j = 0; j < BN / S::CH; ++j) {
                                if (RG)  // rg_pk leaping columns (element stride s_w) x rg images
                                    ptx::tma_load_4d(sa + S::A_STAGE + f * S::B_BYTES + j * S::ATOM, &tmX, &full[stage],
                                                     c.nb * BN + j * S::CH, 0, iw, ih);
                                else
                                    ptx::tma_load_4d(sa + S::A_STAGE + f * S::B_BYTES + j * S::ATOM, &tmX, &full[stage],
                                                     c.nb * BN + j * S::CH, iw, ih, n64 * KIMG);
                            }
                        }
                    }
                }
                __syncwarp();
                if (++stage == S::STAGES) {
                    stage = 0;
                    phase ^= 1;
                }
            }
        }
    } else if (warp == 1) {
        // ---------------- MMA issuer (whole warp, elected lane issues)
        constexpr uint32_t idesc = ptx::instr_desc(128, BN, kTF32, true, true);
        // MN-major: LBO 8 KB between 128 B channel atoms, SBO = one K group (8 x / 4 x 128 B)
        const uint64_t dconst = kTF32 ? ptx::smem_desc_mn_b32(0, S::ATOM, 512) : ptx::smem_desc_sw128(0, S::ATOM, 1024);
        uint32_t stage = 0, phase = 0, acc = 0, acc_phase = 0;
        for (long long t = blockIdx.x; t < p.num_tiles; t += gridDim.x) {
            const WTile c = wdecode<MT, RG>(t, p);
            ptx::mbar_wait(&tempty[acc], acc_phase ^ 1);
            ptx::tc_fence_after();
            const uint32_t d = tmem_base + acc * (MT * BN);
            uint32_t started = 0;  // row tiles: taps that already accumulated in this tile
            for (int kb = c.kb0; kb < c.kb1; ++kb) {
                ptx::mbar_wait(&full[stage], phase);
                ptx::tc_fence_after();
                const uint32_t a_addr = ptx::smem_u32(smem + stage * S::STAGE_BYTES);
                const uint64_t ad = dconst | ptx::desc_addr(a_addr);
                const int ow = c.ows + (PP ? 2 : rpk) * ((kb / p.nblk64) % max(c.wn, 1));
                bool ohok = true;
                if (p.tc > 1) {
                    const int oh = c.ohs + ((kb / p.nblk64) / max(c.wn, 1)) % max(c.hn, 1);
                    ohok = oh >= p.oh_s[c.fh] && oh < p.oh_e[c.fh];
                }
                if (ptx::elect_one()) {
#pragma unroll
                    for (int f = 0; f < MT; ++f) {
                        int kk0 = 0, kk1 = KIMG / S::UK;  // K steps of this tap in the k-block
                        if (PP) {  // X column f: one MMA for tap f of ow (rows 0-63) and tap f-1 of ow+1 (64-127)
                            if (!ohok || ow - p.pw + f < 0 || ow - p.pw + f >= p.Wx) continue;
                        } else if (RG) {
                            // row groups: only the K rows (q * rg + image) of the tap's valid positions q of
                            // the chunk are multiplied -- exact trimming at the range ends
                            const int lo = MT > 1 ? p.ow_s[f] : c.ows, hi = MT > 1 ? p.ow_e[f] : c.ows + c.wr;
                            const int q0 = max(lo - ow, 0), q1 = min(hi - ow, rpk);
                            if (!ohok || q1 <= q0) continue;
                            kk0 = q0 * p.rg / S::UK;
                            kk1 = q1 * p.rg / S::UK;
                        } else if (!ohok || (MT > 1 && !(ow >= p.ow_s[f] && ow < p.ow_e[f]))) {
                            continue;  // trimmed tap
                        }
                        const uint64_t bd = dconst | ptx::desc_addr(a_addr + S::A_STAGE + f * S::B_BYTES);
                        const uint32_t acc0 = MT > 1 ? ((started >> f) & 1u) : uint32_t(kb > c.kb0);
                        if (RG) {  // row groups: the K steps of the tap's valid positions only
#pragma unroll
                            for (int kk = 0; kk < KIMG / S::UK; ++kk)
                                if (kk >= kk0 && kk < kk1)
                                    ptx::mma_ss<kTF32>(d + uint32_t(f * BN), ad + uint64_t(kk * (S::KSTEP >> 4)),
                                                       bd + uint64_t(kk * (S::KSTEP >> 4)), idesc,
                                                       (acc0 | uint32_t(kk - kk0)) != 0);
                        } else {
#pragma unroll
                            for (int kk = 0; kk < KIMG / S::UK; ++kk)  // KIMG images in K16 (bf16) / K8 (tf32) steps
                                ptx::mma_ss<kTF32>(d + uint32_t(f * BN), ad + uint64_t(kk * (S::KSTEP >> 4)),
                                                   bd + uint64_t(kk * (S::KSTEP >> 4)), idesc, (acc0 | uint32_t(kk)) != 0);
                        }
                        started |= 1u << f;
                    }
                    if (p.tcmc)
                        ptx::mma_commit_mc(&empty[stage], tcmask);  // the stage's dY is every cluster CTA's
                    else
                        ptx::mma_commit(&empty[stage]);
                }
                __syncwarp();
                if (++stage == S::STAGES) {
                    stage = 0;
                    phase ^= 1;
                }
            }
            if (ptx::elect_one()) ptx::mma_commit(&tfull[acc]);
            __syncwarp();
            if (++acc == uint32_t(S::NACC)) {
                acc = 0;
                acc_phase ^= 1;
            }
        }
    } else if (warp >= 4) {
        const uint32_t sub = warp & 3;
        const int row = int(sub * 32 + lane);
        const int taps = p.FD * p.FH * p.FW;
        const bool vec4 = (p.C % 4) == 0;
        uint32_t acc = 0, acc_phase = 0;
        for (long long t = blockIdx.x; t < p.num_tiles; t += gridDim.x) {
            const WTile c = wdecode<MT, RG>(t, p);
            const bool zero = c.kb1 <= c.kb0;
            ptx::mbar_wait(&tfull[acc], acc_phase);
            ptx::tc_fence_after();
            const int oc = c.mb * 128 + row;
            const int cbase = c.nb * BN;
            const int cvalid = min(BN, p.C - cbase);
            if constexpr (PP) {
                // tap fw = D_fw[0:64] (position ow, warps 0-1) + D_{fw+1}[64:128] (ow+1, warps 2-3):
                // the halves go to G_Z partial slots 2z and 2z+1 (summed by KB-REDUCE)
                const int h = sub >= 2 ? 1 : 0;
                const int ocr = row - 64 * h;
#pragma unroll 1
                for (int fw = 0; fw < 3; ++fw) {
                    const int j = fw + h;
                    const bool live = !zero && pp_col_has_work(c, p, j);
                    float* dst = ocr < p.OC ? p.out + (2 * c.z + h) * p.part_stride +
                                                  (static_cast<long long>(ocr) * taps + (c.fd * p.FH + c.fh) * p.FW + fw) *
                                                      p.C + cbase
                                            : nullptr;
#pragma unroll 1
                    for (int c0 = 0; c0 < BN; c0 += 32) {
                        uint32_t r[32];
                        ptx::tmem_ld32(tmem_base + ((sub * 32u) << 16) + acc * (MT * BN) + j * BN + c0, r);
                        ptx::tmem_ld_wait();
                        if (dst == nullptr || c0 >= cvalid) continue;
                        if (!live) {
#pragma unroll
                            for (int q = 0; q < 32; ++q) r[q] = 0u;
                        }
                        if (vec4 && c0 + 32 <= cvalid) {
#pragma unroll
                            for (int q = 0; q < 32; q += 4)
                                *reinterpret_cast<float4*>(dst + c0 + q) =
                                    make_float4(__uint_as_float(r[q]), __uint_as_float(r[q + 1]),
                                                __uint_as_float(r[q + 2]), __uint_as_float(r[q + 3]));
                        } else {
#pragma unroll
                            for (int q = 0; q < 32; ++q)
                                if (c0 + q < cvalid) dst[c0 + q] = __uint_as_float(r[q]);
                        }
                    }
                }
                ptx::tc_fence_before();
                ptx::mbar_arrive(&tempty[acc]);
                if (++acc == uint32_t(S::NACC)) {
                    acc = 0;
                    acc_phase ^= 1;
                }
                continue;
            } else {
#pragma unroll 1
            for (int f = 0; f < MT; ++f) {
            const bool fzero = zero || (MT > 1 && !tap_has_work<RG>(c, p, f));
            float* dst = nullptr;
            if (p.zc)  // own smem (the ring is idle: one tile per CTA): column group q = (f*BN + c)/4, [q][128 rows]
                dst = reinterpret_cast<float*>(smem) + (f * (BN / 4)) * 512 + row * 4;
            else if (oc < p.OC)
                dst = p.out + c.z * p.part_stride +
                      (static_cast<long long>(oc) * taps + (c.fd * p.FH + c.fh) * p.FW + (MT > 1 ? f : c.fw)) * p.C +
                      cbase;
#pragma unroll 1
            for (int c0 = 0; c0 < BN; c0 += 32) {
                uint32_t r[32];
                ptx::tmem_ld32(tmem_base + ((sub * 32u) << 16) + acc * (MT * BN) + f * BN + c0, r);
                ptx::tmem_ld_wait();
                if (p.zc) {
                    if (fzero) {
#pragma unroll
                        for (int j = 0; j < 32; ++j) r[j] = 0u;
                    }
#pragma unroll
                    for (int j = 0; j < 32; j += 4)
                        *reinterpret_cast<float4*>(dst + (c0 + j) / 4 * 512) =
                            make_float4(__uint_as_float(r[j]), __uint_as_float(r[j + 1]), __uint_as_float(r[j + 2]),
                                        __uint_as_float(r[j + 3]));
                } else if (dst != nullptr && c0 < cvalid) {
                    if (fzero) {
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
            }
            }  // generic taps
            ptx::tc_fence_before();
            ptx::mbar_arrive(&tempty[acc]);
            if (++acc == uint32_t(S::NACC)) {
                acc = 0;
                acc_phase ^= 1;
            }
        }
    }
    ptx::block_sync();
    if (p.zc) {
        // G_Z map-reduce inside the cluster: CTA z sums column slice z of the
        // tile over the gz segments in fixed order z' = 0..gz-1 and writes dW
        ptx::cluster_sync();
        if (warp >= 4 && blockIdx.x < p.num_tiles) {
            const WTile c = wdecode<MT, RG>(blockIdx.x, p);
            const int row = int(threadIdx.x) - 128;
            const int oc = c.mb * 128 + row;
            const int G = MT * BN / 4;
            const int g0 = (c.z * G) / p.gz, g1 = ((c.z + 1) * G) / p.gz;
            const uint32_t sbase = ptx::smem_u32(smem) + uint32_t(row) * 16u;
            const int taps = p.FD * p.FH * p.FW;
            if (oc < p.OC) {
#pragma unroll 1
                for (int gq = g0; gq < g1; gq += 2) {
                    const bool two = gq + 1 < g1;
                    const uint32_t off = sbase + uint32_t(gq) * 2048u;
                    float4 a[8], b[8];
#pragma unroll
                    for (int z = 0; z < 8; ++z) {
                        if (z < p.gz) {
                            a[z] = ptx::ld_dsmem_f4(ptx::mapa(off, uint32_t(z)));
                            if (two) b[z] = ptx::ld_dsmem_f4(ptx::mapa(off + 2048u, uint32_t(z)));
                        }
                    }
#pragma unroll
                    for (int h = 0; h < 2; ++h) {
                        if (h == 1 && !two) break;
                        float4 v = h ? b[0] : a[0];
#pragma unroll
                        for (int z = 1; z < 8; ++z) {
                            if (z < p.gz) {
                                const float4 w = h ? b[z] : a[z];
                                v.x += w.x;
                                v.y += w.y;
                                v.z += w.z;
                                v.w += w.w;
                            }
                        }
                        const int gg = gq + h;
                        const int f = gg / (BN / 4), ic = c.nb * BN + (gg % (BN / 4)) * 4;
                        if (ic >= p.C) continue;
                        float* o = p.out + (static_cast<long long>(oc) * taps + (c.fd * p.FH + c.fh) * p.FW +
                                            (MT > 1 ? f : c.fw)) * p.C + ic;
                        if ((p.C % 4) == 0) {
                            *reinterpret_cast<float4*>(o) = v;
                        } else {
                            const float e[4] = {v.x, v.y, v.z, v.w};
                            for (int u = 0; u < 4 && ic + u < p.C; ++u) o[u] = e[u];
                        }
                    }
                }
            }
        }
        ptx::cluster_sync();  // peers finished reading this CTA's staging
    } else if (p.tcmc) {
        ptx::cluster_sync();  // no CTA leaves while peers may still multicast into it / commit to it
    }
    if (warp == 2) {
        ptx::tc_fence_after();
        ptx::tmem_dealloc(tmem_base, S::TMEM_COLS);
    }
}

}  // namespace cks
