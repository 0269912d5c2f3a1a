// igemm.cuh -- KB-CONV / KB-KS: the trimmed-window implicit GEMM on
// tcgen05 tensor cores, shared by ConvV2 (Alg. 1) and the fused
// Stage2&3 of KS-deconv-V2 (Alg. 2/2B).
//
// GEMM rows are BATCH IMAGES: an accumulator holds 128 images x BN output
// channels of ONE output pixel, so all its rows share one trimmed filter
// window [ts_h, te_h) x [ts_w, te_w) -- the B200 analogue of P:156 ("all
// threads in the same block have the same trimmed-filters ... no warp-
// divergence"): padded zeros are never loaded or multiplied and the K loop
// has no bounds checks.
//
// A tile is PBW consecutive pixels of one output row (same h window, same
// phase), 128 images, BN channels: PBW accumulators in TMEM.  Its K loop
// runs over "row steps" (filter row ch in the h window) x (channel block
// kc); per row step the producer loads
//   * the B row: the filter taps cw in the union of the pixels' w windows,
//     one (BK x BN) K-major tile each, once for all PBW pixels, and
//   * the A positions: one (128 images x BK) K-major tile per activation
//     column iw in the union of the pixels' windows, each loaded ONCE and
//     multiplied into every (pixel j, tap cw = iw - a0w_j) it serves
// (halo reuse: for unit stride a position feeds up to FW pixels).  Compared
// with one pixel per tile this cuts the L2->SM bytes per MAC by ~1.7x, which
// is what bounds this kernel (TMA ingress ~64 B/clk/SM).
//
//   fwd (ConvV2): act = X, filt = W [OC][FH*FW][C] (slot fh*FW+fw),
//                 a0 = o*s - p, out = o (T1)
//   KS-deconv:    act = dY, filt = packed C_{y,x} [P][C][CHm*CWm][OCp]
//                 (Stage1), a0 = oh_s = u + a_y, out = u*sh + ih_s (T2): the
//                 epilogue is Stage3's phase-strided composition.
//
// Stage1-free KS-deconv (BMN, SURVEY §8(f) NEXT #4 -- the all-in-one variant
// the paper tried and set aside): the B operand is read straight from
// W [OC][FH][FW][IC] per sub-filter row -- one TMA box of taps fw = x, x+sw,
// ... (element stride sw) of filter row fh = y + (CH_y-1-ch)*sh, IC innermost
// -- as an MN-major operand (IC = N contiguous, OC = K); the rot180 of
// Stage1 becomes the slot order (slot j <-> cw = CW_x-1-j), absorbed by keeping
// accumulators in forward pixel order.  No packed sub-filters, no KB-SPLIT.
//
// Under-filled grids split the row steps into Z segments (split-K).  Cluster
// split-K (zc, the default): the Z CTAs of one thread-block cluster compute
// the Z segments of ONE output tile (one tile per CTA), stage their fp32
// accumulators in their own (then idle) shared-memory rings, and after a
// cluster barrier CTA r sums column slice r of the tile over z = 0..Z-1 in
// fixed order through distributed shared memory and stores it
// (deterministic; no global partials, no counters, no extra launch).
// Legacy global split-K: each segment writes fp32 partials and the LAST
// arriving CTA of an output tile sums the Z partials in fixed order.
//
// Warp roles (256 threads, 1 CTA/SM, persistent over tiles):
//   warp 0 lane 0  TMA producer (B-row ring + A-position ring, mbarriers)
//   warp 1 lane 0  MMA issuer   (tcgen05.mma, kind::f16 or kind::tf32)
//   warp 2         TMEM allocator
//   warps 4..7     epilogue     (tcgen05.ld -> fp32 stores / split-K reduce)
#pragma once
#include "ptx.cuh"
#include "../../../include/cks.h"
#include "../cks_plan.h"

namespace cks {

constexpr int kMaxPBW = 8;
constexpr int kProgSlot = 2 + 2 * kProgEntries;  // int4: header {np0, np1, rs0, rs1}, {pos_lo, pos_hi, -, -}, 2 lists

// Division by a launch constant d via a host-computed multiplier:
// n / d = (n * m) >> sh with l = ceil(log2 d), sh = 31 + l, m = ceil(2^sh / d);
// exact for n < 2^31 (error m*d - 2^sh < d <= 2^l, so (m*d - 2^sh) * n < 2^sh).
struct FastDiv {
    uint32_t m, sh, d;
};
__device__ __forceinline__ uint32_t fdivu(uint32_t n, const FastDiv& f) {
    return uint32_t((uint64_t(n) * f.m) >> f.sh);
}

struct KAxis {
    int16_t a0[CKS_MAX_ROWS];   // A coordinate of tap 0
    int16_t out[CKS_MAX_ROWS];  // output coordinate
    uint8_t ts[CKS_MAX_ROWS];   // trimmed tap window [ts, te)
    uint8_t te[CKS_MAX_ROWS];
    uint8_t phase[CKS_MAX_ROWS];
};

// Kernel-parameter form of an axis table: the trimmed windows per row and,
// per phase, the affine row -> (A coordinate of tap 0, output coordinate) maps
// (T1: a0 = o*s - p, out = o; T2 phase y: a0 = oh_s = u + a_y,
// out = u*sh + ih_s).  Expanded into the KAxis table in shared memory at
// kernel start; keeps the launch parameters (with the three tensor maps)
// under the 4 KB classic kernel-parameter limit.
constexpr int kMaxPhases = 16;
struct KAxisC {
    uint8_t ts[CKS_MAX_ROWS], te[CKS_MAX_ROWS];
    int16_t row0[kMaxPhases + 1];  // run x (one phase) holds rows [row0[x], row0[x+1])
    int16_t a00[kMaxPhases], a0st[kMaxPhases], out0[kMaxPhases], outst[kMaxPhases];
    int16_t phid[kMaxPhases];      // phase index of run x (phases without rows have no run)
    int8_t rlen[kMaxPhases];       // row groups: output rows per table row of run x (1 = ungrouped)
    int16_t nph, nrows;
};

struct IgemmParams {
    KAxisC ah, aw;
    // 3-D: the depth axis is a third table; an output
    // "row" is (d row, h row), its row steps run over the (filter depth, filter
    // row) pairs of both trimmed windows.  A / output / B rows are flattened
    // (d * rows_per_depth + h); 2-D = one trivial depth row (a0 0, window [0,1)).
    KAxisC ad;
    int a_rows_h;      // A tensor rows per depth slice (X: H, dY: OH)
    int out_rows_h;    // output rows per depth slice
    int b_rows_h;      // B filter rows per depth slice (fwd: FH; packed KS: CHm; W-direct: FH)
    int phases_h;      // phase = (phase_d * phases_h + phase_h) * phases_w + phase_w
    int bsd;           // W-direct: filter depth of sub-filter depth row cd is bfd0[z] - cd * bsd
    int16_t bfd0[kMaxPhases];
    float* out;
    float* part;  // split-K partials [out_tiles][Z][PBW*BN/4][128 rows][4] (coalesced per warp)
    int* sem;     // split-K arrival counters [out_tiles] (zero on entry, left zero)
    int rows_h;
    int nph_w;                 // w phases
    int16_t wph_off[9], wph_cnt[9], wb_cum[9];
    int wblocks;               // pixel blocks along w
    int pbw, acc_stages;       // pixels per tile, TMEM accumulator buffers
    int nblk, nbs, kc_blocks;  // image blocks, BN blocks, BK channel blocks
    int slot_stride;           // filter tap slot = ch * slot_stride + cw
    int phases_w;              // phase = phase_h * phases_w + phase_w
    int N, out_H, out_W, out_C;
    int a_stages, b_stages;    // smem rings: A positions (16 KB each), B rows
    int b_stage_bytes;         // ntap * BN * 128
    int ntap;                  // filter taps per B row (one TMA box)
    int apos;                  // activation positions per A slot (one TMA box)
    int unit_step;             // consecutive pixels' tap-0 columns differ by 1 (N-merged MMAs)
    int a0_step;               // a0 of pixel j = a0 of pixel 0 + j * a0_step (T1: stride, T2: 1)
    int zsplit;
    int zc;  // cluster split-K: cluster = the zsplit segments of one output tile, DSMEM reduction
    int pair;  // CTA pair (cta_group::2): the even/odd CTA of a cluster hold image blocks 2q / 2q+1 of one
               // tile (M = 256) and B columns [0, BN) / [BN, 2 BN) of its 2 BN outputs; nblk counts pairs
    FastDiv fd_z, fd_nbs, fd_nblk, fd_wb, fd_kc, fd_rh;  // divisors of the tile / row-step decode
    long long num_tiles;  // output tiles x zsplit
    int cm;               // cluster size along the O_C blocks: the A tile of a pixel is multicast (1 = off)
    int unified;          // one A slot per row step: A slot + B row share one full/empty barrier pair
    int tma_store;        // 1: last tile per CTA staged in the idle rings and TMA-stored; 2: also every
                          // other tile, through the per-warp 4 KB epilogue buffers
    int epi_stage;        // 16 KB epilogue staging: transpose 32x32 blocks, store full 128 B lines
    int tmem_cols;        // TMEM columns allocated (only what the accumulators need: a small
                          // layer's CTA can share its SM with the next kernel's CTA)
    int epi_bufs;         // 4 KB TMA-store staging buffers per epilogue warp (1 or 2)
    int epi_warps;        // epilogue warps: 4 (one per TMEM sub-partition) or 8 (two, alternate 32-column chunks)
    int dbg;              // experiment flags (0 in production): 1 skip stores, 2 skip MMA
    // Stage1-free KS-deconv (BMN): per phase_h y the filter row of sub-filter row 0,
    // fh0[y] = y + (CH_y - 1) * sh (row ch is fh0[y] - ch * sh); per phase_w x the
    // sub-filter width CW_x; sh
    int16_t bfh0[kMaxPhases], bcw[kMaxPhases];
    int bsh;
    unsigned long long* trace;  // debug timeline (nullptr in production): [cta<4][role<5][1024]
    // Row groups (small batches, N <= 64): M row r of a tile = image r % rg_ni of output row
    // orow + (r / rg_ni) * rg_ostep (valid for r / rg_ni < the group length); 0 = batch-as-M
    int rg_ni, rg_shift, rg_ostep;
};

__device__ __forceinline__ unsigned long long gtimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}
// debug: per-CTA global-timer milestones -> trace[4*1024*5 + cta*8 + k]
__device__ __forceinline__ void trace_gt(const IgemmParams& p, int k) {
    if (p.trace != nullptr && blockIdx.x < 148) p.trace[4 * 1024 * 5 + blockIdx.x * 8 + k] = gtimer();
}

// debug timeline: entry = (code << 56) | clock64
__device__ __forceinline__ void trace_ev(const IgemmParams& p, int role, int& idx, unsigned code) {
    if (p.trace != nullptr && blockIdx.x < 4 && idx < 1024) {
        const unsigned long long t = clock64();
        p.trace[(blockIdx.x * 5 + role) * 1024 + idx] = (static_cast<unsigned long long>(code) << 56) | (t & 0x00FFFFFFFFFFFFFFull);
        ++idx;
    }
}

// KB = bytes of one K row (32 / 64 / 128 -> SWIZZLE_32B / 64B / 128B): narrow
// channel counts (e.g. I_C = 3 padded to 8) use a narrow K block instead of
// multiplying TMA zero fill.
template <int BN, bool kTF32, int KB = 128>
struct IgemmShape {
    static constexpr int EB = kTF32 ? 4 : 2;
    static constexpr int BK = KB / EB;   // channels per K block
    static constexpr int UK = 32 / EB;   // K per tcgen05.mma (32 bytes)
    static constexpr int A_BYTES = 128 * KB;
    static constexpr int TILE_B = BN * KB;
    static constexpr int SMEM_MAX = 227 * 1024;
};

// Per-tile decode shared by the three roles.  Per-pixel data lives in fixed
// size arrays that are only indexed inside fully unrolled loops (registers).
struct Tile {
    int z, nb, nblk, rh, j0, len, ph;
    int rd, cds, nh;      // depth row, first filter depth of its window, filter rows of the h window
    int orow;             // output row (flattened d * out_rows_h + h)
    int a0d;              // A depth coordinate of filter depth 0
    int rs0, rs1;         // row-step range [rs0, rs1) of this split
    int glen;             // row groups: output rows of this tile's group
    int rot;              // per-CTA rotation of the row-step order (spreads weight reads over L2)
    int chs;              // first filter row of the h window
    int cwlo, cwhi;       // union of the pixels' w windows
    int pos_lo, pos_hi;   // union of A columns
    int a0[kMaxPBW], ts[kMaxPBW], te[kMaxPBW];
    long long out_tile;
};

__device__ __forceinline__ Tile decode_tile(long long t64, const IgemmParams& p, const KAxis& ah, const KAxis& aw,
                                            const KAxis& ad) {
    // 32-bit decode (tile counts < 2^31; 64-bit div/mod is a slow software routine)
    Tile c;
    uint32_t t = uint32_t(t64);
    uint32_t q = fdivu(t, p.fd_z);
    c.z = int(t - q * uint32_t(p.zsplit));
    t = q;
    c.out_tile = t;
    q = fdivu(t, p.fd_nbs);
    c.nb = int(t - q * uint32_t(p.nbs));
    t = q;
    q = fdivu(t, p.fd_nblk);
    c.nblk = int(t - q * uint32_t(p.nblk));
    if (p.pair) c.nblk = 2 * c.nblk + int(blockIdx.x & 1u);  // this CTA's image block of the pair
    t = q;
    q = fdivu(t, p.fd_wb);
    const int wb = int(t - q * uint32_t(p.wblocks));
    {
        const uint32_t r3 = q;  // (depth row, h row)
        const uint32_t rd = fdivu(r3, p.fd_rh);
        c.rd = int(rd);
        c.rh = int(r3 - rd * uint32_t(p.rows_h));
    }
    int x = 0;
    while (x + 1 < p.nph_w && p.wb_cum[x + 1] <= wb) ++x;
    c.j0 = p.wph_off[x] + (wb - p.wb_cum[x]) * p.pbw;
    c.len = min(p.pbw, p.wph_off[x] + p.wph_cnt[x] - c.j0);
    c.ph = (ad.phase[c.rd] * p.phases_h + (ah.phase[c.rh] & 15)) * p.phases_w + aw.phase[c.j0];
    c.glen = (ah.phase[c.rh] >> 4) + 1;
    const int chs = ah.ts[c.rh], che = ah.te[c.rh];
    const int cds = ad.ts[c.rd], cde = ad.te[c.rd];
    c.cds = cds;
    c.nh = che - chs;
    c.a0d = ad.a0[c.rd];
    c.orow = ad.out[c.rd] * p.out_rows_h + ah.out[c.rh];
    c.chs = chs;
    int lo = 1 << 20, hi = -(1 << 20), plo = 1 << 20, phi = -(1 << 20);
#pragma unroll
    for (int j = 0; j < kMaxPBW; ++j) {
        c.a0[j] = 0;
        c.ts[j] = 0;
        c.te[j] = 0;
        if (j < c.len) {
            c.a0[j] = aw.a0[c.j0 + j];
            c.ts[j] = aw.ts[c.j0 + j];
            c.te[j] = aw.te[c.j0 + j];
            if (c.te[j] > c.ts[j]) {
                lo = min(lo, c.ts[j]);
                hi = max(hi, c.te[j]);
                plo = min(plo, c.a0[j] + c.ts[j]);
                phi = max(phi, c.a0[j] + c.te[j]);
            }
        }
    }
    const bool empty = (hi <= lo) || (che <= chs) || (cde <= cds);
    c.cwlo = empty ? 0 : lo;
    c.cwhi = empty ? 0 : hi;
    c.pos_lo = empty ? 0 : plo;
    c.pos_hi = empty ? 0 : phi;
    const int rs = empty ? 0 : (che - chs) * (cde - cds) * p.kc_blocks;
    c.rs0 = p.zsplit == 1 ? 0 : int(fdivu(uint32_t(rs) * uint32_t(c.z), p.fd_z));
    c.rs1 = p.zsplit == 1 ? rs : int(fdivu(uint32_t(rs) * uint32_t(c.z + 1), p.fd_z));
    c.rot = c.rs1 > c.rs0 ? int(((blockIdx.x >> (p.pair ? 1 : 0)) / unsigned(p.cm)) % unsigned(c.rs1 - c.rs0))
                          : 0;  // cluster-uniform
    return c;
}

// i-th row step of tile c (rotated start; every role uses the same order)
__device__ __forceinline__ int row_step(const Tile& c, int i) {
    int r = i + c.rot;
    if (r >= c.rs1) r -= c.rs1 - c.rs0;
    return r;
}

// bitmask of pixels j of the tile that use activation column iw
__device__ __forceinline__ uint32_t pos_mask(const Tile& c, int iw) {
    uint32_t m = 0;
#pragma unroll
    for (int j = 0; j < kMaxPBW; ++j) {
        const int cw = iw - c.a0[j];
        if (cw >= c.ts[j] && cw < c.te[j]) m |= 1u << j;
    }
    return m;
}

template <int BN, bool kTF32, int KB, bool PAIR = false, bool BMN = false>
__global__ void __launch_bounds__(384, 1)
    igemm_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                 const __grid_constant__ CUtensorMap tmY, const __grid_constant__ IgemmParams p) {
    // CTA-pair kernels are separate instantiations: a kernel containing
    // cta_group::2 tcgen05 instructions must be launched with pair clusters
    constexpr bool kPair = PAIR;
    using S = IgemmShape<BN, kTF32, KB>;
    extern __shared__ uint8_t smem_raw[];
    // 1 KB alignment by offset arithmetic (keeps the shared address space visible to the compiler)
    uint8_t* smem = smem_raw + ((1024u - (ptx::smem_u32(smem_raw) & 1023u)) & 1023u);
    const uint32_t a_slot = uint32_t(p.apos) * S::A_BYTES;
    uint8_t* abuf = smem;                                    // a_stages x apos x 16 KB
    uint8_t* bbuf = smem + p.a_stages * a_slot;              // b_stages x b_stage_bytes
    uint64_t* bars = reinterpret_cast<uint64_t*>(bbuf + p.b_stages * p.b_stage_bytes);
    uint64_t* afull = bars;
    uint64_t* aempty = afull + p.a_stages;
    uint64_t* bfull = aempty + p.a_stages;
    uint64_t* bempty = bfull + p.b_stages;
    uint64_t* tfull = bempty + p.b_stages;
    uint64_t* tempty = tfull + 2;
    uint64_t* pfull = tempty + 2;   // MMA programs built by warp 2 (double buffered)
    uint64_t* pempty = pfull + 2;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(pempty + 2);
    int* red_flag = reinterpret_cast<int*>(tmem_slot + 1);
    const uint32_t tmem_cols = uint32_t(p.tmem_cols);  // power of two >= acc_stages x pbw x BNo
    // per-axis plan tables copied to smem once (one parallel pass of independent
    // constant loads instead of dependent cold loads in every role's decode)
    KAxis* tab = reinterpret_cast<KAxis*>(reinterpret_cast<uint8_t*>(bars) + 512);
    // 2 program slots x (2 header + 2 x 64 entries)
    int4* prog = reinterpret_cast<int4*>(reinterpret_cast<uint8_t*>(tab) + 3 * sizeof(KAxis));
    // epilogue staging (p.epi_stage): 4 x 4 KB, 1 KB aligned (128B-swizzled TMA-store source)
    float* epi = reinterpret_cast<float*>(smem + ((ptx::smem_u32(prog + 2 * kProgSlot) - ptx::smem_u32(smem) + 1023u) & ~1023u));
    for (int i = threadIdx.x; i < 3 * CKS_MAX_ROWS; i += blockDim.x) {
        const int which = i / CKS_MAX_ROWS;  // 0: h, 1: w, 2: d
        const KAxisC& ax = which == 0 ? p.ah : (which == 1 ? p.aw : p.ad);
        KAxis& t = tab[which];
        const int r = i & (CKS_MAX_ROWS - 1);
        int x = 0;
        while (x + 1 < ax.nph && ax.row0[x + 1] <= r) ++x;
        const int u = r - ax.row0[x];
        const bool v = r < ax.nrows;
        t.a0[r] = v ? int16_t(ax.a00[x] + u * ax.a0st[x]) : int16_t(0);
        t.out[r] = v ? int16_t(ax.out0[x] + u * ax.outst[x]) : int16_t(0);
        t.ts[r] = v ? ax.ts[r] : uint8_t(0);
        t.te[r] = v ? ax.te[r] : uint8_t(0);
        // phase, and (row groups, h axis) the group length - 1 in bits 4..7
        t.phase[r] = v ? uint8_t(ax.phid[x] | ((ax.rlen[x] - 1) << 4)) : uint8_t(0);
    }

    if (threadIdx.x == 0) trace_gt(p, 0);
    ptx::pdl_launch_dependents();
    const uint32_t warp = ptx::warp_id(), lane = ptx::lane_id();
    if (warp == 0 && lane == 0) {
        ptx::prefetch_tmap(&tmA);
        ptx::prefetch_tmap(&tmB);
        for (int i = 0; i < p.a_stages; ++i) {
            ptx::mbar_init(&afull[i], p.unified ? 2 : 1);  // unified: A and B producers
            ptx::mbar_init(&aempty[i], p.cm);  // every CTA of the cluster consumes the multicast slot
        }
        for (int i = 0; i < p.b_stages; ++i) {
            ptx::mbar_init(&bfull[i], 1);
            ptx::mbar_init(&bempty[i], 1);
        }
        for (int i = 0; i < 2; ++i) {
            ptx::mbar_init(&tfull[i], 1);
            ptx::mbar_init(&tempty[i], 32 * p.epi_warps * (kPair ? 2 : 1));  // pair: both CTAs' epilogues
            ptx::mbar_init(&pfull[i], 32);
            ptx::mbar_init(&pempty[i], 32);
        }
        ptx::fence_barrier_init();
    }
    __syncwarp();  // reconverge the initialising lane's warp before the block barrier
    if (warp == 2) {
        if (kPair)
            ptx::tmem_alloc_pair(tmem_slot, tmem_cols);
        else
            ptx::tmem_alloc(tmem_slot, tmem_cols);
    }
    ptx::tc_fence_before();
    ptx::block_sync();
    if (p.cm > 1 || kPair) ptx::cluster_sync();  // peers' barriers exist before the first multicast / pair op
    ptx::tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;
    const uint32_t crank = p.cm > 1 ? blockIdx.x % uint32_t(p.cm) : 0u;
    const bool leader = !kPair || (blockIdx.x & 1u) == 0;  // pair: the even CTA issues the MMAs
    const long long t0 = kPair ? (blockIdx.x >> 1) : blockIdx.x;
    const long long tstep = kPair ? (gridDim.x >> 1) : gridDim.x;
    const int BNo = kPair ? 2 * BN : BN;  // output channels per tile (MMA N of one pixel)
    const uint16_t cmask = uint16_t((1u << p.cm) - 1u);
    if (threadIdx.x == 0) trace_gt(p, 1);
    ptx::pdl_wait();  // inputs of this op may come from the previous kernel
    if (threadIdx.x == 0) trace_gt(p, 2);

    if (warp == 0 || warp == 3) {
        // ---------------- TMA producers.  The whole warp walks the (uniform)
        // schedule and one elected lane issues: warp 0 loads the A slots (apos
        // consecutive activation columns x 128 images, one box), warp 3 the B
        // rows (all taps of one filter row, one box).
        const bool is_b = warp == 3;
        uint32_t aq = 0, bq = 0;  // A / B sequence numbers
        uint32_t as = 0, aph = 0, bs = 0, bph = 0;  // ring slots / phases, stepped (no runtime division)
        const uint32_t na = uint32_t(p.a_stages), nb = uint32_t(p.b_stages);
        int ti = 0;
        const int trole = warp == 0 ? 0 : 4;
        if (lane == 0) trace_ev(p, trole, ti, 0);
        const uint32_t btx = uint32_t(p.ntap * S::TILE_B);
        for (long long t = t0; t < p.num_tiles; t += tstep) {
            const Tile c = decode_tile(t, p, tab[0], tab[1], tab[2]);
            const int a0h = tab[0].a0[c.rh];
            for (int ri = c.rs0; ri < c.rs1; ++ri) {
                const int r = row_step(c, ri);
                const int rq = int(fdivu(uint32_t(r), p.fd_kc));
                const int kc = r - rq * p.kc_blocks;
                const int rdq = rq / c.nh;  // (filter depth, filter row) of this row step
                const int cd = c.cds + rdq, ch = c.chs + (rq - rdq * c.nh);
                const int arow = (c.a0d + cd) * p.a_rows_h + a0h + ch;  // flattened A row
                const int brow = cd * p.b_rows_h + ch;                   // flattened filter row
                if (is_b) {
                    uint64_t* bf = p.unified ? &afull[bs] : &bfull[bs];
                    ptx::mbar_wait(p.unified ? &aempty[bs] : &bempty[bs], bph ^ 1);
                    if (ptx::elect_one()) {
                        if (kPair) {
                            // this CTA's half of the 2 BN columns; bytes complete on the leader's barrier,
                            // which the leader arms for both CTAs
                            const uint32_t bfc = ptx::mapa(ptx::smem_u32(bf), 0);
                            if (leader) ptx::mbar_arrive_expect_tx_cluster(bfc, 2 * btx);
                            ptx::tma_load_4d_pair(bbuf + bs * p.b_stage_bytes, &tmB, bfc, kc * S::BK,
                                                  c.nb * 2 * BN + int(blockIdx.x & 1u) * BN, brow * p.slot_stride,
                                                  c.ph);
                        } else if ((p.dbg & 4) && bq >= uint32_t(p.b_stages)) {
                            ptx::mbar_arrive(bf);  // experiment: B traffic removed (wrong results)
                        } else if (BMN) {
                            // W-direct: taps fw = x + j*sw (j = slot) of filter row fh, BN input channels
                            // (BN / atom 128-byte N atoms: 5-D map, smem [tap][atom][BK rows][128 B]) x BK
                            // output channels
                            const int zy = c.ph / p.phases_w, x = c.ph - zy * p.phases_w;
                            const int z = zy / p.phases_h, y = zy - z * p.phases_h;
                            const int wrow = (p.bfd0[z] - cd * p.bsd) * p.b_rows_h + p.bfh0[y] - ch * p.bsh;
                            ptx::mbar_arrive_expect_tx(bf, btx);
                            constexpr int ATOMW = 128 / S::EB;
                            if (BN > ATOMW)
                                ptx::tma_load_5d(bbuf + bs * p.b_stage_bytes, &tmB, bf, 0, kc * S::BK,
                                                 c.nb * (BN / ATOMW), x, wrow);
                            else
                                ptx::tma_load_4d(bbuf + bs * p.b_stage_bytes, &tmB, bf, c.nb * BN, kc * S::BK, x,
                                                 wrow);
                        } else {
                            ptx::mbar_arrive_expect_tx(bf, btx);
                            ptx::tma_load_4d(bbuf + bs * p.b_stage_bytes, &tmB, bf, kc * S::BK, c.nb * BN,
                                             brow * p.slot_stride, c.ph);
                        }
                    }
                    __syncwarp();
                    if (lane == 0) trace_ev(p, trole, ti, 1);
                    ++bq;
                    if (++bs == nb) {
                        bs = 0;
                        bph ^= 1u;
                    }
                    continue;
                }
                for (int iw0 = c.pos_lo; iw0 < c.pos_hi; iw0 += p.apos) {
                    ++aq;
                    ptx::mbar_wait(&aempty[as], aph ^ 1);
                    if (ptx::elect_one()) {
                        if (kPair) {
                            // this CTA's 128 images (rows 128*rank.. of the pair's M = 256)
                            const uint32_t afc = ptx::mapa(ptx::smem_u32(&afull[as]), 0);
                            if (leader) ptx::mbar_arrive_expect_tx_cluster(afc, 2 * a_slot);
                            ptx::tma_load_4d_pair(abuf + as * a_slot, &tmA, afc, kc * S::BK, c.nblk * 128, iw0,
                                                  arow);
                        } else if ((p.dbg & 8) && aq > uint32_t(p.a_stages)) {
                            ptx::mbar_arrive(&afull[as]);  // experiment: A traffic removed (wrong results)
                        } else if (p.cm > 1) {
                            // this CTA's 128/cm images of every column, multicast to the cluster
                            ptx::mbar_arrive_expect_tx(&afull[as], a_slot);
                            const int rows = 128 / p.cm;
                            for (int col = 0; col < p.apos; ++col)
                                ptx::tma_load_4d_mc(abuf + as * a_slot + col * S::A_BYTES + crank * rows * KB, &tmA,
                                                    &afull[as], kc * S::BK, c.nblk * 128 + int(crank) * rows,
                                                    iw0 + col, arow, cmask);
                        } else {
                            ptx::mbar_arrive_expect_tx(&afull[as], a_slot);
                            ptx::tma_load_4d(abuf + as * a_slot, &tmA, &afull[as], kc * S::BK, c.nblk * 128, iw0,
                                             arow);
                        }
                    }
                    __syncwarp();
                    if (lane == 0) trace_ev(p, trole, ti, 2);
                    if (++as == na) {
                        as = 0;
                        aph ^= 1u;
                    }
                }
            }
        }
    } else if (warp == 1) {
        {
            // ---------------- MMA issuer (single thread)
            // K-major SW128 descriptor without the start address: LBO 16 B, SBO 1 KB
            const uint64_t dconst = ptx::smem_desc_kmajor(0, KB);
            // B: K-major like A, or (BMN) MN-major: 128 B atoms of N laid out [tap][atom] (LBO = atom
            // bytes, so N-merged MMAs walk consecutive taps), SBO = one K group (8 / 4 rows of 128 B)
            constexpr uint32_t kAtomBytes = uint32_t(S::BK) * 128u;  // one 128-byte-wide N atom of BK K rows
            const uint64_t bconst = !BMN ? dconst
                                         : (kTF32 ? ptx::smem_desc_mn_b32(0, kAtomBytes, 512)
                                                  : ptx::smem_desc_mn(0, kAtomBytes, 1024, 128));
            constexpr uint32_t kBStep = BMN ? (S::UK * 128) >> 4 : 2;  // B descriptor advance per MMA K step
            uint32_t acc = 0, acc_ph = 0;
            uint32_t as = 0, aph = 0, bs = 0, bph = 0;  // ring slots / phases, stepped (no runtime division)
            const uint32_t na = uint32_t(p.a_stages), nb = uint32_t(p.b_stages);
            int ti = 0;
            if (lane == 0) trace_ev(p, 1, ti, 0);
            uint32_t ps = 0, pph = 0;
            for (long long t = t0; t < p.num_tiles && leader; t += tstep) {
                ptx::mbar_wait(&pfull[ps], pph);  // program of this tile (warp 2)
                const int4* pg = prog + ps * kProgSlot;
                const int4 h0 = pg[0], h1 = pg[1];
                const int np0 = h0.x, np1 = h0.y, rs0 = h0.z, rs1 = h0.w, pos_lo = h1.x, pos_hi = h1.y;
                __syncwarp();
                ptx::mbar_wait(&tempty[acc], acc_ph ^ 1);
                if (lane == 0) trace_ev(p, 1, ti, 3);
                ptx::tc_fence_after();
                const uint32_t dbase = tmem_base + acc * uint32_t(p.pbw * BNo);
                __syncwarp();
                const uint32_t idesc0 = ptx::instr_desc(kPair ? 256 : 128, 0, kTF32, false, BMN);
                bool first = true;
                for (int ri = rs0; ri < rs1; ++ri) {
                    if (!p.unified) ptx::mbar_wait(&bfull[bs], bph);  // unified: covered by the A-slot wait
                    if (lane == 0) trace_ev(p, 1, ti, 1);
                    const uint64_t bdesc0 = bconst | ptx::desc_addr(ptx::smem_u32(bbuf + bs * p.b_stage_bytes));
                    const int4* pl = pg + 2 + (first ? 0 : kProgEntries);
                    const int np = first ? np0 : np1;
                    first = false;
                    int e = 0;
                    for (int k = 0; pos_lo + k * p.apos < pos_hi; ++k) {
                        ptx::mbar_wait(&afull[as], aph);
                        if (lane == 0) trace_ev(p, 1, ti, 2);
                        ptx::tc_fence_after();
                        const uint64_t aslot = dconst | ptx::desc_addr(ptx::smem_u32(abuf + as * a_slot));
                        // entries of this A slot; the next entry is loaded while the
                        // current one issues (hides the shared-memory load latency)
                        int4 en = e < np ? pl[e] : make_int4(-1, 0, 0, 0);
                        for (; en.x == k; ++e) {
                            const int4 nx = e + 1 < np ? pl[e + 1] : make_int4(-1, 0, 0, 0);
                            const uint64_t adesc = aslot + uint64_t(uint32_t(en.y) * (S::A_BYTES >> 4));
                            const uint64_t bdesc = bdesc0 + uint64_t(uint32_t(en.w & 0xFF) * (S::TILE_B >> 4));
                            const uint32_t cnt = uint32_t(en.w >> 8) & 0xFFu;
                            const uint32_t idesc = idesc0 | (((cnt * uint32_t(BNo)) >> 3) << 17);
                            const uint32_t d = dbase + uint32_t(en.z);
                            const uint32_t acc0 = uint32_t(en.w >> 16) & 1u;
                            if (!(p.dbg & 2) && ptx::elect_one()) {
                                if (kPair) {
#pragma unroll
                                    for (int kk = 0; kk < S::BK / S::UK; ++kk)
                                        ptx::mma_ss_pair<kTF32>(d, adesc + uint64_t(kk * 2), bdesc + uint64_t(kk * 2),
                                                                idesc, kk ? 1u : acc0);
                                } else {
#pragma unroll
                                    for (int kk = 0; kk < S::BK / S::UK; ++kk)
                                        ptx::mma_ss<kTF32>(d, adesc + uint64_t(kk * 2), bdesc + uint64_t(kk * kBStep),
                                                           idesc, kk ? 1u : acc0);
                                }
                            }
                            __syncwarp();
                            en = nx;
                        }
                        if (ptx::elect_one()) {  // A slot free (in every CTA that multicasts into it)
                            if (kPair)
                                ptx::mma_commit_pair(&aempty[as]);
                            else if (p.cm > 1)
                                ptx::mma_commit_mc(&aempty[as], cmask);
                            else
                                ptx::mma_commit(&aempty[as]);
                        }
                        __syncwarp();
                        if (lane == 0) trace_ev(p, 1, ti, 4);
                        if (++as == na) {
                            as = 0;
                            aph ^= 1u;
                        }
                    }
                    if (!p.unified && ptx::elect_one()) ptx::mma_commit(&bempty[bs]);  // B row free
                    __syncwarp();
                    if (++bs == nb) {
                        bs = 0;
                        bph ^= 1u;
                    }
                }
                ptx::mbar_arrive(&pempty[ps]);  // program slot consumed (all 32 lanes)
                if (++ps == 2) {
                    ps = 0;
                    pph ^= 1;
                }
                if (lane == 0) trace_gt(p, 4);
                if (ptx::elect_one()) {  // accumulators ready (immediately if no MMA)
                    if (kPair)
                        ptx::mma_commit_pair(&tfull[acc]);
                    else
                        ptx::mma_commit(&tfull[acc]);
                }
                __syncwarp();
                if (++acc == uint32_t(p.acc_stages)) {
                    acc = 0;
                    acc_ph ^= 1;
                }
            }
        }
        __syncwarp();
    } else if (warp == 2) {
        // ---------------- MMA-program builder (runs ahead of the MMA warp by one tile)
        {
            uint32_t ps = 0, pph = 0;
            for (long long t = t0; t < p.num_tiles && leader; t += tstep) {
                const Tile c = decode_tile(t, p, tab[0], tab[1], tab[2]);
                ptx::mbar_wait(&pempty[ps], pph ^ 1);
                int4* pg = prog + ps * kProgSlot;
                // ---- MMA program of this tile, built by this warp ahead of the MMA warp: entry =
                // one MMA group (A slot, column in slot, first accumulator column, tap
                // of the group's first B tile, N, accumulate flag).  List 0 serves the
                // first row step (groups split by accumulate state), list 1 the others.
                // Lane = activation column; a pixel is "started" in list 0 once an
                // earlier column used it (warp prefix-OR), entry offsets by warp scan.
                int np0 = 0, np1 = 0;
                {
                    const int ncol = c.pos_hi - c.pos_lo;
                    uint32_t carry = 0;
#pragma unroll 1
                    for (int base = 0; base < ncol; base += 32) {
                        const int qa = base + int(lane);
                        const int iw = c.pos_lo + qa;
                        const uint32_t m = qa < ncol ? pos_mask(c, iw) : 0u;
                        uint32_t incl = m;
#pragma unroll
                        for (int off = 1; off < 32; off <<= 1) {
                            const uint32_t v = __shfl_up_sync(0xffffffffu, incl, off);
                            if (int(lane) >= off) incl |= v;
                        }
                        uint32_t excl = __shfl_up_sync(0xffffffffu, incl, 1);
                        if (lane == 0) excl = 0;
                        excl |= carry;
                        // groups of this column in list li (started state st)
                        auto groups = [&](uint32_t started, int off, bool emit) -> int {
                            uint32_t mm = m;
                            int n = 0;
                            while (mm) {
                                const int jlo = __ffs(mm) - 1;
                                const uint32_t st0 = (started >> jlo) & 1u;
                                int cnt = 1;
                                if (p.unit_step) {
                                    while (jlo + cnt < kMaxPBW && ((mm >> (jlo + cnt)) & 1u) &&
                                           (((started >> (jlo + cnt)) & 1u) == st0) && (cnt + 1) * BN <= 256)
                                        ++cnt;
                                }
                                if (emit) {
                                    const int jhi = jlo + cnt - 1;
                                    if (BMN) {  // forward pixel order; slot of pixel jlo's tap, slots ascend with N
                                        const int cw_hi = iw - (c.a0[0] + jlo * p.a0_step);
                                        const int slot0 = p.bcw[tab[1].phase[c.j0]] - 1 - cw_hi;
                                        pg[2 + off + n] = make_int4(qa / p.apos, qa % p.apos, jlo * BN,
                                                                  slot0 | (cnt << 8) | (int(st0) << 16));
                                    } else {
                                        const int cw_lo = iw - (c.a0[0] + jhi * p.a0_step);
                                        pg[2 + off + n] = make_int4(qa / p.apos, qa % p.apos, (p.pbw - 1 - jhi) * BN,
                                                                  cw_lo | (cnt << 8) | (int(st0) << 16));
                                    }
                                }
                                ++n;
                                mm &= ~(((1u << cnt) - 1u) << jlo);
                            }
                            return n;
                        };
                        const int n0 = groups(excl, 0, false), n1 = groups(0xFFu, 0, false);
                        int s0 = n0, s1 = n1;
#pragma unroll
                        for (int off = 1; off < 32; off <<= 1) {
                            const int v0 = __shfl_up_sync(0xffffffffu, s0, off);
                            const int v1 = __shfl_up_sync(0xffffffffu, s1, off);
                            if (int(lane) >= off) {
                                s0 += v0;
                                s1 += v1;
                            }
                        }
                        groups(excl, np0 + s0 - n0, true);
                        groups(0xFFu, kProgEntries + np1 + s1 - n1, true);
                        np0 += __shfl_sync(0xffffffffu, s0, 31);
                        np1 += __shfl_sync(0xffffffffu, s1, 31);
                        carry |= __shfl_sync(0xffffffffu, incl, 31);
                    }
                }
                if (np0 > kProgEntries || np1 > kProgEntries) __trap();  // plan invariant (prog_entries_bound)
                if (lane == 0) {
                    pg[0] = make_int4(np0, np1, c.rs0, c.rs1);
                    pg[1] = make_int4(c.pos_lo, c.pos_hi, 0, 0);
                }
                __syncwarp();
                ptx::mbar_arrive(&pfull[ps]);  // all 32 lanes
                if (++ps == 2) {
                    ps = 0;
                    pph ^= 1;
                }
            }
        }
        __syncwarp();
    } else if (warp >= 4 && int(warp) < 4 + p.epi_warps) {
        // ---------------- epilogue: TMEM -> registers -> fp32 stores
        // (thread = accumulator row = one image; 16-byte vector stores).  With 8
        // epilogue warps, warps w and w + 4 share TMEM sub-partition w & 3 and
        // take alternate 32-column chunks (twice the stores in flight).
        const uint32_t sub = warp & 3;  // TMEM sub-partition: lanes [32*sub, 32*sub+32)
        const uint32_t ew = warp - 4;   // epilogue warp 0..epi_warps-1
        const uint32_t half = ew >> 2, nhalf = uint32_t(p.epi_warps) >> 2;
        const int row = int(sub * 32 + lane);
        const int et = threadIdx.x - 128;  // 0..32*epi_warps-1
        uint32_t ebuf = 0;                 // TMA-store epilogue buffer sequence
        uint32_t acc = 0, acc_ph = 0;
        const int pw_cols = p.pbw * BNo;
        // accumulator buffer released to the MMA issuer (pair: on the leader's barrier)
        const uint32_t tempty_c = ptx::mapa(ptx::smem_u32(tempty), 0);
        auto release = [&](uint32_t a) {
            if (kPair)
                ptx::mbar_arrive_cluster(tempty_c + 8u * a);
            else
                ptx::mbar_arrive(&tempty[a]);
        };
        const bool split = p.zsplit > 1;
        const bool vec4 = (p.out_C % 4) == 0;
        const bool stage = !split && p.epi_stage && vec4;  // coalesced-store epilogue
        int ti = 0;
        if (et == 0) trace_ev(p, 2, ti, 0);
        for (long long t = t0; t < p.num_tiles; t += tstep) {
            const Tile c = decode_tile(t, p, tab[0], tab[1], tab[2]);
            ptx::mbar_wait(&tfull[acc], acc_ph);
            if (et == 0) trace_ev(p, 2, ti, 1);
            ptx::tc_fence_after();
            // M row -> (image, output row).  Batch-as-M: image nblk*128 + row of output row orow.
            // Row groups (rg_ni >= 32): the warp's 32 rows are images of ONE group row wgr,
            // output row orow + wgr * rg_ostep, stored only if wgr < the group length.
            const int wgr = p.rg_ni ? (int(sub * 32) >> p.rg_shift) : 0;
            const bool wlive_row = wgr < c.glen;
            const int orow_w = c.orow + wgr * p.rg_ostep;
            const int nrow0 = p.rg_ni ? (int(sub * 32) & (p.rg_ni - 1)) : c.nblk * 128 + int(sub) * 32;  // image of lane 0
            const int n = nrow0 + int(lane);
            const int cbase = c.nb * BNo;
            const int cvalid = min(BNo, p.out_C - cbase);
            const bool any = c.rs1 > c.rs0;
            // the CTA's last tile: the smem rings are idle (all MMAs done), so stage
            // 32x32 fp32 blocks there (128B swizzle) and write full lines by TMA store
            // other tiles (p.tma_store == 2): the same 32x32 blocks through this warp's
            // 4 KB epilogue buffer, one TMA store in flight per warp (the buffer is
            // reused once the previous store has read it): async full-line stores
            if (p.tma_store == 2 && !split && t + tstep < p.num_tiles && !(p.dbg & 1)) {
                // epi_bufs 4 KB buffers per warp: with 2, one store may still be reading
                // the other buffer while this one is filled
                const uint32_t nbuf = uint32_t(p.epi_bufs);
#pragma unroll 1
                for (int j = 0; j < c.len; ++j) {
                    const bool live = any && (tab[1].te[c.j0 + j] > tab[1].ts[c.j0 + j]);
#pragma unroll 1
                    for (int c0 = 32 * int(half); c0 < BNo; c0 += 32 * int(nhalf)) {
                        uint32_t r[32];
                        ptx::tmem_ld32(tmem_base + ((sub * 32u) << 16) + acc * uint32_t(pw_cols) + (BMN ? j : p.pbw - 1 - j) * BN +
                                           c0, r);
                        ptx::tmem_ld_wait();
                        if (c0 >= cvalid || !wlive_row) continue;
                        float* blk = epi + (ew * nbuf + (ebuf & (nbuf - 1u))) * 1024;
                        ++ebuf;
                        if (ptx::elect_one()) {  // the store that last used this buffer has read it
                            if (nbuf == 2)
                                ptx::bulk_wait_read1();
                            else
                                ptx::bulk_wait_read0();
                        }
                        __syncwarp();
#pragma unroll
                        for (int q = 0; q < 8; ++q) {
                            const float4 v = live ? make_float4(__uint_as_float(r[4 * q]), __uint_as_float(r[4 * q + 1]),
                                                                __uint_as_float(r[4 * q + 2]), __uint_as_float(r[4 * q + 3]))
                                                  : make_float4(0.f, 0.f, 0.f, 0.f);
                            *reinterpret_cast<float4*>(blk + lane * 32 + ((q ^ (lane & 7)) << 2)) = v;
                        }
                        ptx::fence_proxy_async_smem();
                        __syncwarp();
                        if (ptx::elect_one()) {
                            ptx::tma_store_4d(&tmY, blk, cbase + c0, tab[1].out[c.j0 + j], orow_w, nrow0);
                            ptx::bulk_commit();
                        }
                        __syncwarp();
                    }
                }
                ptx::tc_fence_before();
                release(acc);
                if (++acc == uint32_t(p.acc_stages)) {
                    acc = 0;
                    acc_ph ^= 1;
                }
                continue;
            }
            if (p.tma_store && !split && t + tstep >= p.num_tiles && !(p.dbg & 1)) {
                uint8_t* stg = smem + sub * uint32_t(c.len * (BNo / 32)) * 4096u;
#pragma unroll 1
                for (int j = 0; j < c.len; ++j) {
                    const bool live = any && (tab[1].te[c.j0 + j] > tab[1].ts[c.j0 + j]);
#pragma unroll 1
                    for (int c0 = 32 * int(half); c0 < BNo; c0 += 32 * int(nhalf)) {
                        const int k = j * (BNo / 32) + c0 / 32;
                        uint32_t r[32];
                        ptx::tmem_ld32(tmem_base + ((sub * 32u) << 16) + acc * uint32_t(pw_cols) + (BMN ? j : p.pbw - 1 - j) * BN +
                                           c0, r);
                        ptx::tmem_ld_wait();
                        if (c0 >= cvalid || !wlive_row) continue;
                        float* blk = reinterpret_cast<float*>(stg + k * 4096);
#pragma unroll
                        for (int q = 0; q < 8; ++q) {
                            const float4 v = live ? make_float4(__uint_as_float(r[4 * q]), __uint_as_float(r[4 * q + 1]),
                                                                __uint_as_float(r[4 * q + 2]), __uint_as_float(r[4 * q + 3]))
                                                  : make_float4(0.f, 0.f, 0.f, 0.f);
                            *reinterpret_cast<float4*>(blk + lane * 32 + ((q ^ (lane & 7)) << 2)) = v;
                        }
                        ptx::fence_proxy_async_smem();
                        __syncwarp();
                        if (ptx::elect_one()) {
                            ptx::tma_store_4d(&tmY, blk, cbase + c0, tab[1].out[c.j0 + j], orow_w, nrow0);
                            ptx::bulk_commit();
                        }
                        __syncwarp();
                    }
                }
                if (ptx::elect_one()) ptx::bulk_wait_read0();  // smem must outlive the TMA reads
                __syncwarp();
                ptx::tc_fence_before();
                release(acc);
                if (++acc == uint32_t(p.acc_stages)) {
                    acc = 0;
                    acc_ph ^= 1;
                }
                continue;
            }
#pragma unroll 1
            for (int j = 0; j < c.len; ++j) {
                const bool live = any && (tab[1].te[c.j0 + j] > tab[1].ts[c.j0 + j]);
                float* dst = nullptr;
                if (split && p.zc)  // own smem (idle rings): column group q = (j*BN + c)/4, [q][128 rows] float4
                    dst = reinterpret_cast<float*>(smem) + (j * (BN / 4)) * 512 + row * 4;
                else if (split)  // column group q = (j*BN + c)/4 of row `row`
                    dst = p.part + ((c.out_tile * p.zsplit + c.z) * (pw_cols / 4) + j * (BN / 4)) * 512LL + row * 4;
                else if (n < p.N && wlive_row)
                    dst = p.out + ((static_cast<long long>(n) * p.out_H + orow_w) * p.out_W +
                                   tab[1].out[c.j0 + j]) * p.out_C + cbase;
                const int lim = split ? BN : cvalid;
#pragma unroll 1
                for (int c0 = 32 * int(half); c0 < BNo; c0 += 32 * int(nhalf)) {
                    uint32_t r[32];
                    ptx::tmem_ld32(tmem_base + ((sub * 32u) << 16) + acc * uint32_t(pw_cols) + (BMN ? j : p.pbw - 1 - j) * BN + c0,
                                   r);
                    ptx::tmem_ld_wait();
                    if (c0 >= lim || (p.dbg & 1) || (dst == nullptr && !stage) || (stage && !wlive_row))
                        continue;  // stage: warp-uniform
                    if (!live) {
#pragma unroll
                        for (int q = 0; q < 32; ++q) r[q] = 0u;
                    }
                    if (stage) {
                        // transpose through a 128B-swizzled 32 x 32 block: 8 lanes write one
                        // image's 32 channels (128 B, a full line) per store instruction
                        float* blk = epi + ew * uint32_t(p.epi_bufs) * 1024;
#pragma unroll
                        for (int q = 0; q < 8; ++q)
                            *reinterpret_cast<float4*>(blk + lane * 32 + ((q ^ (lane & 7)) << 2)) =
                                make_float4(__uint_as_float(r[4 * q]), __uint_as_float(r[4 * q + 1]),
                                            __uint_as_float(r[4 * q + 2]), __uint_as_float(r[4 * q + 3]));
                        __syncwarp();
                        const int cq = int(lane & 7);
#pragma unroll
                        for (int k = 0; k < 8; ++k) {
                            const int rr = 4 * k + int(lane >> 3);
                            const float4 v = *reinterpret_cast<const float4*>(blk + rr * 32 + ((cq ^ (rr & 7)) << 2));
                            const int nn = nrow0 + rr;
                            const int cc = c0 + 4 * cq;
                            if (nn < p.N && cc < lim)
                                *reinterpret_cast<float4*>(p.out + ((static_cast<long long>(nn) * p.out_H +
                                                                     orow_w) * p.out_W +
                                                                    tab[1].out[c.j0 + j]) * p.out_C + cbase + cc) = v;
                        }
                        __syncwarp();
                    } else if (split) {
#pragma unroll
                        for (int q = 0; q < 32; q += 4)
                            *reinterpret_cast<float4*>(dst + (c0 + q) / 4 * 512) =
                                make_float4(__uint_as_float(r[q]), __uint_as_float(r[q + 1]),
                                            __uint_as_float(r[q + 2]), __uint_as_float(r[q + 3]));
                    } else if (vec4 && c0 + 32 <= lim) {
#pragma unroll
                        for (int q = 0; q < 32; q += 4)
                            *reinterpret_cast<float4*>(dst + c0 + q) =
                                make_float4(__uint_as_float(r[q]), __uint_as_float(r[q + 1]),
                                            __uint_as_float(r[q + 2]), __uint_as_float(r[q + 3]));
                    } else {
#pragma unroll
                        for (int q = 0; q < 32; ++q)
                            if (c0 + q < lim) dst[c0 + q] = __uint_as_float(r[q]);
                    }
                }
            }
            // TMEM drained: release the accumulator buffer before the split-K reduce
            if (et == 0) trace_ev(p, 2, ti, 2);
            ptx::tc_fence_before();
            release(acc);
            if (++acc == uint32_t(p.acc_stages)) {
                acc = 0;
                acc_ph ^= 1;
            }
            if (split && !p.zc) {
                __threadfence();
                asm volatile("bar.sync 1, %0;" ::"r"(32 * p.epi_warps) : "memory");
                if (et == 0) {
                    const int old = atomicAdd(&p.sem[c.out_tile], 1);
                    const int last = old == p.zsplit - 1;
                    if (last) p.sem[c.out_tile] = 0;  // leave the counter zeroed for the next call
                    *red_flag = last;
                    __threadfence();
                }
                __syncwarp();
                asm volatile("bar.sync 1, %0;" ::"r"(32 * p.epi_warps) : "memory");
                if (et == 0) trace_ev(p, 2, ti, 3);
                if (*red_flag && n < p.N && wlive_row && half == 0) {
                    // last segment: sum the Z partials in order z = 0..Z-1; thread = row,
                    // 8 column groups x Z vector loads in flight, coalesced 512 B per warp load
                    const float4* base = reinterpret_cast<const float4*>(p.part) +
                                         (c.out_tile * p.zsplit) * (pw_cols / 4) * 128LL + row;
                    const long long zs = (pw_cols / 4) * 128LL;
                    for (int j = 0; j < c.len; ++j) {
                        float* orow = p.out + ((static_cast<long long>(n) * p.out_H + orow_w) * p.out_W +
                                               tab[1].out[c.j0 + j]) * p.out_C + cbase;
                        for (int c0 = 0; c0 < cvalid; c0 += 32) {
                            const float4* src = base + (j * BN + c0) / 4 * 128LL;
                            float4 v[8];
#pragma unroll
                            for (int q = 0; q < 8; ++q) v[q] = __ldcg(src + q * 128);
                            for (int z = 1; z < p.zsplit; ++z) {
                                float4 w[8];
#pragma unroll
                                for (int q = 0; q < 8; ++q) w[q] = __ldcg(src + z * zs + q * 128);
#pragma unroll
                                for (int q = 0; q < 8; ++q) {
                                    v[q].x += w[q].x;
                                    v[q].y += w[q].y;
                                    v[q].z += w[q].z;
                                    v[q].w += w[q].w;
                                }
                            }
                            if (vec4 && c0 + 32 <= cvalid) {
#pragma unroll
                                for (int q = 0; q < 8; ++q) *reinterpret_cast<float4*>(orow + c0 + 4 * q) = v[q];
                            } else {
#pragma unroll
                                for (int q = 0; q < 8; ++q) {
                                    const float e[4] = {v[q].x, v[q].y, v[q].z, v[q].w};
#pragma unroll
                                    for (int u = 0; u < 4; ++u)
                                        if (c0 + 4 * q + u < cvalid) orow[c0 + 4 * q + u] = e[u];
                                }
                            }
                        }
                    }
                }
                __syncwarp();
                asm volatile("bar.sync 1, %0;" ::"r"(32 * p.epi_warps) : "memory");  // red_flag reuse guard
                if (et == 0) trace_ev(p, 2, ti, 4);
            }
        }
    }
    ptx::block_sync();
    if (p.zc) {
        // cluster split-K reduce: every rank's segment is staged in its smem
        ptx::cluster_sync();
        if (warp >= 4 && warp < 8 && blockIdx.x < p.num_tiles && !(p.dbg & 1)) {
            const Tile c = decode_tile(blockIdx.x, p, tab[0], tab[1], tab[2]);
            const int row = int(threadIdx.x) - 128;  // accumulator row = image (row groups: see epilogue)
            const int gr = p.rg_ni ? (row >> p.rg_shift) : 0;
            const int n = p.rg_ni ? (row & (p.rg_ni - 1)) : c.nblk * 128 + row;
            const int G = c.len * (BN / 4);  // float4 column groups of the tile
            const int g0 = (c.z * G) / p.zsplit, g1 = ((c.z + 1) * G) / p.zsplit;
            const int cbase = c.nb * BN;
            const int cvalid = min(BN, p.out_C - cbase);
            const uint32_t sbase = ptx::smem_u32(smem) + uint32_t(row) * 16u;
            if (n < p.N && gr < c.glen) {
                // two column groups x Z ranks of DSMEM loads in flight, then the fixed-order sums
#pragma unroll 1
                for (int gq = g0; gq < g1; gq += 2) {
                    const bool two = gq + 1 < g1;
                    const uint32_t off = sbase + uint32_t(gq) * 2048u;
                    float4 a[8], b[8];
#pragma unroll
                    for (int z = 0; z < 8; ++z) {
                        if (z < p.zsplit) {
                            a[z] = ptx::ld_dsmem_f4(ptx::mapa(off, uint32_t(z)));
                            if (two) b[z] = ptx::ld_dsmem_f4(ptx::mapa(off + 2048u, uint32_t(z)));
                        }
                    }
#pragma unroll
                    for (int h = 0; h < 2; ++h) {
                        if (h == 1 && !two) break;
                        float4 v = h ? b[0] : a[0];
#pragma unroll
                        for (int z = 1; z < 8; ++z) {  // fixed order z = 0..Z-1
                            if (z < p.zsplit) {
                                const float4 w = h ? b[z] : a[z];
                                v.x += w.x;
                                v.y += w.y;
                                v.z += w.z;
                                v.w += w.w;
                            }
                        }
                        const int gg = gq + h;
                        const int j = gg / (BN / 4), cc = (gg % (BN / 4)) * 4;
                        if (cc >= cvalid) continue;
                        float* o = p.out + ((static_cast<long long>(n) * p.out_H + c.orow + gr * p.rg_ostep) * p.out_W +
                                            tab[1].out[c.j0 + j]) * p.out_C + cbase + cc;
                        if ((p.out_C % 4) == 0 && cc + 4 <= cvalid) {
                            *reinterpret_cast<float4*>(o) = v;
                        } else {
                            const float e[4] = {v.x, v.y, v.z, v.w};
                            for (int u = 0; u < 4 && cc + u < cvalid; ++u) o[u] = e[u];
                        }
                    }
                }
            }
        }
        ptx::cluster_sync();  // peers finished reading this CTA's staging
    } else if (p.cm > 1 || kPair) {
        ptx::cluster_sync();  // no CTA leaves while peers may still signal it
    }
    if (threadIdx.x == 0) trace_gt(p, 5);
    if (warp == 2) {
        ptx::tc_fence_after();
        if (kPair)
            ptx::tmem_dealloc_pair(tmem_base, tmem_cols);
        else
            ptx::tmem_dealloc(tmem_base, tmem_cols);
    }
}

}  // namespace cks
