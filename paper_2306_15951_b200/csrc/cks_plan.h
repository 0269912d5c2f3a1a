// cks_plan.h -- host-side geometry, index tables and tiling plan (layer L1).
//
// Closed-form versions of the per-axis tables of the C-K-S algorithms
// (PAPER.md Appendix, Alg. 1 / 2 / 2B / 3B) under the readings of
// SURVEY.md §8(c) (c1-c16).  The kernels consume exactly these tables; the
// CPU test suite checks them bit-exactly against the oracle's brute-force
// enumeration (tests/test_plan_abi.py).
#pragma once
#include <cstdint>
#include <cstdlib>
#include <string>
#include <vector>

#include "../../include/cks.h"

namespace cks {

// Experiment knob: getenv(name) in the experiments build (-DCKS_EXPERIMENTS,
// libcks_exp.so), nullptr in the production library (no environment reads).
#ifdef CKS_EXPERIMENTS
inline const char* cks_knob(const char* name) { return getenv(name); }
#else
constexpr const char* cks_knob(const char*) { return nullptr; }
#endif

// Mathematical floor / ceil division (correct for negative numerators; C++
// '/' truncates toward zero, and oh_s can be -1 -- SURVEY.md §7 hard part 6).
inline int64_t fdiv(int64_t a, int64_t b) {
    int64_t q = a / b, r = a % b;
    return (r != 0 && ((r < 0) != (b < 0))) ? q - 1 : q;
}
inline int64_t cdiv(int64_t a, int64_t b) { return -fdiv(-a, b); }
inline int64_t fmod_pos(int64_t a, int64_t b) { return a - fdiv(a, b) * b; }

struct Axis {
    int64_t I, F, s, p, O;
};

struct T1Row { int64_t o, ih_s, f_s, f_e; };
struct T2Row { int64_t u, ih, oh_s, ch_s, ch_e; };
struct T2Phase {
    int64_t y, CH, oph, ih_s, U, a;
    std::vector<T2Row> rows;
};
struct T3Row { int64_t f, ih_s, oh_s, oh_e; };
struct T4Run { int64_t o_start, o_end, f_s, f_e; };

cks_status validate(const cks_geom* g);
Axis axis_h(const cks_geom& g);
Axis axis_w(const cks_geom& g);
int64_t out_extent(int64_t I, int64_t F, int64_t s, int64_t p);

std::vector<T1Row> table_t1(const Axis& a);      // Alg. 1 trim
std::vector<T2Phase> table_t2(const Axis& a);    // Alg. 2 / 2B phases
std::vector<T3Row> table_t3(const Axis& a);      // Alg. 3B taps
std::vector<T4Run> table_t4(const Axis& a);      // trim classes
int64_t axis_valid_pairs(const Axis& a);         // V

// Per-axis row list consumed by the implicit-GEMM kernel (fwd / deconv).
// Row r: A-operand coordinate of tap 0 (a0), trimmed tap window [ts, te),
// output coordinate, phase index.  Fwd: one row per output o (T1).  Deconv:
// the T2 rows of all phases in phase order.
// glen: row groups (below) -- the group holds rows [this, this + glen) of the
// ungrouped table, all with this row's window and phase.
struct KRow { int64_t a0, ts, te, out, phase; int64_t glen = 1; };
std::vector<KRow> krows_fwd(const Axis& a);
std::vector<KRow> krows_deconv(const Axis& a);

// Row groups for small per-GPU batches (N <= 64): the implicit GEMM's M = 128
// rows become rg_ph = 128 / rg_ni consecutive output rows x rg_ni images
// (rg_ni = 32 or 64), so a batch of 32 images fills the tensor-core tile
// instead of a quarter of it.  A group is a run of <= ph rows of one phase
// with the SAME trimmed window (trim-homogeneous), A coordinates a0
// stepping by es (the TMA element stride of the A box) and outputs by ostep.
std::vector<KRow> group_rows(const std::vector<KRow>& rows, int ph, int64_t es, int64_t ostep);
// Start indices of the affine runs of a row table (one phase, one group
// length, a0 and out affine in the run index): the kernel's compact axis form.
std::vector<int> run_starts(const std::vector<KRow>& rows);
int rg_images(int64_t N);  // 32 / 64 images per M tile (row groups), 0 = batch-as-M (N > 64)

// MMA-program capacity of the implicit GEMM (kernels/igemm.cuh): entries per
// list.  Every entry is one MMA group covering >= 1 (pixel, tap) pair of the
// tile and no pair appears twice in a list, so pbw * ntap bounds a tile's
// entries; the plan narrows the pixel block until that fits.
constexpr int kProgEntries = 64;
inline int64_t prog_entries_bound(int64_t pbw, int64_t ntap, int64_t /*a0_step*/, int /*BN*/) { return pbw * ntap; }

// channel padding to 16-byte rows
inline int64_t pad_ch(int64_t c, cks_dtype dt) {
    int64_t q = dt == CKS_BF16 ? 8 : 4;
    return (c + q - 1) / q * q;
}
inline int64_t elem_bytes(cks_dtype dt) { return dt == CKS_BF16 ? 2 : 4; }

// Kernel configuration decisions (shared by workspace query and launch).
// The implicit GEMM tiles PBW consecutive pixels of one output row x 128
// images x BN channels; under-filled grids split the row steps into Z
// segments (deterministic in-kernel split-K).
struct IgemmCfg {
    int BN = 128;       // output-channel tile (32, 64, 128)
    int pbw = 1;        // pixels per tile along w
    int acc_stages = 2; // TMEM accumulator buffers
    int nbs = 1;        // number of BN tiles
    int nblk = 1;       // ceil(N / 128)
    int wblocks = 1;
    int Z = 1;          // split-K segments
    int zc = 0;         // cluster split-K (Z CTAs of one cluster per output tile, DSMEM reduce)
    int epi_warps = 4;  // epilogue warps (4 or 8)
    int epi_bufs = 1;   // TMA-store staging buffers per epilogue warp (1 or 2)
    int pair = 0;       // CTA pair (cta_group::2): nblk counts image-block pairs, BN = this CTA's half
    int kc_blocks = 1;
    int KB = 128;       // bytes per K row: 32 / 64 / 128 (swizzle width)
    int ntap = 1;       // taps per filter row (B box)
    int pa = 1;         // activation positions per row step (A box)
    int stage_bytes = 0, stages = 2;  // B-row ring: bytes per row, rows in flight
    int a_stages = 8;                 // A ring (slots of apos x 16 KB)
    int epi = 0;                      // epilogue staging buffers present
    int cm = 1;                       // cluster size along the BN blocks (A-tile multicast)
    int unified = 0;                  // A slot + B row of a row step share one barrier pair
    int apos = 2;                     // activation columns per A slot
    int unit_step = 1;                // consecutive pixels' tap-0 columns differ by 1
    int a0_step = 1;                  // tap-0 column step between consecutive pixels
    int64_t out_tiles = 0, tiles = 0;
    std::vector<int64_t> wph_cnt;  // rows per w phase
    int rg_ni = 0;                 // row groups: images per M tile (0 = off: M = 128 images)
    int rg_ph = 1;                 // row groups: output rows per M tile (128 / rg_ni)
    int rg_es = 1;                 // row groups: A-row step inside a group (TMA element stride)
    int rg_ostep = 1;              // row groups: output-row step inside a group
};
IgemmCfg igemm_cfg(int64_t rows_h, const std::vector<int64_t>& wph_cnt, int64_t N, int64_t nout, int64_t kchan,
                   int64_t eb, int64_t max_taps_h, int64_t ntap, int64_t a0_step, int num_sms, int force_pbw = 0,
                   int force_bn = 0, int rg_ni = 0);
// Row groups of a 2-D layer: rg_ni for the forward / KS-deconv h axis (0 when
// N > 64 or the grouped table does not fit the kernel's compact axis form),
// and the h-axis rows the igemm runs over (grouped when rg_ni > 0).  A forward
// group's A rows step by s_h (TMA element stride), its outputs by 1; a
// KS-deconv group's A rows step by 1 (one phase), its outputs by s_h.
int rg_plan(const cks_geom& g, bool deconv);
std::vector<KRow> igemm_rows_fwd(const cks_geom& g, int rg_ni);
std::vector<KRow> igemm_rows_deconv(const cks_geom& g, int rg_ni);
constexpr int kSmemBudget = 227 * 1024 - 1024 - 512 - 5376 - 4160;  // minus alignment, barriers, 3 axis tables, MMA programs
constexpr int kEpiStageBytes = 4 * 4096;  // epilogue transpose staging: 4 warps x (32 x 32 fp32)
constexpr int epi_stage_bytes(int epi_warps, int bufs = 1) { return epi_warps * bufs * 4096; }
bool epi_staging();                       // coalesced-store epilogue (default on; CKS_EPI_STAGE=0 disables)
IgemmCfg igemm_cfg_fwd(const cks_geom& g, cks_dtype dt, int num_sms);
IgemmCfg igemm_cfg_deconv(const cks_geom& g, cks_dtype dt, int num_sms);
// Stage1-free KS-deconv: the implicit GEMM reads W
// directly as an MN-major B operand (kernels/igemm.cuh BMN).  Eligible when
// W rows are 16-byte multiples (IC * eb % 16 == 0), sw <= 8 (TMA element
// stride) and the phases fit the kernel tables; ks_direct() is the policy the
// library applies to a cks_deconv2d call given W (not packed sub-filters).
bool ks_direct_eligible(const cks_geom& g, cks_dtype dt);
bool ks_direct(const cks_geom& g, cks_dtype dt, int num_sms);
IgemmCfg igemm_cfg_deconv_w(const cks_geom& g, cks_dtype dt, int num_sms);

// Narrow-channel row path (kernels/narrow.cuh): one filter row's contiguous
// (fw, c) run is one K-block of JB elements (ROWB = JB * element bytes).
// Eligible for FW*C small enough that a run (+ its alignment shift) fits a
// 64-element bf16 / 32-element fp32 row, C <= 16 (bf16) / 8 (fp32), and a
// 16-byte X row pitch (W*C*eb % 16 == 0).
#ifndef CKS_ROW_EPI_BUFS
#define CKS_ROW_EPI_BUFS 2  // KB-CONV-ROW TMA-store staging buffers per epilogue warp (kernels/narrow.cuh)
#endif
constexpr int kRowClasses = 24;  // column classes per launch (kernels/narrow.cuh RowClass table)
struct RowClassH {
    int col0 = 0, cstep = 1, ncols = 0;  // output columns col0 + cstep * i
    int off = 0;                         // box origin = (ow*sw - pw)*C + off
    int kc0 = 0, kc1 = 0;                // 32-byte K chunks holding valid elements (ConvV2)
    int base = 0, cnt = 1;               // ConvV2: CTA range; Sk-dilated: partial range
    int64_t work = 0;                    // tiles (ConvV2) / k-blocks (Sk-dilated) of the class
};
struct RowCfg {
    bool ok = false;
    int ROWB = 0;        // bytes per box row: 32 / 64 / 128
    int JB = 0;          // elements per box row
    int BN = 0;          // OC tile
    int R = 1;           // ConvV2: output rows per tile
    int stages = 0;      // pipeline depth
    int smem = 0;        // dynamic shared memory bytes
    int mb = 1, nbs = 1, gz = 1, nblk = 1;  // wgrad: M-blocks, OC blocks, G_Z (total partials), 64-image blocks
    int q = 1;           // wgrad: output rows per k-block (one X box of FH + sh * (q - 1) rows)
    int rg = 0;          // ConvV2 row groups (N <= 64): images per M tile (32 / 64), 0 = 128-image M tiles
    int rg_pc = 1;       // row groups: class columns per M tile (ConvV2: 128 / rg) / per k-block (wgrad: 64 / rg)
    std::vector<RowClassH> cls;
    int grid = 1;        // CTAs
    int64_t tiles = 0;
};
RowCfg row_cfg_fwd(const cks_geom& g, cks_dtype dt, bool allow_rg = true);
RowCfg row_cfg_wgrad(const cks_geom& g, cks_dtype dt, int gz_req, int num_sms, bool allow_rg = true);
// Products of the row kernels with spatial-padding zeros (host model, per
// image): ConvV2 (the partial last K chunk of right-border columns) and
// Sk-dilated (zero-fill rows inside an issued M-block, box elements beyond
// the image in w).  Reported in DESIGN.md; tests pin the ConvV2 count.
int64_t row_fwd_padding_macs(const cks_geom& g, cks_dtype dt);
int64_t row_wgrad_padding_macs(const cks_geom& g, cks_dtype dt);

struct WgradCfg {
    int BN, nbs, mblocks, nblk64, gz;
    int64_t base_tiles;
    bool row = false;  // narrow-channel row kernel
    int kimg = 64;     // images per k-block (64 or 128)
    int mt = 1;        // taps per tile along w: 1, or F_W (row tiles sharing the dY block)
    int zc = 0;        // cluster reduce: the gz segments of a tile form one cluster (DSMEM sum, no partials)
    int a1 = 0;        // O_C <= 64 (bf16, BN = 64): one dY atom per ring stage
    int tc = 0;        // filter-row group (row tiles: the F_H filter rows of a segment walk the same k-blocks)
    int tcmc = 0;      // the group is a cluster with dY multicast
    int pp = 0;        // position pairs (M = two positions' dY; halves written as 2 G_Z partials per segment)
    int rg = 0;        // row groups (N <= kimg / 2): images per k-block position chunk (16 / 32), 0 = off
    int rg_pk = 1;     // row groups: output positions per k-block (kimg / rg)
    int npart() const { return pp ? 2 * gz : gz; }  // fp32 partials the segments write (>1: KB-REDUCE)
};
WgradCfg wgrad_cfg(const cks_geom& g, cks_dtype dt, int gz_req, int num_sms);

// Workspace layout (byte offsets, 256-aligned) for one op.
struct WsLayout {
    size_t x_pad = 0, w_pad = 0, dy_pad = 0, c_packed = 0, partial = 0, sem = 0, total = 0;
    size_t x_pad_bytes = 0, w_pad_bytes = 0, dy_pad_bytes = 0, c_packed_bytes = 0, partial_bytes = 0, sem_bytes = 0;
    size_t mp_w = 0, mp_y = 0, mp_inner = 0;  // multi-phase KS-deconv: stacked filter, pseudo output, inner ws
    size_t mp_w_bytes = 0, mp_y_bytes = 0, mp_inner_bytes = 0;
};

// Multi-phase KS-deconv for narrow outputs (kernels/aux.cuh ks_mp_*): the
// phases stacked on N of one unit-stride ConvV2 over dY (pseudo geometry
// `pg`: X := dY, OC := NP stacked channels, F := CH x CW, padding ph2, pw2).
struct MpPlan {
    bool ok = false;
    int CH = 0, CW = 0, NP = 0, ph2 = 0, pw2 = 0;
    int16_t ih_s[8], a_y[8], iw_s[8], a_x[8];
    cks_geom pg;
};
MpPlan mp_plan(const cks_geom& g, cks_dtype dt);
WsLayout ws_layout(const cks_geom& g, cks_dtype dt, cks_op op, int gz, bool c_packed_given, int num_sms);
size_t ks_split_bytes(const cks_geom& g, cks_dtype dt);

// 3-D (cks_geom3): the (H, W) plane as a 2-D geometry, the depth axis, plans.
cks_status validate3(const cks_geom3* g);
cks_geom plane_geom(const cks_geom3& g);
Axis axis_d(const cks_geom3& g);
IgemmCfg igemm_cfg_fwd3(const cks_geom3& g, cks_dtype dt, int num_sms);
IgemmCfg igemm_cfg_deconv3(const cks_geom3& g, cks_dtype dt, int num_sms);
WgradCfg wgrad_cfg3(const cks_geom3& g, cks_dtype dt, int gz_req, int num_sms);
WsLayout ws_layout3(const cks_geom3& g, cks_dtype dt, cks_op op, int gz, int num_sms);

// Text form of the plan the library uses for (g, dt, op, gz) -- kernel kind
// and tile configuration as key=value pairs (tests, tools/plan_dump.py).
std::string describe_plan(const cks_geom& g, cks_dtype dt, cks_op op, int gz, int num_sms);

}  // namespace cks
