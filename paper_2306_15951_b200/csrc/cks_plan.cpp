// cks_plan.cpp -- host-side geometry, closed-form index tables, tiling plan.
// See cks_plan.h.  Citations: P:<line> = PAPER.md; readings c1-c16 =
// SURVEY.md §8(c), listed in DESIGN.md.
#include "cks_plan.h"

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <unordered_map>

namespace cks {

int64_t out_extent(int64_t I, int64_t F, int64_t s, int64_t p) {
    return fdiv(I + 2 * p - F, s) + 1;  // Table I shape rule (reading c10)
}

cks_status validate(const cks_geom* g) {
    if (!g) return CKS_ERR_NULL;
    if (g->N < 1 || g->C < 1 || g->H < 1 || g->W < 1 || g->OC < 1 || g->FH < 1 || g->FW < 1)
        return CKS_ERR_GEOMETRY;
    if (g->sh < 1 || g->sw < 1 || g->ph < 0 || g->pw < 0) return CKS_ERR_GEOMETRY;
    if (g->ph >= g->FH || g->pw >= g->FW) return CKS_ERR_GEOMETRY;  // reading c16
    if (g->H + 2 * g->ph - g->FH < 0 || g->W + 2 * g->pw - g->FW < 0) return CKS_ERR_GEOMETRY;
    if (g->dh != 1 || g->dw != 1) return CKS_ERR_UNSUPPORTED;        // dilate == stride
    if (g->FH > 32 || g->FW > 32 || g->sh > 8 || g->sw > 8) return CKS_ERR_UNSUPPORTED;
    if (g->N > (int64_t(1) << 30) || g->H > 65535 || g->W > 65535) return CKS_ERR_UNSUPPORTED;
    return CKS_OK;
}

Axis axis_h(const cks_geom& g) { return {g.H, g.FH, g.sh, g.ph, out_extent(g.H, g.FH, g.sh, g.ph)}; }
Axis axis_w(const cks_geom& g) { return {g.W, g.FW, g.sw, g.pw, out_extent(g.W, g.FW, g.sw, g.pw)}; }

// T1 -- Alg. 1, reading c1: ih_s = o*s - p, [f_s, f_e) with
// f_s = max(-ih_s, 0), f_e = min(I - ih_s, F)  ("ending at (fh_e-1, fw_e-1)").
std::vector<T1Row> table_t1(const Axis& a) {
    std::vector<T1Row> t;
    for (int64_t o = 0; o < a.O; ++o) {
        int64_t ih_s = o * a.s - a.p;
        t.push_back({o, ih_s, std::max<int64_t>(-ih_s, 0), std::min(a.I - ih_s, a.F)});
    }
    return t;
}

// T2 -- Alg. 2 Stage1/Stage2&3 + 2B, readings c2 (C extent
// ceil), c3 (rows while ih < I), c4 (trim end min(O - oh_s, CH_y)), c11
// (empty phases), c12 (phase y writes ih = (y - p) mod s).
std::vector<T2Phase> table_t2(const Axis& a) {
    std::vector<T2Phase> out;
    for (int64_t y = 0; y < a.s; ++y) {
        T2Phase ph;
        ph.y = y;
        ph.CH = a.F > y ? cdiv(a.F - y, a.s) : 0;     // ceil((F_H - y)/sh)
        ph.oph = ph.CH - 1;
        int64_t ih_s = y - a.p;                         // Alg. 2: ih_s = y - ph
        if (ih_s < 0) ih_s += cdiv(-ih_s, a.s) * a.s;  //  += ceil(-ih_s/sh)*sh
        ph.ih_s = ih_s;
        ph.U = ih_s < a.I ? cdiv(a.I - ih_s, a.s) : 0;
        // oh_s(u) = (ih + ph - y)/sh - oph = u + a  (exact division)
        ph.a = (ph.CH > 0 && ph.U > 0) ? fdiv(ih_s + a.p - y, a.s) - ph.oph : 0;  // 0 for empty phases
        for (int64_t u = 0; u < ph.U; ++u) {
            T2Row r{u, u * a.s + ih_s, 0, 0, 0};
            if (ph.CH > 0) {
                r.oh_s = u + ph.a;
                int64_t cs = std::max<int64_t>(-r.oh_s, 0);
                int64_t ce = std::min(a.O - r.oh_s, ph.CH);
                if (ce > cs) { r.ch_s = cs; r.ch_e = ce; }
            }
            ph.rows.push_back(r);
        }
        out.push_back(std::move(ph));
    }
    return out;
}

// T3 -- Alg. 3B, reading c5: ih_s = f - p,
// oh_s = max(ceil(-ih_s/s), 0), oh_e = min(O, ceil((I - ih_s)/s)); empty -> (0,0).
std::vector<T3Row> table_t3(const Axis& a) {
    std::vector<T3Row> t;
    for (int64_t f = 0; f < a.F; ++f) {
        int64_t ih_s = f - a.p;
        int64_t os = std::max<int64_t>(cdiv(-ih_s, a.s), 0);
        int64_t oe = std::min(a.O, cdiv(a.I - ih_s, a.s));
        if (oe <= os) os = oe = 0;
        t.push_back({f, ih_s, os, oe});
    }
    return t;
}

std::vector<T4Run> table_t4(const Axis& a) {
    std::vector<T4Run> runs;
    for (const auto& r : table_t1(a)) {
        if (!runs.empty() && runs.back().f_s == r.f_s && runs.back().f_e == r.f_e && runs.back().o_end == r.o)
            runs.back().o_end = r.o + 1;
        else
            runs.push_back({r.o, r.o + 1, r.f_s, r.f_e});
    }
    return runs;
}

int64_t axis_valid_pairs(const Axis& a) {
    int64_t v = 0;
    for (const auto& r : table_t1(a)) v += std::max<int64_t>(r.f_e - r.f_s, 0);
    return v;
}

std::vector<KRow> krows_fwd(const Axis& a) {
    std::vector<KRow> r;
    for (const auto& t : table_t1(a)) r.push_back({t.ih_s, t.f_s, t.f_e, t.o, 0});
    return r;
}

std::vector<KRow> krows_deconv(const Axis& a) {
    std::vector<KRow> r;
    for (const auto& ph : table_t2(a))
        for (const auto& row : ph.rows) r.push_back({row.oh_s, row.ch_s, row.ch_e, row.ih, ph.y});
    return r;
}

std::vector<KRow> group_rows(const std::vector<KRow>& rows, int ph, int64_t es, int64_t ostep) {
    std::vector<KRow> g;
    for (size_t i = 0; i < rows.size();) {
        KRow r = rows[i];
        size_t j = i + 1;
        while (j < rows.size() && int(j - i) < ph && rows[j].phase == r.phase && rows[j].ts == r.ts &&
               rows[j].te == r.te && rows[j].a0 == r.a0 + int64_t(j - i) * es &&
               rows[j].out == r.out + int64_t(j - i) * ostep)
            ++j;
        r.glen = int64_t(j - i);
        g.push_back(r);
        i = j;
    }
    return g;
}

std::vector<int> run_starts(const std::vector<KRow>& rows) {
    std::vector<int> st;
    size_t s = 0;
    int64_t a0st = 0, outst = 0;
    for (size_t i = 0; i < rows.size(); ++i) {
        const KRow& r = rows[i];
        bool start = i == 0 || r.phase != rows[i - 1].phase || r.glen != rows[i - 1].glen;
        if (!start) {
            const int64_t u = int64_t(i - s);
            if (u == 1) {
                a0st = r.a0 - rows[s].a0;
                outst = r.out - rows[s].out;
            } else if (r.a0 != rows[s].a0 + u * a0st || r.out != rows[s].out + u * outst) {
                start = true;
            }
        }
        if (start) {
            st.push_back(int(i));
            s = i;
            a0st = outst = 0;
        }
    }
    return st;
}

// Experiment knobs (tools/ sweeps only; compiled in only with -DCKS_EXPERIMENTS,
// i.e. the separate libcks_exp.so that CKS_EXPERIMENTS=1 builds and loads), read once
// per process: CKS_IGEMM_CFG="BN,PBW,Z[,APOS,BSTAGES]" overrides the tile
// heuristic, CKS_IGEMM_KB caps the K-block bytes, CKS_EPI_STAGE=0 /
// CKS_UNIFIED=0 disable the coalesced epilogue / unified stage barriers,
// CKS_MCAST=1 enables the (slower) cluster multicast of A.
struct Knobs {
    bool ov = false;
    int bn = 0, pbw = 0, z = 0, apos = 0, bst = 0;
    int kb = 0, epi = 1, unified = 1, mcast = 0, kimg128 = 1, zc = 1, epi8 = 0, wmt = 1, pair = 1, smem_cap = 0,
        gz_max = 64, wzc = 2, epi_bufs = 1, wa1 = 1, wmt_tf32 = 1, wa1_tf32 = 1, wtc = 1, pair_tf32 = 1, tf32_wide = 1, wpp = 1, pair_waves_tf32 = 25, bf16_wide = 1, wmt128 = 1, ks_mp = 1, rg = 1, wrow_q = 0, acc1 = 0, wmt_lmin = -1;
    Knobs() {
        if (const char* e = cks_knob("CKS_IGEMM_CFG")) ov = sscanf(e, "%d,%d,%d,%d,%d", &bn, &pbw, &z, &apos, &bst) >= 3;
        if (const char* e = cks_knob("CKS_IGEMM_KB")) kb = atoi(e);
        if (const char* e = cks_knob("CKS_EPI_STAGE")) epi = atoi(e) != 0;
        if (const char* e = cks_knob("CKS_UNIFIED")) unified = atoi(e) != 0;
        if (const char* e = cks_knob("CKS_MCAST")) mcast = atoi(e) == 1;
        if (const char* e = cks_knob("CKS_WGRAD_KIMG")) kimg128 = atoi(e) == 128;
        if (const char* e = cks_knob("CKS_IGEMM_ZC")) zc = atoi(e) != 0;  // 0: legacy global split-K
        // 1: 8 epilogue warps where free, 2: always (measured: no gain, tools/ab.sh) -- experiments
        if (const char* e = cks_knob("CKS_EPI8")) epi8 = atoi(e);
        if (const char* e = cks_knob("CKS_WGRAD_MT")) wmt = atoi(e) != 0;  // 0: one tap per wgrad tile
        if (const char* e = cks_knob("CKS_PAIR")) pair = atoi(e) != 0;      // 0: no 2-CTA igemm tiles
        if (const char* e = cks_knob("CKS_PAIR_TF32")) pair_tf32 = atoi(e) != 0;  // 0: BF16-only CTA pairs
        if (const char* e = cks_knob("CKS_TF32_WIDE")) tf32_wide = atoi(e) != 0;  // wide TF32 pixel blocks
        if (const char* e = cks_knob("CKS_BF16_WIDE")) bf16_wide = atoi(e) != 0;  // the same for BF16
        if (const char* e = cks_knob("CKS_WGRAD_MT128")) wmt128 = atoi(e) != 0;  // BN = 128 row tiles
        if (const char* e = cks_knob("CKS_KS_MP")) ks_mp = atoi(e) != 0;  // multi-phase narrow-output KS-deconv
        if (const char* e = cks_knob("CKS_WGRAD_PP")) wpp = atoi(e) != 0;  // Sk-dilated position pairs
        if (const char* e = cks_knob("CKS_PAIR_WAVES_TF32")) pair_waves_tf32 = atoi(e);  // TF32 pair grid (1/10 waves)
        if (const char* e = cks_knob("CKS_SMEM_CAP")) smem_cap = atoi(e);    // KB of ring budget (experiments)
        if (const char* e = cks_knob("CKS_GZ_MAX")) gz_max = std::max(1, atoi(e));  // G_Z cap (experiments)
        // 0: G_Z partials + KB-REDUCE; 1: in-cluster reduce when the plan's G_Z fits one
        // wave of clusters; 2 (default): also shrink G_Z (to >= 3/4) to a size that fits
        if (const char* e = cks_knob("CKS_WGRAD_ZC")) wzc = atoi(e);
        if (const char* e = cks_knob("CKS_EPI_BUFS")) epi_bufs = atoi(e) == 2 ? 2 : 1;  // TMA-store staging depth
        if (const char* e = cks_knob("CKS_WGRAD_A1")) wa1 = atoi(e) != 0;  // O_C <= 64: one dY atom per stage
        if (const char* e = cks_knob("CKS_WGRAD_MT_TF32")) wmt_tf32 = atoi(e) != 0;  // TF32 row tiles
        if (const char* e = cks_knob("CKS_WGRAD_A1_TF32")) wa1_tf32 = atoi(e) != 0;  // TF32: 64 OC of dY per stage
        if (const char* e = cks_knob("CKS_WGRAD_TC")) wtc = atoi(e);  // filter-row groups (2: multicast clusters)
        if (const char* e = cks_knob("CKS_RG")) rg = atoi(e) != 0;  // 0: batch-as-M tiles at any N
        if (const char* e = cks_knob("CKS_WROW_Q")) wrow_q = atoi(e);  // narrow Sk-dilated: output rows per k-block
        if (const char* e = cks_knob("CKS_ACC1")) acc1 = atoi(e) != 0;  // single TMEM accumulator buffer (experiments)
        if (const char* e = cks_knob("CKS_WMT_LMIN")) wmt_lmin = atoi(e);  // Sk-dilated row tiles: min k-blocks per tap
    }
};
static const Knobs& knobs() {
    static const Knobs k;
    return k;
}
static int g_ov_apos = 0, g_ov_bst = 0;
static bool cfg_override(int& bn, int& pbw, int& z) {
    const Knobs& k = knobs();
    if (!k.ov) return false;
    bn = k.bn, pbw = k.pbw, z = k.z;
    g_ov_apos = k.apos, g_ov_bst = k.bst;
    return true;
}

bool epi_staging() { return knobs().epi != 0; }

static IgemmCfg igemm_cfg_w(int64_t rows_h, const std::vector<int64_t>& wph_cnt, int64_t N, int64_t nout,
                            int64_t kchan, int64_t eb, int64_t max_taps_h, int64_t ntap, int64_t a0_step, int num_sms,
                            int force_pbw, int epi_warps, bool pair = false, int epi_bufs = 1, int force_bn = 0,
                            int min_bn = 0, int rg_ni = 0) {
    IgemmCfg c;
    if (rg_ni > 0) pair = false;  // row groups: one M tile holds the whole batch
    c.pair = pair ? 1 : 0;
    c.epi_bufs = epi_bufs;
    // coalesced-store epilogue staging only where the output rows allow 16 B vectors
    c.epi = (epi_staging() && nout % 4 == 0) ? 1 : 0;
    c.epi_warps = epi_warps;
    int64_t budget = kSmemBudget - (c.epi ? epi_stage_bytes(epi_warps, epi_bufs) + 1024 : 0);  // + 1 KB alignment
    if (knobs().smem_cap > 0) budget = std::min<int64_t>(budget, int64_t(knobs().smem_cap) * 1024);  // experiments
    c.wph_cnt = wph_cnt;
    c.nblk = int((N + 127) / 128);
    if (rg_ni > 0) {
        c.rg_ni = rg_ni;
        c.rg_ph = 128 / rg_ni;
        c.nblk = 1;
    }
    c.BN = nout <= 32 ? 32 : (nout <= 64 ? 64 : 128);
    int ov_bn = 0, ov_pbw = 0, ov_z = 0;
    const bool ov = cfg_override(ov_bn, ov_pbw, ov_z);
    if (ov && ov_bn > 0) c.BN = ov_bn;
    if (force_bn > 0) c.BN = force_bn;
    if (ov && ov_pbw > 0) force_pbw = ov_pbw;
    if (pair) {  // CTA pair: 2 x 128 images, 2 x 128 output channels, one pixel per tile
        c.BN = 128;
        force_pbw = 1;
        c.nblk = int((c.nblk + 1) / 2);
    }
    c.nbs = int((nout + c.BN - 1) / c.BN);
    // K block: the narrowest swizzle row (32 / 64 / 128 B) holding all channels,
    // else 128 B blocks
    const int64_t kbytes = kchan * eb;
    c.KB = kbytes <= 32 ? 32 : (kbytes <= 64 ? 64 : 128);
    if (knobs().kb > 0) c.KB = std::min(c.KB, knobs().kb);
    c.kc_blocks = int((kchan + (c.KB / eb) - 1) / (c.KB / eb));
    c.ntap = int(ntap);
    int64_t maxrow = 1;
    for (auto v : wph_cnt) maxrow = std::max(maxrow, v);
    auto tiles_for = [&](int bn, int pb) {
        int64_t wb = 0;
        for (auto v : wph_cnt) wb += (v + pb - 1) / pb;
        return rows_h * wb * c.nblk * ((nout + bn - 1) / bn);
    };
    // Heuristic (tools/sweep_cfg.sh, tools/sweep_z.sh on B200): the largest pixel
    // block (reuse of B rows and activation columns) that still gives >= 120
    // tiles; if even one pixel per tile leaves < 64 tiles, narrower BN; split-K
    // (Z = 2) only for long K loops (>= 16 row steps) on grids of < 32 tiles.
    int pbw = int(std::min<int64_t>({256 / c.BN, 8, maxrow}));
    while (pbw > 1 && tiles_for(c.BN, pbw) < 120) --pbw;
    if (!pair && tiles_for(c.BN, pbw) < 64 && c.BN == 128 && !(ov && ov_bn > 0) && force_bn == 0) {
        c.BN = 64;
        pbw = 1;
    }
    if (min_bn > 0 && c.BN < min_bn) {  // Stage1-free KS-deconv: whole 128-byte MN atoms of B
        c.BN = min_bn;
        pbw = std::min<int>(pbw, int(std::min<int64_t>(256 / c.BN, 8)));
    }
    c.nbs = int((nout + c.BN * (pair ? 2 : 1) - 1) / (c.BN * (pair ? 2 : 1)));
    if (force_pbw > 0) pbw = std::min<int>(force_pbw, int(std::min<int64_t>(256 / c.BN, 8)));
    // MMA-program capacity (kernels/igemm.cuh kProgSlot: 64 entries per list):
    // the entries of one tile are bounded by prog_entries_bound(); narrow the
    // pixel block until the worst case fits (a wide filter with stride > 1
    // emits one entry per (pixel, tap)).
    while (pbw > 1 && prog_entries_bound(pbw, ntap, a0_step, c.BN) > kProgEntries) --pbw;
    // smem: ring of B rows (ntap x BN x 128 B) and ring of A slots holding all
    // pa activation columns of a row step (one TMA box, one barrier)
    for (; pbw >= 1; --pbw) {
        c.pa = int((pbw - 1) * a0_step + ntap);
        c.stage_bytes = int(ntap * c.BN * c.KB);
        if (2 * (int64_t(c.pa) * 128 * c.KB + c.stage_bytes) <= budget && c.pa <= 256) break;
    }
    if (pbw < 1) pbw = 1;
    // Wide TF32 tiles: TF32 3x3 layers are bound by TMA ingress of the activation
    // columns (ncu, C3 l1: tensor 42 %); a wider pixel block reuses each column for
    // more (pixel, tap) pairs -- the row step then spans two A slots (a 3-deep A ring
    // of half-row-step slots) instead of double-buffering whole row steps.
    // Measured (warm): TF32 C3 l1 fwd / KS-deconv 143 -> 127 us, l2 122 -> 106 us;
    // BF16 l1 81 -> 73 us, l2 64 -> 57 us (C2's small maps keep < 3 waves: unchanged).
    int wide_apos = 0;
    if ((eb == 4 ? knobs().tf32_wide : knobs().bf16_wide) && !pair && force_pbw == 0 && !(ov && ov_pbw > 0)) {
        const int64_t stage = ntap * c.BN * c.KB, colb = int64_t(128) * c.KB;
        for (int pb = pbw + 1; pb <= std::min<int64_t>({int64_t(256 / c.BN), 8, maxrow}); ++pb) {
            // >= 3 waves of tiles (C3 l4, 7x7: 2-pixel tiles leave 1.5 waves and lose 15 %)
            if (tiles_for(c.BN, pb) < 3 * int64_t(num_sms) || prog_entries_bound(pb, ntap, a0_step, c.BN) > kProgEntries)
                break;
            const int64_t pa_ = (pb - 1) * a0_step + ntap, ap = (pa_ + 1) / 2;
            if (2 * stage + 3 * ap * colb > budget) break;
            pbw = pb;
            wide_apos = int(ap);
        }
    }
    c.pbw = pbw;
    c.pa = int((pbw - 1) * a0_step + ntap);
    c.stage_bytes = int(ntap * c.BN * c.KB);
    c.unit_step = a0_step == 1;
    c.a0_step = int(a0_step);
    // A slot: as many of the pa columns as fit with >= 2 A slots and 2 B rows
    c.stages = 2;
    c.apos = c.pa;
    const int64_t col_bytes = 128 * c.KB;  // one activation column, 128 images
    while (c.apos > 1 && 2 * c.stage_bytes + 2 * int64_t(c.apos) * col_bytes > budget) --c.apos;
    if (wide_apos > 0) c.apos = wide_apos;
    if (2 * c.stage_bytes + 2 * int64_t(c.apos) * col_bytes > budget) c.stages = 1;
    if (ov && g_ov_apos > 0) c.apos = std::min(c.pa, g_ov_apos);
    if (ov && g_ov_bst > 0) c.stages = g_ov_bst;
    // row groups: one activation column per A slot (a box of rg_ph rows x rg_ni
    // images is one 128-row K-major tile only for a single column)
    if (c.rg_ni > 0) c.apos = 1;
    c.a_stages = int(std::min<int64_t>(8, (budget - c.stages * c.stage_bytes) / (int64_t(c.apos) * col_bytes)));
    // one A slot per row step: A slot and B row form one stage (one barrier pair,
    // one commit per row step); as many stages as fit
    if (c.apos == c.pa && knobs().unified) {
        const int64_t st = std::min<int64_t>(8, budget / (int64_t(c.apos) * col_bytes + c.stage_bytes));
        if (st >= 2) {
            c.unified = 1;
            c.stages = c.a_stages = int(st);
        }
    }
    c.acc_stages = 2;
    // experiments: one TMEM accumulator buffer for pixel blocks whose two buffers would exceed
    // the 512 TMEM columns (CKS_ACC1 with a forced CKS_IGEMM_CFG pixel block)
    if (knobs().acc1 && int64_t(2) * c.pbw * c.BN * (pair ? 2 : 1) > 512) c.acc_stages = 1;
    c.wblocks = 0;
    for (auto v : wph_cnt) c.wblocks += int((v + c.pbw - 1) / c.pbw);
    c.out_tiles = rows_h * c.wblocks * c.nblk * c.nbs;
    // split-K to fill the SMs (one wave); at least 2 row steps per segment
    const int64_t rs_full = std::max<int64_t>(max_taps_h * c.kc_blocks, 1);
    c.Z = 1;
    c.zc = 0;
    // cluster split-K (zc): Z in {2, 4, 8} CTAs per output tile while the grid
    // stays one wave (out_tiles * Z <= SMs) with >= 2 row steps per segment and
    // >= 8 row steps saved per tile; the
    // tile's fp32 accumulators are staged in the idle rings for the DSMEM reduce
    const int64_t ring = int64_t(c.a_stages) * c.apos * 128 * c.KB + int64_t(c.stages) * c.stage_bytes;
    const bool zc_ok = !pair && knobs().zc && int64_t(128) * c.pbw * c.BN * 4 <= ring;
    if (zc_ok) {
        int z = 8;
        // one wave of resident clusters (8 GPCs x floor(18 / z) clusters, as for KB-WGRAD)
        while (z > 1 && (c.out_tiles * z > num_sms || c.out_tiles * z > int64_t(8) * (18 / z) * z || rs_full < 2 * z))
            z /= 2;
        // the DSMEM reduce costs a few row steps: split only when >= 8 row steps
        // per tile are saved (tools/sweep_zc.sh on the C2 layers)
        if (z > 1 && rs_full * (z - 1) >= 8 * z) {
            c.Z = z;
            c.zc = 1;
        }
    } else if (!pair && c.out_tiles < 32 && rs_full >= 16) {
        c.Z = 2;  // legacy global split-K: only very under-filled grids (sweep: Z = 2 at < 100 tiles was slower)
    }
    if (ov && ov_z > 0 && !pair) {
        c.Z = int(std::min<int64_t>(ov_z, rs_full));
        c.zc = zc_ok && c.Z > 1 && c.Z <= 8 && c.out_tiles * c.Z <= num_sms;
    }
    c.tiles = c.out_tiles * c.Z;
    // A-tile multicast across the BN blocks of one pixel (thread-block cluster):
    // every CTA loads 128/cm of the images of each activation column
    c.cm = 1;
    if (c.Z == 1 && !pair && knobs().mcast) {  // measured slower on B200: off by default
        if (c.nbs % 4 == 0) c.cm = 4;
        else if (c.nbs % 2 == 0) c.cm = 2;
    }
    return c;
}

// 8 epilogue warps (two per TMEM sub-partition, twice the output stores in
// flight) when their 4 KB staging buffers cost no pipeline depth or tile width.
IgemmCfg igemm_cfg(int64_t rows_h, const std::vector<int64_t>& wph_cnt, int64_t N, int64_t nout, int64_t kchan,
                   int64_t eb, int64_t max_taps_h, int64_t ntap, int64_t a0_step, int num_sms, int force_pbw,
                   int force_bn, int rg_ni) {
    if (rg_ni > 0)  // row groups (N <= 64): single-CTA tiles, one wave model as below
        return igemm_cfg_w(rows_h, wph_cnt, N, nout, kchan, eb, max_taps_h, ntap, a0_step, num_sms, force_pbw, 4,
                           false, 1, std::max(force_bn, 0), force_bn < 0 ? -force_bn : 0, rg_ni);
    // Stage1-free KS-deconv: force_bn > 0 fixes the B width (one 128-byte MN atom per tap),
    // force_bn < 0 asks for B widths of whole atoms of -force_bn channels; no CTA pairs
    if (force_bn != 0)
        return igemm_cfg_w(rows_h, wph_cnt, N, nout, kchan, eb, max_taps_h, ntap, a0_step, num_sms, force_pbw, 4,
                           false, 1, std::max(force_bn, 0), force_bn < 0 ? -force_bn : 0);
    // CTA pairs (cta_group::2, M = 256 images x N = 256 channels per MMA): the same
    // smem stage (this CTA's A slot + half the B row) feeds twice the MMA work of a
    // 128 x 128 tile, so the latency-bound 2-stage ring carries twice the math.
    // BF16, >= 256 output channels and >= 2 image blocks, 128 B K blocks, and a
    // pair grid of >= 1 wave; the stage must leave a 2-deep unified ring.
    // Measured (tools/ab.sh, CKS_PAIR): a win where the single-CTA plan is one
    // pixel wide with >= 2 channel blocks (the pair loads each activation column
    // once instead of once per 128-channel block: C3 l3 -9 %) and the pair grid
    // is >= 2.5 waves; a loss against 2-pixel tiles (C4) and on short grids (C3 l4).
    IgemmCfg c4 = igemm_cfg_w(rows_h, wph_cnt, N, nout, kchan, eb, max_taps_h, ntap, a0_step, num_sms,
                              force_pbw, 4);
    if (knobs().epi_bufs == 2 && c4.epi) {  // double-buffered TMA-store staging where it costs no ring depth
        const IgemmCfg c2 = igemm_cfg_w(rows_h, wph_cnt, N, nout, kchan, eb, max_taps_h, ntap, a0_step, num_sms,
                                        force_pbw, 4, false, 2);
        if (c2.pbw == c4.pbw && c2.apos == c4.apos && c2.stages == c4.stages && c2.a_stages == c4.a_stages &&
            c2.unified == c4.unified && c2.BN == c4.BN && c2.Z == c4.Z && c2.zc == c4.zc)
            c4 = c2;
    }
    if (knobs().pair && (eb == 2 || knobs().pair_tf32) && nout >= 256 && N > 128 && kchan * eb >= 128 &&
        force_pbw == 0 && c4.pbw == 1 &&
        c4.nbs >= 2 && c4.Z == 1) {
        const IgemmCfg cp = igemm_cfg_w(rows_h, wph_cnt, N, nout, kchan, eb, max_taps_h, ntap, a0_step, num_sms,
                                        0, 4, true);
        // pair grid of >= 2.5 waves (BF16); TF32 layers are ingress-bound and gain from the pair's
        // halved activation traffic on shorter grids too (knob: tenths of a wave)
        const int64_t waves10 = eb == 4 ? knobs().pair_waves_tf32 : 25;
        if (cp.unified && cp.stages >= 2 && cp.KB == 128 && cp.out_tiles * 2 * 10 >= int64_t(num_sms) * waves10)
            return cp;
    }
    if (knobs().epi8 == 0) return c4;
    const IgemmCfg c8 = igemm_cfg_w(rows_h, wph_cnt, N, nout, kchan, eb, max_taps_h, ntap, a0_step, num_sms,
                                    force_pbw, 8);
    const bool same = c8.pbw == c4.pbw && c8.apos == c4.apos && c8.stages == c4.stages &&
                      c8.a_stages == c4.a_stages && c8.unified == c4.unified && c8.BN == c4.BN && c8.Z == c4.Z &&
                      c8.zc == c4.zc;
    return (same || knobs().epi8 == 2) ? c8 : c4;
}

static int64_t max_window(const std::vector<KRow>& rows) {
    int64_t m = 0;
    for (auto& r : rows) m = std::max(m, r.te - r.ts);
    return m;
}

int rg_images(int64_t N) {
    if (!knobs().rg || N > 64) return 0;
    return N <= 32 ? 32 : 64;
}

std::vector<KRow> igemm_rows_fwd(const cks_geom& g, int rg_ni) {
    auto rh = krows_fwd(axis_h(g));
    return rg_ni > 0 ? group_rows(rh, 128 / rg_ni, g.sh, 1) : rh;
}

std::vector<KRow> igemm_rows_deconv(const cks_geom& g, int rg_ni) {
    auto rh = krows_deconv(axis_h(g));
    return rg_ni > 0 ? group_rows(rh, 128 / rg_ni, 1, g.sh) : rh;
}

int rg_plan(const cks_geom& g, bool deconv) {
    const int ni = rg_images(g.N);
    if (ni == 0 || (!deconv && g.sh > 8)) return 0;  // TMA element strides <= 8
    const auto rows = deconv ? igemm_rows_deconv(g, ni) : igemm_rows_fwd(g, ni);
    for (auto& r : rows)
        if (r.phase > 15) return 0;  // the kernel packs (phase, group length) into one byte
    return run_starts(rows).size() <= 16 ? ni : 0;  // kernels/igemm.cuh kMaxPhases runs
}

static IgemmCfg igemm_cfg_fwd_plan(const cks_geom& g, cks_dtype dt, int num_sms) {
    Axis aw = axis_w(g);
    const int rg = rg_plan(g, false);
    auto rh = igemm_rows_fwd(g, rg);
    IgemmCfg c = igemm_cfg(int64_t(rh.size()), {aw.O}, g.N, g.OC, pad_ch(g.C, dt), elem_bytes(dt), max_window(rh),
                           g.FW, g.sw, num_sms, 0, 0, rg);
    c.rg_es = int(g.sh);
    c.rg_ostep = 1;
    return c;
}

static IgemmCfg igemm_cfg_deconv_plan(const cks_geom& g, cks_dtype dt, int num_sms) {
    Axis aw = axis_w(g);
    const int rg = rg_plan(g, true);
    auto rh = igemm_rows_deconv(g, rg);
    std::vector<int64_t> cnt;
    for (auto& ph : table_t2(aw)) cnt.push_back(ph.U);
    IgemmCfg c = igemm_cfg(int64_t(rh.size()), cnt, g.N, g.C, pad_ch(g.OC, dt), elem_bytes(dt), max_window(rh),
                           cdiv(g.FW, g.sw), 1, num_sms, 0, 0, rg);
    c.rg_es = 1;
    c.rg_ostep = int(g.sh);
    return c;
}

MpPlan mp_plan(const cks_geom& g, cks_dtype dt) {
    MpPlan m;
    if (knobs().ks_mp == 0) return m;
    // stride > 1 (a single phase is the KS path itself), narrow outputs, equal sub-filters
    if (g.sh * g.sw < 2 || g.C > 8 || g.FH % g.sh || g.FW % g.sw || g.sh > 8 || g.sw > 8) return m;
    const int64_t NP = (int64_t(g.sh) * g.sw * g.C + 3) / 4 * 4;  // stacked channels, 16-byte fp32 rows
    if (NP > 64) return m;
    const Axis ah = axis_h(g), aw = axis_w(g);
    const auto th = table_t2(ah), tw = table_t2(aw);
    int64_t amin_h = 0, amax_h = INT64_MIN, amin_w = 0, amax_w = INT64_MIN;
    for (auto& ph : th) {
        if (ph.CH != g.FH / g.sh || ph.U <= 0) return m;  // every phase the full sub-filter, >= 1 row
        amin_h = std::min(amin_h, ph.a);
        amax_h = std::max(amax_h, ph.a + ph.U);
    }
    for (auto& ph : tw) {
        if (ph.CH != g.FW / g.sw || ph.U <= 0) return m;
        amin_w = std::min(amin_w, ph.a);
        amax_w = std::max(amax_w, ph.a + ph.U);
    }
    m.CH = int(g.FH / g.sh);
    m.CW = int(g.FW / g.sw);
    m.ph2 = int(-amin_h);
    m.pw2 = int(-amin_w);
    if (m.ph2 >= m.CH || m.pw2 >= m.CW) return m;  // ConvV2 validity (p < F)
    m.NP = int(NP);
    cks_geom pg;
    pg.N = g.N, pg.C = g.OC, pg.H = ah.O, pg.W = aw.O, pg.OC = NP, pg.FH = m.CH, pg.FW = m.CW;
    pg.sh = 1, pg.sw = 1, pg.ph = m.ph2, pg.pw = m.pw2, pg.dh = 1, pg.dw = 1;
    if (validate(&pg) != CKS_OK) return m;
    // the pseudo output must reach every phase row / column: o = u + a + p' < O'
    if (amax_h - 1 + m.ph2 >= out_extent(pg.H, pg.FH, 1, pg.ph) || amax_w - 1 + m.pw2 >= out_extent(pg.W, pg.FW, 1, pg.pw))
        return m;
    for (auto& ph : th) m.ih_s[ph.y] = int16_t(ph.ih_s), m.a_y[ph.y] = int16_t(ph.a);
    for (auto& ph : tw) m.iw_s[ph.y] = int16_t(ph.ih_s), m.a_x[ph.y] = int16_t(ph.a);
    m.pg = pg;
    m.ok = true;
    (void)dt;
    return m;
}

bool ks_direct_eligible(const cks_geom& g, cks_dtype dt) {
    const int64_t eb = elem_bytes(dt);
    return (g.C * eb) % 16 == 0 && g.sw <= 8 && g.sh <= 16 && cdiv(g.FW, g.sw) * g.sw <= 256 && g.FH <= 32767;
}

static IgemmCfg igemm_cfg_deconv_w_plan(const cks_geom& g, cks_dtype dt, int num_sms) {
    Axis aw = axis_w(g);
    const int rg = rg_plan(g, true);
    auto rh = igemm_rows_deconv(g, rg);
    std::vector<int64_t> cnt;
    for (auto& ph : table_t2(aw)) cnt.push_back(ph.U);
    const int atomw = int(128 / elem_bytes(dt));  // channels of one 128-byte MN atom
    // several atoms per tap need the IC axis split exactly into atoms (5-D map)
    const int fb = g.C % atomw == 0 ? -atomw : atomw;
    IgemmCfg c = igemm_cfg(int64_t(rh.size()), cnt, g.N, g.C, pad_ch(g.OC, dt), elem_bytes(dt), max_window(rh),
                           cdiv(g.FW, g.sw), 1, num_sms, 0, fb, rg);
    c.rg_es = 1;
    c.rg_ostep = int(g.sh);
    return c;
}

// Policy: Stage1-free where eligible and the W-direct plan keeps the packed
// plan's tile (same BN, no CTA pairs): a narrower W-direct tile re-reads dY
// more often (measured: TF32 C3 with BN forced to 32 was up to 1.4x slower)
// (CKS_KS_DIRECT=0/1 forces it off / on where eligible; experiments build).
bool ks_direct(const cks_geom& g, cks_dtype dt, int num_sms) {
    if (!ks_direct_eligible(g, dt)) return false;
    if (const char* e = cks_knob("CKS_KS_DIRECT")) return atoi(e) != 0;
    const IgemmCfg c = igemm_cfg_deconv(g, dt, num_sms);
    const IgemmCfg d = igemm_cfg_deconv_w(g, dt, num_sms);
    return !c.pair && d.BN == c.BN;
}

// ---------------------------------------------------------------- narrow-channel row path
// Column classes (kernels/narrow.cuh): the (fw, c) run of output column ow
// starts at element start = (ow*sw - pw)*C of the flattened X row; TMA box
// origins must be 16-byte aligned.  Interior columns (whole window inside X)
// are grouped by delta = start mod (16 / eb) -- period P = (16/eb) / gcd(sw*C,
// 16/eb) in ow -- and load from start - delta; every border column is a class
// of its own: a left-border one loads from element 0 (its first valid
// element), a right-border one ends its chunks at (origin chosen so the 32-byte K-chunk grid ends exactly at the
// last element of X).  kc0 / kc1: the 32-byte K chunks of the box row that
// hold valid run elements.
static bool row_classes(const cks_geom& g, cks_dtype dt, std::vector<RowClassH>& cls, int& emax) {
    const int64_t eb = elem_bytes(dt), align = 16 / eb, ke = 32 / eb;
    const int64_t jn = g.FW * g.C, rowlen = g.W * g.C;
    const int64_t OW = out_extent(g.W, g.FW, g.sw, g.pw);
    int64_t q = (int64_t(g.sw) * g.C) % align, a = align;
    while (q) { int64_t t = a % q; a = q; q = t; }  // gcd(sw*C, align)
    const int64_t P = align / a;
    cls.clear();
    emax = 0;
    std::vector<int64_t> interior;
    for (int64_t ow = 0; ow < OW; ++ow) {
        const int64_t start = (ow * g.sw - g.pw) * g.C;
        const int64_t jlo = std::max<int64_t>(0, -start), jhi = std::min<int64_t>(jn, rowlen - start);
        if (jlo == 0 && jhi == jn) { interior.push_back(ow); continue; }
        RowClassH c;
        c.col0 = int(ow), c.cstep = 1, c.ncols = 1;
        // left border: origin 0 (the first valid element starts chunk 0); right border:
        // the chunk grid ends exactly at the row end, origin = rowlen - ke*ceil((rowlen - start)/ke)
        // (16-byte aligned: rowlen*eb and ke*eb = 32 are), so no issued K chunk reaches past X
        c.off = int(start < 0 ? -start : rowlen - ke * cdiv(rowlen - start, ke) - start);
        c.kc0 = int((jlo - c.off) / ke);
        c.kc1 = int(cdiv(jhi - c.off, ke));
        emax = std::max(emax, int(jhi - c.off));
        cls.push_back(c);
    }
    if (!interior.empty()) {  // interior columns are contiguous; residues mod P
        const int64_t lo = interior.front(), hi = interior.back() + 1;
        for (int64_t r = 0; r < P && lo + r < hi; ++r) {
            RowClassH c;
            c.col0 = int(lo + r), c.cstep = int(P), c.ncols = int(cdiv(hi - lo - r, P));
            const int64_t delta = fmod_pos((c.col0 * g.sw - g.pw) * g.C, align);
            c.off = int(-delta);
            c.kc0 = int(delta / ke);
            c.kc1 = int(cdiv(delta + jn, ke));
            emax = std::max(emax, int(delta + jn));
            cls.push_back(c);
        }
    }
    std::sort(cls.begin(), cls.end(), [](const RowClassH& x, const RowClassH& y) { return x.col0 < y.col0; });
    return int(cls.size()) <= kRowClasses;
}

static bool row_setup(const cks_geom& g, cks_dtype dt, RowCfg& c) {
    const int64_t eb = elem_bytes(dt);
    if (g.C > (dt == CKS_BF16 ? 16 : 8)) return false;
    if ((g.W * g.C * eb) % 16 != 0) return false;  // TMA row pitch
    if (g.W * g.C > (int64_t(1) << 31) / eb) return false;
    int emax = 0;
    if (!row_classes(g, dt, c.cls, emax)) return false;
    c.ROWB = emax * eb <= 32 ? 32 : (emax * eb <= 64 ? 64 : (emax * eb <= 128 ? 128 : 0));
    c.JB = int(c.ROWB / eb);
    return c.ROWB != 0;
}

// Spread `total` workers over the classes (>= 1 each, at most `cap(c)` each),
// minimising the largest work / workers.
static void row_spread(std::vector<RowClassH>& cls, int64_t total, const std::vector<int64_t>& cap) {
    for (size_t k = 0; k < cls.size(); ++k) cls[k].cnt = 1;
    int64_t used = int64_t(cls.size());
    while (used < total) {
        int best = -1;
        double bw = 0;
        for (size_t k = 0; k < cls.size(); ++k) {
            if (cls[k].cnt >= cap[k]) continue;
            const double w = double(cls[k].work) / cls[k].cnt;
            if (w > bw) { bw = w; best = int(k); }
        }
        if (best < 0) break;
        ++cls[best].cnt;
        ++used;
    }
    int base = 0;
    for (auto& k : cls) { k.base = base; base += k.cnt; }
}

// Narrow ConvV2: tile = R output rows x one column x 128 images x all OC,
// the class's filter rows resident in shared memory.
static RowCfg row_cfg_fwd_plan(const cks_geom& g, cks_dtype dt, bool allow_rg) {
    RowCfg c;
    if (!row_setup(g, dt, c) || g.OC > (dt == CKS_TF32 ? 128 : 256)) return c;  // instantiated BN range
    c.BN = 32;
    while (c.BN < g.OC) c.BN *= 2;
    const int wbytes = int((g.FH * c.BN * c.ROWB + 1023) / 1024 * 1024);
    const int stage = 128 * c.ROWB;
    const int staging = 4 * CKS_ROW_EPI_BUFS * 4096;  // kernels/narrow.cuh RowFwdShape::STAGING
    const int budget = 227 * 1024 - 1024 - 512;
    c.stages = std::min(16, (budget - wbytes - staging) / stage);
    if (c.stages < 3) return c;
    c.smem = 1024 + wbytes + c.stages * stage + staging + 512;
    c.nblk = int((g.N + 127) / 128);
    // row groups (small batches): an M tile is rg_pc columns of one class x rg images, each
    // column group one TMA box of a per-class tensor map (column stride cstep * sw * C)
    if (allow_rg && rg_images(g.N) > 0) {
        c.rg = rg_images(g.N);
        c.rg_pc = 128 / c.rg;
        c.nblk = 1;
    }
    const int64_t OH = out_extent(g.H, g.FH, g.sh, g.ph);
    auto col_units = [&](const RowClassH& k) { return c.rg ? (k.ncols + c.rg_pc - 1) / c.rg_pc : k.ncols; };
    // output rows per tile: X rows are loaded once per tile (h reuse), as many as
    // TMEM holds while the grid keeps >= 2 tiles per SM
    const int rmax = std::min(8, 256 / c.BN);
    auto tiles_for = [&](int r) {
        int64_t t = 0;
        for (auto& k : c.cls) t += cdiv(OH, r) * col_units(k) * c.nblk;
        return t;
    };
    c.R = 1;
    for (int r = rmax; r >= 1; --r)
        if (r == 1 || (r <= OH && tiles_for(r) >= 2 * 148)) { c.R = r; break; }
    c.tiles = tiles_for(c.R);
    std::vector<int64_t> cap;
    for (auto& k : c.cls) {
        k.work = cdiv(OH, c.R) * col_units(k) * c.nblk;
        cap.push_back(k.work);
    }
    row_spread(c.cls, std::max<int64_t>(int64_t(c.cls.size()), 148), cap);
    c.grid = 0;
    for (auto& k : c.cls) c.grid += k.cnt;
    c.ok = true;
    return c;
}

int64_t row_fwd_padding_macs(const cks_geom& g, cks_dtype dt) {
    const RowCfg c = row_cfg_fwd(g, dt);
    if (!c.ok) return -1;
    const int64_t ke = 32 / elem_bytes(dt), jn = g.FW * g.C, rowlen = g.W * g.C;
    int64_t n = 0;
    for (auto& k : c.cls)
        for (int i = 0; i < k.ncols; ++i) {
            const int64_t start = (int64_t(k.col0 + k.cstep * i) * g.sw - g.pw) * g.C;
            // box elements [kc0*ke, kc1*ke) <-> run j = off + e; padding: j in the window range but X outside
            for (int64_t e = k.kc0 * ke; e < k.kc1 * ke; ++e) {
                const int64_t j = k.off + e, x = start + j;
                if (j >= 0 && j < jn && (x < 0 || x >= rowlen)) ++n;
            }
        }
    const int64_t OH = out_extent(g.H, g.FH, g.sh, g.ph);
    int64_t vh = 0;
    for (int64_t oh = 0; oh < OH; ++oh) {
        const int64_t ih0 = oh * g.sh - g.ph;
        vh += std::min(g.H - ih0, g.FH) - std::max<int64_t>(-ih0, 0);
    }
    return n * vh * g.OC;  // per image; every valid filter row of every output row
}

int64_t row_wgrad_padding_macs(const cks_geom& g, cks_dtype dt) {
    const RowCfg c = row_cfg_wgrad(g, dt, 0, 148);
    if (!c.ok) return -1;
    const int64_t jn = g.FW * g.C, rowlen = g.W * g.C, R = 128 / c.JB;
    const int64_t OH = out_extent(g.H, g.FH, g.sh, g.ph);
    int64_t n = 0;
    for (auto& k : c.cls)
        for (int i = 0; i < k.ncols; ++i) {
            const int64_t start = (int64_t(k.col0 + k.cstep * i) * g.sw - g.pw) * g.C;
            for (int64_t oh = 0; oh < OH; ++oh) {
                const int64_t ih0 = oh * g.sh - g.ph;
                const int64_t fs = std::max<int64_t>(-ih0, 0), fe = std::min(g.H - ih0, g.FH);
                for (int64_t m = 0; m < c.mb; ++m) {
                    if (!(m * R < fe && (m + 1) * R > fs)) continue;  // M-block not issued
                    for (int64_t fh = m * R; fh < std::min<int64_t>((m + 1) * R, g.FH); ++fh)
                        for (int64_t e = 0; e < c.JB; ++e) {
                            const int64_t j = k.off + e, x = start + j;
                            if (j < 0 || j >= jn) continue;  // not a stored dW row
                            if (fh < fs || fh >= fe || x < 0 || x >= rowlen) ++n;
                        }
                }
            }
        }
    return n * g.OC;  // per image
}

// Narrow Sk-dilated: M = (fh, e) rows, 128/JB filter rows per M-block; N = OC
// block; K = (oh, column, 64 images) of one column class, split into
// segments; every segment of every class is one G_Z map-reduce partial.
static RowCfg row_cfg_wgrad_plan(const cks_geom& g, cks_dtype dt, int gz_req, int num_sms, bool allow_rg) {
    RowCfg c;
    if (!row_setup(g, dt, c)) return c;
    if (dt == CKS_TF32) {  // MN-major tf32 needs the 128-byte (BASE32B) swizzle
        c.ROWB = 128;
        c.JB = 32;
    }
    const int64_t eb = elem_bytes(dt);
    const int R = 128 / c.JB;
    c.mb = int((g.FH + R - 1) / R);
    if (c.mb > 4) return c;
    const int cap = 256 / c.mb;  // TMEM: mb accumulators of BN columns
    c.BN = 64;
    while (c.BN < pad_ch(g.OC, dt) && c.BN * 2 <= cap) c.BN *= 2;
    if (c.BN > cap) return c;
    c.nbs = int((pad_ch(g.OC, dt) + c.BN - 1) / c.BN);
    c.nblk = int((g.N + 63) / 64);
    // row groups (N <= 32): a 64-row k-block = rg_pc class columns x rg images (per-class maps,
    // kernels/narrow.cuh RowWXMaps: at most kRowWgradRgClasses = 12 classes)
    if (allow_rg && knobs().rg && 2 * g.N <= 64 && c.cls.size() <= 12) {
        c.rg = g.N <= 16 ? 16 : 32;
        c.rg_pc = 64 / c.rg;
        c.nblk = 1;
    }
    auto col_units = [&](const RowClassH& k) -> int64_t { return c.rg ? (k.ncols + c.rg_pc - 1) / c.rg_pc : k.ncols; };
    const int64_t OH = out_extent(g.H, g.FH, g.sh, g.ph);
    // Output rows per k-block q: one X box of FH + sh*(q-1) rows serves q output rows.  Measured
    // (tools/time_op.py, CKS_WROW_Q): ResNet stem TF32 407 -> 329 us (q = 2), BF16 252 -> 206 (2)
    // -> 190 us (3); DCGAN G32to64 BF16 45 -> 38 us; small maps lose parallelism (C2 vgg32 s2:
    // 12 -> 15 us).  Policy: q = 2 where it saves >= 20 % of the X rows per output row and
    // leaves >= 4 k-blocks per SM; q = 3 only with >= 16 k-blocks per SM; always a >= 2-deep ring.
    {
        const int64_t atom = int64_t(64) * c.ROWB;
        const int64_t ow_cols = out_extent(g.W, g.FW, g.sw, g.pw);
        const int qmax = knobs().wrow_q > 0 ? knobs().wrow_q : 3;
        for (int q = qmax; q >= 1; --q) {
            if (q == 1) {
                c.q = 1;
                break;
            }
            const int64_t stage = ((q - 1) * g.sh + int64_t(c.mb) * R) * atom + int64_t(q) * c.BN * 64 * eb;
            const int64_t kblocks = ((OH + q - 1) / q) * (c.rg ? (ow_cols + c.rg_pc - 1) / c.rg_pc : ow_cols) * c.nblk;
            const bool forced = knobs().wrow_q > 0;
            const bool saves = 5 * (g.FH + g.sh * (q - 1)) <= 4 * q * g.FH;  // <= 80 % of the rows
            const bool enough = kblocks >= int64_t(q == 2 ? 4 : 16) * num_sms;
            if ((227 * 1024 - 2048) / stage >= 2 && (q - 1) * g.sh + g.FH <= 256 && (forced || (saves && enough))) {
                c.q = q;
                break;
            }
        }
    }
    std::vector<int64_t> segcap;
    for (auto& k : c.cls) {
        k.work = ((OH + c.q - 1) / c.q) * col_units(k) * c.nblk;
        segcap.push_back(gz_req > 0 ? k.work : std::max<int64_t>(1, k.work / 8));  // >= 8 k-blocks per segment
    }
    const int64_t want = gz_req > 0 ? gz_req : std::max<int64_t>(1, num_sms / c.nbs);
    row_spread(c.cls, std::max<int64_t>(want, int64_t(c.cls.size())), segcap);
    c.gz = 0;
    for (auto& k : c.cls) c.gz += k.cnt;
    const int stage = int(((c.q - 1) * g.sh + c.mb * R) * 64 * c.ROWB + c.q * c.BN * 64 * eb);
    c.stages = std::min(8, (227 * 1024 - 2048) / stage);
    if (c.stages < 2) return c;
    c.smem = 1024 + c.stages * stage + 256;
    c.tiles = int64_t(c.nbs) * c.gz;
    c.grid = int(std::min<int64_t>(c.tiles, num_sms));
    c.ok = true;
    return c;
}

static std::string row_classes_str(const std::vector<RowClassH>& cls) {
    std::string o;
    char b[96];
    for (size_t k = 0; k < cls.size(); ++k) {
        snprintf(b, sizeof b, "%s%d:%d:%d:%d:%d:%d:%d:%d", k ? "," : "", cls[k].col0, cls[k].cstep, cls[k].ncols,
                 cls[k].off, cls[k].kc0, cls[k].kc1, cls[k].base, cls[k].cnt);
        o += b;
    }
    return o;
}

std::string describe_plan(const cks_geom& g, cks_dtype dt, cks_op op, int gz, int num_sms) {
    char b[512];
    if (op == CKS_OP_FWD || op == CKS_OP_DECONV) {
        if (op == CKS_OP_FWD) {
            const RowCfg r = row_cfg_fwd(g, dt);
            if (r.ok) {
                snprintf(b, sizeof b, "row_fwd ROWB=%d JB=%d BN=%d R=%d stages=%d grid=%d tiles=%lld rg=%d classes=%d cls=",
                         r.ROWB, r.JB, r.BN, r.R, r.stages, r.grid, (long long)r.tiles, r.rg, int(r.cls.size()));
                return std::string(b) + row_classes_str(r.cls);
            }
        }
        const bool direct = op == CKS_OP_DECONV && ks_direct(g, dt, num_sms);
        const IgemmCfg c = op == CKS_OP_FWD ? igemm_cfg_fwd(g, dt, num_sms)
                                            : (direct ? igemm_cfg_deconv_w(g, dt, num_sms) : igemm_cfg_deconv(g, dt, num_sms));
        snprintf(b, sizeof b,
                 "igemm BN=%d pbw=%d KB=%d ntap=%d pa=%d apos=%d stages=%d a_stages=%d unified=%d out_tiles=%lld "
                 "Z=%d zc=%d kc=%d epi_warps=%d pair=%d ks_direct=%d ks_mp=%d rg=%d",
                 c.BN, c.pbw, c.KB, c.ntap, c.pa, c.apos, c.stages, c.a_stages, c.unified, (long long)c.out_tiles, c.Z,
                 c.zc, c.kc_blocks, c.epi_warps, c.pair, direct ? 1 : 0,
                 op == CKS_OP_DECONV && mp_plan(g, dt).ok ? 1 : 0, c.rg_ni);
        return b;
    }
    const WgradCfg w = wgrad_cfg(g, dt, gz, num_sms);
    if (w.row) {
        const RowCfg r = row_cfg_wgrad(g, dt, gz, num_sms);
        snprintf(b, sizeof b,
                 "row_wgrad ROWB=%d JB=%d BN=%d mb=%d nbs=%d gz=%d stages=%d q=%d tiles=%lld rg=%d classes=%d cls=",
                 r.ROWB, r.JB, r.BN, r.mb, r.nbs, r.gz, r.stages, r.q, (long long)r.tiles, r.rg, int(r.cls.size()));
        return std::string(b) + row_classes_str(r.cls);
    }
    snprintf(b, sizeof b,
             "wgrad BN=%d nbs=%d mblocks=%d kimg=%d mt=%d gz=%d zc=%d a1=%d tc=%d pp=%d base_tiles=%lld rg=%d rg_pk=%d",
             w.BN, w.nbs, w.mblocks, w.kimg, w.mt, w.gz, w.zc, w.a1, w.tc, w.pp, (long long)w.base_tiles, w.rg,
             w.rg_pk);
    return b;
}

// G_Z choice: the paper makes G_Z grow with (N_a + N_b)/N_g and
// bounds it above by the SM count.  Here: enough segments that the
// taps x OC-blocks x IC-blocks x G_Z tiles cover the 148 SMs about once,
// with at least 4 K-blocks (256 images*positions) per segment.
// ad: the depth axis of a 3-D Sk-dilated (per-tap kernel only; every tap's K
// range is the product of its trimmed d, h and w ranges)
static WgradCfg wgrad_cfg_plan(const cks_geom& g, cks_dtype dt, int gz_req, int num_sms, const Axis* ad = nullptr) {
    WgradCfg c;
    RowCfg rc = ad ? RowCfg() : row_cfg_wgrad(g, dt, gz_req, num_sms);
    if (rc.ok) {
        c.row = true;
        c.BN = rc.BN;
        c.nbs = rc.nbs;
        c.mblocks = rc.mb;
        c.nblk64 = rc.nblk;
        c.gz = rc.gz;
        c.base_tiles = rc.nbs;
        return c;
    }
    c.mblocks = int((g.OC + 127) / 128);
    c.BN = g.C <= 64 ? 64 : (g.C <= 128 ? 128 : 256);
    c.nbs = int((g.C + c.BN - 1) / c.BN);
    // 128-image k-blocks (half the barrier round trips) where the stage stays
    // small enough for a 4-deep ring (BN = 64); measured slower for BN >= 128
    c.kimg = (g.N >= 128 && c.BN == 64 && knobs().kimg128) ? 128 : 64;
    c.nblk64 = int((g.N + c.kimg - 1) / c.kimg);
    // row tiles (all F_W = 3 taps of a filter row per tile, the dY block shared):
    // bf16, IC <= 64 (three double-buffered 64-column accumulators fit TMEM)
    // TF32 row tiles keep 64-image k-blocks (3 x 16 KB X blocks + 2 dY atoms per stage)
    // BN = 128 row tiles (I_C <= 128): one TMEM accumulator buffer (3 x 128 columns)
    c.mt = ((c.BN == 64 || (c.BN == 128 && knobs().wmt128)) && g.FW == 3 && knobs().wmt &&
            (dt == CKS_BF16 || knobs().wmt_tf32)) ? 3 : 1;
    Axis ah = axis_h(g), aw = axis_w(g);
    auto th = table_t3(ah), tw = table_t3(aw);
    int64_t dmul = 1;  // 3-D: taps x depth windows (the smallest depth window for lmin)
    if (ad) {
        int64_t dmin = INT64_MAX;
        for (auto& d : table_t3(*ad))
            if (d.oh_e > d.oh_s) dmin = std::min(dmin, d.oh_e - d.oh_s);
        dmul = dmin == INT64_MAX ? 0 : dmin;
    }
    int64_t uws = INT64_MAX, uwe = INT64_MIN;
    for (auto& b : tw)
        if (b.oh_e > b.oh_s) { uws = std::min(uws, b.oh_s); uwe = std::max(uwe, b.oh_e); }
    // k-blocks of the shortest tap (segment sizing): positions (row groups: chunks of
    // rg_pk positions) x image blocks
    auto kbw = [&](int64_t wn) { return c.rg ? (wn + c.rg_pk - 1) / c.rg_pk : wn; };
    int64_t lmin = INT64_MAX, ntaps = 0;
    auto compute_lmin = [&] {
        lmin = INT64_MAX;
        ntaps = 0;
        for (auto& a : th) {
            if (c.mt > 1) {
                int64_t L = dmul * (a.oh_e - a.oh_s) * kbw(std::max<int64_t>(uwe - uws, 0)) * c.nblk64;
                if (L > 0) { lmin = std::min(lmin, L); ++ntaps; }
                continue;
            }
            for (auto& b : tw) {
                int64_t L = dmul * (a.oh_e - a.oh_s) * kbw(b.oh_e - b.oh_s) * c.nblk64;
                if (L > 0) { lmin = std::min(lmin, L); ++ntaps; }
            }
        }
        if (ntaps == 0) lmin = 1;
    };
    compute_lmin();
    // small maps: row tiles cost parallelism (C2 sweep slower); one tap per tile.  Measured
    // (tools/time_op.py, CKS_WMT_LMIN): 64-channel row tiles win from ~1e5 (positions x images)
    // per filter row up (C2 vgg32 64->64 s1: TF32 74 -> 39 us, BF16 51 -> 29 us; C5 l2a TF32
    // 104 -> 88 us) and lose on smaller maps (vgg16 64->128 s2: +44-68 %); 128-channel row tiles
    // (one accumulator buffer) keep the former rule (>= 2048 k-blocks)
    const bool small = knobs().wmt_lmin >= 0 ? lmin < knobs().wmt_lmin
                                             : (c.BN == 64 ? lmin * c.kimg < 100000 : lmin < 2048);
    if (c.mt > 1 && small) {
        c.mt = 1;
        compute_lmin();
    }
    if (dt == CKS_TF32 && c.mt > 1) {  // TF32 row tiles: 64-image (BN = 128: 32-image) k-blocks
        const int k = c.BN == 128 ? 32 : 64;
        lmin = lmin * c.kimg / k;
        c.kimg = k;
        c.nblk64 = int((g.N + k - 1) / k);
    }
    // Row groups (position chunks) for small batches: a k-block of kimg K rows holds
    // rg_pk consecutive output positions x rg = kimg / rg_pk images (position-major), so
    // N <= kimg / 2 images do not leave half the k-block as TMA zero fill.  2-D only
    // (the depth axis keeps image blocks), column stride <= 8 (TMA element stride of
    // the X box).
    if (!ad && knobs().rg && g.sw <= 8 && 2 * g.N <= c.kimg) {
        c.rg = g.N <= 16 ? 16 : 32;
        c.rg_pk = c.kimg / c.rg;
        c.nblk64 = 1;
        compute_lmin();
    }
    c.base_tiles = (ad ? ad->F : 1) * int64_t(g.FH) * (c.mt > 1 ? 1 : g.FW) * c.mblocks * c.nbs;
    if (gz_req > 0) {
        c.gz = gz_req;
    } else {
        int64_t want = std::max<int64_t>(1, num_sms / std::max<int64_t>(c.base_tiles, 1));  // one wave
        int64_t cap = std::max<int64_t>(lmin / 4, 1);
        c.gz = int(std::max<int64_t>(1, std::min<int64_t>({want, cap, int64_t(knobs().gz_max)})));
    }
    // cluster reduce (zc): gz <= 8 segments of a tile as one thread-block cluster,
    // one tile per CTA (one wave), the tile's fp32 sums staged in the idle ring
    // (same stage arithmetic as WgradShape) -- no partials in HBM, no KB-REDUCE launch
    c.a1 = (c.BN == 64 && g.OC <= 64 && knobs().wa1 && (dt == CKS_BF16 || knobs().wa1_tf32)) ? 1 : 0;
    {
        const int eb = dt == CKS_TF32 ? 4 : 2, ch = 128 / eb;
        const int64_t atom = int64_t(c.kimg) * 128;
        const int64_t stage = (c.a1 ? 64 / ch : 128 / ch) * atom + int64_t(c.mt) * (c.BN / ch) * atom;
        const int64_t stages = std::min<int64_t>(8, 200 * 1024 / stage);
        const bool fits = int64_t(128) * c.mt * c.BN * 4 <= stages * stage;
        // every cluster must be resident at once (one tile per CTA): B200 GPCs hold
        // 9 pairs but only 4 clusters of 4 / 2 of 8 (measured: 144 CTAs in clusters
        // of 4 or 8 run in two waves and lose; 72 in clusters of 4 and 144 in pairs win)
        // residency model: 8 GPCs of >= 18 SMs hold floor(18 / gz) clusters each
        auto one_wave = [&](int z) {
            const int64_t t = c.base_tiles * z;
            return t <= num_sms && t <= int64_t(8) * (18 / z) * z;
        };
        c.zc = 0;
        if (knobs().wzc && fits && c.gz >= 2) {
            // the library's own G_Z may shrink (to >= 3/4 of it: measured, halving G_Z
            // costs more parallelism than the reduce saves) to the largest cluster
            // size that fits one wave; a requested gz is taken as is
            int z = std::min(c.gz, 8);
            if (gz_req == 0 && knobs().wzc == 2)
                while (z > 2 && !one_wave(z)) --z;
            // short segments (<= 150 k-blocks each at the halved G_Z) may halve it: in the
            // training-step schedule the freed SMs serve the concurrent KS-deconv chain
            // (C2: step 0.593 -> 0.578 ms); long ones keep >= 3/4 (C3 l2 halved: 71 -> 117 us)
            const bool short_seg = lmin / std::max(z, 1) <= 150;
            const bool ok = knobs().wzc == 2 && gz_req == 0 ? (short_seg ? 2 * z >= c.gz : 4 * z >= 3 * c.gz)
                                                            : z == c.gz;
            if (z >= 2 && z <= 8 && one_wave(z) && ok) {
                c.gz = z;
                c.zc = 1;
            }
        }
    }
    // filter-row clusters (row tiles, no in-cluster G_Z reduce): the F_H row tiles of a segment share
    // each dY block by multicast and walk the union of their oh ranges in lockstep
    // (CKS_WGRAD_TC: 0 off, 1 aligned groups, 2 aligned groups as multicast clusters)
    if (knobs().wtc && c.mt > 1 && !c.zc && g.FH >= 2 && g.FH <= 8) {
        c.tc = int(g.FH);
        c.tcmc = knobs().wtc == 2 ? 1 : 0;
    }
    // position pairs: O_C <= 64 row tiles with unit column stride and an even union ow range
    if (knobs().wpp && !c.rg && c.mt == 3 && c.a1 && c.BN == 64 && g.sw == 1 && !c.zc && !c.tcmc && uwe > uws &&
        (uwe - uws) % 2 == 0) {
        c.pp = 1;
        if (c.kimg == 128) {  // 64-image k-blocks: 48 / 96 KB stages (bf16 / tf32), a deeper ring
            c.kimg = 64;
            c.nblk64 = int((g.N + 63) / 64);
        }
    }
    return c;
}

size_t ks_split_bytes(const cks_geom& g, cks_dtype dt) {
    int64_t chm = cdiv(g.FH, g.sh), cwm = cdiv(g.FW, g.sw);
    return size_t(g.sh) * g.sw * g.C * chm * cwm * pad_ch(g.OC, dt) * elem_bytes(dt);
}

static size_t align256(size_t x) { return (x + 255) / 256 * 256; }

static WsLayout ws_layout_plan(const cks_geom& g, cks_dtype dt, cks_op op, int gz, bool c_packed_given, int num_sms) {
    WsLayout L;
    const int64_t eb = elem_bytes(dt);
    const int64_t Cp = pad_ch(g.C, dt), OCp = pad_ch(g.OC, dt);
    const int64_t OH = out_extent(g.H, g.FH, g.sh, g.ph), OW = out_extent(g.W, g.FW, g.sw, g.pw);
    size_t off = 0;
    auto take = [&](size_t bytes, size_t& at, size_t& sz) {
        if (!bytes) return;
        at = off;
        sz = bytes;
        off += align256(bytes);
    };
    const bool row = (op == CKS_OP_FWD && row_cfg_fwd(g, dt).ok) ||
                     (op == CKS_OP_WGRAD && wgrad_cfg(g, dt, gz, num_sms).row);
    if ((op == CKS_OP_FWD || op == CKS_OP_WGRAD) && !row) {  // the row path reads X unpadded
        if (Cp != g.C) take(size_t(g.N) * g.H * g.W * Cp * eb, L.x_pad, L.x_pad_bytes);
    }
    if (op == CKS_OP_FWD && !row) {
        if (Cp != g.C) take(size_t(g.OC) * g.FH * g.FW * Cp * eb, L.w_pad, L.w_pad_bytes);
    }
    if (op == CKS_OP_DECONV || op == CKS_OP_WGRAD) {
        if (OCp != g.OC) take(size_t(g.N) * OH * OW * OCp * eb, L.dy_pad, L.dy_pad_bytes);
    }
    // W given: room for Stage1's packed sub-filters whichever KS-deconv variant runs
    // (cks_deconv2d_ex may force the Stage1 path); split-K scratch for both plans
    if (op == CKS_OP_DECONV && !c_packed_given) take(ks_split_bytes(g, dt), L.c_packed, L.c_packed_bytes);
    if (op == CKS_OP_DECONV && !c_packed_given) {  // multi-phase KS-deconv (narrow outputs)
        const MpPlan m = mp_plan(g, dt);
        if (m.ok) {
            const int64_t OHp = out_extent(m.pg.H, m.pg.FH, 1, m.pg.ph), OWp = out_extent(m.pg.W, m.pg.FW, 1, m.pg.pw);
            take(size_t(m.NP) * m.CH * m.CW * pad_ch(g.OC, dt) * eb, L.mp_w, L.mp_w_bytes);
            take(size_t(g.N) * OHp * OWp * m.NP * 4, L.mp_y, L.mp_y_bytes);
            take(ws_layout(m.pg, dt, CKS_OP_FWD, 0, false, num_sms).total, L.mp_inner, L.mp_inner_bytes);
        }
    }
    if ((op == CKS_OP_FWD && !row) || op == CKS_OP_DECONV) {
        std::vector<IgemmCfg> cs;
        if (op == CKS_OP_FWD) cs.push_back(igemm_cfg_fwd(g, dt, num_sms));
        else cs.push_back(igemm_cfg_deconv(g, dt, num_sms));
        if (op == CKS_OP_DECONV && !c_packed_given && ks_direct_eligible(g, dt)) cs.push_back(igemm_cfg_deconv_w(g, dt, num_sms));
        size_t part = 0, sem = 0;
        for (const IgemmCfg& c : cs)
            if (c.Z > 1 && !c.zc) {
                part = std::max(part, size_t(c.out_tiles) * c.Z * 128 * c.pbw * c.BN * 4);
                sem = std::max(sem, size_t(c.out_tiles) * 4);
            }
        take(part, L.partial, L.partial_bytes);
        take(sem, L.sem, L.sem_bytes);
    }
    if (op == CKS_OP_WGRAD) {
        WgradCfg c = wgrad_cfg(g, dt, gz, num_sms);
        if (c.npart() > 1 && !c.zc) take(size_t(c.npart()) * g.OC * g.FH * g.FW * g.C * 4, L.partial, L.partial_bytes);
    }
    L.total = off;
    return L;
}

}  // namespace cks

// ---------------------------------------------------------------- plan cache
// The paper pre-computes its index tables once; here every plan
// decision (tile configuration, G_Z, workspace layout) is computed once per
// (geometry, dtype, op, G_Z request, SM count) and served from a thread-safe
// cache afterwards, so a training loop's repeated calls skip the planning.
namespace cks {
namespace {
std::string plan_key(const cks_geom& g, int a, int b, int c, int d) {
    const int64_t v[17] = {g.N, g.C, g.H, g.W, g.OC, g.FH, g.FW, g.sh, g.sw, g.ph, g.pw, g.dh, g.dw, a, b, c, d};
    return std::string(reinterpret_cast<const char*>(v), sizeof(v));
}
template <class V>
struct PlanMemo {
    std::mutex mu;
    std::unordered_map<std::string, V> m;
    template <class F>
    V get(const std::string& k, F&& make) {
        {
            std::lock_guard<std::mutex> lk(mu);
            auto it = m.find(k);
            if (it != m.end()) return it->second;
        }
        V v = make();  // computed outside the lock (pure function of the key)
        std::lock_guard<std::mutex> lk(mu);
        if (m.size() >= 4096) m.clear();  // bounded
        m.emplace(k, v);
        return v;
    }
};
}  // namespace

IgemmCfg igemm_cfg_fwd(const cks_geom& g, cks_dtype dt, int num_sms) {
    static PlanMemo<IgemmCfg> memo;
    return memo.get(plan_key(g, dt, 0, 0, num_sms), [&] { return igemm_cfg_fwd_plan(g, dt, num_sms); });
}
IgemmCfg igemm_cfg_deconv(const cks_geom& g, cks_dtype dt, int num_sms) {
    static PlanMemo<IgemmCfg> memo;
    return memo.get(plan_key(g, dt, 1, 0, num_sms), [&] { return igemm_cfg_deconv_plan(g, dt, num_sms); });
}
RowCfg row_cfg_fwd(const cks_geom& g, cks_dtype dt, bool allow_rg) {
    static PlanMemo<RowCfg> memo;
    return memo.get(plan_key(g, dt, 0, allow_rg ? 1 : 0, 0), [&] { return row_cfg_fwd_plan(g, dt, allow_rg); });
}
RowCfg row_cfg_wgrad(const cks_geom& g, cks_dtype dt, int gz_req, int num_sms, bool allow_rg) {
    static PlanMemo<RowCfg> memo;
    return memo.get(plan_key(g, dt, allow_rg ? 2 : 4, gz_req, num_sms),
                    [&] { return row_cfg_wgrad_plan(g, dt, gz_req, num_sms, allow_rg); });
}
IgemmCfg igemm_cfg_deconv_w(const cks_geom& g, cks_dtype dt, int num_sms) {
    static PlanMemo<IgemmCfg> memo;
    return memo.get(plan_key(g, dt, 3, 0, num_sms), [&] { return igemm_cfg_deconv_w_plan(g, dt, num_sms); });
}
WgradCfg wgrad_cfg(const cks_geom& g, cks_dtype dt, int gz_req, int num_sms) {
    static PlanMemo<WgradCfg> memo;
    return memo.get(plan_key(g, dt, 2, gz_req, num_sms), [&] { return wgrad_cfg_plan(g, dt, gz_req, num_sms); });
}
WsLayout ws_layout(const cks_geom& g, cks_dtype dt, cks_op op, int gz, bool c_packed_given, int num_sms) {
    static PlanMemo<WsLayout> memo;
    return memo.get(plan_key(g, dt, int(op), gz * 2 + (c_packed_given ? 1 : 0), num_sms),
                    [&] { return ws_layout_plan(g, dt, op, gz, c_packed_given, num_sms); });
}

// ---------------------------------------------------------------- 3-D plans
cks_status validate3(const cks_geom3* g) {
    if (!g) return CKS_ERR_NULL;
    if (g->D < 1 || g->FD < 1 || g->sd < 1 || g->pd < 0) return CKS_ERR_GEOMETRY;
    if (g->pd >= g->FD || g->D + 2 * g->pd - g->FD < 0) return CKS_ERR_GEOMETRY;
    if (g->FD > 32 || g->sd > 8) return CKS_ERR_UNSUPPORTED;
    const cks_geom g2 = plane_geom(*g);
    cks_status s = validate(&g2);
    if (s != CKS_OK) return s;
    const Axis ad = axis_d(*g), ah = axis_h(g2);
    if (ad.O * ah.O > int64_t(CKS_MAX_ROWS) * 256 || g->D * g->H > int64_t(CKS_MAX_ROWS) * 256 ||
        ad.O > CKS_MAX_ROWS || g->D > CKS_MAX_ROWS)
        return CKS_ERR_UNSUPPORTED;
    return CKS_OK;
}

cks_geom plane_geom(const cks_geom3& g) {
    cks_geom p;
    p.N = g.N, p.C = g.C, p.H = g.H, p.W = g.W, p.OC = g.OC, p.FH = g.FH, p.FW = g.FW;
    p.sh = g.sh, p.sw = g.sw, p.ph = g.ph, p.pw = g.pw, p.dh = 1, p.dw = 1;
    return p;
}

Axis axis_d(const cks_geom3& g) { return Axis{g.D, g.FD, g.sd, g.pd, out_extent(g.D, g.FD, g.sd, g.pd)}; }

static std::string plan_key3(const cks_geom3& g, int a, int b, int c, int d) {
    const int64_t v[19] = {g.N, g.C, g.D, g.H, g.W, g.OC, g.FD, g.FH, g.FW, g.sd, g.sh, g.sw, g.pd, g.ph, g.pw,
                           a, b, c, d};
    return std::string(reinterpret_cast<const char*>(v), sizeof(v));
}

IgemmCfg igemm_cfg_fwd3(const cks_geom3& g, cks_dtype dt, int num_sms) {
    static PlanMemo<IgemmCfg> memo;
    return memo.get(plan_key3(g, dt, 0, 0, num_sms), [&] {
        const cks_geom g2 = plane_geom(g);
        const Axis ad = axis_d(g), aw = axis_w(g2);
        const int rg = rg_plan(g2, false);  // row groups inside a depth slice (h rows of one window)
        const auto rh = igemm_rows_fwd(g2, rg);
        IgemmCfg c = igemm_cfg(ad.O * int64_t(rh.size()), {aw.O}, g.N, g.OC, pad_ch(g.C, dt), elem_bytes(dt),
                               max_window(rh) * max_window(krows_fwd(ad)), g.FW, g.sw, num_sms, 0, 0, rg);
        c.rg_es = int(g.sh);
        c.rg_ostep = 1;
        return c;
    });
}

IgemmCfg igemm_cfg_deconv3(const cks_geom3& g, cks_dtype dt, int num_sms) {
    static PlanMemo<IgemmCfg> memo;
    return memo.get(plan_key3(g, dt, 1, 0, num_sms), [&] {
        const cks_geom g2 = plane_geom(g);
        const Axis ad = axis_d(g), aw = axis_w(g2);
        std::vector<int64_t> cnt;
        for (auto& ph : table_t2(aw)) cnt.push_back(ph.U);
        const int atomw = int(128 / elem_bytes(dt));
        const int fb = g.C % atomw == 0 ? -atomw : atomw;  // Stage1-free: whole 128-byte MN atoms of W
        const int rg = rg_plan(g2, true);
        const auto rh = igemm_rows_deconv(g2, rg);
        IgemmCfg c = igemm_cfg(ad.I * int64_t(rh.size()), cnt, g.N, g.C, pad_ch(g.OC, dt), elem_bytes(dt),
                               max_window(rh) * max_window(krows_deconv(ad)), cdiv(g.FW, g.sw), 1, num_sms, 0, fb,
                               rg);
        c.rg_es = 1;
        c.rg_ostep = int(g.sh);
        return c;
    });
}

WgradCfg wgrad_cfg3(const cks_geom3& g, cks_dtype dt, int gz_req, int num_sms) {
    static PlanMemo<WgradCfg> memo;
    return memo.get(plan_key3(g, dt, 2, gz_req, num_sms), [&] {
        const Axis ad = axis_d(g);
        return wgrad_cfg_plan(plane_geom(g), dt, gz_req, num_sms, &ad);
    });
}

WsLayout ws_layout3(const cks_geom3& g, cks_dtype dt, cks_op op, int gz, int num_sms) {
    WsLayout L;
    const int64_t eb = elem_bytes(dt), Cp = pad_ch(g.C, dt), OCp = pad_ch(g.OC, dt);
    const Axis ad = axis_d(g);
    const cks_geom g2 = plane_geom(g);
    const int64_t OH = axis_h(g2).O, OW = axis_w(g2).O;
    size_t off = 0;
    auto take = [&](size_t bytes, size_t& at, size_t& sz) {
        if (!bytes) return;
        at = off;
        sz = bytes;
        off += align256(bytes);
    };
    if ((op == CKS_OP_FWD || op == CKS_OP_WGRAD) && Cp != g.C)
        take(size_t(g.N) * g.D * g.H * g.W * Cp * eb, L.x_pad, L.x_pad_bytes);
    if (op == CKS_OP_FWD && Cp != g.C) take(size_t(g.OC) * g.FD * g.FH * g.FW * Cp * eb, L.w_pad, L.w_pad_bytes);
    if ((op == CKS_OP_DECONV || op == CKS_OP_WGRAD) && OCp != g.OC)
        take(size_t(g.N) * ad.O * OH * OW * OCp * eb, L.dy_pad, L.dy_pad_bytes);
    if (op == CKS_OP_FWD || op == CKS_OP_DECONV) {
        const IgemmCfg c = op == CKS_OP_FWD ? igemm_cfg_fwd3(g, dt, num_sms) : igemm_cfg_deconv3(g, dt, num_sms);
        if (c.Z > 1 && !c.zc) {
            take(size_t(c.out_tiles) * c.Z * 128 * c.pbw * c.BN * 4, L.partial, L.partial_bytes);
            take(size_t(c.out_tiles) * 4, L.sem, L.sem_bytes);
        }
    }
    if (op == CKS_OP_WGRAD) {
        const WgradCfg c = wgrad_cfg3(g, dt, gz, num_sms);
        if (c.npart() > 1 && !c.zc)
            take(size_t(c.npart()) * g.OC * g.FD * g.FH * g.FW * g.C * 4, L.partial, L.partial_bytes);
    }
    L.total = off;
    return L;
}

}  // namespace cks
