// cks_api.cu -- the C ABI of libcks.so (include/cks.h): validation,
// workspace carving, TMA descriptor encoding and kernel launches (layer L3).
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>
#include <unordered_map>
#include <utility>

#include "../../include/cks.h"
#include "cks_plan.h"
#include "kernels/allreduce.cuh"
#include "kernels/aux.cuh"
#include "kernels/igemm.cuh"
#include "kernels/narrow.cuh"
#include "kernels/wgrad.cuh"

using namespace cks;

namespace {

constexpr int kPlanSMs = 148;  // B200: plan decisions are device-independent

// ------------------------------------------------------------------ driver entry
typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiledFn get_encode() {
    static EncodeTiledFn fn = nullptr;
    static std::once_flag once;
    std::call_once(once, [] {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<EncodeTiledFn>(p);
    });
    return fn;
}

// Tensor-map cache: encoding is a pure function of its arguments (base
// pointer, shape, strides, box, swizzle ...), so a training loop that calls
// an op again on the same buffers reuses the encoded CUtensorMap (thread-safe,
// bounded).
CUresult encode_cached(EncodeTiledFn enc, CUtensorMap* m, CUtensorMapDataType dt, cuuint32_t rank, void* base,
                       const cuuint64_t* gd, const cuuint64_t* gs, const cuuint32_t* bd, const cuuint32_t* es,
                       CUtensorMapInterleave il, CUtensorMapSwizzle sw, CUtensorMapL2promotion l2,
                       CUtensorMapFloatOOBfill oob) {
    static std::mutex mu;
    static std::unordered_map<std::string, CUtensorMap> cache;
    uint64_t k[32];
    int n = 0;
    k[n++] = uint64_t(dt);
    k[n++] = rank;
    k[n++] = reinterpret_cast<uint64_t>(base);
    for (cuuint32_t i = 0; i < rank; ++i) k[n++] = gd[i];
    for (cuuint32_t i = 0; i + 1 < rank; ++i) k[n++] = gs[i];
    for (cuuint32_t i = 0; i < rank; ++i) k[n++] = (uint64_t(bd[i]) << 32) | es[i];
    k[n++] = (uint64_t(il) << 48) | (uint64_t(sw) << 32) | (uint64_t(l2) << 16) | uint64_t(oob);
    const std::string key(reinterpret_cast<const char*>(k), sizeof(uint64_t) * n);
    {
        std::lock_guard<std::mutex> lk(mu);
        auto it = cache.find(key);
        if (it != cache.end()) {
            *m = it->second;
            return CUDA_SUCCESS;
        }
    }
    const CUresult r = enc(m, dt, rank, base, gd, gs, bd, es, il, sw, l2, oob);
    if (r == CUDA_SUCCESS) {
        std::lock_guard<std::mutex> lk(mu);
        if (cache.size() >= 4096) cache.clear();
        cache.emplace(key, *m);
    }
    return r;
}

// cuMemGetAddressRange through the runtime's driver entry point (libcks.so
// links the static runtime only, not libcuda)
typedef CUresult (*MemRangeFn)(CUdeviceptr*, size_t*, CUdeviceptr);
bool mem_range(const void* p, CUdeviceptr* base) {
    static MemRangeFn fn = nullptr;
    static std::once_flag once;
    std::call_once(once, [] {
        void* f = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuMemGetAddressRange", &f, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<MemRangeFn>(f);
    });
    size_t size = 0;
    return fn && fn(base, &size, reinterpret_cast<CUdeviceptr>(p)) == CUDA_SUCCESS;
}

int device_sms() {
    int dev = 0, sms = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) return kPlanSMs;
    if (cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || sms <= 0) return kPlanSMs;
    return sms;
}

// rank-4 tiled tensor map, 128B swizzle, zero OOB fill
bool make_tmap4(CUtensorMap* m, cks_dtype dt, const void* base, const uint64_t dims[4], const uint64_t strides_b[3],
                const uint32_t box[4], int row_bytes = 128, bool atom32 = false, const uint32_t* estr = nullptr) {
    EncodeTiledFn enc = get_encode();
    if (!enc) return false;
    cuuint64_t gd[4] = {dims[0], dims[1], dims[2], dims[3]};
    cuuint64_t gs[3] = {strides_b[0], strides_b[1], strides_b[2]};
    cuuint32_t bd[4] = {box[0], box[1], box[2], box[3]};
    cuuint32_t es[4] = {1, 1, 1, 1};
    if (estr)  // element strides: box[i] = count * estr[i] loads count elements at stride estr[i]
        for (int i = 0; i < 4; ++i) es[i] = estr[i];
    CUresult r = encode_cached(enc, m, dt == CKS_BF16 ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4,
                     const_cast<void*>(base), gd, gs, bd, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                     atom32 ? CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B  // MN-major tf32 (SWIZZLE_128B_BASE32B)
                            : (row_bytes == 128 ? CU_TENSOR_MAP_SWIZZLE_128B
                                                : (row_bytes == 64 ? CU_TENSOR_MAP_SWIZZLE_64B : CU_TENSOR_MAP_SWIZZLE_32B)),
                     CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return r == CUDA_SUCCESS;
}

int debug_flags() {
    static int f = [] {
        const char* e = cks_knob("CKS_DEBUG_FLAGS");  // experiments only; unset in production
        return e ? atoi(e) : 0;
    }();
    return f;
}

// experiments: allocate all 512 TMEM columns per igemm CTA (the former behaviour)
bool tmem_full() {
    static const bool on = cks_knob("CKS_TMEM_FULL") != nullptr;
    return on;
}

// TMA-store epilogue for every igemm tile (0: only the last tile per CTA; experiments)
bool epi_tma_all() {
    static const bool on = [] {
        const char* e = cks_knob("CKS_EPI_TMA");
        return e ? atoi(e) != 0 : true;
    }();
    return on;
}

// rank-5 tiled tensor map with element strides (Stage1-free KS-deconv B operand)
bool make_tmap5(CUtensorMap* m, cks_dtype dt, const void* base, const uint64_t dims[5], const uint64_t strides_b[4],
                const uint32_t box[5], const uint32_t estr[5]) {
    EncodeTiledFn enc = get_encode();
    if (!enc) return false;
    cuuint64_t gd[5] = {dims[0], dims[1], dims[2], dims[3], dims[4]};
    cuuint64_t gs[4] = {strides_b[0], strides_b[1], strides_b[2], strides_b[3]};
    cuuint32_t bd[5] = {box[0], box[1], box[2], box[3], box[4]};
    cuuint32_t es[5] = {estr[0], estr[1], estr[2], estr[3], estr[4]};
    return encode_cached(enc, m, dt == CKS_BF16 ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 5,
                         const_cast<void*>(base), gd, gs, bd, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                         dt == CKS_TF32 ? CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B : CU_TENSOR_MAP_SWIZZLE_128B,
                         CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// fp32 output map (TMA store), 128B swizzle
bool make_tmap4_f32(CUtensorMap* m, const void* base, const uint64_t dims[4], const uint64_t strides_b[3],
                    const uint32_t box[4]) {
    EncodeTiledFn enc = get_encode();
    if (!enc) return false;
    cuuint64_t gd[4] = {dims[0], dims[1], dims[2], dims[3]};
    cuuint64_t gs[3] = {strides_b[0], strides_b[1], strides_b[2]};
    cuuint32_t bd[4] = {box[0], box[1], box[2], box[3]};
    cuuint32_t es[4] = {1, 1, 1, 1};
    return encode_cached(enc, m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, const_cast<void*>(base), gd, gs, bd, es,
               CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
               CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }

cks_status last_cuda() {
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) {
        fprintf(stderr, "[cks] CUDA error: %s\n", cudaGetErrorString(e));
        return CKS_ERR_CUDA;
    }
    return CKS_OK;
}

// Launch with programmatic stream serialization (PDL): the kernel may start
// while its predecessor drains; every kernel calls griddepcontrol.wait before
// touching global memory, so stream order semantics are preserved.
template <typename... KArgs, typename... Args>
cks_status launch_pdl_cluster(void (*kern)(KArgs...), dim3 grid, dim3 block, int smem, cudaStream_t st, int cluster,
                              Args&&... args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = size_t(smem);
    cfg.stream = st;
    // experiments: CKS_NO_PDL=1 launches without programmatic dependent launch (ncu graph probes)
    static const bool no_pdl = cks_knob("CKS_NO_PDL") != nullptr;
    cudaLaunchAttribute attr[2];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = no_pdl ? 0 : 1;
    attr[1].id = cudaLaunchAttributeClusterDimension;
    attr[1].val.clusterDim.x = unsigned(cluster);
    attr[1].val.clusterDim.y = 1;
    attr[1].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = cluster > 1 ? 2 : 1;
    if (cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...) != cudaSuccess) {
        last_cuda();
        return CKS_ERR_CUDA;
    }
    return CKS_OK;
}

template <typename... KArgs, typename... Args>
cks_status launch_pdl(void (*kern)(KArgs...), dim3 grid, dim3 block, int smem, cudaStream_t st, Args&&... args) {
    return launch_pdl_cluster(kern, grid, block, smem, st, 1, std::forward<Args>(args)...);
}

template <typename K>
cks_status set_smem(K kernel, int bytes) {
    // cudaFuncSetAttribute per call is cheap; keep it stateless (multi-device safe)
    if (cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes) != cudaSuccess) {
        last_cuda();
        return CKS_ERR_CUDA;
    }
    return CKS_OK;
}

FastDiv make_fastdiv(uint32_t d) {
    FastDiv f;
    f.d = d;
    uint32_t l = 0;
    while ((uint64_t(1) << l) < d) ++l;
    f.sh = 31 + l;
    f.m = uint32_t(((uint64_t(1) << f.sh) + d - 1) / d);
    return f;
}

// Compact axis table for the kernel parameters (KAxisC): per-row windows and
// per-phase affine (a0, out) maps.  Returns false (-> CKS_ERR_UNSUPPORTED) if
// the rows are not affine per phase or exceed the phase limit; the expansion in
// the kernel reproduces the KRow table exactly.
bool fill_axis(KAxisC& k, const std::vector<KRow>& rows) {
    memset(&k, 0, sizeof(k));
    const std::vector<int> st = run_starts(rows);  // affine runs (one phase, one group length)
    if (st.size() > size_t(kMaxPhases)) return false;
    const int nph = int(st.size());
    for (int x = 0; x < nph; ++x) {
        const KRow& r = rows[st[x]];
        const int e = x + 1 < nph ? st[x + 1] : int(rows.size());
        if (r.phase > 255 || r.glen < 1 || r.glen > 16 || (r.glen > 1 && r.phase > 15)) return false;
        k.row0[x] = int16_t(st[x]);
        k.phid[x] = int16_t(r.phase);
        k.rlen[x] = int8_t(r.glen);
        k.a00[x] = int16_t(r.a0);
        k.out0[x] = int16_t(r.out);
        if (st[x] + 1 < e) {
            k.a0st[x] = int16_t(rows[st[x] + 1].a0 - r.a0);
            k.outst[x] = int16_t(rows[st[x] + 1].out - r.out);
        }
        for (int i = st[x]; i < e; ++i) {
            const int u = i - st[x];
            if (rows[i].a0 != k.a00[x] + int64_t(u) * k.a0st[x] || rows[i].out != k.out0[x] + int64_t(u) * k.outst[x])
                return false;
            k.ts[i] = uint8_t(rows[i].ts);
            k.te[i] = uint8_t(rows[i].te);
        }
    }
    k.row0[nph] = int16_t(rows.size());
    k.nph = int16_t(nph);
    k.nrows = int16_t(rows.size());
    return true;
}

bool rows_ok(const std::vector<KRow>& rows) {
    if (rows.empty() || rows.size() > CKS_MAX_ROWS) return false;
    for (auto& r : rows)
        if (r.a0 < -32768 || r.a0 > 32767 || r.out > 32767 || r.ts < 0 || r.te > 255 || r.phase > 255) return false;
    return true;
}

// ------------------------------------------------------------------ launchers
template <int BN, bool TF, int KB, bool PAIR = false, bool BMN = false>
cks_status launch_igemm_t(const CUtensorMap& a, const CUtensorMap& b, const CUtensorMap& y, const IgemmParams& p,
                          int smem, cudaStream_t st) {
    auto kern = igemm_kernel<BN, TF, KB, PAIR, BMN>;
    if (set_smem(kern, smem) != CKS_OK) return CKS_ERR_CUDA;
    // cluster split-K: one output tile per cluster of zsplit CTAs, one tile per CTA
    const int cl = p.zc ? p.zsplit : (p.pair ? 2 : p.cm);
    long long grid = p.zc ? p.num_tiles
                          : (p.pair ? 2 * std::min<long long>(p.num_tiles, device_sms() / 2)
                                    : std::min<long long>(p.num_tiles, device_sms() / p.cm * p.cm));  // whole clusters
    if (grid < 1) grid = 1;
    if (cl > 1 &&
        cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1) != cudaSuccess)
        return last_cuda();
    return launch_pdl_cluster(kern, dim3(unsigned(grid)), dim3(384), smem, st, cl, a, b, y, p);
}

template <bool TF, int KB>
cks_status launch_igemm_kb(int BN, const CUtensorMap& a, const CUtensorMap& b, const CUtensorMap& y,
                           const IgemmParams& p, int smem, cudaStream_t st) {
    switch (BN) {
        case 32: return launch_igemm_t<32, TF, KB>(a, b, y, p, smem, st);
        case 64: return launch_igemm_t<64, TF, KB>(a, b, y, p, smem, st);
        case 128: return launch_igemm_t<128, TF, KB>(a, b, y, p, smem, st);
    }
    return CKS_ERR_UNSUPPORTED;
}

template <int BN, bool TF>
cks_status launch_igemm_bmn(int KB, const CUtensorMap& a, const CUtensorMap& b, const CUtensorMap& y,
                            const IgemmParams& p, int smem, cudaStream_t st) {
    if (KB == 32) return launch_igemm_t<BN, TF, 32, false, true>(a, b, y, p, smem, st);
    if (KB == 64) return launch_igemm_t<BN, TF, 64, false, true>(a, b, y, p, smem, st);
    return launch_igemm_t<BN, TF, 128, false, true>(a, b, y, p, smem, st);
}

cks_status launch_igemm(int BN, int KB, bool tf32, const CUtensorMap& a, const CUtensorMap& b, const CUtensorMap& y,
                        const IgemmParams& p, int smem, cudaStream_t st, bool bmn = false) {
    if (bmn) {  // Stage1-free KS-deconv: B = one 128-byte MN atom of W per tap (BN = 64 bf16 / 32 tf32)
        if (p.pair || p.cm > 1) return CKS_ERR_UNSUPPORTED;
        if (tf32) {
            switch (BN) {
                case 32: return launch_igemm_bmn<32, true>(KB, a, b, y, p, smem, st);
                case 64: return launch_igemm_bmn<64, true>(KB, a, b, y, p, smem, st);
                case 128: return launch_igemm_bmn<128, true>(KB, a, b, y, p, smem, st);
            }
            return CKS_ERR_UNSUPPORTED;
        }
        if (BN == 64) return launch_igemm_bmn<64, false>(KB, a, b, y, p, smem, st);
        if (BN == 128) return launch_igemm_bmn<128, false>(KB, a, b, y, p, smem, st);
        return CKS_ERR_UNSUPPORTED;
    }
    if (p.pair) {  // CTA pairs: 128 B K blocks, 128 output channels per CTA (plan invariant)
        if (KB != 128 || BN != 128) return CKS_ERR_UNSUPPORTED;
        return tf32 ? launch_igemm_t<128, true, 128, true>(a, b, y, p, smem, st)
                    : launch_igemm_t<128, false, 128, true>(a, b, y, p, smem, st);
    }
    if (tf32) {
        if (KB == 32) return launch_igemm_kb<true, 32>(BN, a, b, y, p, smem, st);
        if (KB == 64) return launch_igemm_kb<true, 64>(BN, a, b, y, p, smem, st);
        return launch_igemm_kb<true, 128>(BN, a, b, y, p, smem, st);
    }
    if (KB == 32) return launch_igemm_kb<false, 32>(BN, a, b, y, p, smem, st);
    if (KB == 64) return launch_igemm_kb<false, 64>(BN, a, b, y, p, smem, st);
    return launch_igemm_kb<false, 128>(BN, a, b, y, p, smem, st);
}

// Depth axis of a 3-D igemm launch (2-D: one trivial depth row).
struct Depth3 {
    std::vector<KRow> rd;  // depth rows (T1 / T2 of the d axis)
    int a_rows_h = 0;      // A rows per depth slice
    int out_rows_h = 0;    // output rows per depth slice
    int b_rows_h = 0;      // filter rows per depth slice (packed / W row index = d * b_rows_h + h)
    int FD = 1, sd = 1;    // W-direct: filter depth and depth stride
};

// Fill IgemmParams from the plan and launch (fwd and deconv share this).
// out_H: output rows in total (3-D: OD * OH, flattened).
cks_status run_igemm(const IgemmCfg& cfg_in, cks_dtype dt, const std::vector<KRow>& rh, const std::vector<KRow>& rw,
                     const CUtensorMap& ta, const CUtensorMap& tb, float* out, int out_H, int out_W, int out_C,
                     int N, int slot_stride, int phases_w, const WsLayout& L, void* ws, cudaStream_t st,
                     const cks_geom* bmn = nullptr, const Depth3* d3 = nullptr) {
    IgemmCfg cfg = cfg_in;
    if (debug_flags() & 16) {  // experiment: no split-K
        cfg.Z = 1;
        cfg.zc = 0;
        cfg.tiles = cfg.out_tiles;
    }
    IgemmParams p;
    memset(&p, 0, sizeof(p));
    if (!fill_axis(p.ah, rh) || !fill_axis(p.aw, rw)) return CKS_ERR_UNSUPPORTED;
    {
        static const std::vector<KRow> trivial = {KRow{0, 0, 1, 0, 0}};
        if (!fill_axis(p.ad, d3 ? d3->rd : trivial)) return CKS_ERR_UNSUPPORTED;
        p.a_rows_h = d3 ? d3->a_rows_h : 0;
        p.out_rows_h = d3 ? d3->out_rows_h : 0;
        p.b_rows_h = d3 ? d3->b_rows_h : 0;
        p.phases_h = bmn ? bmn->sh : 1;
        p.fd_rh = make_fastdiv(uint32_t(rh.size()));
    }
    p.out = out;
    p.rows_h = int(rh.size());
    p.nph_w = int(cfg.wph_cnt.size());
    if (p.nph_w > 8) return CKS_ERR_UNSUPPORTED;
    int off = 0, cum = 0;
    for (int x = 0; x < p.nph_w; ++x) {
        p.wph_off[x] = int16_t(off);
        p.wph_cnt[x] = int16_t(cfg.wph_cnt[x]);
        p.wb_cum[x] = int16_t(cum);
        off += int(cfg.wph_cnt[x]);
        cum += int((cfg.wph_cnt[x] + cfg.pbw - 1) / cfg.pbw);
    }
    p.wb_cum[p.nph_w] = int16_t(cum);
    p.wblocks = cfg.wblocks;
    p.pbw = cfg.pbw;
    p.acc_stages = cfg.acc_stages;
    p.nblk = cfg.nblk;
    p.nbs = cfg.nbs;
    p.kc_blocks = cfg.kc_blocks;
    p.slot_stride = slot_stride;
    p.phases_w = phases_w;
    p.N = N;
    p.out_H = out_H;
    p.out_W = out_W;
    p.out_C = out_C;
    p.zsplit = cfg.Z;
    p.zc = cfg.zc;
    p.pair = cfg.pair;
    if (cfg.rg_ni > 0) {  // row groups: M row r = (group row r / rg_ni, image r % rg_ni)
        if (cfg.rg_ni != 32 && cfg.rg_ni != 64) return CKS_ERR_UNSUPPORTED;
        p.rg_ni = cfg.rg_ni;
        p.rg_shift = cfg.rg_ni == 32 ? 5 : 6;
        p.rg_ostep = cfg.rg_ostep;
    }
    p.epi_warps = cfg.epi ? cfg.epi_warps : 4;
    p.epi_bufs = cfg.epi ? cfg.epi_bufs : 1;
    {
        const int need = cfg.acc_stages * cfg.pbw * cfg.BN * (cfg.pair ? 2 : 1);
        if (need > 512) return CKS_ERR_UNSUPPORTED;  // TMEM holds 512 fp32 columns per SM
        int cols = 32;
        while (cols < need) cols *= 2;
        p.tmem_cols = tmem_full() ? 512 : cols;
    }
    p.fd_z = make_fastdiv(uint32_t(cfg.Z));
    p.fd_nbs = make_fastdiv(uint32_t(cfg.nbs));
    p.fd_nblk = make_fastdiv(uint32_t(cfg.nblk));
    p.fd_wb = make_fastdiv(uint32_t(cfg.wblocks));
    p.fd_kc = make_fastdiv(uint32_t(cfg.kc_blocks));
    p.num_tiles = cfg.tiles;
    p.dbg = debug_flags();
#ifdef CKS_EXPERIMENTS
    // debug timeline (tools/trace_op.py); absent from the production library
    if (const char* tp = cks_knob("CKS_TRACE_PTR")) p.trace = reinterpret_cast<unsigned long long*>(strtoull(tp, nullptr, 0));
#endif
    // shared memory: A-position ring (16 KB slots) + B-row ring (all taps of a filter row)
    p.a_stages = cfg.a_stages;
    p.b_stages = cfg.stages;
    p.b_stage_bytes = cfg.stage_bytes;
    p.ntap = cfg.ntap;
    p.apos = cfg.apos;
    p.unit_step = cfg.unit_step;
    p.a0_step = cfg.a0_step;
    if (p.a_stages < 2 || p.b_stages < 1) return CKS_ERR_UNSUPPORTED;
    p.epi_stage = cfg.epi;
    p.cm = cfg.cm;
    p.unified = cfg.unified;
    const int smem = 1024 + p.a_stages * p.apos * 128 * cfg.KB + p.b_stages * p.b_stage_bytes + 512 +
                     int(3 * sizeof(KAxis)) + 2 * kProgSlot * 16 + (cfg.epi ? epi_stage_bytes(cfg.epi_warps, cfg.epi_bufs) + 1024 : 0);
    if (cfg.Z > 1 && !cfg.zc) {
        if (!L.partial_bytes || !L.sem_bytes) return CKS_ERR_WORKSPACE;
        p.part = reinterpret_cast<float*>(static_cast<uint8_t*>(ws) + L.partial);
        p.sem = reinterpret_cast<int*>(static_cast<uint8_t*>(ws) + L.sem);
        if (cudaMemsetAsync(p.sem, 0, L.sem_bytes, st) != cudaSuccess) return last_cuda();
    }
    // output tensor map (fp32, 32 channels x 32 images boxes, 128B swizzle) for
    // the last-tile TMA-store epilogue; needs 16-byte rows and staging room in
    // the (then idle) A/B rings: 4 warps x PBW x BN/32 blocks of 4 KB
    CUtensorMap ty;
    memset(&ty, 0, sizeof(ty));
    const int64_t stage_need = int64_t(4) * cfg.pbw * (cfg.BN * (cfg.pair ? 2 : 1) / 32) * 4096;
    const int64_t ring = int64_t(p.a_stages) * p.apos * 128 * cfg.KB + int64_t(p.b_stages) * p.b_stage_bytes;
    if (cfg.Z == 1 && out_C % 4 == 0 && stage_need <= ring && !(debug_flags() & 32)) {
        uint64_t d[4] = {uint64_t(out_C), uint64_t(out_W), uint64_t(out_H), uint64_t(N)};
        uint64_t sb[3] = {uint64_t(out_C) * 4, uint64_t(out_W) * out_C * 4, uint64_t(out_H) * out_W * out_C * 4};
        uint32_t box[4] = {32, 1, 1, 32};
        if (make_tmap4_f32(&ty, out, d, sb, box)) p.tma_store = (cfg.epi && epi_tma_all()) ? 2 : 1;
    }
    if (bmn) {  // Stage1-free: per-phase filter-row origin and sub-filter widths (Alg. 2 Stage1's index map)
        if (bmn->sh > kMaxPhases || bmn->sw > kMaxPhases) return CKS_ERR_UNSUPPORTED;
        for (int y = 0; y < bmn->sh; ++y) p.bfh0[y] = int16_t(y + (cdiv(bmn->FH - y, bmn->sh) - 1) * bmn->sh);
        const int FD = d3 ? d3->FD : 1, sd = d3 ? d3->sd : 1;
        if (sd > kMaxPhases) return CKS_ERR_UNSUPPORTED;
        for (int z = 0; z < sd; ++z) p.bfd0[z] = int16_t(z + (cdiv(FD - z, sd) - 1) * sd);
        p.bsd = sd;
        p.b_rows_h = int(bmn->FH);
        for (int x = 0; x < bmn->sw; ++x) p.bcw[x] = int16_t(cdiv(bmn->FW - x, bmn->sw));
        p.bsh = bmn->sh;
    }
    return launch_igemm(cfg.BN, cfg.KB, dt == CKS_TF32, ta, tb, ty, p, smem, st, bmn != nullptr);
}

template <int BN, bool TF, int KIMG, int MT, bool A1, bool PP, bool RG>
cks_status launch_wgrad_k(const CUtensorMap& a, const CUtensorMap& b, const WgradParams& p, cudaStream_t st) {
    using S = WgradShape<BN, TF, KIMG, MT, A1, PP>;
    auto kern = wgrad_kernel<BN, TF, KIMG, MT, A1, PP, RG>;
    if (set_smem(kern, S::SMEM_BYTES) != CKS_OK) return CKS_ERR_CUDA;
    if (p.zc) {  // one tile per CTA, the gz segments of a tile are one cluster
        if (p.gz > 8) return CKS_ERR_UNSUPPORTED;
        return launch_pdl_cluster(kern, dim3(unsigned(p.num_tiles)), dim3(256), S::SMEM_BYTES, st, p.gz, a, b, p);
    }
    if (p.tcmc) {  // filter-row clusters: tc consecutive tiles (the filter rows of one segment) per cluster
        long long grid = std::min<long long>(p.num_tiles, device_sms() / p.tc * p.tc);
        if (grid < p.tc || p.num_tiles % p.tc) return CKS_ERR_UNSUPPORTED;
        return launch_pdl_cluster(kern, dim3(unsigned(grid)), dim3(256), S::SMEM_BYTES, st, p.tc, a, b, p);
    }
    long long grid = std::min<long long>(p.num_tiles, device_sms());
    if (grid < 1) grid = 1;
    return launch_pdl(kern, dim3(unsigned(grid)), dim3(256), S::SMEM_BYTES, st, a, b, p);
}

// row-group (position-chunk) k-blocks are a separate instantiation: the batch-as-K kernels keep
// their exact issue sequence (a runtime flag in the MMA loop cost up to 14 %: C6 5x5 64->64)
template <int BN, bool TF, int KIMG, int MT = 1, bool A1 = false, bool PP = false>
cks_status launch_wgrad_t(const CUtensorMap& a, const CUtensorMap& b, const WgradParams& p, cudaStream_t st) {
    if constexpr (PP) {
        if (p.rg) return CKS_ERR_UNSUPPORTED;
        return launch_wgrad_k<BN, TF, KIMG, MT, A1, PP, false>(a, b, p, st);
    } else {
        return p.rg ? launch_wgrad_k<BN, TF, KIMG, MT, A1, PP, true>(a, b, p, st)
                    : launch_wgrad_k<BN, TF, KIMG, MT, A1, PP, false>(a, b, p, st);
    }
}

cks_status launch_pad(cks_dtype dt, const void* src, void* dst, long long rows, int C, int Cp, cudaStream_t st) {
    long long total = rows * Cp;
    unsigned blocks = unsigned(std::min<long long>((total + 255) / 256, 148LL * 16));
    if (dt == CKS_BF16)
        return launch_pdl(pad_channels_kernel<uint16_t>, dim3(blocks), dim3(256), 0, st,
                          static_cast<const uint16_t*>(src), static_cast<uint16_t*>(dst), rows, C, Cp);
    return launch_pdl(pad_channels_kernel<uint32_t>, dim3(blocks), dim3(256), 0, st, static_cast<const uint32_t*>(src),
                      static_cast<uint32_t*>(dst), rows, C, Cp);
}

cks_status launch_split(const cks_geom& g, cks_dtype dt, const void* w, void* out, cudaStream_t st) {
    const int CHm = int(cdiv(g.FH, g.sh)), CWm = int(cdiv(g.FW, g.sw));
    const int OCp = int(pad_ch(g.OC, dt));
    dim3 grid(unsigned((OCp + 63) / 64), unsigned((g.C + 63) / 64), unsigned(g.sh * g.sw * CHm * CWm));
    dim3 block(256);
    if (dt == CKS_BF16)
        return launch_pdl(ks_split_kernel<uint16_t>, grid, block, 0, st, static_cast<const uint16_t*>(w),
                          static_cast<uint16_t*>(out), int(g.OC), int(g.FH), int(g.FW), int(g.C), g.sh, g.sw, CHm, CWm,
                          OCp);
    return launch_pdl(ks_split_kernel<uint32_t>, grid, block, 0, st, static_cast<const uint32_t*>(w),
                      static_cast<uint32_t*>(out), int(g.OC), int(g.FH), int(g.FW), int(g.C), g.sh, g.sw, CHm, CWm,
                      OCp);
}

// ------------------------------------------------------------------ narrow-channel row path
// X viewed as (W*C elements, N, H, 1): a box (JB, imgs, rows, 1) is the
// contiguous (fw, c) run of `rows` consecutive X rows for `imgs` images,
// element-addressed at (ow*sw - pw)*C + off (past-the-end / negative rows =
// zero fill).  K-major (ConvV2): swizzle of the row width; MN-major tf32
// (Sk-dilated): SWIZZLE_128B_ATOM_32B.
bool make_row_xmap(CUtensorMap* m, const void* x, const cks_geom& g, cks_dtype dt, uint32_t JB, uint32_t imgs,
                   uint32_t rows, bool mn_tf32) {
    const uint64_t eb = uint64_t(elem_bytes(dt));
    uint64_t d[4] = {uint64_t(g.W * g.C), uint64_t(g.N), uint64_t(g.H), 1};
    uint64_t sb[3] = {uint64_t(g.H * g.W * g.C) * eb, uint64_t(g.W * g.C) * eb, uint64_t(g.N * g.H * g.W * g.C) * eb};
    uint32_t box[4] = {JB, imgs, rows, 1};
    return make_tmap4(m, dt, x, d, sb, box, int(JB * eb), mn_tf32);
}

void fill_row_classes(RowClass* dst, const std::vector<RowClassH>& src) {
    for (size_t k = 0; k < src.size(); ++k) {
        dst[k].col0 = int16_t(src[k].col0);
        dst[k].cstep = int16_t(src[k].cstep);
        dst[k].ncols = int16_t(src[k].ncols);
        dst[k].off = int16_t(src[k].off);
        dst[k].kc0 = int8_t(src[k].kc0);
        dst[k].kc1 = int8_t(src[k].kc1);
        dst[k].base = int16_t(src[k].base);
        dst[k].cnt = int16_t(src[k].cnt);
    }
}

template <int ROWB, int BN, bool TF>
cks_status launch_fwd_row_t(const CUtensorMap& tx, const CUtensorMap& ty, const RowFwdParams& p, const RowXMaps& xm,
                            int smem, int grid, cudaStream_t st) {
    // row groups are a separate instantiation (the 128-image path keeps its exact code)
    auto kern = p.rg ? fwd_row_kernel<ROWB, BN, TF, true> : fwd_row_kernel<ROWB, BN, TF, false>;
    if (set_smem(kern, smem) != CKS_OK) return CKS_ERR_CUDA;
    return launch_pdl(kern, dim3(unsigned(grid)), dim3(256), smem, st, tx, ty, p, xm);
}

template <int ROWB, bool TF>
cks_status launch_fwd_row_rb(int BN, const CUtensorMap& tx, const CUtensorMap& ty, const RowFwdParams& p,
                             const RowXMaps& xm, int smem, int grid, cudaStream_t st) {
    switch (BN) {
        case 32: return launch_fwd_row_t<ROWB, 32, TF>(tx, ty, p, xm, smem, grid, st);
        case 64: return launch_fwd_row_t<ROWB, 64, TF>(tx, ty, p, xm, smem, grid, st);
        case 128: return launch_fwd_row_t<ROWB, 128, TF>(tx, ty, p, xm, smem, grid, st);
        case 256:
            if constexpr (!TF) return launch_fwd_row_t<ROWB, 256, TF>(tx, ty, p, xm, smem, grid, st);
            break;
    }
    return CKS_ERR_UNSUPPORTED;
}

cks_status run_fwd_row(const cks_geom& g, cks_dtype dt, const RowCfg& rc_in, const void* x, const void* w, float* y,
                       cudaStream_t st) {
    RowCfg rc = rc_in;
    CUtensorMap tx, ty;
    memset(&ty, 0, sizeof(ty));
    if (!make_row_xmap(&tx, x, g, dt, uint32_t(rc.JB), 128, 1, false)) return CKS_ERR_CUDA;
    static thread_local RowXMaps xm;  // per-class maps of the row-group plan (unused otherwise)
    if (rc.rg) {
        // per class: (W*C elements, N, class column, H), column stride cstep*sw*C, box JB x rg x rg_pc
        const uint64_t eb = uint64_t(elem_bytes(dt));
        bool ok = rc.cls.size() <= size_t(kRowClasses);
        for (size_t k = 0; ok && k < rc.cls.size(); ++k) {
            const RowClassH& c = rc.cls[k];
            const uint64_t cs = c.ncols > 1 ? uint64_t(c.cstep) * g.sw * g.C * eb : 16;
            uint64_t d[4] = {uint64_t(g.W * g.C), uint64_t(g.N), uint64_t(c.ncols), uint64_t(g.H)};
            uint64_t sb[3] = {uint64_t(g.H * g.W * g.C) * eb, cs, uint64_t(g.W * g.C) * eb};
            uint32_t box[4] = {uint32_t(rc.JB), uint32_t(rc.rg), uint32_t(rc.rg_pc), 1};
            ok = cs % 16 == 0 && make_tmap4(&xm.m[k], dt, x, d, sb, box, int(rc.JB * eb), false);
        }
        if (!ok) rc = row_cfg_fwd(g, dt, false);  // a class the row-group boxes cannot address: 128-image tiles
    }
    RowFwdParams p;
    memset(&p, 0, sizeof(p));
    if (rc.rg) {
        p.rg = rc.rg;
        p.rg_shift = rc.rg == 32 ? 5 : 6;
        p.rg_pc = rc.rg_pc;
    }
    p.w = w;
    p.y = y;
    p.N = int(g.N), p.H = int(g.H), p.W = int(g.W), p.C = int(g.C), p.OC = int(g.OC);
    p.FH = int(g.FH), p.FW = int(g.FW), p.sh = g.sh, p.sw = g.sw, p.ph = g.ph, p.pw = g.pw;
    p.OH = int(axis_h(g).O), p.OW = int(axis_w(g).O);
    p.nblk = rc.nblk;
    p.R = rc.R;
    p.ncls = int(rc.cls.size());
    fill_row_classes(p.cls, rc.cls);
    p.stages = rc.stages;
    if (g.OC % 32 == 0) {  // TMA-store epilogue: 32 channels x 32 images boxes
        uint64_t d[4] = {uint64_t(g.OC), uint64_t(p.OW), uint64_t(p.OH), uint64_t(g.N)};
        uint64_t sb[3] = {uint64_t(g.OC) * 4, uint64_t(p.OW) * g.OC * 4, uint64_t(p.OH) * p.OW * g.OC * 4};
        uint32_t box[4] = {32, 1, 1, 32};
        if (make_tmap4_f32(&ty, y, d, sb, box)) p.tma_store = 1;
    }
    const bool tf = dt == CKS_TF32;
    switch (rc.ROWB) {
        case 32: return tf ? launch_fwd_row_rb<32, true>(rc.BN, tx, ty, p, xm, rc.smem, rc.grid, st)
                           : launch_fwd_row_rb<32, false>(rc.BN, tx, ty, p, xm, rc.smem, rc.grid, st);
        case 64: return tf ? launch_fwd_row_rb<64, true>(rc.BN, tx, ty, p, xm, rc.smem, rc.grid, st)
                           : launch_fwd_row_rb<64, false>(rc.BN, tx, ty, p, xm, rc.smem, rc.grid, st);
        case 128: return tf ? launch_fwd_row_rb<128, true>(rc.BN, tx, ty, p, xm, rc.smem, rc.grid, st)
                            : launch_fwd_row_rb<128, false>(rc.BN, tx, ty, p, xm, rc.smem, rc.grid, st);
    }
    return CKS_ERR_UNSUPPORTED;
}

template <int ROWB, int BN, bool TF>
cks_status launch_wgrad_row_t(const CUtensorMap& tx, const CUtensorMap& tdy, const RowWgradParams& p,
                              const RowWXMaps& xm, int smem, cudaStream_t st) {
    // row groups: a separate instantiation (the 64-image path keeps its exact code)
    auto kern = p.rg ? wgrad_row_kernel<ROWB, BN, TF, true> : wgrad_row_kernel<ROWB, BN, TF, false>;
    if (set_smem(kern, smem) != CKS_OK) return CKS_ERR_CUDA;
    long long grid = std::max<long long>(1, std::min<long long>(p.num_tiles, device_sms()));
    return launch_pdl(kern, dim3(unsigned(grid)), dim3(256), smem, st, tx, tdy, p, xm);
}

template <int ROWB, bool TF>
cks_status launch_wgrad_row_rb(int BN, const CUtensorMap& tx, const CUtensorMap& tdy, const RowWgradParams& p,
                               const RowWXMaps& xm, int smem, cudaStream_t st) {
    switch (BN) {
        case 64: return launch_wgrad_row_t<ROWB, 64, TF>(tx, tdy, p, xm, smem, st);
        case 128: return launch_wgrad_row_t<ROWB, 128, TF>(tx, tdy, p, xm, smem, st);
        case 256: return launch_wgrad_row_t<ROWB, 256, TF>(tx, tdy, p, xm, smem, st);
    }
    return CKS_ERR_UNSUPPORTED;
}

cks_status run_wgrad_row(const cks_geom& g, cks_dtype dt, const RowCfg& rc_in, const void* x, const void* dys,
                         int64_t OCp, const CUtensorMap& tdy, float* wout, long long part_stride, cudaStream_t st) {
    const bool tf = dt == CKS_TF32;
    RowCfg rc = rc_in;
    static thread_local RowWXMaps xm;  // per-class maps of the row-group plan (unused otherwise)
    if (rc.rg) {
        // per class: X (W*C, N, class column, H) and dY (OCp, N, class column, OH), column strides
        // cstep*sw*C / cstep*OCp elements; boxes of rg images x rg_pc columns
        const uint64_t eb = uint64_t(elem_bytes(dt));
        const int xr = int(g.FH) + g.sh * (rc.q - 1);
        const int64_t OH = axis_h(g).O, OW = axis_w(g).O;
        bool ok = rc.cls.size() <= size_t(kRowWgradRgClasses);
        for (size_t k = 0; ok && k < rc.cls.size(); ++k) {
            const RowClassH& c = rc.cls[k];
            const uint64_t xs = c.ncols > 1 ? uint64_t(c.cstep) * g.sw * g.C * eb : 16;
            const uint64_t ys = c.ncols > 1 ? uint64_t(c.cstep) * OCp * eb : 16;
            uint64_t dx[4] = {uint64_t(g.W * g.C), uint64_t(g.N), uint64_t(c.ncols), uint64_t(g.H)};
            uint64_t sx[3] = {uint64_t(g.H * g.W * g.C) * eb, xs, uint64_t(g.W * g.C) * eb};
            uint32_t bx[4] = {uint32_t(rc.JB), uint32_t(rc.rg), uint32_t(rc.rg_pc), uint32_t(xr)};
            // dY columns of class k start at output column col0 (the class map's base is shifted there)
            const void* ybase = static_cast<const uint8_t*>(dys) + int64_t(c.col0) * OCp * int64_t(eb);
            uint64_t dy[4] = {uint64_t(OCp), uint64_t(g.N), uint64_t(c.ncols), uint64_t(OH)};
            uint64_t sy[3] = {uint64_t(OH * OW * OCp) * eb, ys, uint64_t(OW * OCp) * eb};
            uint32_t by[4] = {uint32_t(128 / eb), uint32_t(rc.rg), uint32_t(rc.rg_pc), 1};
            ok = xs % 16 == 0 && ys % 16 == 0 && make_tmap4(&xm.x[k], dt, x, dx, sx, bx, int(rc.JB * eb), tf) &&
                 make_tmap4(&xm.dy[k], dt, ybase, dy, sy, by, 128, tf);
        }
        if (!ok) rc = row_cfg_wgrad(g, dt, rc.gz, kPlanSMs, false);  // same partial count: 64-image k-blocks
    }
    CUtensorMap tx;
    const int xrows = int(g.FH) + g.sh * (rc.q - 1);  // one X box serves q output rows
    if (!make_row_xmap(&tx, x, g, dt, uint32_t(rc.JB), 64, uint32_t(xrows), tf)) return CKS_ERR_CUDA;
    RowWgradParams q;
    memset(&q, 0, sizeof(q));
    if (rc.rg) {
        q.rg = rc.rg;
        q.rg_pk = rc.rg_pc;
    }
    q.out = wout;
    q.part_stride = part_stride;
    q.N = int(g.N), q.H = int(g.H), q.W = int(g.W), q.C = int(g.C), q.OC = int(g.OC);
    q.FH = int(g.FH), q.FW = int(g.FW), q.sh = g.sh, q.sw = g.sw, q.ph = g.ph, q.pw = g.pw;
    q.OH = int(axis_h(g).O), q.OW = int(axis_w(g).O);
    q.mb = rc.mb;
    q.nbs = rc.nbs;
    q.ncls = int(rc.cls.size());
    fill_row_classes(q.cls, rc.cls);
    q.gz = rc.gz;
    q.nblk64 = rc.nblk;
    q.num_tiles = int(rc.tiles);
    q.stages = rc.stages;
    q.q = rc.q;
    q.xrows = xrows;
    q.a_bytes = ((rc.q - 1) * g.sh + rc.mb * (128 / rc.JB)) * 64 * rc.ROWB;
    if (tf) return rc.ROWB == 128 ? launch_wgrad_row_rb<128, true>(rc.BN, tx, tdy, q, xm, rc.smem, st) : CKS_ERR_UNSUPPORTED;
    switch (rc.ROWB) {
        case 32: return launch_wgrad_row_rb<32, false>(rc.BN, tx, tdy, q, xm, rc.smem, st);
        case 64: return launch_wgrad_row_rb<64, false>(rc.BN, tx, tdy, q, xm, rc.smem, st);
        case 128: return launch_wgrad_row_rb<128, false>(rc.BN, tx, tdy, q, xm, rc.smem, st);
    }
    return CKS_ERR_UNSUPPORTED;
}

// Staggered filter-row groups (experiments: CKS_WGRAD_STAGGER=0/1)
bool wgrad_stagger() {
    static const bool on = [] {
        const char* e = cks_knob("CKS_WGRAD_STAGGER");
        return e ? atoi(e) != 0 : false;
    }();
    return on;
}

// per-tap Sk-dilated-V2 kernel (KB-WGRAD)
cks_status run_wgrad_taps(const cks_geom& g, cks_dtype dt, const WgradCfg& cfg, const Axis& ah, const Axis& aw,
                          const CUtensorMap& ta, const CUtensorMap& tb, float* wout, long long part_stride,
                          cudaStream_t st, const Axis* ad = nullptr) {
    WgradParams p;
    memset(&p, 0, sizeof(p));
    auto th = table_t3(ah), tw = table_t3(aw);
    if (th.size() > 32 || tw.size() > 32) return CKS_ERR_UNSUPPORTED;
    if (ad) {  // 3-D: T3 of the depth axis
        auto td = table_t3(*ad);
        if (td.size() > 32) return CKS_ERR_UNSUPPORTED;
        for (size_t i = 0; i < td.size(); ++i) {
            p.od_s[i] = int16_t(td[i].oh_s);
            p.od_e[i] = int16_t(td[i].oh_e);
        }
        p.FD = int(ad->F);
        p.sd = int(ad->s);
        p.pd = int(ad->p);
    } else {
        p.od_s[0] = 0;
        p.od_e[0] = 1;
        p.FD = 1;
        p.sd = 1;
        p.pd = 0;
    }
    p.OHr = int(ah.O);
    p.Hr = int(ah.I);
    for (size_t i = 0; i < th.size(); ++i) {
        p.oh_s[i] = int16_t(th[i].oh_s);
        p.oh_e[i] = int16_t(th[i].oh_e);
    }
    for (size_t i = 0; i < tw.size(); ++i) {
        p.ow_s[i] = int16_t(tw[i].oh_s);
        p.ow_e[i] = int16_t(tw[i].oh_e);
    }
    p.out = wout;
    p.FH = int(g.FH);
    p.FW = int(g.FW);
    p.sh = g.sh;
    p.sw = g.sw;
    p.ph = g.ph;
    p.pw = g.pw;
    p.N = int(g.N);
    p.OC = int(g.OC);
    p.C = int(g.C);
    p.mblocks = cfg.mblocks;
    p.nbs = cfg.nbs;
    p.gz = cfg.gz;
    p.nblk64 = cfg.nblk64;
    p.num_tiles = cfg.base_tiles * cfg.gz;
    p.part_stride = part_stride;
    p.zc = cfg.zc;
    p.tc = cfg.tc;
    p.tcmc = cfg.tcmc;
    p.pp = cfg.pp;
    p.rg = cfg.rg;
    p.rg_pk = cfg.rg ? cfg.rg_pk : 1;
    p.stag = (cfg.tc > 1 && g.sh == 1 && !ad && wgrad_stagger()) ? 1 : 0;
    p.Wx = int(g.W);
    p.ouh_s = 1 << 20;
    p.ouh_e = -(1 << 20);
    for (auto& a : th)
        if (a.oh_e > a.oh_s) {
            p.ouh_s = std::min<int>(p.ouh_s, int(a.oh_s));
            p.ouh_e = std::max<int>(p.ouh_e, int(a.oh_e));
        }
    if (p.ouh_e < p.ouh_s) p.ouh_e = p.ouh_s = 0;
    p.ouw_s = 1 << 20;
    p.ouw_e = -(1 << 20);
    for (auto& b : tw)
        if (b.oh_e > b.oh_s) {
            p.ouw_s = std::min<int>(p.ouw_s, int(b.oh_s));
            p.ouw_e = std::max<int>(p.ouw_e, int(b.oh_e));
        }
    if (p.ouw_e < p.ouw_s) p.ouw_e = p.ouw_s = 0;
    const bool tf = dt == CKS_TF32;
    const bool k128 = cfg.kimg == 128;
    if (cfg.pp && cfg.BN == 64) {  // position pairs: two positions' dY on M, four X columns per k-block
        if (tf) return k128 ? launch_wgrad_t<64, true, 128, 4, true, true>(ta, tb, p, st)
                            : launch_wgrad_t<64, true, 64, 4, true, true>(ta, tb, p, st);
        return k128 ? launch_wgrad_t<64, false, 128, 4, true, true>(ta, tb, p, st)
                    : launch_wgrad_t<64, false, 64, 4, true, true>(ta, tb, p, st);
    }
    if (cfg.a1 && !tf && cfg.BN == 64) {  // O_C <= 64: one dY atom per stage
        if (cfg.mt == 3)
            return k128 ? launch_wgrad_t<64, false, 128, 3, true>(ta, tb, p, st)
                        : launch_wgrad_t<64, false, 64, 3, true>(ta, tb, p, st);
        return k128 ? launch_wgrad_t<64, false, 128, 1, true>(ta, tb, p, st)
                    : launch_wgrad_t<64, false, 64, 1, true>(ta, tb, p, st);
    }
    if (cfg.a1 && tf && cfg.BN == 64) {  // TF32, O_C <= 64: two dY atoms per stage
        if (cfg.mt == 3) return launch_wgrad_t<64, true, 64, 3, true>(ta, tb, p, st);
        return k128 ? launch_wgrad_t<64, true, 128, 1, true>(ta, tb, p, st)
                    : launch_wgrad_t<64, true, 64, 1, true>(ta, tb, p, st);
    }
    if (cfg.mt == 3 && tf && cfg.BN == 64) return launch_wgrad_t<64, true, 64, 3>(ta, tb, p, st);
    if (cfg.mt == 3 && cfg.BN == 128)  // BN = 128 row tiles (one accumulator buffer)
        return tf ? launch_wgrad_t<128, true, 32, 3>(ta, tb, p, st) : launch_wgrad_t<128, false, 64, 3>(ta, tb, p, st);
    if (cfg.mt == 3 && !tf && cfg.BN == 64)  // row tiles: the F_W = 3 taps of a filter row share the dY block
        return k128 ? launch_wgrad_t<64, false, 128, 3>(ta, tb, p, st) : launch_wgrad_t<64, false, 64, 3>(ta, tb, p, st);
#define CKS_WG(BN_)                                                                                   \
    (tf ? (k128 ? launch_wgrad_t<BN_, true, 128>(ta, tb, p, st) : launch_wgrad_t<BN_, true, 64>(ta, tb, p, st)) \
        : (k128 ? launch_wgrad_t<BN_, false, 128>(ta, tb, p, st) : launch_wgrad_t<BN_, false, 64>(ta, tb, p, st)))
    switch (cfg.BN) {
        case 64: return CKS_WG(64);
        case 128: return CKS_WG(128);
        case 256: return CKS_WG(256);
    }
#undef CKS_WG
    return CKS_ERR_UNSUPPORTED;
}

cks_status check_ws(const WsLayout& L, void* ws, size_t ws_bytes) {
    if (L.total == 0) return CKS_OK;
    if (!ws || ws_bytes < L.total) return CKS_ERR_WORKSPACE;
    if (!aligned16(ws)) return CKS_ERR_ALIGNMENT;
    return CKS_OK;
}


// ---------------------------------------------------------------- KB-ZINS
// The textbook (zero-inserting / zero-padding) formulation of Eqs (1)-(3),
// run on the same tensor-core kernels so the measured difference is the
// structural zeros alone (SURVEY §8(d) "measured time of the zero-inserted
// formulation"): the staged operand holds every zero of the definition and
// the inner call has nothing to trim.
struct ZinsLayout {
    cks_geom inner;   // geometry of the inner C-K-S call on the staged operand
    cks_op inner_op;
    int64_t Hs, Ws, Cs, Hd, Wd, Cd;  // staging: source / destination extents
    int ish, isw, top, left;         // insertion strides and leading zeros
    size_t stage = 0, filt = 0, inner_ws = 0, total = 0, inner_ws_bytes = 0;
};

size_t al256(size_t x) { return (x + 255) / 256 * 256; }
// fused wgrad + all-reduce: this rank's dW follows the wgrad scratch in the workspace
size_t ar_local_offset(const WsLayout& L) { return al256(L.total); }

ZinsLayout zins_layout(const cks_geom& g, cks_dtype dt, cks_op op) {
    ZinsLayout Z;
    const Axis ah = axis_h(g), aw = axis_w(g);
    const int64_t rh = g.H + 2 * g.ph - g.FH - (ah.O - 1) * g.sh;  // output padding r (reading c10)
    const int64_t rw = g.W + 2 * g.pw - g.FW - (aw.O - 1) * g.sw;
    Z.inner = g;
    if (op == CKS_OP_FWD) {  // Eq (1): explicit Xpad, unpadded conv
        Z.Hs = g.H, Z.Ws = g.W, Z.Cs = Z.Cd = g.C;
        Z.ish = Z.isw = 1, Z.top = g.ph, Z.left = g.pw;
        Z.Hd = g.H + 2 * g.ph, Z.Wd = g.W + 2 * g.pw;
        Z.inner.H = Z.Hd, Z.inner.W = Z.Wd, Z.inner.ph = Z.inner.pw = 0;
        Z.inner_op = CKS_OP_FWD;
    } else if (op == CKS_OP_DECONV) {  // Eq (2): zero_insert(dY) padded q / q + r, conv with W^rot180
        const int64_t qh = g.FH - 1 - g.ph, qw = g.FW - 1 - g.pw;
        Z.Hs = ah.O, Z.Ws = aw.O, Z.Cs = g.OC, Z.Cd = pad_ch(g.OC, dt);
        Z.ish = g.sh, Z.isw = g.sw, Z.top = int(qh), Z.left = int(qw);
        Z.Hd = (ah.O - 1) * g.sh + 1 + 2 * qh + rh, Z.Wd = (aw.O - 1) * g.sw + 1 + 2 * qw + rw;
        Z.inner = cks_geom{g.N, Z.Cd, Z.Hd, Z.Wd, g.C, g.FH, g.FW, 1, 1, 0, 0, 1, 1};
        Z.inner_op = CKS_OP_FWD;
    } else {  // Eq (3): the zero-inserted dY (+ r trailing rows) is the filter of a unit-stride conv
        Z.Hs = ah.O, Z.Ws = aw.O, Z.Cs = Z.Cd = g.OC;
        Z.ish = g.sh, Z.isw = g.sw, Z.top = Z.left = 0;
        Z.Hd = (ah.O - 1) * g.sh + 1 + rh, Z.Wd = (aw.O - 1) * g.sw + 1 + rw;
        Z.inner.sh = Z.inner.sw = 1;
        Z.inner_op = CKS_OP_WGRAD;
    }
    const size_t eb = size_t(elem_bytes(dt));
    size_t off = 0;
    Z.stage = off;
    off += al256(size_t(g.N) * Z.Hd * Z.Wd * Z.Cd * eb);
    Z.filt = off;
    if (op == CKS_OP_DECONV) {
        cks_geom g1 = g;
        g1.sh = g1.sw = 1;  // Stage1 with unit stride = rot180 with channels swapped: [IC][FH*FW][OCp] (OHWI)
        off += al256(ks_split_bytes(g1, dt));
    }
    Z.inner_ws = off;
    Z.inner_ws_bytes = validate(&Z.inner) == CKS_OK ? ws_layout(Z.inner, dt, Z.inner_op, 0, false, kPlanSMs).total : 0;
    Z.total = off + Z.inner_ws_bytes;
    return Z;
}

cks_status launch_zero_insert(const ZinsLayout& Z, cks_dtype dt, int64_t N, const void* src, void* dst,
                              cudaStream_t st) {
    const int64_t eb = elem_bytes(dt);
    const long long rows = N * Z.Hd;
    if (rows > 0x7fffffffLL) return CKS_ERR_UNSUPPORTED;
    if ((Z.Cs * eb) % 16 == 0 && (Z.Cd * eb) % 16 == 0) {
        const int v = int(16 / eb);
        return launch_pdl(zero_insert_kernel<uint4>, dim3(unsigned(rows)), dim3(256), 0, st,
                          static_cast<const uint4*>(src), static_cast<uint4*>(dst), int(Z.Hs), int(Z.Ws),
                          int(Z.Cs / v), int(Z.Hd), int(Z.Wd), int(Z.Cd / v), Z.ish, Z.isw, Z.top, Z.left);
    }
    if (dt == CKS_BF16)
        return launch_pdl(zero_insert_kernel<uint16_t>, dim3(unsigned(rows)), dim3(256), 0, st,
                          static_cast<const uint16_t*>(src), static_cast<uint16_t*>(dst), int(Z.Hs), int(Z.Ws),
                          int(Z.Cs), int(Z.Hd), int(Z.Wd), int(Z.Cd), Z.ish, Z.isw, Z.top, Z.left);
    return launch_pdl(zero_insert_kernel<uint32_t>, dim3(unsigned(rows)), dim3(256), 0, st,
                      static_cast<const uint32_t*>(src), static_cast<uint32_t*>(dst), int(Z.Hs), int(Z.Ws),
                      int(Z.Cs), int(Z.Hd), int(Z.Wd), int(Z.Cd), Z.ish, Z.isw, Z.top, Z.left);
}

cks_status zins_prepare(const cks_geom* g, cks_dtype dt, cks_op op, void* ws, size_t ws_bytes, ZinsLayout* Z) {
    cks_status s = validate(g);
    if (s != CKS_OK) return s;
    *Z = zins_layout(*g, dt, op);
    if ((s = validate(&Z->inner)) != CKS_OK) return s;
    if (!ws || ws_bytes < Z->total) return CKS_ERR_WORKSPACE;
    if (!aligned16(ws)) return CKS_ERR_ALIGNMENT;
    return CKS_OK;
}

}  // namespace

// ====================================================================== C ABI
extern "C" {

int cks_version(void) { return 1; }

const char* cks_status_string(cks_status s) {
    switch (s) {
        case CKS_OK: return "ok";
        case CKS_ERR_NULL: return "null pointer argument";
        case CKS_ERR_GEOMETRY: return "geometry error";
        case CKS_ERR_UNSUPPORTED: return "unsupported configuration";
        case CKS_ERR_ALIGNMENT: return "pointer not 16-byte aligned";
        case CKS_ERR_WORKSPACE: return "workspace too small";
        case CKS_ERR_CUDA: return "CUDA error";
        case CKS_ERR_CAPACITY: return "output capacity too small";
    }
    return "unknown status";
}

cks_status cks_output_shape(const cks_geom* g, int64_t* OH, int64_t* OW) {
    if (!g || !OH || !OW) return CKS_ERR_NULL;
    cks_status s = validate(g);
    if (s != CKS_OK && s != CKS_ERR_UNSUPPORTED) return s;
    *OH = axis_h(*g).O;
    *OW = axis_w(*g).O;
    return CKS_OK;
}

cks_status cks_workspace_size(const cks_geom* g, cks_dtype dt, cks_op op, int gz, size_t* bytes) {
    if (!g || !bytes) return CKS_ERR_NULL;
    cks_status s = validate(g);
    if (s != CKS_OK) return s;
    if (int(op) == CKS_OP_WGRAD_AR) {  // wgrad scratch + this rank's dW (segments reduced by KB-REDUCE-AR)
        const WsLayout L = ws_layout(*g, dt, CKS_OP_WGRAD, gz, false, kPlanSMs);
        *bytes = ar_local_offset(L) + size_t(g->OC * g->FH * g->FW * g->C) * 4;
        return CKS_OK;
    }
    if (op < CKS_OP_FWD || op > CKS_OP_WGRAD) return CKS_ERR_UNSUPPORTED;
    *bytes = ws_layout(*g, dt, op, gz, false, kPlanSMs).total;
    return CKS_OK;
}

cks_status cks_choose_gz(const cks_geom* g, cks_dtype dt, int* gz) {
    if (!g || !gz) return CKS_ERR_NULL;
    cks_status s = validate(g);
    if (s != CKS_OK) return s;
    *gz = wgrad_cfg(*g, dt, 0, kPlanSMs).gz;
    return CKS_OK;
}

cks_status cks_ks_split_size(const cks_geom* g, cks_dtype dt, size_t* bytes) {
    if (!g || !bytes) return CKS_ERR_NULL;
    cks_status s = validate(g);
    if (s != CKS_OK) return s;
    *bytes = ks_split_bytes(*g, dt);
    return CKS_OK;
}

cks_status cks_conv2d_fwd(const cks_geom* g, cks_dtype dt, const void* x, const void* w, float* y, void* ws,
                          size_t ws_bytes, void* stream) {
    if (!g || !x || !w || !y) return CKS_ERR_NULL;
    cks_status s = validate(g);
    if (s != CKS_OK) return s;
    if (!aligned16(x) || !aligned16(w) || !aligned16(y)) return CKS_ERR_ALIGNMENT;
    const Axis ah = axis_h(*g), aw = axis_w(*g);
    auto rh = krows_fwd(ah), rw = krows_fwd(aw);
    if (!rows_ok(rh) || !rows_ok(rw)) return CKS_ERR_UNSUPPORTED;
    WsLayout L = ws_layout(*g, dt, CKS_OP_FWD, 0, false, kPlanSMs);
    if ((s = check_ws(L, ws, ws_bytes)) != CKS_OK) return s;
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    const RowCfg rc = row_cfg_fwd(*g, dt);
    if (rc.ok) return run_fwd_row(*g, dt, rc, x, w, y, st);  // narrow channels: filter-row K-blocks
    const int64_t eb = elem_bytes(dt), Cp = pad_ch(g->C, dt);
    const void* xs = x;
    const void* wsrc = w;
    if (Cp != g->C) {
        void* xp = static_cast<uint8_t*>(ws) + L.x_pad;
        void* wp = static_cast<uint8_t*>(ws) + L.w_pad;
        if ((s = launch_pad(dt, x, xp, g->N * g->H * g->W, int(g->C), int(Cp), st)) != CKS_OK) return s;
        if ((s = launch_pad(dt, w, wp, g->OC * g->FH * g->FW, int(g->C), int(Cp), st)) != CKS_OK) return s;
        xs = xp;
        wsrc = wp;
    }
    IgemmCfg cfg = igemm_cfg_fwd(*g, dt, kPlanSMs);
    if (cfg.rg_ni > 0) rh = igemm_rows_fwd(*g, cfg.rg_ni);  // row groups (N <= 64)
    const uint32_t BK = uint32_t(cfg.KB / eb);
    CUtensorMap ta, tb;
    {   // X viewed as (C, N, W, H): one box = apos columns x 128 images, each column a canonical tile;
        // row groups: one column x rg_ni images x rg_ph rows (element stride s_h) = 128 tile rows
        uint64_t d[4] = {uint64_t(Cp), uint64_t(g->N), uint64_t(g->W), uint64_t(g->H)};
        uint64_t sb[3] = {uint64_t(g->H * g->W * Cp * eb), uint64_t(Cp * eb), uint64_t(g->W * Cp * eb)};
        uint32_t box[4] = {BK, 128u / uint32_t(cfg.cm), cfg.cm > 1 ? 1u : uint32_t(cfg.apos), 1};
        uint32_t es[4] = {1, 1, 1, uint32_t(cfg.rg_es)};
        if (cfg.rg_ni > 0) {
            box[1] = uint32_t(cfg.rg_ni);
            box[3] = uint32_t(cfg.rg_ph * cfg.rg_es);
        }
        if (!make_tmap4(&ta, dt, xs, d, sb, box, cfg.KB, false, cfg.rg_ni > 0 ? es : nullptr)) return CKS_ERR_CUDA;
    }
    {   // W viewed as (C, OC, FH*FW, 1): one box = the FW taps of a filter row x BN filters
        uint64_t d[4] = {uint64_t(Cp), uint64_t(g->OC), uint64_t(g->FH * g->FW), 1};
        uint64_t sb[3] = {uint64_t(g->FH * g->FW * Cp * eb), uint64_t(Cp * eb), uint64_t(g->OC * g->FH * g->FW * Cp * eb)};
        uint32_t box[4] = {BK, uint32_t(cfg.BN), uint32_t(g->FW), 1};
        if (!make_tmap4(&tb, dt, wsrc, d, sb, box, cfg.KB)) return CKS_ERR_CUDA;
    }
    return run_igemm(cfg, dt, rh, rw, ta, tb, y, int(ah.O), int(aw.O), int(g->OC), int(g->N), int(g->FW), 1, L, ws,
                     st);
}

cks_status cks_ks_split(const cks_geom* g, cks_dtype dt, const void* w, void* c_packed, void* stream) {
    if (!g || !w || !c_packed) return CKS_ERR_NULL;
    cks_status s = validate(g);
    if (s != CKS_OK) return s;
    if (!aligned16(w) || !aligned16(c_packed)) return CKS_ERR_ALIGNMENT;
    return launch_split(*g, dt, w, c_packed, static_cast<cudaStream_t>(stream));
}

cks_status cks_deconv2d(const cks_geom* g, cks_dtype dt, const void* dy, const void* w, const void* c_packed,
                        float* dx, void* ws, size_t ws_bytes, void* stream) {
    return cks_deconv2d_ex(g, dt, dy, w, c_packed, dx, ws, ws_bytes, stream, CKS_KS_AUTO);
}

cks_status cks_deconv2d_ex(const cks_geom* g, cks_dtype dt, const void* dy, const void* w, const void* c_packed,
                           float* dx, void* ws, size_t ws_bytes, void* stream, cks_ks_mode mode) {
    if (!g || !dy || !dx) return CKS_ERR_NULL;
    if ((w == nullptr) == (c_packed == nullptr)) return CKS_ERR_NULL;
    if (mode != CKS_KS_AUTO && mode != CKS_KS_STAGE1_FREE && mode != CKS_KS_STAGE1 && mode != CKS_KS_MULTIPHASE)
        return CKS_ERR_UNSUPPORTED;
    if (c_packed && (mode == CKS_KS_STAGE1_FREE || mode == CKS_KS_MULTIPHASE)) return CKS_ERR_UNSUPPORTED;
    cks_status s = validate(g);
    if (s != CKS_OK) return s;
    if (!aligned16(dy) || !aligned16(dx) || (w && !aligned16(w)) || (c_packed && !aligned16(c_packed)))
        return CKS_ERR_ALIGNMENT;
    const Axis ah = axis_h(*g), aw = axis_w(*g);
    auto rh = krows_deconv(ah), rw = krows_deconv(aw);
    if (!rows_ok(rh) || !rows_ok(rw)) return CKS_ERR_UNSUPPORTED;
    WsLayout L = ws_layout(*g, dt, CKS_OP_DECONV, 0, c_packed != nullptr, kPlanSMs);
    if ((s = check_ws(L, ws, ws_bytes)) != CKS_OK) return s;
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    if (!c_packed && (mode == CKS_KS_MULTIPHASE || mode == CKS_KS_AUTO)) {
        const MpPlan m = mp_plan(*g, dt);
        if (m.ok) {  // narrow outputs: the phases stacked on N of one unit-stride ConvV2 over dY
            void* wm = static_cast<uint8_t*>(ws) + L.mp_w;
            float* yp = reinterpret_cast<float*>(static_cast<uint8_t*>(ws) + L.mp_y);
            const long long np = (long long)m.NP * m.CH * m.CW * g->OC;
            const unsigned pb = unsigned(std::min<long long>((np + 255) / 256, 1024));
            if (dt == CKS_BF16)
                s = launch_pdl(ks_mp_pack_kernel<uint16_t>, dim3(pb), dim3(256), 0, st,
                               static_cast<const uint16_t*>(w), static_cast<uint16_t*>(wm), int(g->OC), int(g->FH),
                               int(g->FW), int(g->C), int(g->sh), int(g->sw), m.CH, m.CW, m.NP, int(g->OC));
            else
                s = launch_pdl(ks_mp_pack_kernel<uint32_t>, dim3(pb), dim3(256), 0, st,
                               static_cast<const uint32_t*>(w), static_cast<uint32_t*>(wm), int(g->OC), int(g->FH),
                               int(g->FW), int(g->C), int(g->sh), int(g->sw), m.CH, m.CW, m.NP, int(g->OC));
            if (s != CKS_OK) return s;
            s = cks_conv2d_fwd(&m.pg, dt, dy, wm, yp, static_cast<uint8_t*>(ws) + L.mp_inner, L.mp_inner_bytes, stream);
            if (s != CKS_OK) return s;
            MpPhase t;
            memset(&t, 0, sizeof(t));
            for (int i = 0; i < 8; ++i) t.ih_s[i] = m.ih_s[i], t.a_y[i] = m.a_y[i], t.iw_s[i] = m.iw_s[i], t.a_x[i] = m.a_x[i];
            const int64_t MH = out_extent(m.pg.H, m.pg.FH, 1, m.pg.ph), MW = out_extent(m.pg.W, m.pg.FW, 1, m.pg.pw);
            const long long tot = g->N * g->H * g->W * g->C;
            const unsigned sb = unsigned(std::min<long long>((tot + 255) / 256, 148LL * 16));
            return launch_pdl(ks_mp_scatter_kernel, dim3(sb), dim3(256), 0, st, (const float*)yp, dx, (long long)g->N,
                              int(g->H), int(g->W), int(g->C), int(g->sh), int(g->sw), int(MH), int(MW), m.NP, m.ph2,
                              m.pw2, t);
        }
        if (mode == CKS_KS_MULTIPHASE) return CKS_ERR_UNSUPPORTED;
    }
    const int64_t eb = elem_bytes(dt), OCp = pad_ch(g->OC, dt);
    const int64_t OH = ah.O, OW = aw.O;
    const void* dys = dy;
    if (OCp != g->OC) {
        void* p = static_cast<uint8_t*>(ws) + L.dy_pad;
        if ((s = launch_pad(dt, dy, p, g->N * OH * OW, int(g->OC), int(OCp), st)) != CKS_OK) return s;
        dys = p;
    }
    const int64_t CWm0 = cdiv(g->FW, g->sw);
    if (mode == CKS_KS_STAGE1_FREE && !ks_direct_eligible(*g, dt)) return CKS_ERR_UNSUPPORTED;
    if (!c_packed && (mode == CKS_KS_STAGE1_FREE || (mode == CKS_KS_AUTO && ks_direct(*g, dt, kPlanSMs)))) {
        // Stage1-free: B straight from W (OHWI) viewed as (IC, OC, FW, FH); one box = the
        // CW taps fw = x, x+sw, ... (element stride sw) of one filter row, 128 B of IC x BK OC
        IgemmCfg cfg = igemm_cfg_deconv_w(*g, dt, kPlanSMs);
        if (cfg.rg_ni > 0) rh = igemm_rows_deconv(*g, cfg.rg_ni);  // row groups (N <= 64)
        const uint32_t BK = uint32_t(cfg.KB / eb);
        CUtensorMap ta, tb;
        {
            uint64_t d[4] = {uint64_t(OCp), uint64_t(g->N), uint64_t(OW), uint64_t(OH)};
            uint64_t sb[3] = {uint64_t(OH * OW * OCp * eb), uint64_t(OCp * eb), uint64_t(OW * OCp * eb)};
            uint32_t box[4] = {BK, 128u, uint32_t(cfg.apos), 1};
            if (cfg.rg_ni > 0) {  // one column x rg_ni images x rg_ph consecutive dY rows
                box[1] = uint32_t(cfg.rg_ni);
                box[3] = uint32_t(cfg.rg_ph);
            }
            if (!make_tmap4(&ta, dt, dys, d, sb, box, cfg.KB)) return CKS_ERR_CUDA;
        }
        const int64_t atomw = 128 / eb;
        if (cfg.BN > atomw) {  // (IC in atom, OC, IC atom, FW, FH): smem [tap][atom][BK][128 B]
            uint64_t d[5] = {uint64_t(atomw), uint64_t(g->OC), uint64_t(g->C / atomw), uint64_t(g->FW), uint64_t(g->FH)};
            uint64_t sb[4] = {uint64_t(g->FH * g->FW * g->C * eb), 128u, uint64_t(g->C * eb),
                              uint64_t(g->FW * g->C * eb)};
            uint32_t box[5] = {uint32_t(atomw), BK, uint32_t(cfg.BN / atomw), uint32_t(CWm0 * g->sw), 1};
            uint32_t es[5] = {1, 1, 1, uint32_t(g->sw), 1};
            if (g->C % atomw || !make_tmap5(&tb, dt, w, d, sb, box, es)) return CKS_ERR_CUDA;
        } else {
            uint64_t d[4] = {uint64_t(g->C), uint64_t(g->OC), uint64_t(g->FW), uint64_t(g->FH)};
            uint64_t sb[3] = {uint64_t(g->FH * g->FW * g->C * eb), uint64_t(g->C * eb), uint64_t(g->FW * g->C * eb)};
            uint32_t box[4] = {uint32_t(cfg.BN), BK, uint32_t(CWm0 * g->sw), 1};
            uint32_t es[4] = {1, 1, uint32_t(g->sw), 1};
            if (!make_tmap4(&tb, dt, w, d, sb, box, 128, dt == CKS_TF32, es)) return CKS_ERR_CUDA;
        }
        return run_igemm(cfg, dt, rh, rw, ta, tb, dx, int(g->H), int(g->W), int(g->C), int(g->N), int(CWm0), g->sw, L,
                         ws, st, g);
    }
    const void* cp = c_packed;
    if (!cp) {  // Stage1 into the workspace
        void* p = static_cast<uint8_t*>(ws) + L.c_packed;
        if ((s = launch_split(*g, dt, w, p, st)) != CKS_OK) return s;
        cp = p;
    }
    const int64_t CHm = cdiv(g->FH, g->sh), CWm = cdiv(g->FW, g->sw), P = int64_t(g->sh) * g->sw;
    IgemmCfg cfg = igemm_cfg_deconv(*g, dt, kPlanSMs);
    if (cfg.rg_ni > 0) rh = igemm_rows_deconv(*g, cfg.rg_ni);  // row groups (N <= 64)
    const uint32_t BK = uint32_t(cfg.KB / eb);
    CUtensorMap ta, tb;
    {   // dY viewed as (OC, N, OW, OH): one box = apos columns x 128 images (row groups: one
        // column x rg_ni images x rg_ph consecutive dY rows)
        uint64_t d[4] = {uint64_t(OCp), uint64_t(g->N), uint64_t(OW), uint64_t(OH)};
        uint64_t sb[3] = {uint64_t(OH * OW * OCp * eb), uint64_t(OCp * eb), uint64_t(OW * OCp * eb)};
        uint32_t box[4] = {BK, 128u / uint32_t(cfg.cm), cfg.cm > 1 ? 1u : uint32_t(cfg.apos), 1};
        if (cfg.rg_ni > 0) {
            box[1] = uint32_t(cfg.rg_ni);
            box[3] = uint32_t(cfg.rg_ph);
        }
        if (!make_tmap4(&ta, dt, dys, d, sb, box, cfg.KB)) return CKS_ERR_CUDA;
    }
    {   // packed C_{y,x} viewed as (OCp, C, CHm*CWm, P): one box = the CWm taps of sub-filter row ch
        uint64_t d[4] = {uint64_t(OCp), uint64_t(g->C), uint64_t(CHm * CWm), uint64_t(P)};
        uint64_t sb[3] = {uint64_t(CHm * CWm * OCp * eb), uint64_t(OCp * eb), uint64_t(g->C * CHm * CWm * OCp * eb)};
        uint32_t box[4] = {BK, uint32_t(cfg.BN), uint32_t(CWm), 1};
        if (!make_tmap4(&tb, dt, cp, d, sb, box, cfg.KB)) return CKS_ERR_CUDA;
    }
    return run_igemm(cfg, dt, rh, rw, ta, tb, dx, int(g->H), int(g->W), int(g->C), int(g->N), int(CWm), g->sw, L, ws,
                     st);
}

// Sk-dilated (+ G_Z reduce).  ar != nullptr: the fused data-parallel variant --
// the wgrad kernels write G_Z partials (or, for one segment / the in-cluster
// reduce, this rank's dW) into the workspace, and KB-REDUCE-AR aggregates the
// segments AND the ranks into every rank's dW.

static cks_status wgrad_impl(const cks_geom* g, cks_dtype dt, const void* x, const void* dy, float* dw, int gz,
                             void* ws, size_t ws_bytes, void* stream, const cks_ar_group* ar,
                             ArParams* defer = nullptr, long long* defer_blocks = nullptr) {
    if (!g || !x || !dy || !dw) return CKS_ERR_NULL;
    cks_status s = validate(g);
    if (s != CKS_OK) return s;
    if (gz < 0) return CKS_ERR_UNSUPPORTED;
    if (!aligned16(x) || !aligned16(dy) || !aligned16(dw)) return CKS_ERR_ALIGNMENT;
    if (g->OC > 65535 || g->C > 65535) return CKS_ERR_UNSUPPORTED;
    WsLayout L = ws_layout(*g, dt, CKS_OP_WGRAD, gz, false, kPlanSMs);
    const long long n_dw = g->OC * g->FH * g->FW * g->C;
    if (ar) {
        WsLayout La = L;  // + this rank's dW (one segment / in-cluster reduce) after the wgrad scratch
        La.total = ar_local_offset(L) + size_t(n_dw) * 4;
        if ((s = check_ws(La, ws, ws_bytes)) != CKS_OK) return s;
    } else if ((s = check_ws(L, ws, ws_bytes)) != CKS_OK) {
        return s;
    }
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    const Axis ah = axis_h(*g), aw = axis_w(*g);
    const int64_t eb = elem_bytes(dt), Cp = pad_ch(g->C, dt), OCp = pad_ch(g->OC, dt);
    const void* xs = x;
    const void* dys = dy;
    WgradCfg cfg = wgrad_cfg(*g, dt, gz, kPlanSMs);
    if (Cp != g->C && !cfg.row) {
        void* p = static_cast<uint8_t*>(ws) + L.x_pad;
        if ((s = launch_pad(dt, x, p, g->N * g->H * g->W, int(g->C), int(Cp), st)) != CKS_OK) return s;
        xs = p;
    }
    if (OCp != g->OC) {
        void* p = static_cast<uint8_t*>(ws) + L.dy_pad;
        if ((s = launch_pad(dt, dy, p, g->N * ah.O * aw.O, int(g->OC), int(OCp), st)) != CKS_OK) return s;
        dys = p;
    }
    CUtensorMap ta;  // dY viewed as (OC, OW, OH, N): boxes of 128 B of channels x 64 / 128 images
    if (cfg.rg && !cfg.row) {  // row groups: (OC, N, OW, OH), boxes of rg images x rg_pk positions
        uint64_t d[4] = {uint64_t(OCp), uint64_t(g->N), uint64_t(aw.O), uint64_t(ah.O)};
        uint64_t sb[3] = {uint64_t(ah.O * aw.O * OCp * eb), uint64_t(OCp * eb), uint64_t(aw.O * OCp * eb)};
        uint32_t box[4] = {uint32_t(128 / eb), uint32_t(cfg.rg), uint32_t(cfg.rg_pk), 1};
        if (!make_tmap4(&ta, dt, dys, d, sb, box, 128, dt == CKS_TF32)) return CKS_ERR_CUDA;
    } else {
        uint64_t d[4] = {uint64_t(OCp), uint64_t(aw.O), uint64_t(ah.O), uint64_t(g->N)};
        uint64_t sb[3] = {uint64_t(OCp * eb), uint64_t(aw.O * OCp * eb), uint64_t(ah.O * aw.O * OCp * eb)};
        uint32_t box[4] = {uint32_t(128 / eb), 1, 1, uint32_t(cfg.row ? 64 : cfg.kimg)};
        if (!make_tmap4(&ta, dt, dys, d, sb, box, 128, dt == CKS_TF32)) return CKS_ERR_CUDA;
    }
    const bool partials = cfg.npart() > 1 && !cfg.zc;
    float* wout = partials ? reinterpret_cast<float*>(static_cast<uint8_t*>(ws) + L.partial)
                           : (ar ? reinterpret_cast<float*>(static_cast<uint8_t*>(ws) + ar_local_offset(L)) : dw);
    const long long part_stride = g->OC * g->FH * g->FW * g->C;
    if (cfg.row) {  // narrow channels: (fh, fw, c) rows as the GEMM M dimension
        s = run_wgrad_row(*g, dt, row_cfg_wgrad(*g, dt, gz, kPlanSMs), x, dys, OCp, ta, wout, part_stride, st);
    } else {
        CUtensorMap tb;  // X viewed as (C, W, H, N): leaping rows ih = oh*sh + fh - ph
        if (cfg.rg) {  // row groups: (C, N, W, H), rg images x rg_pk leaping columns (element stride s_w)
            uint64_t d[4] = {uint64_t(Cp), uint64_t(g->N), uint64_t(g->W), uint64_t(g->H)};
            uint64_t sb[3] = {uint64_t(g->H * g->W * Cp * eb), uint64_t(Cp * eb), uint64_t(g->W * Cp * eb)};
            uint32_t box[4] = {uint32_t(128 / eb), uint32_t(cfg.rg), uint32_t(cfg.rg_pk * g->sw), 1};
            uint32_t es[4] = {1, 1, uint32_t(g->sw), 1};
            if (!make_tmap4(&tb, dt, xs, d, sb, box, 128, dt == CKS_TF32, es)) return CKS_ERR_CUDA;
        } else {
            uint64_t d[4] = {uint64_t(Cp), uint64_t(g->W), uint64_t(g->H), uint64_t(g->N)};
            uint64_t sb[3] = {uint64_t(Cp * eb), uint64_t(g->W * Cp * eb), uint64_t(g->H * g->W * Cp * eb)};
            uint32_t box[4] = {uint32_t(128 / eb), 1, 1, uint32_t(cfg.kimg)};
            if (!make_tmap4(&tb, dt, xs, d, sb, box, 128, dt == CKS_TF32)) return CKS_ERR_CUDA;
        }
        s = run_wgrad_taps(*g, dt, cfg, ah, aw, ta, tb, wout, part_stride, st);
    }
    if (s != CKS_OK) return s;
    if (ar) {  // KB-REDUCE-AR: segments and ranks in one kernel (fixed order)
        ArParams q;
        memset(&q, 0, sizeof(q));
        q.part = reinterpret_cast<const float4*>(wout);
        q.nv = n_dw / 4;
        q.world = ar->world;
        q.rank = ar->rank;
        q.slice = (q.nv + ar->world - 1) / ar->world;
        q.gz = partials ? cfg.npart() : 1;
        for (int t = 0; t < ar->world; ++t) {
            q.recv[t] = static_cast<float4*>(ar->recv[t]);
            q.out[t] = reinterpret_cast<float4*>(ar->out[t]);
            q.flag[t] = ar->flag[t];
        }
        q.count = ar->count;
        q.err = ar->err;
        const long long need = std::max(q.nv, q.slice);
        const long long cap = ar->ctas > 0 ? ar->ctas : 148;
        const unsigned blocks = unsigned(std::max<long long>(1, std::min<long long>((need + 255) / 256, cap)));
        if (defer) {  // emulated ranks: the caller launches every rank's reduce in one cooperative grid
            *defer = q;
            *defer_blocks = blocks;
            return CKS_OK;
        }
        return launch_pdl(reduce_allreduce_kernel, dim3(blocks), dim3(256), 0, st, q);
    }
    if (cfg.npart() > 1 && !cfg.zc) {  // fixed-order aggregation of the G_Z segments
        const long long n = part_stride;
        const bool v4 = n % 4 == 0;
        const long long nv = v4 ? n / 4 : n;
        const int np = cfg.npart();
        const unsigned G = unsigned(std::min(16, np));
        const unsigned blocks = unsigned(std::min<long long>((nv + 31) / 32, 148LL * 16));
        if (v4)
            return launch_pdl(reduce_partials_kernel<float4>, dim3(blocks), dim3(32, G), 0, st,
                              reinterpret_cast<const float4*>(wout), reinterpret_cast<float4*>(dw), nv, np);
        return launch_pdl(reduce_partials_kernel<float>, dim3(blocks), dim3(32, G), 0, st, (const float*)wout, dw, nv,
                          np);
    }
    return CKS_OK;
}

cks_status cks_dilated_wgrad(const cks_geom* g, cks_dtype dt, const void* x, const void* dy, float* dw, int gz,
                             void* ws, size_t ws_bytes, void* stream) {
    return wgrad_impl(g, dt, x, dy, dw, gz, ws, ws_bytes, stream, nullptr);
}

// ------------------------------------------------------------------ 3-D C-K-S
cks_status cks_output_shape3(const cks_geom3* g, int64_t* OD, int64_t* OH, int64_t* OW) {
    if (!g || !OD || !OH || !OW) return CKS_ERR_NULL;
    cks_status s = validate3(g);
    if (s != CKS_OK) return s;
    const cks_geom g2 = plane_geom(*g);
    *OD = axis_d(*g).O;
    *OH = axis_h(g2).O;
    *OW = axis_w(g2).O;
    return CKS_OK;
}

cks_status cks_workspace_size3(const cks_geom3* g, cks_dtype dt, cks_op op, int gz, size_t* bytes) {
    if (!g || !bytes) return CKS_ERR_NULL;
    cks_status s = validate3(g);
    if (s != CKS_OK) return s;
    if (op < CKS_OP_FWD || op > CKS_OP_WGRAD) return CKS_ERR_UNSUPPORTED;
    *bytes = ws_layout3(*g, dt, op, gz, kPlanSMs).total;
    return CKS_OK;
}

cks_status cks_op_counts3(const cks_geom3* g, int64_t out[4]) {
    if (!g || !out) return CKS_ERR_NULL;
    cks_status s = validate3(g);
    if (s != CKS_OK) return s;
    const cks_geom g2 = plane_geom(*g);
    const int64_t vd = axis_valid_pairs(axis_d(*g)), vh = axis_valid_pairs(axis_h(g2)),
                  vw = axis_valid_pairs(axis_w(g2));
    out[0] = g->N * g->C * g->OC * vd * vh * vw;
    out[1] = vd;
    out[2] = vh;
    out[3] = vw;
    return CKS_OK;
}

cks_status cks_conv3d_fwd(const cks_geom3* g, cks_dtype dt, const void* x, const void* w, float* y, void* ws,
                          size_t ws_bytes, void* stream) {
    if (!g || !x || !w || !y) return CKS_ERR_NULL;
    cks_status s = validate3(g);
    if (s != CKS_OK) return s;
    if (!aligned16(x) || !aligned16(w) || !aligned16(y)) return CKS_ERR_ALIGNMENT;
    const cks_geom g2 = plane_geom(*g);
    const Axis ad = axis_d(*g), ah = axis_h(g2), aw = axis_w(g2);
    Depth3 d3;
    d3.rd = krows_fwd(ad);
    auto rh = krows_fwd(ah), rw = krows_fwd(aw);
    if (!rows_ok(rh) || !rows_ok(rw) || !rows_ok(d3.rd)) return CKS_ERR_UNSUPPORTED;
    WsLayout L = ws_layout3(*g, dt, CKS_OP_FWD, 0, kPlanSMs);
    if ((s = check_ws(L, ws, ws_bytes)) != CKS_OK) return s;
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    const int64_t eb = elem_bytes(dt), Cp = pad_ch(g->C, dt);
    const void* xs = x;
    const void* wsrc = w;
    if (Cp != g->C) {
        void* xp = static_cast<uint8_t*>(ws) + L.x_pad;
        void* wp = static_cast<uint8_t*>(ws) + L.w_pad;
        if ((s = launch_pad(dt, x, xp, g->N * g->D * g->H * g->W, int(g->C), int(Cp), st)) != CKS_OK) return s;
        if ((s = launch_pad(dt, w, wp, g->OC * g->FD * g->FH * g->FW, int(g->C), int(Cp), st)) != CKS_OK) return s;
        xs = xp;
        wsrc = wp;
    }
    IgemmCfg cfg = igemm_cfg_fwd3(*g, dt, kPlanSMs);
    if (cfg.rg_ni > 0) rh = igemm_rows_fwd(g2, cfg.rg_ni);  // row groups (N <= 64) inside a depth slice
    const uint32_t BK = uint32_t(cfg.KB / eb);
    CUtensorMap ta, tb;
    {   // X viewed as (C, N, W, D*H): depth and row flattened (a row step never crosses a depth slice;
        // row groups: rg_ph rows of one slice at element stride s_h, trailing box rows never stored)
        uint64_t d[4] = {uint64_t(Cp), uint64_t(g->N), uint64_t(g->W), uint64_t(g->D * g->H)};
        uint64_t sb[3] = {uint64_t(g->D * g->H * g->W * Cp * eb), uint64_t(Cp * eb), uint64_t(g->W * Cp * eb)};
        uint32_t box[4] = {BK, 128u, uint32_t(cfg.apos), 1};
        uint32_t es[4] = {1, 1, 1, uint32_t(cfg.rg_es)};
        if (cfg.rg_ni > 0) {
            box[1] = uint32_t(cfg.rg_ni);
            box[3] = uint32_t(cfg.rg_ph * cfg.rg_es);
        }
        if (!make_tmap4(&ta, dt, xs, d, sb, box, cfg.KB, false, cfg.rg_ni > 0 ? es : nullptr)) return CKS_ERR_CUDA;
    }
    {   // W viewed as (C, OC, FD*FH*FW, 1): one box = the FW taps of filter row (fd, fh)
        uint64_t d[4] = {uint64_t(Cp), uint64_t(g->OC), uint64_t(g->FD * g->FH * g->FW), 1};
        uint64_t sb[3] = {uint64_t(g->FD * g->FH * g->FW * Cp * eb), uint64_t(Cp * eb),
                          uint64_t(g->OC * g->FD * g->FH * g->FW * Cp * eb)};
        uint32_t box[4] = {BK, uint32_t(cfg.BN), uint32_t(g->FW), 1};
        if (!make_tmap4(&tb, dt, wsrc, d, sb, box, cfg.KB)) return CKS_ERR_CUDA;
    }
    d3.a_rows_h = int(g->H);
    d3.out_rows_h = int(ah.O);
    d3.b_rows_h = int(g->FH);
    return run_igemm(cfg, dt, rh, rw, ta, tb, y, int(ad.O * ah.O), int(aw.O), int(g->OC), int(g->N), int(g->FW), 1,
                     L, ws, st, nullptr, &d3);
}

cks_status cks_deconv3d(const cks_geom3* g, cks_dtype dt, const void* dy, const void* w, float* dx, void* ws,
                        size_t ws_bytes, void* stream) {
    if (!g || !dy || !w || !dx) return CKS_ERR_NULL;
    cks_status s = validate3(g);
    if (s != CKS_OK) return s;
    if (!aligned16(dy) || !aligned16(dx) || !aligned16(w)) return CKS_ERR_ALIGNMENT;
    const cks_geom g2 = plane_geom(*g);
    if (!ks_direct_eligible(g2, dt)) return CKS_ERR_UNSUPPORTED;  // Stage1-free only: 16-byte W rows
    const Axis ad = axis_d(*g), ah = axis_h(g2), aw = axis_w(g2);
    Depth3 d3;
    d3.rd = krows_deconv(ad);
    auto rh = krows_deconv(ah), rw = krows_deconv(aw);
    if (!rows_ok(rh) || !rows_ok(rw) || !rows_ok(d3.rd)) return CKS_ERR_UNSUPPORTED;
    WsLayout L = ws_layout3(*g, dt, CKS_OP_DECONV, 0, kPlanSMs);
    if ((s = check_ws(L, ws, ws_bytes)) != CKS_OK) return s;
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    const int64_t eb = elem_bytes(dt), OCp = pad_ch(g->OC, dt);
    const int64_t OD = ad.O, OH = ah.O, OW = aw.O;
    const void* dys = dy;
    if (OCp != g->OC) {
        void* p = static_cast<uint8_t*>(ws) + L.dy_pad;
        if ((s = launch_pad(dt, dy, p, g->N * OD * OH * OW, int(g->OC), int(OCp), st)) != CKS_OK) return s;
        dys = p;
    }
    IgemmCfg cfg = igemm_cfg_deconv3(*g, dt, kPlanSMs);
    if (cfg.rg_ni > 0) rh = igemm_rows_deconv(g2, cfg.rg_ni);  // row groups (N <= 64) inside a depth slice
    const uint32_t BK = uint32_t(cfg.KB / eb);
    const int64_t CWm0 = cdiv(g->FW, g->sw), atomw = 128 / eb;
    CUtensorMap ta, tb;
    {   // dY viewed as (OC, N, OW, OD*OH) (row groups: rg_ph consecutive dY rows of one slice)
        uint64_t d[4] = {uint64_t(OCp), uint64_t(g->N), uint64_t(OW), uint64_t(OD * OH)};
        uint64_t sb[3] = {uint64_t(OD * OH * OW * OCp * eb), uint64_t(OCp * eb), uint64_t(OW * OCp * eb)};
        uint32_t box[4] = {BK, 128u, uint32_t(cfg.apos), 1};
        if (cfg.rg_ni > 0) {
            box[1] = uint32_t(cfg.rg_ni);
            box[3] = uint32_t(cfg.rg_ph);
        }
        if (!make_tmap4(&ta, dt, dys, d, sb, box, cfg.KB)) return CKS_ERR_CUDA;
    }
    // W (OHWI) read directly: filter rows (fd, fh) flattened to FD*FH
    if (cfg.BN > atomw) {
        uint64_t d[5] = {uint64_t(atomw), uint64_t(g->OC), uint64_t(g->C / atomw), uint64_t(g->FW),
                         uint64_t(g->FD * g->FH)};
        uint64_t sb[4] = {uint64_t(g->FD * g->FH * g->FW * g->C * eb), 128u, uint64_t(g->C * eb),
                          uint64_t(g->FW * g->C * eb)};
        uint32_t box[5] = {uint32_t(atomw), BK, uint32_t(cfg.BN / atomw), uint32_t(CWm0 * g->sw), 1};
        uint32_t es[5] = {1, 1, 1, uint32_t(g->sw), 1};
        if (g->C % atomw || !make_tmap5(&tb, dt, w, d, sb, box, es)) return CKS_ERR_CUDA;
    } else {
        uint64_t d[4] = {uint64_t(g->C), uint64_t(g->OC), uint64_t(g->FW), uint64_t(g->FD * g->FH)};
        uint64_t sb[3] = {uint64_t(g->FD * g->FH * g->FW * g->C * eb), uint64_t(g->C * eb),
                          uint64_t(g->FW * g->C * eb)};
        uint32_t box[4] = {uint32_t(cfg.BN), BK, uint32_t(CWm0 * g->sw), 1};
        uint32_t es[4] = {1, 1, uint32_t(g->sw), 1};
        if (!make_tmap4(&tb, dt, w, d, sb, box, 128, dt == CKS_TF32, es)) return CKS_ERR_CUDA;
    }
    d3.a_rows_h = int(OH);
    d3.out_rows_h = int(g->H);
    d3.FD = int(g->FD);
    d3.sd = g->sd;
    return run_igemm(cfg, dt, rh, rw, ta, tb, dx, int(g->D * g->H), int(g->W), int(g->C), int(g->N), int(CWm0), g->sw,
                     L, ws, st, &g2, &d3);
}

cks_status cks_dilated_wgrad3d(const cks_geom3* g, cks_dtype dt, const void* x, const void* dy, float* dw, int gz,
                               void* ws, size_t ws_bytes, void* stream) {
    if (!g || !x || !dy || !dw) return CKS_ERR_NULL;
    cks_status s = validate3(g);
    if (s != CKS_OK) return s;
    if (gz < 0) return CKS_ERR_UNSUPPORTED;
    if (!aligned16(x) || !aligned16(dy) || !aligned16(dw)) return CKS_ERR_ALIGNMENT;
    if (g->OC > 65535 || g->C > 65535) return CKS_ERR_UNSUPPORTED;
    WsLayout L = ws_layout3(*g, dt, CKS_OP_WGRAD, gz, kPlanSMs);
    if ((s = check_ws(L, ws, ws_bytes)) != CKS_OK) return s;
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    const cks_geom g2 = plane_geom(*g);
    const Axis ad = axis_d(*g), ah = axis_h(g2), aw = axis_w(g2);
    const int64_t eb = elem_bytes(dt), Cp = pad_ch(g->C, dt), OCp = pad_ch(g->OC, dt);
    const void* xs = x;
    const void* dys = dy;
    const WgradCfg cfg = wgrad_cfg3(*g, dt, gz, kPlanSMs);
    if (Cp != g->C) {
        void* p = static_cast<uint8_t*>(ws) + L.x_pad;
        if ((s = launch_pad(dt, x, p, g->N * g->D * g->H * g->W, int(g->C), int(Cp), st)) != CKS_OK) return s;
        xs = p;
    }
    if (OCp != g->OC) {
        void* p = static_cast<uint8_t*>(ws) + L.dy_pad;
        if ((s = launch_pad(dt, dy, p, g->N * ad.O * ah.O * aw.O, int(g->OC), int(OCp), st)) != CKS_OK) return s;
        dys = p;
    }
    CUtensorMap ta, tb;
    {   // dY viewed as (OC, OW, OD*OH, N)
        uint64_t d[4] = {uint64_t(OCp), uint64_t(aw.O), uint64_t(ad.O * ah.O), uint64_t(g->N)};
        uint64_t sb[3] = {uint64_t(OCp * eb), uint64_t(aw.O * OCp * eb), uint64_t(ad.O * ah.O * aw.O * OCp * eb)};
        uint32_t box[4] = {uint32_t(128 / eb), 1, 1, uint32_t(cfg.kimg)};
        if (!make_tmap4(&ta, dt, dys, d, sb, box, 128, dt == CKS_TF32)) return CKS_ERR_CUDA;
    }
    {   // X viewed as (C, W, D*H, N): leaping rows (id, ih) flattened
        uint64_t d[4] = {uint64_t(Cp), uint64_t(g->W), uint64_t(g->D * g->H), uint64_t(g->N)};
        uint64_t sb[3] = {uint64_t(Cp * eb), uint64_t(g->W * Cp * eb), uint64_t(g->D * g->H * g->W * Cp * eb)};
        uint32_t box[4] = {uint32_t(128 / eb), 1, 1, uint32_t(cfg.kimg)};
        if (!make_tmap4(&tb, dt, xs, d, sb, box, 128, dt == CKS_TF32)) return CKS_ERR_CUDA;
    }
    const long long part_stride = g->OC * g->FD * g->FH * g->FW * g->C;
    float* wout = (cfg.npart() > 1 && !cfg.zc) ? reinterpret_cast<float*>(static_cast<uint8_t*>(ws) + L.partial) : dw;
    s = run_wgrad_taps(g2, dt, cfg, ah, aw, ta, tb, wout, part_stride, st, &ad);
    if (s != CKS_OK) return s;
    if (cfg.npart() > 1 && !cfg.zc) {  // fixed-order aggregation of the G_Z segments
        const long long n = part_stride;
        const bool v4 = n % 4 == 0;
        const long long nv = v4 ? n / 4 : n;
        const int np = cfg.npart();
        const unsigned G = unsigned(std::min(16, np));
        const unsigned blocks = unsigned(std::min<long long>((nv + 31) / 32, 148LL * 16));
        if (v4)
            return launch_pdl(reduce_partials_kernel<float4>, dim3(blocks), dim3(32, G), 0, st,
                              reinterpret_cast<const float4*>(wout), reinterpret_cast<float4*>(dw), nv, np);
        return launch_pdl(reduce_partials_kernel<float>, dim3(blocks), dim3(32, G), 0, st, (const float*)wout, dw, nv,
                          np);
    }
    return CKS_OK;
}

cks_status cks_ar_recv_bytes(const cks_geom* g, int32_t world, size_t* bytes) {
    if (!g || !bytes) return CKS_ERR_NULL;
    cks_status s = validate(g);
    if (s != CKS_OK) return s;
    if (world < 1 || world > CKS_AR_MAX_RANKS) return CKS_ERR_UNSUPPORTED;
    const long long nv = g->OC * g->FH * g->FW * g->C / 4;
    *bytes = size_t(world) * size_t((nv + world - 1) / world) * 16;
    return CKS_OK;
}

static cks_status ar_check(const cks_geom* g, const float* dw, const cks_ar_group* grp) {
    if (!g || !grp || !grp->count || !grp->err) return CKS_ERR_NULL;
    if (grp->world < 1 || grp->world > CKS_AR_MAX_RANKS || grp->rank < 0 || grp->rank >= grp->world)
        return CKS_ERR_UNSUPPORTED;
    if ((g->OC * g->FH * g->FW * g->C) % 4 != 0) return CKS_ERR_UNSUPPORTED;
    for (int t = 0; t < grp->world; ++t) {
        if (!grp->recv[t] || !grp->out[t] || !grp->flag[t]) return CKS_ERR_NULL;
        if (!aligned16(grp->recv[t]) || !aligned16(grp->out[t])) return CKS_ERR_ALIGNMENT;
    }
    if (grp->out[grp->rank] != dw) return CKS_ERR_UNSUPPORTED;
    return CKS_OK;
}

cks_status cks_dilated_wgrad_allreduce(const cks_geom* g, cks_dtype dt, const void* x, const void* dy, float* dw,
                                       int gz, void* ws, size_t ws_bytes, const cks_ar_group* grp, void* stream) {
    const cks_status s = ar_check(g, dw, grp);
    if (s != CKS_OK) return s;
    return wgrad_impl(g, dt, x, dy, dw, gz, ws, ws_bytes, stream, grp);
}

cks_status cks_dilated_wgrad_allreduce_emulated(int32_t world, const cks_geom* g, cks_dtype dt,
                                                const void* const* x, const void* const* dy, float* const* dw,
                                                int gz, void* const* ws, const size_t* ws_bytes,
                                                const cks_ar_group* grps, void* stream) {
    if (!g || !x || !dy || !dw || !ws || !ws_bytes || !grps) return CKS_ERR_NULL;
    if (world < 1 || world > CKS_AR_MAX_RANKS) return CKS_ERR_UNSUPPORTED;
    ArGroupParams P;
    memset(&P, 0, sizeof(P));
    long long blocks = 1;
    for (int r = 0; r < world; ++r) {
        if (grps[r].world != world || grps[r].rank != r) return CKS_ERR_UNSUPPORTED;
        cks_status s = ar_check(&g[r], dw[r], &grps[r]);
        if (s != CKS_OK) return s;
        long long b = 1;
        s = wgrad_impl(&g[r], dt, x[r], dy[r], dw[r], gz, ws[r], ws_bytes[r], stream, &grps[r], &P.r[r], &b);
        if (s != CKS_OK) return s;
        blocks = std::max(blocks, b);  // every rank's barrier counts gridDim.x CTAs
    }
    // all world x blocks CTAs must be co-resident (they spin at the cross-rank barriers)
    int per_sm = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, reduce_allreduce_emul_kernel, 256, 0) != cudaSuccess)
        return last_cuda();
    const long long resident = (long long)per_sm * device_sms();
    blocks = std::max<long long>(1, std::min<long long>(blocks, resident / world));
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(unsigned(blocks), unsigned(world));
    cfg.blockDim = dim3(256);
    cfg.stream = static_cast<cudaStream_t>(stream);
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeCooperative;
    attr[0].val.cooperative = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    if (cudaLaunchKernelEx(&cfg, reduce_allreduce_emul_kernel, P) != cudaSuccess) return last_cuda();
    return CKS_OK;
}

cks_status cks_ipc_export(const void* ptr, cks_ipc_handle* h) {
    if (!ptr || !h) return CKS_ERR_NULL;
    CUdeviceptr base = 0;
    if (!mem_range(ptr, &base)) return CKS_ERR_CUDA;
    cudaIpcMemHandle_t mh;
    if (cudaIpcGetMemHandle(&mh, reinterpret_cast<void*>(base)) != cudaSuccess) return last_cuda();
    const uint64_t off = uint64_t(reinterpret_cast<CUdeviceptr>(ptr) - base);
    static_assert(sizeof(mh) == 64, "cudaIpcMemHandle_t");
    memcpy(h->bytes, &mh, 64);
    memcpy(h->bytes + 64, &off, 8);
    return CKS_OK;
}

// Imported allocations, by handle: a peer's buffers often live in one
// allocation (the caching allocator's segments), and a handle may be opened
// only once per process -- later imports reuse the mapping (refcounted).
static std::mutex g_ipc_mu;
static std::unordered_map<std::string, std::pair<void*, int>> g_ipc_open;

cks_status cks_ipc_import(const cks_ipc_handle* h, void** ptr) {
    if (!h || !ptr) return CKS_ERR_NULL;
    cudaIpcMemHandle_t mh;
    uint64_t off = 0;
    memcpy(&mh, h->bytes, 64);
    memcpy(&off, h->bytes + 64, 8);
    const std::string key(reinterpret_cast<const char*>(h->bytes), 64);
    std::lock_guard<std::mutex> lk(g_ipc_mu);
    auto it = g_ipc_open.find(key);
    if (it == g_ipc_open.end()) {
        void* base = nullptr;
        if (cudaIpcOpenMemHandle(&base, mh, cudaIpcMemLazyEnablePeerAccess) != cudaSuccess) return last_cuda();
        it = g_ipc_open.emplace(key, std::make_pair(base, 0)).first;
    }
    ++it->second.second;
    *ptr = static_cast<uint8_t*>(it->second.first) + off;
    return CKS_OK;
}

cks_status cks_ipc_close(void* ptr) {
    if (!ptr) return CKS_ERR_NULL;
    CUdeviceptr base = 0;
    if (!mem_range(ptr, &base)) return CKS_ERR_CUDA;
    std::lock_guard<std::mutex> lk(g_ipc_mu);
    for (auto it = g_ipc_open.begin(); it != g_ipc_open.end(); ++it) {
        if (reinterpret_cast<CUdeviceptr>(it->second.first) != base) continue;
        if (--it->second.second > 0) return CKS_OK;
        g_ipc_open.erase(it);
        return cudaIpcCloseMemHandle(reinterpret_cast<void*>(base)) == cudaSuccess ? CKS_OK : last_cuda();
    }
    return CKS_ERR_UNSUPPORTED;  // not an imported pointer
}

cks_status cks_axis_table(int64_t I, int64_t F, int32_t s, int32_t p, int table, int64_t* out, size_t cap,
                          size_t* len) {
    if (!len) return CKS_ERR_NULL;
    if (I < 1 || F < 1 || s < 1 || p < 0 || p >= F || I + 2 * p - F < 0) return CKS_ERR_GEOMETRY;
    Axis a{I, F, s, p, out_extent(I, F, s, p)};
    std::vector<int64_t> v;
    switch (table) {
        case 1:
            for (auto& r : table_t1(a)) v.insert(v.end(), {r.o, r.ih_s, r.f_s, r.f_e});
            break;
        case 2:
            for (auto& ph : table_t2(a)) {
                v.insert(v.end(), {ph.y, ph.CH, ph.oph, ph.ih_s, ph.U, ph.a});
                for (auto& r : ph.rows) v.insert(v.end(), {r.u, r.ih, r.oh_s, r.ch_s, r.ch_e});
            }
            break;
        case 3:
            for (auto& r : table_t3(a)) v.insert(v.end(), {r.f, r.ih_s, r.oh_s, r.oh_e});
            break;
        case 4:
            for (auto& r : table_t4(a)) v.insert(v.end(), {r.o_start, r.o_end, r.f_s, r.f_e});
            break;
        default: return CKS_ERR_UNSUPPORTED;
    }
    *len = v.size();
    if (v.size() > cap) return CKS_ERR_CAPACITY;
    if (!v.empty()) {
        if (!out) return CKS_ERR_NULL;
        memcpy(out, v.data(), v.size() * sizeof(int64_t));
    }
    return CKS_OK;
}

cks_status cks_op_counts(const cks_geom* g, cks_dtype dt, int64_t out[8]) {
    if (!g || !out) return CKS_ERR_NULL;
    cks_status s = validate(g);
    if (s != CKS_OK && s != CKS_ERR_UNSUPPORTED) return s;
    const Axis ah = axis_h(*g), aw = axis_w(*g);
    const int64_t VH = axis_valid_pairs(ah), VW = axis_valid_pairs(aw);
    const int64_t OHp = ah.O + (ah.O - 1) * (g->sh - 1), OWp = aw.O + (aw.O - 1) * (g->sw - 1);
    out[0] = g->N * g->C * g->OC * VH * VW;
    out[1] = VH;
    out[2] = VW;
    out[3] = 2 * (g->OC * g->N * ah.O * aw.O * g->FH * g->FW * g->C);
    out[4] = 2 * (g->C * g->N * g->H * g->W * g->FH * g->FW * g->OC);
    out[5] = 2 * (g->OC * g->FH * g->FW * g->C * OHp * OWp) * g->N;
    IgemmCfg cfg = igemm_cfg_fwd(*g, dt, kPlanSMs);
    const int64_t Cp = pad_ch(g->C, dt), BK = cfg.KB / elem_bytes(dt);
    out[6] = int64_t(cfg.nblk) * 128 * int64_t(cfg.nbs) * cfg.BN * VH * VW * ((Cp + BK - 1) / BK * BK);
    out[7] = cfg.tiles;
    return CKS_OK;
}

cks_status cks_launch_count(const cks_geom* g, cks_dtype dt, cks_op op, int gz, int c_packed_given, int* launches) {
    if (!g || !launches) return CKS_ERR_NULL;
    cks_status s = validate(g);
    if (s != CKS_OK) return s;
    const bool cpad = pad_ch(g->C, dt) != g->C, ocpad = pad_ch(g->OC, dt) != g->OC;
    int n = 1;
    if (op == CKS_OP_FWD) n += (cpad && !row_cfg_fwd(*g, dt).ok) ? 2 : 0;
    else if (op == CKS_OP_DECONV) {
        const MpPlan m = c_packed_given ? MpPlan() : mp_plan(*g, dt);
        if (m.ok) {  // pack + the pseudo ConvV2 + scatter
            int inner = 0;
            const cks_status s2 = cks_launch_count(&m.pg, dt, CKS_OP_FWD, 0, 0, &inner);
            if (s2 != CKS_OK) return s2;
            n = 2 + inner;
        } else {
            n += (c_packed_given || ks_direct(*g, dt, kPlanSMs) ? 0 : 1) + (ocpad ? 1 : 0);
        }
    }
    else if (op == CKS_OP_WGRAD || int(op) == CKS_OP_WGRAD_AR) {
        const WgradCfg c = wgrad_cfg(*g, dt, gz, kPlanSMs);
        // + KB-REDUCE for G_Z partials; the fused variant always ends with KB-REDUCE-AR
        n += (cpad && !c.row ? 1 : 0) + (ocpad ? 1 : 0) +
             (int(op) == CKS_OP_WGRAD_AR ? 1 : (c.npart() > 1 && !c.zc ? 1 : 0));
    }
    else return CKS_ERR_UNSUPPORTED;
    *launches = n;
    return CKS_OK;
}

cks_status cks_plan_describe(const cks_geom* g, cks_dtype dt, cks_op op, int gz, char* buf, size_t cap,
                              size_t* len) {
    if (!g || !len) return CKS_ERR_NULL;
    cks_status s = validate(g);
    if (s != CKS_OK) return s;
    if (op < CKS_OP_FWD || op > CKS_OP_WGRAD) return CKS_ERR_UNSUPPORTED;
    const std::string d = describe_plan(*g, dt, op, gz, kPlanSMs);
    *len = d.size() + 1;
    if (d.size() + 1 > cap) return CKS_ERR_CAPACITY;
    if (!buf) return CKS_ERR_NULL;
    memcpy(buf, d.c_str(), d.size() + 1);
    return CKS_OK;
}

cks_status cks_padding_macs(const cks_geom* g, cks_dtype dt, cks_op op, int64_t* macs) {
    if (!g || !macs) return CKS_ERR_NULL;
    cks_status s = validate(g);
    if (s != CKS_OK) return s;
    if (op < CKS_OP_FWD || op > CKS_OP_WGRAD) return CKS_ERR_UNSUPPORTED;
    int64_t per = 0;  // the igemm / per-tap paths iterate trimmed windows only: 0
    if (op == CKS_OP_FWD) per = std::max<int64_t>(row_fwd_padding_macs(*g, dt), 0);
    if (op == CKS_OP_WGRAD && wgrad_cfg(*g, dt, 0, kPlanSMs).row) per = std::max<int64_t>(row_wgrad_padding_macs(*g, dt), 0);
    *macs = per * g->N;
    return CKS_OK;
}

cks_status cks_zins_workspace_size(const cks_geom* g, cks_dtype dt, cks_op op, size_t* bytes) {
    if (!g || !bytes) return CKS_ERR_NULL;
    cks_status s = validate(g);
    if (s != CKS_OK) return s;
    if (op < CKS_OP_FWD || op > CKS_OP_WGRAD) return CKS_ERR_UNSUPPORTED;
    const ZinsLayout Z = zins_layout(*g, dt, op);
    if ((s = validate(&Z.inner)) != CKS_OK) return s;
    *bytes = Z.total;
    return CKS_OK;
}

cks_status cks_zins_conv2d_fwd(const cks_geom* g, cks_dtype dt, const void* x, const void* w, float* y, void* ws,
                               size_t ws_bytes, void* stream) {
    if (!g || !x || !w || !y || !ws) return CKS_ERR_NULL;
    if (!aligned16(x) || !aligned16(w) || !aligned16(y)) return CKS_ERR_ALIGNMENT;
    ZinsLayout Z;
    cks_status s = zins_prepare(g, dt, CKS_OP_FWD, ws, ws_bytes, &Z);
    if (s != CKS_OK) return s;
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    uint8_t* base = static_cast<uint8_t*>(ws);
    if ((s = launch_zero_insert(Z, dt, g->N, x, base + Z.stage, st)) != CKS_OK) return s;
    return cks_conv2d_fwd(&Z.inner, dt, base + Z.stage, w, y, base + Z.inner_ws, Z.inner_ws_bytes, stream);
}

cks_status cks_zins_deconv2d(const cks_geom* g, cks_dtype dt, const void* dy, const void* w, float* dx, void* ws,
                             size_t ws_bytes, void* stream) {
    if (!g || !dy || !w || !dx || !ws) return CKS_ERR_NULL;
    if (!aligned16(dy) || !aligned16(w) || !aligned16(dx)) return CKS_ERR_ALIGNMENT;
    ZinsLayout Z;
    cks_status s = zins_prepare(g, dt, CKS_OP_DECONV, ws, ws_bytes, &Z);
    if (s != CKS_OK) return s;
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    uint8_t* base = static_cast<uint8_t*>(ws);
    cks_geom g1 = *g;
    g1.sh = g1.sw = 1;
    if ((s = launch_split(g1, dt, w, base + Z.filt, st)) != CKS_OK) return s;  // W^rot180, OHWI with O=IC, I=OCp
    if ((s = launch_zero_insert(Z, dt, g->N, dy, base + Z.stage, st)) != CKS_OK) return s;
    return cks_conv2d_fwd(&Z.inner, dt, base + Z.stage, base + Z.filt, dx, base + Z.inner_ws, Z.inner_ws_bytes,
                          stream);
}

cks_status cks_zins_wgrad(const cks_geom* g, cks_dtype dt, const void* x, const void* dy, float* dw, void* ws,
                          size_t ws_bytes, void* stream) {
    if (!g || !x || !dy || !dw || !ws) return CKS_ERR_NULL;
    if (!aligned16(x) || !aligned16(dy) || !aligned16(dw)) return CKS_ERR_ALIGNMENT;
    ZinsLayout Z;
    cks_status s = zins_prepare(g, dt, CKS_OP_WGRAD, ws, ws_bytes, &Z);
    if (s != CKS_OK) return s;
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    uint8_t* base = static_cast<uint8_t*>(ws);
    if ((s = launch_zero_insert(Z, dt, g->N, dy, base + Z.stage, st)) != CKS_OK) return s;
    return cks_dilated_wgrad(&Z.inner, dt, x, base + Z.stage, dw, 0, base + Z.inner_ws, Z.inner_ws_bytes, stream);
}

}  // extern "C"
