/*
 * cks.h -- C ABI of libcks.so: the C-K-S zero-skipping convolution operators
 * of arXiv 2306.15951 ("Reduce Computational Complexity for Convolutional
 * Layers by Skipping Zeros") on NVIDIA B200 (sm_100a).
 *
 * Citations: P:<line> = the paper text (reference PAPER.md), section/eq/alg.
 *
 * Problem statement (Table I, Eqs (1)-(3) P:134-140):
 *   X  in R^{N x I_H x I_W x I_C}   input feature maps, NHWC (C fastest)
 *   W  in R^{O_C x F_H x F_W x I_C} filters, OHWI
 *   Y  in R^{N x O_H x O_W x O_C}   output feature maps, NHWC
 *   O_H = floor((I_H + 2 ph - F_H)/sh) + 1, O_W likewise.
 *   (1) Y  = conv2D(X, W)              -- ConvV2, filter trimming (Alg. 1)
 *   (2) dX = deconv2D(dY, W^rot180)    -- KS-deconv-V2 (Alg. 2/2B)
 *   (3) dW = dilated_conv2D(X, dY)     -- Sk-dilated-V2 (Alg. 3/3B)
 *
 * Conventions (all entry points):
 *   - Every device buffer is owned by the caller.  The library never
 *     allocates device memory on the compute path; scratch space is queried
 *     with cks_workspace_size() and passed in (ws, ws_bytes).
 *   - Device pointers must be 16-byte aligned; tensors are dense (no strides).
 *   - Calls are asynchronous on `stream` (a cudaStream_t; NULL = legacy
 *     default stream) with no implicit synchronisation.  Outputs are
 *     OVERWRITTEN, never accumulated.  The cross-GPU allreduce of dW is the
 *     caller's job.
 *   - Validation errors are returned synchronously before anything is
 *     launched.  Asynchronous CUDA faults surface at the caller's next
 *     synchronisation (or as CKS_ERR_CUDA from the launch check).
 *   - dtype CKS_BF16: X, W, dY are bfloat16 (raw 16-bit storage); the tensor
 *     cores multiply bf16 and accumulate fp32.  CKS_TF32: X, W, dY are fp32
 *     and multiplied as TF32 (hardware truncation).  Y, dX, dW are always
 *     fp32.  Geometry is (N,C,H,W,OC,FH,FW,sh,sw,ph,pw,dh,dw); dh = dw = 1 is
 *     required (the paper's "dilate" is the conv stride; there is no
 *     forward filter dilation), else CKS_ERR_UNSUPPORTED.
 *   - Validity (reading c16): sh,sw >= 1, 0 <= ph < F_H, 0 <= pw < F_W,
 *     O_H, O_W >= 1, all extents >= 1, else CKS_ERR_GEOMETRY.
 *   - Channel counts whose rows are not a 16-byte multiple (I_C or O_C not a
 *     multiple of 8 for bf16 / 4 for tf32) are staged through zero-padded
 *     copies inside the workspace ("last dimensions ... implicitly
 *     padded"); padded-channel products are not counted as zero-free work.
 *   - Supported extents: every spatial row count used by a kernel (O_H, O_W
 *     for the forward; I_H, I_W for the deconvolution) is <= CKS_MAX_ROWS,
 *     F_H, F_W <= 32, sh, sw <= 8, else CKS_ERR_UNSUPPORTED.
 */
#ifndef CKS_H
#define CKS_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define CKS_MAX_ROWS 256

typedef struct cks_geom {
    int64_t N, C, H, W, OC, FH, FW; /* C = I_C; H, W = I_H, I_W (the X side) */
    int32_t sh, sw, ph, pw, dh, dw;
} cks_geom;

typedef enum { CKS_TF32 = 0, CKS_BF16 = 1 } cks_dtype;

typedef enum {
    CKS_OK = 0,
    CKS_ERR_NULL = 1,        /* a required pointer argument is NULL          */
    CKS_ERR_GEOMETRY = 2,    /* invalid Table-I geometry (see above)         */
    CKS_ERR_UNSUPPORTED = 3, /* valid but outside what this build supports   */
    CKS_ERR_ALIGNMENT = 4,   /* device pointer not 16-byte aligned           */
    CKS_ERR_WORKSPACE = 5,   /* ws too small / NULL while ws bytes needed     */
    CKS_ERR_CUDA = 6,        /* a CUDA runtime/driver call failed            */
    CKS_ERR_CAPACITY = 7     /* host output array too small (tables)          */
} cks_status;

typedef enum { CKS_OP_FWD = 0, CKS_OP_DECONV = 1, CKS_OP_WGRAD = 2 } cks_op;

/* Output extent (Table I shape rule, floor rounding).  Host only. */
cks_status cks_output_shape(const cks_geom* g, int64_t* OH, int64_t* OW);

/* Bytes of scratch the op needs (0 if none).  `gz` is the Sk-dilated G_Z
 * segment count for CKS_OP_WGRAD (0 = the library's choice);
 * ignored for the other ops.  For CKS_OP_DECONV the size assumes the caller
 * passes W (Stage1 runs into the workspace); pass c_packed to skip it. */
cks_status cks_workspace_size(const cks_geom* g, cks_dtype dt, cks_op op, int gz, size_t* bytes);

/* The G_Z the library would use for this geometry with gz = 0 (P:212:
 * "G_Z can be positive related to (N_a + N_b)/N_g ... the upper-bound can be
 * decided by the number of streaming multi-processors").  For narrow-channel
 * layers (the filter-row kernel: FW*C plus its alignment shift fits a 64-
 * element bf16 / 32-element fp32 row, C <= 16 bf16 / 8 fp32, 16-byte X row
 * pitch) the segments are per output-column class (interior columns grouped
 * by box alignment, each border column its own class): the returned G_Z is
 * the total segment count, at least the number of classes; a requested gz is
 * spread over the classes the same way.  Host only. */
cks_status cks_choose_gz(const cks_geom* g, cks_dtype dt, int* gz);

/* Eq (1) via ConvV2 (Alg. 1): Y[n,oh,ow,oc] = sum over the TRIMMED
 * window fh in [fh_s, fh_e), fw in [fw_s, fw_e), ic of
 * X[n, oh*sh-ph+fh, ow*sw-pw+fw, ic] * W[oc,fh,fw,ic]; padded zeros are never
 * loaded or multiplied (the narrow-channel filter-row kernel trims at its
 * 32-byte K-chunk granularity with chunk grids aligned to the image edge:
 * cks_padding_macs reports the products, 0 on every config).
 * x: N*H*W*C (dtype), w: OC*FH*FW*C (dtype), y: N*OH*OW*OC fp32 (overwritten). */
cks_status cks_conv2d_fwd(const cks_geom* g, cks_dtype dt, const void* x, const void* w, float* y,
                          void* ws, size_t ws_bytes, void* stream);

/* Bytes of the packed KS-deconv sub-filter tensor for this geometry. */
cks_status cks_ks_split_size(const cks_geom* g, cks_dtype dt, size_t* bytes);

/* KS-deconv Stage1 (Alg. 2 Stage1 P:443, Fig. 5): rotate W by 180
 * degrees and split it into sh*sw dense sub-filters, one per output phase
 * (y, x): C_{y,x}[oc,ch,cw,ic] = W[oc, y+(oph_y-ch)*sh, x+(opw_x-cw)*sw, ic],
 * oph_y = ceil((F_H-y)/sh)-1.  Stored packed and K-major for the tensor cores:
 * c_packed[p = y*sw+x][ic][ch*CWm + cw][ocp], CHm = ceil(F_H/sh),
 * CWm = ceil(F_W/sw), ocp < OCp = O_C rounded up to 16 bytes; slots outside a
 * phase's CH_y x CW_x extent and channels >= O_C are zero.  Cacheable across
 * calls while W is unchanged. */
cks_status cks_ks_split(const cks_geom* g, cks_dtype dt, const void* w, void* c_packed, void* stream);

/* Eq (2) via KS-deconv-V2 (Alg. 2 Stage2&3 + 2B): per phase (y, x)
 * a unit-stride, filter-trimmed convolution of dY with C_{y,x}, its results
 * scattered to dX rows ih = u*sh + ih_s(y) (fused Stage2&3).  No zero
 * is inserted.  Exactly one of w (then Stage1 runs into ws) or c_packed (from
 * cks_ks_split) must be non-NULL.  dy: N*OH*OW*OC (dtype), dx: N*H*W*C fp32
 * (overwritten; rows no output reaches are written as 0, reading c10/c11). */
cks_status cks_deconv2d(const cks_geom* g, cks_dtype dt, const void* dy, const void* w,
                        const void* c_packed, float* dx, void* ws, size_t ws_bytes, void* stream);

/* cks_deconv2d with an explicit Stage1 choice when w is given (c_packed NULL):
 *   CKS_KS_AUTO          the library's policy (what cks_deconv2d does);
 *   CKS_KS_STAGE1_FREE   no Stage1: the implicit GEMM reads W itself, per
 *                        sub-filter row one TMA box of the taps
 *                        fw = x, x+sw, ... of filter row
 *                        fh = y + (CH_y-1-ch)*sh (the all-in-one variant of
 *                        P:186); requires W rows of a
 *                        16-byte multiple (C*elem % 16 == 0) and sw <= 8, else
 *                        CKS_ERR_UNSUPPORTED;
 *   CKS_KS_STAGE1        Stage1 (cks_ks_split) into ws, then Stage2&3.
 * Same results in every mode (the same sums; only the B operand's source
 * differs).  With c_packed given the mode must be AUTO or STAGE1.  ws as
 * queried by cks_workspace_size(CKS_OP_DECONV) covers every mode. */
/*   CKS_KS_MULTIPHASE    narrow outputs (I_C <= 8, F_H % sh == F_W % sw == 0,
 *                        every phase with >= 1 row): the sh*sw phases are
 *                        stacked on the GEMM N dimension -- with each phase's
 *                        row index shifted by its a_y (T2) all phases read the
 *                        same CH x CW window of dY, so the deconvolution is
 *                        one unit-stride ConvV2 over dY with the stacked
 *                        sub-filters, then a phase-strided scatter to dX
 *                        (CKS_ERR_UNSUPPORTED if not eligible).  AUTO picks it
 *                        where eligible.  At the first / last window row and
 *                        column the GEMM also forms the products of the phases
 *                        whose dX row / column does not exist there; they are
 *                        discarded (never stored). */
typedef enum { CKS_KS_AUTO = 0, CKS_KS_STAGE1_FREE = 1, CKS_KS_STAGE1 = 2, CKS_KS_MULTIPHASE = 3 } cks_ks_mode;
cks_status cks_deconv2d_ex(const cks_geom* g, cks_dtype dt, const void* dy, const void* w,
                           const void* c_packed, float* dx, void* ws, size_t ws_bytes, void* stream,
                           cks_ks_mode mode);

/* Eq (3) via Sk-dilated-V2 (Alg. 3/3B P:445): dW[oc,fh,fw,ic] = sum over
 * n and the TRIMMED (oh, ow) range [oh_s, oh_e) x [ow_s, ow_e) of
 * X[n, oh*sh+fh-ph, ow*sw+fw-pw, ic] * dY[n,oh,ow,oc]: leaping access into X
 * with step = stride, no zero-inserted dY.  The G_K = N*O_H*O_W reduction is
 * split into gz segments computed concurrently and aggregated in a fixed
 * order (map-reduce).  x: N*H*W*C (dtype), dy: N*OH*OW*OC (dtype),
 * dw: OC*FH*FW*C fp32 (overwritten).  gz = 0: library choice. */
cks_status cks_dilated_wgrad(const cks_geom* g, cks_dtype dt, const void* x, const void* dy, float* dw,
                             int gz, void* ws, size_t ws_bytes, void* stream);

/* Per-axis integer tables the kernels consume (host only; bit-exact parity
 * with the oracle's brute-force enumeration).  For one axis (I, F, s, p):
 *   table 1 (T1, ConvV2 trim, Alg. 1): O rows of (o, ih_s, f_s, f_e)
 *   table 2 (T2, KS phases, Alg. 2):   s phase records
 *            (y, CH_y, oph_y, ih_s, U_y, a_y) each followed by U_y rows
 *            (u, ih, oh_s, ch_s, ch_e); empty phases (CH_y = 0) have
 *            a_y = oh_s = ch_s = ch_e = 0, and a_y = 0 when U_y = 0;
 *            an empty trimmed window is written ch_s = ch_e = 0
 *   table 3 (T3, Sk taps, Alg. 3B):   F rows of (f, ih_s, oh_s, oh_e)
 *   table 4 (T4, trim classes):       runs (o_start, o_end, f_s, f_e)
 * flattened into `out` (int64).  *len receives the element count; if it
 * exceeds cap, nothing is written and CKS_ERR_CAPACITY is returned. */
cks_status cks_axis_table(int64_t I, int64_t F, int32_t s, int32_t p, int table,
                          int64_t* out, size_t cap, size_t* len);

/* Operation counts (host only), out[0..7]:
 *   0 zero-free MACs N*I_C*O_C*V_H*V_W (identical for all three operators)
 *   1 V_H, 2 V_W (valid (o, f) pairs per axis)
 *   3 T_Conv, 4 T_Deconv, 5 T_Dilated (with N, reading c9) -- Table III
 *     nominal FLOPs
 *   6 MACs issued by the forward kernel incl. padded channels
 *   7 number of tensor-core tiles of the forward kernel */
cks_status cks_op_counts(const cks_geom* g, cks_dtype dt, int64_t out[8]);

/* Number of kernel launches the op issues for this geometry/options (for
 * the bench's gpu_launches claim).  c_packed_given: deconv skips Stage1. */
cks_status cks_launch_count(const cks_geom* g, cks_dtype dt, cks_op op, int gz, int c_packed_given,
                            int* launches);

/* Text description of the plan the library uses for (g, dt, op, gz): the
 * kernel kind ("igemm", "row_fwd", "wgrad", "row_wgrad") followed by its tile
 * configuration as space-separated key=value pairs (host only; for tests and
 * tools).  *len receives strlen + 1; if it exceeds cap, nothing is written
 * and CKS_ERR_CAPACITY is returned. */
cks_status cks_plan_describe(const cks_geom* g, cks_dtype dt, cks_op op, int gz, char* buf, size_t cap,
                             size_t* len);

/* Multiply-accumulates the op's kernels spend on SPATIAL-PADDING zeros for the
 * whole batch (host only; accounting next to cks_op_counts, Table III).  0
 * for the trimmed-window kernels (every ConvV2 / KS-deconv / Sk-dilated tile
 * iterates its valid window only, Alg. 1-3B).  The narrow-channel row kernels
 * trim at the granularity of their tensor-core operands: ConvV2 loads only
 * valid filter rows and issues only the 32-byte K chunks that hold valid
 * elements, with the chunk grid of a border column aligned to the image edge,
 * so its count is 0 unless a window overhangs both ends of the row;
 * Sk-dilated multiplies the zero-filled rows / border elements inside an
 * issued 128-row M-block (M-blocks entirely outside X are skipped). */
cks_status cks_padding_macs(const cks_geom* g, cks_dtype dt, cks_op op, int64_t* macs);

/* ------------------------------------------------------------ KB-ZINS
 * The formulation C-K-S removes, for measurement ("measured
 * time of the zero-inserted formulation vs C-K-S"): each call materialises the
 * operand of the textbook definition with all its structural zeros in the
 * workspace and runs the same tensor-core kernels on it, which then have no
 * zero to skip.  Results equal the C-K-S entry points (same sums, the extra
 * terms are exact zeros); only the time differs.
 *   cks_zins_conv2d_fwd  Eq (1) on Xpad = X zero-padded by (ph, pw) (Fig. 1
 *                        P:47), convolved with stride (sh, sw) and no padding.
 *   cks_zins_deconv2d    Eq (2) as P:114 states it: Z = dY with (sh-1, sw-1)
 *                        zeros inserted between elements, padded by
 *                        q = F-1-p before and q + r after (r = (I+2p-F) mod s,
 *                        reading c10), convolved with stride 1 by W^rot180
 *                        with I_C / O_C swapped (built by Stage1 at unit
 *                        stride into the workspace).
 *   cks_zins_wgrad       Eq (3): the zero-inserted dY (+ r trailing
 *                        rows / columns) is the filter of a unit-stride
 *                        convolution over X padded by (ph, pw).
 * Arguments, layouts, dtypes and errors as for the C-K-S entry point of the
 * same operator; ws must hold cks_zins_workspace_size(op) bytes (staged
 * operand + rotated filter + the inner call's workspace) and is required.
 * Errors of the inner geometry (e.g. a staged extent > CKS_MAX_ROWS rows)
 * are returned as for the inner call. */
cks_status cks_zins_workspace_size(const cks_geom* g, cks_dtype dt, cks_op op, size_t* bytes);
cks_status cks_zins_conv2d_fwd(const cks_geom* g, cks_dtype dt, const void* x, const void* w, float* y,
                               void* ws, size_t ws_bytes, void* stream);
cks_status cks_zins_deconv2d(const cks_geom* g, cks_dtype dt, const void* dy, const void* w, float* dx,
                             void* ws, size_t ws_bytes, void* stream);
cks_status cks_zins_wgrad(const cks_geom* g, cks_dtype dt, const void* x, const void* dy, float* dw,
                          void* ws, size_t ws_bytes, void* stream);

/* ------------------------------------------------------------ 3-D C-K-S
 * The paper's operators with a depth axis ("stride^N and dilate^N times
 * acceleration for N-dimensional deconvolution and dilated-convolution",
 * P:407 "higher-dimensional versions ... analogized to its 2D counterpart";
 * SURVEY §8(f) NEXT #3; reading c17): trimmed windows on all three axes
 * (ConvV2), sd*sh*sw sub-filters (KS-deconv, Stage1-free: W is read directly),
 * leaping access on all three axes (Sk-dilated).  Layouts: X [N][D][H][W][C],
 * W [OC][FD][FH][FW][C], Y / dY [N][OD][OH][OW][OC], outputs fp32, overwritten.
 * Validity as in 2-D per axis (O >= 1, p < F); FD, FH, FW <= 32, strides <= 8;
 * OD*OH and D*H <= CKS_MAX_ROWS * 256.  KS-deconv needs W rows of a 16-byte
 * multiple (C * elem % 16 == 0), else CKS_ERR_UNSUPPORTED.  Workspace:
 * cks_workspace_size3 for the op (G_Z partials, channel padding). */
typedef struct cks_geom3 {
    int64_t N, C, D, H, W, OC, FD, FH, FW;
    int32_t sd, sh, sw, pd, ph, pw;
} cks_geom3;
cks_status cks_output_shape3(const cks_geom3* g, int64_t* OD, int64_t* OH, int64_t* OW);
cks_status cks_workspace_size3(const cks_geom3* g, cks_dtype dt, cks_op op, int gz, size_t* bytes);
/* zero-free MACs N*C*OC*V_D*V_H*V_W (out[0]) and the per-axis V (out[1..3]) */
cks_status cks_op_counts3(const cks_geom3* g, int64_t out[4]);
cks_status cks_conv3d_fwd(const cks_geom3* g, cks_dtype dt, const void* x, const void* w, float* y, void* ws,
                          size_t ws_bytes, void* stream);
cks_status cks_deconv3d(const cks_geom3* g, cks_dtype dt, const void* dy, const void* w, float* dx, void* ws,
                        size_t ws_bytes, void* stream);
cks_status cks_dilated_wgrad3d(const cks_geom3* g, cks_dtype dt, const void* x, const void* dy, float* dw, int gz,
                               void* ws, size_t ws_bytes, void* stream);

/* ------------------------------------------------- fused wgrad + all-reduce
 * Sk-dilated on this rank's batch shard followed by ONE kernel (KB-REDUCE-AR)
 * that performs the G_Z aggregation AND the sum over the ranks of the
 * data-parallel group through peer memory (NVLink P2P stores): the batch
 * shard is the outermost segment of the paper's map-reduce over
 * G_K = N*O_H*O_W.  Element i of dW is owned by rank
 * i / slice (slice = ceil(n/4 / world) float4 vectors, n = OC*FH*FW*C):
 * every rank pushes its aggregated partial of i to the owner's receive
 * buffer, the owner sums the ranks' contributions in fixed order
 * q = 0..world-1 and stores the result into every rank's dW.  Results are
 * bit-identical on every rank and every run.
 *
 * cks_ar_group (all device pointers are valid in the CALLING process: peers'
 * buffers mapped with cks_ipc_import, or plain pointers when every "rank" is
 * on this device, e.g. tests):
 *   recv[t]   rank t's receive buffer, cks_ar_recv_bytes() bytes;
 *   out[t]    rank t's dW (out[rank] must equal dw);
 *   flag[t]   rank t's two signal words (zeroed once; they count up);
 *   count     this rank's three words: two CTA arrival counters and the
 *             call sequence number (zeroed once; kept on the device, so a
 *             CUDA graph that replays the call stays in step);
 *   err       set to 1 (never cleared by the library) if a peer's signal did
 *             not arrive within a bounded wait -- the kernel then finishes
 *             (no hang) and dW is invalid.
 * One (flag, count) set per call site: calls sharing them must be issued in
 * the same order on every rank.
 * Requires world <= CKS_AR_MAX_RANKS, n % 4 == 0.  ws: cks_workspace_size
 * with op CKS_OP_WGRAD_AR.  Every rank must make the call (same geometry);
 * the call returns once the kernels are queued. */
#define CKS_AR_MAX_RANKS 8
#define CKS_OP_WGRAD_AR 3
typedef struct cks_ar_group {
    int32_t world, rank;
    int32_t ctas;  /* KB-REDUCE-AR grid cap (0: library choice); every CTA may spin at the barriers */
    void* recv[CKS_AR_MAX_RANKS];
    float* out[CKS_AR_MAX_RANKS];
    uint32_t* flag[CKS_AR_MAX_RANKS];
    uint32_t* count;
    int32_t* err;
} cks_ar_group;
cks_status cks_ar_recv_bytes(const cks_geom* g, int32_t world, size_t* bytes);
cks_status cks_dilated_wgrad_allreduce(const cks_geom* g, cks_dtype dt, const void* x, const void* dy, float* dw,
                                       int gz, void* ws, size_t ws_bytes, const cks_ar_group* grp, void* stream);

/* cks_dilated_wgrad_allreduce_emulated -- the same operation for `world`
 * ranks that share ONE GPU (tests; any setup with fewer GPUs than ranks).
 * Per-rank arrays of length world: g[r] (the rank's batch shard), x[r],
 * dy[r], dw[r], ws[r] / ws_bytes[r] (cks_workspace_size, CKS_OP_WGRAD_AR),
 * grps[r] (world = world, rank = r; every pointer valid in this process --
 * peers' buffers imported with cks_ipc_import or local).  Every rank's
 * Sk-dilated is queued on `stream`, then ONE cooperative KB-REDUCE-AR launch
 * covers all ranks (grid.y = rank): the CTAs that spin at the cross-rank
 * barriers are co-resident with the CTAs they wait for.  Separate launches
 * (streams, threads or processes) that wait on one another are not
 * guaranteed to run concurrently on one GPU, so the single-rank entry point
 * above must only be used with one rank per GPU.  Results are bit-identical
 * to the one-rank-per-GPU form (same kernels, same fixed order). */
cks_status cks_dilated_wgrad_allreduce_emulated(int32_t world, const cks_geom* g, cks_dtype dt,
                                                const void* const* x, const void* const* dy, float* const* dw,
                                                int gz, void* const* ws, const size_t* ws_bytes,
                                                const cks_ar_group* grps, void* stream);

/* CUDA IPC for the group's buffers (setup, not the hot path): export a
 * device pointer of this process as an opaque 72-byte handle (64-byte
 * cudaIpcMemHandle_t + 8-byte offset of ptr inside its allocation), import a
 * peer process's handle as a pointer valid here (peer access enabled), and
 * release it. */
typedef struct cks_ipc_handle { unsigned char bytes[72]; } cks_ipc_handle;
cks_status cks_ipc_export(const void* ptr, cks_ipc_handle* h);
cks_status cks_ipc_import(const cks_ipc_handle* h, void** ptr);
cks_status cks_ipc_close(void* ptr);

const char* cks_status_string(cks_status s);
int cks_version(void);

#ifdef __cplusplus
}
#endif
#endif /* CKS_H */
