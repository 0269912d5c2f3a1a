// tma_bench.cu -- TMA ingress microbenchmark (bytes/clk/SM) on B200.
// Each CTA (1 per SM) streams boxes of R rows x 128 B into a ring of S slots
// with `nw` issuing warps; no compute.  Pattern 0: rows = images of an NHWC
// tensor (row stride = H*W*C*2, our A operand); pattern 1: contiguous rows
// (row stride 128 B, a plain K-major GEMM tile).
// build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tma_bench tools/tma_bench.cu -lcuda
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
#include <vector>

__device__ __forceinline__ uint32_t su(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t c) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su(b)), "r"(c) : "memory");
}
__device__ __forceinline__ void expect(uint64_t* b, uint32_t n) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su(b)), "r"(n) : "memory");
}
__device__ __forceinline__ void waitp(uint64_t* b, uint32_t ph) {
    uint32_t ok = 0;
    while (!ok)
        asm volatile("{.reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0,1,0,p;}"
                     : "=r"(ok) : "r"(su(b)), "r"(ph) : "memory");
}
__device__ __forceinline__ void tma4(void* dst, const CUtensorMap* m, uint64_t* bar, int c0, int c1, int c2, int c3) {
    asm volatile(
        "cp.async.bulk.tensor.4d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2,%3,%4,%5}], [%6];"
        ::"r"(su(dst)), "l"((uint64_t)m), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(su(bar)) : "memory");
}

// S slots of R*128 B; warp w (< nw) owns slots w, w+nw, ...; iters loads per slot.
__global__ void __launch_bounds__(128, 1) bench(const __grid_constant__ CUtensorMap tm, int R, int S, int nw, int iters,
                                               int nimg, int npos, unsigned long long* cyc) {
    extern __shared__ __align__(1024) uint8_t sm[];
    uint8_t* buf = sm;
    uint64_t* bars = (uint64_t*)(sm + S * R * 128);
    const int w = threadIdx.x / 32, l = threadIdx.x % 32;
    if (threadIdx.x == 0) {
        for (int i = 0; i < S; ++i) mbar_init(&bars[i], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    unsigned long long t0 = clock64();
    if (w < nw && l == 0) {
        int k = 0;
        for (int it = 0; it < iters; ++it) {
            for (int s = w; s < S; s += nw) {
                if (it > 0) waitp(&bars[s], (it - 1) & 1);
                expect(&bars[s], R * 128);
                const int pos = (blockIdx.x * 7 + k++) % npos;
                tma4(buf + s * R * 128, &tm, &bars[s], 0, pos, 0, (k * R) % (nimg - R + 1) * 0);
            }
        }
        for (int s = w; s < S; s += nw) waitp(&bars[s], (iters - 1) & 1);
    }
    __syncthreads();
    if (threadIdx.x == 0) cyc[blockIdx.x] = clock64() - t0;
}

typedef CUresult (*EncFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                          const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                          CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

int main() {
    void* fp;
    cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fp, cudaEnableDefault, &q);
    EncFn enc = (EncFn)fp;
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    // tensor: N=256 images x 16 x 16 positions x 64 channels bf16 (8 MB, L2 resident)
    const int N = 256, HW = 256, C = 64;
    void* d;
    cudaMalloc(&d, (size_t)N * HW * C * 2);
    cudaMemset(d, 0, (size_t)N * HW * C * 2);
    unsigned long long* cyc;
    cudaMalloc(&cyc, sms * 8);
    cudaFuncSetAttribute(bench, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
    printf("pattern R S nw  B/clk/SM\n");
    for (int pat = 0; pat < 5; ++pat)
        for (int R : {32, 64, 128, 256})
            for (int S : {2, 4, 8, 12, 16})
                for (int nw : {1, 2, 4}) {
                    if (pat >= 2 && pat != 4 && R != 128) continue;
                    const int T = pat == 2 ? 3 : 1;  // taps per box
                    if (S * R * 128 * T + 1024 > 210 * 1024 || nw > S) continue;
                    CUtensorMap tm;
                    cuuint64_t dims[4], str[3];
                    cuuint32_t box[4] = {64, (cuuint32_t)R, (cuuint32_t)T, 1}, es[4] = {1, 1, 1, 1};
                    if (pat == 4) { box[1] = 1; box[2] = 1; box[3] = (cuuint32_t)R; }
                    if (pat == 0) {  // (C, N, HW, 1): rows = images at stride HW*C*2
                        dims[0] = C; dims[1] = N; dims[2] = HW; dims[3] = 1;
                        str[0] = (cuuint64_t)HW * C * 2; str[1] = C * 2; str[2] = (cuuint64_t)N * HW * C * 2;
                    } else if (pat == 1) {  // (C, rows contiguous, blocks, 1)
                        dims[0] = C; dims[1] = N; dims[2] = HW; dims[3] = 1;
                        str[0] = C * 2; str[1] = (cuuint64_t)N * C * 2; str[2] = (cuuint64_t)N * HW * C * 2;
                    } else if (pat == 4) {  // natural NHWC (C, W=16, H=16, N): box (64,1,1,R)
                        dims[0] = C; dims[1] = 16; dims[2] = 16; dims[3] = N;
                        str[0] = C * 2; str[1] = 16 * C * 2; str[2] = (cuuint64_t)HW * C * 2;
                    } else {  // filter W [OC=256][9 taps][Cw=256] viewed (64 of Cw, OC, taps, 1)
                        dims[0] = 256; dims[1] = 256; dims[2] = 9; dims[3] = 1;
                        str[0] = 9 * 256 * 2; str[1] = 256 * 2; str[2] = 256 * 9 * 256 * 2;
                    }
                    CUresult r = enc(&tm, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, d, dims, str, box, es,
                                     CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                                     CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
                    if (r != CUDA_SUCCESS) { printf("enc fail %d\n", r); continue; }
                    const int iters = 2000 / S + 10;
                    const int smem = S * R * 128 * T + S * 8 + 64;
                    const int npos = pat == 4 ? 16 : (pat >= 2 ? 7 : HW);
                    bench<<<sms, 128, smem>>>(tm, R * T, S, nw, iters, N, npos, cyc);
                    bench<<<sms, 128, smem>>>(tm, R * T, S, nw, iters, N, npos, cyc);
                    cudaDeviceSynchronize();
                    std::vector<unsigned long long> h(sms);
                    cudaMemcpy(h.data(), cyc, sms * 8, cudaMemcpyDeviceToHost);
                    double mx = 0;
                    for (auto v : h) mx = v > mx ? v : mx;
                    const double bytes = (double)iters * S * R * 128 * T;
                    printf("%d %3d x%d %2d %d  %6.1f\n", pat, R, T, S, nw, bytes / mx);
                }
    cudaError_t e = cudaGetLastError();
    printf("err=%s\n", cudaGetErrorString(e));
    return 0;
}
