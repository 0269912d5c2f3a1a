// lsu_bench.cu -- smem ingress of scattered 128-byte rows (rows = images of an
// NHWC tensor at stride H*W*C*2) via (a) TMA boxes, (b) cp.async 16 B per
// thread from nl loader warps, (c) both at once on disjoint halves.
// build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/lsu_bench tools/lsu_bench.cu -lcuda
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
__device__ __forceinline__ void cpa16(uint32_t dst, const void* src) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst), "l"(src) : "memory");
}

// X: N images x P positions x 64 ch bf16 (row = 128 B at (n, pos)), row stride between images = P*128.
// Each "stage" = R rows (images n0..n0+R-1 at one position) = R*128 bytes.
// mode 0: TMA only (warp 0), mode 1: cp.async only (nl warps), mode 2: TMA half + cp.async half.
__global__ void __launch_bounds__(384, 1) bench(const __grid_constant__ CUtensorMap tm, const uint8_t* X, int P, int R,
                                               int S, int iters, int mode, int nl, unsigned long long* cyc) {
    extern __shared__ __align__(1024) uint8_t sm[];
    const int bytes = R * 128;
    uint64_t* bars = (uint64_t*)(sm + S * bytes);
    const int w = threadIdx.x / 32, l = threadIdx.x % 32;
    if (threadIdx.x == 0) {
        for (int i = 0; i < S; ++i) mbar_init(&bars[i], 1 + (mode >= 1 ? nl * 32 : 0));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    unsigned long long t0 = clock64();
    const int tma_rows = mode == 0 ? R : (mode == 2 ? R / 2 : 0);
    if (w == 0) {
        if (l == 0) {
            for (int it = 0; it < iters; ++it)
                for (int s = 0; s < S; ++s) {
                    if (it > 0) waitp(&bars[s], (it - 1) & 1);
                    expect(&bars[s], tma_rows * 128);
                    const int pos = (blockIdx.x * 7 + it * S + s) % P;
                    if (tma_rows) tma4(sm + s * bytes, &tm, &bars[s], 0, 0, pos, 0);
                }
        }
    } else if (w >= 1 && w <= nl && mode >= 1) {
        const int lt = (w - 1) * 32 + l;
        const int nthr = nl * 32;
        for (int it = 0; it < iters; ++it)
            for (int s = 0; s < S; ++s) {
                if (it > 0) waitp(&bars[s], (it - 1) & 1);
                const int pos = (blockIdx.x * 7 + it * S + s) % P;
                // rows [tma_rows, R): 8 x 16 B chunks each
                for (int q = lt; q < (R - tma_rows) * 8; q += nthr) {
                    const int r = tma_rows + q / 8, c = q % 8;
                    const uint8_t* src = X + ((size_t)r * P + pos) * 128 + c * 16;
                    const uint32_t dst = su(sm + s * bytes + r * 128 + ((c ^ (r & 7)) * 16));
                    cpa16(dst, src);
                }
                asm volatile("cp.async.mbarrier.arrive.noinc.shared.b64 [%0];" ::"r"(su(&bars[s])) : "memory");
            }
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int s = 0; s < S; ++s) waitp(&bars[s], (iters - 1) & 1);
        cyc[blockIdx.x] = clock64() - t0;
    }
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
    const int N = 256, P = 256;  // 256 images x 256 positions x 128 B = 8 MB (L2 resident)
    uint8_t* d;
    cudaMalloc(&d, (size_t)N * P * 128);
    cudaMemset(d, 0, (size_t)N * P * 128);
    unsigned long long* cyc;
    cudaMalloc(&cyc, sms * 8);
    cudaFuncSetAttribute(bench, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
    printf("mode nl R S  B/clk/SM\n");
    for (int mode : {0, 1, 2})
        for (int nl : {2, 4, 8})
            for (int R : {128})
                for (int S : {4, 8}) {
                    if (mode == 0 && nl != 2) continue;
                    CUtensorMap tm;
                    cuuint64_t dims[4] = {64, (cuuint64_t)N, (cuuint64_t)P, 1};
                    cuuint64_t str[3] = {(cuuint64_t)P * 128, 128, (cuuint64_t)N * P * 128};
                    const cuuint32_t rows = mode == 2 ? R / 2 : R;
                    cuuint32_t box[4] = {64, rows, 1, 1}, es[4] = {1, 1, 1, 1};
                    enc(&tm, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, d, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                        CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
                    const int iters = 3000 / S;
                    const int smem = S * R * 128 + S * 8 + 64;
                    bench<<<sms, 384, smem>>>(tm, d, P, R, S, iters, mode, nl, cyc);
                    bench<<<sms, 384, smem>>>(tm, d, P, R, S, iters, mode, nl, cyc);
                    cudaError_t e = cudaDeviceSynchronize();
                    if (e != cudaSuccess) { printf("err %s\n", cudaGetErrorString(e)); return 1; }
                    std::vector<unsigned long long> h(sms);
                    cudaMemcpy(h.data(), cyc, sms * 8, cudaMemcpyDeviceToHost);
                    double mx = 0;
                    for (auto v : h) mx = v > mx ? v : mx;
                    printf("%d %d %3d %2d  %6.1f\n", mode, nl, R, S, (double)iters * S * R * 128 / mx);
                }
    return 0;
}
