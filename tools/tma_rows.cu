// tma_rows.cu -- TMA ingress (B/clk/SM) vs innermost row bytes (32/64/128) for
// boxes (RB/2 elements, R images, T filter rows, 1) over an NHWC-like tensor
// (rows = images at a large stride), S ring slots, nw issuing warps.
// build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/tma_rows tools/tma_rows.cu -lcuda
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

__global__ void __launch_bounds__(128, 1) bench(const __grid_constant__ CUtensorMap tm, int bytes, int S, int nw,
                                               int iters, int W, int H, unsigned long long* cyc) {
    extern __shared__ __align__(1024) uint8_t sm[];
    uint64_t* bars = (uint64_t*)(sm + S * bytes);
    const int w = threadIdx.x / 32, l = threadIdx.x % 32;
    if (threadIdx.x == 0) {
        for (int i = 0; i < S; ++i) mbar_init(&bars[i], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    unsigned long long t0 = clock64();
    if (w < nw && l == 0) {
        int k = 0;
        for (int it = 0; it < iters; ++it)
            for (int s = w; s < S; s += nw) {
                if (it > 0) waitp(&bars[s], (it - 1) & 1);
                expect(&bars[s], bytes);
                const int pos = (blockIdx.x * 7 + k++);
                tma4(sm + s * bytes, &tm, &bars[s], (pos % W) * 8, 0, (pos / W) % H, 0);
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
    // X: N=256 images x H=32 x W=32 x C=8 bf16 viewed (W*C, N, H, 1)  (4 MB, L2 resident)
    const int N = 256, H = 32, W = 32, C = 8;
    void* d;
    cudaMalloc(&d, (size_t)N * H * W * C * 2 * 4);
    cudaMemset(d, 0, (size_t)N * H * W * C * 2);
    unsigned long long* cyc;
    cudaMalloc(&cyc, sms * 8);
    cudaFuncSetAttribute(bench, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
    printf("ctas contig RB R T S nw  B/clk/SM\n");
    for (int ctas : {148})
    for (int contig : {0, 1, 2})
    for (int RB : {64, 128})
        for (int R : {128})
            for (int T : {1, 4})
                for (int S : {4, 8})
                    for (int nw : {1, 2}) {
                        const int bytes = RB * R * T;
                        if (S * bytes + 1024 > 200 * 1024 || nw > S) continue;
                        CUtensorMap tm;
                        cuuint64_t dims[4] = {(cuuint64_t)W * C, (cuuint64_t)N, (cuuint64_t)H, 1};
                        cuuint64_t str[3] = {(cuuint64_t)H * W * C * 2, (cuuint64_t)W * C * 2, (cuuint64_t)N * H * W * C * 2};
                        if (contig) {  // rows of one box contiguous: (W*C, N) with N stride = RB bytes... use a dense [H][N][RB] view
                            // contig 2: rows at a 2*RB pitch (image-innermost layout with twice the channels)
                            const cuuint64_t pitch = (cuuint64_t)RB * contig;
                            dims[0] = RB / 2; dims[1] = N; dims[2] = H; dims[3] = 1;
                            str[0] = pitch; str[1] = (cuuint64_t)N * pitch; str[2] = (cuuint64_t)N * H * pitch;
                        }
                        cuuint32_t box[4] = {(cuuint32_t)RB / 2, (cuuint32_t)R, (cuuint32_t)T, 1}, es[4] = {1, 1, 1, 1};
                        CUresult r = enc(&tm, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, d, dims, str, box, es,
                                         CU_TENSOR_MAP_INTERLEAVE_NONE,
                                         RB == 128 ? CU_TENSOR_MAP_SWIZZLE_128B : (RB == 64 ? CU_TENSOR_MAP_SWIZZLE_64B : CU_TENSOR_MAP_SWIZZLE_32B),
                                         CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
                        if (r != CUDA_SUCCESS) { printf("enc fail %d\n", r); continue; }
                        const int iters = 400000 / (S * bytes / 64) + 4;
                        const int smem = S * bytes + S * 8 + 64;
                        const int wx = contig ? 1 : W - 4;
                        bench<<<ctas, 128, smem>>>(tm, bytes, S, nw, iters, wx, H - 8, cyc);
                        bench<<<ctas, 128, smem>>>(tm, bytes, S, nw, iters, wx, H - 8, cyc);
                        cudaDeviceSynchronize();
                        std::vector<unsigned long long> h(ctas);
                        cudaMemcpy(h.data(), cyc, ctas * 8, cudaMemcpyDeviceToHost);
                        double mx = 0;
                        for (auto v : h) mx = v > mx ? v : mx;
                        printf("%3d %d %3d %3d %d %2d %d  %6.1f\n", ctas, contig, RB, R, T, S, nw, (double)iters * S * bytes / mx);
                    }
    printf("err=%s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
