// aux.cuh -- the memory-bound helper kernels of the path:
//   KB-SPLIT   KS-deconv Stage1 (Alg. 2 Stage1 P:443, Fig. 5)
//   KB-REDUCE  fixed-order G_Z aggregation of Sk-dilated partials
//   KB-PAD     zero-padded channel staging for rows not a 16-byte multiple
//              ("last dimensions ... implicitly padded to multiples of 4")
#pragma once
#include <cstdint>

#include "ptx.cuh"

namespace cks {

// Stage1: rotate W by 180 degrees and split it into sh*sw sub-filters,
//   C_{y,x}[oc,ch,cw,ic] = W[oc, y+(oph_y-ch)*sh, x+(opw_x-cw)*sw, ic],
//   oph_y = ceil((F_H-y)/sh) - 1,
// stored packed and K-major for the KS GEMM: out[p][ic][ch*CWm+cw][ocp].
// Slots outside the phase extent and channels >= OC are written as zero.
// Tile transpose through shared memory: 32 oc x 32 ic per block.
template <typename T>
__global__ void ks_split_kernel(const T* __restrict__ W, T* __restrict__ out, int OC, int FH, int FW, int C, int sh,
                                int sw, int CHm, int CWm, int OCp) {
    __shared__ T tile[32][33];
    ptx::pdl_launch_dependents();
    ptx::pdl_wait();
    const int slots = CHm * CWm;
    const int ps = blockIdx.z;  // (phase, slot)
    const int pidx = ps / slots, slot = ps % slots;
    const int y = pidx / sw, x = pidx % sw;
    const int ch = slot / CWm, cw = slot % CWm;
    const int CH = FH > y ? (FH - y + sh - 1) / sh : 0;
    const int CW = FW > x ? (FW - x + sw - 1) / sw : 0;
    const bool live = ch < CH && cw < CW;
    const int fh = y + (CH - 1 - ch) * sh;
    const int fw = x + (CW - 1 - cw) * sw;
    const int oc0 = blockIdx.x * 32, ic0 = blockIdx.y * 32;
    // load W[oc0+ty][fh][fw][ic0+tx] (coalesced over ic)
    for (int ty = threadIdx.y; ty < 32; ty += blockDim.y) {
        const int oc = oc0 + ty, ic = ic0 + threadIdx.x;
        T v = T(0);
        if (live && oc < OC && ic < C) v = W[((static_cast<long long>(oc) * FH + fh) * FW + fw) * C + ic];
        tile[ty][threadIdx.x] = v;
    }
    __syncthreads();
    // store out[pidx][ic0+ty][slot][oc0+tx] (coalesced over oc)
    for (int ty = threadIdx.y; ty < 32; ty += blockDim.y) {
        const int ic = ic0 + ty, oc = oc0 + threadIdx.x;
        if (ic < C && oc < OCp)
            out[((static_cast<long long>(pidx) * C + ic) * slots + slot) * OCp + oc] = tile[threadIdx.x][ty];
    }
}

// dst[r][0:Cp] = src[r][0:C] with zeros in [C, Cp).
template <typename T>
__global__ void pad_channels_kernel(const T* __restrict__ src, T* __restrict__ dst, long long rows, int C, int Cp) {
    ptx::pdl_launch_dependents();
    ptx::pdl_wait();
    const long long total = rows * Cp;
    for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < total;
         i += static_cast<long long>(gridDim.x) * blockDim.x) {
        const long long r = i / Cp;
        const int c = int(i - r * Cp);
        dst[i] = c < C ? src[r * C + c] : T(0);
    }
}

// out[i] = sum_{z = 0..gz-1} part[z][i], fixed order z = 0, 1, ... (deterministic).
__global__ void reduce_partials_kernel(const float* __restrict__ part, float* __restrict__ out, long long n, int gz) {
    ptx::pdl_launch_dependents();
    ptx::pdl_wait();
    const long long n4 = n / 4;
    const float4* p4 = reinterpret_cast<const float4*>(part);
    float4* o4 = reinterpret_cast<float4*>(out);
    const long long s4 = n / 4;  // partial stride in float4 (n % 4 == 0 on this path)
    for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < n4;
         i += static_cast<long long>(gridDim.x) * blockDim.x) {
        float4 a = p4[i];
        for (int z = 1; z < gz; ++z) {
            const float4 b = p4[z * s4 + i];
            a.x += b.x;
            a.y += b.y;
            a.z += b.z;
            a.w += b.w;
        }
        o4[i] = a;
    }
}

__global__ void reduce_partials_scalar_kernel(const float* __restrict__ part, float* __restrict__ out, long long n,
                                              int gz) {
    ptx::pdl_launch_dependents();
    ptx::pdl_wait();
    for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<long long>(gridDim.x) * blockDim.x) {
        float a = part[i];
        for (int z = 1; z < gz; ++z) a += part[z * n + i];
        out[i] = a;
    }
}

}  // namespace cks
