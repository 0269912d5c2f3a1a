// aux.cuh -- the memory-bound helper kernels of the path:
//   KB-SPLIT   KS-deconv Stage1 (Alg. 2 Stage1 P:443, Fig. 5)
//   KB-REDUCE  fixed-order G_Z aggregation of Sk-dilated partials
//   KB-PAD     zero-padded channel staging for rows not a 16-byte multiple
//              ("last dimensions ... implicitly padded to multiples of 4")
//   KB-ZINS    staging of the zero-inserted / zero-padded operand of the
//              textbook formulation (measurement baseline, not the C-K-S path)
#pragma once
#include <cstdint>

#include "ptx.cuh"

namespace cks {

// Stage1: rotate W by 180 degrees and split it into sh*sw sub-filters,
//   C_{y,x}[oc,ch,cw,ic] = W[oc, y+(oph_y-ch)*sh, x+(opw_x-cw)*sw, ic],
//   oph_y = ceil((F_H-y)/sh) - 1,
// stored packed and K-major for the KS GEMM: out[p][ic][ch*CWm+cw][ocp].
// Slots outside the phase extent and channels >= OC are written as zero.
// Per (phase, slot) this is a transpose of the (oc x ic) plane of one tap:
// 64 x 64 tiles through shared memory, 16-byte global loads / stores when the
// rows allow it (C % 8 == 0, OCp % 8 == 0; 2-byte element type).
template <typename T>
__global__ void __launch_bounds__(256) ks_split_kernel(const T* __restrict__ W, T* __restrict__ out, int OC, int FH,
                                                       int FW, int C, int sh, int sw, int CHm, int CWm, int OCp) {
    __shared__ T tile[64][66];
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
    const int oc0 = blockIdx.x * 64, ic0 = blockIdx.y * 64;
    const int t = threadIdx.x;
    constexpr int V = 16 / sizeof(T);  // elements per 16-byte vector
    const bool vec = (C % V) == 0 && (OCp % V) == 0 && sizeof(T) == 2;
    // load W[oc0+r][fh][fw][ic0 .. ic0+63] -> tile[r][.]
    if (vec) {
        for (int q = t; q < 64 * (64 / V); q += 256) {
            const int r = q / (64 / V), c = (q % (64 / V)) * V;
            const int oc = oc0 + r, ic = ic0 + c;
            uint4 v = make_uint4(0u, 0u, 0u, 0u);
            if (live && oc < OC && ic < C)
                v = *reinterpret_cast<const uint4*>(W + ((static_cast<long long>(oc) * FH + fh) * FW + fw) * C + ic);
            const T* e = reinterpret_cast<const T*>(&v);
#pragma unroll
            for (int k = 0; k < V; ++k) tile[r][c + k] = e[k];
        }
    } else {
        for (int q = t; q < 64 * 64; q += 256) {
            const int r = q / 64, c = q % 64;
            const int oc = oc0 + r, ic = ic0 + c;
            T v = T(0);
            if (live && oc < OC && ic < C) v = W[((static_cast<long long>(oc) * FH + fh) * FW + fw) * C + ic];
            tile[r][c] = v;
        }
    }
    __syncthreads();
    // store out[pidx][ic0+r][slot][oc0 .. oc0+63] <- tile[.][r]
    if (vec) {
        for (int q = t; q < 64 * (64 / V); q += 256) {
            const int r = q / (64 / V), c = (q % (64 / V)) * V;
            const int ic = ic0 + r, oc = oc0 + c;
            if (ic < C && oc < OCp) {
                uint4 v;
                T* e = reinterpret_cast<T*>(&v);
#pragma unroll
                for (int k = 0; k < V; ++k) e[k] = tile[c + k][r];
                *reinterpret_cast<uint4*>(out + ((static_cast<long long>(pidx) * C + ic) * slots + slot) * OCp + oc) = v;
            }
        }
    } else {
        for (int q = t; q < 64 * 64; q += 256) {
            const int r = q / 64, c = q % 64;
            const int ic = ic0 + r, oc = oc0 + c;
            if (ic < C && oc < OCp)
                out[((static_cast<long long>(pidx) * C + ic) * slots + slot) * OCp + oc] = tile[c][r];
        }
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

// KB-ZINS staging (the formulation C-K-S avoids: zero insertion P:114, Fig. 1
// and zero padding, Eqs (1)-(3) as written).  One block per destination row
// (n, i); in units of V (a 16-byte vector when both channel counts allow it):
//   dst[n][i][j][c] = src[n][(i-top)/sh][(j-left)/sw][c]  if i-top, j-left are
//                     non-negative multiples of sh, sw inside the source and
//                     c < Cs,  else 0.
template <typename V>
__global__ void __launch_bounds__(256) zero_insert_kernel(const V* __restrict__ src, V* __restrict__ dst, int Hs,
                                                          int Ws, int Cs, int Hd, int Wd, int Cd, int sh, int sw,
                                                          int top, int left) {
    ptx::pdl_launch_dependents();
    ptx::pdl_wait();
    const long long row = blockIdx.x;  // n * Hd + i
    const int n = int(row / Hd), i = int(row - static_cast<long long>(n) * Hd);
    const int di = i - top;
    const int si = di >= 0 && di % sh == 0 ? di / sh : -1;
    const bool live_row = si >= 0 && si < Hs;
    V* out = dst + row * Wd * Cd;
    const V* in = src + (static_cast<long long>(n) * Hs + (live_row ? si : 0)) * Ws * Cs;
    const V zero = V();  // V is a raw bit type: uint4, uint32_t (fp32) or uint16_t (bf16)
    for (int q = threadIdx.x; q < Wd * Cd; q += blockDim.x) {
        const int j = q / Cd, c = q - j * Cd;
        const int dj = j - left;
        V v = zero;
        if (live_row && dj >= 0 && dj % sw == 0 && dj / sw < Ws && c < Cs) v = in[(dj / sw) * Cs + c];
        out[q] = v;
    }
}

// Multi-phase KS-deconv for narrow outputs (I_C <= 8, F % s == 0 on both
// axes, so every phase has the same CH x CW sub-filter): the sh*sw phases are
// stacked on the GEMM N dimension.  With the phase row index shifted by a_y
// (T2), every phase reads the SAME CH x CW window of dY at window origin r, so
// the deconvolution is one unit-stride ConvV2 over dY with the stacked filter
//   Wm[n = (y*sw + x)*IC + ic][ch][cw][oc] = C_{y,x}[oc,ch,cw,ic]
//                                          = W[oc, y+(CH-1-ch)*sh, x+(CW-1-cw)*sw, ic]
// (zeros for n >= sh*sw*IC, oc >= OC) and a phase-strided scatter of its
// output Y'[n][o][q][.] to dX rows u*sh + ih_s(y), u = o - ph' - a_y.
template <typename T>
__global__ void __launch_bounds__(256) ks_mp_pack_kernel(const T* __restrict__ W, T* __restrict__ out, int OC,
                                                         int FH, int FW, int IC, int sh, int sw, int CH, int CW,
                                                         int NP, int OCp) {
    ptx::pdl_launch_dependents();
    ptx::pdl_wait();
    const long long total = static_cast<long long>(NP) * CH * CW * OCp;
    for (long long i = blockIdx.x * 256LL + threadIdx.x; i < total; i += gridDim.x * 256LL) {
        const int oc = int(i % OCp);
        long long r = i / OCp;
        const int cw = int(r % CW);
        r /= CW;
        const int ch = int(r % CH);
        const int n = int(r / CH);
        const int pidx = n / IC, ic = n % IC;
        T v = T(0);
        if (pidx < sh * sw && oc < OC) {
            const int y = pidx / sw, x = pidx % sw;
            const int fh = y + (CH - 1 - ch) * sh, fw = x + (CW - 1 - cw) * sw;
            v = W[((static_cast<long long>(oc) * FH + fh) * FW + fw) * IC + ic];
        }
        out[i] = v;
    }
}

// dX[n][u*sh + ih_s(y)][v*sw + iw_s(x)][ic] = Y'[n][u + a_y + ph'][v + a_x + pw'][(y*sw+x)*IC + ic]
// for every phase and row / column of the phase (the phases partition dX, so
// every element of dX is written exactly once).  Thread = one dX element.
struct MpPhase {
    int16_t ih_s[8], a_y[8], iw_s[8], a_x[8];
};
__global__ void __launch_bounds__(256) ks_mp_scatter_kernel(const float* __restrict__ yp, float* __restrict__ dx,
                                                            long long N, int H, int W, int IC, int sh, int sw, int MH,
                                                            int MW, int NP, int ph2, int pw2, MpPhase t) {
    ptx::pdl_launch_dependents();
    ptx::pdl_wait();
    const long long total = N * H * W * IC;
    for (long long i = blockIdx.x * 256LL + threadIdx.x; i < total; i += gridDim.x * 256LL) {
        const int ic = int(i % IC);
        long long r = i / IC;
        const int iw = int(r % W);
        r /= W;
        const int ih = int(r % H);
        const long long n = r / H;
        // phase of this element: ih = u*sh + ih_s(y) with ih_s(y) in [0, sh)
        int y = 0, x = 0;
        while (y + 1 < sh && t.ih_s[y] != ih % sh) ++y;
        while (x + 1 < sw && t.iw_s[x] != iw % sw) ++x;
        const int u = (ih - t.ih_s[y]) / sh, v = (iw - t.iw_s[x]) / sw;
        const int o = u + t.a_y[y] + ph2, q = v + t.a_x[x] + pw2;
        float val = 0.f;
        if (o >= 0 && o < MH && q >= 0 && q < MW)
            val = yp[((n * MH + o) * MW + q) * NP + (y * sw + x) * IC + ic];
        dx[i] = val;
    }
}

// out[i] = sum_{z = 0..gz-1} part[z][i] with a FIXED association
// (deterministic): z-group g = threadIdx.y sums z = g, g+G, g+2G, ... in
// increasing z, then the G group sums are added in order g = 0..G-1.
// blockDim = (32, G); one block covers 32 vector elements.
__device__ __forceinline__ float4 vadd(float4 a, float4 b) { return make_float4(a.x + b.x, a.y + b.y, a.z + b.z, a.w + b.w); }
__device__ __forceinline__ float vadd(float a, float b) { return a + b; }
template <typename V>
__device__ __forceinline__ V vzero();
template <>
__device__ __forceinline__ float4 vzero<float4>() { return make_float4(0.f, 0.f, 0.f, 0.f); }
template <>
__device__ __forceinline__ float vzero<float>() { return 0.f; }

template <typename V>
__global__ void reduce_partials_kernel(const V* __restrict__ part, V* __restrict__ out, long long nv, int gz) {
    __shared__ V acc[16][32];
    ptx::pdl_launch_dependents();
    ptx::pdl_wait();
    const int G = int(blockDim.y), g = int(threadIdx.y), x = int(threadIdx.x);
    for (long long i0 = blockIdx.x * 32LL; i0 < nv; i0 += gridDim.x * 32LL) {
        const long long i = i0 + x;
        V a = vzero<V>();
        if (i < nv) {
            int z = g;
            for (; z + 3 * G < gz; z += 4 * G) {  // 4 independent loads in flight
                const V v0 = part[z * nv + i], v1 = part[(z + G) * nv + i];
                const V v2 = part[(z + 2 * G) * nv + i], v3 = part[(z + 3 * G) * nv + i];
                a = vadd(vadd(vadd(vadd(a, v0), v1), v2), v3);
            }
            for (; z < gz; z += G) a = vadd(a, part[z * nv + i]);
        }
        acc[g][x] = a;
        __syncthreads();
        if (g == 0 && i < nv) {
            V r = acc[0][x];
            for (int q = 1; q < G; ++q) r = vadd(r, acc[q][x]);
            out[i] = r;
        }
        __syncthreads();
    }
}

}  // namespace cks
