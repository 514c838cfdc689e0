// tem_simt.cu -- SIMT (CUDA-core) implementation of the BSN-TEM step.
//
// First correct path: implicit-GEMM convolutions on CUDA cores with fp32
// accumulation, fused bias/ReLU/halo epilogues, a
// per-video fused head kernel (conv3 + sigmoid + weighted logistic loss + dz +
// head backward, rows a3-a5) and deterministic split-K weight gradients.
// All reductions run in a fixed order, so a rank's gradient is bitwise
// reproducible run to run.
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <math.h>

#include "kernels.h"

namespace tem {
namespace {

constexpr int BM = 128, BN = 128, BK = 16, NT = 256;

enum Mode { FWD = 0, DGRAD = 1, WGRAD = 2 };

TEM_DEV bool is_halo(int p, int Tp) {
    const int t = p % Tp;
    return t == 0 || t == Tp - 1;
}

// One 128x128 output tile of an implicit GEMM; 256 threads, 8x8 outputs each
// (rows ty*4+{0..3} and 64+ty*4+{0..3}; columns likewise with tx).
//
// FWD   : out[p][o]  = act(bias[o] + sum_{j,c} in[p+j-1][c] * W[o][j][c])       (rows a1/a2)
// DGRAD : dA1[p][c]  = 1[h1>0] * sum_{j,o} dA2[p+1-j][o] * W[o][j][c]           (row a6)
// WGRAD : part[s][o][j*Cin+c] = sum_{p in split s} dA[p][o] * in[p+j-1][c]      (rows a7/a8)
//         and part[s][Cout*3*Cin + o] = sum_p dA[p][o]  (bias gradient)
template <int MODE, typename TA, typename TB, typename TOut>
__global__ void __launch_bounds__(NT) simt_conv_kernel(
    const TA* __restrict__ A, const TB* __restrict__ Bm, const float* __restrict__ bias,
    const void* __restrict__ mask, TOut* __restrict__ out, int R, int Tp, int Cin, int Cout,
    int k_split) {
    __shared__ __align__(16) float As[2][BK][BM];
    __shared__ __align__(16) float Bs[2][BK][BN];
    const int tid = threadIdx.x;
    const int tx = tid % 16, ty = tid / 16;

    int m0, n0, kb_begin, kb_end;
    int p_begin = 0, p_end = 0;
    if (MODE == WGRAD) {
        m0 = blockIdx.x * BM;  // o
        n0 = blockIdx.y * BN;  // j*Cin + c
        p_begin = blockIdx.z * k_split;
        p_end = min(R, p_begin + k_split);
        kb_begin = 0;
        kb_end = (p_end - p_begin + BK - 1) / BK;
    } else {
        m0 = blockIdx.x * BM;  // p
        n0 = blockIdx.y * BN;  // o (FWD) or c (DGRAD)
        kb_begin = 0;
        kb_end = 3 * (Cin / BK);  // (tap j, channel block)
    }
    const int NW = 3 * Cin;  // WGRAD column count

    float ra[8], rb[8];
    // ---- global -> registers for k-block kb ----
    auto load = [&](int kb) {
        if (MODE == FWD || MODE == DGRAD) {
            const int cpb = Cin / BK;
            const int j = kb / cpb, c0 = (kb % cpb) * BK;
            {   // A: row m = tid/2, 8 k-values at (tid%2)*8
                const int m = tid >> 1, kh = (tid & 1) * 8;
                const int row = (MODE == FWD) ? (m0 + m + j - 1) : (m0 + m + 1 - j);
                if (m0 + m < R && row >= 0 && row < R)
                    load8(A + (size_t)row * Cin + c0 + kh, ra);
                else
#pragma unroll
                    for (int q = 0; q < 8; ++q) ra[q] = 0.f;
            }
            if (MODE == FWD) {  // B: W[o][j][c], row o = tid/2
                const int n = tid >> 1, kh = (tid & 1) * 8;
                if (n0 + n < Cout)
                    load8(Bm + ((size_t)(n0 + n) * 3 + j) * Cin + c0 + kh, rb);
                else
#pragma unroll
                    for (int q = 0; q < 8; ++q) rb[q] = 0.f;
            } else {  // DGRAD B: W[o0+k][j][n0 + n8 .. +7], k = tid/16 (channel index c = n)
                const int k = tid >> 4, n8 = (tid & 15) * 8;
                const int C = Cout;  // W is [Cin_o][3][C]; here "Cin" = #o, Cout = #c
                load8(Bm + ((size_t)(c0 + k) * 3 + j) * C + n0 + n8, rb);
            }
        } else {  // WGRAD
            const int k = tid >> 4, x8 = (tid & 15) * 8;
            const int p = p_begin + kb * BK + k;
            // A: dA[p][m0 + x8 ..]
            if (p < p_end)
                load8(A + (size_t)p * Cout + m0 + x8, ra);
            else
#pragma unroll
                for (int q = 0; q < 8; ++q) ra[q] = 0.f;
            // B: in[p + j - 1][c], n = j*Cin + c
            const int n = n0 + x8;
            const int j = n / Cin, c = n - j * Cin;
            const int row = p + j - 1;
            if (p < p_end && n < NW && row >= 0 && row < R)
                load8(Bm + (size_t)row * Cin + c, rb);
            else
#pragma unroll
                for (int q = 0; q < 8; ++q) rb[q] = 0.f;
        }
    };
    auto store = [&](int buf) {
        if (MODE == FWD || MODE == DGRAD) {
            const int m = tid >> 1, kh = (tid & 1) * 8;
#pragma unroll
            for (int q = 0; q < 8; ++q) As[buf][kh + q][m] = ra[q];
            if (MODE == FWD) {
#pragma unroll
                for (int q = 0; q < 8; ++q) Bs[buf][kh + q][m] = rb[q];
            } else {
                const int k = tid >> 4, n8 = (tid & 15) * 8;
                *reinterpret_cast<float4*>(&Bs[buf][k][n8]) = make_float4(rb[0], rb[1], rb[2], rb[3]);
                *reinterpret_cast<float4*>(&Bs[buf][k][n8 + 4]) = make_float4(rb[4], rb[5], rb[6], rb[7]);
            }
        } else {
            const int k = tid >> 4, x8 = (tid & 15) * 8;
            *reinterpret_cast<float4*>(&As[buf][k][x8]) = make_float4(ra[0], ra[1], ra[2], ra[3]);
            *reinterpret_cast<float4*>(&As[buf][k][x8 + 4]) = make_float4(ra[4], ra[5], ra[6], ra[7]);
            *reinterpret_cast<float4*>(&Bs[buf][k][x8]) = make_float4(rb[0], rb[1], rb[2], rb[3]);
            *reinterpret_cast<float4*>(&Bs[buf][k][x8 + 4]) = make_float4(rb[4], rb[5], rb[6], rb[7]);
        }
    };

    float acc[8][8];
#pragma unroll
    for (int i = 0; i < 8; ++i)
#pragma unroll
        for (int j = 0; j < 8; ++j) acc[i][j] = 0.f;
    float bsum = 0.f;  // WGRAD bias column sum (threads < BM of n-tile 0)

    if (kb_begin < kb_end) {
        load(kb_begin);
        store(0);
    }
    __syncthreads();
    for (int kb = kb_begin; kb < kb_end; ++kb) {
        const int cur = (kb - kb_begin) & 1;
        if (kb + 1 < kb_end) load(kb + 1);
#pragma unroll
        for (int k = 0; k < BK; ++k) {
            const float4 a0 = *reinterpret_cast<const float4*>(&As[cur][k][ty * 4]);
            const float4 a1 = *reinterpret_cast<const float4*>(&As[cur][k][ty * 4 + 64]);
            const float4 b0 = *reinterpret_cast<const float4*>(&Bs[cur][k][tx * 4]);
            const float4 b1 = *reinterpret_cast<const float4*>(&Bs[cur][k][tx * 4 + 64]);
            const float a[8] = {a0.x, a0.y, a0.z, a0.w, a1.x, a1.y, a1.z, a1.w};
            const float b[8] = {b0.x, b0.y, b0.z, b0.w, b1.x, b1.y, b1.z, b1.w};
#pragma unroll
            for (int i = 0; i < 8; ++i)
#pragma unroll
                for (int j = 0; j < 8; ++j) acc[i][j] = fmaf(a[i], b[j], acc[i][j]);
        }
        if (MODE == WGRAD && blockIdx.y == 0 && tid < BM) {
#pragma unroll
            for (int k = 0; k < BK; ++k) bsum += As[cur][k][tid];
        }
        if (kb + 1 < kb_end) store(cur ^ 1);
        __syncthreads();
    }

    // ---- epilogue ----
#pragma unroll
    for (int i = 0; i < 8; ++i) {
        const int m = m0 + (i < 4 ? ty * 4 + i : 64 + ty * 4 + (i - 4));
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const int n = n0 + tx * 4 + h * 64;
            float v[4] = {acc[i][h * 4], acc[i][h * 4 + 1], acc[i][h * 4 + 2], acc[i][h * 4 + 3]};
            if (MODE == FWD) {
                if (m >= R || n >= Cout) continue;
                const bool halo = is_halo(m, Tp);
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    float t = v[q] + bias[n + q];
                    t = t > 0.f ? t : 0.f;
                    out[(size_t)m * Cout + n + q] = from_f<TOut>(halo ? 0.f : t);
                }
            } else if (MODE == DGRAD) {
                if (m >= R || n >= Cout) continue;
                const bool halo = is_halo(m, Tp);
                const TA* h1 = reinterpret_cast<const TA*>(mask);
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    const float hv = to_f(h1[(size_t)m * Cout + n + q]);
                    out[(size_t)m * Cout + n + q] = from_f<TOut>((!halo && hv > 0.f) ? v[q] : 0.f);
                }
            } else {
                // WGRAD: m = o (< Cout), n = j*Cin + c (< NW); partial slice for split z
                if (n >= NW) continue;
                float* dst = reinterpret_cast<float*>(out) + (size_t)blockIdx.z * ((size_t)Cout * NW + Cout);
#pragma unroll
                for (int q = 0; q < 4; ++q) dst[(size_t)m * NW + n + q] = v[q];
            }
        }
    }
    if (MODE == WGRAD && blockIdx.y == 0 && tid < BM) {
        float* dst = reinterpret_cast<float*>(out) + (size_t)blockIdx.z * ((size_t)Cout * NW + Cout);
        dst[(size_t)Cout * NW + m0 + tid] = bsum;
    }
}

// part[s][0..n) summed over s in ascending order -> dst[0..n).  n multiple of 4.
__global__ void reduce_splits_kernel(const float* __restrict__ part, float* __restrict__ dst,
                                     int64_t n, int S) {
    const int64_t nv = n / 4;
    for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < nv;
         v += (int64_t)gridDim.x * blockDim.x) {
        float4 a = reinterpret_cast<const float4*>(part)[v];
        for (int s = 1; s < S; ++s) {
            const float4 b = reinterpret_cast<const float4*>(part + (size_t)s * n)[v];
            a.x += b.x; a.y += b.y; a.z += b.z; a.w += b.w;
        }
        reinterpret_cast<float4*>(dst)[v] = a;
    }
}

// x [B][T][Cin] -> xp [B][T+2][Cin] with zero halo rows (same operand type).
template <typename T>
__global__ void prep_x_kernel(const T* __restrict__ x, T* __restrict__ xp, int B, int Tn, int Cin) {
    const int vec = 16 / sizeof(T);
    // 32-bit index math, one 16-byte group per thread (grid sized by the launcher)
    const int per_row = Cin / vec;
    const int total = B * (Tn + 2) * per_row;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < total; i += gridDim.x * blockDim.x) {
        const int p = i / per_row;
        const int cv = i - p * per_row;
        const int v = p / (Tn + 2);
        const int t = p - v * (Tn + 2);
        uint4 val = make_uint4(0, 0, 0, 0);
        if (t >= 1 && t <= Tn)
            val = reinterpret_cast<const uint4*>(x + ((size_t)v * Tn + (t - 1)) * Cin)[cv];
        reinterpret_cast<uint4*>(xp + (size_t)p * Cin)[cv] = val;
    }
}

__global__ void cast_shadow_kernel(const float* __restrict__ w, __nv_bfloat16* __restrict__ s, int64_t n) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x)
        s[i] = __float2bfloat16_rn(w[i]);
}

template <typename T>
cudaError_t conv_launches(const Geom& g, const RankBufs& b, const float* labels, const float lam[3],
                          float* loss_out, Status* status, int* nl, const EvRec& rec, cudaStream_t s) {
    const int R = g.R, Tp = g.T + 2;
    const T* xp = static_cast<const T*>(b.xp);
    T* h1 = static_cast<T*>(b.h1);
    T* dA2 = static_cast<T*>(b.dA2);
    T* dA1 = static_cast<T*>(b.dA1);
    const T* W = static_cast<const T*>(b.wop);
    const T* W1 = W + g.off_W1;
    const T* W2 = W + g.off_W2;
    const dim3 blk(NT);
    int n = 0;
    if (g.B == 0) {  // empty shard: zero gradient, zero loss (the update is then a no-op)
        cudaMemsetAsync(b.grad, 0, (size_t)g.Kpad * sizeof(float), s);
        return launch_head(g, b, labels, lam, loss_out, status, rec, s, nl);
    }
    // a1: conv1 + bias + ReLU -> h1
    rec.begin(SLOT_CONV1);
    simt_conv_kernel<FWD, T, T, T><<<dim3((R + BM - 1) / BM, (g.C + BN - 1) / BN), blk, 0, s>>>(
        xp, W1, b.params + g.off_b1, nullptr, h1, R, Tp, g.Cin, g.C, 0);
    rec.end(SLOT_CONV1);
    ++n;
    // a2: conv2 + bias + ReLU -> h2 (fp32; consumed by the fp32 head)
    rec.begin(SLOT_CONV2);
    simt_conv_kernel<FWD, T, T, float><<<dim3((R + BM - 1) / BM, (g.C + BN - 1) / BN), blk, 0, s>>>(
        h1, W2, b.params + g.off_b2, nullptr, b.h2, R, Tp, g.C, g.C, 0);
    rec.end(SLOT_CONV2);
    ++n;
    // a3-a5: head
    {
        cudaError_t e = launch_head(g, b, labels, lam, loss_out, status, rec, s, &n);
        if (e != cudaSuccess) return e;
    }
    // a6: conv2 dgrad -> dA1
    rec.begin(SLOT_DGRAD);
    simt_conv_kernel<DGRAD, T, T, T><<<dim3((R + BM - 1) / BM, (g.C + BN - 1) / BN), blk, 0, s>>>(
        dA2, W2, nullptr, h1, dA1, R, Tp, g.C, g.C, 0);
    rec.end(SLOT_DGRAD);
    ++n;
    // a7: conv2 wgrad (+ db2), a8: conv1 wgrad (+ db1)
    const int S = simt_wgrad_splits(g);
    const int ksplit = ((R + S - 1) / S + BK - 1) / BK * BK;
    const int S_eff = (R + ksplit - 1) / ksplit;
    rec.begin(SLOT_WGRAD2);
    simt_conv_kernel<WGRAD, T, T, float><<<dim3(g.C / BM, (3 * g.C + BN - 1) / BN, S_eff), blk, 0, s>>>(
        dA2, h1, nullptr, nullptr, b.wpart, R, Tp, g.C, g.C, ksplit);
    rec.end(SLOT_WGRAD2);
    ++n;
    {
        const int64_t nn = (int64_t)g.C * 3 * g.C + g.C;
        rec.begin(SLOT_RED2);
        launch_reduce_splits(b.wpart, b.grad + g.off_W2, nn, S_eff, s);
        rec.end(SLOT_RED2);
        ++n;
    }
    rec.begin(SLOT_WGRAD1);
    simt_conv_kernel<WGRAD, T, T, float><<<dim3(g.C / BM, (3 * g.Cin + BN - 1) / BN, S_eff), blk, 0, s>>>(
        dA1, xp, nullptr, nullptr, b.wpart, R, Tp, g.Cin, g.C, ksplit);
    rec.end(SLOT_WGRAD1);
    ++n;
    {
        const int64_t nn = (int64_t)g.C * 3 * g.Cin + g.C;
        rec.begin(SLOT_RED1);
        launch_reduce_splits(b.wpart, b.grad + g.off_W1, nn, S_eff, s);
        rec.end(SLOT_RED1);
        ++n;
    }
    *nl += n;
    return cudaGetLastError();
}

}  // namespace

cudaError_t launch_reduce_splits(const float* part, float* dst, int64_t n, int S, cudaStream_t s) {
    reduce_splits_kernel<<<296, 256, 0, s>>>(part, dst, n, S);
    return cudaGetLastError();
}

int simt_wgrad_splits(const Geom& g) {
    const int tiles = (g.C / BM) * ((3 * g.Cin + BN - 1) / BN);
    int S = (2 * 148 + tiles - 1) / tiles;
    const int maxS = (g.R + BK - 1) / BK;
    if (S > maxS) S = maxS;
    if (S < 1) S = 1;
    return S;
}

cudaError_t launch_prep_x(const Geom& g, const void* x, void* xp, cudaStream_t s) {
    const int vec = g.prec == TEM_BF16 ? 8 : 4;
    const int groups = g.B * (g.T + 2) * (g.Cin / vec);
    const int grid = groups <= 0 ? 1 : (groups + 255) / 256 > 148 * 16 ? 148 * 16 : (groups + 255) / 256;
    if (g.prec == TEM_BF16)
        prep_x_kernel<__nv_bfloat16><<<grid, 256, 0, s>>>(static_cast<const __nv_bfloat16*>(x),
                                                          static_cast<__nv_bfloat16*>(xp), g.B, g.T, g.Cin);
    else
        prep_x_kernel<float><<<grid, 256, 0, s>>>(static_cast<const float*>(x), static_cast<float*>(xp),
                                                  g.B, g.T, g.Cin);
    return cudaGetLastError();
}

template <typename T>
__global__ void relu_decisions_kernel(const T* __restrict__ h1, const float* __restrict__ h2,
                                      uint8_t* __restrict__ out, int B, int Tn, int C) {
    const int64_t n = (int64_t)B * Tn * C;
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n;
         e += (int64_t)gridDim.x * blockDim.x) {
        const int64_t r = e / C;
        const int c = (int)(e - r * C);
        const int64_t v = r / Tn, t = r - v * Tn;
        const int64_t p = v * (Tn + 2) + t + 1;
        out[e] = to_f(h1[p * C + c]) > 0.f ? 1 : 0;
        out[n + e] = h2[p * C + c] > 0.f ? 1 : 0;
    }
}

cudaError_t launch_relu_decisions(const Geom& g, const RankBufs& b, uint8_t* out, cudaStream_t s) {
    if (g.op_bf16)
        relu_decisions_kernel<__nv_bfloat16><<<296, 256, 0, s>>>(static_cast<const __nv_bfloat16*>(b.h1), b.h2,
                                                                 out, g.B, g.T, g.C);
    else
        relu_decisions_kernel<float><<<296, 256, 0, s>>>(static_cast<const float*>(b.h1), b.h2, out, g.B, g.T, g.C);
    return cudaGetLastError();
}

cudaError_t launch_cast_shadow(const float* params, __nv_bfloat16* shadow, int64_t n, cudaStream_t s) {
    cast_shadow_kernel<<<296, 256, 0, s>>>(params, shadow, n);
    return cudaGetLastError();
}

cudaError_t simt_compute(const Geom& g, const RankBufs& b, const float* labels, const float lam[3],
                         float* loss_out, Status* status, int* nlaunch, const EvRec& rec, cudaStream_t s) {
    if (g.prec == TEM_BF16)
        return conv_launches<__nv_bfloat16>(g, b, labels, lam, loss_out, status, nlaunch, rec, s);
    return conv_launches<float>(g, b, labels, lam, loss_out, status, nlaunch, rec, s);
}

const char* slot_name(int slot) {
    static const char* names[NUM_SLOTS] = {"prep_x", "conv1_fwd", "conv2_fwd", "head_loss", "head_finalize",
                                           "conv2_dgrad", "conv2_wgrad", "conv2_wgrad_reduce",
                                           "conv1_wgrad", "conv1_wgrad_reduce", "exchange", "pem",
                                           "pem_reduce", "exchange_w2", "pgm"};
    return (slot >= 0 && slot < NUM_SLOTS) ? names[slot] : "?";
}

}  // namespace tem
