// prep.cu -- input preparation and small helpers of the TEM step (no GEMMs: those are the
// tcgen05 kernels of tem_umma.cu).
//   prep_x        x [B][T][Cin] -> the halo-padded operand layout [B][T+2][Cin] (bf16 path;
//                 the fp32 path splits into hi / lo planes in prep_x_split_kernel instead)
//   cast_shadow   bf16 operand copy of the weights
//   relu_decisions  the step's ReLU decisions 1[h1 > 0], 1[h2 > 0] (parity tests, reading R7b)
//   empty shard   B = 0: zero gradient, zero loss (the rank still joins the exchange)
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <math.h>

#include "kernels.h"

namespace tem {
namespace {

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

}  // namespace

cudaError_t launch_reduce_splits(const float* part, float* dst, int64_t n, int S, cudaStream_t s) {
    reduce_splits_kernel<<<296, 256, 0, s>>>(part, dst, n, S);
    return cudaGetLastError();
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
                                      const uint64_t* __restrict__ dec2, uint8_t* __restrict__ out, int B,
                                      int Tn, int C) {
    const int64_t n = (int64_t)B * Tn * C;
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n;
         e += (int64_t)gridDim.x * blockDim.x) {
        const int64_t r = e / C;
        const int c = (int)(e - r * C);
        const int64_t v = r / Tn, t = r - v * Tn;
        const int64_t p = v * (Tn + 2) + t + 1;
        out[e] = to_f(h1[p * C + c]) > 0.f ? 1 : 0;
        out[n + e] = dec2 ? (uint8_t)((dec2[p * (C / 64) + c / 64] >> (c % 64)) & 1u)  // fused head
                          : (h2[p * C + c] > 0.f ? 1 : 0);
    }
}

cudaError_t launch_relu_decisions(const Geom& g, const RankBufs& b, uint8_t* out, cudaStream_t s) {
    relu_decisions_kernel<__nv_bfloat16><<<296, 256, 0, s>>>(static_cast<const __nv_bfloat16*>(b.h1), b.h2,
                                                             b.dec2_valid ? b.dec2 : nullptr, out, g.B, g.T, g.C);
    return cudaGetLastError();
}

cudaError_t launch_cast_shadow(const float* params, __nv_bfloat16* shadow, int64_t n, cudaStream_t s) {
    cast_shadow_kernel<<<296, 256, 0, s>>>(params, shadow, n);
    return cudaGetLastError();
}

cudaError_t empty_shard_compute(const Geom& g, const RankBufs& b, const float* labels, const float lam[3],
                                float* loss_out, Status* status, int* nl, const EvRec& rec, cudaStream_t s) {
    cudaError_t e = cudaMemsetAsync(b.grad, 0, (size_t)g.Kpad * sizeof(float), s);
    if (e != cudaSuccess) return e;
    return launch_head(g, b, labels, lam, loss_out, status, rec, s, nl);  // zero loss terms
}

const char* slot_name(int slot) {
    static const char* names[NUM_SLOTS] = {"prep_x", "conv1_fwd", "conv2_fwd", "head_loss", "head_finalize",
                                           "conv2_dgrad", "conv2_wgrad", "conv2_wgrad_reduce",
                                           "conv1_wgrad", "conv1_wgrad_reduce", "exchange", "pem",
                                           "pem_reduce", "exchange_w2", "pgm", "backward"};
    return (slot >= 0 && slot < NUM_SLOTS) ? names[slot] : "?";
}

}  // namespace tem
