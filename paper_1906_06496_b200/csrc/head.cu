// head.cu -- the TEM head and its deterministic reduction.
//
// head_rows_kernel: CTA j owns padded rows [j*RPC, (j+1)*RPC) of the halo layout (a chunk
// spans at most three videos); 8 warps, one snippet row per warp iteration:
//   z_o  = b3[o] + sum_c W3[o][c] h2[c]                           (conv3, k = 1)
//   p_o  = sigmoid(z_o); b = [g > 0.5]; alpha+/- = T / max(l+/-, 1) per video and channel
//   L_o += alpha+ b log p + alpha- (1-b) log(1-p), log p = -softplus(-z), log(1-p) = -softplus(z)
//   dz_o = lambda_o / (B T) * (alpha- (1-b) p - alpha+ b (1-p))    (row a4)
//   dA2  = 1[h2 > 0] * (W3^T dz), stored in the operand format of the path (row a5);
//          halo rows of dA2 are written as zeros
// and per-CTA partials of dW3 = sum dz h2^T, db3 = sum dz, -(1/T) sum L terms, and
// db2 = sum dA2 (the conv2 bias gradient sums the same rounded operand the conv2 weight
// gradient uses).  head_reduce_kernel sums the partials in a fixed order (two levels; the
// last CTA to finish does the second) into the gradient and the four loss outputs, and
// latches NONFINITE.
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <math.h>
#include <stdlib.h>

#include "kernels.h"

namespace tem {
namespace {

constexpr int HEAD_WARPS = 8;
constexpr int NZP_MAX = 8;  // fused-logit partials per row (C / BN of the conv2 epilogue)


TEM_DEV void store4(float* dst, const float (&v)[4]) {
    *reinterpret_cast<float4*>(dst) = make_float4(v[0], v[1], v[2], v[3]);
}
TEM_DEV void store4(__nv_bfloat16* dst, const __nv_bfloat16 (&v)[4]) {
    __nv_bfloat162 a, b;
    a.x = v[0]; a.y = v[1]; b.x = v[2]; b.y = v[3];
    *reinterpret_cast<uint2*>(dst) = make_uint2(*reinterpret_cast<uint32_t*>(&a), *reinterpret_cast<uint32_t*>(&b));
}

// Latency structure: every global load the CTA needs that does not depend on another (W3
// columns, the first batch of h2 rows, the labels, the fused logits) is issued before the
// first barrier, so a CTA costs about one memory round trip plus its arithmetic.  <= 85
// registers: 3 CTAs (768 threads) per SM, and head_rows_per_cta sizes the grid to one wave.
template <typename TOp>
__global__ void __launch_bounds__(256, 3) head_rows_kernel(
    const float* __restrict__ h2, const float* __restrict__ W3, const float* __restrict__ b3,
    const float* __restrict__ labels, float lam0, float lam1, float lam2, TOp* __restrict__ dA2,
    TOp* __restrict__ dA2_lo, float* __restrict__ z_out, float* __restrict__ part, int B, int Tn, int C,
    int RPC, const float* __restrict__ zpart, int nzp) {
    extern __shared__ __align__(16) float sm[];
    trace_begin(SLOT_HEAD);
    pdl_trigger();
    pdl_wait();
    TEM_PHASE_STAMP(2 * NUM_SLOTS, 0);
    float* sW3 = sm;           // [3][C] (only the nzp == 0 path reads it)
    float* sdz = sm + 3 * C;   // [RPC][3] dz of this CTA's rows (0 on halo rows)
    __shared__ float s_ap[3][3], s_an[3][3], s_misc[HEAD_WARPS][6];
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int Tp = Tn + 2, R = B * Tp;
    const int p0 = blockIdx.x * RPC, p1 = min(R, p0 + RPC);
    const int v0 = p0 / Tp, nv = (p1 - 1) / Tp - v0 + 1;  // <= 3 videos
    const float lam[3] = {lam0, lam1, lam2};

    // ---- phase-2 operands first: thread = 4 consecutive columns x one of RP row phases ----
    const int CG = C / 4;            // column groups (<= 128)
    const int RP = blockDim.x / CG;  // row phases (>= 2)
    const int cg = tid % CG, rp = tid / CG;
    const int c0 = 4 * cg;
    const bool act2 = rp < RP;
    constexpr int U = 4;
    float w[3][4];
    float4 hv[U];
    if (act2) {
#pragma unroll
        for (int o = 0; o < 3; ++o) {
            const float4 t = __ldg(reinterpret_cast<const float4*>(W3 + (size_t)o * C + c0));
            w[o][0] = t.x; w[o][1] = t.y; w[o][2] = t.z; w[o][3] = t.w;
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int p = p0 + rp + u * RP;
            hv[u] = p < p1 ? *reinterpret_cast<const float4*>(h2 + (size_t)p * C + c0) : make_float4(0.f, 0.f, 0.f, 0.f);
        }
    }
    // ---- label statistics: one warp per (video, channel); l+ counts strict > 0.5 (R5) ----
    for (int pr = warp; pr < nv * 3; pr += HEAD_WARPS) {
        const int k = pr / 3, o = pr - 3 * k;
        const float* lab = labels + ((size_t)(v0 + k) * 3 + o) * Tn;
        int lp = 0;
#pragma unroll 4
        for (int t0 = 0; t0 < Tn; t0 += 32) {
            const bool pos = (t0 + lane < Tn) && lab[t0 + lane] > 0.5f;
            lp += __popc(__ballot_sync(0xffffffffu, pos));
        }
        if (lane == 0) {
            const int ln = Tn - lp;
            s_ap[k][o] = (float)Tn / (float)(lp > 1 ? lp : 1);
            s_an[k][o] = (float)Tn / (float)(ln > 1 ? ln : 1);
        }
    }
    if (nzp == 0)
        for (int i = tid; i < 3 * C; i += blockDim.x) sW3[i] = W3[i];
    __syncthreads();
    TEM_PHASE_STAMP(2 * NUM_SLOTS, 1);
    // ---- phase 1: z, loss terms, dz -> smem ----
    const int NQ = C / 32;  // <= 16
    float lsum[3] = {0.f, 0.f, 0.f}, dbs[3] = {0.f, 0.f, 0.f};
    const float inv_bt = 1.0f / ((float)B * (float)Tn);
    auto row_loss = [&](int p, const float (&z)[3]) {  // rows a3/a4 for one snippet row
        const int v = p / Tp, t = p - v * Tp - 1, k = v - v0;
        float* dzr = sdz + (p - p0) * 3;
#pragma unroll
        for (int o = 0; o < 3; ++o) {
            const float g = labels[((size_t)v * 3 + o) * Tn + t];
            const float bt = g > 0.5f ? 1.f : 0.f;
            const float ap = s_ap[k][o], an = s_an[k][o];
            float lt, dz;
            head_row_terms(z[o], bt, ap, an, lam[o] * inv_bt, lt, dz);
            lsum[o] += lt;
            dbs[o] += dz;
            dzr[o] = dz;
            z_out[((size_t)v * Tn + t) * 3 + o] = z[o];
        }
    };
    if (nzp > 0) {
        // logits precomputed by the conv2 epilogue: one row per THREAD, partials summed in
        // ascending n-tile order (all loads issued together)
        for (int p = p0 + tid; p < p1; p += blockDim.x) {
            const int tp = p % Tp;
            if (tp == 0 || tp == Tp - 1) {
                sdz[(p - p0) * 3] = sdz[(p - p0) * 3 + 1] = sdz[(p - p0) * 3 + 2] = 0.f;
                continue;
            }
            float zz[NZP_MAX][3];
#pragma unroll
            for (int kk = 0; kk < NZP_MAX; ++kk)
#pragma unroll
                for (int o = 0; o < 3; ++o) zz[kk][o] = kk < nzp ? zpart[((size_t)kk * R + p) * 3 + o] : 0.f;
            float z[3];
#pragma unroll
            for (int o = 0; o < 3; ++o) {
                float sz = zz[0][o];
#pragma unroll
                for (int kk = 1; kk < NZP_MAX; ++kk)
                    if (kk < nzp) sz += zz[kk][o];
                z[o] = sz + b3[o];
            }
            row_loss(p, z);
        }
        // warp-level fixed-order reduction of the per-thread loss / db3 sums
#pragma unroll
        for (int o = 0; o < 3; ++o)
#pragma unroll
            for (int off = 16; off > 0; off >>= 1) {
                lsum[o] += __shfl_xor_sync(0xffffffffu, lsum[o], off);
                dbs[o] += __shfl_xor_sync(0xffffffffu, dbs[o], off);
            }
    } else {
        // one row per warp: z = W3 . h2 by a warp reduction, then the row's loss (lanes redundant)
        for (int p = p0 + warp; p < p1; p += HEAD_WARPS) {
            const int tp = p % Tp;
            if (tp == 0 || tp == Tp - 1) {
                if (lane < 3) sdz[(p - p0) * 3 + lane] = 0.f;
                continue;
            }
            float z[3] = {0.f, 0.f, 0.f};
            for (int q = 0; q < NQ; ++q) {
                const float h = h2[(size_t)p * C + lane + 32 * q];
#pragma unroll
                for (int o = 0; o < 3; ++o) z[o] = fmaf(sW3[o * C + lane + 32 * q], h, z[o]);
            }
#pragma unroll
            for (int o = 0; o < 3; ++o) {
#pragma unroll
                for (int off = 16; off > 0; off >>= 1) z[o] += __shfl_xor_sync(0xffffffffu, z[o], off);
                z[o] += b3[o];
            }
            if (lane == 0) row_loss(p, z);
        }
    }
    if (lane == 0) {
#pragma unroll
        for (int o = 0; o < 3; ++o) {
            s_misc[warp][o] = lsum[o];
            s_misc[warp][3 + o] = dbs[o];
        }
    }
    __syncthreads();
    TEM_PHASE_STAMP(2 * NUM_SLOTS, 2);
    // ---- phase 2: dA2 = 1[h2>0] W3^T dz (halo rows: dz = 0 -> 0); dW3 += dz h2; db2 += stored dA2 ----
    float* dst = part + (size_t)blockIdx.x * (4 * C + 8);  // row stride padded to 16 bytes
    float acc[3][4], bs[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        bs[i] = 0.f;
        acc[0][i] = acc[1][i] = acc[2][i] = 0.f;
    }
    if (act2) {
        for (int pb = p0 + rp; pb < p1; pb += U * RP) {
            if (pb != p0 + rp) {
#pragma unroll
                for (int u = 0; u < U; ++u) {
                    const int p = pb + u * RP;
                    hv[u] = p < p1 ? *reinterpret_cast<const float4*>(h2 + (size_t)p * C + c0)
                                   : make_float4(0.f, 0.f, 0.f, 0.f);
                }
            }
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const int p = pb + u * RP;
                if (p >= p1) break;
                const float* dzr = sdz + (p - p0) * 3;
                const float d0 = dzr[0], d1 = dzr[1], d2 = dzr[2];
                const float h[4] = {hv[u].x, hv[u].y, hv[u].z, hv[u].w};
                TOp dh[4], dl[4];
#pragma unroll
                for (int i = 0; i < 4; ++i) {
                    float d = w[0][i] * d0;
                    d = fmaf(w[1][i], d1, d);
                    d = fmaf(w[2][i], d2, d);
                    const float dv = h[i] > 0.f ? d : 0.f;
                    dh[i] = from_f<TOp>(dv);
                    float st = to_f(dh[i]);
                    if (dA2_lo) {
                        dl[i] = from_f<TOp>(dv - st);
                        st += to_f(dl[i]);
                    }
                    bs[i] += st;
                    acc[0][i] = fmaf(d0, h[i], acc[0][i]);
                    acc[1][i] = fmaf(d1, h[i], acc[1][i]);
                    acc[2][i] = fmaf(d2, h[i], acc[2][i]);
                }
                store4(dA2 + (size_t)p * C + c0, dh);
                if (dA2_lo) store4(dA2_lo + (size_t)p * C + c0, dl);
            }
        }
    }
    // combine the row phases in a fixed order through shared memory (sdz is dead after the sync)
    float* red = sdz;  // [RP][CG][16]
    __syncthreads();
    TEM_PHASE_STAMP(2 * NUM_SLOTS, 3);
    if (act2) {
        float* r = red + ((size_t)rp * CG + cg) * 16;
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            r[i] = acc[0][i];
            r[4 + i] = acc[1][i];
            r[8 + i] = acc[2][i];
            r[12 + i] = bs[i];
        }
    }
    __syncthreads();
    TEM_PHASE_STAMP(2 * NUM_SLOTS, 4);
    if (rp == 0) {
        float sum[16];
#pragma unroll
        for (int k = 0; k < 16; ++k) sum[k] = red[(size_t)cg * 16 + k];
        for (int ph = 1; ph < RP; ++ph)
#pragma unroll
            for (int k = 0; k < 16; ++k) sum[k] += red[((size_t)ph * CG + cg) * 16 + k];
        // partial row layout: [dW3 (3C)][db3 (3)][L (3)][db2 (C)]
        store4(dst + c0, {sum[0], sum[1], sum[2], sum[3]});
        store4(dst + C + c0, {sum[4], sum[5], sum[6], sum[7]});
        store4(dst + 2 * C + c0, {sum[8], sum[9], sum[10], sum[11]});
#pragma unroll
        for (int i = 0; i < 4; ++i) dst[3 * C + 6 + c0 + i] = sum[12 + i];  // offset 3C+6: 8-byte aligned only
    }
    if (tid < 3) {
        float l = s_misc[0][tid], d = s_misc[0][3 + tid];
        for (int w2 = 1; w2 < HEAD_WARPS; ++w2) {
            l += s_misc[w2][tid];
            d += s_misc[w2][3 + tid];
        }
        dst[3 * C + tid] = d;
        dst[3 * C + 3 + tid] = -l / (float)Tn;
    }
    TEM_PHASE_STAMP(2 * NUM_SLOTS, 5);
    trace_end(SLOT_HEAD);
}

// Two-level fixed-order reduction of the P partial rows (n = 4C+6 entries each, stride 4C+8).
// Level 1: CTA (x, y) sums rows [y*P/G, (y+1)*P/G) of entries x*256.. into lvl1[y].
// Level 2: per column block x, the last of its G CTAs sums lvl1[0..G) in order and writes
// those outputs; the block holding the three loss sums also writes loss_out.
__global__ void head_reduce_kernel(const float* __restrict__ part, int P, int C, float* __restrict__ lvl1,
                                   unsigned* __restrict__ counter, float* __restrict__ gW3,
                                   float* __restrict__ gb2, float* __restrict__ loss_out, int B, float lam0,
                                   float lam1, float lam2, Status* status, int64_t* stepctr) {
    trace_begin(SLOT_HEADFIN);
    pdl_trigger();
    pdl_wait();
    const int n = 4 * C + 6, stride = 4 * C + 8;  // entries / padded row stride
    const int G = gridDim.y;
    const int e = blockIdx.x * blockDim.x + threadIdx.x;
    const int r0 = (int)((int64_t)blockIdx.y * P / G), r1 = (int)((int64_t)(blockIdx.y + 1) * P / G);
    if (e < n) {
        float s = 0.f;
#pragma unroll 8
        for (int r = r0; r < r1; ++r) s += part[(size_t)r * stride + e];
        lvl1[(size_t)blockIdx.y * n + e] = s;
    }
    __threadfence();
    __syncthreads();
    __shared__ unsigned s_last;
    if (threadIdx.x == 0) s_last = (atomicAdd(&counter[blockIdx.x], 1u) == (unsigned)G - 1) ? 1u : 0u;
    __syncthreads();
    if (!s_last) return;
    __threadfence();
    __shared__ float s_L[3];
    const int lb = 3 * C + 3;  // first loss entry
    const bool has_loss = (lb >= (int)(blockIdx.x * blockDim.x)) && (lb < (int)((blockIdx.x + 1) * blockDim.x));
    if (e < n) {
        float s = 0.f;
#pragma unroll 8
        for (int g = 0; g < G; ++g) s += __ldcg(&lvl1[(size_t)g * n + e]);
        if (e < 3 * C + 3) gW3[e] = s;                 // dW3 then db3 (contiguous in the flat order)
        else if (e < 3 * C + 6) s_L[e - 3 * C - 3] = s;  // sum over videos of L_o
        else gb2[e - 3 * C - 6] = s;                   // db2
    }
    __syncthreads();
    if (threadIdx.x == 0) counter[blockIdx.x] = 0u;
    if (has_loss && threadIdx.x == 0) {
        float L[3];
        for (int o = 0; o < 3; ++o) L[o] = B > 0 ? s_L[o] / (float)B : 0.f;
        const float tot = lam0 * L[0] + lam1 * L[1] + lam2 * L[2];
        loss_out[0] = tot;
        loss_out[1] = L[0];
        loss_out[2] = L[1];
        loss_out[3] = L[2];
        const int64_t step = *stepctr;
        *stepctr = step + 1;
        if (!isfinite(tot)) latch(status, TEM_ERR_NONFINITE, step);
    }
    trace_end(SLOT_HEADFIN);
}

}  // namespace

TEM_TRACE_SETTER(trace_set_head)

namespace {

int head_rows_per_cta(const Geom& g) {
    // (more, smaller CTAs -- 32 or 16 rows -- measured slower: 37 / 54 vs 27 us at c3)
    int rpc = (g.R + 443) / 444;  // one wave at 3 CTAs per SM
    rpc = (rpc + 7) / 8 * 8;
    if (rpc < 8) rpc = 8;
    if (rpc > 128) rpc = 128;
    return rpc;
}

}  // namespace

int head_ctas(const Geom& g) { return g.R > 0 ? (g.R + head_rows_per_cta(g) - 1) / head_rows_per_cta(g) : 0; }

cudaError_t launch_head_rows(const Geom& g, const RankBufs& b, const float* labels, const float lam[3],
                             const EvRec& rec, cudaStream_t s, int* n) {
    const int P = head_ctas(g);
    const int rpc = head_rows_per_cta(g);
    const size_t red = (size_t)256 * 16;  // phase-2 row-phase reduction [RP][C/4][16]
    const size_t hsm = (size_t)(3 * g.C + (3 * rpc > (int)red ? 3 * rpc : red)) * sizeof(float);
    if (P == 0) return cudaSuccess;
    rec.begin(SLOT_HEAD);
    auto k = head_rows_kernel<__nv_bfloat16>;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)hsm);
    cudaError_t e = launch_pdl(k, dim3(P), dim3(256), hsm, s, false, (const float*)b.h2,
                               (const float*)(b.params + g.off_W3), (const float*)(b.params + g.off_b3), labels, lam[0],
                               lam[1], lam[2], static_cast<__nv_bfloat16*>(b.dA2),
                               static_cast<__nv_bfloat16*>(b.dA2_lo), b.z, b.headpart, g.B, g.T, g.C, rpc,
                               (const float*)b.zpart, b.nzpart);
    rec.end(SLOT_HEAD);
    ++*n;
    return e;
}

cudaError_t launch_head_reduce(const Geom& g, const RankBufs& b, const float lam[3], float* loss_out,
                               Status* status, const EvRec& rec, cudaStream_t s, int* n) {
    return launch_head_reduce_rows(g, b, head_ctas(g), lam, loss_out, status, rec, s, n);
}

// Sum `P` partial rows ([P][4C + 8]: head_rows CTAs, or the fused-head row tiles).
cudaError_t launch_head_reduce_rows(const Geom& g, const RankBufs& b, int P, const float lam[3], float* loss_out,
                                    Status* status, const EvRec& rec, cudaStream_t s, int* n) {
    rec.begin(SLOT_HEADFIN);
    const int nent = 4 * g.C + 6;
    const int G = P >= 128 ? 16 : (P >= 16 ? 4 : 1);
    cudaError_t e = launch_pdl(head_reduce_kernel, dim3((nent + 255) / 256, G), dim3(256), 0, s, true,
                               (const float*)b.headpart, P, g.C, b.headlvl1, b.counter, b.grad + g.off_W3,
                               b.grad + g.off_b2, loss_out, g.B, lam[0], lam[1], lam[2], status, b.stepctr);
    rec.end(SLOT_HEADFIN);
    ++*n;
    return e;
}

cudaError_t launch_head(const Geom& g, const RankBufs& b, const float* labels, const float lam[3],
                        float* loss_out, Status* status, const EvRec& rec, cudaStream_t s, int* n) {
    cudaError_t e = launch_head_rows(g, b, labels, lam, rec, s, n);
    if (e != cudaSuccess) return e;
    return launch_head_reduce(g, b, lam, loss_out, status, rec, s, n);
}

}  // namespace tem
