// pem.cu -- BSN's proposal evaluation module (PEM), the second model of the joint TEM + PEM
// data-parallel step (BASELINE configs[4]; readings R19-R21).
//
// Per proposal m (M = B * P per rank) with BSP feature f_m (F = 32) and IoU target g_m:
//   a = W1 f_m + b1 (H = 512),  h = ReLU(a),  y = sigmoid(w2 . h + b2),
//   L = (1/M) sum_m (y - g)^2,  dz = (2/M)(y - g) y (1 - y),
//   dw2 += dz h,  db2 += dz,  dh = 1[a > 0] dz w2,  dW1 += dh f^T,  db1 += dh.
//
// pem_kernel: CTA j owns a contiguous range of proposals; each of its 256 threads owns two
// hidden units (j = tid, tid + 256) with their W1 rows in registers, so the forward dot
// products and the dW1 outer-product accumulation need no shared-memory traffic beyond the
// 8-row feature tile.  The logit of a row is a fixed-order reduction (warp xor tree, then the
// 8 warps in order).  Each CTA writes one partial row [dW1 | db1 | dw2 | db2 | sum (y-g)^2];
// pem_reduce_kernel sums the partial rows in CTA order (deterministic) into the gradient and
// the loss.  The work is 4 F H = 65,536 FLOP per proposal: a SIMT (ALU) kernel -- K = 32 is
// too short a contraction for the tensor cores to pay, and it runs on the side branch beside
// the TEM GEMMs.
#include <cuda_runtime.h>
#include <math.h>
#include <stdlib.h>

#include "kernels.h"

namespace tem {
namespace {

// PEM_U hidden units per thread (PEM_U = 1: 512 threads at ~110 registers, 16 warps per SM;
// PEM_U = 2 ran 256 threads at 222 registers, 8 warps, latency-bound at IPC 0.6)
constexpr int PEM_F = 32, PEM_H = 512, PEM_U = 1, PEM_THREADS = PEM_H / PEM_U, PEM_RB = 8;  // rows per batch

__global__ void __launch_bounds__(PEM_THREADS, 1) pem_kernel(const float* __restrict__ f, const float* __restrict__ g,
                                                          const float* __restrict__ prm, int M, int rows_per_cta,
                                                          float* __restrict__ part, uint8_t* __restrict__ dec_out) {
    trace_begin(SLOT_PEM);
    pdl_trigger();
    pdl_wait();
    constexpr int KP = PEM_H * PEM_F + 2 * PEM_H + 1;
    __shared__ float fs[PEM_RB][PEM_F];
    __shared__ float zred[PEM_RB][PEM_THREADS / 32];
    __shared__ float dzs[PEM_RB];
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    extern __shared__ float w1s[];  // [H][F + 1]: W1 staging, then the dW1 partial's transpose
    const float* W1 = prm;
    const float* b1 = prm + PEM_H * PEM_F;
    const float* w2 = b1 + PEM_H;
    const float b2 = w2[PEM_H];
    float w[PEM_U][PEM_F], acc[PEM_U][PEM_F];
    float bb[PEM_U], ww[PEM_U], gb[PEM_U], gw[PEM_U];
#pragma unroll
    for (int u = 0; u < PEM_U; ++u) gb[u] = gw[u] = 0.f;
    {
        // W1 rows via shared memory: fully coalesced loads (consecutive threads, consecutive
        // floats), then each thread reads its rows from a 33-float padded layout (conflict
        // free).  Direct row loads were 32 cache lines per warp instruction.
        // All loads of a thread are issued before its first shared store (the rolled loop
        // waited on every load: 40 % of the kernel's stall samples).  Scalar: W1 starts at the
        // flat offset off_pem, not 16-byte aligned.
        constexpr int NV = PEM_H * PEM_F / PEM_THREADS;
        float v[NV];
#pragma unroll
        for (int q = 0; q < NV; ++q) v[q] = __ldg(W1 + tid + q * PEM_THREADS);
#pragma unroll
        for (int q = 0; q < NV; ++q) {
            const int i = tid + q * PEM_THREADS, j = i / PEM_F, k = i - j * PEM_F;
            w1s[j * (PEM_F + 1) + k] = v[q];
        }
        __syncthreads();
#pragma unroll
        for (int u = 0; u < PEM_U; ++u) {
            const int j = tid + u * PEM_THREADS;
#pragma unroll
            for (int k = 0; k < PEM_F; ++k) w[u][k] = w1s[j * (PEM_F + 1) + k];
#pragma unroll
            for (int k = 0; k < PEM_F; ++k) acc[u][k] = 0.f;
            bb[u] = b1[j];
            ww[u] = w2[j];
        }
    }
    float gb2 = 0.f, lsum = 0.f;  // thread 0
    const int m0 = blockIdx.x * rows_per_cta, m1 = min(M, m0 + rows_per_cta);
    const float twoM = 2.0f / (float)M;
    for (int mb = m0; mb < m1; mb += PEM_RB) {
        const int nr = min(PEM_RB, m1 - mb);
        // feature tile: 8 rows x 32 = 256 floats, one per thread
        if (tid < PEM_RB * PEM_F) {
            const int r = tid / PEM_F, k = tid % PEM_F;
            fs[r][k] = r < nr ? f[(size_t)(mb + r) * PEM_F + k] : 0.f;
        }
        __syncthreads();
        float h[PEM_RB][PEM_U];
        bool pos[PEM_RB][PEM_U];
#pragma unroll
        for (int r = 0; r < PEM_RB; ++r) {
            float zp = 0.f;
#pragma unroll
            for (int u = 0; u < PEM_U; ++u) {
                float a = bb[u];
#pragma unroll
                for (int k = 0; k < PEM_F; ++k) a = fmaf(w[u][k], fs[r][k], a);
                pos[r][u] = a > 0.f;
                h[r][u] = pos[r][u] ? a : 0.f;
                if (dec_out && r < nr) dec_out[(size_t)(mb + r) * PEM_H + tid + u * PEM_THREADS] = pos[r][u] ? 1 : 0;
            }
            zp = ww[0] * h[r][0];
#pragma unroll
            for (int u = 1; u < PEM_U; ++u) zp = fmaf(ww[u], h[r][u], zp);
#pragma unroll
            for (int off = 16; off > 0; off >>= 1) zp += __shfl_xor_sync(0xffffffffu, zp, off);
            if (lane == 0) zred[r][warp] = zp;
        }
        __syncthreads();
        if (tid < nr) {
            float z = b2;
#pragma unroll
            for (int q = 0; q < PEM_THREADS / 32; ++q) z += zred[tid][q];
            const float y = 1.f / (1.f + expf(-z));
            const float e = y - g[mb + tid];
            dzs[tid] = twoM * e * y * (1.f - y);
            zred[tid][0] = e * e;  // loss term of row tid (the row's reduction is consumed)
        }
        __syncthreads();
        if (tid == 0)
            for (int r = 0; r < nr; ++r) {
                lsum += zred[r][0];
                gb2 += dzs[r];
            }
#pragma unroll
        for (int r = 0; r < PEM_RB; ++r) {
            if (r >= nr) break;
            const float d = dzs[r];
#pragma unroll
            for (int u = 0; u < PEM_U; ++u) {
                gw[u] = fmaf(d, h[r][u], gw[u]);
                const float dh = pos[r][u] ? d * ww[u] : 0.f;
                gb[u] += dh;
#pragma unroll
                for (int k = 0; k < PEM_F; ++k) acc[u][k] = fmaf(dh, fs[r][k], acc[u][k]);
            }
        }
        __syncthreads();  // fs / zred / dzs reused by the next batch
    }
    float* dst = part + (size_t)blockIdx.x * (KP + 1);
    // dW1 rows through the padded shared buffer so the global stores are coalesced (a thread's
    // own 32-float row was 32 sectors per warp store)
#pragma unroll
    for (int u = 0; u < PEM_U; ++u) {
        const int j = tid + u * PEM_THREADS;
#pragma unroll
        for (int k = 0; k < PEM_F; ++k) w1s[j * (PEM_F + 1) + k] = acc[u][k];
        dst[PEM_H * PEM_F + j] = gb[u];
        dst[PEM_H * PEM_F + PEM_H + j] = gw[u];
    }
    __syncthreads();
    for (int i = tid; i < PEM_H * PEM_F; i += PEM_THREADS) {
        const int j = i / PEM_F, k = i - j * PEM_F;
        dst[i] = w1s[j * (PEM_F + 1) + k];
    }
    if (tid == 0) {
        dst[KP - 1] = gb2;
        dst[KP] = lsum;
    }
    trace_end(SLOT_PEM);
}

// grad[e] = sum over the G CTA partials; loss = sum_j L_j / M; NONFINITE latch.  A CTA of 8
// warps owns 32 consecutive elements: warp w sums the partials j = w, w + 8, ... in ascending j
// (coalesced 128-byte rows), then the 8 warp sums are added in warp order -- a fixed order,
// so the result is deterministic.  (One thread per element summing all G serially was
// 10.6 us for 10 MB at c5.)
constexpr int PEMRED_W = 8;
__global__ void __launch_bounds__(32 * PEMRED_W) pem_reduce_kernel(const float* __restrict__ part, int G, int M,
                                                                   float* __restrict__ grad, float* __restrict__ loss_out,
                                                                   Status* status, const int64_t* stepctr) {
    trace_begin(SLOT_PEMRED);
    pdl_trigger();
    pdl_wait();
    constexpr int KP = PEM_H * PEM_F + 2 * PEM_H + 1;
    __shared__ float ws[PEMRED_W][32];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int e = blockIdx.x * 32 + lane;
    float s = 0.f;
    if (e <= KP) {
        int j = warp;
        for (; j + 3 * PEMRED_W < G; j += 4 * PEMRED_W) {  // 4 loads in flight per lane
            const float a0 = __ldcs(part + (size_t)j * (KP + 1) + e);
            const float a1 = __ldcs(part + (size_t)(j + PEMRED_W) * (KP + 1) + e);
            const float a2 = __ldcs(part + (size_t)(j + 2 * PEMRED_W) * (KP + 1) + e);
            const float a3 = __ldcs(part + (size_t)(j + 3 * PEMRED_W) * (KP + 1) + e);
            s += a0;
            s += a1;
            s += a2;
            s += a3;
        }
        for (; j < G; j += PEMRED_W) s += __ldcs(part + (size_t)j * (KP + 1) + e);
    }
    ws[warp][lane] = s;
    __syncthreads();
    if (warp == 0 && e <= KP) {
        float t = ws[0][lane];
#pragma unroll
        for (int w = 1; w < PEMRED_W; ++w) t += ws[w][lane];
        if (e < KP) {
            grad[e] = t;
        } else {
            const float L = M > 0 ? t / (float)M : 0.f;
            *loss_out = L;
            if (!isfinite(L)) latch(status, TEM_ERR_NONFINITE, stepctr ? *stepctr : 0);
        }
    }
    trace_end(SLOT_PEMRED);
}


// ---------------------------------------------------------------------------------------
// Hidden-unit split (opt-in, TEM_PEM_UNITSPLIT=1; slower, see pem_rowsplit()): CTA j owns the PEM_US hidden units [PEM_US j, PEM_US j + PEM_US)
// for ALL M proposals, so dW1 / db1 / dw2 of its units are complete inside the CTA and no
// per-CTA partial rows of the whole gradient are written or reduced (the row split wrote
// 147 x 70 KB and summed them: ~25 us at c5).  Three kernels:
//   pem_fwd_kernel : zpart[j][m] = sum_{u in j} w2_u ReLU(a_mu), a_mu = b1_u + W1_u . f_m
//   pem_dz_kernel  : z_m = b2 + sum_j zpart[j][m] (j ascending), y, dz_m, per-CTA (db2, sum e^2)
//   pem_bwd_kernel : recomputes a_mu with the same code (same decisions), dh = 1[a>0] dz w2_u,
//                    dW1_u = sum_m dh f_m, db1_u = sum_m dh, dw2_u = sum_m dz h; CTA 0 adds db2
//                    and the loss.  Every sum is a fixed-order tree (deterministic).
constexpr int PEM_US = 4, PEM_UG = PEM_H / PEM_US, PEM_T2 = 256;

// a = b + W . f for one unit, W row from shared memory (broadcast reads), fixed k order
TEM_DEV float pem_preact(const float* __restrict__ wrow, float b, const float (&f)[PEM_F]) {
    float a = b;
#pragma unroll
    for (int k = 0; k < PEM_F; ++k) a = fmaf(wrow[k], f[k], a);
    return a;
}

// Rows [m0, m0 + PEM_T2) of f into a padded shared tile with coalesced loads (a thread loading
// its own 128-byte row touched 32 lines per warp load: ~50 us per kernel at c5); then every
// thread reads its row conflict-free.  All threads call (two barriers).
TEM_DEV void pem_tile(const float* __restrict__ f, int M, int m0, float (*ft)[PEM_F + 1]) {
    __syncthreads();  // the previous tile is consumed
    const int nrow = min(PEM_T2, M - m0);
    constexpr int NV = PEM_T2 * PEM_F / 4 / PEM_T2;  // float4 per thread, all in flight at once
    float4 v[NV];
    const float4* src = reinterpret_cast<const float4*>(f + (size_t)m0 * PEM_F);
#pragma unroll
    for (int q = 0; q < NV; ++q) {
        const int i = threadIdx.x + q * PEM_T2;  // float4 index in the tile
        v[q] = (i * 4) / PEM_F < nrow ? __ldg(src + i) : make_float4(0.f, 0.f, 0.f, 0.f);
    }
#pragma unroll
    for (int q = 0; q < NV; ++q) {
        const int i = 4 * (threadIdx.x + q * PEM_T2), r = i / PEM_F, k = i - r * PEM_F;
        ft[r][k] = v[q].x;
        ft[r][k + 1] = v[q].y;
        ft[r][k + 2] = v[q].z;
        ft[r][k + 3] = v[q].w;
    }
    __syncthreads();
}

TEM_DEV void pem_load_row(const float* __restrict__ fm, float (&f)[PEM_F]) {
#pragma unroll
    for (int k = 0; k < PEM_F; ++k) f[k] = fm[k];
}

__global__ void __launch_bounds__(PEM_T2) pem_fwd_kernel(const float* __restrict__ f, const float* __restrict__ prm,
                                                         int M, float* __restrict__ zpart,
                                                         uint8_t* __restrict__ dec_out) {
    trace_begin(SLOT_PEM);
    pdl_trigger();
    pdl_wait();
    __shared__ float ws[PEM_US][PEM_F];
    const int j = blockIdx.x, u0 = j * PEM_US, tid = threadIdx.x;
    const float* W1 = prm;
    const float* b1 = prm + PEM_H * PEM_F;
    const float* w2 = b1 + PEM_H;
    if (tid < PEM_US * PEM_F) ws[tid / PEM_F][tid % PEM_F] = W1[(size_t)u0 * PEM_F + tid];
    __syncthreads();
    float bb[PEM_US], ww[PEM_US];
#pragma unroll
    for (int u = 0; u < PEM_US; ++u) {
        bb[u] = b1[u0 + u];
        ww[u] = w2[u0 + u];
    }
    __shared__ float ft[PEM_T2][PEM_F + 1];
    for (int m0 = 0; m0 < M; m0 += PEM_T2) {
        pem_tile(f, M, m0, ft);
        const int m = m0 + tid;
        if (m >= M) continue;
        float fr[PEM_F];
        pem_load_row(ft[tid], fr);
        float zp = 0.f;
#pragma unroll
        for (int u = 0; u < PEM_US; ++u) {
            const float a = pem_preact(ws[u], bb[u], fr);
            if (dec_out) dec_out[(size_t)m * PEM_H + u0 + u] = a > 0.f ? 1 : 0;
            zp = fmaf(ww[u], a > 0.f ? a : 0.f, zp);
        }
        zpart[(size_t)j * M + m] = zp;
    }
    trace_end(SLOT_PEM);
}

// 32 rows per CTA: warp w sums the unit-group partials j = w, w + 8, ... of its lanes' rows
// (coalesced, 4 loads in flight), then the 8 warp sums in warp order (fixed order)
constexpr int PEMDZ_ROWS = 32;
__global__ void __launch_bounds__(PEM_T2) pem_dz_kernel(const float* __restrict__ zpart, const float* __restrict__ g,
                                                        const float* __restrict__ prm, int M, float* __restrict__ dz,
                                                        float* __restrict__ cpart) {
    pdl_trigger();
    pdl_wait();
    constexpr int NW = PEM_T2 / 32;
    __shared__ float zs[NW][PEMDZ_ROWS];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int m = blockIdx.x * PEMDZ_ROWS + lane;
    float zp = 0.f;
    if (m < M) {
        int j = warp;
        for (; j + 3 * NW < PEM_UG; j += 4 * NW) {
            const float a0 = zpart[(size_t)j * M + m], a1 = zpart[(size_t)(j + NW) * M + m];
            const float a2 = zpart[(size_t)(j + 2 * NW) * M + m], a3 = zpart[(size_t)(j + 3 * NW) * M + m];
            zp += a0;
            zp += a1;
            zp += a2;
            zp += a3;
        }
        for (; j < PEM_UG; j += NW) zp += zpart[(size_t)j * M + m];
    }
    zs[warp][lane] = zp;
    __syncthreads();
    if (warp == 0) {
        float d = 0.f, l2 = 0.f;
        if (m < M) {
            float z = prm[PEM_H * PEM_F + 2 * PEM_H];  // b2
#pragma unroll
            for (int w = 0; w < NW; ++w) z += zs[w][lane];
            const float y = 1.f / (1.f + expf(-z));
            const float e = y - g[m];
            d = (2.0f / (float)M) * e * y * (1.f - y);
            l2 = e * e;
            dz[m] = d;
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            d += __shfl_xor_sync(0xffffffffu, d, o);
            l2 += __shfl_xor_sync(0xffffffffu, l2, o);
        }
        if (lane == 0) {
            cpart[2 * blockIdx.x] = d;
            cpart[2 * blockIdx.x + 1] = l2;
        }
    }
}

__global__ void __launch_bounds__(PEM_T2) pem_bwd_kernel(const float* __restrict__ f, const float* __restrict__ prm,
                                                         const float* __restrict__ dz, const float* __restrict__ cpart,
                                                         int ncp, int M, float* __restrict__ grad,
                                                         float* __restrict__ loss_out, Status* status,
                                                         const int64_t* stepctr) {
    trace_begin(SLOT_PEMRED);
    pdl_trigger();
    pdl_wait();
    constexpr int NV = PEM_US * PEM_F + 2 * PEM_US;  // dW1 slice, db1, dw2 of this CTA's units
    __shared__ float ws[PEM_US][PEM_F];
    __shared__ float wsum[PEM_T2 / 32][NV];
    const int j = blockIdx.x, u0 = j * PEM_US, tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const float* W1 = prm;
    const float* b1 = prm + PEM_H * PEM_F;
    const float* w2 = b1 + PEM_H;
    if (tid < PEM_US * PEM_F) ws[tid / PEM_F][tid % PEM_F] = W1[(size_t)u0 * PEM_F + tid];
    __syncthreads();
    float bb[PEM_US], ww[PEM_US];
#pragma unroll
    for (int u = 0; u < PEM_US; ++u) {
        bb[u] = b1[u0 + u];
        ww[u] = w2[u0 + u];
    }
    float acc[NV];
#pragma unroll
    for (int q = 0; q < NV; ++q) acc[q] = 0.f;
    __shared__ float ft[PEM_T2][PEM_F + 1];
    for (int m0 = 0; m0 < M; m0 += PEM_T2) {
        pem_tile(f, M, m0, ft);
        const int m = m0 + tid;
        if (m >= M) continue;
        float fr[PEM_F];
        pem_load_row(ft[tid], fr);
        const float d = dz[m];
#pragma unroll
        for (int u = 0; u < PEM_US; ++u) {
            const float a = pem_preact(ws[u], bb[u], fr);  // same code as pem_fwd_kernel
            const bool pos = a > 0.f;
            const float dh = pos ? d * ww[u] : 0.f;
#pragma unroll
            for (int k = 0; k < PEM_F; ++k) acc[u * PEM_F + k] = fmaf(dh, fr[k], acc[u * PEM_F + k]);
            acc[PEM_US * PEM_F + u] += dh;
            acc[PEM_US * PEM_F + PEM_US + u] = fmaf(d, pos ? a : 0.f, acc[PEM_US * PEM_F + PEM_US + u]);
        }
    }
    // fixed-order CTA reduction: warp xor trees, then the warps in order
#pragma unroll
    for (int q = 0; q < NV; ++q) {
        float v = acc[q];
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
        if (lane == 0) wsum[warp][q] = v;
    }
    __syncthreads();
    if (tid < NV) {
        float t = 0.f;
#pragma unroll
        for (int w = 0; w < PEM_T2 / 32; ++w) t += wsum[w][tid];
        if (tid < PEM_US * PEM_F) grad[(size_t)u0 * PEM_F + tid] = t;                   // W1 rows u0..
        else if (tid < PEM_US * PEM_F + PEM_US) grad[PEM_H * PEM_F + u0 + (tid - PEM_US * PEM_F)] = t;  // b1
        else grad[PEM_H * PEM_F + PEM_H + u0 + (tid - PEM_US * PEM_F - PEM_US)] = t;    // w2
    }
    if (j == 0 && tid == 0) {  // db2 and the loss from the dz kernel's CTA partials, in order
        float sd = 0.f, sl = 0.f;
        for (int q = 0; q < ncp; ++q) {
            sd += cpart[2 * q];
            sl += cpart[2 * q + 1];
        }
        grad[PEM_H * PEM_F + 2 * PEM_H] = sd;
        const float L = M > 0 ? sl / (float)M : 0.f;
        *loss_out = L;
        if (!isfinite(L)) latch(status, TEM_ERR_NONFINITE, stepctr ? *stepctr : 0);
    }
    trace_end(SLOT_PEMRED);
}

}  // namespace

void trace_set_pem(unsigned long long* p) { cudaMemcpyToSymbol(g_trace, &p, sizeof(p)); }

int pem_rowsplit_ctas(const Geom& g);

// Partial-buffer rows (of K_pem + 1 floats) the workspace reserves: the row split's per-CTA
// partials, or the unit split's zpart [PEM_UG][M] + dz [M] + dz-kernel partials.
int pem_ctas(const Geom& g) {
    const int M = g.B * g.pem_P;
    if (M <= 0) return 0;
    const int64_t row = pem_num_params_of(g) + 1;
    const int64_t unit = (int64_t)PEM_UG * M + M + 2 * ((M + 31) / 32);
    const int rows_split = pem_rowsplit_ctas(g);
    const int unit_rows = (int)((unit + row - 1) / row);
    return rows_split > unit_rows ? rows_split : unit_rows;
}

static bool pem_rowsplit() {
    // the hidden-unit split (TEM_PEM_UNITSPLIT=1) measured slower at c5: fwd + dz 21.3 us and
    // bwd 20.8 us with 4 units per CTA (23 + 23 with 2) vs 18.7 + 8.5 us for the row split --
    // one CTA per SM re-reading all M feature rows is latency-bound at 8 warps
    return getenv("TEM_PEM_UNITSPLIT") == nullptr;  // read per launch (tests switch it)
}

int pem_rowsplit_ctas(const Geom& g) {
    const int M = g.B * g.pem_P;
    if (M <= 0) return 0;
    // All SMs, on the critical path right after prep_x.  Measured alternatives
    // (scripts/probes/step_trace.py --workload c5): on a graph branch of its own (16 CTAs
    // beside the TEM step) steps were ~20 us slower and occasionally stalled for milliseconds;
    // more CTAs there took SMs conv2's 8-CTA clusters need.
    static const int rows_env = [] {
        const char* e = getenv("TEM_PEM_ROWS");  // (experiments) proposals per CTA
        return e ? atoi(e) : 0;
    }();
    const int per = rows_env > 0 ? rows_env : 14;
    int G = (M + per - 1) / per;
    if (G > 148) G = 148;
    return G;
}

cudaError_t launch_pem(const Geom& g, const float* f, const float* iou, const float* params, float* part,
                       float* grad, float* loss_out, Status* status, const int64_t* stepctr, uint8_t* dec_out,
                       cudaStream_t s, cudaStream_t s_red, cudaEvent_t fork, int* n, const EvRec& rec) {
    const int M = g.B * g.pem_P;
    if (pem_ctas(g) == 0) {
        cudaError_t e = cudaMemsetAsync(grad, 0, sizeof(float) * (size_t)pem_num_params_of(g), s);
        if (e == cudaSuccess) e = cudaMemsetAsync(loss_out, 0, sizeof(float), s);
        return e;
    }
    if (!pem_rowsplit()) {  // hidden-unit split (experiment)
        float* zpart = part;
        float* dz = zpart + (size_t)PEM_UG * M;
        float* cpart = dz + M;
        const int ndz = (M + PEMDZ_ROWS - 1) / PEMDZ_ROWS;
        rec.begin(SLOT_PEM);
        cudaError_t e = launch_pdl(pem_fwd_kernel, dim3(PEM_UG), dim3(PEM_T2), 0, s, false, f, params, M, zpart, dec_out);
        if (e == cudaSuccess)
            e = launch_pdl(pem_dz_kernel, dim3(ndz), dim3(PEM_T2), 0, s, false, (const float*)zpart, iou, params, M, dz,
                           cpart);
        rec.end(SLOT_PEM);
        if (e != cudaSuccess) return e;
        *n += 2;
        rec.begin(SLOT_PEMRED);
        e = launch_pdl(pem_bwd_kernel, dim3(PEM_UG), dim3(PEM_T2), 0, s, false, f, params, (const float*)dz,
                       (const float*)cpart, ndz, M, grad, loss_out, status, stepctr);
        rec.end(SLOT_PEMRED);
        if (e == cudaSuccess) ++*n;
        return e;
    }
    const int G = pem_rowsplit_ctas(g);
    const int rows = (M + G - 1) / G;
    // pem_kernel on the caller's (critical-path) stream with programmatic dependent launch;
    // pem_reduce follows a cross-stream event and launches without it
    constexpr size_t W1S = sizeof(float) * PEM_H * (PEM_F + 1);  // 67.6 KB staging
    static bool attr = false;
    if (!attr) {
        cudaError_t ea = cudaFuncSetAttribute(pem_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)W1S);
        if (ea != cudaSuccess) return ea;
        attr = true;
    }
    rec.begin(SLOT_PEM);
    cudaError_t e = launch_pdl(pem_kernel, dim3(G), dim3(PEM_THREADS), W1S, s, false, f, iou, params, M, rows, part,
                               dec_out);
    rec.end(SLOT_PEM);
    if (e != cudaSuccess) return e;
    ++*n;
    if (s_red != s && fork &&
        (cudaEventRecord(fork, s) != cudaSuccess || cudaStreamWaitEvent(s_red, fork, 0) != cudaSuccess))
        return cudaErrorUnknown;
    const int KP = (int)pem_num_params_of(g);
    rec.begin(SLOT_PEMRED);
    e = launch_pdl(pem_reduce_kernel, dim3((KP + 1 + 31) / 32), dim3(32 * PEMRED_W), 0, s_red, true, (const float*)part, G, M, grad,
                   loss_out, status, stepctr);
    rec.end(SLOT_PEMRED);
    if (e == cudaSuccess) ++*n;
    return e;
}

}  // namespace tem
