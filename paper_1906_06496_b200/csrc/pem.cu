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


}  // namespace

TEM_TRACE_SETTER(trace_set_pem)

// Partial-buffer rows (of K_pem + 1 floats) the workspace reserves: one per CTA.
// All SMs, on the critical path right after prep_x.  Measured alternatives
// (scripts/probes/step_trace.py --workload c5): on a graph branch of its own (16 CTAs beside
// the TEM step) steps were ~20 us slower and occasionally stalled for milliseconds; more CTAs
// there took SMs conv2's 8-CTA clusters need.  A hidden-unit split (CTA j owns 4 units over
// all proposals) measured slower (21.3 + 20.8 vs 18.7 + 8.5 us) and was removed.
int pem_ctas(const Geom& g) {
    const int M = g.B * g.pem_P;
    if (M <= 0) return 0;
    int G = (M + 13) / 14;  // 14 proposals per CTA
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
    const int G = pem_ctas(g);
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
