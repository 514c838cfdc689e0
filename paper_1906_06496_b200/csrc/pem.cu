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

#include "kernels.h"

namespace tem {
namespace {

constexpr int PEM_F = 32, PEM_H = 512, PEM_THREADS = 256, PEM_RB = 8;  // rows per batch

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
    const float* W1 = prm;
    const float* b1 = prm + PEM_H * PEM_F;
    const float* w2 = b1 + PEM_H;
    const float b2 = w2[PEM_H];
    float w[2][PEM_F], acc[2][PEM_F];
    float bb[2], ww[2], gb[2] = {0.f, 0.f}, gw[2] = {0.f, 0.f};
    {
        // W1 rows via shared memory: fully coalesced loads (consecutive threads, consecutive
        // floats), then each thread reads its two rows from a 33-float padded layout (conflict
        // free).  Direct row loads were 32 cache lines per warp instruction.
        extern __shared__ float w1s[];  // [H][F + 1]
        for (int i = tid; i < PEM_H * PEM_F; i += PEM_THREADS) {
            const int j = i / PEM_F, k = i - j * PEM_F;
            w1s[j * (PEM_F + 1) + k] = __ldg(W1 + i);
        }
        __syncthreads();
#pragma unroll
        for (int u = 0; u < 2; ++u) {
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
        {
            const int r = tid / PEM_F, k = tid % PEM_F;
            fs[r][k] = r < nr ? f[(size_t)(mb + r) * PEM_F + k] : 0.f;
        }
        __syncthreads();
        float h[PEM_RB][2];
        bool pos[PEM_RB][2];
#pragma unroll
        for (int r = 0; r < PEM_RB; ++r) {
            float zp = 0.f;
#pragma unroll
            for (int u = 0; u < 2; ++u) {
                float a = bb[u];
#pragma unroll
                for (int k = 0; k < PEM_F; ++k) a = fmaf(w[u][k], fs[r][k], a);
                pos[r][u] = a > 0.f;
                h[r][u] = pos[r][u] ? a : 0.f;
                if (dec_out && r < nr) dec_out[(size_t)(mb + r) * PEM_H + tid + u * PEM_THREADS] = pos[r][u] ? 1 : 0;
            }
            zp = fmaf(ww[1], h[r][1], ww[0] * h[r][0]);
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
            for (int u = 0; u < 2; ++u) {
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
#pragma unroll
    for (int u = 0; u < 2; ++u) {
        const int j = tid + u * PEM_THREADS;
#pragma unroll
        for (int k = 0; k < PEM_F; ++k) dst[(size_t)j * PEM_F + k] = acc[u][k];
        dst[PEM_H * PEM_F + j] = gb[u];
        dst[PEM_H * PEM_F + PEM_H + j] = gw[u];
    }
    if (tid == 0) {
        dst[KP - 1] = gb2;
        dst[KP] = lsum;
    }
    trace_end(SLOT_PEM);
}

// grad[e] = sum over CTA partials in CTA order; loss = sum_j L_j / M; NONFINITE latch.
__global__ void pem_reduce_kernel(const float* __restrict__ part, int G, int M, float* __restrict__ grad,
                                  float* __restrict__ loss_out, Status* status, const int64_t* stepctr) {
    trace_begin(SLOT_PEMRED);
    pdl_trigger();
    pdl_wait();
    constexpr int KP = PEM_H * PEM_F + 2 * PEM_H + 1;
    const int e = blockIdx.x * blockDim.x + threadIdx.x;
    if (e <= KP) {
        float s = 0.f;
        for (int j = 0; j < G; ++j) s += part[(size_t)j * (KP + 1) + e];
        if (e < KP) {
            grad[e] = s;
        } else {
            const float L = M > 0 ? s / (float)M : 0.f;
            *loss_out = L;
            if (!isfinite(L)) latch(status, TEM_ERR_NONFINITE, stepctr ? *stepctr : 0);
        }
    }
    trace_end(SLOT_PEMRED);
}

}  // namespace

void trace_set_pem(unsigned long long* p) { cudaMemcpyToSymbol(g_trace, &p, sizeof(p)); }

int pem_ctas(const Geom& g) {
    const int M = g.B * g.pem_P;
    if (M <= 0) return 0;
    // All SMs, on the critical path right after prep_x.  Measured alternatives
    // (scripts/probes/step_trace.py --workload c5): on a graph branch of its own (16 CTAs
    // beside the TEM step) steps were ~20 us slower and occasionally stalled for milliseconds;
    // more CTAs there took SMs conv2's 8-CTA clusters need.
    int G = (M + 13) / 14;
    if (G > 148) G = 148;
    return G;
}

cudaError_t launch_pem(const Geom& g, const float* f, const float* iou, const float* params, float* part,
                       float* grad, float* loss_out, Status* status, const int64_t* stepctr, uint8_t* dec_out,
                       cudaStream_t s, cudaStream_t s_red, cudaEvent_t fork, int* n, const EvRec& rec) {
    const int M = g.B * g.pem_P;
    const int G = pem_ctas(g);
    if (G == 0) {
        cudaError_t e = cudaMemsetAsync(grad, 0, sizeof(float) * (size_t)pem_num_params_of(g), s);
        if (e == cudaSuccess) e = cudaMemsetAsync(loss_out, 0, sizeof(float), s);
        return e;
    }
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
    e = launch_pdl(pem_reduce_kernel, dim3((KP + 1 + 255) / 256), dim3(256), 0, s_red, true, (const float*)part, G, M, grad,
                   loss_out, status, stepctr);
    rec.end(SLOT_PEMRED);
    if (e == cudaSuccess) ++*n;
    return e;
}

}  // namespace tem
