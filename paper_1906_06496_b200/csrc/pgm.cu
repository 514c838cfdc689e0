// pgm.cu -- BSN's proposal generation module (PGM) on the GPU: candidate boundaries, ranked
// proposals, 32-d Boundary-Sensitive Proposal features and IoU targets, the data path that
// feeds PEM (reading R24; the paper names the stage at P:85).
//
// One CTA of 1024 threads per video (T <= 128):
//   1. p_a, p_s, p_e into shared memory; max of p_s / p_e by warp shuffles; candidate flags
//      p[t] > fl(0.9 max) or a strict interior peak, compacted in ascending t with ballots;
//   2. every (start, end) candidate pair -> one 64-bit key ((~bits(c)) << 32 | t_s << 16 | t_e),
//      c = fl(p_s[t_s] p_e[t_e]) >= 0, so ascending keys = (c desc, t_s asc, t_e asc); pairs
//      with t_s >= t_e get the key ~0 (last);
//   3. bitonic sort of the keys in shared memory (<= 16384 keys, 128 KB);
//   4. the first P keys -> (t_s, t_e), IoU target and the 32 interpolated samples of p_a,
//      one thread per (proposal, sample).
// Decisions (flags, scores, order) are fp32 and bit-identical to the oracle; features / IoU
// are fp32 (oracle fp64, tolerance in reading R24).  The work is tiny (B CTAs); the kernel is
// latency-bound by design: it runs once per step on the side of the training step.
#include <cuda_runtime.h>
#include <stdint.h>

#include "kernels.h"

namespace tem {
namespace {

constexpr int PGM_THREADS = 1024, PGM_TMAX = 128;
constexpr int PGM_NS = 8, PGM_NC = 16, PGM_NE = 8, PGM_F = PGM_NS + PGM_NC + PGM_NE;

__device__ __forceinline__ float pgm_at(const float* p, int T, int j) { return (j >= 0 && j < T) ? p[j] : 0.0f; }

__device__ __forceinline__ float pgm_interp(const float* pa, int T, float x) {
    const float fi = floorf(x);
    const int i = (int)fi;
    const float f = x - fi;
    return (1.0f - f) * pgm_at(pa, T, i) + f * pgm_at(pa, T, i + 1);
}

__device__ float block_max(float v, float* red) {
    for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
    const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
    __syncthreads();
    if (l == 0) red[w] = v;
    __syncthreads();
    if (w == 0) {
        v = l < PGM_THREADS / 32 ? red[l] : -INFINITY;
        for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
        if (l == 0) red[0] = v;
    }
    __syncthreads();
    const float r = red[0];
    __syncthreads();
    return r;
}

__global__ void __launch_bounds__(PGM_THREADS) pgm_kernel(int T, int G, int P, const float* __restrict__ prob,
                                                          const float* __restrict__ gt,
                                                          const int32_t* __restrict__ n_gt,
                                                          float* __restrict__ feat, float* __restrict__ iou,
                                                          int32_t* __restrict__ ts_out, int32_t* __restrict__ te_out,
                                                          int32_t* __restrict__ count) {
    extern __shared__ unsigned long long keys[];  // [npow2]
    __shared__ float pa[PGM_TMAX], ps[PGM_TMAX], pe[PGM_TMAX];
    __shared__ float red[32];
    __shared__ int cs[PGM_TMAX], ce[PGM_TMAX];
    __shared__ int wcount[2][PGM_TMAX / 32];
    __shared__ int nvalid;
    const int v = blockIdx.x, tid = threadIdx.x;
    const float* pv = prob + (size_t)v * 3 * T;
    if (tid < T) {
        pa[tid] = pv[tid];
        ps[tid] = pv[T + tid];
        pe[tid] = pv[2 * T + tid];
    }
    if (tid == 0) nvalid = 0;
    __syncthreads();
    // 1. candidates
    const float ms = block_max(tid < T ? ps[tid] : -INFINITY, red);
    const float me = block_max(tid < T ? pe[tid] : -INFINITY, red);
    const float ths = __fmul_rn(0.9f, ms), the = __fmul_rn(0.9f, me);
    bool fs = false, fe = false;
    if (tid < T) {
        const bool inner = tid > 0 && tid < T - 1;
        fs = ps[tid] > ths || (inner && ps[tid] > ps[tid - 1] && ps[tid] > ps[tid + 1]);
        fe = pe[tid] > the || (inner && pe[tid] > pe[tid - 1] && pe[tid] > pe[tid + 1]);
    }
    const int w = tid >> 5, l = tid & 31;
    const unsigned bs = __ballot_sync(0xffffffffu, fs), be = __ballot_sync(0xffffffffu, fe);
    if (w < PGM_TMAX / 32 && l == 0) {
        wcount[0][w] = __popc(bs);
        wcount[1][w] = __popc(be);
    }
    __syncthreads();
    int offs = 0, offe = 0, nS = 0, nE = 0;
    for (int q = 0; q < (T + 31) / 32; ++q) {
        if (q < w) {
            offs += wcount[0][q];
            offe += wcount[1][q];
        }
        nS += wcount[0][q];
        nE += wcount[1][q];
    }
    const unsigned below = (1u << l) - 1u;
    if (fs) cs[offs + __popc(bs & below)] = tid;
    if (fe) ce[offe + __popc(be & below)] = tid;
    __syncthreads();
    // 2. keys of all candidate pairs, padded to a power of two with ~0
    const int npair = nS * nE;
    int npow = 1;
    while (npow < npair) npow <<= 1;
    int myvalid = 0;
    for (int i = tid; i < npow; i += PGM_THREADS) {
        unsigned long long k = ~0ull;
        if (i < npair) {
            const int a = cs[i / nE], b = ce[i % nE];
            if (a < b) {
                const float c = __fmul_rn(ps[a], pe[b]);
                k = ((unsigned long long)(~__float_as_uint(c)) << 32) | ((unsigned long long)a << 16) |
                    (unsigned long long)b;
                ++myvalid;
            }
        }
        keys[i] = k;
    }
    if (myvalid) atomicAdd(&nvalid, myvalid);
    __syncthreads();
    // 3. bitonic sort, ascending
    for (int kk = 2; kk <= npow; kk <<= 1)
        for (int j = kk >> 1; j > 0; j >>= 1) {
            for (int i = tid; i < npow; i += PGM_THREADS) {
                const int ixj = i ^ j;
                if (ixj > i) {
                    const unsigned long long x = keys[i], y = keys[ixj];
                    const bool up = (i & kk) == 0;
                    if ((x > y) == up) {
                        keys[i] = y;
                        keys[ixj] = x;
                    }
                }
            }
            __syncthreads();
        }
    // 4. outputs
    const int n = min(P, nvalid);
    if (tid == 0) count[v] = n;
    const int ng = min(n_gt[v], G);
    for (int i = tid; i < P; i += PGM_THREADS) {
        int a = -1, b = -1;
        float g = 0.0f;
        if (i < n) {
            const unsigned long long k = keys[i];
            a = (int)((k >> 16) & 0xffff);
            b = (int)(k & 0xffff);
            const float s1 = (float)a + 0.5f, e1 = (float)b + 0.5f;
            for (int q = 0; q < ng; ++q) {
                const float s2 = gt[((size_t)v * G + q) * 2], e2 = gt[((size_t)v * G + q) * 2 + 1];
                const float inter = fmaxf(0.0f, fminf(e1, e2) - fmaxf(s1, s2));
                const float uni = (e1 - s1) + (e2 - s2) - inter;
                if (uni > 0.0f) g = fmaxf(g, inter / uni);
            }
        }
        ts_out[(size_t)v * P + i] = a;
        te_out[(size_t)v * P + i] = b;
        iou[(size_t)v * P + i] = g;
    }
    for (int idx = tid; idx < P * PGM_F; idx += PGM_THREADS) {
        const int i = idx / PGM_F, k = idx - i * PGM_F;
        float val = 0.0f;
        if (i < n) {
            const unsigned long long key = keys[i];
            const int a = (int)((key >> 16) & 0xffff), b = (int)(key & 0xffff);
            const float d = (float)(b - a);
            float lo, hi;
            int kk, nn;
            if (k < PGM_NS) {
                lo = a - d / 5.0f, hi = a + d / 5.0f, kk = k, nn = PGM_NS;
            } else if (k < PGM_NS + PGM_NC) {
                lo = (float)a, hi = (float)b, kk = k - PGM_NS, nn = PGM_NC;
            } else {
                lo = b - d / 5.0f, hi = b + d / 5.0f, kk = k - PGM_NS - PGM_NC, nn = PGM_NE;
            }
            val = pgm_interp(pa, T, lo + (kk + 0.5f) * (hi - lo) / nn);
        }
        feat[(size_t)v * P * PGM_F + idx] = val;
    }
}

}  // namespace

cudaError_t launch_pgm(int B, int T, int G, int P, const float* prob, const float* gt, const int32_t* n_gt,
                       float* feat, float* iou, int32_t* ts, int32_t* te, int32_t* count, cudaStream_t s) {
    if (B == 0) return cudaSuccess;
    int npow = 1;
    while (npow < T * T) npow <<= 1;
    const size_t smem = sizeof(unsigned long long) * npow;
    static size_t attr = 0;
    if (smem > attr) {
        cudaError_t e = cudaFuncSetAttribute(pgm_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return e;
        attr = smem;
    }
    pgm_kernel<<<B, PGM_THREADS, smem, s>>>(T, G, P, prob, gt, n_gt, feat, iou, ts, te, count);
    return cudaGetLastError();
}

}  // namespace tem

// C ABI (include/tem.h)
tem_status tem_pgm(int32_t B, int32_t T, int32_t G, int32_t P, const float* prob, const float* gt,
                   const int32_t* n_gt, float* features, float* iou, int32_t* ts, int32_t* te, int32_t* count,
                   void* stream) {
    if (B < 0 || T < 1 || T > 128 || G < 0 || P < 1 || P > 65536) return TEM_ERR_INVALID_ARG;
    if (B > 0 && (!prob || !n_gt || (G > 0 && !gt) || !features || !iou || !ts || !te || !count))
        return TEM_ERR_INVALID_ARG;
    return tem::launch_pgm(B, T, G, P, prob, gt, n_gt, features, iou, ts, te, count, (cudaStream_t)stream) ==
                   cudaSuccess
               ? TEM_OK
               : TEM_ERR_CUDA;
}
