// pgm.cu -- BSN's proposal generation module (PGM) on the GPU: candidate boundaries, ranked
// proposals, 32-d Boundary-Sensitive Proposal features and IoU targets, the data path that
// feeds PEM (reading R24; the paper names the stage at P:85).
//
// One CTA of 1024 threads per video (T <= 128):
//   1. p_a, p_s, p_e into shared memory; max of p_s / p_e by warp shuffles; candidate flags
//      p[t] > fl(0.9 max) or a strict interior peak, compacted in ascending t with ballots;
//   2. every (start, end) candidate pair with t_s < t_e has the 64-bit key
//      ((~bits(c)) << 32 | t_s << 16 | t_e), c = fl(p_s[t_s] p_e[t_e]) >= 0, so ascending keys =
//      (c desc, t_s asc, t_e asc); a 4-pass 8-bit radix select finds the P-th smallest ~bits(c);
//   3. the pairs at or below it (P plus ties) are collected and bitonic-sorted in shared memory
//      (<= 16384 keys, 128 KB; a full sort measured 103 us per step at c6, the select ~10x less);
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

constexpr int PGM_THREADS = 1024, PGM_TMAX = 128, PGM_SELMAX = 4096;
constexpr int PGM_NS = 8, PGM_NC = 16, PGM_NE = 8, PGM_F = PGM_NS + PGM_NC + PGM_NE;

__device__ __forceinline__ float pgm_at(const float* p, int T, int j) { return (j >= 0 && j < T) ? p[j] : 0.0f; }

__device__ __forceinline__ float pgm_interp(const float* pa, int T, float x) {
    const float fi = floorf(x);
    const int i = (int)fi;
    const float f = x - fi;
    return (1.0f - f) * pgm_at(pa, T, i) + f * pgm_at(pa, T, i + 1);
}

// Slot of this lane in a shared array filled by a counter: one atomic per warp (all lanes call).
__device__ __forceinline__ int warp_slot(bool take, int* counter) {
    const unsigned m = __ballot_sync(0xffffffffu, take);
    const int lane = threadIdx.x & 31;
    int base = 0;
    if (lane == 0 && m) base = atomicAdd(counter, __popc(m));
    base = __shfl_sync(0xffffffffu, base, 0);
    return base + __popc(m & ((1u << lane) - 1u));
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
                                                          const float* __restrict__ z, float* __restrict__ prob_out,
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
    __shared__ int nvalid, nsel, sel[2];
    __shared__ unsigned hist[256];
    const int v = blockIdx.x, tid = threadIdx.x;
    if (z) {  // in-step use: p = sigmoid(z) of TEM's logits z [B][T][3], kept in prob_out [B][3][T]
        if (tid < T) {
            const float* zv = z + ((size_t)v * T + tid) * 3;
            float* po = prob_out + (size_t)v * 3 * T;
            pa[tid] = po[tid] = 1.0f / (1.0f + expf(-zv[0]));
            ps[tid] = po[T + tid] = 1.0f / (1.0f + expf(-zv[1]));
            pe[tid] = po[2 * T + tid] = 1.0f / (1.0f + expf(-zv[2]));
        }
    } else {
        const float* pv = prob + (size_t)v * 3 * T;
        if (tid < T) {
            pa[tid] = pv[tid];
            ps[tid] = pv[T + tid];
            pe[tid] = pv[2 * T + tid];
        }
    }
    if (tid == 0) nvalid = nsel = 0;
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
    // 2. the valid pairs' keys into shared memory (order irrelevant: they are ranked below);
    //    then a radix select on u = ~bits(c), 8 bits per pass, finds the P-th smallest u
    //    (ascending u = descending c)
    unsigned long long* all = keys;                      // [T*T] pair keys
    unsigned long long* top = keys + PGM_TMAX * PGM_TMAX;  // [PGM_SELMAX] selected keys
    // warp w takes start candidates w, w + 32, ...; its lanes walk the end candidates after
    // t_s (ce is ascending: the first index with ce > t_s by binary search), warp-aggregated
    // compaction into `all`
    for (int si = w; si < nS; si += PGM_THREADS / 32) {
        const int a = cs[si];
        int lo = 0, hi = nE;
        while (lo < hi) {
            const int mid = (lo + hi) >> 1;
            if (ce[mid] > a) hi = mid;
            else lo = mid + 1;
        }
        for (int e0 = lo; e0 < nE; e0 += 32) {
            const int ei = e0 + l;
            const bool ok = ei < nE;
            const int pos = warp_slot(ok, &nvalid);
            if (ok) {
                const int b = ce[ei];
                const unsigned u = ~__float_as_uint(__fmul_rn(ps[a], pe[b]));
                all[pos] = ((unsigned long long)u << 32) | ((unsigned long long)a << 16) | (unsigned long long)b;
            }
        }
    }
    __syncthreads();
    const int nv = nvalid;
    unsigned prefix = 0xffffffffu;  // nv <= P: every valid pair is kept
    if (nv > P) {
        prefix = 0u;
        unsigned mask = 0u;
        int rank = P;  // 1-based rank still to locate among the pairs matching prefix / mask
        for (int shift = 24; shift >= 0; shift -= 8) {
            for (int q = tid; q < 256; q += PGM_THREADS) hist[q] = 0u;
            __syncthreads();
            for (int i = tid; i < nv; i += PGM_THREADS) {
                const unsigned u = (unsigned)(all[i] >> 32);
                if ((u & mask) == prefix) atomicAdd(&hist[(u >> shift) & 255u], 1u);
            }
            __syncthreads();
            if (tid < 32) {  // smallest digit whose cumulative count reaches rank
                unsigned loc[8], sum = 0;
#pragma unroll
                for (int q = 0; q < 8; ++q) {
                    loc[q] = hist[8 * tid + q];
                    sum += loc[q];
                }
                unsigned incl = sum;
#pragma unroll
                for (int o = 1; o < 32; o <<= 1) {
                    const unsigned y = __shfl_up_sync(0xffffffffu, incl, o);
                    if (tid >= o) incl += y;
                }
                const unsigned excl = incl - sum;
                const unsigned hit = __ballot_sync(0xffffffffu, incl >= (unsigned)rank);
                const int lane = __ffs(hit) - 1;
                if (tid == lane) {
                    unsigned c = excl;
                    int d = -1;
#pragma unroll
                    for (int q = 0; q < 8; ++q)
                        if (d < 0) {
                            if (c + loc[q] >= (unsigned)rank) d = q;
                            else c += loc[q];
                        }
                    sel[0] = 8 * lane + d;
                    sel[1] = rank - (int)c;
                }
            }
            __syncthreads();
            prefix |= (unsigned)sel[0] << shift;
            mask |= 255u << shift;
            rank = sel[1];
            __syncthreads();
        }
    }
    // 3. the pairs at or below the P-th u (P plus its ties) are ranked by the full key with a
    //    bitonic sort; with more than PGM_SELMAX of them (massive ties) all pairs are sorted
    for (int i0 = 0; i0 < nv; i0 += PGM_THREADS) {
        const int i = i0 + tid;
        const unsigned long long k = i < nv ? all[i] : ~0ull;
        const bool ok = i < nv && (unsigned)(k >> 32) <= prefix;
        const int pos = warp_slot(ok, &nsel);
        if (ok && pos < PGM_SELMAX) top[pos] = k;
    }
    __syncthreads();
    const int m = nsel;
    unsigned long long* srt = m <= PGM_SELMAX ? top : all;
    const int ns = m <= PGM_SELMAX ? m : nv;
    int npow = 1;
    while (npow < ns) npow <<= 1;
    for (int i = ns + tid; i < npow; i += PGM_THREADS) srt[i] = ~0ull;
    __syncthreads();
    for (int kk = 2; kk <= npow; kk <<= 1)
        for (int jj = kk >> 1; jj > 0; jj >>= 1) {
            for (int i = tid; i < npow; i += PGM_THREADS) {
                const int ixj = i ^ jj;
                if (ixj > i) {
                    const unsigned long long x = srt[i], y = srt[ixj];
                    const bool up = (i & kk) == 0;
                    if ((x > y) == up) {
                        srt[i] = y;
                        srt[ixj] = x;
                    }
                }
            }
            __syncthreads();
        }
    // 4. outputs
    const int n = min(P, nv);
    if (tid == 0) count[v] = n;
    const int ng = min(n_gt[v], G);
    for (int i = tid; i < P; i += PGM_THREADS) {
        int a = -1, b = -1;
        float g = 0.0f;
        if (i < n) {
            const unsigned long long k = srt[i];
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
            const unsigned long long key = srt[i];
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
                       float* feat, float* iou, int32_t* ts, int32_t* te, int32_t* count, cudaStream_t s,
                       const float* z, float* prob_out) {
    if (B == 0) return cudaSuccess;
    // all pairs [PGM_TMAX^2] (padded to a power of two for the tie fallback) + the selection
    const size_t smem = sizeof(unsigned long long) * (PGM_TMAX * PGM_TMAX + PGM_SELMAX);
    static size_t attr = 0;
    if (smem > attr) {
        cudaError_t e = cudaFuncSetAttribute(pgm_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return e;
        attr = smem;
    }
    pgm_kernel<<<B, PGM_THREADS, smem, s>>>(T, G, P, prob, z, prob_out, gt, n_gt, feat, iou, ts, te, count);
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
