// ring.cu -- KR1: the paper's ring allreduce over NVLink peer memory,
// with the 1/N mean and the optimizer update fused into the block owner (SURVEY 8(a)
// rows a9-a12), plus the NVSwitch two-shot variant and the parameter-server comparator KP1
// (P:115-124).
//
// Handshake (every collective kernel): before any data moves, channel g of rank n
// writes a 16-byte header {K_lo, epoch, K_hi | kind | op | mode, epoch} into slot [n][g] of
// EVERY rank's heap, then reads the N headers [0..N-1][g] of its own heap.  Every rank
// therefore compares the same N descriptors: if any differs, all ranks latch PROTOCOL and
// abort before the first data store; a header that does not arrive within spin_ns latches
// TRANSPORT.
//
// Ring protocol (one launch per rank per collective; grid = G channels x local ranks):
//   * The gradient of K_pad elements is split into N equal blocks (row a9).  Inside a block,
//     float4 position v belongs to channel (v / THREADS) mod G -- interleaved, so the chain
//     order of every element (fixed by its block alone) is independent of G.
//   * Messages travel as LL lines (common.cuh): each float4 becomes two 16-byte lines
//     {d0, epoch, d1, epoch}, stored into the right neighbour's LL slot (phase, round).  The
//     receiving thread polls its own lines until both flags carry this collective's epoch: no
//     block barrier, no fence, and the hand-off is per thread, so round i+1 at rank n+1 starts
//     on the first positions while rank n still sends the rest of round i.
//   * Scatter round i = 0..N-2: rank n sends block s = (n-i) mod N: own[s] plus the
//     partial received in round i-1.  So block b is summed along g_b + g_{b+1} + ... +
//     g_{b+N-1}, bit-identical to the oracle's round-by-round replay.
//   * Owner: after round N-2 rank n owns block (n+1) mod N: last add, mean
//     s * fl(1/N), optimizer update (mode 1), bf16 operand copies; the result is gather
//     round 0's message.
//   * Gather round k = 1..N-2 (reading R10): store the block received in round k-1
//     and forward it (send (n+1-k) mod N) -- replace, never add; then store the last one.
//   * Epochs: per-channel counters in the workspace, advanced by one per collective on every
//     rank (G is fixed per context, so all channels advance together); LL slots have a fixed
//     stride (sized for the largest collective) and alternate between two halves by epoch
//     parity, so a line of collective t+1 never lands on an unread line of collective t
//     (DESIGN.md 6.6).
// The same device code serves production (one process per GPU, peers over NVLink) and the
// single-device emulation used by the tests (N ranks = N CTA groups of one cooperative
// launch, "peer" heaps on the same device).
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <algorithm>

#include "kernels.h"
#include "optim.cuh"

namespace tem {
namespace {

constexpr int RING_THREADS = 512;
constexpr int RING_UNROLL = 4;  // float4 positions in flight per thread

TEM_DEV int modn(int a, int n) {
    const int r = a % n;
    return r < 0 ? r + n : r;
}

TEM_DEV uint64_t flag_value(uint32_t epoch) { return (uint64_t)epoch << 32; }

// Bounded spin: after `kSpinCheck` polls, checks the wall clock (and the CTA's abort word) every
// kSpinCheck polls; past spin_ns it latches TRANSPORT and tells the CTA to abort.
constexpr int kSpinCheck = 64;
struct Spin {
    uint64_t t0 = 0;
    int n = 0;
    // true: keep polling; false: give up (timed out, or another thread of the CTA did)
    TEM_DEV bool again(Status* st, uint64_t spin_ns, volatile int* s_abort) {
        if (++n < kSpinCheck) return true;
        n = 0;
        if (*s_abort) return false;
        const uint64_t t = globaltimer();
        if (t0 == 0) {
            t0 = t;
            return true;
        }
        if (t - t0 > spin_ns) {
            latch(st, TEM_ERR_TRANSPORT, -1);
            *s_abort = 1;
            return false;
        }
        return true;
    }
};

// Thread 0 waits for `flag` to reach `epoch` (two-shot / PS phase flags); returns false
// (CTA-uniform) on timeout.
TEM_DEV bool wait_flag(const uint64_t* flag, uint32_t epoch, Status* st, uint64_t spin_ns, int* s_abort) {
    if (threadIdx.x == 0) {
        Spin sp;
        while ((uint32_t)(ld_acquire_sys(flag) >> 32) < epoch)
            if (!sp.again(st, spin_ns, s_abort)) break;
    }
    __syncthreads();
    return *s_abort == 0;
}

TEM_DEV void signal_flag(uint64_t* flag, uint32_t epoch) {
    __syncthreads();  // every thread's data stores precede thread 0's release (cumulative)
    if (threadIdx.x == 0) st_release_sys(flag, flag_value(epoch));
}

// The collective's descriptor in the header (kind: 0 ring, 1 two-shot, 2 PS).
TEM_DEV uint4 header_value(int64_t K, uint32_t epoch, int kind, int op, int mode) {
    const uint32_t hi = (uint32_t)((uint64_t)K >> 32) & 0xFFu;
    return make_uint4((uint32_t)K, epoch, hi | ((uint32_t)kind << 8) | ((uint32_t)op << 16) | ((uint32_t)mode << 24),
                      epoch);
}

// Symmetric pre-data check (see the file comment).  CTA-uniform result; false = abort.
TEM_DEV bool handshake(const RingLocal& L, int N, int n, int g, uint32_t epoch, uint4 mine, int64_t off_hdr,
                       Status* st, uint64_t spin_ns, int* s_abort) {
    const int tid = threadIdx.x;
    // slots [epoch parity][src][channel]: consecutive collectives use disjoint halves
    auto slot = [&](int heap_rank, int src) {
        return reinterpret_cast<uint4*>(L.heaps[heap_rank] + off_hdr) +
               ((int64_t)(epoch & 1u) * TEM_MAX_RANKS + src) * kMaxChannels + g;
    };
    if (tid < N) st_volatile4(slot(tid, n), mine);
    if (tid < N) {
        const uint4* p = slot(n, tid);
        uint4 h = ld_volatile4(p);
        Spin sp;
        while (h.y != epoch || h.w != epoch) {
            if (!sp.again(st, spin_ns, s_abort)) break;
            h = ld_volatile4(p);
        }
        if (h.y == epoch && h.w == epoch && (h.x != mine.x || h.z != mine.z)) {
            latch(st, TEM_ERR_PROTOCOL, -1);
            *s_abort = 1;
        }
    }
    __syncthreads();
    return *s_abort == 0;
}

// Adam's running products beta^t (reading R22), one thread, after the step's update kernels.
__global__ void opt_scalars_kernel(float* scal, float beta1, float beta2) {
    pdl_trigger();
    pdl_wait();
    scal[0] = __fmul_rn(scal[0], beta1);
    scal[1] = __fmul_rn(scal[1], beta2);
}

// Masked vector helpers for ring_allreduce with K < K_pad (elements >= K untouched).
TEM_DEV float4 ld4_masked(const float* p, int64_t e, int64_t K) {
    if (e + 4 <= K) return *reinterpret_cast<const float4*>(p + e);
    float4 r = make_float4(0.f, 0.f, 0.f, 0.f);
    if (e + 0 < K) r.x = p[e + 0];
    if (e + 1 < K) r.y = p[e + 1];
    if (e + 2 < K) r.z = p[e + 2];
    return r;
}
TEM_DEV float4 ldcg4_masked(const float* p, int64_t e, int64_t K) {
    if (e + 4 <= K) return ld_cg4(p + e);
    float4 r = make_float4(0.f, 0.f, 0.f, 0.f);
    if (e + 0 < K) r.x = __ldcg(p + e + 0);
    if (e + 1 < K) r.y = __ldcg(p + e + 1);
    if (e + 2 < K) r.z = __ldcg(p + e + 2);
    return r;
}
TEM_DEV void st4_masked(float* p, int64_t e, int64_t K, float4 v) {
    if (e + 4 <= K) {
        *reinterpret_cast<float4*>(p + e) = v;
        return;
    }
    if (e + 0 < K) p[e + 0] = v.x;
    if (e + 1 < K) p[e + 1] = v.y;
    if (e + 2 < K) p[e + 2] = v.z;
}

// LL message of one float4 position: two lines {d0, e, d1, e}, {d2, e, d3, e}.
TEM_DEV void ll_send(uint4* p, float4 a, uint32_t e) {
    st_volatile4(p, make_uint4(__float_as_uint(a.x), e, __float_as_uint(a.y), e));
    st_volatile4(p + 1, make_uint4(__float_as_uint(a.z), e, __float_as_uint(a.w), e));
}
// Receive the LL messages of up to RING_UNROLL positions (lines p[u], p[u] + 1; p[u] == nullptr:
// no position): every line is loaded first, then only the lines still carrying an old epoch are
// polled again -- one memory latency per batch, not per position.  false: abort (timeout).
TEM_DEV bool ll_recv(const uint4* const (&p)[RING_UNROLL], uint32_t e, float4 (&out)[RING_UNROLL], Status* st,
                     uint64_t spin_ns, volatile int* s_abort) {
    uint4 a[RING_UNROLL], b[RING_UNROLL];
#pragma unroll
    for (int u = 0; u < RING_UNROLL; ++u)
        if (p[u]) {
            a[u] = ld_volatile4(p[u]);
            b[u] = ld_volatile4(p[u] + 1);
        }
    Spin sp;
    while (true) {
        bool done = true;
#pragma unroll
        for (int u = 0; u < RING_UNROLL; ++u) {
            if (!p[u]) continue;
            if (a[u].y != e || a[u].w != e) {
                done = false;
                a[u] = ld_volatile4(p[u]);
            }
            if (b[u].y != e || b[u].w != e) {
                done = false;
                b[u] = ld_volatile4(p[u] + 1);
            }
        }
        if (done) break;
        if (!sp.again(st, spin_ns, s_abort)) return false;
    }
#pragma unroll
    for (int u = 0; u < RING_UNROLL; ++u)
        out[u] = make_float4(__uint_as_float(a[u].x), __uint_as_float(a[u].z), __uint_as_float(b[u].x),
                             __uint_as_float(b[u].z));
    return true;
}

__global__ void __launch_bounds__(RING_THREADS) ring_kernel(const __grid_constant__ RingParams P) {
    __shared__ uint32_t s_epoch;
    __shared__ int s_abort;
    const int l = blockIdx.y, g = blockIdx.x, tid = threadIdx.x;
    const int N = P.N, n = P.rank_base + l, G = P.G;
    const RingLocal& L = P.loc[l];
    const int right = modn(n + 1, N);
    const int64_t K = P.K, Bk = P.Kpad / N, nvec = Bk / 4;
    const float inv_n = 1.0f / (float)N;
    if (tid == 0) {
        s_epoch = L.epochs[g] + 1;
        s_abort = 0;
    }
    __syncthreads();
    const uint32_t epoch = s_epoch;
    if (!handshake(L, N, n, g, epoch, header_value(K, epoch, 0, P.op, P.mode), P.off_hdr, P.status, P.spin_ns,
                   &s_abort))
        return;
    volatile int* abort = &s_abort;
    const uint4* ll_self = reinterpret_cast<const uint4*>(L.heaps[n] + P.off_ll);
    uint4* ll_right = reinterpret_cast<uint4*>(L.heaps[right] + P.off_ll);
    // line of float4 position v in LL slot (epoch parity, phase, round): fixed stride P.ll_stride
    // lines; consecutive collectives use disjoint halves
    const int64_t half = (int64_t)(epoch & 1u) * 2 * (N - 1);
    auto slot = [&](int phase, int round) { return (half + phase * (N - 1) + round) * P.ll_stride; };
    const float* src = L.src;
    float* dst = L.dst_self;
    const int64_t stride = (int64_t)G * RING_THREADS;
    const int64_t v_begin = (int64_t)g * RING_THREADS + tid;

    // ---------------- scatter: rounds 0..N-2 ----------------
    for (int i = 0; i <= N - 2; ++i) {
        const int64_t blk = (int64_t)modn(n - i, N) * Bk;
        for (int64_t v0 = v_begin; v0 < nvec; v0 += RING_UNROLL * stride) {
            float4 a[RING_UNROLL];
#pragma unroll
            for (int u = 0; u < RING_UNROLL; ++u) {
                const int64_t v = v0 + u * stride;
                if (v < nvec) a[u] = ld4_masked(src, blk + 4 * v, K);
            }
            if (i > 0) {
                const uint4* q[RING_UNROLL];
                float4 b[RING_UNROLL];
#pragma unroll
                for (int u = 0; u < RING_UNROLL; ++u) {
                    const int64_t v = v0 + u * stride;
                    q[u] = v < nvec ? ll_self + slot(0, i - 1) + 2 * v : nullptr;
                }
                if (!ll_recv(q, epoch, b, P.status, P.spin_ns, abort)) return;
#pragma unroll
                for (int u = 0; u < RING_UNROLL; ++u) {
                    a[u].x = a[u].x + b[u].x; a[u].y = a[u].y + b[u].y; a[u].z = a[u].z + b[u].z; a[u].w = a[u].w + b[u].w;
                }
            }
#pragma unroll
            for (int u = 0; u < RING_UNROLL; ++u) {
                const int64_t v = v0 + u * stride;
                if (v < nvec) ll_send(ll_right + slot(0, i) + 2 * v, a[u], epoch);
            }
        }
    }
    // ---------------- owner: last add, mean, update; gather round 0's message ----------------
    {
        const int64_t blk = (int64_t)modn(n + 1, N) * Bk;
        for (int64_t v0 = v_begin; v0 < nvec; v0 += RING_UNROLL * stride) {
            float4 a[RING_UNROLL], w[RING_UNROLL];
#pragma unroll
            for (int u = 0; u < RING_UNROLL; ++u) {
                const int64_t v = v0 + u * stride;
                if (v >= nvec) continue;
                a[u] = ld4_masked(src, blk + 4 * v, K);
                if (P.mode == 1) w[u] = *reinterpret_cast<const float4*>(dst + blk + 4 * v);
            }
            float4 r[RING_UNROLL];
            if (N > 1) {
                const uint4* q[RING_UNROLL];
#pragma unroll
                for (int u = 0; u < RING_UNROLL; ++u) {
                    const int64_t v = v0 + u * stride;
                    q[u] = v < nvec ? ll_self + slot(0, N - 2) + 2 * v : nullptr;
                }
                if (!ll_recv(q, epoch, r, P.status, P.spin_ns, abort)) return;
            }
#pragma unroll
            for (int u = 0; u < RING_UNROLL; ++u) {
                const int64_t v = v0 + u * stride;
                if (v >= nvec) continue;
                const int64_t e = blk + 4 * v;
                float4 x = a[u];
                if (N > 1) {
                    x.x = x.x + r[u].x; x.y = x.y + r[u].y; x.z = x.z + r[u].z; x.w = x.w + r[u].w;
                }
                if (P.op == TEM_MEAN) {
                    x.x = x.x * inv_n; x.y = x.y * inv_n; x.z = x.z * inv_n; x.w = x.w * inv_n;
                }
                if (P.mode == 1) {
                    x = owner_update(P.oc, L.opt, e, x, w[u]);
                    if (L.shadow) store_shadow4(L.shadow, L.shadow_lo, e, x);
                }
                st4_masked(dst, e, K, x);
                if (N > 1) ll_send(ll_right + slot(1, 0) + 2 * v, x, epoch);
            }
        }
    }
    // ---------------- gather rounds 1..N-2: store what arrived, forward it; then the last ------
    for (int k = 1; k <= N - 1; ++k) {
        const int64_t blk = (int64_t)modn(n + 1 - k, N) * Bk;  // received in round k-1 (R10)
        for (int64_t v0 = v_begin; v0 < nvec; v0 += RING_UNROLL * stride) {
            const uint4* q[RING_UNROLL];
            float4 x[RING_UNROLL];
#pragma unroll
            for (int u = 0; u < RING_UNROLL; ++u) {
                const int64_t v = v0 + u * stride;
                q[u] = v < nvec ? ll_self + slot(1, k - 1) + 2 * v : nullptr;
            }
            if (!ll_recv(q, epoch, x, P.status, P.spin_ns, abort)) return;
#pragma unroll
            for (int u = 0; u < RING_UNROLL; ++u) {
                const int64_t v = v0 + u * stride;
                if (v >= nvec) continue;
                const int64_t e = blk + 4 * v;
                if (k <= N - 2) ll_send(ll_right + slot(1, k) + 2 * v, x[u], epoch);
                st4_masked(dst, e, K, x[u]);
                if (L.shadow) store_shadow4(L.shadow, L.shadow_lo, e, x[u]);
            }
        }
    }
    if (tid == 0) L.epochs[g] = epoch;
}

// Two-shot allreduce over NVSwitch: the same result bits as the
// ring, in two communication phases instead of 2(N-1) dependent rounds.
//   phase 0: every rank stages its gradient in its own heap (skipped when the source already
//            is its heap's user region) and raises, per channel, a ready flag in every peer.
//   phase 1: rank n owns block b = (n+1) mod N (the ring's owner).  Channel g waits for
//            the ready flags of all N sources, reads its piece of block b from every rank's
//            heap and sums along the ring's chain g_b + g_{b+1} + ... + g_{b+N-1} (SURVEY 8(c)
//            c.1) -- so every element is bit-identical to the ring and to the oracle -- applies
//            mean (and SGD), writes the result into EVERY rank's destination (direct NVLink
//            stores) and raises a done flag in every peer.
//   then:    each rank waits for the done flags of the N-1 other owners and refreshes its bf16
//            operand copies of those blocks.
// Flags: epoch words (after the handshake); ready[src][channel], done[owner][channel] at off_flags.
__global__ void __launch_bounds__(RING_THREADS) twoshot_kernel(const __grid_constant__ RingParams P) {
    __shared__ uint32_t s_epoch;
    __shared__ int s_abort;
    const int l = blockIdx.y, g = blockIdx.x, tid = threadIdx.x;
    const int N = P.N, n = P.rank_base + l, G = P.G;
    const RingLocal& L = P.loc[l];
    const int64_t K = P.K, Bk = P.Kpad / N, nvec = Bk / 4;
    const float inv_n = 1.0f / (float)N;
    auto heap = [&](int r) { return L.heaps[r]; };
    auto stage = [&](int r) -> float* {  // rank r's readable copy of its gradient
        return P.off_stage >= 0 ? reinterpret_cast<float*>(heap(r) + P.off_stage) : reinterpret_cast<float*>(heap(r) + P.off_src);
    };
    auto flag = [&](int r, int phase, int who) -> uint64_t* {
        return reinterpret_cast<uint64_t*>(heap(r) + P.off_flags) + ((int64_t)phase * TEM_MAX_RANKS + who) * kMaxChannels + g;
    };
    if (tid == 0) {
        s_epoch = L.epochs[g] + 1;
        s_abort = 0;
    }
    __syncthreads();
    const uint32_t epoch = s_epoch;
    if (!handshake(L, N, n, g, epoch, header_value(K, epoch, 1, P.op, P.mode), P.off_hdr, P.status, P.spin_ns,
                   &s_abort))
        return;
    // channel g's piece of every block: vectors [v0, v1) of each block
    const int64_t v0 = (int64_t)g * nvec / G, v1 = (int64_t)(g + 1) * nvec / G;
    // ---------------- phase 0: stage (own heap) + ready flags ----------------
    if (P.off_stage >= 0) {
        float* st = stage(n);
        for (int b = 0; b < N; ++b)
            for (int64_t v = v0 + tid; v < v1; v += RING_THREADS) {
                const int64_t e = (int64_t)b * Bk + 4 * v;
                if (e >= K) continue;
                st4_masked(st, e, K, ld4_masked(L.src, e, K));
            }
    }
    __syncthreads();
    if (tid < N) st_release_sys(flag(tid, 0, n), flag_value(epoch));  // ready: my piece g is readable
    // ---------------- phase 1: owner reduce (chain order) + mean/SGD + broadcast ----------------
    const int b = modn(n + 1, N);
    for (int r = 0; r < N; ++r)
        if (!wait_flag(flag(n, 0, r), epoch, P.status, P.spin_ns, &s_abort)) return;
    for (int64_t v = v0 + tid; v < v1; v += RING_THREADS) {
        const int64_t e = (int64_t)b * Bk + 4 * v;
        if (e >= K) continue;
        float4 a = ldcg4_masked(stage(b), e, K);  // chain start: rank b
        for (int q = 1; q < N; ++q) {
            const float4 t = ldcg4_masked(stage(modn(b + q, N)), e, K);
            a.x = a.x + t.x; a.y = a.y + t.y; a.z = a.z + t.z; a.w = a.w + t.w;
        }
        if (P.op == TEM_MEAN) {
            a.x = a.x * inv_n; a.y = a.y * inv_n; a.z = a.z * inv_n; a.w = a.w * inv_n;
        }
        float4 out = a;
        if (P.mode == 1) {
            out = owner_update(P.oc, L.opt, e, a, *reinterpret_cast<const float4*>(L.dst_self + e));
            if (L.shadow) store_shadow4(L.shadow, L.shadow_lo, e, out);
        }
        for (int r = 0; r < N; ++r) st4_masked(reinterpret_cast<float*>(heap(r) + P.off_dst), e, K, out);
    }
    __syncthreads();
    if (tid < N) st_release_sys(flag(tid, 1, n), flag_value(epoch));  // done: block b piece g written
    // ---------------- receive: the other owners' blocks, refresh operand copies ----------------
    for (int q = 1; q < N; ++q) {
        const int owner = modn(n + q, N), blk = modn(owner + 1, N);
        if (!wait_flag(flag(n, 1, owner), epoch, P.status, P.spin_ns, &s_abort)) return;
        if (L.shadow) {
            for (int64_t v = v0 + tid; v < v1; v += RING_THREADS) {
                const int64_t e = (int64_t)blk * Bk + 4 * v;
                store_shadow4(L.shadow, L.shadow_lo, e, ld_cg4(L.dst_self + e));
            }
        }
    }
    // no rank may restage (next collective) before every owner has read this one: the done
    // flags above cover it -- an owner raises done only after reading all N stages
    if (tid == 0) L.epochs[g] = epoch;
}

// N = 1: the ring is the identity; the owner update alone.
__global__ void sgd_single_kernel(const float* __restrict__ g, float* __restrict__ w,
                                  __nv_bfloat16* __restrict__ shadow, __nv_bfloat16* __restrict__ shadow_lo,
                                  int64_t n, int op, OptCfg oc, OptState os) {
    trace_begin(SLOT_EXCHANGE);
    pdl_trigger();
    pdl_wait();
    const int64_t nv = n / 4;
    for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < nv;
         v += (int64_t)gridDim.x * blockDim.x) {
        float4 a = reinterpret_cast<const float4*>(g)[v];
        if (op == TEM_MEAN) {  // fl(1/1) = 1: a * 1 is exact
            a.x = a.x * 1.0f; a.y = a.y * 1.0f; a.z = a.z * 1.0f; a.w = a.w * 1.0f;
        }
        const float4 x = owner_update(oc, os, 4 * v, a, reinterpret_cast<float4*>(w)[v]);
        reinterpret_cast<float4*>(w)[v] = x;
        if (shadow) store_shadow4(shadow, shadow_lo, 4 * v, x);
    }
    trace_end(SLOT_EXCHANGE);
}

// launch shape of the fused update: 8 x 148 CTAs of 256 threads, ~1.2 element groups per thread
// (measured at c2: 229.8 k samples/s vs 228.1 k with 296 x 512, 228.6 k with 148 x 1024)
constexpr int UPD_THREADS = 256, UPD_CTAS = 8 * 148;
template <int KIND>
__global__ void __launch_bounds__(UPD_THREADS) sgd_fused_kernel(float* __restrict__ g, float* __restrict__ w, __nv_bfloat16* __restrict__ shadow,
                                 __nv_bfloat16* __restrict__ shadow_lo, int64_t e0, int64_t e1, OptCfg oc,
                                 OptState os,
                                 const float* __restrict__ p1, int64_t stride1, int64_t n1, int S1,
                                 const float* __restrict__ p2, int64_t stride2, int64_t off2, int64_t n2, int S2,
                                 int mode) {
    // mode 1: update + keep the summed local gradient in g; 2: update only (tem_local_grad
    // sums the partials again on demand, same order); 0: only sum the partials into g
    const int slot = e0 > 0 ? SLOT_EXCH2 : SLOT_EXCHANGE;  // the split update's W2.. range
    trace_begin(slot);
    pdl_trigger();
    pdl_wait();
    const int64_t nv = e1 / 4;
    for (int64_t v = e0 / 4 + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < nv;
         v += (int64_t)gridDim.x * blockDim.x) {
        const int64_t e = 4 * v;
        const float* src = nullptr;
        int64_t stride = 0;
        int S = 1;
        if (e < n1) {
            src = p1 + e;
            stride = stride1;
            S = S1;
        } else if (e >= off2 && e < off2 + n2) {
            src = p2 + (e - off2);
            stride = stride2;
            S = S2;
        }
        // every load of the element group is issued before the first use (one memory latency
        // per iteration): the weights, then up to 4 partials unrolled
        const float4 wv = mode ? reinterpret_cast<const float4*>(w)[v] : make_float4(0.f, 0.f, 0.f, 0.f);
        float4 a;
        if (src) {  // split-K partials, summed in ascending s (as reduce_wgrad_kernel)
            constexpr int SU = 4;
            float4 p[SU];
#pragma unroll
            for (int s = 0; s < SU; ++s)
                if (s < S) p[s] = __ldcs(reinterpret_cast<const float4*>(src + (size_t)s * stride));
            a = p[0];
#pragma unroll
            for (int s = 1; s < SU; ++s)
                if (s < S) {
                    a.x += p[s].x; a.y += p[s].y; a.z += p[s].z; a.w += p[s].w;
                }
            for (int s = SU; s < S; ++s) {
                const float4 q = __ldcs(reinterpret_cast<const float4*>(src + (size_t)s * stride));
                a.x += q.x; a.y += q.y; a.z += q.z; a.w += q.w;
            }
            if (mode != 2) reinterpret_cast<float4*>(g)[v] = a;  // the local gradient
        } else {
            if (mode == 0) continue;
            a = reinterpret_cast<const float4*>(g)[v];
        }
        if (mode == 0) continue;
        // TEM_MEAN at N = 1: a * fl(1/1) is exact
        const float4 x = owner_update<KIND>(oc, os, e, a, wv);
        reinterpret_cast<float4*>(w)[v] = x;
        if (shadow) store_shadow4(shadow, shadow_lo, e, x);
    }
    trace_end(slot);
}

// KP1 parameter-server comparator: every rank pushes its buffer into
// its slot of rank 0's heap; rank 0 sums slots in ascending rank order,
// applies op, writes the result into every rank's buffer; then a release flag per
// rank.  Channel g handles a contiguous slice of K.
__global__ void __launch_bounds__(RING_THREADS) ps_kernel(const __grid_constant__ PsParams P) {
    __shared__ uint32_t s_epoch;
    __shared__ int s_abort;
    const int l = blockIdx.y, g = blockIdx.x, tid = threadIdx.x;
    const int N = P.N, n = P.rank_base + l, G = P.G;
    const RingLocal& L = P.loc[l];
    char* heap0 = L.heaps[0];
    const int64_t K = P.K;
    const int64_t Kv = (K + 3) / 4;
    const int64_t v0 = g * Kv / G, v1 = (g + 1) * Kv / G;
    const float inv_n = 1.0f / (float)N;
    if (tid == 0) {
        s_epoch = L.epochs[g] + 1;
        s_abort = 0;
    }
    __syncthreads();
    const uint32_t epoch = s_epoch;
    if (!handshake(L, N, n, g, epoch, header_value(K, epoch, 2, P.op, P.mode), P.off_hdr, P.status, P.spin_ns,
                   &s_abort))
        return;
    // K_slot stride: slots hold K rounded up to 4
    const int64_t slot_stride = Kv * 4;
    // phase 0: push to server slot n (uplink: N*M)
    {
        float* slot = reinterpret_cast<float*>(heap0 + P.off_slots) + (int64_t)n * slot_stride;
        for (int64_t v = v0 + tid; v < v1; v += RING_THREADS) {
            const int64_t e = 4 * v;
            st4_masked(slot, e, K, ld4_masked(L.src, e, K));
        }
        uint64_t* f = reinterpret_cast<uint64_t*>(heap0 + P.off_flags) + (int64_t)n * kMaxChannels + g;
        signal_flag(f, epoch);
    }
    if (n == 0) {
        // server: wait for all N pushes of this channel, then reduce in ascending rank order
        for (int r = 0; r < N; ++r) {
            const uint64_t* f = reinterpret_cast<const uint64_t*>(heap0 + P.off_flags) + (int64_t)r * kMaxChannels + g;
            if (!wait_flag(f, epoch, P.status, P.spin_ns, &s_abort)) return;
        }
        const float* slots = reinterpret_cast<const float*>(heap0 + P.off_slots);
        for (int64_t v = v0 + tid; v < v1; v += RING_THREADS) {
            const int64_t e = 4 * v;
            float4 a = ldcg4_masked(slots, e, K);
            for (int r = 1; r < N; ++r) {
                const float4 b = ldcg4_masked(slots + (int64_t)r * slot_stride, e, K);
                a.x = a.x + b.x; a.y = a.y + b.y; a.z = a.z + b.z; a.w = a.w + b.w;
            }
            if (P.op == TEM_MEAN) {
                a.x = a.x * inv_n; a.y = a.y * inv_n; a.z = a.z * inv_n; a.w = a.w * inv_n;
            }
            if (P.mode == 1)  // the server holds and upgrades the weights
                a = owner_update(P.oc, L.opt, e, a, *reinterpret_cast<const float4*>(L.dst_self + e));
            for (int r = 0; r < N; ++r)  // downlink broadcast (gbar, or w' in SGD mode)
                st4_masked(reinterpret_cast<float*>(L.heaps[r] + P.off_dst), e, K, a);
        }
        __syncthreads();
        for (int r = 0; r < N; ++r) {
            uint64_t* f = reinterpret_cast<uint64_t*>(L.heaps[r] + P.off_flags) + (int64_t)(TEM_MAX_RANKS + r) * kMaxChannels + g;
            signal_flag(f, epoch);
        }
    }
    // everybody: wait for the downlink of this channel
    {
        const uint64_t* f = reinterpret_cast<const uint64_t*>(L.heaps[n] + P.off_flags) + (int64_t)(TEM_MAX_RANKS + n) * kMaxChannels + g;
        if (!wait_flag(f, epoch, P.status, P.spin_ns, &s_abort)) return;
    }
    if (L.shadow)  // refresh this rank's operand copies of the new weights (its channel slice)
        for (int64_t v = v0 + tid; v < v1; v += RING_THREADS)
            store_shadow4(L.shadow, L.shadow_lo, 4 * v, ld_cg4(L.dst_self + 4 * v));
    if (tid == 0) L.epochs[g] = epoch;
}

}  // namespace

cudaError_t launch_ring(const RingParams& p, cudaStream_t s) {
    dim3 grid(p.G, p.nlocal), block(RING_THREADS);
    if (p.nlocal > 1) {
        // single-device emulation: CTAs of different emulated ranks wait on one another,
        // so they must be co-resident -> cooperative launch (fails instead of hanging).
        void* args[] = {const_cast<RingParams*>(&p)};
        return cudaLaunchCooperativeKernel((const void*)ring_kernel, grid, block, args, 0, s);
    }
    ring_kernel<<<grid, block, 0, s>>>(p);
    return cudaGetLastError();
}

cudaError_t launch_sgd_single(const float* g, float* w, __nv_bfloat16* shadow, __nv_bfloat16* shadow_lo,
                              int64_t n, int op, const OptCfg& oc, const OptState& os, cudaStream_t s) {
    return launch_pdl(sgd_single_kernel, dim3(296), dim3(512), 0, s, false, g, w, shadow, shadow_lo, n, op, oc, os);
}

cudaError_t launch_opt_scalars(float* scal, float beta1, float beta2, cudaStream_t s) {
    return launch_pdl(opt_scalars_kernel, dim3(1), dim3(1), 0, s, false, scal, beta1, beta2);
}

TEM_TRACE_SETTER(trace_set_ring)

cudaError_t launch_sgd_fused(float* g, float* w, __nv_bfloat16* shadow, __nv_bfloat16* shadow_lo, int64_t e0,
                             int64_t e1, const OptCfg& oc, const OptState& os, const float* p1, int64_t stride1,
                             int64_t n1, int S1, const float* p2, int64_t stride2, int64_t off2, int64_t n2, int S2,
                             cudaStream_t s, bool side, int ctas, int mode) {
    // UPD_CTAS x UPD_THREADS, grid-stride (round 1 measured 2 x 512 threads per SM faster;
    // with the round-2 step, 8 x 256 per SM is)
    auto k = oc.kind == TEM_OPT_ADAM       ? sgd_fused_kernel<TEM_OPT_ADAM>
             : oc.kind == TEM_OPT_MOMENTUM ? sgd_fused_kernel<TEM_OPT_MOMENTUM>
                                           : sgd_fused_kernel<TEM_OPT_SGD>;
    return launch_pdl(k, dim3(ctas > 0 ? ctas : UPD_CTAS), dim3(UPD_THREADS), 0, s, side, g, w, shadow, shadow_lo, e0, e1, oc, os, p1,
                      stride1, n1, S1, p2, stride2, off2, n2, S2, mode);
}

cudaError_t launch_twoshot(const RingParams& p, cudaStream_t s) {
    dim3 grid(p.G, p.nlocal), block(RING_THREADS);
    if (p.nlocal > 1) {
        void* args[] = {const_cast<RingParams*>(&p)};
        return cudaLaunchCooperativeKernel((const void*)twoshot_kernel, grid, block, args, 0, s);
    }
    twoshot_kernel<<<grid, block, 0, s>>>(p);
    return cudaGetLastError();
}

cudaError_t launch_ps(const PsParams& p, cudaStream_t s) {
    dim3 grid(p.G, p.nlocal), block(RING_THREADS);
    if (p.nlocal > 1) {
        void* args[] = {const_cast<PsParams*>(&p)};
        return cudaLaunchCooperativeKernel((const void*)ps_kernel, grid, block, args, 0, s);
    }
    ps_kernel<<<grid, block, 0, s>>>(p);
    return cudaGetLastError();
}

}  // namespace tem
