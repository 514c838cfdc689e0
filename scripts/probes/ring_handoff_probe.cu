// Ring hand-off latency probe (single device, emulated ranks): R CTAs in a ring pass a
// message of S bytes around M laps; each CTA waits for its left neighbour's message, adds its
// own contribution and forwards it to the right (the dependent chain of the ring's scatter).
// Reports ns per hop for hand-off protocols:
//   V0  data stores; __syncthreads; thread 0 st.release.sys flag | thread 0 polls
//       ld.acquire.sys with __nanosleep(64); __syncthreads; ld.cg data  (round-1 ring)
//   V1  V0 without the sleep
//   V2  V1 with .gpu scope (what the same-device emulation needs; production needs .sys)
//   V3  LL: every 4-byte datum travels with a 4-byte flag in one 8-byte store; each thread
//       polls its own words (ld.volatile), no block barrier, no fence
//   V4  LL with 16-byte stores {d0, f, d1, f}: 8 data bytes per 16-byte store
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o ring_handoff_probe ring_handoff_probe.cu
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <vector>
#include <cuda_runtime.h>
#include <cooperative_groups.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); exit(1); } } while (0)

constexpr int THREADS = 512;

__device__ __forceinline__ uint64_t gtimer() {
    uint64_t t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}
__device__ __forceinline__ uint32_t ld_acq_sys(const uint32_t* p) {
    uint32_t v; asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory"); return v;
}
__device__ __forceinline__ uint32_t ld_acq_gpu(const uint32_t* p) {
    uint32_t v; asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory"); return v;
}
__device__ __forceinline__ void st_rel_sys(uint32_t* p, uint32_t v) {
    asm volatile("st.release.sys.global.u32 [%0], %1;" :: "l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ void st_rel_gpu(uint32_t* p, uint32_t v) {
    asm volatile("st.release.gpu.global.u32 [%0], %1;" :: "l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ uint2 ld_vol2(const uint2* p) {
    uint2 v; asm volatile("ld.volatile.global.v2.u32 {%0,%1}, [%2];" : "=r"(v.x), "=r"(v.y) : "l"(p) : "memory"); return v;
}
__device__ __forceinline__ void st_vol2(uint2* p, uint2 v) {
    asm volatile("st.volatile.global.v2.u32 [%0], {%1,%2};" :: "l"(p), "r"(v.x), "r"(v.y) : "memory");
}
__device__ __forceinline__ uint4 ld_vol4(const uint4* p) {
    uint4 v; asm volatile("ld.volatile.global.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(p) : "memory"); return v;
}
__device__ __forceinline__ void st_vol4(uint4* p, uint4 v) {
    asm volatile("st.volatile.global.v4.u32 [%0], {%1,%2,%3,%4};" :: "l"(p), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w) : "memory");
}

struct Args {
    int R, M, nwords;       // ranks, laps, 4-byte data words per message
    float* own;             // [R][nwords]
    float* inbox;           // [R][nwords]  (V0-V2)
    uint32_t* flags;        // [R]          (V0-V2)
    uint2* ll;              // [R][nwords]  (V3)
    uint4* ll4;             // [R][nwords/2] (V4)
    unsigned long long* t;  // [2]
};

template <int V>
__global__ void __launch_bounds__(THREADS) ring_probe(Args a) {
    const int r = blockIdx.x, R = a.R, right = (r + 1) % R, tid = threadIdx.x;
    const int n = a.nwords;
    __shared__ int s_dummy;
    if (r == 0 && tid == 0) a.t[0] = gtimer();
    for (int lap = 0; lap < a.M; ++lap) {
        const uint32_t seq = lap + 1;
        const bool first = (r == 0 && lap == 0);
        if (V <= 2) {
            if (!first) {
                if (tid == 0) {
                    const uint32_t want = (r == 0) ? seq - 1 : seq;
                    while (true) {
                        const uint32_t f = V == 2 ? ld_acq_gpu(a.flags + r) : ld_acq_sys(a.flags + r);
                        if (f >= want) break;
                        if (V == 0) __nanosleep(64);
                    }
                }
                __syncthreads();
            }
            float* out = a.inbox + (size_t)right * n;
            const float* in = a.inbox + (size_t)r * n;
            for (int i = tid * 4; i < n; i += THREADS * 4) {
                float4 v = *reinterpret_cast<const float4*>(a.own + (size_t)r * n + i);
                if (!first) {
                    const float4 u = __ldcg(reinterpret_cast<const float4*>(in + i));
                    v.x += u.x; v.y += u.y; v.z += u.z; v.w += u.w;
                }
                *reinterpret_cast<float4*>(out + i) = v;
            }
            __syncthreads();
            if (tid == 0) {
                if (V == 2) st_rel_gpu(a.flags + right, seq); else st_rel_sys(a.flags + right, seq);
            }
        } else if (V == 3) {
            const uint32_t want = (r == 0) ? seq - 1 : seq;
            uint2* out = a.ll + (size_t)right * n;
            const uint2* in = a.ll + (size_t)r * n;
            for (int i = tid; i < n; i += THREADS) {
                float v = a.own[(size_t)r * n + i];
                if (!first) {
                    uint2 w;
                    do { w = ld_vol2(in + i); } while (w.y < want);
                    v += __uint_as_float(w.x);
                }
                st_vol2(out + i, make_uint2(__float_as_uint(v), seq));
            }
        } else {
            const uint32_t want = (r == 0) ? seq - 1 : seq;
            uint4* out = a.ll4 + (size_t)right * (n / 2);
            const uint4* in = a.ll4 + (size_t)r * (n / 2);
            for (int i = tid; i < n / 2; i += THREADS) {
                float v0 = a.own[(size_t)r * n + 2 * i], v1 = a.own[(size_t)r * n + 2 * i + 1];
                if (!first) {
                    uint4 w;
                    do { w = ld_vol4(in + i); } while (w.y < want || w.w < want);
                    v0 += __uint_as_float(w.x);
                    v1 += __uint_as_float(w.z);
                }
                st_vol4(out + i, make_uint4(__float_as_uint(v0), seq, __float_as_uint(v1), seq));
            }
        }
    }
    (void)s_dummy;
    // rank 0 waits for the last lap's message to come back
    if (r == 0) {
        const uint32_t want = a.M;
        if (V <= 2) {
            if (tid == 0) while ((V == 2 ? ld_acq_gpu(a.flags) : ld_acq_sys(a.flags)) < want) {}
            __syncthreads();
        } else if (V == 3) {
            for (int i = tid; i < n; i += THREADS) while (ld_vol2(a.ll + i).y < want) {}
            __syncthreads();
        } else {
            for (int i = tid; i < n / 2; i += THREADS) while (ld_vol4(a.ll4 + i).y < want) {}
            __syncthreads();
        }
        if (tid == 0) a.t[1] = gtimer();
    }
}

template <int V>
double run(int R, int M, int nwords) {
    Args a;
    a.R = R; a.M = M; a.nwords = nwords;
    CK(cudaMalloc(&a.own, (size_t)R * nwords * 4));
    CK(cudaMalloc(&a.inbox, (size_t)R * nwords * 4));
    CK(cudaMalloc(&a.flags, (size_t)R * 4));
    CK(cudaMalloc(&a.ll, (size_t)R * nwords * 8));
    CK(cudaMalloc(&a.ll4, (size_t)R * nwords * 8));
    CK(cudaMalloc(&a.t, 16));
    CK(cudaMemset(a.own, 0, (size_t)R * nwords * 4));
    double best = 1e30;
    for (int rep = 0; rep < 3; ++rep) {
        CK(cudaMemset(a.flags, 0, (size_t)R * 4));
        CK(cudaMemset(a.ll, 0, (size_t)R * nwords * 8));
        CK(cudaMemset(a.ll4, 0, (size_t)R * nwords * 8));
        void* args[] = {&a};
        CK(cudaLaunchCooperativeKernel((const void*)ring_probe<V>, dim3(R), dim3(THREADS), args, 0, 0));
        CK(cudaDeviceSynchronize());
        unsigned long long t[2];
        CK(cudaMemcpy(t, a.t, 16, cudaMemcpyDeviceToHost));
        const double ns = (double)(t[1] - t[0]) / ((double)M * R);
        if (ns < best) best = ns;
    }
    cudaFree(a.own); cudaFree(a.inbox); cudaFree(a.flags); cudaFree(a.ll); cudaFree(a.ll4); cudaFree(a.t);
    return best;
}

int main() {
    const int R = 8, M = 200;
    printf("ns per hop, R=%d ranks (CTAs), %d laps, 512 threads\n", R, M);
    printf("%10s %10s %10s %10s %10s %10s\n", "bytes", "V0 rel.sys", "V1 nosleep", "V2 .gpu", "V3 LL8", "V4 LL16");
    for (int bytes : {512, 2048, 8192, 32768, 131072}) {
        const int nw = bytes / 4;
        printf("%10d %10.0f %10.0f %10.0f %10.0f %10.0f\n", bytes, run<0>(R, M, nw), run<1>(R, M, nw), run<2>(R, M, nw),
               run<3>(R, M, nw), run<4>(R, M, nw));
    }
    return 0;
}
