// mma_cadence_probe.cu -- the fp32 dual-accumulator MMA pattern issued by a CONVERGED warp
// (elect.sync, as the kernels now do), with the per-tap synchronisation the halo kernel needs:
//   mode 0: none; 1: commit per tap; 2: commit + mbarrier wait (completed phase) per tap;
//   3: commit + named-barrier sync with a helper warp that did the mbarrier wait per tap.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_1906_06496_b200/csrc \
//        scripts/probes/mma_cadence_probe.cu -o /tmp/mma_cad && /tmp/mma_cad
#include <cstdio>
#include <cuda_runtime.h>
#include "umma.cuh"
using namespace tem::umma;

template <int MODE>
__global__ void __launch_bounds__(128, 1) probe(long long* out, int nk) {
    extern __shared__ __align__(1024) uint8_t sm[];
    uint8_t* s = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(sm) + 1023) & ~uintptr_t(1023));
    __shared__ uint64_t bar, bar2, ring[6];
    __shared__ uint32_t slot;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    for (int i = threadIdx.x; i < 200 * 1024 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(s)[i] = 0;
    if (threadIdx.x == 0) {
        mbar_init(&bar, 1); mbar_init(&bar2, 1);
        for (int q = 0; q < 6; ++q) mbar_init(&ring[q], 1);
        fence_barrier_init();
    }
    if (warp == 0) tmem_alloc<512>(&slot);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    if (threadIdx.x == 0) for (int q = 0; q < 6; ++q) mbar_arrive_local(&ring[q]);  // phase 0 complete
    __syncthreads();
    const uint32_t tb = slot;
    const int ntap = nk / 4;
    if (warp == 1) {  // helper: waits on the (completed) ring phase, then releases the MMA warp
        if (MODE == 3)
            for (int t = 0; t < ntap; ++t) {
                mbar_wait(&ring[t % 6], 0);
                asm volatile("bar.arrive 1, 64;" ::: "memory");
            }
    } else if (warp == 0) {
        const bool issuer = elect_one_sync();
        constexpr uint32_t id2 = make_idesc_bf16(128, 128, false, false), id1 = make_idesc_bf16(128, 64, false, false);
        long long t0 = clock64();
        for (int t = 0; t < ntap; ++t) {
            if (MODE == 2) mbar_wait(&ring[t % 6], 0);
            if (MODE == 3) asm volatile("bar.sync 1, 64;" ::: "memory");
            if (MODE >= 2) tc_fence_after();
            const int st = t % 6;
            const uint32_t ahi = smem_u32(s) + (st % 3) * 34816 + 128, alo = ahi + 17408;
            const uint32_t bhl = smem_u32(s) + 104448 + st * 16384;
            const uint64_t a0 = make_desc(ahi, 16, 1024), a1 = make_desc(alo, 16, 1024), b0 = make_desc(bhl, 16, 1024);
#pragma unroll
            for (int k = 0; k < 4; ++k)
                if (issuer) {
                    mma_bf16(tb, a0 + 2 * k, b0 + 2 * k, id2, (t | k) ? 1u : 0u);
                    mma_bf16(tb + 128, a1 + 2 * k, b0 + 2 * k, id1, (t | k) ? 1u : 0u);
                }
            if (MODE >= 1 && issuer) mma_commit(&bar2);
        }
        long long t1 = clock64();
        if (issuer) mma_commit(&bar);
        mbar_wait(&bar, 0);
        long long t2 = clock64();
        if (blockIdx.x == 0 && lane == 0) { out[0] = t1 - t0; out[1] = t2 - t0; }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 0) { tc_fence_after(); tmem_dealloc<512>(tb); }
}

template <int MODE>
void run(long long* d) {
    const int nk = 4096;
    auto k = probe<MODE>;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 210 * 1024);
    k<<<1, 128, 210 * 1024>>>(d, nk);
    k<<<1, 128, 210 * 1024>>>(d, nk);
    cudaError_t e = cudaDeviceSynchronize();
    long long h[2];
    cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
    printf("converged warp, mode %d: %.1f clk per K-step pair %s\n", MODE, (double)h[1] / nk, cudaGetErrorString(e));
    fflush(stdout);
}

int main() {
    long long* d;
    cudaMalloc(&d, 16);
    run<0>(d); run<1>(d); run<2>(d);  // mode 3 (named barrier with a helper warp) hung; see DESIGN 6.3b
    return 0;
}
