// mma_dual_probe.cu -- rate of the fp32 path's MMA pattern (R16): per K-step of
// 16, A_hi x [B_hi | B_lo] at N = 2*BN into accumulator 0, then A_lo x B_hi at N = BN into
// accumulator 1, with the A descriptors at a halo row offset (tap j: +j*128 B).  Isolated from
// TMA: operands static in shared memory.  Build + run on the GPU box:
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_1906_06496_b200/csrc \
//        scripts/probes/mma_dual_probe.cu -o /tmp/mma_dual && /tmp/mma_dual
#include <cstdio>
#include <cuda_runtime.h>
#include "umma.cuh"
using namespace tem::umma;

__device__ __forceinline__ uint32_t mbar_test(uint64_t* bar, uint32_t parity) {
    uint32_t ok;
    asm volatile("{\n.reg .pred p;\nmbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\nselp.u32 %0, 1, 0, p;\n}\n"
                 : "=r"(ok) : "r"(smem_u32(bar)), "r"(parity) : "memory");
    return ok;
}

template <int BN, int TAPOFF, int NSTAGE = 1, int CADENCE = 0, bool BMN = false>
__global__ void __launch_bounds__(128, 1) probe(long long* out, int nk) {
    extern __shared__ __align__(1024) uint8_t sm[];
    uint8_t* s = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(sm) + 1023) & ~uintptr_t(1023));
    __shared__ uint64_t bar, bar2, bar3, ring[6];
    __shared__ uint32_t slot;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    for (int i = threadIdx.x; i < 200 * 1024 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(s)[i] = 0;
    if (threadIdx.x == 0) {
        mbar_init(&bar, 1); mbar_init(&bar2, 1); mbar_init(&bar3, 1);
        for (int q = 0; q < 6; ++q) mbar_init(&ring[q], 1);
        fence_barrier_init();
    }
    if (warp == 0) tmem_alloc<512>(&slot);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tb = slot;
    if (warp == 0 && lane == 0) {
        constexpr uint32_t id2 = make_idesc_bf16(128, 2 * BN, false, BMN), id1 = make_idesc_bf16(128, BN, false, BMN);
        // A_hi window at 0, A_lo at 24 KB (130 rows x 128 B each + pad), B [hi|lo] at 48 KB
        if (CADENCE == 3)
            for (int q = 0; q < 5; ++q) mbar_arrive_local(&ring[q]);  // taps 0..4 "loaded" up front
        if (CADENCE == 4 || CADENCE == 5 || CADENCE == 7)
            for (int q = 0; q < 6; ++q) mbar_arrive_local(&ring[q]);  // taps 0..5 "loaded" up front
        long long t0 = clock64();
        uint32_t ready = 1;
        for (int i = 0; i < nk; ++i) {
            const int k = i & 3;
            if (CADENCE == 7 && k == 1) ready = mbar_test(&ring[((i >> 2) + 1) % 6], 0);  // early check, completed phase
            if (CADENCE == 4 && k == 1) {  // check the next tap's barrier early (non-blocking)
                const int t = (i >> 2) + 1;
                ready = mbar_test(&ring[t % 6], (t / 6) & 1);
            }
            // NSTAGE > 1: walk distinct operand buffers (A stages 34 KB apart, B stages 16 KB apart)
            const int st = (i >> 2) % NSTAGE;
            const uint32_t ahi = smem_u32(s) + (NSTAGE > 1 ? st % 3 : 0) * 34816 + TAPOFF * 128;
            const uint32_t alo = ahi + 17408;
            const uint32_t bhl = smem_u32(s) + (NSTAGE > 1 ? 104448 + (st % 6) * 16384 : 49152);
            const uint64_t a0 = make_desc(ahi + k * 32, 16, 1024), a1 = make_desc(alo + k * 32, 16, 1024);
            // BMN: DGRAD's MN-major B (LBO = one 64-column panel of K rows, K-steps of 16 rows)
            const uint64_t b0 = BMN ? make_desc(bhl + k * 2048, 64 * 128, 1024) : make_desc(bhl + k * 32, 16, 1024);
            mma_bf16(tb, a0, b0, id2, i ? 1u : 0u);
            mma_bf16(tb + 2 * BN, a1, b0, id1, i ? 1u : 0u);
            if (CADENCE && k == 3) {  // the kernel's per-tap cadence: commit, then wait + fence
                mma_commit(&bar2);
                if (CADENCE == 2) { mbar_arrive_local(&bar3); mbar_wait(&bar3, (i >> 2) & 1); }
                if (CADENCE == 5) mbar_wait(&ring[(i >> 2) % 6], 0);  // completed phase: the wait alone
                if (CADENCE == 7 && !ready) mbar_wait(&ring[((i >> 2) + 1) % 6], 0);
                if (CADENCE == 6) tc_fence_after();                     // (commit + fence only, = cadence 1)
                if (CADENCE == 4) {
                    const int t = i >> 2;
                    mbar_arrive_local(&ring[(t + 6) % 6]);  // "load" of tap t + 6 (same slot as t)
                    if (!ready) mbar_wait(&ring[(t + 1) % 6], ((t + 1) / 6) & 1);
                }
                if (CADENCE == 3) {  // wait on a phase completed 5 taps earlier (as the kernel's rings)
                    const int t = i >> 2;
                    mbar_arrive_local(&ring[(t + 5) % 6]);
                    mbar_wait(&ring[t % 6], (t / 6) & 1);
                }
                tc_fence_after();
            }
        }
        long long t1 = clock64();
        mma_commit(&bar);
        mbar_wait(&bar, 0);
        long long t2 = clock64();
        if (blockIdx.x == 0) { out[0] = t1 - t0; out[1] = t2 - t0; }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 0) { tc_fence_after(); tmem_dealloc<512>(tb); }
}

template <int BN, int TAPOFF, int NSTAGE = 1, int CADENCE = 0, bool BMN = false>
void run(long long* d, int grid) {
    const int nk = 4096;
    auto k = probe<BN, TAPOFF, NSTAGE, CADENCE, BMN>;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 210 * 1024);
    k<<<grid, 128, 210 * 1024>>>(d, nk);
    k<<<grid, 128, 210 * 1024>>>(d, nk);
    cudaError_t e = cudaDeviceSynchronize();
    long long h[2];
    cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
    const int floor_clk = 128 * 2 * BN / 256 + 128 * BN / 256;
    printf("BN=%3d tap=%d stages=%d cadence=%d bmn=%d grid=%3d: %.1f clk per K-step pair (MMA floor %d) %s\n", BN, TAPOFF, NSTAGE, CADENCE, (int)BMN, grid,
           (double)h[1] / nk, floor_clk, cudaGetErrorString(e));
}

int main() {
    long long* d;
    cudaMalloc(&d, 16);
    for (int grid : {1, 104}) {
        run<64, 1, 6, 0>(d, grid); run<64, 1, 6, 1>(d, grid); run<64, 1, 6, 2>(d, grid); run<64, 1, 6, 3>(d, grid);
        run<64, 1, 6, 4>(d, grid); run<64, 1, 6, 5>(d, grid); run<64, 1, 6, 7>(d, grid);
    }
    return 0;
}
