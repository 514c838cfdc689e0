// mma_probe.cu -- tcgen05.mma issue/execution rate from shared-memory operands (SS mode)
// versus N, with the issuing thread doing nothing else.  Build + run on the GPU box:
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_1906_06496_b200/csrc \
//        scripts/probes/mma_probe.cu -o /tmp/mma_probe -lcuda && /tmp/mma_probe
#include <cstdio>
#include <cuda_runtime.h>
#include "umma.cuh"
using namespace tem::umma;

template <int N, int NMMA, bool PRECOMP>
__global__ void __launch_bounds__(128, 1) probe(long long* out) {
    extern __shared__ __align__(1024) uint8_t sm[];
    uint8_t* s = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(sm) + 1023) & ~uintptr_t(1023));
    __shared__ uint64_t bar;
    __shared__ uint32_t slot;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    for (int i = threadIdx.x; i < 64 * 1024 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(s)[i] = 0;
    if (threadIdx.x == 0) { mbar_init(&bar, 1); fence_barrier_init(); }
    if (warp == 0) tmem_alloc<512>(&slot);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tb = slot;
    if (warp == 0 && lane == 0) {
        constexpr uint32_t idesc = make_idesc_bf16(128, N, false, false);
        const uint32_t a = smem_u32(s), b = smem_u32(s + 16384);
        const uint64_t ad0 = make_desc(a, 16, 1024), bd0 = make_desc(b, 16, 1024);
        long long t0 = clock64();
        #pragma unroll 4
        for (int i = 0; i < NMMA; ++i) {
            const int k = i & 3;
            uint64_t ad, bd;
            if (PRECOMP) { ad = ad0 + (uint64_t)(k * 2); bd = bd0 + (uint64_t)(k * 2); }
            else { ad = make_desc(a + k * 32, 16, 1024); bd = make_desc(b + k * 32, 16, 1024); }
            mma_bf16(tb, ad, bd, idesc, i ? 1u : 0u);
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

template <int N, bool PRECOMP>
void run(long long* d, int grid) {
    constexpr int NMMA = 4096;
    auto k = probe<N, NMMA, PRECOMP>;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 80 * 1024);
    k<<<grid, 128, 80 * 1024>>>(d);
    k<<<grid, 128, 80 * 1024>>>(d);
    cudaError_t e = cudaDeviceSynchronize();
    long long h[2];
    cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
    printf("N=%3d precomp=%d grid=%3d: issue %.1f clk/mma, complete %.1f clk/mma (floor %d) %s\n", N, PRECOMP, grid,
           (double)h[0] / NMMA, (double)h[1] / NMMA, 128 * N / 256, cudaGetErrorString(e));
}

int main() {
    long long* d;
    cudaMalloc(&d, 16);
    for (int grid : {1, 148}) {
        run<32, false>(d, grid); run<64, false>(d, grid); run<64, true>(d, grid);
        run<128, false>(d, grid); run<128, true>(d, grid); run<256, false>(d, grid); run<256, true>(d, grid);
    }
    return 0;
}
