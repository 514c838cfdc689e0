// tem_umma.cu -- tcgen05 / TMA implicit-GEMM convolutions of the BSN-TEM step (sm_100a).
//
// One warp-specialised kernel template serves the five dense contractions of the step
// (SURVEY 8(a) rows a1, a2, a6, a7, a8):
//   FWD   out[p][o] = act(bias[o] + sum_{j,c} in[p+j-1][c] * W[o][j][c])   A K-major, B K-major
//   DGRAD dA1[p][c] = 1[h1>0] sum_{j,o} dA2[p+1-j][o] * W2[o][j][c]         A K-major, B MN-major
//   WGRAD part[s][o][j*Cin+c] = sum_{p in split s} dA[p][o] * in[p+j-1][c]  A MN-major, B MN-major
// Activations use the halo-padded row layout [B][T+2][C] (zero rows at every video
// boundary), so each k=3 tap is a plain TMA row offset; out-of-range rows/columns are
// zero-filled by TMA.  Operands are bf16 in 128B-swizzled shared memory; accumulators
// live in TMEM (128 lanes x BN fp32 columns).
//
// Precision:  NPASS = 1 -> bf16 operands, fp32 accumulate (TEM_BF16, reading R8).
//             NPASS = 3 -> "fp32" path: every operand is split x = hi + lo with
//             hi = bf16(x), lo = bf16(x - hi) (|x - hi - lo| <= 2^-17 |x|), and the product
//             is hi*hi + hi*lo + lo*hi accumulated in fp32 -- ~2^-16 relative per product,
//             inside the 1e-4 contract.
//
// Warp roles (192 threads): warp 0 = TMA producer, warp 1 = TMEM allocator + MMA issuer
// (one elected lane), warps 2..5 = epilogue (TMEM -> registers -> global).
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>

#include "kernels.h"
#include "umma.cuh"

namespace tem {
namespace umma {

constexpr int BM = 128;
constexpr int BK = 64;   // bf16 elements per k-block = one 128-byte swizzle row
constexpr int UK = 16;   // K per tcgen05.mma (kind::f16)
constexpr int NTHREADS = 192;

template <int BN, int NPASS, int STAGES>
struct Cfg {
    static constexpr int NPL = NPASS == 3 ? 2 : 1;
    static constexpr uint32_t A_BYTES = BM * BK * 2;
    static constexpr uint32_t B_BYTES = BN * BK * 2;
    static constexpr uint32_t STAGE_BYTES = NPL * (A_BYTES + B_BYTES);
    static constexpr uint32_t SMEM = STAGES * STAGE_BYTES + 1024 /*align*/ + 256 /*barriers*/ +
                                     4 * BN * 4 /*epilogue column sums*/;
    static constexpr int TMEM_COLS = BN < 32 ? 32 : BN;
};

TEM_DEV bool halo_row(int p, int Tp) {
    const int t = p % Tp;
    return t == 0 || t == Tp - 1;
}

TEM_DEV uint32_t pack_bf16x2(float a, float b) {
    __nv_bfloat162 v = __floats2bfloat162_rn(a, b);
    return *reinterpret_cast<uint32_t*>(&v);
}

// Store 16 consecutive values as bf16 (hi) and optionally the residual plane (lo).
TEM_DEV void store16_planes(__nv_bfloat16* hi, __nv_bfloat16* lo, const float (&v)[16]) {
    uint32_t h[8], l[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) {
        const __nv_bfloat16 h0 = __float2bfloat16_rn(v[2 * i]), h1 = __float2bfloat16_rn(v[2 * i + 1]);
        __nv_bfloat162 hh;
        hh.x = h0;
        hh.y = h1;
        h[i] = *reinterpret_cast<uint32_t*>(&hh);
        if (lo) l[i] = pack_bf16x2(v[2 * i] - __bfloat162float(h0), v[2 * i + 1] - __bfloat162float(h1));
    }
    uint4* dh = reinterpret_cast<uint4*>(hi);
    dh[0] = make_uint4(h[0], h[1], h[2], h[3]);
    dh[1] = make_uint4(h[4], h[5], h[6], h[7]);
    if (lo) {
        uint4* dl = reinterpret_cast<uint4*>(lo);
        dl[0] = make_uint4(l[0], l[1], l[2], l[3]);
        dl[1] = make_uint4(l[4], l[5], l[6], l[7]);
    }
}

// Column sums of a 32-row x 16-column register tile (one row per lane): a reduce-scatter
// over the warp in a fixed order.  Returns, in lanes L and L^1, the 32-row sum of
// column ((L>>4)&1)*8 + ((L>>3)&1)*4 + ((L>>2)&1)*2 + ((L>>1)&1).
TEM_DEV float warp_colsum16(const float (&v)[16], int lane, int* col) {
    const bool b4 = lane & 16, b3 = lane & 8, b2 = lane & 4, b1 = lane & 2;
    float a[8], b[4], c[2];
#pragma unroll
    for (int i = 0; i < 8; ++i) {
        const float keep = b4 ? v[i + 8] : v[i], send = b4 ? v[i] : v[i + 8];
        a[i] = keep + __shfl_xor_sync(0xffffffffu, send, 16);
    }
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        const float keep = b3 ? a[i + 4] : a[i], send = b3 ? a[i] : a[i + 4];
        b[i] = keep + __shfl_xor_sync(0xffffffffu, send, 8);
    }
#pragma unroll
    for (int i = 0; i < 2; ++i) {
        const float keep = b2 ? b[i + 2] : b[i], send = b2 ? b[i] : b[i + 2];
        c[i] = keep + __shfl_xor_sync(0xffffffffu, send, 4);
    }
    float d = (b1 ? c[1] : c[0]) + __shfl_xor_sync(0xffffffffu, b1 ? c[0] : c[1], 2);
    d += __shfl_xor_sync(0xffffffffu, d, 1);
    *col = (b4 ? 8 : 0) + (b3 ? 4 : 0) + (b2 ? 2 : 0) + (b1 ? 1 : 0);
    return d;
}

template <int MODE, int BN, int NPASS, int STAGES>
__global__ void __launch_bounds__(NTHREADS, 1) umma_conv_kernel(const __grid_constant__ UmmaParams P) {
    using C_ = Cfg<BN, NPASS, STAGES>;
    constexpr int NPL = C_::NPL;
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + STAGES * C_::STAGE_BYTES);
    uint64_t* empty = full + STAGES;
    uint64_t* tfull = empty + STAGES;
    uint32_t* tslot = reinterpret_cast<uint32_t*>(tfull + 1);
    float* csum = reinterpret_cast<float*>(smem + STAGES * C_::STAGE_BYTES + 256);  // [4][BN]

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int m0 = blockIdx.x * BM;
    const int ntile = blockIdx.y;
    const int split = blockIdx.z;

    // k-block range
    int nkb, p_begin = 0;
    if (MODE == WGRAD_) {
        p_begin = split * P.ksplit_rows;
        const int p_end = min(P.R, p_begin + P.ksplit_rows);
        nkb = (p_end - p_begin + BK - 1) / BK;
    } else {
        nkb = 3 * P.cpb;
    }

    if (warp == 0 && lane == 0) {
        for (int i = 0; i < 2; ++i) {
            tma_prefetch(&P.a[i]);
            tma_prefetch(&P.b[i]);
        }
        for (int s = 0; s < STAGES; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], 1);
        }
        mbar_init(tfull, 1);
        fence_barrier_init();
    }
    if (warp == 1) tmem_alloc<C_::TMEM_COLS>(tslot);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tbase = *tslot;

    if (warp == 0) {
        if (lane == 0) {
            // ===================== TMA producer =====================
            for (int kb = 0; kb < nkb; ++kb) {
                const int s = kb % STAGES;
                const uint32_t ph = (kb / STAGES) & 1;
                mbar_wait(&empty[s], ph ^ 1);
                uint8_t* st = smem + s * C_::STAGE_BYTES;
                mbar_arrive_expect_tx(&full[s], C_::STAGE_BYTES);
#pragma unroll
                for (int pl = 0; pl < NPL; ++pl) {
                    uint8_t* sa = st + pl * C_::A_BYTES;
                    uint8_t* sb = st + NPL * C_::A_BYTES + pl * C_::B_BYTES;
                    if (MODE == FWD_) {
                        const int j = kb / P.cpb, c0 = (kb % P.cpb) * BK;
                        tma_load_2d(sa, &P.a[pl], &full[s], c0, m0 + j - 1);
                        tma_load_2d(sb, &P.b[pl], &full[s], j * P.Kc + c0, ntile * BN);
                    } else if (MODE == DGRAD_) {
                        const int j = kb / P.cpb, o0 = (kb % P.cpb) * BK;
                        tma_load_2d(sa, &P.a[pl], &full[s], o0, m0 + 1 - j);
#pragma unroll
                        for (int q = 0; q < BN / 64; ++q)
                            tma_load_3d(sb + q * (BK * 128), &P.b[pl], &full[s], ntile * BN + 64 * q, j, o0);
                    } else {  // WGRAD
                        const int p0 = p_begin + kb * BK;
#pragma unroll
                        for (int q = 0; q < BM / 64; ++q)
                            tma_load_2d(sa + q * (BK * 128), &P.a[pl], &full[s], m0 + 64 * q, p0);
#pragma unroll
                        for (int q = 0; q < BN / 64; ++q) {
                            int g = ntile * (BN / 64) + q;
                            if (P.ones_chunk && g == 3 * P.cpj) {
                                // all-ones B chunk (lo plane: zeros): column 0 of D = sum_p dA[p][o],
                                // the bias gradient, on the tensor core in the same split precision
                                tma_load_2d(sb + q * (BK * 128), &P.ones, &full[s], 64 * pl, p0);
                                continue;
                            }
                            if (g >= 3 * P.cpj) g = 3 * P.cpj - 1;  // dummy chunk, discarded by the epilogue
                            const int j = g / P.cpj, c0 = (g % P.cpj) * 64;
                            tma_load_2d(sb + q * (BK * 128), &P.b[pl], &full[s], c0, p0 + j - 1);
                        }
                    }
                }
            }
        }
    } else if (warp == 1) {
        if (lane == 0) {
            // ===================== MMA issuer =====================
            constexpr bool A_MN = (MODE == WGRAD_);
            constexpr bool B_MN = (MODE != FWD_);
            constexpr uint32_t idesc = make_idesc_bf16(BM, BN, A_MN, B_MN);
            for (int kb = 0; kb < nkb; ++kb) {
                const int s = kb % STAGES;
                const uint32_t ph = (kb / STAGES) & 1;
                mbar_wait(&full[s], ph);
                tc_fence_after();
                const uint32_t st = smem_u32(smem + s * C_::STAGE_BYTES);
#pragma unroll
                for (int k = 0; k < BK / UK; ++k) {
#pragma unroll
                    for (int pass = 0; pass < NPASS; ++pass) {
                        const int pa = (pass == 2) ? 1 : 0;  // hi*hi, hi*lo, lo*hi
                        const int pb = (pass == 1) ? 1 : 0;
                        const uint32_t a_addr = st + pa * C_::A_BYTES;
                        const uint32_t b_addr = st + NPL * C_::A_BYTES + pb * C_::B_BYTES;
                        uint64_t ad, bd;
                        if (A_MN) ad = make_desc(a_addr + k * (UK * 128), BK * 128, 1024);
                        else ad = make_desc(a_addr + k * (UK * 2), 16, 1024);
                        if (B_MN) bd = make_desc(b_addr + k * (UK * 128), BK * 128, 1024);
                        else bd = make_desc(b_addr + k * (UK * 2), 16, 1024);
                        mma_bf16(tbase, ad, bd, idesc, (kb | k | pass) != 0 ? 1u : 0u);
                    }
                }
                mma_commit(&empty[s]);  // frees the smem stage once these MMAs are done
            }
            mma_commit(tfull);  // accumulator complete
        }
        __syncwarp();
    } else {
        // ===================== epilogue (warps 2..5) =====================
        const int q = warp & 3;  // TMEM lane quarter accessible to this warp
        const int row = m0 + 32 * q + lane;
        mbar_wait(tfull, 0);
        tc_fence_after();
#pragma unroll 1
        for (int c16 = 0; c16 < BN / 16; ++c16) {
            uint32_t r[16];
            tmem_ld16(tbase + ((uint32_t)(32 * q) << 16) + (uint32_t)(c16 * 16), r);
            tmem_ld_wait();
            float v[16];
#pragma unroll
            for (int i = 0; i < 16; ++i) v[i] = __uint_as_float(r[i]);
            if (MODE == FWD_ || MODE == DGRAD_) {
                const int n = ntile * BN + c16 * 16;  // Nout is a multiple of BN
                const bool valid = row < P.R;
                const bool halo = !valid || halo_row(row, P.Tp);
                if (MODE == FWD_) {
#pragma unroll
                    for (int i = 0; i < 16; ++i) {
                        const float t = v[i] + P.bias[n + i];
                        v[i] = (!halo && t > 0.f) ? t : 0.f;
                    }
                } else {
                    uint32_t mw[8] = {0, 0, 0, 0, 0, 0, 0, 0};
                    if (!halo) {
                        const uint4* mk = reinterpret_cast<const uint4*>(
                            static_cast<const __nv_bfloat16*>(P.mask) + (size_t)row * P.Nout + n);
                        const uint4 m0v = mk[0], m1v = mk[1];
                        mw[0] = m0v.x; mw[1] = m0v.y; mw[2] = m0v.z; mw[3] = m0v.w;
                        mw[4] = m1v.x; mw[5] = m1v.y; mw[6] = m1v.z; mw[7] = m1v.w;
                    }
#pragma unroll
                    for (int i = 0; i < 8; ++i) {
                        const bool p0 = __uint_as_float(mw[i] << 16) > 0.f;
                        const bool p1 = __uint_as_float(mw[i] & 0xFFFF0000u) > 0.f;
                        v[2 * i] = p0 ? v[2 * i] : 0.f;
                        v[2 * i + 1] = p1 ? v[2 * i + 1] : 0.f;
                    }
                    if (P.bsum) {
                        // bias gradient of conv1 (row a8): column sums of the STORED operand
                        // (bf16(v) [+ bf16(v - bf16(v))]), reduced over this CTA's 128 rows
                        float sv[16];
#pragma unroll
                        for (int i = 0; i < 16; ++i) {
                            const float h = __bfloat162float(__float2bfloat16_rn(v[i]));
                            sv[i] = P.out_lo ? h + __bfloat162float(__float2bfloat16_rn(v[i] - h)) : h;
                        }
                        int col;
                        const float cs = warp_colsum16(sv, lane, &col);
                        if ((lane & 1) == 0) csum[q * BN + c16 * 16 + col] = cs;
                    }
                }
                if (!valid) continue;
                if (P.out_f32) {
                    float4* d = reinterpret_cast<float4*>(static_cast<float*>(P.out_hi) + (size_t)row * P.Nout + n);
#pragma unroll
                    for (int i = 0; i < 4; ++i) d[i] = make_float4(v[4 * i], v[4 * i + 1], v[4 * i + 2], v[4 * i + 3]);
                } else {
                    __nv_bfloat16* hi = static_cast<__nv_bfloat16*>(P.out_hi) + (size_t)row * P.Nout + n;
                    __nv_bfloat16* lo = P.out_lo ? static_cast<__nv_bfloat16*>(P.out_lo) + (size_t)row * P.Nout + n
                                                 : nullptr;
                    store16_planes(hi, lo, v);
                }
            } else {  // WGRAD partial: row = o, columns -> (j, c)
                const int nl = c16 * 16;
                const int g = ntile * (BN / 64) + nl / 64;
                if (P.ones_chunk && g == 3 * P.cpj) {
                    if (nl % 64 == 0)  // column 0 of the ones chunk: bias gradient partial
                        P.part[(size_t)split * P.part_stride + (size_t)P.Nout * P.NW + row] = v[0];
                    continue;
                }
                if (g >= 3 * P.cpj) continue;
                const int j = g / P.cpj, c = (g % P.cpj) * 64 + (nl % 64);
                if (c >= P.Cin_w) continue;
                float* dst = P.part + (size_t)split * P.part_stride + (size_t)row * P.NW + (size_t)j * P.Cin_w + c;
                if (c + 16 <= P.Cin_w) {
#pragma unroll
                    for (int i = 0; i < 4; ++i)
                        reinterpret_cast<float4*>(dst)[i] = make_float4(v[4 * i], v[4 * i + 1], v[4 * i + 2], v[4 * i + 3]);
                } else {
#pragma unroll
                    for (int i = 0; i < 16; ++i)
                        if (c + i < P.Cin_w) dst[i] = v[i];
                }
            }
        }
        if (MODE == DGRAD_ && P.bsum) {
            // combine the 4 row-quarters in a fixed order -> bsum[m-tile][n]
            asm volatile("bar.sync 1, 128;" ::: "memory");
            const int et = threadIdx.x - 64;  // 0..127
            for (int cidx = et; cidx < BN; cidx += 128) {
                const float s = ((csum[cidx] + csum[BN + cidx]) + csum[2 * BN + cidx]) + csum[3 * BN + cidx];
                P.bsum[(size_t)blockIdx.x * P.Nout + ntile * BN + cidx] = s;
            }
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 1) {
        tc_fence_after();
        tmem_dealloc<C_::TMEM_COLS>(tbase);
    }
}

// ------------------------------------------------------------------ companions
// x [B][T][Cin] fp32 -> halo-padded hi/lo bf16 planes [B][T+2][Cin].
__global__ void prep_x_split_kernel(const float* __restrict__ x, __nv_bfloat16* __restrict__ hi,
                                    __nv_bfloat16* __restrict__ lo, int B, int Tn, int Cin) {
    const int per_row = Cin / 4;
    const int64_t total = (int64_t)B * (Tn + 2) * per_row;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
         i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t p = i / per_row;
        const int cv = (int)(i - p * per_row);
        const int t = (int)(p % (Tn + 2));
        const int64_t v = p / (Tn + 2);
        float4 a = make_float4(0.f, 0.f, 0.f, 0.f);
        if (t >= 1 && t <= Tn) a = reinterpret_cast<const float4*>(x + ((size_t)v * Tn + (t - 1)) * Cin)[cv];
        const __nv_bfloat16 h0 = __float2bfloat16_rn(a.x), h1 = __float2bfloat16_rn(a.y),
                            h2 = __float2bfloat16_rn(a.z), h3 = __float2bfloat16_rn(a.w);
        __nv_bfloat162 ha, hb;
        ha.x = h0; ha.y = h1; hb.x = h2; hb.y = h3;
        uint2 hv, lv;
        hv.x = *reinterpret_cast<uint32_t*>(&ha);
        hv.y = *reinterpret_cast<uint32_t*>(&hb);
        lv.x = pack_bf16x2(a.x - __bfloat162float(h0), a.y - __bfloat162float(h1));
        lv.y = pack_bf16x2(a.z - __bfloat162float(h2), a.w - __bfloat162float(h3));
        reinterpret_cast<uint2*>(hi + (size_t)p * Cin)[cv] = hv;
        reinterpret_cast<uint2*>(lo + (size_t)p * Cin)[cv] = lv;
    }
}

// Weight gradient = sum of the S split-K partials (ascending s); optionally followed by the
// bias gradient = sum of nbp per-m-tile column sums (ascending m).  Both fixed order.
__global__ void reduce_wgrad_kernel(const float* __restrict__ part, int64_t part_stride, int S, int64_t nW,
                                    const float* __restrict__ bpart, int nbp, int C, float* __restrict__ dst) {
    const int64_t nvw = nW / 4, nvb = nbp > 0 ? C / 4 : 0;
    for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < nvw + nvb;
         v += (int64_t)gridDim.x * blockDim.x) {
        float4 a;
        if (v < nvw) {
            a = reinterpret_cast<const float4*>(part)[v];
            for (int s = 1; s < S; ++s) {
                const float4 b = reinterpret_cast<const float4*>(part + (size_t)s * part_stride)[v];
                a.x += b.x; a.y += b.y; a.z += b.z; a.w += b.w;
            }
        } else {
            const int64_t cv = v - nvw;
            a = reinterpret_cast<const float4*>(bpart)[cv];
            for (int m = 1; m < nbp; ++m) {
                const float4 b = reinterpret_cast<const float4*>(bpart + (size_t)m * C)[cv];
                a.x += b.x; a.y += b.y; a.z += b.z; a.w += b.w;
            }
        }
        reinterpret_cast<float4*>(dst)[v] = a;
    }
}

// [R][128] bf16: columns 0..63 = 1.0, 64..127 = 0 (the bias-gradient "ones" operand)
__global__ void fill_ones_kernel(__nv_bfloat16* __restrict__ o, int64_t rows) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < rows * 128;
         i += (int64_t)gridDim.x * blockDim.x)
        o[i] = __float2bfloat16_rn((i & 127) < 64 ? 1.f : 0.f);
}

__global__ void cast_shadow_split_kernel(const float* __restrict__ w, __nv_bfloat16* __restrict__ hi,
                                         __nv_bfloat16* __restrict__ lo, int64_t n) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        const float v = w[i];
        const __nv_bfloat16 h = __float2bfloat16_rn(v);
        hi[i] = h;
        if (lo) lo[i] = __float2bfloat16_rn(v - __bfloat162float(h));
    }
}

}  // namespace umma

// ------------------------------------------------------------------ host side
namespace {

PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
    static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
    if (!fn) {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
    }
    return fn;
}

// bf16 2D tensor [outer][inner] (row-major), box {64, box_rows}, 128B swizzle, zero OOB fill.
bool map2d(CUtensorMap* m, const void* base, uint64_t inner, uint64_t outer, uint32_t box_rows) {
    auto fn = encode_fn();
    if (!fn || !base) return false;
    cuuint64_t dims[2] = {inner, outer};
    cuuint64_t strides[1] = {inner * 2};
    cuuint32_t box[2] = {64, box_rows};
    cuuint32_t es[2] = {1, 1};
    return fn(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims, strides, box, es,
              CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
              CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}
// W2 [o][j][c] as 3D (c, j, o), box {64, 1, BK}: an MN-major (c-contiguous) tile of BK o-rows.
bool map_w_mn(CUtensorMap* m, const void* base, uint64_t C) {
    auto fn = encode_fn();
    if (!fn || !base) return false;
    cuuint64_t dims[3] = {C, 3, C};
    cuuint64_t strides[2] = {C * 2, 3 * C * 2};
    cuuint32_t box[3] = {64, 1, (cuuint32_t)umma::BK};
    cuuint32_t es[3] = {1, 1, 1};
    return fn(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void*>(base), dims, strides, box, es,
              CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
              CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

template <int MODE, int BN, int NPASS, int STAGES>
cudaError_t launch_one(const UmmaParams& p, dim3 grid, cudaStream_t s) {
    using C_ = umma::Cfg<BN, NPASS, STAGES>;
    auto k = umma::umma_conv_kernel<MODE, BN, NPASS, STAGES>;
    static bool attr = false;
    if (!attr) {
        cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)C_::SMEM);
        if (e != cudaSuccess) return e;
        attr = true;
    }
    k<<<grid, umma::NTHREADS, C_::SMEM, s>>>(p);
    return cudaGetLastError();
}

}  // namespace

int umma_wgrad_splits(const Geom& g) {
    const int tiles = (g.C / umma::BM) * 6;
    int S = (148 + tiles - 1) / tiles;
    const int nkb = (g.R + umma::BK - 1) / umma::BK;
    if (S > nkb) S = nkb;
    if (S < 1) S = 1;
    return S;
}

bool umma_plan(const Geom& g, const RankBufs& b, UmmaPlan* plan) {
    const int npl = g.prec == TEM_FP32 ? 2 : 1;
    UmmaPlan& P = *plan;
    memset(&P, 0, sizeof(P));
    if (g.R == 0) return true;  // empty shard: nothing to plan (tem_compute takes the B = 0 branch)
    if (cudaStreamCreateWithFlags(&P.aux, cudaStreamNonBlocking) != cudaSuccess ||
        cudaEventCreateWithFlags(&P.fork, cudaEventDisableTiming) != cudaSuccess ||
        cudaEventCreateWithFlags(&P.join, cudaEventDisableTiming) != cudaSuccess)
        return false;
    P.npass = npl == 2 ? 3 : 1;
    const int R = g.R, Tp = g.T + 2;
    // tile widths: split (fp32) path uses narrower N tiles for more CTAs at small batch
    P.bn_fwd = (npl == 2 || (R + 127) / 128 * (g.C / 256) < 148) ? 128 : 256;
    if (npl == 2 && (R + 127) / 128 * (g.C / 128) < 148) P.bn_fwd = 64;
    const void* xp[2] = {b.xp, b.xp_lo};
    const void* h1[2] = {b.h1, b.h1_lo};
    const void* dA2[2] = {b.dA2, b.dA2_lo};
    const void* dA1[2] = {b.dA1, b.dA1_lo};
    const __nv_bfloat16* W[2] = {b.shadow, b.shadow_lo};
    bool ok = true;
    for (int pl = 0; pl < npl; ++pl) {
        const __nv_bfloat16* W1 = W[pl] + g.off_W1;
        const __nv_bfloat16* W2 = W[pl] + g.off_W2;
        // conv1 FWD: A = xp [R][Cin], B = W1 [C][3*Cin]
        ok &= map2d(&P.conv1.a[pl], xp[pl], g.Cin, R, umma::BM);
        ok &= map2d(&P.conv1.b[pl], W1, 3 * (uint64_t)g.Cin, g.C, P.bn_fwd);
        // conv2 FWD: A = h1 [R][C], B = W2 [C][3*C]
        ok &= map2d(&P.conv2.a[pl], h1[pl], g.C, R, umma::BM);
        ok &= map2d(&P.conv2.b[pl], W2, 3 * (uint64_t)g.C, g.C, P.bn_fwd);
        // DGRAD: A = dA2 [R][C] (K-major), B = W2 MN-major (3D)
        ok &= map2d(&P.dgrad.a[pl], dA2[pl], g.C, R, umma::BM);
        ok &= map_w_mn(&P.dgrad.b[pl], W2, g.C);
        // WGRAD2: A = dA2 MN-major box {64, BK}, B = h1 MN-major box {64, BK}
        ok &= map2d(&P.wgrad2.a[pl], dA2[pl], g.C, R, umma::BK);
        ok &= map2d(&P.wgrad2.b[pl], h1[pl], g.C, R, umma::BK);
        // WGRAD1: A = dA1, B = xp
        ok &= map2d(&P.wgrad1.a[pl], dA1[pl], g.C, R, umma::BK);
        ok &= map2d(&P.wgrad1.b[pl], xp[pl], g.Cin, R, umma::BK);
    }
    const int S = umma_wgrad_splits(g);
    const int nkb = (R + umma::BK - 1) / umma::BK;
    const int kb_per = (nkb + S - 1) / S;
    P.ksplit_rows = kb_per * umma::BK;
    P.S = (R + P.ksplit_rows - 1) / P.ksplit_rows;
    auto common = [&](UmmaParams& q) {
        q.R = R;
        q.Tp = Tp;
        q.ksplit_rows = P.ksplit_rows;
    };
    common(P.conv1);
    P.conv1.Kc = g.Cin;
    P.conv1.cpb = (g.Cin + umma::BK - 1) / umma::BK;
    P.conv1.Nout = g.C;
    P.conv1.bias = b.params + g.off_b1;
    P.conv1.out_hi = b.h1;
    P.conv1.out_lo = b.h1_lo;
    common(P.conv2);
    P.conv2.Kc = g.C;
    P.conv2.cpb = g.C / umma::BK;
    P.conv2.Nout = g.C;
    P.conv2.bias = b.params + g.off_b2;
    P.conv2.out_hi = b.h2;
    P.conv2.out_f32 = 1;
    common(P.dgrad);
    P.dgrad.Kc = g.C;
    P.dgrad.cpb = g.C / umma::BK;
    P.dgrad.Nout = g.C;
    P.dgrad.mask = b.h1;
    P.dgrad.out_hi = b.dA1;
    P.dgrad.out_lo = b.dA1_lo;
    P.dgrad.bsum = nullptr;  // db1 comes from the ones column of the conv1 wgrad GEMM
    const int64_t wmax = (int64_t)g.C * 3 * (g.Cin > g.C ? g.Cin : g.C) + g.C;
    common(P.wgrad2);
    P.wgrad2.Nout = g.C;
    P.wgrad2.Cin_w = g.C;
    P.wgrad2.cpj = (g.C + 63) / 64;
    P.wgrad2.NW = 3 * g.C;
    P.wgrad2.part = b.wpart2;
    P.wgrad2.part_stride = (int64_t)g.C * 3 * g.C + g.C;
    common(P.wgrad1);
    P.wgrad1.Nout = g.C;
    P.wgrad1.Cin_w = g.Cin;
    P.wgrad1.cpj = (g.Cin + 63) / 64;
    P.wgrad1.NW = 3 * g.Cin;
    P.wgrad1.part = b.wpart;
    P.wgrad1.part_stride = (int64_t)g.C * 3 * g.Cin + g.C;
    P.wgrad1.ones_chunk = 1;
    ok &= map2d(&P.wgrad1.ones, b.ones, 128, R, umma::BK);
    (void)wmax;
    return ok;
}

void umma_plan_destroy(UmmaPlan* plan) {
    if (!plan) return;
    if (plan->aux) cudaStreamDestroy(plan->aux);
    if (plan->fork) cudaEventDestroy(plan->fork);
    if (plan->join) cudaEventDestroy(plan->join);
    delete plan;
}

template <int MODE>
static cudaError_t dispatch(const UmmaParams& p, int bn, int npass, dim3 grid, cudaStream_t s) {
    if (npass == 3) {
        if (bn == 64) return launch_one<MODE, 64, 3, 4>(p, grid, s);
        if (bn == 128) return launch_one<MODE, 128, 3, 3>(p, grid, s);
        return launch_one<MODE, 256, 3, 2>(p, grid, s);
    }
    if (bn == 64) return launch_one<MODE, 64, 1, 6>(p, grid, s);
    if (bn == 128) return launch_one<MODE, 128, 1, 6>(p, grid, s);
    return launch_one<MODE, 256, 1, 4>(p, grid, s);
}

cudaError_t umma_compute(const Geom& g, const RankBufs& b, const UmmaPlan& P, const float* labels,
                         const float lam[3], float* loss_out, Status* status, int* nl, const EvRec& rec,
                         cudaStream_t s) {
    const int R = g.R;
    const int mt = (R + umma::BM - 1) / umma::BM;
    int n = 0;
    cudaError_t e;
    rec.begin(SLOT_CONV1);
    e = dispatch<FWD_>(P.conv1, P.bn_fwd, P.npass, dim3(mt, g.C / P.bn_fwd, 1), s);
    rec.end(SLOT_CONV1);
    if (e != cudaSuccess) return e;
    ++n;
    rec.begin(SLOT_CONV2);
    e = dispatch<FWD_>(P.conv2, P.bn_fwd, P.npass, dim3(mt, g.C / P.bn_fwd, 1), s);
    rec.end(SLOT_CONV2);
    if (e != cudaSuccess) return e;
    ++n;
    e = launch_head(g, b, labels, lam, loss_out, status, rec, s, &n);
    if (e != cudaSuccess) return e;
    // Fork: conv2 wgrad (+ its reduction) on the aux stream runs alongside conv2 dgrad ->
    // conv1 wgrad on s; both only read dA2 / h1 / xp (captured as parallel graph branches).
    const int wbn = 256;
    const EvRec rec2{rec.ev, P.aux};
    if (cudaEventRecord(P.fork, s) != cudaSuccess || cudaStreamWaitEvent(P.aux, P.fork, 0) != cudaSuccess)
        return cudaErrorUnknown;
    rec2.begin(SLOT_WGRAD2);
    e = dispatch<WGRAD_>(P.wgrad2, wbn, P.npass, dim3(g.C / umma::BM, (3 * P.wgrad2.cpj + 3) / 4, P.S), P.aux);
    rec2.end(SLOT_WGRAD2);
    if (e != cudaSuccess) return e;
    ++n;
    rec2.begin(SLOT_RED2);
    umma::reduce_wgrad_kernel<<<296, 256, 0, P.aux>>>(b.wpart2, P.wgrad2.part_stride, P.S, (int64_t)g.C * 3 * g.C,
                                                      nullptr, 0, g.C, b.grad + g.off_W2);
    e = cudaGetLastError();
    rec2.end(SLOT_RED2);
    if (e != cudaSuccess) return e;
    ++n;
    if (cudaEventRecord(P.join, P.aux) != cudaSuccess) return cudaErrorUnknown;
    rec.begin(SLOT_DGRAD);
    e = dispatch<DGRAD_>(P.dgrad, P.bn_fwd, P.npass, dim3(mt, g.C / P.bn_fwd, 1), s);
    rec.end(SLOT_DGRAD);
    if (e != cudaSuccess) return e;
    ++n;
    rec.begin(SLOT_WGRAD1);
    e = dispatch<WGRAD_>(P.wgrad1, wbn, P.npass, dim3(g.C / umma::BM, (3 * P.wgrad1.cpj + 3) / 4, P.S), s);
    rec.end(SLOT_WGRAD1);
    if (e != cudaSuccess) return e;
    ++n;
    rec.begin(SLOT_RED1);
    umma::reduce_wgrad_kernel<<<296, 256, 0, s>>>(b.wpart, P.wgrad1.part_stride, P.S,
                                                  (int64_t)g.C * 3 * g.Cin + g.C, nullptr, 0, g.C, b.grad + g.off_W1);
    e = cudaGetLastError();
    rec.end(SLOT_RED1);
    if (e != cudaSuccess) return e;
    ++n;
    if (cudaStreamWaitEvent(s, P.join, 0) != cudaSuccess) return cudaErrorUnknown;  // join
    *nl += n;
    return cudaSuccess;
}

cudaError_t launch_prep_x_split(const Geom& g, const float* x, void* hi, void* lo, cudaStream_t s) {
    umma::prep_x_split_kernel<<<296, 256, 0, s>>>(x, static_cast<__nv_bfloat16*>(hi), static_cast<__nv_bfloat16*>(lo),
                                                 g.B, g.T, g.Cin);
    return cudaGetLastError();
}

cudaError_t launch_fill_ones(void* ones, int64_t rows, cudaStream_t s) {
    if (rows <= 0) return cudaSuccess;
    umma::fill_ones_kernel<<<296, 256, 0, s>>>(static_cast<__nv_bfloat16*>(ones), rows);
    return cudaGetLastError();
}

cudaError_t launch_cast_shadow_split(const float* params, __nv_bfloat16* hi, __nv_bfloat16* lo, int64_t n,
                                     cudaStream_t s) {
    umma::cast_shadow_split_kernel<<<296, 256, 0, s>>>(params, hi, lo, n);
    return cudaGetLastError();
}

}  // namespace tem
