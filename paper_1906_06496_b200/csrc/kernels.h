// kernels.h -- internal launcher declarations of libtem (host side).
#pragma once
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "common.cuh"

namespace tem {

// Geometry of one rank's TEM step.  Activations use the halo-padded row layout
// [B][T+2][C]: row p = v*(T+2) + t + 1 holds snippet t of video v; rows v*(T+2)
// and v*(T+2)+T+1 are zero, so every k=3 tap is a plain row shift (reading R1's
// zero "same" padding) and tiles may span video boundaries.
struct Geom {
    int B, T, Cin, C, Co;
    int R;          // B*(T+2) padded rows
    int prec;       // TEM_FP32 / TEM_BF16
    int64_t K, Kpad;
    int64_t off_W1, off_b1, off_W2, off_b2, off_W3, off_b3;
};

// Per-rank device buffers (all inside the caller's workspace except params).
struct RankBufs {
    const float* params;  // fp32 master weights [Kpad] (symmetric heap)
    const void* wop;      // operand copy of the weights: params (fp32) or bf16 shadow
    void* xp;             // [R][Cin] operand type
    void* h1;             // [R][C]   operand type
    float* h2;            // [R][C]
    void* dA2;            // [R][C]   operand type
    void* dA1;            // [R][C]   operand type
    float* z;             // [B][T][3]
    float* grad;          // [Kpad] local gradient (flat order W1 b1 W2 b2 W3 b3 pad)
    float* headpart;      // [B][3C + 6]
    float* wpart;         // [S][max(C*3*Cin + C, C*3*C + C)]
    int64_t* stepctr;     // step counter for NONFINITE reporting
    __nv_bfloat16* shadow;  // [Kpad] bf16 weights (TEM_BF16) or nullptr
};

// --- SIMT path (tem_simt.cu) ---------------------------------------------------------
int simt_wgrad_splits(const Geom& g);
cudaError_t launch_prep_x(const Geom& g, const void* x, void* xp, cudaStream_t s);
cudaError_t launch_cast_shadow(const float* params, __nv_bfloat16* shadow, int64_t n, cudaStream_t s);
cudaError_t launch_relu_decisions(const Geom& g, const RankBufs& b, uint8_t* out, cudaStream_t s);
// Enqueue the whole forward + loss + backward; returns number of kernels launched via *nlaunch.
// Kernel slots of one step (for tem_timing_*): every launch is bracketed by
// ev[2*slot] / ev[2*slot+1] when ev != nullptr.
enum Slot { SLOT_PREP = 0, SLOT_CONV1, SLOT_CONV2, SLOT_HEAD, SLOT_HEADFIN, SLOT_DGRAD, SLOT_WGRAD2,
            SLOT_RED2, SLOT_WGRAD1, SLOT_RED1, SLOT_EXCHANGE, NUM_SLOTS };
const char* slot_name(int slot);
struct EvRec {
    cudaEvent_t* ev;  // [NUM_SLOTS*2] or nullptr
    cudaStream_t s;
    void begin(int slot) const { if (ev) cudaEventRecord(ev[2 * slot], s); }
    void end(int slot) const { if (ev) cudaEventRecord(ev[2 * slot + 1], s); }
};
cudaError_t simt_compute(const Geom& g, const RankBufs& b, const float* labels,
                         const float lam[3], float* loss_out, Status* status, int* nlaunch,
                         const EvRec& rec, cudaStream_t s);

// --- ring / exchange (ring.cu) --------------------------------------------------------
struct RingLocal {
    const float* src;       // contribution of this rank (local grads, or the user buffer)
    float* dst_self;        // result on this rank (params, or the user buffer)
    __nv_bfloat16* shadow;  // bf16 copy of dst to refresh (TEM_BF16 weights) or nullptr
    uint32_t* epochs;       // [kMaxChannels] per-channel collective counters (workspace)
    char* heaps[TEM_MAX_RANKS];  // every rank's heap base as mapped in this process
};
constexpr int kMaxChannels = 128;
constexpr int kMaxChunks = 16;
struct RingParams {
    RingLocal loc[TEM_MAX_RANKS];
    int N, rank_base, nlocal, G, C, op, mode;  // mode 0 = allreduce, 1 = SGD
    int64_t K, Kpad;
    float lr;
    int64_t off_dst, off_stage, off_flags;
    Status* status;
    uint64_t spin_ns;
};
cudaError_t launch_ring(const RingParams& p, cudaStream_t s);
cudaError_t launch_sgd_single(const float* g, float* w, __nv_bfloat16* shadow, int64_t n,
                              int op, float lr, cudaStream_t s);
struct PsParams {
    RingLocal loc[TEM_MAX_RANKS];
    int N, rank_base, nlocal, G, op;
    int64_t K;
    int64_t off_dst, off_slots, off_flags;
    Status* status;
    uint64_t spin_ns;
};
cudaError_t launch_ps(const PsParams& p, cudaStream_t s);

}  // namespace tem
