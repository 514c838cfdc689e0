// kernels.h -- internal launcher declarations of libtem (host side).
#pragma once
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <cuda.h>
#include <stdlib.h>

#include "common.cuh"

namespace tem {

// Kernel launch with programmatic dependent launch allowed (unless TEM_NO_PDL is set): the
// kernel's prologue overlaps the tail of its stream predecessor (see pdl_wait/pdl_trigger).
bool pdl_enabled();
// Launch priority of the step's graph branches: the critical path (prep -> convs -> head ->
// dgrad -> conv1 wgrad -> exchange) high, the side branches (head reduction, conv2 wgrad, PEM)
// low, so the block scheduler hands them the SMs the critical path leaves idle.
// Returns the number of attributes written (0, or 1 where the device has priorities).
int launch_priority_attr(cudaLaunchAttribute* a, bool side_branch);
template <typename... KArgs, typename... Args>
cudaError_t launch_pdl(void (*k)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s, bool side,
                       Args... args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute a[2];
    int na = 0;
    // side-branch kernels follow a cross-stream event: no early launch (their CTAs would sit on
    // SMs the critical path needs)
    if (pdl_enabled() && !side) {
        a[na].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        a[na++].val.programmaticStreamSerializationAllowed = 1;
    }
    na += launch_priority_attr(&a[na], side);
    cfg.attrs = a;
    cfg.numAttrs = na;
    return cudaLaunchKernelEx(&cfg, k, static_cast<KArgs>(args)...);
}

// Geometry of one rank's TEM step.  Activations use the halo-padded row layout
// [B][T+2][C]: row p = v*(T+2) + t + 1 holds snippet t of video v; rows v*(T+2)
// and v*(T+2)+T+1 are zero, so every k=3 tap is a plain row shift (reading R1's
// zero "same" padding) and tiles may span video boundaries.
struct Geom {
    int B, T, Cin, C, Co;
    int R;          // B*(T+2) padded rows
    int prec;       // TEM_FP32 / TEM_BF16
    int split;      // hi/lo residual planes present (TEM_FP32: the 3-pass bf16 split, R16)
    int64_t K, Kpad;
    int64_t off_W1, off_b1, off_W2, off_b2, off_W3, off_b3;
    // PEM (joint TEM + PEM step, BASELINE configs[4]): pem_P proposals per video, 0 = off;
    // its parameters follow TEM's in the flat vector at off_pem (reading R21)
    int pem_P, pem_F, pem_H;
    int pgm_G;  // > 0: PEM's inputs come from PGM on this step's TEM output (reading R24)
    int64_t off_pem;
};
inline int64_t pem_num_params_of(const Geom& g) {
    return g.pem_P > 0 ? (int64_t)g.pem_H * g.pem_F + 2 * (int64_t)g.pem_H + 1 : 0;
}

// Owner update (tem_step exchanges): SGD, or Adam with per-rank moments (reading R22).
struct OptCfg {
    int kind;  // TEM_OPT_SGD / TEM_OPT_ADAM
    float lr, beta1, beta2, c1, c2, eps;  // c1 = fl(1 - beta1), c2 = fl(1 - beta2)
    float mu;                             // momentum (TEM_OPT_MOMENTUM)
};
struct OptState {
    float* m;           // [K_pad] first moments / momentum buffer (each rank touches only the blocks it owns)
    float* v;           // [K_pad] second moments
    const float* scal;  // [beta1^t, beta2^t] of this step (opt_scalars_kernel, before the exchange)
};

// One kernel path: tcgen05/TMA bf16 tensor-core GEMMs, one plane of bf16 operands (TEM_BF16)
// or hi/lo planes (TEM_FP32, 3-pass split).  (The round-1 CUDA-core path was removed: no
// multi-backend dispatch in the product library.)

// The fp32 backward as ONE persistent launch (tem_umma.cu, bwd_kernel): conv2 DGRAD, conv2
// WGRAD and conv1 WGRAD tiles on a static per-CTA task list, one CTA per SM (cooperative
// launch: all co-resident), conv1 WGRAD tiles waiting on the DGRAD tiles they read through
// per-tile flags.  Device state in the workspace (RankBufs::bwd).
struct BwdState {
    int* tasks;          // [grid][max_tasks] task words (type << 24 | m << 16 | n << 8 | split), -1 ends a list
    unsigned* flags;     // [dgrad m-tiles x n-tiles] epoch at which each DGRAD tile was stored
    unsigned* epoch;     // [0] epoch of the last completed launch, [1] exit ticket (self-resetting)
};
constexpr int BWD_MAX_TASKS = 8;
constexpr int BWD_MAX_DG_TILES = 1024;

// Per-rank device buffers (all inside the caller's workspace except params).
// Operand tensors are bf16 ("hi"; "_lo" = residual plane x - bf16(x), present only on the
// fp32 path).
struct RankBufs {
    float* pempart;       // PEM per-CTA partial rows [pem_ctas][K_pem + 1]
    uint8_t* pemdec;      // PEM ReLU decisions [B*P][H] of the last step (recorded on request)
    const float* params;  // fp32 master weights [Kpad] (symmetric heap)
    void* xp;             // [R][Cin] operand type
    void* h1;             // [R][C]   operand type
    float* h2;            // [R][C]
    void* dA2;            // [R][C]   operand type
    void* dA1;            // [R][C]   operand type
    void* xp_lo;
    void* h1_lo;
    void* dA2_lo;
    void* dA1_lo;
    float* z;             // [B][T][3]
    float* grad;          // [Kpad] local gradient (flat order W1 b1 W2 b2 W3 b3 pad)
    float* headpart;      // [ctas][4C + 8] head partials (dW3, db3, L, db2; 2 pad)
    float* headlvl1;      // [32][4C + 6] first-level sums
    unsigned* counter;    // last-CTA ticket of the head reduction (self-resetting)
    float* bpart;         // [m-tiles][C] conv1 bias-gradient partials (tcgen05 DGRAD epilogue)
    void* ones;           // [R][128] bf16 ones/zeros operand for the bias-gradient column
    float* zpart;         // [C/BN][R][3] partial logits from the conv2 epilogue (tcgen05), or nullptr
    int nzpart;           // number of partial-logit planes (C / conv2 tile width); 0 = head computes z
    float* wpart;         // [S][C*3*Cin + C] split-K partials of conv1 wgrad (and its bias column)
    float* wpart2;        // [S][C*3*C + C] split-K partials of the tcgen05 conv2 wgrad
    int64_t* stepctr;     // step counter for NONFINITE reporting
    uint64_t* dec2;       // [R][C / 64] conv2 ReLU decision masks (fused head: h2 is not stored)
    int dec2_valid;       // 1 when the plan fuses the head (dec2 holds the decisions, not h2)
    BwdState bwd;         // persistent-backward task lists / flags (workspace)
    // bf16 operand copies of the weights, TWO sets [2][Kpad] (ping-pong): a step's GEMMs read
    // set `wset` while its updates write set 1 - wset, so an update may run while a GEMM of
    // the same step still reads the old weights
    __nv_bfloat16* shadow;     // hi plane, set 0 (set 1 at + shadow_set)
    __nv_bfloat16* shadow_lo;  // residual plane (fp32 path) or nullptr
    int64_t shadow_set;        // elements between the sets (K_pad)
};
inline __nv_bfloat16* shadow_hi(const RankBufs& b, int set) { return b.shadow + set * b.shadow_set; }
inline __nv_bfloat16* shadow_lo(const RankBufs& b, int set) {
    return b.shadow_lo ? b.shadow_lo + set * b.shadow_set : nullptr;
}

// --- tcgen05 path (tem_umma.cu) ---------------------------------------------------------
enum UmmaMode { FWD_ = 0, DGRAD_ = 1, WGRAD_ = 2 };
struct UmmaParams {
    CUtensorMap a[2];  // A operand, hi / lo planes
    CUtensorMap b[2];  // B operand, hi / lo planes
    CUtensorMap out[2];  // epilogue TMA-store maps (output hi / lo plane, fp32 output, or split-K partials)
    int R, Tp;         // padded rows, T + 2
    int Kc, cpb;       // FWD/DGRAD: channels per tap along K, k-blocks per tap
    int Nout;          // output columns (row stride of outputs / mask)
    const float* bias; // FWD
    const void* mask;  // DGRAD: h1 (bf16 hi plane)
    void* out_hi;      // FWD/DGRAD output plane (bf16) or fp32 (out_f32)
    void* out_lo;      // residual plane or nullptr
    int out_f32;
    float* bsum;       // DGRAD: per-m-tile column sums of the stored dA1 [m-tiles][Nout] or nullptr
    const float* w3;   // FWD conv2: W3 [3][Nout] (fp32) for the fused partial logits
    float* zpart;      // FWD conv2: [Nout/BN][R][3] partial logits, or nullptr
    float* part;       // WGRAD split partials
    int64_t part_stride;
    int NW, Cin_w, cpj;  // WGRAD: 3*Cin, Cin, 64-wide chunks per tap
    int ksplit_rows;
    int mtiles, ntiles, nsplit;  // tile grid (persistent kernels walk it cluster tile by cluster tile)
    int ones_chunk;      // WGRAD: chunk slot 3*cpj reads the all-ones map (bias gradient column)
    int slot;            // trace / timing slot (Slot)
    int side;            // 1: launched on the side branch (low priority)
    int no_pdl;          // 1: launched without programmatic dependent launch (its CTAs would sit
                         // on SMs the concurrent side branch could use while waiting)
    // conv2 FWD with the fused head (fp32 single-wave path, clusters of ntiles CTAs):
    int fused_head;
    uint64_t* dec2;        // [R][Nout / 64] conv2 ReLU decisions (bit i: column 64 k + i), fused head
    CUtensorMap out2[2];   // dA2 hi / lo store maps
    const float* labels;   // [B][3][T] (per call)
    float lam[3];          // per call
    const float* b3;
    float* z_out;          // [B][T][3]
    float* headpart;       // [mtiles][4C + 8] partial rows (head_reduce input)
    int Bv, Tn;
    CUtensorMap ones;    // [R][128] bf16: columns 0..63 = 1, 64..127 = 0
};
struct UmmaPlan {
    UmmaParams conv1, conv2, dgrad, wgrad1, wgrad2;
    int bwd_grid;               // > 0: the backward runs as bwd_kernel on this many CTAs
    BwdState bwd;
    CUtensorMap wmap[3][2][2];  // B maps of conv1 (W1), conv2 (W2), dgrad (W2) [set][plane]
    int npass, bn_fwd, S, ksplit_rows;
    int S1, S2;  // split-K factors of conv1 / conv2 wgrad (<= S, the workspace's)
    cudaStream_t aux;         // second stream: conv2 wgrad runs beside conv2 dgrad / conv1 wgrad
    cudaEvent_t fork, join;
    cudaStream_t pem;         // third stream: the PEM (configs[4]) beside the whole TEM step
    cudaEvent_t pem_fork, pem_join;
    bool pem_pending;         // a PEM launch on `pem` awaits its join before the exchange
};
void umma_plan_destroy(UmmaPlan* plan);
bool umma_bwd_active(const UmmaPlan& P);  // the backward runs as one persistent launch
void* umma_tstamp_buffer(int64_t* nbytes, int on);  // split-K phase timestamps (diagnostics)
void* umma_tclk_buffer(int64_t* nbytes);            // SM clock stamps (diagnostics)
void umma_set_probe_skip(int bits);                  // operand-skip probe (diagnostics build only)
int umma_wgrad_splits(const Geom& g);
bool umma_plan(const Geom& g, const RankBufs& b, UmmaPlan* plan);
cudaError_t launch_fill_ones(void* ones, int64_t rows, cudaStream_t s);
cudaError_t launch_prep_x_split(const Geom& g, const float* x, void* hi, void* lo, cudaStream_t s);
cudaError_t launch_cast_shadow_split(const float* params, __nv_bfloat16* hi, __nv_bfloat16* lo, int64_t n,
                                     cudaStream_t s);

// --- input preparation and helpers (prep.cu) -------------------------------------------
int head_ctas(const Geom& g);
cudaError_t launch_prep_x(const Geom& g, const void* x, void* xp, cudaStream_t s);
cudaError_t launch_cast_shadow(const float* params, __nv_bfloat16* shadow, int64_t n, cudaStream_t s);
cudaError_t launch_relu_decisions(const Geom& g, const RankBufs& b, uint8_t* out, cudaStream_t s);
// Enqueue the whole forward + loss + backward; returns number of kernels launched via *nlaunch.
// Kernel slots of one step (for tem_timing_*): every launch is bracketed by
// ev[2*slot] / ev[2*slot+1] when ev != nullptr.
enum Slot { SLOT_PREP = 0, SLOT_CONV1, SLOT_CONV2, SLOT_HEAD, SLOT_HEADFIN, SLOT_DGRAD, SLOT_WGRAD2,
            SLOT_RED2, SLOT_WGRAD1, SLOT_RED1, SLOT_EXCHANGE, SLOT_PEM, SLOT_PEMRED, SLOT_EXCH2, SLOT_PGM,
            SLOT_BWD, NUM_SLOTS };
const char* slot_name(int slot);
// kernel-span trace buffers (diagnostics): one setter per translation unit with traced kernels
void trace_set_umma(unsigned long long* p);
void trace_set_head(unsigned long long* p);
void trace_set_ring(unsigned long long* p);
void trace_set_pem(unsigned long long* p);
struct EvRec {
    cudaEvent_t* ev;  // [NUM_SLOTS*2] or nullptr
    cudaStream_t s;
    void begin(int slot) const { if (ev) cudaEventRecord(ev[2 * slot], s); }
    void end(int slot) const { if (ev) cudaEventRecord(ev[2 * slot + 1], s); }
};
// Empty shard (B = 0): zero gradient and zero loss, so the exchange still runs.
cudaError_t empty_shard_compute(const Geom& g, const RankBufs& b, const float* labels, const float lam[3],
                                float* loss_out, Status* status, int* nlaunch, const EvRec& rec, cudaStream_t s);
// defer_reduce: skip the two split-K reductions; the N = 1 exchange sums the partials itself
// (launch_sgd_fused) -- used by tem_step only, so tem_compute still leaves the full gradient.
// split: (bucketed exchange, N > 1) the [bnd, K_pad) bucket's exchange is launched on the side
// branch once conv2 dgrad is done, beside conv1 wgrad (reading R25).
struct SplitUpdate;
// wset: the operand set (RankBufs::shadow) of the weights this step reads.  defer_reduce (N = 1
// tem_step): the split-K partials are left for the update kernel, which sums them itself.
cudaError_t umma_compute(const Geom& g, const RankBufs& b, const UmmaPlan& P, const float* labels,
                         const float lam[3], float* loss_out, Status* status, int* nlaunch,
                         const EvRec& rec, cudaStream_t s, int wset, bool defer_reduce = false,
                         float* loss_host = nullptr, const SplitUpdate* split = nullptr);
// head (conv3 + sigmoid + loss + dz + dA2) and its deterministic finalisation (rows a3-a5);
// writes dA2 as b.dA2 (+ b.dA2_lo when present) in the operand type of the path.
cudaError_t launch_head(const Geom& g, const RankBufs& b, const float* labels, const float lam[3],
                        float* loss_out, Status* status, const EvRec& rec, cudaStream_t s, int* n);
cudaError_t launch_head_rows(const Geom& g, const RankBufs& b, const float* labels, const float lam[3],
                             const EvRec& rec, cudaStream_t s, int* n);
// PEM forward + loss + backward (pem.cu): the gradient at grad (K_pem floats, the PEM block of
// the flat gradient) and the loss at *loss_out; dec_out (nullable): ReLU decisions [M][H].
int pem_ctas(const Geom& g);
// pem_kernel runs on `s`; pem_reduce on `s_red` (forked from `s` through `fork` when they differ).
cudaError_t launch_pem(const Geom& g, const float* f, const float* iou, const float* params, float* part,
                       float* grad, float* loss_out, Status* status, const int64_t* stepctr, uint8_t* dec_out,
                       cudaStream_t s, cudaStream_t s_red, cudaEvent_t fork, int* n, const EvRec& rec);
cudaError_t launch_head_reduce_rows(const Geom& g, const RankBufs& b, int nrows, const float lam[3],
                                   float* loss_out, Status* status, const EvRec& rec, cudaStream_t s, int* n);
cudaError_t launch_head_reduce(const Geom& g, const RankBufs& b, const float lam[3], float* loss_out,
                               Status* status, const EvRec& rec, cudaStream_t s, int* n);
cudaError_t launch_reduce_splits(const float* part, float* dst, int64_t n, int S, cudaStream_t s);

// --- ring / exchange (ring.cu) --------------------------------------------------------
struct RingParams;
struct SplitUpdate {
    OptCfg oc;
    OptState os;
    const RingParams* early = nullptr;  // N > 1 bucketed exchange: the [bnd, K_pad) bucket's
    int early_kind = 0;                 // ring (TEM_EXCHANGE_RING) / two-shot, launched after dgrad
    int n1_w2 = 0;  // N = 1 tem_step: update [off_W2, K_pad) on the side branch after conv2 wgrad
};
struct RingLocal {
    OptState opt;
    const float* src;       // contribution of this rank (local grads, or the user buffer)
    float* dst_self;        // result on this rank (params, or the user buffer)
    __nv_bfloat16* shadow;  // bf16 copy of dst to refresh (operand weights) or nullptr
    __nv_bfloat16* shadow_lo;  // residual plane dst - bf16(dst) or nullptr
    uint32_t* epochs;       // [kMaxChannels] per-channel collective counters (workspace)
    char* heaps[TEM_MAX_RANKS];  // every rank's heap base as mapped in this process
};
// PGM (pgm.cu, reading R24): proposals, BSP features, IoU targets of B videos (T <= 128)
cudaError_t launch_pgm(int B, int T, int G, int P, const float* prob, const float* gt, const int32_t* n_gt,
                       float* feat, float* iou, int32_t* ts, int32_t* te, int32_t* count, cudaStream_t s,
                       const float* z = nullptr, float* prob_out = nullptr);
constexpr int kMaxChannels = 128;
struct RingParams {
    RingLocal loc[TEM_MAX_RANKS];
    int N, rank_base, nlocal, G, op, mode;  // mode 0 = allreduce, 1 = optimizer step
    int64_t K, Kpad;
    OptCfg oc;
    int64_t off_dst, off_stage, off_flags;
    int64_t off_hdr;    // handshake headers [TEM_MAX_RANKS][kMaxChannels] x 16 B (every kernel)
    int64_t off_ll;     // ring: LL slots [2 phases][N-1 rounds][ll_stride lines] x 16 B
    int64_t ll_stride;  // lines per LL slot (2 per float4 of the largest block)
    int64_t off_src;  // two-shot: heap offset of the source when it already lives in the heap
                      // (off_stage < 0), i.e. ring_allreduce's user region
    Status* status;
    uint64_t spin_ns;
};
cudaError_t launch_ring(const RingParams& p, cudaStream_t s);
cudaError_t launch_twoshot(const RingParams& p, cudaStream_t s);  // NVSwitch two-shot (NEXT #3(i))
// Owner update of elements [e0, e1) at N = 1 (e0, e1 multiples of 4): the gradient is
// sum_s part1[s][e] on [0, n1), sum_s part2[s][e - off2] on [off2, off2 + n2) (split-K partials in
// ascending s, the order of the fused WGRAD reduction), else grad[e].  mode 1: update (and store
// the summed partials into grad), 2: update only, 0: only sum the partials into grad
// (tem_local_grad after an N = 1 tem_step, whose W1 / W2 gradient exists only as partials).
cudaError_t launch_sgd_fused(float* g, float* w, __nv_bfloat16* shadow, __nv_bfloat16* shadow_lo, int64_t e0,
                             int64_t e1, const OptCfg& oc, const OptState& os, const float* p1, int64_t stride1, int64_t n1,
                             int S1, const float* p2, int64_t stride2, int64_t off2, int64_t n2, int S2,
                             cudaStream_t s, bool side = false, int ctas = 0, int mode = 1);
cudaError_t launch_sgd_single(const float* g, float* w, __nv_bfloat16* shadow, __nv_bfloat16* shadow_lo,
                              int64_t n, int op, const OptCfg& oc, const OptState& os, cudaStream_t s);
// Adam: scal[0] *= beta1, scal[1] *= beta2 (fp32, once per step, before the exchange kernel).
cudaError_t launch_opt_scalars(float* scal, float beta1, float beta2, cudaStream_t s);
struct PsParams {
    RingLocal loc[TEM_MAX_RANKS];
    int N, rank_base, nlocal, G, op, mode;  // mode 0 = allreduce, 1 = optimizer step (server)
    OptCfg oc;
    int64_t K;
    int64_t off_dst, off_slots, off_flags, off_hdr;
    Status* status;
    uint64_t spin_ns;
};
cudaError_t launch_ps(const PsParams& p, cudaStream_t s);

}  // namespace tem
