/* ============================================================================
 * tem.h -- C ABI of libtem.so: the data-parallel BSN-TEM training step of
 * arXiv 1906.06496 with its ring allreduce, for NVIDIA B200 (sm_100a).
 *
 * Citations: "P:n" = PAPER.md line n; "S:n" = SPEC.md line n; "SURVEY 8(x)" =
 * the hot-path scope table in SURVEY.md section 8.  Readings R1..R16 of the
 * paper are listed in DESIGN.md section 3.
 *
 * Plain C: every pointer is a raw host or device address, every size a plain
 * integer.  `stream` arguments are a cudaStream_t passed as void* (NULL = the
 * legacy default stream).  No torch type appears here.
 *
 * Ownership.  The CALLER owns all device memory: parameters, the symmetric
 * heap of every rank, the workspace, inputs and outputs.  The library borrows
 * these pointers for the lifetime of the context and allocates no device
 * memory itself; it heap-allocates only its opaque host-side context (and a
 * 64-byte pinned, device-mapped status word through which kernels latch
 * errors).
 *
 * Asynchrony and errors.  Calls enqueue work on `stream` and return after
 * enqueue.  Host-detectable errors return immediately (INVALID_ARG, CUDA,
 * STATE).  Errors detected on the device (PROTOCOL, TRANSPORT, NONFINITE) are
 * latched in the context and returned by the NEXT call on that context (or by
 * tem_shutdown / tem_sync); after such an error the contents of params / buf
 * are unspecified.  No function throws, aborts or exits.
 *
 * Collective semantics.  With world_size N > 1 every rank calls
 * tem_step / tem_exchange / ring_allreduce in the same order with equal
 * arguments; calls on one context are not reentrant.
 * ==========================================================================*/
#ifndef TEM_H_
#define TEM_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
    TEM_OK = 0,
    TEM_ERR_INVALID_ARG = 1, /* bad dims, N <= 0, pointer outside the symmetric heap   */
    TEM_ERR_PROTOCOL = 2,    /* ranks disagree on the collective (K, kind, op): every
                                rank reads all N ranks' headers before any data moves, so all
                                ranks latch it and none writes a result                      */
    TEM_ERR_TRANSPORT = 3,   /* a peer header / message did not arrive within spin_timeout_ms
                                                                                      */
    TEM_ERR_CUDA = 4,        /* a CUDA launch / API call failed                               */
    TEM_ERR_NONFINITE = 5,   /* non-finite loss; tem_sync reports the step index      */
    TEM_ERR_STATE = 6        /* call on a shut-down or NULL context                           */
} tem_status;

typedef enum { TEM_SUM = 0, TEM_MEAN = 1 } tem_reduce_op;
typedef enum { TEM_FP32 = 0, TEM_BF16 = 1 } tem_precision;    /* BASELINE configs[1]/[2]   */

#define TEM_MAX_RANKS 8

typedef struct tem_ctx tem_ctx; /* opaque, owned by the library */

typedef struct {
    /* --- cluster (SPEC WorkerId / ClusterConfig; "N is the number of GPU") */
    int32_t rank;        /* this process's first rank, 0 <= rank < world_size               */
    int32_t world_size;  /* N, 1 <= N <= TEM_MAX_RANKS                                       */
    int32_t device;      /* CUDA device ordinal                                              */
    int32_t local_ranks; /* ranks driven by this process on `device`: 1 in production (one
                            process per GPU); == world_size for the single-device emulation
                            used by the tests, where the N ranks run as CTA groups of one
                            cooperative launch over same-device "peer" heaps               */
    /* --- model ("temporal network with 3 convolution layers"; shapes BASELINE.json)  */
    int32_t batch_per_rank; /* B >= 0 videos per rank per step (P:113 data parallelism)     */
    int32_t seq_len;        /* T >= 1 snippets per video (100 in the paper's setup)          */
    int32_t c_in;           /* 400 two-stream feature dims; multiple of 16           */
    int32_t c_hidden;       /* 512; multiple of 128, at most 512                             */
    int32_t c_out;          /* 3: actionness, start, end (reading R4); must be 3             */
    int32_t precision;      /* tem_precision: TEM_FP32 (fp32 operands, fp32 accumulate) or
                               TEM_BF16 (bf16 operands, fp32 accumulate; reading R8)          */
    float lr;               /* SGD step size >= 0 (S:272 vs S:278 resolved: 0 allowed)       */
    float loss_weight[3];   /* lambda_action, lambda_start, lambda_end (reading R6)          */
    /* --- symmetric memory (one heap per rank, all mapped in this process)                  */
    void* const* peer_bufs; /* [world_size] base of each rank's heap as mapped here (for
                               local_ranks == world_size all are on `device`)                 */
    size_t sym_bytes;       /* capacity of each heap, >= tem_sym_bytes(cfg)                   */
    int64_t max_allreduce_elems; /* largest K ring_allreduce will be called with (sizes the
                                    staging area); 0 -> the TEM gradient size               */
    /* --- workspace                                                                         */
    void* workspace;        /* device, 256-byte aligned, >= tem_workspace_bytes(cfg)          */
    size_t workspace_bytes;
    /* --- collective tuning (0 = automatic)                                                 */
    int32_t ring_channels;  /* G: CTAs per rank of every collective kernel (default 16; the
                               emulation caps it at SMs / local_ranks); equal on every rank  */
    int32_t spin_timeout_ms; /* bound on any wait for a peer (0 -> 20000 ms); past it the
                               collective latches TEM_ERR_TRANSPORT                           */
    /* --- gradient exchange of tem_step / tem_exchange                                      */
    int32_t exchange;       /* TEM_EXCHANGE_RING (the paper's ring; default) or
                               TEM_EXCHANGE_PS (the parameter-server comparator, P:115-124:
                               ranks push gradients to rank 0, which sums them in ascending
                               rank order, applies mean + SGD to its weights and pushes w'
                               back to every rank) or TEM_EXCHANGE_TWOSHOT (NVSwitch two-shot,
                               SURVEY 8(f) NEXT #3(i): each block's owner reads the block from
                               every rank and sums in the ring's chain order -- bit-identical
                               to the ring -- then writes w' into every rank: 2 phases instead
                               of 2(N-1) rounds)                                              */
    /* --- PEM: joint TEM + PEM training (BASELINE configs[4]).  BSN's
     *     proposal evaluation module: per proposal a BSP feature f (F) -> ReLU(W1 f + b1) (H)
     *     -> sigmoid(w2 . h + b2), MSE to the proposal's IoU (readings R19-R20).  Its
     *     F*H + 2H + 1 parameters follow TEM's in the flat vector (R21), so tem_num_params
     *     grows by 17,409 and one exchange carries both gradients.                           */
    int32_t pem_proposals;  /* P proposals per video per step; 0 = TEM only                  */
    int32_t pem_features;   /* F: 32 (required when pem_proposals > 0)                       */
    int32_t pem_hidden;     /* H: 512 (required when pem_proposals > 0)                      */
    /* --- optimizer of the owner update                                */
    int32_t optimizer;      /* TEM_OPT_SGD (default: w = fma(-lr, gbar, w), R12) or TEM_OPT_ADAM
                               (reading R22: m, v sharded by block ownership -- the owner of a
                               block keeps its moments; bias correction by running fp32 products
                               beta^t; every op single-rounded, so replicas stay bitwise equal
                               and the result equals the oracle's orc_ring_adam_f32)            */
    float beta1, beta2, eps; /* Adam: 0 <= beta < 1, eps > 0 (ignored otherwise)               */
    float momentum;         /* TEM_OPT_MOMENTUM (reading R23): heavy ball u = fma(mu, u, gbar),
                               w = fma(-lr, u, w); 0 <= mu < 1; u sharded by block ownership
                               like Adam's moments                                            */
    int32_t exchange_buckets; /* 0 or 1: one exchange over the whole gradient (the paper's ring);
                               2 (ring / two-shot, world_size > 1, reading
                               R25): two buckets [0, bnd) and [bnd, K_pad), bnd = roundup(off_W2,
                               4N), each exchanged with R9's partition of its own length; with one
                               rank per process the [bnd, K_pad) bucket (W2 .. b3, PEM) starts
                               as soon as conv2 dgrad is done, beside conv1 wgrad              */
    int32_t pgm_gt_max;     /* > 0 (requires pem_proposals > 0, seq_len <= 128): PGM-fed PEM --
                               tem_step_pgm runs PGM (tem_pgm) on this step's TEM probabilities
                               sigmoid(z) and trains PEM on its BSP features and IoU targets
                               against the caller's ground truth (<= pgm_gt_max instances per
                               video); 0: PEM inputs from the caller (tem_step_pem)           */
} tem_config;

enum { TEM_EXCHANGE_RING = 0, TEM_EXCHANGE_PS = 1, TEM_EXCHANGE_TWOSHOT = 2 };
enum { TEM_OPT_SGD = 0, TEM_OPT_ADAM = 1, TEM_OPT_MOMENTUM = 2 };

/* --- sizes -----------------------------------------------------------------------------
 * K      = c_hidden*3*c_in + c_hidden + c_hidden*3*c_hidden + c_hidden + 3*c_hidden + 3
 *          (flat order [W1, b1, W2, b2, W3, b3]; W1 [c_hidden][3][c_in],
 *          W2 [c_hidden][3][c_hidden], W3 [3][c_hidden]; reading R3)
 * K_pad  = roundup(K, 4*world_size)  (N equal 16-byte aligned blocks)
 * Return 0 on invalid cfg. */
int64_t tem_num_params(const tem_config* cfg);
int64_t tem_kpad(const tem_config* cfg, int64_t K);
size_t tem_workspace_bytes(const tem_config* cfg);
/* Per-rank symmetric heap layout (offsets are identical on every rank):
 *   [0, 4*K_pad)                 params (fp32 master weights)
 *   [off_user, off_user + 4*max) user region for ring_allreduce buffers
 *   then library-private areas: two-shot staging, PS slots, the handshake headers, the
 *   two-shot / PS phase flags and the ring's LL slots.
 * The caller zero-fills the whole heap once before tem_init on every rank.
 *
 * Wire protocol between ranks (what one rank stores into a peer's heap):
 *   handshake  before any data moves, channel g of rank s stores the 16-byte header
 *              {K mod 2^32, epoch, (K >> 32) | kind << 8 | op << 16 | mode << 24, epoch}
 *              (kind 0 ring, 1 two-shot, 2 PS; mode 1 = tem_step exchange) into header slot
 *              (epoch & 1, s, g) of every rank, and every rank compares all N headers of channel g:
 *              any difference -> PROTOCOL on every rank, nothing written.
 *   ring       LL lines of 16 bytes {d0, epoch, d1, epoch} (each 8-byte half written
 *              atomically): float4 position v of a block message travels as lines 2v, 2v+1
 *              of slot (epoch & 1, phase, round) -- scatter phase 0 rounds 0..N-2, gather
 *              phase 1 rounds 0..N-2; slot stride tem_ll_slot_lines(cfg) lines -- in the
 *              receiver's LL area at tem_sym_ll_offset(cfg).  Header slot [s][g] lies at
 *              tem_sym_hdr_offset(cfg) + 16 * (((epoch & 1) * 8 + s) * 128 + g).  `epoch`
 *              counts the collectives of the context from 1, identical on every rank. */
size_t tem_sym_hdr_offset(const tem_config* cfg);
size_t tem_sym_ll_offset(const tem_config* cfg);
int64_t tem_ll_slot_lines(const tem_config* cfg);
size_t tem_sym_bytes(const tem_config* cfg);
size_t tem_sym_user_offset(const tem_config* cfg);

/* --- lifecycle ---------------------------------------------------------------------------
 * tem_init: validates cfg, lays out workspace and heap, and binds `params`, which must be
 * the first 4*K_pad bytes of this rank's heap (peer_bufs[rank]) and hold the initial
 * weights, bitwise identical on every rank ("all of GPUs have the same CNN model").
 * For local_ranks > 1, params of rank r are peer_bufs[r]; `params` must equal
 * peer_bufs[rank].  Returns INVALID_ARG / CUDA; *out = NULL on failure. */
tem_status tem_init(const tem_config* cfg, float* params, tem_ctx** out);

/* tem_step = tem_compute + tem_exchange: one synchronous data-parallel SGD step.
 *   x       device, [local_ranks][B][T][c_in], fp32 (TEM_FP32) or bf16 bits (TEM_BF16),
 *           row-major channels-last; rank r's shard of the global batch.
 *   labels  device, [local_ranks][B][3][T] fp32 in [0,1] (channel 0 action, 1 start, 2 end).
 *   loss_out device, [local_ranks][4] fp32: total, action, start, end -- the LOCAL batch
 *           mean (reading R5/R6) of this step, before the update.
 * After the call completes, params are bitwise identical on every rank because the
 * ring's gather carries the updated weights. */
tem_status tem_step(tem_ctx* ctx, const void* x, const float* labels, float* loss_out,
                    void* stream);
/* t1 of P:163 only: forward + loss + backward into the local gradient buffer. */
tem_status tem_compute(tem_ctx* ctx, const void* x, const float* labels, float* loss_out,
                       void* stream);
/* t2 of P:163 only: ring allreduce (Mean) of the local gradients fused with the owner's
 * SGD update w = fma(-lr, gbar, w) and the gather of the updated weights. */
tem_status tem_exchange(tem_ctx* ctx, void* stream);
/* Joint TEM + PEM step / compute (cfg->pem_proposals > 0; tem_step / tem_compute return
 * TEM_ERR_INVALID_ARG on such a config).  x, labels as tem_step; bsp: device [B][P][F] fp32 BSP
 * features; iou: device [B][P] fp32 IoU targets (R19).  loss_out: device, 5 * local_ranks
 * floats: the tem_step losses (4 per local rank), then one PEM MSE per local rank.  The TEM
 * and PEM gradients go through one exchange of the concatenated vector. */
tem_status tem_step_pem(tem_ctx* ctx, const void* x, const float* labels, const float* bsp, const float* iou,
                        float* loss_out, void* stream);
tem_status tem_compute_pem(tem_ctx* ctx, const void* x, const float* labels, const float* bsp,
                           const float* iou, float* loss_out, void* stream);
/* PEM ReLU decisions of the last tem_*_pem call of local rank `local_rank`: out[m][j] =
 * 1[a_mj > 0] (uint8, M = B*P rows, H columns) into the caller's device buffer (R7b). */
tem_status tem_pem_relu_decisions(tem_ctx* ctx, int32_t local_rank, uint8_t* out, void* stream);

/* tem_step with HOST buffers (pinned recommended; local_ranks == 1; TEM-only configs): the
 * end-to-end path a user calls.  Copies x and labels host->device into one of two staging sets
 * in the workspace on a private copy stream, runs the step on `stream` once the copy is done,
 * and copies the loss (4 floats) device->host.  Everything is complete when `stream`'s work of
 * this call is; the host buffers may be reused from then on.  Consecutive calls overlap the
 * copy of a step with the compute of the previous one (the staging set of call k is reused by
 * call k+2, after the step of call k is done). */
tem_status tem_step_host(tem_ctx* ctx, const void* x_host, const float* labels_host,
                         float* loss_host, void* stream);
/* Same for a PEM config (pem_proposals > 0): also copies the BSP features [B][P][F] and IoU
 * targets [B][P]; loss_host receives 5 floats: the 4 TEM values of tem_step, then L_PEM.
 * With pgm_gt_max > 0 (PGM-fed, tem_step_pgm) the two extra inputs are instead the ground
 * truth [B][pgm_gt_max][2] fp32 and its counts [B] int32. */
tem_status tem_step_pem_host(tem_ctx* ctx, const void* x_host, const float* labels_host,
                             const float* bsp_host, const float* iou_host, float* loss_host, void* stream);

/* ring_allreduce: in-place allreduce of K fp32 elements.
 *   buf   device; must be the user region of this rank's heap, i.e.
 *         peer_bufs[rank] + tem_sym_user_offset(cfg) (the same offset on every rank);
 *         for local_ranks > 1 every emulated rank's user region is reduced.
 *   K     1 <= K <= max_allreduce_elems (equal on every rank, else PROTOCOL).  The partition
 *         pads K to K_pad = roundup(K, 4N); elements >= K are neither read nor written.
 *   op    TEM_SUM or TEM_MEAN (mean = s * fl(1/N), once, on the block owner; reading R11).
 * Result is bitwise identical on every rank and equals the oracle's ring replay bit for bit:
 * block b is summed along the chain g_b + g_{b+1} + ... + g_{b+N-1}. */
tem_status ring_allreduce(tem_ctx* ctx, float* buf, int64_t K, int32_t op, void* stream);

/* Parameter-server comparator: every rank pushes its buffer into
 * rank 0's heap; rank 0 sums in ascending rank order, applies op, and pushes the
 * result back to every rank.  Same buffer rules as ring_allreduce. */
tem_status ps_allreduce(tem_ctx* ctx, float* buf, int64_t K, int32_t op, void* stream);

/* Two-shot allreduce over NVSwitch: the owner of block b reads block b
 * from every rank's heap and sums along the ring's chain g_b + g_{b+1} + ... + g_{b+N-1}, applies
 * op once and stores the result into every rank's buffer.  Same buffer rules, partition (R9)
 * and result bits as ring_allreduce, with two communication phases instead of 2(N-1). */
tem_status twoshot_allreduce(tem_ctx* ctx, float* buf, int64_t K, int32_t op, void* stream);

/* Joint TEM + PGM + PEM step (pgm_gt_max > 0): TEM forward / backward, then PGM on the
 * sigmoid of this step's logits (stop-gradient), then PEM on the proposals' BSP features with
 * their IoU targets, and the exchange of the joint gradient.  gt [local_ranks][B][G][2] fp32
 * instances (snippet units), n_gt [local_ranks][B] int32, device; loss_out as tem_step_pem.
 * The step's PGM outputs: tem_debug_buffer "pgm_prob" ([B][3][T]), "pgm_feat", "pgm_iou",
 * "pgm_ts", "pgm_te", "pgm_count" (the tem_pgm layouts). */
tem_status tem_step_pgm(tem_ctx* ctx, const void* x, const float* labels, const float* gt, const int32_t* n_gt,
                        float* loss_out, void* stream);
tem_status tem_compute_pgm(tem_ctx* ctx, const void* x, const float* labels, const float* gt,
                           const int32_t* n_gt, float* loss_out, void* stream);

/* PGM, BSN's proposal generation (reading R24; the paper names the
 * stage at P:85): for each of B videos, candidate boundaries of TEM's start / end probability
 * sequences, the P best (start, end) proposals and their 32-d Boundary-Sensitive Proposal
 * features -- the input of PEM -- with IoU targets.  Context-free; all pointers device, on
 * `stream`, written completely (unused proposal rows: ts = te = -1, zero features / IoU).
 *   prob      [B][3][T] fp32: 0 actionness, 1 start, 2 end probabilities (R4); 1 <= T <= 128
 *   gt, n_gt  [B][G][2] fp32 ground-truth instances (start, end) in snippet units and [B]
 *             int32 counts (n_gt[v] > G is clamped to G); G >= 0
 *   P         proposals per video, 1 <= P <= 65536
 *   features  [B][P][32] fp32: 8 samples of the start region, 16 of the proposal, 8 of the end
 *             region of the actionness sequence (linear interpolation, zero outside [0, T-1])
 *   iou       [B][P] fp32: max IoU of [ts + 1/2, te + 1/2] with the instances
 *   ts, te    [B][P] int32 proposal boundaries, ranked by (score desc, ts asc, te asc), score
 *             = fl32(p_start[ts] * p_end[te]); count [B] int32 = proposals found (<= P)
 * Candidates, scores and ranking are fp32 decisions, bit-identical to the oracle.
 * Errors: INVALID_ARG (shapes / null pointers), CUDA (launch). */
tem_status tem_pgm(int32_t B, int32_t T, int32_t G, int32_t P, const float* prob, const float* gt,
                   const int32_t* n_gt, float* features, float* iou, int32_t* ts, int32_t* te, int32_t* count,
                   void* stream);

/* Blocks until all work of ctx on `stream` is done; returns the latched device status.
 * For NONFINITE, *bad_step (if non-NULL) receives the 0-based step index. */
tem_status tem_sync(tem_ctx* ctx, void* stream, int64_t* bad_step);

/* Teardown: the "closing" half of the paper's preparation time t3 / P ("the
 * preparation time for opening and closing deep learning platform"; tem_init is the opening).
 * Synchronises the device, frees the host context, the pinned status word, the graphs and the
 * library's streams / events; the caller's device memory is untouched (it owns it).  Every rank
 * calls it after its last collective; it issues no collective itself.  NULL is a no-op
 * (returns TEM_OK).  Returns any latched error (PROTOCOL / TRANSPORT / NONFINITE / CUDA). */
tem_status tem_shutdown(tem_ctx* ctx);

/* --- introspection for tests and benchmarks (device pointers owned by the workspace) --- */
/* [K_pad] fp32 local gradient of the last tem_compute / tem_step (call after it completed).
 * After an N = 1 tem_step the W1 / W2 parts exist only as split-K partials (the update sums
 * them itself); this call then sums them into the buffer first, in the update's order, on the
 * legacy default stream, and synchronises it. */
float* tem_local_grad(tem_ctx* ctx, int32_t local_rank);
float* tem_logits(tem_ctx* ctx, int32_t local_rank);     /* [B][T][3] fp32 z, last compute */
/* Device address and size of an internal workspace tensor of local rank `local_rank`, for
 * tests: "xp", "h1", "h2", "dA2", "dA1" (halo-padded [B][T+2][C] rows in the path's operand
 * type; h2 fp32, not written when the head is fused into conv2), their residual planes "xp_lo", "h1_lo", "dA2_lo", "dA1_lo", and the weight
 * operand copies "shadow", "shadow_lo" ([K_pad] bf16).  Diagnostics: "tstamp_on" / "tstamp"
 * enable / disable the split-K GEMM phase timestamps ([1024][16] u64 ns).  NULL / 0 if absent. */
void* tem_debug_buffer(tem_ctx* ctx, int32_t local_rank, const char* name, int64_t* nbytes);
/* ReLU decisions of the last tem_compute of local rank `local_rank`: writes
 * out[layer][b][t][c] = 1[a_layer > 0] (uint8, layer 0 = conv1, 1 = conv2) into the
 * caller's device buffer of 2*B*T*c_hidden bytes, on `stream` (reading R7b). */
tem_status tem_relu_decisions(tem_ctx* ctx, int32_t local_rank, uint8_t* out, void* stream);
/* Number of kernels one tem_step / tem_exchange / ring_allreduce(K) enqueues. */
int32_t tem_launches_per_step(tem_ctx* ctx);
int32_t tem_launches_per_exchange(tem_ctx* ctx);
const char* tem_status_string(int32_t status);
/* Per-kernel timing for benchmarks (local_ranks == 1 only).  tem_timing_begin creates
 * host-side CUDA events for up to max_steps subsequent tem_step / tem_step_host calls and
 * brackets every kernel of each step with a start/stop event on the launching stream.
 * tem_timing_end synchronises those events, writes the per-slot SUM over recorded steps
 * (milliseconds) into sum_ms[tem_timing_slots()], the number of recorded steps into
 * *steps, destroys the events and disables timing. */
int32_t tem_timing_slots(tem_ctx* ctx);
const char* tem_timing_slot_name(tem_ctx* ctx, int32_t slot);
tem_status tem_timing_begin(tem_ctx* ctx, int32_t max_steps);
tem_status tem_timing_end(tem_ctx* ctx, float* sum_ms, int32_t* steps);
/* Kernel-path description ("tcgen05-bf16x3-fp32" or "tcgen05-bf16") for reports. */
const char* tem_kernel_path(tem_ctx* ctx);

#ifdef __cplusplus
}
#endif
#endif /* TEM_H_ */
