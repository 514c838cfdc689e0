// tem_capi.cu -- host side of the C ABI declared in include/tem.h.
//
// Validates configurations, lays out the caller-owned workspace and symmetric
// heaps, and enqueues the kernels of prep.cu / tem_umma.cu / head.cu / pem.cu / pgm.cu / ring.cu.  No
// device memory is allocated here.
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>
#include <stdlib.h>

#include <string.h>

#include <algorithm>
#include <new>

#include "kernels.h"

using namespace tem;

bool tem::pdl_enabled() {
    static const int on = getenv("TEM_NO_PDL") ? 0 : 1;
    return on != 0;
}

int tem::launch_priority_attr(cudaLaunchAttribute* a, bool side) {
    static int lo = 1, hi = 1, on = -1;  // numerically lower = higher priority
    if (on < 0) {
        on = 1;
        if (cudaDeviceGetStreamPriorityRange(&lo, &hi) != cudaSuccess) {
            cudaGetLastError();
            on = 0;
        }
    }
    if (!on || lo == hi) return 0;
    // critical path high, side branches (head reduction, conv2 wgrad, PEM) low.  Measured: with
    // the PEM branch at high or equal priority, single c5 steps stalled for 2-22 ms; neutral
    // for c2.
    a->id = cudaLaunchAttributePriority;
    a->val.priority = side ? lo : hi;
    return 1;
}

namespace {

constexpr size_t kAlign = 256;
constexpr uint64_t kSpinMsDefault = 20000;  // flag-wait bound when cfg->spin_timeout_ms == 0
#ifdef TEM_DIAG
constexpr size_t kTraceWords = 2 * NUM_SLOTS + 4096 * 8;    // diagnostics trace area
#endif

size_t align_up(size_t x, size_t a) { return (x + a - 1) / a * a; }
int64_t roundup(int64_t x, int64_t q) { return (x + q - 1) / q * q; }

struct HeapLayout {
    size_t off_user, user_bytes, off_stage, off_ps, off_hdr, off_psflags, off_tsflags, off_ll, total;
    int64_t ll_stride;  // LL lines per ring slot
};

struct WsLayout {
    size_t xp, h1, h2, dA2, dA1, xp_lo, h1_lo, dA2_lo, dA1_lo, z, grad, headpart, headlvl1, counter, bpart, wpart, wpart2, shadow,
        shadow_lo, ones, zpart, epochs, stepctr, dec2, bwd_tasks, bwd_flags, bwd_epoch, xstage, labstage, lossstage, bspstage, ioustage, pempart, pemdec, opt_m, opt_v, opt_scal,
        pgm_prob, pgm_feat, pgm_iou, pgm_ts, pgm_te, pgm_count, trace, per_rank;
};

bool cfg_valid(const tem_config* c) {
    if (!c) return false;
    if (c->world_size < 1 || c->world_size > TEM_MAX_RANKS) return false;
    if (c->rank < 0 || c->rank >= c->world_size) return false;
    if (!(c->local_ranks == 1 || (c->local_ranks == c->world_size && c->rank == 0))) return false;
    if (c->batch_per_rank < 0 || c->seq_len < 1) return false;
    if (c->c_in < 16 || c->c_in % 16 != 0) return false;
    if (c->c_hidden < 128 || c->c_hidden % 128 != 0 || c->c_hidden > 512) return false;
    if (c->c_out != 3) return false;
    if (c->precision != TEM_FP32 && c->precision != TEM_BF16) return false;
    if (!(c->lr >= 0.0f) || !isfinite(c->lr)) return false;
    for (int o = 0; o < 3; ++o)
        if (!isfinite(c->loss_weight[o])) return false;
    if (c->max_allreduce_elems < 0) return false;
    if (c->ring_channels < 0 || c->ring_channels > kMaxChannels) return false;
    if (c->spin_timeout_ms < 0) return false;
    if (c->exchange != TEM_EXCHANGE_RING && c->exchange != TEM_EXCHANGE_PS && c->exchange != TEM_EXCHANGE_TWOSHOT)
        return false;
    if (c->pem_proposals < 0) return false;
    if (c->pem_proposals > 0 && (c->pem_features != 32 || c->pem_hidden != 512)) return false;  // kernel shape
    if (c->exchange_buckets < 0 || c->exchange_buckets > 2) return false;
    if (c->exchange_buckets == 2 && c->exchange == TEM_EXCHANGE_PS) return false;
    if (c->pgm_gt_max < 0 || (c->pgm_gt_max > 0 && (c->pem_proposals <= 0 || c->seq_len > 128))) return false;
    if (c->optimizer != TEM_OPT_SGD && c->optimizer != TEM_OPT_ADAM && c->optimizer != TEM_OPT_MOMENTUM) return false;
    if (c->optimizer == TEM_OPT_MOMENTUM && !(c->momentum >= 0.0f && c->momentum < 1.0f)) return false;
    if (c->optimizer == TEM_OPT_ADAM &&
        !(c->beta1 >= 0.0f && c->beta1 < 1.0f && c->beta2 >= 0.0f && c->beta2 < 1.0f && c->eps > 0.0f &&
          isfinite(c->eps)))
        return false;
    return true;
}

int64_t tem_params_only(const tem_config* c) {
    const int64_t C = c->c_hidden, Ci = c->c_in, Co = c->c_out;
    return C * 3 * Ci + C + C * 3 * C + C + Co * C + Co;
}
int64_t num_params(const tem_config* c) {  // [TEM | PEM] (reading R21)
    const int64_t pem = c->pem_proposals > 0
                            ? (int64_t)c->pem_hidden * c->pem_features + 2 * (int64_t)c->pem_hidden + 1
                            : 0;
    return tem_params_only(c) + pem;
}

Geom make_geom(const tem_config* c) {
    Geom g;
    g.B = c->batch_per_rank;
    g.T = c->seq_len;
    g.Cin = c->c_in;
    g.C = c->c_hidden;
    g.Co = c->c_out;
    g.R = g.B * (g.T + 2);
    g.prec = c->precision;
    g.split = g.prec == TEM_FP32 ? 1 : 0;
    g.K = num_params(c);
    g.Kpad = roundup(g.K, 4 * (int64_t)c->world_size);
    g.off_W1 = 0;
    g.off_b1 = g.off_W1 + (int64_t)g.C * 3 * g.Cin;
    g.off_W2 = g.off_b1 + g.C;
    g.off_b2 = g.off_W2 + (int64_t)g.C * 3 * g.C;
    g.off_W3 = g.off_b2 + g.C;
    g.off_b3 = g.off_W3 + (int64_t)g.Co * g.C;
    g.pem_P = c->pem_proposals;
    g.pgm_G = c->pgm_gt_max;
    g.pem_F = c->pem_proposals > 0 ? c->pem_features : 0;
    g.pem_H = c->pem_proposals > 0 ? c->pem_hidden : 0;
    g.off_pem = tem_params_only(c);
    return g;
}

int64_t max_ar(const tem_config* c) {
    return c->max_allreduce_elems > 0 ? c->max_allreduce_elems : num_params(c);
}

HeapLayout heap_layout(const tem_config* c) {
    HeapLayout h;
    const int64_t N = c->world_size;
    const int64_t kpad = roundup(num_params(c), 4 * N);
    const int64_t kar = roundup(max_ar(c), 4 * N);
    h.off_user = align_up((size_t)kpad * 4, 4096);
    h.user_bytes = (size_t)kar * 4;
    h.off_stage = align_up(h.off_user + h.user_bytes, 4096);
    const size_t stage_bytes = (size_t)(kpad > kar ? kpad : kar) * 4;
    h.off_ps = align_up(h.off_stage + stage_bytes, 4096);
    const int64_t kps = roundup(num_params(c) > max_ar(c) ? num_params(c) : max_ar(c), 4);
    h.off_hdr = align_up(h.off_ps + (size_t)N * kps * 4, 4096);
    h.off_psflags = h.off_hdr + (size_t)2 * TEM_MAX_RANKS * kMaxChannels * 16;
    h.off_tsflags = h.off_psflags + (size_t)2 * TEM_MAX_RANKS * kMaxChannels * 8;
    // ring LL slots: [2 epoch parities][2 phases][N-1 rounds][2 lines per float4 of the
    // largest block] x 16 B
    h.ll_stride = (kpad > kar ? kpad : kar) / N / 2;
    h.off_ll = align_up(h.off_tsflags + (size_t)2 * TEM_MAX_RANKS * kMaxChannels * 8, 4096);
    h.total = align_up(h.off_ll + (size_t)4 * (N - 1) * h.ll_stride * 16, 4096);
    return h;
}

int64_t shadow_set_elems(const Geom& g) { return roundup(g.Kpad, 256); }

WsLayout ws_layout(const tem_config* c) {
    const Geom g = make_geom(c);
    const size_t esz = 2;                           // operand planes are bf16
    const size_t xsz = g.prec == TEM_BF16 ? 2 : 4;  // caller's x element size
    WsLayout w;
    size_t o = 0;
    auto take = [&](size_t bytes) {
        const size_t at = o;
        o = align_up(o + bytes, kAlign);
        return at;
    };
    const int S = umma_wgrad_splits(g);
    const size_t wmax = (size_t)g.C * 3 * (g.Cin > g.C ? g.Cin : g.C) + g.C;
    w.xp = take((size_t)g.R * g.Cin * esz);
    w.h1 = take((size_t)g.R * g.C * esz);
    w.h2 = take((size_t)g.R * g.C * 4);
    w.dA2 = take((size_t)g.R * g.C * esz);
    w.dA1 = take((size_t)g.R * g.C * esz);
    const size_t lo = g.split ? 1 : 0;
    w.xp_lo = take(lo * g.R * g.Cin * esz);
    w.h1_lo = take(lo * g.R * g.C * esz);
    w.dA2_lo = take(lo * g.R * g.C * esz);
    w.dA1_lo = take(lo * g.R * g.C * esz);
    w.z = take((size_t)g.B * g.T * 3 * 4);
    w.grad = take((size_t)g.Kpad * 4);
    w.headpart = take((size_t)head_ctas(g) * (4 * g.C + 8) * 4);
    w.headlvl1 = take((size_t)32 * (4 * g.C + 6) * 4);
    w.counter = take(64);
    w.bpart = take((size_t)((g.R + 127) / 128) * g.C * 4);
    w.wpart = take((size_t)S * wmax * 4);
    w.wpart2 = take((size_t)S * ((size_t)g.C * 3 * g.C + g.C) * 4);
    w.pempart = take((size_t)pem_ctas(g) * (pem_num_params_of(g) + 1) * 4);
    w.pemdec = take(g.pem_P > 0 ? (size_t)g.B * g.pem_P * g.pem_H : 0);  // last ReLU decisions (tests)
    // two operand sets (ping-pong, RankBufs::shadow), each 512-byte aligned (TMA bases)
    w.shadow = take(2 * (size_t)shadow_set_elems(g) * 2);
    w.shadow_lo = take(lo * 2 * (size_t)shadow_set_elems(g) * 2);
    w.ones = take((size_t)g.R * 128 * 2);
    w.zpart = take((size_t)(g.C / 64) * g.R * 3 * 4);
    w.epochs = take((size_t)kMaxChannels * 4);
    w.stepctr = take(8);
    w.dec2 = take((size_t)g.R * (g.C / 64) * 8);
    w.bwd_tasks = take((size_t)1024 * BWD_MAX_TASKS * 4);  // persistent backward (UmmaPlan::bwd_grid)
    w.bwd_flags = take((size_t)BWD_MAX_DG_TILES * 4);
    w.bwd_epoch = take(2 * 4);
    // host-input staging (tem_step_host / tem_step_pem_host), double-buffered: the copy of step
    // k+1 lands in the other set while step k computes
    w.xstage = take(2 * (size_t)g.B * g.T * g.Cin * xsz);
    w.labstage = take(2 * (size_t)g.B * 3 * g.T * 4);
    w.lossstage = take(8 * 4);
    w.bspstage = take(2 * (size_t)g.B * g.pem_P * g.pem_F * 4);
    w.ioustage = take(2 * (size_t)g.B * g.pem_P * 4);
    const size_t adam = c->optimizer == TEM_OPT_ADAM ? 1 : 0;  // reading R22
    const size_t state1 = c->optimizer != TEM_OPT_SGD ? 1 : 0;  // Adam's m / momentum's u (R23)
    w.opt_m = take(state1 * (size_t)g.Kpad * 4);
    w.opt_v = take(adam * (size_t)g.Kpad * 4);
    w.opt_scal = take(adam * 8);
    const size_t pgm = g.pgm_G > 0 ? 1 : 0;  // PGM-fed PEM (reading R24)
    w.pgm_prob = take(pgm * (size_t)g.B * 3 * g.T * 4);
    w.pgm_feat = take(pgm * (size_t)g.B * g.pem_P * 32 * 4);
    w.pgm_iou = take(pgm * (size_t)g.B * g.pem_P * 4);
    w.pgm_ts = take(pgm * (size_t)g.B * g.pem_P * 4);
    w.pgm_te = take(pgm * (size_t)g.B * g.pem_P * 4);
    w.pgm_count = take(pgm * (size_t)g.B * 4);
#ifdef TEM_DIAG
    w.trace = take(sizeof(unsigned long long) * kTraceWords);  // diagnostics build only
#endif
    w.per_rank = o;
    return w;
}

}  // namespace

struct tem_ctx {
    tem_config cfg;
    void* peers[TEM_MAX_RANKS];
    Geom g;
    HeapLayout hl;
    WsLayout wl;
    int N, nlocal, rank;
    int G;                     // channels (CTAs per rank) of every collective: fixed per context,
                               // so the per-channel epochs advance together
    uint64_t spin_ns;          // flag-wait bound
    RankBufs rb[TEM_MAX_RANKS];
    UmmaPlan* plan[TEM_MAX_RANKS];
    uint32_t* epochs[TEM_MAX_RANKS];
    char* ws_base[TEM_MAX_RANKS];
    Status* st_host;
    Status* st_dev;
    int launches_step, launches_exchange;
    bool alive;
    int wpar;              // operand set (RankBufs::shadow) holding the current weights: a step's
                           // GEMMs read it, its update writes 1 - wpar, then it flips
    bool reduce_deferred;  // last compute left the split-K partials for the fused N = 1 exchange
    bool split_n1;         // ... and updated [off_W2, K_pad) itself on its side branch
    bool early_done;       // bucketed exchange: the [bnd, K_pad) bucket ran inside the compute
    bool grad_lazy;        // N = 1 tem_step left the W1 / W2 gradient as split-K partials only;
                           // tem_local_grad sums them on demand (same order as the update)
    // per-kernel timing (tem_timing_*)
    cudaEvent_t* tev;  // [max_steps][NUM_SLOTS*2]
    int t_max, t_idx;
    // CUDA-graph replay of whole steps (one graph per input pointer set), run on a private
    // non-blocking stream ordered with the caller's stream by events
    float* loss_host_pending;  // tem_step_host: host loss buffer the compute reads back into
    bool loss_host_done;
    const float* pem_bsp;      // tem_*_pem: this call's PEM inputs (nullptr: TEM-only call)
    const float* pem_iou;
    const float* pgm_gt;       // tem_*_pgm: this call's ground truth [nlocal][B][G][2] / counts
    const int32_t* pgm_ngt;
    bool pem_record_dec;       // record the PEM ReLU decisions (tem_pem_relu_decisions)
    struct GraphEntry {
        const void* x;
        const void* lab;
        const void* bsp;
        const void* iou;
        const void* gt;
        const void* ngt;
        int wpar;
        void* loss;
        void* loss_host;
        cudaGraphExec_t exec;
        int launches;
        bool grad_lazy;  // the captured step leaves the W1 / W2 gradient as partials
    };
    static constexpr int kMaxGraphs = 16;
    GraphEntry graphs[kMaxGraphs];
    int ngraphs;
    bool use_graphs;
    cudaStream_t gstream;
    cudaEvent_t ev_in, ev_out;
    // host-input pipeline (tem_step_host): copy stream, per staging set "copied" / "consumed"
    cudaStream_t cstream;
    cudaEvent_t ev_copied[2], ev_consumed[2];
    int hslot;
};

namespace {
// Replay (capturing on first use) the step for this pointer set.  Returns TEM_OK, or an error
// from capture; `fn` enqueues the step on the stream it is given and reports its launches.
template <typename F>
tem_status graph_step(tem_ctx* c, const void* x, const void* lab, void* loss, cudaStream_t s, F&& fn) {
    tem_ctx::GraphEntry* e = nullptr;
    for (int i = 0; i < c->ngraphs; ++i)
        if (c->graphs[i].x == x && c->graphs[i].lab == lab && c->graphs[i].loss == loss &&
            c->graphs[i].loss_host == c->loss_host_pending && c->graphs[i].bsp == c->pem_bsp &&
            c->graphs[i].iou == c->pem_iou && c->graphs[i].gt == c->pgm_gt && c->graphs[i].ngt == c->pgm_ngt &&
            c->graphs[i].wpar == c->wpar)
            e = &c->graphs[i];
    if (!e) {
        if (c->ngraphs == tem_ctx::kMaxGraphs) {  // evict the oldest
            cudaGraphExecDestroy(c->graphs[0].exec);
            for (int i = 1; i < c->ngraphs; ++i) c->graphs[i - 1] = c->graphs[i];
            --c->ngraphs;
        }
        cudaGraph_t graph = nullptr;
        if (cudaStreamBeginCapture(c->gstream, cudaStreamCaptureModeRelaxed) != cudaSuccess) return TEM_ERR_CUDA;
        int nl = 0;
        const tem_status st = fn(c->gstream, &nl);
        const cudaError_t ce = cudaStreamEndCapture(c->gstream, &graph);
        if (st != TEM_OK || ce != cudaSuccess) {
            if (graph) cudaGraphDestroy(graph);
            cudaGetLastError();
            return st != TEM_OK ? st : TEM_ERR_CUDA;
        }
        cudaGraphExec_t exec = nullptr;
        // per-node launch priorities (critical path vs side branch) only apply with this flag
        const cudaError_t ie = cudaGraphInstantiateWithFlags(&exec, graph, cudaGraphInstantiateFlagUseNodePriority);
        cudaGraphDestroy(graph);
        if (ie != cudaSuccess) return TEM_ERR_CUDA;
        cudaGraphUpload(exec, s);
        e = &c->graphs[c->ngraphs++];
        e->x = x;
        e->lab = lab;
        e->loss = loss;
        e->loss_host = c->loss_host_pending;
        e->bsp = c->pem_bsp;
        e->iou = c->pem_iou;
        e->gt = c->pgm_gt;
        e->ngt = c->pgm_ngt;
        e->wpar = c->wpar;
        e->exec = exec;
        e->launches = nl;
        e->grad_lazy = c->grad_lazy;
    }
    // Captured on the private stream, replayed directly on the caller's stream (stream order
    // gives the dependencies; no cross-stream event handoff per step).
    if (cudaGraphLaunch(e->exec, s) != cudaSuccess) return TEM_ERR_CUDA;
    c->grad_lazy = e->grad_lazy;
    if (e->loss_host && c->g.B > 0) c->loss_host_done = true;
    c->launches_step = e->launches;
    return TEM_OK;
}
}  // namespace

extern "C" {

const char* tem_status_string(int32_t s) {
    switch (s) {
        case TEM_OK: return "TEM_OK";
        case TEM_ERR_INVALID_ARG: return "TEM_ERR_INVALID_ARG";
        case TEM_ERR_PROTOCOL: return "TEM_ERR_PROTOCOL";
        case TEM_ERR_TRANSPORT: return "TEM_ERR_TRANSPORT";
        case TEM_ERR_CUDA: return "TEM_ERR_CUDA";
        case TEM_ERR_NONFINITE: return "TEM_ERR_NONFINITE";
        case TEM_ERR_STATE: return "TEM_ERR_STATE";
        default: return "TEM_ERR_UNKNOWN";
    }
}

int64_t tem_num_params(const tem_config* cfg) { return cfg_valid(cfg) ? num_params(cfg) : 0; }

int64_t tem_kpad(const tem_config* cfg, int64_t K) {
    if (!cfg_valid(cfg) || K < 0) return 0;
    return roundup(K, 4 * (int64_t)cfg->world_size);
}

size_t tem_workspace_bytes(const tem_config* cfg) {
    if (!cfg_valid(cfg)) return 0;
    return ws_layout(cfg).per_rank * (size_t)cfg->local_ranks;
}

size_t tem_sym_bytes(const tem_config* cfg) { return cfg_valid(cfg) ? heap_layout(cfg).total : 0; }

size_t tem_sym_user_offset(const tem_config* cfg) { return cfg_valid(cfg) ? heap_layout(cfg).off_user : 0; }

size_t tem_sym_hdr_offset(const tem_config* cfg) { return cfg_valid(cfg) ? heap_layout(cfg).off_hdr : 0; }

size_t tem_sym_ll_offset(const tem_config* cfg) { return cfg_valid(cfg) ? heap_layout(cfg).off_ll : 0; }

int64_t tem_ll_slot_lines(const tem_config* cfg) { return cfg_valid(cfg) ? heap_layout(cfg).ll_stride : 0; }

tem_status tem_init(const tem_config* cfg, float* params, tem_ctx** out) {
    if (!out) return TEM_ERR_INVALID_ARG;
    *out = nullptr;
    if (!cfg_valid(cfg) || !cfg->peer_bufs || !params || !cfg->workspace) return TEM_ERR_INVALID_ARG;
    const HeapLayout hl = heap_layout(cfg);
    const WsLayout wl = ws_layout(cfg);
    if (cfg->sym_bytes < hl.total) return TEM_ERR_INVALID_ARG;
    if (cfg->workspace_bytes < wl.per_rank * (size_t)cfg->local_ranks) return TEM_ERR_INVALID_ARG;
    if (((uintptr_t)cfg->workspace) % kAlign) return TEM_ERR_INVALID_ARG;
    for (int r = 0; r < cfg->world_size; ++r)
        if (!cfg->peer_bufs[r] || ((uintptr_t)cfg->peer_bufs[r]) % 4096) return TEM_ERR_INVALID_ARG;
    if ((void*)params != cfg->peer_bufs[cfg->rank]) return TEM_ERR_INVALID_ARG;
    if (cudaSetDevice(cfg->device) != cudaSuccess) return TEM_ERR_CUDA;

    tem_ctx* c = new (std::nothrow) tem_ctx();
    if (!c) return TEM_ERR_CUDA;
    c->cfg = *cfg;
    for (int r = 0; r < cfg->world_size; ++r) c->peers[r] = cfg->peer_bufs[r];
    c->cfg.peer_bufs = c->peers;
    c->g = make_geom(cfg);
    c->hl = hl;
    c->wl = wl;
    c->N = cfg->world_size;
    c->nlocal = cfg->local_ranks;
    c->rank = cfg->rank;
    // channels of every collective (identical on every rank: depends on cfg only, never on a
    // call's K)
    c->G = cfg->ring_channels > 0 ? cfg->ring_channels : 16;
    c->spin_ns = (uint64_t)(cfg->spin_timeout_ms > 0 ? cfg->spin_timeout_ms : kSpinMsDefault) * 1000000ull;
    if (c->nlocal > 1) {  // emulation: all CTAs of all emulated ranks must be co-resident
        int dev_sms = 148;
        cudaDeviceGetAttribute(&dev_sms, cudaDevAttrMultiProcessorCount, cfg->device);
        const int cap = dev_sms / c->nlocal;
        if (c->G > cap) c->G = cap;
    }
    if (cudaHostAlloc((void**)&c->st_host, 64, cudaHostAllocMapped) != cudaSuccess) {
        delete c;
        return TEM_ERR_CUDA;
    }
    memset((void*)c->st_host, 0, 64);
    if (cudaHostGetDevicePointer((void**)&c->st_dev, c->st_host, 0) != cudaSuccess) {
        cudaFreeHost(c->st_host);
        delete c;
        return TEM_ERR_CUDA;
    }
    for (int l = 0; l < c->nlocal; ++l) {
        char* base = (char*)cfg->workspace + wl.per_rank * l;
        c->ws_base[l] = base;
        RankBufs& b = c->rb[l];
        b.params = (const float*)c->peers[c->rank + l];
        b.xp = base + wl.xp;
        b.h1 = base + wl.h1;
        b.h2 = (float*)(base + wl.h2);
        b.dA2 = base + wl.dA2;
        b.dA1 = base + wl.dA1;
        b.z = (float*)(base + wl.z);
        b.grad = (float*)(base + wl.grad);
        b.headpart = (float*)(base + wl.headpart);
        b.headlvl1 = (float*)(base + wl.headlvl1);
        b.counter = (unsigned*)(base + wl.counter);
        b.bpart = (float*)(base + wl.bpart);
        b.ones = base + wl.ones;
        b.zpart = (float*)(base + wl.zpart);
        b.nzpart = 0;  // set by the tcgen05 plan
        b.wpart = (float*)(base + wl.wpart);
        b.wpart2 = (float*)(base + wl.wpart2);
        b.pempart = (float*)(base + wl.pempart);
        b.pemdec = (uint8_t*)(base + wl.pemdec);
        b.stepctr = (int64_t*)(base + wl.stepctr);
        b.dec2 = (uint64_t*)(base + wl.dec2);
        b.bwd.tasks = (int*)(base + wl.bwd_tasks);
        b.bwd.flags = (unsigned*)(base + wl.bwd_flags);
        b.bwd.epoch = (unsigned*)(base + wl.bwd_epoch);
        b.xp_lo = c->g.split ? base + wl.xp_lo : nullptr;
        b.h1_lo = c->g.split ? base + wl.h1_lo : nullptr;
        b.dA2_lo = c->g.split ? base + wl.dA2_lo : nullptr;
        b.dA1_lo = c->g.split ? base + wl.dA1_lo : nullptr;
        b.shadow = (__nv_bfloat16*)(base + wl.shadow);
        b.shadow_lo = c->g.split ? (__nv_bfloat16*)(base + wl.shadow_lo) : nullptr;
        b.shadow_set = shadow_set_elems(c->g);
        c->plan[l] = nullptr;
        c->epochs[l] = (uint32_t*)(base + wl.epochs);
        cudaError_t e = cudaMemsetAsync(base, 0, wl.per_rank, 0);
        if (e == cudaSuccess && cfg->optimizer == TEM_OPT_ADAM) {  // beta^0 = 1 (reading R22)
            static const float one2[2] = {1.0f, 1.0f};
            e = cudaMemcpy(base + wl.opt_scal, one2, sizeof(one2), cudaMemcpyHostToDevice);
        }
        if (e == cudaSuccess) e = launch_cast_shadow_split(b.params, b.shadow, b.shadow_lo, c->g.Kpad, 0);
        if (e == cudaSuccess) e = launch_fill_ones(b.ones, c->g.R, 0);
        if (e == cudaSuccess) {
            c->plan[l] = new (std::nothrow) UmmaPlan();
            if (!c->plan[l] || !umma_plan(c->g, b, c->plan[l])) e = cudaErrorInvalidValue;
            else b.nzpart = c->plan[l]->conv2.zpart ? c->plan[l]->conv2.ntiles : 0;
            b.dec2_valid = c->plan[l] && c->plan[l]->conv2.fused_head ? 1 : 0;
        }
        if (e != cudaSuccess) {
            for (int q = 0; q <= l; ++q) umma_plan_destroy(c->plan[q]);
            cudaFreeHost(c->st_host);
            delete c;
            return TEM_ERR_CUDA;
        }
    }
    if (cudaStreamSynchronize(0) != cudaSuccess) {
        cudaFreeHost(c->st_host);
        delete c;
        return TEM_ERR_CUDA;
    }
    c->launches_step = 0;
    c->launches_exchange = 0;
    c->ngraphs = 0;
    c->wpar = 0;  // tem_init cast the weights into set 0
    // graphs: one rank per process only (the emulation's cooperative launch is not captured)
    const char* ng = getenv("TEM_NO_GRAPH");
    c->use_graphs = c->nlocal == 1 && !(ng && ng[0] == '1');
    c->gstream = nullptr;
    if (c->use_graphs &&
        (cudaStreamCreateWithFlags(&c->gstream, cudaStreamNonBlocking) != cudaSuccess ||
         cudaEventCreateWithFlags(&c->ev_in, cudaEventDisableTiming) != cudaSuccess ||
         cudaEventCreateWithFlags(&c->ev_out, cudaEventDisableTiming) != cudaSuccess)) {
        cudaGetLastError();
        c->use_graphs = false;
    }
    c->alive = true;
    *out = c;
    return TEM_OK;
}

static tem_status check_ctx(tem_ctx* c) {
    if (!c || !c->alive) return TEM_ERR_STATE;
    const int32_t code = *(volatile int32_t*)&c->st_host->code;
    if (code != 0) return (tem_status)code;
    return TEM_OK;
}

static cudaEvent_t* timing_slot_events(tem_ctx* c) {
    if (!c->tev || c->t_idx >= c->t_max || c->nlocal != 1) return nullptr;
    return c->tev + (size_t)c->t_idx * NUM_SLOTS * 2;
}

static OptCfg opt_cfg(const tem_ctx* c) {
    OptCfg o;
    o.kind = c->cfg.optimizer;
    o.lr = c->cfg.lr;
    o.beta1 = c->cfg.beta1;
    o.beta2 = c->cfg.beta2;
    o.c1 = 1.0f - c->cfg.beta1;  // fp32 subtraction (the oracle's c1)
    o.c2 = 1.0f - c->cfg.beta2;
    o.eps = c->cfg.eps;
    o.mu = c->cfg.momentum;
    return o;
}

static OptState opt_state(const tem_ctx* c, int l) {
    OptState o{nullptr, nullptr, nullptr};
    if (c->cfg.optimizer == TEM_OPT_MOMENTUM) o.m = (float*)(c->ws_base[l] + c->wl.opt_m);
    if (c->cfg.optimizer == TEM_OPT_ADAM) {
        o.m = (float*)(c->ws_base[l] + c->wl.opt_m);
        o.v = (float*)(c->ws_base[l] + c->wl.opt_v);
        o.scal = (const float*)(c->ws_base[l] + c->wl.opt_scal);
    }
    return o;
}

static RingLocal ring_local(tem_ctx* c, int l, const float* src, float* dst, __nv_bfloat16* shadow,
                            __nv_bfloat16* shadow_lo);

// bucketed exchange (reading R25): [0, bnd) and [bnd, K_pad), bnd = roundup(off_W2, 4N)
static int64_t bucket_bound(const tem_ctx* c) {
    const int64_t q = 4 * (int64_t)c->N;
    return (c->g.off_W2 + q - 1) / q * q;
}
static bool bucketed(const tem_ctx* c) { return c->cfg.exchange_buckets == 2 && c->N > 1; }

static void set_heap_offsets(const tem_ctx* c, RingParams* p) {
    p->off_stage = (int64_t)c->hl.off_stage;
    p->off_flags = (int64_t)c->hl.off_tsflags;  // two-shot phase flags (the ring needs none)
    p->off_hdr = (int64_t)c->hl.off_hdr;
    p->off_ll = (int64_t)c->hl.off_ll;
    p->ll_stride = c->hl.ll_stride;
    p->status = c->st_dev;
    p->spin_ns = c->spin_ns;
}

// The tem_step exchange of elements [e0, e1) of the flat gradient: every pointer and the heap
// destination offset shifted by e0, the ring's partition taken over e1 - e0 (a multiple of 4N).
static RingParams step_ring(tem_ctx* c, int64_t e0, int64_t e1) {
    RingParams p;
    memset(&p, 0, sizeof(p));
    for (int l = 0; l < c->nlocal; ++l) {
        const RankBufs& b = c->rb[l];
        __nv_bfloat16* sl = shadow_lo(b, 1 - c->wpar);  // the update writes the other operand set
        p.loc[l] = ring_local(c, l, b.grad + e0, (float*)b.params + e0, shadow_hi(b, 1 - c->wpar) + e0,
                              sl ? sl + e0 : nullptr);
        if (p.loc[l].opt.m) p.loc[l].opt.m += e0;
        if (p.loc[l].opt.v) p.loc[l].opt.v += e0;
    }
    p.N = c->N;
    p.rank_base = c->rank;
    p.nlocal = c->nlocal;
    p.G = c->G;
    p.op = TEM_MEAN;
    p.mode = 1;
    p.K = e1 - e0;
    p.Kpad = e1 - e0;
    p.oc = opt_cfg(c);
    p.off_dst = e0 * (int64_t)sizeof(float);
    set_heap_offsets(c, &p);
    return p;
}

static cudaError_t launch_step_ring(tem_ctx* c, const RingParams& p, cudaStream_t s) {
    return c->cfg.exchange == TEM_EXCHANGE_TWOSHOT ? launch_twoshot(p, s) : launch_ring(p, s);
}

// fuse_reduce (tem_step): at N = 1 the split-K reductions are left to the update kernel
static tem_status compute_impl(tem_ctx* c, const void* x, const float* labels, float* loss_out,
                               cudaStream_t s, int* nl, bool fuse_reduce = false) {
    const EvRec rec{timing_slot_events(c), s};
    const Geom& g = c->g;
    const size_t esz = g.prec == TEM_BF16 ? 2 : 4;  // caller's x element size
    const float lam[3] = {c->cfg.loss_weight[0], c->cfg.loss_weight[1], c->cfg.loss_weight[2]};
    for (int l = 0; l < c->nlocal; ++l) {
        const char* xl = (const char*)x + (size_t)l * g.B * g.T * g.Cin * esz;
        const float* labl = labels + (size_t)l * g.B * 3 * g.T;
        rec.begin(SLOT_PREP);
        cudaError_t e = g.split ? launch_prep_x_split(g, (const float*)xl, c->rb[l].xp, c->rb[l].xp_lo, s)
                                : launch_prep_x(g, xl, c->rb[l].xp, s);
        rec.end(SLOT_PREP);
        if (e != cudaSuccess) return TEM_ERR_CUDA;
        ++*nl;
        const bool defer = fuse_reduce && c->N == 1 && g.B > 0;
        c->reduce_deferred = defer;
        c->grad_lazy = false;  // this compute's partials overwrite the last step's
        SplitUpdate su{opt_cfg(c), opt_state(c, l)};
        // N = 1: [off_W2, K_pad) is updated on the side branch as soon as conv2 wgrad and the head
        // are done (measured c2 195.5k -> 200.4k samples/s with the default 296-CTA grid; 16-64
        // CTAs were slower), the exchange then updates [0, off_W2) only.  Not with PGM-fed PEM,
        // whose gradient is produced after the compute.
        // the persistent backward has no side-branch WGRAD to hang the split update / early
        // bucket off: the exchange then updates (or exchanges) the whole vector after it
        const bool bwd = g.B > 0 && umma_bwd_active(*c->plan[l]);
        c->split_n1 = defer && g.pgm_G == 0 && !bwd;
        su.n1_w2 = c->split_n1 ? 1 : 0;
        // bucketed exchange with one rank per process: the [bnd, K_pad) bucket starts inside the
        // compute (not with PGM-fed PEM, whose gradient is produced after it)
        RingParams early;
        c->early_done = false;
        if (bucketed(c) && c->nlocal == 1 && fuse_reduce && g.B > 0 && g.pgm_G == 0 && !bwd) {
            early = step_ring(c, bucket_bound(c), g.Kpad);
            su.early = &early;
            su.early_kind = c->cfg.exchange;
            c->early_done = true;
        }
        float* lh = (c->nlocal == 1) ? c->loss_host_pending : nullptr;
        if (g.pem_P > 0 && g.pgm_G == 0) {
            // PEM (configs[4]): both kernels on the critical path right after prep_x, on all SMs
            // (on a side stream beside the TEM GEMMs it measured slower and stalled)
            const int M = g.B * g.pem_P;
            e = launch_pem(g, c->pem_bsp + (size_t)l * M * g.pem_F, c->pem_iou + (size_t)l * M,
                           c->rb[l].params + g.off_pem, c->rb[l].pempart, c->rb[l].grad + g.off_pem,
                           loss_out + 4 * c->nlocal + l, c->st_dev, c->rb[l].stepctr,
                           c->pem_record_dec ? c->rb[l].pemdec : nullptr, s, s, nullptr, nl, rec);
            if (e != cudaSuccess) return TEM_ERR_CUDA;
        }
        if (g.B > 0) {
            e = umma_compute(g, c->rb[l], *c->plan[l], labl, lam, loss_out + 4 * l, c->st_dev, nl, rec, s, c->wpar,
                             defer, lh, (c->early_done || c->split_n1) ? &su : nullptr);
            if (lh) c->loss_host_done = true;
        } else {
            e = empty_shard_compute(g, c->rb[l], labl, lam, loss_out + 4 * l, c->st_dev, nl, rec, s);
        }
        if (e != cudaSuccess) return TEM_ERR_CUDA;
        if (g.pem_P > 0 && g.pgm_G > 0 && g.B > 0) {
            // PGM-fed PEM (reading R24): proposals and BSP features from this step's logits
            // (stop-gradient), then PEM on them -- after the TEM compute, on the step's stream
            char* base = c->ws_base[l];
            float* feat = (float*)(base + c->wl.pgm_feat);
            float* iou = (float*)(base + c->wl.pgm_iou);
            rec.begin(SLOT_PGM);
            e = launch_pgm(g.B, g.T, g.pgm_G, g.pem_P, nullptr, c->pgm_gt + (size_t)l * g.B * g.pgm_G * 2,
                           c->pgm_ngt + (size_t)l * g.B, feat, iou, (int32_t*)(base + c->wl.pgm_ts),
                           (int32_t*)(base + c->wl.pgm_te), (int32_t*)(base + c->wl.pgm_count), s, c->rb[l].z,
                           (float*)(base + c->wl.pgm_prob));
            rec.end(SLOT_PGM);
            if (e != cudaSuccess) return TEM_ERR_CUDA;
            ++*nl;
            e = launch_pem(g, feat, iou, c->rb[l].params + g.off_pem, c->rb[l].pempart, c->rb[l].grad + g.off_pem,
                           loss_out + 4 * c->nlocal + l, c->st_dev, c->rb[l].stepctr,
                           c->pem_record_dec ? c->rb[l].pemdec : nullptr, s, s, nullptr, nl, rec);
            if (e != cudaSuccess) return TEM_ERR_CUDA;
        }
    }
    return TEM_OK;
}

// Adam: advance every local rank's beta^t before the update reads it
static tem_status opt_scalars(tem_ctx* c, cudaStream_t s, int* nl) {
    if (c->cfg.optimizer != TEM_OPT_ADAM) return TEM_OK;
    for (int l = 0; l < c->nlocal; ++l) {
        if (launch_opt_scalars((float*)(c->ws_base[l] + c->wl.opt_scal), c->cfg.beta1, c->cfg.beta2, s) !=
            cudaSuccess)
            return TEM_ERR_CUDA;
        ++*nl;
    }
    return TEM_OK;
}

static RingLocal ring_local(tem_ctx* c, int l, const float* src, float* dst, __nv_bfloat16* shadow,
                            __nv_bfloat16* shadow_lo) {
    RingLocal L;
    L.opt = opt_state(c, l);
    L.src = src;
    L.dst_self = dst;
    L.shadow = shadow;
    L.shadow_lo = shadow_lo;
    L.epochs = c->epochs[l];
    for (int r = 0; r < TEM_MAX_RANKS; ++r) L.heaps[r] = r < c->N ? (char*)c->peers[r] : nullptr;
    return L;
}

static tem_status exchange_impl(tem_ctx* c, cudaStream_t s, int* nl) {
    const Geom& g = c->g;
    const EvRec rec{timing_slot_events(c), s};
    rec.begin(SLOT_EXCHANGE);
    const OptCfg oc = opt_cfg(c);
    const int wr = 1 - c->wpar;  // every update writes the other operand set (RankBufs::shadow)
    if (c->N == 1 && c->reduce_deferred) {  // tem_step: split-K reductions fused into the update
        const RankBufs& b = c->rb[0];
        const UmmaPlan& P = *c->plan[0];
        c->reduce_deferred = false;
        // the summed W1 / W2 gradient is not stored (5.6 MB of writes): tem_local_grad rebuilds
        // it from the partials on demand, in the same order
        const int64_t e1 = c->split_n1 ? g.off_W2 : g.Kpad;
        c->split_n1 = false;
        if (launch_sgd_fused(b.grad, (float*)b.params, shadow_hi(b, wr), shadow_lo(b, wr), 0, e1, oc,
                             opt_state(c, 0), b.wpart, P.wgrad1.part_stride, g.off_W2, P.S1, b.wpart2,
                             P.wgrad2.part_stride, g.off_W2, (int64_t)3 * g.C * g.C, P.S2, s, false,
                             g.prec == TEM_BF16 ? 592 : 0, 2) != cudaSuccess)  // bf16: 592 x 256 measured faster
            return TEM_ERR_CUDA;
        ++*nl;
        c->grad_lazy = true;
        rec.end(SLOT_EXCHANGE);
        return opt_scalars(c, s, nl);
    }
    if (c->N == 1) {
        for (int l = 0; l < c->nlocal; ++l) {
            if (launch_sgd_single(c->rb[l].grad, (float*)c->rb[l].params, shadow_hi(c->rb[l], wr),
                                  shadow_lo(c->rb[l], wr), g.Kpad, TEM_MEAN, oc, opt_state(c, l), s) != cudaSuccess)
                return TEM_ERR_CUDA;
            ++*nl;
        }
        rec.end(SLOT_EXCHANGE);
        return opt_scalars(c, s, nl);
    }
    if (bucketed(c)) {  // reading R25: [bnd, K_pad) (unless it ran in the compute), then [0, bnd)
        const int64_t bnd = bucket_bound(c);
        if (!c->early_done) {
            if (launch_step_ring(c, step_ring(c, bnd, g.Kpad), s) != cudaSuccess) return TEM_ERR_CUDA;
            ++*nl;
        }
        c->early_done = false;
        if (launch_step_ring(c, step_ring(c, 0, bnd), s) != cudaSuccess) return TEM_ERR_CUDA;
        ++*nl;
        rec.end(SLOT_EXCHANGE);
        return opt_scalars(c, s, nl);
    }
    RingParams p;
    memset(&p, 0, sizeof(p));
    for (int l = 0; l < c->nlocal; ++l)
        p.loc[l] = ring_local(c, l, c->rb[l].grad, (float*)c->rb[l].params, shadow_hi(c->rb[l], wr),
                              shadow_lo(c->rb[l], wr));
    p.N = c->N;
    p.rank_base = c->rank;
    p.nlocal = c->nlocal;
    p.G = c->G;
    p.op = TEM_MEAN;
    p.mode = 1;
    p.K = g.Kpad;
    p.Kpad = g.Kpad;
    p.oc = oc;
    p.off_dst = 0;
    set_heap_offsets(c, &p);
    if (c->cfg.exchange == TEM_EXCHANGE_PS) {  // comparator: push / server update / pull
        PsParams q;
        memset(&q, 0, sizeof(q));
        for (int l = 0; l < c->nlocal; ++l) q.loc[l] = p.loc[l];
        q.N = c->N;
        q.rank_base = c->rank;
        q.nlocal = c->nlocal;
        q.G = c->G;
        q.op = TEM_MEAN;
        q.mode = 1;
        q.oc = oc;
        q.K = g.Kpad;
        q.off_dst = 0;
        q.off_slots = (int64_t)c->hl.off_ps;
        q.off_flags = (int64_t)c->hl.off_psflags;
        q.off_hdr = (int64_t)c->hl.off_hdr;
        q.status = c->st_dev;
        q.spin_ns = c->spin_ns;
        if (launch_ps(q, s) != cudaSuccess) return TEM_ERR_CUDA;
    } else if (c->cfg.exchange == TEM_EXCHANGE_TWOSHOT) {  // NVSwitch two-shot (NEXT #3(i))
        if (launch_twoshot(p, s) != cudaSuccess) return TEM_ERR_CUDA;
    } else if (launch_ring(p, s) != cudaSuccess) {
        return TEM_ERR_CUDA;
    }
    rec.end(SLOT_EXCHANGE);
    ++*nl;
    return opt_scalars(c, s, nl);
}

tem_status tem_compute(tem_ctx* c, const void* x, const float* labels, float* loss_out, void* stream) {
    tem_status st = check_ctx(c);
    if (st != TEM_OK) return st;
    if (c->g.pem_P > 0 && !c->pem_bsp) return TEM_ERR_INVALID_ARG;  // PEM config: tem_compute_pem
    if ((!x || !labels) && c->g.B > 0) return TEM_ERR_INVALID_ARG;
    if (!loss_out) return TEM_ERR_INVALID_ARG;
    int nl = 0;
    st = compute_impl(c, x, labels, loss_out, (cudaStream_t)stream, &nl);
    return st;
}

tem_status tem_exchange(tem_ctx* c, void* stream) {
    tem_status st = check_ctx(c);
    if (st != TEM_OK) return st;
    int nl = 0;
    st = exchange_impl(c, (cudaStream_t)stream, &nl);
    c->launches_exchange = nl;
    if (st == TEM_OK) c->wpar ^= 1;  // the update wrote the other operand set
    return st;
}

tem_status tem_step(tem_ctx* c, const void* x, const float* labels, float* loss_out, void* stream) {
    tem_status st = check_ctx(c);
    if (st != TEM_OK) return st;
    if (c->g.pem_P > 0 && !c->pem_bsp) return TEM_ERR_INVALID_ARG;  // PEM config: tem_step_pem
    if ((!x || !labels) && c->g.B > 0) return TEM_ERR_INVALID_ARG;
    if (!loss_out) return TEM_ERR_INVALID_ARG;
    if (c->use_graphs && !c->tev) {  // one graph per pointer set and operand-set parity
        st = graph_step(c, x, labels, loss_out, (cudaStream_t)stream, [&](cudaStream_t gs, int* n) {
            int a = 0, b = 0;
            tem_status r = compute_impl(c, x, labels, loss_out, gs, &a, true);
            if (r == TEM_OK) r = exchange_impl(c, gs, &b);
            *n = a + b;
            c->launches_exchange = b;
            return r;
        });
        if (st == TEM_OK) c->wpar ^= 1;
        return st;
    }
    int nl = 0;
    st = compute_impl(c, x, labels, loss_out, (cudaStream_t)stream, &nl, true);
    if (st != TEM_OK) return st;
    int ne = 0;
    st = exchange_impl(c, (cudaStream_t)stream, &ne);
    c->launches_step = nl + ne;
    c->launches_exchange = ne;
    if (c->tev && c->t_idx < c->t_max) ++c->t_idx;
    if (st == TEM_OK) c->wpar ^= 1;
    return st;
}

// Joint TEM + PEM (configs[4]): the PEM inputs ride along in the ctx for this call only.
static bool pem_args_ok(tem_ctx* c, const float* bsp, const float* iou) {
    return c->g.pem_P > 0 && c->g.pgm_G == 0 && ((bsp && iou) || c->g.B == 0);
}

static bool pgm_args_ok(tem_ctx* c, const float* gt, const int32_t* n_gt) {
    return c->g.pgm_G > 0 && ((gt && n_gt) || c->g.B == 0);
}

tem_status tem_step_pgm(tem_ctx* c, const void* x, const float* labels, const float* gt, const int32_t* n_gt,
                        float* loss_out, void* stream) {
    tem_status st = check_ctx(c);
    if (st != TEM_OK) return st;
    if (!pgm_args_ok(c, gt, n_gt)) return TEM_ERR_INVALID_ARG;
    static const float kDummy = 0.f;
    c->pem_bsp = &kDummy;  // marks a PEM call
    c->pgm_gt = gt;
    c->pgm_ngt = n_gt;
    st = tem_step(c, x, labels, loss_out, stream);
    c->pem_bsp = nullptr;
    c->pgm_gt = nullptr;
    c->pgm_ngt = nullptr;
    return st;
}

tem_status tem_compute_pgm(tem_ctx* c, const void* x, const float* labels, const float* gt, const int32_t* n_gt,
                           float* loss_out, void* stream) {
    tem_status st = check_ctx(c);
    if (st != TEM_OK) return st;
    if (!pgm_args_ok(c, gt, n_gt)) return TEM_ERR_INVALID_ARG;
    static const float kDummy = 0.f;
    c->pem_bsp = &kDummy;
    c->pgm_gt = gt;
    c->pgm_ngt = n_gt;
    st = tem_compute(c, x, labels, loss_out, stream);
    c->pem_bsp = nullptr;
    c->pgm_gt = nullptr;
    c->pgm_ngt = nullptr;
    return st;
}

tem_status tem_step_pem(tem_ctx* c, const void* x, const float* labels, const float* bsp, const float* iou,
                        float* loss_out, void* stream) {
    tem_status st = check_ctx(c);
    if (st != TEM_OK) return st;
    if (!pem_args_ok(c, bsp, iou)) return TEM_ERR_INVALID_ARG;
    static const float kDummy = 0.f;
    c->pem_bsp = bsp ? bsp : &kDummy;  // non-null marks a PEM call (B = 0: no PEM inputs read)
    c->pem_iou = iou;
    st = tem_step(c, x, labels, loss_out, stream);
    c->pem_bsp = c->pem_iou = nullptr;
    return st;
}

tem_status tem_compute_pem(tem_ctx* c, const void* x, const float* labels, const float* bsp, const float* iou,
                           float* loss_out, void* stream) {
    tem_status st = check_ctx(c);
    if (st != TEM_OK) return st;
    if (!pem_args_ok(c, bsp, iou)) return TEM_ERR_INVALID_ARG;
    static const float kDummy = 0.f;
    c->pem_bsp = bsp ? bsp : &kDummy;
    c->pem_iou = iou;
    st = tem_compute(c, x, labels, loss_out, stream);
    c->pem_bsp = c->pem_iou = nullptr;
    return st;
}

tem_status tem_pem_relu_decisions(tem_ctx* c, int32_t l, uint8_t* out, void* stream) {
    if (!c || !c->alive) return TEM_ERR_STATE;
    if (c->g.pem_P <= 0 || l < 0 || l >= c->nlocal) return TEM_ERR_INVALID_ARG;
    if (!out) {  // start recording for the following steps (recording changes no result)
        c->pem_record_dec = true;
        for (int i = 0; i < c->ngraphs; ++i) cudaGraphExecDestroy(c->graphs[i].exec);
        c->ngraphs = 0;
        return TEM_OK;
    }
    if (!c->pem_record_dec) return TEM_ERR_STATE;
    const size_t n = (size_t)c->g.B * c->g.pem_P * c->g.pem_H;
    return n == 0 || cudaMemcpyAsync(out, c->rb[l].pemdec, n, cudaMemcpyDeviceToDevice, (cudaStream_t)stream) ==
                         cudaSuccess
               ? TEM_OK
               : TEM_ERR_CUDA;
}

// Host-input pipeline shared by tem_step_host / tem_step_pem_host: this call's inputs are
// copied on a private copy stream into staging set `hslot`, which the step on `s` waits for;
// the set is reused two calls later, once the step that consumed it is done.  A caller that
// issues steps back to back therefore overlaps the copy of step k+1 with the compute of step k.
static tem_status host_stage(tem_ctx* c, cudaStream_t s, const void* x_host, const float* labels_host,
                             const void* bsp_host, size_t bb, const void* iou_host, size_t ib, int* slot, void** xd,
                             float** ld, float** bd, float** id) {
    const Geom& g = c->g;
    if (!c->cstream) {
        if (cudaStreamCreateWithFlags(&c->cstream, cudaStreamNonBlocking) != cudaSuccess) return TEM_ERR_CUDA;
        for (int i = 0; i < 2; ++i)
            if (cudaEventCreateWithFlags(&c->ev_copied[i], cudaEventDisableTiming) != cudaSuccess ||
                cudaEventCreateWithFlags(&c->ev_consumed[i], cudaEventDisableTiming) != cudaSuccess)
                return TEM_ERR_CUDA;
    }
    const int i = c->hslot;
    c->hslot ^= 1;
    *slot = i;
    const size_t esz = g.prec == TEM_BF16 ? 2 : 4;
    const size_t xb = (size_t)g.B * g.T * g.Cin * esz, lb = (size_t)g.B * 3 * g.T * 4;
    // the extra inputs' staging sets hold [B][P][F] / [B][P] floats (>= PGM's gt / counts)
    const size_t bcap = (size_t)g.B * g.pem_P * g.pem_F * 4, icap = (size_t)g.B * g.pem_P * 4;
    if (bb > bcap || ib > icap) return TEM_ERR_INVALID_ARG;
    char* base = c->ws_base[0];
    *xd = base + c->wl.xstage + i * xb;
    *ld = (float*)(base + c->wl.labstage + i * lb);
    *bd = (float*)(base + c->wl.bspstage + i * bcap);
    *id = (float*)(base + c->wl.ioustage + i * icap);
    cudaStream_t cs = c->cstream;
    // one copy per tensor (measured: splitting x over parallel copy streams is slower)
    if (cudaStreamWaitEvent(cs, c->ev_consumed[i], 0) != cudaSuccess) return TEM_ERR_CUDA;
    if (xb && cudaMemcpyAsync(*xd, x_host, xb, cudaMemcpyHostToDevice, cs) != cudaSuccess) return TEM_ERR_CUDA;
    if (lb && cudaMemcpyAsync(*ld, labels_host, lb, cudaMemcpyHostToDevice, cs) != cudaSuccess) return TEM_ERR_CUDA;
    if (bsp_host && bb && cudaMemcpyAsync(*bd, bsp_host, bb, cudaMemcpyHostToDevice, cs) != cudaSuccess)
        return TEM_ERR_CUDA;
    if (iou_host && ib && cudaMemcpyAsync(*id, iou_host, ib, cudaMemcpyHostToDevice, cs) != cudaSuccess)
        return TEM_ERR_CUDA;
    if (cudaEventRecord(c->ev_copied[i], cs) != cudaSuccess || cudaStreamWaitEvent(s, c->ev_copied[i], 0) != cudaSuccess)
        return TEM_ERR_CUDA;
    return TEM_OK;
}

tem_status tem_step_host(tem_ctx* c, const void* x_host, const float* labels_host, float* loss_host,
                         void* stream) {
    tem_status st = check_ctx(c);
    if (st != TEM_OK) return st;
    if (!loss_host || ((!x_host || !labels_host) && c->g.B > 0)) return TEM_ERR_INVALID_ARG;
    if (c->nlocal != 1) return TEM_ERR_INVALID_ARG;  // host path: one rank per process
    if (c->g.pem_P > 0) return TEM_ERR_INVALID_ARG;  // PEM configs: tem_step_pem_host
    cudaStream_t s = (cudaStream_t)stream;
    int slot;
    void* xd;
    float *ld, *bd, *id;
    st = host_stage(c, s, x_host, labels_host, nullptr, 0, nullptr, 0, &slot, &xd, &ld, &bd, &id);
    if (st != TEM_OK) return st;
    float* lossd = (float*)(c->ws_base[0] + c->wl.lossstage);
    c->loss_host_pending = loss_host;  // the tcgen05 path reads the loss back inside the step
    c->loss_host_done = false;
    st = tem_step(c, xd, ld, lossd, stream);
    const bool done = c->loss_host_done;
    c->loss_host_pending = nullptr;
    c->loss_host_done = false;
    if (st != TEM_OK) return st;
    if (!done && cudaMemcpyAsync(loss_host, lossd, 16, cudaMemcpyDeviceToHost, s) != cudaSuccess) return TEM_ERR_CUDA;
    if (cudaEventRecord(c->ev_consumed[slot], s) != cudaSuccess) return TEM_ERR_CUDA;
    return TEM_OK;
}

tem_status tem_step_pem_host(tem_ctx* c, const void* x_host, const float* labels_host, const float* bsp_host,
                             const float* iou_host, float* loss_host, void* stream) {
    tem_status st = check_ctx(c);
    if (st != TEM_OK) return st;
    if (!loss_host || ((!x_host || !labels_host || !bsp_host || !iou_host) && c->g.B > 0)) return TEM_ERR_INVALID_ARG;
    if (c->nlocal != 1 || c->g.pem_P <= 0) return TEM_ERR_INVALID_ARG;
    cudaStream_t s = (cudaStream_t)stream;
    int slot;
    void* xd;
    float *ld, *bd, *id;
    const Geom& g = c->g;
    const bool pgm = g.pgm_G > 0;  // PGM-fed: the extra inputs are the instances and their counts
    const size_t bb = pgm ? (size_t)g.B * g.pgm_G * 2 * 4 : (size_t)g.B * g.pem_P * g.pem_F * 4;
    const size_t ib = pgm ? (size_t)g.B * 4 : (size_t)g.B * g.pem_P * 4;
    st = host_stage(c, s, x_host, labels_host, bsp_host, bb, iou_host, ib, &slot, &xd, &ld, &bd, &id);
    if (st != TEM_OK) return st;
    float* lossd = (float*)(c->ws_base[0] + c->wl.lossstage);
    st = pgm ? tem_step_pgm(c, xd, ld, bd, (const int32_t*)id, lossd, stream) : tem_step_pem(c, xd, ld, bd, id, lossd, stream);
    if (st != TEM_OK) return st;
    // [4 TEM | 1 PEM] floats, after the step
    if (cudaMemcpyAsync(loss_host, lossd, 5 * sizeof(float), cudaMemcpyDeviceToHost, s) != cudaSuccess ||
        cudaEventRecord(c->ev_consumed[slot], s) != cudaSuccess)
        return TEM_ERR_CUDA;
    return TEM_OK;
}

tem_status ring_allreduce(tem_ctx* c, float* buf, int64_t K, int32_t op, void* stream) {
    tem_status st = check_ctx(c);
    if (st != TEM_OK) return st;
    if (op != TEM_SUM && op != TEM_MEAN) return TEM_ERR_INVALID_ARG;
    if (K < 1 || K > max_ar(&c->cfg)) return TEM_ERR_INVALID_ARG;
    if ((char*)buf != (char*)c->peers[c->rank] + c->hl.off_user) return TEM_ERR_INVALID_ARG;
    RingParams p;
    memset(&p, 0, sizeof(p));
    for (int l = 0; l < c->nlocal; ++l) {
        float* ub = (float*)((char*)c->peers[c->rank + l] + c->hl.off_user);
        p.loc[l] = ring_local(c, l, ub, ub, nullptr, nullptr);
    }
    p.N = c->N;
    p.rank_base = c->rank;
    p.nlocal = c->nlocal;
    p.Kpad = roundup(K, 4 * (int64_t)c->N);
    p.G = c->G;
    p.op = op;
    p.mode = 0;
    p.K = K;
    p.off_dst = (int64_t)c->hl.off_user;
    set_heap_offsets(c, &p);
    if (launch_ring(p, (cudaStream_t)stream) != cudaSuccess) return TEM_ERR_CUDA;
    return TEM_OK;
}

tem_status twoshot_allreduce(tem_ctx* c, float* buf, int64_t K, int32_t op, void* stream) {
    tem_status st = check_ctx(c);
    if (st != TEM_OK) return st;
    if (op != TEM_SUM && op != TEM_MEAN) return TEM_ERR_INVALID_ARG;
    if (K < 1 || K > max_ar(&c->cfg)) return TEM_ERR_INVALID_ARG;
    if ((char*)buf != (char*)c->peers[c->rank] + c->hl.off_user) return TEM_ERR_INVALID_ARG;
    RingParams p;
    memset(&p, 0, sizeof(p));
    for (int l = 0; l < c->nlocal; ++l) {
        float* ub = (float*)((char*)c->peers[c->rank + l] + c->hl.off_user);
        p.loc[l] = ring_local(c, l, ub, ub, nullptr, nullptr);
    }
    p.N = c->N;
    p.rank_base = c->rank;
    p.nlocal = c->nlocal;
    p.Kpad = roundup(K, 4 * (int64_t)c->N);
    p.G = c->G;
    p.op = op;
    p.mode = 0;
    p.K = K;
    p.off_dst = (int64_t)c->hl.off_user;
    set_heap_offsets(c, &p);
    p.off_stage = -1;  // in place: the user region is the readable source
    p.off_src = (int64_t)c->hl.off_user;
    if (launch_twoshot(p, (cudaStream_t)stream) != cudaSuccess) return TEM_ERR_CUDA;
    return TEM_OK;
}

tem_status ps_allreduce(tem_ctx* c, float* buf, int64_t K, int32_t op, void* stream) {
    tem_status st = check_ctx(c);
    if (st != TEM_OK) return st;
    if (op != TEM_SUM && op != TEM_MEAN) return TEM_ERR_INVALID_ARG;
    if (K < 1 || K > max_ar(&c->cfg)) return TEM_ERR_INVALID_ARG;
    if ((char*)buf != (char*)c->peers[c->rank] + c->hl.off_user) return TEM_ERR_INVALID_ARG;
    PsParams p;
    memset(&p, 0, sizeof(p));
    for (int l = 0; l < c->nlocal; ++l) {
        float* ub = (float*)((char*)c->peers[c->rank + l] + c->hl.off_user);
        p.loc[l] = ring_local(c, l, ub, ub, nullptr, nullptr);
    }
    p.N = c->N;
    p.rank_base = c->rank;
    p.nlocal = c->nlocal;
    p.G = c->G;
    p.op = op;
    p.K = K;
    p.off_dst = (int64_t)c->hl.off_user;
    p.off_slots = (int64_t)c->hl.off_ps;
    p.off_flags = (int64_t)c->hl.off_psflags;
    p.off_hdr = (int64_t)c->hl.off_hdr;
    p.status = c->st_dev;
    p.spin_ns = c->spin_ns;
    if (launch_ps(p, (cudaStream_t)stream) != cudaSuccess) return TEM_ERR_CUDA;
    return TEM_OK;
}

tem_status tem_sync(tem_ctx* c, void* stream, int64_t* bad_step) {
    if (!c || !c->alive) return TEM_ERR_STATE;
    if (cudaStreamSynchronize((cudaStream_t)stream) != cudaSuccess) return TEM_ERR_CUDA;
    const int32_t code = *(volatile int32_t*)&c->st_host->code;
    if (bad_step) *bad_step = *(volatile int64_t*)&c->st_host->step;
    return (tem_status)code;
}

tem_status tem_shutdown(tem_ctx* c) {
    if (!c) return TEM_OK;
    if (!c->alive) return TEM_ERR_STATE;
    tem_status st = TEM_OK;
    if (cudaSetDevice(c->cfg.device) != cudaSuccess || cudaDeviceSynchronize() != cudaSuccess)
        st = TEM_ERR_CUDA;
    const int32_t code = *(volatile int32_t*)&c->st_host->code;
    if (st == TEM_OK && code != 0) st = (tem_status)code;
    cudaFreeHost(c->st_host);
    for (int l = 0; l < c->nlocal; ++l) umma_plan_destroy(c->plan[l]);
    for (int i = 0; i < c->ngraphs; ++i) cudaGraphExecDestroy(c->graphs[i].exec);
    if (c->cstream) {
        cudaStreamDestroy(c->cstream);
        for (int i = 0; i < 2; ++i) {
            cudaEventDestroy(c->ev_copied[i]);
            cudaEventDestroy(c->ev_consumed[i]);
        }
    }
    if (c->gstream) {
        cudaStreamDestroy(c->gstream);
        cudaEventDestroy(c->ev_in);
        cudaEventDestroy(c->ev_out);
    }
    if (c->tev) {
        for (size_t i = 0; i < (size_t)c->t_max * NUM_SLOTS * 2; ++i) cudaEventDestroy(c->tev[i]);
        delete[] c->tev;
    }
    c->alive = false;
    delete c;
    return st;
}

float* tem_local_grad(tem_ctx* c, int32_t l) {
    if (!c || !c->alive || l < 0 || l >= c->nlocal) return nullptr;
    if (c->grad_lazy && l == 0) {  // sum the split-K partials of the last N = 1 tem_step into grad
        const Geom& g = c->g;
        const RankBufs& b = c->rb[0];
        const UmmaPlan& P = *c->plan[0];
        if (launch_sgd_fused(b.grad, nullptr, nullptr, nullptr, 0, g.Kpad, opt_cfg(c), opt_state(c, 0), b.wpart,
                             P.wgrad1.part_stride, g.off_W2, P.S1, b.wpart2, P.wgrad2.part_stride, g.off_W2,
                             (int64_t)3 * g.C * g.C, P.S2, 0, false, 0, 0) != cudaSuccess ||
            cudaStreamSynchronize(0) != cudaSuccess)
            return nullptr;
        c->grad_lazy = false;
    }
    return c->rb[l].grad;
}

float* tem_logits(tem_ctx* c, int32_t l) {
    if (!c || !c->alive || l < 0 || l >= c->nlocal) return nullptr;
    return c->rb[l].z;
}

void* tem_debug_buffer(tem_ctx* c, int32_t l, const char* name, int64_t* nbytes) {
    if (nbytes) *nbytes = 0;
    if (!c || !c->alive || l < 0 || l >= c->nlocal || !name) return nullptr;
#ifdef TEM_DIAG
    if (strcmp(name, "trace_on") == 0 || strcmp(name, "trace_off") == 0 || strcmp(name, "trace") == 0) {
        // diagnostics build only: [NUM_SLOTS][2] kernel spans + [4096][8] head phase stamps (ns)
        // in the trace area at the end of the caller's workspace (tem_workspace_bytes reserves it)
        unsigned long long* buf = (unsigned long long*)(c->ws_base[0] + c->wl.trace);
        if (strcmp(name, "trace") != 0) {
            unsigned long long* p = strcmp(name, "trace_on") == 0 ? buf : nullptr;
            trace_set_umma(p);
            trace_set_head(p);
            trace_set_ring(p);
            trace_set_pem(p);
        }
        if (nbytes) *nbytes = (int64_t)(sizeof(unsigned long long) * kTraceWords);
        return buf;
    }
#endif
    if (strcmp(name, "tstamp_on") == 0 || strcmp(name, "tstamp") == 0)
        return umma_tstamp_buffer(nbytes, strcmp(name, "tstamp_on") == 0 ? 1 : 0);
#ifdef TEM_DIAG
    if (strcmp(name, "tclk") == 0) return umma_tclk_buffer(nbytes);
    if (strncmp(name, "probe_skip:", 11) == 0) {  // diagnostics: skip FWD/DGRAD operand loads
        umma_set_probe_skip(atoi(name + 11));
        return nullptr;
    }
#endif
    if (strncmp(name, "tstamp_slot:", 12) == 0)  // stamps of one launch: "tstamp_slot:<Slot>"
        return umma_tstamp_buffer(nbytes, 100 + atoi(name + 12));
    const Geom& g = c->g;
    const RankBufs& b = c->rb[l];
    const int64_t esz = 2;
    const int64_t act = (int64_t)g.R * g.C * esz, xin = (int64_t)g.R * g.Cin * esz;
    struct Item { const char* n; const void* p; int64_t bytes; };
    const Item items[] = {
        {"xp", b.xp, xin}, {"h1", b.h1, act}, {"h2", b.h2, (int64_t)g.R * g.C * 4}, {"dA2", b.dA2, act},
        {"dA1", b.dA1, act}, {"xp_lo", b.xp_lo, xin}, {"h1_lo", b.h1_lo, act}, {"dA2_lo", b.dA2_lo, act},
        {"dA1_lo", b.dA1_lo, act}, {"shadow", shadow_hi(b, c->wpar), g.Kpad * 2},
        {"shadow_lo", shadow_lo(b, c->wpar), g.Kpad * 2},
        {"pgm_prob", c->ws_base[l] + c->wl.pgm_prob, g.pgm_G > 0 ? (int64_t)g.B * 3 * g.T * 4 : 0},
        {"pgm_feat", c->ws_base[l] + c->wl.pgm_feat, g.pgm_G > 0 ? (int64_t)g.B * g.pem_P * 32 * 4 : 0},
        {"pgm_iou", c->ws_base[l] + c->wl.pgm_iou, g.pgm_G > 0 ? (int64_t)g.B * g.pem_P * 4 : 0},
        {"pgm_ts", c->ws_base[l] + c->wl.pgm_ts, g.pgm_G > 0 ? (int64_t)g.B * g.pem_P * 4 : 0},
        {"pgm_te", c->ws_base[l] + c->wl.pgm_te, g.pgm_G > 0 ? (int64_t)g.B * g.pem_P * 4 : 0},
        {"pgm_count", c->ws_base[l] + c->wl.pgm_count, g.pgm_G > 0 ? (int64_t)g.B * 4 : 0},
        {"bwd_tasks", b.bwd.tasks, (int64_t)1024 * BWD_MAX_TASKS * 4}};
    for (const Item& it : items)
        if (strcmp(it.n, name) == 0) {
            if (!it.p) return nullptr;
            if (nbytes) *nbytes = it.bytes;
            return const_cast<void*>(it.p);
        }
    return nullptr;
}

tem_status tem_relu_decisions(tem_ctx* c, int32_t l, uint8_t* out, void* stream) {
    if (!c || !c->alive) return TEM_ERR_STATE;
    if (l < 0 || l >= c->nlocal || (!out && c->g.B > 0)) return TEM_ERR_INVALID_ARG;
    if (c->g.B == 0) return TEM_OK;
    return launch_relu_decisions(c->g, c->rb[l], out, (cudaStream_t)stream) == cudaSuccess ? TEM_OK
                                                                                           : TEM_ERR_CUDA;
}

int32_t tem_timing_slots(tem_ctx* c) { return c ? NUM_SLOTS : 0; }

const char* tem_timing_slot_name(tem_ctx* c, int32_t slot) { return c ? slot_name(slot) : "?"; }

tem_status tem_timing_begin(tem_ctx* c, int32_t max_steps) {
    if (!c || !c->alive) return TEM_ERR_STATE;
    if (max_steps < 1 || c->nlocal != 1 || c->tev) return TEM_ERR_INVALID_ARG;
    const size_t n = (size_t)max_steps * NUM_SLOTS * 2;
    c->tev = new (std::nothrow) cudaEvent_t[n];
    if (!c->tev) return TEM_ERR_CUDA;
    for (size_t i = 0; i < n; ++i)
        if (cudaEventCreate(&c->tev[i]) != cudaSuccess) return TEM_ERR_CUDA;
    c->t_max = max_steps;
    c->t_idx = 0;
    return TEM_OK;
}

tem_status tem_timing_end(tem_ctx* c, float* sum_ms, int32_t* steps) {
    if (!c || !c->alive) return TEM_ERR_STATE;
    if (!c->tev) return TEM_ERR_INVALID_ARG;
    tem_status st = TEM_OK;
    for (int k = 0; k < NUM_SLOTS; ++k) sum_ms[k] = 0.f;
    for (int i = 0; i < c->t_idx; ++i)
        for (int k = 0; k < NUM_SLOTS; ++k) {
            cudaEvent_t a = c->tev[((size_t)i * NUM_SLOTS + k) * 2], b = c->tev[((size_t)i * NUM_SLOTS + k) * 2 + 1];
            if (cudaEventSynchronize(b) != cudaSuccess) { st = TEM_ERR_CUDA; continue; }
            float ms = 0.f;
            if (cudaEventElapsedTime(&ms, a, b) == cudaSuccess) sum_ms[k] += ms;
            // slots never recorded this step (e.g. head with B = 0) report "not ready": skip
            cudaGetLastError();
        }
    if (steps) *steps = c->t_idx;
    const size_t n = (size_t)c->t_max * NUM_SLOTS * 2;
    for (size_t i = 0; i < n; ++i) cudaEventDestroy(c->tev[i]);
    delete[] c->tev;
    c->tev = nullptr;
    c->t_max = c->t_idx = 0;
    return st;
}

int32_t tem_launches_per_step(tem_ctx* c) { return c ? c->launches_step : 0; }
int32_t tem_launches_per_exchange(tem_ctx* c) { return c ? c->launches_exchange : 0; }

const char* tem_kernel_path(tem_ctx* c) {
    if (!c) return "none";
    return c->g.prec == TEM_BF16 ? "tcgen05-bf16" : "tcgen05-bf16x3-fp32";
}

}  // extern "C"
