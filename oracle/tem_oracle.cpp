// ============================================================================
// tem_oracle.cpp -- the CPU ORACLE for the data-parallel BSN-TEM step and the
// ring allreduce of arXiv 1906.06496.
//
// TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and the
// cpu_baseline / --impl reference legs of bench.py may load this library.
// The product path (paper_1906_06496_b200/) never imports, links or executes
// anything under oracle/, and this file shares no code, header, table or
// helper with paper_1906_06496_b200/csrc/.
//
// Plain, slow, obviously correct.  Built with
//   g++ -O2 -std=c++17 -ffp-contract=off -fno-fast-math -shared -fPIC
// so that every fp32 add/mul/fma below rounds exactly once, in the order
// written (no contraction, no reassociation, no FTZ/DAZ).
//
// Citations: "P:n" = /root/reference/PAPER.md line n (section / equation);
// "S:n" = SPEC.md line n; "SURVEY 8(x)" = /root/repo/SURVEY.md section 8 row.
// Readings where the paper is silent are listed in DESIGN.md section 3.
//
// Pins (tests/test_oracle_*.py) -- nothing below is "parity unpinned":
//   schedules      : P:135 instantiation, exhaustive completion N=2..16
//   ring sum       : integer-exact inputs vs brute force; one-hot N=3;
//                    hand-derived order witness; recursive-summation error bound
//   volume         : 2 K_pad (N-1)/N elements sent per rank
//   mean / SGD     : lr = 0 identity; power-of-two N exactness; fused == unfused
//   TEM forward    : torch.nn.functional.conv1d float64 (library routine)
//   TEM loss       : closed form 2 ln 2 per channel at z == 0
//   TEM backward   : central finite differences + torch.autograd float64
//   DP equivalence : N ranks x B (mean) == 1 rank x N*B
//   PEM            : torch.autograd float64 (library routine); closed form at W1 = 0;
//                    central finite differences (tests/test_oracle_pem.py)
// ============================================================================
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <vector>

extern "C" {

// ---------------------------------------------------------------------------
// Block partition ("divide weights in every GPU into
// N parts").  Reading R9: K is zero-padded to K_pad = roundup(K, N*V) with
// V = 4 fp32 elements (one 16-byte vector) so that the N blocks are equal and
// every block starts 16-byte aligned.  Block b = [b*K_pad/N, (b+1)*K_pad/N).
// ---------------------------------------------------------------------------
int64_t orc_kpad(int64_t K, int N, int V) {
    if (K < 0 || N < 1 || V < 1) return -1;
    const int64_t q = (int64_t)N * V;
    return ((K + q - 1) / q) * q;
}

static int mod_nonneg(int a, int n) { int r = a % n; return r < 0 ? r + n : r; }

// "The n-th GPU passes its own (n-i)%N-th block ... to its right
// neighbor and receives (n-i-1)%N-th block ... from its left neighbor, where i
// is the round of scatter."  Rounds i = 0..N-2 (0-based; the only origin under
// which P:143's owner (n+1)%N follows).  Non-negative residue.
int orc_scatter_schedule(int rank, int N, int round, int* send_blk, int* recv_blk) {
    if (N < 2 || rank < 0 || rank >= N || round < 0 || round > N - 2) return 1;
    *send_blk = mod_nonneg(rank - round, N);
    *recv_blk = mod_nonneg(rank - round - 1, N);
    return 0;
}

// P:151-152 gather.  The printed indices (n-i-1)%N / (n-i-2)%N do not complete
// for N >= 4 with i starting at 0 or 1.  Reading R10:
// round k = 0..N-2, send (n+1-k)%N, receive (n-k)%N, i.e. the printed
// formula with i = k - 2 (mod N).  Round 0 sends the block completed in the
// scatter, (n+1)%N.  Received blocks REPLACE.
int orc_gather_schedule(int rank, int N, int round, int* send_blk, int* recv_blk) {
    if (N < 2 || rank < 0 || rank >= N || round < 0 || round > N - 2) return 1;
    *send_blk = mod_nonneg(rank + 1 - round, N);
    *recv_blk = mod_nonneg(rank - round, N);
    return 0;
}

// ---------------------------------------------------------------------------
// Ring allreduce replay, fp32, round by round.
//   bufs      : N rank buffers of K_pad floats each, rank-major, IN PLACE.
//   op        : 0 = Sum, 1 = Mean (mean applied once, on the owner,
//               after the scatter, as s * fl(1/N) -- reading R11).
//   params    : NULL for a plain allreduce.  Otherwise N rank parameter
//               buffers (K_pad each, identical on entry): the owner of each
//               block applies SGD  w = fma(-lr, gbar, w)  ("upgrade
//               parameters"; reading R12) and the GATHER then carries the
//               updated weights instead of the gradient; bufs then hold, on
//               every rank, the reduced (op-applied) gradient of the blocks the
//               rank owns only -- use orc_ring_allreduce_f32 for gradients.
//   sent      : optional [N] counters of elements sent per rank.
// Every message is a copy of a whole block taken at the start of the round
// (all ranks send simultaneously, then all receive), as in P:135 / P:152.
// ---------------------------------------------------------------------------
static int ring_replay(float* bufs, float* params, int N, int64_t K_pad, int op, float lr,
                       int64_t* sent) {
    if (N < 1 || K_pad < 0 || K_pad % N != 0 || (op != 0 && op != 1)) return 1;
    const int64_t Bk = K_pad / N;
    if (sent) for (int r = 0; r < N; ++r) sent[r] = 0;
    const float inv_n = 1.0f / (float)N;
    if (N == 1) {  // identity collective; mean multiplies by fl(1/1) = 1
        for (int64_t e = 0; e < K_pad; ++e) {
            float g = bufs[e];
            if (op == 1) g = g * inv_n;
            bufs[e] = g;
            if (params) params[e] = std::fma(-lr, g, params[e]);
        }
        return 0;
    }
    std::vector<float> msg((size_t)N * Bk);
    // --- scatter (reduce) rounds i = 0..N-2 ---
    for (int i = 0; i <= N - 2; ++i) {
        for (int n = 0; n < N; ++n) {  // everybody sends first
            int s, rcv;
            orc_scatter_schedule(n, N, i, &s, &rcv);
            std::memcpy(&msg[(size_t)n * Bk], bufs + (size_t)n * K_pad + (size_t)s * Bk,
                        sizeof(float) * Bk);
            if (sent) sent[n] += Bk;
        }
        for (int n = 0; n < N; ++n) {  // ... then receives from the left and ADDS
            int s, rcv;
            orc_scatter_schedule(n, N, i, &s, &rcv);
            const int left = mod_nonneg(n - 1, N);
            float* own = bufs + (size_t)n * K_pad + (size_t)rcv * Bk;
            const float* in = &msg[(size_t)left * Bk];
            for (int64_t e = 0; e < Bk; ++e) own[e] = own[e] + in[e];
        }
    }
    // --- owner: mean once + (optionally) SGD on block (n+1)%N ---
    for (int n = 0; n < N; ++n) {
        const int b = mod_nonneg(n + 1, N);
        float* own = bufs + (size_t)n * K_pad + (size_t)b * Bk;
        for (int64_t e = 0; e < Bk; ++e) {
            float g = own[e];
            if (op == 1) g = g * inv_n;
            own[e] = g;
            if (params) {
                float* w = params + (size_t)n * K_pad + (size_t)b * Bk;
                w[e] = std::fma(-lr, g, w[e]);
            }
        }
    }
    // --- gather (replace) rounds k = 0..N-2 ---
    float* carry = params ? params : bufs;
    for (int k = 0; k <= N - 2; ++k) {
        for (int n = 0; n < N; ++n) {
            int s, rcv;
            orc_gather_schedule(n, N, k, &s, &rcv);
            std::memcpy(&msg[(size_t)n * Bk], carry + (size_t)n * K_pad + (size_t)s * Bk,
                        sizeof(float) * Bk);
            if (sent) sent[n] += Bk;
        }
        for (int n = 0; n < N; ++n) {
            int s, rcv;
            orc_gather_schedule(n, N, k, &s, &rcv);
            const int left = mod_nonneg(n - 1, N);
            std::memcpy(carry + (size_t)n * K_pad + (size_t)rcv * Bk, &msg[(size_t)left * Bk],
                        sizeof(float) * Bk);
        }
    }
    return 0;
}

int orc_ring_allreduce_f32(float* bufs, int N, int64_t K_pad, int op, int64_t* sent) {
    return ring_replay(bufs, nullptr, N, K_pad, op, 0.0f, sent);
}

// Ring allreduce fused with the owner's SGD update.
// grads: N x K_pad (read-only here; copied), params: N x K_pad in place.
int orc_ring_sgd_f32(const float* grads, float* params, int N, int64_t K_pad, int op, float lr) {
    std::vector<float> g(grads, grads + (size_t)N * K_pad);
    return ring_replay(g.data(), params, N, K_pad, op, lr, nullptr);
}

// Direct per-element chain form of the same result:
// block b is accumulated as (((g_b + g_{b+1}) + g_{b+2}) + ... + g_{b+N-1}),
// rank indices mod N.  out: K_pad floats (identical on every rank).
int orc_ring_chain_f32(const float* grads, int N, int64_t K_pad, int op, float* out) {
    if (N < 1 || K_pad < 0 || K_pad % N != 0 || (op != 0 && op != 1)) return 1;
    const int64_t Bk = K_pad / N;
    const float inv_n = 1.0f / (float)N;
    for (int b = 0; b < N; ++b)
        for (int64_t e = b * Bk; e < (b + 1) * Bk; ++e) {
            float s = grads[(size_t)b * K_pad + e];
            for (int j = 1; j < N; ++j) s = s + grads[(size_t)mod_nonneg(b + j, N) * K_pad + e];
            if (op == 1) s = s * inv_n;
            out[e] = s;
        }
    return 0;
}

// Ring allreduce fused with an Adam owner update (reading R22): the mean
// gradient gbar of every element comes from the ring's chain (orc_ring_chain_f32), then, in
// fp32 with every operation rounded once, in this order (t = this step, b1t = beta1^t and
// b2t = beta2^t kept as running fp32 products, updated BEFORE use: b1t *= beta1, b2t *= beta2):
//   m    = beta1 * m + (1 - beta1) * gbar          (products, then the sum)
//   v    = beta2 * v + (1 - beta2) * (gbar * gbar)
//   mhat = m / (1 - b1t),   vhat = v / (1 - b2t)
//   w    = w - lr * (mhat / (sqrt(vhat) + eps))
// (1 - beta1), (1 - beta2) are fp32 constants.  The optimizer state is sharded by ownership
// on the GPU (the owner of a block holds its m, v); here it is one array.
// scal: [b1t, b2t] in/out.  All replicas receive the same w.
int orc_ring_adam_f32(const float* grads, float* params, float* m, float* v, float* scal, int N, int64_t K_pad,
                      float lr, float beta1, float beta2, float eps) {
    std::vector<float> gbar((size_t)K_pad);
    const int rc = orc_ring_chain_f32(grads, N, K_pad, 1, gbar.data());
    if (rc) return rc;
    const float b1t = scal[0] * beta1, b2t = scal[1] * beta2;
    scal[0] = b1t;
    scal[1] = b2t;
    const float c1 = 1.0f - beta1, c2 = 1.0f - beta2;
    const float d1 = 1.0f - b1t, d2 = 1.0f - b2t;
    for (int64_t e = 0; e < K_pad; ++e) {
        const float g = gbar[(size_t)e];
        const float a1 = beta1 * m[e];
        const float a2 = c1 * g;
        m[e] = a1 + a2;
        const float gg = g * g;
        const float q1 = beta2 * v[e];
        const float q2 = c2 * gg;
        v[e] = q1 + q2;
        const float mhat = m[e] / d1;
        const float vhat = v[e] / d2;
        const float den = std::sqrt(vhat) + eps;
        const float step = mhat / den;
        const float upd = lr * step;
        params[e] = params[e] - upd;
    }
    return 0;
}

// Ring mean + SGD with heavy-ball momentum (reading R23), fp32 with
// explicit fused multiply-adds as the SGD step of R12:
//   gbar = ring chain mean (as orc_ring_chain_f32, op = mean)
//   u    = fma(mu, u, gbar)          (momentum buffer, zero before the first step)
//   w    = fma(-lr, u, w)
// mu = 0 reduces to orc_ring_sgd_f32 bit for bit.  All replicas receive the same w.
int orc_ring_momentum_f32(const float* grads, float* params, float* u, int N, int64_t K_pad, float lr, float mu) {
    std::vector<float> gbar((size_t)K_pad);
    const int rc = orc_ring_chain_f32(grads, N, K_pad, 1, gbar.data());
    if (rc) return rc;
    for (int64_t e = 0; e < K_pad; ++e) {
        u[e] = std::fma(mu, u[e], gbar[(size_t)e]);
        params[e] = std::fma(-lr, u[e], params[e]);
    }
    return 0;
}

// Parameter-server comparator ("accumulates all N buffers in
// ascending-rank order").  out = ((g_0 + g_1) + g_2) + ... ; mean once.
int orc_ps_allreduce_f32(const float* grads, int N, int64_t K, int op, float* out) {
    if (N < 1 || K < 0 || (op != 0 && op != 1)) return 1;
    const float inv_n = 1.0f / (float)N;
    for (int64_t e = 0; e < K; ++e) {
        float s = grads[e];
        for (int r = 1; r < N; ++r) s = s + grads[(size_t)r * K + e];
        if (op == 1) s = s * inv_n;
        out[e] = s;
    }
    return 0;
}

// ---------------------------------------------------------------------------
// bf16 round-to-nearest-even of an fp32 value (reading R8: the c3 path rounds
// exactly the tensor-core operands).  Bit rule: add 0x7FFF + lsb, truncate.
// ---------------------------------------------------------------------------
uint16_t orc_bf16_bits(float f) {
    uint32_t u;
    std::memcpy(&u, &f, 4);
    const uint32_t lsb = (u >> 16) & 1u;
    u += 0x7FFFu + lsb;
    return (uint16_t)(u >> 16);
}
static float bf16_to_f32(uint16_t h) {
    uint32_t u = (uint32_t)h << 16;
    float f;
    std::memcpy(&f, &u, 4);
    return f;
}
// fp64 value -> fp32 (RNE) -> bf16 (RNE): the GPU accumulates in fp32 and
// rounds the fp32 result, so the oracle rounds through fp32 too.
static double bf16_round(double v) { return (double)bf16_to_f32(orc_bf16_bits((float)v)); }

// ---------------------------------------------------------------------------
// BSN-TEM forward + loss + backward, fp64.
//   P:68 "a temporal network with 3 convolution layers"; shapes from
//   BASELINE.json north_star: conv1d Cin->C k3 ReLU, C->C k3 ReLU, C->Co k1
//   sigmoid, over T snippets.  Readings R1-R7:
//   cross-correlation, stride 1, zero "same" padding 1, biases present;
//   x [B][T][Cin]; W [Cout][k][Cin]; labels [B][Co][T]; channel o: 0 action,
//   1 start, 2 end; b_t = [g_t > 0.5]; per video and channel
//   alpha+ = T/max(l+,1), alpha- = T/max(l-,1);
//   L_o = -(1/T) sum_t [alpha+ b log p + alpha- (1-b) log(1-p)],
//   log p = -softplus(-z), log(1-p) = -softplus(z);  L = (1/B) sum_v sum_o lambda_o L_o.
//   ReLU'(0) = 0.
//
//   prec = 0 : fp64 throughout (ground truth for the fp32 path, c1/c2)
//   prec = 1 : bf16 operand emulation (c3, reading R8): x, W1, W2, h1, dA2,
//              dA1 are rounded to bf16 where they enter a convolution; every
//              sum is fp64; h2, W3, z, p, dz and all gradients unrounded.
//              Bias gradients sum the same (rounded) operand the weight
//              gradient of that layer uses.
//   params flat: [W1 (C*3*Cin), b1 (C), W2 (C*3*C), b2 (C), W3 (Co*C), b3 (Co)]
//   loss_out [1 + Co]: total, then per-channel batch means of L_o (unweighted).
//   z_out [B][T][Co] logits (may be NULL); grad_out flat, same order as params.
// ---------------------------------------------------------------------------
int64_t orc_tem_num_params(int Cin, int C, int Co) {
    return (int64_t)C * 3 * Cin + C + (int64_t)C * 3 * C + C + (int64_t)Co * C + Co;
}

static double softplus(double u) { return u > 0 ? u + std::log1p(std::exp(-u)) : std::log1p(std::exp(u)); }

// ReLU decisions (reading R7b).  The ReLU mask 1[a > 0] is a decision taken by
// floating point: when |a| is within the rounding error of the accumulation, fp32
// and fp64 may legitimately disagree.  The extended entry point therefore
//   * reports every pre-activation with |a| <= tau * S, S = |bias| + sum |w x|
//     (the magnitude the rounding error scales with; tau = kink_tau for a1, kink_tau2
//     for a2: the layers' rounding bands differ on the bf16 path), as index
//     layer*(B*T*C) + (b*T + t)*C + c  (layer 0 = a1, 1 = a2), and
//   * accepts a sorted list `flips` of such indices whose decision is inverted.
// With no flips it is exactly the plain definition.
int orc_tem_fwd_bwd_ex(int prec, int B, int T, int Cin, int C, int Co,
                       const double* x, const double* params, const double* labels,
                       const double* lambda, double* loss_out, double* z_out, double* grad_out,
                       const int64_t* flips, int64_t nflips, double kink_tau, double kink_tau2,
                       int64_t* kinks_out, int64_t kinks_cap, int64_t* nkinks,
                       uint8_t* decisions_out) {
    if (B < 0 || T < 1 || Cin < 1 || C < 1 || Co < 1 || (prec != 0 && prec != 1)) return 1;
    if (nkinks) *nkinks = 0;
    const int64_t layer_stride = (int64_t)B * T * C;
    auto flipped = [&](int64_t idx) {
        return nflips > 0 && std::binary_search(flips, flips + nflips, idx);
    };
    auto note_kink = [&](int64_t idx, double a, double S) {
        const double tau = idx < layer_stride ? kink_tau : kink_tau2;
        if (tau > 0 && std::fabs(a) <= tau * S && nkinks) {
            if (*nkinks < kinks_cap && kinks_out) kinks_out[*nkinks] = idx;
            ++*nkinks;
        }
    };
    const int K3 = 3;
    const double* W1 = params;
    const double* b1 = W1 + (size_t)C * K3 * Cin;
    const double* W2 = b1 + C;
    const double* b2 = W2 + (size_t)C * K3 * C;
    const double* W3 = b2 + C;
    const double* b3 = W3 + (size_t)Co * C;
    double* dW1 = grad_out;
    double* db1 = dW1 + (size_t)C * K3 * Cin;
    double* dW2 = db1 + C;
    double* db2 = dW2 + (size_t)C * K3 * C;
    double* dW3 = db2 + C;
    double* db3 = dW3 + (size_t)Co * C;
    const int64_t K = orc_tem_num_params(Cin, C, Co);
    for (int64_t e = 0; e < K; ++e) grad_out[e] = 0.0;
    for (int o = 0; o <= Co; ++o) loss_out[o] = 0.0;
    if (B == 0) return 0;

    auto op = [&](double v) { return prec == 1 ? bf16_round(v) : v; };  // operand rounding
    const size_t BT = (size_t)B * T;
    std::vector<double> xq(BT * Cin), W1q((size_t)C * K3 * Cin), W2q((size_t)C * K3 * C);
    for (size_t e = 0; e < xq.size(); ++e) xq[e] = op(x[e]);
    for (size_t e = 0; e < W1q.size(); ++e) W1q[e] = op(W1[e]);
    for (size_t e = 0; e < W2q.size(); ++e) W2q[e] = op(W2[e]);

    // a1: conv1 (row a1)
    std::vector<double> a1(BT * C), h1q(BT * C), a2(BT * C), h2(BT * C);
    std::vector<char> d1(BT * C), d2(BT * C);  // ReLU decisions
    for (int b = 0; b < B; ++b)
        for (int t = 0; t < T; ++t)
            for (int o = 0; o < C; ++o) {
                double acc = b1[o], S = std::fabs(b1[o]);
                for (int j = 0; j < K3; ++j) {
                    const int tt = t + j - 1;
                    if (tt < 0 || tt >= T) continue;  // zero "same" padding
                    const double* wr = &W1q[((size_t)o * K3 + j) * Cin];
                    const double* xr = &xq[((size_t)b * T + tt) * Cin];
                    for (int c = 0; c < Cin; ++c) {
                        acc += wr[c] * xr[c];
                        S += std::fabs(wr[c] * xr[c]);
                    }
                }
                const size_t e = ((size_t)b * T + t) * C + o;
                a1[e] = acc;
                note_kink((int64_t)e, acc, S);
                d1[e] = (char)((acc > 0) != flipped((int64_t)e));
            }
    for (size_t e = 0; e < a1.size(); ++e) h1q[e] = op(d1[e] ? a1[e] : 0.0);
    // a2: conv2 (row a2)
    for (int b = 0; b < B; ++b)
        for (int t = 0; t < T; ++t)
            for (int o = 0; o < C; ++o) {
                double acc = b2[o], S = std::fabs(b2[o]);
                for (int j = 0; j < K3; ++j) {
                    const int tt = t + j - 1;
                    if (tt < 0 || tt >= T) continue;
                    const double* wr = &W2q[((size_t)o * K3 + j) * C];
                    const double* hr = &h1q[((size_t)b * T + tt) * C];
                    for (int c = 0; c < C; ++c) {
                        acc += wr[c] * hr[c];
                        S += std::fabs(wr[c] * hr[c]);
                    }
                }
                const size_t e = ((size_t)b * T + t) * C + o;
                a2[e] = acc;
                note_kink(layer_stride + (int64_t)e, acc, S);
                d2[e] = (char)((acc > 0) != flipped(layer_stride + (int64_t)e));
            }
    for (size_t e = 0; e < a2.size(); ++e) h2[e] = d2[e] ? a2[e] : 0.0;
    if (decisions_out)
        for (size_t e = 0; e < BT * C; ++e) {
            decisions_out[e] = (uint8_t)d1[e];
            decisions_out[BT * C + e] = (uint8_t)d2[e];
        }
    // z: conv3 k1 (row a3)
    std::vector<double> z(BT * Co), dz(BT * Co);
    for (size_t r = 0; r < BT; ++r)
        for (int o = 0; o < Co; ++o) {
            double acc = b3[o];
            for (int c = 0; c < C; ++c) acc += W3[(size_t)o * C + c] * h2[r * C + c];
            z[r * Co + o] = acc;
        }
    if (z_out) for (size_t e = 0; e < z.size(); ++e) z_out[e] = z[e];
    // loss + dz (row a4)
    for (int b = 0; b < B; ++b)
        for (int o = 0; o < Co; ++o) {
            const double* g = labels + ((size_t)b * Co + o) * T;
            int lpos = 0;
            for (int t = 0; t < T; ++t) lpos += (g[t] > 0.5) ? 1 : 0;
            const int lneg = T - lpos;
            const double ap = (double)T / (double)(lpos > 1 ? lpos : 1);
            const double an = (double)T / (double)(lneg > 1 ? lneg : 1);
            double Lo = 0.0;
            for (int t = 0; t < T; ++t) {
                const double zz = z[((size_t)b * T + t) * Co + o];
                const double bt = (g[t] > 0.5) ? 1.0 : 0.0;
                const double logp = -softplus(-zz), log1mp = -softplus(zz);
                Lo += ap * bt * logp + an * (1.0 - bt) * log1mp;
                const double p = 1.0 / (1.0 + std::exp(-zz));
                dz[((size_t)b * T + t) * Co + o] =
                    lambda[o] / ((double)B * T) * (an * (1.0 - bt) * p - ap * bt * (1.0 - p));
            }
            Lo = -Lo / (double)T;
            loss_out[1 + o] += Lo / (double)B;
            loss_out[0] += lambda[o] * Lo / (double)B;
        }
    // head backward (row a5)
    std::vector<double> dA2q(BT * C);
    for (size_t r = 0; r < BT; ++r)
        for (int o = 0; o < Co; ++o) {
            db3[o] += dz[r * Co + o];
            for (int c = 0; c < C; ++c) dW3[(size_t)o * C + c] += dz[r * Co + o] * h2[r * C + c];
        }
    for (size_t r = 0; r < BT; ++r)
        for (int c = 0; c < C; ++c) {
            double acc = 0.0;
            for (int o = 0; o < Co; ++o) acc += W3[(size_t)o * C + c] * dz[r * Co + o];
            dA2q[r * C + c] = op(d2[r * C + c] ? acc : 0.0);
        }
    // conv2 wgrad (row a7)
    for (int b = 0; b < B; ++b)
        for (int t = 0; t < T; ++t)
            for (int o = 0; o < C; ++o) {
                const double d = dA2q[((size_t)b * T + t) * C + o];
                db2[o] += d;
                for (int j = 0; j < K3; ++j) {
                    const int tt = t + j - 1;
                    if (tt < 0 || tt >= T) continue;
                    const double* hr = &h1q[((size_t)b * T + tt) * C];
                    double* wr = &dW2[((size_t)o * K3 + j) * C];
                    for (int c = 0; c < C; ++c) wr[c] += d * hr[c];
                }
            }
    // conv2 dgrad (row a6): dh1[t] = sum_j sum_o W2[o][j][:] dA2[t-j+1][o]
    std::vector<double> dA1q(BT * C);
    for (int b = 0; b < B; ++b)
        for (int t = 0; t < T; ++t)
            for (int c = 0; c < C; ++c) {
                double acc = 0.0;
                for (int j = 0; j < K3; ++j) {
                    const int ts = t - j + 1;
                    if (ts < 0 || ts >= T) continue;
                    for (int o = 0; o < C; ++o)
                        acc += W2q[((size_t)o * K3 + j) * C + c] * dA2q[((size_t)b * T + ts) * C + o];
                }
                const size_t r = (size_t)b * T + t;
                dA1q[r * C + c] = op(d1[r * C + c] ? acc : 0.0);
            }
    // conv1 wgrad (row a8); no dX (inputs are precomputed features)
    for (int b = 0; b < B; ++b)
        for (int t = 0; t < T; ++t)
            for (int o = 0; o < C; ++o) {
                const double d = dA1q[((size_t)b * T + t) * C + o];
                db1[o] += d;
                for (int j = 0; j < K3; ++j) {
                    const int tt = t + j - 1;
                    if (tt < 0 || tt >= T) continue;
                    const double* xr = &xq[((size_t)b * T + tt) * Cin];
                    double* wr = &dW1[((size_t)o * K3 + j) * Cin];
                    for (int c = 0; c < Cin; ++c) wr[c] += d * xr[c];
                }
            }
    return 0;
}

int orc_tem_fwd_bwd(int prec, int B, int T, int Cin, int C, int Co,
                    const double* x, const double* params, const double* labels,
                    const double* lambda, double* loss_out, double* z_out, double* grad_out) {
    return orc_tem_fwd_bwd_ex(prec, B, T, Cin, C, Co, x, params, labels, lambda, loss_out, z_out,
                              grad_out, nullptr, 0, 0.0, 0.0, nullptr, 0, nullptr, nullptr);
}

// ============================================================================ PEM
// BSN's proposal evaluation module, trained jointly with TEM in BASELINE configs[4] (SURVEY
// 8(f) NEXT #1; the paper shows BSN's stages only in Fig. 1b, P:63 -- the module itself is
// BSN's, readings R19-R21 in DESIGN.md).  Per proposal m with BSP feature f_m (F = 32) and
// IoU target g_m:
//   a_m = W1 f_m + b1 (H = 512),  h_m = ReLU(a_m),  z_m = w2 . h_m + b2,  y_m = sigmoid(z_m)
//   L   = (1/M) sum_m (y_m - g_m)^2                                   (R20: plain MSE)
// Backward (chain rule):  dz_m = (2/M)(y_m - g_m) y_m (1 - y_m);  dw2 = sum_m dz_m h_m;
//   db2 = sum_m dz_m;  dh_m = 1[a_m > 0] dz_m w2;  dW1 = sum_m dh_m f_m^T;  db1 = sum_m dh_m.
// Parameters (and gradient) flat [W1 (H x F, row [j][k]), b1 (H), w2 (H), b2 (1)] (R21).
// flips / kinks / decisions: as orc_tem_fwd_bwd_ex (reading R7b), index m*H + j.
int64_t orc_pem_num_params(int F, int H) { return (int64_t)H * F + 2 * (int64_t)H + 1; }

int orc_pem_fwd_bwd(int M, int F, int H, const double* f, const double* params, const double* g,
                    double* loss_out, double* y_out, double* grad_out, const int64_t* flips, int64_t nflips,
                    double kink_tau, int64_t* kinks_out, int64_t kinks_cap, int64_t* nkinks,
                    uint8_t* decisions_out) {
    if (M < 0 || F < 1 || H < 1 || !params || !loss_out || !grad_out) return 1;
    const double* W1 = params;
    const double* b1 = W1 + (int64_t)H * F;
    const double* w2 = b1 + H;
    const double b2 = w2[H];
    const int64_t K = orc_pem_num_params(F, H);
    for (int64_t i = 0; i < K; ++i) grad_out[i] = 0.0;
    double* gW1 = grad_out;
    double* gb1 = gW1 + (int64_t)H * F;
    double* gw2 = gb1 + H;
    double* gb2 = gw2 + H;
    std::vector<double> h(H);
    std::vector<uint8_t> pos(H);
    int64_t nk = 0;
    double L = 0.0;
    for (int m = 0; m < M; ++m) {
        const double* fm = f + (int64_t)m * F;
        for (int j = 0; j < H; ++j) {
            double a = b1[j], mag = std::fabs(b1[j]);
            for (int k = 0; k < F; ++k) {
                a += W1[(int64_t)j * F + k] * fm[k];
                mag += std::fabs(W1[(int64_t)j * F + k] * fm[k]);
            }
            const int64_t idx = (int64_t)m * H + j;
            bool p = a > 0.0;
            if (flips && nflips > 0 && std::binary_search(flips, flips + nflips, idx)) p = !p;
            if (kink_tau > 0.0 && std::fabs(a) <= kink_tau * mag) {
                if (kinks_out && nk < kinks_cap) kinks_out[nk] = idx;
                ++nk;
            }
            if (decisions_out) decisions_out[idx] = p ? 1 : 0;
            pos[j] = p ? 1 : 0;
            h[j] = p ? a : 0.0;
        }
        double z = b2;
        for (int j = 0; j < H; ++j) z += w2[j] * h[j];
        const double y = 1.0 / (1.0 + std::exp(-z));
        if (y_out) y_out[m] = y;
        L += (y - g[m]) * (y - g[m]);
        const double dz = (2.0 / M) * (y - g[m]) * y * (1.0 - y);
        *gb2 += dz;
        for (int j = 0; j < H; ++j) {
            gw2[j] += dz * h[j];
            const double dh = pos[j] ? dz * w2[j] : 0.0;
            gb1[j] += dh;
            for (int k = 0; k < F; ++k) gW1[(int64_t)j * F + k] += dh * fm[k];
        }
    }
    loss_out[0] = M > 0 ? L / M : 0.0;
    if (nkinks) *nkinks = nk;
    return 0;
}

}  // extern "C"

