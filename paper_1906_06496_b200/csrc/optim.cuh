// optim.cuh -- the owner's optimizer update and the refresh of the weights' bf16 operand
// copies, used by every kernel that applies an update (ring.cu: the collectives and the N = 1
// update kernels).
#pragma once
#include <cuda_bf16.h>

#include "kernels.h"

namespace tem {

// Refresh the operand copies of the weights: sh = bf16(w), and (3-pass fp32 path)
// sl = bf16(w - bf16(w)).
TEM_DEV void store_shadow4(__nv_bfloat16* sh, __nv_bfloat16* sl, int64_t e, float4 w) {
    const __nv_bfloat162 a = __floats2bfloat162_rn(w.x, w.y);
    const __nv_bfloat162 b = __floats2bfloat162_rn(w.z, w.w);
    uint2 u;
    u.x = *reinterpret_cast<const uint32_t*>(&a);
    u.y = *reinterpret_cast<const uint32_t*>(&b);
    *reinterpret_cast<uint2*>(sh + e) = u;
    if (sl) {
        const __nv_bfloat162 c = __floats2bfloat162_rn(w.x - __low2float(a), w.y - __high2float(a));
        const __nv_bfloat162 d = __floats2bfloat162_rn(w.z - __low2float(b), w.w - __high2float(b));
        uint2 v;
        v.x = *reinterpret_cast<const uint32_t*>(&c);
        v.y = *reinterpret_cast<const uint32_t*>(&d);
        *reinterpret_cast<uint2*>(sl + e) = v;
    }
}

// The owner's optimizer step on 4 elements at e (tem_step exchanges, K = K_pad).
//   SGD  (R12): w' = fma(-lr, g, w), one rounding.
//   Adam (R22): m' = b1*m + c1*g; v' = b2*v + c2*(g*g); w' = w - lr*((m'/(1-b1^t)) /
//               (sqrt(v'/(1-b2^t)) + eps)), every operation single-rounded (no contraction), in
//               the oracle's order (orc_ring_adam_f32); the moments live in the owner's OptState;
//               scal holds beta^(t-1) during the step.
TEM_DEV float adam1(const OptCfg& o, float d1, float d2, float g, float& m, float& v, float w) {
    m = __fadd_rn(__fmul_rn(o.beta1, m), __fmul_rn(o.c1, g));
    v = __fadd_rn(__fmul_rn(o.beta2, v), __fmul_rn(o.c2, __fmul_rn(g, g)));
    const float mhat = __fdiv_rn(m, d1), vhat = __fdiv_rn(v, d2);
    const float step = __fdiv_rn(mhat, __fadd_rn(__fsqrt_rn(vhat), o.eps));
    return __fsub_rn(w, __fmul_rn(o.lr, step));
}
// KIND = -1: chosen at run time from o.kind; TEM_OPT_SGD / TEM_OPT_ADAM: fixed at compile time
template <int KIND = -1>
TEM_DEV float4 owner_update(const OptCfg& o, const OptState& st, int64_t e, float4 g, float4 w) {
    if (KIND == TEM_OPT_MOMENTUM || (KIND < 0 && o.kind == TEM_OPT_MOMENTUM)) {  // reading R23
        float4 u = *reinterpret_cast<const float4*>(st.m + e);
        u.x = __fmaf_rn(o.mu, u.x, g.x);
        u.y = __fmaf_rn(o.mu, u.y, g.y);
        u.z = __fmaf_rn(o.mu, u.z, g.z);
        u.w = __fmaf_rn(o.mu, u.w, g.w);
        *reinterpret_cast<float4*>(st.m + e) = u;
        g = u;  // w = fma(-lr, u, w) below
    } else if (KIND == TEM_OPT_ADAM || (KIND < 0 && o.kind == TEM_OPT_ADAM)) {
        // this step's beta^t = fl(beta^(t-1) * beta): every thread forms the same product; the
        // stored pair advances after the step's last update (opt_scalars_kernel)
        const float d1 = __fsub_rn(1.0f, __fmul_rn(st.scal[0], o.beta1));
        const float d2 = __fsub_rn(1.0f, __fmul_rn(st.scal[1], o.beta2));
        float4 m = *reinterpret_cast<const float4*>(st.m + e), v = *reinterpret_cast<const float4*>(st.v + e);
        float4 r;
        r.x = adam1(o, d1, d2, g.x, m.x, v.x, w.x);
        r.y = adam1(o, d1, d2, g.y, m.y, v.y, w.y);
        r.z = adam1(o, d1, d2, g.z, m.z, v.z, w.z);
        r.w = adam1(o, d1, d2, g.w, m.w, v.w, w.w);
        *reinterpret_cast<float4*>(st.m + e) = m;
        *reinterpret_cast<float4*>(st.v + e) = v;
        return r;
    }
    return make_float4(__fmaf_rn(-o.lr, g.x, w.x), __fmaf_rn(-o.lr, g.y, w.y), __fmaf_rn(-o.lr, g.z, w.z),
                       __fmaf_rn(-o.lr, g.w, w.w));
}

}  // namespace tem
