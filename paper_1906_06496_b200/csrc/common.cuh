// common.cuh -- device helpers private to libtem (never shared with oracle/).
#pragma once
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/tem.h"

#define TEM_DEV __device__ __forceinline__

namespace tem {

// Operand storage types.  fp32 path: float everywhere; bf16 path: bf16 operands
// (reading R8), fp32 accumulate.
TEM_DEV float to_f(float v) { return v; }
TEM_DEV float to_f(__nv_bfloat16 v) { return __bfloat162float(v); }
template <typename T> TEM_DEV T from_f(float v);
template <> TEM_DEV float from_f<float>(float v) { return v; }
template <> TEM_DEV __nv_bfloat16 from_f<__nv_bfloat16>(float v) { return __float2bfloat16_rn(v); }

// Load 8 consecutive operand elements as floats (16B / 32B aligned).
TEM_DEV void load8(const float* p, float* v) {
    float4 a = *reinterpret_cast<const float4*>(p);
    float4 b = *reinterpret_cast<const float4*>(p + 4);
    v[0] = a.x; v[1] = a.y; v[2] = a.z; v[3] = a.w;
    v[4] = b.x; v[5] = b.y; v[6] = b.z; v[7] = b.w;
}
TEM_DEV void load8(const __nv_bfloat16* p, float* v) {
    uint4 u = *reinterpret_cast<const uint4*>(p);
    const uint32_t w[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        v[2 * i] = __uint_as_float(w[i] << 16);
        v[2 * i + 1] = __uint_as_float(w[i] & 0xFFFF0000u);
    }
}

// ---- system-scope flag primitives (ring protocol, cross-GPU over NVLink) ----------------
TEM_DEV uint64_t ld_acquire_sys(const uint64_t* p) {
    uint64_t v;
    asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
TEM_DEV void st_release_sys(uint64_t* p, uint64_t v) {
    asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
// LL ("low latency") lines: 16 bytes {d0, flag, d1, flag}.  Each 8-byte half {datum, flag} is
// written by one 8-byte-atomic half of a volatile 16-byte store, so a reader that sees both
// flags equal to the expected epoch also sees both data words -- no fence, no barrier.
TEM_DEV uint4 ld_volatile4(const uint4* p) {
    uint4 v;
    asm volatile("ld.volatile.global.v4.u32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
                 : "l"(p)
                 : "memory");
    return v;
}
TEM_DEV void st_volatile4(uint4* p, uint4 v) {
    asm volatile("st.volatile.global.v4.u32 [%0], {%1,%2,%3,%4};" ::"l"(p), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w)
                 : "memory");
}
TEM_DEV uint64_t globaltimer() {
    uint64_t t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}
// One snippet row of the head (readings R5-R7) for output channel o:
// the loss term alpha+ b log p + alpha- (1-b) log(1-p) and dz = lam/(B T) (alpha- (1-b) p -
// alpha+ b (1-p)).  With e = exp(-|z|): p and 1-p are 1/(1+e) and e/(1+e) (which one depends on
// the sign of z; no cancellation), log p = -softplus(-z), log(1-p) = -softplus(z) and
// softplus(+-z) = max(+-z, 0) + log1p(e) -- one exp and one log per row and channel, both the
// hardware approximations (ex2 / lg2: ~2^-22 relative for exp, ~2^-21 absolute for log, and
// log(1 + e) loses at most ~2^-24 absolute when 1 + e rounds): the loss and dz stay ~1e-7
// relative to the fp64 oracle, far inside the 1e-4 contract, at a fraction of the latency of
// the libm versions on this latency-bound, one-warp-per-scheduler path.
TEM_DEV void head_row_terms(float z, float bt, float ap, float an, float lam_over_bt, float& lt, float& dz) {
    const float e = __expf(-fabsf(z));
    const float r = __frcp_rn(1.f + e);
    const float er = e * r;
    const float p = z >= 0.f ? r : er, q = z >= 0.f ? er : r;  // p, 1 - p
    const float l1 = __logf(1.f + e);
    const float logp = -(fmaxf(-z, 0.f) + l1), log1mp = -(fmaxf(z, 0.f) + l1);
    lt = ap * bt * logp + an * (1.f - bt) * log1mp;
    dz = lam_over_bt * (an * (1.f - bt) * p - ap * bt * q);
}

// Kernel-span trace (diagnostics build only, -DTEM_DIAG; scripts/probes/step_trace.py): while
// g_trace is set (one copy per translation unit, set by trace_set_<unit>), each traced kernel
// records the minimum start and maximum end globaltimer over its CTAs in g_trace[2 slot],
// g_trace[2 slot + 1].  The product library compiles these to nothing.
#ifdef TEM_DIAG
static __device__ unsigned long long* g_trace;
TEM_DEV void trace_begin(int slot) {
    if (g_trace != nullptr && threadIdx.x == 0) atomicMin(&g_trace[2 * slot], (unsigned long long)globaltimer());
}
TEM_DEV void trace_end(int slot) {  // all threads of the CTA, at its end
    if (g_trace != nullptr) {
        __syncthreads();
        if (threadIdx.x == 0) atomicMax(&g_trace[2 * slot + 1], (unsigned long long)globaltimer());
    }
}
// per-CTA phase stamp k of a kernel (g_trace[2 NUM_SLOTS + cta * 8 + k])
#define TEM_PHASE_STAMP(base, k)                                                                  \
    do {                                                                                          \
        if (g_trace != nullptr && threadIdx.x == 0) g_trace[(base) + blockIdx.x * 8 + (k)] = globaltimer(); \
    } while (0)
#define TEM_TRACE_SETTER(name) \
    void name(unsigned long long* p) { cudaMemcpyToSymbol(g_trace, &p, sizeof(p)); }
#else
TEM_DEV void trace_begin(int) {}
TEM_DEV void trace_end(int) {}
#define TEM_PHASE_STAMP(base, k) \
    do {                         \
    } while (0)
#define TEM_TRACE_SETTER(name) \
    void name(unsigned long long*) {}
#endif

// L2-coherent 128-bit load (bypasses L1: data written by a peer GPU lands in our L2).
TEM_DEV float4 ld_cg4(const float* p) { return __ldcg(reinterpret_cast<const float4*>(p)); }

// Programmatic dependent launch (PDL): a kernel launched with the programmatic-serialization
// attribute may start while its stream predecessor is still running; it must call pdl_wait()
// before touching global memory that the predecessor writes or reads.  pdl_trigger() lets
// the NEXT kernel launch now (its CTAs still block in their own pdl_wait).  Both are no-ops
// for a kernel launched without the attribute.
TEM_DEV void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
TEM_DEV void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

// Device-side error latch (host-mapped pinned word): first error wins.
struct Status {
    int32_t code;      // tem_status
    int32_t pad;
    int64_t step;      // step index for NONFINITE
};
TEM_DEV void latch(Status* s, int32_t code, int64_t step) {
    if (atomicCAS(&s->code, 0, code) == 0) {
        s->step = step;
        __threadfence_system();
    }
}

}  // namespace tem
