// sm_100a kernels of the gradient exchange + blended update (arXiv 1711.04325).
//
// Everything here is HBM- or NVLink-bound streaming work:
// there is no dense contraction, so no tensor cores.  The kernels move 8 elements per
// thread per trip (one 256-bit access per fp32 row where the buffers are 32-byte aligned,
// else two 128-bit ones; 16-byte fp16 wire vectors), use evict-first streaming hints for
// data touched once (g, theta, Delta, m), and keep the fp16 wire buffers on the
// default policy so a consumer launched right after the producer hits L2.
//
// Cross-GPU ordering (world > 1) uses epoch-valued flags in each rank's CUDA-IPC
// exchange buffer: a producer (the last block of a phase, found with a ticket
// counter, or the block completing a chunk) issues one system-scope fence and then
// relaxed system-scope stores of the step's epoch into every rank's flag slot;
// consumers spin with ld.acquire.sys, bounded by a %globaltimer timeout that turns a
// missing rank into LMSGD_ERR_TIMEOUT instead of a hang.
#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <initializer_list>
#include <utility>

#include "lmsgd_internal.h"
#include "device_common.cuh"

namespace lmsgd {
namespace {

constexpr int kThreads = 256;   // LMSGD_LB below spells the same block size
#ifndef LMSGD_XGATHER_OWN_IN_REDUCE
#define LMSGD_XGATHER_OWN_IN_REDUCE 0   // A/B knob: lmsgd_exchange with the own shard of R_out written by the reduce (profiles/r2/ab/exchange_own_shard.txt: no gain)
#endif
#ifndef LMSGD_XUNITS
#define LMSGD_XUNITS 2   // A/B at k = 4 (profiles/r1/ab/xunits_n4.txt): 201.9 vs 206.8 us per step with 1
#endif
constexpr int kXUnits = LMSGD_XUNITS;   // k_xupdate: 2048-element units per block
enum { FLAG_A = 0, FLAG_B = 1, FLAG_C = 2, FLAG_D = 3 };  // A / B: a rank's phase 0 / 1 push is done; C: BN staged;
                                             // D (local): this step's skip decision is stored

// Minimum resident blocks per SM asked of ptxas (register caps), A/B knobs set with
// LMSGD_NVCC_EXTRA in build.py; 0 = ptxas' default heuristic (which is NOT the same as
// an explicit 1: that lets ptxas use up to 255 registers, 76 for k_update).  Measured
// (profiles/r1/ab/update_caps.txt, one box, 5 runs): k_xupdate capped at 6 or 5
// blocks/SM moves the k = 4 step by -3.5 .. +0.6 us (noise), k_update capped at 5 by
// +0.7 us, k_fused1 capped at 5 by +7 us -- all stay at the default.  Only k_xstep1
// gains from its cap (LMSGD_XSTEP_MINB).
#ifndef LMSGD_UPD_MINB
#define LMSGD_UPD_MINB 0    // k_update
#endif
#ifndef LMSGD_FUSED_MINB
#define LMSGD_FUSED_MINB 0  // k_fused1
#endif
#ifndef LMSGD_XUPD_MINB
#define LMSGD_XUPD_MINB 0   // k_xupdate
#endif
#define LMSGD_LB_0 __launch_bounds__(256)
#define LMSGD_LB_1 __launch_bounds__(256, 1)
#define LMSGD_LB_2 __launch_bounds__(256, 2)
#define LMSGD_LB_3 __launch_bounds__(256, 3)
#define LMSGD_LB_4 __launch_bounds__(256, 4)
#define LMSGD_LB_5 __launch_bounds__(256, 5)
#define LMSGD_LB_6 __launch_bounds__(256, 6)
#define LMSGD_LB_7 __launch_bounds__(256, 7)
#define LMSGD_LB_8 __launch_bounds__(256, 8)
#define LMSGD_LB_(b) LMSGD_LB_##b
#define LMSGD_LB(b) LMSGD_LB_(b)

// ------------------------------------------------------------------ helpers

__device__ __forceinline__ bool nonfinite(float x) {
    return (__float_as_uint(x) & 0x7f800000u) == 0x7f800000u;
}

// Two fp32 -> one f16x2 word, RNE, saturating to +-65504 (R7).  `lo` lands in
// the low 16 bits (lower address).
__device__ __forceinline__ uint32_t cvt_sat_f16x2(float lo, float hi) {
    uint32_t r;
    asm("cvt.rn.satfinite.f16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(hi), "f"(lo));
    return r;
}

__device__ __forceinline__ float h2f(uint32_t w, int hi) {
    return __half2float(__ushort_as_half(static_cast<unsigned short>(hi ? (w >> 16) : (w & 0xffffu))));
}

// binary16 of an exact float64 sum: clamp (saturation, R7) then one RNE rounding.
__device__ __forceinline__ unsigned short sat16_f64(double a, unsigned& sat) {
    if (fabs(a) > 65504.0) ++sat;
    a = fmin(fmax(a, -65504.0), 65504.0);
    return __half_as_ushort(__double2half(a));
}

__device__ __forceinline__ uint32_t ld_acquire_sys(const uint32_t* p) {
    uint32_t v;
    asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}

// NVLS (NVLink SHARP through the NVSwitch; lmsgd_nvls_*): `mc` is a multicast address,
// i.e. the same offset in every rank's copy of the bound buffer.
//   ld_reduce: the switch reads the 16 bytes (8 fp16) from every rank's copy and returns
//              their sum, accumulated in fp32 (.acc::f32; SASS LDGMC.E.HPADD.F16x8) and
//              rounded once to fp16 -- R = sat16(S) up to the fp32 accumulation (R8').
//   st:        one store, replicated by the switch into every rank's copy.
__device__ __forceinline__ uint4 mm_ld_reduce_f16x8(const void* mc) {
    uint4 r;
    asm volatile("multimem.ld_reduce.relaxed.sys.global.add.acc::f32.v4.f16x2 {%0, %1, %2, %3}, [%4];"
                 : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
                 : "l"(mc)
                 : "memory");
    return r;
}
__device__ __forceinline__ void mm_st_16B(void* mc, uint4 v) {
    asm volatile("multimem.st.relaxed.sys.global.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(mc), "r"(v.x), "r"(v.y),
                 "r"(v.z), "r"(v.w)
                 : "memory");
}
// R7 on the switch's result: an fp16 infinity is a sum beyond the fp16 range (the inputs
// are finite, saturated at pack); count it and saturate to +-65504.
__device__ __forceinline__ uint32_t sat_inf_f16x2(uint32_t w, unsigned& sat) {
#pragma unroll
    for (int i = 0; i < 2; ++i) {
        const uint32_t h = (w >> (16 * i)) & 0xffffu;
        if ((h & 0x7fffu) == 0x7c00u) {
            ++sat;
            w = (w & ~(0xffffu << (16 * i))) | (((h & 0x8000u) | 0x7bffu) << (16 * i));
        }
    }
    return w;
}


// 8 consecutive fp32 at p with the evict-first streaming hint: one 256-bit access
// (V8: LDG/STG.E.EF.ENL2.256, sm_100; p 32-byte aligned) or two 128-bit ones (p 16-byte
// aligned).  The host picks V8 when every state / gradient pointer of the launch is
// 32-byte aligned (a torch allocation is).  Measured (N = 1, R50, profiles/r2/ab/v8_n1.txt):
// the in-place single pass 114.8 -> 106.0 us, the guarded in-place step 131.9 -> 123.7 us,
// the SGD-phase step with m frozen 101.7 -> 93.6 us; the out-of-place step unchanged.
template <bool V8>
__device__ __forceinline__ void ld8cs(const float* p, float v[8]) {
    if constexpr (V8) {
    asm volatile("ld.global.cs.v8.f32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];"
                 : "=f"(v[0]), "=f"(v[1]), "=f"(v[2]), "=f"(v[3]), "=f"(v[4]), "=f"(v[5]), "=f"(v[6]), "=f"(v[7])
                 : "l"(p));
    } else {
    const float4 a = __ldcs(reinterpret_cast<const float4*>(p));
    const float4 b = __ldcs(reinterpret_cast<const float4*>(p) + 1);
    v[0] = a.x; v[1] = a.y; v[2] = a.z; v[3] = a.w;
    v[4] = b.x; v[5] = b.y; v[6] = b.z; v[7] = b.w;
    }
}
template <bool V8>
__device__ __forceinline__ void st8cs(float* p, const float v[8]) {
    if constexpr (V8) {
    asm volatile("st.global.cs.v8.f32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8};" ::"l"(p), "f"(v[0]), "f"(v[1]),
                 "f"(v[2]), "f"(v[3]), "f"(v[4]), "f"(v[5]), "f"(v[6]), "f"(v[7])
                 : "memory");
    } else {
    __stcs(reinterpret_cast<float4*>(p), make_float4(v[0], v[1], v[2], v[3]));
    __stcs(reinterpret_cast<float4*>(p) + 1, make_float4(v[4], v[5], v[6], v[7]));
    }
}

// 8 consecutive fp32 from j0 (j0 % 8 == 0), zero beyond n.  Streaming loads.
template <bool V8 = false>
__device__ __forceinline__ void load8_g(const float* __restrict__ g, int64_t j0, int64_t n,
                                        float x[8]) {
    if (j0 + 8 <= n) {
        ld8cs<V8>(g + j0, x);
    } else {
#pragma unroll
        for (int i = 0; i < 8; ++i) x[i] = (j0 + i < n) ? g[j0 + i] : 0.0f;
    }
}

// h = sat16_RNE(s * g) for 8 values; records the first non-finite g index and
// the count of finite g with |s g| > 65504.
__device__ __forceinline__ uint4 pack8(const float x[8], float s, int64_t j0, int64_t& first,
                                       unsigned& sat) {
    float y[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) {
        const bool bad = nonfinite(x[i]);
        if (bad) first = (j0 + i) < first ? (j0 + i) : first;
        y[i] = s * x[i];
        sat += (!bad && fabsf(y[i]) > 65504.0f) ? 1u : 0u;
    }
    return make_uint4(cvt_sat_f16x2(y[0], y[1]), cvt_sat_f16x2(y[2], y[3]),
                      cvt_sat_f16x2(y[4], y[5]), cvt_sat_f16x2(y[6], y[7]));
}

// Warp-aggregated status flush: one atomic per warp (and none when clean).
__device__ __forceinline__ void flush_status(int64_t first, unsigned sat, int64_t* st, int sat_slot) {
    const unsigned full = 0xffffffffu;
    const unsigned satw = __reduce_add_sync(full, sat);
    const bool anyf = __any_sync(full, first != kNone);
    if (anyf) {
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            const int64_t other = __shfl_xor_sync(full, first, o);
            first = other < first ? other : first;
        }
    }
    if ((threadIdx.x & 31) == 0) {
        if (satw) atomicAdd(reinterpret_cast<unsigned long long*>(st + sat_slot), (unsigned long long)satw);
        if (anyf) atomicMin(reinterpret_cast<long long*>(st + ST_FIRST), (long long)first);
    }
}

// The blended update of one element, fp32:
//   m1 = mu2 m + (1-mu2) gh^2;  coef = a_SGD + a_RMS / (sqrt(m1) + eps)
//   d1 = mu1 d - coef gh;       th1 = th + eta d1
// RMS == false is the alpha_RMSprop == 0 specialisation (bit-identical: the
// dropped term is exactly 0 because sqrt(m1) + eps >= eps > 0).
template <bool RMS>
__device__ __forceinline__ void upd1(float gh, float& th, float& d, float& m, const UpdConst& c) {
    const float m1 = fmaf(c.mu2, m, c.omm2 * (gh * gh));
    float coef = c.a_sgd;
    if (RMS) coef = c.a_sgd + c.a_rms / (sqrtf(m1) + c.eps);
    const float d1 = fmaf(c.mu1, d, -(coef * gh));
    th = fmaf(c.eta, d1, th);
    d = d1;
    m = m1;
}

// Update 8 consecutive elements from j0 given their 8 fp16 wire values.  WD: the
// weight-decay variant (R12, g += lambda theta on [0, n_wd)); a separate
// instantiation so the default path carries no per-element test.
// KM == false (LMSGD_FLAG_FREEZE_M, only with alpha_RMSprop == 0, RMS == false): m
// is neither read nor written -- it does not enter Delta or theta then.
template <bool RMS, bool WD, bool KM = true, bool V8 = false>
__device__ __forceinline__ void update8(uint4 r, int64_t j0, int64_t n, const UpdConst& c,
                                        float* __restrict__ th, float* __restrict__ d,
                                        float* __restrict__ m) {
    const uint32_t w[4] = {r.x, r.y, r.z, r.w};
    if (j0 + 8 <= n) {
        static_assert(KM || !RMS, "m is only frozen when alpha_RMSprop == 0");
        float tv[8], dv[8], mv[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
        ld8cs<V8>(th + j0, tv);
        ld8cs<V8>(d + j0, dv);
        if (KM) ld8cs<V8>(m + j0, mv);
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            float gh = h2f(w[i >> 1], i & 1) * c.inv_ks;
            if (WD && j0 + i < c.n_wd) gh = fmaf(c.wd, tv[i], gh);
            upd1<RMS>(gh, tv[i], dv[i], mv[i], c);
        }
        st8cs<V8>(th + j0, tv);
        st8cs<V8>(d + j0, dv);
        if (KM) st8cs<V8>(m + j0, mv);
    } else {
        for (int i = 0; i < 8 && j0 + i < n; ++i) {
            float gh = h2f(w[i >> 1], i & 1) * c.inv_ks;
            float t = th[j0 + i], dd = d[j0 + i], mm = KM ? m[j0 + i] : 0.f;
            if (WD && j0 + i < c.n_wd) gh = fmaf(c.wd, t, gh);
            upd1<RMS>(gh, t, dd, mm, c);
            th[j0 + i] = t; d[j0 + i] = dd;
            if (KM) m[j0 + i] = mm;
        }
    }
}

__device__ __forceinline__ void reset_words(int64_t* st) {  // one thread per word
    st[threadIdx.x] = (threadIdx.x == ST_FIRST || threadIdx.x == ST_G_FIRST) ? kNone : 0;
}
__device__ __forceinline__ void reset_status(int64_t* st) {
    if (st && blockIdx.x == 0 && threadIdx.x < ST_WORDS) reset_words(st);
}

__device__ __forceinline__ void write_last(int64_t* last, int64_t first, int64_t psat, int64_t ssat,
                                           int64_t err, int64_t skipped) {
    if (last && blockIdx.x == 0 && threadIdx.x == 0) store_last(last, first, psat, ssat, err, skipped);
}

// R[j0 .. j0+8) = sat16_RNE(sum_{p<k} slot_p[j0 .. j0+8)), slots `stride` elements apart:
// widened to fp64 and summed in slot order (exact, so order-free), one rounding.
__device__ __forceinline__ void reduce8(const uint16_t* __restrict__ slots, int64_t stride, int k, int64_t j0,
                                        uint16_t* __restrict__ R, unsigned& sat) {
    double acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    for (int p = 0; p < k; ++p) {
        const uint4 q = *reinterpret_cast<const uint4*>(slots + (int64_t)p * stride + j0);
        const uint32_t w[4] = {q.x, q.y, q.z, q.w};
#pragma unroll
        for (int e = 0; e < 8; ++e) acc[e] += (double)h2f(w[e >> 1], e & 1);
    }
    unsigned short o[8];
#pragma unroll
    for (int e = 0; e < 8; ++e) o[e] = sat16_f64(acc[e], sat);
    *reinterpret_cast<uint4*>(R + j0) = make_uint4(o[0] | (uint32_t)o[1] << 16, o[2] | (uint32_t)o[3] << 16,
                                                  o[4] | (uint32_t)o[5] << 16, o[6] | (uint32_t)o[7] << 16);
}

// reduce8, also returning the 8 reduced values (the update consumes them directly)
__device__ __forceinline__ uint4 reduce8_val(const uint16_t* __restrict__ slots, int64_t stride, int k, int64_t j0,
                                             uint16_t* __restrict__ R, unsigned& sat) {
    reduce8(slots, stride, k, j0, R, sat);
    return *reinterpret_cast<const uint4*>(R + j0);   // this thread's own store
}

__device__ __forceinline__ int64_t gtid() { return (int64_t)blockIdx.x * blockDim.x + threadIdx.x; }
__device__ __forceinline__ int64_t gstride() { return (int64_t)gridDim.x * blockDim.x; }

// ------------------------------------------------------------------ single GPU

__global__ void k_status_reset(int64_t* st, int words) {
    if ((int)threadIdx.x < words) reset_words(st);
}

// graph mode: this step's status slot pair from the device step counter
__device__ __forceinline__ int dev_parity(const Dev1& dv) {
    return (int)((*reinterpret_cast<volatile const uint32_t*>(dv.epoch) + 1u) & 1u);
}

template <bool V8>
__global__ void __launch_bounds__(kThreads) k_pack(const float* __restrict__ g, int64_t n,
                                                   int64_t n_pad, float s, uint16_t* __restrict__ h,
                                                   int64_t* st, Dev1 dv) {
    pdl_enter();
    if (dv.epoch) st = dv.st_base + dev_parity(dv) * ST_WORDS;
    int64_t first = kNone;
    unsigned sat = 0;
    const int64_t nv = n_pad >> 3;
    for (int64_t v = gtid(); v < nv; v += gstride()) {
        const int64_t j0 = v << 3;
        float x[8];
        load8_g<V8>(g, j0, n, x);
        *reinterpret_cast<uint4*>(h + j0) = pack8(x, s, j0, first, sat);
    }
    flush_status(first, sat, st, ST_PACK_SAT);
}

__global__ void __launch_bounds__(kThreads) k_reduce_local(const uint16_t* __restrict__ h, int k,
                                                           int64_t n_pad, uint16_t* __restrict__ R,
                                                           int64_t* st) {
    pdl_enter();
    unsigned sat = 0;
    const int64_t nv = n_pad >> 3;
    for (int64_t v = gtid(); v < nv; v += gstride()) reduce8(h, n_pad, k, v << 3, R, sat);
    if (st) flush_status(kNone, sat, st, ST_SUM_SAT);
}

template <bool RMS, bool WD, bool KM, bool V8>
__global__ void LMSGD_LB(LMSGD_UPD_MINB) k_update(const uint16_t* __restrict__ R, int64_t n, UpdConst c,
                                                     float* __restrict__ th, float* __restrict__ d,
                                                     float* __restrict__ m, const int64_t* st,
                                                     int64_t* st_reset, int64_t* last, Dev1 dv) {
    pdl_enter();
    int64_t first = kNone, psat = 0, ssat = 0, err = 0;
    if (dv.epoch) {   // graph mode: slots from the device counter, coefficients from the table
        const int par = dev_parity(dv);
        st = dv.st_base + par * ST_WORDS;
        st_reset = dv.st_base + (par ^ 1) * ST_WORDS;
        const int64_t idx = *reinterpret_cast<volatile const int64_t*>(dv.cursor);
        if (idx >= dv.count) err = (int64_t)LMSGD_ERR_RANGE;
        else c = dv.ctab[idx];
    }
    if (st) {
        first = st[ST_FIRST]; psat = st[ST_PACK_SAT]; ssat = st[ST_SUM_SAT];
        err = err ? err : st[ST_ERROR];
    }
    const bool skip = first != kNone || err != 0;
    write_last(last, first, psat, ssat, err, skip);
    reset_status(st_reset);
    if (skip) return;
    const int64_t nv = (n + 7) >> 3;
    for (int64_t v = gtid(); v < nv; v += gstride()) {
        const int64_t j0 = v << 3;
        const uint4 r = *reinterpret_cast<const uint4*>(R + j0);
        update8<RMS, WD, KM, V8>(r, j0, n, c, th, d, m);
    }
}

// k = 1 single pass (LMSGD_FLAG_NO_SKIP): h = sat16(s g) kept in registers,
// ghat = fp32(h) / s, update.  28 B/elem of HBM traffic.
template <bool RMS, bool WD, bool KM, bool V8>
__global__ void LMSGD_LB(LMSGD_FUSED_MINB) k_fused1(const float* __restrict__ g, int64_t n, float s,
                                                     UpdConst c, float* __restrict__ th,
                                                     float* __restrict__ d, float* __restrict__ m,
                                                     int64_t* st, int64_t* st_reset, Dev1 dv) {
    pdl_enter();
    if (dv.epoch) {   // graph mode (see k_update)
        const int par = dev_parity(dv);
        st = dv.st_base + par * ST_WORDS;
        st_reset = dv.st_base + (par ^ 1) * ST_WORDS;
        const int64_t idx = *reinterpret_cast<volatile const int64_t*>(dv.cursor);
        if (idx >= dv.count) return;   // table exhausted: k_advance1 reports LMSGD_ERR_RANGE
        c = dv.ctab[idx];
    }
    reset_status(st_reset);
    int64_t first = kNone;
    unsigned sat = 0;
    const int64_t nv = (n + 7) >> 3;
    for (int64_t v = gtid(); v < nv; v += gstride()) {
        const int64_t j0 = v << 3;
        float x[8];
        load8_g<V8>(g, j0, n, x);
        const uint4 r = pack8(x, s, j0, first, sat);
        update8<RMS, WD, KM, V8>(r, j0, n, c, th, d, m);
    }
    flush_status(first, sat, st, ST_PACK_SAT);
}

// Out-of-place variant of update8 (lmsgd_step_out_of_place): reads theta, Delta, m
// from the *_in buffers and writes the new values to the *_out buffers.
template <bool RMS, bool V8>
__device__ __forceinline__ void update8_oop(uint4 r, int64_t j0, int64_t n, const UpdConst& c,
                                            const float* __restrict__ thi, const float* __restrict__ di,
                                            const float* __restrict__ mi, float* __restrict__ tho,
                                            float* __restrict__ dout, float* __restrict__ mo) {
    const uint32_t w[4] = {r.x, r.y, r.z, r.w};
    if (j0 + 8 <= n) {
        float tv[8], dv[8], mv[8];
        ld8cs<V8>(thi + j0, tv);
        ld8cs<V8>(di + j0, dv);
        ld8cs<V8>(mi + j0, mv);
#pragma unroll
        for (int i = 0; i < 8; ++i) upd1<RMS>(h2f(w[i >> 1], i & 1) * c.inv_ks, tv[i], dv[i], mv[i], c);
        st8cs<V8>(tho + j0, tv);
        st8cs<V8>(dout + j0, dv);
        st8cs<V8>(mo + j0, mv);
    } else {
        for (int i = 0; i < 8 && j0 + i < n; ++i) {
            float t = thi[j0 + i], dd = di[j0 + i], mm = mi[j0 + i];
            upd1<RMS>(h2f(w[i >> 1], i & 1) * c.inv_ks, t, dd, mm, c);
            tho[j0 + i] = t; dout[j0 + i] = dd; mo[j0 + i] = mm;
        }
    }
}

// lmsgd_step_out_of_place, k = 1: the guarded step in ONE pass over the state (28 B/elem,
// like k_fused1) -- the new state goes to separate buffers, so a non-finite gradient,
// found only at the end, costs nothing but a repair copy (k_repair1).
#ifndef LMSGD_OOP_LATE_TRIGGER
#define LMSGD_OOP_LATE_TRIGGER 0
#endif
template <bool RMS, bool V8>
__global__ void LMSGD_LB(LMSGD_FUSED_MINB) k_fused1_oop(const float* __restrict__ g, int64_t n, float s,
                                                         UpdConst c, const float* __restrict__ thi,
                                                         const float* __restrict__ di, const float* __restrict__ mi,
                                                         float* __restrict__ tho, float* __restrict__ dout,
                                                         float* __restrict__ mo, int64_t* st, int64_t* st_reset,
                                                         int64_t* trace) {
    // wait for the previous step and let k_repair1 launch (LMSGD_OOP_LATE_TRIGGER = 1: only
    // once every block has finished its elements -- measured neutral with one repair block,
    // +0.7 us per clean step with 148, profiles/r2/ab/repair_n1.txt)
    asm volatile("griddepcontrol.wait;" ::: "memory");
    if (!LMSGD_OOP_LATE_TRIGGER) asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    // lmsgd_trace_enable: block 0's start (it runs in the first wave) ...
    if (trace && blockIdx.x == 0 && threadIdx.x == 0) trace[TR_PACK_START] = (int64_t)globaltimer();
    reset_status(st_reset);
    int64_t first = kNone;
    unsigned sat = 0;
    const int64_t nv = (n + 7) >> 3;
    for (int64_t v = gtid(); v < nv; v += gstride()) {
        const int64_t j0 = v << 3;
        float x[8];
        load8_g<V8>(g, j0, n, x);
        update8_oop<RMS, V8>(pack8(x, s, j0, first, sat), j0, n, c, thi, di, mi, tho, dout, mo);
    }
    flush_status(first, sat, st, ST_PACK_SAT);
    if (LMSGD_OOP_LATE_TRIGGER) asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}

// After k_fused1_oop: block 0 publishes the status record; if a gradient was non-finite
// the step is skipped and the output set receives the unchanged input set (theta, Delta,
// m; a grid-stride copy by every block, 24 B/elem).  On a clean step every block returns
// at once.  LMSGD_REPAIR_BLOCKS blocks of 512 threads (0 = one per SM), launched with
// programmatic dependent launch.  Measured (N = 1, R50, 3 runs each, repair_n1.txt): one
// block (round 1) 105.3 us per clean step but 18.7 ms per skipped step; 32 blocks 105.4 us
// and 0.78 ms; 148 blocks behind an end-of-block trigger 106.0 us and 0.29 ms.
__global__ void __launch_bounds__(512) k_repair1(const int64_t* st, const float* __restrict__ thi,
                                                 const float* __restrict__ di, const float* __restrict__ mi,
                                                 float* __restrict__ tho, float* __restrict__ dout,
                                                 float* __restrict__ mo, int64_t n, int64_t* last, int64_t* trace) {
    pdl_enter();
    // ... and the end of k_fused1_oop: griddepcontrol.wait returns once every k_fused1_oop
    // block has completed and its memory is visible (lmsgd_trace_enable)
    if (trace && blockIdx.x == 0 && threadIdx.x == 0) trace[TR_UPD_END] = (int64_t)globaltimer();
    const int64_t first = *reinterpret_cast<volatile const int64_t*>(st + ST_FIRST);
    if (blockIdx.x == 0 && threadIdx.x == 0)
        store_last(last, first, st[ST_PACK_SAT], 0, st[ST_ERROR], first != kNone ? 1 : 0);
    if (first == kNone) return;
    const int64_t nv = n >> 2;
    for (int64_t v = gtid(); v < nv; v += gstride()) {
        __stcs(reinterpret_cast<float4*>(tho) + v, __ldcs(reinterpret_cast<const float4*>(thi) + v));
        __stcs(reinterpret_cast<float4*>(dout) + v, __ldcs(reinterpret_cast<const float4*>(di) + v));
        __stcs(reinterpret_cast<float4*>(mo) + v, __ldcs(reinterpret_cast<const float4*>(mi) + v));
    }
    for (int64_t j = (nv << 2) + gtid(); j < n; j += gstride()) {
        tho[j] = thi[j]; dout[j] = di[j]; mo[j] = mi[j];
    }
}

// Publishes the fused step's status (never skipped) into the public `last` record.
// A separate 1-warp launch: a per-block fence + ticket in k_fused1 cost 16% of it.
__global__ void k_finalize_fused(const int64_t* st, int64_t* last) {
    pdl_enter();
    if (threadIdx.x == 0) store_last(last, st[ST_FIRST], st[ST_PACK_SAT], st[ST_SUM_SAT], st[ST_ERROR], 0);
}

// Graph mode, k = 1: after the step's kernels, publish the fused step's status and
// advance the device step counter and coefficient cursor (one warp).
__global__ void k_advance1(Dev1 dv, int64_t* last, int fused) {
    pdl_enter();
    if (threadIdx.x != 0) return;
    const uint32_t e = *dv.epoch + 1u;
    const int64_t* st = dv.st_base + (int)(e & 1u) * ST_WORDS;
    const bool range = *dv.cursor >= dv.count;
    if (fused)
        store_last(last, st[ST_FIRST], st[ST_PACK_SAT], st[ST_SUM_SAT],
                   range ? (int64_t)LMSGD_ERR_RANGE : st[ST_ERROR], range);
    *dv.cursor += 1;
    *dv.epoch = e;
}

// ------------------------------------------------------------------ world > 1

// The step's (or BN call's) epoch and status parity.  Host mode passes them as
// arguments (x.epoch > 0); graph mode passes epoch 0 and the kernel reads the device
// counter (*dev_epoch + 1) once per block.  The branch is uniform; the XArgs
// themselves always stay in the kernel parameter space.
struct Ep {
    uint32_t e;
    int par;
};
__device__ __forceinline__ Ep get_ep(const XArgs& x) {
    if (x.epoch != 0u) return Ep{x.epoch, x.parity};
    __shared__ uint32_t s_e;
    if (threadIdx.x == 0) s_e = *reinterpret_cast<volatile const uint32_t*>(x.dev_epoch) + 1u;
    __syncthreads();
    return Ep{s_e, (int)(s_e & 1u)};
}

__device__ __forceinline__ uint32_t* flag_slot(const XArgs& x, int owner, int which) {
    return reinterpret_cast<uint32_t*>(x.peers.base[owner] + x.lay.off_flags + which * 128);
}
__device__ __forceinline__ int64_t* status_of(const XArgs& x, const Ep& ep, int owner) {
    return reinterpret_cast<int64_t*>(x.peers.base[owner] + x.lay.off_status) + ep.par * ST_WORDS;
}

__device__ __forceinline__ void stamp(const XArgs& x, int which) {
    if (x.trace) x.trace[which] = (int64_t)globaltimer();
}


// A block's place in its rank's grid.  A real launch is one rank's grid (b = blockIdx.x,
// g = gridDim.x).  An emulated-group launch (lmsgd_*_group: the ranks of a world
// emulated on ONE GPU, every rank's blocks in the same launch so that ranks that wait
// for one another are co-scheduled) interleaves `nsim` ranks' grids: block blockIdx.x
// plays rank blockIdx.x % nsim as that rank's block blockIdx.x / nsim.
// Emulated group: the per-rank launch arguments, a device array indexed by rank slot.
struct Sim {
    const void* args;   // XStep[nsim] or BnArgs[nsim]
    int nsim;
};
// (read from the special registers each time: nothing held in registers for a real launch)
template <bool SIM>
struct Grid {
    const Sim& s;
    __device__ __forceinline__ int64_t b() const { return SIM ? (int64_t)(blockIdx.x / s.nsim) : (int64_t)blockIdx.x; }
    __device__ __forceinline__ int64_t g() const { return SIM ? (int64_t)(gridDim.x / s.nsim) : (int64_t)gridDim.x; }
};
// This block's arguments: the kernel parameter itself (real launch) or its rank's entry
// of the group array, staged once in shared memory.
template <bool SIM, typename T>
__device__ __forceinline__ const T& rank_args(const T& param, const Sim& sim, T& smem) {
    if (!SIM) return param;
    if (threadIdx.x == 0) smem = static_cast<const T*>(sim.args)[blockIdx.x % sim.nsim];
    __syncthreads();
    return smem;
}

// Grid-wide "done" ticket: returns true in exactly one thread (thread 0 of the last
// block to finish), after all blocks' writes are fenced at system scope.
__device__ bool grid_last(const XArgs& x, int which, int64_t grid) {
    __threadfence_system();
    __syncthreads();
    if (threadIdx.x == 0) {
        const unsigned t = atomicAdd(x.ticket + which, 1u);
        if (t == grid - 1) {
            x.ticket[which] = 0;
            __threadfence_system();
            return true;
        }
    }
    return false;
}

__device__ __forceinline__ void st_relaxed_sys(uint32_t* p, uint32_t v) {
    asm volatile("st.relaxed.sys.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

// Release `value` into slot p of every rank: one system-scope fence, then relaxed
// stores (= a release pattern).  k st.release.sys cost ~1.5 us each on NVLink 5
// (tools/flagbench.cu); the single fence + relaxed stores ~1 us total.
__device__ void publish(const XArgs& x, const Ep& ep, int which) {
    __threadfence_system();
    for (int p = 0; p < x.world; ++p) st_relaxed_sys(flag_slot(x, p, which) + x.rank, ep.e);
}


// Warp 0: wait until every rank has published `which` for this epoch, lane p polling
// rank p's slot (the k acquire round trips overlap instead of running back to back).
// Bounded spin; on timeout record LMSGD_ERR_TIMEOUT in this rank's words.  Call with all
// 32 lanes of warp 0; every lane returns the same result.
__device__ bool warp_wait_all(const XArgs& x, const Ep& ep, int which, bool trace_seen = false) {
    const int p = threadIdx.x & 31;
    bool ok = true;
    if (p < x.world) {
        const uint32_t* f = flag_slot(x, x.rank, which) + p;
        const uint64_t t0 = globaltimer();
        while ((int32_t)(ld_acquire_sys(f) - ep.e) < 0) {
            __nanosleep(64);
            if ((int64_t)(globaltimer() - t0) > x.timeout_ns) {
                ok = false;
                break;
            }
        }
        if (ok && trace_seen && x.trace) x.trace[TR_A_SEEN + p] = (int64_t)globaltimer();   // diagnostics
    }
    ok = __all_sync(0xffffffffu, ok);
    if (!ok && p == 0) {
        int64_t* mine = status_of(x, ep, x.rank);
        mine[ST_ERROR] = (int64_t)LMSGD_ERR_TIMEOUT;
        mine[ST_G_ERROR] = (int64_t)LMSGD_ERR_TIMEOUT;
        __threadfence_system();
    }
    // no trailing fence: each lane's ld.acquire.sys orders its later accesses, and the
    // callers' bar.sync extends that to the rest of the block
    return ok;
}

// Work units of the exchange kernels: a unit is kThreads consecutive 8-element groups
// (2048 elements) of one shard.  k_xstep1's push sweeps them owner-interleaved -- unit u
// belongs to owner (u + rank) % world -- so that the blocks in flight on every rank touch
// all owners evenly (no owner's links are a hot spot); the update and gather kernels take
// them chunk-major (see k_xupdate).

// ------------------------------------------------------------------ world > 1, one kernel

__device__ __forceinline__ uint32_t* cflag(const XArgs& x, int r, int c, int owner) {
    return reinterpret_cast<uint32_t*>(x.peers.base[r] + x.lay.off_cflags) + (int64_t)c * LMSGD_MAX_WORLD + owner;
}

__device__ __forceinline__ bool spin_flag(const XArgs& x, const Ep& ep, const uint32_t* f) {
    const uint64_t t0 = globaltimer();
    while ((int32_t)(ld_acquire_sys(f) - ep.e) < 0) {
        __nanosleep(32);
        if ((int64_t)(globaltimer() - t0) > x.timeout_ns) return false;
    }
    return true;
}

// Chunk flags carry the step's skip decision with the epoch: value 2 e + skip.  A
// consumer then needs one acquire load (no separate wait for flag D and no status
// reads before its update).  The value is exactly 2 e or 2 e + 1 once ready: the next
// step's reduce cannot publish before every rank has finished this step's update.
// Polling backs off exponentially from 32 ns to LMSGD_CFLAG_BACKOFF ns, so that update
// blocks resident long before their chunk (the phased k_xstep1) do not flood L2 with polls.
#ifndef LMSGD_CFLAG_BACKOFF
#define LMSGD_CFLAG_BACKOFF 32
#endif
__device__ __forceinline__ bool spin_cflag(const XArgs& x, const Ep& ep, const uint32_t* f, uint32_t& v) {
    const uint64_t t0 = globaltimer();
    const uint32_t want = ep.e << 1;
    unsigned ns = 32;
    while ((int32_t)((v = ld_acquire_sys(f)) - want) < 0) {
        __nanosleep(ns);
        ns = ns < LMSGD_CFLAG_BACKOFF ? 2 * ns : ns;
        if ((int64_t)(globaltimer() - t0) > x.timeout_ns) return false;
    }
    return true;
}

// The chunk-flag value of this step: waits for the local decision (flag D, stored by
// block 0 long before any chunk completes) and encodes skip.
__device__ __forceinline__ uint32_t cflag_value(const XArgs& x, const Ep& ep) {
    if (!spin_flag(x, ep, flag_slot(x, x.rank, FLAG_D))) return (ep.e << 1) | 1u;
    const volatile int64_t* vm = status_of(x, ep, x.rank);
    const bool skip = vm[ST_G_FIRST] != kNone || vm[ST_G_ERROR] != 0;
    return (ep.e << 1) | (skip ? 1u : 0u);
}

// The world > 1 step in two kernels.
//
// k_xstep1 -- persistent, cooperatively launched (all blocks co-resident, so blocks
// may wait on each other and on other GPUs):
//   1. pack + push: fp16 payload written straight into every owner's receive slot;
//      one system fence per block; the last block releases flag A to every rank;
//   2. every block acquires A of all ranks; block 0 computes the global skip
//      decision from the (now final) pack status words of all ranks, stores it and
//      releases the local flag D;
//   3. exact reduce of this rank's shard, unit u on block u % grid; a 64K-element
//      chunk is released to every rank (cflag[c][rank] = 2 epoch + skip) once all
//      its units are reduced and fenced.
// k_xupdate -- flat grid, launched with programmatic dependent launch so its blocks
// take SMs as soon as k_xstep1's blocks retire: kXUnits units per block, chunk-major
// and owner-major inside a chunk; a block waits only for its units' chunk flags (which
// carry the skip decision), so the update of early chunks overlaps the reduce of later
// ones; R is pulled from the owner inside the update (the all-gather).
// k_xfinalize -- one warp: the step's public status record.
// Chunk counters in a.ctr are reset by the block that completes them.
#ifndef LMSGD_XSTEP_MINB
#define LMSGD_XSTEP_MINB 8   // k_xstep1 capped at 32 registers: 8 blocks/SM (A/B at k = 4: 214.9 vs
                             // 225.6 us per step with no cap, 48 registers, 5 blocks/SM)
#endif
// NV (lmsgd_nvls_*, LMSGD_NVLS_*): 0 = peer memory as above; 1 = the pack is written to this
// rank's own wire (no push) and phase 3 is the switch's reduction (multimem.ld_reduce) of
// this rank's shard into R; 2 = as 1, and the reduced shard is multicast (multimem.st) back
// into every rank's wire in place, so every rank then holds the whole all-reduce result
// locally.
// LMSGD_XPHASES (A/B knob, 1): the shard's units split at chunk boundaries into this many
// phases, each pushed, barriered and reduced in turn, so that k_xupdate (launched behind
// this kernel with programmatic dependent launch, on the SMs left free: LMSGD_XSTEP_BPS
// blocks per SM) updates phase 0's chunks while phase 1 is pushed.  The update is in
// place, so the global skip decision must precede it: phase 0 then also scans the later
// phases' gradient for non-finite values.  tools/xbench.cu suggested the overlap (push ||
// update 134 us against 70 + 99 us serial at k = 4), but in the step two phases measured
// 242-294 us against 203 us (k = 4, 2-6 blocks per SM, with or without backed-off flag
// polling; profiles/r2/ab/phases_n4.txt): the second barrier, the scan and the push with
// fewer blocks beside a busy update cost more than the overlap saves.  Parity-tested at 2.
#ifndef LMSGD_XPHASES
#define LMSGD_XPHASES 1
#endif
static_assert(LMSGD_XPHASES == 1 || LMSGD_XPHASES == 2, "phase flags: A (phase 0) and B (phase 1)");
// k_xstep1 blocks per SM (the rest of each SM is left to k_xupdate when the phases overlap)
#ifndef LMSGD_XSTEP_BPS_DEFAULT
#define LMSGD_XSTEP_BPS_DEFAULT (LMSGD_XPHASES > 1 ? 2 : 8)
#endif
// LMSGD_REDUCE_IN_UPDATE (A/B knob, off): in a step (not lmsgd_exchange) on the peer path
// with one phase, k_xstep1 ends after the skip decision and every rank reduces its own
// shard's units inside k_xupdate (own units first in each chunk, released per block),
// so the update does not wait for a separate reduce pass and its hand-over.  Parity green
// at world 2-8 (emulated and real), but 405.7 vs 202.6 us per step at k = 4 and 332.9 vs
// 180.8 us at k = 2 (profiles/r2/ab/reduce_in_update.txt): the blocks waiting for other
// owners' chunks hold the SMs while only 1/k of the blocks produce R, each behind a system
// fence.  Both kernels decide it the same way.
#ifndef LMSGD_REDUCE_IN_UPDATE
#define LMSGD_REDUCE_IN_UPDATE 0
#endif
__device__ __forceinline__ bool riu_active(const XStep& a) {
    const int nph = a.x.lay.nchunks >= LMSGD_XPHASES ? LMSGD_XPHASES : 1;
    return LMSGD_REDUCE_IN_UPDATE && a.riu && a.x.nv == 0 && nph == 1;
}

template <bool SIM, int NV>
__global__ void LMSGD_LB(LMSGD_XSTEP_MINB) k_xstep1(XStep a_, Sim sim) {
    static_assert(!(SIM && NV), "NVLS needs one GPU per rank");
    pdl_enter();   // wait for the previous step / caller work; let k_xupdate queue up
    __shared__ XStep s_a;
    const XStep& a = rank_args<SIM>(a_, sim, s_a);
    const Grid<SIM> G{sim};
    const XArgs& x = a.x;
    const Ep ep = get_ep(x);
    __shared__ int s_ok;
    __shared__ uint32_t s_fv;   // this step's chunk-flag value (thread 0; 0 = not read yet)
    const bool t0 = threadIdx.x == 0;
    if (t0) s_fv = 0;
    if (G.b() == 0 && t0) stamp(x, TR_PACK_START);
    const int64_t gsh = x.lay.shard >> 3;
    const int64_t ups = (gsh + kThreads - 1) / kThreads;
    int64_t* mine = status_of(x, ep, x.rank);
    const uint16_t* recv = reinterpret_cast<const uint16_t*>(x.peers.base[x.rank] + x.lay.off_recv);
    uint16_t* R = reinterpret_cast<uint16_t*>(x.peers.base[x.rank] + x.lay.off_R);
    // phase p covers the shard units [ulo(p), ulo(p + 1)), chunk-aligned (identical on every rank)
    const int nph = x.lay.nchunks >= LMSGD_XPHASES ? LMSGD_XPHASES : 1;
    auto ulo = [&](int p) -> int64_t {
        const int64_t u = ((int64_t)x.lay.nchunks * p / nph) * x.lay.cu;
        return u < ups ? u : ups;
    };
    // unit u of a phase's all-owner sweep: owner-interleaved (unit u -> owner (u + rank) % world)
    // so that every rank's blocks in flight touch all owners evenly; -1 past the shard
    auto sweep = [&](int64_t lo, int64_t u, int& owner) -> int64_t {
        owner = (int)((u % x.world + x.rank) % x.world);
        const int64_t gi = (lo + u / x.world) * kThreads + threadIdx.x;
        return gi < gsh ? gi : -1;
    };
    // thread 0, after a bar.sync and a system fence that order this block's R writes of
    // unit u (cumulativity): count the unit into its chunk; the block completing a chunk
    // releases it to every rank (cflag[c][rank] = 2 epoch + skip)
    auto count_unit = [&](int64_t u) {
        const int c = (int)(u / x.lay.cu);
        const int64_t rem = ups - (int64_t)c * x.lay.cu;
        const unsigned cnt = (unsigned)(rem < x.lay.cu ? rem : x.lay.cu);
        if (atomicAdd(a.ctr + 4 + c, 1u) + 1u == cnt) {
            a.ctr[4 + c] = 0;
            // the other blocks fenced their R writes before their tickets; this fence
            // orders the observed tickets (hence those writes) before the flag stores
            // peers acquire (cumulativity), as publish() does after its ticket
            __threadfence_system();
            if (!s_fv) s_fv = cflag_value(x, ep);
            for (int p = 0; p < x.world; ++p) st_relaxed_sys(cflag(x, p, c, x.rank), s_fv);
        }
    };

    for (int ph = 0; ph < nph; ++ph) {
        const int64_t lo = ulo(ph), hi = ulo(ph + 1);
        // ---- 1. pack + push of this phase's units (16-byte SM stores to the owners;
        //         pushing each packed unit as one 4 KB cp.async.bulk, or 32-byte stores,
        //         measured the same: the all-to-all is NVLink-bound)
        {
            int64_t first = kNone;
            unsigned sat = 0;
            const int64_t units = (int64_t)x.world * (hi - lo);
            for (int64_t u = G.b(); u < units; u += G.g()) {
                int owner;
                const int64_t gi = sweep(lo, u, owner);
                if (gi < 0) continue;
                const int64_t j0 = ((int64_t)owner * gsh + gi) << 3;
                float xv[8];
                load8_g(a.g, j0, x.n, xv);
                uint16_t* dst = NV ? reinterpret_cast<uint16_t*>(x.nv_uc) + j0   // own wire, [n_pad] layout
                                   : reinterpret_cast<uint16_t*>(x.peers.base[owner] + x.lay.off_recv) +
                                         (int64_t)x.rank * x.lay.shard + (gi << 3);
                *reinterpret_cast<uint4*>(dst) = pack8(xv, a.scale, j0, first, sat);
            }
            if (ph == 0 && nph > 1) {   // the later phases' gradient: finiteness only
                const int64_t units2 = (int64_t)x.world * (ups - hi);
                for (int64_t u = G.b(); u < units2; u += G.g()) {
                    int owner;
                    const int64_t gi = sweep(hi, u, owner);
                    if (gi < 0) continue;
                    const int64_t j0 = ((int64_t)owner * gsh + gi) << 3;
                    float xv[8];
                    load8_g(a.g, j0, x.n, xv);
#pragma unroll
                    for (int i = 0; i < 8; ++i)
                        if (nonfinite(xv[i]) && j0 + i < first) first = j0 + i;
                }
            }
            flush_status(first, sat, mine, ST_PACK_SAT);
        }
        // this block's pushes and status atomics, then its ticket: bar.sync + one thread's
        // system fence (cumulativity; the grid-sync pattern); flag A (phase 0) or B
        const int which = ph == 0 ? FLAG_A : FLAG_B;
        unsigned int* tk = a.ctr + (ph == 0 ? 0 : 2);
        __syncthreads();
        if (t0) __threadfence_system();
        if (t0 && atomicAdd(tk, 1u) + 1u == G.g()) {
            *tk = 0;
            if (ph == 0) stamp(x, TR_PACK_END);
            publish(x, ep, which);
            if (ph == 0) stamp(x, TR_PUB_END);
        }

        // ---- 2. all ranks pushed this phase; after phase 0 block 0 makes the global skip
        //         decision (every rank's first non-finite index is final: phase 0 scanned
        //         the rest) and releases the local flag D.  The reduce does not need it.
        if (threadIdx.x < 32) {
            const bool ok = warp_wait_all(x, ep, which, G.b() == 0 && ph == 0);
            if (t0) s_ok = ok ? 1 : 0;
        }
        __syncthreads();
        if (ph == 0 && G.b() == 0) {
            __shared__ int64_t s_st[2 * LMSGD_MAX_WORLD];
            if (threadIdx.x < x.world) {   // every rank's first index and error, read in parallel
                const volatile int64_t* sp = status_of(x, ep, threadIdx.x);
                s_st[2 * threadIdx.x] = sp[ST_FIRST];
                s_st[2 * threadIdx.x + 1] = sp[ST_ERROR];
            }
            __syncthreads();
            if (t0) {
                int64_t gfirst = kNone, err = s_ok ? 0 : (int64_t)LMSGD_ERR_TIMEOUT;
                for (int p = 0; p < x.world; ++p) {
                    gfirst = s_st[2 * p] < gfirst ? s_st[2 * p] : gfirst;
                    err = err ? err : s_st[2 * p + 1];
                }
                mine[ST_G_FIRST] = gfirst;
                mine[ST_G_ERROR] = err;
                int64_t* nxt = reinterpret_cast<int64_t*>(x.peers.base[x.rank] + x.lay.off_status) +
                               (ep.par ^ 1) * ST_WORDS;   // next step's slot: every rank has read it
                for (int w = 0; w < ST_WORDS; ++w) nxt[w] = (w == ST_FIRST || w == ST_G_FIRST) ? kNone : 0;
                __threadfence();
                asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(flag_slot(x, x.rank, FLAG_D)), "r"(ep.e)
                             : "memory");
                stamp(x, TR_RED_START);
            }
        }
        if (!s_ok) {
            if (t0) atomicAdd(a.ctr + 1, 1u);
            return;
        }
        if (riu_active(a)) {   // the reduce happens in k_xupdate
            if (G.b() == 0 && t0) stamp(x, TR_RED_GO);
            break;
        }

        // ---- 3. exact reduce of this phase's units of the own shard (unit u on block
        //         u % grid); a chunk is released when the last block holding one of its
        //         units has finished all its units of the phase.  Runs even for a step
        //         that will be skipped (its R is then never read).
        if (ph == 0 && G.b() == 0 && t0) stamp(x, TR_RED_GO);
        unsigned sat = 0;
        if (NV) {
            // this shard's 8-element groups summed by the switch over every rank's wire,
            // NVU units per trip with all their ld_reduce issued first (more bytes in flight)
            constexpr int NVU = 2;
            for (int64_t u0 = lo + G.b(); u0 < hi; u0 += NVU * G.g()) {
                uint4 v[NVU];
                int64_t off[NVU];
#pragma unroll
                for (int i = 0; i < NVU; ++i) {
                    const int64_t su = u0 + i * G.g();
                    const int64_t gi = su * kThreads + threadIdx.x;
                    off[i] = (su < hi && gi < gsh) ? ((int64_t)x.rank * x.lay.shard + (gi << 3)) * 2 : -1;
                    if (off[i] >= 0) v[i] = mm_ld_reduce_f16x8(x.nv_mc + off[i]);
                }
#pragma unroll
                for (int i = 0; i < NVU; ++i) {
                    if (off[i] < 0) continue;
                    v[i].x = sat_inf_f16x2(v[i].x, sat); v[i].y = sat_inf_f16x2(v[i].y, sat);
                    v[i].z = sat_inf_f16x2(v[i].z, sat); v[i].w = sat_inf_f16x2(v[i].w, sat);
                    if (NV == 2) mm_st_16B(x.nv_mc + off[i], v[i]);   // into every rank's wire, in place
                    else *reinterpret_cast<uint4*>(R + (off[i] / 2 - (int64_t)x.rank * x.lay.shard)) = v[i];
                }
            }
        } else if (LMSGD_XGATHER_OWN_IN_REDUCE && a.rout) {
            // lmsgd_exchange: the own shard of the caller's output is written here, so the
            // all-gather (k_xgather) only pulls the other owners' shards
            for (int64_t su = lo + G.b(); su < hi; su += G.g()) {
                const int64_t gi = su * kThreads + threadIdx.x;
                if (gi < gsh)
                    __stcs(reinterpret_cast<uint4*>(a.rout + (int64_t)x.rank * x.lay.shard + (gi << 3)),
                           reduce8_val(recv, x.lay.shard, x.world, gi << 3, R, sat));
            }
        } else {
            for (int64_t su = lo + G.b(); su < hi; su += G.g()) {
                const int64_t gi = su * kThreads + threadIdx.x;
                if (gi < gsh) reduce8(recv, x.lay.shard, x.world, gi << 3, R, sat);
            }
        }
        flush_status(kNone, sat, mine, ST_SUM_SAT);
        // one system fence per block (one thread, after bar.sync), then count this block's
        // units of the phase into their chunks.  (Releasing after every round of units
        // measured slower: the early update blocks compete with the reduce for HBM,
        // profiles/r2/ab/reduce_release_n4.txt.)
        __syncthreads();
        if (t0) {
            __threadfence_system();
            for (int64_t su = lo + G.b(); su < hi; su += G.g()) count_unit(su);
        }
    }
    if (G.b() == 0 && t0) stamp(x, TR_RED_END);

    if (t0) atomicAdd(a.ctr + 1, 1u);   // k_xfinalize waits for every block of this grid
}

// R of a unit: pulled from its owner's R (the all-gather fused into the update), or, after an
// NVLS all-reduce in place (NV == 2, LOCALR), read from this rank's own wire.
__device__ __forceinline__ const uint16_t* r_src(const XArgs& x, bool localr, int owner, int64_t gi) {
    return localr ? reinterpret_cast<const uint16_t*>(x.nv_uc) + (int64_t)owner * x.lay.shard + (gi << 3)
                  : reinterpret_cast<const uint16_t*>(x.peers.base[owner] + x.lay.off_R) + (gi << 3);
}

template <bool RMS, bool WD, bool KM, bool SIM, bool LOCALR, bool V8>
__global__ void LMSGD_LB(LMSGD_XUPD_MINB) k_xupdate(XStep a_, Sim sim) {
    // no griddepcontrol.wait: ordering with k_xstep1 is by the chunk flags.
    // kXUnits units per block (LMSGD_XUNITS): with one acquire per unit (chunk flags
    // carrying the decision), 2 units beat 1 in the step; with the older flag-D protocol
    // 1 had been faster (225 vs 215 us at k = 4).
    __shared__ XStep s_a;
    const XStep& a = rank_args<SIM>(a_, sim, s_a);
    const Grid<SIM> G{sim};
    const XArgs& x = a.x;
    const Ep ep = get_ep(x);
    __shared__ UpdConst s_c;
    __shared__ int s_range;
    if (threadIdx.x == 0) {   // graph mode: this step's coefficients from the device table
        s_c = a.c;
        s_range = 0;
        if (a.ctab) {
            const int64_t idx = *reinterpret_cast<volatile const int64_t*>(a.cursor);
            s_range = idx >= a.ctab_count;
            s_c = a.ctab[s_range ? a.ctab_count - 1 : idx];
        }
    }
    __shared__ int s_ok[kXUnits];
    const int64_t gsh = x.lay.shard >> 3;
    const int64_t ups = (gsh + kThreads - 1) / kThreads;
    const int64_t kcu = (int64_t)x.world * x.lay.cu;
    // chunk-major; inside a chunk owner-major starting with this rank's own units, so that
    // the blocks reducing own units (reduce in the update) come before the blocks of the
    // same chunk that wait for other owners -- also when an emulated group interleaves
    // every rank's blocks in one grid.  (A resident window of ~900 blocks spans dozens of
    // 32-unit owner segments, so every owner's links still see traffic at once.)
    auto unit_of = [&](int v, int& owner, int64_t& u, int& c) {
        const int64_t i = G.b() * kXUnits + v;
        c = (int)(i / kcu);
        const int64_t r = i - (int64_t)c * kcu;
        owner = (int)((r / x.lay.cu + x.rank) % x.world);
        u = c < x.lay.nchunks ? (int64_t)c * x.lay.cu + r % x.lay.cu : ups;   // ups: past the last unit
    };
    int owner[kXUnits];
    int64_t us[kXUnits];
    int cch[kXUnits];
#pragma unroll
    for (int v = 0; v < kXUnits; ++v) unit_of(v, owner[v], us[v], cch[v]);
    // Reduce in the update (riu_active: the step at world > 1 on the peer path): a unit of
    // this rank's own shard is reduced here, from the receive slots every rank pushed
    // before its flag A (warp v acquires all of them, then flag D for the decision), and
    // its R is released to the other ranks per chunk as k_xstep1's reduce does otherwise.
    // Own units are reduced, updated and released BEFORE the block waits for any other
    // owner's chunk: otherwise two ranks' blocks could each hold an own unit while waiting
    // for the other's.
    const int w = threadIdx.x >> 5;
    const bool riu = riu_active(a);
    bool own[kXUnits];
    bool any_own = false;
#pragma unroll
    for (int v = 0; v < kXUnits; ++v) {
        own[v] = riu && owner[v] == x.rank && us[v] < ups;
        any_own = any_own || own[v];
    }
    __shared__ int s_skip;
    if (threadIdx.x == 0) {
        s_skip = 0;
        if (G.b() == 0) stamp(x, TR_UPD_START);
    }
#pragma unroll
    for (int v = 0; v < kXUnits; ++v) s_ok[v] = 1;   // (written by thread 0 of each warp below)
    __syncthreads();
    const UpdConst c = s_c;
    uint4 rv[kXUnits];
    int64_t j0v[kXUnits];
#pragma unroll
    for (int v = 0; v < kXUnits; ++v) {
        const int64_t gi = us[v] * kThreads + threadIdx.x;
        j0v[v] = (us[v] < ups && gi < gsh) ? ((int64_t)owner[v] * gsh + gi) << 3 : x.n;
    }
    if (any_own) {
        // ---- own units: every rank's push is in (flag A), the decision is stored (flag D)
        if (w < kXUnits && own[w]) {
            int ok = warp_wait_all(x, ep, FLAG_A) ? 1 : 0;
            if ((threadIdx.x & 31) == 0) {
                if (ok && !spin_flag(x, ep, flag_slot(x, x.rank, FLAG_D))) {
                    ok = 0;
                    status_of(x, ep, x.rank)[ST_G_ERROR] = (int64_t)LMSGD_ERR_TIMEOUT;
                }
                if (ok) {
                    const volatile int64_t* vm = status_of(x, ep, x.rank);
                    if (vm[ST_G_FIRST] != kNone || vm[ST_G_ERROR] != 0) s_skip = 1;
                }
                s_ok[w] = ok;
            }
        }
        __syncthreads();
        int go = 1;
#pragma unroll
        for (int v = 0; v < kXUnits; ++v) go &= s_ok[v];
        if (!go) return;   // timeout: recorded; the peers time out on this rank's chunks too
        const bool skip = s_skip || s_range;
        unsigned sat = 0;
        if (!skip) {
#pragma unroll
            for (int v = 0; v < kXUnits; ++v) {
                if (!own[v] || j0v[v] >= x.n) continue;
                const int64_t gi = us[v] * kThreads + threadIdx.x;
                rv[v] = reduce8_val(reinterpret_cast<const uint16_t*>(x.peers.base[x.rank] + x.lay.off_recv),
                                    x.lay.shard, x.world, gi << 3,
                                    reinterpret_cast<uint16_t*>(x.peers.base[x.rank] + x.lay.off_R), sat);
                update8<RMS, WD, KM, V8>(rv[v], j0v[v], x.n, c, a.th, a.d, a.m);
            }
        }
        // (padding groups of the last unit -- gi >= gsh -- hold no data: nothing to reduce)
        flush_status(kNone, sat, status_of(x, ep, x.rank), ST_SUM_SAT);
        __syncthreads();
        if (threadIdx.x == 0) {   // release: one fence after bar.sync, then the chunk tickets
            __threadfence_system();
#pragma unroll
            for (int v = 0; v < kXUnits; ++v) {
                if (!own[v]) continue;
                const int64_t rem = ups - (int64_t)cch[v] * x.lay.cu;
                const unsigned cnt = (unsigned)(rem < x.lay.cu ? rem : x.lay.cu);
                if (atomicAdd(a.ctr + 4 + cch[v], 1u) + 1u == cnt) {
                    a.ctr[4 + cch[v]] = 0;
                    __threadfence_system();   // the observed tickets' R writes before the flags
                    const uint32_t fv = cflag_value(x, ep);
                    for (int p = 0; p < x.world; ++p) st_relaxed_sys(cflag(x, p, cch[v], x.rank), fv);
                }
            }
        }
    }
    // ---- other owners' units: lane 0 of warp v waits for unit v's chunk flag (the waits
    //      overlap), even when the step is skipped: the step may end only after every
    //      owner has finished reading its receive slots.  The flag carries the decision.
    bool any_remote = false;
#pragma unroll
    for (int v = 0; v < kXUnits; ++v) any_remote = any_remote || (!own[v] && us[v] < ups);
    if (!any_remote) return;
    if ((threadIdx.x & 31) == 0 && w < kXUnits && !own[w]) {
        int ow, cc;
        int64_t u;
        unit_of(w, ow, u, cc);
        int ok = 1;
        if (u < ups) {
            uint32_t fv;
            if (!spin_cflag(x, ep, cflag(x, x.rank, cc, ow), fv)) {
                ok = 0;
                status_of(x, ep, x.rank)[ST_G_ERROR] = (int64_t)LMSGD_ERR_TIMEOUT;
            } else if (fv & 1u) {
                s_skip = 1;   // skipped step
            }
        }
        s_ok[w] = ok;
    }
    __syncthreads();
    int go = 1;
#pragma unroll
    for (int v = 0; v < kXUnits; ++v) go &= s_ok[v];
    if (G.b() == 0 && threadIdx.x == 0) stamp(x, TR_UPD_GO);
    if (!go || s_skip || s_range) return;
    // every remote unit's R (a peer load) issued before the first update
    // (LMSGD_XUPD_PREFETCH; 0 = load each unit's R right before its update)
#ifndef LMSGD_XUPD_PREFETCH
#define LMSGD_XUPD_PREFETCH 1
#endif
#pragma unroll
    for (int v = 0; v < kXUnits; ++v)
        if (LMSGD_XUPD_PREFETCH && !own[v] && j0v[v] < x.n)
            rv[v] = *reinterpret_cast<const uint4*>(r_src(x, LOCALR, owner[v], us[v] * kThreads + threadIdx.x));
#pragma unroll
    for (int v = 0; v < kXUnits; ++v) {
        if (own[v] || j0v[v] >= x.n) continue;
        if (!LMSGD_XUPD_PREFETCH)
            rv[v] = *reinterpret_cast<const uint4*>(r_src(x, LOCALR, owner[v], us[v] * kThreads + threadIdx.x));
        update8<RMS, WD, KM, V8>(rv[v], j0v[v], x.n, c, a.th, a.d, a.m);
    }
}

// lmsgd_exchange, world > 1: the all-gather half of the fp16 all-reduce (row a4) on
// its own, as a flat pull into the caller's buffer.  Same unit order and waits as
// k_xupdate (chunk-major, owner-interleaved; the owner's chunk flag),
// then one 16-byte peer load and one local store per thread.  The reduced values
// are copied whether or not a gradient was non-finite (the status says so).
// Measured (k = 2, 51 MB): 123 us for the whole exchange, against 137 us with the
// gather done inside k_xstep1's persistent grid after its reduce; 2, 4 or 8 units per
// block with overlapped flag waits change nothing (k = 4, 158.5-159.7 us,
// profiles/r1/ab/gather_units_n4.txt): the pull is NVLink-bound (~600 GB/s in).  The
// exchange moves 2 x 2 N (k-1)/k bytes out of every GPU (push, then R served to the
// peers), 76.7 MB at k = 4: 118 us at the ~650 GB/s an SM store stream reaches.
#ifndef LMSGD_XGATHER_UNITS
#define LMSGD_XGATHER_UNITS 1   // units per k_xgather block (A/B knob)
#endif
constexpr int kGUnits = LMSGD_XGATHER_UNITS;
template <bool SIM, bool LOCALR>
__global__ void __launch_bounds__(kThreads) k_xgather(XStep a_, Sim sim) {
    __shared__ XStep s_a;
    const XStep& a = rank_args<SIM>(a_, sim, s_a);
    const XArgs& x = a.x;
    const Ep ep = get_ep(x);
    const int64_t gsh = x.lay.shard >> 3;
    const int64_t ups = (gsh + kThreads - 1) / kThreads;
    const int64_t kcu = (int64_t)x.world * x.lay.cu;
    // kGUnits consecutive units of the chunk-major, owner-interleaved order per block; lane
    // v of warp 0 waits for unit v's chunk flag (the waits overlap), then every thread
    // issues its units' peer loads before the local stores
    auto unit_of = [&](int v, int& owner, int64_t& u, int& c) {
        const int64_t i = Grid<SIM>{sim}.b() * kGUnits + v;
        c = (int)(i / kcu);
        const int64_t r = i - (int64_t)c * kcu;
        owner = (int)((r % x.world + x.rank) % x.world);
        u = c < x.lay.nchunks ? (int64_t)c * x.lay.cu + r / x.world : ups;
    };
    // the own shard was written by k_xstep1's reduce (peer path)
    auto own_done = [&](int owner) { return LMSGD_XGATHER_OWN_IN_REDUCE && x.nv == 0 && owner == x.rank; };
    __shared__ int s_go;
    if (threadIdx.x == 0 && Grid<SIM>{sim}.b() == 0) stamp(x, TR_UPD_START);
    if (threadIdx.x < 32) {
        int go = 1;
        if ((int)threadIdx.x < kGUnits) {
            int owner, c;
            int64_t u;
            unit_of(threadIdx.x, owner, u, c);
            uint32_t fv;
            if (u < ups && !own_done(owner) && !spin_cflag(x, ep, cflag(x, x.rank, c, owner), fv)) {
                go = 0;
                status_of(x, ep, x.rank)[ST_G_ERROR] = (int64_t)LMSGD_ERR_TIMEOUT;
            }
        }
        go = __all_sync(0xffffffffu, go);
        if (threadIdx.x == 0) s_go = go;
        if (threadIdx.x == 0 && Grid<SIM>{sim}.b() == 0) stamp(x, TR_UPD_GO);
    }
    __syncthreads();
    if (!s_go) return;
    uint4 v[kGUnits];
    int64_t dst[kGUnits];
#pragma unroll
    for (int q = 0; q < kGUnits; ++q) {
        int owner, c;
        int64_t u;
        unit_of(q, owner, u, c);
        const int64_t gi = u * kThreads + threadIdx.x;
        dst[q] = (u < ups && gi < gsh && !own_done(owner)) ? (((int64_t)owner * gsh + gi) << 3) : -1;
        if (dst[q] >= 0) v[q] = *reinterpret_cast<const uint4*>(r_src(x, LOCALR, owner, gi));
    }
#pragma unroll
    for (int q = 0; q < kGUnits; ++q)
        if (dst[q] >= 0) __stcs(reinterpret_cast<uint4*>(a.rout + dst[q]), v[q]);
}

// lmsgd_exchange, world == 1: the step's public status record (R = h, no second
// rounding), and the next call's status slot cleared.
__global__ void k_xfinal1(const int64_t* st, int64_t* st_next, int64_t* last) {
    pdl_enter();
    if (threadIdx.x == 0)
        store_last(last, st[ST_FIRST], st[ST_PACK_SAT], 0, st[ST_ERROR], st[ST_FIRST] != kNone ? 1 : 0);
    if (threadIdx.x < ST_WORDS) reset_words(st_next);
}

// lmsgd_status_accumulate: merge one context's last status record (lmsgd_step_status
// layout) into a sub-step accumulator {first (kNone = none), pack_sat, sum_sat, error}.
__global__ void k_status_acc(const int64_t* last, int64_t offset, int64_t* acc) {
    if (threadIdx.x != 0) return;
    const int64_t first = last[0];
    if (first >= 0 && offset + first < acc[ST_FIRST]) acc[ST_FIRST] = offset + first;
    acc[ST_PACK_SAT] += last[1];
    acc[ST_SUM_SAT] += last[2];
    const int32_t err = reinterpret_cast<const int32_t*>(last + 3)[1];
    if (err != 0 && err != (int32_t)LMSGD_ERR_NONFINITE && acc[ST_ERROR] == 0) acc[ST_ERROR] = err;
}

// The step's public status record; runs after k_xupdate (every owner's reduce has
// been observed by then, so every rank's sum saturation count is final).
template <bool SIM>
__global__ void k_xfinalize(XStep a_, Sim sim, unsigned int xstep1_blocks) {
    pdl_enter();
    __shared__ XStep s_a;
    const XStep& a = rank_args<SIM>(a_, sim, s_a);
    const XArgs& x = a.x;
    const Ep ep = get_ep(x);
    if (threadIdx.x != 0) return;
    // k_xupdate may complete before k_xstep1 (it never waits for its grid): the step
    // ends only once every k_xstep1 block has retired its last memory operation
    while (ld_acquire_sys(a.ctr + 1) < xstep1_blocks) __nanosleep(64);
    a.ctr[1] = 0;
    const volatile int64_t* mine = status_of(x, ep, x.rank);
    const int64_t gfirst = mine[ST_G_FIRST];
    int64_t err = mine[ST_G_ERROR];
    if (!err && a.ctab && *a.cursor >= a.ctab_count) err = (int64_t)LMSGD_ERR_RANGE;   // table exhausted
    const bool skip = gfirst != kNone || err != 0;
    // every rank's phases have been pushed and reduced by now: its pack and sum saturation
    // counts are final (a skipped step reports no sum saturations)
    int64_t ssat = 0, psat = 0;
    for (int p = 0; p < x.world; ++p) {
        const volatile int64_t* sp = status_of(x, ep, p);
        psat += sp[ST_PACK_SAT];
        if (!skip) ssat += sp[ST_SUM_SAT];
    }
    store_last(a.last, gfirst, psat, ssat, err, skip);
    stamp(x, TR_UPD_END);
    // the step is complete on this GPU: advance the device step counter (and cursor)
    if (a.cursor) *a.cursor += 1;
    *a.x.dev_epoch = ep.e;
}

// BN statistics without moving averages, one cooperative kernel
// (all blocks co-resident): stage [mean | var] in this rank's exchange buffer, one
// system fence per block, the last block releases flag C, every block acquires C of
// all ranks, then averages its slice over the ranks' staging buffers in rank order,
// in fp64, one rounding to fp32 (R16).  Double-buffered by call parity.
template <bool SIM>
__global__ void __launch_bounds__(kThreads) k_bn_allreduce(BnArgs a_, Sim sim) {
    __shared__ BnArgs s_a;
    const BnArgs& a = rank_args<SIM>(a_, sim, s_a);
    const Grid<SIM> G{sim};
    const XArgs& x = a.x;
    float* __restrict__ mean = a.mean;
    float* __restrict__ var = a.var;
    const int64_t C = a.C;
    const int64_t gt = G.b() * blockDim.x + threadIdx.x, gs = G.g() * blockDim.x;
    const Ep ep = get_ep(x);
    __shared__ int s_ok;
    const int64_t Cp = (C + 3) & ~int64_t(3);   // var staged at a 16-B aligned offset
    const int64_t off = (int64_t)ep.par * 2 * LMSGD_MAX_BN_CHANNELS;
    float* stage = reinterpret_cast<float*>(x.peers.base[x.rank] + x.lay.off_bn) + off;
    for (int64_t i = gt; i < C; i += gs) {
        stage[i] = mean[i];
        stage[Cp + i] = var[i];
    }
    if (grid_last(x, FLAG_C, G.g())) {
        publish(x, ep, FLAG_C);
        *x.dev_epoch = ep.e;   // every block has read the call counter by now
    }
    if (threadIdx.x < 32) {
        const bool ok = warp_wait_all(x, ep, FLAG_C);
        if (threadIdx.x == 0) s_ok = ok ? 1 : 0;
    }
    __syncthreads();
    if (!s_ok) return;
    // one float4 of every rank per thread, all peer loads issued before the sums
    for (int64_t f = gt; f < Cp / 2; f += gs) {
        float4 v[LMSGD_MAX_WORLD];
#pragma unroll
        for (int p = 0; p < LMSGD_MAX_WORLD; ++p)
            if (p < x.world)
                v[p] = reinterpret_cast<const float4*>(reinterpret_cast<const float*>(x.peers.base[p] + x.lay.off_bn) + off)[f];
        double a0 = 0, a1 = 0, a2 = 0, a3 = 0;
#pragma unroll
        for (int p = 0; p < LMSGD_MAX_WORLD; ++p)
            if (p < x.world) { a0 += v[p].x; a1 += v[p].y; a2 += v[p].z; a3 += v[p].w; }
        const double kk = (double)x.world;
        const float o[4] = {(float)(a0 / kk), (float)(a1 / kk), (float)(a2 / kk), (float)(a3 / kk)};
        const int64_t e0 = f * 4;
        for (int e = 0; e < 4; ++e) {
            const int64_t i = e0 + e;
            if (i < C) mean[i] = o[e];
            else if (i >= Cp && i - Cp < C) var[i - Cp] = o[e];
        }
    }
}

// Flat grids: one 8-element group per thread, one wave of short-lived blocks.
// Measured (tools/ubench.cu, B200): 98 us for the 25.6M update vs 124 us for a
// persistent grid-stride grid of SMs x resident blocks.
int grid_for(const Launch&, int64_t work_items) {
    int64_t blocks = (work_items + kThreads - 1) / kThreads;
    if (blocks > 0x7fffffff) blocks = 0x7fffffff;  // grid-stride loops cover the rest
    return blocks < 1 ? 1 : (int)blocks;
}

}  // namespace

// ------------------------------------------------------------------ launchers

// The update's kernel instantiation for a step: RMS (alpha_RMSprop != 0, or unknown
// on the host in graph mode), WD (weight decay on), KM (m kept: not FREEZE_M).
struct UpdateK { template <bool R, bool W, bool K, bool V> static constexpr auto get() { return k_update<R, W, K, V>; } };
struct Fused1K { template <bool R, bool W, bool K, bool V> static constexpr auto get() { return k_fused1<R, W, K, V>; } };
template <bool SIM, bool LOCALR>
struct XUpdateK {
    template <bool R, bool W, bool K, bool V> static constexpr auto get() { return k_xupdate<R, W, K, SIM, LOCALR, V>; }
};
template <typename K>
auto pick_variant(const UpdConst& c, bool graph, bool v8) {
    const bool rms = c.a_rms != 0.0f || graph, wd = c.n_wd > 0, km = rms || !c.freeze_m;
    if (v8) {
        if (rms) return wd ? K::template get<true, true, true, true>() : K::template get<true, false, true, true>();
        if (km) return wd ? K::template get<false, true, true, true>() : K::template get<false, false, true, true>();
        return wd ? K::template get<false, true, false, true>() : K::template get<false, false, false, true>();
    }
    if (rms) return wd ? K::template get<true, true, true, false>() : K::template get<true, false, true, false>();
    if (km) return wd ? K::template get<false, true, true, false>() : K::template get<false, false, true, false>();
    return wd ? K::template get<false, true, false, false>() : K::template get<false, false, false, false>();
}

// 256-bit accesses need 32-byte aligned rows: every pointer of the launch (NULLs ignored)
__host__ inline bool aligned32(std::initializer_list<const void*> ps) {
    for (const void* p : ps)
        if (p && (reinterpret_cast<uintptr_t>(p) & 31u)) return false;
    return true;
}

// Launch with the programmatic-stream-serialization attribute (see pdl_enter).
template <typename... KArgs, typename... Args>
cudaError_t launch_pdl_if(bool pdl, void (*kernel)(KArgs...), int grid, int block, cudaStream_t s,
                          Args&&... args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)grid);
    cfg.blockDim = dim3((unsigned)block);
    cfg.dynamicSmemBytes = 0;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = pdl ? 1 : 0;
    return cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...);
}
#define launch_pdl(...) launch_pdl_if((L.pdl_mask & 1) != 0, __VA_ARGS__)



int xstep_default_bps() { return LMSGD_XSTEP_BPS_DEFAULT; }

int xstep_blocks_per_sm(bool sim) {
    int b = 0;
    // every instantiation shares the grid size: take the smallest occupancy
    auto occ = [&](auto k) {
        int v = 0;
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&v, k, kThreads, 0);
        b = (b == 0 || v < b) ? v : b;
    };
    if (sim) {
        occ(k_xstep1<true, 0>);
    } else {
        occ(k_xstep1<false, 0>);
        occ(k_xstep1<false, 1>);
        occ(k_xstep1<false, 2>);
    }
    return b > 0 ? b : 1;
}

// One world > 1 step (or exchange) of this rank: k_xstep1 (cooperative + PDL), then
// k_xupdate or k_xgather (PDL), then k_xfinalize.  Group mode (d_group != NULL): the
// same kernels' SIM instantiations carry `nsim` emulated ranks' grids in each launch;
// `a` is then any rank's arguments (sizes, kernel variant), the kernels read their
// rank's entry of d_group.
cudaError_t launch_xstep(cudaStream_t s, const Launch& L, const XStep& a, const XStep* d_group, int nsim) {
    const bool sim = d_group != nullptr;
    if (!sim) nsim = 1;
    const Sim sm{d_group, nsim};
    // per-rank k_xstep1 grid: all nsim grids co-resident
    const int bps_sim = xstep_blocks_per_sm(true) < LMSGD_XSTEP_BPS_DEFAULT ? xstep_blocks_per_sm(true)
                                                                          : LMSGD_XSTEP_BPS_DEFAULT;
    const int per_rank = sim ? (L.sm_count * bps_sim) / nsim : L.grid_xstep;
    XStep arg = a;
    cudaError_t e;
    {
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3((unsigned)(per_rank * nsim));
        cfg.blockDim = dim3(kThreads);
        cfg.stream = s;
        cudaLaunchAttribute attr[2];
        attr[0].id = cudaLaunchAttributeCooperative;   // all blocks co-resident: they wait on each other
        attr[0].val.cooperative = 1;
        attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        attr[1].val.programmaticStreamSerializationAllowed = 1;
        cfg.attrs = attr;
        cfg.numAttrs = (L.pdl_mask & 2) ? 2 : 1;   // + programmatic dependent launch (hides the launch latency)
        const int nv = sim ? 0 : a.x.nv;
        e = sim       ? cudaLaunchKernelEx(&cfg, k_xstep1<true, 0>, arg, sm)
            : nv == 1 ? cudaLaunchKernelEx(&cfg, k_xstep1<false, 1>, arg, sm)
            : nv == 2 ? cudaLaunchKernelEx(&cfg, k_xstep1<false, 2>, arg, sm)
                      : cudaLaunchKernelEx(&cfg, k_xstep1<false, 0>, arg, sm);
    }
    if (e != cudaSuccess) return e;
    const bool pdl = (L.pdl_mask & 4) == 0;   // bit 4 (diagnostics): launch k_xupdate after k_xstep1 completes
    const bool localr = !sim && a.x.nv == 2;   // NVLS all-reduce in place: R is in the own wire
    if (a.rout) {   // lmsgd_exchange: the all-gather into the caller's buffer instead of the update
        const int grid = (int)(((int64_t)a.x.lay.nchunks * a.x.world * a.x.lay.cu + kGUnits - 1) / kGUnits) * nsim;
        e = sim      ? launch_pdl_if(pdl, k_xgather<true, false>, grid, kThreads, s, a, sm)
            : localr ? launch_pdl_if(pdl, k_xgather<false, true>, grid, kThreads, s, a, sm)
                     : launch_pdl_if(pdl, k_xgather<false, false>, grid, kThreads, s, a, sm);
    } else {
        const int grid = (int)(((int64_t)a.x.lay.nchunks * a.x.world * a.x.lay.cu + kXUnits - 1) / kXUnits) * nsim;
        const bool g = a.ctab != nullptr;
        // the 256-bit variant needs every rank's state 32-byte aligned (a.v8: set by the caller
        // over all ranks of an emulated group); not with m frozen, where it measured slower
        // at k > 1 (172.6 vs 169.7 us at k = 4, profiles/r2/ab/v8_xupdate.txt)
        const bool frozen = a.c.freeze_m && a.c.a_rms == 0.0f && !g;
        const bool v8 = a.v8 && aligned32({a.th, a.d, a.m}) && !frozen;
        e = sim      ? launch_pdl_if(pdl, pick_variant<XUpdateK<true, false>>(a.c, g, v8), grid, kThreads, s, a, sm)
            : localr ? launch_pdl_if(pdl, pick_variant<XUpdateK<false, true>>(a.c, g, v8), grid, kThreads, s, a, sm)
                     : launch_pdl_if(pdl, pick_variant<XUpdateK<false, false>>(a.c, g, v8), grid, kThreads, s, a, sm);
    }
    if (e != cudaSuccess) return e;
    return sim ? launch_pdl_if(true, k_xfinalize<true>, nsim, 32, s, a, sm, (unsigned int)per_rank)
               : launch_pdl_if(true, k_xfinalize<false>, 1, 32, s, a, sm, (unsigned int)per_rank);
}


int stream_blocks_per_sm() {
    int worst = 1 << 30, b = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, k_update<true, false, true, false>, kThreads, 0);
    worst = b < worst ? b : worst;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, k_fused1<true, false, true, false>, kThreads, 0);  // NOLINT
    worst = b < worst ? b : worst;
    return worst > 0 ? worst : 1;
}

cudaError_t launch_status_reset(cudaStream_t s, int64_t* st) {
    k_status_reset<<<1, 32, 0, s>>>(st, 4);  // the public sub-step status is int64[4]
    return cudaGetLastError();
}

cudaError_t launch_pack(cudaStream_t s, const Launch& L, const float* g, int64_t n, int64_t n_pad,
                        float scale, uint16_t* h, int64_t* st, const Dev1& dv) {
    return launch_pdl(aligned32({g}) ? k_pack<true> : k_pack<false>, grid_for(L, n_pad >> 3), kThreads, s, g, n,
                      n_pad, scale, h, st, dv);
}

cudaError_t launch_reduce_local(cudaStream_t s, const Launch& L, const uint16_t* h, int k,
                                int64_t n_pad, uint16_t* R, int64_t* st) {
    return launch_pdl(k_reduce_local, grid_for(L, n_pad >> 3), kThreads, s, h, k, n_pad, R, st);
}

cudaError_t launch_update(cudaStream_t s, const Launch& L, const uint16_t* R, int64_t n,
                          const UpdConst& c, float* th, float* d, float* m, const int64_t* st,
                          int64_t* st_reset, int64_t* last, const Dev1& dv) {
    const int grid = grid_for(L, (n + 7) >> 3);
    // graph mode: alpha_RMSprop is only known on the device
    return launch_pdl(pick_variant<UpdateK>(c, dv.epoch != nullptr, aligned32({th, d, m})), grid, kThreads, s, R, n,
                      c, th, d, m, st,
                      st_reset, last, dv);
}

cudaError_t launch_fused1(cudaStream_t s, const Launch& L, const float* g, int64_t n, float scale,
                          const UpdConst& c, float* th, float* d, float* m, int64_t* st,
                          int64_t* st_reset, int64_t* /*last: see launch_finalize_fused*/, const Dev1& dv) {
    const int grid = grid_for(L, (n + 7) >> 3);
    return launch_pdl(pick_variant<Fused1K>(c, dv.epoch != nullptr, aligned32({g, th, d, m})), grid, kThreads, s, g,
                      n, scale, c, th, d, m,
                      st, st_reset, dv);
}

int64_t host_units(const XArgs& x) {
    const int64_t gsh = x.lay.shard >> 3;
    return (int64_t)x.world * ((gsh + kThreads - 1) / kThreads);
}

cudaError_t launch_advance1(cudaStream_t s, const Dev1& dv, int64_t* last, bool fused) {
    return launch_pdl_if(true, k_advance1, 1, 32, s, dv, last, fused ? 1 : 0);
}

cudaError_t launch_xfinal1(cudaStream_t s, const int64_t* st, int64_t* st_next, int64_t* last) {
    return launch_pdl_if(true, k_xfinal1, 1, 32, s, st, st_next, last);
}

cudaError_t launch_step_oop1(cudaStream_t s, const Launch& L, const float* g, int64_t n, float scale,
                             const UpdConst& c, const float* thi, const float* di, const float* mi, float* tho,
                             float* dout, float* mo, int64_t* st, int64_t* st_reset, int64_t* last,
                             int64_t* trace) {
    const int grid = grid_for(L, (n + 7) >> 3);
    const bool v8 = aligned32({g, thi, di, mi, tho, dout, mo});
    cudaError_t e = launch_pdl(c.a_rms != 0.0f ? (v8 ? k_fused1_oop<true, true> : k_fused1_oop<true, false>)
                                               : (v8 ? k_fused1_oop<false, true> : k_fused1_oop<false, false>),
                               grid, kThreads, s, g, n,
                               scale, c, thi, di, mi, tho, dout, mo, st, st_reset, trace);
    if (e != cudaSuccess) return e;
#ifndef LMSGD_REPAIR_BLOCKS
#define LMSGD_REPAIR_BLOCKS 32   // 0: one block per SM
#endif
    const int rb = LMSGD_REPAIR_BLOCKS > 0 ? LMSGD_REPAIR_BLOCKS : L.sm_count;
    return launch_pdl_if(true, k_repair1, rb, 512, s, (const int64_t*)st, thi, di, mi, tho, dout, mo, n, last, trace);
}

cudaError_t launch_status_accumulate(cudaStream_t s, const int64_t* last, int64_t offset, int64_t* acc) {
    k_status_acc<<<1, 32, 0, s>>>(last, offset, acc);
    return cudaGetLastError();
}

cudaError_t launch_finalize_fused(cudaStream_t s, const int64_t* st, int64_t* last) {
    return launch_pdl_if(true, k_finalize_fused, 1, 32, s, st, last);
}




cudaError_t launch_bn_allreduce(cudaStream_t s, const BnArgs& a, const BnArgs* d_group, int nsim) {
    const bool sim = d_group != nullptr;
    if (!sim) nsim = 1;
    int grid = (int)(((a.C + 3) / 4 * 2 + kThreads - 1) / kThreads);   // one float4 per thread
    grid = grid > 148 ? 148 : (grid < 1 ? 1 : grid);
    if (sim) {   // every emulated rank's grid co-resident
        int b = 0;
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, k_bn_allreduce<true>, kThreads, 0);
        int dev = 0, sms = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        const int cap = (b > 0 ? b : 1) * sms / nsim;
        grid = grid > cap ? cap : grid;
    }
    BnArgs arg = a;
    Sim sm{d_group, nsim};
    void* params[] = {&arg, &sm};
    return cudaLaunchCooperativeKernel(sim ? (const void*)k_bn_allreduce<true> : (const void*)k_bn_allreduce<false>,
                                       dim3((unsigned)(grid * nsim)), dim3(kThreads), params, 0, s);
}

}  // namespace lmsgd
