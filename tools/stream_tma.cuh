// Bulk-copy (TMA engine, cp.async.bulk) staged streaming kernels for sm_100a.
//
// Included by kernels.cu inside lmsgd::{anon} after the per-element helpers
// (upd1, pack8, flush_status).  One CTA per SM: warp 8 lane 0 is the producer and
// streams tiles of the wire values (fp16 R, or fp32 g for the fused k = 1 step) and
// of theta, Delta, m into a STAGES-deep shared-memory ring with
// cp.async.bulk ... mbarrier::complete_tx; warps 0-7 compute the blended update in
// place in shared memory and one elected thread writes theta, Delta, m back with
// cp.async.bulk shared -> global.  No register staging of the loads, so the bytes
// in flight per SM are set by the ring depth, not by occupancy.
#pragma once

// Development variant (tools/ubench.cu), not linked into liblmsgd.so: on B200 the
// flat LDG.128 kernels measured faster.

// pack of 4 values (j0 % 4 == 0), same rule as pack8.
__device__ __forceinline__ uint2 pack4(float4 x, float s, int64_t j0, int64_t& first, unsigned& sat) {
    const float v[4] = {x.x, x.y, x.z, x.w};
    float y[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        const bool bad = nonfinite(v[i]);
        if (bad) first = (j0 + i) < first ? (j0 + i) : first;
        y[i] = s * v[i];
        sat += (!bad && fabsf(y[i]) > 65504.0f) ? 1u : 0u;
    }
    return make_uint2(cvt_sat_f16x2(y[0], y[1]), cvt_sat_f16x2(y[2], y[3]));
}


__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, unsigned count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}

__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, unsigned bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
}

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred P1;\n"
        "LAB_WAIT:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
        "@P1 bra DONE;\n\t"
        "bra LAB_WAIT;\n"
        "DONE:\n}\n" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}

__device__ __forceinline__ uint64_t policy_evict_first() {
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
    return p;
}

__device__ __forceinline__ uint64_t policy_evict_last() {
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
    return p;
}

// global -> shared bulk copy completing on an mbarrier, with an L2 eviction policy.
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes, uint64_t* bar,
                                         uint64_t pol) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
            smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(pol)
        : "memory");
}

// shared -> global bulk copy (bulk async-group of the issuing thread).
__device__ __forceinline__ void bulk_s2g(void* dst, const void* src, unsigned bytes, uint64_t pol) {
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group.L2::cache_hint [%0], [%1], %2, %3;" ::"l"(dst),
                 "r"(smem_u32(src)), "r"(bytes), "l"(pol)
                 : "memory");
}

__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }

template <int N>
__device__ __forceinline__ void bulk_wait_read() {
    asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(N) : "memory");
}

template <int N>
__device__ __forceinline__ void bulk_wait() {
    asm volatile("cp.async.bulk.wait_group %0;" ::"n"(N) : "memory");
}

__device__ __forceinline__ void fence_proxy_async_smem() {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

__device__ __forceinline__ void consumer_bar() {  // warps 0-7 only
    asm volatile("bar.sync 1, 256;" ::: "memory");
}

constexpr int kTmaConsumers = 256;
constexpr int kTmaThreads = kTmaConsumers + 32;

template <bool FUSED, int TE>
__host__ __device__ constexpr int tma_stage_bytes() {
    return TE * ((FUSED ? 4 : 2) + 12);
}

// Blended update of [0, n8) (n8 = n rounded down to a multiple of 8) from the
// fp16 wire R (FUSED = false) or from g packed in registers (FUSED = true); the
// last n - n8 elements are done by CTA 0 with plain loads.  Same per-element
// arithmetic as update8 (upd1), hence bit-identical results.
template <bool RMS, bool FUSED, int TE, int STAGES>
__global__ void __launch_bounds__(kTmaThreads, 1)
    k_stream_tma(const void* __restrict__ wire, int64_t n, float s, UpdConst c, float* __restrict__ th,
                 float* __restrict__ d, float* __restrict__ m, const int64_t* st_in, int64_t* st_out) {
    extern __shared__ __align__(128) unsigned char smem[];
    __shared__ __align__(8) uint64_t full[STAGES], empty[STAGES];
    constexpr int WB = FUSED ? 4 : 2;
    constexpr int SB = tma_stage_bytes<FUSED, TE>();
    if (!FUSED && st_in && (st_in[ST_FIRST] != kNone || st_in[ST_ERROR] != 0)) return;  // guarded skip
    const int64_t n8 = n & ~int64_t(7);
    const int64_t ntiles = (n8 + TE - 1) / TE;
    if (threadIdx.x == 0) {
        for (int i = 0; i < STAGES; ++i) {
            mbar_init(&full[i], 1);
            mbar_init(&empty[i], 1);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    const int warp = threadIdx.x >> 5;
    int64_t first = kNone;
    unsigned sat = 0;
    if (warp == 8) {
        if ((threadIdx.x & 31) == 0) {  // producer
            const uint64_t pol = policy_evict_first();
            int it = 0;
            for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x, ++it) {
                const int si = it % STAGES;
                const uint32_t u = it / STAGES;
                if (it >= STAGES) mbar_wait(&empty[si], (u & 1) ^ 1);
                const int64_t e0 = tile * TE;
                const unsigned cnt = (unsigned)((n8 - e0) < TE ? (n8 - e0) : TE);
                unsigned char* sb = smem + si * SB;
                mbar_expect_tx(&full[si], cnt * (WB + 12));
                bulk_g2s(sb, static_cast<const char*>(wire) + e0 * WB, cnt * WB, &full[si], pol);
                bulk_g2s(sb + TE * WB, th + e0, cnt * 4, &full[si], pol);
                bulk_g2s(sb + TE * WB + TE * 4, d + e0, cnt * 4, &full[si], pol);
                bulk_g2s(sb + TE * WB + TE * 8, m + e0, cnt * 4, &full[si], pol);
            }
        }
    } else {
        const int tid = threadIdx.x;
        const uint64_t pol = policy_evict_first();
        int it = 0;
        for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x, ++it) {
            const int si = it % STAGES;
            const uint32_t u = it / STAGES;
            mbar_wait(&full[si], u & 1);
            const int64_t e0 = tile * TE;
            const int cnt = (int)((n8 - e0) < TE ? (n8 - e0) : TE);
            unsigned char* sb = smem + si * SB;
            float* ts = reinterpret_cast<float*>(sb + TE * WB);
            float* ds = ts + TE;
            float* ms = ds + TE;
            static_assert(TE % (4 * kTmaConsumers) == 0, "tile = whole float4 rows of the consumers");
#pragma unroll
            for (int q = 0; q < TE / (4 * kTmaConsumers); ++q) {
                const int e = q * 4 * kTmaConsumers + tid * 4;
                if (e < cnt) {
                    float gh[4];
                    if (FUSED) {
                        const float4 gv = reinterpret_cast<const float4*>(sb)[e >> 2];
                        const uint2 h = pack4(gv, s, e0 + e, first, sat);
                        gh[0] = h2f(h.x, 0) * c.inv_ks; gh[1] = h2f(h.x, 1) * c.inv_ks;
                        gh[2] = h2f(h.y, 0) * c.inv_ks; gh[3] = h2f(h.y, 1) * c.inv_ks;
                    } else {
                        const uint2 r = reinterpret_cast<const uint2*>(sb)[e >> 2];
                        gh[0] = h2f(r.x, 0) * c.inv_ks; gh[1] = h2f(r.x, 1) * c.inv_ks;
                        gh[2] = h2f(r.y, 0) * c.inv_ks; gh[3] = h2f(r.y, 1) * c.inv_ks;
                    }
                    float4 tv = reinterpret_cast<float4*>(ts)[e >> 2];
                    float4 dv = reinterpret_cast<float4*>(ds)[e >> 2];
                    float4 mv = reinterpret_cast<float4*>(ms)[e >> 2];
                    upd1<RMS>(gh[0], tv.x, dv.x, mv.x, c);
                    upd1<RMS>(gh[1], tv.y, dv.y, mv.y, c);
                    upd1<RMS>(gh[2], tv.z, dv.z, mv.z, c);
                    upd1<RMS>(gh[3], tv.w, dv.w, mv.w, c);
                    reinterpret_cast<float4*>(ts)[e >> 2] = tv;
                    reinterpret_cast<float4*>(ds)[e >> 2] = dv;
                    reinterpret_cast<float4*>(ms)[e >> 2] = mv;
                }
            }
            fence_proxy_async_smem();
            consumer_bar();
            if (tid == 0) {
                bulk_s2g(th + e0, ts, cnt * 4, pol);
                bulk_s2g(d + e0, ds, cnt * 4, pol);
                bulk_s2g(m + e0, ms, cnt * 4, pol);
                bulk_commit();
                bulk_wait_read<0>();
                mbar_arrive(&empty[si]);
            }
        }
        if (tid == 0) bulk_wait<0>();
    }
    // ragged tail (< 8 elements): CTA 0, one thread, plain loads
    if (blockIdx.x == 0 && threadIdx.x == 0 && n8 < n) {
        float x8[8];
        if (FUSED) {
            const float* g = static_cast<const float*>(wire);
            for (int i = 0; i < 8; ++i) x8[i] = (n8 + i < n) ? g[n8 + i] : 0.0f;
            const uint4 h = pack8(x8, s, n8, first, sat);
            update8<RMS, false>(h, n8, n, c, th, d, m);
        } else {
            const uint4 r = *reinterpret_cast<const uint4*>(static_cast<const uint16_t*>(wire) + n8);
            update8<RMS, false>(r, n8, n, c, th, d, m);
        }
    }
    if (FUSED && st_out) {
        // warps 0..8 all reach here; flush_status needs full warps
        flush_status(first, sat, st_out, ST_PACK_SAT);
    }
}
