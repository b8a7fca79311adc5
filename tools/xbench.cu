// Multi-GPU exchange-kernel micro-benchmark (development tool): one process drives
// every visible GPU (<= 8) with peer access; data is static, so no flags are needed.
// Measures the phases of the world > 1 step in isolation, all GPUs concurrently.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I include \
//        -I paper_1711_04325_b200/csrc tools/xbench.cu -o tools/xbench
#include "../paper_1711_04325_b200/csrc/kernels.cu"

namespace lmsgd {
namespace {
#include "stream_tma.cuh"   // tools/: the TMA-staged development variant
}  // namespace
}  // namespace lmsgd

#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <functional>
#include <vector>

using namespace lmsgd;

#define CKE(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s at %d\n", cudaGetErrorString(e), __LINE__); exit(1);} } while (0)

namespace xb {

// exact reduce with integer accumulation: fp16 -> fixed point (units of 2^-24)
__device__ __forceinline__ long long h2fix(uint32_t b) {
    const int e = (b >> 10) & 31;
    const long long f = b & 1023;
    long long v = e ? ((1024 + f) << (e - 1)) : f;
    return (b & 0x8000) ? -v : v;
}

template <int MODE>   // 0: fp64 flat (production arithmetic), 1: int64 flat, 2: int64 persistent
__global__ void __launch_bounds__(256) k_reduce(const uint16_t* __restrict__ recv, int k, int64_t shard,
                                                uint16_t* __restrict__ R) {
    const int64_t nv = shard >> 3;
    for (int64_t v = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; v < nv; v += (int64_t)gridDim.x * blockDim.x) {
        const int64_t j0 = v << 3;
        unsigned short o[8];
        unsigned sat = 0;
        if (MODE == 0) {
            double acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
            for (int p = 0; p < k; ++p) {
                const uint4 q = *reinterpret_cast<const uint4*>(recv + (int64_t)p * shard + j0);
                const uint32_t w[4] = {q.x, q.y, q.z, q.w};
#pragma unroll
                for (int e = 0; e < 8; ++e) acc[e] += (double)h2f(w[e >> 1], e & 1);
            }
#pragma unroll
            for (int e = 0; e < 8; ++e) o[e] = sat16_f64(acc[e], sat);
        } else {
            long long acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
            for (int p = 0; p < k; ++p) {
                const uint4 q = *reinterpret_cast<const uint4*>(recv + (int64_t)p * shard + j0);
                const uint32_t w[4] = {q.x, q.y, q.z, q.w};
#pragma unroll
                for (int e = 0; e < 8; ++e) acc[e] += h2fix((e & 1) ? (w[e >> 1] >> 16) : (w[e >> 1] & 0xffff));
            }
#pragma unroll
            for (int e = 0; e < 8; ++e) o[e] = sat16_f64((double)acc[e] * 0x1p-24, sat);
        }
        *reinterpret_cast<uint4*>(R + j0) = make_uint4(o[0] | (uint32_t)o[1] << 16, o[2] | (uint32_t)o[3] << 16,
                                                      o[4] | (uint32_t)o[5] << 16, o[6] | (uint32_t)o[7] << 16);
    }
}

struct Ptrs { const uint16_t* R[8]; };

// update with R pulled from owners (interleaved units), like k_update_gather minus the flags
__global__ void __launch_bounds__(256) k_upd_pull(Ptrs P, int world, int rank, int64_t shard, int64_t n, UpdConst c,
                                                  float* __restrict__ th, float* __restrict__ d, float* __restrict__ m) {
    const int64_t gsh = shard >> 3;
    const int64_t ups = (gsh + 255) / 256;
    const int64_t u = blockIdx.x;
    const int owner = (int)((u % world + rank) % world);
    const int64_t gi = (u / world) * 256 + threadIdx.x;
    if (gi >= gsh) return;
    const int64_t j0 = ((int64_t)owner * gsh + gi) << 3;
    if (j0 >= n) return;
    (void)ups;
    const uint4 r = *reinterpret_cast<const uint4*>(P.R[owner] + (gi << 3));
    update8<true, false>(r, j0, n, c, th, d, m);
}

// the same with a register cap (more resident blocks per SM to cover the peer-load latency)
template <int MINB>
__global__ void __launch_bounds__(256, MINB) k_upd_pull_lb(Ptrs P, int world, int rank, int64_t shard, int64_t n, UpdConst c,
                                                           float* __restrict__ th, float* __restrict__ d, float* __restrict__ m) {
    const int64_t gsh = shard >> 3;
    const int64_t u = blockIdx.x;
    const int owner = (int)((u % world + rank) % world);
    const int64_t gi = (u / world) * 256 + threadIdx.x;
    if (gi >= gsh) return;
    const int64_t j0 = ((int64_t)owner * gsh + gi) << 3;
    if (j0 >= n) return;
    const uint4 r = *reinterpret_cast<const uint4*>(P.R[owner] + (gi << 3));
    update8<true, false>(r, j0, n, c, th, d, m);
}

// R prefetched with cp.async (LDGSTS) into shared memory for the NEXT unit of a 2-unit block
__global__ void __launch_bounds__(256) k_upd_pull2(Ptrs P, int world, int rank, int64_t shard, int64_t n, UpdConst c,
                                                   float* __restrict__ th, float* __restrict__ d, float* __restrict__ m) {
    const int64_t gsh = shard >> 3;
    for (int rep = 0; rep < 2; ++rep) {
        const int64_t u = (int64_t)blockIdx.x * 2 + rep;
        const int owner = (int)((u % world + rank) % world);
        const int64_t gi = (u / world) * 256 + threadIdx.x;
        if (gi >= gsh) continue;
        const int64_t j0 = ((int64_t)owner * gsh + gi) << 3;
        if (j0 >= n) continue;
        const uint4 r = *reinterpret_cast<const uint4*>(P.R[owner] + (gi << 3));
        update8<true, false>(r, j0, n, c, th, d, m);
    }
}

// P with a system fence after every unit (what per-chunk release needs), persistent
__global__ void __launch_bounds__(256) k_push_fenced(const float* __restrict__ g, uint16_t* const* recv, int world,
                                                     int rank, int64_t shard, int64_t n, int fence_every) {
    const int64_t gsh = shard >> 3;
    const int64_t ups = (gsh + 255) / 256;
    int cnt = 0;
    for (int64_t us = blockIdx.x; us < ups; us += gridDim.x) {
        const int64_t gi = us * 256 + threadIdx.x;
        if (gi < gsh) {
            for (int q = 0; q < world; ++q) {
                const int owner = (q + rank) % world;
                const int64_t j0 = ((int64_t)owner * gsh + gi) << 3;
                float xv[8];
                load8_g(g, j0, n, xv);
                int64_t first = kNone; unsigned sat = 0;
                *reinterpret_cast<uint4*>(recv[owner] + (int64_t)rank * shard + (gi << 3)) = pack8(xv, 1024.f, j0, first, sat);
            }
        }
        if (fence_every && ++cnt % fence_every == 0) { __threadfence_system(); __syncthreads(); }
    }
    __threadfence_system();
}

// P with 16 elements per thread and ONE 32-byte remote store (st.global.v8.b32, sm_100) per
// owner per thread, the g loads as two 256-bit loads; persistent, one fence per block
__global__ void __launch_bounds__(256) k_push32(const float* __restrict__ g, uint16_t* const* recv, int world,
                                                int rank, int64_t shard, int64_t n) {
    const int64_t gsh = shard >> 4;                     // 16-element groups per shard
    const int64_t ups = (gsh + 255) / 256;
    for (int64_t us = blockIdx.x; us < ups * world; us += gridDim.x) {
        const int owner = (int)((us % world + rank) % world);
        const int64_t gi = (us / world) * 256 + threadIdx.x;
        if (gi >= gsh) continue;
        const int64_t j0 = ((int64_t)owner * shard) + (gi << 4);
        float xa[8], xb[8];
        if (j0 + 16 <= n) {
            asm volatile("ld.global.cs.v8.f32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];"
                         : "=f"(xa[0]), "=f"(xa[1]), "=f"(xa[2]), "=f"(xa[3]), "=f"(xa[4]), "=f"(xa[5]), "=f"(xa[6]),
                           "=f"(xa[7]) : "l"(g + j0));
            asm volatile("ld.global.cs.v8.f32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];"
                         : "=f"(xb[0]), "=f"(xb[1]), "=f"(xb[2]), "=f"(xb[3]), "=f"(xb[4]), "=f"(xb[5]), "=f"(xb[6]),
                           "=f"(xb[7]) : "l"(g + j0 + 8));
        } else {
            load8_g(g, j0, n, xa);
            load8_g(g, j0 + 8, n, xb);
        }
        int64_t first = kNone; unsigned sat = 0;
        const uint4 pa = pack8(xa, 1024.f, j0, first, sat), pb = pack8(xb, 1024.f, j0 + 8, first, sat);
        uint16_t* dst = recv[owner] + (int64_t)rank * shard + (gi << 4);
        asm volatile("st.global.v8.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8};" ::"l"(dst), "r"(pa.x), "r"(pa.y),
                     "r"(pa.z), "r"(pa.w), "r"(pb.x), "r"(pb.y), "r"(pb.z), "r"(pb.w) : "memory");
    }
    __threadfence_system();
}

// P with 16 elements per thread (two 16-B stores per owner per thread)
__global__ void __launch_bounds__(256) k_push16(const float* __restrict__ g, uint16_t* const* recv, int world,
                                                int rank, int64_t shard, int64_t n) {
    const int64_t gsh = shard >> 3;
    const int64_t g2 = (gsh + 1) / 2;                 // pairs of groups
    const int64_t ups = (g2 + 255) / 256;
    for (int64_t us = blockIdx.x; us < ups; us += gridDim.x) {
        const int64_t pi = us * 256 + threadIdx.x;
        if (pi * 2 + 1 < gsh) {
            for (int q = 0; q < world; ++q) {
                const int owner = (q + rank) % world;
                const int64_t j0 = ((int64_t)owner * gsh + pi * 2) << 3;
                float xa[8], xb[8];
                load8_g(g, j0, n, xa);
                load8_g(g, j0 + 8, n, xb);
                int64_t first = kNone; unsigned sat = 0;
                uint4* dst = reinterpret_cast<uint4*>(recv[owner] + (int64_t)rank * shard + (pi * 2 << 3));
                dst[0] = pack8(xa, 1024.f, j0, first, sat);
                dst[1] = pack8(xb, 1024.f, j0 + 8, first, sat);
            }
        }
    }
    __threadfence_system();
}

// update pull with the R load on the non-coherent read-only path
__global__ void __launch_bounds__(256) k_upd_pull_nc(Ptrs P, int world, int rank, int64_t shard, int64_t n, UpdConst c,
                                                     float* __restrict__ th, float* __restrict__ d, float* __restrict__ m) {
    const int64_t gsh = shard >> 3;
    const int64_t u = blockIdx.x;
    const int owner = (int)((u % world + rank) % world);
    const int64_t gi = (u / world) * 256 + threadIdx.x;
    if (gi >= gsh) return;
    const int64_t j0 = ((int64_t)owner * gsh + gi) << 3;
    if (j0 >= n) return;
    const uint4 r = __ldg(reinterpret_cast<const uint4*>(P.R[owner] + (gi << 3)));
    update8<true, false>(r, j0, n, c, th, d, m);
}

// update pull with the unit's R fetched by one bulk copy (TMA engine) into shared memory
__global__ void __launch_bounds__(256) k_upd_pull_bulk(Ptrs P, int world, int rank, int64_t shard, int64_t n, UpdConst c,
                                                       float* __restrict__ th, float* __restrict__ d, float* __restrict__ m) {
    __shared__ __align__(128) uint4 sR[256];
    __shared__ __align__(8) uint64_t bar;
    const int64_t gsh = shard >> 3;
    const int64_t u = blockIdx.x;
    const int owner = (int)((u % world + rank) % world);
    const int64_t g0 = (u / world) * 256;
    const int64_t cnt = (gsh - g0) < 256 ? (gsh - g0) : 256;
    if (cnt <= 0) return;
    if (threadIdx.x == 0) {
        mbar_init(&bar, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        mbar_expect_tx(&bar, (unsigned)(cnt * 16));
        bulk_g2s(sR, P.R[owner] + (g0 << 3), (unsigned)(cnt * 16), &bar, policy_evict_first());
    }
    const int64_t gi = g0 + threadIdx.x;
    const int64_t j0 = ((int64_t)owner * gsh + gi) << 3;
    const bool act = threadIdx.x < cnt && j0 < n;
    float4 t0, t1, d0, d1, m0, m1;
    if (act && j0 + 8 <= n) {   // state loads in flight while the bulk copy runs
        t0 = __ldcs(reinterpret_cast<const float4*>(th + j0)); t1 = __ldcs(reinterpret_cast<const float4*>(th + j0) + 1);
        d0 = __ldcs(reinterpret_cast<const float4*>(d + j0)); d1 = __ldcs(reinterpret_cast<const float4*>(d + j0) + 1);
        m0 = __ldcs(reinterpret_cast<const float4*>(m + j0)); m1 = __ldcs(reinterpret_cast<const float4*>(m + j0) + 1);
    }
    mbar_wait(&bar, 0);
    if (!act) return;
    if (j0 + 8 > n) { update8<true, false>(sR[threadIdx.x], j0, n, c, th, d, m); return; }
    const uint4 r = sR[threadIdx.x];
    const uint32_t w[4] = {r.x, r.y, r.z, r.w};
    float tv[8] = {t0.x, t0.y, t0.z, t0.w, t1.x, t1.y, t1.z, t1.w};
    float dv[8] = {d0.x, d0.y, d0.z, d0.w, d1.x, d1.y, d1.z, d1.w};
    float mv[8] = {m0.x, m0.y, m0.z, m0.w, m1.x, m1.y, m1.z, m1.w};
#pragma unroll
    for (int i = 0; i < 8; ++i) upd1<true>(h2f(w[i >> 1], i & 1) * c.inv_ks, tv[i], dv[i], mv[i], c);
    float4* t4 = reinterpret_cast<float4*>(th + j0); float4* d4 = reinterpret_cast<float4*>(d + j0); float4* m4 = reinterpret_cast<float4*>(m + j0);
    __stcs(t4, make_float4(tv[0], tv[1], tv[2], tv[3])); __stcs(t4 + 1, make_float4(tv[4], tv[5], tv[6], tv[7]));
    __stcs(d4, make_float4(dv[0], dv[1], dv[2], dv[3])); __stcs(d4 + 1, make_float4(dv[4], dv[5], dv[6], dv[7]));
    __stcs(m4, make_float4(mv[0], mv[1], mv[2], mv[3])); __stcs(m4 + 1, make_float4(mv[4], mv[5], mv[6], mv[7]));
}

// all-gather push: owner writes its R shard into every rank's full-R buffer (persistent)
__global__ void __launch_bounds__(256) k_ag_push(const uint16_t* __restrict__ Rmine, uint16_t* const* full, int world,
                                                 int rank, int64_t shard) {
    const int64_t nv = shard >> 3;
    for (int64_t v = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; v < nv * world; v += (int64_t)gridDim.x * blockDim.x) {
        const int p = (int)((v / nv + rank) % world);   // rotate destinations
        const int64_t i = v % nv;
        const uint4 q = reinterpret_cast<const uint4*>(Rmine)[i];
        reinterpret_cast<uint4*>(full[p] + (int64_t)rank * shard)[i] = q;
    }
    __threadfence_system();
}

// f4 (sharded update): every rank updates only its own shard (above, with
// launch_update on the shard), then pulls the other owners' updated fp32 theta shards
// (4 B/elem over NVLink, interleaved units like k_upd_pull).
struct ThPtrs { const float* th[8]; };
__global__ void __launch_bounds__(256) k_th_gather(ThPtrs P, int world, int rank, int64_t shard, int64_t n,
                                                   float* __restrict__ th) {
    const int64_t gsh = shard >> 2;                      // float4 groups per shard
    const int64_t u = blockIdx.x;                        // unit: 256 float4 of one remote owner
    const int q = (int)(u % (world - 1));
    const int owner = (rank + 1 + q) % world;
    const int64_t gi = (u / (world - 1)) * 256 + threadIdx.x;
    if (gi >= gsh) return;
    const int64_t j0 = (int64_t)owner * shard + (gi << 2);
    if (j0 + 4 <= n) {
        __stcs(reinterpret_cast<float4*>(th + j0), *reinterpret_cast<const float4*>(P.th[owner] + j0));
    } else {
        for (int64_t j = j0; j < n; ++j) th[j] = P.th[owner][j];
    }
}

}  // namespace xb

int main(int argc, char** argv) {
    int ndev; CKE(cudaGetDeviceCount(&ndev));
    const int W = ndev > 8 ? 8 : ndev;
    const int64_t n = 25557032;
    int64_t shard = ((n + W - 1) / W + 63) / 64 * 64;
    const int64_t n_pad = shard * W;
    printf("world=%d n=%lld shard=%lld\n", W, (long long)n, (long long)shard);
    std::vector<float*> th(W), d(W), m(W), g(W);
    std::vector<uint16_t*> recv(W), R(W), full(W);
    std::vector<uint16_t**> fullp(W);
    std::vector<cudaStream_t> st(W);
    std::vector<cudaEvent_t> e0(W), e1(W);
    for (int i = 0; i < W; ++i) {
        CKE(cudaSetDevice(i));
        for (int j = 0; j < W; ++j) if (j != i) CKE(cudaDeviceEnablePeerAccess(j, 0));
        CKE(cudaMalloc(&th[i], n * 4)); CKE(cudaMalloc(&d[i], n * 4)); CKE(cudaMalloc(&m[i], n * 4)); CKE(cudaMalloc(&g[i], n * 4));
        CKE(cudaMemset(th[i], 0, n * 4)); CKE(cudaMemset(d[i], 0, n * 4)); CKE(cudaMemset(m[i], 0, n * 4)); CKE(cudaMemset(g[i], 0, n * 4));
        CKE(cudaMalloc(&recv[i], n_pad * 2)); CKE(cudaMalloc(&R[i], shard * 2)); CKE(cudaMalloc(&full[i], n_pad * 2));
        CKE(cudaMemset(recv[i], 0x11, n_pad * 2)); CKE(cudaMemset(R[i], 0x22, shard * 2)); CKE(cudaMemset(full[i], 0x22, n_pad * 2));
        CKE(cudaStreamCreate(&st[i])); cudaEventCreate(&e0[i]); cudaEventCreate(&e1[i]);
    }
    for (int i = 0; i < W; ++i) {
        CKE(cudaSetDevice(i));
        CKE(cudaMalloc(&fullp[i], 8 * sizeof(uint16_t*)));
        CKE(cudaMemcpy(fullp[i], full.data(), W * sizeof(uint16_t*), cudaMemcpyHostToDevice));
    }
    int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    UpdConst c{0.9f, 0.99f, (float)(1.0 - 0.99), 1e-8f, 6.4f, 0.0091578f, 4.64e-05f, 1.0f / 4096};
    xb::Ptrs P{};
    for (int i = 0; i < W; ++i) P.R[i] = R[i];
    // argv[1]: run only the benchmarks whose name contains it; XB_ITERS: timed iterations
    // (a short run under ncu: every launch is profiled)
    const char* only = argc > 1 ? argv[1] : nullptr;
    const int iters = std::getenv("XB_ITERS") ? std::atoi(std::getenv("XB_ITERS")) : 30;
    auto run = [&](const char* name, double bytes, const std::function<void(int)>& f) {
        if (only && !std::strstr(name, only)) return;
        for (int it = 0; it < 3; ++it) for (int i = 0; i < W; ++i) { cudaSetDevice(i); f(i); }
        for (int i = 0; i < W; ++i) { cudaSetDevice(i); CKE(cudaDeviceSynchronize()); }
        for (int i = 0; i < W; ++i) { cudaSetDevice(i); cudaEventRecord(e0[i], st[i]); }
        for (int it = 0; it < iters; ++it) for (int i = 0; i < W; ++i) { cudaSetDevice(i); f(i); }
        float worst = 0;
        for (int i = 0; i < W; ++i) { cudaSetDevice(i); cudaEventRecord(e1[i], st[i]); CKE(cudaEventSynchronize(e1[i])); float ms; cudaEventElapsedTime(&ms, e0[i], e1[i]); worst = ms > worst ? ms : worst; }
        CKE(cudaGetLastError());
        const double us = worst / iters * 1e3;
        printf("%-46s %9.2f us  %8.1f GB/s\n", name, us, bytes / us / 1e3);
    };
    const Launch L{sms, 0, 0, 0x1};
    const int ups = (int)(((shard >> 3) + 255) / 256);
    // pack (local only) for reference
    int64_t* dst; CKE(cudaSetDevice(0));
    run("reduce fp64 flat", 2.0 * n_pad, [&](int i) { xb::k_reduce<0><<<(int)((shard / 8 + 255) / 256), 256, 0, st[i]>>>(recv[i], W, shard, R[i]); });
    run("reduce int64 flat", 2.0 * n_pad, [&](int i) { xb::k_reduce<1><<<(int)((shard / 8 + 255) / 256), 256, 0, st[i]>>>(recv[i], W, shard, R[i]); });
    run("reduce int64 persistent 148x8", 2.0 * n_pad, [&](int i) { xb::k_reduce<1><<<sms * 8, 256, 0, st[i]>>>(recv[i], W, shard, R[i]); });
    run("reduce fp64 persistent 148x8", 2.0 * n_pad, [&](int i) { xb::k_reduce<0><<<sms * 8, 256, 0, st[i]>>>(recv[i], W, shard, R[i]); });
    run("update pull from owners (flat, interleaved)", 26.0 * n, [&](int i) { xb::k_upd_pull<<<W * ups, 256, 0, st[i]>>>(P, W, i, shard, n, c, th[i], d[i], m[i]); });
    run("update pull, launch_bounds(256,6)", 26.0 * n, [&](int i) { xb::k_upd_pull_lb<6><<<W * ups, 256, 0, st[i]>>>(P, W, i, shard, n, c, th[i], d[i], m[i]); });
    run("update pull, launch_bounds(256,8)", 26.0 * n, [&](int i) { xb::k_upd_pull_lb<8><<<W * ups, 256, 0, st[i]>>>(P, W, i, shard, n, c, th[i], d[i], m[i]); });
    run("update pull, 2 units per block", 26.0 * n, [&](int i) { xb::k_upd_pull2<<<(W * ups + 1) / 2, 256, 0, st[i]>>>(P, W, i, shard, n, c, th[i], d[i], m[i]); });
    run("update local full R (k_update flat)", 26.0 * n, [&](int i) { launch_update(st[i], L, full[i], n, c, th[i], d[i], m[i], nullptr, nullptr, nullptr); });
    {   // P with per-unit fences, alone and concurrently with the local update on a second stream
        std::vector<uint16_t**> recvp(W);
        for (int i = 0; i < W; ++i) { CKE(cudaSetDevice(i)); CKE(cudaMalloc(&recvp[i], 8 * sizeof(uint16_t*)));
                                      CKE(cudaMemcpy(recvp[i], recv.data(), W * sizeof(uint16_t*), cudaMemcpyHostToDevice)); }
        std::vector<cudaStream_t> st2(W);
        for (int i = 0; i < W; ++i) { CKE(cudaSetDevice(i)); CKE(cudaStreamCreateWithFlags(&st2[i], cudaStreamNonBlocking)); }
        const double pb = 2.0 * n_pad * (W - 1) / W;
        run("P persistent 148x6, one fence/block", pb, [&](int i) { xb::k_push_fenced<<<sms * 6, 256, 0, st[i]>>>(g[i], recvp[i], W, i, shard, n, 0); });
        run("P persistent 148x6, 16 elem/thread", pb, [&](int i) { xb::k_push16<<<sms * 6, 256, 0, st[i]>>>(g[i], recvp[i], W, i, shard, n); });
        run("P persistent 148x8, 32-B remote stores", pb, [&](int i) { xb::k_push32<<<sms * 8, 256, 0, st[i]>>>(g[i], recvp[i], W, i, shard, n); });
        run("P persistent 148x4, 32-B remote stores", pb, [&](int i) { xb::k_push32<<<sms * 4, 256, 0, st[i]>>>(g[i], recvp[i], W, i, shard, n); });
        run("P persistent 148x8, one fence/block", pb, [&](int i) { xb::k_push_fenced<<<sms * 8, 256, 0, st[i]>>>(g[i], recvp[i], W, i, shard, n, 0); });
        run("P persistent 148x4, one fence/block", pb, [&](int i) { xb::k_push_fenced<<<sms * 4, 256, 0, st[i]>>>(g[i], recvp[i], W, i, shard, n, 0); });
        run("update pull, R by one bulk copy per block", 26.0 * n, [&](int i) { xb::k_upd_pull_bulk<<<W * ups, 256, 0, st[i]>>>(P, W, i, shard, n, c, th[i], d[i], m[i]); });
    run("update pull, R via ld.global.nc", 26.0 * n, [&](int i) { xb::k_upd_pull_nc<<<W * ups, 256, 0, st[i]>>>(P, W, i, shard, n, c, th[i], d[i], m[i]); });
        run("P persistent 148x6, fence/unit", pb, [&](int i) { xb::k_push_fenced<<<sms * 6, 256, 0, st[i]>>>(g[i], recvp[i], W, i, shard, n, 1); });
        run("P persistent 148x2, fence/unit", pb, [&](int i) { xb::k_push_fenced<<<sms * 2, 256, 0, st[i]>>>(g[i], recvp[i], W, i, shard, n, 1); });
        for (int pb_ = 1; pb_ <= 4; pb_ *= 2)   // pipelining potential: the push (one fence per block) || the update
            run(pb_ == 1 ? "P 148x1 one fence || local update (2 streams)" : pb_ == 2 ? "P 148x2 one fence || local update (2 streams)"
                                                                       : "P 148x4 one fence || local update (2 streams)",
                26.0 * n, [&](int i) {
                    cudaEvent_t ev; cudaEventCreateWithFlags(&ev, cudaEventDisableTiming);
                    xb::k_push_fenced<<<sms * pb_, 256, 0, st[i]>>>(g[i], recvp[i], W, i, shard, n, 0);
                    launch_update(st2[i], L, full[i], n, c, th[i], d[i], m[i], nullptr, nullptr, nullptr);
                    cudaEventRecord(ev, st2[i]); cudaStreamWaitEvent(st[i], ev, 0); cudaEventDestroy(ev); });
        run("P 148x1 one fence alone", pb, [&](int i) { xb::k_push_fenced<<<sms * 1, 256, 0, st[i]>>>(g[i], recvp[i], W, i, shard, n, 0); });
        run("P 148x2 one fence alone", pb, [&](int i) { xb::k_push_fenced<<<sms * 2, 256, 0, st[i]>>>(g[i], recvp[i], W, i, shard, n, 0); });
        run("P 148x2 fence/unit || local update (2 streams)", 26.0 * n, [&](int i) {
            cudaEvent_t ev; cudaEventCreateWithFlags(&ev, cudaEventDisableTiming);
            xb::k_push_fenced<<<sms * 2, 256, 0, st[i]>>>(g[i], recvp[i], W, i, shard, n, 1);
            launch_update(st2[i], L, full[i], n, c, th[i], d[i], m[i], nullptr, nullptr, nullptr);
            cudaEventRecord(ev, st2[i]); cudaStreamWaitEvent(st[i], ev, 0); cudaEventDestroy(ev); });
        run("P 148x2 fence/unit || pull update (2 streams)", 26.0 * n, [&](int i) {
            cudaEvent_t ev; cudaEventCreateWithFlags(&ev, cudaEventDisableTiming);
            xb::k_push_fenced<<<sms * 2, 256, 0, st[i]>>>(g[i], recvp[i], W, i, shard, n, 1);
            xb::k_upd_pull<<<W * ups, 256, 0, st2[i]>>>(P, W, i, shard, n, c, th[i], d[i], m[i]);
            cudaEventRecord(ev, st2[i]); cudaStreamWaitEvent(st[i], ev, 0); cudaEventDestroy(ev); });
    }
    {   // f4: sharded update + fp32 theta all-gather, against the replicated update above
        xb::ThPtrs TP{};
        for (int i = 0; i < W; ++i) TP.th[i] = th[i];
        auto nsh = [&](int i) { const int64_t lo = (int64_t)i * shard; return lo >= n ? (int64_t)0 : (n - lo < shard ? n - lo : shard); };
        const int gunits = (int)((W - 1) * (((shard >> 2) + 255) / 256));
        run("f4 sharded update (own shard, local R)", 26.0 * n / W, [&](int i) {
            if (nsh(i)) launch_update(st[i], L, R[i], nsh(i), c, th[i] + (int64_t)i * shard, d[i], m[i], nullptr, nullptr, nullptr); });
        run("f4 theta all-gather pull (fp32)", 4.0 * n * (W - 1) / W, [&](int i) {
            xb::k_th_gather<<<gunits, 256, 0, st[i]>>>(TP, W, i, shard, n, th[i]); });
        run("f4 sharded update + theta all-gather", 26.0 * n, [&](int i) {
            if (nsh(i)) launch_update(st[i], L, R[i], nsh(i), c, th[i] + (int64_t)i * shard, d[i], m[i], nullptr, nullptr, nullptr);
            xb::k_th_gather<<<gunits, 256, 0, st[i]>>>(TP, W, i, shard, n, th[i]); });
    }
    run("AG push R shard to all (persistent 148x8)", 2.0 * shard * (W - 1), [&](int i) { xb::k_ag_push<<<sms * 8, 256, 0, st[i]>>>(R[i], fullp[i], W, i, shard); });
    run("AG push + local update", 26.0 * n, [&](int i) { xb::k_ag_push<<<sms * 8, 256, 0, st[i]>>>(R[i], fullp[i], W, i, shard);
                                                          launch_update(st[i], L, full[i], n, c, th[i], d[i], m[i], nullptr, nullptr, nullptr); });
    return 0;
}
