// NVLink peer-memory micro-benchmark (development tool): remote store / load
// bandwidth of SM-driven kernels vs the copy engine, single process, 2+ GPUs.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 tools/p2pbench.cu -o tools/p2pbench
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <functional>
#include <vector>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s at %d\n", cudaGetErrorString(e), __LINE__); exit(1);} } while (0)

__device__ __forceinline__ uint32_t cvt2(float lo, float hi) {
    uint32_t r; asm("cvt.rn.satfinite.f16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(hi), "f"(lo)); return r;
}

// pack 8 fp32 -> 8 fp16, store to dst (remote or local); optional per-block fence + ticket
template <int MODE>  // 0 plain, 1 fence.sys per block, 2 fence + ticket
__global__ void k_push(const float* __restrict__ g, uint16_t* __restrict__ dst, int64_t nv, unsigned* ticket) {
    for (int64_t v = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; v < nv; v += (int64_t)gridDim.x * blockDim.x) {
        const float4 a = __ldcs(reinterpret_cast<const float4*>(g) + 2 * v);
        const float4 b = __ldcs(reinterpret_cast<const float4*>(g) + 2 * v + 1);
        reinterpret_cast<uint4*>(dst)[v] = make_uint4(cvt2(a.x, a.y), cvt2(a.z, a.w), cvt2(b.x, b.y), cvt2(b.z, b.w));
    }
    if (MODE >= 1) { __threadfence_system(); __syncthreads(); }
    if (MODE == 2 && threadIdx.x == 0) atomicAdd(ticket, 1u);
}

// pull: R = src_local + src_remote (fp16 each), exact-ish sum in fp32 (timing only)
__global__ void k_pull(const uint16_t* __restrict__ a, const uint16_t* __restrict__ b, uint16_t* __restrict__ out, int64_t nv) {
    for (int64_t v = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; v < nv; v += (int64_t)gridDim.x * blockDim.x) {
        const uint4 x = reinterpret_cast<const uint4*>(a)[v];
        const uint4 y = reinterpret_cast<const uint4*>(b)[v];
        uint4 o;
        const __half2* hx = reinterpret_cast<const __half2*>(&x);
        const __half2* hy = reinterpret_cast<const __half2*>(&y);
        __half2* ho = reinterpret_cast<__half2*>(&o);
        for (int i = 0; i < 4; ++i) ho[i] = __hadd2(hx[i], hy[i]);
        reinterpret_cast<uint4*>(out)[v] = o;
    }
}

// remote read only (sink into a local buffer)
__global__ void k_read(const uint4* __restrict__ src, uint4* __restrict__ dst, int64_t nv) {
    for (int64_t v = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; v < nv; v += (int64_t)gridDim.x * blockDim.x) dst[v] = src[v];
}

int main(int argc, char** argv) {
    int ndev; CK(cudaGetDeviceCount(&ndev));
    if (ndev < 2) { printf("need 2 GPUs\n"); return 0; }
    const int64_t n = argc > 1 ? atoll(argv[1]) : 25557504;   // fp16 elements pushed (the full R50 payload)
    const int64_t nv = n / 8;
    float* g[2]; uint16_t* h[2]; uint16_t* o[2]; unsigned* tk[2];
    for (int d = 0; d < 2; ++d) {
        CK(cudaSetDevice(d));
        CK(cudaDeviceEnablePeerAccess(1 - d, 0));
        CK(cudaMalloc(&g[d], n * 4)); CK(cudaMemset(g[d], 0, n * 4));
        CK(cudaMalloc(&h[d], n * 2)); CK(cudaMalloc(&o[d], n * 2)); CK(cudaMemset(h[d], 0, n * 2));
        CK(cudaMalloc(&tk[d], 4));
    }
    cudaStream_t st[2]; cudaEvent_t e0[2], e1[2];
    for (int d = 0; d < 2; ++d) { cudaSetDevice(d); cudaStreamCreate(&st[d]); cudaEventCreate(&e0[d]); cudaEventCreate(&e1[d]); }
    int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    auto run = [&](const char* name, int nd, double bytes, const std::function<void(int)>& f) {
        for (int it = 0; it < 3; ++it) for (int d = 0; d < nd; ++d) { cudaSetDevice(d); f(d); }
        for (int d = 0; d < nd; ++d) { cudaSetDevice(d); CK(cudaDeviceSynchronize()); }
        const int iters = 20;
        for (int d = 0; d < nd; ++d) { cudaSetDevice(d); cudaEventRecord(e0[d], st[d]); }
        for (int it = 0; it < iters; ++it) for (int d = 0; d < nd; ++d) { cudaSetDevice(d); f(d); }
        float worst = 0;
        for (int d = 0; d < nd; ++d) { cudaSetDevice(d); cudaEventRecord(e1[d], st[d]); CK(cudaEventSynchronize(e1[d])); float ms; cudaEventElapsedTime(&ms, e0[d], e1[d]); worst = ms > worst ? ms : worst; }
        const double us = worst / iters * 1e3;
        printf("%-44s %2s %9.2f us %8.1f GB/s per GPU per dir\n", name, nd == 2 ? "x2" : "x1", us, bytes / us / 1e3);
    };
    const int flat = (int)((nv + 255) / 256);
    for (int nd = 1; nd <= 2; ++nd) {
        run("push flat (remote store)", nd, n * 2.0, [&](int d) { k_push<0><<<flat, 256, 0, st[d]>>>(g[d], h[1 - d], nv, tk[d]); });
        run("push flat + fence.sys/block", nd, n * 2.0, [&](int d) { k_push<1><<<flat, 256, 0, st[d]>>>(g[d], h[1 - d], nv, tk[d]); });
        run("push flat + fence + ticket", nd, n * 2.0, [&](int d) { k_push<2><<<flat, 256, 0, st[d]>>>(g[d], h[1 - d], nv, tk[d]); });
        run("push persistent 148x8 + fence", nd, n * 2.0, [&](int d) { k_push<1><<<sms * 8, 256, 0, st[d]>>>(g[d], h[1 - d], nv, tk[d]); });
        run("push persistent 148x2 + fence", nd, n * 2.0, [&](int d) { k_push<1><<<sms * 2, 256, 0, st[d]>>>(g[d], h[1 - d], nv, tk[d]); });
        run("push local (reference)", nd, n * 2.0, [&](int d) { k_push<0><<<flat, 256, 0, st[d]>>>(g[d], h[d], nv, tk[d]); });
        run("pull flat: local+remote -> local", nd, n * 2.0, [&](int d) { k_pull<<<flat, 256, 0, st[d]>>>(h[d], h[1 - d], o[d], nv); });
        run("pull persistent 148x8", nd, n * 2.0, [&](int d) { k_pull<<<sms * 8, 256, 0, st[d]>>>(h[d], h[1 - d], o[d], nv); });
        run("read remote flat", nd, n * 2.0, [&](int d) { k_read<<<flat, 256, 0, st[d]>>>((const uint4*)h[1 - d], (uint4*)o[d], nv); });
        run("write remote copy (local->remote) flat", nd, n * 2.0, [&](int d) { k_read<<<flat, 256, 0, st[d]>>>((const uint4*)h[d], (uint4*)o[1 - d], nv); });
        run("cudaMemcpyPeerAsync push", nd, n * 2.0, [&](int d) { cudaMemcpyPeerAsync(o[1 - d], 1 - d, h[d], d, n * 2, st[d]); });
        run("cudaMemcpyAsync push (UVA)", nd, n * 2.0, [&](int d) { cudaMemcpyAsync(o[1 - d], h[d], n * 2, cudaMemcpyDefault, st[d]); });
    }
    return 0;
}
