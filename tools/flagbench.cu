// Cross-GPU flag latency micro-benchmark (development tool): ping-pong between GPU 0
// and GPU 1 through peer-mapped flags, several store/load flavours.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 tools/flagbench.cu -o tools/flagbench
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>
#include <cstdlib>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s at %d\n", cudaGetErrorString(e), __LINE__); exit(1);} } while (0)

__device__ __forceinline__ uint64_t gt() { uint64_t t; asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t)); return t; }
__device__ __forceinline__ uint32_t ld_acq(const uint32_t* p) { uint32_t v; asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory"); return v; }
__device__ __forceinline__ uint32_t ld_rlx(const uint32_t* p) { uint32_t v; asm volatile("ld.relaxed.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory"); return v; }
__device__ __forceinline__ uint32_t ld_vol(const uint32_t* p) { return *(volatile const uint32_t*)p; }
__device__ __forceinline__ void st_rel(uint32_t* p, uint32_t v) { asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory"); }
__device__ __forceinline__ void st_rlx(uint32_t* p, uint32_t v) { asm volatile("st.relaxed.sys.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory"); }

// mode 0: release/acquire; 1: relaxed store + relaxed load; 2: volatile; 3: fence.sys + relaxed store, acquire load
template <int MODE>
__global__ void pingpong(uint32_t* my_flag, uint32_t* peer_flag, int iters, int leader, uint64_t* out) {
    uint64_t t0 = gt();
    for (int i = 1; i <= iters; ++i) {
        if (leader) {
            if (MODE == 0) st_rel(peer_flag, i); else if (MODE == 3) { __threadfence_system(); st_rlx(peer_flag, i); } else if (MODE == 1) st_rlx(peer_flag, i); else *(volatile uint32_t*)peer_flag = i;
            while ((MODE == 0 || MODE == 3 ? ld_acq(my_flag) : MODE == 1 ? ld_rlx(my_flag) : ld_vol(my_flag)) < (uint32_t)i) {}
        } else {
            while ((MODE == 0 || MODE == 3 ? ld_acq(my_flag) : MODE == 1 ? ld_rlx(my_flag) : ld_vol(my_flag)) < (uint32_t)i) {}
            if (MODE == 0) st_rel(peer_flag, i); else if (MODE == 3) { __threadfence_system(); st_rlx(peer_flag, i); } else if (MODE == 1) st_rlx(peer_flag, i); else *(volatile uint32_t*)peer_flag = i;
        }
    }
    *out = gt() - t0;
}

// publish cost after a burst of remote stores by the whole grid (like the pack's tail)
__global__ void burst_then_publish(uint4* remote, int64_t n16, uint32_t* peer_flag, uint32_t v, unsigned* tick, uint64_t* out) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n16; i += (int64_t)gridDim.x * blockDim.x) remote[i] = make_uint4(1, 2, 3, 4);
    __threadfence_system();
    __syncthreads();
    if (threadIdx.x == 0 && atomicAdd(tick, 1u) == gridDim.x - 1) {
        *tick = 0;
        uint64_t a = gt();
        st_rel(peer_flag, v);
        uint64_t b = gt();
        out[0] = b - a;
    }
}

template <int MODE>
static void run(const char* name, uint32_t* f0, uint32_t* f1, uint64_t* o0, uint64_t* o1) {
    const int iters = 2000;
    CK(cudaSetDevice(0)); CK(cudaMemset(f0, 0, 4));
    CK(cudaSetDevice(1)); CK(cudaMemset(f1, 0, 4));
    CK(cudaSetDevice(0)); CK(cudaDeviceSynchronize());
    CK(cudaSetDevice(1)); CK(cudaDeviceSynchronize());
    CK(cudaSetDevice(1)); pingpong<MODE><<<1, 1>>>(f1, f0, iters, 0, o1);
    CK(cudaSetDevice(0)); pingpong<MODE><<<1, 1>>>(f0, f1, iters, 1, o0);
    CK(cudaSetDevice(0)); CK(cudaDeviceSynchronize());
    CK(cudaSetDevice(1)); CK(cudaDeviceSynchronize());
    uint64_t t; CK(cudaSetDevice(0)); CK(cudaMemcpy(&t, o0, 8, cudaMemcpyDeviceToHost));
    printf("%-40s round trip %8.2f us\n", name, t / 1e3 / iters);
}

int main() {
    int n; CK(cudaGetDeviceCount(&n)); if (n < 2) { printf("need 2 GPUs\n"); return 0; }
    uint32_t *f0, *f1; uint64_t *o0, *o1; uint4* buf1; unsigned* tick; 
    CK(cudaSetDevice(0)); CK(cudaDeviceEnablePeerAccess(1, 0)); CK(cudaMalloc(&f0, 128)); CK(cudaMalloc(&o0, 64)); CK(cudaMalloc(&tick, 4)); CK(cudaMemset(tick, 0, 4));
    CK(cudaSetDevice(1)); CK(cudaDeviceEnablePeerAccess(0, 0)); CK(cudaMalloc(&f1, 128)); CK(cudaMalloc(&o1, 64)); CK(cudaMalloc(&buf1, 64 << 20));
    run<0>("release.sys / acquire.sys", f0, f1, o0, o1);
    run<3>("fence.sys+relaxed st / acquire.sys", f0, f1, o0, o1);
    run<1>("relaxed.sys / relaxed.sys", f0, f1, o0, o1);
    run<2>("volatile / volatile", f0, f1, o0, o1);
    CK(cudaSetDevice(0));
    for (int rep = 0; rep < 3; ++rep) {
        cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
        cudaEventRecord(a);
        burst_then_publish<<<148 * 6, 256>>>(buf1, (64 << 20) / 16, f1, 7, tick, o0);
        cudaEventRecord(b); CK(cudaEventSynchronize(b));
        float ms; cudaEventElapsedTime(&ms, a, b);
        uint64_t t; CK(cudaMemcpy(&t, o0, 8, cudaMemcpyDeviceToHost));
        printf("burst 64MB remote + publish: kernel %.1f us, release store %.2f us\n", ms * 1e3, t / 1e3);
    }
    return 0;
}
