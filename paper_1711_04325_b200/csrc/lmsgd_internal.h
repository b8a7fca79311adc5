// Internal interfaces between the C ABI (api.cpp) and the sm_100a kernels
// (kernels.cu).  Not installed; not part of the ABI.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "lmsgd.h"

namespace lmsgd {

constexpr int64_t kNone = INT64_MAX;  // "no non-finite index" in device status words

// Device status words of a step: this rank's {first_nonfinite, pack_saturations,
// sum_saturations, error} and, world > 1, the global decision {first, pack_sat,
// error} that the rank's reduce computes from every rank's words.  The public
// sub-step status (lmsgd_status_reset) is the first four words.
enum { ST_FIRST = 0, ST_PACK_SAT = 1, ST_SUM_SAT = 2, ST_ERROR = 3,
       ST_G_FIRST = 4, ST_G_PACK_SAT = 5, ST_G_ERROR = 6, ST_G_SUM_SAT = 7, ST_WORDS = 8 };

// fp32 constants of the update, each rounded once from double (R15).
struct UpdConst {
    float mu1, mu2, omm2, eps;   // omm2 = fp32(1 - mu2), computed in double
    float eta, a_sgd, a_rms;
    float inv_ks;                // fp32(1 / (k s)), exact for power-of-two k s
    float wd;                    // weight decay lambda (R12), 0 = off
    int32_t freeze_m;            // host-side only: LMSGD_FLAG_FREEZE_M and a_rms == 0 (kernel choice)
    int64_t n_wd;                // elements [0, n_wd) are decayed
};

// Layout of one rank's exchange buffer (CUDA IPC-shared when world > 1).
struct Layout {
    int64_t shard;        // elements per rank shard (multiple of 64)
    int64_t off_recv;     // uint16 [world][shard]: slot p = rank p's packed values of MY shard
    int64_t off_R;        // uint16 [shard]: this rank's reduced shard (wire-2 payload)
    int64_t off_status;   // int64 [2 parity][ST_WORDS]
    int64_t off_flags;    // uint32: A at +0, B at +128 B, C at +256 B, D at +384 B, each [LMSGD_MAX_WORLD]
    int64_t off_bn;       // float [2 parity][2 * LMSGD_MAX_BN_CHANNELS]
    int64_t off_cflags;   // uint32 [nchunks][LMSGD_MAX_WORLD]: owner o's "R chunk c ready" = epoch
    int32_t cu;           // work units (2048 elements) per reduce chunk
    int32_t nchunks;      // chunks per shard
    int64_t bytes;
};

struct Peers {
    char* base[LMSGD_MAX_WORLD];  // exchange buffer of every rank (own included)
};

struct Ticket {
    unsigned int* counters;  // device, zero-initialised, reset by the last block
};

struct Launch {
    int sm_count;
    int grid_cap_stream;   // SMs x resident blocks of the streaming kernels (informational)
    int grid_xstep;        // SMs x resident blocks of k_xstep (cooperative, all co-resident)
    int pdl_mask;          // programmatic dependent launch: bit 1 = the k = 1 kernels,
                           // bit 2 = k_xstep1 (cooperative + PDL)
};

// Graph mode of the world == 1 step (lmsgd_step_graph): everything that changes
// between steps is read from device memory at fixed addresses, so a captured CUDA
// graph replays as the next step.  epoch == NULL selects host mode (arguments).
struct Dev1 {
    uint32_t* epoch;         // completed steps; this step is *epoch + 1 (parity = its low bit)
    int64_t* st_base;        // the two status slots [2][ST_WORDS]
    const UpdConst* ctab;    // coefficient table (lmsgd_schedule_upload)
    int64_t count;
    int64_t* cursor;         // index of this step's coefficients
};

// ---- single-GPU building blocks (sub-step ABI and world == 1)
cudaError_t launch_status_reset(cudaStream_t s, int64_t* st);
cudaError_t launch_pack(cudaStream_t s, const Launch& L, const float* g, int64_t n, int64_t n_pad,
                        float scale, uint16_t* h, int64_t* st, const Dev1& dv = Dev1{});
cudaError_t launch_reduce_local(cudaStream_t s, const Launch& L, const uint16_t* h, int k,
                                int64_t n_pad, uint16_t* R, int64_t* st);
cudaError_t launch_update(cudaStream_t s, const Launch& L, const uint16_t* R, int64_t n,
                          const UpdConst& c, float* th, float* d, float* m, const int64_t* st,
                          int64_t* st_reset, int64_t* last, const Dev1& dv = Dev1{});
cudaError_t launch_fused1(cudaStream_t s, const Launch& L, const float* g, int64_t n, float scale,
                          const UpdConst& c, float* th, float* d, float* m, int64_t* st,
                          int64_t* st_reset, int64_t* last, const Dev1& dv = Dev1{});
// graph mode, k = 1: publish the fused step's status (fused) and advance the counters
cudaError_t launch_advance1(cudaStream_t s, const Dev1& dv, int64_t* last, bool fused);
cudaError_t launch_finalize_fused(cudaStream_t s, const int64_t* st, int64_t* last);
// lmsgd_step_out_of_place, k = 1: one pass in -> out, then the status / repair kernel
cudaError_t launch_step_oop1(cudaStream_t s, const Launch& L, const float* g, int64_t n, float scale,
                             const UpdConst& c, const float* thi, const float* di, const float* mi, float* tho,
                             float* dout, float* mo, int64_t* st, int64_t* st_reset, int64_t* last,
                             int64_t* trace = nullptr);   // trace: TR_PACK_START / TR_UPD_END stamps
// lmsgd_exchange at world == 1: status record of the pack, next slot cleared
cudaError_t launch_xfinal1(cudaStream_t s, const int64_t* st, int64_t* st_next, int64_t* last);
// lmsgd_status_accumulate: merge a step status record into a sub-step accumulator
cudaError_t launch_status_accumulate(cudaStream_t s, const int64_t* last, int64_t offset, int64_t* acc);
int stream_blocks_per_sm();

// ---- world > 1 exchange over peer memory (NVLink / NVSwitch)
struct XArgs {
    Peers peers;
    Layout lay;
    int world, rank;
    uint32_t epoch;      // step number (>= 1), the flag value of this step
    int parity;          // epoch & 1: status slot of this step
    int64_t n;
    int64_t timeout_ns;
    unsigned int* ticket;
    int64_t* trace;      // NULL, or this step's TR_WORDS %globaltimer stamps (lmsgd_trace_enable)
    uint32_t* dev_epoch; // device counter of completed steps (world > 1) or BN calls: the kernels
                         // use epoch = *dev_epoch + 1 and the phase's last kernel advances it,
                         // so a step captured in a CUDA graph replays as the next step
    // NVLS (lmsgd_nvls_*): this rank's packed wire [n_pad] fp16 as a local (unicast) view and
    // as the multicast view every rank's copy is bound to; nv = LMSGD_NVLS_* mode, 0 = off
    char* nv_uc;
    char* nv_mc;
    int nv;
};

// Trace stamps of one world > 1 step (ns, this GPU's %globaltimer): pack start,
// pack end (its last block), all ranks' packs observed, reduce start, reduce end,
// all ranks' reduces observed, update start, update end.
enum { TR_PACK_START = 0, TR_PACK_END, TR_RED_START, TR_RED_GO, TR_RED_END, TR_UPD_START, TR_UPD_GO,
       TR_UPD_END, TR_PUB_END, TR_A_SEEN /* + rank, 8 words */ = 9, TR_WORDS = 17 };
// One persistent cooperative kernel for the whole world > 1 step (pack+push, exact
// reduce of the own shard with per-chunk release, update with the all-gather fused).
struct XStep {
    XArgs x;
    const float* g;
    float scale;
    UpdConst c;
    float *th, *d, *m;
    int64_t* last;
    unsigned int* ctr;   // local counters, reset by their completer: [0] pack blocks done,
                         // [1] k_xstep1 blocks retired, [2..3] unused, [4 + c] reduce units of chunk c
    const UpdConst* ctab;    // graph mode: device coefficient table (lmsgd_schedule_upload), else NULL
    int64_t ctab_count;
    int64_t* cursor;         // graph mode: device index of the next step's coefficients
    uint16_t* rout;          // lmsgd_exchange: the caller's [n_pad] all-reduce output (k_xgather
                             // replaces k_xupdate); NULL for a step
    int32_t v8;              // 1: the update may use 256-bit accesses if th/d/m are 32-byte aligned
                             // (an emulated group sets it only if every rank's are)
    int32_t riu;             // 1: a step whose own-shard units are reduced inside k_xupdate
                             // (kernels.cu riu_active: peer path, one phase); 0 for lmsgd_exchange
};
// d_group / nsim: emulated-group mode (lmsgd_*_group): device array of the nsim ranks'
// XStep, every rank's blocks in one launch per kernel; NULL for a real (one-rank) launch
cudaError_t launch_xstep(cudaStream_t s, const Launch& L, const XStep& a, const XStep* d_group = nullptr,
                         int nsim = 1);
int xstep_blocks_per_sm(bool sim = false);   // occupancy of k_xstep1 (all co-resident)
int xstep_default_bps();                      // blocks per SM it is launched with by default

struct BnArgs {
    XArgs x;
    float *mean, *var;
    int64_t C;
};
cudaError_t launch_bn_allreduce(cudaStream_t s, const BnArgs& a, const BnArgs* d_group = nullptr, int nsim = 1);

}  // namespace lmsgd
