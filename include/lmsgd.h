/*
 * lmsgd.h -- C ABI of the B200-native gradient exchange + blended update of
 * arXiv 1711.04325 (Akiba et al., "Extremely Large Minibatch SGD: Training
 * ResNet-50 on ImageNet in 15 Minutes").
 *
 * One synchronous data-parallel iteration
 * after the backward pass, on k = world GPUs of one node:
 *
 *   pack     h   = sat16_RNE(s * g)                  fp32 -> fp16 wire
 *   exchange R   = sat16_RNE(sum_ranks h)            fp16 all-reduce, exact accumulation
 *   unpack   ghat = fp32(R) * (1 / (k s))            "casts back and averages"
 *   update   m     = mu2 m + (1 - mu2) ghat^2
 *            Delta = mu1 Delta - (a_SGD + a_RMS / (sqrt(m) + eps)) ghat
 *            theta = theta + eta Delta
 *
 * with (eta, a_SGD, a_RMS) from the slow-start / RMSprop-warm-up schedule
 * (PAPER.md:174-196, 216-230), and the BN last-minibatch statistics average before
 * validation.  Readings of ambiguous passages: DESIGN.md R1-R20.
 *
 * Conventions for every function below
 *  - Return value: LMSGD_OK (0) or a negative lmsgd_status.  Argument errors are
 *    detected synchronously, before anything is enqueued, and leave all buffers
 *    untouched.  lmsgd_last_error(ctx) gives a one-line message.
 *  - "device" pointers are CUDA device pointers on the context's device
 *    (cudaMalloc / torch CUDA tensors), fp32, contiguous, 16-byte aligned.
 *    "host" pointers are ordinary or pinned host memory as stated.
 *  - All device work is enqueued on the caller's `stream` (a cudaStream_t passed
 *    as void*; NULL = legacy default stream) and the call returns before it
 *    completes.  Caller-owned buffers must stay alive until the stream passes.
 *  - Ownership: the caller owns params/grads/delta/m/mean/var.  The library owns
 *    its fusion (fp16 wire) buffers, flags, status words and peer mappings.
 *  - Thread safety: one context per rank per host thread.
 *  - Determinism: identical inputs give bit-identical outputs on every rank and
 *    every run (the fp16 sum is exact, the update is elementwise; in the optional NVLS
 *    modes the switch's fp32-accumulated sum is not exact but still deterministic and
 *    computed once per element by its owner, so replicas stay bit-identical).
 */
#ifndef LMSGD_H
#define LMSGD_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif
#if defined(LMSGD_BUILD) && defined(__GNUC__)
#pragma GCC visibility push(default)  /* the library is built with -fvisibility=hidden */
#endif

#define LMSGD_ABI_VERSION 1
#define LMSGD_MAX_WORLD 8            /* one NVSwitch node */
#define LMSGD_IPC_HANDLE_BYTES 64    /* sizeof(cudaIpcMemHandle_t) */
#define LMSGD_MAX_BN_CHANNELS (1 << 20)

typedef enum {
    LMSGD_OK = 0,
    LMSGD_ERR_INVALID_ARG = -1,   /* null/misaligned pointer, bad size, t < 1, eta <= 0 ... */
    LMSGD_ERR_CUDA = -2,          /* a CUDA runtime call failed (message in last_error)   */
    LMSGD_ERR_NONFINITE = -4,     /* a gradient entry was NaN/Inf: the step was skipped    */
    LMSGD_ERR_STATE = -5,         /* call out of order (e.g. step before connect)          */
    LMSGD_ERR_UNSUPPORTED = -6,   /* e.g. world > LMSGD_MAX_WORLD, no peer access          */
    LMSGD_ERR_TIMEOUT = -7,       /* a cross-GPU wait exceeded the timeout; step skipped   */
    LMSGD_ERR_RANGE = -8          /* schedule asked past its last epoch / table exhausted  */
} lmsgd_status;

/* Hyperparameters, PAPER.md:167 (mu1, mu2, eps), PAPER.md:190 (beta_center,
 * beta_period), PAPER.md:192 (eta_RMSprop).  lmsgd_hyper_default fills
 * 0.9, 0.99, 1e-8, 3e-4, 10, 5. */
typedef struct lmsgd_hyper {
    double mu1, mu2, eps, eta_rmsprop, beta_center, beta_period;
} lmsgd_hyper;

/* Logical cluster shape that drives eta_base = 0.1 * n_workers * b_local / 256
 * (PAPER.md:217-221).  Independent of the physical world size k: the paper's
 * 32k run is n_workers = 1024, b_local = 32.  n_train = images per epoch (the
 * paper does not print it; ImageNet-1k = 1,281,167, R5).
 * schedule: 0 = slow-start, 1 = Goyal et al..
 * transition: the alpha_SGD warm-up function:
 *   LMSGD_TRANSITION_ELU (0, the paper's, reading R1), and the alternatives the paper
 *   examined without printing them (reading R20, each 1/2 at beta_center with slope
 *   1/beta_period there): LINEAR clamp(1/2 + (e - bc)/bp, 0, 1), SIGMOID
 *   1/(1 + exp(-4 (e - bc)/bp)), SUDDEN 0 below bc, 1 from bc on. */
#define LMSGD_TRANSITION_ELU 0
#define LMSGD_TRANSITION_LINEAR 1
#define LMSGD_TRANSITION_SIGMOID 2
#define LMSGD_TRANSITION_SUDDEN 3
typedef struct lmsgd_cluster {
    int64_t n_workers, b_local, n_train;
    int32_t schedule;
    int32_t transition;
} lmsgd_cluster;

/* Per-step coefficients.  lmsgd_schedule_at is the canonical source; a caller may
 * pass its own (eta > 0, 0 <= alpha_sgd <= 1, alpha_rmsprop >= 0). */
typedef struct lmsgd_coeffs {
    double epoch;          /* (t-1) b_total / n_train, start of step (R2, R3)  */
    double eta;            /* eta_SGD of the current phase      */
    double alpha_sgd;      /* ELU-like transition, slope 1/beta_period (R1)    */
    double alpha_rmsprop;  /* ((1 - alpha_sgd) eta_RMSprop) / eta */
    int32_t phase;         /* LR phase index 0..3 */
    int32_t reserved;
} lmsgd_coeffs;

/* Result of the most recent step (all ranks see the same values). */
typedef struct lmsgd_step_status {
    int64_t first_nonfinite;   /* smallest flat index j with non-finite g_j on any rank; -1 none */
    int64_t pack_saturations;  /* sum over ranks of #{j : |s g_j| > 65504}              */
    int64_t sum_saturations;   /* #{j : |sum_ranks h_j| > 65504} (wire-2 clamp)          */
    int32_t skipped;           /* 1 if the update was not applied (non-finite / timeout) */
    int32_t error;             /* 0, LMSGD_ERR_NONFINITE or LMSGD_ERR_TIMEOUT             */
} lmsgd_step_status;

typedef struct lmsgd_ctx lmsgd_ctx;   /* opaque, library-owned */

/* init flags */
#define LMSGD_FLAG_NO_SKIP 0x1u   /* k = 1: single-pass fused pack+update (28 B/elem); non-finite
                                     gradients are detected and reported but NOT skipped.
                                     Ignored for world > 1, where the skip decision is free
                                     (the reduce needs every rank's payload anyway). */
#define LMSGD_FLAG_FREEZE_M 0x2u  /* lmsgd_step only: on steps with alpha_rmsprop == 0 (SGD after the
                                     warm-up) m is neither read nor written -- it
                                     does not enter Delta or theta then, so theta and Delta are
                                     bit-identical to the full rule while the update moves 18 instead
                                     of 26 B/elem.  m then holds its value from the last RMSprop step
                                     (NOT the paper's m_t); off by default.  lmsgd_step_graph ignores it. */

/* ---------------------------------------------------------------- host-only */

int lmsgd_abi_version(void);
const char* lmsgd_status_string(lmsgd_status s);

/* Fill the paper's hyperparameters (see lmsgd_hyper).  Never fails except for NULL. */
lmsgd_status lmsgd_hyper_default(lmsgd_hyper* out);

/* Schedule coefficients of iteration t >= 1, pure host
 * function, IEEE double in the operation order of DESIGN.md "Schedule":
 *   epoch = ((t-1) b_total) / n_train;  phase p = first with (t-1) b_total < E_p n_train
 *   eta = mult_p * (0.1 * b_total / 256);  a_SGD = alpha(epoch);
 *   a_RMS = ((1 - a_SGD) eta_RMSprop) / eta
 * Errors: INVALID_ARG (NULL, t < 1, non-positive sizes, beta_period <= 0),
 *         RANGE (t past the last epoch). */
lmsgd_status lmsgd_schedule_at(const lmsgd_hyper* hyper, const lmsgd_cluster* cluster,
                               int64_t t, lmsgd_coeffs* out);

/* Number of iterations T the schedule covers (90 epochs). */
lmsgd_status lmsgd_schedule_steps(const lmsgd_cluster* cluster, int64_t* T);

/* Exchange layout for world ranks and n parameters (host-only): shard =
 * ceil(n / world) rounded up to 64 elements (128 B of fp16), n_pad = world * shard.
 * Rank r owns the reduction of elements [r shard, (r+1) shard); elements >= n are
 * zero padding. */
lmsgd_status lmsgd_layout(int world, int64_t n, int64_t* shard, int64_t* n_pad);

/* ---------------------------------------------------------------- context */

/* Create the context of rank `rank` of `world` (1..LMSGD_MAX_WORLD) on CUDA
 * `device` for n_params parameters.  loss_scale s: a positive power of two, the
 * same on all ranks (R11).  hyper may be NULL (paper defaults).  Allocates the
 * fusion buffers: world == 1 needs nothing else; world > 1 must then call
 * lmsgd_ipc_handle + lmsgd_connect.  Synchronous. */
lmsgd_status lmsgd_init(lmsgd_ctx** out, int world, int rank, int device, int64_t n_params,
                        float loss_scale, const lmsgd_hyper* hyper, uint32_t flags);

/* world > 1: this rank's CUDA IPC handle of its exchange buffer
 * (LMSGD_IPC_HANDLE_BYTES host bytes).  The caller all-gathers the handles by any
 * means (e.g. torch.distributed) -- the library does no host networking. */
lmsgd_status lmsgd_ipc_handle(lmsgd_ctx* ctx, uint8_t* out);

/* world > 1: map every peer's exchange buffer.  handles = world * LMSGD_IPC_HANDLE_BYTES
 * host bytes in rank order (this rank's own entry is ignored).  Synchronous;
 * must be called by all ranks before the first step. */
lmsgd_status lmsgd_connect(lmsgd_ctx* ctx, const uint8_t* handles);

/* ---------------------------------------------------------------- NVLS (optional)
 * The fp16 all-reduce of PAPER.md:82-87 through the NVSwitch's in-switch reduction
 * (NVLink SHARP, "NVLS") instead of the peer-memory reduce-scatter.  Every rank's
 * packed wire [n_pad] fp16 lives in memory bound to one multicast object; the owner of
 * shard r reads the switch's sum of shard r over all ranks with
 * multimem.ld_reduce.add.acc::f32 (fp32 accumulation inside the switch, one rounding
 * to fp16 -- reading R8' in DESIGN.md: NOT the exact fp64 sum of the default path, so
 * R may differ from the oracle's by one fp16 rounding of an inexact fp32 sum; the
 * tolerance is 1e-3 |ghat| + 2^-24/(k s)), and counts an fp16 infinity in the result
 * as a sum saturation (saturating it to +-65504, R7).  Flags, the global skip, the
 * status words and the update are those of the default path.
 *
 * Modes (lmsgd_nvls_bind / lmsgd_nvls_mode):
 *   LMSGD_NVLS_OFF       the default peer-memory path (push + exact fp64 reduce);
 *   LMSGD_NVLS_RS        pack into the own wire (HBM only), the switch reduces each
 *                        owner's shard into its R, the update pulls R from the owners;
 *   LMSGD_NVLS_ALLREDUCE as RS, and the owner multicasts its reduced shard back into
 *                        every rank's wire in place (multimem.st), so the update (and
 *                        lmsgd_exchange's copy-out) reads R from local HBM.
 * Bootstrap (one GPU per rank; collective, in this order, with a barrier where noted):
 *   rank 0: lmsgd_nvls_create -> LMSGD_NVLS_HANDLE_BYTES host bytes, broadcast them;
 *   every rank: lmsgd_nvls_connect(handle)   [the multicast object is shared as a POSIX
 *               file descriptor, passed from rank 0 over an abstract unix socket named in
 *               the handle]; barrier;
 *   every rank: lmsgd_nvls_bind(mode); barrier before the first step.
 * Errors: UNSUPPORTED (world == 1, no multicast support on the device, group-connected
 * context), STATE (out of order), CUDA (driver call failed; the message names it). */
#define LMSGD_NVLS_HANDLE_BYTES 64
#define LMSGD_NVLS_OFF 0
#define LMSGD_NVLS_RS 1
#define LMSGD_NVLS_ALLREDUCE 2
/* *supported = 1 if `device` supports multicast objects (CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED). */
lmsgd_status lmsgd_nvls_supported(int device, int* supported);
lmsgd_status lmsgd_nvls_create(lmsgd_ctx* ctx, uint8_t* handle_out);
lmsgd_status lmsgd_nvls_connect(lmsgd_ctx* ctx, const uint8_t* handle);
lmsgd_status lmsgd_nvls_bind(lmsgd_ctx* ctx, int mode);
/* Switch between modes after lmsgd_nvls_bind (every rank the same mode, between steps). */
lmsgd_status lmsgd_nvls_mode(lmsgd_ctx* ctx, int mode);

/* Synchronizes the device, unmaps peers, frees library buffers.  NULL is a no-op.
 * world > 1: collective -- every rank must have finished its last step (e.g. a
 * barrier after lmsgd_query_status) before any rank finalizes, since peers write
 * into this rank's buffer during a step. */
lmsgd_status lmsgd_finalize(lmsgd_ctx* ctx);

/* Message of the last failing call on ctx ("" if none); valid until the next call. */
const char* lmsgd_last_error(const lmsgd_ctx* ctx);

/* Weight decay inherited from Goyal et al. ("the same settings are
 * used unless otherwise specified"; reading R12): from the next step on,
 * ghat_j <- ghat_j + lambda theta_j for j < n_decay (-1 = all n_params) before the
 * m update -- the torch.optim convention, so the caller puts the decayed tensors
 * (e.g. conv/fc weights) first and BN / bias parameters after them.  lambda = 0
 * (default) disables it.  Graph mode: set before lmsgd_schedule_upload. */
lmsgd_status lmsgd_set_weight_decay(lmsgd_ctx* ctx, double lambda, int64_t n_decay);

/* ---------------------------------------------------------------- hot path */

/* One synchronous data-parallel iteration on this rank (all ranks must call it
 * with the same coeffs, in the same order):
 *   params [n] device in/out theta;  grads [n] device in g (this rank's);
 *   delta [n], m [n] device in/out optimizer state (zero before the first step).
 * Enqueued on `stream`; returns before completion.  A non-finite gradient on ANY
 * rank leaves params/delta/m untouched on EVERY rank (reported by
 * lmsgd_query_status), unless LMSGD_FLAG_NO_SKIP at world == 1. */
lmsgd_status lmsgd_step(lmsgd_ctx* ctx, void* stream, float* params, const float* grads,
                        float* delta, float* m, const lmsgd_coeffs* coeffs);

/* The same iteration out of place, world == 1: reads theta, Delta, m from the *_in
 * buffers and writes the new state to the *_out buffers (device fp32 [n] each; outputs
 * must not overlap the inputs or grads).  The non-finite guard of lmsgd_step then costs
 * no extra pass: pack and update run as ONE pass (28 instead of 32 B/elem of HBM
 * traffic), and if a gradient turns out non-finite the outputs receive a copy of the
 * inputs (skipped = 1, LMSGD_ERR_NONFINITE from lmsgd_query_status).  Either way the
 * *_out buffers hold the state after the step, so the caller alternates two buffer sets
 * (ping-pong) without synchronising.  Results are bit-identical to lmsgd_step.
 * Like lmsgd_step it bakes the step's status slot into its launches: not for CUDA-graph
 * capture.  Errors: INVALID_ARG (NULL / misaligned / overlapping buffers, bad coeffs),
 * UNSUPPORTED (world > 1 -- there lmsgd_step's skip decision is free --, weight decay
 * set, or a context created with flags != 0: the call always guards and keeps m), STATE (a context that runs lmsgd_step_graph). */
lmsgd_status lmsgd_step_out_of_place(lmsgd_ctx* ctx, void* stream, const float* params_in, float* params_out,
                                     const float* grads, const float* delta_in, float* delta_out,
                                     const float* m_in, float* m_out, const lmsgd_coeffs* coeffs);

/* The same iteration with the gradient in HOST memory (pinned for full speed), end
 * to end: copies grads_host -> device, runs lmsgd_step, then copies the step's
 * parameters theta_t (n fp32, if params_host != NULL) and status record back into
 * params_host / *status_host (valid once `stream` has passed this point).  The
 * host->device copy runs on a library-owned copy stream into one of two device
 * staging buffers and may start as soon as the call is made (grads_host must be
 * complete then, and unchanged until `stream` passes this point); `stream` waits
 * for it, and the device->host copies run on `stream` after the step.  Consecutive
 * calls therefore overlap the host->device copy of step t+1 with the kernels and the
 * device->host copy of step t.  Errors as lmsgd_step, INVALID_ARG for NULL
 * grads_host / status_host. */
lmsgd_status lmsgd_step_host(lmsgd_ctx* ctx, void* stream, float* params, const float* grads_host,
                             float* delta, float* m, const lmsgd_coeffs* coeffs, float* params_host,
                             lmsgd_step_status* status_host);

/* lmsgd_step_out_of_place end to end from host memory, as lmsgd_step_host: grads_host
 * -> device, the one-pass guarded step (world == 1), then params_out (theta_t) ->
 * params_host (if not NULL) and the status record -> *status_host on `stream`.  The
 * entry point bench.py times as "e2e" at N = 1.  Errors as lmsgd_step_out_of_place. */
lmsgd_status lmsgd_step_out_of_place_host(lmsgd_ctx* ctx, void* stream, const float* params_in, float* params_out,
                                          const float* grads_host, const float* delta_in, float* delta_out,
                                          const float* m_in, float* m_out, const lmsgd_coeffs* coeffs,
                                          float* params_host, lmsgd_step_status* status_host);

/* The fp16 all-reduce of the step on its own -- rows a2-a4 (pack, reduce-scatter,
 * all-gather) without the update; PAPER.md:82-87 ("half-precision floats for
 * communication" in the all-reduce), readings R7-R10 and R19:
 *   R_out[j] = sat16_RNE( sum_{r<k} sat16_RNE(s * g_r[j]) )  for j < n_params,
 *   R_out[j] = 0                                               for n_params <= j < n_pad,
 * binary16 bits, the exact sum rounded once (the payload lmsgd_step averages as
 * fp32(R) / (k s)).  grads: device fp32 [n_params], this rank's gradient;
 * R_out: device uint16 [n_pad] (lmsgd_layout(world, n_params)), caller-owned,
 * identical on every rank afterwards.  Collective: every rank calls it, in the same
 * order relative to lmsgd_step (both advance the context's step counter).
 * Enqueued on `stream`.  lmsgd_query_status reports the saturation counts and the
 * first non-finite index; a non-finite gradient sets skipped = 1 and error =
 * LMSGD_ERR_NONFINITE and leaves R_out's values unspecified.  world == 1: R_out is
 * the packed gradient (k_pack + a one-warp status kernel).  Errors: INVALID_ARG (NULL / misaligned),
 * STATE (before lmsgd_connect, or on a context that runs lmsgd_step_graph). */
lmsgd_status lmsgd_exchange(lmsgd_ctx* ctx, void* stream, const float* grads, uint16_t* R_out);

/* Bucketed exchange (the exchange of a layer bucket overlapped with
 * the rest of backward, Fig. 1): one context per bucket of the flat
 * gradient, lmsgd_exchange per bucket as its gradients complete, then ONE lmsgd_update
 * (sub-step) over the concatenated R with the buckets' statuses merged:
 *   merge ctx's last exchange status into the sub-step accumulator dstatus (device
 *   int64[4], see lmsgd_status_reset): first = min(first, offset + the bucket's first
 *   non-finite index), saturation counts added, the first non-NONFINITE error kept.
 *   Stream-ordered (one thread; no host sync).  offset: the bucket's first flat index. */
lmsgd_status lmsgd_status_accumulate(lmsgd_ctx* ctx, void* stream, int64_t offset, int64_t* dstatus);
/* Cap the persistent exchange kernel (k_xstep1) of this context at `blocks` blocks
 * (0 = the default, every SM x its resident blocks), so that an exchange overlapped with
 * other work (backward) occupies only part of the GPU.  Every rank the same value. */
lmsgd_status lmsgd_set_exchange_blocks(lmsgd_ctx* ctx, int blocks);

/* ---------------------------------------------------------------- CUDA graphs
 * lmsgd_step bakes its per-step arguments (coefficients, step number) into the
 * launches, so a captured lmsgd_step would replay the same step.  The graph entry
 * point keeps everything that changes between steps in device memory instead: */

/* Upload the coefficients of iterations t_first .. t_first + count - 1
 * (lmsgd_schedule_at, hyper may be NULL) to a device table and point the device
 * cursor at its first entry.  Synchronous.  Errors: INVALID_ARG, RANGE (a step past
 * the schedule), CUDA. */
lmsgd_status lmsgd_schedule_upload(lmsgd_ctx* ctx, const lmsgd_hyper* hyper, const lmsgd_cluster* cluster,
                                   int64_t t_first, int64_t count);

/* One iteration like lmsgd_step, with the coefficients taken from the uploaded table at
 * the device cursor and the step number from a device counter; both advance on the
 * device at the end of the step.  Safe to capture in a CUDA graph (e.g.
 * torch.cuda.graph): every replay runs the next iteration.  Past the end of the table
 * the update is skipped and the status reports LMSGD_ERR_RANGE.  A context uses
 * either lmsgd_step / lmsgd_exchange or lmsgd_step_graph (LMSGD_ERR_STATE otherwise). */
lmsgd_status lmsgd_step_graph(lmsgd_ctx* ctx, void* stream, float* params, const float* grads,
                              float* delta, float* m);

/* BN statistics without moving averages (R16): on every rank,
 *   mean[c] <- fp32( (sum_{r=0..k-1} mean_r[c]) / k ),  var likewise,
 * summed in fp64 in rank order, one rounding.  mean, var: device fp32 [C],
 * 0 < C <= LMSGD_MAX_BN_CHANNELS, in/out.  world == 1: identity (no kernel). */
lmsgd_status lmsgd_bn_stats_allreduce(lmsgd_ctx* ctx, void* stream, float* mean, float* var,
                                      int64_t C);

/* Wait for the last step on its stream and report its status.  Returns
 * LMSGD_ERR_NONFINITE / LMSGD_ERR_TIMEOUT if that step was skipped. */
lmsgd_status lmsgd_query_status(lmsgd_ctx* ctx, lmsgd_step_status* out);

/* ---------------------------------------------------------------- profiling
 * Per-kernel device timing of lmsgd_step, measured with CUDA events recorded on
 * the step's stream around each kernel launch (used by bench.py for the roofline
 * of the dominant kernel).  Phases: 0 = pack (k_pack / k_fused1), 2 = update
 * (k_update; for world > 1 the whole step, whose kernels overlap -- use tracing). */

/* max_launches > 0: start recording (event pool sized for that many kernel
 * launches; further launches are not timed).  0: stop and discard.  Synchronous. */
lmsgd_status lmsgd_profile_enable(lmsgd_ctx* ctx, int64_t max_launches);

/* Wait for the recorded launches, return the summed device milliseconds and the
 * launch count of each phase (arrays of 3), and clear the record. */
lmsgd_status lmsgd_profile_read(lmsgd_ctx* ctx, double* ms, int64_t* launches);

/* Tracing of world > 1 steps: 17 %globaltimer stamps (ns, this GPU's clock) per step
 * -- pack start, pack end (last block, before its flag release), decision made
 * (all ranks' packs observed), reduce start, reduce end, update start, update go,
 * update end, flag release done, and the arrival of each rank's pack flag (8) --
 * into a ring of max_steps steps (0 disables).  lmsgd_step_out_of_place (world 1)
 * records two of them: word 0 = k_fused1_oop's start (block 0, after its dependency
 * wait) and word 7 = its end (seen by k_repair1 after its dependency wait), so the
 * kernel's duration is measured inside the step stream without events between the
 * kernels.  Synchronous. */
lmsgd_status lmsgd_trace_enable(lmsgd_ctx* ctx, int64_t max_steps);

/* Copy up to max_steps recorded steps (17 int64 each, oldest first until the ring
 * wraps) into host `out`; *steps = how many were copied.  Synchronizes the device. */
lmsgd_status lmsgd_trace_read(lmsgd_ctx* ctx, int64_t* out, int64_t max_steps, int64_t* steps);

/* ---------------------------------------------------------------- emulated groups
 * The world > 1 path (the exchange of PAPER.md:79-87 and the BN average of
 * PAPER.md:68-71) with every rank of the world as a context of ONE process on ONE GPU.
 * Ranks that wait for one another must run at the same time; separate launches (in
 * one or several streams or processes) on one GPU do not guarantee that.  So a group
 * call launches each kernel of the path ONCE for all the listed ranks: the same
 * kernels (their group instantiations) with every rank's blocks interleaved in one
 * grid -- cooperative where blocks wait on each other -- each block playing its rank
 * with that rank's arguments, buffers, flags, counters and status slots.  Results
 * are those of the same world run one process per GPU (tested bit-identical).  Used to
 * test the world > 1 kernels where there are fewer GPUs than ranks.
 *
 * lmsgd_connect_group: ctxs[0 .. world-1] are the world's contexts (lmsgd_init with
 * the same world, n_params, loss scale and device, ranks 0 .. world-1 in any order);
 * connects them in-process (peers = each other's exchange buffers, no CUDA IPC).  A
 * group-connected context accepts only the group calls (the single-rank calls return
 * LMSGD_ERR_STATE).  Errors: INVALID_ARG (NULL, mismatched contexts, duplicate rank,
 * not the whole world), STATE (already connected). */
lmsgd_status lmsgd_connect_group(lmsgd_ctx* const* ctxs, int world);

/* One lmsgd_step of the `count` listed ranks (1 <= count <= world, each rank at most
 * once; arrays indexed like ctxs): params[i], grads[i], delta[i], m[i] are rank
 * ctxs[i]'s device fp32 [n_params] buffers, coeffs is shared.  Ranks that are not
 * listed do not step, so the listed ones time out (LMSGD_ERR_TIMEOUT, as when a peer
 * process stops).  Enqueued on `stream`; lmsgd_query_status(ctxs[i]) reports rank i.
 * Errors as lmsgd_step, INVALID_ARG / STATE as lmsgd_connect_group. */
lmsgd_status lmsgd_step_group(lmsgd_ctx* const* ctxs, int count, void* stream, float* const* params,
                              const float* const* grads, float* const* delta, float* const* m,
                              const lmsgd_coeffs* coeffs);

/* lmsgd_exchange of the listed ranks: R_out[i] is rank ctxs[i]'s device uint16
 * [n_pad] output. */
lmsgd_status lmsgd_exchange_group(lmsgd_ctx* const* ctxs, int count, void* stream, const float* const* grads,
                                  uint16_t* const* R_out);

/* lmsgd_step_graph of the listed ranks (each after lmsgd_schedule_upload).  The first
 * call with a given set of buffers must be made outside stream capture (it uploads the
 * ranks' arguments, synchronously); later calls with the same buffers may be captured
 * (LMSGD_ERR_STATE if they would need an upload during capture). */
lmsgd_status lmsgd_step_graph_group(lmsgd_ctx* const* ctxs, int count, void* stream, float* const* params,
                                    const float* const* grads, float* const* delta, float* const* m);

/* lmsgd_bn_stats_allreduce of the listed ranks: mean[i], var[i] device fp32 [C] of rank
 * ctxs[i], averaged in place. */
lmsgd_status lmsgd_bn_stats_allreduce_group(lmsgd_ctx* const* ctxs, int count, void* stream, float* const* mean,
                                            float* const* var, int64_t C);

/* ---------------------------------------------------------------- sub-steps
 * Context-free single-GPU kernels, exported for parity tests and for the
 * simulated-k mode (k workers' payloads on one GPU).  `dstatus` is a device
 * int64[4] accumulator {first_nonfinite (INT64_MAX = none), pack_saturations,
 * sum_saturations, error}; reset it with lmsgd_status_reset. */

lmsgd_status lmsgd_status_reset(void* stream, int64_t* dstatus);

/* h[j] = sat16_RNE(s * g[j]) for j < n, h[j] = 0 for n <= j < n_pad.
 * g: device fp32 [n]; h: device uint16 (binary16 bits) [n_pad], n_pad >= n, n_pad % 8 == 0. */
lmsgd_status lmsgd_pack(void* stream, const float* g, int64_t n, int64_t n_pad, float loss_scale,
                        uint16_t* h, int64_t* dstatus);

/* R[j] = sat16_RNE(sum_{i<k} h[i * n_pad + j]) (exact fp64 sum), j < n_pad.
 * h: device uint16 [k][n_pad]; R: device uint16 [n_pad]; 1 <= k <= 8192. */
lmsgd_status lmsgd_reduce_local(void* stream, const uint16_t* h, int k, int64_t n_pad,
                                uint16_t* R, int64_t* dstatus);

/* ghat = fp32(R[j]) * fp32(1/(k s)) and the blended update on params/delta/m [n].
 * If dstatus != NULL and dstatus[0] != INT64_MAX (a non-finite gradient was
 * packed) the update is skipped. */
lmsgd_status lmsgd_update(void* stream, const uint16_t* R, int64_t n, int k, float loss_scale,
                          const lmsgd_hyper* hyper, const lmsgd_coeffs* coeffs,
                          float* params, float* delta, float* m, const int64_t* dstatus);

/* k = 1 single pass: pack + unpack + update without the fp16 buffer (28 B/elem). */
lmsgd_status lmsgd_fused_step1(void* stream, const float* g, int64_t n, float loss_scale,
                               const lmsgd_hyper* hyper, const lmsgd_coeffs* coeffs,
                               float* params, float* delta, float* m, int64_t* dstatus);

#if defined(LMSGD_BUILD) && defined(__GNUC__)
#pragma GCC visibility pop
#endif
#ifdef __cplusplus
}
#endif
#endif /* LMSGD_H */
