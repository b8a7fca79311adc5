#!/usr/bin/env python
"""bench.py -- throughput of the arXiv 1711.04325 hot path on B200.

One step = one synchronous data-parallel iteration after backward (all SURVEY
section 8(a) rows): pack fp32 gradients to loss-scaled fp16, fp16 all-reduce with
exact accumulation (N > 1), unpack + average, blended RMSprop/SGD update of the
25,557,032-parameter ResNet-50 buffer (BASELINE.json configs[1] at N = 1,
configs[2] at N = 2/4/8), schedule coefficients from the slow-start / RMSprop
warm-up schedule of the 32k run.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl lmsgd|reference]
    torchrun --nproc-per-node N bench.py --gpus N ...

Prints ONE JSON line on rank 0.  value = global synchronous update steps/s (one step
= every rank's gradient exchanged and every replica updated; per-GPU work is fixed
as N grows: weak scaling).  The N-replica figure (steps/s x N) and the aggregate
gradient elements/s are separate keys.
"""
from __future__ import annotations

import argparse
import ctypes
import json
import os
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "update steps/s on 25.6M-param grad buffer at 1/2/4/8 B200; HBM & NVLink GB/s vs peak"
UNIT = "steps/s"
LOSS_SCALE = 1024.0
UPDATE_BYTES_PER_ELEM = 26      # R (2) + theta, Delta, m read (12) + written (12)
PACK_BYTES_PER_ELEM = 6         # g read (4) + fp16 write (2)
FUSED_BYTES_PER_ELEM = 28       # g (4) + state read (12) + written (12)
L2_BYTES = 126 * 2 ** 20


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=2000)
    p.add_argument("--warmup", type=int, default=20)
    p.add_argument("--impl", choices=["lmsgd", "reference"], default="lmsgd")
    p.add_argument("--depth", type=int, default=50, choices=[50, 152])
    p.add_argument("--mode", choices=["out_of_place", "guarded", "fused"], default="out_of_place",
                   help="N=1: out_of_place = the guarded step in one pass, state ping-ponging between two "
                        "buffer sets (lmsgd_step_out_of_place, the default; what LMSGD uses at world 1); "
                        "guarded = in-place lmsgd_step, pack + update with the global non-finite skip; "
                        "fused = in-place single pass without the skip (LMSGD_FLAG_NO_SKIP)")
    p.add_argument("--t-start", type=int, default=1, help="first schedule step timed (1 = RMSprop warm-up)")
    p.add_argument("--nvls", choices=["off", "rs", "allreduce"], default="off",
                   help="N>1: exchange mode of the headline step (include/lmsgd.h NVLS): off = peer-memory "
                        "push + exact fp64 owner reduce (default); rs = NVSwitch reduction (fp32 accumulation) "
                        "into the owner's R; allreduce = rs + multicast of R back into every rank's wire. "
                        "Every available mode is timed in the nvlink section either way")
    p.add_argument("--nvls-ab", action="store_true",
                   help="N>1: also bind the NVLS multicast wire and time every exchange mode (nvlink.modes); "
                        "implied by --nvls rs|allreduce")
    p.add_argument("--e2e-steps", type=int, default=50)
    p.add_argument("--full-schedule", action="store_true",
                   help="config C5: time the whole 90-epoch schedule (T = 3,519 steps at 32k from t = 1) with the "
                        "BN statistics average at every epoch crossing; use with --depth 152")
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--no-profile", action="store_true", help="do not record per-kernel events")
    p.add_argument("--trace", action="store_true", help="(kept for compatibility; N>1 always traces the profile pass)")
    return p.parse_args()


def workload_name(depth: int, world: int, mode: str) -> str:
    """config.workload, identical on both arms (the oracle computes the same step)."""
    if world == 1:
        return f"resnet{depth}_grad_buffer_fused_pack_update_1gpu_{mode}"
    return f"resnet{depth}_grad_buffer_fp16_allreduce_update"


def env_rank():
    return int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)), int(os.environ.get("LOCAL_RANK", 0))


def measured_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


def committed_traffic(kernel: str):
    """DRAM bytes (read + write) per launch of `kernel` from the committed ncu
    capture (profiles/traffic.json, written by tools/ncu_summary.py), else None."""
    try:
        with open(os.path.join(ROOT, "profiles", "traffic.json")) as f:
            t = json.load(f)
    except Exception:
        return None
    for name, v in t.items():
        if name == kernel or name.startswith(kernel + "<"):
            return v
    return None


# ------------------------------------------------------------------ clocks (NVML)

class ClockSampler:
    REASONS = {0x4: "sw_power_cap", 0x8: "hw_slowdown", 0x20: "sw_thermal_slowdown",
               0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown", 0x2: "applications_clocks_setting",
               0x10: "sync_boost"}

    def __init__(self, index: int, period_s: float = 0.002):
        self.index, self.period = index, period_s
        self.samples, self.reasons = [], set()
        self.max_mhz = None
        self._stop = threading.Event()
        self._t = None
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
        except Exception as e:  # noqa: BLE001
            self.nv, self.err = None, str(e)

    def _run(self):
        nv = self.nv
        get_r = getattr(nv, "nvmlDeviceGetCurrentClocksEventReasons", None) or \
            nv.nvmlDeviceGetCurrentClocksThrottleReasons
        while not self._stop.is_set():
            try:
                self.samples.append(nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM))
                r = get_r(self.h)
                for bit, name in self.REASONS.items():
                    if r & bit:
                        self.reasons.add(name)
            except Exception:  # noqa: BLE001
                pass
            time.sleep(self.period)

    def start(self):
        if self.nv:
            self._t = threading.Thread(target=self._run, daemon=True)
            self._t.start()

    def stop(self):
        if self._t:
            self._stop.set()
            self._t.join()
        s = sorted(self.samples)
        return {"sm_mhz": s[len(s) // 2] if s else None, "sm_max_mhz": self.max_mhz,
                "reasons": sorted(self.reasons), "samples": len(s)}


class NvlinkCounters:
    """NVLink traffic of one GPU (all links) between two snapshots, from NVML:
    the field counters NVML_FI_DEV_NVLINK_COUNT_XMIT/RCV_BYTES (202/204, bytes) or
    NVML_FI_DEV_NVLINK_THROUGHPUT_DATA_TX/RX (138/139, KiB), scope UINT_MAX (every link)
    or link by link; else the GPM metrics NVML_GPM_METRIC_NVLINK_TOTAL_TX/RX_PER_SEC
    (61/60) between two GPM samples times the host time between them.  `kind` says which;
    None (and `err` says why) where the driver exposes none of them."""
    SETS = (((202, "tx"), (204, "rx"), 1), ((138, "tx"), (139, "rx"), 1024))
    LINKS = 18   # NVLink 5: 18 links per B200

    def __init__(self, index: int):
        self.kind, self.err = None, None
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv, self.h = pynvml, pynvml.nvmlDeviceGetHandleByIndex(index)
        except Exception as e:  # noqa: BLE001
            self.err = str(e)
            return
        errs = []
        for per_link in (False, True):
            for tx, rx, unit in self.SETS:
                self.fields, self.per_link = (tx, rx, unit), per_link
                try:
                    self._fields()
                    self.kind = f"nvml fields {tx[0]}/{rx[0]}" + (" per link" if per_link else "")
                    return
                except Exception as e:  # noqa: BLE001
                    errs.append(("per-link " if per_link else "") + str(e))
        try:
            sup = self.nv.nvmlGpmQueryDeviceSupport(self.h)
            if not sup.isSupportedDevice:
                raise RuntimeError("GPM not supported on this device")
            a, b = self.snapshot_gpm(), None
            time.sleep(0.01)
            b = self.snapshot_gpm()
            self._gpm_delta(a, b)
            self.kind = "nvml gpm metrics 61/60 x host time"
            return
        except Exception as e:  # noqa: BLE001
            errs.append("gpm " + str(e))
        self.err = "; ".join(errs)

    def _fields(self):
        tx, rx, unit = self.fields
        scopes = list(range(self.LINKS)) if self.per_link else [0xFFFFFFFF]
        req = [(f[0], sc) for f in (tx, rx) for sc in scopes]
        vals = self.nv.nvmlDeviceGetFieldValues(self.h, req)
        out, ok = {"tx": 0, "rx": 0}, 0
        for v, (fid, _) in zip(vals, req):
            if v.nvmlReturn == 0:
                ok += 1
                out["tx" if fid == tx[0] else "rx"] += int(v.value.ullVal) * unit
        if ok == 0:
            raise RuntimeError(f"NVML fields {tx[0]}/{rx[0]}: return {vals[0].nvmlReturn}")
        return out

    def snapshot_gpm(self):
        smp = self.nv.nvmlGpmSampleAlloc()
        self.nv.nvmlGpmSampleGet(self.h, smp)
        return smp, time.perf_counter()

    def _gpm_delta(self, a, b):
        nv = self.nv
        mg = nv.c_nvmlGpmMetricsGet_t()
        mg.version = nv.NVML_GPM_METRICS_GET_VERSION
        mg.numMetrics = 2
        mg.sample1, mg.sample2 = a[0], b[0]
        mg.metrics[0].metricId = nv.NVML_GPM_METRIC_NVLINK_TOTAL_TX_PER_SEC
        mg.metrics[1].metricId = nv.NVML_GPM_METRIC_NVLINK_TOTAL_RX_PER_SEC
        nv.nvmlGpmMetricsGet(mg)
        for i in range(2):
            if mg.metrics[i].nvmlReturn != 0:
                raise RuntimeError(f"gpm metric {mg.metrics[i].metricId}: return {mg.metrics[i].nvmlReturn}")
        dt = b[1] - a[1]
        for smp in (a[0], b[0]):
            nv.nvmlGpmSampleFree(smp)
        # NVML reports these two metrics in MiB/s
        return {"tx": mg.metrics[0].value * 2 ** 20 * dt, "rx": mg.metrics[1].value * 2 ** 20 * dt}

    def snapshot(self):
        if self.kind is None:
            return None
        return self.snapshot_gpm() if self.kind.startswith("nvml gpm") else self._fields()

    def delta(self, a, b):
        if a is None or b is None:
            return None
        if self.kind.startswith("nvml gpm"):
            out = self._gpm_delta(a, b)
        else:
            out = {k: b[k] - a[k] for k in ("tx", "rx")}
        out["source"] = self.kind
        return out


# ------------------------------------------------------------------ oracle timing (CPU)

def oracle_steps(k: int, n_full: int, budget_s: float, n_steps: int | None = None, depth: int = 50,
                 n_warm: int = 0):
    """Time the CPU oracle (as it stands) on whole steps of the workload: k workers'
    pack + exact reduce + fp16 wire + fp64 update of the n_full-element buffer.  If a
    full-size step does not fit the budget (n_steps steps in budget_s seconds, or at
    least 2 steps), each step runs on the largest leading slice that does and the
    rate is extrapolated per element.  Returns (steps/s, elems per step, steps,
    seconds, extrapolated)."""
    import numpy as np

    import synth
    from oracle import exchange, schedule, update
    # calibrate the per-element cost on a 1M slice (one step)
    cal = min(n_full, 1 << 20)
    gc = synth.grads(k, 1, cal)
    t0 = time.perf_counter()
    ex = exchange.exchange(list(gc), LOSS_SCALE)
    c = schedule.coeffs_at(1)
    update.step(np.zeros(cal), ex.ghat, np.zeros(cal), np.zeros(cal), c.eta, c.alpha_sgd, c.alpha_rmsprop)
    per_elem = (time.perf_counter() - t0) / cal
    want = n_steps if n_steps else max(2, int(budget_s / (per_elem * n_full)))
    ns = n_full if per_elem * n_full * want <= budget_s * 1.25 else \
        max(1 << 16, int(budget_s / want / per_elem))
    g = synth.grads(k, 1, ns)
    th = synth.theta0(n_full, depth)[:ns].astype(np.float64)
    d, m = np.zeros(ns), np.zeros(ns)
    for i in range(n_warm):    # untimed
        c = schedule.coeffs_at(1 + i)
        ex = exchange.exchange(list(g), LOSS_SCALE)
        th, d, m = update.step(th, ex.ghat, m, d, c.eta, c.alpha_sgd, c.alpha_rmsprop)
    t0 = time.perf_counter()
    for i in range(want):
        c = schedule.coeffs_at(1 + i)
        ex = exchange.exchange(list(g), LOSS_SCALE)
        th, d, m = update.step(th, ex.ghat, m, d, c.eta, c.alpha_sgd, c.alpha_rmsprop)
    el = time.perf_counter() - t0
    return (ns * want / el) / n_full, ns, want, el, ns < n_full


def cpu_cores_used():
    return 1   # NumPy elementwise ufuncs run on one thread


def run_reference(args):
    rank, world, _ = env_rank()
    if rank != 0:
        return 0
    import synth
    k = max(1, args.gpus)
    n = synth.resnet_n_params(args.depth)
    # one untimed warm-up step (the oracle has nothing to warm beyond page faults), then
    # exactly --steps timed oracle steps; whole steps of the full workload unless the
    # timed steps would exceed ~3 minutes
    rate, ns, calls, el, extrap = oracle_steps(k, n, 180.0, args.steps, args.depth, n_warm=min(args.warmup, 1))
    what = (f"pack x{k} workers + exact fp64 reduce + fp16 wire + fp64 update, NumPy on one core, "
            f"{calls} steps on ")
    sample = what + (f"a {ns}-element leading slice of the {n}-param buffer, extrapolated per element"
                     if extrap else f"the whole {n}-param buffer (no extrapolation)")
    line = {
        "impl": "reference", "metric": METRIC, "value": rate, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 / rate,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": DATA,
        "config": bench_config(args, k, n),
        "cpu_baseline": {"value": rate, "unit": UNIT, "cores": cpu_cores_used(), "kind": "oracle",
                         "sample": sample},
        "e2e": {"value": rate, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


def bench_config(args, world: int, n: int) -> dict:
    """config of the JSON line -- static, identical on both arms."""
    return {"workload": workload_name(args.depth, world, args.mode), "n_params": n, "k": world, "wire": "f16",
            "loss_scale": LOSS_SCALE, "schedule": "slow-start 32k (n=1024, b_local=32), t from %d" % args.t_start,
            "l2": f"inputs {n * 16 / 1e9:.2f} GB > 126 MB L2 (no flush needed)"}


DATA = "synthetic (paper-shaped: ResNet layout, minibatch-32 noise)"


# ------------------------------------------------------------------ GPU arm

def main():
    args = parse()
    if args.impl == "reference":
        return run_reference(args)
    import numpy as np
    import torch
    import torch.distributed as dist

    import paper_1711_04325_b200 as L
    import synth

    rank, world, local = env_rank()
    assert world == args.gpus, f"--gpus {args.gpus} but WORLD_SIZE {world}"
    torch.cuda.set_device(local)
    devc = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=devc)
    n = synth.resnet_n_params(args.depth)
    flags = L.LMSGD_FLAG_NO_SKIP if (args.mode == "fused" and world == 1) else 0
    ctx = L.lmsgd_init(world, rank, local, n, LOSS_SCALE, None, flags)
    L.connect_process_group(ctx)
    NV_MODES = {"off": L.LMSGD_NVLS_OFF, "rs": L.LMSGD_NVLS_RS, "allreduce": L.LMSGD_NVLS_ALLREDUCE}
    nvls_ok = False
    if world > 1:
        sup = torch.tensor([1 if L.lmsgd_nvls_supported(local) else 0], device=devc)
        dist.all_reduce(sup, op=dist.ReduceOp.MIN)
        nvls_ok = bool(sup.item()) and (args.nvls_ab or args.nvls != "off")
        if nvls_ok:   # bind the multicast wire once; the headline mode is --nvls
            L.connect_nvls(ctx, NV_MODES[args.nvls])
    assert args.nvls == "off" or nvls_ok, "--nvls needs multicast support on every GPU"

    # inputs, resident in HBM before timing (synthetic, paper-shaped; see synth / DESIGN.md)
    gen = torch.Generator(device=devc)
    gen.manual_seed(1711 + rank)
    theta = torch.from_numpy(synth.theta0(n, args.depth)).to(devc)
    a = 10.0 ** (torch.rand(n, generator=gen, device=devc) * 4.0 - 5.0)
    gen_c = torch.Generator(device=devc)
    gen_c.manual_seed(1711)
    c_sig = torch.randn(n, generator=gen_c, device=devc)
    grads = (a * (c_sig + torch.randn(n, generator=gen, device=devc) / 32 ** 0.5)).float().contiguous()
    del a, c_sig
    delta = torch.zeros(n, device=devc)
    m = torch.zeros(n, device=devc)
    cl = L.make_cluster()
    T = L.lmsgd_schedule_steps(cl)
    if args.full_schedule:
        args.steps, args.t_start = T, 1
    coeffs = [L.lmsgd_schedule_at(None, cl, (args.t_start - 1 + i) % T + 1) for i in range(args.warmup + args.steps)]
    # BN sync points of the full-schedule run: steps whose epoch crosses an integer
    bn_at = set()
    if args.full_schedule:
        ep = [c.epoch for c in coeffs[args.warmup:]] + [90.0]
        bn_at = {i for i in range(args.steps) if int(ep[i + 1]) > int(ep[i])}
        C_bn = sum(synth.resnet_bn_channels(args.depth))
        bn_mean = torch.randn(C_bn, device=devc)
        bn_var = torch.rand(C_bn, device=devc) + 0.1
    stream = torch.cuda.current_stream()
    sp = ctypes.c_void_p(stream.cuda_stream)
    P = ctypes.c_void_p
    ptrs = (P(theta.data_ptr()), P(grads.data_ptr()), P(delta.data_ptr()), P(m.data_ptr()))
    lib = L.lib()

    oop = args.mode == "out_of_place" and world == 1
    if oop:   # the second buffer set of the out-of-place step (the state alternates)
        theta2, delta2, m2 = torch.empty_like(theta), torch.empty_like(delta), torch.empty_like(m)
        sets = (ptrs, (P(theta2.data_ptr()), ptrs[1], P(delta2.data_ptr()), P(m2.data_ptr())))

    def step(i):
        if oop:
            a_, b_ = sets[i & 1], sets[(i & 1) ^ 1]
            st = lib.lmsgd_step_out_of_place(ctx.ptr, sp, a_[0], b_[0], ptrs[1], a_[2], b_[2], a_[3], b_[3],
                                             ctypes.byref(coeffs[i]))
        else:
            st = lib.lmsgd_step(ctx.ptr, sp, *ptrs, ctypes.byref(coeffs[i]))
        if st != 0:
            raise L.LmsgdError(st, lib.lmsgd_last_error(ctx.ptr).decode())

    def barrier():
        if world > 1:
            dist.barrier(device_ids=[local])

    def max_over_ranks(x: float) -> float:
        if world == 1:
            return x
        t = torch.tensor([x], device=devc, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    for i in range(args.warmup):
        step(i)
    torch.cuda.synchronize()
    if args.warmup > 0:
        code, st = L.lmsgd_query_status(ctx)
        assert code == 0, f"warm-up step status {code}"

    # kernels launched per step: out of place = k_fused1_oop + k_repair1 (status; copies
    # only on a skipped step); fused = k_fused1 + status finalize; guarded k=1 = k_pack
    # + k_update; world > 1 = k_xstep1 + k_xupdate + k_xfinalize
    kernels_per_step = 2 if (flags or oop) else (2 if world == 1 else 3)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)

    host_s = [0.0]

    def timed(profile: bool):
        if profile:
            L.lmsgd_profile_enable(ctx, kernels_per_step * args.steps)
        barrier()
        torch.cuda.synchronize()
        e0.record(stream)
        h0 = time.perf_counter()
        for i in range(args.steps):
            step(args.warmup + i)
            if i in bn_at:
                L.lmsgd_bn_stats_allreduce(ctx, bn_mean, bn_var)
        host_s[0] = time.perf_counter() - h0
        e1.record(stream)
        torch.cuda.synchronize()
        barrier()
        out = max_over_ranks(e0.elapsed_time(e1))
        prof = L.lmsgd_profile_read(ctx) if profile else {}
        if profile:
            L.lmsgd_profile_enable(ctx, 0)
        code, st = L.lmsgd_query_status(ctx)
        assert code == 0 and st.skipped == 0, f"timed step status {code}"
        return out, prof

    # 1) the headline: K steps, nothing but the steps in the stream
    clocks = ClockSampler(local)
    clocks.start()
    ms, _ = timed(False)
    ck = clocks.stop()
    host_us_per_step = host_s[0] / args.steps * 1e6   # enqueue cost; < device time => not host-bound
    # 2) the same K steps again with CUDA events around every kernel (per-kernel roofline)
    # 2) per-kernel durations of the same K steps, measured in a second pass:
    #    N = 1: CUDA events around every kernel (lmsgd_profile_enable);
    #    N > 1: %globaltimer stamps inside the kernels (lmsgd_trace_enable) -- events
    #    between the step's kernels would serialise their overlap.
    prof, trace, ms_prof = {}, None, None
    if not args.no_profile:
        if oop:
            # k_fused1_oop's start (block 0) and end (k_repair1 past its dependency wait)
            # as %globaltimer stamps inside the step stream: no events between the
            # kernels, so the per-step durations sum to at most the pass's elapsed time
            import statistics
            L.lmsgd_trace_enable(ctx, args.steps)
            ms_prof, _ = timed(False)
            tr = L.lmsgd_trace_read(ctx, args.steps)
            L.lmsgd_trace_enable(ctx, 0)
            dur = [(t["update_end"] - t["pack_start"]) / 1e3 for t in tr]
            prof = {"pack": (sum(dur) * 1e-3, len(dur))}
            trace = {"k_fused1_oop_us": {"mean": sum(dur) / len(dur), "median": statistics.median(dur),
                                         "min": min(dur), "max": max(dur), "launches": len(dur)},
                     "source": "in-kernel %globaltimer: k_fused1_oop block 0 start -> k_repair1 start (after "
                               "its griddepcontrol.wait, i.e. every k_fused1_oop block done)"}
        elif world == 1:
            ms_prof, prof = timed(True)
        else:
            import statistics
            L.lmsgd_trace_enable(ctx, args.steps)
            ms_prof, _ = timed(False)
            tr = L.lmsgd_trace_read(ctx, args.steps)
            L.lmsgd_trace_enable(ctx, 0)
            # stamps: see lmsgd_trace_enable (pack start/end, decision, reduce start/end,
            # update kernel start, first unit released, status record written)
            segs = {"pack": ("pack_start", "pack_end"), "wait_all_packs": ("pack_end", "reduce_start"),
                    "reduce_block0": ("reduce_go", "reduce_end"), "update_first_wait": ("update_start", "update_go"),
                    "update": ("update_go", "update_end"), "step": ("pack_start", "update_end"),
                    # the update kernel's whole span: its first block's start (which may
                    # precede the last reduce blocks) to the status record -- used for the
                    # roofline; "update" starts at block 0's go and can undercount, because
                    # other blocks run while block 0 still waits for its chunks
                    "update_span": ("update_start", "update_end"),
                    "publish": ("pack_end", "publish_end")}
            segs.update({f"flag_A_from_{p}": ("pack_end", f"a_seen_{p}") for p in range(world)})
            body = tr[len(tr) // 4:]
            mine = {k: statistics.median((t[b] - t[a]) / 1e3 for t in body) for k, (a, b) in segs.items()}
            allr = [None] * world
            dist.all_gather_object(allr, mine)
            trace = {"us_median_per_rank": allr}
            worst = {k: max(r[k] for r in allr) for k in ("pack", "update_span", "step")}
            prof = {"pack": (worst["pack"] * 1e-3, 1), "update": (worst["update_span"] * 1e-3, 1)}
    # 3) per-step distribution (median, p10, p90): a CUDA event pair
    #    around each of up to 500 steps, the max over ranks per step
    dist_us = None
    if not args.no_profile and not args.full_schedule:
        ks = min(args.steps, 500)
        evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(ks)]
        barrier()
        torch.cuda.synchronize()
        for i in range(ks):
            evs[i][0].record(stream)
            step(args.warmup + i)
            evs[i][1].record(stream)
        torch.cuda.synchronize()
        per = torch.tensor([a.elapsed_time(b) * 1e3 for a, b in evs], dtype=torch.float64, device=devc)
        if world > 1:
            dist.all_reduce(per, op=dist.ReduceOp.MAX)
        q = torch.quantile(per.cpu(), torch.tensor([0.1, 0.5, 0.9], dtype=torch.float64)).tolist()
        dist_us = {"steps": ks, "p10": q[0], "median": q[1], "p90": q[2],
                   "note": "one event pair per step (breaks the launch overlap between steps); max over ranks"}
    ms_per_step = ms / args.steps
    global_steps_per_s = 1e3 / ms_per_step
    value = global_steps_per_s      # synchronous steps/s of the whole job (every replica updated)

    # per-kernel roofline (dominant kernel = the update; fused kernel when --mode fused)
    peak, peak_src = measured_peaks()
    phases = {}
    for ph, (pms, cnt) in prof.items():
        if cnt:
            src = ("in-kernel %globaltimer stamps (k_fused1_oop start -> end), mean over the timed steps" if oop
                   else "cuda events around each kernel" if world == 1 else
                   "in-kernel %globaltimer trace, max over ranks; update = the k_xupdate span from its first "
                   "block's start" if ph == "update" else "in-kernel %globaltimer trace, max over ranks")
            phases[ph] = {"us_per_launch": (max_over_ranks(pms / cnt * 1e3) if world == 1 else pms * 1e3),
                          "launches": cnt if world == 1 else args.steps, "source": src}
    if oop:   # phase 0 = k_fused1_oop alone (in-kernel stamps)
        dom, dom_bytes, kname = "pack", FUSED_BYTES_PER_ELEM, "k_fused1_oop"
    elif flags:
        dom, dom_bytes, kname = "pack", FUSED_BYTES_PER_ELEM, "k_fused1"   # phase 0 = the fused kernel
    else:
        dom, dom_bytes, kname = "update", UPDATE_BYTES_PER_ELEM, "k_update" if world == 1 else "k_xupdate"
    roofline = None
    if dom in phases:
        us = phases[dom]["us_per_launch"]
        achieved = dom_bytes * n / (us * 1e-6) / 1e9
        roofline = {"bound": "hbm", "kernel": kname, "achieved": achieved, "peak": peak, "unit": "GB/s",
                    "frac": achieved / peak, "traffic": committed_traffic(kname),
                    "traffic_source": "profiles/traffic.json (ncu --set full capture, dram__bytes_read.sum + "
                                      "dram__bytes_write.sum per launch)",
                    "algorithmic_bytes_per_launch": dom_bytes * n, "bytes_per_elem": dom_bytes, "elems": n,
                    "us_per_launch": us, "peak_source": peak_src,
                    # the kernel's share of the step it was measured in (profile pass) and of the
                    # headline pass
                    "share_of_step": us * 1e-3 / (ms_prof / args.steps if ms_prof else ms_per_step),
                    "share_of_headline_step": us * 1e-3 / ms_per_step}
    if "pack" in phases and not flags and not oop and world == 1:
        phases["pack"]["gbs_algorithmic"] = PACK_BYTES_PER_ELEM * n / (phases["pack"]["us_per_launch"] * 1e-6) / 1e9
    if "update" in phases:
        phases["update"]["gbs_algorithmic"] = UPDATE_BYTES_PER_ELEM * n / (phases["update"]["us_per_launch"] * 1e-6) / 1e9
    nvlink = None
    if world > 1:
        n_pad = -(-n // (64 * world)) * 64 * world
        bus_bytes = 2 * (2 * n_pad) * (world - 1) / world     # nccl-tests busbw convention, fp16 payload
        nvlink = {"allreduce_bus_bytes_per_step": bus_bytes,
                  "step_bus_gbs": bus_bytes / (ms_per_step * 1e-3) / 1e9, "peak_gbs_per_dir": 900.0,
                  "measured_peer_gbs_per_dir": 770.0}
        if "pack" in phases:
            # the pack+push phase moves 2 B x N_pad x (k-1)/k out of (and into) every GPU
            push = 2 * n_pad * (world - 1) / world
            nvlink["pack_push_us"] = phases["pack"]["us_per_launch"]
            nvlink["pack_push_gbs_per_dir"] = push / (phases["pack"]["us_per_launch"] * 1e-6) / 1e9
            nvlink["pack_push_frac_of_measured_peer"] = nvlink["pack_push_gbs_per_dir"] / 770.0
        # yardstick: NCCL fp16 all-reduce of the same payload alone (not part of our path)
        buf = torch.zeros(n_pad, dtype=torch.float16, device=devc)
        for _ in range(5):
            dist.all_reduce(buf)
        torch.cuda.synchronize()
        barrier()
        y0, y1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        y0.record(stream)
        for _ in range(20):
            dist.all_reduce(buf)
        y1.record(stream)
        torch.cuda.synchronize()
        nccl_ms = max_over_ranks(y0.elapsed_time(y1) / 20)
        nvlink["nccl_fp16_allreduce_us"] = nccl_ms * 1e3
        nvlink["nccl_fp16_allreduce_bus_gbs"] = bus_bytes / (nccl_ms * 1e-3) / 1e9
        del buf
        # our fp16 all-reduce alone (lmsgd_exchange: pack -> reduce -> all-gather into a
        # local buffer), same payload, same convention, in every exchange mode; the step too.
        # NVLink payload bytes from the NVML counters around each timed loop.
        counters = NvlinkCounters(local)
        rout = torch.empty(n_pad, dtype=torch.int16, device=devc)
        modes = ["off"] + (["rs", "allreduce"] if nvls_ok else [])
        per_mode = {}

        def timed_loop(fn, iters):
            for i in range(5):
                fn(i)
            torch.cuda.synchronize()
            barrier()
            c0 = counters.snapshot()
            y0.record(stream)
            for i in range(iters):
                fn(i)
            y1.record(stream)
            torch.cuda.synchronize()
            c1 = counters.snapshot()
            code, _ = L.lmsgd_query_status(ctx)
            assert code == 0, f"status {code}"
            t_ms = max_over_ranks(y0.elapsed_time(y1) / iters)
            link = None
            dl = counters.delta(c0, c1)   # taken after a device sync on both sides: these iters only
            if dl:
                link = {"tx": dl["tx"] / iters, "rx": dl["rx"] / iters, "source": dl["source"]}
            return t_ms, link

        push_alg = 2 * n_pad * (world - 1) / world           # one direction, per GPU, reduce-scatter
        for md in modes:
            if nvls_ok:
                L.lmsgd_nvls_mode(ctx, NV_MODES[md])
            x_ms, link = timed_loop(lambda i: L.lmsgd_exchange(ctx, grads, rout), 50)
            s_ms, slink = timed_loop(lambda i: step(args.warmup + i % args.steps), 50)
            per_mode[md] = {"exchange_us": x_ms * 1e3, "exchange_bus_gbs": bus_bytes / (x_ms * 1e-3) / 1e9,
                            "exchange_bus_frac_of_900": bus_bytes / (x_ms * 1e-3) / 1e9 / 900.0,
                            "step_us": s_ms * 1e3,
                            "nvml_link_bytes_per_exchange": link, "nvml_link_bytes_per_step": slink}
        if counters.kind is None:
            nvlink["nvml_counters_error"] = counters.err
        if nvls_ok:
            L.lmsgd_nvls_mode(ctx, NV_MODES[args.nvls])
        # phases of the exchange alone (in-kernel stamps, medians, max over ranks):
        # pack+push, the wait for every rank's push, the reduce, and the all-gather pull
        # (k_xgather) up to the status record
        import statistics
        L.lmsgd_trace_enable(ctx, 50)
        for _ in range(50):
            L.lmsgd_exchange(ctx, grads, rout)
        tr = L.lmsgd_trace_read(ctx, 50)
        L.lmsgd_trace_enable(ctx, 0)
        xsegs = {"pack_push": ("pack_start", "pack_end"), "wait_all_pushes": ("pack_end", "reduce_start"),
                 "reduce": ("reduce_go", "reduce_end"), "gather_after_reduce": ("reduce_end", "update_end"),
                 "gather_block0_start": ("reduce_end", "update_start"),
                 "gather_block0_first_chunk": ("update_start", "update_go"),
                 "gather_from_first_chunk": ("update_go", "update_end"),
                 "exchange": ("pack_start", "update_end")}
        mine_x = {k_: statistics.median((t[b] - t[a]) / 1e3 for t in tr[10:]) for k_, (a, b) in xsegs.items()}
        allx = [None] * world
        dist.all_gather_object(allx, mine_x)
        nvlink["exchange_trace_us"] = {k_: max(r[k_] for r in allx) for k_ in xsegs}
        nvlink["modes"] = per_mode
        nvlink["algorithmic_link_bytes_per_gpu"] = {
            "off": {"tx": 2 * push_alg, "rx": 2 * push_alg,
                    "note": "push 2 N_pad (k-1)/k out + R served to the peers' all-gather 2 N_pad (k-1)/k"},
            "rs_allreduce": {"note": "switch reads every rank's wire (2 N_pad out per GPU, of which 2 N_pad/k "
                                     "may stay local), returns the owner's reduced shard (2 N_pad/k in); "
                                     "allreduce adds the multicast of R: 2 N_pad/k out, 2 N_pad in"}}
        hd = per_mode[args.nvls]
        nvlink["lmsgd_exchange_us"] = hd["exchange_us"]
        nvlink["lmsgd_exchange_bus_gbs"] = hd["exchange_bus_gbs"]
        nvlink["lmsgd_exchange_bus_frac_of_900"] = hd["exchange_bus_frac_of_900"]
        best = min(per_mode, key=lambda k_: per_mode[k_]["exchange_us"])
        nvlink["fastest_exchange_mode"] = best
        nvlink["fastest_step_mode"] = min(per_mode, key=lambda k_: per_mode[k_]["step_us"])
        del rout
        # X-A2A yardstick (NCCL, not our path): our pack -> NCCL all-to-all of the fp16
        # shards -> our exact local reduce of the k received slots -> NCCL all-gather of R
        shard = n_pad // world
        h16 = torch.empty(n_pad, dtype=torch.int16, device=devc)
        recv = torch.empty(n_pad, dtype=torch.int16, device=devc)
        Rsh = torch.empty(shard, dtype=torch.int16, device=devc)
        outg = torch.empty(n_pad, dtype=torch.int16, device=devc)
        f16 = lambda t: t.view(torch.float16)   # NCCL has no int16; the collectives only move bits  # noqa: E731
        dstat = torch.empty(4, dtype=torch.int64, device=devc)

        def a2a(i):
            L.lmsgd_status_reset(dstat)
            L.lmsgd_pack(grads, n_pad, LOSS_SCALE, h16, dstat)
            dist.all_to_all_single(f16(recv), f16(h16))
            L.lmsgd_reduce_local(recv, world, shard, Rsh, dstat)
            dist.all_gather_into_tensor(f16(outg), f16(Rsh))

        for i in range(5):
            a2a(i)
        torch.cuda.synchronize()
        barrier()
        y0.record(stream)
        for i in range(20):
            a2a(i)
        y1.record(stream)
        torch.cuda.synchronize()
        a_ms = max_over_ranks(y0.elapsed_time(y1) / 20)
        nvlink["x_a2a_yardstick_us"] = a_ms * 1e3
        nvlink["x_a2a_yardstick_bus_gbs"] = bus_bytes / (a_ms * 1e-3) / 1e9
        nvlink["x_a2a_note"] = ("lmsgd_pack + NCCL all_to_all_single (fp16) + lmsgd_reduce_local (exact) + NCCL "
                                "all_gather_into_tensor: the NCCL route that keeps >= fp32 accumulation")
        del h16, recv, Rsh, outg

    # config C4: BN last-minibatch statistics average over the ranks (53 layers, 26,560
    # channels for ResNet-50), latency-bound; device time per call, max over ranks
    bn = None
    if world > 1:
        C = sum(synth.resnet_bn_channels(args.depth))
        mean = torch.randn(C, device=devc)
        var = torch.rand(C, device=devc) + 0.1
        for _ in range(20):
            L.lmsgd_bn_stats_allreduce(ctx, mean, var)
        torch.cuda.synchronize()
        barrier()
        nb = 1000
        e0.record(stream)
        for _ in range(nb):
            L.lmsgd_bn_stats_allreduce(ctx, mean, var)
        e1.record(stream)
        torch.cuda.synchronize()
        bn_us = max_over_ranks(e0.elapsed_time(e1) / nb * 1e3)
        y = torch.cat([mean, var])
        for _ in range(20):
            dist.all_reduce(y)
        torch.cuda.synchronize()
        e0.record(stream)
        for _ in range(200):
            dist.all_reduce(y)
            y.mul_(1.0 / world)
        e1.record(stream)
        torch.cuda.synchronize()
        bn = {"channels": C, "bytes": 8 * C, "us_per_call": bn_us,
              "nccl_fp32_allreduce_plus_scale_us": max_over_ranks(e0.elapsed_time(e1) / 200 * 1e3)}

    # e2e through the public host-buffer entry points, every step: H2D of this step's
    # gradient from pinned memory, the whole step, D2H of theta_t and the status record
    # (N = 1: lmsgd_step_out_of_place_host, the one-pass guarded step; N > 1:
    # lmsgd_step_host)
    g_host = grads.cpu().pin_memory()
    st_host = torch.zeros(4, dtype=torch.int64).pin_memory()
    th_host = torch.empty(n, dtype=torch.float32).pin_memory()
    gp, sh, thp = P(g_host.data_ptr()), P(st_host.data_ptr()), P(th_host.data_ptr())
    ke = max(1, min(args.e2e_steps, args.steps))

    def step_host(i):
        if oop:
            a_, b_ = sets[i & 1], sets[(i & 1) ^ 1]
            s_ = lib.lmsgd_step_out_of_place_host(ctx.ptr, sp, a_[0], b_[0], gp, a_[2], b_[2], a_[3], b_[3],
                                                  ctypes.byref(coeffs[i % len(coeffs)]), thp, sh)
        else:
            s_ = lib.lmsgd_step_host(ctx.ptr, sp, ptrs[0], gp, ptrs[2], ptrs[3], ctypes.byref(coeffs[i % len(coeffs)]),
                                     thp, sh)
        if s_ != 0:
            raise L.LmsgdError(s_, lib.lmsgd_last_error(ctx.ptr).decode())

    for i in range(4):
        step_host(i)
    torch.cuda.synchronize()
    barrier()
    torch.cuda.synchronize()
    e0.record(stream)
    for i in range(ke):
        step_host(i)
    e1.record(stream)
    torch.cuda.synchronize()
    barrier()
    assert L.decode_status(st_host).error == 0
    e2e_ms = max_over_ranks(e0.elapsed_time(e1)) / ke
    e2e = {"value": 1e3 / e2e_ms, "unit": UNIT, "h2d_bytes_per_step": 4 * n,
           "d2h_bytes_per_step": 4 * n + ctypes.sizeof(L.StepStatus), "ms_per_step": e2e_ms, "steps": ke,
           "api": "lmsgd_step_out_of_place_host" if oop else "lmsgd_step_host",
           # PCIe-bound: the H2D of step t+1 overlaps the kernels and the D2H of step t
           "pcie_gbs_per_dir": 4 * n / (e2e_ms * 1e-3) / 1e9}

    # N = 1: also time the in-place single-pass variant without the skip (LMSGD_FLAG_NO_SKIP,
    # BASELINE.json configs[1] "fused fp16-pack + blended update") and the guarded mode the
    # headline does not use
    variants = None
    if world == 1 and not flags and not args.no_profile:
        ctxf = L.lmsgd_init(1, 0, local, n, LOSS_SCALE, None, L.LMSGD_FLAG_NO_SKIP)
        thf, df, mf = theta.clone(), delta.clone(), m.clone()
        pf = (P(thf.data_ptr()), P(grads.data_ptr()), P(df.data_ptr()), P(mf.data_ptr()))
        for i in range(args.warmup):
            lib.lmsgd_step(ctxf.ptr, sp, *pf, ctypes.byref(coeffs[i]))
        torch.cuda.synchronize()
        e0.record(stream)
        for i in range(args.steps):
            lib.lmsgd_step(ctxf.ptr, sp, *pf, ctypes.byref(coeffs[args.warmup + i]))
        e1.record(stream)
        torch.cuda.synchronize()
        fms = e0.elapsed_time(e1) / args.steps
        codef, _ = L.lmsgd_query_status(ctxf)
        assert codef == 0
        variants = {"fused_no_skip": {"ms_per_step": fms, "value": 1e3 / fms, "unit": UNIT,
                                      "hbm_gbs_algorithmic": FUSED_BYTES_PER_ELEM * n / (fms * 1e-3) / 1e9,
                                      "frac_of_measured_hbm": FUSED_BYTES_PER_ELEM * n / (fms * 1e-3) / 1e9 / peak,
                                      "note": "single pass (pack+update, 28 B/elem); non-finite gradients are "
                                              "reported but not skipped"}}
        L.lmsgd_finalize(ctxf)
        del thf, df, mf
        # the guarded step the headline does not run: in place (lmsgd_step, pack + update,
        # 32 B/elem) when the headline is out of place, and vice versa
        ctxo = L.lmsgd_init(1, 0, local, n, LOSS_SCALE)
        vs = [(theta.clone(), delta.clone(), m.clone()), (torch.empty_like(theta), torch.empty_like(delta),
                                                          torch.empty_like(m))]
        pset = [tuple(P(x.data_ptr()) for x in st_) for st_ in vs]
        gp_ = P(grads.data_ptr())

        def step_other(i):
            a_, b_ = pset[i & 1], pset[(i & 1) ^ 1]
            if oop:
                r_ = lib.lmsgd_step(ctxo.ptr, sp, a_[0], gp_, a_[1], a_[2], ctypes.byref(coeffs[i]))
            else:
                r_ = lib.lmsgd_step_out_of_place(ctxo.ptr, sp, a_[0], b_[0], gp_, a_[1], b_[1], a_[2], b_[2],
                                                 ctypes.byref(coeffs[i]))
            if r_ != 0:
                raise L.LmsgdError(r_, lib.lmsgd_last_error(ctxo.ptr).decode())

        for i in range(args.warmup):
            step_other(i)
        torch.cuda.synchronize()
        e0.record(stream)
        for i in range(args.steps):
            step_other(args.warmup + i)
        e1.record(stream)
        torch.cuda.synchronize()
        oms = e0.elapsed_time(e1) / args.steps
        codeo, _ = L.lmsgd_query_status(ctxo)
        assert codeo == 0
        vb = UPDATE_BYTES_PER_ELEM + PACK_BYTES_PER_ELEM if oop else FUSED_BYTES_PER_ELEM
        variants["guarded_in_place" if oop else "guarded_out_of_place"] = {
            "ms_per_step": oms, "value": 1e3 / oms, "unit": UNIT,
            "hbm_gbs_algorithmic": vb * n / (oms * 1e-3) / 1e9,
            "frac_of_measured_hbm": vb * n / (oms * 1e-3) / 1e9 / peak, "gpu_launches_per_step": 2,
            "note": ("lmsgd_step in place: k_pack + k_update (32 B/elem), the same results and skip" if oop else
                     "lmsgd_step_out_of_place: the same results and skip in one pass (28 B/elem), the state "
                     "alternating between two buffer sets")}
        L.lmsgd_finalize(ctxo)
        del vs

    # N = 1 out of place: a skipped step (a non-finite gradient) = the fused pass + the
    # repair copy in -> out by k_repair1 (24 B/elem more)
    if oop and not args.no_profile:
        bad = grads.clone()
        bad[n // 2] = float("nan")
        pb = P(bad.data_ptr())
        kk = 20
        torch.cuda.synchronize()
        e0.record(stream)
        for i in range(kk):
            a_, b_ = sets[i & 1], sets[(i & 1) ^ 1]
            lib.lmsgd_step_out_of_place(ctx.ptr, sp, a_[0], b_[0], pb, a_[2], b_[2], a_[3], b_[3],
                                        ctypes.byref(coeffs[i]))
        e1.record(stream)
        torch.cuda.synchronize()
        sk_ms = e0.elapsed_time(e1) / kk
        codes, sts = L.lmsgd_query_status(ctx)
        assert codes == L.LMSGD_ERR_NONFINITE and sts.skipped == 1
        variants = variants or {}
        variants["out_of_place_skipped_step"] = {
            "ms_per_step": sk_ms, "steps": kk,
            "hbm_gbs_algorithmic": (FUSED_BYTES_PER_ELEM + 24) * n / (sk_ms * 1e-3) / 1e9,
            "note": "every step has a non-finite gradient: k_fused1_oop (28 B/elem) + k_repair1's copy in -> out "
                    "(24 B/elem, one block per SM)"}
        del bad

    # SGD phase (alpha_RMSprop = 0, t >= 490 at 32k: 86% of the 3,519 steps), with and
    # without LMSGD_FLAG_FREEZE_M (m not touched: 18 instead of 26 B/elem in the update)
    if not args.no_profile and not args.full_schedule:
        variants = variants or {}
        t_sgd = 1000
        csgd = [L.lmsgd_schedule_at(None, cl, t_sgd + i) for i in range(args.warmup + args.steps)]
        for name, vflags in (("sgd_phase", flags), ("sgd_phase_freeze_m", flags | L.LMSGD_FLAG_FREEZE_M)):
            ctxv = L.lmsgd_init(world, rank, local, n, LOSS_SCALE, None, vflags)
            L.connect_process_group(ctxv)
            if nvls_ok and args.nvls != "off":
                L.connect_nvls(ctxv, NV_MODES[args.nvls])
            thv, dv_, mv = theta.clone(), delta.clone(), m.clone()
            pv = (P(thv.data_ptr()), P(grads.data_ptr()), P(dv_.data_ptr()), P(mv.data_ptr()))
            vo = oop and name == "sgd_phase"   # the headline's own mode, out of place at N = 1
            if vo:
                thw, dw, mw = torch.empty_like(thv), torch.empty_like(dv_), torch.empty_like(mv)
                pw = (P(thw.data_ptr()), pv[1], P(dw.data_ptr()), P(mw.data_ptr()))

            def vstep(i):
                if vo:
                    a_, b_ = (pv, pw) if i % 2 == 0 else (pw, pv)
                    lib.lmsgd_step_out_of_place(ctxv.ptr, sp, a_[0], b_[0], pv[1], a_[2], b_[2], a_[3], b_[3],
                                                ctypes.byref(csgd[i]))
                else:
                    lib.lmsgd_step(ctxv.ptr, sp, *pv, ctypes.byref(csgd[i]))

            for i in range(args.warmup):
                vstep(i)
            torch.cuda.synchronize()
            barrier()
            torch.cuda.synchronize()
            e0.record(stream)
            for i in range(args.steps):
                vstep(args.warmup + i)
            e1.record(stream)
            torch.cuda.synchronize()
            barrier()
            vms = max_over_ranks(e0.elapsed_time(e1)) / args.steps
            codev, _ = L.lmsgd_query_status(ctxv)
            assert codev == 0
            variants[name] = {"ms_per_step": vms, "value": 1e3 / vms, "unit": UNIT, "t_from": t_sgd,
                              "note": ("alpha_RMSprop = 0: the SGD instantiation of the same step"
                                       if name == "sgd_phase" else
                                       "LMSGD_FLAG_FREEZE_M (in-place lmsgd_step): theta and Delta bit-identical "
                                       "to the full rule, m left at its last RMSprop-phase value (not the "
                                       "paper's m_t)")}
            barrier()
            L.lmsgd_finalize(ctxv)
            del thv, dv_, mv

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        rate, ns, calls, el, extrap = oracle_steps(1, n, 15.0, None, args.depth)
        cpu = {"value": rate, "unit": UNIT, "cores": cpu_cores_used(), "kind": "oracle",
               "sample": f"{calls} whole oracle steps (pack + exact reduce + fp16 wire + fp64 update, k=1) on "
                         + (f"a {ns}-element slice of the {n}-param buffer, extrapolated per element" if extrap
                            else f"the whole {n}-param buffer") + f", {el:.1f} s",
               "host_cores_available": len(os.sched_getaffinity(0))}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f32", "data": DATA,
            "config": bench_config(args, world, n),
            # every step updates N replicas of the n-element buffer from N gradients
            "replica_update_steps_per_s": global_steps_per_s * world,
            "grad_elems_per_s": global_steps_per_s * world * n,
            "roofline": roofline, "phases": phases, "nvlink": nvlink, "bn_stats_allreduce": bn,
            "variants": variants,
            "cpu_baseline": cpu, "e2e": e2e,
            "clocks": ck, "gpu_launches": kernels_per_step * args.steps,
            "profile_pass_ms_per_step": (ms_prof / args.steps) if ms_prof else None,
            "step_us_distribution": dist_us,
            "host_enqueue_us_per_step": host_us_per_step,
            "full_schedule": ({"steps": args.steps, "bn_syncs": len(bn_at), "total_s": ms / 1e3,
                               "note": "config C5: whole 90-epoch slow-start / RMSprop warm-up schedule"}
                              if args.full_schedule else None),
            "trace": trace,
        }
        print(json.dumps(line), flush=True)
    L.lmsgd_finalize(ctx)
    if world > 1:
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
