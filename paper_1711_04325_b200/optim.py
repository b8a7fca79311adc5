"""torch-style front end of the hot path: ``LMSGD`` (plumbing only).

What a training script calls instead of ``torch.optim.SGD``: it lays the model's
parameters and gradients out as views of two flat fp32 device buffers (SURVEY
section 8(a) row a1, zero-copy: autograd accumulates straight into the flat gradient),
takes each iteration's coefficients from the host schedule (row a0,
``lmsgd_schedule_at``: slow-start LR + RMSprop warm-up)
and runs the exchange + blended update through ``lmsgd_step`` (rows a2-a6, the
sm_100a kernels).  Nothing here touches a gradient or a parameter value.

Weight decay (reading R12): the decayed parameters (by default every
tensor with more than one dimension -- conv and fc weights; BN and biases excluded,
Goyal et al.'s convention) are placed first in the flat buffer so the library's
decayed prefix covers exactly them.

Out of place (``out_of_place=True``; opt-in, world 1, no weight decay, no flags): the
parameters, Delta and m live in two buffer sets; each step reads one set and writes
the other through ``lmsgd_step_out_of_place`` (the guarded step in one pass over HBM,
28 instead of 32 B/elem), then the parameters' ``.data`` are re-pointed at the new
set.  Results are bit-identical to the in-place step.  The price: every parameter's
storage address alternates between two buffers from step to step, so anything that
caches a parameter's storage -- a forward/backward captured in a CUDA graph, a
saved ``p.data`` or ``flat_p`` -- would keep reading the stale set.  That is why the
mode is off by default; use the in-place step (the default) with captured graphs.

Checkpoint/resume: ``state_dict`` holds the step counter t and the optimizer state
(Delta, m) -- with the parameters, everything the next step depends on.
"""
from __future__ import annotations

from typing import Callable, Iterable

import torch

from . import lmsgd as L


def _default_decay(p: torch.Tensor) -> bool:
    return p.dim() > 1


class LMSGD:
    def __init__(self, params: Iterable[torch.Tensor], *, cluster: L.Cluster | None = None,
                 hyper: L.Hyper | None = None, loss_scale: float = 1024.0, weight_decay: float = 0.0,
                 decay: Callable[[torch.Tensor], bool] = _default_decay, flags: int = 0,
                 group=None, t_start: int = 1, out_of_place: bool = False):
        params = [p for p in params if p.requires_grad]
        if not params:
            raise ValueError("no trainable parameters")
        dev = params[0].device
        if dev.type != "cuda" or any(p.device != dev or p.dtype != torch.float32 for p in params):
            raise ValueError("LMSGD needs fp32 parameters on one CUDA device")
        decayed = [p for p in params if weight_decay and decay(p)]
        ids = {id(p) for p in decayed}
        self.params = decayed + [p for p in params if id(p) not in ids]
        self.n = sum(p.numel() for p in self.params)
        self.n_decay = sum(p.numel() for p in decayed)
        import torch.distributed as dist
        dist_on = dist.is_available() and dist.is_initialized()
        world = dist.get_world_size(group) if dist_on else 1
        rank = dist.get_rank(group) if dist_on else 0
        if out_of_place and (world != 1 or weight_decay or flags):
            raise ValueError("out_of_place needs world == 1, no weight decay and flags == 0")
        self.out_of_place = bool(out_of_place)
        nsets = 2 if self.out_of_place else 1
        self._p = [torch.empty(self.n, dtype=torch.float32, device=dev) for _ in range(nsets)]
        self.flat_g = torch.zeros(self.n, dtype=torch.float32, device=dev)
        self._cur = 0
        self._views = [[] for _ in range(nsets)]
        off = 0
        with torch.no_grad():
            for p in self.params:   # row a1: parameters and gradients become views
                k = p.numel()
                self._p[0][off:off + k].copy_(p.reshape(-1))
                for b in range(nsets):
                    self._views[b].append(self._p[b][off:off + k].view_as(p))
                p.data = self._views[0][-1]
                p.grad = self.flat_g[off:off + k].view_as(p)
                off += k
        self.cluster = cluster if cluster is not None else L.make_cluster()
        self.hyper = hyper
        self.world, self.rank, self.group, self.loss_scale = world, rank, group, loss_scale
        self.device = dev.index if dev.index is not None else torch.cuda.current_device()
        self._init_exchange(flags, weight_decay)
        self._d = [torch.zeros(self.n, dtype=torch.float32, device=dev) for _ in range(nsets)]
        self._m = [torch.zeros(self.n, dtype=torch.float32, device=dev) for _ in range(nsets)]
        self.t = int(t_start)
        self.steps_total = L.lmsgd_schedule_steps(self.cluster)

    def _init_exchange(self, flags, weight_decay):
        self.ctx = L.lmsgd_init(self.world, self.rank, self.device, self.n, self.loss_scale, self.hyper, flags)
        L.connect_process_group(self.ctx, self.group)
        if weight_decay:
            L.lmsgd_set_weight_decay(self.ctx, weight_decay, self.n_decay)

    # the current buffer set (the one the parameters view)
    @property
    def flat_p(self) -> torch.Tensor:
        return self._p[self._cur]

    @property
    def delta(self) -> torch.Tensor:
        return self._d[self._cur]

    @property
    def m(self) -> torch.Tensor:
        return self._m[self._cur]

    # ------------------------------------------------------------------ training
    def zero_grad(self):
        """Zero the flat gradient (the per-parameter .grad views stay attached)."""
        self.flat_g.zero_()

    def _check_views(self):
        base, end = self.flat_g.data_ptr(), self.flat_g.data_ptr() + 4 * self.n
        for p in self.params:
            g = p.grad
            if g is None or not (base <= g.data_ptr() < end):
                raise RuntimeError("a parameter's .grad left the flat gradient buffer (was "
                                   "model.zero_grad(set_to_none=True) called?); use LMSGD.zero_grad()")

    def coeffs(self, t: int | None = None) -> L.Coeffs:
        return L.lmsgd_schedule_at(self.hyper, self.cluster, self.t if t is None else t)

    def step(self, stream=None) -> L.Coeffs:
        """One iteration: coefficients of step t, exchange + update (enqueued on the
        current stream; returns before completion)."""
        self._check_views()
        c = self.coeffs()
        if self.out_of_place:
            a, b = self._cur, self._cur ^ 1
            L.lmsgd_step_out_of_place(self.ctx, self._p[a], self._p[b], self.flat_g, self._d[a], self._d[b],
                                      self._m[a], self._m[b], c, stream)
            for p, v in zip(self.params, self._views[b]):   # the step's output is the new parameter set
                p.data = v
            self._cur = b
        else:
            L.lmsgd_step(self.ctx, self.flat_p, self.flat_g, self.delta, self.m, c, stream)
        self.t += 1
        return c

    def status(self):
        """(code, lmsgd_step_status) of the last step; synchronizes its stream."""
        return L.lmsgd_query_status(self.ctx)

    # ------------------------------------------------------------------ checkpoint / resume
    def state_dict(self) -> dict:
        return {"t": self.t, "n": self.n, "n_decay": self.n_decay,
                "delta": self.delta.detach().clone(), "m": self.m.detach().clone()}

    def load_state_dict(self, sd: dict):
        if sd["n"] != self.n or sd["n_decay"] != self.n_decay:
            raise ValueError("checkpoint was written for another parameter layout")
        self.t = int(sd["t"])
        self.delta.copy_(sd["delta"])
        self.m.copy_(sd["m"])

    def close(self):
        L.lmsgd_finalize(self.ctx)


def bucket_bounds(n: int, world: int, bucket_elems: int) -> list[tuple[int, int]]:
    """[lo, hi) flat ranges of the buckets, from the END of the buffer (the last layers'
    gradients are complete first): every boundary but n is a multiple of 64 * world, so
    each bucket's exchange output (n_pad = its size rounded up to 64 * world) is a
    contiguous slice of one R buffer; buckets hold about bucket_elems elements."""
    if n < 1 or world < 1 or bucket_elems < 1:
        raise ValueError("bucket_bounds: n, world and bucket_elems must be positive")
    unit = 64 * world
    bounds, hi = [], n
    while hi > 0:
        lo = max(0, (hi - bucket_elems) // unit * unit)
        if lo == hi:
            lo = max(0, hi - unit)
        bounds.append((lo, hi))
        hi = lo
    return bounds


class BucketedLMSGD(LMSGD):
    """``LMSGD`` with the exchange split into buckets of the flat gradient and overlapped
    with backward (the communication/iteration overlap of
    PAPER.md:113-116 Fig. 1).  Plumbing only:

    * the flat buffer is cut, from its end, into buckets of about ``bucket_elems``
      elements whose boundaries are multiples of 64 k (so every bucket's exchange output
      is a contiguous slice of one R buffer [n_pad]); one context per bucket;
    * a post-accumulate-grad hook counts each bucket's parameters; when the last one's
      gradient is in, the bucket's ``lmsgd_exchange`` (pack -> fp16 all-reduce with exact
      accumulation) is enqueued on a communication stream behind the backward work so
      far, and its status is merged into one accumulator (``lmsgd_status_accumulate``);
      ``exchange_blocks`` caps the exchange kernel's grid so it shares the GPU with
      backward (``lmsgd_set_exchange_blocks``);
    * ``step()`` enqueues any bucket not yet exchanged, waits for the communication
      stream and runs ONE ``lmsgd_update`` over the whole R (unpack, average and the
      blended update of PAPER.md:154-156, skipped on every rank if any bucket saw a
      non-finite gradient), then resets the accumulator.

    The arithmetic is that of ``LMSGD``'s step (the same fp16 all-reduce sum per element,
    the same update kernel body), so the results are bit-identical to it.  No weight
    decay, no out-of-place mode (the sub-step update has neither).

    One backward per step: a bucket is exchanged as soon as its gradients are in, so a
    second backward before ``step()`` (gradient accumulation) must run inside
    ``no_sync()`` -- the hooks then do nothing and ``step()`` exchanges every bucket."""

    def __init__(self, params, *, bucket_elems: int = 1 << 22, exchange_blocks: int = 0, overlap: bool = True,
                 **kw):
        if kw.get("weight_decay") or kw.get("out_of_place") or kw.get("flags"):
            raise ValueError("BucketedLMSGD: no weight decay, out-of-place mode or flags")
        self.bucket_elems, self.exchange_blocks, self.overlap = int(bucket_elems), int(exchange_blocks), overlap
        super().__init__(params, **kw)

    def _init_exchange(self, flags, weight_decay):
        dev = self.flat_g.device
        bounds = bucket_bounds(self.n, self.world, self.bucket_elems)
        self.buckets = []
        top_pad = 0
        for lo, hi in bounds:
            ctx = L.lmsgd_init(self.world, self.rank, self.device, hi - lo, self.loss_scale, self.hyper, 0)
            L.connect_process_group(ctx, self.group)
            if self.exchange_blocks:
                L.lmsgd_set_exchange_blocks(ctx, self.exchange_blocks)
            n_pad = L.lmsgd_layout(self.world, hi - lo)[1]
            top_pad = max(top_pad, lo + n_pad)
            self.buckets.append({"lo": lo, "hi": hi, "n_pad": n_pad, "ctx": ctx})
        self.ctx = self.buckets[0]["ctx"]      # any connected context serves BN (bn_sync)
        self.R = torch.zeros(top_pad, dtype=torch.int16, device=dev)
        self.dstatus = torch.empty(4, dtype=torch.int64, device=dev)
        self.last_status = torch.empty(4, dtype=torch.int64, device=dev)
        L.lmsgd_status_reset(self.dstatus)
        L.lmsgd_status_reset(self.last_status)   # status() before the first step: clean
        self.comm = torch.cuda.Stream(device=dev)
        self._upd_done = torch.cuda.Event()
        self._upd_done.record(torch.cuda.current_stream(dev))
        # parameter i -> the buckets its flat range overlaps; bucket b <- its parameter count
        self._p2b, off = [], 0
        npar = [0] * len(self.buckets)
        for p in self.params:
            k = p.numel()
            bs = [b for b, bk in enumerate(self.buckets) if bk["lo"] < off + k and off < bk["hi"]]
            self._p2b.append(bs)
            for b in bs:
                npar[b] += 1
            off += k
        self._npar = npar
        self._pending = list(npar)
        self._launched = [False] * len(self.buckets)
        self._hooks = []
        if self.overlap:
            for i, p in enumerate(self.params):
                self._hooks.append(p.register_post_accumulate_grad_hook(lambda _p, i=i: self._grad_ready(i)))

    def no_sync(self):
        """Context manager: backward passes inside it only accumulate (no bucket exchange)."""
        import contextlib

        @contextlib.contextmanager
        def _ctx():
            self._paused = True
            try:
                yield
            finally:
                self._paused = False
        return _ctx()

    def _grad_ready(self, i: int):
        if getattr(self, "_paused", False):
            return
        for b in self._p2b[i]:
            self._pending[b] -= 1
            if self._pending[b] < 0:
                raise RuntimeError("BucketedLMSGD: a second backward before step() -- its bucket was already "
                                   "exchanged; accumulate gradients inside opt.no_sync()")
            if self._pending[b] == 0:
                self._launch(b, torch.cuda.current_stream(self.flat_g.device))

    def _launch(self, b: int, after: torch.cuda.Stream):
        if self._launched[b]:
            return
        self._launched[b] = True
        bk = self.buckets[b]
        ev = torch.cuda.Event()
        ev.record(after)                       # this bucket's gradients are complete on `after`
        self.comm.wait_event(ev)
        self.comm.wait_event(self._upd_done)   # R and the accumulator are free again
        lo, hi = bk["lo"], bk["hi"]
        L.lmsgd_exchange(bk["ctx"], self.flat_g[lo:hi], self.R[lo:lo + bk["n_pad"]], self.comm)
        L.lmsgd_status_accumulate(bk["ctx"], lo, self.dstatus, self.comm)

    def step(self, stream=None) -> L.Coeffs:
        self._check_views()
        cur = stream if stream is not None else torch.cuda.current_stream(self.flat_g.device)
        for b in range(len(self.buckets)):     # buckets whose hooks did not fire (or overlap off)
            self._launch(b, cur)
        cur.wait_stream(self.comm)
        c = self.coeffs()
        L.lmsgd_update(self.R, self.n, self.world, self.loss_scale, self.hyper, c, self.flat_p, self.delta, self.m,
                       self.dstatus, cur)
        self.last_status.copy_(self.dstatus)
        L.lmsgd_status_reset(self.dstatus, cur)
        self._upd_done.record(cur)
        self._pending = list(self._npar)
        self._launched = [False] * len(self.buckets)
        self.t += 1
        return c

    def status(self):
        """(code, lmsgd_step_status) of the last step, from the merged bucket statuses."""
        torch.cuda.synchronize(self.flat_g.device)
        first, psat, ssat, err = (int(v) for v in self.last_status.cpu().tolist())
        st = L.StepStatus()
        st.first_nonfinite = -1 if first == (1 << 63) - 1 else first
        st.pack_saturations, st.sum_saturations = psat, ssat
        st.skipped = 1 if (st.first_nonfinite >= 0 or err) else 0
        st.error = err if err else (L.LMSGD_ERR_NONFINITE if st.first_nonfinite >= 0 else 0)
        return st.error, st

    def close(self):
        for h in self._hooks:
            h.remove()
        torch.cuda.synchronize(self.flat_g.device)
        for bk in self.buckets:
            L.lmsgd_finalize(bk["ctx"])
