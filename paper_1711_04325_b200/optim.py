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
        self.ctx = L.lmsgd_init(world, rank, dev.index if dev.index is not None else torch.cuda.current_device(),
                                self.n, loss_scale, hyper, flags)
        L.connect_process_group(self.ctx, group)
        if weight_decay:
            L.lmsgd_set_weight_decay(self.ctx, weight_decay, self.n_decay)
        self._d = [torch.zeros(self.n, dtype=torch.float32, device=dev) for _ in range(nsets)]
        self._m = [torch.zeros(self.n, dtype=torch.float32, device=dev) for _ in range(nsets)]
        self.t = int(t_start)
        self.steps_total = L.lmsgd_schedule_steps(self.cluster)

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
