"""BatchNorm without moving averages, end to end.

"we only considered the last minibatch, instead of the moving average, and used
all-reduce communication on these statistics to obtain the average over all
workers before validation."

* ``last_minibatch_bn(model)`` sets ``momentum = 1.0`` on every BatchNorm layer, so
  its running statistics are exactly the last training minibatch's (no moving
  average).
* ``BNStatsSync(model, ctx)`` re-points every layer's ``running_mean`` /
  ``running_var`` buffer at a view of two flat fp32 device buffers (no copies), and
  ``sync()`` averages them over the ranks with ``lmsgd_bn_stats_allreduce`` (one
  sm_100a kernel, fp64 sum in rank order, one rounding -- reading R16).

torch stores the unbiased minibatch variance in ``running_var``; the library averages
what it is given (R16: the bias convention is the caller's).  Plumbing only: the
average itself runs in the library.
"""
from __future__ import annotations

import torch

from . import lmsgd as L

_BN = (torch.nn.BatchNorm1d, torch.nn.BatchNorm2d, torch.nn.BatchNorm3d)


def bn_layers(model: torch.nn.Module):
    return [m for m in model.modules() if isinstance(m, _BN) and m.track_running_stats]


def last_minibatch_bn(model: torch.nn.Module) -> torch.nn.Module:
    for m in bn_layers(model):
        m.momentum = 1.0
    return model


class BNStatsSync:
    def __init__(self, model: torch.nn.Module, ctx: L.Context):
        self.ctx = ctx
        self.layers = bn_layers(model)
        if not self.layers:
            raise ValueError("model has no BatchNorm layers with running statistics")
        dev = self.layers[0].running_mean.device
        C = sum(m.num_features for m in self.layers)
        if C > L.LMSGD_MAX_BN_CHANNELS:
            raise ValueError("more BN channels than LMSGD_MAX_BN_CHANNELS")
        self.mean = torch.empty(C, dtype=torch.float32, device=dev)
        self.var = torch.empty(C, dtype=torch.float32, device=dev)
        off = 0
        for m in self.layers:
            c = m.num_features
            self.mean[off:off + c].copy_(m.running_mean)
            self.var[off:off + c].copy_(m.running_var)
            m._buffers["running_mean"] = self.mean[off:off + c]
            m._buffers["running_var"] = self.var[off:off + c]
            off += c
        self.channels = C

    def sync(self, stream=None):
        """Average every layer's last-minibatch statistics over the ranks (before
        validation).  Enqueued on the current stream."""
        L.lmsgd_bn_stats_allreduce(self.ctx, self.mean, self.var, stream)
