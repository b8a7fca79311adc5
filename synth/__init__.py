"""Seeded synthetic inputs shared by the oracle tests, the GPU parity tests and bench.py.

This module holds NO arithmetic of the method (no fp16 rounding, no schedule, no
update, no reduction).  It only produces inputs with the structure of the paper's
workload (ResNet-50 / ResNet-152 trained with per-worker minibatch 32, PAPER.md:17,
PAPER.md:108, fp32 parameters PAPER.md:85):

* ``resnet_param_sizes(depth)`` -- the per-tensor element counts of torchvision's
  ResNet in ``named_parameters()`` order (the flat fusion-buffer layout).
* ``resnet_bn_channels(depth)`` -- channels of every BatchNorm layer (the BN
  statistics payload).
* ``theta0`` -- initial fp32 parameters (conv ~ N(0, 2/fan_in), BN gamma=1,
  beta=0, fc ~ N(0, 0.01^2)).
* ``grads`` -- per-worker, per-step fp32 gradients
  g[i,t,j] = a_j * (c[t,j] + z[i,t,j] / sqrt(32)), a_j = 10**U(-5,-1):
  a signal shared by all workers plus minibatch-32 noise per worker
  (recipe stated in DESIGN.md "Input recipe").
* ``bn_stats`` -- per-worker last-minibatch (mean, var) vectors.

Random streams are numpy ``SeedSequence([1711, ...])`` so host inputs are
reproducible on any machine.  Device-resident copies for timing are made by the
caller (bench.py) with torch; that is plumbing, not arithmetic of the method.
"""
from __future__ import annotations

import numpy as np

SEED = 1711
B_LOCAL = 32  # per-worker minibatch

_BLOCKS = {50: (3, 4, 6, 3), 101: (3, 4, 23, 3), 152: (3, 8, 36, 3)}


def _resnet_tensors(depth: int):
    """(kind, shape) of every parameter tensor of a torchvision bottleneck ResNet,
    in named_parameters() order.  kind in {conv, bn_w, bn_b, fc_w, fc_b}."""
    blocks = _BLOCKS[depth]
    out = [("conv", (64, 3, 7, 7)), ("bn_w", (64,)), ("bn_b", (64,))]
    inplanes = 64
    for li, nb in enumerate(blocks):
        width = 64 * (2 ** li)
        for b in range(nb):
            out += [("conv", (width, inplanes, 1, 1)), ("bn_w", (width,)), ("bn_b", (width,)),
                    ("conv", (width, width, 3, 3)), ("bn_w", (width,)), ("bn_b", (width,)),
                    ("conv", (width * 4, width, 1, 1)), ("bn_w", (width * 4,)), ("bn_b", (width * 4,))]
            if b == 0:
                out += [("conv", (width * 4, inplanes, 1, 1)), ("bn_w", (width * 4,)),
                        ("bn_b", (width * 4,))]
            inplanes = width * 4
    out += [("fc_w", (1000, 2048)), ("fc_b", (1000,))]
    return out


def resnet_param_sizes(depth: int = 50) -> list[int]:
    return [int(np.prod(s)) for _, s in _resnet_tensors(depth)]


def resnet_n_params(depth: int = 50) -> int:
    return sum(resnet_param_sizes(depth))


def resnet_bn_channels(depth: int = 50) -> list[int]:
    return [s[0] for k, s in _resnet_tensors(depth) if k == "bn_w"]


def _rng(*key: int) -> np.random.Generator:
    return np.random.default_rng(np.random.SeedSequence([SEED, *key]))


def theta0(n: int, depth: int | None = 50) -> np.ndarray:
    """Initial fp32 parameters of length n.  If depth is given and n equals that
    ResNet's size, the per-tensor init follows the tensor kinds; otherwise a
    plain N(0, 0.05^2) vector (used for small parity sizes)."""
    r = _rng(0, 0)
    if depth is not None and n == resnet_n_params(depth):
        parts = []
        for kind, shape in _resnet_tensors(depth):
            cnt = int(np.prod(shape))
            if kind == "conv":
                fan_in = int(np.prod(shape[1:]))
                parts.append(r.standard_normal(cnt) * np.sqrt(2.0 / fan_in))
            elif kind == "bn_w":
                parts.append(np.ones(cnt))
            elif kind in ("bn_b", "fc_b"):
                parts.append(np.zeros(cnt))
            else:
                parts.append(r.standard_normal(cnt) * 0.01)
        return np.concatenate(parts).astype(np.float32)
    return (r.standard_normal(n) * 0.05).astype(np.float32)


def grad_scale(n: int) -> np.ndarray:
    """a_j = 10**U(-5,-1): per-element gradient magnitude, drawn once."""
    return 10.0 ** _rng(1, 0).uniform(-5.0, -1.0, n)


def grads(k: int, t: int, n: int, a: np.ndarray | None = None) -> np.ndarray:
    """fp32 [k, n] gradients of k workers at step t (t >= 1)."""
    if a is None:
        a = grad_scale(n)
    c = _rng(2, t).standard_normal(n)
    out = np.empty((k, n), dtype=np.float32)
    for i in range(k):
        z = _rng(3, t, i).standard_normal(n)
        out[i] = (a * (c + z / np.sqrt(B_LOCAL))).astype(np.float32)
    return out


def bn_stats(k: int, channels: int, seed: int = 0) -> tuple[np.ndarray, np.ndarray]:
    """fp32 [k, C] last-minibatch means ~ N(0, 0.5^2) and biased vars ~ 0.1+Exp(1)
    (vars are non-negative, as a minibatch variance is)."""
    r = _rng(4, seed)
    mean = (r.standard_normal((k, channels)) * 0.5).astype(np.float32)
    var = (0.1 + r.exponential(1.0, (k, channels))).astype(np.float32)
    return mean, var
