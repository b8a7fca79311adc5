"""fp16 gradient exchange across k synchronous data-parallel workers
(oracle; test infrastructure).

PAPER.md:79-80 (synchronous data parallelism, ChainerMN) and PAPER.md:85-87
("we used half-precision floats for communication").  BASELINE.json north_star:
"flattens fp32 gradients, casts and scales them to fp16 for communication,
all-reduces them across workers, casts back and averages ... always with fp32
accumulation".

The algorithm, step by step (readings R7-R11):
  pack    h_ij = sat16_RNE(fp32(s) * g_ij)          s = loss scale, a power of two
  reduce  S_j  = sum_i h_ij, summed in float64 in worker order
                 (exact: every binary16 value is a multiple of 2^-24 below 2^16 in
                 magnitude, so any sum of <= 2^13 of them needs < 53 bits)
  wire-2  R_j  = sat16_RNE(S_j)                       the fp16 all-reduce SUM (R9, R10)
  unpack  ghat_j = fp32(R_j) * fp32(1 / (k s))       an IEEE fp32 multiply (R10)

``ideal`` gives sum_i g_ij / k in float64 with no wire rounding (to report the
fp16-wire deviation).
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import binary16


@dataclass
class ExchangeResult:
    ghat: np.ndarray      # fp32 [n], what the update consumes
    R: np.ndarray         # uint16 [n], all-reduced fp16 sum (wire-2 payload)
    S: np.ndarray         # float64 [n], exact sum of the k fp16 payloads
    pack_saturations: int
    sum_saturations: int


def _check_scale(s: float):
    m, e = np.frexp(s)
    if not (s > 0 and m == 0.5):
        raise ValueError("loss scale must be a positive power of two")


def pack(g, s: float = 1.0):
    """h = sat16_RNE(fp32(s) * g) for one worker's fp32 gradient.
    Raises binary16.NonFiniteError(first index) if g has a non-finite entry
    (R7: non-finite gradient is an error).  Returns (bits uint16, saturations)."""
    _check_scale(s)
    g = np.asarray(g, dtype=np.float32)
    bad = ~np.isfinite(g)
    if bad.any():
        raise binary16.NonFiniteError(int(np.argmax(bad)))
    with np.errstate(over="ignore"):
        x = np.float32(s) * g                 # the fp32 product (exact for finite results)
    x64 = x.astype(np.float64)
    x64 = np.where(np.isinf(x64), np.sign(x64) * 2.0 * binary16.MAX_FINITE, x64)  # fp32 overflow saturates too
    return binary16.to_binary16(x64, return_saturation=True)


def reduce_sum(h_workers) -> np.ndarray:
    """S_j = sum over workers i (in index order) of the widened fp16 values, float64."""
    S = np.zeros(np.asarray(h_workers[0]).shape, dtype=np.float64)
    for h in h_workers:
        S = S + binary16.from_binary16(h)
    return S


def unpack_average(R, k: int, s: float = 1.0) -> np.ndarray:
    """ghat = fp32(R) * fp32(1/(k s)) as one IEEE fp32 multiply."""
    inv = np.float32(1.0 / (k * s))
    return binary16.from_binary16(R).astype(np.float32) * inv


def check_finite(g_workers):
    """Reading R7: a non-finite gradient on any worker is an error; the reported
    index is the smallest flat index j at which any worker's g_j is non-finite."""
    first = None
    for g in g_workers:
        bad = ~np.isfinite(np.asarray(g, dtype=np.float32))
        if bad.any():
            j = int(np.argmax(bad))
            first = j if first is None else min(first, j)
    if first is not None:
        raise binary16.NonFiniteError(first)


def exchange(g_workers, s: float = 1.0) -> ExchangeResult:
    """The whole exchange for k = len(g_workers) workers."""
    k = len(g_workers)
    check_finite(g_workers)
    packed = [pack(g, s) for g in g_workers]
    S = reduce_sum([p[0] for p in packed])
    R, sat2 = binary16.to_binary16(S, return_saturation=True)
    ghat = unpack_average(R, k, s)
    return ExchangeResult(ghat, R, S, sum(p[1] for p in packed), sat2)


def ideal(g_workers) -> np.ndarray:
    """sum_i g_i / k in float64 (no fp16 wire)."""
    g = np.asarray(g_workers, dtype=np.float64)
    return g.sum(axis=0) / g.shape[0]
