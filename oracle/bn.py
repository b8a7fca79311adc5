"""BatchNorm statistics without moving averages (oracle; test infrastructure).

PAPER.md:68-71 (section 2): "we only considered the last minibatch, instead of the
moving average, and used all-reduce communication on these statistics to obtain
the average over all workers before validation."

Reading R16: the simple arithmetic mean over workers of the per-channel
means and, separately, of the per-channel (biased) variances -- not the pooled
variance; fp32 in and out, summed in float64 in worker order, divided by k in
float64, rounded to fp32 once.
"""
from __future__ import annotations

import numpy as np


def average(stats_workers) -> np.ndarray:
    """stats_workers: [k, C] fp32 (means or vars of each worker).  Returns fp32 [C]."""
    x = np.asarray(stats_workers, dtype=np.float32)
    k = x.shape[0]
    acc = np.zeros(x.shape[1:], dtype=np.float64)
    for i in range(k):
        acc = acc + x[i].astype(np.float64)
    return (acc / k).astype(np.float32)


def sync_statistics(means, vars_):
    """(mean_c, var_c) averaged over workers."""
    return average(means), average(vars_)
