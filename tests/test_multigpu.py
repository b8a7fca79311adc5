"""Multi-GPU parity (world = every visible GPU, >= 2) through torchrun; see
tests/mgpu_worker.py for what is checked.  Skipped on a 1-GPU box."""
import os
import subprocess
import sys

import pytest

torch = pytest.importorskip("torch")

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
pytestmark = [pytest.mark.gpu, pytest.mark.multigpu]


NGPU = torch.cuda.device_count() if torch.cuda.is_available() else 0


def _run(k, port, extra_env=None):
    env = dict(os.environ, LMSGD_TIMEOUT_MS="20000", PYTHONPATH=ROOT)
    env.update(extra_env or {})
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={k}",
           "--master-addr=127.0.0.1", f"--master-port={port}", os.path.join(ROOT, "tests", "mgpu_worker.py")]
    r = subprocess.run(cmd, env=env, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0 and f"MGPU_OK world={k}" in r.stdout, r.stdout[-4000:] + r.stderr[-4000:]


@pytest.mark.skipif(NGPU < 2, reason="needs >= 2 GPUs")
def test_exchange_on_all_gpus():
    _run(NGPU, 29533)


@pytest.mark.skipif(NGPU < 3, reason="needs >= 3 GPUs")
def test_exchange_three_ranks():
    # k = 3: 1/(k s) is not a power of two, shards of a ragged size
    _run(3, 29534)


@pytest.mark.skipif(NGPU < 2, reason="needs >= 2 GPUs")
def test_exchange_two_ranks_and_timeout():
    # a rank that never steps makes the other time out (status, no hang)
    _run(2, 29535, {"LMSGD_TEST_TIMEOUT": "1", "LMSGD_TIMEOUT_MS": "3000"})


@pytest.mark.skipif(not (2 <= NGPU < 8), reason="needs 2..7 GPUs (8 GPUs run world 8 natively)")
def test_world8_oversubscribed():
    # world = 8 code paths with two or more ranks per GPU (time-sliced; correctness only)
    env = dict(os.environ, LMSGD_TIMEOUT_MS="120000", PYTHONPATH=ROOT)
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=8",
           "--master-addr=127.0.0.1", "--master-port=29536", os.path.join(ROOT, "tests", "oversub_worker.py")]
    r = subprocess.run(cmd, env=env, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0 and "OVERSUB_OK world=8" in r.stdout, r.stdout[-4000:] + r.stderr[-4000:]
