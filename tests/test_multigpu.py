"""Multi-GPU parity (world = every visible GPU, >= 2) through torchrun; see
tests/mgpu_worker.py for what is checked.  Skipped on a 1-GPU box."""
import os
import subprocess
import sys

import pytest

torch = pytest.importorskip("torch")

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
pytestmark = [pytest.mark.gpu, pytest.mark.multigpu]


@pytest.mark.skipif(not torch.cuda.is_available() or torch.cuda.device_count() < 2, reason="needs >= 2 GPUs")
def test_exchange_on_all_gpus():
    k = torch.cuda.device_count()
    env = dict(os.environ, LMSGD_TIMEOUT_MS="20000", PYTHONPATH=ROOT)
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={k}",
           "--master-addr=127.0.0.1", "--master-port=29533", os.path.join(ROOT, "tests", "mgpu_worker.py")]
    r = subprocess.run(cmd, env=env, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0 and f"MGPU_OK world={k}" in r.stdout, r.stdout[-4000:] + r.stderr[-4000:]
