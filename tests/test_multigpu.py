"""World > 1 parity through torchrun; see tests/mgpu_worker.py for what is checked.

Two ways to get world > 1 ranks:
  * one GPU per rank (NGPU >= world): NCCL bootstrap, the exchange over NVLink;
  * oversubscribed (world > NGPU, including a 1-GPU box): rank r on GPU r % NGPU,
    gloo bootstrap, the exchange's peer mappings are CUDA-IPC mappings of another
    process's buffer on the same device.  Every world > 1 kernel (k_xstep1, k_xupdate,
    k_xgather, k_xfinalize, k_bn_allreduce) then runs its full cross-rank protocol --
    flags, epochs, status slots, owner-computes exact reduce, fused all-gather -- with
    the GPU time-slicing between the ranks' contexts (correctness only, no timing).
The oversubscribed runs are OPT-IN (LMSGD_OVERSUB=1): kernels that wait on one another
are not guaranteed to be co-scheduled when they are separate launches on one GPU, and the
pool's profiling guide records Xid 109 (context-switch timeout) for 2 and 4 such ranks as
processes on one B200.  They passed on a 1-GPU box once
(profiles/r2/pytest_gpu_1gpu_oversub_processes.txt); the default coverage of the world > 1
kernels with fewer GPUs than ranks is tests/test_group_gpu.py (every rank's blocks in one
launch).
"""
import os
import subprocess
import sys

import pytest

torch = pytest.importorskip("torch")

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
pytestmark = [pytest.mark.gpu, pytest.mark.multigpu]


NGPU = torch.cuda.device_count() if torch.cuda.is_available() else 0
OVERSUB = os.environ.get("LMSGD_OVERSUB") == "1"
needs_gpu = pytest.mark.skipif(NGPU < 1, reason="needs a GPU")


def oversub(world):
    return pytest.mark.skipif(world > NGPU and not OVERSUB,
                              reason="more ranks than GPUs: opt-in (LMSGD_OVERSUB=1); see test_group_gpu.py")


def _run(k, port, worker="mgpu_worker.py", extra_env=None, ok=None, timeout=900):
    env = dict(os.environ, LMSGD_TIMEOUT_MS="60000" if k > NGPU else "20000", PYTHONPATH=ROOT)
    env.update(extra_env or {})
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={k}",
           "--master-addr=127.0.0.1", f"--master-port={port}", os.path.join(ROOT, "tests", worker)]
    r = subprocess.run(cmd, env=env, capture_output=True, text=True, timeout=timeout)
    ok = ok or f"MGPU_OK world={k}"
    assert r.returncode == 0 and ok in r.stdout, r.stdout[-4000:] + r.stderr[-4000:]


@pytest.mark.skipif(NGPU < 2, reason="needs >= 2 GPUs (one per rank)")
def test_exchange_on_all_gpus():
    _run(NGPU, 29533)


@pytest.mark.skipif(NGPU < 3, reason="needs >= 3 GPUs")
def test_exchange_three_ranks():
    # k = 3: 1/(k s) is not a power of two, shards of a ragged size
    _run(3, 29534)


@needs_gpu
@oversub(2)
def test_exchange_two_ranks_and_timeout():
    # a rank that never steps makes the other time out (status, no hang); oversubscribed
    # on a 1-GPU box
    _run(2, 29535, extra_env={"LMSGD_TEST_TIMEOUT": "1", "LMSGD_TIMEOUT_MS": "3000"})


@needs_gpu
@oversub(2)
@pytest.mark.skipif(NGPU >= 2, reason="NGPU >= 2 runs world 2 natively (test_exchange_on_all_gpus)")
def test_world2_oversubscribed():
    # the whole mgpu_worker suite at world 2 with both ranks on GPU 0 (gloo bootstrap)
    _run(2, 29537)


@needs_gpu
@oversub(4)
@pytest.mark.skipif(NGPU >= 4, reason="NGPU >= 4 runs world 4 with one GPU per rank")
def test_world4_oversubscribed():
    # the whole mgpu_worker suite at world 4, ranks time-sharing the visible GPUs
    _run(4, 29538, extra_env={"LMSGD_STRESS_STEPS": "200"})


@needs_gpu
@oversub(8)
@pytest.mark.skipif(NGPU >= 8, reason="8 GPUs run world 8 natively")
def test_world8_oversubscribed():
    # world = 8 code paths (8 flag slots, 8-way exact reduce, shard layout) with several
    # ranks per GPU (time-sliced; correctness only)
    _run(8, 29536, worker="oversub_worker.py", extra_env={"LMSGD_TIMEOUT_MS": "120000"},
         ok="OVERSUB_OK world=8")


def _nvls_supported():
    if NGPU < 2:
        return False
    import paper_1711_04325_b200 as L
    return L.lmsgd_nvls_supported(0)


@pytest.mark.skipif(NGPU < 2, reason="NVLS needs >= 2 GPUs (one per rank, one multicast object)")
def test_nvls_on_all_gpus():
    # the NVSwitch-reduction exchange (LMSGD_NVLS_RS / _ALLREDUCE): tests/nvls_worker.py
    if not _nvls_supported():
        pytest.skip("no multicast support on this box")
    _run(NGPU, 29539, worker="nvls_worker.py", ok=f"NVLS_OK world={NGPU}")
