"""Host logic of the N > 1 path on CPU (world_size 2, gloo): IPC-handle bootstrap
plumbing in the binding, the exchange layout, and bench.py's reference arm under a
multi-rank launch (rank 0 prints one line, other ranks exit 0)."""
import json
import os
import subprocess
import sys

import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

import paper_1711_04325_b200 as L

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    seen = {}
    import paper_1711_04325_b200.lmsgd as mod
    mod.lmsgd_ipc_handle = lambda ctx: bytes([ctx.rank + 1]) * L.LMSGD_IPC_HANDLE_BYTES
    mod.lmsgd_connect = lambda ctx, handles: seen.setdefault("h", handles)
    ctx = L.Context(None, world, rank, 0, 10)
    mod.connect_process_group(ctx)
    q.put((rank, seen["h"]))
    dist.destroy_process_group()


def test_connect_process_group_gathers_handles_in_rank_order():
    world, q = 2, mp.get_context("spawn").SimpleQueue()
    mp.start_processes(_worker, args=(world, 29611, q), nprocs=world, start_method="spawn")
    got = dict(q.get() for _ in range(world))
    want = b"".join(bytes([r + 1]) * L.LMSGD_IPC_HANDLE_BYTES for r in range(world))
    assert got[0] == want and got[1] == want


@pytest.mark.parametrize("world", [1, 2, 3, 4, 8])
@pytest.mark.parametrize("n", [1, 63, 64 * 8 + 1, 25_557_032, 60_192_808])
def test_layout_partitions_the_buffer(world, n):
    shard, n_pad = L.lmsgd_layout(world, n)
    assert shard % 64 == 0 and n_pad == shard * world and n <= n_pad < n + 64 * world
    bounds = [(r * shard, (r + 1) * shard) for r in range(world)]
    assert bounds[0][0] == 0 and bounds[-1][1] == n_pad
    assert all(b[1] == c[0] for b, c in zip(bounds, bounds[1:]))
    assert all((b[0] * 2) % 128 == 0 for b in bounds)      # 128-B aligned fp16 shards


def test_bench_reference_arm_multi_rank():
    env = dict(os.environ, PYTHONPATH=ROOT)
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
           "--master-addr=127.0.0.1", "--master-port=29612", os.path.join(ROOT, "bench.py"),
           "--impl", "reference", "--gpus", "2", "--steps", "3", "--warmup", "1"]
    r = subprocess.run(cmd, env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert d["impl"] == "reference" and d["n_gpus"] == 2 and d["cpu_baseline"]["kind"] == "oracle"
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["value"] > 0
