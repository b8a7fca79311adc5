"""World-8 functional check on fewer GPUs (two or more ranks per GPU), launched by
tests/test_multigpu.py through torchrun.  The driver's scaling run uses 8 GPUs,
which a development box may not have: this worker runs the world = 8 code paths
(shard layout, 8 flag slots, 8-way exact reduce, owner interleaving) with rank r on
GPU r % ngpu.  Ranks that share a GPU are separate processes, so the GPU
time-slices between them: correctness only, no timing.  Bootstrap and the replica
checks use gloo (NCCL refuses two ranks on one device); CUDA IPC works between
processes on the same device.

Checks, through the C ABI: R of lmsgd_exchange bit-exact vs the oracle's 8-worker
exchange; the state after each step within the one-step tolerance (oracle resynced);
replicas bit-identical; a non-finite gradient on one rank skips the step everywhere;
the BN statistics average bit-exact.  Prints "OVERSUB_OK world=8" on rank 0.
"""
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import paper_1711_04325_b200 as L  # noqa: E402
import synth  # noqa: E402
from mgpu_worker import check_state  # noqa: E402
from oracle import bn, exchange, schedule  # noqa: E402

S = 1024.0
C1 = schedule.Cluster(n_workers=2, b_local=32, n_train=64)
C1_C = L.make_cluster(2, 32, 64)


def identical_everywhere(x: torch.Tensor):
    h = x.cpu().contiguous().view(torch.int32)
    out = [torch.empty_like(h) for _ in range(dist.get_world_size())]
    dist.all_gather(out, h)
    assert all(torch.equal(o, out[0]) for o in out), "replica divergence"


def main():
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    ngpu = torch.cuda.device_count()
    local = rank % ngpu
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    dist.init_process_group("gloo")
    D = lambda x: torch.from_numpy(np.ascontiguousarray(x)).to(dev)  # noqa: E731
    H = lambda x: x.cpu().numpy()  # noqa: E731

    for n in (64 * world + 3, 100_003):
        ctx = L.lmsgd_init(world, rank, local, n, S)
        L.connect_process_group(ctx)
        a = synth.grad_scale(n)
        th0 = synth.theta0(n, None)
        th, d, m = D(th0), D(np.zeros(n, np.float32)), D(np.zeros(n, np.float32))
        _, n_pad = L.lmsgd_layout(world, n)
        rbuf = torch.empty(n_pad, dtype=torch.int16, device=dev)
        for t in (1, 2, 12):
            g = synth.grads(world, t, n, a)
            g[:, 3] = 9000.0 / S                      # 8 x 9000 > 65504: the sum saturates
            ex = exchange.exchange(list(g), S)
            L.lmsgd_exchange(ctx, D(g[rank]), rbuf)
            code, st = L.lmsgd_query_status(ctx)
            R = H(rbuf).view(np.uint16)
            assert code == 0 and np.array_equal(R[:n], ex.R) and not R[n:].any(), (n, t, code)
            assert st.sum_saturations == ex.sum_saturations >= 1
            prev = H(th), H(d), H(m)
            L.lmsgd_step(ctx, th, D(g[rank]), d, m, L.lmsgd_schedule_at(None, C1_C, t))
            code, st = L.lmsgd_query_status(ctx)
            assert code == 0 and st.skipped == 0, (n, t, code)
            check_state(H(th), H(d), H(m), *prev, ex.ghat, schedule.coeffs_at(t, schedule.Hyper(), C1))
            for x in (th, d, m):
                identical_everywhere(x)
        # non-finite on the last rank: every rank skips, same first index
        g = synth.grads(world, 13, n, a)
        g[world - 1, n // 2] = np.inf
        before = H(th)
        L.lmsgd_step(ctx, th, D(g[rank]), d, m, L.lmsgd_schedule_at(None, C1_C, 13))
        code, st = L.lmsgd_query_status(ctx)
        assert code == L.LMSGD_ERR_NONFINITE and st.first_nonfinite == n // 2, (code, st.first_nonfinite)
        assert np.array_equal(H(th), before)
        # BN statistics average (53 layers of ResNet-50)
        C = sum(synth.resnet_bn_channels(50))
        mean_all, var_all = synth.bn_stats(world, C, seed=5)
        mean, var = D(mean_all[rank]), D(var_all[rank])
        L.lmsgd_bn_stats_allreduce(ctx, mean, var)
        torch.cuda.synchronize()
        om, ov = bn.sync_statistics(mean_all, var_all)
        assert np.array_equal(H(mean), om) and np.array_equal(H(var), ov), "BN average not bit-exact"
        dist.barrier()
        L.lmsgd_finalize(ctx)

    dist.barrier()
    if rank == 0:
        print(f"OVERSUB_OK world={world}", flush=True)
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
