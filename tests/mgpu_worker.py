"""Multi-GPU parity worker, launched by tests/test_multigpu.py through torchrun
(one process per GPU, NCCL process group for bootstrap only).

Oversubscribed mode (world > visible GPUs, e.g. world 2 or 4 on a 1-GPU box): rank r
runs on GPU r % ngpu and the process group is gloo (NCCL refuses two ranks on one
device); the exchange itself is unchanged -- CUDA IPC maps another process's buffer
on the same device as it does a peer's -- so every world > 1 kernel (k_xstep1,
k_xupdate, k_xgather, k_xfinalize, k_bn_allreduce) runs its real cross-rank flag
protocol, the GPU time-slicing between the ranks' contexts.  Correctness only; the
skew stress runs LMSGD_STRESS_STEPS steps (default 10^4 with one GPU per rank, 400
oversubscribed).

Checks on world = k real GPUs over NVLink, through the C ABI:
  * R (fp16 all-reduce sum) and ghat bit-exact vs the oracle's k-worker exchange;
  * state after each step within the one-step tolerance (oracle resynced);
  * replica bit-identity of theta / Delta / m on every rank after every step;
  * a non-finite gradient on one rank skips the step on every rank, same status;
  * saturation counts summed over ranks;
  * BN statistics average bit-exact vs the oracle;
  * lmsgd_exchange (the fp16 all-reduce alone): R bit-exact, interleaved with steps;
  * 10^4 steps under random per-rank device skew: replicas bit-identical and equal to
    the same sequence without skew (the flag / epoch / status-slot protocol);
  * the full 25.6M ResNet-50 buffer (sampled check) in bench.py's launch configuration.
Exit code 0 and "MGPU_OK" on rank 0 when everything passes.
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
from oracle import binary16, bn, exchange, run, schedule  # noqa: E402

S = 1024.0
C1 = schedule.Cluster(n_workers=2, b_local=32, n_train=64)
C1_C = L.make_cluster(2, 32, 64)


def check_state(th_g, d_g, m_g, th0, d0, m0, ghat, c, tol=1e-6, wd=0.0, n_wd=None):
    hyper = schedule.Hyper()
    th_o, d_o, m_o = run.resync_step(th0, d0, m0, ghat, c, hyper, wd, n_wd)
    # |g| + |lambda theta|: the fp32 g + lambda theta is exact to that scale, not to
    # the (possibly cancelled) sum (R12)
    gh = np.abs(np.asarray(ghat, dtype=np.float64))
    if wd:
        k = gh.size if n_wd is None else n_wd
        gh[:k] += wd * np.abs(np.asarray(th0, np.float64)[:k])
    coef = c.alpha_sgd + c.alpha_rmsprop / (np.sqrt(m_o) + hyper.eps)
    scale_d = hyper.mu1 * np.abs(np.asarray(d0, np.float64)) + coef * gh
    # wd = 0: m_t is a sum of non-negative fp32 terms, so m_t itself bounds its rounding;
    # with wd the fp32 g + lambda theta is exact only to (|g| + lambda|theta|) (R12)
    scale_m = m_o + (1.0 - hyper.mu2) * gh * gh if wd else m_o
    e = (run.scaled_error(m_g, m_o, scale_m), run.scaled_error(d_g, d_o, scale_d),
         run.scaled_error(th_g, th_o, np.abs(np.asarray(th0, np.float64)) + c.eta * scale_d))
    assert max(e) <= tol, e


# collectives of the checks run on the device with NCCL, on host copies with gloo
COLL_ON_HOST = False


def _coll(t):
    return t.cpu() if COLL_ON_HOST else t


def replicas_identical(*tensors):
    for t in tensors:
        t = _coll(t)
        ref = t.clone()
        dist.broadcast(ref, 0)
        assert torch.equal(ref, t), "replica divergence"


def all_gather_host(t):
    """Every rank's copy of t as numpy arrays, in rank order."""
    t = _coll(t.contiguous())
    out = [torch.empty_like(t) for _ in range(dist.get_world_size())]
    dist.all_gather(out, t)
    return [o.cpu().numpy() for o in out]


def timeout_case(rank, world, local, D, H):
    """A rank that does not step: the others time out instead of hanging."""
    n = 4096
    ctx = L.lmsgd_init(world, rank, local, n, S)
    L.connect_process_group(ctx)
    th, d, m = D(np.zeros(n, np.float32)), D(np.zeros(n, np.float32)), D(np.zeros(n, np.float32))
    if rank == 0:
        L.lmsgd_step(ctx, th, D(np.ones(n, np.float32)), d, m, L.make_coeffs(1.0, 1.0, 0.0))
        code, st = L.lmsgd_query_status(ctx)
        assert code == L.LMSGD_ERR_TIMEOUT and st.skipped == 1, (code, st.skipped)
        assert not H(th).any()
    dist.barrier()
    L.lmsgd_finalize(ctx)


def main():
    global COLL_ON_HOST
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    ngpu = torch.cuda.device_count()
    oversub = world > ngpu
    local = int(os.environ["LOCAL_RANK"]) % ngpu
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if oversub:
        COLL_ON_HOST = True
        dist.init_process_group("gloo")
    else:
        dist.init_process_group("nccl", device_id=dev)
    stress_steps = int(os.environ.get("LMSGD_STRESS_STEPS", 400 if oversub else 10_000))
    D = lambda x: torch.from_numpy(np.ascontiguousarray(x)).to(dev)  # noqa: E731
    H = lambda x: x.cpu().numpy()  # noqa: E731

    if os.environ.get("LMSGD_TEST_TIMEOUT") == "1":   # only the timeout case
        timeout_case(rank, world, local, D, H)
        dist.barrier()
        if rank == 0:
            print(f"MGPU_OK world={world}", flush=True)
        dist.destroy_process_group()
        return

    # ---- exchange + update parity on ragged sizes, across the warm-up
    for n in (1, 100, 64 * world + 3, 123_457, (1 << 20) + 13):
        ctx = L.lmsgd_init(world, rank, local, n, S)
        L.connect_process_group(ctx)
        a = synth.grad_scale(n)
        r = np.random.default_rng(n)
        th0 = synth.theta0(n, None)
        d0 = (r.standard_normal(n) * 1e-3).astype(np.float32)
        m0 = (r.random(n) * 1e-6).astype(np.float32)
        th, d, m = D(th0), D(d0), D(m0)
        for t in (1, 2, 11, 12, 15):
            g = synth.grads(world, t, n, a)
            prev = H(th), H(d), H(m)
            L.lmsgd_step(ctx, th, D(g[rank]), d, m, L.lmsgd_schedule_at(None, C1_C, t))
            code, st = L.lmsgd_query_status(ctx)
            assert code == 0 and st.skipped == 0 and st.first_nonfinite == -1, (code, st.skipped)
            ex = exchange.exchange(list(g), S)
            assert st.pack_saturations == ex.pack_saturations and st.sum_saturations == ex.sum_saturations
            check_state(H(th), H(d), H(m), *prev, ex.ghat, schedule.coeffs_at(t, schedule.Hyper(), C1))
            replicas_identical(th, d, m)
        L.lmsgd_finalize(ctx)

    # ---- weight decay on a prefix (R12), exchange + update across the ranks
    n = 50_021
    ctx = L.lmsgd_init(world, rank, local, n, S)
    L.connect_process_group(ctx)
    L.lmsgd_set_weight_decay(ctx, 1e-4, 30_000)
    th0 = synth.theta0(n, None)
    th, d, m = D(th0), D(np.zeros(n, np.float32)), D(np.zeros(n, np.float32))
    g = synth.grads(world, 2, n)
    L.lmsgd_step(ctx, th, D(g[rank]), d, m, L.lmsgd_schedule_at(None, C1_C, 2))
    code, st = L.lmsgd_query_status(ctx)
    assert code == 0
    z = np.zeros(n, np.float32)
    check_state(H(th), H(d), H(m), th0, z, z, exchange.exchange(list(g), S).ghat,
                schedule.coeffs_at(2, schedule.Hyper(), C1), wd=1e-4, n_wd=30_000)
    replicas_identical(th, d, m)
    L.lmsgd_finalize(ctx)

    # ---- LMSGD_FLAG_FREEZE_M: theta, Delta bit-identical to the full rule; m untouched on SGD steps
    ref = L.lmsgd_init(world, rank, local, n, S)
    L.connect_process_group(ref)
    frz = L.lmsgd_init(world, rank, local, n, S, None, L.LMSGD_FLAG_FREEZE_M)
    L.connect_process_group(frz)
    a = [D(th0), D(np.zeros(n, np.float32)), D(np.zeros(n, np.float32))]
    b = [x.clone() for x in a]
    for t in (3, 12, 13):
        co = L.lmsgd_schedule_at(None, C1_C, t)
        gt = D(synth.grads(world, t, n)[rank])
        m_before = b[2].clone()
        L.lmsgd_step(ref, a[0], gt, a[1], a[2], co)
        L.lmsgd_step(frz, b[0], gt, b[1], b[2], co)
        torch.cuda.synchronize()
        assert torch.equal(a[0], b[0]) and torch.equal(a[1], b[1]), t
        assert torch.equal(b[2], m_before) if co.alpha_rmsprop == 0.0 else torch.equal(a[2], b[2]), t
    replicas_identical(*b)
    L.lmsgd_query_status(ref)
    L.lmsgd_query_status(frz)
    dist.barrier()
    L.lmsgd_finalize(ref)
    L.lmsgd_finalize(frz)

    # ---- the torch-style front end (LMSGD) on a small net, one minibatch per rank
    torch.manual_seed(0)
    net = torch.nn.Sequential(torch.nn.Conv2d(3, 8, 3), torch.nn.BatchNorm2d(8), torch.nn.ReLU(),
                              torch.nn.Flatten(), torch.nn.Linear(8 * 6 * 6, 10)).to(dev)
    opt = L.LMSGD(net.parameters(), cluster=C1_C, loss_scale=S, weight_decay=1e-4)
    for t in (1, 2, 3):
        gen = torch.Generator(device="cpu").manual_seed(1000 * t + rank)
        x, y = torch.randn(32, 3, 8, 8, generator=gen).to(dev), torch.randint(0, 10, (32,), generator=gen).to(dev)
        opt.zero_grad()
        torch.nn.functional.cross_entropy(net(x), y).backward()
        allg = all_gather_host(opt.flat_g)
        prev = H(opt.flat_p), H(opt.delta), H(opt.m)
        opt.step()
        assert opt.status()[0] == 0
        check_state(H(opt.flat_p), H(opt.delta), H(opt.m), *prev,
                    exchange.exchange(allg, S).ghat, schedule.coeffs_at(t, schedule.Hyper(), C1),
                    wd=1e-4, n_wd=opt.n_decay)
        replicas_identical(opt.flat_p, opt.delta, opt.m)
    dist.barrier()
    opt.close()

    # ---- row f1: the bucketed exchange overlapped with backward (BucketedLMSGD) gives
    #      bit-identically LMSGD's state, and the oracle's one-step state, on every rank
    def deep(seed):
        torch.manual_seed(seed)
        return torch.nn.Sequential(torch.nn.Conv2d(3, 16, 3), torch.nn.ReLU(), torch.nn.Conv2d(16, 32, 3),
                                   torch.nn.ReLU(), torch.nn.Flatten(), torch.nn.Linear(32 * 4 * 4, 10)).to(dev)
    torch.backends.cudnn.deterministic, torch.backends.cudnn.benchmark = True, False   # identical grads
    na, nb = deep(3), deep(3)
    oa = L.LMSGD(na.parameters(), cluster=C1_C, loss_scale=S)
    ob = L.BucketedLMSGD(nb.parameters(), cluster=C1_C, loss_scale=S, bucket_elems=2048, exchange_blocks=32)
    assert len(ob.buckets) > 2
    for t in (1, 2, 3):
        gen = torch.Generator(device="cpu").manual_seed(500 * t + rank)
        x, y = torch.randn(16, 3, 8, 8, generator=gen).to(dev), torch.randint(0, 10, (16,), generator=gen).to(dev)
        for net_, opt_ in ((na, oa), (nb, ob)):
            opt_.zero_grad()
            torch.nn.functional.cross_entropy(net_(x), y).backward()
        allg = all_gather_host(ob.flat_g)
        prev = H(ob.flat_p), H(ob.delta), H(ob.m)
        oa.step()
        ob.step()
        assert ob.status()[0] == 0 and oa.status()[0] == 0
        assert torch.equal(oa.flat_p, ob.flat_p) and torch.equal(oa.delta, ob.delta) and torch.equal(oa.m, ob.m), t
        check_state(H(ob.flat_p), H(ob.delta), H(ob.m), *prev, exchange.exchange(allg, S).ghat,
                    schedule.coeffs_at(t, schedule.Hyper(), C1))
        replicas_identical(ob.flat_p, ob.delta, ob.m)
    dist.barrier()
    oa.close()
    ob.close()

    # ---- ghat bit-exact (mu1 = 0, (a_SGD, a_RMS) = (1, 0) => Delta = -ghat), with saturation
    n = 200_003
    hyp = L.lmsgd_hyper_default()
    hyp.mu1 = 0.0
    ctx = L.lmsgd_init(world, rank, local, n, S, hyp)
    L.connect_process_group(ctx)
    g = synth.grads(world, 7, n)
    g[:, 0] = 60000.0 / S          # every rank near the top: the sum saturates at wire-2
    g[0, 1] = 70000.0 / S          # rank 0 saturates at pack
    z = lambda: D(np.zeros(n, np.float32))  # noqa: E731
    th, d, m = z(), z(), z()
    L.lmsgd_step(ctx, th, D(g[rank]), d, m, L.make_coeffs(1.0, 1.0, 0.0))
    code, st = L.lmsgd_query_status(ctx)
    ex = exchange.exchange(list(g), S)
    assert np.array_equal(-H(d), ex.ghat), "ghat not bit-exact"
    assert st.pack_saturations == ex.pack_saturations >= 1 and st.sum_saturations == ex.sum_saturations >= 1

    # ---- non-finite on one rank: every rank skips, same first index (the global minimum)
    th0, d0, m0 = H(th), H(d), H(m)
    g = synth.grads(world, 8, n)
    g[world - 1, 4321] = np.nan
    g[0, 9999] = np.inf
    L.lmsgd_step(ctx, th, D(g[rank]), d, m, L.make_coeffs(1.0, 1.0, 0.0))
    code, st = L.lmsgd_query_status(ctx)
    assert code == L.LMSGD_ERR_NONFINITE and st.skipped == 1 and st.first_nonfinite == 4321, (code, st.first_nonfinite)
    assert np.array_equal(H(th), th0) and np.array_equal(H(d), d0) and np.array_equal(H(m), m0)
    try:
        exchange.exchange(list(g), S)
        raise AssertionError("oracle accepted a non-finite gradient")
    except binary16.NonFiniteError as e:
        assert e.index == 4321
    # and the next clean step goes through
    g = synth.grads(world, 9, n)
    L.lmsgd_step(ctx, th, D(g[rank]), d, m, L.make_coeffs(1.0, 1.0, 0.0))
    code, st = L.lmsgd_query_status(ctx)
    assert code == 0 and np.array_equal(-H(d), exchange.exchange(list(g), S).ghat)

    # ---- the fp16 all-reduce alone (lmsgd_exchange, rows a2-a4): R bit-exact on every
    #      rank, interleaved with steps on the same context (one epoch counter)
    _, n_pad = L.lmsgd_layout(world, n)
    Rg = torch.full((n_pad,), -1, dtype=torch.int16, device=dev)
    for t in (10, 11):
        g = synth.grads(world, t, n)
        g[:, 5] = 60000.0 / S                  # the sum saturates
        L.lmsgd_exchange(ctx, D(g[rank]), Rg)
        code, st = L.lmsgd_query_status(ctx)
        ex = exchange.exchange(list(g), S)
        R = H(Rg).view(np.uint16)
        assert code == 0 and st.skipped == 0 and np.array_equal(R[:n], ex.R), "exchange R not bit-exact"
        assert not R[n:].any(), "exchange padding not zero"
        assert st.pack_saturations == ex.pack_saturations and st.sum_saturations == ex.sum_saturations >= 1
        replicas_identical(Rg.view(torch.int32))   # NCCL has no int16
        L.lmsgd_step(ctx, th, D(g[rank]), d, m, L.make_coeffs(1.0, 1.0, 0.0))   # a step in between
        code, st = L.lmsgd_query_status(ctx)
        assert code == 0 and np.array_equal(-H(d), ex.ghat)
    g = synth.grads(world, 12, n)
    g[world - 1, 777] = np.inf
    L.lmsgd_exchange(ctx, D(g[rank]), Rg)
    code, st = L.lmsgd_query_status(ctx)
    assert code == L.LMSGD_ERR_NONFINITE and st.skipped == 1 and st.first_nonfinite == 777, (code, st.first_nonfinite)
    for nx in (1, 100, 64 * world + 3, 123_457):
        cx = L.lmsgd_init(world, rank, local, nx, S)
        L.connect_process_group(cx)
        _, npx = L.lmsgd_layout(world, nx)
        Rx = torch.full((npx,), -1, dtype=torch.int16, device=dev)
        g = synth.grads(world, 3, nx)
        L.lmsgd_exchange(cx, D(g[rank]), Rx)
        code, st = L.lmsgd_query_status(cx)
        R = H(Rx).view(np.uint16)
        assert code == 0 and np.array_equal(R[:nx], exchange.exchange(list(g), S).R) and not R[nx:].any(), nx
        dist.barrier()
        L.lmsgd_finalize(cx)

    # ---- BN last-minibatch statistics average
    for C in (1, 64, sum(synth.resnet_bn_channels(50))):
        mean_all, var_all = synth.bn_stats(world, C, seed=C)
        mean, var = D(mean_all[rank]), D(var_all[rank])
        L.lmsgd_bn_stats_allreduce(ctx, mean, var)
        torch.cuda.synchronize()
        om, ov = bn.sync_statistics(mean_all, var_all)
        assert np.array_equal(H(mean), om) and np.array_equal(H(var), ov), "BN average not bit-exact"
    L.lmsgd_finalize(ctx)

    # ---- BN without moving averages end to end: momentum = 1 BN
    #      layers, a different minibatch per rank, then the average before validation
    from paper_1711_04325_b200 import bn_sync
    torch.manual_seed(5)   # identical weights on every rank
    net = torch.nn.Sequential(torch.nn.Conv2d(3, 16, 3), torch.nn.BatchNorm2d(16), torch.nn.ReLU(),
                              torch.nn.Conv2d(16, 32, 3), torch.nn.BatchNorm2d(32), torch.nn.ReLU(),
                              torch.nn.Flatten(), torch.nn.LazyLinear(10), torch.nn.BatchNorm1d(10)).to(dev)
    bn_sync.last_minibatch_bn(net)
    ctx = L.lmsgd_init(world, rank, local, 1000, S)
    L.connect_process_group(ctx)
    net.train()
    net(torch.randn(32, 3, 12, 12, device=dev))          # materialise the lazy layer
    sync = bn_sync.BNStatsSync(net, ctx)
    gen = torch.Generator(device=dev)
    gen.manual_seed(100 + rank)
    xb = torch.randn(32, 3, 12, 12, device=dev, generator=gen) * (1 + rank)
    net(xb)                                              # last training minibatch of this rank
    layers = bn_sync.bn_layers(net)
    mine_mean = torch.cat([m.running_mean for m in layers]).clone()
    mine_var = torch.cat([m.running_var for m in layers]).clone()
    # momentum = 1: running statistics are exactly this minibatch's (first BN layer)
    h = net[0](xb)
    assert torch.allclose(layers[0].running_mean, h.mean(dim=(0, 2, 3)), rtol=1e-5, atol=1e-6)
    all_mean = all_gather_host(mine_mean)
    all_var = all_gather_host(mine_var)
    sync.sync()
    torch.cuda.synchronize()
    om, ov = bn.sync_statistics(np.stack(all_mean), np.stack(all_var))
    assert np.array_equal(H(sync.mean), om) and np.array_equal(H(sync.var), ov)
    assert np.array_equal(H(layers[1].running_var), ov[16:48])      # the modules see the averages
    net.eval()
    net(torch.randn(4, 3, 12, 12, device=dev))           # validation uses the synced statistics
    replicas_identical(sync.mean, sync.var)
    L.lmsgd_finalize(ctx)

    # ---- CUDA-graph entry point: device coefficient table + device step counter,
    #      eagerly, then captured once and replayed
    n = 77_777
    ctx = L.lmsgd_init(world, rank, local, n, S)
    L.connect_process_group(ctx)
    a = synth.grad_scale(n)
    th0 = synth.theta0(n, None)
    th, d, m = D(th0), D(np.zeros(n, np.float32)), D(np.zeros(n, np.float32))
    L.lmsgd_schedule_upload(ctx, None, C1_C, 1, 10)          # steps 1 .. 10
    gbuf = D(np.zeros(n, np.float32))
    side = torch.cuda.Stream()
    graph = None
    for t in range(1, 8):
        g = synth.grads(world, t, n, a)
        prev = H(th), H(d), H(m)
        gbuf.copy_(D(g[rank]))
        if t <= 3:
            L.lmsgd_step_graph(ctx, th, gbuf, d, m)
        else:
            if graph is None:
                graph = torch.cuda.CUDAGraph()
                torch.cuda.synchronize()
                with torch.cuda.stream(side):
                    with torch.cuda.graph(graph, stream=side):
                        L.lmsgd_step_graph(ctx, th, gbuf, d, m, stream=side)
            graph.replay()
        torch.cuda.synchronize()
        code, st = L.lmsgd_query_status(ctx)
        assert code == 0 and st.skipped == 0, (t, code)
        check_state(H(th), H(d), H(m), *prev, exchange.exchange(list(g), S).ghat,
                    schedule.coeffs_at(t, schedule.Hyper(), C1))
        replicas_identical(th, d, m)
    L.lmsgd_finalize(ctx)

    # ---- longer run: random schedule steps, replica bit-identity every step,
    #      resync parity every 10th step
    n = 333_331
    ctx = L.lmsgd_init(world, rank, local, n, S)
    L.connect_process_group(ctx)
    a = synth.grad_scale(n)
    th0 = synth.theta0(n, None)
    th, d, m = D(th0), D(np.zeros(n, np.float32)), D(np.zeros(n, np.float32))
    rng = np.random.default_rng(11)
    for it in range(40):
        t = int(rng.integers(1, 3519))
        g = synth.grads(world, t, n, a)
        prev = (H(th), H(d), H(m)) if it % 10 == 9 else None
        L.lmsgd_step(ctx, th, D(g[rank]), d, m, L.lmsgd_schedule_at(None, L.make_cluster(), t))
        if prev is not None:
            code, st = L.lmsgd_query_status(ctx)
            assert code == 0
            check_state(H(th), H(d), H(m), *prev, exchange.exchange(list(g), S).ghat, schedule.coeffs_at(t))
        replicas_identical(th, d, m)
    L.lmsgd_finalize(ctx)

    # ---- cross-GPU flag protocol under skew: 10^4 steps
    #      (stress_steps),
    #      random per-rank device delays before a step, exchanges and non-finite steps
    #      interleaved; the final state must be bit-identical on every rank AND to the same
    #      sequence run without delays
    n = 100_003
    gen = torch.Generator(device=dev)
    gen.manual_seed(77 + rank)
    pool = [torch.randn(n, generator=gen, device=dev) * 1e-3 for _ in range(8)]
    bad = pool[0].clone()
    bad[12_345] = float("nan")
    rbuf = torch.empty(L.lmsgd_layout(world, n)[1], dtype=torch.int16, device=dev)
    finals = []
    for delayed in (False, True):
        ctx = L.lmsgd_init(world, rank, local, n, S)
        L.connect_process_group(ctx)
        th = D(synth.theta0(n, None))
        d, m = torch.zeros(n, device=dev), torch.zeros(n, device=dev)
        rng = np.random.default_rng(1234 + (rank if delayed else 0))
        for it in range(stress_steps):
            if delayed and rng.random() < 0.3:
                torch.cuda._sleep(int(rng.integers(1, 200_000)))   # up to ~100 us of device skew
            if it % 97 == 13:
                L.lmsgd_exchange(ctx, pool[it % 8], rbuf)
            elif it % 501 == 7:
                L.lmsgd_step(ctx, th, bad if rank == it % world else pool[it % 8], d, m,
                             L.lmsgd_schedule_at(None, C1_C, 1 + it % 30))
                code, st = L.lmsgd_query_status(ctx)
                assert code == L.LMSGD_ERR_NONFINITE and st.first_nonfinite == 12_345, (it, code)
            else:
                L.lmsgd_step(ctx, th, pool[it % 8], d, m, L.lmsgd_schedule_at(None, C1_C, 1 + it % 30))
        code, st = L.lmsgd_query_status(ctx)
        assert code == 0 and st.skipped == 0, code
        finals.append((th.clone(), d.clone(), m.clone()))
        replicas_identical(th, d, m)
        dist.barrier()
        L.lmsgd_finalize(ctx)
    for a_, b_ in zip(*finals):
        assert torch.equal(a_, b_), "state depends on cross-GPU timing"

    # ---- full ResNet-50 buffer, sampled check
    n = synth.resnet_n_params(50)
    ctx = L.lmsgd_init(world, rank, local, n, S)
    L.connect_process_group(ctx)
    th0 = synth.theta0(n, 50)
    g = synth.grads(world, 1, n)
    th, d, m = D(th0), D(np.zeros(n, np.float32)), D(np.zeros(n, np.float32))
    cfull = L.lmsgd_schedule_at(None, L.make_cluster(), 1)
    L.lmsgd_step(ctx, th, D(g[rank]), d, m, cfull)
    code, st = L.lmsgd_query_status(ctx)
    assert code == 0
    idx = np.unique(np.concatenate([np.arange(2000), np.arange(n - 2000, n),
                                    np.random.default_rng(3).integers(0, n, 100_000)]))
    ex = exchange.exchange([gi[idx] for gi in g], S)
    z = np.zeros(idx.size, np.float32)
    check_state(H(th)[idx], H(d)[idx], H(m)[idx], th0[idx], z, z, ex.ghat, schedule.coeffs_at(1))
    replicas_identical(th, d, m)
    L.lmsgd_finalize(ctx)

    dist.barrier()
    if rank == 0:
        print(f"MGPU_OK world={world}", flush=True)
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
