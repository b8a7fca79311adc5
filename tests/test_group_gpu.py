"""World > 1 parity on ONE GPU through the emulated-group calls (include/lmsgd.h
"emulated groups"): the world's ranks are contexts of this process, connected
in-process, and every kernel of the world > 1 path -- k_xstep1 (pack + push, global
skip decision, owner-computes exact reduce), k_xupdate (update with the all-gather
fused in), k_xgather, k_xfinalize, k_bn_allreduce -- runs ONCE per call with all ranks'
blocks in its grid, so ranks that wait on each other's flags are co-scheduled.  This is
what lets a 1-GPU box check rows a3 (reduce-scatter), a4 (all-gather) and a7 (BN
average) against the oracle; tests/test_multigpu.py runs the same checks one process
per GPU where there are enough GPUs.

Bar: R and ghat bit-exact, status words exact, the state
after each step within 1e-6 scaled of the oracle resynced to the GPU's previous state,
every rank's replica bit-identical, the BN average bit-exact.
"""
import os

import numpy as np
import pytest

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA GPU", allow_module_level=True)

import paper_1711_04325_b200 as L  # noqa: E402
import synth  # noqa: E402
from oracle import binary16, bn, exchange, schedule  # noqa: E402
from test_gpu_parity import check_state  # noqa: E402

pytestmark = pytest.mark.gpu
DEV = torch.device("cuda:0")
S = 1024.0
C1 = schedule.Cluster(n_workers=2, b_local=32, n_train=64)
C1_C = L.make_cluster(2, 32, 64)


def dev(x):
    return torch.from_numpy(np.ascontiguousarray(x)).to(DEV)


def host(x):
    return x.cpu().numpy()


def group(k, n, hyper=None, flags=0, timeout_ms=None):
    old = os.environ.get("LMSGD_TIMEOUT_MS")
    os.environ["LMSGD_TIMEOUT_MS"] = str(timeout_ms or 20_000)
    try:
        ctxs = [L.lmsgd_init(k, r, 0, n, S, hyper, flags) for r in range(k)]
    finally:
        if old is None:
            del os.environ["LMSGD_TIMEOUT_MS"]
        else:
            os.environ["LMSGD_TIMEOUT_MS"] = old
    L.lmsgd_connect_group(ctxs)
    return ctxs


def close(ctxs):
    torch.cuda.synchronize()
    for c in ctxs:
        L.lmsgd_finalize(c)


def statuses(ctxs):
    return [L.lmsgd_query_status(c) for c in ctxs]


def identical(per_rank):
    return all(torch.equal(x, per_rank[0]) for x in per_rank[1:])


@pytest.mark.parametrize("k", [2, 3, 4, 8])
@pytest.mark.parametrize("n", [1, 100, 64 * 8 + 3, 123_457, (1 << 20) + 13])
def test_group_exchange_and_step(k, n):
    """R bit-exact (lmsgd_exchange), then steps across the warm-up: state parity,
    saturation counts, replica bit-identity; the two calls share the epoch counter."""
    ctxs = group(k, n)
    a = synth.grad_scale(n)
    r = np.random.default_rng(n + k)
    th0 = synth.theta0(n, None)
    d0 = (r.standard_normal(n) * 1e-3).astype(np.float32)
    m0 = (r.random(n) * 1e-6).astype(np.float32)
    th = [dev(th0) for _ in range(k)]
    d = [dev(d0) for _ in range(k)]
    m = [dev(m0) for _ in range(k)]
    _, n_pad = L.lmsgd_layout(k, n)
    for t in (1, 2, 11, 12, 15):
        g = synth.grads(k, t, n, a)
        g[:, 0] = 9000.0 / S                     # k >= 8 x 9000 > 65504: the sum saturates
        gd = [dev(g[i]) for i in range(k)]
        ex = exchange.exchange(list(g), S)
        if t in (1, 12):
            Rs = [torch.full((n_pad,), -1, dtype=torch.int16, device=DEV) for _ in range(k)]
            L.lmsgd_exchange_group(ctxs, gd, Rs)
            for (code, st), R in zip(statuses(ctxs), Rs):
                Rh = host(R).view(np.uint16)
                assert code == 0 and st.skipped == 0 and np.array_equal(Rh[:n], ex.R) and not Rh[n:].any()
                assert st.pack_saturations == ex.pack_saturations and st.sum_saturations == ex.sum_saturations
        prev = host(th[0]), host(d[0]), host(m[0])
        L.lmsgd_step_group(ctxs, th, gd, d, m, L.lmsgd_schedule_at(None, C1_C, t))
        for code, st in statuses(ctxs):
            assert code == 0 and st.skipped == 0 and st.first_nonfinite == -1, (t, code)
            assert st.pack_saturations == ex.pack_saturations and st.sum_saturations == ex.sum_saturations
        check_state(host(th[0]), host(d[0]), host(m[0]), *prev, ex.ghat, schedule.coeffs_at(t, schedule.Hyper(), C1))
        assert identical(th) and identical(d) and identical(m), t
    close(ctxs)


@pytest.mark.parametrize("k", [2, 4, 8])
def test_group_ghat_bit_exact_and_global_skip(k):
    n = 200_003
    h = L.lmsgd_hyper_default()
    h.mu1 = 0.0                     # (a_SGD, a_RMS) = (1, 0), mu1 = 0: Delta = -ghat exactly
    ctxs = group(k, n, h)
    z = lambda: [dev(np.zeros(n, np.float32)) for _ in range(k)]  # noqa: E731
    th, d, m = z(), z(), z()
    g = synth.grads(k, 7, n)
    g[:, 0] = 60000.0 / S           # the sum saturates at wire-2
    g[0, 1] = 70000.0 / S           # rank 0 saturates at pack
    L.lmsgd_step_group(ctxs, th, [dev(x) for x in g], d, m, L.make_coeffs(1.0, 1.0, 0.0))
    ex = exchange.exchange(list(g), S)
    for (code, st), di in zip(statuses(ctxs), d):
        assert code == 0 and np.array_equal(-host(di), ex.ghat)
        assert st.pack_saturations == ex.pack_saturations >= 1 and st.sum_saturations == ex.sum_saturations >= 1
    # non-finite on two ranks: every rank skips, first index = the global minimum
    before = [host(x) for x in th + d + m]
    g = synth.grads(k, 8, n)
    g[k - 1, 4321] = np.nan
    g[0, 9999] = np.inf
    L.lmsgd_step_group(ctxs, th, [dev(x) for x in g], d, m, L.make_coeffs(1.0, 1.0, 0.0))
    for code, st in statuses(ctxs):
        assert code == L.LMSGD_ERR_NONFINITE and st.skipped == 1 and st.first_nonfinite == 4321, (code, st.first_nonfinite)
    assert all(np.array_equal(a, host(b)) for a, b in zip(before, th + d + m))
    with pytest.raises(binary16.NonFiniteError) as e:
        exchange.exchange(list(g), S)
    assert e.value.index == 4321
    # the exchange alone reports it too; the next clean step goes through
    _, n_pad = L.lmsgd_layout(k, n)
    Rs = [torch.empty(n_pad, dtype=torch.int16, device=DEV) for _ in range(k)]
    L.lmsgd_exchange_group(ctxs, [dev(x) for x in g], Rs)
    for code, st in statuses(ctxs):
        assert code == L.LMSGD_ERR_NONFINITE and st.first_nonfinite == 4321
    g = synth.grads(k, 9, n)
    L.lmsgd_step_group(ctxs, th, [dev(x) for x in g], d, m, L.make_coeffs(1.0, 1.0, 0.0))
    for (code, st), di in zip(statuses(ctxs), d):
        assert code == 0 and np.array_equal(-host(di), exchange.exchange(list(g), S).ghat)
    close(ctxs)


@pytest.mark.parametrize("k", [2, 3, 8])
def test_group_bn_stats_bit_exact(k):
    ctxs = group(k, 1000)
    for C in (1, 64, 1001, sum(synth.resnet_bn_channels(50))):
        mean_all, var_all = synth.bn_stats(k, C, seed=C)
        mean = [dev(mean_all[i]) for i in range(k)]
        var = [dev(var_all[i]) for i in range(k)]
        L.lmsgd_bn_stats_allreduce_group(ctxs, mean, var)
        torch.cuda.synchronize()
        om, ov = bn.sync_statistics(mean_all, var_all)
        for i in range(k):
            assert np.array_equal(host(mean[i]), om) and np.array_equal(host(var[i]), ov), (k, C, i)
    close(ctxs)


def test_group_timeout_when_a_rank_does_not_step():
    n = 4096
    ctxs = group(2, n, timeout_ms=2000)
    th, d, m = dev(np.zeros(n, np.float32)), dev(np.zeros(n, np.float32)), dev(np.zeros(n, np.float32))
    L.lmsgd_step_group(ctxs[:1], [th], [dev(np.ones(n, np.float32))], [d], [m], L.make_coeffs(1.0, 1.0, 0.0))
    code, st = L.lmsgd_query_status(ctxs[0])
    assert code == L.LMSGD_ERR_TIMEOUT and st.skipped == 1, (code, st.skipped)
    assert not host(th).any()
    close(ctxs)


def test_group_rejects_single_rank_calls_and_bad_groups():
    n = 1000
    ctxs = group(2, n)
    t = dev(np.zeros(n, np.float32))
    with pytest.raises(L.LmsgdError) as e:
        L.lmsgd_step(ctxs[0], t, t.clone(), t.clone(), t.clone(), L.make_coeffs(0.1, 1.0, 0.0))
    assert e.value.status == L.LMSGD_ERR_STATE
    with pytest.raises(L.LmsgdError) as e:
        L.lmsgd_step_group([ctxs[0], ctxs[0]], [t] * 2, [t] * 2, [t] * 2, [t] * 2, L.make_coeffs(0.1, 1.0, 0.0))
    assert e.value.status == L.LMSGD_ERR_INVALID_ARG
    close(ctxs)
    loose = [L.lmsgd_init(2, r, 0, n, S) for r in range(2)]
    with pytest.raises(L.LmsgdError) as e:                 # not connected
        L.lmsgd_step_group(loose, [t] * 2, [t] * 2, [t] * 2, [t] * 2, L.make_coeffs(0.1, 1.0, 0.0))
    assert e.value.status == L.LMSGD_ERR_STATE
    other = L.lmsgd_init(2, 1, 0, n + 1, S)
    with pytest.raises(L.LmsgdError) as e:                 # mismatched n_params
        L.lmsgd_connect_group([loose[0], other])
    assert e.value.status == L.LMSGD_ERR_INVALID_ARG
    close(loose + [other])


def test_group_weight_decay_and_freeze_m():
    k, n = 2, 50_021
    th0 = synth.theta0(n, None)
    ctxs = group(k, n)
    for c in ctxs:
        L.lmsgd_set_weight_decay(c, 1e-4, 30_000)
    th = [dev(th0) for _ in range(k)]
    d = [dev(np.zeros(n, np.float32)) for _ in range(k)]
    m = [dev(np.zeros(n, np.float32)) for _ in range(k)]
    g = synth.grads(k, 2, n)
    L.lmsgd_step_group(ctxs, th, [dev(x) for x in g], d, m, L.lmsgd_schedule_at(None, C1_C, 2))
    assert all(code == 0 for code, _ in statuses(ctxs))
    z = np.zeros(n, np.float32)
    check_state(host(th[0]), host(d[0]), host(m[0]), th0, z, z, exchange.exchange(list(g), S).ghat,
                schedule.coeffs_at(2, schedule.Hyper(), C1), wd=1e-4, n_wd=30_000)
    assert identical(th) and identical(d) and identical(m)
    close(ctxs)
    # FREEZE_M: theta, Delta bit-identical to the full rule; m untouched on SGD steps
    ref, frz = group(k, n), group(k, n, None, L.LMSGD_FLAG_FREEZE_M)
    A = [[dev(th0) for _ in range(k)], [dev(z) for _ in range(k)], [dev(z) for _ in range(k)]]
    B = [[x.clone() for x in col] for col in A]
    for t in (3, 12, 13):
        co = L.lmsgd_schedule_at(None, C1_C, t)
        gt = [dev(x) for x in synth.grads(k, t, n)]
        m_before = [x.clone() for x in B[2]]
        L.lmsgd_step_group(ref, *A[:1], gt, A[1], A[2], co)
        L.lmsgd_step_group(frz, *B[:1], gt, B[1], B[2], co)
        torch.cuda.synchronize()
        for i in range(k):
            assert torch.equal(A[0][i], B[0][i]) and torch.equal(A[1][i], B[1][i]), t
            assert torch.equal(B[2][i], m_before[i]) if co.alpha_rmsprop == 0.0 else torch.equal(A[2][i], B[2][i])
    close(ref + frz)


@pytest.mark.parametrize("k", [2, 4])
def test_group_graph_mode_captured_and_replayed(k):
    n = 77_777
    ctxs = group(k, n)
    for c in ctxs:
        L.lmsgd_schedule_upload(c, None, C1_C, 1, 10)       # steps 1 .. 10
    a = synth.grad_scale(n)
    th0 = synth.theta0(n, None)
    th = [dev(th0) for _ in range(k)]
    d = [dev(np.zeros(n, np.float32)) for _ in range(k)]
    m = [dev(np.zeros(n, np.float32)) for _ in range(k)]
    gbuf = [dev(np.zeros(n, np.float32)) for _ in range(k)]
    side = torch.cuda.Stream()
    graph = None
    for t in range(1, 9):
        g = synth.grads(k, t, n, a)
        for i in range(k):
            gbuf[i].copy_(dev(g[i]))
        prev = host(th[0]), host(d[0]), host(m[0])
        if t <= 3:
            L.lmsgd_step_graph_group(ctxs, th, gbuf, d, m)
        else:
            if graph is None:
                graph = torch.cuda.CUDAGraph()
                torch.cuda.synchronize()
                with torch.cuda.stream(side):
                    with torch.cuda.graph(graph, stream=side):
                        L.lmsgd_step_graph_group(ctxs, th, gbuf, d, m, stream=side)
            graph.replay()
        torch.cuda.synchronize()
        for code, st in statuses(ctxs):
            assert code == 0 and st.skipped == 0, (t, code)
        check_state(host(th[0]), host(d[0]), host(m[0]), *prev, exchange.exchange(list(g), S).ghat,
                    schedule.coeffs_at(t, schedule.Hyper(), C1))
        assert identical(th) and identical(d) and identical(m), t
    close(ctxs)


def test_group_long_run_replicas_and_resync():
    """100 group steps at random schedule points (k = 4) with exchanges and skipped
    steps interleaved: replicas bit-identical after every step, oracle parity every
    10th step."""
    k, n = 4, 100_003
    ctxs = group(k, n)
    a = synth.grad_scale(n)
    th = [dev(synth.theta0(n, None)) for _ in range(k)]
    d = [dev(np.zeros(n, np.float32)) for _ in range(k)]
    m = [dev(np.zeros(n, np.float32)) for _ in range(k)]
    _, n_pad = L.lmsgd_layout(k, n)
    Rs = [torch.empty(n_pad, dtype=torch.int16, device=DEV) for _ in range(k)]
    rng = np.random.default_rng(11)
    for it in range(100):
        t = int(rng.integers(1, 3519))
        g = synth.grads(k, t, n, a)
        if it % 17 == 5:
            g[it % k, it * 7] = np.nan
        gd = [dev(x) for x in g]
        if it % 13 == 3:
            L.lmsgd_exchange_group(ctxs, gd, Rs)
        prev = (host(th[0]), host(d[0]), host(m[0]))
        L.lmsgd_step_group(ctxs, th, gd, d, m, L.lmsgd_schedule_at(None, L.make_cluster(), t))
        code, st = L.lmsgd_query_status(ctxs[k - 1])
        if it % 17 == 5:
            assert code == L.LMSGD_ERR_NONFINITE and st.first_nonfinite == it * 7
            assert np.array_equal(host(th[0]), prev[0])
        else:
            assert code == 0
            if it % 10 == 9:
                check_state(host(th[0]), host(d[0]), host(m[0]), *prev, exchange.exchange(list(g), S).ghat,
                            schedule.coeffs_at(t))
        assert identical(th) and identical(d) and identical(m), it
    close(ctxs)


@pytest.mark.parametrize("k", [2, 4, 8])
def test_group_resnet50_full_size_sampled(k):
    """The 25,557,032-element ResNet-50 buffer (BASELINE configs[2]) at world k, the
    whole path on sampled indices (elementwise, so the oracle on the sample is exact),
    replicas compared in full."""
    n = synth.resnet_n_params(50)
    ctxs = group(k, n)
    th0 = synth.theta0(n, 50)
    g = synth.grads(k, 1, n)
    th = [dev(th0) for _ in range(k)]
    d = [torch.zeros(n, device=DEV) for _ in range(k)]
    m = [torch.zeros(n, device=DEV) for _ in range(k)]
    L.lmsgd_step_group(ctxs, th, [dev(x) for x in g], d, m, L.lmsgd_schedule_at(None, L.make_cluster(), 1))
    for code, _ in statuses(ctxs):
        assert code == 0
    idx = np.unique(np.concatenate([np.arange(2000), np.arange(n - 2000, n),
                                    np.random.default_rng(3).integers(0, n, 100_000)]))
    ex = exchange.exchange([gi[idx] for gi in g], S)
    z = np.zeros(idx.size, np.float32)
    check_state(host(th[0])[idx], host(d[0])[idx], host(m[0])[idx], th0[idx], z, z, ex.ghat, schedule.coeffs_at(1))
    assert identical(th) and identical(d) and identical(m)
    close(ctxs)
