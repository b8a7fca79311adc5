"""GPU parity of the CUDA path (through the C ABI) against the CPU oracle.

Bar (BASELINE.json north_star):
  * fp16 wire payloads R and the averaged gradient ghat: bit-exact (the sum is exact);
  * schedule: bit-exact (tests/test_lib_host.py);
  * fp32 state after one step, oracle resynced to the GPU's previous state:
    |x_gpu - x_oracle| <= 1e-6 * scale_x with scale_m = m_t (+ (1-mu2)(|ghat| + lambda|theta|)^2 with weight decay),
    scale_Delta = mu1 |Delta_{t-1}| + |c ghat|, scale_theta = |theta_{t-1}| + eta scale_Delta;
  * status words (first non-finite index, saturation counts): exact.
"""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA GPU", allow_module_level=True)

import paper_1711_04325_b200 as L  # noqa: E402
import synth  # noqa: E402
from oracle import binary16, exchange, run, schedule  # noqa: E402

pytestmark = pytest.mark.gpu
DEV = torch.device("cuda:0")
TOL = 1e-6
C1 = schedule.Cluster(n_workers=2, b_local=32, n_train=64)
C1_C = L.make_cluster(2, 32, 64)
K32 = schedule.Cluster()
K32_C = L.make_cluster()


def dev(x):
    return torch.from_numpy(np.ascontiguousarray(x)).to(DEV)


def host(x):
    return x.cpu().numpy()


def check_state(th_g, d_g, m_g, th0, d0, m0, ghat, c, hyper=schedule.Hyper(), tol=TOL, wd=0.0, n_wd=None):
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
    e = {
        "m": run.scaled_error(m_g, m_o, scale_m),
        "delta": run.scaled_error(d_g, d_o, scale_d),
        # Delta's own rounding (relative to scale_d) propagates through eta: DESIGN.md "Tolerances"
        "theta": run.scaled_error(th_g, th_o, np.abs(np.asarray(th0, np.float64)) + c.eta * scale_d),
    }
    assert max(e.values()) <= tol, e
    return e


def init_state(n, seed=0):
    r = np.random.default_rng(seed)
    th = synth.theta0(n, None)
    d = (r.standard_normal(n) * 1e-3).astype(np.float32)
    m = (r.random(n) * 1e-6).astype(np.float32)
    return th, d, m


# ------------------------------------------------------------------ k = 1 context path

@pytest.mark.parametrize("n", [1, 7, 8, 9, 63, 64, 65, 1000, 10_007, (1 << 20) + 13])
@pytest.mark.parametrize("flags", [0, L.LMSGD_FLAG_NO_SKIP])
def test_k1_step_ragged_sizes(n, flags):
    s = 1024.0
    th0, d0, m0 = init_state(n)
    ctx = L.lmsgd_init(1, 0, 0, n, s, None, flags)
    th, d, m = dev(th0), dev(d0), dev(m0)
    a = synth.grad_scale(n)
    for t in (1, 12, 15):   # exp branch (RMS on), linear branch, SGD (RMS off)
        coeffs = L.lmsgd_schedule_at(None, C1_C, t)
        c = schedule.coeffs_at(t, schedule.Hyper(), C1)
        g = synth.grads(1, t, n, a)
        prev = host(th), host(d), host(m)
        L.lmsgd_step(ctx, th, dev(g[0]), d, m, coeffs)
        code, st = L.lmsgd_query_status(ctx)
        assert code == 0 and st.skipped == 0 and st.first_nonfinite == -1
        ex = exchange.exchange(list(g), s)
        assert st.pack_saturations == ex.pack_saturations and st.sum_saturations in (0, ex.sum_saturations)
        check_state(host(th), host(d), host(m), *prev, ex.ghat, c)
    L.lmsgd_finalize(ctx)


@pytest.mark.parametrize("flags", [0, L.LMSGD_FLAG_NO_SKIP])
@pytest.mark.parametrize("s", [1.0, 1024.0])
def test_k1_ghat_bit_exact(flags, s):
    """With mu1 = 0 and (a_SGD, a_RMS) = (1, 0): Delta_t = -ghat exactly in fp32,
    which exposes the GPU's ghat for a bit-exact comparison with the oracle."""
    n = 200_003
    h = L.lmsgd_hyper_default()
    h.mu1 = 0.0
    ctx = L.lmsgd_init(1, 0, 0, n, s, h, flags)
    g = synth.grads(1, 5, n)
    # include subnormal / saturating / tie values
    g[0, :6] = np.array([3e-8, 6e-8, 65504.0 / s, 65520.0 / s, 1e6, -2.0 ** -25 * 3 / s], dtype=np.float32)
    th, d, m = dev(np.zeros(n, np.float32)), dev(np.zeros(n, np.float32)), dev(np.zeros(n, np.float32))
    L.lmsgd_step(ctx, th, dev(g[0]), d, m, L.make_coeffs(1.0, 1.0, 0.0))
    code, st = L.lmsgd_query_status(ctx)
    ex = exchange.exchange(list(g), s)
    assert np.array_equal(-host(d), ex.ghat)
    assert st.pack_saturations == ex.pack_saturations >= 2
    L.lmsgd_finalize(ctx)


def test_k1_nonfinite_skips_and_reports_first_index():
    n = 100_000
    ctx = L.lmsgd_init(1, 0, 0, n, 1024.0)
    th0, d0, m0 = init_state(n)
    th, d, m = dev(th0), dev(d0), dev(m0)
    g = synth.grads(1, 1, n)[0]
    g[77_777] = np.inf
    g[99_999] = np.nan
    g[31] = -np.inf
    L.lmsgd_step(ctx, th, dev(g), d, m, L.lmsgd_schedule_at(None, K32_C, 1))
    code, st = L.lmsgd_query_status(ctx)
    assert code == L.LMSGD_ERR_NONFINITE and st.skipped == 1 and st.first_nonfinite == 31
    with pytest.raises(binary16.NonFiniteError) as e:
        exchange.exchange([g], 1024.0)
    assert e.value.index == st.first_nonfinite
    assert np.array_equal(host(th), th0) and np.array_equal(host(d), d0) and np.array_equal(host(m), m0)
    # the next clean step proceeds normally (status slots are per step)
    g2 = synth.grads(1, 2, n)
    L.lmsgd_step(ctx, th, dev(g2[0]), d, m, L.lmsgd_schedule_at(None, K32_C, 2))
    code, st = L.lmsgd_query_status(ctx)
    assert code == 0 and st.skipped == 0 and st.first_nonfinite == -1
    check_state(host(th), host(d), host(m), th0, d0, m0, exchange.exchange(list(g2), 1024.0).ghat,
                schedule.coeffs_at(2))
    L.lmsgd_finalize(ctx)


def test_k1_no_skip_flag_reports_but_applies():
    n = 4096
    ctx = L.lmsgd_init(1, 0, 0, n, 1.0, None, L.LMSGD_FLAG_NO_SKIP)
    th0, d0, m0 = init_state(n)
    th, d, m = dev(th0), dev(d0), dev(m0)
    g = synth.grads(1, 1, n)[0]
    g[100] = np.nan
    L.lmsgd_step(ctx, th, dev(g), d, m, L.lmsgd_schedule_at(None, K32_C, 1))
    code, st = L.lmsgd_query_status(ctx)
    assert code == L.LMSGD_ERR_NONFINITE and st.first_nonfinite == 100 and st.skipped == 0
    assert not np.array_equal(host(th)[:100], th0[:100])
    L.lmsgd_finalize(ctx)


def test_zero_gradient_fixed_point_and_endpoints():
    n = 5000
    th0, _, _ = init_state(n)
    z = np.zeros(n, np.float32)
    ctx = L.lmsgd_init(1, 0, 0, n, 1.0)
    th, d, m = dev(th0), dev(z), dev(z)
    L.lmsgd_step(ctx, th, dev(z), d, m, L.lmsgd_schedule_at(None, K32_C, 1))
    assert np.array_equal(host(th), th0) and not host(d).any() and not host(m).any()
    # pure momentum SGD (alpha_RMS = 0) and pure RMSprop (alpha_SGD = 0)
    g = synth.grads(1, 1, n)
    for a_sgd, a_rms in ((1.0, 0.0), (0.0, 1.0), (0.3, 2e-5)):
        th, d, m = dev(th0), dev(z), dev(z)
        L.lmsgd_step(ctx, th, dev(g[0]), d, m, L.make_coeffs(0.1, a_sgd, a_rms))
        c = schedule.Coeffs(0.0, 0.1, a_sgd, a_rms, 0)
        check_state(host(th), host(d), host(m), th0, z, z, exchange.exchange(list(g), 1.0).ghat, c)
    L.lmsgd_finalize(ctx)


def test_delta_independent_of_eta_on_gpu():
    """Delta_t carries no eta -- bit-equal under different LR sequences."""
    n = 65_536
    ctxs = [L.lmsgd_init(1, 0, 0, n, 1024.0) for _ in range(2)]
    th0, d0, m0 = init_state(n)
    st = [[dev(th0), dev(d0), dev(m0)] for _ in range(2)]
    a = synth.grad_scale(n)
    for t in range(1, 8):
        g = dev(synth.grads(1, t, n, a)[0])
        c = L.lmsgd_schedule_at(None, C1_C, t)
        for i, eta in enumerate((0.5, 7.0 + t)):
            ci = L.make_coeffs(eta, c.alpha_sgd, c.alpha_rmsprop)
            L.lmsgd_step(ctxs[i], st[i][0], g, st[i][1], st[i][2], ci)
        torch.cuda.synchronize()
        assert torch.equal(st[0][1], st[1][1]) and torch.equal(st[0][2], st[1][2])
    for c in ctxs:
        L.lmsgd_finalize(c)


def test_determinism_and_step_host_matches_step():
    n = 300_001
    th0, d0, m0 = init_state(n)
    g = synth.grads(1, 4, n)[0]
    outs = []
    for use_host in (False, False, True, "oop"):
        ctx = L.lmsgd_init(1, 0, 0, n, 1024.0)
        th, d, m = dev(th0), dev(d0), dev(m0)
        c = L.lmsgd_schedule_at(None, K32_C, 4)
        if use_host:
            gh = torch.from_numpy(g).pin_memory()
            stbuf = torch.zeros(4, dtype=torch.int64).pin_memory()
            ph = torch.full((n,), -1.0).pin_memory()
            if use_host == "oop":
                out = [torch.empty_like(x) for x in (th, d, m)]
                L.lmsgd_step_out_of_place_host(ctx, th, out[0], gh, d, out[1], m, out[2], c, stbuf, ph)
                th, d, m = out
            else:
                L.lmsgd_step_host(ctx, th, gh, d, m, c, stbuf, ph)
            torch.cuda.synchronize()
            s = L.decode_status(stbuf)
            assert s.first_nonfinite == -1 and s.skipped == 0
            assert torch.equal(ph, th.cpu())          # theta_t came back to the host
        else:
            L.lmsgd_step(ctx, th, dev(g), d, m, c)
        outs.append([host(x) for x in (th, d, m)])
        L.lmsgd_finalize(ctx)
    for o in outs[1:]:
        for a, b in zip(o, outs[0]):
            assert np.array_equal(a, b)


def test_c1_twenty_steps_resynced():
    """Config C1: 4,096 params, 2 workers x minibatch 32, 20 steps across the whole
    RMSprop -> SGD warm-up (simulated k = 2 on one GPU), every step checked."""
    n, k, s = 4096, 2, 1024.0
    n_pad = 4096
    a = synth.grad_scale(n)
    th0, d0, m0 = synth.theta0(n, None), np.zeros(n, np.float32), np.zeros(n, np.float32)
    th, d, m = dev(th0), dev(d0), dev(m0)
    hbuf = torch.empty(k * n_pad, dtype=torch.int16, device=DEV)
    R = torch.empty(n_pad, dtype=torch.int16, device=DEV)
    dst = torch.empty(4, dtype=torch.int64, device=DEV)
    free = run.run(th0, lambda t: synth.grads(k, t, n, a), k, 20, s, cluster=C1)
    for t in range(1, 21):
        g = synth.grads(k, t, n, a)
        prev = host(th), host(d), host(m)
        L.lmsgd_status_reset(dst)
        for i in range(k):
            L.lmsgd_pack(dev(g[i]), n_pad, s, hbuf[i * n_pad:(i + 1) * n_pad], dst)
        L.lmsgd_reduce_local(hbuf, k, n_pad, R, dst)
        L.lmsgd_update(R, n, k, s, None, L.lmsgd_schedule_at(None, C1_C, t), th, d, m, dst)
        ex = exchange.exchange(list(g), s)
        assert np.array_equal(host(R).view(np.uint16), ex.R)
        assert np.array_equal(ex.ghat, free.ghat[t - 1])
        check_state(host(th), host(d), host(m), *prev, ex.ghat, schedule.coeffs_at(t, schedule.Hyper(), C1))
    # free-running drift over 20 steps stays small (fp32 vs fp64 compounding)
    scale = np.abs(free.theta) + 1e-3
    # bound: 20 steps x momentum gain 1/(1-mu1) = 10 x per-step 5e-7
    assert run.scaled_error(host(th), free.theta, scale) < 1e-4


def test_full_schedule_resynced_every_step():
    """The whole 90-epoch 32k schedule (T = 3,519 iterations: the RMSprop warm-up, the
    switch to SGD at t = 490 and the LR drops at t = 1565, 2738, 3325) through the
    context path, every step checked against the oracle resynced to the GPU's state;
    then the same run through the CUDA-graph entry point (coefficients from the device
    table) must end bit-identical."""
    n, s = 4099, 1024.0
    T = L.lmsgd_schedule_steps(K32_C)
    assert T == 3519
    a = synth.grad_scale(n)
    th0 = synth.theta0(n, None)
    z = np.zeros(n, np.float32)
    grads = [None] + [synth.grads(1, t, n, a)[0] for t in range(1, T + 1)]
    ctx = L.lmsgd_init(1, 0, 0, n, s)
    th, d, m = dev(th0), dev(z), dev(z)
    worst = 0.0
    for t in range(1, T + 1):
        prev = host(th), host(d), host(m)
        L.lmsgd_step(ctx, th, dev(grads[t]), d, m, L.lmsgd_schedule_at(None, K32_C, t))
        e = check_state(host(th), host(d), host(m), *prev, exchange.exchange([grads[t]], s).ghat,
                        schedule.coeffs_at(t))
        worst = max(worst, max(e.values()))
    code, _ = L.lmsgd_query_status(ctx)
    assert code == 0 and worst <= TOL
    L.lmsgd_finalize(ctx)
    # graph entry point over the same schedule, eagerly (the table and counters are on the device)
    ctxg = L.lmsgd_init(1, 0, 0, n, s)
    L.lmsgd_schedule_upload(ctxg, None, K32_C, 1, T)
    thg, dg, mg = dev(th0), dev(z), dev(z)
    gbuf = dev(z)
    for t in range(1, T + 1):
        gbuf.copy_(dev(grads[t]))
        L.lmsgd_step_graph(ctxg, thg, gbuf, dg, mg)
    code, _ = L.lmsgd_query_status(ctxg)
    assert code == 0
    assert torch.equal(thg, th) and torch.equal(dg, d) and torch.equal(mg, m)
    L.lmsgd_finalize(ctxg)


# ------------------------------------------------------------------ sub-steps / simulated k

def _pack_codec_case(x32, s):
    n = x32.size
    n_pad = (n + 7) // 8 * 8
    h = torch.empty(n_pad, dtype=torch.int16, device=DEV)
    dst = torch.empty(4, dtype=torch.int64, device=DEV)
    L.lmsgd_status_reset(dst)
    L.lmsgd_pack(dev(x32), n_pad, s, h, dst)
    return host(h).view(np.uint16)[:n], host(dst)


def test_pack_vs_oracle_codec_boundary_classes():
    exps = np.arange(127 - 40, 127 + 17, dtype=np.uint32)
    mant = np.concatenate([np.arange(0, 1 << 23, 8191, dtype=np.uint32),
                           ((np.arange(1 << 10, dtype=np.uint32) << 13)[:, None]
                            + np.array([0xFFF, 0x1000, 0x1001], dtype=np.uint32)).ravel()])
    pat = (exps[:, None] << 23 | mant[None, :]).ravel()
    pat = np.concatenate([pat, pat | np.uint32(0x80000000),
                          np.random.default_rng(1).integers(0, 2 ** 32, 1 << 22, dtype=np.uint64).astype(np.uint32)])
    x = pat.view(np.float32)
    x = x[np.isfinite(x)]
    for s in (1.0, 1024.0, 0.5):
        got, st = _pack_codec_case(x, s)
        ref, sat = exchange.pack(x, s)
        bad = np.nonzero(got != ref)[0]
        assert bad.size == 0, (s, x[bad[:4]], got[bad[:4]], ref[bad[:4]])
        assert st[1] == sat and st[0] == np.iinfo(np.int64).max


@pytest.mark.skipif(__import__("os").environ.get("LMSGD_EXHAUSTIVE") != "1", reason="set LMSGD_EXHAUSTIVE=1")
def test_pack_all_fp32_patterns_vs_oracle():
    # k_pack (s = 1) on every one of the 2^32 fp32 bit patterns against the oracle codec,
    # 2^24 patterns per launch; non-finite patterns: only the first-index status counts
    step = 1 << 24
    for hi in range(0, 1 << 32, step):
        pat = np.arange(hi, hi + step, dtype=np.uint64).astype(np.uint32)
        x = pat.view(np.float32)
        got, st = _pack_codec_case(x, 1.0)
        fin = np.isfinite(x)
        ref, sat = binary16.to_binary16(x[fin], return_saturation=True)
        assert np.array_equal(got[fin], ref), hex(hi)
        assert st[1] == sat
        first = np.iinfo(np.int64).max if fin.all() else int(np.argmin(fin))
        assert st[0] == first, hex(hi)


def test_pack_nonfinite_first_index():
    x = np.ones(1000, np.float32)
    x[[500, 17, 999]] = [np.nan, np.inf, -np.inf]
    _, st = _pack_codec_case(x, 1.0)
    assert st[0] == 17


@pytest.mark.parametrize("k", [2, 3, 4, 8])
def test_simulated_k_exchange_bit_exact(k):
    n, s = 123_457, 1024.0
    n_pad = (n + 64 * k - 1) // (64 * k) * 64 * k
    g = synth.grads(k, 9, n)
    g[0, :3] = [60000.0 / s, 60000.0 / s, -1.0]
    g[1, :3] = [60000.0 / s, 1000.0 / s, 1.0]
    hbuf = torch.empty(k * n_pad, dtype=torch.int16, device=DEV)
    R = torch.empty(n_pad, dtype=torch.int16, device=DEV)
    dst = torch.empty(4, dtype=torch.int64, device=DEV)
    L.lmsgd_status_reset(dst)
    for i in range(k):
        L.lmsgd_pack(dev(g[i]), n_pad, s, hbuf[i * n_pad:(i + 1) * n_pad], dst)
    L.lmsgd_reduce_local(hbuf, k, n_pad, R, dst)
    ex = exchange.exchange(list(g), s)
    Rg = host(R).view(np.uint16)
    assert np.array_equal(Rg[:n], ex.R) and not Rg[n:].any()
    stg = host(dst)
    assert stg[1] == ex.pack_saturations and stg[2] == ex.sum_saturations >= 1
    # ghat bit-exact via mu1 = 0, (1, 0) => Delta = -ghat
    hyp = L.lmsgd_hyper_default()
    hyp.mu1 = 0.0
    z = lambda: dev(np.zeros(n, np.float32))  # noqa: E731
    th, d, m = z(), z(), z()
    L.lmsgd_update(R, n, k, s, hyp, L.make_coeffs(1.0, 1.0, 0.0), th, d, m, dst)
    assert np.array_equal(-host(d), ex.ghat)


def test_k1_exchange_through_ctx():
    # lmsgd_exchange at world 1: R = the packed gradient, status of the pack,
    # interleaved with steps on the same context
    n, s = 100_003, 1024.0
    _, n_pad = L.lmsgd_layout(1, n)
    ctx = L.lmsgd_init(1, 0, 0, n, s)
    Rg = torch.full((n_pad,), -1, dtype=torch.int16, device=DEV)
    th, d, m = (dev(np.zeros(n, np.float32)) for _ in range(3))
    for t in (1, 2, 3):
        g = synth.grads(1, t, n)
        g[0, 7] = 70000.0 / s
        L.lmsgd_exchange(ctx, dev(g[0]), Rg)
        code, st = L.lmsgd_query_status(ctx)
        ex = exchange.exchange(list(g), s)
        R = host(Rg).view(np.uint16)
        assert code == 0 and st.skipped == 0 and np.array_equal(R[:n], ex.R) and not R[n:].any()
        assert st.pack_saturations == ex.pack_saturations == 1 and st.sum_saturations == 0
        L.lmsgd_step(ctx, th, dev(g[0]), d, m, L.make_coeffs(1.0, 1.0, 0.0))
        code, st = L.lmsgd_query_status(ctx)
        assert code == 0 and st.skipped == 0 and st.pack_saturations == 1
    g = synth.grads(1, 4, n)
    g[0, [99, 12]] = [np.nan, -np.inf]
    L.lmsgd_exchange(ctx, dev(g[0]), Rg)
    code, st = L.lmsgd_query_status(ctx)
    assert code == L.LMSGD_ERR_NONFINITE and st.skipped == 1 and st.first_nonfinite == 12
    g = synth.grads(1, 5, n)
    L.lmsgd_exchange(ctx, dev(g[0]), Rg)          # the next call is clean again
    code, st = L.lmsgd_query_status(ctx)
    assert code == 0 and st.first_nonfinite == -1 and np.array_equal(host(Rg).view(np.uint16)[:n],
                                                                       exchange.exchange(list(g), s).R)
    L.lmsgd_schedule_upload(ctx, None, C1_C, 1, 4)
    with pytest.raises(L.LmsgdError) as e:        # host-mode epochs: no switch to graph mode
        L.lmsgd_step_graph(ctx, th, dev(g[0]), d, m)
    assert e.value.status == L.LMSGD_ERR_STATE
    L.lmsgd_finalize(ctx)


@pytest.mark.parametrize("n", [1, 9, 65, 10_007, (1 << 20) + 13])
def test_step_out_of_place_matches_step(n):
    # one-pass guarded step, ping-pong buffers: bit-identical to the in-place lmsgd_step,
    # a non-finite gradient leaves out = in (skipped), the next step continues from there
    s = 1024.0
    th0, d0, m0 = init_state(n)
    ref = L.lmsgd_init(1, 0, 0, n, s)
    oop = L.lmsgd_init(1, 0, 0, n, s)
    th, d, m = dev(th0), dev(d0), dev(m0)
    bufs = [[dev(th0), dev(d0), dev(m0)], [dev(np.zeros(n, np.float32)) for _ in range(3)]]
    a = synth.grad_scale(n)
    cur = 0
    for i, t in enumerate((1, 12, 15, 16, 17)):
        g = synth.grads(1, t, n, a)[0]
        if i == 3:
            g[n // 2] = np.nan
        co = L.lmsgd_schedule_at(None, C1_C, t)
        prev = host(th), host(d), host(m)
        L.lmsgd_step(ref, th, dev(g), d, m, co)
        code_r, _ = L.lmsgd_query_status(ref)
        src, dst = bufs[cur], bufs[cur ^ 1]
        L.lmsgd_step_out_of_place(oop, src[0], dst[0], dev(g), src[1], dst[1], src[2], dst[2], co)
        code, st = L.lmsgd_query_status(oop)
        cur ^= 1
        assert code == code_r
        assert all(torch.equal(x, y) for x, y in zip(dst, (th, d, m))), t
        if i == 3:
            assert code == L.LMSGD_ERR_NONFINITE and st.skipped == 1 and st.first_nonfinite == n // 2
            assert all(torch.equal(x, y) for x, y in zip(dst, src))
        else:
            assert code == 0 and st.skipped == 0
            check_state(host(dst[0]), host(dst[1]), host(dst[2]), *prev, exchange.exchange([g], s).ghat,
                        schedule.coeffs_at(t, schedule.Hyper(), C1))
    with pytest.raises(L.LmsgdError) as e:        # outputs overlapping the inputs
        L.lmsgd_step_out_of_place(oop, bufs[0][0], bufs[0][0], dev(g), bufs[0][1], bufs[1][1], bufs[0][2],
                                  bufs[1][2], co)
    assert e.value.status == L.LMSGD_ERR_INVALID_ARG
    L.lmsgd_set_weight_decay(oop, 1e-4)
    with pytest.raises(L.LmsgdError) as e:
        L.lmsgd_step_out_of_place(oop, *(bufs[0][0], bufs[1][0]), dev(g), bufs[0][1], bufs[1][1], bufs[0][2],
                                  bufs[1][2], co)
    assert e.value.status == L.LMSGD_ERR_UNSUPPORTED
    for fl in (L.LMSGD_FLAG_NO_SKIP, L.LMSGD_FLAG_FREEZE_M):   # the call always guards and keeps m
        cf = L.lmsgd_init(1, 0, 0, n, s, None, fl)
        with pytest.raises(L.LmsgdError) as e:
            L.lmsgd_step_out_of_place(cf, bufs[0][0], bufs[1][0], dev(g), bufs[0][1], bufs[1][1], bufs[0][2],
                                      bufs[1][2], co)
        assert e.value.status == L.LMSGD_ERR_UNSUPPORTED
        L.lmsgd_finalize(cf)
    L.lmsgd_finalize(ref)
    L.lmsgd_finalize(oop)


def test_fused_step1_matches_pack_update():
    n = 777_777
    th0, d0, m0 = init_state(n)
    g = dev(synth.grads(1, 2, n)[0])
    c = L.lmsgd_schedule_at(None, K32_C, 2)
    n_pad = (n + 7) // 8 * 8
    a = [dev(x) for x in (th0, d0, m0)]
    b = [dev(x) for x in (th0, d0, m0)]
    dst = torch.empty(4, dtype=torch.int64, device=DEV)
    L.lmsgd_status_reset(dst)
    L.lmsgd_fused_step1(g, 1024.0, None, c, *a, dst)
    h = torch.empty(n_pad, dtype=torch.int16, device=DEV)
    dst2 = torch.empty(4, dtype=torch.int64, device=DEV)
    L.lmsgd_status_reset(dst2)
    L.lmsgd_pack(g, n_pad, 1024.0, h, dst2)
    L.lmsgd_update(h, n, 1, 1024.0, None, c, *b, dst2)
    for x, y in zip(a, b):
        assert torch.equal(x, y)


# ------------------------------------------------------------------ full size (BASELINE configs)

@pytest.mark.parametrize("depth,t,flags", [(50, 1, 0), (50, 392, 0), (50, 1000, 0), (152, 1, 0), (152, 3519, 0),
                                          (50, 1, L.LMSGD_FLAG_NO_SKIP), (152, 2, L.LMSGD_FLAG_NO_SKIP)])
def test_resnet_full_size_sampled(depth, t, flags):
    """C2 / C5 sizes: the 25,557,032-element ResNet-50 and 60,192,808-element
    ResNet-152 buffers, k = 1, in the launch configuration bench.py times; outputs
    compared on a sample of indices (the path is elementwise, so the oracle on the
    sampled indices is exact)."""
    n = synth.resnet_n_params(depth)
    s = 1024.0
    r = np.random.default_rng(t)
    idx = np.unique(np.concatenate([np.arange(1000), np.arange(n - 1000, n), r.integers(0, n, 200_000)]))
    th0 = synth.theta0(n, depth)
    d0 = (r.standard_normal(n) * 1e-3).astype(np.float32)
    m0 = (r.random(n) * 1e-6).astype(np.float32)
    g = synth.grads(1, t, n)
    ctx = L.lmsgd_init(1, 0, 0, n, s, None, flags)
    th, d, m = dev(th0), dev(d0), dev(m0)
    L.lmsgd_step(ctx, th, dev(g[0]), d, m, L.lmsgd_schedule_at(None, K32_C, t))
    code, st = L.lmsgd_query_status(ctx)
    assert code == 0
    ex = exchange.exchange([g[0][idx]], s)
    check_state(host(th)[idx], host(d)[idx], host(m)[idx], th0[idx], d0[idx], m0[idx], ex.ghat,
                schedule.coeffs_at(t))
    L.lmsgd_finalize(ctx)


@pytest.mark.parametrize("depth,t0", [(50, 1), (50, 489), (152, 1), (152, 3517)])
def test_resnet_full_size_out_of_place_sampled(depth, t0):
    """The N = 1 headline kernel pair (k_fused1_oop + k_repair1, lmsgd_step_out_of_place)
    at the C2 / C5 sizes, in bench.py's launch configuration, over three steps with the
    state ping-ponging between two buffer sets: a clean step (sampled oracle parity and
    full-buffer bit-identity with the in-place lmsgd_step), a step with one non-finite
    gradient (skipped: the output set equals the input set bit for bit, status exact),
    and a clean step continuing from the repaired set (sampled parity again)."""
    n = synth.resnet_n_params(depth)
    s = 1024.0
    r = np.random.default_rng(t0)
    idx = np.unique(np.concatenate([np.arange(1000), np.arange(n - 1000, n), r.integers(0, n, 200_000)]))
    th0 = synth.theta0(n, depth)
    d0 = (r.standard_normal(n) * 1e-3).astype(np.float32)
    m0 = (r.random(n) * 1e-6).astype(np.float32)
    oop = L.lmsgd_init(1, 0, 0, n, s)
    ref = L.lmsgd_init(1, 0, 0, n, s)
    sets = [[dev(th0), dev(d0), dev(m0)], [torch.empty(n, device=DEV) for _ in range(3)]]
    inplace = [dev(th0), dev(d0), dev(m0)]
    a = synth.grad_scale(n)
    cur = 0
    for i, t in enumerate((t0, t0 + 1, t0 + 2)):
        g = synth.grads(1, t, n, a)[0]
        if i == 1:
            g[n - 5] = np.nan                    # inside the last (ragged) vector group
            g[n // 3] = -np.inf
        co = L.lmsgd_schedule_at(None, K32_C, t)
        src, dst = sets[cur], sets[cur ^ 1]
        prev = [host(x)[idx] for x in src]
        gd = dev(g)
        L.lmsgd_step_out_of_place(oop, src[0], dst[0], gd, src[1], dst[1], src[2], dst[2], co)
        code, st = L.lmsgd_query_status(oop)
        L.lmsgd_step(ref, inplace[0], gd, inplace[1], inplace[2], co)
        code_r, _ = L.lmsgd_query_status(ref)
        assert code == code_r
        assert all(torch.equal(x, y) for x, y in zip(dst, inplace)), (depth, t)
        if i == 1:
            assert code == L.LMSGD_ERR_NONFINITE and st.skipped == 1 and st.first_nonfinite == n // 3
            assert all(torch.equal(x, y) for x, y in zip(dst, src))
        else:
            assert code == 0 and st.skipped == 0 and st.first_nonfinite == -1
            ex = exchange.exchange([g[idx]], s)
            assert st.pack_saturations == exchange.exchange([g], s).pack_saturations
            check_state(host(dst[0])[idx], host(dst[1])[idx], host(dst[2])[idx], *prev, ex.ghat,
                        schedule.coeffs_at(t))
        cur ^= 1
    L.lmsgd_finalize(oop)
    L.lmsgd_finalize(ref)


# ------------------------------------------------------------------ API behaviour on the GPU

def test_api_errors_on_gpu():
    n = 1000
    ctx = L.lmsgd_init(1, 0, 0, n, 1.0)
    th = torch.zeros(n + 1, device=DEV)
    g = torch.zeros(n, device=DEV)
    import ctypes
    st = L.lib().lmsgd_step(ctx.ptr, None, ctypes.c_void_p(th.data_ptr() + 4), ctypes.c_void_p(g.data_ptr()),
                            ctypes.c_void_p(g.data_ptr()), ctypes.c_void_p(g.data_ptr()),
                            ctypes.byref(L.make_coeffs(0.1, 1.0, 0.0)))
    assert st == L.LMSGD_ERR_INVALID_ARG                  # misaligned (offset 4 B) params
    assert b"aligned" in L.lib().lmsgd_last_error(ctx.ptr)
    for bad in (L.make_coeffs(0.0, 1.0, 0.0), L.make_coeffs(0.1, 1.5, 0.0), L.make_coeffs(0.1, 1.0, -1.0)):
        with pytest.raises(L.LmsgdError) as e:
            L.lmsgd_step(ctx, th[:n], g, g.clone(), g.clone(), bad)
        assert e.value.status == L.LMSGD_ERR_INVALID_ARG
    with pytest.raises(L.LmsgdError) as e:
        L.lmsgd_query_status(ctx)                   # no step yet
    assert e.value.status == L.LMSGD_ERR_STATE
    mean, var = torch.randn(64, device=DEV), torch.rand(64, device=DEV)
    m0, v0 = mean.clone(), var.clone()
    L.lmsgd_bn_stats_allreduce(ctx, mean, var)     # world 1: identity
    assert torch.equal(mean, m0) and torch.equal(var, v0)
    L.lmsgd_finalize(ctx)
    ctx2 = L.lmsgd_init(2, 0, 0, n, 1.0)             # world 2, never connected
    with pytest.raises(L.LmsgdError) as e:
        L.lmsgd_step(ctx2, th[:n], g, g.clone(), g.clone(), L.make_coeffs(0.1, 1.0, 0.0))
    assert e.value.status == L.LMSGD_ERR_STATE
    L.lmsgd_finalize(ctx2)


def test_goyal_schedule_through_ctx():
    """The Goyal et al. schedule selected in the cluster struct."""
    n = 50_000
    cl_c = L.make_cluster(1024, 32, 1_281_167, L.SCHEDULE_GOYAL)
    cl_o = schedule.Cluster(schedule="goyal")
    th0, d0, m0 = init_state(n)
    ctx = L.lmsgd_init(1, 0, 0, n, 1024.0)
    th, d, m = dev(th0), dev(d0), dev(m0)
    for t in (1, 1200, 2400, 3200):
        g = synth.grads(1, t, n)
        prev = host(th), host(d), host(m)
        L.lmsgd_step(ctx, th, dev(g[0]), d, m, L.lmsgd_schedule_at(None, cl_c, t))
        check_state(host(th), host(d), host(m), *prev, exchange.exchange(list(g), 1024.0).ghat,
                    schedule.coeffs_at(t, schedule.Hyper(), cl_o))
    L.lmsgd_finalize(ctx)


def test_bn_sync_world1_is_last_minibatch():
    """f2 at world 1: momentum-1 BN keeps the last minibatch's statistics; the sync is
    the identity (the average of one worker)."""
    from paper_1711_04325_b200 import bn_sync
    torch.manual_seed(0)
    net = torch.nn.Sequential(torch.nn.Conv2d(3, 8, 3), torch.nn.BatchNorm2d(8)).to(DEV)
    bn_sync.last_minibatch_bn(net)
    ctx = L.lmsgd_init(1, 0, 0, 100, 1.0)
    sync = bn_sync.BNStatsSync(net, ctx)
    net.train()
    for _ in range(3):
        xb = torch.randn(16, 3, 10, 10, device=DEV)
        net(xb)
    h = net[0](xb)
    before = sync.mean.clone()
    sync.sync()
    torch.cuda.synchronize()
    assert torch.equal(sync.mean, before)
    assert torch.allclose(net[1].running_mean, h.mean(dim=(0, 2, 3)), rtol=1e-5, atol=1e-6)
    assert torch.allclose(net[1].running_var, h.var(dim=(0, 2, 3), unbiased=True), rtol=1e-4, atol=1e-6)
    L.lmsgd_finalize(ctx)


# ------------------------------------------------------------------ CUDA graphs

@pytest.mark.parametrize("flags", [0, L.LMSGD_FLAG_NO_SKIP])
def test_graph_step_matches_host_step_and_replays(flags):
    """lmsgd_step_graph (device coefficient table + device step counter) equals
    lmsgd_step bit for bit, also when captured once in a CUDA graph and replayed."""
    n, s = 300_007, 1024.0
    th0, d0, m0 = init_state(n)
    a = synth.grad_scale(n)
    grads = [dev(synth.grads(1, t, n, a)[0]) for t in range(1, 7)]
    ref = L.lmsgd_init(1, 0, 0, n, s, None, flags)
    rt, rd, rm = dev(th0), dev(d0), dev(m0)
    refs = []
    for t in range(1, 7):
        L.lmsgd_step(ref, rt, grads[t - 1], rd, rm, L.lmsgd_schedule_at(None, C1_C, t))
        torch.cuda.synchronize()
        refs.append((rt.clone(), rd.clone(), rm.clone()))
    L.lmsgd_finalize(ref)

    ctx = L.lmsgd_init(1, 0, 0, n, s, None, flags)
    L.lmsgd_schedule_upload(ctx, None, C1_C, 1, 6)
    th, d, m = dev(th0), dev(d0), dev(m0)
    gbuf = grads[0].clone()
    L.lmsgd_step_graph(ctx, th, gbuf, d, m)                  # step 1 eagerly
    torch.cuda.synchronize()
    assert all(torch.equal(x, y) for x, y in zip((th, d, m), refs[0]))
    side = torch.cuda.Stream()
    graph = torch.cuda.CUDAGraph()
    with torch.cuda.stream(side):
        with torch.cuda.graph(graph, stream=side):
            L.lmsgd_step_graph(ctx, th, gbuf, d, m, stream=side)
    for t in range(2, 7):                                     # each replay = the next step
        gbuf.copy_(grads[t - 1])
        graph.replay()
        torch.cuda.synchronize()
        assert all(torch.equal(x, y) for x, y in zip((th, d, m), refs[t - 1])), t
        code, st = L.lmsgd_query_status(ctx)
        assert code == 0 and st.skipped == 0
    gbuf.copy_(grads[0])
    before = (th.clone(), d.clone(), m.clone())
    graph.replay()                                            # past the uploaded table
    torch.cuda.synchronize()
    code, st = L.lmsgd_query_status(ctx)
    assert code == L.LMSGD_ERR_RANGE and st.skipped == 1
    assert all(torch.equal(x, y) for x, y in zip((th, d, m), before))
    with pytest.raises(L.LmsgdError) as e:                    # no mixing at world 1
        L.lmsgd_step(ctx, th, gbuf, d, m, L.make_coeffs(0.1, 1.0, 0.0))
    assert e.value.status == L.LMSGD_ERR_STATE
    L.lmsgd_finalize(ctx)


@pytest.mark.parametrize("flags", [0, L.LMSGD_FLAG_NO_SKIP])
def test_weight_decay_prefix(flags):
    """R12: weight decay on the first n_decay elements (PAPER.md:52-53 via Goyal)."""
    n, s, lam, nd = 100_003, 1024.0, 1e-4, 60_001
    th0, d0, m0 = init_state(n)
    ctx = L.lmsgd_init(1, 0, 0, n, s, None, flags)
    L.lmsgd_set_weight_decay(ctx, lam, nd)
    th, d, m = dev(th0), dev(d0), dev(m0)
    for t in (1, 15):
        g = synth.grads(1, t, n)
        prev = host(th), host(d), host(m)
        L.lmsgd_step(ctx, th, dev(g[0]), d, m, L.lmsgd_schedule_at(None, C1_C, t))
        check_state(host(th), host(d), host(m), *prev, exchange.exchange(list(g), s).ghat,
                    schedule.coeffs_at(t, schedule.Hyper(), C1), wd=lam, n_wd=nd)
    with pytest.raises(L.LmsgdError):
        L.lmsgd_set_weight_decay(ctx, -1.0)
    L.lmsgd_finalize(ctx)
    # graph mode: the uploaded table carries lambda (and selects the decay kernel)
    gctx = L.lmsgd_init(1, 0, 0, n, s, None, flags)
    L.lmsgd_set_weight_decay(gctx, lam, nd)
    L.lmsgd_schedule_upload(gctx, None, C1_C, 1, 1)
    gt, gd, gm = dev(th0), dev(d0), dev(m0)
    hctx = L.lmsgd_init(1, 0, 0, n, s, None, flags)
    L.lmsgd_set_weight_decay(hctx, lam, nd)
    ht, hd, hm = dev(th0), dev(d0), dev(m0)
    g1 = dev(synth.grads(1, 1, n)[0])
    L.lmsgd_step_graph(gctx, gt, g1, gd, gm)
    L.lmsgd_step(hctx, ht, g1, hd, hm, L.lmsgd_schedule_at(None, C1_C, 1))
    torch.cuda.synchronize()
    assert torch.equal(gt, ht) and torch.equal(gd, hd) and torch.equal(gm, hm)
    octx = L.lmsgd_init(1, 0, 0, n, s, None, flags)      # no decay: same suffix, other prefix
    ot, od, om = dev(th0), dev(d0), dev(m0)
    L.lmsgd_step(octx, ot, g1, od, om, L.lmsgd_schedule_at(None, C1_C, 1))
    torch.cuda.synchronize()
    assert torch.equal(gm[nd:], om[nd:]) and not torch.equal(gm[:nd], om[:nd])
    L.lmsgd_finalize(octx)
    L.lmsgd_finalize(gctx)
    L.lmsgd_finalize(hctx)


@pytest.mark.parametrize("flags", [0, L.LMSGD_FLAG_NO_SKIP])
def test_freeze_m_sgd_phase(flags):
    """LMSGD_FLAG_FREEZE_M: RMSprop steps are the full rule; on alpha_RMSprop = 0 steps
    theta and Delta are bit-identical to the full rule and m is not touched."""
    n, s = 100_003, 1024.0
    th0, d0, m0 = init_state(n)
    ref = L.lmsgd_init(1, 0, 0, n, s, None, flags)
    frz = L.lmsgd_init(1, 0, 0, n, s, None, flags | L.LMSGD_FLAG_FREEZE_M)
    a, b = [dev(th0), dev(d0), dev(m0)], [dev(th0), dev(d0), dev(m0)]
    for t in (1, 9, 12, 15, 16):   # exp branch, alpha = 1/2 (a_RMS > 0), then SGD
        co = L.lmsgd_schedule_at(None, C1_C, t)
        g = dev(synth.grads(1, t, n)[0])
        m_before = b[2].clone()
        L.lmsgd_step(ref, *a[:1], g, *a[1:], co)
        L.lmsgd_step(frz, *b[:1], g, *b[1:], co)
        torch.cuda.synchronize()
        assert torch.equal(a[0], b[0]) and torch.equal(a[1], b[1]), t
        if co.alpha_rmsprop == 0.0:
            assert torch.equal(b[2], m_before) and not torch.equal(a[2], b[2]), t
        else:
            assert torch.equal(a[2], b[2]), t
    L.lmsgd_finalize(ref)
    L.lmsgd_finalize(frz)


def test_out_of_place_skip_is_repaired_in_stream_order_and_fast():
    """A skipped out-of-place step repairs its output set (k_repair1's copy, 32 blocks): the
    next step, enqueued with no host synchronisation in between, must read the repaired set
    (bit-identical to the in-place reference), and the skipped step must cost well under a
    millisecond, not round 1's 18.7 ms single-block copy."""
    n = synth.resnet_n_params(50)
    s = 1024.0
    th0 = synth.theta0(n, 50)
    r = np.random.default_rng(5)
    d0 = (r.standard_normal(n) * 1e-3).astype(np.float32)
    m0 = (r.random(n) * 1e-6).astype(np.float32)
    oop, ref = L.lmsgd_init(1, 0, 0, n, s), L.lmsgd_init(1, 0, 0, n, s)
    sets = [[dev(th0), dev(d0), dev(m0)], [torch.zeros(n, device=DEV) for _ in range(3)]]
    inplace = [dev(th0), dev(d0), dev(m0)]
    a = synth.grad_scale(n)
    gs = [dev(synth.grads(1, t, n, a)[0]) for t in (1, 2, 3, 4)]
    bad = gs[1].clone()
    bad[n // 2] = float("nan")
    seq = [gs[0], bad, gs[2], bad, bad, gs[3]]
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(len(seq) + 1)]
    torch.cuda.synchronize()
    cur = 0
    ev[0].record()
    for i, g in enumerate(seq):          # no host synchronisation between the steps
        co = L.lmsgd_schedule_at(None, K32_C, i + 1)
        src, dst = sets[cur], sets[cur ^ 1]
        L.lmsgd_step_out_of_place(oop, src[0], dst[0], g, src[1], dst[1], src[2], dst[2], co)
        ev[i + 1].record()
        cur ^= 1
    torch.cuda.synchronize()
    for i, g in enumerate(seq):
        L.lmsgd_step(ref, inplace[0], g, inplace[1], inplace[2], L.lmsgd_schedule_at(None, K32_C, i + 1))
    torch.cuda.synchronize()
    assert all(torch.equal(x, y) for x, y in zip(sets[cur], inplace))
    us = [ev[i].elapsed_time(ev[i + 1]) * 1e3 for i in range(len(seq))]
    clean, skipped = us[5], max(us[3], us[4])    # steps after warm-up
    # a skipped step = the fused pass + the repair copy by 32 blocks: ~0.8 ms at R50 (round
    # 1's one-block copy took 18.7 ms)
    assert skipped < 12.0 * clean and skipped < 2000.0, (us, clean, skipped)
    L.lmsgd_finalize(oop)
    L.lmsgd_finalize(ref)


@pytest.mark.parametrize("n", [1000, 100_003])
def test_16_byte_aligned_buffers_match_32_byte_aligned(n):
    """The streaming kernels use 256-bit accesses (LDG/STG.E.EF.ENL2.256) when every pointer
    of a launch is 32-byte aligned and 128-bit ones otherwise (the ABI only requires 16-byte
    alignment).  Both paths give bit-identical results: in-place guarded (k_pack + k_update),
    in-place fused (k_fused1), out of place (k_fused1_oop), emulated world 2 (k_xupdate)."""
    s = 1024.0
    th0 = synth.theta0(n, None)
    r = np.random.default_rng(n)
    d0 = (r.standard_normal(n) * 1e-3).astype(np.float32)
    m0 = (r.random(n) * 1e-6).astype(np.float32)
    g = synth.grads(2, 3, n)
    co = L.lmsgd_schedule_at(None, C1_C, 3)

    def bufs(off):   # theta, Delta, m, g0, g1 at a float offset into fresh allocations
        out = []
        for x in (th0, d0, m0, g[0], g[1]):
            b = torch.zeros(n + 8, device=DEV)
            b[off:off + n] = dev(x)
            out.append(b[off:off + n])
        return out

    results = []
    for off in (0, 4):   # 0: 32-byte aligned (torch allocations are), 4: 16-byte only
        a = bufs(off)
        assert (a[0].data_ptr() % 32 == 0) == (off == 0)
        out = {}
        ctx = L.lmsgd_init(1, 0, 0, n, s)
        th, d, m = (x.clone() for x in a[:3])
        L.lmsgd_step(ctx, th, a[3], d, m, co)
        out["guarded"] = (th, d, m)
        ctxf = L.lmsgd_init(1, 0, 0, n, s, None, L.LMSGD_FLAG_NO_SKIP)
        th, d, m = (x.clone() for x in a[:3])
        L.lmsgd_step(ctxf, th, a[3], d, m, co)
        out["fused"] = (th, d, m)
        b = bufs(off)
        ctxo = L.lmsgd_init(1, 0, 0, n, s)
        L.lmsgd_step_out_of_place(ctxo, a[0], b[0], a[3], a[1], b[1], a[2], b[2], co)
        out["oop"] = tuple(b[:3])
        ctxs = [L.lmsgd_init(2, r_, 0, n, s) for r_ in range(2)]
        L.lmsgd_connect_group(ctxs)
        st2 = [[x.clone() for x in bufs(off)[:3]] for _ in range(2)]
        L.lmsgd_step_group(ctxs, [x[0] for x in st2], [a[3], a[4]], [x[1] for x in st2], [x[2] for x in st2], co)
        out["group"] = tuple(st2[0])
        torch.cuda.synchronize()
        for c_ in [ctx, ctxf, ctxo] + ctxs:
            assert L.lmsgd_query_status(c_)[0] == 0
            L.lmsgd_finalize(c_)
        results.append({k: tuple(x.cpu() for x in v) for k, v in out.items()})
    for k in results[0]:
        assert all(torch.equal(x, y) for x, y in zip(results[0][k], results[1][k])), k
