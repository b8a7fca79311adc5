"""The torch-style front end (paper_1711_04325_b200.optim.LMSGD) on a small conv net:
zero-copy flat buffers (row a1), schedule (a0), weight-decay ordering (R12),
one-step parity against the oracle on every step, checkpoint/resume bit-exact."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA GPU", allow_module_level=True)

import paper_1711_04325_b200 as L  # noqa: E402
from oracle import exchange, schedule  # noqa: E402
from test_gpu_parity import check_state  # noqa: E402

pytestmark = pytest.mark.gpu
DEV = torch.device("cuda:0")
C1 = schedule.Cluster(n_workers=2, b_local=32, n_train=64)


def _net(seed=0):
    torch.manual_seed(seed)
    return torch.nn.Sequential(torch.nn.Conv2d(3, 8, 3), torch.nn.BatchNorm2d(8), torch.nn.ReLU(),
                               torch.nn.Flatten(), torch.nn.Linear(8 * 6 * 6, 10)).to(DEV)


def _batch(t):
    g = torch.Generator(device="cpu").manual_seed(100 + t)
    return (torch.randn(32, 3, 8, 8, generator=g).to(DEV), torch.randint(0, 10, (32,), generator=g).to(DEV))


def _train_step(net, opt, t):
    x, y = _batch(t)
    opt.zero_grad()
    torch.nn.functional.cross_entropy(net(x), y).backward()


def test_lmsgd_optimizer_matches_oracle_and_resumes(monkeypatch):
    # bit-exact resume needs a deterministic backward (cuDNN's default conv wgrad may use atomics)
    monkeypatch.setattr(torch.backends.cudnn, "deterministic", True)
    monkeypatch.setattr(torch.backends.cudnn, "benchmark", False)
    lam, s = 1e-4, 1024.0
    net = _net()
    opt = L.LMSGD(net.parameters(), cluster=L.make_cluster(2, 32, 64), loss_scale=s, weight_decay=lam)
    # R12 ordering: conv and fc weights first (decayed), BN and biases after
    assert opt.n_decay == 8 * 3 * 3 * 3 + 10 * 8 * 6 * 6
    assert opt.n == sum(p.numel() for p in net.parameters())
    for t in range(1, 6):   # exp branch: alpha_RMS > 0
        _train_step(net, opt, t)
        g = opt.flat_g.cpu().numpy()[None]
        prev = opt.flat_p.cpu().numpy(), opt.delta.cpu().numpy(), opt.m.cpu().numpy()
        c = opt.step()
        code, st = opt.status()
        assert code == 0 and st.skipped == 0 and c.epoch == schedule.coeffs_at(t, schedule.Hyper(), C1).epoch
        check_state(opt.flat_p.cpu().numpy(), opt.delta.cpu().numpy(), opt.m.cpu().numpy(), *prev,
                    exchange.exchange(list(g), s).ghat, schedule.coeffs_at(t, schedule.Hyper(), C1),
                    wd=lam, n_wd=opt.n_decay)
    # the module's parameters ARE the flat buffer (zero copy)
    assert net[0].weight.data_ptr() == opt.flat_p.data_ptr()
    # checkpoint, continue 3 steps; restore into a fresh model + optimizer, same 3 steps
    ck_model = {k: v.clone() for k, v in net.state_dict().items()}
    ck_opt = opt.state_dict()
    for t in range(6, 9):
        _train_step(net, opt, t)
        opt.step()
    torch.cuda.synchronize()
    net2 = _net(seed=1)
    opt2 = L.LMSGD(net2.parameters(), cluster=L.make_cluster(2, 32, 64), loss_scale=s, weight_decay=lam)
    net2.load_state_dict(ck_model)
    opt2.load_state_dict(ck_opt)
    assert opt2.t == 6
    for t in range(6, 9):
        _train_step(net2, opt2, t)
        opt2.step()
    torch.cuda.synchronize()
    assert torch.equal(opt.flat_p, opt2.flat_p) and torch.equal(opt.delta, opt2.delta) and torch.equal(opt.m, opt2.m)
    opt.close()
    opt2.close()


def test_lmsgd_detached_grad_fails_loudly():
    net = _net()
    opt = L.LMSGD(net.parameters(), cluster=L.make_cluster(2, 32, 64))
    _train_step(net, opt, 1)
    net.zero_grad(set_to_none=True)
    x, y = _batch(2)
    torch.nn.functional.cross_entropy(net(x), y).backward()
    with pytest.raises(RuntimeError, match="flat gradient"):
        opt.step()
    opt.close()


def test_lmsgd_rejects_cpu_params():
    with pytest.raises(ValueError):
        L.LMSGD(torch.nn.Linear(4, 4).parameters())


def test_lmsgd_out_of_place_matches_in_place(monkeypatch):
    # out_of_place=True (opt-in, world 1, no weight decay): the parameters alternate
    # between two flat buffers, results bit-identical to in place (the default)
    monkeypatch.setattr(torch.backends.cudnn, "deterministic", True)
    monkeypatch.setattr(torch.backends.cudnn, "benchmark", False)
    nets = [_net(), _net()]
    opts = [L.LMSGD(nets[0].parameters(), cluster=L.make_cluster(2, 32, 64), out_of_place=True),
            L.LMSGD(nets[1].parameters(), cluster=L.make_cluster(2, 32, 64))]
    assert opts[0].out_of_place and not opts[1].out_of_place
    for t in range(1, 8):
        for net, opt in zip(nets, opts):
            _train_step(net, opt, t)
            opt.step()
        torch.cuda.synchronize()
        assert torch.equal(opts[0].flat_p, opts[1].flat_p), t
        assert torch.equal(opts[0].delta, opts[1].delta) and torch.equal(opts[0].m, opts[1].m), t
        # the module sees the step's output buffer
        assert nets[0][0].weight.data_ptr() == opts[0].flat_p.data_ptr()
        assert all(torch.equal(a, b) for a, b in zip(nets[0].parameters(), nets[1].parameters()))
    for o in opts:
        o.close()


def test_lmsgd_out_of_place_resume(monkeypatch):
    # checkpoint/resume in the out-of-place mode: the state lives in whichever buffer set
    # is current; a fresh optimizer restored from the checkpoint continues bit-identically
    monkeypatch.setattr(torch.backends.cudnn, "deterministic", True)
    monkeypatch.setattr(torch.backends.cudnn, "benchmark", False)
    net = _net()
    opt = L.LMSGD(net.parameters(), cluster=L.make_cluster(2, 32, 64), out_of_place=True)
    assert opt.out_of_place
    for t in range(1, 4):   # odd number of steps: the current set is the second one
        _train_step(net, opt, t)
        opt.step()
    ck_model = {k: v.clone() for k, v in net.state_dict().items()}
    ck_opt = opt.state_dict()
    for t in range(4, 7):
        _train_step(net, opt, t)
        opt.step()
    torch.cuda.synchronize()
    net2 = _net(seed=1)
    opt2 = L.LMSGD(net2.parameters(), cluster=L.make_cluster(2, 32, 64), out_of_place=True)
    net2.load_state_dict(ck_model)
    opt2.load_state_dict(ck_opt)
    for t in range(4, 7):
        _train_step(net2, opt2, t)
        opt2.step()
    torch.cuda.synchronize()
    assert torch.equal(opt.flat_p, opt2.flat_p) and torch.equal(opt.delta, opt2.delta) and torch.equal(opt.m, opt2.m)
    opt.close()
    opt2.close()


def test_lmsgd_default_in_place_with_captured_forward(monkeypatch):
    # the default (in place) keeps every parameter's storage fixed, so a forward pass
    # captured once in a CUDA graph sees the updated weights on every replay
    monkeypatch.setattr(torch.backends.cudnn, "benchmark", False)
    net = _net()
    opt = L.LMSGD(net.parameters(), cluster=L.make_cluster(2, 32, 64))
    assert not opt.out_of_place
    ptrs = [p.data_ptr() for p in net.parameters()]
    x = torch.randn(4, 3, 8, 8, device="cuda")
    side = torch.cuda.Stream()
    side.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(side):
        net(x)   # warm-up on the capture stream
    torch.cuda.current_stream().wait_stream(side)
    graph = torch.cuda.CUDAGraph()
    with torch.cuda.graph(graph):
        y_static = net(x)
    for t in range(1, 4):
        graph.replay()
        before = y_static.clone()
        _train_step(net, opt, t)
        opt.step()
        graph.replay()
        torch.cuda.synchronize()
        with torch.no_grad():
            eager = net(x)
        # the replay used the new weights (eager and captured kernels may differ in rounding)
        assert not torch.equal(y_static, before), t
        assert torch.allclose(y_static, eager, rtol=1e-4, atol=1e-5), t
    assert [p.data_ptr() for p in net.parameters()] == ptrs
    opt.close()


def test_lmsgd_out_of_place_rejects_flags():
    with pytest.raises(ValueError):
        L.LMSGD(_net().parameters(), out_of_place=True, flags=L.LMSGD_FLAG_FREEZE_M)


def _deep_net(seed=0):
    torch.manual_seed(seed)
    return torch.nn.Sequential(torch.nn.Conv2d(3, 16, 3), torch.nn.BatchNorm2d(16), torch.nn.ReLU(),
                               torch.nn.Conv2d(16, 32, 3), torch.nn.BatchNorm2d(32), torch.nn.ReLU(),
                               torch.nn.Conv2d(32, 32, 3), torch.nn.ReLU(), torch.nn.Flatten(),
                               torch.nn.Linear(32 * 2 * 2, 64), torch.nn.ReLU(), torch.nn.Linear(64, 10)).to(DEV)


@pytest.mark.parametrize("overlap,bucket", [(True, 1000), (True, 64), (False, 5000), (True, 1 << 22)])
def test_bucketed_lmsgd_matches_lmsgd_and_oracle(monkeypatch, overlap, bucket):
    """Row f1: the bucketed exchange (one lmsgd_exchange per bucket from a post-accumulate
    hook, on a side stream, then one lmsgd_update) gives bit-identically the state of the
    unbucketed LMSGD step, and the oracle's one-step state; a non-finite gradient in one
    bucket skips the whole step (first index global)."""
    monkeypatch.setattr(torch.backends.cudnn, "deterministic", True)
    monkeypatch.setattr(torch.backends.cudnn, "benchmark", False)
    s = 1024.0
    net_a, net_b = _deep_net(), _deep_net()
    opt_a = L.LMSGD(net_a.parameters(), cluster=L.make_cluster(2, 32, 64), loss_scale=s)
    opt_b = L.BucketedLMSGD(net_b.parameters(), cluster=L.make_cluster(2, 32, 64), loss_scale=s,
                            bucket_elems=bucket, exchange_blocks=16, overlap=overlap)
    bks = sorted((bk["lo"], bk["hi"]) for bk in opt_b.buckets)   # the buckets tile [0, n) at 64 k boundaries
    assert bks[0][0] == 0 and bks[-1][1] == opt_b.n and all(a[1] == b[0] for a, b in zip(bks, bks[1:]))
    assert all(lo % 64 == 0 for lo, _ in bks) and (len(bks) > 1) == (bucket < opt_b.n)
    for t in range(1, 5):
        x, y = torch.randn(16, 3, 8, 8, generator=torch.Generator().manual_seed(t)).to(DEV), \
            torch.randint(0, 10, (16,), generator=torch.Generator().manual_seed(t)).to(DEV)
        for net, opt in ((net_a, opt_a), (net_b, opt_b)):
            opt.zero_grad()
            torch.nn.functional.cross_entropy(net(x), y).backward()
        g = opt_b.flat_g.cpu().numpy()[None]
        assert np.array_equal(g[0], opt_a.flat_g.cpu().numpy())
        prev = opt_b.flat_p.cpu().numpy(), opt_b.delta.cpu().numpy(), opt_b.m.cpu().numpy()
        opt_a.step()
        opt_b.step()
        code, st = opt_b.status()
        assert code == 0 and st.skipped == 0
        assert torch.equal(opt_a.flat_p, opt_b.flat_p) and torch.equal(opt_a.delta, opt_b.delta) and \
            torch.equal(opt_a.m, opt_b.m), t
        check_state(opt_b.flat_p.cpu().numpy(), opt_b.delta.cpu().numpy(), opt_b.m.cpu().numpy(), *prev,
                    exchange.exchange(list(g), s).ghat, schedule.coeffs_at(t, schedule.Hyper(), C1))
    # a NaN in one parameter's gradient (a tensor hook, i.e. inside backward): every bucket
    # is exchanged, the update is skipped, the first index is the global flat index
    w = net_b[3].weight
    off = sum(p.numel() for p in opt_b.params[:[id(p) for p in opt_b.params].index(id(w))])
    h = w.register_hook(lambda gr: gr.index_put((torch.tensor([1], device=DEV),), torch.tensor(float("nan"),
                                                                                            device=DEV)))
    before = opt_b.flat_p.clone(), opt_b.delta.clone(), opt_b.m.clone()
    opt_b.zero_grad()
    torch.nn.functional.cross_entropy(net_b(x), y).backward()
    opt_b.step()
    code, st = opt_b.status()
    h.remove()
    row = w.shape[1] * w.shape[2] * w.shape[3]
    assert code == L.LMSGD_ERR_NONFINITE and st.skipped == 1 and st.first_nonfinite == off + row, \
        (code, st.first_nonfinite, off + row)
    assert torch.equal(before[0], opt_b.flat_p) and torch.equal(before[1], opt_b.delta) and torch.equal(before[2], opt_b.m)
    # and the next clean step goes through
    opt_b.zero_grad()
    torch.nn.functional.cross_entropy(net_b(x), y).backward()
    opt_b.step()
    assert opt_b.status()[0] == 0
    opt_a.close()
    opt_b.close()


def test_bucketed_lmsgd_accumulation_needs_no_sync(monkeypatch):
    """Two backward passes before one step: inside no_sync() the first only accumulates and
    the step equals LMSGD's on the summed gradient; without it the second backward is
    refused (its buckets were already exchanged)."""
    monkeypatch.setattr(torch.backends.cudnn, "deterministic", True)
    monkeypatch.setattr(torch.backends.cudnn, "benchmark", False)
    s = 1024.0
    net_a, net_b = _deep_net(), _deep_net()
    opt_a = L.LMSGD(net_a.parameters(), cluster=L.make_cluster(2, 32, 64), loss_scale=s)
    opt_b = L.BucketedLMSGD(net_b.parameters(), cluster=L.make_cluster(2, 32, 64), loss_scale=s, bucket_elems=2048)
    xs = [torch.randn(8, 3, 8, 8, generator=torch.Generator().manual_seed(i)).to(DEV) for i in range(2)]
    y = torch.zeros(8, dtype=torch.long, device=DEV)
    for net, opt in ((net_a, opt_a), (net_b, opt_b)):
        opt.zero_grad()
        if opt is opt_b:
            with opt_b.no_sync():
                torch.nn.functional.cross_entropy(net(xs[0]), y).backward()
        else:
            torch.nn.functional.cross_entropy(net(xs[0]), y).backward()
        torch.nn.functional.cross_entropy(net(xs[1]), y).backward()
        opt.step()
    assert opt_b.status()[0] == 0
    assert torch.equal(opt_a.flat_p, opt_b.flat_p) and torch.equal(opt_a.delta, opt_b.delta)
    opt_b.zero_grad()
    torch.nn.functional.cross_entropy(net_b(xs[0]), y).backward()
    with pytest.raises(RuntimeError, match="no_sync"):
        torch.nn.functional.cross_entropy(net_b(xs[1]), y).backward()
    opt_a.close()
    opt_b.close()
