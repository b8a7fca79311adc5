"""NVLS parity worker (include/lmsgd.h "NVLS"), launched by tests/test_multigpu.py
through torchrun with one process per GPU (world >= 2 GPUs of one NVSwitch node).

The switch accumulates the fp16 wire in fp32 (multimem.ld_reduce ... .acc::f32), so R
is the oracle's exact-sum R up to one fp16 rounding of an inexact fp32 sum (reading
R8').  Checked for both NVLS modes (RS: the switch reduces into the owner's
R, the update pulls it; ALLREDUCE: the owner multicasts R back into every wire):
  * lmsgd_exchange: R within one fp16 ulp of the oracle's R on every element, at most
    1e-3 of the elements differing at all, padding zero, R identical on every rank and
    identical between two calls on the same input (the switch's sum is deterministic);
  * ghat within 1e-3 |ghat| + 2^-24/(k s) of the oracle (north_star / SURVEY 8(c));
  * the state after each step within 1e-6 scaled of the oracle resynced to the GPU's
    previous state AND to the GPU's R (the one-step bar, with the NVLS R as input);
  * replicas bit-identical after every step; status words: pack saturations exact,
    sum saturations = the oracle's count for sums far past 65504;
  * a non-finite gradient on one rank skips the step on every rank;
  * a CUDA-graph capture of the step replays correctly;
  * 2,000 steps under random per-rank device skew end bit-identical to the same
    sequence without skew, and the modes switch between steps (OFF <-> RS <-> ALLREDUCE);
  * the full ResNet-50 buffer on sampled indices.
Prints "NVLS_OK world=k" on rank 0 when everything passes.
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
from mgpu_worker import check_state, replicas_identical  # noqa: E402
from oracle import binary16, exchange, schedule  # noqa: E402

S = 1024.0
S_SCALE = S
C1 = schedule.Cluster(n_workers=2, b_local=32, n_train=64)
C1_C = L.make_cluster(2, 32, 64)
MODES = (L.LMSGD_NVLS_RS, L.LMSGD_NVLS_ALLREDUCE)


def f16_ulp_apart(a, b):
    """Distance in fp16 ulps of two arrays of binary16 bit patterns (monotone integer map)."""
    def key(u):
        u = u.astype(np.int64)
        return np.where(u & 0x8000, -(u & 0x7FFF), u & 0x7FFF)
    return np.abs(key(a) - key(b))


STATS = {"elems": 0, "not_rne": 0, "toward_zero": 0}


def check_R(R, n, ex, k):
    """R of the NVLS all-reduce against the oracle's exact sum S: R must be a faithful
    fp16 rounding of S (one of the two fp16 values bracketing S; the RNE value the
    oracle picks is one of them), or +-65504 where |S| > 65504 (R7); ghat within the
    stated tolerance.  How often R is not the RNE value, and in which direction, is
    recorded (STATS) for DESIGN.md."""
    Rn = R[:n]
    assert not R[n:].any(), "padding not zero"
    hw = binary16.from_binary16(Rn)
    rne = binary16.from_binary16(ex.R)
    S = ex.S
    inrange = np.abs(S) <= 65504.0
    d = f16_ulp_apart(Rn, ex.R)
    # faithful: hw == rne, or hw is rne's neighbour on the other side of S
    other_side = np.sign(hw - S) != np.sign(rne - S)
    ok = (d == 0) | ((d == 1) & other_side & inrange)
    assert ok.all(), f"R not a faithful rounding of the exact sum at {np.flatnonzero(~ok)[:5]}"
    STATS["elems"] += int(n)
    STATS["not_rne"] += int((d > 0).sum())
    STATS["toward_zero"] += int(((d > 0) & (np.abs(hw) < np.abs(S))).sum())
    gh = hw.astype(np.float32) * np.float32(1.0 / (k * S_SCALE))
    tol = 1e-3 * np.abs(ex.ghat.astype(np.float64)) + 2.0 ** -24 / (k * S_SCALE)
    assert np.all(np.abs(gh.astype(np.float64) - ex.ghat) <= tol), "ghat outside 1e-3 |ghat| + 2^-24/(k s)"
    return gh


def nvls_ctx(world, rank, local, n, mode, hyper=None):
    ctx = L.lmsgd_init(world, rank, local, n, S, hyper)
    L.connect_process_group(ctx)
    L.connect_nvls(ctx, mode)
    return ctx


def main():
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    local = int(os.environ["LOCAL_RANK"])
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    dist.init_process_group("nccl", device_id=dev)
    D = lambda x: torch.from_numpy(np.ascontiguousarray(x)).to(dev)  # noqa: E731
    H = lambda x: x.cpu().numpy()  # noqa: E731
    assert L.lmsgd_nvls_supported(local), "device has no multicast support"

    def exchange_R(ctx, g, n_pad):
        R = torch.full((n_pad,), -1, dtype=torch.int16, device=dev)
        L.lmsgd_exchange(ctx, g, R)
        code, st = L.lmsgd_query_status(ctx)
        return code, st, H(R).view(np.uint16)

    for mode in MODES:
        # ---- exchange + update on ragged sizes, across the warm-up
        for n in (1, 100, 64 * world + 3, 123_457, (1 << 20) + 13):
            ctx = nvls_ctx(world, rank, local, n, mode)
            _, n_pad = L.lmsgd_layout(world, n)
            a = synth.grad_scale(n)
            r = np.random.default_rng(n)
            th0 = synth.theta0(n, None)
            th, d, m = D(th0), D((r.standard_normal(n) * 1e-3).astype(np.float32)), D((r.random(n) * 1e-6).astype(np.float32))
            for t in (1, 2, 11, 12, 15):
                g = synth.grads(world, t, n, a)
                gd = D(g[rank])
                ex = exchange.exchange(list(g), S)
                code, st, R = exchange_R(ctx, gd, n_pad)
                assert code == 0 and st.skipped == 0 and st.pack_saturations == ex.pack_saturations, (mode, n, t, code)
                gh = check_R(R, n, ex, world)
                code2, _, R2 = exchange_R(ctx, gd, n_pad)
                assert code2 == 0 and np.array_equal(R, R2), "switch sum not deterministic"
                replicas_identical(torch.from_numpy(R.view(np.int32).copy()).to(dev))   # n_pad is even
                prev = H(th), H(d), H(m)
                L.lmsgd_step(ctx, th, gd, d, m, L.lmsgd_schedule_at(None, C1_C, t))
                code, st = L.lmsgd_query_status(ctx)
                assert code == 0 and st.skipped == 0 and st.first_nonfinite == -1, (code, st.skipped)
                check_state(H(th), H(d), H(m), *prev, gh, schedule.coeffs_at(t, schedule.Hyper(), C1))
                replicas_identical(th, d, m)
            dist.barrier()
            L.lmsgd_finalize(ctx)

        # ---- saturation, non-finite skip, mode switching
        n = 200_003
        hyp = L.lmsgd_hyper_default()
        hyp.mu1 = 0.0                   # (1, 0), mu1 = 0: Delta = -ghat exactly
        ctx = nvls_ctx(world, rank, local, n, mode, hyp)
        z = lambda: D(np.zeros(n, np.float32))  # noqa: E731
        th, d, m = z(), z(), z()
        g = synth.grads(world, 7, n)
        g[:, 0] = 60000.0 / S           # the sum is far past 65504 on every k >= 2: inf -> saturated
        g[0, 1] = 70000.0 / S           # rank 0 saturates at pack
        L.lmsgd_step(ctx, th, D(g[rank]), d, m, L.make_coeffs(1.0, 1.0, 0.0))
        code, st = L.lmsgd_query_status(ctx)
        ex = exchange.exchange(list(g), S)
        assert code == 0 and st.pack_saturations == ex.pack_saturations >= 1
        assert st.sum_saturations == ex.sum_saturations >= 1, (st.sum_saturations, ex.sum_saturations)
        gh = -H(d)
        assert gh[0] == np.float32(65504.0 / (world * S)), gh[0]
        tol = 1e-3 * np.abs(ex.ghat.astype(np.float64)) + 2.0 ** -24 / (world * S)
        assert np.all(np.abs(gh.astype(np.float64) - ex.ghat) <= tol)
        th0, d0, m0 = H(th), H(d), H(m)
        g = synth.grads(world, 8, n)
        g[world - 1, 4321] = np.nan
        g[0, 9999] = np.inf
        L.lmsgd_step(ctx, th, D(g[rank]), d, m, L.make_coeffs(1.0, 1.0, 0.0))
        code, st = L.lmsgd_query_status(ctx)
        assert code == L.LMSGD_ERR_NONFINITE and st.skipped == 1 and st.first_nonfinite == 4321, (code, st.first_nonfinite)
        assert np.array_equal(H(th), th0) and np.array_equal(H(d), d0) and np.array_equal(H(m), m0)
        for md in (L.LMSGD_NVLS_OFF, mode, L.LMSGD_NVLS_RS, L.LMSGD_NVLS_ALLREDUCE, L.LMSGD_NVLS_OFF):
            L.lmsgd_nvls_mode(ctx, md)
            g = synth.grads(world, 9 + md, n)
            L.lmsgd_step(ctx, th, D(g[rank]), d, m, L.make_coeffs(1.0, 1.0, 0.0))
            code, st = L.lmsgd_query_status(ctx)
            ex = exchange.exchange(list(g), S)
            assert code == 0
            if md == L.LMSGD_NVLS_OFF:
                assert np.array_equal(-H(d), ex.ghat), "peer path after NVLS: ghat not bit-exact"
            else:
                tol = 1e-3 * np.abs(ex.ghat.astype(np.float64)) + 2.0 ** -24 / (world * S)
                assert np.all(np.abs(-H(d).astype(np.float64) - ex.ghat) <= tol)
            replicas_identical(th, d, m)
        dist.barrier()
        L.lmsgd_finalize(ctx)

        # ---- CUDA graph: eager graph-mode steps, then one capture replayed
        n = 77_777
        ctx = nvls_ctx(world, rank, local, n, mode)
        _, n_pad = L.lmsgd_layout(world, n)
        a = synth.grad_scale(n)
        th, d, m = D(synth.theta0(n, None)), D(np.zeros(n, np.float32)), D(np.zeros(n, np.float32))
        L.lmsgd_schedule_upload(ctx, None, C1_C, 1, 10)
        gbuf = D(np.zeros(n, np.float32))
        side = torch.cuda.Stream()
        graph = None
        ref = L.lmsgd_init(world, rank, local, n, S)      # R of the same input through lmsgd_exchange
        L.connect_process_group(ref)
        L.connect_nvls(ref, mode)
        for t in range(1, 7):
            g = synth.grads(world, t, n, a)
            gbuf.copy_(D(g[rank]))
            _, _, R = exchange_R(ref, gbuf, n_pad)
            gh = check_R(R, n, exchange.exchange(list(g), S), world)
            prev = H(th), H(d), H(m)
            if t <= 2:
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
            check_state(H(th), H(d), H(m), *prev, gh, schedule.coeffs_at(t, schedule.Hyper(), C1))
            replicas_identical(th, d, m)
        dist.barrier()
        L.lmsgd_finalize(ctx)
        L.lmsgd_finalize(ref)

    # ---- skew stress: per-rank device delays, exchanges, non-finite steps and mode
    #      switches interleaved; bit-identical replicas and no dependence on timing
    n = 100_003
    gen = torch.Generator(device=dev)
    gen.manual_seed(77 + rank)
    pool = [torch.randn(n, generator=gen, device=dev) * 1e-3 for _ in range(8)]
    bad = pool[0].clone()
    bad[12_345] = float("nan")
    rbuf = torch.empty(L.lmsgd_layout(world, n)[1], dtype=torch.int16, device=dev)
    steps = int(os.environ.get("LMSGD_STRESS_STEPS", 2000))
    finals = []
    for delayed in (False, True):
        ctx = nvls_ctx(world, rank, local, n, L.LMSGD_NVLS_ALLREDUCE)
        th = D(synth.theta0(n, None))
        d, m = torch.zeros(n, device=dev), torch.zeros(n, device=dev)
        rng = np.random.default_rng(1234 + (rank if delayed else 0))
        for it in range(steps):
            if it % 250 == 0:
                L.lmsgd_nvls_mode(ctx, (L.LMSGD_NVLS_ALLREDUCE, L.LMSGD_NVLS_RS, L.LMSGD_NVLS_OFF)[(it // 250) % 3])
            if delayed and rng.random() < 0.3:
                torch.cuda._sleep(int(rng.integers(1, 200_000)))
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

    # ---- full ResNet-50 buffer, sampled: R against the oracle, the state against the
    #      oracle resynced to the GPU's R
    n = synth.resnet_n_params(50)
    for mode in MODES:
        ctx = nvls_ctx(world, rank, local, n, mode)
        _, n_pad = L.lmsgd_layout(world, n)
        th0 = synth.theta0(n, 50)
        g = synth.grads(world, 1, n)
        gd = D(g[rank])
        code, st, R = exchange_R(ctx, gd, n_pad)
        assert code == 0
        idx = np.unique(np.concatenate([np.arange(2000), np.arange(n - 2000, n),
                                        np.random.default_rng(3).integers(0, n, 100_000)]))
        ex = exchange.exchange([gi[idx] for gi in g], S)
        Rs = np.zeros(idx.size + 1, np.uint16)      # check_R wants padding after the sampled values
        Rs[:idx.size] = R[idx]
        gh = check_R(Rs, idx.size, ex, world)
        th, d, m = D(th0), D(np.zeros(n, np.float32)), D(np.zeros(n, np.float32))
        L.lmsgd_step(ctx, th, gd, d, m, L.lmsgd_schedule_at(None, L.make_cluster(), 1))
        code, st = L.lmsgd_query_status(ctx)
        assert code == 0
        zz = np.zeros(idx.size, np.float32)
        check_state(H(th)[idx], H(d)[idx], H(m)[idx], th0[idx], zz, zz, gh, schedule.coeffs_at(1))
        replicas_identical(th, d, m)
        dist.barrier()
        L.lmsgd_finalize(ctx)

    dist.barrier()
    if rank == 0:
        print(f"NVLS R vs the exact-sum RNE R: {STATS['not_rne']} of {STATS['elems']} elements differ "
              f"({STATS['not_rne'] / max(1, STATS['elems']):.4f}), {STATS['toward_zero']} of them toward zero",
              flush=True)
        print(f"NVLS_OK world={world}", flush=True)
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
