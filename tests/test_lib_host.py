"""Host-side checks of the C ABI library (no GPU needed): it loads, exports every
function include/lmsgd.h declares, rejects bad arguments synchronously, and its C++
schedule is bit-identical to the oracle's doubles."""
import ctypes
import math
import os
import re
import struct
import subprocess

import pytest

import paper_1711_04325_b200 as L
from oracle import schedule as sch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared():
    src = open(os.path.join(ROOT, "include", "lmsgd.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(lmsgd_[a-z0-9_]+)\s*\(", src)))


def test_every_declared_symbol_is_exported():
    names = _declared()
    assert len(names) >= 19
    lib = ctypes.CDLL(L.LIB_PATH)
    for n in names:
        assert hasattr(lib, n), n
    out = subprocess.run(["nm", "-D", "--defined-only", L.LIB_PATH], capture_output=True, text=True).stdout
    exported = set(re.findall(r" T (lmsgd_\w+)", out))
    assert exported == set(names)   # nothing undeclared leaks out either


def test_library_is_sm100a():
    out = subprocess.run(["cuobjdump", "-lelf", L.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_abi_version_and_defaults():
    assert L.lmsgd_abi_version() == 1
    h = L.lmsgd_hyper_default()
    assert (h.mu1, h.mu2, h.eps, h.eta_rmsprop, h.beta_center, h.beta_period) == (0.9, 0.99, 1e-8, 3e-4, 10.0, 5.0)


def _bits(x):
    return struct.pack("<d", x)


def _f32(x):
    return struct.pack("<f", x)


@pytest.mark.parametrize("cfg", [
    dict(n_workers=1024, b_local=32, n_train=1_281_167, schedule="slow_start"),
    dict(n_workers=1024, b_local=32, n_train=1_281_167, schedule="goyal"),
    dict(n_workers=2, b_local=32, n_train=64, schedule="slow_start"),
    dict(n_workers=8, b_local=32, n_train=1_281_167, schedule="slow_start"),
    dict(n_workers=1000, b_local=7, n_train=999_983, schedule="slow_start"),
    dict(n_workers=1024, b_local=32, n_train=1_281_167, schedule="slow_start", transition="linear"),
    dict(n_workers=1024, b_local=32, n_train=1_281_167, schedule="slow_start", transition="sigmoid"),
    dict(n_workers=1024, b_local=32, n_train=1_281_167, schedule="goyal", transition="sudden"),
    dict(n_workers=2, b_local=32, n_train=64, schedule="slow_start", transition="sigmoid"),
    dict(n_workers=2, b_local=32, n_train=64, schedule="slow_start", transition="linear"),
])
def test_schedule_bit_exact_vs_oracle(cfg):
    ocl = sch.Cluster(**cfg)
    tr = {"elu": 0, "linear": 1, "sigmoid": 2, "sudden": 3}[cfg.get("transition", "elu")]
    ccl = L.make_cluster(cfg["n_workers"], cfg["b_local"], cfg["n_train"],
                         0 if cfg["schedule"] == "slow_start" else 1, tr)
    T = sch.n_steps(ocl)
    assert L.lmsgd_schedule_steps(ccl) == T
    step = max(1, T // 4000)
    ts = sorted(set(list(range(1, T + 1, step)) + [T, 1, 2]))
    for t in ts:
        o = sch.coeffs_at(t, sch.Hyper(), ocl)
        c = L.lmsgd_schedule_at(None, ccl, t)
        for f in ("epoch", "eta", "alpha_sgd", "alpha_rmsprop"):
            assert _bits(getattr(c, f)) == _bits(getattr(o, f)), (t, f, getattr(c, f), getattr(o, f))
            assert _f32(getattr(c, f)) == _f32(getattr(o, f))
        assert c.phase == o.phase
    with pytest.raises(L.LmsgdError) as e:
        L.lmsgd_schedule_at(None, ccl, T + 1)
    assert e.value.status == L.LMSGD_ERR_RANGE


def test_schedule_all_steps_32k_bit_exact():
    ocl = sch.Cluster()
    ccl = L.make_cluster()
    for t in range(1, 3520):
        o = sch.coeffs_at(t)
        c = L.lmsgd_schedule_at(None, ccl, t)
        assert (c.epoch, c.eta, c.alpha_sgd, c.alpha_rmsprop, c.phase) == \
               (o.epoch, o.eta, o.alpha_sgd, o.alpha_rmsprop, o.phase)


def test_schedule_custom_hyper():
    h = L.lmsgd_hyper_default()
    h.beta_center, h.beta_period, h.eta_rmsprop = 3.0, 2.0, 1e-3
    oh = sch.Hyper(beta_center=3.0, beta_period=2.0, eta_rmsprop=1e-3)
    cl = L.make_cluster(2, 32, 64)
    for t in range(1, 30):
        o = sch.coeffs_at(t, oh, sch.Cluster(2, 32, 64))
        c = L.lmsgd_schedule_at(h, cl, t)
        assert (c.alpha_sgd, c.alpha_rmsprop) == (o.alpha_sgd, o.alpha_rmsprop)


def test_schedule_arg_errors():
    cl = L.make_cluster()
    for bad_t in (0, -5):
        with pytest.raises(L.LmsgdError) as e:
            L.lmsgd_schedule_at(None, cl, bad_t)
        assert e.value.status == L.LMSGD_ERR_INVALID_ARG
    for bad in (L.make_cluster(0, 32), L.make_cluster(8, 0), L.make_cluster(8, 32, 0), L.make_cluster(schedule=7),
                L.make_cluster(transition=4), L.make_cluster(transition=-1)):
        with pytest.raises(L.LmsgdError):
            L.lmsgd_schedule_at(None, bad, 1)
    h = L.lmsgd_hyper_default()
    h.beta_period = 0.0
    with pytest.raises(L.LmsgdError):
        L.lmsgd_schedule_at(h, cl, 1)


@pytest.mark.parametrize("kw,err", [
    (dict(world=0, rank=0), L.LMSGD_ERR_UNSUPPORTED),
    (dict(world=9, rank=0), L.LMSGD_ERR_UNSUPPORTED),
    (dict(world=2, rank=2), L.LMSGD_ERR_INVALID_ARG),
    (dict(world=1, rank=0, n_params=0), L.LMSGD_ERR_INVALID_ARG),
    (dict(world=1, rank=0, loss_scale=3.0), L.LMSGD_ERR_INVALID_ARG),
    (dict(world=1, rank=0, loss_scale=0.0), L.LMSGD_ERR_INVALID_ARG),
    (dict(world=1, rank=0, flags=0x80), L.LMSGD_ERR_INVALID_ARG),
])
def test_init_rejects_bad_args_before_touching_cuda(kw, err):
    args = dict(world=1, rank=0, device=0, n_params=100, loss_scale=1.0, flags=0)
    args.update(kw)
    with pytest.raises(L.LmsgdError) as e:
        L.lmsgd_init(**args)
    assert e.value.status == err


def test_no_oracle_in_product_path():
    pkg = os.path.join(ROOT, "paper_1711_04325_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cpp", ".h", ".cuh")):
                src = open(os.path.join(dirpath, f)).read()
                assert not re.search(r"^\s*(import|from)\s+(oracle|synth)\b", src, re.M), f
                assert "oracle/" not in src and "oracle." not in src.replace("oracle.  ", ""), f


def test_no_undefined_library_symbols():
    out = subprocess.run(["nm", "-D", "--undefined-only", L.LIB_PATH], capture_output=True, text=True).stdout
    bad = [ln for ln in out.splitlines() if " U " in ln and "@" not in ln]   # weak (w) refs are fine
    assert not bad, bad


@pytest.mark.parametrize("n,world,b", [(1, 1, 1), (1000, 2, 64), (23_314, 1, 1000), (25_557_032, 4, 1 << 22),
                                       (25_557_032, 8, 2 << 20), (100, 8, 1 << 30), (513, 8, 512)])
def test_bucket_bounds_tile_the_buffer(n, world, b):
    """BucketedLMSGD's partition (host logic): the buckets tile [0, n) from its end, every
    boundary except n is a multiple of 64 * world (so the buckets' padded exchange outputs
    are disjoint slices of one R buffer), and no bucket is far from the requested size."""
    from paper_1711_04325_b200.optim import bucket_bounds
    bk = bucket_bounds(n, world, b)
    assert bk[0][1] == n and bk[-1][0] == 0
    assert all(a[0] == c[1] for a, c in zip(bk, bk[1:]))          # contiguous, descending
    assert all(lo % (64 * world) == 0 for lo, _ in bk)
    assert all(hi % (64 * world) == 0 for _, hi in bk[1:])
    unit = 64 * world
    for lo, hi in bk[:-1]:
        assert hi - lo >= min(b, n), (lo, hi)
        assert hi - lo < max(b, unit) + unit, (lo, hi)
    _, n_pad_top = L.lmsgd_layout(world, bk[0][1] - bk[0][0])
    assert bk[0][0] + n_pad_top >= n


def test_nvls_entry_points_without_a_gpu():
    """The NVLS calls are exported and fail soft on a machine without a GPU: the support
    query answers False (no driver entry points / no device) instead of raising, and the
    binding rejects a malformed handle before calling into the library."""
    assert L.lmsgd_nvls_supported(0) in (False, True)
    with pytest.raises(ValueError):
        L.lmsgd_nvls_connect(L.Context(None, 2, 0, 0, 10), b"short")
    # NULL context: an argument error, not a crash
    assert L.lib().lmsgd_nvls_create(None, ctypes.create_string_buffer(64)) == L.LMSGD_ERR_INVALID_ARG
    assert L.lib().lmsgd_nvls_bind(None, 1) == L.LMSGD_ERR_INVALID_ARG
    assert L.lib().lmsgd_nvls_mode(None, 1) == L.LMSGD_ERR_INVALID_ARG
    assert L.lib().lmsgd_status_accumulate(None, None, 0, None) == L.LMSGD_ERR_INVALID_ARG
    assert L.lib().lmsgd_set_exchange_blocks(None, 4) == L.LMSGD_ERR_INVALID_ARG
