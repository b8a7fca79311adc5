"""Thin ctypes binding of liblmsgd.so (include/lmsgd.h), same names as the C ABI.

Argument marshalling only: torch tensors are turned into device pointers and the
current CUDA stream into a cudaStream_t; every step of the path runs in the
library's sm_100a kernels.  There is no fallback: if liblmsgd.so is missing or
fails to load, importing this module raises.
"""
from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass

_PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_PKG, "liblmsgd.so")

LMSGD_OK = 0
LMSGD_ERR_INVALID_ARG = -1
LMSGD_ERR_CUDA = -2
LMSGD_ERR_NONFINITE = -4
LMSGD_ERR_STATE = -5
LMSGD_ERR_UNSUPPORTED = -6
LMSGD_ERR_TIMEOUT = -7
LMSGD_ERR_RANGE = -8
LMSGD_MAX_WORLD = 8
LMSGD_IPC_HANDLE_BYTES = 64
LMSGD_MAX_BN_CHANNELS = 1 << 20
LMSGD_FLAG_NO_SKIP = 0x1
LMSGD_FLAG_FREEZE_M = 0x2
LMSGD_NVLS_HANDLE_BYTES = 64
LMSGD_NVLS_OFF = 0
LMSGD_NVLS_RS = 1
LMSGD_NVLS_ALLREDUCE = 2
SCHEDULE_SLOW_START = 0
SCHEDULE_GOYAL = 1
TRANSITION_ELU, TRANSITION_LINEAR, TRANSITION_SIGMOID, TRANSITION_SUDDEN = 0, 1, 2, 3   # R20


class Hyper(ctypes.Structure):
    _fields_ = [("mu1", ctypes.c_double), ("mu2", ctypes.c_double), ("eps", ctypes.c_double),
                ("eta_rmsprop", ctypes.c_double), ("beta_center", ctypes.c_double),
                ("beta_period", ctypes.c_double)]


class Cluster(ctypes.Structure):
    _fields_ = [("n_workers", ctypes.c_int64), ("b_local", ctypes.c_int64), ("n_train", ctypes.c_int64),
                ("schedule", ctypes.c_int32), ("transition", ctypes.c_int32)]


class Coeffs(ctypes.Structure):
    _fields_ = [("epoch", ctypes.c_double), ("eta", ctypes.c_double), ("alpha_sgd", ctypes.c_double),
                ("alpha_rmsprop", ctypes.c_double), ("phase", ctypes.c_int32), ("reserved", ctypes.c_int32)]


class StepStatus(ctypes.Structure):
    _fields_ = [("first_nonfinite", ctypes.c_int64), ("pack_saturations", ctypes.c_int64),
                ("sum_saturations", ctypes.c_int64), ("skipped", ctypes.c_int32), ("error", ctypes.c_int32)]


class LmsgdError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"lmsgd status {status}: {msg}")
        self.status = status


def _load() -> ctypes.CDLL:
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} is missing: run `python -m paper_1711_04325_b200.build` "
                          "(there is no CPU fallback)")
    lib = ctypes.CDLL(LIB_PATH)
    P, I64, I32, F32, U32 = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int, ctypes.c_float, ctypes.c_uint32
    sig = {
        "lmsgd_abi_version": (I32, []),
        "lmsgd_status_string": (ctypes.c_char_p, [I32]),
        "lmsgd_hyper_default": (I32, [ctypes.POINTER(Hyper)]),
        "lmsgd_schedule_at": (I32, [ctypes.POINTER(Hyper), ctypes.POINTER(Cluster), I64, ctypes.POINTER(Coeffs)]),
        "lmsgd_schedule_steps": (I32, [ctypes.POINTER(Cluster), ctypes.POINTER(I64)]),
        "lmsgd_layout": (I32, [I32, I64, ctypes.POINTER(I64), ctypes.POINTER(I64)]),
        "lmsgd_init": (I32, [ctypes.POINTER(P), I32, I32, I32, I64, F32, ctypes.POINTER(Hyper), U32]),
        "lmsgd_ipc_handle": (I32, [P, ctypes.c_char_p]),
        "lmsgd_connect": (I32, [P, ctypes.c_char_p]),
        "lmsgd_nvls_supported": (I32, [I32, ctypes.POINTER(I32)]),
        "lmsgd_nvls_create": (I32, [P, ctypes.c_char_p]),
        "lmsgd_nvls_connect": (I32, [P, ctypes.c_char_p]),
        "lmsgd_nvls_bind": (I32, [P, I32]),
        "lmsgd_nvls_mode": (I32, [P, I32]),
        "lmsgd_status_accumulate": (I32, [P, P, I64, P]),
        "lmsgd_set_exchange_blocks": (I32, [P, I32]),
        "lmsgd_finalize": (I32, [P]),
        "lmsgd_last_error": (ctypes.c_char_p, [P]),
        "lmsgd_step": (I32, [P, P, P, P, P, P, ctypes.POINTER(Coeffs)]),
        "lmsgd_exchange": (I32, [P, P, P, P]),
        "lmsgd_step_out_of_place": (I32, [P, P, P, P, P, P, P, P, P, ctypes.POINTER(Coeffs)]),
        "lmsgd_step_host": (I32, [P, P, P, P, P, P, ctypes.POINTER(Coeffs), P, P]),
        "lmsgd_step_out_of_place_host": (I32, [P, P, P, P, P, P, P, P, P, ctypes.POINTER(Coeffs), P, P]),
        "lmsgd_bn_stats_allreduce": (I32, [P, P, P, P, I64]),
        "lmsgd_set_weight_decay": (I32, [P, ctypes.c_double, I64]),
        "lmsgd_schedule_upload": (I32, [P, ctypes.POINTER(Hyper), ctypes.POINTER(Cluster), I64, I64]),
        "lmsgd_step_graph": (I32, [P, P, P, P, P, P]),
        "lmsgd_query_status": (I32, [P, ctypes.POINTER(StepStatus)]),
        "lmsgd_profile_enable": (I32, [P, I64]),
        "lmsgd_profile_read": (I32, [P, ctypes.POINTER(ctypes.c_double), ctypes.POINTER(I64)]),
        "lmsgd_trace_enable": (I32, [P, I64]),
        "lmsgd_trace_read": (I32, [P, ctypes.POINTER(I64), I64, ctypes.POINTER(I64)]),
        "lmsgd_connect_group": (I32, [ctypes.POINTER(P), I32]),
        "lmsgd_step_group": (I32, [ctypes.POINTER(P), I32, P, ctypes.POINTER(P), ctypes.POINTER(P),
                                   ctypes.POINTER(P), ctypes.POINTER(P), ctypes.POINTER(Coeffs)]),
        "lmsgd_exchange_group": (I32, [ctypes.POINTER(P), I32, P, ctypes.POINTER(P), ctypes.POINTER(P)]),
        "lmsgd_step_graph_group": (I32, [ctypes.POINTER(P), I32, P, ctypes.POINTER(P), ctypes.POINTER(P),
                                         ctypes.POINTER(P), ctypes.POINTER(P)]),
        "lmsgd_bn_stats_allreduce_group": (I32, [ctypes.POINTER(P), I32, P, ctypes.POINTER(P), ctypes.POINTER(P),
                                                 I64]),
        "lmsgd_status_reset": (I32, [P, P]),
        "lmsgd_pack": (I32, [P, P, I64, I64, F32, P, P]),
        "lmsgd_reduce_local": (I32, [P, P, I32, I64, P, P]),
        "lmsgd_update": (I32, [P, P, I64, I32, F32, ctypes.POINTER(Hyper), ctypes.POINTER(Coeffs), P, P, P, P]),
        "lmsgd_fused_step1": (I32, [P, P, I64, F32, ctypes.POINTER(Hyper), ctypes.POINTER(Coeffs), P, P, P, P]),
    }
    for name, (res, args) in sig.items():
        f = getattr(lib, name)
        f.restype, f.argtypes = res, args
    return lib


_lib = _load()
EXPORTED = tuple(sorted(n for n in dir(_lib) if n.startswith("lmsgd_")))


def lib() -> ctypes.CDLL:
    return _lib


def _check(status: int, ctx=None):
    if status != LMSGD_OK:
        msg = _lib.lmsgd_last_error(ctx.ptr if isinstance(ctx, Context) else ctx)
        raise LmsgdError(status, (msg or b"").decode() or _lib.lmsgd_status_string(status).decode())


# ------------------------------------------------------------------ host-only

def lmsgd_abi_version() -> int:
    return _lib.lmsgd_abi_version()


def lmsgd_hyper_default() -> Hyper:
    h = Hyper()
    _check(_lib.lmsgd_hyper_default(ctypes.byref(h)))
    return h


def make_cluster(n_workers=1024, b_local=32, n_train=1_281_167, schedule=SCHEDULE_SLOW_START,
                 transition=TRANSITION_ELU) -> Cluster:
    return Cluster(n_workers, b_local, n_train, schedule, transition)


def lmsgd_schedule_at(hyper: Hyper | None, cluster: Cluster, t: int) -> Coeffs:
    hyper = hyper if hyper is not None else lmsgd_hyper_default()
    c = Coeffs()
    _check(_lib.lmsgd_schedule_at(ctypes.byref(hyper), ctypes.byref(cluster), int(t), ctypes.byref(c)))
    return c


def lmsgd_schedule_steps(cluster: Cluster) -> int:
    T = ctypes.c_int64()
    _check(_lib.lmsgd_schedule_steps(ctypes.byref(cluster), ctypes.byref(T)))
    return T.value


def lmsgd_layout(world: int, n: int) -> tuple[int, int]:
    """(shard, n_pad) of the exchange layout."""
    sh, npad = ctypes.c_int64(), ctypes.c_int64()
    _check(_lib.lmsgd_layout(int(world), int(n), ctypes.byref(sh), ctypes.byref(npad)))
    return sh.value, npad.value


def make_coeffs(eta: float, alpha_sgd: float, alpha_rmsprop: float, epoch: float = 0.0, phase: int = 0) -> Coeffs:
    return Coeffs(epoch, eta, alpha_sgd, alpha_rmsprop, phase, 0)


# ------------------------------------------------------------------ tensors

def _ptr(t, dtype=None, name="tensor"):
    import torch
    if not isinstance(t, torch.Tensor):
        raise TypeError(f"{name} must be a torch.Tensor")
    if not t.is_cuda:
        raise ValueError(f"{name} must be a CUDA tensor")
    if dtype is not None and t.dtype != dtype:
        raise TypeError(f"{name} must be {dtype}, got {t.dtype}")
    if not t.is_contiguous():
        raise ValueError(f"{name} must be contiguous")
    return ctypes.c_void_p(t.data_ptr())


def _stream(stream):
    import torch
    if stream is None:
        stream = torch.cuda.current_stream()
    return ctypes.c_void_p(stream.cuda_stream if hasattr(stream, "cuda_stream") else int(stream))


# ------------------------------------------------------------------ context

@dataclass
class Context:
    ptr: ctypes.c_void_p
    world: int
    rank: int
    device: int
    n: int

    def __del__(self):
        if self.ptr:
            try:
                _lib.lmsgd_finalize(self.ptr)
            except Exception:
                pass
            self.ptr = None


def lmsgd_init(world: int, rank: int, device: int, n_params: int, loss_scale: float = 1.0,
               hyper: Hyper | None = None, flags: int = 0) -> Context:
    p = ctypes.c_void_p()
    st = _lib.lmsgd_init(ctypes.byref(p), int(world), int(rank), int(device), int(n_params),
                         float(loss_scale), ctypes.byref(hyper) if hyper is not None else None, int(flags))
    _check(st)
    return Context(p, world, rank, device, n_params)


def lmsgd_ipc_handle(ctx: Context) -> bytes:
    buf = ctypes.create_string_buffer(LMSGD_IPC_HANDLE_BYTES)
    _check(_lib.lmsgd_ipc_handle(ctx.ptr, buf), ctx)
    return buf.raw


def lmsgd_connect(ctx: Context, handles: bytes):
    if len(handles) != ctx.world * LMSGD_IPC_HANDLE_BYTES:
        raise ValueError("handles must be world * LMSGD_IPC_HANDLE_BYTES bytes in rank order")
    _check(_lib.lmsgd_connect(ctx.ptr, handles), ctx)


def connect_process_group(ctx: Context, group=None):
    """Bootstrap plumbing: all-gather the IPC handles over torch.distributed and
    connect.  (The library itself does no host networking.)"""
    import torch.distributed as dist
    if ctx.world == 1:
        return
    mine = lmsgd_ipc_handle(ctx)
    out = [None] * ctx.world
    dist.all_gather_object(out, mine, group=group)
    lmsgd_connect(ctx, b"".join(out))
    dist.barrier(group=group)


def lmsgd_nvls_supported(device: int) -> bool:
    v = ctypes.c_int()
    _check(_lib.lmsgd_nvls_supported(int(device), ctypes.byref(v)))
    return bool(v.value)


def lmsgd_nvls_create(ctx: Context) -> bytes:
    buf = ctypes.create_string_buffer(LMSGD_NVLS_HANDLE_BYTES)
    _check(_lib.lmsgd_nvls_create(ctx.ptr, buf), ctx)
    return buf.raw


def lmsgd_nvls_connect(ctx: Context, handle: bytes):
    if len(handle) != LMSGD_NVLS_HANDLE_BYTES:
        raise ValueError("handle must be LMSGD_NVLS_HANDLE_BYTES bytes")
    _check(_lib.lmsgd_nvls_connect(ctx.ptr, handle), ctx)


def lmsgd_nvls_bind(ctx: Context, mode: int):
    _check(_lib.lmsgd_nvls_bind(ctx.ptr, int(mode)), ctx)


def lmsgd_nvls_mode(ctx: Context, mode: int):
    _check(_lib.lmsgd_nvls_mode(ctx.ptr, int(mode)), ctx)


def connect_nvls(ctx: Context, mode: int = None, group=None):
    """Bootstrap plumbing of the NVLS exchange (include/lmsgd.h "NVLS"): rank 0 creates
    the multicast object, its handle is broadcast over torch.distributed, every rank
    joins, a barrier, every rank binds its wire, a barrier.  Call after
    connect_process_group."""
    import torch.distributed as dist
    mode = LMSGD_NVLS_ALLREDUCE if mode is None else mode
    h = [lmsgd_nvls_create(ctx) if ctx.rank == 0 else None]
    dist.broadcast_object_list(h, src=dist.get_global_rank(group, 0) if group is not None else 0, group=group)
    lmsgd_nvls_connect(ctx, h[0])
    dist.barrier(group=group)
    lmsgd_nvls_bind(ctx, mode)
    dist.barrier(group=group)


def lmsgd_finalize(ctx: Context):
    if ctx.ptr:
        _check(_lib.lmsgd_finalize(ctx.ptr))
        ctx.ptr = None


def lmsgd_step(ctx: Context, params, grads, delta, m, coeffs: Coeffs, stream=None):
    import torch
    for t, nm in ((params, "params"), (grads, "grads"), (delta, "delta"), (m, "m")):
        if t.numel() != ctx.n:
            raise ValueError(f"{nm} must have n_params = {ctx.n} elements")
    _check(_lib.lmsgd_step(ctx.ptr, _stream(stream), _ptr(params, torch.float32, "params"),
                           _ptr(grads, torch.float32, "grads"), _ptr(delta, torch.float32, "delta"),
                           _ptr(m, torch.float32, "m"), ctypes.byref(coeffs)), ctx)


def lmsgd_step_out_of_place(ctx: Context, params_in, params_out, grads, delta_in, delta_out, m_in, m_out,
                            coeffs: Coeffs, stream=None):
    """world == 1: the guarded step in one pass, state read from *_in and written to *_out."""
    import torch
    ts = ((params_in, "params_in"), (params_out, "params_out"), (grads, "grads"), (delta_in, "delta_in"),
          (delta_out, "delta_out"), (m_in, "m_in"), (m_out, "m_out"))
    for t, nm in ts:
        if t.numel() != ctx.n:
            raise ValueError(f"{nm} must have n_params = {ctx.n} elements")
    _check(_lib.lmsgd_step_out_of_place(ctx.ptr, _stream(stream), *(_ptr(t, torch.float32, nm) for t, nm in ts),
                                        ctypes.byref(coeffs)), ctx)


def lmsgd_exchange(ctx: Context, grads, R_out, stream=None):
    """fp16 all-reduce alone (rows a2-a4): R_out [n_pad] (int16/uint16 tensor of
    binary16 bits) <- sat16(sum over ranks of sat16(s g)), identical on every rank."""
    import torch
    if grads.numel() != ctx.n:
        raise ValueError(f"grads must have n_params = {ctx.n} elements")
    _, n_pad = lmsgd_layout(ctx.world, ctx.n)
    if R_out.numel() != n_pad or R_out.element_size() != 2:
        raise ValueError(f"R_out must be a 2-byte tensor of n_pad = {n_pad} elements")
    _check(_lib.lmsgd_exchange(ctx.ptr, _stream(stream), _ptr(grads, torch.float32, "grads"),
                               _ptr(R_out, None, "R_out")), ctx)


def lmsgd_status_accumulate(ctx: Context, offset: int, dstatus, stream=None):
    import torch
    _check(_lib.lmsgd_status_accumulate(ctx.ptr, _stream(stream), int(offset), _ptr(dstatus, torch.int64, "dstatus")),
           ctx)


def lmsgd_set_exchange_blocks(ctx: Context, blocks: int):
    _check(_lib.lmsgd_set_exchange_blocks(ctx.ptr, int(blocks)), ctx)


def lmsgd_set_weight_decay(ctx: Context, lam: float, n_decay: int = -1):
    _check(_lib.lmsgd_set_weight_decay(ctx.ptr, float(lam), int(n_decay)), ctx)


def lmsgd_schedule_upload(ctx: Context, hyper: Hyper | None, cluster: Cluster, t_first: int, count: int):
    _check(_lib.lmsgd_schedule_upload(ctx.ptr, ctypes.byref(hyper) if hyper is not None else None,
                                      ctypes.byref(cluster), int(t_first), int(count)), ctx)


def lmsgd_step_graph(ctx: Context, params, grads, delta, m, stream=None):
    """Graph-capturable step (coefficients and step number on the device)."""
    import torch
    for t, nm in ((params, "params"), (grads, "grads"), (delta, "delta"), (m, "m")):
        if t.numel() != ctx.n:
            raise ValueError(f"{nm} must have n_params = {ctx.n} elements")
    _check(_lib.lmsgd_step_graph(ctx.ptr, _stream(stream), _ptr(params, torch.float32, "params"),
                                 _ptr(grads, torch.float32, "grads"), _ptr(delta, torch.float32, "delta"),
                                 _ptr(m, torch.float32, "m")), ctx)


def _host_buf(t, n, name):
    import torch
    if t is None:
        return None
    if t.is_cuda or t.dtype != torch.float32 or not t.is_contiguous() or t.numel() != n:
        raise ValueError(f"{name} must be a contiguous CPU float32 tensor of n_params elements")
    return ctypes.c_void_p(t.data_ptr())


def _status_buf(status_host):
    if status_host.is_cuda or status_host.numel() * status_host.element_size() < ctypes.sizeof(StepStatus):
        raise ValueError("status_host must be a CPU buffer of >= 32 bytes")
    return ctypes.c_void_p(status_host.data_ptr())


def lmsgd_step_host(ctx: Context, params, grads_host, delta, m, coeffs: Coeffs, status_host,
                    params_host=None, stream=None):
    """grads_host: CPU float32 tensor (pinned for full speed); status_host: a pinned
    CPU int64 tensor of 4 elements (lmsgd_step_status layout); params_host (optional):
    a pinned CPU float32 tensor that receives theta_t.  Both are filled when the stream
    passes this point."""
    import torch
    _check(_lib.lmsgd_step_host(ctx.ptr, _stream(stream), _ptr(params, torch.float32, "params"),
                                _host_buf(grads_host, ctx.n, "grads_host"), _ptr(delta, torch.float32, "delta"),
                                _ptr(m, torch.float32, "m"), ctypes.byref(coeffs),
                                _host_buf(params_host, ctx.n, "params_host"), _status_buf(status_host)), ctx)


def lmsgd_step_out_of_place_host(ctx: Context, params_in, params_out, grads_host, delta_in, delta_out, m_in, m_out,
                                 coeffs: Coeffs, status_host, params_host=None, stream=None):
    """lmsgd_step_out_of_place from a host gradient, theta_t (optional) and the status
    copied back to the host on the stream."""
    import torch
    ts = ((params_in, "params_in"), (params_out, "params_out"), (delta_in, "delta_in"), (delta_out, "delta_out"),
          (m_in, "m_in"), (m_out, "m_out"))
    for t, nm in ts:
        if t.numel() != ctx.n:
            raise ValueError(f"{nm} must have n_params = {ctx.n} elements")
    p = [_ptr(t, torch.float32, nm) for t, nm in ts]
    _check(_lib.lmsgd_step_out_of_place_host(ctx.ptr, _stream(stream), p[0], p[1],
                                             _host_buf(grads_host, ctx.n, "grads_host"), p[2], p[3], p[4], p[5],
                                             ctypes.byref(coeffs), _host_buf(params_host, ctx.n, "params_host"),
                                             _status_buf(status_host)), ctx)


def decode_status(buf) -> StepStatus:
    """StepStatus from a 4 x int64 host buffer written by lmsgd_step_host."""
    return StepStatus.from_buffer_copy(bytes(buf.numpy().tobytes()))


def lmsgd_bn_stats_allreduce(ctx: Context, mean, var, stream=None):
    import torch
    if mean.numel() != var.numel():
        raise ValueError("mean and var must have the same length")
    _check(_lib.lmsgd_bn_stats_allreduce(ctx.ptr, _stream(stream), _ptr(mean, torch.float32, "mean"),
                                         _ptr(var, torch.float32, "var"), mean.numel()), ctx)


def lmsgd_query_status(ctx: Context) -> tuple[int, StepStatus]:
    """(status code, StepStatus) of the last step; LMSGD_ERR_NONFINITE / TIMEOUT /
    RANGE (graph mode, table exhausted) are returned, not raised."""
    s = StepStatus()
    st = _lib.lmsgd_query_status(ctx.ptr, ctypes.byref(s))
    if st not in (LMSGD_OK, LMSGD_ERR_NONFINITE, LMSGD_ERR_TIMEOUT, LMSGD_ERR_RANGE) or (st != LMSGD_OK and s.error == 0):
        _check(st, ctx)
    return st, s


def lmsgd_profile_enable(ctx: Context, max_launches: int):
    _check(_lib.lmsgd_profile_enable(ctx.ptr, int(max_launches)), ctx)


PHASES = ("pack", "reduce", "update")


def lmsgd_profile_read(ctx: Context) -> dict:
    """{phase: (summed device ms, launches)} of the recorded step kernels."""
    ms = (ctypes.c_double * 3)()
    n = (ctypes.c_int64 * 3)()
    _check(_lib.lmsgd_profile_read(ctx.ptr, ms, n), ctx)
    return {PHASES[i]: (ms[i], n[i]) for i in range(3)}


# pack start, pack end, all ranks' packs observed (reduce_start), reduce kernel start
# (reduce_go), reduce end, all ranks' reduces observed (update_start), update kernel
# start (update_go), update end
TRACE_FIELDS = ("pack_start", "pack_end", "reduce_start", "reduce_go", "reduce_end",
                "update_start", "update_go", "update_end", "publish_end") + tuple(f"a_seen_{p}" for p in range(8))
TRACE_WORDS = len(TRACE_FIELDS)


def lmsgd_trace_enable(ctx: Context, max_steps: int):
    _check(_lib.lmsgd_trace_enable(ctx.ptr, int(max_steps)), ctx)


def lmsgd_trace_read(ctx: Context, max_steps: int):
    """List of per-step dicts {field: ns} (world > 1 steps only)."""
    buf = (ctypes.c_int64 * (TRACE_WORDS * max_steps))()
    got = ctypes.c_int64()
    _check(_lib.lmsgd_trace_read(ctx.ptr, buf, int(max_steps), ctypes.byref(got)), ctx)
    return [dict(zip(TRACE_FIELDS, buf[TRACE_WORDS * i:TRACE_WORDS * (i + 1)])) for i in range(got.value)]


# ------------------------------------------------------------------ emulated groups
# (include/lmsgd.h "emulated groups"): a world's ranks as contexts of this process on
# one GPU, each kernel launched once for all of them.

def _ptrs(items, fn):
    arr = (ctypes.c_void_p * len(items))()
    for i, x in enumerate(items):
        arr[i] = fn(x).value if x is not None else None
    return arr


def _ctxs(ctxs):
    return _ptrs(ctxs, lambda c: c.ptr)


def lmsgd_connect_group(ctxs):
    _check(_lib.lmsgd_connect_group(_ctxs(ctxs), len(ctxs)), ctxs[0])


def lmsgd_step_group(ctxs, params, grads, delta, m, coeffs: Coeffs, stream=None):
    import torch
    f = lambda nm: (lambda t: _ptr(t, torch.float32, nm))  # noqa: E731
    for c, ts in zip(ctxs, zip(params, grads, delta, m)):
        if any(t.numel() != c.n for t in ts):
            raise ValueError(f"every buffer must have n_params = {c.n} elements")
    _check(_lib.lmsgd_step_group(_ctxs(ctxs), len(ctxs), _stream(stream), _ptrs(params, f("params")),
                                 _ptrs(grads, f("grads")), _ptrs(delta, f("delta")), _ptrs(m, f("m")),
                                 ctypes.byref(coeffs)), ctxs[0])


def lmsgd_exchange_group(ctxs, grads, R_out, stream=None):
    import torch
    _, n_pad = lmsgd_layout(ctxs[0].world, ctxs[0].n)
    for c, g, r in zip(ctxs, grads, R_out):
        if g.numel() != c.n or r.numel() != n_pad or r.element_size() != 2:
            raise ValueError(f"grads [n_params] fp32, R_out [n_pad = {n_pad}] 2-byte tensors")
    _check(_lib.lmsgd_exchange_group(_ctxs(ctxs), len(ctxs), _stream(stream),
                                     _ptrs(grads, lambda t: _ptr(t, torch.float32, "grads")),
                                     _ptrs(R_out, lambda t: _ptr(t, None, "R_out"))), ctxs[0])


def lmsgd_step_graph_group(ctxs, params, grads, delta, m, stream=None):
    import torch
    f = lambda nm: (lambda t: _ptr(t, torch.float32, nm))  # noqa: E731
    _check(_lib.lmsgd_step_graph_group(_ctxs(ctxs), len(ctxs), _stream(stream), _ptrs(params, f("params")),
                                       _ptrs(grads, f("grads")), _ptrs(delta, f("delta")), _ptrs(m, f("m"))),
           ctxs[0])


def lmsgd_bn_stats_allreduce_group(ctxs, mean, var, stream=None):
    import torch
    C = mean[0].numel()
    if any(t.numel() != C for t in list(mean) + list(var)):
        raise ValueError("every mean / var must have the same length")
    f = lambda nm: (lambda t: _ptr(t, torch.float32, nm))  # noqa: E731
    _check(_lib.lmsgd_bn_stats_allreduce_group(_ctxs(ctxs), len(ctxs), _stream(stream), _ptrs(mean, f("mean")),
                                               _ptrs(var, f("var")), C), ctxs[0])


# ------------------------------------------------------------------ sub-steps

def lmsgd_status_reset(dstatus, stream=None):
    import torch
    _check(_lib.lmsgd_status_reset(_stream(stream), _ptr(dstatus, torch.int64, "dstatus")))


def lmsgd_pack(g, n_pad: int, loss_scale: float, h, dstatus, stream=None):
    import torch
    _check(_lib.lmsgd_pack(_stream(stream), _ptr(g, torch.float32, "g"), g.numel(), int(n_pad),
                           float(loss_scale), _ptr(h, None, "h"), _ptr(dstatus, torch.int64, "dstatus")))


def lmsgd_reduce_local(h, k: int, n_pad: int, R, dstatus=None, stream=None):
    import torch
    _check(_lib.lmsgd_reduce_local(_stream(stream), _ptr(h, None, "h"), int(k), int(n_pad), _ptr(R, None, "R"),
                                   _ptr(dstatus, torch.int64, "dstatus") if dstatus is not None else None))


def lmsgd_update(R, n: int, k: int, loss_scale: float, hyper, coeffs: Coeffs, params, delta, m,
                 dstatus=None, stream=None):
    import torch
    hyper = hyper if hyper is not None else lmsgd_hyper_default()
    _check(_lib.lmsgd_update(_stream(stream), _ptr(R, None, "R"), int(n), int(k), float(loss_scale),
                             ctypes.byref(hyper), ctypes.byref(coeffs), _ptr(params, torch.float32, "params"),
                             _ptr(delta, torch.float32, "delta"), _ptr(m, torch.float32, "m"),
                             _ptr(dstatus, torch.int64, "dstatus") if dstatus is not None else None))


def lmsgd_fused_step1(g, loss_scale: float, hyper, coeffs: Coeffs, params, delta, m, dstatus, stream=None):
    import torch
    hyper = hyper if hyper is not None else lmsgd_hyper_default()
    _check(_lib.lmsgd_fused_step1(_stream(stream), _ptr(g, torch.float32, "g"), g.numel(), float(loss_scale),
                                  ctypes.byref(hyper), ctypes.byref(coeffs), _ptr(params, torch.float32, "params"),
                                  _ptr(delta, torch.float32, "delta"), _ptr(m, torch.float32, "m"),
                                  _ptr(dstatus, torch.int64, "dstatus")))
