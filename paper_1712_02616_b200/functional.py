"""Torch-facing wrappers of the C ABI (argument marshalling only).

Every step of the hot path runs in libiabn.so's CUDA kernels; this module only
turns torch tensors into (pointer, desc, stream) triples, caches the scratch
workspace, and raises on a non-OK status.  Tensors are contiguous CUDA
tensors: layout "NCHW" means shape [N, C, *spatial], layout "NHWC" means
[N, *spatial, C] in memory (a 4-D channels_last tensor qualifies, see
``layout_of``).  Per-channel vectors are fp32 [C].

Paper: arXiv 1712.02616 -- Alg. 1 forward (:204-214), Alg. 2
variant I backward (:215-223), in-place buffers (:200), InPlace-ABN^sync (:315).
"""
from __future__ import annotations

import ctypes
from dataclasses import dataclass

import torch

from . import _lib as L

_DTYPES = {torch.float32: L.F32, torch.bfloat16: L.BF16}
_GAMMA = {"abs_eps": 0, "plain": L.GAMMA_PLAIN, "fixed_one": L.GAMMA_FIXED_ONE}
_LAYOUT = {"NCHW": L.NCHW, "NHWC": L.NHWC}


def layout_of(x: torch.Tensor) -> tuple[str, torch.Tensor]:
    """(layout, storage-order view) of a 4-D tensor: NCHW-contiguous or channels_last."""
    if x.is_contiguous():
        return "NCHW", x
    if x.dim() == 4 and x.is_contiguous(memory_format=torch.channels_last):
        return "NHWC", x.permute(0, 2, 3, 1)
    raise ValueError("tensor must be contiguous (NCHW) or channels_last (NHWC)")


def _geom(x: torch.Tensor, layout: str) -> tuple[int, int, int]:
    if not x.is_cuda:
        raise ValueError("InPlace-ABN tensors must be CUDA tensors (there is no CPU path)")
    if not x.is_contiguous():
        raise ValueError("activation tensors must be contiguous in the given layout")
    if x.dtype not in _DTYPES:
        raise ValueError(f"unsupported dtype {x.dtype} (float32 or bfloat16)")
    if x.dim() < 2:
        raise ValueError("need at least [N, C]")
    n = x.shape[0]
    c = x.shape[1] if layout == "NCHW" else x.shape[-1]
    hw = x.numel() // max(n * c, 1) if n * c > 0 else 0
    return n, c, hw


_DESCS: dict[tuple, L.Desc] = {}


def _desc(x: torch.Tensor, layout: str) -> L.Desc:
    """Descriptor of x, cached per (shape, dtype, layout): a layer calls with the same
    shape every step, and building the ctypes struct is part of the per-call host cost."""
    key = (x.shape, x.dtype, layout, x.is_cuda)
    d = _DESCS.get(key)
    if d is not None and x.is_contiguous():
        return d
    n, c, hw = _geom(x, layout)
    d = L.desc(n, c, hw, _DTYPES[x.dtype], _LAYOUT[layout])
    if len(_DESCS) < 4096:
        _DESCS[key] = d
    return d


_WS: dict[tuple, torch.Tensor] = {}
_WSB: dict[tuple, int] = {}  # workspace bytes per geometry (pure function of the desc)


def workspace(d: L.Desc, device: torch.device, stream=None) -> tuple[int, int]:
    """Scratch space of the call: one buffer per (device, stream), grown on demand.
    Calls on one stream are ordered, so they may share it; calls on different
    streams get different buffers (the library's calls are stream-ordered only)."""
    dk = (d.n, d.c, d.hw, d.dtype, d.layout)
    nbytes = _WSB.get(dk)
    if nbytes is None:
        nbytes = _WSB[dk] = max(L.workspace_bytes(d), 16)
    key = (device.index, _stream(stream, device))
    ws = _WS.get(key)
    if ws is None or ws.numel() < nbytes:
        if stream is None:
            ws = torch.empty(nbytes, dtype=torch.uint8, device=device)
        else:
            # allocated from the explicit stream's pool: when it is later replaced, the
            # caching allocator reuses it only after the work queued on that stream
            with torch.cuda.stream(stream):
                ws = torch.empty(nbytes, dtype=torch.uint8, device=device)
        _WS[key] = ws
    return ws.data_ptr(), ws.numel()


def _empty_c(C: int, device: torch.device, stream) -> torch.Tensor:
    """A per-channel fp32 output, allocated on the stream the kernels write it from."""
    if stream is None:
        return torch.empty(C, dtype=torch.float32, device=device)
    with torch.cuda.stream(stream):
        return torch.empty(C, dtype=torch.float32, device=device)


def _ptr(t: torch.Tensor | None) -> int | None:
    return None if t is None else t.data_ptr()


def _f32(t: torch.Tensor | None, C: int, name: str) -> torch.Tensor | None:
    if t is None:
        return None
    if t.dtype != torch.float32 or t.numel() != C or not t.is_contiguous() or not t.is_cuda:
        raise ValueError(f"{name} must be a contiguous CUDA float32 tensor of {C} elements")
    return t


_RAW_STREAM = getattr(torch._C, "_cuda_getCurrentRawStream", None)
_CUR_DEV = getattr(torch._C, "_cuda_getDevice", None)


def _stream(stream, device: torch.device | None = None) -> int:
    """The CUDA stream handle of a call: the explicit one, else the current stream of the
    tensors' device (not of the current device)."""
    if stream is not None:
        return stream.cuda_stream
    idx = device.index if device is not None and device.index is not None else None
    if _RAW_STREAM is not None:  # same value, without building a Stream object
        return _RAW_STREAM(idx if idx is not None else _CUR_DEV())
    return torch.cuda.current_stream(idx).cuda_stream


def _flags(gamma_mode: str, running_var_biased: bool = False, extra: int = 0) -> int:
    return _GAMMA[gamma_mode] | (L.RUNNING_VAR_BIASED if running_var_biased else 0) | extra


# f after BN; sigmoid / tanh: fp32, iabn_forward / iabn_backward only
ACTIVATIONS = {"leaky_relu": 0, "sigmoid": L.ACT_SIGMOID, "tanh": L.ACT_TANH}


def _act(activation: str) -> int:
    if activation not in ACTIVATIONS:
        raise ValueError(f"activation must be one of {sorted(ACTIVATIONS)}, got {activation!r}")
    return ACTIVATIONS[activation]


def broadcast_unique_id(group, make_id) -> bytes:
    """Rank 0 of `group` calls make_id(); every rank returns rank 0's 128 bytes."""
    import torch.distributed as dist
    rank = dist.get_rank(group)
    obj = [make_id() if rank == 0 else None]
    src = dist.get_global_rank(group, 0) if group is not None else 0
    dist.broadcast_object_list(obj, src=src, group=group)
    uid = obj[0]
    if not isinstance(uid, (bytes, bytearray)) or len(uid) != 128:
        raise RuntimeError("bad communicator id")
    return bytes(uid)


@dataclass
class Comm:
    """NCCL communicator of the synchronized variant (iabn_comm)."""
    handle: ctypes.c_void_p
    nranks: int
    rank: int

    @classmethod
    def create(cls, nranks: int, rank: int, uid: bytes) -> "Comm":
        h = ctypes.c_void_p()
        L.call("iabn_comm_init", ctypes.byref(h), nranks, rank, uid)
        return cls(h, nranks, rank)

    @staticmethod
    def unique_id() -> bytes:
        buf = ctypes.create_string_buffer(128)
        L.call("iabn_comm_get_unique_id", buf)
        return buf.raw

    @classmethod
    def from_process_group(cls, group=None) -> "Comm":
        """Rank 0 draws the NCCL id; torch.distributed broadcasts it (plumbing)."""
        import torch.distributed as dist
        uid = broadcast_unique_id(group, cls.unique_id)
        return cls.create(dist.get_world_size(group), dist.get_rank(group), uid)

    def set_timing(self, on: bool = True) -> None:
        """Record per-phase CUDA events in the synchronized calls (iabn_comm_set_timing)."""
        L.call("iabn_comm_set_timing", self.handle, 1 if on else 0)

    def phase_ms(self) -> dict:
        """Device time of the last timed forward / backward, per phase (iabn_comm_phase_ms):
        {"forward": {"reduce", "allreduce", "apply"}, "backward": {...}} in ms."""
        buf = (ctypes.c_float * 6)()
        L.call("iabn_comm_phase_ms", self.handle, buf)
        names = ("reduce", "allreduce", "apply")
        return {p: {n: float(buf[3 * i + k]) for k, n in enumerate(names)}
                for i, p in enumerate(("forward", "backward"))}

    def close(self) -> None:
        if self.handle:
            L.call("iabn_comm_destroy", self.handle)
            self.handle = ctypes.c_void_p()


def forward(x: torch.Tensor, gamma: torch.Tensor, beta: torch.Tensor,
            running_mean: torch.Tensor | None = None, running_var: torch.Tensor | None = None, *,
            momentum: float = 0.1, eps: float = 1e-5, slope: float = 0.01,
            out: torch.Tensor | None = None, training: bool = True, gamma_mode: str = "abs_eps",
            running_var_biased: bool = False, layout: str = "NCHW", flags: int = 0,
            comm: Comm | None = None, stream=None, activation: str = "leaky_relu"):
    """Alg. 1: z = f(BN_{gamma,beta}(x)), written over x unless ``out`` is given; f is
    leaky ReLU with ``slope`` (default), sigmoid or tanh (``activation``).
    Returns (z, save_mean, save_var); in eval mode save_* are None."""
    d = _desc(x, layout)
    C = d.c
    z = x if out is None else out
    if z.shape != x.shape or z.dtype != x.dtype or not z.is_contiguous():
        raise ValueError("out must match x in shape, dtype and contiguity")
    gamma, beta = _f32(gamma, C, "gamma"), _f32(beta, C, "beta")
    running_mean = _f32(running_mean, C, "running_mean")
    running_var = _f32(running_var, C, "running_var")
    fl = _flags(gamma_mode, running_var_biased, flags | _act(activation)) | \
        (0 if training else L.EVAL)
    if training:
        save_mean = _empty_c(C, x.device, stream)
        save_var = _empty_c(C, x.device, stream)
    else:
        save_mean = save_var = None
    ws, nb = workspace(d, x.device, stream)
    args = [ctypes.byref(d), x.data_ptr(), z.data_ptr(), gamma.data_ptr(), beta.data_ptr(),
            _ptr(running_mean), _ptr(running_var), _ptr(save_mean), _ptr(save_var), momentum, eps,
            slope, fl, ws, nb, _stream(stream, x.device)]
    if comm is None:
        L.call("iabn_forward", *args)
    else:
        L.call("iabn_forward_sync", *args, comm.handle)
    return z, save_mean, save_var


def backward(z: torch.Tensor, dz: torch.Tensor, gamma: torch.Tensor, beta: torch.Tensor,
             save_var: torch.Tensor, *, save_mean: torch.Tensor | None = None, eps: float = 1e-5,
             slope: float = 0.01, dx: torch.Tensor | None = None, gamma_mode: str = "abs_eps",
             layout: str = "NCHW", flags: int = 0, comm: Comm | None = None,
             global_param_grads: bool = False, stream=None, activation: str = "leaky_relu"):
    """Alg. 2: from z and dL/dz only (variant II / BN-dagger in the channel-resident
    kernels, I in the streaming ones and with IABN_VARIANT_I; R6).  dx is
    written over dz unless ``dx`` is given.  Returns (dx, dgamma, dbeta)."""
    d = _desc(z, layout)
    C = d.c
    if dz.shape != z.shape or dz.dtype != z.dtype or not dz.is_contiguous():
        raise ValueError("dz must match z in shape, dtype and contiguity")
    dx = dz if dx is None else dx
    gamma, beta = _f32(gamma, C, "gamma"), _f32(beta, C, "beta")
    save_var = _f32(save_var, C, "save_var")
    dgamma = _empty_c(C, z.device, stream)
    dbeta = _empty_c(C, z.device, stream)
    fl = _flags(gamma_mode, False, flags | _act(activation)) | \
        (L.SYNC_GLOBAL_PARAM_GRADS if global_param_grads else 0)
    ws, nb = workspace(d, z.device, stream)
    args = [ctypes.byref(d), z.data_ptr(), dz.data_ptr(), dx.data_ptr(), gamma.data_ptr(),
            beta.data_ptr(), _ptr(save_mean), save_var.data_ptr(), dgamma.data_ptr(),
            dbeta.data_ptr(), eps, slope, fl, ws, nb, _stream(stream, z.device)]
    if comm is None:
        L.call("iabn_backward", *args)
    else:
        L.call("iabn_backward_sync", *args, comm.handle)
    return dx, dgamma, dbeta


# ---------------------------------------------------------------- fused-collective sync, one GPU
def forward_sync_emulated(x: torch.Tensor, nranks: int, gamma: torch.Tensor, beta: torch.Tensor,
                          running_mean: torch.Tensor | None = None,
                          running_var: torch.Tensor | None = None, *, momentum: float = 0.1,
                          eps: float = 1e-5, slope: float = 0.01, out: torch.Tensor | None = None,
                          gamma_mode: str = "abs_eps", running_var_biased: bool = False,
                          flags: int = 0, stream=None):
    """InPlace-ABN^sync over ``nranks`` equal shards of ``x`` (along N), emulated on one
    GPU by the fused-collective kernel (include/iabn.h, iabn_forward_sync_emulated).
    Returns (z, save_mean, save_var) with global statistics."""
    if x.dim() < 2 or x.shape[0] % nranks:
        raise ValueError("x.shape[0] must be a multiple of nranks")
    d = _desc(x, "NCHW")
    C = d.c
    shard = L.Desc(d.n // nranks, d.c, d.hw, d.dtype, d.layout)
    z = x if out is None else out
    if z.shape != x.shape or z.dtype != x.dtype or not z.is_contiguous():
        raise ValueError("out must match x in shape, dtype and contiguity")
    gamma, beta = _f32(gamma, C, "gamma"), _f32(beta, C, "beta")
    running_mean = _f32(running_mean, C, "running_mean")
    running_var = _f32(running_var, C, "running_var")
    save_mean = torch.empty(C, dtype=torch.float32, device=x.device)
    save_var = torch.empty(C, dtype=torch.float32, device=x.device)
    ws, nb = workspace(d, x.device, stream)
    L.call("iabn_forward_sync_emulated", ctypes.byref(shard), nranks, x.data_ptr(), z.data_ptr(),
           gamma.data_ptr(), beta.data_ptr(), _ptr(running_mean), _ptr(running_var),
           save_mean.data_ptr(), save_var.data_ptr(), momentum, eps, slope,
           _flags(gamma_mode, running_var_biased, flags), ws, nb, _stream(stream, x.device))
    return z, save_mean, save_var


def backward_sync_emulated(z: torch.Tensor, dz: torch.Tensor, nranks: int, gamma: torch.Tensor,
                           beta: torch.Tensor, save_var: torch.Tensor, *, eps: float = 1e-5,
                           slope: float = 0.01, dx: torch.Tensor | None = None,
                           gamma_mode: str = "abs_eps", flags: int = 0,
                           global_param_grads: bool = False, stream=None):
    """Backward of :func:`forward_sync_emulated`.  Returns (dx, dgamma, dbeta) with
    dgamma/dbeta of shape [nranks, C] (row r = shard r's contribution)."""
    if z.dim() < 2 or z.shape[0] % nranks:
        raise ValueError("z.shape[0] must be a multiple of nranks")
    if dz.shape != z.shape or dz.dtype != z.dtype or not dz.is_contiguous():
        raise ValueError("dz must match z in shape, dtype and contiguity")
    d = _desc(z, "NCHW")
    C = d.c
    shard = L.Desc(d.n // nranks, d.c, d.hw, d.dtype, d.layout)
    dx = dz if dx is None else dx
    dgamma = torch.empty(nranks, C, dtype=torch.float32, device=z.device)
    dbeta = torch.empty(nranks, C, dtype=torch.float32, device=z.device)
    fl = _flags(gamma_mode, False, flags) | (L.SYNC_GLOBAL_PARAM_GRADS if global_param_grads else 0)
    ws, nb = workspace(d, z.device, stream)
    L.call("iabn_backward_sync_emulated", ctypes.byref(shard), nranks, z.data_ptr(), dz.data_ptr(),
           dx.data_ptr(), _f32(gamma, C, "gamma").data_ptr(), _f32(beta, C, "beta").data_ptr(),
           None, _f32(save_var, C, "save_var").data_ptr(), dgamma.data_ptr(), dbeta.data_ptr(),
           eps, slope, fl, ws, nb, _stream(stream, z.device))
    return dx, dgamma, dbeta


# ---------------------------------------------------------------- split phase
def forward_reduce(x: torch.Tensor, *, layout: str = "NCHW", stream=None) -> torch.Tensor:
    """Local raw moments, fp64 [C, 3] = (count, sum, sum of squares)."""
    d = _desc(x, layout)
    stats = torch.empty(d.c, 3, dtype=torch.float64, device=x.device)
    ws, nb = workspace(d, x.device, stream)
    L.call("iabn_forward_reduce", ctypes.byref(d), x.data_ptr(), stats.data_ptr(), ws, nb,
           _stream(stream, x.device))
    return stats


def forward_apply(x: torch.Tensor, stats_global: torch.Tensor, gamma, beta, running_mean=None,
                  running_var=None, *, momentum=0.1, eps=1e-5, slope=0.01, out=None,
                  gamma_mode="abs_eps", running_var_biased=False, layout="NCHW", flags=0,
                  stream=None):
    d = _desc(x, layout)
    C = d.c
    z = x if out is None else out
    save_mean = torch.empty(C, dtype=torch.float32, device=x.device)
    save_var = torch.empty(C, dtype=torch.float32, device=x.device)
    ws, nb = workspace(d, x.device, stream)
    assert stats_global.dtype == torch.float64 and stats_global.numel() == 3 * C
    L.call("iabn_forward_apply", ctypes.byref(d), x.data_ptr(), z.data_ptr(),
           stats_global.data_ptr(), _f32(gamma, C, "gamma").data_ptr(),
           _f32(beta, C, "beta").data_ptr(), _ptr(_f32(running_mean, C, "running_mean")),
           _ptr(_f32(running_var, C, "running_var")), save_mean.data_ptr(), save_var.data_ptr(),
           momentum, eps, slope, _flags(gamma_mode, running_var_biased, flags), ws, nb,
           _stream(stream, x.device))
    return z, save_mean, save_var


def backward_reduce(z, dz, gamma, beta, *, eps=1e-5, slope=0.01, gamma_mode="abs_eps",
                    layout="NCHW", flags=0, stream=None) -> torch.Tensor:
    """Local gradient sums, fp64 [2C + 1] = ([C][2] (sum dy, sum dy x^), count)."""
    d = _desc(z, layout)
    C = d.c
    sums = torch.empty(2 * C + 1, dtype=torch.float64, device=z.device)
    ws, nb = workspace(d, z.device, stream)
    L.call("iabn_backward_reduce", ctypes.byref(d), z.data_ptr(), dz.data_ptr(),
           _f32(gamma, C, "gamma").data_ptr(), _f32(beta, C, "beta").data_ptr(), sums.data_ptr(),
           eps, slope, _flags(gamma_mode, False, flags), ws, nb, _stream(stream, z.device))
    return sums


def backward_apply(z, dz, sums_global, sums_local, gamma, beta, save_var, *, eps=1e-5,
                   slope=0.01, dx=None, gamma_mode="abs_eps", layout="NCHW", flags=0,
                   global_param_grads=False, stream=None):
    d = _desc(z, layout)
    C = d.c
    dx = dz if dx is None else dx
    dgamma = torch.empty(C, dtype=torch.float32, device=z.device)
    dbeta = torch.empty(C, dtype=torch.float32, device=z.device)
    ws, nb = workspace(d, z.device, stream)
    fl = _flags(gamma_mode, False, flags) | (L.SYNC_GLOBAL_PARAM_GRADS if global_param_grads else 0)
    L.call("iabn_backward_apply", ctypes.byref(d), z.data_ptr(), dz.data_ptr(), dx.data_ptr(),
           sums_global.data_ptr(), _ptr(sums_local), _f32(gamma, C, "gamma").data_ptr(),
           _f32(beta, C, "beta").data_ptr(), _f32(save_var, C, "save_var").data_ptr(),
           dgamma.data_ptr(), dbeta.data_ptr(), eps, slope, fl, ws, nb, _stream(stream, z.device))
    return dx, dgamma, dbeta


def fold_conv(weight: torch.Tensor, bias: torch.Tensor | None, running_mean: torch.Tensor,
              running_var: torch.Tensor, gamma: torch.Tensor, beta: torch.Tensor, *,
              eps: float = 1e-5, gamma_mode: str = "abs_eps", inplace: bool = False,
              stream=None) -> tuple[torch.Tensor, torch.Tensor]:
    """Test-time BN of a conv's output channels absorbed into the conv (PAPER.md:85,
    iabn_fold_conv): returns (weight', bias') with conv(x; weight', bias') =
    BN_eval(conv(x; weight, bias)).  weight: contiguous CUDA float32 [cout, ...]."""
    if weight.dtype != torch.float32 or not weight.is_cuda or not weight.is_contiguous():
        raise ValueError("weight must be a contiguous CUDA float32 tensor")
    cout = weight.shape[0]
    kper = weight.numel() // cout
    for name, t in (("running_mean", running_mean), ("running_var", running_var),
                    ("gamma", gamma), ("beta", beta), ("bias", bias)):
        _f32(t, cout, name)
    w_out = weight if inplace else torch.empty_like(weight)
    b_out = bias if (inplace and bias is not None) else torch.empty(cout, dtype=torch.float32,
                                                                    device=weight.device)
    L.call("iabn_fold_conv", cout, kper, _ptr(weight), _ptr(bias), _ptr(running_mean),
           _ptr(running_var), _ptr(gamma), _ptr(beta), eps, _flags(gamma_mode), _ptr(w_out),
           _ptr(b_out), _stream(stream, weight.device))
    return w_out, b_out


def schedule(x_shape_desc: L.Desc, pass_: int, flags: int = 0) -> tuple[str, int]:
    s, k = L.query_schedule(x_shape_desc, pass_, flags)
    return ("fused" if s == 1 else "streaming"), k


# ---------------------------------------------------------------- autograd
class InPlaceABNFunction(torch.autograd.Function):
    """z = InPlace-ABN(x); x's storage is reused for z (mark_dirty), and the
    backward reads only z and sigma_B (Alg. 1 l.3)."""

    @staticmethod
    def forward(ctx, x, gamma, beta, running_mean, running_var, momentum, eps, slope, training,
                gamma_mode, layout, comm, grad_inplace=True, activation="leaky_relu"):
        z, _, save_var = forward(x, gamma.detach(), beta.detach(), running_mean, running_var,
                                 momentum=momentum, eps=eps, slope=slope, training=training,
                                 gamma_mode=gamma_mode, layout=layout, comm=comm,
                                 activation=activation)
        ctx.mark_dirty(x)
        ctx.save_for_backward(z, gamma, beta, save_var)
        ctx.cfg = (eps, slope, gamma_mode, layout, comm, training, grad_inplace, activation)
        return z

    @staticmethod
    def backward(ctx, dz):
        z, gamma, beta, save_var = ctx.saved_tensors
        eps, slope, gamma_mode, layout, comm, training, grad_inplace, activation = ctx.cfg
        if not training:
            raise RuntimeError("backward through eval-mode InPlace-ABN is not supported")
        dz = dz.contiguous()
        # gradient sharing: dL/dx is written over dL/dz unless disabled
        dx, dgamma, dbeta = backward(z, dz, gamma.detach(), beta.detach(), save_var, eps=eps,
                                     slope=slope, dx=None if grad_inplace else torch.empty_like(dz),
                                     gamma_mode=gamma_mode, layout=layout, comm=comm,
                                     activation=activation)
        return (dx, dgamma, dbeta, None, None, None, None, None, None, None, None, None, None,
                None)


def inplace_abn(x, gamma, beta, running_mean=None, running_var=None, *, momentum=0.1, eps=1e-5,
                slope=0.01, training=True, gamma_mode="abs_eps", layout="NCHW", comm=None,
                grad_inplace=True, activation="leaky_relu"):
    """Autograd entry: z written over x (mark_dirty) and, with ``grad_inplace`` (default,
    the paper's gradient sharing), dL/dx written over the incoming dL/dz.
    The incoming gradient buffer is then consumed: pass ``grad_inplace=False`` if a
    caller keeps its own reference to the gradient it feeds in (e.g. z.backward(g) with
    a g it reuses)."""
    return InPlaceABNFunction.apply(x, gamma, beta, running_mean, running_var, momentum, eps,
                                    slope, training, gamma_mode, layout, comm, grad_inplace,
                                    activation)


class InPlaceABN(torch.nn.Module):
    """The plug-in BN+LeakyReLU layer of PAPER.md:200 (fp32 gamma/beta, running stats);
    ``activation`` = "sigmoid" / "tanh" for the other invertible activations of
    PAPER.md:142 (fp32 activations, no comm)."""

    def __init__(self, num_features: int, *, eps=1e-5, momentum=0.1, slope=0.01,
                 gamma_mode="abs_eps", comm: Comm | None = None, device=None,
                 grad_inplace: bool = True, activation: str = "leaky_relu"):
        super().__init__()
        _act(activation)
        self.activation = activation
        self.grad_inplace = grad_inplace
        self.weight = torch.nn.Parameter(torch.ones(num_features, device=device))
        self.bias = torch.nn.Parameter(torch.zeros(num_features, device=device))
        self.register_buffer("running_mean", torch.zeros(num_features, device=device))
        self.register_buffer("running_var", torch.ones(num_features, device=device))
        self.eps, self.momentum, self.slope, self.gamma_mode, self.comm = (eps, momentum, slope,
                                                                           gamma_mode, comm)

    def forward(self, x):
        layout, _ = layout_of(x)
        xs = x if layout == "NCHW" else x.permute(0, 2, 3, 1)
        z = inplace_abn(xs, self.weight, self.bias, self.running_mean, self.running_var,
                        momentum=self.momentum, eps=self.eps, slope=self.slope,
                        training=self.training, gamma_mode=self.gamma_mode, layout=layout,
                        comm=self.comm, grad_inplace=self.grad_inplace,
                        activation=self.activation)
        return z if layout == "NCHW" else z.permute(0, 3, 1, 2)
