"""CPU double-precision oracle for the InPlace-ABN hot path -- TEST INFRASTRUCTURE.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py`` (its ``cpu_baseline``
leg and ``--impl reference``) may import this package.  The product package
``paper_1712_02616_b200`` never imports it, and it never imports the product.

The arithmetic lives in ``oracle/oracle.c`` (plain C, double, each function
citing the PAPER.md passage it follows); this module only compiles it with gcc
and marshals numpy float64 arrays through ctypes.  Layout ``"NCHW"`` means
``x[n][c][s]``, ``"NHWC"`` means ``x[n][s][c]`` (s = flattened H*W).
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "oracle.c")
LIB_PATH = os.path.join(_HERE, "liboracle.so")

GAMMA_MODES = {"abs_eps": 0, "plain": 1, "fixed_one": 2}
ACTS = {"leaky": 0, "sigmoid": 1, "tanh": 2}
LAYOUTS = {"NCHW": 0, "NHWC": 1}

_D = ctypes.POINTER(ctypes.c_double)
_I64 = ctypes.c_int64


def build(mutant: int = 0, out: str | None = None, force: bool = False) -> str:
    """Compile oracle.c with gcc (-O2 -fopenmp, no fast-math).  ``mutant`` > 0
    builds a deliberately wrong variant for the test-of-tests."""
    out = out or (LIB_PATH if mutant == 0 else os.path.join(_HERE, f"liboracle_mut{mutant}.so"))
    deps = [_SRC, os.path.join(_HERE, "oracle.h")]
    if (not force and os.path.exists(out)
            and os.path.getmtime(out) >= max(os.path.getmtime(d) for d in deps)):
        return out
    tmp = out + f".tmp{os.getpid()}"
    cmd = ["gcc", "-O2", "-std=c11", "-fopenmp", "-fPIC", "-shared", "-Wall", "-Wextra",
           "-fno-fast-math", "-ffp-contract=off", f"-DORACLE_MUTANT={mutant}",
           "-o", tmp, _SRC, "-lm"]
    subprocess.run(cmd, check=True)
    os.replace(tmp, out)
    return out


def _bind(lib: ctypes.CDLL) -> ctypes.CDLL:
    i, d = ctypes.c_int, ctypes.c_double
    lib.oracle_channel_stats.argtypes = [_I64, _I64, _I64, i, _D, _D, _D]
    lib.oracle_forward.argtypes = [_I64, _I64, _I64, i, _D, _D, _D, i, d, d, d, i, _D, _D, _D,
                                   _D, _D]
    lib.oracle_forward_eval.argtypes = [_I64, _I64, _I64, i, _D, _D, _D, i, d, d, _D, _D, _D]
    lib.oracle_backward_standard.argtypes = [_I64, _I64, _I64, i, _D, _D, _D, _D, i, d, d, _D,
                                             _D, _D]
    for f in (lib.oracle_backward_inplace_I, lib.oracle_backward_inplace_II):
        f.argtypes = [_I64, _I64, _I64, i, _D, _D, _D, _D, _D, i, d, d, _D, _D, _D]
    lib.oracle_merge_stats.argtypes = [_I64, _I64, _D, _D, _D, _D, _D, _D]
    lib.oracle_fold_conv.argtypes = [_I64, _I64, _D, _D, _D, _D, _D, _D, i, d, _D, _D]
    for f in (lib.oracle_channel_stats, lib.oracle_forward, lib.oracle_forward_eval,
              lib.oracle_backward_standard, lib.oracle_backward_inplace_I,
              lib.oracle_backward_inplace_II, lib.oracle_merge_stats, lib.oracle_fold_conv):
        f.restype = None
    lib.oracle_param_grads_sharded.argtypes = [_I64, _I64, _I64, i, _D, _D, _D, _D, i, d, d, _I64,
                                               ctypes.POINTER(_I64), _D, _D]
    lib.oracle_param_grads_sharded.restype = None
    lib.oracle_forward_act.argtypes = [_I64, _I64, _I64, i, _D, _D, _D, i, d, i, d, _D, _D, _D]
    lib.oracle_backward_standard_act.argtypes = [_I64, _I64, _I64, i, _D, _D, _D, _D, i, d, i,
                                                 d, _D, _D, _D]
    lib.oracle_backward_inplace_act.argtypes = [_I64, _I64, _I64, i, _D, _D, _D, _D, _D, i, d, i,
                                                d, _D, _D, _D]
    for f in (lib.oracle_forward_act, lib.oracle_backward_standard_act,
              lib.oracle_backward_inplace_act):
        f.restype = None
    lib.oracle_mutant_id.restype = ctypes.c_int
    return lib


_LIBS: dict[str, "Oracle"] = {}


def load(mutant: int = 0) -> "Oracle":
    path = build(mutant)
    if path not in _LIBS:
        _LIBS[path] = Oracle(_bind(ctypes.CDLL(path)))
    return _LIBS[path]


def _p(a: np.ndarray | None):
    if a is None:
        return None
    assert a.dtype == np.float64 and a.flags["C_CONTIGUOUS"], "oracle wants C-contiguous float64"
    return a.ctypes.data_as(_D)


def _f64(a) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(a, dtype=np.float64))


def _shape(x: np.ndarray, layout: str) -> tuple[int, int, int]:
    """x is given 3-D: NCHW -> [N, C, HW]; NHWC -> [N, HW, C]."""
    assert x.ndim == 3, "pass x as [N, C, HW] (NCHW) or [N, HW, C] (NHWC)"
    if layout == "NCHW":
        return x.shape[0], x.shape[1], x.shape[2]
    return x.shape[0], x.shape[2], x.shape[1]


@dataclass
class ForwardResult:
    z: np.ndarray
    mean: np.ndarray
    var: np.ndarray
    running_mean: np.ndarray | None
    running_var: np.ndarray | None


class Oracle:
    def __init__(self, lib: ctypes.CDLL):
        self.lib = lib
        self.mutant = lib.oracle_mutant_id()

    def channel_stats(self, x, layout="NCHW"):
        x = _f64(x)
        N, C, HW = _shape(x, layout)
        mean, var = np.empty(C), np.empty(C)
        self.lib.oracle_channel_stats(N, C, HW, LAYOUTS[layout], _p(x), _p(mean), _p(var))
        return mean, var

    def forward(self, x, gamma, beta, *, eps=1e-5, slope=0.01, momentum=0.1,
                running_mean=None, running_var=None, gamma_mode="abs_eps",
                running_var_biased=False, layout="NCHW") -> ForwardResult:
        x, gamma, beta = _f64(x), _f64(gamma), _f64(beta)
        N, C, HW = _shape(x, layout)
        rm = None if running_mean is None else _f64(running_mean).copy()
        rv = None if running_var is None else _f64(running_var).copy()
        z, mean, var = np.empty_like(x), np.empty(C), np.empty(C)
        self.lib.oracle_forward(N, C, HW, LAYOUTS[layout], _p(x), _p(gamma), _p(beta),
                                GAMMA_MODES[gamma_mode], eps, slope, momentum,
                                int(running_var_biased), _p(rm), _p(rv), _p(z), _p(mean), _p(var))
        return ForwardResult(z, mean, var, rm, rv)

    def forward_eval(self, x, gamma, beta, running_mean, running_var, *, eps=1e-5, slope=0.01,
                     gamma_mode="abs_eps", layout="NCHW") -> np.ndarray:
        x = _f64(x)
        N, C, HW = _shape(x, layout)
        z = np.empty_like(x)
        self.lib.oracle_forward_eval(N, C, HW, LAYOUTS[layout], _p(x), _p(_f64(gamma)),
                                     _p(_f64(beta)), GAMMA_MODES[gamma_mode], eps, slope,
                                     _p(_f64(running_mean)), _p(_f64(running_var)), _p(z))
        return z

    def fold_conv(self, w, bias, running_mean, running_var, gamma, beta, *, eps=1e-5,
                  gamma_mode="abs_eps"):
        """Test-time BN absorbed into the preceding conv: w [cout, ...],
        bias [cout] or None -> (w', bias')."""
        w = _f64(w)
        cout = w.shape[0]
        kper = int(w.size // cout)
        w_out, b_out = np.empty_like(w), np.empty(cout)
        b = None if bias is None else _f64(bias)
        self.lib.oracle_fold_conv(cout, kper, _p(w), None if b is None else _p(b),
                                  _p(_f64(running_mean)), _p(_f64(running_var)), _p(_f64(gamma)),
                                  _p(_f64(beta)), GAMMA_MODES[gamma_mode], eps, _p(w_out),
                                  _p(b_out))
        return w_out, b_out

    def backward_standard(self, x, dz, gamma, beta, *, eps=1e-5, slope=0.01,
                          gamma_mode="abs_eps", layout="NCHW"):
        x, dz = _f64(x), _f64(dz)
        N, C, HW = _shape(x, layout)
        dx, dg, db = np.empty_like(x), np.empty(C), np.empty(C)
        self.lib.oracle_backward_standard(N, C, HW, LAYOUTS[layout], _p(x), _p(dz),
                                          _p(_f64(gamma)), _p(_f64(beta)),
                                          GAMMA_MODES[gamma_mode], eps, slope, _p(dx), _p(dg),
                                          _p(db))
        return dx, dg, db

    def _bwd_from_z(self, fn, z, dz, var, gamma, beta, eps, slope, gamma_mode, layout):
        z, dz = _f64(z), _f64(dz)
        N, C, HW = _shape(z, layout)
        dx, dg, db = np.empty_like(z), np.empty(C), np.empty(C)
        fn(N, C, HW, LAYOUTS[layout], _p(z), _p(dz), _p(_f64(var)), _p(_f64(gamma)),
           _p(_f64(beta)), GAMMA_MODES[gamma_mode], eps, slope, _p(dx), _p(dg), _p(db))
        return dx, dg, db

    def backward_inplace_I(self, z, dz, var, gamma, beta, *, eps=1e-5, slope=0.01,
                           gamma_mode="abs_eps", layout="NCHW"):
        return self._bwd_from_z(self.lib.oracle_backward_inplace_I, z, dz, var, gamma, beta, eps,
                                slope, gamma_mode, layout)

    def backward_inplace_II(self, z, dz, var, gamma, beta, *, eps=1e-5, slope=0.01,
                            gamma_mode="abs_eps", layout="NCHW"):
        return self._bwd_from_z(self.lib.oracle_backward_inplace_II, z, dz, var, gamma, beta, eps,
                                slope, gamma_mode, layout)

    def param_grads_sharded(self, x, dz, gamma, beta, shards, *, eps=1e-5, slope=0.01,
                            gamma_mode="abs_eps", layout="NCHW"):
        """Per-shard (dgamma, dbeta), each [len(shards), C], of the synchronized layer over
        the concatenated batch x (shard k = the next shards[k] samples along N; R7)."""
        x, dz = _f64(x), _f64(dz)
        N, C, HW = _shape(x, layout)
        assert sum(shards) == N
        K = len(shards)
        sn = (_I64 * K)(*[int(s) for s in shards])
        dg, db = np.empty((K, C)), np.empty((K, C))
        self.lib.oracle_param_grads_sharded(N, C, HW, LAYOUTS[layout], _p(x), _p(dz),
                                            _p(_f64(gamma)), _p(_f64(beta)),
                                            GAMMA_MODES[gamma_mode], eps, slope, K, sn, _p(dg),
                                            _p(db))
        return dg, db

    # ------------------------------------------- other invertible activations
    def forward_act(self, x, gamma, beta, *, act="sigmoid", eps=1e-5, slope=0.01,
                    gamma_mode="abs_eps", layout="NCHW"):
        """(z, mean, biased var) of BN followed by `act` (leaky / sigmoid / tanh)."""
        x = _f64(x)
        N, C, HW = _shape(x, layout)
        z, mean, var = np.empty_like(x), np.empty(C), np.empty(C)
        self.lib.oracle_forward_act(N, C, HW, LAYOUTS[layout], _p(x), _p(_f64(gamma)),
                                    _p(_f64(beta)), GAMMA_MODES[gamma_mode], eps, ACTS[act],
                                    slope, _p(z), _p(mean), _p(var))
        return z, mean, var

    def backward_standard_act(self, x, dz, gamma, beta, *, act="sigmoid", eps=1e-5, slope=0.01,
                              gamma_mode="abs_eps", layout="NCHW"):
        x, dz = _f64(x), _f64(dz)
        N, C, HW = _shape(x, layout)
        dx, dg, db = np.empty_like(x), np.empty(C), np.empty(C)
        self.lib.oracle_backward_standard_act(N, C, HW, LAYOUTS[layout], _p(x), _p(dz),
                                              _p(_f64(gamma)), _p(_f64(beta)),
                                              GAMMA_MODES[gamma_mode], eps, ACTS[act], slope,
                                              _p(dx), _p(dg), _p(db))
        return dx, dg, db

    def backward_inplace_act(self, z, dz, var, gamma, beta, *, act="sigmoid", eps=1e-5,
                             slope=0.01, gamma_mode="abs_eps", layout="NCHW"):
        z, dz = _f64(z), _f64(dz)
        N, C, HW = _shape(z, layout)
        dx, dg, db = np.empty_like(z), np.empty(C), np.empty(C)
        self.lib.oracle_backward_inplace_act(N, C, HW, LAYOUTS[layout], _p(z), _p(dz),
                                             _p(_f64(var)), _p(_f64(gamma)), _p(_f64(beta)),
                                             GAMMA_MODES[gamma_mode], eps, ACTS[act], slope,
                                             _p(dx), _p(dg), _p(db))
        return dx, dg, db

    def merge_stats(self, counts, means, vars_):
        counts, means, vars_ = _f64(counts), _f64(means), _f64(vars_)
        K, C = means.shape
        cnt = ctypes.c_double(0.0)
        mean, var = np.empty(C), np.empty(C)
        self.lib.oracle_merge_stats(K, C, _p(counts), _p(means), _p(vars_), ctypes.byref(cnt),
                                    _p(mean), _p(var))
        return cnt.value, mean, var
