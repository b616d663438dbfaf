"""C-ABI library: loads without a GPU, exports every symbol include/iabn.h
declares, and validates arguments synchronously before touching the device
(so every error path below is exercised here, on CPU, with fake pointers that
are never dereferenced)."""
import ctypes
import os
import re

import pytest
import torch

from paper_1712_02616_b200 import _lib as L

# Calls that pass every host-side check would launch kernels on fake pointers
# if a GPU were present; they only run where there is none.
no_gpu = pytest.mark.skipif(torch.cuda.is_available(),
                            reason="would launch kernels on fake pointers")

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "iabn.h")

P = 0x10000  # fake, 16-byte aligned "device" addresses (never dereferenced)


def declared_symbols():
    src = open(HEADER).read()
    return sorted(set(re.findall(r"IABN_API\s+[\w\s\*]+?\b(iabn_\w+)\s*\(", src)))


def test_exports_every_declared_symbol():
    decl = declared_symbols()
    assert len(decl) >= 17
    assert sorted(decl) == sorted(L.EXPORTS)
    for name in decl:
        assert hasattr(L.lib, name), name


def test_version_and_status_strings():
    assert L.lib.iabn_version() == 1
    names = [L.lib.iabn_status_string(s).decode() for s in range(8)]
    assert names[0] == "IABN_OK" and names[3] == "IABN_ERR_ALIAS" and names[7] == "IABN_ERR_NCCL"


def _fwd(d, x=P, z=P, gamma=P, beta=P, rm=P, rv=P, sm=P, sv=P, momentum=0.1, eps=1e-5,
         slope=0.01, flags=0, ws=P * 16, ws_bytes=None):
    if ws_bytes is None:
        ws_bytes = L.workspace_bytes(d)
    return L.lib.iabn_forward(ctypes.byref(d), x, z, gamma, beta, rm, rv, sm, sv, momentum, eps,
                              slope, flags, ws, ws_bytes, None)


def _bwd(d, z=P, dz=P * 4096, dx=P * 4096, gamma=P, beta=P, sv=P, dg=P, db=P, eps=1e-5,
         slope=0.01, flags=0, ws=P * 16, ws_bytes=None):
    if ws_bytes is None:
        ws_bytes = L.workspace_bytes(d)
    return L.lib.iabn_backward(ctypes.byref(d), z, dz, dx, gamma, beta, None, sv, dg, db, eps,
                               slope, flags, ws, ws_bytes, None)


def test_workspace_bytes():
    assert L.workspace_bytes(L.desc(0, 4, 4, L.F32, L.NCHW)) == 0
    assert L.workspace_bytes(L.desc(2, 8, 16, L.F32, L.NCHW)) > 0
    a = L.workspace_bytes(L.desc(64, 1024, 196, L.F32, L.NCHW))
    b = L.workspace_bytes(L.desc(16, 4096, 12544, L.BF16, L.NCHW))
    assert a > 0 and b > 0 and b < 16 << 20  # O(C) scratch, never O(E)


@pytest.mark.parametrize("n,c,hw", [(0, 4, 4), (2, 0, 4), (2, 4, 0), (-1, 4, 4)])
def test_empty_shapes_rejected(n, c, hw):
    d = L.desc(n, c, hw, L.F32, L.NCHW)
    assert _fwd(d, ws_bytes=1 << 20) == L.ERR_INVALID_ARG
    assert "empty" in L.lib.iabn_last_error().decode()


def test_unknown_dtype_layout():
    assert _fwd(L.desc(2, 4, 4, 7, L.NCHW), ws_bytes=1 << 20) == L.ERR_UNSUPPORTED
    assert _fwd(L.desc(2, 4, 4, L.F32, 5), ws_bytes=1 << 20) == L.ERR_UNSUPPORTED


@pytest.mark.parametrize("kw,status", [
    (dict(eps=0.0), L.ERR_INVALID_ARG), (dict(eps=-1e-5), L.ERR_INVALID_ARG),
    (dict(eps=float("inf")), L.ERR_INVALID_ARG), (dict(eps=float("nan")), L.ERR_INVALID_ARG),
    (dict(slope=0.0), L.ERR_INVALID_ARG), (dict(slope=1.5), L.ERR_INVALID_ARG),
    (dict(momentum=-0.1), L.ERR_INVALID_ARG), (dict(momentum=1.1), L.ERR_INVALID_ARG),
    (dict(x=0), L.ERR_INVALID_ARG), (dict(gamma=0), L.ERR_INVALID_ARG),
    (dict(sm=0), L.ERR_INVALID_ARG), (dict(rm=0), L.ERR_INVALID_ARG),
    (dict(x=P + 4), L.ERR_UNSUPPORTED), (dict(z=P + 8), L.ERR_ALIAS),
    (dict(ws=0), L.ERR_WORKSPACE), (dict(ws_bytes=16), L.ERR_WORKSPACE),
])
def test_forward_validation(kw, status):
    d = L.desc(2, 8, 16, L.F32, L.NCHW)
    if kw.get("z") == P + 8:  # 8 bytes past x: misaligned is checked first, so use +16
        kw["z"] = P + 16
    assert _fwd(d, **kw) == status, L.lib.iabn_last_error()


def test_forward_degenerate_single_value():
    d = L.desc(1, 8, 1, L.F32, L.NCHW)  # m = 1 value per channel
    assert _fwd(d) == L.ERR_DEGENERATE


@no_gpu
def test_forward_momentum_zero_accepted_and_reaches_device():
    d = L.desc(2, 8, 16, L.F32, L.NCHW)
    # all host checks pass -> the call gets as far as the device (absent here)
    st = _fwd(d, momentum=0.0, rm=0, rv=0)
    assert st in (L.ERR_CUDA, L.OK)
    if st == L.ERR_CUDA:
        assert "cuda" in L.lib.iabn_last_error().decode().lower()


@no_gpu
def test_forward_in_place_allowed():
    d = L.desc(2, 8, 16, L.F32, L.NCHW)
    assert _fwd(d, x=P, z=P) in (L.ERR_CUDA, L.OK)
    assert _fwd(d, x=P, z=P + 2 * 8 * 16 * 4) in (L.ERR_CUDA, L.OK)  # disjoint


@pytest.mark.parametrize("kw,status", [
    (dict(dx=P * 4096 + 16), L.ERR_ALIAS),  # partial overlap of dx and dz
    (dict(dx=P), L.ERR_ALIAS),  # dx overlaps z
    (dict(sv=0), L.ERR_INVALID_ARG), (dict(dg=0), L.ERR_INVALID_ARG),
    (dict(slope=2.0), L.ERR_INVALID_ARG), (dict(z=P + 2), L.ERR_UNSUPPORTED),
])
def test_backward_validation(kw, status):
    d = L.desc(2, 8, 16, L.F32, L.NCHW)
    assert _bwd(d, **kw) == status, L.lib.iabn_last_error()


@no_gpu
def test_backward_in_place_reaches_device():
    d = L.desc(2, 8, 16, L.BF16, L.NHWC)
    assert _bwd(d) in (L.ERR_CUDA, L.OK)


@no_gpu
def test_eval_needs_running_stats():
    d = L.desc(2, 8, 16, L.F32, L.NCHW)
    assert _fwd(d, rm=0, flags=L.EVAL) == L.ERR_INVALID_ARG
    assert _fwd(d, sm=0, sv=0, flags=L.EVAL) in (L.ERR_CUDA, L.OK)


@no_gpu
def test_launch_count_is_zero_without_launches():
    assert L.launch_count() == 0


def _fold(cout=4, k=27, w=P, bias=P * 2, rm=P * 3, rv=P * 4, gamma=P * 5, beta=P * 6, eps=1e-5,
          flags=0, w_out=P * 64, b_out=P * 128):
    return L.lib.iabn_fold_conv(cout, k, w, bias, rm, rv, gamma, beta, eps, flags, w_out, b_out,
                                None)


@pytest.mark.parametrize("kw,status", [
    (dict(cout=0), L.ERR_INVALID_ARG), (dict(k=-1), L.ERR_INVALID_ARG),
    (dict(w=0), L.ERR_INVALID_ARG), (dict(rv=0), L.ERR_INVALID_ARG),
    (dict(b_out=0), L.ERR_INVALID_ARG), (dict(eps=0.0), L.ERR_INVALID_ARG),
    (dict(eps=float("nan")), L.ERR_INVALID_ARG), (dict(w=P + 4), L.ERR_UNSUPPORTED),
    (dict(w_out=P + 16), L.ERR_ALIAS),  # partial overlap of w and w_out
    (dict(b_out=P * 64 + 8), L.ERR_ALIAS),  # bias_out inside w_out
    (dict(b_out=P * 2 + 4), L.ERR_ALIAS),  # partial overlap of bias and bias_out
])
def test_fold_conv_validation(kw, status):
    assert _fold(**kw) == status, L.lib.iabn_last_error()


@no_gpu
def test_fold_conv_in_place_reaches_device():
    assert _fold(w_out=P, b_out=P * 2) in (L.ERR_CUDA, L.OK)
    assert _fold(bias=0) in (L.ERR_CUDA, L.OK)  # no conv bias


# ---------------------------------------------------------------- fused-collective sync emulation
def _fwd_emu(d, nranks, flags=0, ws_bytes=None, x=P, z=P):
    gd = L.desc(d.n * nranks, d.c, d.hw, d.dtype, d.layout) if 1 <= nranks <= 64 else d
    if ws_bytes is None:
        ws_bytes = L.workspace_bytes(gd)
    return L.lib.iabn_forward_sync_emulated(ctypes.byref(d), nranks, x, z, P, P, P, P, P, P, 0.1,
                                            1e-5, 0.01, flags, P * 16, ws_bytes, None)


@pytest.mark.parametrize("nranks", [0, -1, 9])
def test_sync_emulated_rank_count(nranks):
    d = L.desc(2, 8, 16, L.F32, L.NCHW)
    assert _fwd_emu(d, nranks) == L.ERR_INVALID_ARG, L.lib.iabn_last_error()


def test_sync_emulated_validation():
    d = L.desc(2, 8, 16, L.F32, L.NCHW)
    assert _fwd_emu(d, 2, flags=L.EVAL) == L.ERR_INVALID_ARG
    assert _fwd_emu(L.desc(2, 8, 16, L.F32, L.NHWC), 2) == L.ERR_UNSUPPORTED
    # the workspace is sized for the whole tensor (nranks shards), not one shard
    assert _fwd_emu(d, 4, ws_bytes=L.workspace_bytes(d) - 1) == L.ERR_WORKSPACE
    # z overlapping part of the whole tensor (not only of the first shard)
    assert _fwd_emu(d, 4, z=P + 3 * 8 * 16 * 4) == L.ERR_ALIAS
    dz = P * 4096
    st = L.lib.iabn_backward_sync_emulated(ctypes.byref(d), 2, P, dz, dz, P, P, None, 0, P, P,
                                           1e-5, 0.01, 0, P * 16,
                                           L.workspace_bytes(L.desc(4, 8, 16, L.F32, L.NCHW)), None)
    assert st == L.ERR_INVALID_ARG  # save_var NULL


def test_build_entry_does_not_import_package_before_library_exists():
    """build() must work from a fresh checkout (libiabn.so is git-ignored): the build
    script is loaded by path, so the package (which raises without the library) is not
    imported before the library is built."""
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    code = ("import importlib.util, sys, os;"
            "spec = importlib.util.spec_from_file_location('_b', "
            "os.path.join(sys.argv[1], 'paper_1712_02616_b200', 'build.py'));"
            "m = importlib.util.module_from_spec(spec); spec.loader.exec_module(m);"
            "assert 'paper_1712_02616_b200' not in sys.modules;"
            "assert callable(m.build) and m.LIB.endswith('libiabn.so')")
    subprocess.run([sys.executable, "-c", code, root], check=True, cwd="/")


# ---------------------------------------------------------------- sigmoid / tanh
def test_activation_flag_validation():
    f32, bf16 = L.desc(2, 8, 16, L.F32, L.NCHW), L.desc(2, 8, 16, L.BF16, L.NHWC)
    both = L.ACT_SIGMOID | L.ACT_TANH
    assert _fwd(f32, flags=both) == L.ERR_INVALID_ARG
    assert _bwd(f32, flags=both) == L.ERR_INVALID_ARG
    for act in (L.ACT_SIGMOID, L.ACT_TANH):
        assert _fwd(bf16, flags=act) == L.ERR_UNSUPPORTED  # fp32 storage only
        assert _bwd(bf16, flags=act) == L.ERR_UNSUPPORTED
        assert _fwd_emu(f32, 2, flags=act) == L.ERR_UNSUPPORTED  # single-GPU entries only
        assert L.lib.iabn_forward_apply(ctypes.byref(f32), P, P, P, P, P, P, P, P, P, 0.1, 1e-5,
                                        0.01, act, P * 16, L.workspace_bytes(f32),
                                        None) == L.ERR_UNSUPPORTED


def test_activation_names():
    import paper_1712_02616_b200 as Pk
    from paper_1712_02616_b200 import functional as F
    assert F._act("leaky_relu") == 0 and F._act("sigmoid") == L.ACT_SIGMOID
    with pytest.raises(ValueError):
        F._act("relu")  # not invertible
    with pytest.raises(ValueError):
        Pk.InPlaceABN(4, activation="gelu")


def test_nhwc_bulk_ring_plan_host_logic():
    """The NHWC bulk-ring reduction plan (iabn_debug_nb_records, host only): records = whole
    clusters of 8 CTAs, at most 32 (256 CTAs), >= 8 stages of 16 KB; not for rows over 4 KB,
    NCHW, or rows that are not 16-byte aligned."""
    f = L.lib.iabn_debug_nb_records
    f.argtypes = [ctypes.c_void_p]
    f.restype = ctypes.c_int

    def rec(n, c, hw, dt=L.BF16, ly=L.NHWC):
        d = L.desc(n, c, hw, dt, ly)
        return f(ctypes.addressof(d))
    assert rec(32, 128, 3136) == 32                 # 25.7 MB: capped at 32 clusters
    assert rec(1, 64, 1024) == 1                    # 128 KB: 8 CTAs of one 16 KB stage
    assert rec(4, 64, 1024) == 4                    # 512 KB: 32 CTAs
    assert rec(1, 64, 512) == 0                     # 64 KB: 4 CTAs, no whole cluster
    assert rec(32, 2048, 49) > 0                    # 4 KB rows: still bulk
    assert rec(32, 2080, 49) == 0                   # > 4 KB rows
    assert rec(32, 128, 3136, ly=L.NCHW) == 0       # NCHW: never
    assert rec(32, 7, 3136, dt=L.F32) == 0          # 28-byte rows: not 16-byte aligned
