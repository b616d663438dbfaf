"""Seeded synthetic inputs shared by the oracle side and the CUDA side.

This module holds NO arithmetic of the method: it only draws random numbers
with torch's generator (CPU by default, so tests and the oracle see the same
values on any machine) and lays them out.  The recipe is DESIGN.md
"Input recipe" (after SURVEY.md section 8(d)): conv-output-like per-channel
heterogeneity,

  x[., c, .] ~ N(mu_c, s_c^2),  mu_c ~ U(-2, 2),  s_c log-uniform in [0.25, 4]
  gamma_c = +-U(0.5, 1.5) with 20% negative;  beta_c = U(-0.5, 0.5) * |gamma_c|
  dz ~ N(0, 1);  running mean 0, running var 1

bf16 storage is the RNE rounding of the fp32 draws.  Stress variants:
``offset`` (|mean|/std = 1e3, cancellation), ``constant`` (channel 0 constant).
Tensors are 3-D: NCHW -> [N, C, HW], NHWC -> [N, HW, C] (contiguous).
"""
from __future__ import annotations

import math
from dataclasses import dataclass

import torch

DTYPES = {"f32": torch.float32, "bf16": torch.bfloat16}


@dataclass
class Params:
    gamma: torch.Tensor
    beta: torch.Tensor
    running_mean: torch.Tensor
    running_var: torch.Tensor


def _gen(seed: int, device="cpu") -> torch.Generator:
    g = torch.Generator(device=device)
    g.manual_seed(int(seed))
    return g


def make_params(C: int, seed: int, device="cpu") -> Params:
    g = _gen(10_000 + seed, device)
    mag = torch.rand(C, generator=g, device=device) + 0.5
    neg = torch.rand(C, generator=g, device=device) < 0.2
    gamma = torch.where(neg, -mag, mag)
    beta = (torch.rand(C, generator=g, device=device) - 0.5) * mag
    return Params(gamma.float().contiguous(), beta.float().contiguous(),
                  torch.zeros(C, device=device), torch.ones(C, device=device))


def channel_moments(C: int, seed: int, device="cpu", stress: str | None = None):
    g = _gen(20_000 + seed, device)
    mu = torch.rand(C, generator=g, device=device) * 4.0 - 2.0
    lo, hi = math.log(0.25), math.log(4.0)
    s = torch.exp(torch.rand(C, generator=g, device=device) * (hi - lo) + lo)
    if stress == "offset":
        mu = torch.where(mu >= 0, 1.0, -1.0).to(device) * 1e3 * s
    return mu, s


def make_x(N: int, C: int, HW: int, seed: int, *, layout="NCHW", dtype="f32", device="cpu",
           stress: str | None = None) -> torch.Tensor:
    mu, s = channel_moments(C, seed, device, stress)
    g = _gen(30_000 + seed, device)
    x = torch.randn(N, C, HW, generator=g, device=device)
    x.mul_(s.view(1, C, 1)).add_(mu.view(1, C, 1))
    if stress == "constant":
        x[:, 0, :] = mu[0]
    if layout == "NHWC":
        x = x.permute(0, 2, 1).contiguous()
    return x.to(DTYPES[dtype]).contiguous()


def make_dz(N: int, C: int, HW: int, seed: int, *, layout="NCHW", dtype="f32",
            device="cpu") -> torch.Tensor:
    g = _gen(40_000 + seed, device)
    dz = torch.randn(N, C, HW, generator=g, device=device)
    if layout == "NHWC":
        dz = dz.permute(0, 2, 1).contiguous()
    return dz.to(DTYPES[dtype]).contiguous()


def to_nchw(t: torch.Tensor, layout: str) -> torch.Tensor:
    """[N, HW, C] -> [N, C, HW] (pure re-indexing)."""
    return t if layout == "NCHW" else t.permute(0, 2, 1)


# Shapes of BASELINE.json's configs (SURVEY.md section 8 preamble).
CONFIGS = {
    "tiny": dict(N=2, C=8, HW=16, dtype="f32", layout="NCHW"),
    "r50s3": dict(N=64, C=1024, HW=196, dtype="f32", layout="NCHW"),
    "wrn38": dict(N=16, C=4096, HW=112 * 112, dtype="bf16", layout="NCHW"),
}

# ResNeXt-101 32x4d pre-activation BN+Act layers at 224^2: (C, HW, count)
# (SURVEY.md section 8, cfg3 table); N = 32 per GPU.
RX101_LAYERS = [(64, 112 * 112, 1), (64, 56 * 56, 1), (128, 56 * 56, 6), (256, 56 * 56, 4),
                (256, 28 * 28, 7), (512, 28 * 28, 5), (512, 14 * 14, 45), (1024, 14 * 14, 24),
                (1024, 7 * 7, 5), (2048, 7 * 7, 3)]


def densenet264_layers() -> list[tuple[int, int]]:
    """(C, HW) of every BN of DenseNet-BC-264 (growth 32, blocks 6/12/64/48, bottleneck
    4*32) at 224^2, in network order: stem BN, per dense layer BN(concat) + BN(128),
    transition BNs, final BN (C 64..2688)."""
    k, out = 32, [(64, 112 * 112)]
    c, hw = 64, 56 * 56
    for bi, n in enumerate((6, 12, 64, 48)):
        for i in range(n):
            out.append((c + i * k, hw))
            out.append((4 * k, hw))
        c += n * k
        if bi < 3:
            out.append((c, hw))  # transition BN
            c //= 2
            hw //= 4
    out.append((c, hw))  # final BN
    return out


def rx101_layers() -> list[tuple[int, int]]:
    """(C, HW) of the 101 BN+Act layers of ResNeXt-101 32x4d in network order."""
    return [(c, hw) for c, hw, n in RX101_LAYERS for _ in range(n)]

