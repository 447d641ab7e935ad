"""Seeded synthetic gradient generators (SURVEY.md §8(d) "Synthetic inputs").

Holds NONE of LowDiff's arithmetic: only random numbers with the shapes and
value distributions of the paper's workloads.  The tensors are produced once
(on whatever device the caller asks for) and the very same bytes are handed to
the CUDA path and, copied to the host, to the oracle -- so both sides always see
bit-identical inputs (task rule ③).

Distributions:
  D1  Gaussian with a per-layer scale s_l = 10**(-4 + 3 u_l), u_l = hash(seed, l)
  D2  heavy tail (Student-t with 3 degrees of freedom) with the same scales
  D3  D1 quantised to bf16-representable fp32 (low 16 mantissa bits zeroed): tie stress
  D4  D1 with embedding-row sparsity (GPT-2 wte rows active w.p. 0.16, BERT word rows
      w.p. 0.3) and 1-D (LayerNorm / bias) tensors scaled by 0.1
  D5  rank correlation: g_r = alpha * z_shared + sqrt(1 - alpha^2) * z_r
The bench default is D4 with alpha = 0.5 (D1 o D4 o D5).
"""
from __future__ import annotations

import math

import torch

SEED = 2509040840  # < 2**32; the arXiv id
_MASK64 = (1 << 64) - 1


def splitmix64(x: int) -> int:
    x = (x + 0x9E3779B97F4A7C15) & _MASK64
    z = x
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & _MASK64
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & _MASK64
    return z ^ (z >> 31)


def mix(*vals: int) -> int:
    h = 0
    for v in vals:
        h = splitmix64(h ^ (v & _MASK64))
    return h


def layer_scales(n_layers: int, seed: int = SEED) -> list[float]:
    """s_l = 10**(-4 + 3 u_l) with u_l in [0,1) from hash(seed, l)."""
    return [10.0 ** (-4.0 + 3.0 * (mix(seed, 0x5CA1E, l) >> 11) / float(1 << 53)) for l in range(n_layers)]


def _gen(device, *key: int) -> torch.Generator:
    g = torch.Generator(device=device)
    g.manual_seed(mix(*key) & ((1 << 63) - 1))
    return g


# row structure of the embedding tables, by layer-table name (D4)
ROW_SPARSITY = {
    "gpt2_xl": {0: (1600, 0.16)},      # wte: ~8K distinct tokens of 50,257 per batch
    "bert_large": {0: (1024, 0.30)},   # word embeddings
}


def gradient(sizes: list[int], rank: int, iteration: int, *, dist: str = "D4",
             alpha: float = 0.5, model: str | None = None, seed: int = SEED,
             device="cpu", out: torch.Tensor | None = None) -> torch.Tensor:
    """One rank's dense fp32 gradient for one iteration, flat over the layer table."""
    psi = sum(sizes)
    if out is None:
        out = torch.empty(psi, dtype=torch.float32, device=device)
    device = out.device
    scales = layer_scales(len(sizes), seed)
    stream = {"D1": 1, "D2": 2, "D3": 3, "D4": 4, "D5": 5}[dist]
    g_own = _gen(device, seed, stream, rank, iteration)
    g_shared = _gen(device, seed, stream, 0xFFFF, iteration)
    a = float(alpha)
    b = math.sqrt(max(0.0, 1.0 - a * a))
    rows = ROW_SPARSITY.get(model or "", {}) if dist == "D4" else {}
    off = 0
    for l, n in enumerate(sizes):
        seg = out[off:off + n]
        z = torch.randn(n, generator=g_own, device=device, dtype=torch.float32)
        if a != 0.0:
            zs = torch.randn(n, generator=g_shared, device=device, dtype=torch.float32)
            z.mul_(b).add_(zs, alpha=a)
        if dist == "D2":
            chi = torch.randn((3, n), generator=g_own, device=device, dtype=torch.float32)
            z.div_(chi.square().mean(0).sqrt_().clamp_min_(1e-3))
        z.mul_(scales[l])
        if dist == "D4":
            if l in rows:
                row_len, p = rows[l]
                nrow = n // row_len
                act = torch.rand(nrow, generator=g_own, device=device) < p
                z.view(nrow, row_len).mul_(act[:, None].to(torch.float32))
            elif n <= 6400:  # 1-D LayerNorm / bias tensors
                z.mul_(0.1)
        if dist == "D3":
            z = (z.view(torch.int32) & ~0xFFFF).view(torch.float32)
        seg.copy_(z)
        off += n
    return out


def adversarial_layers() -> list[tuple[str, torch.Tensor]]:
    """Hand-built layers for the tie / degenerate cases of SURVEY §8(d) parity suite."""
    g = _gen("cpu", SEED, 99)
    cases = [
        ("all_zero", torch.zeros(3000)),
        ("all_equal", torch.full((2500,), 0.25)),
        ("signed_equal", torch.tensor([0.5, -0.5] * 1200)),
        ("single_nonzero", torch.zeros(4097).index_fill_(0, torch.tensor([1234]), -3.0)),
        ("n_is_1", torch.tensor([0.75])),
        ("neg_zero", torch.tensor([-0.0, 0.0] * 700)),
        ("denormals", torch.tensor([1e-45, -2e-45, 3e-44, 1e-40] * 300)),
        ("bf16_ties", (torch.randn(20000, generator=g).view(torch.int32) & ~0xFFFFF).view(torch.float32)),
    ]
    return cases
