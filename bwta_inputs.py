"""Seeded synthetic inputs shared by the tests, smoke() and bench.py.

Holds NO arithmetic of the BWTA method (no quantization, packing, dot
products or epilogues): only random tensors with the distributions of the
paper's workloads and the scale statistics its recipe prescribes
(DESIGN.md "Input recipe").  Tensors are generated on the CPU with a seeded
torch.Generator, so the CUDA path and the CPU oracle see identical bytes.

Recipe:
  * activations X ~ N(0, 1) in FP16 (Gaussian activations);
  * weights W ~ 0.02 N(0, 1); mu = mean(W); per-channel weight scale
    s_w[n] = mean |W_n - mu| (north star "per-channel weight scale");
  * activation scale s_A = 2 mean|X| (the init s_A^0 = (2/n)||A||_1),
    which yields ~57.5% zeros;
  * attention probabilities P = softmax(z), z ~ N(0, 1) per row (power-law-like
    probabilities), s_Att = 2 mean(P) = 2/Tk -> ~31% ones;
  * post-ReLU FFN2 input relu(N(0, 1)), s = 2 mean|x|.
"""
from __future__ import annotations

import torch


def _gen(seed: int) -> torch.Generator:
    g = torch.Generator(device="cpu")
    g.manual_seed(int(seed))
    return g


def normal(shape, seed: int, dtype=torch.float16, std: float = 1.0) -> torch.Tensor:
    x = torch.randn(tuple(shape), generator=_gen(seed), dtype=torch.float32)
    if std != 1.0:
        x = x * std
    return x.to(dtype)


def activations(shape, seed: int, dtype=torch.float16) -> torch.Tensor:
    return normal(shape, seed, dtype)


def relu_activations(shape, seed: int, dtype=torch.float16) -> torch.Tensor:
    return torch.clamp_min(normal(shape, seed, torch.float32), 0.0).to(dtype)


def weights(n: int, k: int, seed: int, dtype=torch.float16) -> torch.Tensor:
    return normal((n, k), seed, dtype, std=0.02)


def attention_probs(shape, seed: int, dtype=torch.float16) -> torch.Tensor:
    z = normal(shape, seed, torch.float32)
    return torch.softmax(z, dim=-1).to(dtype)


def act_scale(x: torch.Tensor) -> float:
    """s_A = 2 mean|x|, computed in float64, returned as a float32 value."""
    v = 2.0 * x.detach().to("cpu", torch.float64).abs().mean().item()
    return float(torch.tensor(v, dtype=torch.float32).item())


def weight_stats(w: torch.Tensor):
    """(mu, s_w): mu = mean(W) as float32; s_w[n] = mean|W_n - mu| float32 [N]."""
    w64 = w.detach().to("cpu", torch.float64)
    mu = float(torch.tensor(w64.mean().item(), dtype=torch.float32).item())
    s_w = (w64 - mu).abs().mean(dim=1).to(torch.float32)
    return mu, s_w


def uniform_codes(shape, seed: int, low: int, high: int) -> torch.Tensor:
    """Random integer codes in [low, high] (int8), for plane-level tests."""
    return torch.randint(low, high + 1, tuple(shape), generator=_gen(seed), dtype=torch.int8)


def random_words(shape, seed: int) -> torch.Tensor:
    """Random uint32 words (as int32 bit patterns)."""
    return torch.randint(-2**31, 2**31 - 1, tuple(shape), generator=_gen(seed), dtype=torch.int64).to(torch.int32)
