"""Seeded synthetic inputs shared by the tests, ``bench.py`` and ``smoke()``.

This module holds NO arithmetic of the method (no RMSNorm, no transform, no
attention, no absorption).  It only draws numbers and rounds them to the bf16
storage format, so that the CUDA path and the CPU oracle consume bit-identical
inputs.  Neither ``oracle/`` nor the product package
is imported here.

Every array that stands for a bf16 tensor is returned as ``uint16`` bit
patterns; callers widen them (the oracle to fp64, the product to a torch bf16
view).  Recipe (SURVEY.md §8(d) "Synthetic inputs"):

* raw latent rows ``c_KV`` ~ N(0, diag(sigma^2)) with a power-law spectrum
  ``sigma_i^2 ∝ 1/(i+1)`` plus 4 outlier channels x10 (the per-channel imbalance
  the Hadamard transform targets, §4.3.1), optionally rotated by
  a random orthogonal basis ``V`` so that the population PCA basis is ``V``
  (§4.3.2: PCA concentrates energy in leading components);
* RoPE keys ``k_pe`` and queries ``q_nope``, ``q_pe`` ~ N(0, 1);
* weights W^UK, W^UV ~ N(0, 1/d_h) and N(0, 1/d_c); W^O ~ N(0, 1/(h_q d_h));
  gamma ~ 1 + 0.1 N(0, 1) (§3.3 P:97-100 shapes).

Each sequence ``b`` draws from its own stream ``(seed, b)`` so any single
sequence of a 32K-token batch can be regenerated cheaply for sampled parity.
"""
from __future__ import annotations

import dataclasses
import numpy as np

__all__ = [
    "ModelDims", "PRESETS", "bf16_bits", "bf16_to_f32", "Weights", "gen_weights",
    "gen_raw_ckv", "gen_kpe", "gen_queries", "gen_seq_lens", "random_orthogonal",
    "latent_spectrum",
]


@dataclasses.dataclass(frozen=True)
class ModelDims:
    """Attention-layer dimensions (§3.1/§3.3 symbols)."""
    name: str
    h_q: int          # query heads
    d_c: int          # latent width (= 4 d_h in the paper)
    d_r: int          # decoupled RoPE width
    d_h: int          # head dim
    D: int            # hidden size

    @property
    def n_outlier(self) -> int:
        return min(4, self.d_c // 8)


# Presets: BASELINE.json configs (BJ:7-11) and SURVEY.md §8(d).
PRESETS = {
    # configs[0] "tiny": 4 heads, latent 64 + RoPE 16 (d_h=16, D=128)
    "tiny": ModelDims("tiny", h_q=4, d_c=64, d_r=16, d_h=16, D=128),
    # odd tiny: catches transposes hidden by tiny's d_c = h_q*d_h coincidence
    "odd": ModelDims("odd", h_q=6, d_c=64, d_r=16, d_h=16, D=96),
    # DeepSeek-V3 attention layer (D=7168 is [ext])
    "dsv3": ModelDims("dsv3", h_q=128, d_c=512, d_r=64, d_h=128, D=7168),
    # Kimi-K2 attention layer: 64 heads, same latent shape
    "kimi": ModelDims("kimi", h_q=64, d_c=512, d_r=64, d_h=128, D=7168),
}


def bf16_bits(x: np.ndarray) -> np.ndarray:
    """fp32 -> bf16 bit patterns, round-to-nearest-even (storage rounding only)."""
    f = np.ascontiguousarray(x, dtype=np.float32)
    u = f.view(np.uint32).astype(np.uint64)
    rounded = (u + 0x7FFF + ((u >> 16) & 1)) >> 16
    return rounded.astype(np.uint16)


def bf16_to_f32(b: np.ndarray) -> np.ndarray:
    """bf16 bit patterns -> fp32 (exact widening)."""
    return (np.ascontiguousarray(b, dtype=np.uint16).astype(np.uint32) << 16).view(np.float32)


def _rng(seed: int, *stream: int) -> np.random.Generator:
    return np.random.default_rng(np.random.SeedSequence([int(seed) & 0xFFFFFFFF, *[int(s) for s in stream]]))


def random_orthogonal(d: int, seed: int) -> np.ndarray:
    """A random orthogonal matrix (QR of a Gaussian, sign-fixed), fp64."""
    a = _rng(seed, 7001).standard_normal((d, d))
    q, r = np.linalg.qr(a)
    return q * np.sign(np.diag(r))[None, :]


def latent_spectrum(d_c: int, n_outlier: int) -> np.ndarray:
    """Per-channel std of the raw latent: power law 1/sqrt(i+1), outliers x10."""
    sig = 1.0 / np.sqrt(np.arange(1, d_c + 1, dtype=np.float64))
    # outliers at fixed, spread-out channels (not the leading ones)
    for t in range(n_outlier):
        sig[(t * d_c) // max(n_outlier, 1) + d_c // (2 * max(n_outlier, 1))] *= 10.0
    return sig


@dataclasses.dataclass
class Weights:
    """Checkpoint-side weights (bf16 bits).  Shapes follow PAPER.md §3.3:
    W_UK, W_UV in R^{4d_h x (h_q d_h)}; W_O in R^{(h_q d_h) x D}; gamma in R^{4d_h}."""
    W_UK: np.ndarray
    W_UV: np.ndarray
    gamma: np.ndarray
    W_O: np.ndarray


def gen_weights(dims: ModelDims, seed: int, *, gamma_one: bool = False) -> Weights:
    r = _rng(seed, 1)
    W_UK = r.standard_normal((dims.d_c, dims.h_q * dims.d_h), dtype=np.float32) / np.float32(np.sqrt(dims.d_h))
    W_UV = r.standard_normal((dims.d_c, dims.h_q * dims.d_h), dtype=np.float32) / np.float32(np.sqrt(dims.d_c))
    if gamma_one:
        gamma = np.ones(dims.d_c, np.float32)
    else:
        gamma = (1.0 + 0.1 * r.standard_normal(dims.d_c)).astype(np.float32)
    W_O = r.standard_normal((dims.h_q * dims.d_h, dims.D), dtype=np.float32) / np.float32(np.sqrt(dims.h_q * dims.d_h))
    return Weights(bf16_bits(W_UK), bf16_bits(W_UV), bf16_bits(gamma), bf16_bits(W_O))


def gen_raw_ckv(dims: ModelDims, n: int, seed: int, seq: int, *, basis: np.ndarray | None = None,
                scale: float = 1.0) -> np.ndarray:
    """Raw (pre-RMSNorm) latent rows for sequence ``seq``: [n, d_c] bf16 bits."""
    r = _rng(seed, 2, seq)
    z = r.standard_normal((n, dims.d_c), dtype=np.float32)
    z *= latent_spectrum(dims.d_c, dims.n_outlier).astype(np.float32)[None, :] * np.float32(scale)
    if basis is not None:
        z = (z.astype(np.float64) @ basis.T).astype(np.float32)
    return bf16_bits(z)


def gen_kpe(dims: ModelDims, n: int, seed: int, seq: int) -> np.ndarray:
    """Post-RoPE shared keys k^PE for sequence ``seq``: [n, d_r] bf16 bits."""
    r = _rng(seed, 3, seq)
    return bf16_bits(r.standard_normal((n, dims.d_r), dtype=np.float32))


def gen_queries(dims: ModelDims, B: int, seed: int, step: int = 0, *, peak: float = 1.0):
    """q_nope [B, h_q, d_h] and post-RoPE q_pe [B, h_q, d_r] (bf16 bits)."""
    r = _rng(seed, 4, step)
    q = r.standard_normal((B, dims.h_q, dims.d_h), dtype=np.float32) * np.float32(peak)
    qpe = r.standard_normal((B, dims.h_q, dims.d_r), dtype=np.float32) * np.float32(peak)
    return bf16_bits(q), bf16_bits(qpe)


def gen_seq_lens(B: int, S: int, seed: int, *, ragged: bool) -> np.ndarray:
    """Uniform lengths S, or ragged U[S/2, S] (SURVEY.md §8(d) "Lengths")."""
    if not ragged:
        return np.full(B, S, np.int32)
    r = _rng(seed, 5)
    return r.integers(max(1, S // 2), S + 1, size=B).astype(np.int32)
