"""Scalar building blocks of the oracle (fp64).  TEST INFRASTRUCTURE ONLY."""
from __future__ import annotations

import numpy as np

MASK64 = (1 << 64) - 1


def bf16_to_f64(bits: np.ndarray) -> np.ndarray:
    """Widen bf16 bit patterns to float64 (exact)."""
    u = np.asarray(bits, dtype=np.uint16).astype(np.uint32) << 16
    return u.view(np.float32).astype(np.float64)


def round_bf16(x: np.ndarray) -> np.ndarray:
    """Round float64 values to the nearest bf16 value (ties to even), returned as float64.

    Done in two exact steps: fp64 -> fp32 would double-round, so the rounding is
    taken directly on the fp64 mantissa: keep 8 significant bits.
    """
    x = np.asarray(x, dtype=np.float64)
    m, e = np.frexp(x)                 # x = m * 2^e, 0.5 <= |m| < 1
    scaled = m * 256.0                 # 8 significant bits in the integer part
    r = np.round(scaled)               # numpy rounds half to even
    return np.ldexp(r / 256.0, e)


def rms(x: np.ndarray, eps: float) -> np.ndarray:
    """RMS(x) = sqrt(1/d * sum_i x_i^2 + eps) over the last axis (§4.1)."""
    x = np.asarray(x, dtype=np.float64)
    d = x.shape[-1]
    return np.sqrt(np.sum(x * x, axis=-1) / d + eps)


def rmsnorm(gamma: np.ndarray, x: np.ndarray, eps: float) -> np.ndarray:
    """RMSNorm(gamma, x) = x / RMS(x) ⊙ gamma (§4.1)."""
    return x / rms(x, eps)[..., None] * np.asarray(gamma, dtype=np.float64)


def softmax(s: np.ndarray) -> np.ndarray:
    """softmax over the last axis; the max shift is the usual exact rewrite of
    exp(s_t) / sum_u exp(s_u)."""
    s = np.asarray(s, dtype=np.float64)
    z = np.exp(s - np.max(s, axis=-1, keepdims=True))
    return z / np.sum(z, axis=-1, keepdims=True)


def splitmix64(seed: int, n: int) -> list[int]:
    """The first ``n`` outputs of SplitMix64 seeded with ``seed`` (Steele, Lea &
    Flood 2014; Vigna's reference C).  Used to draw the random ±1 diagonal D of
    the Hadamard reparameterisation (§4.3.1, reading G7)."""
    out = []
    state = seed & MASK64
    for _ in range(n):
        state = (state + 0x9E3779B97F4A7C15) & MASK64
        z = state
        z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & MASK64
        z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & MASK64
        z = z ^ (z >> 31)
        out.append(z)
    return out


def sign_vector(seed: int, d: int) -> np.ndarray:
    """s_i = -1 if the top bit of splitmix64 output i is set, else +1 (reading R7)."""
    return np.array([-1.0 if (z >> 63) else 1.0 for z in splitmix64(seed, d)], dtype=np.float64)
