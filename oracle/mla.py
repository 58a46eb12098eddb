"""Multi-head Latent Attention decode, two independent formulations (fp64).

TEST INFRASTRUCTURE ONLY.

* ``mla_decode_full``: the non-absorbed pipeline with decoupled RoPE, Eq.
  isolate_rope (§3.3): keys and values are materialised per
  head from the normalised latent, k = ĉ W^UK, v = ĉ W^UV (right-multiplied,
  reading R9), logits (q kᵀ + q^PE k^PEᵀ)·sm_scale.
* ``mla_decode_absorbed``: Eq. mla_softmax / mla (§3.1) after the
  absorption of §3.3: Q = q W^UKᵀ attends directly to ĉ, and the
  output goes through W^VO kept factored as W^UV then W^O (reading R10).

The queries q (= c^Q W^UQ) and q^PE (= RoPE(c^Q W^QR)) and the post-RoPE key
k^PE are inputs: the projections before them are the caller's.
Softmax scale ``sm_scale`` is one scalar for NoPE and RoPE logits (reading R1).
"""
from __future__ import annotations

import numpy as np

from .numerics import rmsnorm, softmax


def mla_decode_full(q_nope, q_pe, c_raw, k_pe, W_UK, W_UV, gamma, W_O, *, h_q, d_h, eps, sm_scale):
    """One decode token of one sequence.

    q_nope [h_q, d_h], q_pe [h_q, d_r], c_raw [S, d_c] (pre-norm c^KV), k_pe [S, d_r],
    W_UK, W_UV [d_c, h_q*d_h], gamma [d_c], W_O [h_q*d_h, D].  Returns (out [D], p [h_q, S]).
    """
    c_hat = rmsnorm(gamma, c_raw, eps)                 # ĉ = RMSNorm(c^KV)
    k = c_hat @ W_UK                                   # k = ĉ W^UK
    v = c_hat @ W_UV                                   # v = ĉ W^UV (R9)
    S = c_raw.shape[0]
    O = np.zeros(h_q * d_h)
    P = np.zeros((h_q, S))
    for h in range(h_q):
        kh = k[:, h * d_h:(h + 1) * d_h]               # [S, d_h]
        vh = v[:, h * d_h:(h + 1) * d_h]
        logits = (kh @ q_nope[h] + k_pe @ q_pe[h]) * sm_scale   # (q kᵀ + q^PE k^PEᵀ)/√(d_h+d_r)
        p = softmax(logits)
        P[h] = p
        O[h * d_h:(h + 1) * d_h] = p @ vh              # softmax(...) v
    return O @ W_O, P                                  # Õ = O W^O


def mla_decode_absorbed(q_nope, q_pe, c_raw, k_pe, W_UK, W_UV, gamma, W_O, *, h_q, d_h, eps, sm_scale):
    """Absorbed form: O_h = softmax(Q_h ĉᵀ·scale + RoPE) ĉ, Õ = Σ_h O_h W^UV_h W^O_h.

    Same arguments/return as ``mla_decode_full``; also returns O [h_q, d_c].
    """
    c_hat = rmsnorm(gamma, c_raw, eps)                 # ĉ^KV = RMSNorm(c^KV)
    D = W_O.shape[1]
    out = np.zeros(D)
    S, d_c = c_raw.shape
    P = np.zeros((h_q, S))
    O_lat = np.zeros((h_q, d_c))
    for h in range(h_q):
        W_UK_h = W_UK[:, h * d_h:(h + 1) * d_h]        # [d_c, d_h]
        Q_h = W_UK_h @ q_nope[h]                       # Q = q W^UKᵀ (absorbed)
        logits = (c_hat @ Q_h + k_pe @ q_pe[h]) * sm_scale
        p = softmax(logits)                            # Eq. mla_softmax
        P[h] = p
        O_h = p @ c_hat                                # O = softmax(·) ĉ
        O_lat[h] = O_h
        W_VO_h = W_UV[:, h * d_h:(h + 1) * d_h] @ W_O[h * d_h:(h + 1) * d_h, :]   # W^VO (factored)
        out += O_h @ W_VO_h                            # Õ = O W^VO
    return out, P, O_lat
