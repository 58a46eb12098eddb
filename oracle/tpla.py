"""Tensor-Parallel Latent Attention decode, step by step (fp64).

TEST INFRASTRUCTURE ONLY.

Follows PAPER.md §4 generalised to (k, g) by §4.4, with the
reparameterisation of §4.1-§4.3:

1. convert (offline): W^UKV_new = Uᵀ W_γ W^UKV; slice latent rows of
   group j and the heads of block i; fold mu_j into the W^UK slice (Condition 2,
   P:256; reading R6: mu scales the NoPE logits only).
2. cache rows: c' = c U; the device's slice c'_j is
   normalised by the sliced RMS sqrt(alpha_j/d_c ||c'_j||² + eps) (SLICED, the
   paper's TPLA), or by the full RMS (EXACT, the PD-separation prefill rows
   P:421, reading R11); the replicated RoPE key rides along.
3. decode per device (Eq. tpla_softmax_one_device): Q'_j = q W^UK'_jᵀ,
   s_t = sm_scale (Q'_j ĉ_{j,t} + q^PE k^PE_t), softmax over this shard only (no
   cross-device statistics), O_j = Σ_t p_t ĉ_{j,t}, Õ_j = O_j W^VO_j
   with W^VO_j kept factored as W^UV'_j then W^O rows.
4. O = AllReduce(Σ_r Õ_r), summed in ascending rank order.
"""
from __future__ import annotations

import dataclasses

import numpy as np

from .numerics import softmax
from .plan import DevicePlan, make_plan

SLICED, EXACT, NONE = "sliced", "exact", "none"


@dataclasses.dataclass
class DeviceWeights:
    """Per-device converted weights (fp64, unrounded)."""
    W_UK: np.ndarray    # [H_loc, W_lat, d_h], mu_j folded in
    W_UV: np.ndarray    # [H_loc, W_lat, d_h]
    W_O: np.ndarray     # [H_loc*d_h, D]  (rows of W^O for this head block)


def reparam_weights(W_UK, W_UV, gamma, U):
    """W^UKV_new = Uᵀ W_γ W^UKV.  Returns (W_UK_new, W_UV_new), [d_c, h_q*d_h]."""
    W_gamma = np.diag(np.asarray(gamma, dtype=np.float64))
    return U.T @ W_gamma @ W_UK, U.T @ W_gamma @ W_UV


def convert_weights(W_UK, W_UV, gamma, W_O, U, plan: DevicePlan, mu_j: float, *, d_h: int) -> DeviceWeights:
    """Offline conversion for one device."""
    W_UK_new, W_UV_new = reparam_weights(W_UK, W_UV, gamma, U)
    rows = slice(plan.lat_begin, plan.lat_end)
    H = plan.h_loc
    uk = np.empty((H, plan.w_lat, d_h))
    uv = np.empty((H, plan.w_lat, d_h))
    for a, h in enumerate(range(plan.head_begin, plan.head_end)):
        cols = slice(h * d_h, (h + 1) * d_h)
        uk[a] = mu_j * W_UK_new[rows, cols]
        uv[a] = W_UV_new[rows, cols]
    wo = W_O[plan.head_begin * d_h:plan.head_end * d_h, :]
    return DeviceWeights(uk, uv, np.array(wo, dtype=np.float64))


def cache_rows(c_raw, k_pe, U, plan: DevicePlan, alpha_j: float, eps: float, mode: str):
    """Device row [ĉ_j ‖ k^PE] for each raw latent row.

    c_raw [n, d_c] pre-norm latents, k_pe [n, d_r] post-RoPE keys.  Returns [n, W_lat + d_r] fp64.
    """
    c_raw = np.asarray(c_raw, dtype=np.float64)
    d_c = c_raw.shape[1]
    c_t = c_raw @ U                                             # c' = c U
    c_j = c_t[:, plan.lat_begin:plan.lat_end]                   # device slice (cU)_j
    if mode == SLICED:                                          # sqrt(alpha/d ||(cU)_j||² + eps)
        r = np.sqrt(alpha_j / d_c * np.sum(c_j * c_j, axis=1) + eps)
    elif mode == EXACT:                                         # sqrt(1/d ||c||² + eps)
        r = np.sqrt(np.sum(c_t * c_t, axis=1) / d_c + eps)
    elif mode == NONE:                                          # layout tests only
        r = np.ones(c_raw.shape[0])
    else:
        raise ValueError(mode)
    return np.concatenate([c_j / r[:, None], np.asarray(k_pe, dtype=np.float64)], axis=1)


def absorb_query(q_nope_b, dw: DeviceWeights):
    """Q'_j[h, :] = W^UK'_j[h] q[h] for the device's heads: [H_loc, W_lat]."""
    return np.einsum("hld,hd->hl", dw.W_UK, q_nope_b)


def shard_attention(Qp, qpe, rows, w_lat: int, sm_scale: float):
    """Attention of one shard for one sequence (Eq. tpla_softmax_one_device P:137-138 with the
    replicated RoPE logits of P:238-242): Qp [H, W_lat] (mu_j included), qpe [H, d_r],
    rows [S, W_lat + d_r].  Returns O [H, W_lat] = softmax(s) ĉ_j, lse [H] = log Σ_t exp(s_t),
    p [H, S] and the RoPE logits [H, S]."""
    c_hat = rows[:, :w_lat]                     # ĉ_j  [S, W_lat]
    kpe = rows[:, w_lat:]                       # k^PE [S, d_r] (replicated)
    nope = Qp @ c_hat.T                         # Q'_j ĉ_jᵀ (mu_j already in Q'_j)
    rope = qpe @ kpe.T                          # q^PE k^PEᵀ, unscaled by mu (R6)
    s = sm_scale * (nope + rope)
    p = softmax(s)                              # per-shard softmax
    smax = np.max(s, axis=1)
    lse = smax + np.log(np.sum(np.exp(s - smax[:, None]), axis=1))
    return p @ c_hat, lse, p, rope


def decode_device(q_nope, q_pe, rows, dw: DeviceWeights, plan: DevicePlan, *, sm_scale, return_parts=False):
    """One device's decode step over a batch (Eq. tpla_softmax_one_device).

    q_nope [B, h_q, d_h] and q_pe [B, h_q, d_r] hold ALL heads (the device takes its block);
    rows: list of B arrays [S_b, W_lat + d_r] (this device's cache rows of each sequence).
    Returns y [B, D] (= Õ_j), and optionally dict(O=[B, H_loc, W_lat], P=list of [H_loc, S_b],
    rope_logits=list of [H_loc, S_b]).
    """
    B = q_nope.shape[0]
    W_lat = plan.w_lat
    H = plan.h_loc
    d_h = dw.W_UK.shape[2]
    D = dw.W_O.shape[1]
    y = np.zeros((B, D))
    O_all = np.zeros((B, H, W_lat))
    P_all, R_all = [], []
    heads = slice(plan.head_begin, plan.head_end)
    for b in range(B):
        Qp = absorb_query(q_nope[b, heads], dw)     # Q'_j [H, W_lat]
        O, _, p, rope = shard_attention(Qp, q_pe[b, heads], rows[b], W_lat, sm_scale)   # O_j [H, W_lat]
        v = np.einsum("hl,hld->hd", O, dw.W_UV)     # O_j W^UV'_j per head   [H, d_h]
        y[b] = v.reshape(H * d_h) @ dw.W_O          # Õ_j = O_j W^VO_j
        O_all[b] = O
        P_all.append(p)
        R_all.append(rope)
    if return_parts:
        return y, dict(O=O_all, P=P_all, rope_logits=R_all)
    return y


def all_reduce(parts):
    """O = AllReduce(Σ_r Õ_r): fixed ascending-rank summation."""
    acc = np.zeros_like(parts[0])
    for p in parts:
        acc = acc + p
    return acc


@dataclasses.dataclass
class Problem:
    """All fp64 inputs of one TPLA decode step (what the caller hands the library)."""
    W_UK: np.ndarray
    W_UV: np.ndarray
    gamma: np.ndarray
    W_O: np.ndarray
    U: np.ndarray
    alpha: np.ndarray   # [g]
    mu: np.ndarray      # [g]
    c_raw: list         # B arrays [S_b, d_c]
    k_pe: list          # B arrays [S_b, d_r]
    modes: list         # B arrays of row modes (SLICED / EXACT / NONE), one per token
    q_nope: np.ndarray  # [B, h_q, d_h]
    q_pe: np.ndarray    # [B, h_q, d_r]
    h_q: int
    d_h: int
    eps: float
    sm_scale: float


def device_rows(pb: Problem, plan: DevicePlan, alpha_j: float, *, round_rows=None):
    """Cache rows of every sequence for one device, row mode per token."""
    out = []
    for b in range(len(pb.c_raw)):
        modes = pb.modes[b]
        rows = np.empty((pb.c_raw[b].shape[0], plan.row_width))
        for m in set(modes):
            sel = np.array([mm == m for mm in modes])
            rows[sel] = cache_rows(pb.c_raw[b][sel], pb.k_pe[b][sel], pb.U, plan, alpha_j, pb.eps, m)
        if round_rows is not None:
            rows = round_rows(rows)
        out.append(rows)
    return out


def tpla_decode_step(pb: Problem, k: int, g: int, *, round_rows=None, return_parts=False):
    """Full step over all k devices + all-reduce.  Returns o [B, D] (and per-rank parts)."""
    d_c, d_r = pb.U.shape[0], pb.k_pe[0].shape[1]
    ys, parts = [], []
    for r in range(k):
        plan = make_plan(k, g, pb.h_q, d_c, d_r, r)
        dw = convert_weights(pb.W_UK, pb.W_UV, pb.gamma, pb.W_O, pb.U, plan, pb.mu[plan.shard], d_h=pb.d_h)
        rows = device_rows(pb, plan, pb.alpha[plan.shard], round_rows=round_rows)
        y, pr = decode_device(pb.q_nope, pb.q_pe, rows, dw, plan, sm_scale=pb.sm_scale, return_parts=True)
        pr["rows"] = rows
        pr["plan"] = plan
        ys.append(y)
        parts.append(pr)
    o = all_reduce(ys)
    return (o, ys, parts) if return_parts else o


def tpla_decode_exact_logits(pb: Problem, g: int, *, round_rows=None):
    """Exact-softmax variant (SURVEY.md pin c10; the all-gather / row-parallel route of
    P:232-236 and the "norm only" ablation): partial NoPE logits of the g shards are
    summed (mu = 1) BEFORE one softmax; RoPE logits added once.  k = g (one device per shard)."""
    d_c, d_r = pb.U.shape[0], pb.k_pe[0].shape[1]
    plans = [make_plan(g, g, pb.h_q, d_c, d_r, r) for r in range(g)]
    dws = [convert_weights(pb.W_UK, pb.W_UV, pb.gamma, pb.W_O, pb.U, pl, 1.0, d_h=pb.d_h) for pl in plans]
    rows = [device_rows(pb, pl, pb.alpha[pl.shard], round_rows=round_rows) for pl in plans]   # (R19: bf16 cache)
    B = pb.q_nope.shape[0]
    out = np.zeros((B, pb.W_O.shape[1]))
    for b in range(B):
        logits = 0.0
        for j, pl in enumerate(plans):
            Qp = absorb_query(pb.q_nope[b], dws[j])                   # all heads (k = g)
            logits = logits + Qp @ rows[j][b][:, :pl.w_lat].T          # Σ_j Q'_j ĉ_jᵀ
        logits = logits + pb.q_pe[b] @ rows[0][b][:, plans[0].w_lat:].T
        p = softmax(pb.sm_scale * logits)
        for j, pl in enumerate(plans):
            O = p @ rows[j][b][:, :pl.w_lat]
            v = np.einsum("hl,hld->hd", O, dws[j].W_UV)
            out[b] += v.reshape(-1) @ dws[j].W_O                      # X1 A1 + X2 A2
    return out


def gla_decode_step(pb: Problem, g: int, *, mu=None):
    """MLA -> GLA conversion (§3.2; contrast of §4.4 P:334 and Fig. 3):
    the latent axis is cut into g shards AND the heads into g blocks; device i keeps only the
    diagonal block — heads block i attend to latent shard i alone (Q_{i,i}, W^VO_{i,i}), each
    shard normalised by its own RMSNorm (the sliced RMS of the shard, i.e. the SLICED
    rows with alpha = g), its own softmax, and O = AllReduce(Σ_i Õ_i).  The off-diagonal
    blocks Q_{i,j}, j != i, do not contribute ("unable to access the off-diagonal head slices",
    P:334).  mu: NoPE logit scale per shard (default 1: the GLA equations carry none).
    Device i is the TPLA plan of rank i at (k = g, g) restricted to heads block i of g."""
    d_c, d_r = pb.U.shape[0], pb.k_pe[0].shape[1]
    mu = np.ones(g) if mu is None else np.asarray(mu, float)
    ys = []
    for i in range(g):
        full = make_plan(g, g, pb.h_q, d_c, d_r, i)                 # latent shard i, all heads
        h_blk = pb.h_q // g
        plan = DevicePlan(i, i, i, i * h_blk, (i + 1) * h_blk, full.lat_begin, full.lat_end, full.row_width)
        dw = convert_weights(pb.W_UK, pb.W_UV, pb.gamma, pb.W_O, pb.U, plan, mu[i], d_h=pb.d_h)
        rows = device_rows(pb, plan, pb.alpha[i])
        ys.append(decode_device(pb.q_nope, pb.q_pe, rows, dw, plan, sm_scale=pb.sm_scale))
    return all_reduce(ys)
