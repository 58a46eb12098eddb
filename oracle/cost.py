"""Per-device KV widths, bytes and attention FLOPs (§1, §4.5, §5.4.1).

TEST INFRASTRUCTURE ONLY.  Integer arithmetic, exact.
"""
from __future__ import annotations


def kv_width_mla(d_c: int, d_r: int) -> int:
    """MLA replicates the whole latent + RoPE key on every device: "64 + 512 = 576"."""
    return d_c + d_r


def kv_width_tpla(d_c: int, d_r: int, g: int) -> int:
    """TPLA keeps a d_c/g latent slice plus the replicated RoPE key: "(64+256)"."""
    return d_c // g + d_r


def kv_width_gqa(n_kv_heads: int, d_h: int, k: int) -> int:
    """GQA K+V per token per device: 2 × kv_heads × d_h / TP, e.g. 2×8×128 = 2048 → 512 at TP=4."""
    return 2 * n_kv_heads * d_h // k


def nope_flops_tpla(L_q: int, S: int, h_q: int, d_h: int, g: int) -> int:
    """O(L_q × S × h_q × (4d_h/g) × 2) per device (P:363 for g = 2: h_q × 2d_h × 2)."""
    return L_q * S * h_q * (4 * d_h // g) * 2


def nope_flops_mla(L_q: int, S: int, h_q: int, d_h: int, k: int) -> int:
    """O(L_q × S × (h_q/k) × 4d_h × 2) per device (P:363 for k = 2)."""
    return L_q * S * (h_q // k) * 4 * d_h * 2


def decode_attention_flops(S_total: int, h_loc: int, w_lat: int, d_r: int) -> int:
    """Multiply-add count ×2 of one device's absorbed decode attention over S_total cached tokens:
    QKᵀ over [latent slice ‖ RoPE] (w_lat + d_r) plus PV over the latent slice (w_lat)."""
    return 2 * S_total * h_loc * (2 * w_lat + d_r)


def decode_cache_bytes(S_total: int, w_lat: int, d_r: int, elem_bytes: int = 2) -> int:
    """Bytes of cache one device must read per decode step ("reading the entire ... KV cache")."""
    return S_total * (w_lat + d_r) * elem_bytes
