"""Baseline fairness (verdict r1 item 9): the replicated-MLA (g = 1) decode attention of this library
(K3p + the CTA-pair tcgen05 K3 + K4) against flashinfer's sm100 MLA decode (trtllm-gen backend), same
shape, same bf16 cache contents, same queries: DeepSeek-V3 absorbed MLA, latent 512 + RoPE 64, 32K
context, batch 32, with all 128 heads on one device (mla1) and 64 (the paper's MLA TP = 2, mla2).
Also ONE TPLA shard of configs[1] (g = 2: latent 256 + 64, 128 heads), which flashinfer's kernel runs
too (kv_lora_rank 256).  Reports µs per launch, the HBM fraction of each, and the max row error
between the two outputs (an independent cross-check of K3).
flashinfer is LIBRARY code (timed here as a comparison only; nothing in the product calls it).

    python tools/flashinfer_mla.py [--B 32] [--S 32768]
"""
import argparse
import json
import math
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402
from paper_2508_15881_b200.runtime import LayerSpec, TplaRank  # noqa: E402


def timed(fn, iters=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(iters):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) * 1e3 / iters


def run(B, S, H, hbm, gg=1):
    """gg = 1: the replicated-MLA baseline (latent 512); gg = 2: ONE TPLA shard (latent 256, the c1 K3)."""
    dev = torch.device("cuda:0")
    dims = synth.PRESETS["dsv3"]
    k = dims.h_q // H * gg
    wl = 512 // gg
    rk = TplaRank(LayerSpec(dims.h_q, dims.d_c, dims.d_r, dims.d_h, dims.D), k=k, g=gg, rank=0, batch=B,
                  max_seq_len=S, device=dev)
    g = torch.Generator(device=dev)
    g.manual_seed(11)
    rk.cache_buf[..., :wl + 64].normal_(generator=g)
    q_lat = torch.randn((B, H, wl), generator=g, device=dev).to(torch.bfloat16)
    q_pe_all = torch.randn((B, dims.h_q, 64), generator=g, device=dev).to(torch.bfloat16)
    lens = torch.full((B,), S, dtype=torch.int32, device=dev)
    scale = 1.0 / math.sqrt(dims.d_h + dims.d_r)
    O = torch.empty((B, H, wl), dtype=torch.float32, device=dev)
    us_ours = timed(lambda: rk.decode_attention(q_lat, q_pe_all, lens, O))
    nbytes = B * S * (wl + 64) * 2
    res = {"B": B, "S": S, "heads": H, "latent": wl, "tpla_lib_us": us_ours, "tpla_lib_hbm_frac": nbytes / (us_ours * 1e-6) / 1e9 / hbm}
    try:
        import flashinfer.mla as fm
        q = torch.cat([q_lat, q_pe_all[:, :H]], dim=-1).unsqueeze(1).contiguous()      # [B, 1, H, 576]
        kv = rk.cache_buf[..., :wl + 64]                                                 # [pages, 64, W]
        if rk.row_stride != wl + 64:
            kv = kv.contiguous()
        ws = torch.zeros(256 * 1024 * 1024, dtype=torch.uint8, device=dev)

        def fi():
            return fm.trtllm_batch_decode_with_kv_cache_mla(q, kv, ws, 128, wl, 64, rk.block_table, lens, S,
                                                            bmm1_scale=scale, bmm2_scale=1.0)
        ref = fi().float().squeeze(1)
        us_fi = timed(fi)
        torch.cuda.synchronize()
        err = ((O - ref).abs().amax(-1) / ref.abs().amax(-1)).max().item()
        res.update({"flashinfer_trtllm_us": us_fi, "flashinfer_hbm_frac": nbytes / (us_fi * 1e-6) / 1e9 / hbm,
                    "max_row_rel_diff": err, "tpla_lib_over_flashinfer_time": us_ours / us_fi})
    except Exception as e:                                   # (no cubins offline, API drift, ...)
        res["flashinfer"] = f"unavailable: {type(e).__name__}: {str(e)[:300]}"
    return res


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--B", type=int, default=32)
    ap.add_argument("--S", type=int, default=32768)
    a = ap.parse_args()
    hbm = 6553.6
    try:
        hbm = json.load(open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                                          "MEASURED_PEAKS.json")))["hbm_gbs"]
    except Exception:
        pass
    for H in (128, 64):
        print(json.dumps(run(a.B, a.S, H, hbm)), flush=True)
    print(json.dumps(run(a.B, a.S, 128, hbm, gg=2)), flush=True)     # the TPLA c1 shard itself


if __name__ == "__main__":
    main()
