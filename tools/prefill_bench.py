"""prefill attention time of one prompt, PD-separated MLA prefill (g = 1, heads split
over k) against TPLA prefill (g = k), DSV3 shape, both ranks of the TP group on this GPU
(per-device time = total / k).  The paper reports TTFT 1.4x in favour of the PD-separated MLA
prefill at 1K context (its hardware); this measures the attention + up-projection
part of the prefill on B200 (the K1 cache write of the prompt included, MoE/FFN excluded).

    python tools/prefill_bench.py [--L 1024 4096] [--k 2] [--iters 20]
"""
import argparse
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402
from paper_2508_15881_b200 import abi  # noqa: E402
from paper_2508_15881_b200.runtime import LayerSpec, TplaRank  # noqa: E402


def run(L, k, g, iters, dev):
    dims = synth.PRESETS["dsv3"]
    spec = LayerSpec(dims.h_q, dims.d_c, dims.d_r, dims.d_h, dims.D)
    w = synth.gen_weights(dims, 7)
    gen = torch.Generator(device=dev)
    gen.manual_seed(7)
    sig = torch.tensor(synth.latent_spectrum(dims.d_c, dims.n_outlier), dtype=torch.float32, device=dev)
    ck = (torch.randn((L, dims.d_c), generator=gen, device=dev) * sig).to(torch.bfloat16)
    kp = torch.randn((L, dims.d_r), generator=gen, device=dev).to(torch.bfloat16)
    q = torch.randn((L, dims.h_q, dims.d_h), generator=gen, device=dev).to(torch.bfloat16)
    qp = torch.randn((L, dims.h_q, dims.d_r), generator=gen, device=dev).to(torch.bfloat16)
    seq = torch.zeros(L, dtype=torch.int32, device=dev)
    pos = torch.arange(L, dtype=torch.int32, device=dev)
    xf = abi.XFORM_HADAMARD if g > 1 else abi.XFORM_IDENTITY
    ranks = []
    for r in range(k):
        rk = TplaRank(spec, k=k, g=g, rank=r, batch=1, max_seq_len=L, device=dev)
        rk.convert(w.W_UK, w.W_UV, w.gamma, w.W_O, xform=xf, sign_seed=7)
        ranks.append(rk)
    y = torch.zeros((L, dims.D), dtype=torch.float32, device=dev)
    out = torch.empty((L, dims.D), dtype=torch.bfloat16, device=dev)

    def step():
        for j, rk in enumerate(ranks):
            rk.prefill(ck, kp, seq, pos)                       # K1: the prompt's rows (EXACT)
            rk.prefill_attention(q, qp, 0, y, out if j == k - 1 else None, accumulate=j > 0)

    for _ in range(3):
        step()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(iters):
        step()
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / iters
    return {"L": L, "k": k, "g": g, "us_all_ranks": ms * 1e3, "us_per_device": ms * 1e3 / k,
            "prompt_tokens_per_s_per_device": L / (ms / k / 1e3)}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--L", type=int, nargs="+", default=[1024, 4096])
    ap.add_argument("--k", type=int, default=2)
    ap.add_argument("--iters", type=int, default=20)
    a = ap.parse_args()
    dev = torch.device("cuda:0")
    rows = []
    for L in a.L:
        mla = run(L, a.k, 1, a.iters, dev)
        tp = run(L, a.k, a.k, a.iters, dev)
        rows.append({"L": L, "mla_pdsep": mla, "tpla": tp, "tpla_over_mla_time": tp["us_per_device"] / mla["us_per_device"]})
        print(json.dumps(rows[-1]), flush=True)


if __name__ == "__main__":
    main()
