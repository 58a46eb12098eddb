"""Small decode steps for compute-sanitizer (memcheck / racecheck / synccheck): K1 (Hadamard, sliced),
K3p, K2, K3 at W_lat 64 (g = 8, split issuers + ping-pong softmax), 256 (g = 2) and 512 (g = 1, CTA
pairs with the DSMEM logit exchange), K45, the tcgen05 W^O GEMM K5 and its reduce, the co-located
sum (tpla_project_out_sum), and the legacy mma.sync shapes (tiny).  Every output is checked finite.

    compute-sanitizer --tool racecheck python tools/sanitize_cases.py
"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402
from paper_2508_15881_b200 import abi  # noqa: E402
from paper_2508_15881_b200.runtime import LayerSpec, TplaRank, bf16_from_bits  # noqa: E402


def case(dname, k, g, S_list, shared):
    d = torch.device("cuda:0")
    dims = synth.PRESETS[dname]
    B = len(S_list)
    spec = LayerSpec(dims.h_q, dims.d_c, dims.d_r, dims.d_h, dims.D)
    w = synth.gen_weights(dims, 3)
    q, qpe = synth.gen_queries(dims, B, 4)
    q, qpe = bf16_from_bits(q, d), bf16_from_bits(qpe, d)
    seq = torch.from_numpy(np.concatenate([np.full(S, b, np.int32) for b, S in enumerate(S_list)])).to(d)
    pos = torch.from_numpy(np.concatenate([np.arange(S, dtype=np.int32) for S in S_list])).to(d)
    ck = bf16_from_bits(np.concatenate([synth.gen_raw_ckv(dims, S, 5, b) for b, S in enumerate(S_list)]), d)
    kp = bf16_from_bits(np.concatenate([synth.gen_kpe(dims, S, 5, b) for b, S in enumerate(S_list)]), d)
    lens = torch.tensor(S_list, dtype=torch.int32, device=d)
    y = torch.zeros((B, dims.D), dtype=torch.float32, device=d)
    out = torch.empty((B, dims.D), dtype=torch.bfloat16, device=d)
    ranks = []
    for r in range(k):
        rk = TplaRank(spec, k=k, g=g, rank=r, batch=B, max_seq_len=max(S_list), device=d, page_perm_seed=r)
        rk.convert(w.W_UK, w.W_UV, w.gamma, w.W_O, xform=abi.XFORM_HADAMARD, sign_seed=9)
        rk.append(ck, kp, seq, pos, abi.RMS_SLICED)
        ranks.append(rk)
    if shared:
        vs = [torch.zeros(ranks[0].v_acc_shape(B), dtype=torch.float32, device=d) for _ in ranks]
        for rk, v in zip(ranks, vs):
            rk.decode_v(q, qpe, lens, v)
        ranks[0].project_out_sum(vs, y, out)
    else:
        for j, rk in enumerate(ranks):
            rk.decode(q, qpe, lens, y, out if j == k - 1 else None, accumulate=j > 0)
    abi.tpla_sync(0)
    assert torch.isfinite(y).all() and y.abs().max() > 0, (dname, k, g)
    print(f"{dname} k={k} g={g} S={S_list} shared={shared}: ok")


if __name__ == "__main__":
    case("tiny", 2, 2, [77, 130], False)
    case("dsv3", 2, 2, [129, 300], False)
    case("dsv3", 8, 8, [200, 65], True)
    case("dsv3", 1, 1, [257, 64], False)
    print("SANITIZE CASES OK")
