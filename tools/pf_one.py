"""One non-absorbed MLA prefill forward (K8/K9) of a 4K prompt, DSV3 heads split over 2 devices (rank 0)
for ncu captures:  ncu --kernel-name regex:attn_fwd -c 1 python tools/pf_one.py"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402
from paper_2508_15881_b200.runtime import LayerSpec, PrefillRank  # noqa: E402

L = int(os.environ.get("PF_L", "4096"))
dev = torch.device("cuda:0")
dims = synth.PRESETS["dsv3"]
w = synth.gen_weights(dims, 7)
pr = PrefillRank(LayerSpec(dims.h_q, dims.d_c, dims.d_r, dims.d_h, dims.D), k=2, rank=0, max_len=L, device=dev)
pr.convert(w.W_UK, w.W_UV, w.gamma, w.W_O)
g = torch.Generator(device=dev)
g.manual_seed(7)
ck = torch.randn((L, dims.d_c), generator=g, device=dev).to(torch.bfloat16)
kp = torch.randn((L, dims.d_r), generator=g, device=dev).to(torch.bfloat16)
q = torch.randn((L, dims.h_q, dims.d_h), generator=g, device=dev).to(torch.bfloat16)
qp = torch.randn((L, dims.h_q, dims.d_r), generator=g, device=dev).to(torch.bfloat16)
y = torch.zeros((L, dims.D), dtype=torch.float32, device=dev)
for _ in range(2):
    pr.forward(ck, kp, q, qp, y)
torch.cuda.synchronize()
print("PF OK")
