"""SM clock and power while K3 runs back to back (is K3 power-capped?).

    python tools/k3_clock_probe.py [--workload c1] [--seconds 3]

Builds one rank of the workload (random cache), replays a CUDA graph of 20 K3 launches for about
--seconds, samples NVML SM clock / power / throttle reasons meanwhile, and prints the K3 time per
launch together with the median clock, so time can be converted to cycles."""
import argparse
import os
import sys
import threading
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import synth  # noqa: E402
from paper_2508_15881_b200 import _abi as abi  # noqa: E402
from paper_2508_15881_b200.runtime import LayerSpec, TplaRank  # noqa: E402

WL = {"c1": ("dsv3", 32, 32768, 2), "c3": ("dsv3", 16, 131072, 8), "h8": ("dsv3", 32, 32768, 8),
      "c2": ("kimi", 64, 32768, 4)}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="c1", choices=sorted(WL))
    ap.add_argument("--seconds", type=float, default=3.0)
    a = ap.parse_args()
    model, B, S, g = WL[a.workload]
    dims = synth.PRESETS[model]
    dev = torch.device("cuda:0")
    r = TplaRank(LayerSpec(dims.h_q, dims.d_c, dims.d_r, dims.d_h, dims.D), k=g, g=g, rank=0, batch=B,
                 max_seq_len=S, device=dev)
    r.cache_buf.copy_(torch.randn(r.cache_buf.shape, device=dev).to(torch.bfloat16))
    pl = r.plan
    q = torch.randn((B, pl.h_loc, pl.w_lat), device=dev).to(torch.bfloat16)
    qpe = torch.randn((B, dims.h_q, dims.d_r), device=dev).to(torch.bfloat16)
    lens = torch.full((B,), S, dtype=torch.int32, device=dev)
    for _ in range(3):
        r.decode_attention(q, qpe, lens, None)
    torch.cuda.synchronize()
    graph = torch.cuda.CUDAGraph()
    with torch.cuda.graph(graph):
        for _ in range(20):
            r.decode_attention(q, qpe, lens, None)
    import pynvml
    pynvml.nvmlInit()
    h = pynvml.nvmlDeviceGetHandleByIndex(0)
    clocks, power, reasons = [], [], 0
    stop = threading.Event()

    def sample():
        nonlocal reasons
        while not stop.is_set():
            clocks.append(pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM))
            power.append(pynvml.nvmlDeviceGetPowerUsage(h) / 1000.0)
            reasons |= pynvml.nvmlDeviceGetCurrentClocksEventReasons(h)
            time.sleep(0.002)

    t = threading.Thread(target=sample, daemon=True)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    n = 0
    t.start()
    e0.record()
    t_end = time.time() + a.seconds
    while time.time() < t_end:
        graph.replay()
        n += 20
        if n % 200 == 0:
            torch.cuda.synchronize()
    e1.record()
    torch.cuda.synchronize()
    stop.set()
    t.join()
    us = e0.elapsed_time(e1) * 1e3 / n
    mhz = float(np.median(clocks[len(clocks) // 4:]))
    bytes_ = B * S * pl.row_width * 2
    print(f"{a.workload}: K3 {us:.1f} us/launch  {bytes_ / us / 1e3:.0f} GB/s  SM clock median {mhz:.0f} MHz "
          f"(= {us * mhz:.0f} cycles/launch)  power median {np.median(power):.0f} W max {max(power):.0f} W  "
          f"reasons 0x{reasons:x}")


if __name__ == "__main__":
    main()
