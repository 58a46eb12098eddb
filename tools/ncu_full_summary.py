"""Summarise an 'ncu --set full' raw CSV export (one row per profiled launch) as markdown, and
write profiles/ncu_traffic.json (DRAM bytes per launch by library kernel name, read by bench.py
for roofline.traffic).
    python tools/ncu_full_summary.py gpurun_out/prof_full_raw.csv WORKLOAD > profiles/rNN_ncu_full.md"""
import csv
import json
import os
import re
import sys

NAMES = {"attn_tc_kernel": "K3_attn_tc", "skinny_tc_kernel": "K5_W_O_tc", "combine_wuv_kernel": "K45_combine_W_UV",
         "attn_plan_kernel": "K3p_attn_plan", "nt_gemm_kernel": "K2_absorb_q", "pre_attn_kernel": "K3p_K2_pre_attn", "attn_fwd_causal_kernel": "K8_prefill_fa",
         "gemm_tn_kernel": "K9_prefill_gemm"}
METRICS = [
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "DRAM throughput % of peak"),
    ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed", "tensor pipe active % (elapsed)"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM throughput %"),
    ("lts__t_sector_hit_rate.pct", "L2 hit rate %"),
    ("sm__cycles_elapsed.avg.per_second", "SM clock"),
    ("launch__registers_per_thread", "registers/thread"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
]
SCALE = {"Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "byte": 1.0}

rows = list(csv.reader(open(sys.argv[1])))
workload = sys.argv[2] if len(sys.argv) > 2 else "c1"
hdr, units, data = rows[0], rows[1], rows[2:]
ki = hdr.index("Kernel Name")
stall_cols = [i for i, h in enumerate(hdr) if re.match(r"smsp__average_warps_issue_stalled_.*_per_issue_active.ratio$", h)]
traffic = {}
print("| metric | " + " | ".join(NAMES.get(re.search(r"::(\w+)", r[ki]).group(1), r[ki][:30]) for r in data) + " |")
print("|---|" + "---|" * len(data))
for m, label in METRICS:
    if m not in hdr:
        continue
    i = hdr.index(m)
    print(f"| {label} ({units[i]}) | " + " | ".join(r[i] for r in data) + " |")
for r in data:
    short = re.search(r"::(\w+)", r[ki]).group(1)
    name = NAMES.get(short, short)
    rb = float(r[hdr.index("dram__bytes_read.sum")]) * SCALE.get(units[hdr.index("dram__bytes_read.sum")], 1)
    wb = float(r[hdr.index("dram__bytes_write.sum")]) * SCALE.get(units[hdr.index("dram__bytes_write.sum")], 1)
    traffic[name] = {"workload": workload, "dram_bytes_per_launch": rb + wb, "dram_read": rb, "dram_write": wb,
                     "source": os.path.basename(sys.argv[1])}
print()
print("Top issue-stall reasons (warps stalled per issued instruction):")
print()
for r in data:
    short = re.search(r"::(\w+)", r[ki]).group(1)
    st = sorted(((float(r[i] or 0), re.sub(r"smsp__average_warps_issue_stalled_|_per_issue_active.ratio", "", hdr[i]))
                 for i in stall_cols), reverse=True)[:5]
    print(f"- {NAMES.get(short, short)}: " + ", ".join(f"{n} {v:.2f}" for v, n in st))
out = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "profiles", "ncu_traffic.json")
json.dump(traffic, open(out, "w"), indent=1)
