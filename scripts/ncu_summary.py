#!/usr/bin/env python
"""Summarise an `ncu --set full` report (per kernel launch): duration, DRAM traffic, tensor-pipe
activity, SM / L2 throughput.  usage: python scripts/ncu_summary.py REPORT.ncu-rep > out.md"""
import csv
import io
import subprocess
import sys

M = [("gpu__time_duration.sum", "dur_us", 1e-3),
     ("dram__bytes_read.sum", "dram_rd_MB", 1e-6),
     ("dram__bytes_write.sum", "dram_wr_MB", 1e-6),
     ("lts__t_bytes.sum", "l2_MB", 1e-6),
     ("l1tex__m_xbar2l1tex_read_bytes_mem_global_op_tma_ld.sum", "tma_ld_MB", 1e-6),
     ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed", "tensor_pct", 1),
     ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active", "tensor_act_pct", 1),
     ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "sm_pct", 1),
     ("FBSP.TriageCompute.dram__throughput.avg.pct_of_peak_sustained_elapsed", "dram_pct", 1),
     ("launch__grid_size", "grid", 1),
     ("launch__registers_per_thread", "regs", 1)]

out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr, units, data = rows[0], rows[1], rows[2:]
idx = {h: i for i, h in enumerate(hdr)}
print("| kernel | " + " | ".join(n for _, n, _ in M) + " |")
print("|---|" + "---|" * len(M))
for r in data:
    name = r[idx["Kernel Name"]].split("(")[0].replace("void ", "")[:70]
    vals = []
    for key, _, sc in M:
        i = idx.get(key)
        if i is None or not r[i]:
            vals.append("-")
            continue
        try:
            v = float(r[i].replace(",", ""))
        except ValueError:
            vals.append("-")
            continue
        u = units[i]
        if key == "gpu__time_duration.sum" and u == "us":
            sc = 1
        if key.endswith("bytes_read.sum") or key.endswith("bytes_write.sum") or key.endswith("bytes.sum") or "tma_ld" in key:
            mult = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(u, 1)
            v *= mult
        vals.append(f"{v * sc:.2f}" if sc != 1 else f"{v:.1f}")
    print(f"| {name} | " + " | ".join(vals) + " |")
