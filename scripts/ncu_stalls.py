"""Sum ncu source-page warp-stall samples over every profiled instance of a kernel and print the
hottest SASS lines with their CUDA source line (ncu --page source --csv --print-source sass,cuda
is not available in one pass, so the SASS page is aggregated by address offset)."""
import csv
import sys
from collections import defaultdict

rows = list(csv.reader(open(sys.argv[1])))
name = sys.argv[2] if len(sys.argv) > 2 else ""
kern, hdr, agg, text, inst = None, None, defaultdict(int), {}, 0
base = None
for r in rows:
    if r and r[0] == "Kernel Name":
        kern = r[1]
        hdr = None
        base = None
        if name in kern:
            inst += 1
        continue
    if kern is None or name not in kern:
        continue
    if hdr is None:
        hdr = r
        continue
    if len(r) != len(hdr):
        continue
    try:
        addr = int(r[0], 16)
        samples = int(r[2] or 0)
    except ValueError:
        continue
    if base is None:
        base = addr
    off = addr - base
    agg[off] += samples
    text[off] = r[1]
tot = sum(agg.values())
print(f"{inst} instances, {tot} samples")
for off, v in sorted(agg.items(), key=lambda kv: -kv[1])[:int(sys.argv[3]) if len(sys.argv) > 3 else 40]:
    print(f"  +{off:05x} {v:6d} {100.0 * v / max(tot, 1):5.1f}%  {text[off][:100]}")
