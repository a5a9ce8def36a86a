"""Summarise an ncu --csv launch list (gpu__time_duration.sum per launch) by kernel."""
import collections
import csv
import sys


def summarise(path):
    hdr, data = None, []
    for r in csv.reader(open(path)):
        if r and r[0] == "ID":
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            data.append(dict(zip(hdr, r)))
    agg = collections.defaultdict(list)
    for d in data:
        k = d["Kernel Name"]
        name = k.split("(")[0]
        agg[name].append(float(d["Metric Value"]) / (1000.0 if d["Metric Unit"] == "ns" else 1.0))
    tot = sum(sum(v) for v in agg.values())
    rows = []
    for k, v in sorted(agg.items(), key=lambda kv: -sum(kv[1])):
        rows.append((k[:90], len(v), sum(v) / len(v), sum(v) / tot))
    return rows, tot, len(data)


if __name__ == "__main__":
    rows, tot, n = summarise(sys.argv[1])
    print(f"{n} launches, {tot:.1f} us total (serialised, cold)")
    for k, c, avg, sh in rows:
        print(f"{k:92s} n={c:5d} avg={avg:8.2f}us share={sh:.3f}")
