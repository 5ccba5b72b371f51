"""Summarise an ncu --metrics gpu__time_duration.sum CSV launch list: time share per kernel name.

    python tools/launch_summary.py gpurun_out/launches_gpt.csv [top]
"""
import csv
import re
import sys
from collections import defaultdict


def short(name: str) -> str:
    name = re.sub(r"^void ", "", name)
    name = re.sub(r"^(pd::)?(<unnamed>::|\(anonymous namespace\)::)?", "", name)
    m = re.match(r"([A-Za-z_0-9]+)(<[^(]*>)?", name)
    if not m:
        return name[:60]
    base = m.group(1)
    tmpl = m.group(2) or ""
    return (base + tmpl)[:110]


def main():
    path = sys.argv[1]
    top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
    rows = list(csv.reader(l for l in open(path) if not l.startswith("==")))
    hdr = rows[0]
    ki, mi, vi = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value")
    tot = defaultdict(float)
    cnt = defaultdict(int)
    for r in rows[1:]:
        if len(r) <= vi or r[mi] != "gpu__time_duration.sum":
            continue
        v = float(r[vi].replace(",", ""))
        k = short(r[ki])
        tot[k] += v
        cnt[k] += 1
    total = sum(tot.values())
    print(f"{'share':>6} {'total_ms':>9} {'n':>6} {'avg_us':>8}  kernel")
    for k, v in sorted(tot.items(), key=lambda kv: -kv[1])[:top]:
        print(f"{100 * v / total:6.2f} {v / 1e6:9.3f} {cnt[k]:6d} {v / cnt[k] / 1e3:8.2f}  {k}")
    print(f"total {total / 1e6:.3f} ms over {sum(cnt.values())} launches")


if __name__ == "__main__":
    main()
