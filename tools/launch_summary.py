"""Summarise an ncu launch list (`--metrics gpu__time_duration.sum --csv`).

python tools/launch_summary.py LAUNCHES.csv OUT.md "title" "command"
Per kernel: launches, total and mean device time, share of the listed time.
ncu serialises launches with cold caches: compare shares, not absolutes.
"""

from __future__ import annotations

import csv
import re
import sys
from collections import defaultdict


def short(name: str) -> str:
    base = name.split("(")[0].replace("void ", "")
    base = re.sub(r"gsv::<unnamed>::", "", base)
    if "cub::" in base:
        base = base.split("::")[-1][:48]
    return base


def main():
    src, out, title, cmd = sys.argv[1:5]
    lines = [ln for ln in open(src) if ln.startswith('"')]
    rows = list(csv.DictReader(lines))
    tot = defaultdict(float)
    cnt = defaultdict(int)
    for r in rows:
        if r["Metric Name"] != "gpu__time_duration.sum":
            continue
        k = short(r["Kernel Name"])
        scale = {"ns": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3}.get(r["Metric Unit"], 1e-3)
        tot[k] += float(r["Metric Value"].replace(",", "")) * scale
        cnt[k] += 1
    allt = sum(tot.values())
    md = [f"# {title}", "", f"Command: `{cmd}`.",
          "Per-launch times are cold-cache and serialised (ncu): compare shares, not absolutes.",
          "", "| kernel | launches | total us | mean us | share |", "|---|---|---|---|---|"]
    for k, t in sorted(tot.items(), key=lambda kv: -kv[1]):
        md.append(f"| `{k}` | {cnt[k]} | {t:.1f} | {t / cnt[k]:.1f} | {100 * t / allt:.1f}% |")
    open(out, "w").write("\n".join(md) + "\n")
    print(f"wrote {out} ({len(rows)} launches, {allt:.0f} us)")


if __name__ == "__main__":
    main()
