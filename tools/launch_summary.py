"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv) as a
markdown table: launches, total and mean duration and share per kernel.

usage: python tools/launch_summary.py launches.csv [title]
"""
import collections
import csv
import sys


def main():
    path = sys.argv[1]
    title = sys.argv[2] if len(sys.argv) > 2 else path
    lines = [ln for ln in open(path) if ln.startswith('"')]
    rows = list(csv.DictReader(lines))
    tot = collections.Counter()
    cnt = collections.Counter()
    for r in rows:
        if r.get("Metric Name") != "gpu__time_duration.sum":
            continue
        scale = {"ns": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}.get(r["Metric Unit"], 1e-3)
        v = float(r["Metric Value"].replace(",", "")) * scale
        name = r["Kernel Name"][:70]
        tot[name] += v
        cnt[name] += 1
    all_us = sum(tot.values())
    print(f"# {title}\n")
    print("| kernel | launches | total us | mean us | share |")
    print("|---|---|---|---|---|")
    for k, v in tot.most_common():
        print(f"| `{k}` | {cnt[k]} | {v:.1f} | {v / cnt[k]:.2f} | {100 * v / all_us:.1f}% |")
    print(f"\ntotal {all_us:.1f} us over {sum(cnt.values())} launches")


if __name__ == "__main__":
    main()
