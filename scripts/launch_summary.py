"""Aggregate an ncu launch list (--metrics gpu__time_duration.sum --csv) per
kernel: launches, total us, share.  Usage: launch_summary.py launches.csv [steps]"""
import csv
import io
import sys
from collections import defaultdict


def main(path, steps=1.0):
    text = open(path).read()
    start = text.index('"ID"')
    rows = list(csv.DictReader(io.StringIO(text[start:])))
    tot, cnt = defaultdict(float), defaultdict(int)
    for r in rows:
        if r.get("Metric Name") != "gpu__time_duration.sum":
            continue
        name = r["Kernel Name"].split("(")[0].split("<")[0].replace("void ", "").strip()
        name = name.split("::")[-1]
        v = float(r["Metric Value"].replace(",", ""))
        unit = r.get("Metric Unit", "ns")
        tot[name] += v / 1000.0 if unit in ("ns", "nsecond") else v
        cnt[name] += 1
    all_us = sum(tot.values())
    print(f"| kernel | launches/step | us/step | share |\n|---|---|---|---|")
    for k in sorted(tot, key=lambda k: -tot[k]):
        print(f"| {k} | {cnt[k] / steps:.1f} | {tot[k] / steps:.1f} | {100 * tot[k] / all_us:.1f} % |")
    print(f"| total | {sum(cnt.values()) / steps:.1f} | {all_us / steps:.1f} | |")


if __name__ == "__main__":
    main(sys.argv[1], float(sys.argv[2]) if len(sys.argv) > 2 else 1.0)
