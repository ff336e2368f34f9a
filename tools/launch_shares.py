"""Summarize an ncu launch list (--metrics gpu__time_duration.sum --csv):
per kernel, launches, total device time and share of the listed time.

    python tools/launch_shares.py gpurun_out/launches_<tag>.csv
"""

import collections
import csv
import re
import sys


def main(path: str) -> None:
    tot = collections.defaultdict(float)
    cnt = collections.Counter()
    with open(path) as f:
        lines = [ln for ln in f if ln.startswith('"')]
    for row in csv.DictReader(lines):
        if row.get("Metric Name") != "gpu__time_duration.sum":
            continue
        name = re.sub(r"\(.*", "", row["Kernel Name"]).replace("gsw::", "")
        v = float(row["Metric Value"])
        if row.get("Metric Unit") == "us":
            v *= 1e3
        elif row.get("Metric Unit") == "ms":
            v *= 1e6
        tot[name] += v
        cnt[name] += 1
    s = sum(tot.values())
    print(f"{'kernel':40s} {'launches':>8s} {'total_ms':>10s} {'share':>7s}")
    for k, v in sorted(tot.items(), key=lambda kv: -kv[1]):
        print(f"{k:40s} {cnt[k]:8d} {v / 1e6:10.3f} {v / s:7.3f}")
    print(f"{'TOTAL':40s} {sum(cnt.values()):8d} {s / 1e6:10.3f}")


if __name__ == "__main__":
    main(sys.argv[1])
