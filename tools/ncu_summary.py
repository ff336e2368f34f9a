"""One line per ncu capture of tools/profile.sh (run where the .ncu-rep files are).

    python tools/ncu_summary.py gpurun_out > profiles/<tag>_ncu_current_kernels.txt
    python tools/ncu_summary.py gpurun_out/prof_srad.ncu-rep ...

Per capture: kernel, device time, DRAM bytes and rate, issue-active and
SM-throughput %, warps-active %, registers, grid, the top stall reasons.
"""

from __future__ import annotations

import csv
import glob
import io
import os
import subprocess
import sys

SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-9, "us": 1e-6, "ms": 1e-3, "s": 1.0,
         "nsecond": 1e-9, "usecond": 1e-6, "msecond": 1e-3, "second": 1.0}


def main() -> int:
    args = sys.argv[1:] or ["gpurun_out"]
    reps = [a for a in args if a.endswith(".ncu-rep")]
    for a in args:
        if os.path.isdir(a):
            reps += sorted(glob.glob(os.path.join(a, "prof_*.ncu-rep")))
    for rep in reps:
        out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
        rows = list(csv.reader(io.StringIO(out)))
        if len(rows) < 3:
            print(f"{os.path.basename(rep)}: no data")
            continue
        h, u, v = rows[0], rows[1], rows[2]
        d = dict(zip(h, v))
        units = dict(zip(h, u))

        def num(k):
            try:
                return float(d[k].replace(",", "")) * SCALE.get(units.get(k, ""), 1.0)
            except (KeyError, ValueError):
                return float("nan")

        t = num("gpu__time_duration.sum")
        dram = num("dram__bytes_read.sum") + num("dram__bytes_write.sum")
        stalls = sorted(((num(k), k) for k in h if "issue_stalled" in k and k.endswith("per_issue_active.ratio")),
                        reverse=True)[:4]
        st = ", ".join(f"{k.split('issue_stalled_')[1].split('_per')[0]} {x:.2f}" for x, k in stalls)
        name = d.get("Kernel Name", "?").split("(")[0]
        print(f"{os.path.basename(rep)[5:-8]:8s} {name:40s} time={t * 1e6:10.1f}us dram={dram / 1e6:9.1f}MB "
              f"dram_GBps={dram / t / 1e9 if t > 0 else 0:7.1f} "
              f"issue%={num('sm__issue_active.avg.pct_of_peak_sustained_elapsed'):5.1f} "
              f"sm%={num('sm__throughput.avg.pct_of_peak_sustained_elapsed'):5.1f} "
              f"warps%={num('sm__warps_active.avg.pct_of_peak_sustained_active'):5.1f} "
              f"regs={d.get('launch__registers_per_thread', '?')} grid={d.get('launch__grid_size', '?')} "
              f"stalls: {st}")
    return 0


if __name__ == "__main__":
    sys.exit(main())
