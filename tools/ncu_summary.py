"""One line per ncu report: DRAM bytes, duration, achieved DRAM GB/s,
occupancy and pipe utilisation (the numbers profiles/ cites).

    python tools/ncu_summary.py gpurun_out/prof_*.ncu-rep
"""

import csv
import io
import subprocess
import sys

METRICS = ["dram__bytes_read.sum", "dram__bytes_write.sum", "gpu__time_duration.sum", "launch__registers_per_thread",
           "launch__grid_size", "launch__block_size", "sm__warps_active.avg.pct_of_peak_sustained_active",
           "dram__throughput.avg.pct_of_peak_sustained_elapsed", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
           "sm__pipe_tensor_op_hmma_cycles_active.avg.pct_of_peak_sustained_active",
           "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active"]
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-9, "us": 1e-6, "usecond": 1e-6,
         "ms": 1e-3, "msecond": 1e-3, "nsecond": 1e-9}


def summarize(path: str) -> str:
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv", "--metrics", ",".join(METRICS)],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    if len(rows) < 3:
        return f"{path}: no data"
    h, u, v = rows[0], rows[1], rows[2]
    d = {h[i]: (v[i], u[i]) for i in range(len(h))}

    def num(k):
        if k not in d or d[k][0] in ("", "n/a"):
            return None
        return float(d[k][0].replace(",", "")) * SCALE.get(d[k][1], 1.0)

    rd, wr, t = num("dram__bytes_read.sum"), num("dram__bytes_write.sum"), num("gpu__time_duration.sum")
    name = d["Kernel Name"][0].split("(")[0].replace("gsw::", "")
    parts = [f"{name:28s}", f"time={t * 1e6:10.1f}us" if t else "time=?"]
    if rd is not None and wr is not None:
        parts.append(f"dram={(rd + wr) / 1e6:10.1f}MB")
        if t:
            parts.append(f"dram_GBps={(rd + wr) / t / 1e9:7.1f}")
    for k, lab in [("dram__throughput.avg.pct_of_peak_sustained_elapsed", "dram%"),
                   ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "sm%"),
                   ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps%"),
                   ("sm__pipe_tensor_op_hmma_cycles_active.avg.pct_of_peak_sustained_active", "tensor%"),
                   ("launch__registers_per_thread", "regs"), ("launch__grid_size", "grid")]:
        if k in d and d[k][0] not in ("", "n/a"):
            parts.append(f"{lab}={d[k][0]}")
    return " ".join(parts)


if __name__ == "__main__":
    for p in sys.argv[1:]:
        print(summarize(p))
