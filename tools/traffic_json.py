"""profiles/traffic.json from the ncu captures of tools/profile.sh: DRAM
bytes (read + write) of one launch of each kind's main kernel next to that
launch's algorithmic bytes (catalog.algorithmic_work per launch).

    python tools/traffic_json.py gpurun_out [tag]
"""

import csv
import io
import json
import os
import subprocess
import sys

# kind -> (capture name, kernel, size note, algorithmic bytes of ONE launch)
KINDS = {
    "hotspot": ("hotspot", "hotspot_pass4", "24576^2, one four-step pass", 12.0 * 24576 ** 2),
    "srad": ("srad", "srad_stream", "24576^2, one iteration", 8.0 * 24576 ** 2),
    "kmeans": ("kmeans", "kmeans_assign<34>", "32M x 34, one iteration", 4.0 * 32e6 * 34 + 4.0 * 32e6),
    "backprop": ("bpadj", "bp_adjust", "48M x 16", None),
    "needle": ("needle", "needle_bands", "24576^2", 8.0 * 24577 ** 2),
    "bfs": ("bfs", "bfs_expand", "128M vertices, one dense level", None),
    "lud": ("lud", "lud_internal", "6144, one mid-factorization trailing update", None),
}


def dram(rep: str):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv", "--metrics",
                          "dram__bytes_read.sum,dram__bytes_write.sum"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    if len(rows) < 3:
        return None
    h, u, v = rows[0], rows[1], rows[2]
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
    tot = 0.0
    for k in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
        i = h.index(k)
        tot += float(v[i].replace(",", "")) * scale.get(u[i], 1)
    return int(tot)


def main():
    src = sys.argv[1] if len(sys.argv) > 1 else "gpurun_out"
    tag = sys.argv[2] if len(sys.argv) > 2 else "r02"
    out = {"_source": f"tools/traffic_json.py over tools/profile.sh {tag} captures: dram__bytes_read.sum + "
                      "dram__bytes_write.sum of one launch (ncu --set full, B200); algorithmic = SURVEY.md §8d "
                      "per-unit figure x units of that launch"}
    for kind, (cap, kern, size, alg) in KINDS.items():
        rep = os.path.join(src, f"prof_{cap}.ncu-rep")
        if not os.path.exists(rep):
            continue
        out[kind] = {"kernel": kern, "size": size, "dram_bytes_per_launch": dram(rep),
                     "algorithmic_bytes_per_launch": int(alg) if alg else None}
    json.dump(out, open(os.path.join("profiles", "traffic.json"), "w"), indent=2)
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
