"""Host<->device copy bandwidth from pinned memory (the e2e ceiling).

    python tools/pcie_bw.py
"""

import json

import torch


def bw(src, dst, reps=5):
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    best = 1e9
    for _ in range(reps):
        e0.record()
        dst.copy_(src, non_blocking=True)
        e1.record()
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1))
    return src.numel() * src.element_size() / (best * 1e-3) / 1e9


n = 1 << 30  # 4 GiB of float32
h = torch.empty(n, dtype=torch.float32, pin_memory=True)
d = torch.empty(n, dtype=torch.float32, device="cuda")
h2d = bw(h, d)
d2h = bw(d, h)
# both directions at once on two streams
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
h2 = torch.empty(n, dtype=torch.float32, pin_memory=True)
d2 = torch.empty(n, dtype=torch.float32, device="cuda")
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
with torch.cuda.stream(s1):
    d.copy_(h, non_blocking=True)
with torch.cuda.stream(s2):
    h2.copy_(d2, non_blocking=True)
torch.cuda.current_stream().wait_stream(s1)
torch.cuda.current_stream().wait_stream(s2)
e1.record()
torch.cuda.synchronize()
both = 2 * 4 * n / (e0.elapsed_time(e1) * 1e-3) / 1e9
print(json.dumps({"h2d_GBps": round(h2d, 1), "d2h_GBps": round(d2h, 1), "bidir_total_GBps": round(both, 1),
                  "bytes_each": 4 * n}))
