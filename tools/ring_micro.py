"""Raw C-ABI round trip of one decision (gs_submit) in launch and ring
mode, without the Python shim: where the drop-in's per-call time goes."""
import ctypes, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2107_08538_b200 import _native as nat  # noqa: E402
from paper_2107_08538_b200.gpushare import DeviceState, Scheduler, device_spec, parse_policy  # noqa: E402

spec = device_spec("b200")
for ring in (False, True):
    devs = [DeviceState(spec, i) for i in range(8)]
    sched = Scheduler(devs, parse_policy("mgb-warps"))
    if ring:
        sched.start_ring(max_pending=5000, max_handles=5000, max_jobs=8)
    lib = nat.lib()
    dec = nat.GsDecision()
    n = 2000
    probes = [nat.GsProbe(1 << 20, 0, 8, 1.0, 1, 8, 256, 32, 0, i % 4000, -1, 2) for i in range(n)]
    t = time.perf_counter()
    for p in probes:
        lib.gs_submit(sched._ptr, ctypes.byref(p), ctypes.byref(dec))
    us = (time.perf_counter() - t) / n * 1e6
    print(("ring" if ring else "launch"), f"{us:.1f} us per gs_submit", flush=True)
    if ring:
        sched.stop_ring()
