"""One mgb-warps (or argv[1]) placement sweep of argv[2] probes (for ncu)."""
import ctypes, os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2107_08538_b200 import _native as nat  # noqa: E402
from paper_2107_08538_b200.gpushare import DeviceState, Scheduler, device_spec, parse_policy  # noqa: E402
from paper_2107_08538_b200.sweep import gen_probes  # noqa: E402

policy = sys.argv[1] if len(sys.argv) > 1 else "mgb-warps"
n = int(sys.argv[2]) if len(sys.argv) > 2 else 20000
spec = device_spec("b200")
probes = gen_probes(n, seed=1)
devs = [DeviceState(spec, i) for i in range(8)]
sched = Scheduler(devs, parse_policy(policy))
cap = 2 * n + 16
ev = np.zeros((cap, 3), dtype=np.int32)
ne, ms = ctypes.c_int64(), ctypes.c_float()
nat.check(nat.lib().gs_sweep(sched._ptr, probes.ctypes.data, n, 32, ev.ctypes.data, cap, ctypes.byref(ne), ctypes.byref(ms)))
print(policy, n, "events", ne.value, "ms", ms.value, "ns/probe", ms.value * 1e6 / n)
