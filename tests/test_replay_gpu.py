"""Golden-stream parity of the GPU engine (pytest -m gpu).

* every recorded reference SimEngine run replayed through the drop-in API;
* the cfg 4 sweeps run in one gs_sweep launch vs the reference's events;
* 10^5 / 10^6-probe sweeps vs the (golden-pinned) C oracle.
"""

import ctypes

import numpy as np
import pytest

from replay import DropinBackend, load_sim_runs, load_sweeps, replay_run

pytestmark = pytest.mark.gpu

RUNS = list(load_sim_runs())
SWEEPS = load_sweeps()
LABELS = sorted(k for k in SWEEPS if "." not in k)


@pytest.mark.parametrize("chunk", range(8))
def test_dropin_replays_reference_streams(chunk):
    n = 0
    for run in RUNS[chunk::8]:
        n += replay_run(DropinBackend(), run)
    assert n > 0


def run_gpu_sweep(spec, n_dev, probes, max_res, policy):
    from paper_2107_08538_b200 import _native as nat
    from paper_2107_08538_b200.gpushare import DeviceState, Scheduler, parse_policy

    devs = [DeviceState(spec, i) for i in range(n_dev)]
    sched = Scheduler(devs, parse_policy(policy))
    cap = 2 * len(probes) + 16
    ev = np.zeros((cap, 3), dtype=np.int32)
    ne, ms = ctypes.c_int64(), ctypes.c_float()
    nat.check(nat.lib().gs_sweep(sched._ptr, probes.ctypes.data, len(probes), max_res, ev.ctypes.data, cap,
                                 ctypes.byref(ne), ctypes.byref(ms)))
    final = np.array([[d.free_mem, d.in_use_warps, d.rr_cursor, d.version,
                       __import__("replay").sm_crc((d.sm_warps, d.sm_tbs, d.sm_regs, d.sm_smem))]
                      for d in devs], dtype=np.int64)
    return ev[: ne.value], final, ms.value


def sweep_inputs(label):
    from paper_2107_08538_b200.gpushare.device_model import DeviceSpec
    from paper_2107_08538_b200.sweep import gen_probes

    meta = SWEEPS[label + ".meta"]
    n_dev, n, seed, max_res, pol = (int(x) for x in meta[:5])
    spec = DeviceSpec("s", *[int(x) for x in meta[5:]])
    return spec, n_dev, gen_probes(n, seed), max_res, ("mgb-warps" if pol == 0 else "mgb-sm")


@pytest.mark.parametrize("label", LABELS)
def test_gpu_sweep_matches_reference(label):
    spec, n_dev, probes, max_res, policy = sweep_inputs(label)
    ev, final, _ = run_gpu_sweep(spec, n_dev, probes, max_res, policy)
    np.testing.assert_array_equal(ev, SWEEPS[label])
    np.testing.assert_array_equal(final, SWEEPS[label + ".final"])


@pytest.mark.parametrize("n,policy", [(100_000, "mgb-sm"), (1_000_000, "mgb-warps"),
                                      (200_000, "mgb-sm")])
def test_gpu_sweep_matches_oracle_at_scale(n, policy):
    from oracle import oracle as O
    from paper_2107_08538_b200.gpushare import device_spec
    from paper_2107_08538_b200.sweep import gen_probes

    spec = device_spec("b200")
    probes = gen_probes(n, seed=11)
    ev, final, ms = run_gpu_sweep(spec, 8, probes, 32, policy)
    devs = [O.OracleDevice(spec, i) for i in range(8)]
    oev = O.OracleScheduler(devs, 2 if policy == "mgb-sm" else 3, 6, True).sweep(probes, 32)
    np.testing.assert_array_equal(ev, oev)
    np.testing.assert_array_equal(final, np.array([d.snapshot() for d in devs], dtype=np.int64))


@pytest.mark.parametrize("chunk", range(16))
def test_ring_mode_replays_reference_streams(chunk):
    """Every golden stream served by the persistent decision kernel over the
    host-mapped command ring (16 chunks cover all recorded runs)."""
    n = 0
    for run in RUNS[chunk::16]:
        be = DropinBackend(ring=True)
        try:
            n += replay_run(be, run)
        finally:
            be.close()
    assert n > 0


def _sweep_state(spec, n_dev, probes, max_res, policy, general, monkeypatch):
    """Events plus every byte of state a sweep leaves: ledger headers and
    the residency row of every handle on every device."""
    from paper_2107_08538_b200 import _native as nat
    from paper_2107_08538_b200.gpushare import DeviceState, Scheduler, parse_policy

    monkeypatch.setenv("GS_SWEEP_GENERAL", "1" if general else "0")
    devs = [DeviceState(spec, i) for i in range(n_dev)]
    sched = Scheduler(devs, parse_policy(policy))
    cap = 2 * len(probes) + 16
    ev = np.zeros((cap, 3), dtype=np.int32)
    ne, ms = ctypes.c_int64(), ctypes.c_float()
    lib = nat.lib()
    nat.check(lib.gs_sweep(sched._ptr, probes.ctypes.data, len(probes), max_res, ev.ctypes.data, cap,
                           ctypes.byref(ne), ctypes.byref(ms)))
    hdr = [ctypes.string_at(ctypes.addressof(d._led), 56) for d in devs]  # all but rr_cursor/sm_count
    rows = []
    row = nat.GsResidency()
    for d in devs:
        for h in range(len(probes)):
            nat.check(lib.gs_residency_read(d._ptr, h, ctypes.byref(row), None))
            rows.append(ctypes.string_at(ctypes.addressof(row), ctypes.sizeof(row)) if row.present else b"")
    return ev[: ne.value], hdr, rows, lib.gs_pending_count(sched._ptr)


@pytest.mark.parametrize("label", ["b200x2-warps-3k", "p100x2-warps-2k", "b200x8-warps-1k"])
def test_gpu_sweep_fast_chain_matches_general_path(label, monkeypatch):
    """The specialised mgb-warps sweep chain leaves exactly the state the
    general interpreter path does: events, ledger headers (free/in-use,
    version, held sums, grow epoch) and residency rows — including the
    streams that defer and hand over to the general path mid-sweep."""
    spec, n_dev, probes, max_res, policy = sweep_inputs(label)
    fast = _sweep_state(spec, n_dev, probes, max_res, policy, False, monkeypatch)
    slow = _sweep_state(spec, n_dev, probes, max_res, policy, True, monkeypatch)
    np.testing.assert_array_equal(fast[0], slow[0])
    np.testing.assert_array_equal(fast[0], SWEEPS[label])
    assert fast[1] == slow[1]
    assert fast[2] == slow[2]
    assert fast[3] == slow[3]


@pytest.mark.parametrize("case", ["non_fresh", "wide_key"])
def test_gpu_sweep_fast_chain_rejects_and_hands_over(case):
    """Oversized probes are rejected inside the fast chain; a non-fresh probe,
    or in-use warps beyond the packed 32-bit key, hands the rest of the
    stream to the general path — all vs the oracle."""
    from oracle import oracle as O
    from paper_2107_08538_b200.gpushare import device_spec
    from paper_2107_08538_b200.sweep import gen_probes

    spec = device_spec("b200")
    probes = gen_probes(5000, seed=5)
    probes["mem_bytes"][::97] = spec.mem_bytes + 1  # impossible everywhere
    if case == "non_fresh":
        probes["level"][4000] = 0                    # not fresh (still a new handle)
    else:
        probes["total_warps"][3000:3400] = 1 << 24   # in_use_warps passes 2^26
    ev, final, _ = run_gpu_sweep(spec, 8, probes, 32, "mgb-warps")
    devs = [O.OracleDevice(spec, i) for i in range(8)]
    oev = O.OracleScheduler(devs, 3, 6, True).sweep(probes, 32)
    np.testing.assert_array_equal(ev, oev)
    assert (ev[:, 0] == 2).sum() == len(range(0, 5000, 97))
    np.testing.assert_array_equal(final, np.array([d.snapshot() for d in devs], dtype=np.int64))


@pytest.mark.parametrize("max_res,ev_cap", [(0, None), (1, None), (5, 700), (31, 100)])
def test_gpu_sweep_fast_chain_fifo_edges(max_res, ev_cap, monkeypatch):
    """FIFO depths where the oldest resident is the task just pushed
    (max_resident 0) or a few slots back, and event logs shorter than the
    stream: the specialised chain and the general path agree on the events,
    the event count and the final ledgers, and both match the oracle."""
    from oracle import oracle as O
    from paper_2107_08538_b200 import _native as nat
    from paper_2107_08538_b200.gpushare import DeviceState, Scheduler, device_spec, parse_policy
    from paper_2107_08538_b200.sweep import gen_probes

    spec = device_spec("b200")
    probes = gen_probes(3000, seed=21, mem_gib=(10, 60))

    def run(general):
        monkeypatch.setenv("GS_SWEEP_GENERAL", "1" if general else "0")
        devs = [DeviceState(spec, i) for i in range(3)]
        sched = Scheduler(devs, parse_policy("mgb-warps"))
        cap = ev_cap or 2 * len(probes) + 16
        ev = np.zeros((cap, 3), dtype=np.int32)
        ne, ms = ctypes.c_int64(), ctypes.c_float()
        nat.check(nat.lib().gs_sweep(sched._ptr, probes.ctypes.data, len(probes), max_res, ev.ctypes.data, cap,
                                     ctypes.byref(ne), ctypes.byref(ms)))
        hdr = [ctypes.string_at(ctypes.addressof(d._led), 56) for d in devs]
        return ev[: min(ne.value, cap)], ne.value, hdr

    fast, slow = run(False), run(True)
    np.testing.assert_array_equal(fast[0], slow[0])
    assert fast[1] == slow[1]
    assert fast[2] == slow[2]
    devs = [O.OracleDevice(spec, i) for i in range(3)]
    oev = O.OracleScheduler(devs, 3, 6, True).sweep(probes, max_res)
    assert fast[1] == len(oev)
    np.testing.assert_array_equal(fast[0], oev[: len(fast[0])])


def test_sweep_consumes_the_scheduler():
    """Tasks a sweep leaves resident keep their reservations and their
    handles never reach the caller: a second sweep or a submit on the same
    scheduler is a contract violation, not a silent leak of capacity."""
    from paper_2107_08538_b200 import _native as nat
    from paper_2107_08538_b200.gpushare import DeviceState, Scheduler, device_spec, parse_policy
    from paper_2107_08538_b200.sweep import gen_probes

    spec = device_spec("b200")
    probes = gen_probes(500, seed=3)
    devs = [DeviceState(spec, i) for i in range(2)]
    sched = Scheduler(devs, parse_policy("mgb-warps"))
    cap = 2 * len(probes) + 16
    ev = np.zeros((cap, 3), dtype=np.int32)
    ne, ms = ctypes.c_int64(), ctypes.c_float()
    lib = nat.lib()
    nat.check(lib.gs_sweep(sched._ptr, probes.ctypes.data, len(probes), 32, ev.ctypes.data, cap,
                           ctypes.byref(ne), ctypes.byref(ms)))
    assert sum(d.in_use_warps for d in devs) > 0  # residents still hold capacity
    rc = lib.gs_sweep(sched._ptr, probes.ctypes.data, len(probes), 32, ev.ctypes.data, cap,
                      ctypes.byref(ne), ctypes.byref(ms))
    assert rc == nat.GS_ERR_CONTRACT
    dec = nat.GsDecision()
    p = nat.GsProbe()
    p.handle, p.job = len(probes) + 1, 0
    assert lib.gs_submit(sched._ptr, ctypes.byref(p), ctypes.byref(dec)) == nat.GS_ERR_CONTRACT
