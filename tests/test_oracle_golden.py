"""The C oracle against golden streams recorded from the reference (CPU).

This pins the oracle (oracle/gs_oracle.c) before it is trusted as the
checker for the GPU engine at sizes the golden files do not cover.
"""

import numpy as np
import pytest

from replay import OracleBackend, load_sim_runs, load_sweeps, replay_run

RUNS = list(load_sim_runs())


def test_golden_corpus_shape():
    labels = [r["label"] for r in RUNS]
    assert len(RUNS) >= 300
    assert any(lbl.startswith("strict") for lbl in labels)
    assert any("b200x8" in lbl for lbl in labels)
    assert sum(len(r["events"]) for r in RUNS) > 40000


@pytest.mark.parametrize("chunk", range(8))
def test_oracle_replays_reference_streams(chunk):
    n = 0
    for run in RUNS[chunk::8]:
        n += replay_run(OracleBackend(), run)
    assert n > 0


SWEEPS = load_sweeps()
LABELS = sorted(k for k in SWEEPS if "." not in k)


def sweep_inputs(label):
    from paper_2107_08538_b200.gpushare.device_model import DeviceSpec
    from paper_2107_08538_b200.sweep import gen_probes

    meta = SWEEPS[label + ".meta"]
    n_dev, n, seed, max_res, pol = (int(x) for x in meta[:5])
    spec = DeviceSpec("s", *[int(x) for x in meta[5:]])
    return spec, n_dev, gen_probes(n, seed), max_res, (3 if pol == 0 else 2)


@pytest.mark.parametrize("label", LABELS)
def test_oracle_sweep_matches_reference(label):
    from oracle import oracle as O

    spec, n_dev, probes, max_res, code = sweep_inputs(label)
    devs = [O.OracleDevice(spec, i) for i in range(n_dev)]
    sched = O.OracleScheduler(devs, code, 6, True)
    ev = sched.sweep(probes, max_res)
    np.testing.assert_array_equal(ev, SWEEPS[label])
    final = np.array([d.snapshot() for d in devs], dtype=np.int64)
    np.testing.assert_array_equal(final, SWEEPS[label + ".final"])
