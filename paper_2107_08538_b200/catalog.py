"""Rodinia-class job catalog and seeded job mixes (BASELINE cfg 1).

The reference's catalog (gpushare/data/catalog.json) describes each job by
footprint and duration only; here each template is an executable job with a
small and a large size class (the reference's 1-4 GiB / 4-13 GiB classes,
catalog.json:3).  `gen_mix` follows gpushare/workload_gen.py:177-214: larges
rounded up, picks drawn from random.Random(f"{seed}|{mix}|{n}"), then
shuffled, job ids j00..jNN.

Jobs of one template are identical instances, as in the reference (a
template is one fixed program: footprint, kernels, duration): their
synthetic inputs come from a per-template data seed, so a mix needs one
staged copy of each template's inputs, not one per job.
"""

from __future__ import annotations

import math
import os
import random
from dataclasses import dataclass

from .workloads import Job

# kind -> (small kwargs, large kwargs).  Footprints (host_footprint) follow
# the reference catalog's classes, small 1-4 GiB and large 4-13 GiB
# (catalog.json:3): bfs 1.8 / 7.2, hotspot 3.0 / 6.8, srad 2.0 / 4.5, kmeans
# 1.1 / 4.2, backprop 2.0 / 5.9, needle 2.0 / 4.5 GiB.  lud is the exception
# (0.06 / 0.15 GiB): its work is O(n^3) — a 1 GiB matrix (n = 16384) is
# 2.9 TFLOP, ~150 ms on a B200 and minutes on the CPU oracle.
RODINIA = {
    "bfs": (dict(n=32_000_000), dict(n=128_000_000)),
    "hotspot": (dict(n=16384, iters=40), dict(n=24576, iters=40)),
    "srad": (dict(n=16384, iters=10), dict(n=24576, iters=10)),
    "kmeans": (dict(n=8_000_000, m=34, iters=10), dict(n=32_000_000, m=34, iters=10)),
    "backprop": (dict(n=16_000_000, m=16, iters=2), dict(n=48_000_000, m=16, iters=2)),
    "needle": (dict(n=16384), dict(n=24576)),
    "lud": (dict(n=4096), dict(n=6144)),
}

# Darknet YOLOv3-tiny inference jobs (BASELINE cfg 2): image edge, batch
DARKNET = {
    "yolo": (dict(n=416, m=8), dict(n=608, m=32)),
    "resnet": (dict(n=224, m=8), dict(n=224, m=64)),
}

# the 8-job CPU-runnable mix of cfg 0 (2x bfs, hotspot, srad, kmeans, repeated)
CFG0 = [("bfs", dict(n=1_000_000)), ("bfs", dict(n=1_000_000)), ("hotspot", dict(n=1024, iters=20)),
        ("srad", dict(n=2048, iters=5)), ("kmeans", dict(n=494_020, m=34, iters=5))]


@dataclass(frozen=True)
class MixJob:
    job_id: str
    template: str
    job_class: str
    job: Job


def parse_mix(mix: str) -> tuple[int, int]:
    rl, rs = (int(x) for x in mix.split(":"))
    if rl < 0 or rs < 0 or rl + rs == 0:
        raise ValueError(f"bad mix {mix!r}")
    return rl, rs


def gen_mix(mix: str = "3:1", n: int = 32, seed: int = 1, kinds: tuple[str, ...] = tuple(RODINIA)) -> list[MixJob]:
    """Seeded job mix, larges:smalls (workload_gen.py:177-214 selection)."""
    rl, rs = parse_mix(mix)
    n_large = math.ceil(rl / (rl + rs) * n)
    n_small = n - n_large
    rng = random.Random(f"{seed}|{mix}|{n}")
    picks = [(rng.choice(kinds), "small") for _ in range(n_small)]
    picks += [(rng.choice(kinds), "large") for _ in range(n_large)]
    rng.shuffle(picks)
    width = max(2, len(str(n - 1)))
    out = []
    for i, (kind, cls) in enumerate(picks):
        kw = RODINIA[kind][0 if cls == "small" else 1]
        out.append(MixJob(f"j{i:0{width}d}", f"{kind}_{cls}", cls,
                          Job(kind, seed=template_seed(seed, kind, cls), **kw)))
    return out


def template_seed(seed: int, kind: str, cls: str) -> int:
    """Data seed of a template's instances in mix `seed`."""
    return seed * 1000 + 2 * list(RODINIA).index(kind) + (cls == "large")


def cfg0_mix(seed: int = 1) -> list[MixJob]:
    """BASELINE cfg 0: 8 jobs (2x bfs, hotspot, srad, kmeans, repeated to 8)."""
    out = []
    for i in range(8):
        kind, kw = CFG0[i % len(CFG0)]
        out.append(MixJob(f"j{i:02d}", kind, "small", Job(kind, seed=seed * 1000 + i, **kw)))
    return out


# yolov3-tiny conv layers as (edge divisor, cin, cout, k) in plan order
# (csrc/gs_darknet.cu yolo_plan); pools / upsample move no GEMM work
YOLO_CONVS = [(1, 3, 16, 3), (2, 16, 32, 3), (4, 32, 64, 3), (8, 64, 128, 3), (16, 128, 256, 3),
              (32, 256, 512, 3), (32, 512, 1024, 3), (32, 1024, 256, 1), (32, 256, 512, 3), (32, 512, 255, 1),
              (32, 256, 128, 1), (16, 384, 256, 3), (16, 256, 255, 1)]


def implicit_conv(cin: int, k: int) -> bool:
    """The executor runs this convolution as an implicit GEMM (no im2row
    workspace): csrc/gs_darknet.cu NetBuilder::implicit_conv."""
    return k in (1, 3) and cin in (8, 16, 32, 64, 128)


def yolo_buffers(S: int, N: int) -> list[int]:
    """Byte sizes of the YOLOv3-tiny job's buffers (yolo_plan order)."""
    act = lambda d, c: N * (S // d) ** 2 * c * 2  # noqa: E731  bf16 NHWC
    w = 0
    ws = 0
    for d, cin, cout, k in YOLO_CONVS:
        kpad = (k * k * cin + 7) // 8 * 8
        w = (w + cout * kpad + 7) // 8 * 8
        if k != 1 and not implicit_conv(cin, k):
            ws = max(ws, N * (S // d) ** 2 * kpad * 2)
    bias = sum(c[2] for c in YOLO_CONVS) * 4
    det = (N * (S // 32) ** 2 + N * (S // 16) ** 2) * 255 * 4
    acts = [act(1, 16), act(2, 16), act(2, 32), act(4, 32), act(4, 64), act(8, 64), act(8, 128), act(16, 128),
            act(16, 384), act(32, 256), act(32, 512), act(32, 512), act(32, 1024), act(32, 256), act(32, 512),
            act(32, 128), act(16, 256)]
    return [N * S * S * 3 * 2, w * 2, bias, det, max(ws, 16)] + acts


def yolo_flops(S: int, N: int) -> float:
    return float(sum(2 * N * (S // d) ** 2 * k * k * cin * cout for d, cin, cout, k in YOLO_CONVS))


def resnet50_convs(S: int) -> list[tuple[int, int, int, int, int, str]]:
    """ResNet-50 convolutions in plan order (csrc/gs_darknet.cu resnet50_plan):
    (in_hw, cin, cout, k, stride, out_buffer) with out_buffer "act" (a new
    resident activation) or "det" (the logits)."""
    out = [(S, 3, 64, 7, 2, "act")]
    hw = S // 4
    cin = 64
    for mid, blocks in ((64, 3), (128, 4), (256, 6), (512, 3)):
        for bi in range(blocks):
            stride = 2 if (mid != 64 and bi == 0) else 1
            out.append((hw, cin, mid, 1, 1, "act"))
            out.append((hw, mid, mid, 3, stride, "act"))
            if bi == 0:
                out.append((hw, cin, 4 * mid, 1, stride, "act"))
            out.append((hw // stride, mid, 4 * mid, 1, 1, "act"))
            hw //= stride
            cin = 4 * mid
    out.append((1, 2048, 1000, 1, 1, "det"))
    return out


def resnet_buffers(S: int, N: int) -> list[int]:
    """Byte sizes of the ResNet-50 job's buffers (resnet50_plan order)."""
    w = b = ws = 0
    acts = []
    for hw, cin, cout, k, stride, kind in resnet50_convs(S):
        kdim = k * k * cin
        kpad = (kdim + 7) // 8 * 8
        w = (w + cout * kpad + 7) // 8 * 8
        b += cout
        ohw = hw // stride if kind == "act" else 1
        if not (k == 1 and stride == 1) and not implicit_conv(cin, k):
            ws = max(ws, N * ohw * ohw * kpad * 2)
        if kind == "act":
            acts.append(N * ohw * ohw * cout * 2)
            if len(acts) == 1:  # the stem is followed by the 3x3/2 max-pool
                acts.append(N * (S // 4) ** 2 * 64 * 2)
    acts.append(N * 2048 * 2)  # global average pool
    return [N * S * S * 3 * 2, w * 2, b * 4, N * 1000 * 4, max(ws, 16)] + acts


def resnet_flops(S: int, N: int) -> float:
    tot = 0
    for hw, cin, cout, k, stride, kind in resnet50_convs(S):
        ohw = hw // stride if kind == "act" else 1
        tot += 2 * N * ohw * ohw * k * k * cin * cout
    return float(tot)


def host_footprint(job: Job) -> int:
    """The probe's mem_bytes computed on the host alone (same rule as
    gs_job_probe: buffers and the control block rounded to 2 MiB + the
    8 MiB task heap) — used by
    the CPU reference arm, which must not touch the GPU engine."""
    g = 2 << 20
    n, m = job.n, job.m
    sizes = {
        "bfs": [(n + 1) * 4, n * 24, n * 4] + [(n // 32 + 4) // 4 * 16] * 3 + [8 * 17, (n + 1) * 4, n * 24],
        "hotspot": [n * n * 4] * 3,
        "srad": [n * n * 4] * 2 + [16],
        "kmeans": [n * m * 4, n * 4, 5 * m * 4, 5 * m * 8, 40],
        "backprop": [(n + 1) * 4, m * (n + 1) * 4, m * (n + 1) * 4, 320, -(-(n + 1) // 8192) * 16 * 8],
        "needle": [n * n * 4, (n + 1) * (n + 4) * 4, 2 * n * 8],
        "lud": [n * n * 4],
        "yolo": yolo_buffers(n, m) if job.kind == "yolo" else [],
        "resnet": resnet_buffers(n, m) if job.kind == "resnet" else [],
    }[job.kind]
    sizes = sizes + [32]  # the job's control block (output digest + tile tickets)
    return (8 << 20) + sum((s + g - 1) // g * g for s in sizes)


def survey_bytes(job: Job) -> float:
    """SURVEY.md §8(d)'s per-unit byte counts as written (per iteration of
    the unfused Rodinia kernels): hotspot 12·N² per step, srad 24·N² per
    iteration, needle 8·N².  The executed algorithms move less (two hotspot
    steps per pass, srad's fused coefficient/update): algorithmic_work."""
    n, it = job.n, max(job.iters, 1)
    if job.kind == "hotspot":
        return 12.0 * n * n * it
    if job.kind == "srad":
        return 24.0 * n * n * it
    if job.kind == "needle":
        return 8.0 * n * n
    return algorithmic_work(job)[0]


def algorithmic_work(job: Job) -> tuple[float, str]:
    """(work, unit) per job run — SURVEY.md §8d's per-unit figures times the
    units a run processes: bytes for HBM-bound kernels, flops for lud."""
    n, it, m = job.n, max(job.iters, 1), job.m
    if job.kind == "hotspot":
        # read T and P, write T once per pass; passes of four steps
        # (hotspot_pass4) while four remain, then two-step passes, then an
        # odd single step (csrc/gs_work.cu run_kernels; GS_HOTSPOT_STEPS=2
        # runs two-step passes only)
        passes = it // 4 + (it % 4) // 2 + it % 2
        if os.environ.get("GS_HOTSPOT_STEPS", "")[:1] == "2":
            passes = it // 2 + it % 2
        return 12.0 * n * n * passes, "B"
    if job.kind == "srad":  # fused coefficient + update: read J, write J
        return 8.0 * n * n * it, "B"
    if job.kind == "bfs":
        return 4.0 * 6 * n + 13.0 * n, "B"
    if job.kind == "kmeans":
        return (4.0 * n * m + 4.0 * n) * it, "B"
    if job.kind == "backprop":
        return 16.0 * (n + 1) * (m + 1) * it, "B"
    if job.kind == "needle":
        return 8.0 * (n + 1) * (n + 1), "B"
    if job.kind == "lud":
        return 2.0 / 3.0 * n ** 3, "FLOP"
    if job.kind == "yolo":
        return yolo_flops(n, m) * it, "TC_FLOP"
    if job.kind == "resnet":
        return resnet_flops(n, m) * it, "TC_FLOP"
    return 0.0, "B"


def darknet_mix(n: int, seed: int, sizes=(416, 608, 832, 1024), batches=(1, 2, 4, 8, 16, 32, 64),
                resnet_sizes=(224, 448)) -> list[Job]:
    """Half YOLOv3-tiny, half ResNet-50 inference jobs (BASELINE cfg 2)."""
    rng = random.Random(f"{seed}|darknet|{n}")
    out = []
    for i in range(n):
        B = rng.choice(batches)
        if rng.random() < 0.5:
            out.append(Job("yolo", n=rng.choice(sizes), m=B, iters=1, seed=seed * 1000 + i))
        else:
            out.append(Job("resnet", n=rng.choice(resnet_sizes), m=B, iters=1, seed=seed * 1000 + i))
    return out


# cfg 2: jobs large enough that 8 co-running ones exceed the device (Darknet
# keeps every layer's output resident: 8-33 GB per YOLO job, 7-28 GB per
# ResNet-50 job at these sizes)
CFG2_SIZES, CFG2_BATCHES, CFG2_RESNET = (1280, 1536, 1792), (32, 64), (896, 1152)
