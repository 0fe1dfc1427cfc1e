"""Benchmark harness for the CLI (mirror of the reference's bench.py module).

Same entry points as the reference (bench.py:24-200 there) -- BenchResult,
run_strong_scaling, run_edge_sweep, speedups, linear_fit, emit_report --
timing the GPU edge pass instead of the CPU worker pool:

  * the timed region is one pass (histogram + pull) over a graph already
    resident and prepared in HBM, measured with CUDA events on each
    device's launching stream, max over devices; graph generation, CSR
    build and shard preparation stay outside, as the reference keeps
    build_csr and the projection outside (bench.py:1-7, 79-82);
  * repetitions are interleaved round-robin across configurations after one
    untimed warm-up each (bench.py:49-69);
  * the strong-scaling axis is the GPU (row shard) count;
  * results.csv keeps the reference's columns (name,n,s,k,workers,atomics,
    median_s,reps; workers = GPUs) and appends gpus, variant, geps and
    roofline_frac (B_min of SURVEY.md 8(d) / time / measured HBM peak x GPUs).
    No plots are drawn (matplotlib is not installed).
"""

import csv
import json
import logging
import os
from dataclasses import dataclass, field

import numpy as np

from .errors import ValidationError

logger = logging.getLogger(__name__)

CSV_COLUMNS = ["name", "n", "s", "k", "workers", "atomics", "median_s", "reps", "gpus", "variant", "geps",
               "roofline_frac"]


def _hbm_peak_gbs():
    here = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    try:
        with open(os.path.join(here, "MEASURED_PEAKS.json")) as fh:
            return float(json.load(fh)["hbm_gbs"])
    except Exception:
        return 6650.0  # B200_PROFILING.md fallback


@dataclass
class BenchResult:
    """Timing record for one (graph, GPU count) configuration (bench.py:27-47)."""

    name: str
    n: int
    s: int
    k: int
    gpus: int
    weighted: bool = False
    variant: str = "pull"
    times: list = field(default_factory=list)

    def __post_init__(self):
        if len(self.times) < 3:
            raise ValidationError("a reported number needs at least 3 repetitions")
        if any(t <= 0 for t in self.times):
            raise ValidationError("per-rep times must be positive")

    @property
    def workers(self) -> int:
        return self.gpus

    @property
    def reps(self) -> int:
        return len(self.times)

    @property
    def median_s(self) -> float:
        return float(np.median(self.times))

    @property
    def geps(self) -> float:
        return self.s / self.median_s / 1e9

    @property
    def bmin_bytes(self) -> int:
        return self.s * (8 + 4 * int(self.weighted)) + 4 * self.n + 4 * self.n * self.k

    @property
    def roofline_frac(self) -> float:
        return self.bmin_bytes / self.median_s / 1e9 / (_hbm_peak_gbs() * self.gpus)


def _timed_rounds(passes, reps):
    """Warm each prepared pass once, then time reps rounds round-robin;
    a pass's time is the max over its devices (seconds)."""
    for p in passes:
        p.run()
    times = [[] for _ in passes]
    for _ in range(reps):
        for i, p in enumerate(passes):
            ms = p.run()
            times[i].append(max(ms.values()) * 1e-3 if ms else 0.0)
    return times


def run_strong_scaling(graph, y, gpu_counts, reps=5, name="graph"):
    """Time the pass at each GPU count on a fixed graph (bench.py:72-96)."""
    from .multi import ShardedPass

    if reps < 3:
        raise ValidationError("reps must be at least 3")
    passes = [ShardedPass(graph, y, g) for g in gpu_counts]
    times = _timed_rounds(passes, reps)
    results = []
    for g, p, t in zip(gpu_counts, passes, times):
        results.append(BenchResult(name=name, n=p.n, s=p.s, k=y.k, gpus=g, weighted=p.weighted, times=t))
        logger.info("%s gpus=%d median=%.6fs", name, g, results[-1].median_s)
    return results


def speedups(results):
    """Map GPU count -> speedup relative to the 1-GPU median (bench.py:99-105)."""
    base = [r for r in results if r.gpus == 1]
    if not base:
        raise ValidationError("speedups need a 1-GPU measurement")
    t1 = base[0].median_s
    return {r.gpus: t1 / r.median_s for r in results}


def run_edge_sweep(sizes, n_per_s, k, seed, reps=5, fraction=0.1, gpus=1):
    """Time the pass on ER graphs of growing edge count (bench.py:108-142)."""
    from .graph import generate_erdos_renyi
    from .labeling import random_labels
    from .multi import ShardedPass

    if len(sizes) == 0:
        raise ValidationError("sizes must be nonempty")
    if any(b <= a for a, b in zip(sizes, sizes[1:])):
        raise ValidationError("sizes must be increasing")
    if reps < 3:
        raise ValidationError("reps must be at least 3")
    passes = []
    for i, s in enumerate(sizes):
        n = max(1, int(round(s * n_per_s)))
        el = generate_erdos_renyi(n, s, seed + i)
        y = random_labels(n, k, fraction, seed + 1000 + i)
        passes.append(ShardedPass(el, y, gpus))
    times = _timed_rounds(passes, reps)
    results = []
    for s, p, t in zip(sizes, passes, times):
        results.append(BenchResult(name=f"er-{s}", n=p.n, s=s, k=k, gpus=gpus, weighted=False, times=t))
        logger.info("er s=%d median=%.6fs", s, results[-1].median_s)
    return results


def linear_fit(sizes, times):
    """Least-squares line through (sizes, times); returns (slope, icept, r2) (bench.py:145-154)."""
    x = np.asarray(sizes, dtype=np.float64)
    t = np.asarray(times, dtype=np.float64)
    slope, icept = np.polyfit(x, t, 1)
    pred = slope * x + icept
    ss_res = float(np.sum((t - pred) ** 2))
    ss_tot = float(np.sum((t - t.mean()) ** 2))
    r2 = 1.0 if ss_tot == 0 else 1.0 - ss_res / ss_tot
    return float(slope), float(icept), r2


def emit_report(results, out_dir):
    """Write results.csv into out_dir (the reference's columns + GPU columns)."""
    os.makedirs(out_dir, exist_ok=True)
    with open(os.path.join(out_dir, "results.csv"), "w", newline="", encoding="utf-8") as fh:
        w = csv.writer(fh)
        w.writerow(CSV_COLUMNS)
        for r in results:
            w.writerow([r.name, r.n, r.s, r.k, r.workers, "false", f"{r.median_s:.9g}", r.reps, r.gpus, r.variant,
                        f"{r.geps:.6g}", f"{r.roofline_frac:.6g}"])
