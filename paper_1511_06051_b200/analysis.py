"""Speedup analysis and sweep drivers — host mirror of analysis.hpp.

The formulas (naive_speedup, sparknet_speedup, best_tau_speedup, first_reach, the
overhead curves) are the reference's closed forms (analysis.hpp:14-69, 283-300); the
sweeps (sweep_heatmap / sweep_overhead / sweep_tau, analysis.hpp:178-418) drive the B200
run_serial / run_sparknet of schemes.py.  Each sweep cell also carries the MEASURED wall
clock of its run (compute per step C(b) and per-round synchronisation S), kept next to the
simulated clock and written to its own CSV (csvio.write_measured), never as new columns.
Cells run one after another: every run already spreads its K workers over the GPUs.
"""
from __future__ import annotations

from dataclasses import dataclass, field, replace
from typing import List, Optional, Sequence, Tuple

from .schemes import (EvalRecord, RunTrace, SchemeContext, run_serial, run_sparknet)


def naive_speedup(compute_seconds: float, workers: int, sync_seconds: float) -> float:
    """analysis.hpp:19-24: C / (C/K + S)."""
    if not compute_seconds > 0.0:
        raise ValueError("naive_speedup: C(b) must be > 0")
    if workers < 1:
        raise ValueError("naive_speedup: K must be >= 1")
    if sync_seconds < 0.0:
        raise ValueError("naive_speedup: S must be >= 0")
    return compute_seconds / (compute_seconds / float(workers) + sync_seconds)


def sparknet_speedup(serial_iters_to_target: float, compute_seconds: float, tau: float,
                     sync_seconds: float, rounds_to_target: float) -> float:
    """analysis.hpp:29-37: N_a C / ((tau C + S) M_a)."""
    if (not serial_iters_to_target > 0.0 or not compute_seconds > 0.0 or not tau > 0.0
            or not rounds_to_target > 0.0 or sync_seconds < 0.0):
        raise ValueError("sparknet_speedup: inputs must be positive (S may be zero)")
    return (serial_iters_to_target * compute_seconds /
            ((tau * compute_seconds + sync_seconds) * rounds_to_target))


@dataclass
class TauMeasurement:
    """analysis.hpp:40-44."""
    tau: int = 0
    rounds_to_target: int = 0
    reached: bool = True


@dataclass
class BestTau:
    tau: int = -1
    speedup: float = 0.0


def best_tau_speedup(measurements: Sequence[TauMeasurement], serial_iters_to_target: int,
                     compute_seconds: float, sync_seconds: float) -> BestTau:
    """analysis.hpp:54-69: ties prefer the smaller tau; unreached entries are skipped."""
    if not measurements:
        raise ValueError("best_tau_speedup: no measurements")
    best = BestTau()
    for m in measurements:
        if not m.reached:
            continue
        s = sparknet_speedup(float(serial_iters_to_target), compute_seconds, float(m.tau),
                             sync_seconds, float(m.rounds_to_target))
        if s > best.speedup or (s == best.speedup and best.tau != -1 and m.tau < best.tau):
            best = BestTau(m.tau, s)
    return best


def first_reach(trace: RunTrace, accuracy: float) -> Optional[EvalRecord]:
    """analysis.hpp:71-76."""
    for r in trace.records:
        if r.accuracy >= accuracy:
            return r
    return None


@dataclass
class SpeedupPoint:
    """analysis.hpp:80-90 (+ the measured wall clock of the run behind the point)."""
    workers: int = 1
    tau: int = 1
    sync_seconds: float = 0.0
    compute_seconds: float = 1.0
    seed: int = 0
    serial_iters_to_target: int = 0
    rounds_to_target: int = -1
    reached: bool = False
    speedup: float = 0.0
    measured_step_ms: float = 0.0   # wall clock: tau local steps / tau (median round)
    measured_sync_ms: float = 0.0   # wall clock: one average, S (median round)


@dataclass
class SweepGrid:
    """analysis.hpp:94-105."""
    workers: List[int] = field(default_factory=list)
    taus: List[int] = field(default_factory=list)
    target: float = 0.0
    cells: List[SpeedupPoint] = field(default_factory=list)
    runs: List[SpeedupPoint] = field(default_factory=list)

    def cell(self, worker_index: int, tau_index: int) -> SpeedupPoint:
        return self.cells[worker_index * len(self.taus) + tau_index]


@dataclass
class HeatmapSpec:
    """analysis.hpp:107-119 (threads accepted for API parity)."""
    workers: List[int] = field(default_factory=list)
    taus: List[int] = field(default_factory=list)
    seeds: List[int] = field(default_factory=list)
    serial_iter_budget: int = 0
    serial_eval_every: int = 10
    max_parallel_iters: int = 0
    warm_start_iters: int = 0
    target_accuracy: Optional[float] = None
    target_at_serial_iters: Optional[int] = None
    threads: int = 1


@dataclass
class HeatmapResult:
    grid: SweepGrid = field(default_factory=SweepGrid)
    target: float = 0.0
    baselines: List[Tuple[int, int]] = field(default_factory=list)
    serial_traces: List[RunTrace] = field(default_factory=list)


def lower_median(v):
    """analysis.hpp:128-132."""
    s = sorted(v)
    return s[(len(s) - 1) // 2]


def rounds_budget(max_parallel_iters: int, tau: int) -> int:
    return (max_parallel_iters + tau - 1) // tau


def baseline_trace(base: SchemeContext, seed: int, budget: int, eval_every: int) -> RunTrace:
    """analysis.hpp:140-146: serial baseline with early stopping disabled."""
    ctx = replace(base, seed=seed, target_accuracy=2.0,
                  devices=[base.devices[0]] if base.devices else None)
    return run_serial(ctx, budget, eval_every)


def accuracy_at_iters(trace: RunTrace, iters: int) -> float:
    """analysis.hpp:151-166: median accuracy within +-10% of iteration `iters`."""
    window = iters // 10
    near, past = [], False
    for r in trace.records:
        if iters - window <= r.serial_iters <= iters + window:
            near.append(r.accuracy)
        past |= r.serial_iters >= iters
    if not past or not near:
        raise RuntimeError("sweep: serial budget smaller than the target-derivation point")
    return lower_median(near)


def _for_workers(ctx: SchemeContext, k: int) -> SchemeContext:
    """Worker k on GPU k when the context lists >= K devices, else all on the first."""
    if ctx.devices and len(ctx.devices) > 1:
        return replace(ctx, devices=list(ctx.devices[:k]) if k <= len(ctx.devices)
                       else [ctx.devices[0]])
    return ctx


def _measured(trace: RunTrace, tau: int) -> Tuple[float, float]:
    if not trace.compute_ms:
        return 0.0, 0.0
    # median over rounds after the first, which also pays the one-time CUDA-graph capture
    # and the communicators' connection setup (the first round alone if it is the only one)
    comp = trace.compute_ms[1:] or trace.compute_ms
    sync = trace.sync_ms[1:] or trace.sync_ms
    return lower_median(comp) / tau, lower_median(sync)


def sweep_heatmap(base: SchemeContext, spec: HeatmapSpec) -> HeatmapResult:
    """analysis.hpp:178-280."""
    if not spec.workers or not spec.taus or not spec.seeds:
        raise ValueError("heatmap: worker, tau and seed axes must be nonempty")
    if spec.serial_iter_budget < 1 or spec.max_parallel_iters < 1:
        raise ValueError("heatmap: budgets must be >= 1")
    if spec.target_accuracy is None and spec.target_at_serial_iters is None:
        raise ValueError("heatmap: no target accuracy and no derivation point")
    res = HeatmapResult()
    res.serial_traces = [baseline_trace(base, s, spec.serial_iter_budget, spec.serial_eval_every)
                         for s in spec.seeds]
    if spec.target_accuracy is not None:
        target = spec.target_accuracy
    else:
        target = lower_median([accuracy_at_iters(t, spec.target_at_serial_iters)
                               for t in res.serial_traces])
    res.target = target
    for seed, t in zip(spec.seeds, res.serial_traces):
        hit = first_reach(t, target)
        if hit is None:
            raise RuntimeError(f"heatmap: serial baseline for seed {seed} did not reach target "
                               f"{target:.6f} within {spec.serial_iter_budget} iterations")
        res.baselines.append((seed, hit.serial_iters))
    grid = res.grid
    grid.workers, grid.taus, grid.target = list(spec.workers), list(spec.taus), target
    nk, nt = len(spec.workers), len(spec.taus)
    grid.runs = [SpeedupPoint() for _ in range(len(spec.seeds) * nk * nt)]
    for si, seed in enumerate(spec.seeds):
        for ki, k in enumerate(spec.workers):
            for ti, tau in enumerate(spec.taus):
                ctx = _for_workers(replace(base, seed=seed, target_accuracy=target), k)
                trace = run_sparknet(ctx, k, tau, rounds_budget(spec.max_parallel_iters, tau),
                                     spec.warm_start_iters)
                p = SpeedupPoint(workers=k, tau=tau, sync_seconds=base.cost.sync_seconds,
                                 compute_seconds=base.cost.compute_seconds, seed=seed,
                                 serial_iters_to_target=res.baselines[si][1])
                hit = first_reach(trace, target)
                if hit is not None:
                    p.reached = True
                    p.rounds_to_target = hit.rounds
                    p.speedup = float(p.serial_iters_to_target) / (float(tau) * float(hit.rounds))
                p.measured_step_ms, p.measured_sync_ms = _measured(trace, tau)
                grid.runs[(si * nk + ki) * nt + ti] = p
    grid.cells = []
    for ki in range(nk):
        for ti in range(nt):
            runs = [grid.runs[(si * nk + ki) * nt + ti] for si in range(len(spec.seeds))]
            runs = sorted(runs, key=lambda q: q.speedup)  # stable, unreached (0) first
            grid.cells.append(runs[(len(runs) - 1) // 2])
    return res


@dataclass
class OverheadPoint:
    """analysis.hpp:276-281."""
    sync_seconds: float = 0.0
    naive: float = 0.0
    sparknet: float = 0.0
    best_tau: int = -1


def compute_overhead_curves(serial_iters_to_target: int, measurements: Sequence[TauMeasurement],
                            workers: int, sync_values: Sequence[float]) -> List[OverheadPoint]:
    """analysis.hpp:286-301 with C(b) normalised to 1."""
    pts = []
    for s in sync_values:
        best = best_tau_speedup(measurements, serial_iters_to_target, 1.0, s)
        pts.append(OverheadPoint(s, naive_speedup(1.0, workers, s), best.speedup, best.tau))
    return pts


@dataclass
class OverheadSpec:
    """analysis.hpp:303-315."""
    sync_values: List[float] = field(default_factory=list)
    workers: int = 1
    taus: List[int] = field(default_factory=list)
    seed: int = 0
    serial_iter_budget: int = 0
    serial_eval_every: int = 10
    max_parallel_iters: int = 0
    warm_start_iters: int = 0
    target_accuracy: Optional[float] = None
    target_at_serial_iters: Optional[int] = None
    threads: int = 1


@dataclass
class OverheadResult:
    target: float = 0.0
    serial_iters_to_target: int = 0
    measurements: List[TauMeasurement] = field(default_factory=list)
    points: List[OverheadPoint] = field(default_factory=list)
    measured: List[Tuple[int, float, float]] = field(default_factory=list)  # (tau, C ms, S ms)


def sweep_overhead(base: SchemeContext, spec: OverheadSpec) -> OverheadResult:
    """analysis.hpp:327-368."""
    if not spec.sync_values or not spec.taus:
        raise ValueError("overhead: sync and tau axes must be nonempty")
    if spec.workers < 1:
        raise ValueError("overhead: need at least one worker")
    if spec.target_accuracy is None and spec.target_at_serial_iters is None:
        raise ValueError("overhead: no target accuracy and no derivation point")
    res = OverheadResult()
    baseline = baseline_trace(base, spec.seed, spec.serial_iter_budget, spec.serial_eval_every)
    res.target = (spec.target_accuracy if spec.target_accuracy is not None
                  else accuracy_at_iters(baseline, spec.target_at_serial_iters))
    hit = first_reach(baseline, res.target)
    if hit is None:
        raise RuntimeError(f"overhead: serial baseline did not reach target {res.target:.6f}")
    res.serial_iters_to_target = hit.serial_iters
    for tau in spec.taus:
        ctx = _for_workers(replace(base, seed=spec.seed, target_accuracy=res.target),
                           spec.workers)
        trace = run_sparknet(ctx, spec.workers, tau, rounds_budget(spec.max_parallel_iters, tau),
                             spec.warm_start_iters)
        h = first_reach(trace, res.target)
        res.measurements.append(TauMeasurement(tau, h.rounds, True) if h is not None
                                else TauMeasurement(tau, 0, False))
        res.measured.append((tau,) + _measured(trace, tau))
    res.points = compute_overhead_curves(res.serial_iters_to_target, res.measurements,
                                         spec.workers, spec.sync_values)
    return res


@dataclass
class TauSweepSpec:
    """analysis.hpp:370-378."""
    taus: List[int] = field(default_factory=list)
    workers: int = 5
    seed: int = 0
    max_parallel_iters: int = 0
    warm_start_iters: int = 0
    target_accuracy: float = 2.0
    threads: int = 1


def sweep_tau(base: SchemeContext, spec: TauSweepSpec) -> List[RunTrace]:
    """analysis.hpp:383-404: one full trace per tau (shared seed -> shared warm start)."""
    if not spec.taus:
        raise ValueError("tau sweep: tau axis must be nonempty")
    out = []
    for tau in spec.taus:
        ctx = _for_workers(replace(base, seed=spec.seed, target_accuracy=spec.target_accuracy),
                           spec.workers)
        out.append(run_sparknet(ctx, spec.workers, tau,
                                rounds_budget(spec.max_parallel_iters, tau),
                                spec.warm_start_iters))
    return out
