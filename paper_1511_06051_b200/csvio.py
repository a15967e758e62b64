"""trace.csv / heatmap.csv / overhead.csv — the reference's schemas (csv.hpp:19-125),
byte-identical output for the same values, plus measured.csv: the wall-clock C(b) and S
of each run, kept in its own file so the reference's files are unchanged.
"""
from __future__ import annotations

import io
import math
from typing import Iterable, List, Sequence, TextIO

from .analysis import OverheadPoint, SpeedupPoint, SweepGrid
from .schemes import EvalRecord, RunTrace


def format_double(v: float) -> str:
    """csv.hpp:22-33: the shortest '%.*g' (precision 1..17) that parses back exactly."""
    if math.isinf(v):
        return "inf" if v > 0 else "-inf"
    best = ""
    for p in range(1, 18):
        s = "%.*g" % (p, v)
        if float(s) == v and (not best or len(s) < len(best)):
            best = s
    return best


TRACE_HEADER = "scheme,K,tau,b,round,serial_iters,parallel_iters,sim_time,accuracy"


def write_trace(out: TextIO, traces) -> None:
    """csv.hpp:38-47."""
    if isinstance(traces, RunTrace):
        traces = [traces]
    out.write(TRACE_HEADER + "\n")
    for t in traces:
        for r in t.records:
            out.write(f"{t.scheme},{t.workers},{t.tau},{t.batch},{r.rounds},{r.serial_iters},"
                      f"{r.parallel_iters},{format_double(r.sim_time)},"
                      f"{format_double(r.accuracy)}\n")


def parse_trace(inp: TextIO) -> List[RunTrace]:
    """csv.hpp:56-92: consecutive rows with the same (scheme, K, tau, b) form one run."""
    lines = inp.read().split("\n")
    if not lines or lines == [""]:
        raise RuntimeError("trace csv: empty file")
    if lines[0] != TRACE_HEADER:
        raise RuntimeError("trace csv: unexpected header")
    traces: List[RunTrace] = []
    for line in lines[1:]:
        if not line:
            continue
        cells = line.split(",")
        if len(cells) != 9:
            raise RuntimeError("trace csv: malformed row: " + line)
        k, tau, b = int(cells[1]), int(cells[2]), int(cells[3])
        if (not traces or traces[-1].scheme != cells[0] or traces[-1].workers != k
                or traces[-1].tau != tau or traces[-1].batch != b):
            traces.append(RunTrace(scheme=cells[0], workers=k, tau=tau, batch=b))
        traces[-1].records.append(EvalRecord(serial_iters=int(cells[5]),
                                             parallel_iters=int(cells[6]), rounds=int(cells[4]),
                                             sim_time=float(cells[7]), accuracy=float(cells[8])))
    return traces


HEATMAP_HEADER = "K,tau,N_a,M_a,speedup,reached"


def _heatmap_point(p: SpeedupPoint) -> str:
    m = str(p.rounds_to_target) if p.reached else "inf"
    return (f"{p.workers},{p.tau},{p.serial_iters_to_target},{m},{format_double(p.speedup)},"
            f"{1 if p.reached else 0}\n")


def write_heatmap(out: TextIO, grid: SweepGrid) -> None:
    """csv.hpp:106-109."""
    out.write(HEATMAP_HEADER + "\n")
    for p in grid.cells:
        out.write(_heatmap_point(p))


def write_heatmap_runs(out: TextIO, grid: SweepGrid) -> None:
    """csv.hpp:112-118."""
    out.write("seed," + HEATMAP_HEADER + "\n")
    for p in grid.runs:
        out.write(f"{p.seed},{_heatmap_point(p)}")


OVERHEAD_HEADER = "S,naive_speedup,sparknet_speedup,best_tau"


def write_overhead(out: TextIO, points: Sequence[OverheadPoint]) -> None:
    """csv.hpp:120-125."""
    out.write(OVERHEAD_HEADER + "\n")
    for p in points:
        out.write(f"{format_double(p.sync_seconds)},{format_double(p.naive)},"
                  f"{format_double(p.sparknet)},{p.best_tau}\n")


MEASURED_HEADER = "seed,K,tau,b,step_ms,sync_ms,sync_fraction"


def write_measured(out: TextIO, points: Iterable[SpeedupPoint], batch: int) -> None:
    """Measured wall clock per sweep run: C(b) per local step and S per average (ms), and
    S / (tau C(b) + S), the share of a round spent averaging."""
    out.write(MEASURED_HEADER + "\n")
    for p in points:
        rnd = p.tau * p.measured_step_ms + p.measured_sync_ms
        frac = p.measured_sync_ms / rnd if rnd > 0 else 0.0
        out.write(f"{p.seed},{p.workers},{p.tau},{batch},{format_double(p.measured_step_ms)},"
                  f"{format_double(p.measured_sync_ms)},{format_double(frac)}\n")


def trace_text(traces) -> str:
    buf = io.StringIO()
    write_trace(buf, traces)
    return buf.getvalue()
