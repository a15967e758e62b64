"""analysis.hpp closed forms and csv.hpp schemas, CPU only: the
reference's analysis_test.cpp cases, csv format_double pinned to reference-generated golden
strings, and (where oracle/_ref exists) live comparisons with the reference's functions."""
import io
import math

import numpy as np
import pytest

from paper_1511_06051_b200 import analysis as an
from paper_1511_06051_b200 import csvio
from paper_1511_06051_b200.schemes import EvalRecord, RunTrace


def test_naive_speedup_formula():
    """analysis_test.cpp:30-48."""
    assert an.naive_speedup(1.0, 5, 0.0) == 5.0
    assert an.naive_speedup(2.0, 5, 20.0) == pytest.approx(2.0 / 20.4, rel=1e-12)
    rng = np.random.default_rng(61)
    for _ in range(200):
        c = rng.uniform(0.1, 10.0)
        k = int(1 + rng.integers(16))
        s = rng.uniform(0.0, 10.0)
        v = an.naive_speedup(c, k, s)
        assert v > 0.0
        if s > 0.0:
            assert v <= c / s
        if s >= c:
            assert v < 1.0 + 1e-12
        assert v > an.naive_speedup(c, k, s + 0.5)
        assert an.naive_speedup(c, k + 1, s) > v
    with pytest.raises(ValueError):
        an.naive_speedup(0.0, 2, 1.0)


def test_sparknet_speedup_formula():
    """analysis_test.cpp:50-71."""
    assert an.sparknet_speedup(10000, 1.0, 50, 20.0, 40) == pytest.approx(10000 / 2800, rel=1e-12)
    assert an.sparknet_speedup(1200, 2.0, 10, 0.0, 30) == pytest.approx(4.0, rel=1e-12)
    v = an.sparknet_speedup(500, 2.0, 50, 20.0, 10)
    assert v == pytest.approx(100.0 / 120.0, rel=1e-12) and v <= 1.0
    rng = np.random.default_rng(67)
    for _ in range(100):
        n, m, tau, s = (rng.uniform(100, 1e4), rng.uniform(1, 100), rng.uniform(1, 100),
                        rng.uniform(0, 50))
        assert an.sparknet_speedup(n, 1.0, tau, s, m) > an.sparknet_speedup(n, 1.0, tau, s + 1, m)


def test_best_tau():
    """analysis_test.cpp:73-106."""
    best = an.best_tau_speedup([an.TauMeasurement(50, 40)], 10000, 1.0, 20.0)
    assert best.tau == 50 and best.speedup == pytest.approx(10000 / 2800)
    tied = [an.TauMeasurement(2, 9), an.TauMeasurement(1, 10)]
    best = an.best_tau_speedup(tied, 900, 1.0, 8.0)
    assert best.speedup == pytest.approx(10.0) and best.tau == 1
    rng = np.random.default_rng(71)
    for _ in range(50):
        allm = [an.TauMeasurement(t, int(1 + rng.integers(200)))
                for t in (1, 2, 5, 10, 25, 100, 500, 1000, 2500)]
        s = rng.uniform(0, 100)
        assert (an.best_tau_speedup(allm, 5000, 1.0, s).speedup >=
                an.best_tau_speedup(allm[:4], 5000, 1.0, s).speedup)
    mixed = [an.TauMeasurement(1, 0, False), an.TauMeasurement(5, 10)]
    assert an.best_tau_speedup(mixed, 100, 1.0, 0.0).tau == 5
    assert an.best_tau_speedup([an.TauMeasurement(1, 0, False)], 100, 1.0, 0.0).tau == -1


def test_overhead_curves():
    """analysis_test.cpp:108-128."""
    ms = [an.TauMeasurement(1, 100), an.TauMeasurement(10, 12), an.TauMeasurement(100, 2)]
    pts = an.compute_overhead_curves(1000, ms, 5, [0.0, 1.0, 10.0, 100.0])
    assert len(pts) == 4 and pts[0].naive == 5.0 and pts[1].naive < 1.0
    for a, b in zip(pts, pts[1:]):
        assert b.naive < a.naive and b.sparknet <= a.sparknet
    for p in pts:
        for m in ms:
            if m.tau == p.best_tau:
                assert p.sparknet == pytest.approx(
                    an.sparknet_speedup(1000, 1.0, m.tau, p.sync_seconds, m.rounds_to_target))


def test_first_reach_and_medians():
    """analysis_test.cpp:231-238; lower median / accuracy_at_iters (analysis.hpp:128-166)."""
    t = RunTrace(records=[EvalRecord(10, 0, 0, 10.0, 0.2), EvalRecord(20, 0, 0, 20.0, 0.5),
                          EvalRecord(30, 0, 0, 30.0, 0.4)])
    assert an.first_reach(t, 0.5).serial_iters == 20
    assert an.first_reach(t, 0.45).serial_iters == 20
    assert an.first_reach(t, 0.9) is None
    assert an.lower_median([3, 1, 2, 4]) == 2
    assert an.accuracy_at_iters(t, 20) == 0.5
    with pytest.raises(RuntimeError):
        an.accuracy_at_iters(t, 100)
    assert an.rounds_budget(10, 3) == 4


def test_format_double_pinned_to_reference(golden):
    vals = golden["fmt_values"]
    want = str(golden["fmt_strings"]).split("|")
    assert [csvio.format_double(float(v)) for v in vals] == want
    assert csvio.format_double(math.inf) == "inf" and csvio.format_double(-math.inf) == "-inf"


def test_format_double_and_speedups_live_reference(ref_lib):
    rng = np.random.default_rng(5)
    for v in np.concatenate([rng.normal(size=50), 10.0 ** rng.uniform(-30, 30, 50)]):
        assert csvio.format_double(float(v)) == ref_lib.format_double(float(v))
    for _ in range(50):
        c, k, s = rng.uniform(0.1, 5), int(rng.integers(1, 9)), rng.uniform(0, 5)
        assert an.naive_speedup(c, k, s) == ref_lib.naive_speedup(c, k, s)
        n, tau, m = rng.uniform(10, 1e4), rng.uniform(1, 100), rng.uniform(1, 100)
        assert an.sparknet_speedup(n, c, tau, s, m) == ref_lib.sparknet_speedup(n, c, tau, s, m)


def test_trace_csv_round_trip():
    """csv.hpp:35-92: write then parse gives back the same runs and values."""
    a = RunTrace(scheme="sparknet", workers=2, tau=5, batch=10,
                 records=[EvalRecord(3, 5, 1, 19.0, 0.25), EvalRecord(3, 10, 2, 1 / 3, 0.5)])
    b = RunTrace(scheme="serial", workers=1, tau=0, batch=10,
                 records=[EvalRecord(10, 0, 0, 10.0, 0.9)])
    text = csvio.trace_text([a, b])
    assert text.splitlines()[0] == csvio.TRACE_HEADER
    assert text.splitlines()[1] == "sparknet,2,5,10,1,3,5,19,0.25"
    back = csvio.parse_trace(io.StringIO(text))
    assert [(t.scheme, t.workers, t.tau, t.batch) for t in back] == [
        ("sparknet", 2, 5, 10), ("serial", 1, 0, 10)]
    assert back[0].records[1].sim_time == 1 / 3 and back[1].records[0].accuracy == 0.9
    with pytest.raises(RuntimeError, match="unexpected header"):
        csvio.parse_trace(io.StringIO("x\n"))
    with pytest.raises(RuntimeError, match="malformed row"):
        csvio.parse_trace(io.StringIO(csvio.TRACE_HEADER + "\n1,2\n"))


def test_heatmap_and_overhead_csv():
    """csv.hpp:94-125 row formats (unreached -> M_a 'inf', reached flag)."""
    g = an.SweepGrid(workers=[2], taus=[1, 5], target=0.9, cells=[
        an.SpeedupPoint(2, 1, serial_iters_to_target=40, rounds_to_target=30, reached=True,
                        speedup=40 / 30, seed=3),
        an.SpeedupPoint(2, 5, serial_iters_to_target=40, seed=3)])
    g.runs = list(g.cells)
    buf = io.StringIO()
    csvio.write_heatmap(buf, g)
    assert buf.getvalue().splitlines() == [csvio.HEATMAP_HEADER,
                                           "2,1,40,30,1.3333333333333333,1", "2,5,40,inf,0,0"]
    buf = io.StringIO()
    csvio.write_heatmap_runs(buf, g)
    assert buf.getvalue().splitlines()[1] == "3,2,1,40,30,1.3333333333333333,1"
    buf = io.StringIO()
    csvio.write_overhead(buf, [an.OverheadPoint(0.0, 5.0, 4.5, 10)])
    assert buf.getvalue().splitlines() == [csvio.OVERHEAD_HEADER, "0,5,4.5,10"]
