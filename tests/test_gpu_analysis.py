"""Sweep drivers (analysis.hpp:178-418) on the B200 schemes: the reference's
analysis_test.cpp properties on its tiny problem, plus the measured wall clock each cell
carries."""
import io

import pytest

from paper_1511_06051_b200 import analysis as an
from paper_1511_06051_b200 import csvio
from paper_1511_06051_b200 import netspec as ns

pytestmark = pytest.mark.gpu


def _ctx(sep, seed):
    from paper_1511_06051_b200 import schemes
    from paper_1511_06051_b200.data import Dataset
    from paper_1511_06051_b200.model import SgdOptions
    train = Dataset.synthetic(2, 1, 1, 16, 150, sep, seed, 0)
    evald = Dataset.synthetic(2, 1, 1, 16, 20, sep, seed, 1)
    return schemes.SchemeContext(net=ns.make_mlp(10, 1, 1, 16, 2, 4), train_data=train,
                                 eval_data=evald, batch=10, sgd=SgdOptions(0.1, 0.0), seed=1,
                                 cost=schemes.CostModel(1.0, 0.0, 1.0), target_accuracy=2.0,
                                 eval_steps=4, precision="fp32")


def test_heatmap_single_cell_grid():
    """analysis_test.cpp:130-160."""
    spec = an.HeatmapSpec(workers=[1], taus=[1, 5], seeds=[3, 4, 5], serial_iter_budget=400,
                          serial_eval_every=5, max_parallel_iters=800, target_accuracy=0.9)
    res = an.sweep_heatmap(_ctx(6.0, 301), spec)
    assert len(res.grid.cells) == 2 and len(res.grid.runs) == 6
    for cell in res.grid.cells:
        assert cell.reached
        assert cell.speedup == cell.serial_iters_to_target / (cell.tau * cell.rounds_to_target)
        assert 0.5 < cell.speedup < 2.0
        assert cell.measured_step_ms > 0.0 and cell.measured_sync_ms >= 0.0
    assert all(n_a >= 1 for _, n_a in res.baselines)
    buf = io.StringIO()
    csvio.write_heatmap(buf, res.grid)
    assert buf.getvalue().splitlines()[0] == csvio.HEATMAP_HEADER
    buf = io.StringIO()
    csvio.write_measured(buf, res.grid.runs, 10)
    assert len(buf.getvalue().splitlines()) == 7


def test_heatmap_derived_target_and_unreachable_baseline():
    """analysis_test.cpp:162-188."""
    spec = an.HeatmapSpec(workers=[1], taus=[1], seeds=[3], serial_iter_budget=400,
                          serial_eval_every=5, max_parallel_iters=800, target_at_serial_iters=100)
    res = an.sweep_heatmap(_ctx(6.0, 301), spec)
    assert 0.5 < res.target <= 1.0
    hopeless = an.HeatmapSpec(workers=[1], taus=[1], seeds=[3], serial_iter_budget=20,
                              serial_eval_every=5, max_parallel_iters=40,
                              target_accuracy=0.999999)
    with pytest.raises(RuntimeError):
        an.sweep_heatmap(_ctx(0.0, 301), hopeless)


def test_overhead_sweep():
    """analysis_test.cpp:190-208."""
    spec = an.OverheadSpec(sync_values=[0.0, 1.0, 4.0], workers=2, taus=[1, 5], seed=6,
                           serial_iter_budget=400, serial_eval_every=5, max_parallel_iters=800,
                           target_accuracy=0.9)
    res = an.sweep_overhead(_ctx(6.0, 303), spec)
    assert len(res.points) == 3 and res.points[0].naive == 2.0
    assert len(res.measurements) == 2 and all(m.reached for m in res.measurements)
    assert all(c > 0.0 for _, c, _ in res.measured)


def test_tau_sweep_shares_warm_start():
    """analysis_test.cpp:210-229."""
    spec = an.TauSweepSpec(taus=[1, 5, 10], workers=2, seed=8, max_parallel_iters=100,
                           warm_start_iters=10)
    traces = an.sweep_tau(_ctx(6.0, 305), spec)
    assert len(traces) == 3
    for t in traces:
        assert t.warm_digest == traces[0].warm_digest
        prev = 0.0
        for r in t.records:
            assert r.sim_time > prev
            prev = r.sim_time
    back = csvio.parse_trace(io.StringIO(csvio.trace_text(traces)))
    assert [len(t.records) for t in back] == [len(t.records) for t in traces]
