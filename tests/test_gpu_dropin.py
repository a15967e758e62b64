"""The C++ drop-in (include/parasgd_b200: Net + run_sparknet over the C ABI), driven by
reference-style C++ (tests/cpp/dropin_test.cpp), against the pinned CPU oracle."""
import json
import os
import subprocess

import numpy as np
import pytest

from oracle.pyoracle import max_relative_deviation
from paper_1511_06051_b200 import netspec as ns

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_cpp_dropin_run_sparknet_matches_oracle(oracle_lib):
    exe = os.path.join(ROOT, "tests", "cpp", "dropin_test")
    if not os.path.exists(exe):
        pytest.skip("dropin_test not built (needs the reference headers at build time)")
    out = subprocess.run([exe], capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stderr[-2000:]
    res = json.loads(out.stdout.strip().splitlines()[-1])
    assert res["failures"] == 0
    train = oracle_lib.generate_synthetic(10, 1, 16, 16, 24, 2.0, 12345, 0)
    evald = oracle_lib.generate_synthetic(10, 1, 16, 16, 6, 2.0, 12345, 1)
    spec = ns.make_lenet_small(10, 1, 16, 16, 10)
    recs, _, rw = oracle_lib.run_sparknet(spec, train, evald, 10, 0.05, 0.9, 1, 2, 2, 3, 2,
                                          eval_steps=2, cost=(2.0, 10.0), want_weights=True)
    got = res["records"]
    assert [r[:4] for r in got] == [list(r[:4]) for r in recs]   # iters / rounds / sim clock
    for g, w in zip(got, recs):
        assert abs(g[4] - w[4]) <= 0.1                            # accuracy (fp32 vs fp64 argmax)
    # 8 SGD steps of fp32 vs fp64 from the same (fp32-representable) data
    for r in range(3):
        assert max_relative_deviation(np.array(res["round_weights"][r]), rw[r]) <= 1e-4
    # run_naive through the drop-in vs the oracle's (reference-pinned) run_naive
    _, sw = oracle_lib.run_naive(spec, train, evald, 10, 0.05, 0.9, 1, 2, 4, 2, eval_steps=2,
                                 cost=(2.0, 10.0, 1.0), want_weights=True)
    assert len(res["naive_weights"]) == 4
    for s in range(4):
        assert max_relative_deviation(np.array(res["naive_weights"][s]), sw[s]) <= 2e-4
