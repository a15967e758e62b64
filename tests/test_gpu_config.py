"""`train` from config files on the GPUs: the reference's own cmd_train (experiment.hpp:185-231,
unmodified, through include/parasgd_shim) on the B200 drop-in (tests/cpp/config_test).
  * reference keys only (lenet-small): the trace equals the oracle's run_sparknet on the
    same configuration (iteration counts, rounds and simulated clock exactly; accuracies
    within the fp32-vs-fp64 argmax margin);
  * B200 keys (cifar10_quick preset, weight decay, TF32, NCCL average mode): the trace equals
    the Python API's run_sparknet on the same context, record for record."""
import csv
import os
import subprocess

import numpy as np
import pytest

from paper_1511_06051_b200 import netspec as ns

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
EXE = os.path.join(ROOT, "tests", "cpp", "config_test")
CFG = os.path.join(ROOT, "tests", "configs")


def train(cfg, tmp_path):
    if not os.path.exists(EXE):
        pytest.skip("config_test not built (needs the reference headers at build time)")
    env = dict(os.environ, PARASGD_OUT=str(tmp_path))
    out = subprocess.run([EXE, "train", os.path.join(CFG, cfg)], env=env, capture_output=True,
                         text=True, timeout=600)
    assert out.returncode == 0, out.stderr[-2000:] + out.stdout[-2000:]
    assert "wrote" in out.stdout
    with open(tmp_path / "trace.csv") as f:
        rows = list(csv.DictReader(f))
    return [(r["scheme"], int(r["K"]), int(r["tau"]), int(r["b"]), int(r["round"]),
             int(r["serial_iters"]), int(r["parallel_iters"]), float(r["sim_time"]),
             float(r["accuracy"])) for r in rows]


def test_reference_config_trains_like_the_oracle(tmp_path, oracle_lib):
    got = train("sparknet_lenet.cfg", tmp_path)
    tr = oracle_lib.generate_synthetic(10, 1, 16, 16, 60, 2.0, 12345, 0)
    ev = oracle_lib.generate_synthetic(10, 1, 16, 16, 20, 2.0, 12345, 1)
    recs, _, _ = oracle_lib.run_sparknet(ns.make_lenet_small(20, 1, 16, 16, 10), tr, ev, 20,
                                         0.05, 0.9, 1, 2, 5, 3, 5, eval_steps=2,
                                         cost=(1.0, 10.0), want_weights=True)
    assert len(got) == len(recs) == 3
    for g, w in zip(got, recs):
        assert g[:4] == ("sparknet", 2, 5, 20)
        assert (g[5], g[6], g[4], g[7]) == (w[0], w[1], w[2], w[3])
        assert abs(g[8] - w[4]) <= 0.1


def test_b200_config_keys_train_like_the_python_api(tmp_path):
    got = train("sparknet_cifar10_quick_tf32.cfg", tmp_path)
    from paper_1511_06051_b200 import schemes
    from paper_1511_06051_b200.data import Dataset, generate_synthetic
    from paper_1511_06051_b200.model import SgdOptions
    img, lab = generate_synthetic(10, 3, 32, 32, 60, 2.0, 12345, 0)
    train_ds = Dataset(img, lab, 10)
    img, lab = generate_synthetic(10, 3, 32, 32, 20, 2.0, 12345, 1)
    eval_ds = Dataset(img, lab, 10)
    ctx = schemes.SchemeContext(net=ns.make_cifar10_quick(20), train_data=train_ds,
                                eval_data=eval_ds, batch=20, sgd=SgdOptions(0.01, 0.9, 0.004),
                                seed=1, cost=schemes.CostModel(1.0, 10.0, 1.0),
                                target_accuracy=2.0, eval_steps=4, precision="tf32")
    ctx.average_mode = "fast"
    t = schemes.run_sparknet(ctx, 2, 10, 4, 10)
    assert len(got) == len(t.records) == 4
    for g, r in zip(got, t.records):
        assert g[:4] == ("sparknet", 2, 10, 20)
        assert (g[5], g[6], g[4]) == (r.serial_iters, r.parallel_iters, r.rounds)
        assert g[7] == r.sim_time
        assert g[8] == pytest.approx(r.accuracy, abs=1e-12)
    assert all(0.0 <= g[8] <= 1.0 for g in got) and np.isfinite(got[-1][8])
