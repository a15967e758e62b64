"""K x tau sweep on the box's GPUs (analysis.hpp sweep_heatmap /
sweep_tau): writes the reference's heatmap.csv / heatmap_runs.csv / trace.csv schemas plus
measured.csv — the wall-clock C(b) per local step and S per average of every run, next to
the simulated clock.  Worker k runs on GPU k when K <= #GPUs.

  python tools/sweep.py --workers 1,2,4,8 --taus 1,10,50 --out sweep_out
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_1511_06051_b200 import analysis as an  # noqa: E402
from paper_1511_06051_b200 import csvio, netspec, schemes  # noqa: E402
from paper_1511_06051_b200.data import DeviceSyntheticDataset  # noqa: E402
from paper_1511_06051_b200.model import SgdOptions  # noqa: E402


def main():
    p = argparse.ArgumentParser()
    p.add_argument("--net", default="cifar10_quick", choices=["cifar10_quick", "cq-valid"])
    p.add_argument("--workers", default="1,2")
    p.add_argument("--taus", default="1,10")
    p.add_argument("--seeds", default="1")
    p.add_argument("--batch", type=int, default=100)
    p.add_argument("--per-class", type=int, default=500)
    p.add_argument("--serial-budget", type=int, default=300)
    p.add_argument("--eval-every", type=int, default=20)
    p.add_argument("--max-parallel-iters", type=int, default=300)
    p.add_argument("--target", type=float, default=None,
                   help="fixed target accuracy (default: derived at half the serial budget)")
    p.add_argument("--lr", type=float, default=0.01)
    p.add_argument("--separation", type=float, default=2.0,
                   help="generate_synthetic class separation (distance between class means)")
    p.add_argument("--precision", default="tf32")
    p.add_argument("--out", default="sweep_out")
    a = p.parse_args()
    import torch
    ngpu = max(1, torch.cuda.device_count())
    spec = (netspec.make_cifar10_quick(a.batch) if a.net == "cifar10_quick"
            else netspec.make_cq_valid(a.batch))
    train = DeviceSyntheticDataset(10, 3, 32, 32, a.per_class, a.separation, 12345, 0)
    evald = DeviceSyntheticDataset(10, 3, 32, 32, max(1, a.per_class // 10), a.separation, 12345, 1)
    ctx = schemes.SchemeContext(net=spec, train_data=train, eval_data=evald, batch=a.batch,
                                sgd=SgdOptions(a.lr, 0.9, 0.004 if a.net == "cifar10_quick"
                                               else 0.0),
                                seed=1, cost=schemes.CostModel(1.0, 0.0, 1.0), eval_steps=5,
                                devices=list(range(ngpu)), precision=a.precision,
                                average_mode="fast")
    hs = an.HeatmapSpec(workers=[int(x) for x in a.workers.split(",")],
                        taus=[int(x) for x in a.taus.split(",")],
                        seeds=[int(x) for x in a.seeds.split(",")],
                        serial_iter_budget=a.serial_budget, serial_eval_every=a.eval_every,
                        max_parallel_iters=a.max_parallel_iters, target_accuracy=a.target,
                        target_at_serial_iters=None if a.target else a.serial_budget // 2)
    res = an.sweep_heatmap(ctx, hs)
    os.makedirs(a.out, exist_ok=True)
    with open(os.path.join(a.out, "heatmap.csv"), "w") as f:
        csvio.write_heatmap(f, res.grid)
    with open(os.path.join(a.out, "heatmap_runs.csv"), "w") as f:
        csvio.write_heatmap_runs(f, res.grid)
    with open(os.path.join(a.out, "measured.csv"), "w") as f:
        csvio.write_measured(f, res.grid.runs, a.batch)
    with open(os.path.join(a.out, "trace.csv"), "w") as f:
        csvio.write_trace(f, res.serial_traces)
    print(f"target accuracy {res.target:.4f}; N_a per seed {res.baselines}")
    for name in ("heatmap.csv", "measured.csv"):
        print(open(os.path.join(a.out, name)).read())


if __name__ == "__main__":
    main()
