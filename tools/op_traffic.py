"""Per-op DRAM traffic of one training step, for bench.py's roofline "traffic" field.

  # on the GPU box: one profiled step of the bench workload under ncu (eager launches)
  PSG_EAGER=1 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
      --csv --log-file gpurun_out/ops.csv python tools/op_traffic.py run --workload alexnet \
      --ops gpurun_out/ops.json
  # anywhere: map the step's launches onto the op list
  python tools/op_traffic.py summarize gpurun_out/ops.csv gpurun_out/ops.json \
      profiles/round1/alexnet_op_traffic.json

`run` trains two steps, then calls profile_step(repeats=1): its warm-up and timed
repetitions are each one full step in op order, so the last sum(launches) kernels of the
ncu log are the timed step.  ncu times are cold-cache and serialised: use them for bytes
and shares, not absolute speed.
"""
import argparse
import csv
import io
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def run(a):
    sys.argv = [sys.argv[0]]
    import bench
    from paper_1511_06051_b200 import data as pdata
    from paper_1511_06051_b200 import model
    spec, b = bench.make_spec(a.workload)
    _, _, _, _, lr, mu, wd = bench.WORKLOADS[a.workload]
    ds = bench.build_dataset(a.workload, 1)
    net = model.Net(spec, 1, precision=a.precision)
    net.set_sgd(model.SgdOptions(lr, mu, wd))
    net.set_training_data(pdata.make_worker_iterator(pdata.shard(ds, 1, 1), 0, b, 1))
    net.train(2)
    ops = net.profile_step(repeats=1)
    with open(a.ops, "w") as f:
        json.dump({"workload": a.workload, "precision": a.precision, "ops": ops}, f, indent=1)


def load_ncu(path):
    text = open(path).read()
    rows = list(csv.DictReader(io.StringIO(text[text.find('"ID"'):])))
    kern = {}
    for r in rows:
        k = int(r["ID"])
        d = kern.setdefault(k, {"name": r["Kernel Name"].split("(")[0]})
        v = float(r["Metric Value"].replace(",", ""))
        unit = r["Metric Unit"]
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-3, "nsecond": 1e-3,
                 "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}.get(unit, 1.0)
        d[r["Metric Name"]] = v * scale
    return [kern[k] for k in sorted(kern)]


def _wavg(kernels, metric):
    t = sum(k.get("gpu__time_duration.sum", 0) for k in kernels if metric in k)
    if not t:
        return None
    return sum(k[metric] * k.get("gpu__time_duration.sum", 0) for k in kernels if metric in k) / t


def summarize(a):
    ks = load_ncu(a.csv)
    prof = json.load(open(a.ops))
    ops = prof["ops"]
    need = sum(o["launches"] for o in ops)
    if len(ks) < need:
        raise SystemExit(f"ncu log has {len(ks)} kernels, the step needs {need}")
    step = ks[-need:]
    out, i = [], 0
    for o in ops:
        mine = step[i:i + o["launches"]]
        i += o["launches"]
        out.append({"op": o["name"], "launches": o["launches"],
                    "kernels": [k["name"] for k in mine],
                    "dram_bytes": sum(k.get("dram__bytes_read.sum", 0) +
                                      k.get("dram__bytes_write.sum", 0) for k in mine),
                    "ncu_us": sum(k.get("gpu__time_duration.sum", 0) for k in mine),
                    # tcgen05 pipe activity of the op's GEMM (time-weighted over its kernels)
                    "tensor_pipe_pct": _wavg(mine, "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed"),
                    "tc_pipe_pct": _wavg(mine, "sm__pipe_tc_cycles_active.avg.pct_of_peak_sustained_elapsed"),
                    "algorithmic_flops": o["flops"], "algorithmic_bytes": o["bytes"]})
    total = sum(x["ncu_us"] for x in out)
    for x in out:
        x["ncu_share"] = x["ncu_us"] / total if total else 0.0
    with open(a.out, "w") as f:
        json.dump({"workload": prof["workload"], "precision": prof["precision"],
                   "source": os.path.basename(a.csv), "ops": out}, f, indent=1)
    for x in sorted(out, key=lambda x: -x["ncu_us"])[:12]:
        print(f"{x['op']:28s} {x['ncu_us']:9.1f} us  {x['ncu_share']:5.1%}  "
              f"dram {x['dram_bytes'] / 1e6:9.1f} MB  algo {x['algorithmic_bytes'] / 1e6:9.1f} MB")


def main():
    p = argparse.ArgumentParser()
    sub = p.add_subparsers(dest="cmd", required=True)
    r = sub.add_parser("run")
    r.add_argument("--workload", default="cifar10_quick")
    r.add_argument("--precision", default="tf32")
    r.add_argument("--ops", required=True)
    s = sub.add_parser("summarize")
    s.add_argument("csv")
    s.add_argument("ops")
    s.add_argument("out")
    a = p.parse_args()
    run(a) if a.cmd == "run" else summarize(a)


if __name__ == "__main__":
    main()
