"""Where does a tcgen05 GEMM's time go?  Runs training steps of a bench workload with
PSG_TC_PROF=1 (per-launch clock64 counters in the kernel, TcArgs::prof) and prints, per GEMM
launch of one step, the leader CTAs' share of the MMA-loop time spent waiting for a loaded
stage (operand supply) or for a free accumulator (epilogue), the producer's share waiting for
an empty slot, and the cycles per MMA instruction.

    PSG_TC_PROF=1 python tools/tc_prof.py [--workload alexnet] [--steps 5]
"""
import argparse
import ctypes
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="alexnet")
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--json", default="")
    a = ap.parse_args()
    os.environ["PSG_TC_PROF"] = "1"
    sys.argv = [sys.argv[0]]
    import bench
    from paper_1511_06051_b200 import _lib
    from paper_1511_06051_b200 import data as pdata
    from paper_1511_06051_b200 import model
    lib = _lib.lib()
    spec, b = bench.make_spec(a.workload)
    _, _, _, _, lr, mu, wd = bench.WORKLOADS[a.workload]
    ds = bench.build_dataset(a.workload, 1)
    shards = pdata.shard(ds, 1, 1)
    net = model.Net(spec, 1, device=0, precision="tf32")
    net.set_sgd(model.SgdOptions(lr, mu, wd))
    net.set_training_data(pdata.make_worker_iterator(shards, 0, b, 1))
    net.train(3)  # builds and captures the step graph: one label per launch
    net.sync()
    buf = ctypes.create_string_buffer(1 << 20)
    lib.psg_debug_tc_prof(buf, len(buf), 1)
    net.train(a.steps)
    net.sync()
    lib.psg_debug_tc_prof(buf, len(buf), 0)
    rows = []
    for line in buf.value.decode().strip().splitlines():
        idx, label, nums = line.split("|")
        c = [int(x) for x in nums.split()]
        loop, wf, wt, nst, pw, pl, ew, el = c
        if loop == 0:
            continue
        rows.append({
            "launch": int(idx), "plan": label,
            "mma_wait_full": wf / loop, "mma_wait_acc": wt / loop,
            "prod_wait_empty": pw / pl if pl else 0.0, "epi_wait_acc": ew / el if el else 0.0,
            "loop_cycles": loop, "stages": nst,
            "cycles_per_stage": loop / max(nst, 1),
        })
        f = dict((t.rstrip("0123456789"), t[len(t.rstrip("0123456789")):]) for t in label.split()
                 if t[-1].isdigit() and "x" not in t)
        rows[-1]["cycles_per_mma"] = rows[-1]["cycles_per_stage"] / (int(f["kps"]) * int(f["kblk"]) // 8)
    print(f"{'#':>3} {'plan':70} {'wait_full':>9} {'wait_acc':>8} {'prod_wait':>9} "
          f"{'epi_wait':>8} {'cyc/stage':>9} {'cyc/mma':>7}")
    for r in rows:
        print(f"{r['launch']:3d} {r['plan'][:70]:70} {r['mma_wait_full']:9.3f} "
              f"{r['mma_wait_acc']:8.3f} {r['prod_wait_empty']:9.3f} {r['epi_wait_acc']:8.3f} "
              f"{r['cycles_per_stage']:9.0f} {r['cycles_per_mma']:7.1f}")
    if a.json:
        with open(a.json, "w") as f:
            json.dump({"workload": a.workload, "steps": a.steps, "launches": rows}, f, indent=1)


if __name__ == "__main__":
    main()
