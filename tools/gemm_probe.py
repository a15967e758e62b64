"""Pipeline wait counters (PSG_TC_PROF) of the tcgen05 GEMM on one linear layer whose operands
stay L2-resident: separates the kernel's own pipeline behaviour from the operand supply of the
AlexNet layers (tools/tc_prof.py).

    PSG_TC_PROF=1 python tools/gemm_probe.py [batch] [D] [O]
"""
import ctypes
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
os.environ["PSG_TC_PROF"] = "1"

from paper_1511_06051_b200 import _lib  # noqa: E402
from paper_1511_06051_b200 import model  # noqa: E402
from paper_1511_06051_b200 import netspec as ns  # noqa: E402


def main():
    b, d, o = (int(x) for x in (sys.argv[1:4] if len(sys.argv) > 3 else (1024, 2048, 2048)))
    spec = ns.NetSpec([ns.data_layer("data", b, d, 1, 1), ns.label_layer("label", b),
                       ns.linear_layer("fc", "data", o),
                       ns.softmax_loss_layer("loss", "fc", "label")])
    net = model.Net(spec, 1, precision="tf32")
    rng = np.random.default_rng(0)
    x = rng.uniform(-1, 1, size=(b, d, 1, 1)).astype(np.float32).astype(np.float64)
    y = rng.integers(0, o, size=b).astype(np.int32)
    lib = _lib.lib()
    buf = ctypes.create_string_buffer(1 << 16)
    net.backward_flat(model.Batch(x, y))
    net.sync()
    lib.psg_debug_tc_prof(buf, len(buf), 1)
    for _ in range(5):
        net.backward_flat(model.Batch(x, y))
    net.sync()
    lib.psg_debug_tc_prof(buf, len(buf), 0)
    print(f"linear b={b} D={d} O={o}: fwd M={b} N={o} K={d}")
    print(f"{'plan':70} {'wait_full':>9} {'wait_acc':>8} {'prod_wait':>9} {'epi_wait':>8} "
          f"{'cyc/mma':>7}")
    for line in buf.value.decode().strip().splitlines():
        _, label, nums = line.split("|")
        loop, wf, wt, nst, pw, pl, ew, el = (int(v) for v in nums.split())
        if not loop:
            continue
        f = dict((t.rstrip("0123456789"), t[len(t.rstrip("0123456789")):]) for t in label.split()
                 if t[-1].isdigit() and "x" not in t)
        mmas = max(nst, 1) * int(f["kps"]) * int(f["kblk"]) // 8
        print(f"{label[:70]:70} {wf / loop:9.3f} {wt / loop:8.3f} {pw / max(pl, 1):9.3f} "
              f"{ew / max(el, 1):8.3f} {loop / mmas:7.1f}")


if __name__ == "__main__":
    main()
