"""Two nets on one GPU driven concurrently from two host threads (each net has its own
stream): net B's gradients must equal B's gradients computed alone, bitwise.  Probes whether
concurrently running grids of the same tcgen05 kernel instantiation interfere (DESIGN §3,
open issue).  Shapes: A = a linear layer (fc-like wgrad), B = a grouped conv (caffe_mix's c2).

    python tools/concurrency_check.py [iterations]
"""
import os
import sys
import threading

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_1511_06051_b200 import model  # noqa: E402
from paper_1511_06051_b200 import netspec as ns  # noqa: E402


def net_a():
    kind = os.environ.get("CC_A", "linear")
    if kind == "conv":  # a plain conv (fprop EPI 0 / wgrad EPI 2 multi-tap)
        return ns.NetSpec([ns.data_layer("data", 3, 32, 8, 8), ns.label_layer("label", 3),
                           ns.conv_layer("c", "data", 3, 3, 32, pad=1),
                           ns.linear_layer("fc", "c", 12),
                           ns.softmax_loss_layer("loss", "fc", "label")])
    if kind == "simt":  # a linear layer too small for the tensor-core path
        return ns.NetSpec([ns.data_layer("data", 3, 6, 1, 1), ns.label_layer("label", 3),
                           ns.linear_layer("fc", "data", 12),
                           ns.softmax_loss_layer("loss", "fc", "label")])
    return ns.NetSpec([ns.data_layer("data", 3, 8, 2, 2), ns.label_layer("label", 3),
                       ns.linear_layer("fc", "data", 12), ns.softmax_loss_layer("loss", "fc", "label")])


def net_b():
    return ns.NetSpec([ns.data_layer("data", 3, 8, 5, 5), ns.label_layer("label", 3),
                       ns.conv_layer("c2", "data", 3, 3, 8, pad=1, group=2),
                       ns.linear_layer("out", "c2", 5), ns.softmax_loss_layer("loss", "out", "label")])


def batch(spec, seed, classes):
    rng = np.random.default_rng(seed)
    d = spec.data_spec().shape
    return model.Batch(rng.uniform(-1, 1, size=tuple(d)).astype(np.float32).astype(np.float64),
                       rng.integers(0, classes, size=d[0]).astype(np.int32))


def main():
    iters = int(sys.argv[1]) if len(sys.argv) > 1 else 200
    a = model.Net(net_a(), 1, precision="tf32")
    b = model.Net(net_b(), 2, precision="tf32")
    ba, bb = batch(net_a(), 1, 12), batch(net_b(), 2, 5)
    ref = b.backward_flat(bb)[1]
    stop = [False]

    def hammer():
        while not stop[0]:
            a.backward_flat(ba)

    t = threading.Thread(target=hammer)
    t.start()
    bad = 0
    names = [f"{n}:{i}" for n, ts in b._structure for i, _ in enumerate(ts)]
    which = {}
    for _ in range(iters):
        g = b.backward_flat(bb)[1]
        if not np.array_equal(g, ref):
            bad += 1
            for nm, (o, c) in zip(names, b.segments()):
                if not np.array_equal(g[o:o + c], ref[o:o + c]):
                    which[nm] = which.get(nm, 0) + 1
    stop[0] = True
    t.join()
    print(f"concurrent backward of B: {bad} / {iters} differ from B alone {which}")


if __name__ == "__main__":
    main()
