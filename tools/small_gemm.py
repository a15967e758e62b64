"""One small TF32 linear layer (the GoogLeNet classifier shape) run forward+backward a few
times: used to profile the GEMM kernel's fixed per-launch cost (ncu -k tc_gemm)."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_1511_06051_b200 import model  # noqa: E402
from paper_1511_06051_b200 import netspec as ns  # noqa: E402


def main():
    b, d, o = (int(x) for x in (sys.argv[1:4] if len(sys.argv) > 3 else (32, 1024, 1000)))
    spec = ns.NetSpec([ns.data_layer("data", b, d, 1, 1), ns.label_layer("label", b),
                       ns.linear_layer("fc", "data", o), ns.softmax_loss_layer("loss", "fc", "label")])
    net = model.Net(spec, 1, precision="tf32")
    rng = np.random.default_rng(0)
    x = rng.uniform(-1, 1, size=(b, d, 1, 1)).astype(np.float32).astype(np.float64)
    y = rng.integers(0, o, size=b).astype(np.int32)
    for _ in range(3):
        net.backward_flat(model.Batch(x, y))
    print("ok")


if __name__ == "__main__":
    main()
