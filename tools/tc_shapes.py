"""TF32 (tcgen05) vs strict fp32 on single-layer nets with the AlexNet / cifar10_quick layer
geometries (small batch).  Prints the per-pass relative deviation; run under gpurun."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from oracle.pyoracle import max_relative_deviation  # noqa: E402
from paper_1511_06051_b200 import model  # noqa: E402
from paper_1511_06051_b200 import netspec as ns  # noqa: E402

# name: (batch, C, H, W, F, k, pad, group[, stride]) ; C < 0 marks a linear layer (D = -C, O = F)
SHAPES = {
    "ax_conv1": (2, 3, 227, 227, 96, 11, 0, 1, 4),
    "cq_conv1": (8, 3, 32, 32, 32, 5, 2, 1),
    "ax_conv2": (4, 96, 27, 27, 256, 5, 2, 2),
    "ax_conv3": (4, 256, 13, 13, 384, 3, 1, 1),
    "ax_conv4": (4, 384, 13, 13, 384, 3, 1, 2),
    "ax_conv5": (4, 384, 13, 13, 256, 3, 1, 2),
    "cq_conv2": (8, 32, 16, 16, 32, 5, 2, 1),
    "cq_conv3": (8, 32, 8, 8, 64, 5, 2, 1),
    "gn_4b_5x5": (4, 24, 14, 14, 64, 5, 2, 1),        # C/G = 24: padded channel blocks
    "gn_4b_5x5_red": (4, 512, 14, 14, 24, 1, 0, 1),   # F = 24: padded filter blocks (dgrad)
    "grp_c24": (4, 48, 13, 13, 96, 3, 1, 2),          # grouped, C/G = 24
    "grp_f24": (4, 64, 9, 9, 48, 3, 1, 2),            # grouped, F/G = 24 (4-D W^T view)
    "ax_fc6": (64, -9216, 1, 1, 4096, 1, 0, 1),
    "ax_fc8": (64, -4096, 1, 1, 1000, 1, 0, 1),
}


def spec_for(name):
    b, c, h, w, f, k, p, g = SHAPES[name][:8]
    stride = SHAPES[name][8] if len(SHAPES[name]) > 8 else 1
    if c < 0:
        body = [ns.data_layer("data", b, 1, 1, -c), ns.label_layer("label", b),
                ns.linear_layer("l", "data", f)]
    else:
        body = [ns.data_layer("data", b, c, h, w), ns.label_layer("label", b),
                ns.conv_layer("pre", "data", 1, 1, c), ns.conv_layer("l", "pre", k, k, f, pad=p,
                                                                    group=g, stride=stride)]
    body += [ns.linear_layer("cls", "l", 16), ns.softmax_loss_layer("loss", "cls", "label")]
    return ns.NetSpec(body)


def main(names):
    worst = 0.0
    for name in names:
        spec = spec_for(name)
        d = spec.data_spec().shape
        rng = np.random.default_rng(1)
        x = rng.uniform(-1, 1, size=tuple(d)).astype(np.float32).astype(np.float64)
        y = rng.integers(0, 16, size=d[0]).astype(np.int32)
        out = {}
        for prec in ("fp32", "tf32"):
            net = model.Net(spec, 3, precision=prec)
            _, g = net.backward_flat(model.Batch(x, y))
            li = spec.index_of("l")
            out[prec] = (net.layer_output(li), net.layer_grad(li), g,
                         net.layer_grad(li - 1) if spec.layers[li - 1].kind == ns.CONV else None)
            segs = net.segments()
        fwd = max_relative_deviation(out["tf32"][0], out["fp32"][0])
        grads = max_relative_deviation(out["tf32"][2], out["fp32"][2], segs)
        dgrad = (max_relative_deviation(out["tf32"][3], out["fp32"][3])
                 if out["fp32"][3] is not None else 0.0)
        worst = max(worst, fwd, grads, dgrad)
        print(f"{name:10s} fwd {fwd:.2e} dgrad {dgrad:.2e} param-grads {grads:.2e}", flush=True)
    print("WORST", worst)
    return 0 if worst < 1e-2 else 1


if __name__ == "__main__":
    sys.exit(main(sys.argv[1:] or list(SHAPES)))
