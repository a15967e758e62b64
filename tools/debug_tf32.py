"""Per-layer TF32-vs-oracle deviation report (debug aid; run under gpurun)."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

from oracle.pyoracle import OracleLib, max_relative_deviation  # noqa: E402
from paper_1511_06051_b200 import model  # noqa: E402
from paper_1511_06051_b200 import netspec as ns  # noqa: E402
from test_gpu_tf32 import tc_nets  # noqa: E402


def f32(x):
    return np.asarray(x, np.float64).astype(np.float32).astype(np.float64)


def main(names):
    orc_lib = OracleLib()
    for name in names:
        spec = tc_nets()[name]
        net = model.Net(spec, 31, precision="tf32", fuse=False)
        orc = orc_lib.net(spec, 31)
        orc.set_weights(net.get_weights_flat())
        rng = np.random.default_rng(11)
        d = spec.data_spec().shape
        x = f32(rng.uniform(-1, 1, size=tuple(d)))
        y = rng.integers(0, net.num_classes(), size=d[0]).astype(np.int32)
        loss, g = net.backward_flat(model.Batch(x, y))
        n = d[0]
        print(f"== {name}: loss {loss:.6f}")
        for li, l in enumerate(spec.layers):
            if l.kind in (ns.DATA, ns.LABEL, ns.SOFTMAX_LOSS):
                continue
            inputs = [net.layer_output(spec.index_of(i)) for i in l.inputs]
            want = orc.layer_forward(li, n, inputs)
            fwd = max_relative_deviation(net.layer_output(li), want)
            dy = net.layer_grad(li)
            src = spec.layers[spec.index_of(l.inputs[0])]
            dx_want, dp_want = orc.layer_backward(li, n, dy, want_dx=src.kind != ns.DATA)
            dg = (max_relative_deviation(net.layer_grad(spec.index_of(l.inputs[0])), dx_want)
                  if src.kind != ns.DATA else float("nan"))
            off, cnt = orc.layer_params(li)
            wk = wb = float("nan")
            if cnt:
                kc = cnt - (l.num_filters if l.kind == ns.CONV else l.num_outputs)
                wk = max_relative_deviation(g[off:off + kc], dp_want[:kc])
                wb = max_relative_deviation(g[off + kc:off + cnt], dp_want[kc:])
                if wk > 1e-2:
                    got = g[off:off + kc]
                    print("   kernel grad got[:8]", got[:8], "want[:8]", dp_want[:8],
                          "nonzero", np.count_nonzero(got), "/", kc)
            print(f"  {l.name:6s} fwd {fwd:.2e} dgrad {dg:.2e} wgrad {wk:.2e} bias {wb:.2e}")


if __name__ == "__main__":
    main(sys.argv[1:] or list(tc_nets()))
