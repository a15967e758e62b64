"""Out-of-bounds writes (compute-sanitizer is closed on the GPU pool): the production
kernel variants run in a subprocess with PSG_GUARD=1, where every net buffer (activations,
gradients, routes, parameters, split-K workspaces, im2col / space-to-depth scratch) sits
between two 4 KB guard bands of 0xA5; afterwards no guard byte may have changed.  Covers
AlexNet (TF32 CTA pairs and single-CTA, fused and unfused), GoogLeNet, cifar10_quick (strict
and TF32), the parity micro nets (strict / TF32, fused / unfused) and the grouped C/G = 48
transposed-weight dgrad."""
import os
import subprocess
import sys
import textwrap

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

SCRIPT = textwrap.dedent("""
    import ctypes, sys
    import numpy as np
    sys.path.insert(0, %r)
    from paper_1511_06051_b200 import _lib, data, model, netspec as ns
    def run(spec, precision, pair, fuse, classes=10):
        d = spec.data_spec().shape
        rng = np.random.default_rng(0)
        n = 2 * d[0]
        img = rng.uniform(-1, 1, size=(n,) + tuple(d[1:])).astype(np.float32).astype(np.float64)
        ds = data.Dataset(img, (np.arange(n) %% classes).astype(np.int32), classes)
        net = model.Net(spec, 1, precision=precision, fuse=fuse, tc_pair=pair)
        net.set_sgd(model.SgdOptions(0.01, 0.9, 0.0005))
        net.set_training_data(data.make_worker_iterator(data.shard(ds, 1, 1), 0, d[0], 1))
        net.train(2)
        net.backward_flat(model.Batch(img[:d[0]], ds.labels[:d[0]]))
        del net
    grouped = ns.NetSpec([
        ns.data_layer("data", 2, 96, 9, 9), ns.label_layer("label", 2),
        ns.conv_layer("c0", "data", 1, 1, 96), ns.relu_layer("r0", "c0"),
        ns.conv_layer("c1", "r0", 5, 5, 256, pad=2, group=2), ns.relu_layer("r1", "c1"),
        ns.pool_layer("p", "r1", 3, 3, 2, 2, ceil_mode=True),
        ns.linear_layer("fc", "p", 16), ns.softmax_loss_layer("loss", "fc", "label")])
    for pair in ("always", "never"):
        for fuse in (True, False):
            run(ns.make_alexnet(2), "tf32", pair, fuse, 1000)
            run(ns.make_cifar10_quick(8), "tf32", pair, fuse)
            run(grouped, "tf32", pair, fuse, 16)
    sys.path.insert(0, %r + "/tests")
    import test_gpu_parity as T
    for name, spec in T.micro_nets().items():
        for precision in ("fp32", "tf32"):
            for fuse in (True, False):
                run(spec, precision, "auto", fuse, 5 if name == "caffe_mix" else 10)
    run(ns.make_googlenet(2), "tf32", "always", True, 1000)
    run(ns.make_cifar10_quick(8), "fp32", "auto", True)
    run(ns.make_alexnet(2), "fp32", "auto", False, 1000)
    bad = ctypes.c_ulonglong()
    first = ctypes.create_string_buffer(256)
    _lib.call("psg_debug_guard_violations", ctypes.byref(bad), first, 256)
    print("GUARD", bad.value, first.value.decode())
""") % (ROOT, ROOT)


def test_no_kernel_writes_outside_its_buffers():
    env = dict(os.environ, PSG_GUARD="1")
    r = subprocess.run([sys.executable, "-c", SCRIPT], env=env, capture_output=True, text=True,
                       timeout=900)
    assert r.returncode == 0, r.stderr[-3000:]
    line = [ln for ln in r.stdout.splitlines() if ln.startswith("GUARD")][-1]
    assert line.split()[1] == "0", line
