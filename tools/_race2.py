import os, sys
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "tests"))
from paper_1511_06051_b200 import data, model as gpu
import test_gpu_parity as T
from oracle import pyoracle
orc = pyoracle.OracleLib()
def run(fuse, lane, steps):
    if lane: os.environ["PSG_WGRAD_LANE"] = "2"; os.environ["PSG_WGRAD_LANE_LAYER"] = "fc"
    else: os.environ.pop("PSG_WGRAD_LANE", None)
    spec = T.micro_nets()["caffe_mix"]
    d = spec.data_spec().shape
    img, lab = orc.generate_synthetic(10, d[1], d[2], d[3], 6, 2.0, 12345, 0)
    ds = data.Dataset(T.f32(img), lab % 5, 5)
    net = gpu.Net(spec, 3, precision="tf32", fuse=fuse)
    net.set_sgd(gpu.SgdOptions(0.01, 0.9, 0.001))
    net.set_training_data(data.make_worker_iterator(data.shard(ds, 1, 1), 0, d[0], 1))
    out = []
    for s in range(steps):
        net.train(1)
        out.append(net.get_weights_flat())
    return net, out
for trial in range(3):
    for fuse in (True, False):
        net, a = run(fuse, False, 4)
        _, b = run(fuse, True, 4)
        names = [f"{n}:{i}" for n, ts in net._structure for i, _ in enumerate(ts)]
        segs = net.segments()
        first = [(s, [names[i] for i, (o, c) in enumerate(segs) if not np.array_equal(a[s][o:o+c], b[s][o:o+c])]) for s in range(4)]
        print(trial, fuse, [(s, x) for s, x in first if x][:2])
