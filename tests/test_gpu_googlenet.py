"""GoogLeNet (BASELINE.json configs[3]: bvlc_googlenet with both auxiliary heads) on the
device vs the oracle: concat layers, a DAG with multi-consumer activations and three
weighted softmax losses.  Per-layer isolation as in test_gpu_parity (each layer fed the
GPU's own inputs and upstream gradient), strict fp32 1e-5 and TF32 1e-2."""
import numpy as np
import pytest

from oracle.pyoracle import max_relative_deviation
from paper_1511_06051_b200 import netspec as ns

pytestmark = pytest.mark.gpu

BARS = {"fp32": 1e-5, "tf32": 1e-2}


def f32(x):
    return np.asarray(x, np.float64).astype(np.float32).astype(np.float64)


@pytest.fixture(scope="module")
def spec():
    return ns.make_googlenet(2, num_classes=1000)


def test_googlenet_structure(spec, oracle_lib):
    from paper_1511_06051_b200.model import Net
    assert ns.param_count(spec) == 13_378_280
    assert sum(ns.forward_macs(spec).values()) == 1_591_044_096
    net = Net(spec, 5)
    orc = oracle_lib.net(spec, 5)
    assert net.P == orc.P == 13_378_280
    np.testing.assert_array_equal(net.get_weights_flat(), f32(orc.get_weights()))


@pytest.mark.parametrize("precision", ["fp32", "tf32"])
def test_googlenet_per_layer_parity(spec, oracle_lib, precision):
    from paper_1511_06051_b200.model import Batch, Net
    bar = BARS[precision]
    net = Net(spec, 11, precision=precision, fuse=False)
    orc = oracle_lib.net(spec, 11)
    orc.set_weights(net.get_weights_flat())
    rng = np.random.default_rng(3)
    x = f32(rng.uniform(-1, 1, size=(2, 3, 224, 224)))
    y = np.array([7, 911], np.int32)
    loss, g = net.backward_flat(Batch(x, y))
    consumers = {}
    for l in spec.layers:
        for i in l.inputs:
            consumers[i] = consumers.get(i, 0) + 1
    checked = 0
    for li, l in enumerate(spec.layers):
        if l.kind in (ns.DATA, ns.LABEL, ns.SOFTMAX_LOSS):
            continue
        inputs = [net.layer_output(spec.index_of(i)) for i in l.inputs]
        orc.set_dropout_step(0)
        want = orc.layer_forward(li, 2, inputs)
        assert max_relative_deviation(net.layer_output(li), want) <= bar, f"forward {l.name}"
        if l.kind not in (ns.CONV, ns.LINEAR):
            continue
        dy = net.layer_grad(li)
        src = spec.layers[spec.index_of(l.inputs[0])]
        single = consumers[src.name] == 1 and src.kind != ns.DATA
        dx_want, dp_want = orc.layer_backward(li, 2, dy, want_dx=single)
        if single:  # the producer's gradient is exactly this layer's dx
            got_dx = net.layer_grad(spec.index_of(l.inputs[0]))
            assert max_relative_deviation(got_dx, dx_want) <= bar, f"dgrad {l.name}"
        off, cnt = orc.layer_params(li)
        kc = cnt - (l.num_filters if l.kind == ns.CONV else l.num_outputs)
        assert max_relative_deviation(g[off:off + cnt], dp_want, [(0, kc), (kc, cnt - kc)]) \
            <= bar, f"wgrad {l.name}"
        checked += 1
    assert checked == 64  # 59 convs + 5 linear layers (2 per aux head + the classifier)


def test_googlenet_weighted_losses_strict(spec, oracle_lib):
    """Total loss = loss3 + 0.3 (loss1 + loss2); the probabilities are loss3's."""
    from paper_1511_06051_b200.model import Batch, Net
    net = Net(spec, 13)
    orc = oracle_lib.net(spec, 13)
    orc.set_weights(net.get_weights_flat())
    rng = np.random.default_rng(8)
    x = f32(rng.uniform(-1, 1, size=(2, 3, 224, 224)))
    y = np.array([1, 999], np.int32)
    r = net.forward(Batch(x, y))
    lo, po = orc.forward(x, y)
    assert abs(r.loss - lo) <= 1e-5 * abs(lo)
    assert max_relative_deviation(r.probabilities, po) <= 1e-5
    assert r.probabilities.shape == (2, 1000)


def test_googlenet_trains_tf32():
    """tau local steps on an HBM-resident shard stay finite (the bench path)."""
    from paper_1511_06051_b200 import data
    from paper_1511_06051_b200.model import Net, SgdOptions
    spec = ns.make_googlenet(8)
    ds = data.DeviceSyntheticDataset(10, 3, 224, 224, 4, 2.0, 12345, 0, label_classes=1000)
    net = Net(spec, 1, precision="tf32")
    net.set_sgd(SgdOptions(0.01, 0.9, 0.0002))
    net.set_training_data(data.make_worker_iterator(data.shard(ds, 1, 1), 0, 8, 1))
    net.train(4)
    assert np.isfinite(net.last_loss())


def test_googlenet_branch_lanes_bitwise(monkeypatch):
    """GoogLeNet (TF32, b = 2) with its inception branches and auxiliary heads on their own
    streams trains bitwise like one stream (PSG_LANES=0), twice in a row."""
    from paper_1511_06051_b200 import data, model
    from paper_1511_06051_b200 import netspec as ns
    spec = ns.make_googlenet(2)
    d = spec.data_spec().shape
    rng = np.random.default_rng(3)
    img = rng.uniform(-1, 1, size=(8,) + tuple(d[1:])).astype(np.float32).astype(np.float64)
    ds = data.Dataset(img, (np.arange(8) % 1000).astype(np.int32), 1000)
    out = []
    for lanes in ("1", "0", "1"):
        monkeypatch.setenv("PSG_LANES", lanes)
        net = model.Net(spec, 5, precision="tf32")
        net.set_sgd(model.SgdOptions(0.01, 0.9, 0.0002))
        net.set_training_data(data.make_worker_iterator(data.shard(ds, 1, 1), 0, d[0], 1))
        net.train(3)
        out.append(net.get_weights_flat())
    np.testing.assert_array_equal(out[0], out[1])
    np.testing.assert_array_equal(out[0], out[2])

