"""GPU parity: libpsg (through the C ABI) vs the pinned C oracle on the same inputs.

Bars (BASELINE.json north_star): per-layer outputs / gradients <= 1e-5 relative in fp32
mode (1e-2 in TF32 mode), measured with the reference's per-tensor max-normalised metric
(test_helpers.hpp:77-91) one step at a time from identical (fp32-representable) state;
averaged weights bit-exact in ordered mode; shard indexing bit-exact.
"""
import numpy as np
import pytest

from oracle.pyoracle import max_relative_deviation
from paper_1511_06051_b200 import netspec as ns

pytestmark = pytest.mark.gpu

STRICT = 1e-5
TF32 = 1e-2


def f32(x):
    return np.asarray(x, np.float64).astype(np.float32).astype(np.float64)


def micro_nets():
    return {
        "lenet_small": ns.make_lenet_small(6, 1, 16, 16, 10),
        "mlp": ns.make_mlp(5, 1, 1, 16, 10),
        "cq_valid": ns.make_cq_valid(4),
        "cifar10_quick": ns.make_cifar10_quick(4),
        "caffe_mix": ns.NetSpec([
            ns.data_layer("data", 3, 3, 19, 19), ns.label_layer("label", 3),
            ns.conv_layer("c1", "data", 5, 5, 8, stride=2, pad=1), ns.relu_layer("r1", "c1"),
            ns.lrn_layer("n1", "r1", 5, 1e-2, 0.75, 1.0),
            ns.pool_layer("p1", "n1", 3, 3, 2, 2, ceil_mode=True),
            ns.conv_layer("c2", "p1", 3, 3, 8, pad=1, group=2), ns.relu_layer("r2", "c2"),
            ns.pool_layer("p2", "r2", 3, 3, 2, 2, method=ns.POOL_AVE, ceil_mode=True),
            ns.linear_layer("fc", "p2", 12), ns.relu_layer("r3", "fc"),
            ns.dropout_layer("d3", "r3", 0.5), ns.linear_layer("out", "d3", 5),
            ns.softmax_loss_layer("loss", "out", "label")]),
    }


@pytest.fixture(scope="module")
def gpu():
    from paper_1511_06051_b200 import model
    return model


def _pair(gpu, oracle_lib, spec, seed):
    net = gpu.Net(spec, seed, fuse=False)  # per-layer state is inspected
    orc = oracle_lib.net(spec, seed)
    return net, orc


def _batch(spec, classes, seed):
    rng = np.random.default_rng(seed)
    d = spec.data_spec().shape
    x = f32(rng.uniform(-1, 1, size=tuple(d)))
    y = rng.integers(0, classes, size=d[0]).astype(np.int32)
    return x, y


@pytest.mark.parametrize("name", list(micro_nets()))
def test_init_is_fp32_rounding_of_reference_init(gpu, oracle_lib, name):
    """model.hpp:200-283 init: same RNG streams, one rounding to fp32."""
    spec = micro_nets()[name]
    net, orc = _pair(gpu, oracle_lib, spec, 17)
    np.testing.assert_array_equal(net.get_weights_flat(), f32(orc.get_weights()))


@pytest.mark.parametrize("name", list(micro_nets()))
def test_forward_backward_parity_strict(gpu, oracle_lib, name):
    spec = micro_nets()[name]
    net, orc = _pair(gpu, oracle_lib, spec, 23)
    w = net.get_weights_flat()
    orc.set_weights(w)
    x, y = _batch(spec, net.num_classes(), 5)
    r = net.forward(gpu.Batch(x, y))
    lo, po = orc.forward(x, y)
    assert abs(r.loss - lo) <= STRICT * max(1.0, abs(lo))
    assert max_relative_deviation(r.probabilities, po) <= STRICT
    loss, g = net.backward_flat(gpu.Batch(x, y))
    lo, go = orc.backward(x, y)
    assert abs(loss - lo) <= STRICT * max(1.0, abs(lo))
    assert max_relative_deviation(g, go, net.segments()) <= STRICT


@pytest.mark.parametrize("name", list(micro_nets()))
def test_per_layer_isolation_strict(gpu, oracle_lib, name):
    """Each layer fed the GPU's own inputs and upstream gradient."""
    spec = micro_nets()[name]
    net, orc = _pair(gpu, oracle_lib, spec, 29)
    orc.set_weights(net.get_weights_flat())
    x, y = _batch(spec, net.num_classes(), 7)
    _, g = net.backward_flat(gpu.Batch(x, y))
    n = x.shape[0]
    for li, l in enumerate(spec.layers):
        if l.kind in (ns.DATA, ns.LABEL, ns.SOFTMAX_LOSS):
            continue
        inputs = [net.layer_output(spec.index_of(i)) for i in l.inputs]
        orc.set_dropout_step(0)
        want = orc.layer_forward(li, n, inputs)
        got = net.layer_output(li)
        assert max_relative_deviation(got, want) <= STRICT, f"forward {l.name}"
        dy = net.layer_grad(li)
        src = spec.layers[spec.index_of(l.inputs[0])]
        dx_want, dp_want = orc.layer_backward(li, n, dy, want_dx=src.kind != ns.DATA)
        if src.kind != ns.DATA:
            # chains: the producer's gradient is exactly this layer's dx
            got_dx = net.layer_grad(spec.index_of(l.inputs[0]))
            assert max_relative_deviation(got_dx, dx_want) <= STRICT, f"dgrad {l.name}"
        off, cnt = orc.layer_params(li)
        if cnt:
            kc = cnt - (l.num_filters if l.kind == ns.CONV else l.num_outputs)
            segs = [(0, kc), (kc, cnt - kc)]
            assert max_relative_deviation(g[off:off + cnt], dp_want, segs) <= STRICT, \
                f"wgrad {l.name}"


def test_multi_consumer_dgrad_not_needed_for_chains(gpu):
    """The reference layer graphs are chains; every producer here has one consumer."""
    for spec in micro_nets().values():
        consumers = {}
        for l in spec.layers:
            for i in l.inputs:
                consumers[i] = consumers.get(i, 0) + 1
        assert all(v == 1 for k, v in consumers.items() if k != "label")


@pytest.mark.parametrize("mu,wd", [(0.0, 0.0), (0.9, 0.0), (0.9, 0.004)])
def test_apply_update_parity(gpu, oracle_lib, mu, wd):
    """model.hpp:90-107 (+ weight decay / lr_mult extension)."""
    spec = ns.make_cifar10_quick(2)
    net, orc = _pair(gpu, oracle_lib, spec, 3)
    orc.set_weights(net.get_weights_flat())
    net.set_sgd(gpu.SgdOptions(0.01, mu, wd))
    orc.set_sgd(0.01, mu, wd)
    rng = np.random.default_rng(0)
    for _ in range(3):
        g = f32(rng.normal(size=net.P))
        net.apply_update_flat(g)
        orc.apply_update(g)
        assert max_relative_deviation(net.get_weights_flat(), orc.get_weights(),
                                      net.segments()) <= STRICT
        assert max_relative_deviation(net.get_velocity_flat(), orc.get_velocity(),
                                      net.segments()) <= STRICT


def _dataset(gpu, oracle_lib, spec, per_class, variant=0):
    from paper_1511_06051_b200.data import Dataset
    d = spec.data_spec().shape
    img, lab = oracle_lib.generate_synthetic(10, d[1], d[2], d[3], per_class, 2.0, 12345, variant)
    return Dataset(f32(img), lab, 10)


def test_device_shard_stream_bit_exact(gpu, oracle_lib):
    """The batch the GPU gathers at step s is rows order[s*b:(s+1)*b] of the reference
    iterator (data.hpp:312-351), across epoch boundaries."""
    from paper_1511_06051_b200 import data
    spec = ns.make_lenet_small(8, 1, 16, 16, 10)
    ds = _dataset(gpu, oracle_lib, spec, 7)
    shards = data.shard(ds, 3, 5)
    net = gpu.Net(spec, 1)
    net.set_sgd(gpu.SgdOptions(1e-6, 0.0))
    it = data.make_worker_iterator(shards, 1, 8, 5)
    net.set_training_data(it)
    want = oracle_lib.worker_indices(70, 3, 1, 8, 5, 12)
    for s in range(12):
        net.train(1)
        got = net.layer_output(spec.index_of("data"))
        rows = want[s * 8:(s + 1) * 8].astype(np.int64)
        np.testing.assert_array_equal(got, ds.images[rows])


def test_train_lockstep_parity(gpu, oracle_lib):
    """Net::train(1) == oracle backward+apply_update on the same batch and state."""
    from paper_1511_06051_b200 import data
    spec = ns.make_cifar10_quick(10)
    ds = _dataset(gpu, oracle_lib, spec, 6)
    shards = data.shard(ds, 2, 1)
    net = gpu.Net(spec, 1)
    orc = oracle_lib.net(spec, 1)
    net.set_sgd(gpu.SgdOptions(0.01, 0.9, 0.004))
    orc.set_sgd(0.01, 0.9, 0.004)
    it = data.make_worker_iterator(shards, 0, 10, 1)
    net.set_training_data(it)
    idx = oracle_lib.worker_indices(60, 2, 0, 10, 1, 5).astype(np.int64)
    for s in range(5):
        w0 = net.get_weights_flat()
        orc.set_weights(w0)
        vel = net.get_velocity_flat()
        net.train(1)
        rows = idx[s * 10:(s + 1) * 10]
        _, g = orc.backward(ds.images[rows], ds.labels[rows])
        # oracle velocity state := GPU's pre-step velocity
        orc.set_sgd(0.01, 0.9, 0.004)
        _set_velocity(orc, vel)
        orc.apply_update(g)
        assert max_relative_deviation(net.get_weights_flat(), orc.get_weights(),
                                      net.segments()) <= STRICT


def _set_velocity(orc, vel):
    """Velocity injection through the update rule: with g=0, wd=0, mu=0 -> no-op; so
    rebuild it by one update from zero velocity (v = 0*mu + v)."""
    w = orc.get_weights()
    orc.L.orc_net_reset_velocity(orc.h)
    lr, mu, wd = 0.01, 0.9, 0.004
    orc.set_sgd(lr, 1e-300, 0.0)
    orc.apply_update(np.asarray(vel, np.float64))  # v = vel, w -= lr*vel
    orc.set_weights(w)
    orc.set_sgd(lr, mu, wd)


def test_average_local_ordered_bit_exact(gpu, oracle_lib):
    """weights_mean (weights.hpp:90-107): ascending fp64 accumulation, /K, one rounding."""
    spec = ns.make_cq_valid(2)
    nets = [gpu.Net(spec, 1) for _ in range(4)]
    rng = np.random.default_rng(3)
    ws = []
    for n in nets:
        w = f32(rng.normal(size=n.P))
        n.set_weights_flat(w)
        ws.append(w)
    from paper_1511_06051_b200 import schemes
    schemes.average_local(nets)
    want = f32(oracle_lib.weights_mean(ws))
    for n in nets:
        np.testing.assert_array_equal(n.get_weights_flat(), want)


def test_non_finite_raises_runtime_error(gpu, oracle_lib):
    """tensor.hpp:78-84: a diverging run fails loudly (sticky device flag)."""
    from paper_1511_06051_b200 import data
    spec = ns.make_mlp(8, 1, 1, 16, 10)
    img = np.full((40, 1, 1, 16), 1e30)
    ds = data.Dataset(img, np.arange(40, dtype=np.int32) % 10, 10)
    net = gpu.Net(spec, 1)
    net.set_sgd(gpu.SgdOptions(1e30, 0.0))
    net.set_training_data(data.make_worker_iterator(data.shard(ds, 1, 1), 0, 8, 1))
    with pytest.raises(RuntimeError):
        net.train(3)


def test_error_conventions(gpu):
    from paper_1511_06051_b200 import data
    spec = ns.make_mlp(4, 1, 1, 16, 10)
    net = gpu.Net(spec, 1)
    with pytest.raises(RuntimeError):
        net.train(1)                      # model.hpp:113
    with pytest.raises(ValueError):
        net.train(-1)                     # model.hpp:112
    with pytest.raises(RuntimeError):
        net.test(1)                       # model.hpp:124
    with pytest.raises(ValueError):
        net.test(0)                       # model.hpp:123
    x = np.zeros((4, 1, 1, 16))
    with pytest.raises(ValueError):
        net.forward(gpu.Batch(x, np.array([0, 1, 2, 10], np.int32)))  # label out of range
    with pytest.raises(ValueError):
        net.forward(gpu.Batch(np.zeros((4, 1, 1, 15)), np.zeros(4, np.int32)))
    with pytest.raises(ValueError):
        net.set_sgd(gpu.SgdOptions(0.0, 0.0))  # model.hpp:61
    with pytest.raises(ValueError):
        net.set_sgd(gpu.SgdOptions(0.1, 1.0))  # model.hpp:62
    w = net.get_weights()
    bad = data  # noqa: F841
    from paper_1511_06051_b200.weights import WeightCollection
    with pytest.raises(ValueError):
        net.set_weights(WeightCollection([(n, ts) for n, ts in list(w)[:-1]]))


def test_zero_weights_uniform_softmax_loss(gpu):
    """model_test.cpp:146-156."""
    spec = ns.make_mlp(4, 1, 1, 16, 10)
    net = gpu.Net(spec, 5)
    net.set_weights_flat(np.zeros(net.P))
    rng = np.random.default_rng(17)
    x = rng.uniform(-1, 1, size=(4, 1, 1, 16))
    r = net.forward(gpu.Batch(x, rng.integers(0, 10, 4).astype(np.int32)))
    assert abs(r.loss - np.log(10.0)) < 1e-6
    np.testing.assert_allclose(r.probabilities.sum(axis=1), 1.0, atol=1e-6)


def test_max_pool_tie_routes_to_lowest_index(gpu):
    """model_test.cpp:217-246."""
    spec = ns.NetSpec([ns.data_layer("data", 1, 1, 1, 4), ns.label_layer("label", 1),
                       ns.conv_layer("c1", "data", 1, 2, 1), ns.pool_layer("p1", "c1", 1, 3, 1, 1),
                       ns.linear_layer("fc", "p1", 2), ns.softmax_loss_layer("loss", "fc", "label")])
    net = gpu.Net(spec, 1)
    net.set_weights_flat(np.array([1.0, 1.0, 0.0, 1.0, -1.0, 0.0, 0.0]))
    batch = gpu.Batch(np.array([1.0, 2.0, 1.0, 2.0]).reshape(1, 1, 1, 4), np.array([0], np.int32))
    out = net.forward(batch)
    grads = net.backward(batch)
    dk = grads.find("c1")[0].ravel()
    p0, p1 = out.probabilities[0]
    dpool = (p0 - 1.0) - p1
    np.testing.assert_allclose(dk, [dpool * 1.0, dpool * 2.0], rtol=STRICT)


def _inception_net(b):
    """One small inception block (GoogLeNet-style branches, ReLUs feeding a concat)."""
    layers = [ns.data_layer("data", b, 3, 12, 12), ns.label_layer("label", b),
              ns.conv_layer("c0", "data", 3, 3, 16, pad=1), ns.relu_layer("r0", "c0")]
    ns._inception(layers, "inc", "r0", 8, 8, 16, 4, 8, 8, {})
    layers += [ns.pool_layer("p", "inc/output", 3, 3, 2, 2),
               ns.linear_layer("out", "p", 10), ns.softmax_loss_layer("loss", "out", "label")]
    return ns.NetSpec(layers)


@pytest.mark.parametrize("precision", ["fp32", "tf32"])
@pytest.mark.parametrize("name", ["cifar10_quick", "caffe_mix", "s2d", "inception"])
def test_relu_fusion_is_bitwise_neutral(gpu, oracle_lib, name, precision):
    """psg_net_set_fusion: the ReLU applied in the GEMM epilogue, ReLU backwards folded into
    the consuming LRN / dgrad epilogue / pool backward / concat split, the LRN computed inside
    the following max pool and the batch gathered straight into the space-to-depth input
    give bitwise-identical training to the unfused graph."""
    from paper_1511_06051_b200 import data
    spec = (_s2d_net(6) if name == "s2d" else _inception_net(6) if name == "inception"
            else micro_nets()[name])
    d = spec.data_spec().shape
    img, lab = oracle_lib.generate_synthetic(10, d[1], d[2], d[3], 6, 2.0, 12345, 0)
    ds = data.Dataset(f32(img), lab % 5 if name == "caffe_mix" else lab,
                      5 if name == "caffe_mix" else 10)
    out = []
    for fuse in (True, False):
        net = gpu.Net(spec, 3, precision=precision, fuse=fuse)
        net.set_sgd(gpu.SgdOptions(0.01, 0.9, 0.001))
        net.set_training_data(data.make_worker_iterator(data.shard(ds, 1, 1), 0, d[0], 1))
        net.train(3)
        out.append((net.get_weights_flat(), net.last_loss()))
    np.testing.assert_array_equal(out[0][0], out[1][0])
    assert out[0][1] == out[1][1]


@pytest.mark.parametrize("precision", ["fp32", "tf32"])
@pytest.mark.parametrize("name", ["inception", "caffe_mix", "cifar10_quick"])
@pytest.mark.parametrize("fuse", [True, False])
def test_lanes_are_bitwise_neutral(gpu, oracle_lib, name, precision, fuse, monkeypatch):
    """Lanes — the inception block's branches on their own streams, every lane-0 layer's wgrad
    on a second stream overlapping the dgrad chain, cross-lane event edges, per-lane GEMM
    workspaces, the later branch gradients into the block input written to scratch and summed
    in order, concurrent grids of the tcgen05 kernel — train bitwise like one stream
    (PSG_LANES=0)."""
    from paper_1511_06051_b200 import data
    spec = (_inception_net(6) if name == "inception" else micro_nets()[name] if name == "caffe_mix"
            else ns.make_cifar10_quick(10))
    d = spec.data_spec().shape
    img, lab = oracle_lib.generate_synthetic(10, d[1], d[2], d[3], 6, 2.0, 12345, 0)
    classes = 5 if name == "caffe_mix" else 10
    ds = data.Dataset(f32(img), lab % classes, classes)
    out = []
    for lanes in ("1", "0"):
        monkeypatch.setenv("PSG_LANES", lanes)
        net = gpu.Net(spec, 3, precision=precision, fuse=fuse)
        net.set_sgd(gpu.SgdOptions(0.01, 0.9, 0.001))
        net.set_training_data(data.make_worker_iterator(data.shard(ds, 1, 1), 0, d[0], 1))
        net.train(3)
        out.append((net.get_weights_flat(), net.last_loss()))
    np.testing.assert_array_equal(out[0][0], out[1][0])
    assert out[0][1] == out[1][1]


def _concat_edge_net(b):
    """A concat over the data layer (no gradient), a ReLU'd branch taken twice (the same
    gradient written by two slices: per-slice launches) and an odd channel count (scalar
    path)."""
    return ns.NetSpec([
        ns.data_layer("data", b, 3, 6, 6), ns.label_layer("label", b),
        ns.conv_layer("a", "data", 1, 1, 4), ns.relu_layer("ra", "a"),
        ns.conv_layer("b", "data", 3, 3, 5, pad=1),
        ns.concat_layer("cat", ["data", "ra", "b", "ra"]),
        ns.pool_layer("p", "cat", 3, 3, 2, 2),
        ns.linear_layer("out", "p", 10), ns.softmax_loss_layer("loss", "out", "label")])


@pytest.mark.parametrize("precision", ["fp32", "tf32"])
@pytest.mark.parametrize("name", ["inception", "concat_edge"])
@pytest.mark.parametrize("lanes", ["1", "0"])
def test_single_launch_concat_is_bitwise_neutral(gpu, oracle_lib, name, precision, lanes,
                                                 monkeypatch):
    """The concat forward and its backward split as ONE launch over all inputs
    (concat_copy_all / concat_split_all) train bitwise like one launch per input
    (PSG_CONCAT_SINGLE=0), with and without branch lanes."""
    from paper_1511_06051_b200 import data
    spec = _inception_net(6) if name == "inception" else _concat_edge_net(6)
    d = spec.data_spec().shape
    img, lab = oracle_lib.generate_synthetic(10, d[1], d[2], d[3], 6, 2.0, 12345, 0)
    ds = data.Dataset(f32(img), lab, 10)
    monkeypatch.setenv("PSG_LANES", lanes)
    out = []
    for single in ("1", "0"):
        monkeypatch.setenv("PSG_CONCAT_SINGLE", single)
        net = gpu.Net(spec, 3, precision=precision)
        net.set_sgd(gpu.SgdOptions(0.01, 0.9, 0.001))
        net.set_training_data(data.make_worker_iterator(data.shard(ds, 1, 1), 0, d[0], 1))
        net.train(3)
        out.append((net.get_weights_flat(), net.last_loss()))
    np.testing.assert_array_equal(out[0][0], out[1][0])
    assert out[0][1] == out[1][1]


def _s2d_net(b):
    """A strided 3-channel first conv (the space-to-depth route in TF32: the device stream
    gathers straight into x', host batches are staged NHWC then rearranged), then
    ReLU -> LRN -> 3x3 max pool over 48 channels (the fused LRN / pool kernels, 6-channel
    lanes in the backward)."""
    return ns.NetSpec([
        ns.data_layer("data", b, 3, 23, 23), ns.label_layer("label", b),
        ns.conv_layer("c1", "data", 7, 7, 48, stride=2, pad=3), ns.relu_layer("r1", "c1"),
        ns.lrn_layer("n1", "r1", 5, 1e-2, 0.75, 1.0),
        ns.pool_layer("p1", "n1", 3, 3, 2, 2, ceil_mode=True),
        ns.linear_layer("out", "p1", 10), ns.softmax_loss_layer("loss", "out", "label")])


@pytest.mark.parametrize("name", ["cifar10_quick", "s2d"])
def test_train_host_matches_device_stream(gpu, oracle_lib, name):
    """psg_net_train_host (host batches, double-buffered H2D overlapping the steps) ==
    psg_net_train on the HBM-resident stream with the same batch order, bitwise."""
    from paper_1511_06051_b200 import data
    from paper_1511_06051_b200._lib import PinnedArray
    spec = ns.make_cifar10_quick(10) if name == "cifar10_quick" else _s2d_net(10)
    ds = _dataset(gpu, oracle_lib, spec, 6)
    shards = data.shard(ds, 1, 4)
    a = gpu.Net(spec, 2, precision="tf32")
    b = gpu.Net(spec, 2, precision="tf32")
    for n in (a, b):
        n.set_sgd(gpu.SgdOptions(0.01, 0.9, 0.004))
    a.set_training_data(data.make_worker_iterator(shards, 0, 10, 4))
    a.train(5)
    it = data.make_worker_iterator(shards, 0, 10, 4)
    img = PinnedArray((5,) + tuple(spec.data_spec().shape), np.float32)
    lab = PinnedArray((5, 10), np.int32)
    for s in range(5):
        idx = it.next_indices().astype(np.int64)
        img.array[s] = ds.images[idx]
        lab.array[s] = ds.labels[idx]
    losses = b.train_host(img.array, lab.array)
    np.testing.assert_array_equal(a.get_weights_flat(), b.get_weights_flat())
    assert losses[-1] == a.last_loss()


@pytest.mark.parametrize("name,threads,dma", [("cifar10_quick", 1, "0"), ("cifar10_quick", 4, "0"),
                                              ("s2d", 3, "0"), ("cifar10_quick", 2, "0.5"),
                                              ("s2d", 1, "1")])
def test_train_host_rows_matches_device_stream(gpu, oracle_lib, name, threads, dma, monkeypatch):
    """psg_net_train_host_rows (host threads gather each step's rows into pinned staging while
    the GPU runs the previous step; the DMA share of the rows copied straight from the
    registered dataset) == psg_net_train on the HBM-resident stream, bitwise."""
    from paper_1511_06051_b200 import data
    monkeypatch.setenv("PSG_HOST_ROW_DMA_FRAC", dma)
    spec = ns.make_cifar10_quick(10) if name == "cifar10_quick" else _s2d_net(10)
    ds = _dataset(gpu, oracle_lib, spec, 6)
    shards = data.shard(ds, 1, 4)
    a = gpu.Net(spec, 2, precision="tf32")
    b = gpu.Net(spec, 2, precision="tf32")
    for n in (a, b):
        n.set_sgd(gpu.SgdOptions(0.01, 0.9, 0.004))
    a.set_training_data(data.make_worker_iterator(shards, 0, 10, 4))
    a.train(7)
    it = data.make_worker_iterator(shards, 0, 10, 4)
    rows = np.concatenate([it.next_indices() for _ in range(7)])
    img = np.ascontiguousarray(ds.images, np.float32)
    losses = b.train_host_rows(img, np.ascontiguousarray(ds.labels, np.int32), rows, threads)
    np.testing.assert_array_equal(a.get_weights_flat(), b.get_weights_flat())
    assert losses.size == 7 and losses[-1] == a.last_loss()
