"""AlexNet (BASELINE.json configs[2], the north-star workload) at its production geometry —
227x227 input, conv1 11x11/4 on the space-to-depth route (s2d_x_k<12>), conv2 5x5 p2 g2
with 48 channels per group (K-major transposed-weight dgrad), conv3-5, fc6 9216 -> 4096 with
split K, LRN -> 3x3 max pool over 96 and 256 channels — on the production tcgen05 kernel
variants, checked against the oracle (model.hpp:334-585 + the Caffe extensions).

The batch is small (b = 2) so the fp64 oracle finishes in seconds; at b = 2 the throughput
heuristic would not pick CTA pairs, so the pair policy is forced (psg_net_set_tc_options):
"always" runs every K-major-A GEMM as a cta_group::2 pair (tc_gemm_kernel<KBLK, true, EPI>,
the kernels AlexNet's b = 256 step launches), "never" the single-CTA kernels.

* per-layer isolation: each layer fed the GPU's own inputs and upstream
  gradient, strict fp32 1e-5 / TF32 1e-2, per-tensor max-normalised (test_helpers.hpp:77-91);
* the fused graph (ReLU in the GEMM epilogue, ReLU backward as the dgrad epilogue mask —
  tc_gemm_kernel<32, true, 1> —, LRN inside the max pool and its backward gathered through
  the pool's route at 96 / 256 channels, the batch gathered straight into the space-to-depth
  input) trains bitwise like the unfused graph the isolation test checks;
* the host-fed (e2e) path stages NCHW batches into the space-to-depth input and trains
  bitwise like the HBM-resident stream.
"""
import numpy as np
import pytest

from oracle.pyoracle import max_relative_deviation
from paper_1511_06051_b200 import netspec as ns

pytestmark = pytest.mark.gpu

BARS = {"fp32": 1e-5, "tf32": 1e-2}
B = 2


def f32(x):
    return np.asarray(x, np.float64).astype(np.float32).astype(np.float64)


@pytest.fixture(scope="module")
def spec():
    return ns.make_alexnet(B)


def test_alexnet_structure(spec, oracle_lib):
    from paper_1511_06051_b200.model import Net
    assert ns.param_count(spec) == 60_965_224
    net = Net(spec, 5)
    orc = oracle_lib.net(spec, 5)
    assert net.P == orc.P == 60_965_224
    np.testing.assert_array_equal(net.get_weights_flat(), f32(orc.get_weights()))


@pytest.mark.parametrize("precision,pair", [("tf32", "always"), ("tf32", "never"),
                                            ("fp32", "auto")])
def test_alexnet_per_layer_parity(spec, oracle_lib, precision, pair):
    from paper_1511_06051_b200.model import Batch, Net
    bar = BARS[precision]
    net = Net(spec, 11, precision=precision, fuse=False, tc_pair=pair)
    orc = oracle_lib.net(spec, 11)
    orc.set_weights(net.get_weights_flat())
    rng = np.random.default_rng(3)
    x = f32(rng.uniform(-1, 1, size=(B, 3, 227, 227)))
    y = np.array([7, 911], np.int32)
    loss, g = net.backward_flat(Batch(x, y))
    checked = []
    for li, l in enumerate(spec.layers):
        if l.kind in (ns.DATA, ns.LABEL, ns.SOFTMAX_LOSS):
            continue
        inputs = [net.layer_output(spec.index_of(i)) for i in l.inputs]
        orc.set_dropout_step(0)
        want = orc.layer_forward(li, B, inputs)
        assert max_relative_deviation(net.layer_output(li), want) <= bar, f"forward {l.name}"
        dy = net.layer_grad(li)
        src = spec.layers[spec.index_of(l.inputs[0])]
        dx_want, dp_want = orc.layer_backward(li, B, dy, want_dx=src.kind != ns.DATA)
        if src.kind != ns.DATA:  # a chain: the producer's gradient is exactly this dx
            got = net.layer_grad(spec.index_of(l.inputs[0]))
            assert max_relative_deviation(got, dx_want) <= bar, f"dgrad {l.name}"
        off, cnt = orc.layer_params(li)
        if cnt:
            kc = cnt - (l.num_filters if l.kind == ns.CONV else l.num_outputs)
            assert max_relative_deviation(g[off:off + cnt], dp_want,
                                          [(0, kc), (kc, cnt - kc)]) <= bar, f"wgrad {l.name}"
        checked.append(l.name)
    assert len(checked) == 22  # 5 conv, 3 fc, 7 relu, 2 lrn, 3 pool, 2 dropout


def _dataset(oracle_lib, rows_per_class=1):
    from paper_1511_06051_b200 import data
    img, lab = oracle_lib.generate_synthetic(10, 3, 227, 227, rows_per_class, 2.0, 12345, 0)
    return data.Dataset(f32(img), lab * 97, 1000)  # spread the labels over 1000 classes


def test_alexnet_fused_pairs_train_bitwise_like_unfused(spec, oracle_lib):
    from paper_1511_06051_b200 import data
    from paper_1511_06051_b200.model import Net, SgdOptions
    ds = _dataset(oracle_lib)
    out = []
    for fuse in (True, False):
        net = Net(spec, 3, precision="tf32", fuse=fuse, tc_pair="always")
        net.set_sgd(SgdOptions(0.01, 0.9, 0.0005))
        net.set_training_data(data.make_worker_iterator(data.shard(ds, 1, 1), 0, B, 1))
        net.train(2)
        out.append((net.get_weights_flat(), net.last_loss(), net.kernels_per_step()))
    np.testing.assert_array_equal(out[0][0], out[1][0])
    assert out[0][1] == out[1][1]
    assert out[0][2] < out[1][2]  # the fused graph launches fewer kernels


def test_alexnet_host_fed_matches_device_stream(spec, oracle_lib):
    """psg_net_train_host stages the NCHW host batch straight into conv1's space-to-depth
    input (s2d_x_k<12> over an NCHW source); bitwise equal to the device-gathered stream."""
    from paper_1511_06051_b200 import data
    from paper_1511_06051_b200._lib import PinnedArray
    from paper_1511_06051_b200.model import Net, SgdOptions
    ds = _dataset(oracle_lib)
    shards = data.shard(ds, 1, 4)
    a = Net(spec, 2, precision="tf32", tc_pair="always")
    b = Net(spec, 2, precision="tf32", tc_pair="always")
    for n in (a, b):
        n.set_sgd(SgdOptions(0.01, 0.9, 0.0005))
    a.set_training_data(data.make_worker_iterator(shards, 0, B, 4))
    a.train(3)
    it = data.make_worker_iterator(shards, 0, B, 4)
    img = PinnedArray((3, B, 3, 227, 227), np.float32)
    lab = PinnedArray((3, B), np.int32)
    for s in range(3):
        idx = it.next_indices().astype(np.int64)
        img.array[s] = ds.images[idx]
        lab.array[s] = ds.labels[idx]
    losses = b.train_host(img.array, lab.array)
    np.testing.assert_array_equal(a.get_weights_flat(), b.get_weights_flat())
    assert losses[-1] == a.last_loss()
