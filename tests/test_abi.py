"""CPU checks of the drop-in boundary: libpsg.so loads without a GPU and exports every
entry point include/psg.h declares; host-side (integer) semantics are bit-exact with the
pinned oracle; the Python mirror's validation matches net_spec.hpp."""
import ctypes
import os
import re

import numpy as np
import pytest

from paper_1511_06051_b200 import _lib
from paper_1511_06051_b200 import netspec as ns

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    text = open(os.path.join(ROOT, "include", "psg.h")).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(psg_[a-z0-9_]+)\s*\(", text)))


def test_library_exports_every_declared_symbol():
    L = ctypes.CDLL(_lib.LIB_PATH)
    missing = [s for s in declared_symbols() if not hasattr(L, s)]
    assert not missing, missing
    assert set(declared_symbols()) == set(_lib.SIGNATURES), \
        set(declared_symbols()) ^ set(_lib.SIGNATURES)


def test_abi_version_and_layer_desc_layout():
    L = _lib.lib()
    assert L.psg_abi_version() == 1
    d = ns.CLayerDesc()
    L.psg_layer_desc_init(ctypes.byref(d), ns.CONV, b"conv1")
    assert d.name == b"conv1" and d.stride_h == 1 and d.group == 1 and d.loss_weight == 1.0
    assert d.lr_mult_w == d.lr_mult_b == d.decay_mult_w == d.decay_mult_b == 1.0


def test_device_calls_fail_loudly_without_gpu():
    """No CPU fallback: without a CUDA device the C ABI reports PSG_ECUDA."""
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    n = ctypes.c_int(-1)
    rc = _lib.lib().psg_device_count(ctypes.byref(n))
    assert rc == _lib.ECUDA
    with pytest.raises(_lib.CudaError):
        from paper_1511_06051_b200.model import Net
        Net(ns.make_mlp(2, 1, 1, 4, 3), 1)


@pytest.mark.parametrize("n,k,seed", [(111, 4, 3), (5500, 8, 1), (7, 7, 2)])
def test_host_shard_matches_oracle(oracle_lib, n, k, seed):
    from paper_1511_06051_b200.data import Dataset, shard
    ds = Dataset(np.zeros((n, 1, 1, 1)), np.zeros(n, np.int32), 1)
    got = shard(ds, k, seed)
    want = oracle_lib.shard(n, k, seed)
    for a, b in zip(got, want):
        np.testing.assert_array_equal(a.indices, b)


def test_host_iterator_matches_oracle(oracle_lib):
    from paper_1511_06051_b200.data import Dataset, make_worker_iterator, shard
    ds = Dataset(np.zeros((111, 1, 1, 1)), np.zeros(111, np.int32), 1)
    it = make_worker_iterator(shard(ds, 4, 3), 2, 5, 3)
    got = np.concatenate([it.next_indices() for _ in range(40)])
    np.testing.assert_array_equal(got, oracle_lib.worker_indices(111, 4, 2, 5, 3, 40))


def test_host_generator_matches_golden(golden):
    from golden_util import equal
    from paper_1511_06051_b200.data import generate_synthetic
    img, lab = generate_synthetic(3, 3, 8, 8, 2, 4.0, 7, 0)
    assert equal(golden, "synth_3_3_8_8_2_4_7_0_images", img)
    assert equal(golden, "synth_3_3_8_8_2_4_7_0_labels", lab)


def test_shard_errors():
    from paper_1511_06051_b200.data import Dataset, shard
    ds = Dataset(np.zeros((3, 1, 1, 1)), np.zeros(3, np.int32), 1)
    with pytest.raises(ValueError):
        shard(ds, 0, 1)
    with pytest.raises(ValueError):
        shard(ds, 4, 1)


def test_netspec_validation_mirrors_reference():
    with pytest.raises(ValueError):
        ns.NetSpec([ns.data_layer("d", 1, 1, 4, 4), ns.label_layer("l", 1),
                    ns.conv_layer("c", "x", 3, 3, 2),
                    ns.softmax_loss_layer("loss", "c", "l")]).validate()
    with pytest.raises(ValueError):
        ns.NetSpec([ns.data_layer("d", 1, 1, 4, 4), ns.label_layer("l", 1)]).validate()
    with pytest.raises(ValueError):
        ns.NetSpec([ns.data_layer("d", 1, 1, 4, 4), ns.data_layer("d", 1, 1, 4, 4)]).validate()


def test_param_counts_match_survey():
    """P for cq / AlexNet."""
    assert ns.param_count(ns.make_cifar10_quick(100)) == 145578
    assert ns.param_count(ns.make_alexnet(256)) == 60965224
    assert ns.param_count(ns.make_lenet_small(50, 1, 16, 16, 10)) == 5162
    assert ns.param_count(ns.make_cq_valid(100)) == 63658


def test_work_units_match_baseline():
    """fwd MACs / train FLOPs per image."""
    cq = ns.make_cifar10_quick(100)
    assert sum(ns.forward_macs(cq).values()) == 12_354_176  # "12.35 M"
    assert abs(ns.train_flops_per_image(cq) / 1e6 - 69.2) < 0.05
    ax = ns.make_alexnet(256)
    assert abs(sum(ns.forward_macs(ax).values()) / 1e6 - 724.41) < 0.01
    assert abs(ns.train_flops_per_image(ax) / 1e9 - 4.136) < 0.002


def test_weights_mean_host_semantics(golden):
    from paper_1511_06051_b200.weights import WeightCollection, weights_mean
    from golden_util import equal
    items = golden["mean_4_items"]
    cols = [WeightCollection([("t", [items[k]])]) for k in range(4)]
    m = weights_mean(cols)
    assert equal(golden, "mean_4_out", m.entry(0)[1][0])
    with pytest.raises(ValueError):
        weights_mean([])
    with pytest.raises(ValueError):
        weights_mean([cols[0], WeightCollection([("u", [items[0]])])])
    assert m.same_structure(cols[0])


def test_weight_collection_digest_matches_reference(golden, oracle_lib):
    """FNV-1a digest (weights.hpp:66-82) of the lenet-small golden weights."""
    from paper_1511_06051_b200.weights import WeightCollection
    spec = ns.make_lenet_small(6, 1, 16, 16, 10)
    orc = oracle_lib.net(spec, 42)
    flat = orc.get_weights()
    orc.apply_update(np.zeros_like(flat))
    w = WeightCollection()
    pos = 0
    shapes = {"conv1": [(8, 1, 5, 5), (8,)], "conv2": [(16, 8, 5, 5), (16,)],
              "ip1": [(64, 16), (64,)], "ip2": [(10, 64), (10,)]}
    for l in spec.layers:
        ts = []
        for shp in shapes.get(l.name, []):
            cnt = int(np.prod(shp))
            ts.append(flat[pos:pos + cnt].reshape(shp))
            pos += cnt
        w.add(l.name, ts)
    assert w.digest() == orc.digest(flat)


def test_cpp_dropin_builds_against_reference_headers():
    """include/parasgd_b200 compiles as a drop-in next to the reference's own headers."""
    import __graft_entry__ as ge
    if not os.path.isdir(ge.REF_INC):
        pytest.skip("reference headers absent (GPU box): the binary is prebuilt")
    ge.build_cpp_dropin()
    assert os.path.exists(os.path.join(ROOT, "tests", "cpp", "dropin_test"))
