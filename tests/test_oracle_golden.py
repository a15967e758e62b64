"""The C oracle is pinned, bit for bit, to golden vectors produced by the unmodified
reference (tests/golden/make_golden.py).  CPU only."""
import numpy as np
import pytest

from golden_util import equal, net_input_rng
from paper_1511_06051_b200 import netspec as ns

NETS = ["lenet_small", "mlp", "cq_valid", "micro", "conv_pool_conv"]


def _spec(name):
    import importlib.util
    import os
    path = os.path.join(os.path.dirname(__file__), "golden", "make_golden.py")
    spec = importlib.util.spec_from_file_location("make_golden", path)
    mod = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mod)
    return mod.NETS[name]


@pytest.mark.parametrize("n,k,seed", [(111, 4, 3), (5500, 8, 1), (50, 1, 9), (7, 7, 2)])
def test_shard_bit_exact(oracle_lib, golden, n, k, seed):
    """data.hpp:261-288; data_test.cpp:188-226."""
    shards = oracle_lib.shard(n, k, seed)
    for i, s in enumerate(shards):
        assert equal(golden, f"shard_{n}_{k}_{seed}_{i}", s.astype(np.uint32))
    allidx = np.sort(np.concatenate(shards))
    assert np.array_equal(allidx, np.arange(n))
    sizes = [s.size for s in shards]
    assert max(sizes) - min(sizes) <= 1


@pytest.mark.parametrize("n,k,w,b,seed,steps", [(111, 4, 2, 5, 3, 40), (5500, 4, 0, 50, 1, 60),
                                                 (5500, 4, 3, 50, 1, 60), (120, 1, 0, 8, 11, 50)])
def test_worker_stream_bit_exact(oracle_lib, golden, n, k, w, b, seed, steps):
    """ShardBatchIterator (data.hpp:312-351): per-epoch reshuffle, drop-last."""
    idx = oracle_lib.worker_indices(n, k, w, b, seed, steps)
    assert equal(golden, f"stream_{n}_{k}_{w}_{b}_{seed}_{steps}", idx.astype(np.uint32))


def test_epoch_partitions_shard(oracle_lib):
    """data_test.cpp:228-268: an epoch's batches are disjoint and come from the shard."""
    shard = oracle_lib.shard(103, 3, 5)[1]
    b = 7
    idx = oracle_lib.worker_indices(103, 3, 1, b, 5, shard.size // b)
    assert len(set(idx.tolist())) == idx.size
    assert set(idx.tolist()) <= set(shard.tolist())


@pytest.mark.parametrize("cls,c,h,w,per,sep,seed,var", [(10, 1, 16, 16, 2, 2.0, 12345, 0),
                                                         (10, 1, 16, 16, 2, 2.0, 12345, 1),
                                                         (3, 3, 8, 8, 2, 4.0, 7, 0)])
def test_synthetic_bit_exact(oracle_lib, golden, cls, c, h, w, per, sep, seed, var):
    """generate_synthetic (data.hpp:111-155)."""
    img, lab = oracle_lib.generate_synthetic(cls, c, h, w, per, sep, seed, var)
    key = f"synth_{cls}_{c}_{h}_{w}_{per}_{int(sep)}_{seed}_{var}"
    assert equal(golden, key + "_images", img)
    assert equal(golden, key + "_labels", lab)


@pytest.mark.parametrize("k", [1, 2, 3, 4, 8])
def test_weights_mean_bit_exact(oracle_lib, golden, k):
    """weights.hpp:90-107 + tensor.hpp:166-179."""
    items = golden[f"mean_{k}_items"]
    out = oracle_lib.weights_mean(list(items))
    assert equal(golden, f"mean_{k}_out", out)


@pytest.mark.parametrize("idx,name", list(enumerate(NETS)))
def test_net_bit_exact(oracle_lib, golden, idx, name):
    """Net init / forward / backward / per-layer state / apply_update (model.hpp)."""
    mk, seed = _spec(name)
    spec = mk()
    net = oracle_lib.net(spec, seed)
    d = spec.data_spec().shape
    classes = net.classes
    rng = net_input_rng(idx)
    x = rng.uniform(-1, 1, size=tuple(d))
    y = rng.integers(0, classes, size=d[0]).astype(np.int32)
    assert equal(golden, f"{name}_x", x)
    assert equal(golden, f"{name}_w0", net.get_weights())
    loss, probs = net.forward(x, y)
    assert equal(golden, f"{name}_loss", np.array([loss]))
    assert equal(golden, f"{name}_probs", probs)
    loss, grads = net.backward(x, y)
    assert equal(golden, f"{name}_grads", grads)
    for li, l in enumerate(spec.layers):
        if l.kind == ns.LABEL:
            continue
        assert equal(golden, f"{name}_out_{li}", net.layer_out(li, d[0]).ravel()), l.name
        if l.kind not in (ns.DATA, ns.SOFTMAX_LOSS):
            # (the data-layer gradient is never observable and is not compared)
            g = net.layer_grad(li, d[0]).ravel()
            assert equal(golden, f"{name}_grad_{li}", g), l.name
    net.set_sgd(0.05, 0.9)
    net.apply_update(grads)
    net.apply_update(grads)
    assert equal(golden, f"{name}_w_after2", net.get_weights())
    assert int(golden[f"{name}_digest"][0]) == net.digest()


@pytest.mark.parametrize("K,tau,rounds,warm,mu", [(1, 3, 3, 2, 0.0), (2, 2, 3, 0, 0.9),
                                                   (4, 3, 2, 4, 0.5)])
def test_run_sparknet_bit_exact(oracle_lib, golden, K, tau, rounds, warm, mu):
    """run_sparknet (schemes.hpp:274-351): per-round averages, records, warm digest."""
    train = oracle_lib.generate_synthetic(10, 1, 16, 16, 24, 2.0, 12345, 0)
    evald = oracle_lib.generate_synthetic(10, 1, 16, 16, 6, 2.0, 12345, 1)
    assert equal(golden, "run_train_images", train[0])
    spec = ns.make_lenet_small(10, 1, 16, 16, 10)
    recs, digest, rw = oracle_lib.run_sparknet(spec, train, evald, 10, 0.05, mu, 1, K, tau,
                                               rounds, warm, threads=2, eval_steps=2,
                                               cost=(2.0, 10.0), want_weights=True)
    key = f"run_{K}_{tau}_{rounds}_{warm}_{int(mu * 10)}"
    assert equal(golden, key + "_records", np.array(recs, np.float64))
    assert int(golden[key + "_digest"][0]) == digest
    assert equal(golden, key + "_weights", rw)


def test_oracle_matches_live_reference_cq_valid(oracle_lib, ref_lib):
    """Where oracle/_ref exists (this container), check the restatement live on a fresh
    seed: the cifar10_quick analog expressible by the reference."""
    spec = ns.make_cq_valid(2)
    a, b = oracle_lib.net(spec, 77), ref_lib.net(spec, 77)
    rng = np.random.default_rng(5)
    x = rng.normal(size=(2, 3, 32, 32))
    y = np.array([3, 7], np.int32)
    la, ga = a.backward(x, y)
    lb, gb = b.backward(x, y)
    assert la == lb and np.array_equal(ga, gb)


@pytest.mark.parametrize("K,iters,every,mu,sub", [(1, 4, 2, 0.0, 1.0), (2, 5, 2, 0.9, 1.0),
                                                  (5, 3, 3, 0.5, 0.7)])
def test_run_naive_bit_exact(oracle_lib, golden, K, iters, every, mu, sub):
    """run_naive (schemes.hpp:201-262): per-step weights and the evaluation records."""
    train = oracle_lib.generate_synthetic(10, 1, 16, 16, 24, 2.0, 12345, 0)
    evald = oracle_lib.generate_synthetic(10, 1, 16, 16, 6, 2.0, 12345, 1)
    spec = ns.make_lenet_small(10, 1, 16, 16, 10)
    recs, sw = oracle_lib.run_naive(spec, train, evald, 10, 0.05, mu, 1, K, iters, every,
                                    eval_steps=2, cost=(2.0, 10.0, sub), want_weights=True)
    key = f"naive_{K}_{iters}_{every}_{int(mu * 10)}"
    assert equal(golden, key + "_records", np.array(recs, np.float64))
    assert equal(golden, key + "_weights", sw)
