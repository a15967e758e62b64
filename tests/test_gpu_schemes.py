"""GPU schemes beyond run_sparknet: run_naive (schemes.hpp:201-262), run_serial
(schemes.hpp:154-193) and sharded per-round evaluation, checked
against the pinned C oracle (whose run_naive is bit-exact to the reference,
tests/test_oracle_golden.py::test_run_naive_bit_exact)."""
import numpy as np
import pytest

from oracle.pyoracle import max_relative_deviation
from paper_1511_06051_b200 import netspec as ns

pytestmark = pytest.mark.gpu

STRICT = 1e-5


def f32(x):
    return np.asarray(x, np.float64).astype(np.float32).astype(np.float64)


def _data(oracle_lib, per_class, variant):
    from paper_1511_06051_b200.data import Dataset
    img, lab = oracle_lib.generate_synthetic(10, 1, 16, 16, per_class, 2.0, 12345, variant)
    return Dataset(f32(img), lab, 10), (f32(img), lab)


def _ctx(spec, train, evald, batch, mu, devices=None):
    from paper_1511_06051_b200 import schemes
    from paper_1511_06051_b200.model import SgdOptions
    return schemes.SchemeContext(net=spec, train_data=train, eval_data=evald, batch=batch,
                                 sgd=SgdOptions(0.05, mu), seed=1,
                                 cost=schemes.CostModel(2.0, 10.0, 1.0), target_accuracy=2.0,
                                 eval_steps=2, devices=devices, precision="fp32")


@pytest.mark.parametrize("K,mu", [(1, 0.0), (2, 0.9), (5, 0.5)])
def test_run_naive_step_parity(oracle_lib, K, mu):
    """Every step: the K part gradients (K nets on one GPU) averaged in the reference's
    order and applied == the oracle's run_naive, step by step from the same start.
    Per-step deviations stay at the fp32 level; records match the reference's clock."""
    from paper_1511_06051_b200 import schemes
    spec = ns.make_lenet_small(10, 1, 16, 16, 10)
    train, th = _data(oracle_lib, 24, 0)
    evald, eh = _data(oracle_lib, 6, 1)
    steps = 4
    want_recs, want_w = oracle_lib.run_naive(spec, th, eh, 10, 0.05, mu, 1, K, steps, 2,
                                             eval_steps=2, cost=(2.0, 10.0, 1.0),
                                             want_weights=True)
    got_w = []
    obs = schemes.SchemeObserver(on_step=lambda it, net: got_w.append(net.get_weights_flat()))
    trace = schemes.run_naive(_ctx(spec, train, evald, 10, mu), K, steps, 2, obs)
    assert trace.scheme == "naive" and len(trace.records) == len(want_recs) == 2
    for r, w in zip(trace.records, want_recs):
        assert (r.serial_iters, r.parallel_iters, r.rounds) == tuple(w[:3])
        assert r.sim_time == w[3]
    segs = None
    for s in range(steps):
        dev = max_relative_deviation(got_w[s], want_w[s], segs)
        # fp32 vs fp64 trajectories drift slowly; the first step is the isolated bar
        assert dev <= (STRICT if s == 0 else 20 * STRICT), (s, dev)


def test_run_naive_matches_serial_full_batch(oracle_lib):
    """schemes.hpp:196-200: run_naive is algorithmically run_serial on the same stream."""
    from paper_1511_06051_b200 import schemes
    spec = ns.make_lenet_small(10, 1, 16, 16, 10)
    train, _ = _data(oracle_lib, 24, 0)
    evald, _ = _data(oracle_lib, 6, 1)
    got = {}
    for name, run in (("naive", lambda c, o: schemes.run_naive(c, 2, 3, 3, o)),
                      ("serial", lambda c, o: schemes.run_serial(c, 3, 3, o))):
        ws = []
        run(_ctx(spec, train, evald, 10, 0.9),
            schemes.SchemeObserver(on_step=lambda it, net: ws.append(net.get_weights_flat())))
        got[name] = ws
    for a, b in zip(got["naive"], got["serial"]):
        assert max_relative_deviation(a, b) <= 10 * STRICT


def test_sharded_eval_equals_single_net(oracle_lib):
    """Sharded evaluation (K nets with the same weights, batches k, k+K, ...) gives the
    same integer counts as one net's test(steps), including iterator wrap-around."""
    from paper_1511_06051_b200 import schemes
    from paper_1511_06051_b200.model import Net
    spec = ns.make_lenet_small(10, 1, 16, 16, 10)
    evald, _ = _data(oracle_lib, 5, 1)  # 50 rows, b = 10 -> wraps after 5 batches
    nets = [Net(spec, 1) for _ in range(3)]
    w = nets[0].get_weights_flat()
    for n in nets[1:]:
        n.set_weights_flat(w)
    ctx = _ctx(spec, evald, evald, 10, 0.0)
    for steps in (1, 2, 3, 7, 11):
        ctx.eval_steps = steps
        single = schemes.evaluate(nets[0], ctx)
        assert schemes.evaluate_sharded(nets, ctx) == single
        assert schemes.evaluate_sharded(nets[:2], ctx) == single


def test_sharded_eval_counts_match_oracle_argmax(oracle_lib):
    """The fused device argmax/count agrees with the oracle's evaluate on fp32-exact
    weights (strict fp32 forward; argmax ties to the lowest index)."""
    from paper_1511_06051_b200 import schemes
    from paper_1511_06051_b200.model import Net
    spec = ns.make_lenet_small(10, 1, 16, 16, 10)
    train, th = _data(oracle_lib, 24, 0)
    evald, eh = _data(oracle_lib, 6, 1)
    # a trained state so predictions are not degenerate
    recs, rw = oracle_lib.run_naive(spec, th, eh, 10, 0.05, 0.9, 1, 1, 6, 6, eval_steps=6,
                                    want_weights=True)
    nets = [Net(spec, 1) for _ in range(2)]
    for n in nets:
        n.set_weights_flat(f32(rw[-1]))
    ctx = _ctx(spec, train, evald, 10, 0.0)
    ctx.eval_steps = 6
    acc = schemes.evaluate_sharded(nets, ctx)
    orc = oracle_lib.net(spec, 1)
    orc.set_weights(f32(rw[-1]))
    _, probs = orc.forward(eh[0][:60], eh[1][:60])
    want = float(np.mean(np.argmax(probs, axis=1) == eh[1][:60]))
    # a near-tie can flip between fp32 and fp64 on at most a couple of the 60 rows
    assert abs(acc - want) <= 2.0 / 60 + 1e-12


def _gpus():
    try:
        import torch
        return torch.cuda.device_count()
    except Exception:
        return 0


@pytest.mark.parametrize("mode", ["ordered", "fast"])
def test_run_naive_two_gpus_matches_one_gpu(oracle_lib, mode):
    """Across GPUs the part gradients are averaged by NCCL (ordered: bit-identical to the
    single-GPU ordered kernel); evaluation is sharded across the workers."""
    if _gpus() < 2:
        pytest.skip("needs >= 2 GPUs")
    from paper_1511_06051_b200 import schemes
    spec = ns.make_lenet_small(10, 1, 16, 16, 10)
    train, _ = _data(oracle_lib, 24, 0)
    evald, _ = _data(oracle_lib, 6, 1)
    runs = {}
    for devs in (None, [0, 1]):
        ws = []
        ctx = _ctx(spec, train, evald, 10, 0.9, devices=devs)
        ctx.average_mode = mode
        t = schemes.run_naive(ctx, 2, 4, 2, schemes.SchemeObserver(
            on_step=lambda it, net: ws.append(net.get_weights_flat())))
        runs[str(devs)] = (ws, [r.accuracy for r in t.records])
    (w1, a1), (w2, a2) = runs["None"], runs["[0, 1]"]
    for a, b in zip(w1, w2):
        if mode == "ordered":
            np.testing.assert_array_equal(a, b)
        else:
            assert max_relative_deviation(a, b) <= STRICT
    if mode == "ordered":
        assert a1 == a2


def _mlp_fixture():
    """schemes_test.cpp:17-37: mlp 8-4-2 on generate_synthetic(2, 1, 1, 8, 60, 3.0, 501),
    plain SGD lr 0.05 (mu = 0)."""
    from paper_1511_06051_b200 import schemes
    from paper_1511_06051_b200.data import Dataset, generate_synthetic
    from paper_1511_06051_b200.model import SgdOptions
    img, lab = generate_synthetic(2, 1, 1, 8, 60, 3.0, 501, 0)
    train = Dataset(f32(img), lab, 2)
    img, lab = generate_synthetic(2, 1, 1, 8, 20, 3.0, 501, 1)
    evald = Dataset(f32(img), lab, 2)

    def ctx(seed, batch=8, devices=None, mode="ordered"):
        c = schemes.SchemeContext(net=ns.make_mlp(batch, 1, 1, 8, 2, 4), train_data=train,
                                  eval_data=evald, batch=batch, sgd=SgdOptions(0.05, 0.0),
                                  seed=seed, cost=schemes.CostModel(1.0, 0.0, 1.0),
                                  target_accuracy=2.0, eval_steps=5, devices=devices,
                                  precision="fp32")
        c.average_mode = mode
        return c
    return train, ctx


def test_tau1_equals_big_batch_serial():
    """schemes_test.cpp:178-213 / acceptance 1b on the device: run_sparknet with K = 2
    workers, tau = 1, b = 4 (ordered K-way average) == serial SGD with batch K*b on the
    concatenated worker batches, same initial weights and lr (mu = 0).  The reference's
    fp64 bar is 1e-10; in fp32 the two paths sum the same gradient terms in different
    orders (mean of 4, then mean of 2, vs mean of 8): per-round deviations stay at the fp32
    level."""
    from paper_1511_06051_b200 import data, schemes
    from paper_1511_06051_b200.model import Batch, Net, SgdOptions
    train, ctx = _mlp_fixture()
    c = ctx(13, batch=4)
    rounds = []
    schemes.run_sparknet(c, 2, 1, 30, 0, 1, schemes.SchemeObserver(
        on_round=lambda r, w: rounds.append(np.concatenate([t.ravel() for _, ts in w
                                                             for t in ts]))))
    big = Net(ns.make_mlp(8, 1, 1, 8, 2, 4), 13)
    big.set_sgd(SgdOptions(0.05, 0.0))
    shards = data.shard(train, 2, 13)
    streams = [data.make_worker_iterator(shards, k, 4, 13) for k in range(2)]
    worst = 0.0
    for r in range(30):
        idx = np.concatenate([s.next_indices() for s in streams]).astype(np.int64)
        _, g = big.backward_flat(Batch(train.images[idx], train.labels[idx]))
        big.apply_update_flat(g)
        worst = max(worst, max_relative_deviation(rounds[r], big.get_weights_flat()))
    assert len(rounds) == 30
    assert worst <= 1e-5, worst


def test_run_sparknet_k_gpus_bitwise_equals_k_nets_on_one_gpu():
    """schemes_test.cpp:249-260 (threaded == sequential, bitwise) on B200s: K = 2 workers
    on 2 GPUs with the ordered NCCL average (all-to-all, ascending-k fp64 reduce, allgather)
    produce bit-identical rounds, warm start and accuracies to the K nets on one GPU
    (ordered local average)."""
    if _gpus() < 2:
        pytest.skip("needs >= 2 GPUs")
    from paper_1511_06051_b200 import schemes
    _, ctx = _mlp_fixture()
    runs = []
    for devs in (None, [0, 1]):
        ws = []
        t = schemes.run_sparknet(ctx(19, devices=devs), 2, 3, 10, 5, 1, schemes.SchemeObserver(
            on_round=lambda r, w: ws.append(np.concatenate([x.ravel() for _, xs in w
                                                            for x in xs]))))
        runs.append((ws, t))
    (wa, ta), (wb, tb) = runs
    assert len(wa) == len(wb) == 10
    for a, b in zip(wa, wb):
        np.testing.assert_array_equal(a, b)
    assert ta.warm_digest == tb.warm_digest
    assert [r.accuracy for r in ta.records] == [r.accuracy for r in tb.records]
