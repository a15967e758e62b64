"""Pins for the oracle's Caffe extensions the reference cannot express:
pad/stride/group conv, AVE + ceil-mode pooling, LRN, dropout, weight decay, multipliers.

Method: the reference's own central finite-difference oracle (test_helpers.hpp:44-73,
step 1e-5, relative_error floor 1e-5, bar 1e-5), plus the exact identities
  * pad p conv == valid conv on a zero-padded input (forward and dK),
  * stride s conv == the stride-1 output subsampled,
  * group G conv == G independent convs on channel slices,
where the right-hand sides run on the reference-expressible subset, itself pinned bit for
bit to the unmodified reference (test_oracle_golden.py)."""
import zlib

import numpy as np
import pytest

from paper_1511_06051_b200 import netspec as ns


def relative_error(a, b, floor=1e-5):
    return abs(a - b) / max(abs(a), abs(b), floor)


def max_gradient_error(net, x, y, step=1e-5, stride=1):
    """test_helpers.hpp:51-73 on the oracle (train phase: dropout masks fixed)."""
    _, analytic = net.backward(x, y)
    w0 = net.get_weights()
    worst = 0.0
    for i in range(0, w0.size, stride):
        p = w0.copy()
        p[i] += step
        net.set_weights(p)
        up, _ = net.forward(x, y, train=True)
        p[i] -= 2 * step
        net.set_weights(p)
        down, _ = net.forward(x, y, train=True)
        fd = (up - down) / (2 * step)
        worst = max(worst, relative_error(fd, analytic[i]))
    net.set_weights(w0)
    return worst


def _batch(rng, spec, classes):
    d = spec.data_spec().shape
    x = rng.uniform(-1, 1, size=tuple(d))
    y = rng.integers(0, classes, size=d[0]).astype(np.int32)
    return x, y


EXT_NETS = {
    "pad_stride_conv": ns.NetSpec([
        ns.data_layer("data", 2, 2, 7, 7), ns.label_layer("label", 2),
        ns.conv_layer("c1", "data", 3, 3, 4, stride=2, pad=1), ns.relu_layer("r1", "c1"),
        ns.linear_layer("fc", "r1", 3), ns.softmax_loss_layer("loss", "fc", "label")]),
    "group_conv": ns.NetSpec([
        ns.data_layer("data", 2, 4, 6, 6), ns.label_layer("label", 2),
        ns.conv_layer("c1", "data", 3, 3, 4, pad=1, group=2),
        ns.conv_layer("c2", "c1", 3, 3, 6, group=2), ns.linear_layer("fc", "c2", 3),
        ns.softmax_loss_layer("loss", "fc", "label")]),
    "ave_ceil_pool": ns.NetSpec([
        ns.data_layer("data", 2, 1, 8, 8), ns.label_layer("label", 2),
        ns.conv_layer("c1", "data", 3, 3, 3, pad=2),
        ns.pool_layer("p1", "c1", 3, 3, 2, 2, method=ns.POOL_AVE, ceil_mode=True),
        ns.pool_layer("p2", "p1", 3, 3, 2, 2, method=ns.POOL_MAX, ceil_mode=True, pad=1),
        ns.linear_layer("fc", "p2", 3), ns.softmax_loss_layer("loss", "fc", "label")]),
    "lrn": ns.NetSpec([
        ns.data_layer("data", 2, 2, 5, 5), ns.label_layer("label", 2),
        ns.conv_layer("c1", "data", 3, 3, 7), ns.relu_layer("r1", "c1"),
        ns.lrn_layer("n1", "r1", 5, 0.5, 0.75, 1.0),
        ns.linear_layer("fc", "n1", 3), ns.softmax_loss_layer("loss", "fc", "label")]),
    "dropout": ns.NetSpec([
        ns.data_layer("data", 3, 1, 1, 12), ns.label_layer("label", 3),
        ns.linear_layer("ip1", "data", 16), ns.relu_layer("r1", "ip1"),
        ns.dropout_layer("d1", "r1", 0.5), ns.linear_layer("ip2", "d1", 4),
        ns.softmax_loss_layer("loss", "ip2", "label", loss_weight=0.7)]),
    # GoogLeNet-style branch + concat + an auxiliary weighted loss head
    "inception_concat_aux": ns.NetSpec([
        ns.data_layer("data", 2, 3, 6, 6), ns.label_layer("label", 2),
        ns.conv_layer("a1", "data", 1, 1, 2), ns.relu_layer("ra", "a1"),
        ns.conv_layer("b1", "data", 1, 1, 2), ns.conv_layer("b3", "b1", 3, 3, 3, pad=1),
        ns.pool_layer("pp", "data", 3, 3, 1, 1, pad=1, ceil_mode=True),
        ns.conv_layer("pj", "pp", 1, 1, 2),
        ns.concat_layer("cat", ["ra", "b3", "pj"]),
        ns.linear_layer("aux", "b1", 3),
        ns.softmax_loss_layer("aux_loss", "aux", "label", loss_weight=0.3),
        ns.pool_layer("gp", "cat", 6, 6, 1, 1, method=ns.POOL_AVE),
        ns.linear_layer("fc", "gp", 3), ns.softmax_loss_layer("loss", "fc", "label")]),
}


@pytest.mark.parametrize("name", list(EXT_NETS))
def test_extension_gradients_match_finite_differences(oracle_lib, name):
    spec = EXT_NETS[name]
    rng = np.random.default_rng(zlib.crc32(name.encode()))
    for trial in range(2):
        net = oracle_lib.net(spec, 100 + trial)
        net.set_dropout_step(trial + 3)
        x, y = _batch(rng, spec, net.classes)
        assert max_gradient_error(net, x, y) < 1e-5


def _single_conv(b, c, h, w, f, k, **kw):
    return ns.NetSpec([ns.data_layer("data", b, c, h, w), ns.label_layer("label", b),
                       ns.conv_layer("c1", "data", k, k, f, **kw),
                       ns.linear_layer("fc", "c1", 2), ns.softmax_loss_layer("loss", "fc", "label")])


def test_pad_equals_valid_conv_on_padded_input(oracle_lib):
    rng = np.random.default_rng(1)
    p = 2
    a = oracle_lib.net(_single_conv(2, 3, 6, 6, 4, 5, pad=p), 9)
    b = oracle_lib.net(_single_conv(2, 3, 6 + 2 * p, 6 + 2 * p, 4, 5), 9)
    oa, ca = a.layer_params(2)
    wk = a.get_weights()[oa:oa + ca]
    x = rng.normal(size=(2, 3, 6, 6))
    xp = np.pad(x, ((0, 0), (0, 0), (p, p), (p, p)))
    wb = b.get_weights()
    ob, _ = b.layer_params(2)
    wb[ob:ob + ca] = wk
    b.set_weights(wb)
    ya = a.layer_forward(2, 2, [x])
    yb = b.layer_forward(2, 2, [xp])
    np.testing.assert_array_equal(ya, yb)
    dy = rng.normal(size=ya.shape)
    _, dpa = a.layer_backward(2, 2, dy, want_dx=False)
    _, dpb = b.layer_backward(2, 2, dy, want_dx=False)
    np.testing.assert_allclose(dpa, dpb, rtol=0, atol=1e-13)


def test_stride_equals_subsampled_stride1(oracle_lib):
    rng = np.random.default_rng(2)
    a = oracle_lib.net(_single_conv(2, 3, 11, 11, 4, 3, stride=4), 3)
    b = oracle_lib.net(_single_conv(2, 3, 11, 11, 4, 3), 3)
    b.set_weights(np.concatenate([a.get_weights()[:4 * 3 * 9 + 4],
                                  b.get_weights()[4 * 3 * 9 + 4:]]))
    x = rng.normal(size=(2, 3, 11, 11))
    ya = a.layer_forward(2, 2, [x])
    yb = b.layer_forward(2, 2, [x])
    np.testing.assert_array_equal(ya, yb[:, :, ::4, ::4])


def test_group_equals_sliced_convs(oracle_lib):
    rng = np.random.default_rng(3)
    g = oracle_lib.net(_single_conv(2, 4, 5, 5, 6, 3, group=2), 4)
    og, cg = g.layer_params(2)
    wg = g.get_weights()[og:og + cg]
    kern, bias = wg[:6 * 2 * 9].reshape(6, 2, 3, 3), wg[6 * 2 * 9:]
    x = rng.normal(size=(2, 4, 5, 5))
    y = g.layer_forward(2, 2, [x])
    for grp in range(2):
        s = oracle_lib.net(_single_conv(2, 2, 5, 5, 3, 3), 4)
        ws = s.get_weights()
        ws[:3 * 2 * 9] = kern[3 * grp:3 * grp + 3].ravel()
        ws[3 * 2 * 9:3 * 2 * 9 + 3] = bias[3 * grp:3 * grp + 3]
        s.set_weights(ws)
        ys = s.layer_forward(2, 2, [x[:, 2 * grp:2 * grp + 2]])
        np.testing.assert_array_equal(y[:, 3 * grp:3 * grp + 3], ys)


def test_ave_pool_matches_direct_numpy(oracle_lib):
    spec = EXT_NETS["ave_ceil_pool"]
    net = oracle_lib.net(spec, 1)
    rng = np.random.default_rng(4)
    x = rng.normal(size=(2, 3, 10, 10))
    y = net.layer_forward(3, 2, [x])
    # Caffe AVE, ceil mode: 10 -> ceil((10-3)/2)+1 = 5, last window clipped, divisor clipped to H+pad
    assert y.shape == (2, 3, 5, 5)
    want = np.zeros_like(y)
    for i in range(5):
        for j in range(5):
            hs, ws = 2 * i, 2 * j
            he, we = min(hs + 3, 10), min(ws + 3, 10)
            want[:, :, i, j] = x[:, :, hs:he, ws:we].sum(axis=(2, 3)) / ((he - hs) * (we - ws))
    np.testing.assert_allclose(y, want, rtol=1e-14, atol=1e-14)


def test_dropout_mask_rate_and_test_phase_identity(oracle_lib):
    spec = EXT_NETS["dropout"]
    net = oracle_lib.net(spec, 5)
    x = np.random.default_rng(6).normal(size=(3, 1, 1, 12))
    y = np.zeros(3, np.int32)
    net.forward(x, y, train=True)
    before = net.layer_out(3, 3)
    after = net.layer_out(4, 3)
    kept = after != 0
    np.testing.assert_allclose(after[kept], 2.0 * before[kept])
    # test phase is the identity
    net.forward(x, y, train=False)
    np.testing.assert_array_equal(net.layer_out(4, 3), net.layer_out(3, 3))


def test_weight_decay_and_multipliers(oracle_lib):
    """v = mu v + (g + lambda * decay_mult * w); w -= lr * lr_mult * v; lambda=0 == reference."""
    spec = ns.NetSpec([ns.data_layer("data", 2, 1, 1, 4), ns.label_layer("label", 2),
                       ns.linear_layer("ip", "data", 3, lr_mult=(1.0, 2.0), decay_mult=(1.0, 0.0)),
                       ns.softmax_loss_layer("loss", "ip", "label")])
    net = oracle_lib.net(spec, 2)
    w = net.get_weights()
    g = np.random.default_rng(7).normal(size=w.size)
    net.set_sgd(0.1, 0.9, 0.01)
    net.apply_update(g)
    want = w.copy()
    nk = 12
    want[:nk] = w[:nk] - 0.1 * (g[:nk] + 0.01 * w[:nk])
    want[nk:] = w[nk:] - 0.2 * g[nk:]
    np.testing.assert_allclose(net.get_weights(), want, rtol=1e-15, atol=1e-15)


def test_concat_forward_is_channel_stacking(oracle_lib):
    """concat output == the inputs stacked along channels (NCHW)."""
    spec = ns.NetSpec([ns.data_layer("data", 2, 2, 3, 3), ns.label_layer("label", 2),
                       ns.conv_layer("a", "data", 1, 1, 3), ns.conv_layer("b", "data", 3, 3, 2, pad=1),
                       ns.concat_layer("cat", ["a", "b", "a"]), ns.linear_layer("fc", "cat", 2),
                       ns.softmax_loss_layer("loss", "fc", "label")])
    net = oracle_lib.net(spec, 4)
    rng = np.random.default_rng(2)
    x, y = _batch(rng, spec, 2)
    net.forward(x, y)
    a, b, cat = (net.layer_out(spec.index_of(k), 2) for k in ("a", "b", "cat"))
    np.testing.assert_array_equal(cat, np.concatenate([a, b, a], axis=1))


def test_multiple_losses_sum_weighted(oracle_lib):
    """Total loss = sum of loss_weight x mean cross-entropy over the loss layers; the
    gradient of a weighted aux head is that weight times its unit-weight gradient."""
    def spec(w_aux):
        return ns.NetSpec([ns.data_layer("data", 3, 1, 1, 5), ns.label_layer("label", 3),
                           ns.linear_layer("h", "data", 4),
                           ns.linear_layer("aux", "h", 3),
                           ns.softmax_loss_layer("l1", "aux", "label", loss_weight=w_aux),
                           ns.linear_layer("fc", "h", 3),
                           ns.softmax_loss_layer("l2", "fc", "label")])
    rng = np.random.default_rng(9)
    x = rng.normal(size=(3, 1, 1, 5))
    y = np.array([0, 2, 1], np.int32)
    n0 = oracle_lib.net(spec(0.0), 3)
    n1 = oracle_lib.net(spec(1.0), 3)
    nw = oracle_lib.net(spec(0.3), 3)
    l0, g0 = n0.backward(x, y)
    l1, g1 = n1.backward(x, y)
    lw, gw = nw.backward(x, y)
    aux_only = l1 - l0
    assert lw == pytest.approx(l0 + 0.3 * aux_only, rel=1e-12)
    np.testing.assert_allclose(gw - g0, 0.3 * (g1 - g0), rtol=1e-9, atol=1e-12)
