"""Generate the golden fixtures in tests/golden/ from the UNMODIFIED reference.

The reference (/root/reference/proj/include, header-only C++) is compiled in place by
oracle/Makefile into oracle/_ref/libparasgd_ref_strict.so (no FP contraction) and driven
through its own public API (plus the private per-layer state via the scoped access
override described in SURVEY §8(c)).  Run from the repo root:

    make -C oracle && python tests/golden/make_golden.py

The fixtures pin the C oracle (oracle/oracle.c) bit for bit; the GPU parity tests then
compare libpsg against the pinned oracle.
"""
from __future__ import annotations

import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

from oracle.pyoracle import RefLib  # noqa: E402
from paper_1511_06051_b200 import netspec as ns  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))


def micro_conv_linear():
    """model_test.cpp:20-36 style micro net: data 1x4x4 -> conv 3x3 (2) -> fc 2."""
    return ns.NetSpec([
        ns.data_layer("data", 1, 1, 4, 4), ns.label_layer("label", 1),
        ns.conv_layer("c1", "data", 3, 3, 2), ns.linear_layer("fc", "c1", 2),
        ns.softmax_loss_layer("loss", "fc", "label")])


def conv_pool_conv():
    """model_test.cpp:186-192."""
    return ns.NetSpec([
        ns.data_layer("data", 2, 1, 8, 8), ns.label_layer("label", 2),
        ns.conv_layer("c1", "data", 3, 3, 2), ns.pool_layer("p1", "c1", 2, 2, 2, 2),
        ns.conv_layer("c2", "p1", 2, 2, 3), ns.linear_layer("fc", "c2", 2),
        ns.softmax_loss_layer("loss", "fc", "label")])


NETS = {
    "lenet_small": (lambda: ns.make_lenet_small(6, 1, 16, 16, 10), 42),
    "mlp": (lambda: ns.make_mlp(5, 1, 1, 16, 10), 5),
    "cq_valid": (lambda: ns.make_cq_valid(3), 11),
    "micro": (micro_conv_linear, 3),
    "conv_pool_conv": (conv_pool_conv, 200),
}


BIG = 4096


def net_input_rng(idx: int) -> np.random.Generator:
    """Inputs of the idx-th NETS entry (PCG64 streams are stable across numpy versions)."""
    return np.random.default_rng(1000 + idx)


def digest_array(a: np.ndarray) -> str:
    """sha256 over the raw little-endian bytes (bitwise identity check)."""
    import hashlib
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def compact(g: dict) -> dict:
    """Large arrays are stored as sha256 + dtype + shape + the first 64 values; bitwise
    equality of a recomputed array is equality of its digest."""
    out = {}
    for k, v in g.items():
        v = np.asarray(v)
        if v.size > BIG:
            out[k + "__sha256"] = np.array(digest_array(v))
            out[k + "__dtype"] = np.array(str(v.dtype))
            out[k + "__shape"] = np.array(v.shape, np.int64)
            out[k + "__head"] = v.ravel()[:64]
        else:
            out[k] = v
    return out


def main() -> None:
    ref = RefLib(strict=True)
    g = {}
    # rng.hpp: splitmix64 / derive_seed via the shard permutation and iterator streams.
    for (n, k, seed) in [(111, 4, 3), (5500, 8, 1), (50, 1, 9), (7, 7, 2)]:
        for i, s in enumerate(ref.shard(n, k, seed)):
            g[f"shard_{n}_{k}_{seed}_{i}"] = s.astype(np.uint32)
    for (n, k, w, b, seed, steps) in [(111, 4, 2, 5, 3, 40), (5500, 4, 0, 50, 1, 60),
                                      (5500, 4, 3, 50, 1, 60), (120, 1, 0, 8, 11, 50)]:
        g[f"stream_{n}_{k}_{w}_{b}_{seed}_{steps}"] = ref.worker_indices(
            n, k, w, b, seed, steps).astype(np.uint32)
    # data.hpp generate_synthetic (variants 0 / 1)
    for (cls, c, h, w, per, sep, seed, var) in [(10, 1, 16, 16, 2, 2.0, 12345, 0),
                                                (10, 1, 16, 16, 2, 2.0, 12345, 1),
                                                (3, 3, 8, 8, 2, 4.0, 7, 0)]:
        img, lab = ref.generate_synthetic(cls, c, h, w, per, sep, seed, var)
        key = f"synth_{cls}_{c}_{h}_{w}_{per}_{int(sep)}_{seed}_{var}"
        g[key + "_images"] = img
        g[key + "_labels"] = lab
    # weights.hpp weights_mean, ascending order
    rng = np.random.default_rng(2024)
    for k in (1, 2, 3, 4, 8):
        items = [rng.uniform(-1, 1, 257) for _ in range(k)]
        g[f"mean_{k}_items"] = np.stack(items)
        g[f"mean_{k}_out"] = ref.weights_mean(items)
    # model.hpp: init, forward, backward, per-layer state, SGD update
    for idx, (name, (mk, seed)) in enumerate(NETS.items()):
        spec = mk()
        rng = net_input_rng(idx)
        net = ref.net(spec, seed)
        d = spec.data_spec().shape
        classes = [l for l in spec.layers if l.kind == ns.LINEAR][-1].num_outputs
        x = rng.uniform(-1, 1, size=tuple(d))
        y = rng.integers(0, classes, size=d[0]).astype(np.int32)
        g[f"{name}_w0"] = net.get_weights()
        g[f"{name}_x"] = x
        g[f"{name}_y"] = y
        loss, probs = net.forward(x, y, classes)
        g[f"{name}_loss"] = np.array([loss])
        g[f"{name}_probs"] = probs
        loss, grads = net.backward(x, y)
        g[f"{name}_grads"] = grads
        for li, l in enumerate(spec.layers):
            if l.kind in (ns.LABEL,):
                continue
            g[f"{name}_out_{li}"] = net.layer_out(li)
            if l.kind not in (ns.DATA, ns.SOFTMAX_LOSS):
                g[f"{name}_grad_{li}"] = net.layer_grad(li)
        net.set_sgd(0.05, 0.9)
        net.apply_update(grads)
        net.apply_update(grads)
        g[f"{name}_w_after2"] = net.get_weights()
        g[f"{name}_digest"] = np.array([net.digest()], np.uint64)
    # schemes.hpp run_sparknet: lenet-small on synthetic 1x16x16, per-round averages
    train = ref.generate_synthetic(10, 1, 16, 16, 24, 2.0, 12345, 0)
    evald = ref.generate_synthetic(10, 1, 16, 16, 6, 2.0, 12345, 1)
    g["run_train_images"], g["run_train_labels"] = train
    g["run_eval_images"], g["run_eval_labels"] = evald
    spec = ns.make_lenet_small(10, 1, 16, 16, 10)
    for (K, tau, rounds, warm, mu) in [(1, 3, 3, 2, 0.0), (2, 2, 3, 0, 0.9), (4, 3, 2, 4, 0.5)]:
        recs, digest, rw = ref.run_sparknet(spec, train, evald, 10, 0.05, mu, 1, K, tau, rounds,
                                            warm, threads=K, eval_steps=2, cost=(2.0, 10.0),
                                            want_weights=True)
        key = f"run_{K}_{tau}_{rounds}_{warm}_{int(mu * 10)}"
        g[key + "_records"] = np.array(recs, np.float64)
        g[key + "_digest"] = np.array([digest], np.uint64)
        g[key + "_weights"] = rw
    # schemes.hpp run_naive: the batch split into K part gradients, averaged, applied
    for (K, iters, every, mu, sub) in [(1, 4, 2, 0.0, 1.0), (2, 5, 2, 0.9, 1.0),
                                       (5, 3, 3, 0.5, 0.7)]:
        recs, sw = ref.run_naive(spec, train, evald, 10, 0.05, mu, 1, K, iters, every,
                                 eval_steps=2, cost=(2.0, 10.0, sub), want_weights=True)
        key = f"naive_{K}_{iters}_{every}_{int(mu * 10)}"
        g[key + "_records"] = np.array(recs, np.float64)
        g[key + "_weights"] = sw
    # csv.hpp format_double: the shortest round-tripping '%.*g' (trace / heatmap schemas)
    rng = np.random.default_rng(77)
    vals = np.concatenate([[0.0, 1.0, 0.1, 1.0 / 3.0, 100.0, 1e-5, 2.5e-300, 123456789.0,
                            -0.75, 1e300, 0.9, 4.0 * (2.0 * 2.0 + 10.0)],
                           rng.uniform(-10, 10, 40), 10.0 ** rng.uniform(-20, 20, 40)])
    g["fmt_values"] = vals
    g["fmt_strings"] = np.array("|".join(ref.format_double(float(v)) for v in vals))
    path = os.path.join(OUT, "reference_golden.npz")
    np.savez_compressed(path, **compact(g))
    print(f"wrote {path}: {len(g)} arrays, {os.path.getsize(path) / 1e6:.2f} MB")


if __name__ == "__main__":
    main()
