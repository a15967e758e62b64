"""TEST INFRASTRUCTURE ONLY: ctypes bindings to the CPU oracle (liboracle.so) and to the
unmodified reference compiled in place (oracle/_ref/libparasgd_ref*.so).

Only tests/, __graft_entry__.smoke() and bench.py's CPU legs may import this module; the
product package (paper_1511_06051_b200) never does.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from typing import Optional, Sequence

import numpy as np

from paper_1511_06051_b200.netspec import CLayerDesc, NetSpec

HERE = os.path.dirname(os.path.abspath(__file__))
_D = ctypes.POINTER(ctypes.c_double)
_I32 = ctypes.POINTER(ctypes.c_int32)
_U64 = ctypes.POINTER(ctypes.c_uint64)


class Record(ctypes.Structure):
    _fields_ = [("serial_iters", ctypes.c_long), ("parallel_iters", ctypes.c_long),
                ("rounds", ctypes.c_long), ("sim_time", ctypes.c_double),
                ("accuracy", ctypes.c_double)]


class SparknetArgs(ctypes.Structure):
    _fields_ = [
        ("layers", ctypes.POINTER(CLayerDesc)), ("n_layers", ctypes.c_int),
        ("train_images", _D), ("train_labels", _I32), ("train_n", ctypes.c_size_t),
        ("eval_images", _D), ("eval_labels", _I32), ("eval_n", ctypes.c_size_t),
        ("c", ctypes.c_int), ("h", ctypes.c_int), ("w", ctypes.c_int),
        ("batch", ctypes.c_size_t),
        ("lr", ctypes.c_double), ("momentum", ctypes.c_double), ("weight_decay", ctypes.c_double),
        ("seed", ctypes.c_uint64),
        ("compute_seconds", ctypes.c_double), ("sync_seconds", ctypes.c_double),
        ("target_accuracy", ctypes.c_double), ("eval_steps", ctypes.c_long),
        ("workers", ctypes.c_int), ("tau", ctypes.c_int),
        ("rounds", ctypes.c_long), ("warm", ctypes.c_long), ("threads", ctypes.c_int),
        ("skip_eval", ctypes.c_int), ("sublinearity", ctypes.c_double),
    ]


def build() -> None:
    """Compile liboracle.so (and oracle/_ref when /root/reference is present)."""
    subprocess.run(["make", "-s", "-C", HERE], check=True)


def _dp(a: np.ndarray):
    return a.ctypes.data_as(_D)


def _ip(a: np.ndarray):
    return a.ctypes.data_as(_I32)


def _up(a: np.ndarray):
    return a.ctypes.data_as(_U64)


class _Lib:
    def __init__(self, path: str):
        if not os.path.exists(path):
            raise FileNotFoundError(path)
        self.lib = ctypes.CDLL(path)


class OracleLib(_Lib):
    """liboracle.so — the C restatement."""

    def __init__(self, path: Optional[str] = None):
        super().__init__(path or os.path.join(HERE, "liboracle.so"))
        L = self.lib
        L.orc_net_create.restype = ctypes.c_void_p
        L.orc_net_create.argtypes = [ctypes.POINTER(CLayerDesc), ctypes.c_int, ctypes.c_uint64]
        L.orc_last_error.restype = ctypes.c_char_p
        L.orc_net_destroy.argtypes = [ctypes.c_void_p]
        L.orc_net_param_count.restype = ctypes.c_size_t
        L.orc_net_param_count.argtypes = [ctypes.c_void_p]
        L.orc_net_num_classes.argtypes = [ctypes.c_void_p]
        for fn in ("orc_net_get_weights", "orc_net_set_weights", "orc_net_get_velocity"):
            getattr(L, fn).argtypes = [ctypes.c_void_p, _D]
        L.orc_net_reset_velocity.argtypes = [ctypes.c_void_p]
        L.orc_net_set_sgd.argtypes = [ctypes.c_void_p, ctypes.c_double, ctypes.c_double,
                                      ctypes.c_double]
        L.orc_net_set_dropout_step.argtypes = [ctypes.c_void_p, ctypes.c_uint64]
        L.orc_net_forward.argtypes = [ctypes.c_void_p, _D, _I32, ctypes.c_size_t, ctypes.c_int,
                                      _D, _D]
        L.orc_net_backward.argtypes = [ctypes.c_void_p, _D, _I32, ctypes.c_size_t, _D, _D]
        L.orc_net_apply_update.argtypes = [ctypes.c_void_p, _D]
        L.orc_net_layer_dims.argtypes = [ctypes.c_void_p, ctypes.c_int,
                                         ctypes.POINTER(ctypes.c_int64)]
        L.orc_net_layer_out.restype = _D
        L.orc_net_layer_out.argtypes = [ctypes.c_void_p, ctypes.c_int]
        L.orc_net_layer_grad.restype = _D
        L.orc_net_layer_grad.argtypes = [ctypes.c_void_p, ctypes.c_int]
        L.orc_layer_forward.argtypes = [ctypes.c_void_p, ctypes.c_int, ctypes.c_size_t,
                                        ctypes.POINTER(_D), _D]
        L.orc_layer_backward.argtypes = [ctypes.c_void_p, ctypes.c_int, ctypes.c_size_t, _D, _D,
                                         _D]
        L.orc_net_layer_params.argtypes = [ctypes.c_void_p, ctypes.c_int,
                                           ctypes.POINTER(ctypes.c_size_t),
                                           ctypes.POINTER(ctypes.c_size_t)]
        L.orc_weights_mean.argtypes = [ctypes.POINTER(_D), ctypes.c_int, ctypes.c_size_t, _D]
        L.orc_generate_synthetic.argtypes = [ctypes.c_int, ctypes.c_size_t, ctypes.c_size_t,
                                             ctypes.c_size_t, ctypes.c_size_t, ctypes.c_double,
                                             ctypes.c_uint64, ctypes.c_uint64, _D, _I32]
        L.orc_shard.argtypes = [ctypes.c_size_t, ctypes.c_int, ctypes.c_uint64, _U64, _U64]
        L.orc_worker_stream_seed.restype = ctypes.c_uint64
        L.orc_worker_stream_seed.argtypes = [ctypes.c_uint64, ctypes.c_int]
        L.orc_epoch_order.argtypes = [_U64, ctypes.c_size_t, ctypes.c_uint64, ctypes.c_uint64,
                                      _U64]
        L.orc_splitmix64.restype = ctypes.c_uint64
        L.orc_splitmix64.argtypes = [ctypes.c_uint64]
        L.orc_derive_seed.restype = ctypes.c_uint64
        L.orc_derive_seed.argtypes = [ctypes.c_uint64, _U64, ctypes.c_int]
        L.orc_run_sparknet.restype = ctypes.c_long
        L.orc_run_sparknet.argtypes = [ctypes.POINTER(SparknetArgs), ctypes.POINTER(Record),
                                       ctypes.c_long, _U64, _D]
        L.orc_run_naive.restype = ctypes.c_long
        L.orc_run_naive.argtypes = [ctypes.POINTER(SparknetArgs), ctypes.c_long, ctypes.c_long,
                                    ctypes.POINTER(Record), ctypes.c_long, _D]
        L.orc_weights_digest.restype = ctypes.c_uint64
        L.orc_weights_digest.argtypes = [ctypes.c_void_p, _D]

    def error(self) -> str:
        return self.lib.orc_last_error().decode()

    def generate_synthetic(self, classes, c, h, w, per_class, separation, seed, variant=0):
        n = classes * per_class
        images = np.empty((n, c, h, w), np.float64)
        labels = np.empty(n, np.int32)
        self.lib.orc_generate_synthetic(classes, c, h, w, per_class, separation, seed, variant,
                                        _dp(images), _ip(labels))
        return images, labels

    def shard(self, n, workers, seed):
        perm = np.empty(n, np.uint64)
        offs = np.empty(workers + 1, np.uint64)
        rc = self.lib.orc_shard(n, workers, seed, _up(perm), _up(offs))
        if rc:
            raise ValueError(self.error())
        return [perm[offs[k]:offs[k + 1]].copy() for k in range(workers)]

    def worker_stream_seed(self, seed, k):
        return self.lib.orc_worker_stream_seed(seed, k)

    def epoch_order(self, shard, seed, epoch):
        shard = np.ascontiguousarray(shard, np.uint64)
        out = np.empty_like(shard)
        self.lib.orc_epoch_order(_up(shard), shard.size, seed, epoch, _up(out))
        return out

    def worker_indices(self, n, workers, k, batch, seed, steps):
        """Indices a ShardBatchIterator emits over `steps` next() calls (data.hpp:312-351)."""
        shard = self.shard(n, workers, seed)[k]
        sseed = self.worker_stream_seed(seed, k)
        out = []
        epoch, order, cursor = 0, self.epoch_order(shard, sseed, 0), 0
        for _ in range(steps):
            if (cursor + 1) * batch > shard.size:
                epoch += 1
                order, cursor = self.epoch_order(shard, sseed, epoch), 0
            out.append(order[cursor * batch:(cursor + 1) * batch])
            cursor += 1
        return np.concatenate(out) if out else np.empty(0, np.uint64)

    def weights_mean(self, items: Sequence[np.ndarray]) -> np.ndarray:
        arrs = [np.ascontiguousarray(a, np.float64) for a in items]
        ptrs = (_D * len(arrs))(*[_dp(a) for a in arrs])
        out = np.empty_like(arrs[0])
        self.lib.orc_weights_mean(ptrs, len(arrs), arrs[0].size, _dp(out))
        return out

    def net(self, spec: NetSpec, seed: int) -> "OracleNet":
        return OracleNet(self, spec, seed)

    def run_sparknet(self, spec: NetSpec, train, evald, batch, lr, momentum, seed, workers, tau,
                     rounds, warm, threads=1, weight_decay=0.0, target=2.0, eval_steps=1,
                     cost=(1.0, 0.0), want_weights=False, skip_eval=False):
        return _run_sparknet(self.lib.orc_run_sparknet, spec, train, evald, batch, lr, momentum,
                             seed, workers, tau, rounds, warm, threads, weight_decay, target,
                             eval_steps, cost, want_weights, skip_eval,
                             lambda: self.error(), P=_param_count(self, spec, seed))

    def run_naive(self, spec: NetSpec, train, evald, batch, lr, momentum, seed, workers, iters,
                  eval_every, weight_decay=0.0, target=2.0, eval_steps=1, cost=(1.0, 0.0, 1.0),
                  want_weights=False):
        return _run_naive(self.lib.orc_run_naive, spec, train, evald, batch, lr, momentum, seed,
                          workers, iters, eval_every, weight_decay, target, eval_steps, cost,
                          want_weights, lambda: self.error(), P=_param_count(self, spec, seed))


def _run_naive(fn, spec, train, evald, batch, lr, momentum, seed, workers, iters, eval_every,
               weight_decay, target, eval_steps, cost, want_weights, err, P):
    """Shared driver of orc_run_naive / ref_run_naive: returns (records, step_weights)."""
    timg = np.ascontiguousarray(train[0], np.float64)
    tlab = np.ascontiguousarray(train[1], np.int32)
    eimg = np.ascontiguousarray(evald[0], np.float64)
    elab = np.ascontiguousarray(evald[1], np.int32)
    layers = spec.to_c()
    a = SparknetArgs()
    a.layers = layers
    a.n_layers = len(spec.layers)
    a.train_images, a.train_labels, a.train_n = _dp(timg), _ip(tlab), tlab.size
    a.eval_images, a.eval_labels, a.eval_n = _dp(eimg), _ip(elab), elab.size
    a.c, a.h, a.w = timg.shape[1], timg.shape[2], timg.shape[3]
    a.batch, a.lr, a.momentum, a.weight_decay = batch, lr, momentum, weight_decay
    a.seed = seed
    a.compute_seconds, a.sync_seconds = cost[0], cost[1]
    a.sublinearity = cost[2] if len(cost) > 2 else 1.0
    a.target_accuracy, a.eval_steps = target, eval_steps
    a.workers = workers
    nmax = max(1, (iters + eval_every - 1) // eval_every)
    recs = (Record * nmax)()
    sw = np.zeros((max(iters, 1), P), np.float64) if want_weights else None
    n = fn(ctypes.byref(a), iters, eval_every, recs, nmax, _dp(sw) if want_weights else None)
    if n < 0:
        raise RuntimeError(err())
    out = [(r.serial_iters, r.parallel_iters, r.rounds, r.sim_time, r.accuracy)
           for r in recs[:min(n, nmax)]]
    return out, (sw[:iters] if want_weights else None)


def _param_count(lib, spec, seed):
    n = lib.net(spec, seed)
    return n.P


def _run_sparknet(fn, spec, train, evald, batch, lr, momentum, seed, workers, tau, rounds, warm,
                  threads, weight_decay, target, eval_steps, cost, want_weights, skip_eval, err, P):
    timg, tlab = train
    eimg, elab = evald
    timg = np.ascontiguousarray(timg, np.float64)
    eimg = np.ascontiguousarray(eimg, np.float64)
    tlab = np.ascontiguousarray(tlab, np.int32)
    elab = np.ascontiguousarray(elab, np.int32)
    layers = spec.to_c()
    a = SparknetArgs()
    a.layers = layers
    a.n_layers = len(spec.layers)
    a.train_images, a.train_labels, a.train_n = _dp(timg), _ip(tlab), tlab.size
    a.eval_images, a.eval_labels, a.eval_n = _dp(eimg), _ip(elab), elab.size
    a.c, a.h, a.w = timg.shape[1], timg.shape[2], timg.shape[3]
    a.batch, a.lr, a.momentum, a.weight_decay = batch, lr, momentum, weight_decay
    a.seed = seed
    a.compute_seconds, a.sync_seconds = cost
    a.target_accuracy, a.eval_steps = target, eval_steps
    a.workers, a.tau, a.rounds, a.warm, a.threads = workers, tau, rounds, warm, threads
    a.skip_eval = int(skip_eval)
    recs = (Record * max(rounds, 1))()
    digest = np.zeros(1, np.uint64)
    rw = np.zeros((max(rounds, 1), P), np.float64) if want_weights else None
    n = fn(ctypes.byref(a), recs, rounds, _up(digest), _dp(rw) if want_weights else None)
    if n < 0:
        raise RuntimeError(err())
    records = [(r.serial_iters, r.parallel_iters, r.rounds, r.sim_time, r.accuracy)
               for r in recs[:n]]
    return records, int(digest[0]), (rw[:n] if want_weights else None)


class OracleNet:
    def __init__(self, lib: OracleLib, spec: NetSpec, seed: int):
        self.owner = lib
        self.L = lib.lib
        self.spec = spec
        self._layers = spec.to_c()
        self.h = self.L.orc_net_create(self._layers, len(spec.layers), seed)
        if not self.h:
            raise ValueError(lib.error())
        self.P = self.L.orc_net_param_count(self.h)
        self.classes = self.L.orc_net_num_classes(self.h)

    def __del__(self):
        if getattr(self, "h", None):
            self.L.orc_net_destroy(self.h)
            self.h = None

    def _check(self, rc):
        if rc == 1:
            raise ValueError(self.owner.error())
        if rc:
            raise RuntimeError(self.owner.error())

    def get_weights(self):
        out = np.empty(self.P, np.float64)
        self.L.orc_net_get_weights(self.h, _dp(out))
        return out

    def set_weights(self, w):
        w = np.ascontiguousarray(w, np.float64)
        assert w.size == self.P
        self.L.orc_net_set_weights(self.h, _dp(w))

    def get_velocity(self):
        out = np.empty(self.P, np.float64)
        self.L.orc_net_get_velocity(self.h, _dp(out))
        return out

    def set_sgd(self, lr, momentum=0.0, weight_decay=0.0):
        self.L.orc_net_set_sgd(self.h, lr, momentum, weight_decay)

    def set_dropout_step(self, step):
        self.L.orc_net_set_dropout_step(self.h, step)

    def forward(self, images, labels, train=False):
        images = np.ascontiguousarray(images, np.float64)
        labels = np.ascontiguousarray(labels, np.int32)
        loss = ctypes.c_double()
        probs = np.empty((labels.size, self.classes), np.float64)
        self._check(self.L.orc_net_forward(self.h, _dp(images), _ip(labels), labels.size,
                                           int(train), ctypes.byref(loss), _dp(probs)))
        return loss.value, probs

    def backward(self, images, labels):
        images = np.ascontiguousarray(images, np.float64)
        labels = np.ascontiguousarray(labels, np.int32)
        loss = ctypes.c_double()
        grads = np.empty(self.P, np.float64)
        self._check(self.L.orc_net_backward(self.h, _dp(images), _ip(labels), labels.size,
                                            ctypes.byref(loss), _dp(grads)))
        return loss.value, grads

    def apply_update(self, grads):
        grads = np.ascontiguousarray(grads, np.float64)
        self._check(self.L.orc_net_apply_update(self.h, _dp(grads)))

    def layer_dims(self, li):
        d = (ctypes.c_int64 * 3)()
        self.L.orc_net_layer_dims(self.h, li, d)
        return tuple(d)

    def layer_out(self, li, n):
        c, h, w = self.layer_dims(li)
        p = self.L.orc_net_layer_out(self.h, li)
        return np.ctypeslib.as_array(p, shape=(n * c * h * w,)).copy().reshape(n, c, h, w)

    def layer_grad(self, li, n):
        c, h, w = self.layer_dims(li)
        p = self.L.orc_net_layer_grad(self.h, li)
        return np.ctypeslib.as_array(p, shape=(n * c * h * w,)).copy().reshape(n, c, h, w)

    def layer_params(self, li):
        off, cnt = ctypes.c_size_t(), ctypes.c_size_t()
        self.L.orc_net_layer_params(self.h, li, ctypes.byref(off), ctypes.byref(cnt))
        return off.value, cnt.value

    def layer_forward(self, li, n, inputs):
        arrs = [np.ascontiguousarray(a, np.float64) for a in inputs]
        ptrs = (_D * len(arrs))(*[_dp(a) for a in arrs])
        c, h, w = self.layer_dims(li)
        out = np.empty((n, c, h, w), np.float64)
        self._check(self.L.orc_layer_forward(self.h, li, n, ptrs, _dp(out)))
        return out

    def layer_backward(self, li, n, dy, want_dx=True):
        dy = np.ascontiguousarray(dy, np.float64)
        src = self.spec.index_of(self.spec.layers[li].inputs[0])
        c, h, w = self.layer_dims(src)
        dx = np.empty((n, c, h, w), np.float64) if want_dx else None
        _, cnt = self.layer_params(li)
        dp = np.empty(max(cnt, 1), np.float64)
        self._check(self.L.orc_layer_backward(self.h, li, n, _dp(dy),
                                              _dp(dx) if want_dx else None, _dp(dp)))
        return dx, dp[:cnt]

    def digest(self, flat=None):
        flat = self.get_weights() if flat is None else np.ascontiguousarray(flat, np.float64)
        return self.L.orc_weights_digest(self.h, _dp(flat))


class RefLib(_Lib):
    """The unmodified reference compiled in place (oracle/_ref)."""

    def __init__(self, strict: bool = True, path: Optional[str] = None):
        name = "libparasgd_ref_strict.so" if strict else "libparasgd_ref.so"
        super().__init__(path or os.path.join(HERE, "_ref", name))
        L = self.lib
        L.ref_last_error.restype = ctypes.c_char_p
        L.ref_net_create.restype = ctypes.c_void_p
        L.ref_net_create.argtypes = [ctypes.POINTER(CLayerDesc), ctypes.c_int, ctypes.c_uint64]
        L.ref_net_destroy.argtypes = [ctypes.c_void_p]
        L.ref_net_param_count.restype = ctypes.c_size_t
        L.ref_net_param_count.argtypes = [ctypes.c_void_p]
        L.ref_net_set_sgd.argtypes = [ctypes.c_void_p, ctypes.c_double, ctypes.c_double]
        L.ref_net_get_weights.argtypes = [ctypes.c_void_p, _D]
        L.ref_net_set_weights.argtypes = [ctypes.c_void_p, _D]
        L.ref_net_forward.argtypes = [ctypes.c_void_p, _D, _I32, ctypes.c_size_t, _D, _D]
        L.ref_net_backward.argtypes = [ctypes.c_void_p, _D, _I32, ctypes.c_size_t, _D, _D]
        L.ref_net_apply_update.argtypes = [ctypes.c_void_p, _D]
        L.ref_net_layer_size.restype = ctypes.c_size_t
        L.ref_net_layer_size.argtypes = [ctypes.c_void_p, ctypes.c_int]
        L.ref_net_layer_out.argtypes = [ctypes.c_void_p, ctypes.c_int, _D]
        L.ref_net_layer_grad.argtypes = [ctypes.c_void_p, ctypes.c_int, _D]
        L.ref_shard.argtypes = [ctypes.c_size_t, ctypes.c_int, ctypes.c_uint64, _U64, _U64]
        L.ref_worker_indices.argtypes = [ctypes.c_size_t, ctypes.c_int, ctypes.c_int,
                                         ctypes.c_size_t, ctypes.c_uint64, ctypes.c_long, _U64]
        L.ref_generate_synthetic.argtypes = [ctypes.c_int, ctypes.c_size_t, ctypes.c_size_t,
                                             ctypes.c_size_t, ctypes.c_size_t, ctypes.c_double,
                                             ctypes.c_uint64, ctypes.c_uint64, _D, _I32]
        L.ref_weights_mean.argtypes = [ctypes.POINTER(_D), ctypes.c_int, ctypes.c_size_t, _D]
        L.ref_net_digest.restype = ctypes.c_uint64
        L.ref_net_digest.argtypes = [ctypes.c_void_p]
        L.ref_format_double.restype = ctypes.c_int
        L.ref_format_double.argtypes = [ctypes.c_double, ctypes.c_char_p, ctypes.c_int]
        L.ref_naive_speedup.restype = ctypes.c_double
        L.ref_naive_speedup.argtypes = [ctypes.c_double, ctypes.c_int, ctypes.c_double]
        L.ref_sparknet_speedup.restype = ctypes.c_double
        L.ref_sparknet_speedup.argtypes = [ctypes.c_double] * 5
        L.ref_run_naive.restype = ctypes.c_long
        L.ref_run_naive.argtypes = [ctypes.POINTER(SparknetArgs), ctypes.c_long, ctypes.c_long,
                                    ctypes.POINTER(Record), ctypes.c_long, _D]
        L.ref_run_sparknet.restype = ctypes.c_long
        L.ref_run_sparknet.argtypes = [ctypes.POINTER(SparknetArgs), ctypes.POINTER(Record),
                                       ctypes.c_long, _U64, _D]

    def error(self) -> str:
        return self.lib.ref_last_error().decode()

    def generate_synthetic(self, classes, c, h, w, per_class, separation, seed, variant=0):
        n = classes * per_class
        images = np.empty((n, c, h, w), np.float64)
        labels = np.empty(n, np.int32)
        self.lib.ref_generate_synthetic(classes, c, h, w, per_class, separation, seed, variant,
                                        _dp(images), _ip(labels))
        return images, labels

    def shard(self, n, workers, seed):
        perm = np.empty(n, np.uint64)
        offs = np.empty(workers + 1, np.uint64)
        if self.lib.ref_shard(n, workers, seed, _up(perm), _up(offs)):
            raise ValueError(self.error())
        return [perm[offs[k]:offs[k + 1]].copy() for k in range(workers)]

    def worker_indices(self, n, workers, k, batch, seed, steps):
        out = np.empty(steps * batch, np.uint64)
        if self.lib.ref_worker_indices(n, workers, k, batch, seed, steps, _up(out)):
            raise ValueError(self.error())
        return out

    def weights_mean(self, items):
        arrs = [np.ascontiguousarray(a, np.float64) for a in items]
        ptrs = (_D * len(arrs))(*[_dp(a) for a in arrs])
        out = np.empty_like(arrs[0])
        self.lib.ref_weights_mean(ptrs, len(arrs), arrs[0].size, _dp(out))
        return out

    def net(self, spec: NetSpec, seed: int) -> "RefNet":
        return RefNet(self, spec, seed)

    def run_sparknet(self, spec, train, evald, batch, lr, momentum, seed, workers, tau, rounds,
                     warm, threads=1, target=2.0, eval_steps=1, cost=(1.0, 0.0),
                     want_weights=False):
        P = RefNet(self, spec, seed).P
        return _run_sparknet(self.lib.ref_run_sparknet, spec, train, evald, batch, lr, momentum,
                             seed, workers, tau, rounds, warm, threads, 0.0, target, eval_steps,
                             cost, want_weights, False, lambda: self.error(), P=P)

    def format_double(self, v: float) -> str:
        buf = ctypes.create_string_buffer(64)
        if self.lib.ref_format_double(v, buf, 64) < 0:
            raise RuntimeError("format_double: buffer")
        return buf.value.decode()

    def naive_speedup(self, c, k, s):
        return self.lib.ref_naive_speedup(c, k, s)

    def sparknet_speedup(self, n, c, tau, s, m):
        return self.lib.ref_sparknet_speedup(n, c, tau, s, m)

    def run_naive(self, spec, train, evald, batch, lr, momentum, seed, workers, iters, eval_every,
                  target=2.0, eval_steps=1, cost=(1.0, 0.0, 1.0), want_weights=False):
        P = RefNet(self, spec, seed).P
        return _run_naive(self.lib.ref_run_naive, spec, train, evald, batch, lr, momentum, seed,
                          workers, iters, eval_every, 0.0, target, eval_steps, cost, want_weights,
                          lambda: self.error(), P=P)


class RefNet:
    def __init__(self, lib: RefLib, spec: NetSpec, seed: int):
        self.owner = lib
        self.L = lib.lib
        self.spec = spec
        self._layers = spec.to_c()
        self.h = self.L.ref_net_create(self._layers, len(spec.layers), seed)
        if not self.h:
            raise ValueError(lib.error())
        self.P = self.L.ref_net_param_count(self.h)
        self.classes = None

    def __del__(self):
        if getattr(self, "h", None):
            self.L.ref_net_destroy(self.h)
            self.h = None

    def _check(self, rc):
        if rc == 1:
            raise ValueError(self.owner.error())
        if rc:
            raise RuntimeError(self.owner.error())

    def set_sgd(self, lr, momentum=0.0):
        self._check(self.L.ref_net_set_sgd(self.h, lr, momentum))

    def get_weights(self):
        out = np.empty(self.P, np.float64)
        self.L.ref_net_get_weights(self.h, _dp(out))
        return out

    def set_weights(self, w):
        w = np.ascontiguousarray(w, np.float64)
        self._check(self.L.ref_net_set_weights(self.h, _dp(w)))

    def forward(self, images, labels, classes):
        images = np.ascontiguousarray(images, np.float64)
        labels = np.ascontiguousarray(labels, np.int32)
        loss = ctypes.c_double()
        probs = np.empty((labels.size, classes), np.float64)
        self._check(self.L.ref_net_forward(self.h, _dp(images), _ip(labels), labels.size,
                                           ctypes.byref(loss), _dp(probs)))
        return loss.value, probs

    def backward(self, images, labels):
        images = np.ascontiguousarray(images, np.float64)
        labels = np.ascontiguousarray(labels, np.int32)
        loss = ctypes.c_double()
        grads = np.empty(self.P, np.float64)
        self._check(self.L.ref_net_backward(self.h, _dp(images), _ip(labels), labels.size,
                                            ctypes.byref(loss), _dp(grads)))
        return loss.value, grads

    def apply_update(self, grads):
        grads = np.ascontiguousarray(grads, np.float64)
        self._check(self.L.ref_net_apply_update(self.h, _dp(grads)))

    def layer_out(self, li):
        n = self.L.ref_net_layer_size(self.h, li)
        out = np.empty(n, np.float64)
        self._check(self.L.ref_net_layer_out(self.h, li, _dp(out)))
        return out

    def layer_grad(self, li):
        n = self.L.ref_net_layer_size(self.h, li)
        out = np.empty(n, np.float64)
        self._check(self.L.ref_net_layer_grad(self.h, li, _dp(out)))
        return out

    def digest(self):
        return self.L.ref_net_digest(self.h)


def max_relative_deviation(got: np.ndarray, want: np.ndarray, segments=None) -> float:
    """test_helpers.hpp:77-91: per-tensor max |a-b| / max(1e-12, max|b|).

    ``segments`` = list of (offset, count) tensors inside flat vectors; None = one tensor."""
    got = np.asarray(got, np.float64).ravel()
    want = np.asarray(want, np.float64).ravel()
    if segments is None:
        segments = [(0, want.size)]
    worst = 0.0
    for off, cnt in segments:
        b = want[off:off + cnt]
        a = got[off:off + cnt]
        if cnt == 0:
            continue
        scale = max(1e-12, float(np.max(np.abs(b))))
        worst = max(worst, float(np.max(np.abs(a - b))) / scale)
    return worst
