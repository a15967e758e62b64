"""class Net on a B200 — host mirror of model.hpp:50-171 over the C ABI.

Same names, argument meaning and error behaviour as the reference: ValueError for
std::invalid_argument, RuntimeError for std::runtime_error (non-finite values, missing
data).  CamelCase aliases of SparkNet's Scala API (setTrainingData, getWeights, ...) are
provided alongside.
"""
from __future__ import annotations

import ctypes
from dataclasses import dataclass
from typing import Optional

import numpy as np

from . import _lib
from .data import SequentialBatchIterator, ShardBatchIterator
from .netspec import NetSpec
from .weights import WeightCollection


@dataclass
class Batch:
    """batch.hpp:11-16: images [n, c, h, w] + labels."""
    images: np.ndarray
    labels: np.ndarray

    def size(self) -> int:
        return int(np.asarray(self.labels).size)


@dataclass
class ForwardResult:
    """model.hpp:18-21."""
    loss: float
    probabilities: np.ndarray


@dataclass
class SgdOptions:
    """model.hpp:23-26 (+ weight decay extension; 0 reproduces the reference)."""
    learning_rate: float = 0.01
    momentum: float = 0.0
    weight_decay: float = 0.0


class Context:
    """One CUDA device + stream (psg_ctx)."""
    _cache = {}

    def __init__(self, device: int = 0):
        self.device = device
        h = ctypes.c_void_p()
        _lib.call("psg_ctx_create", device, ctypes.byref(h))
        self.handle = h

    @classmethod
    def get(cls, device: int = 0) -> "Context":
        if device not in cls._cache:
            cls._cache[device] = cls(device)
        return cls._cache[device]

    def sync(self) -> None:
        _lib.call("psg_ctx_sync", self.handle)


def device_count() -> int:
    n = ctypes.c_int()
    _lib.call("psg_device_count", ctypes.byref(n))
    return n.value


class Net:
    """A trainable realisation of a NetSpec on one GPU (model.hpp:50)."""

    def __init__(self, spec: NetSpec, seed: int, device: int = 0, precision: str = "fp32",
                 fuse: bool = True, tc_pair: str = "auto"):
        """fuse: ReLU fusion (psg_net_set_fusion; bitwise-identical results).  Pass False
        to read every layer's pre-activation output / gradient (per-layer parity tests).
        tc_pair: tcgen05 CTA-pair policy of the TF32 GEMMs ("auto" | "never" | "always",
        psg_net_set_tc_options) — the parity tests force each kernel variant."""
        spec.validate()
        self._spec = spec
        self._seed = seed
        self.ctx = Context.get(device)
        self._layers = spec.to_c()
        h = ctypes.c_void_p()
        _lib.call("psg_net_create", self.ctx.handle, self._layers, len(spec.layers), seed,
                  ctypes.byref(h))
        self.handle = h
        n = ctypes.c_size_t()
        _lib.call("psg_net_param_count", h, ctypes.byref(n))
        self.P = n.value
        c = ctypes.c_int()
        _lib.call("psg_net_num_classes", h, ctypes.byref(c))
        self._classes = c.value
        self._sgd = SgdOptions()
        self._train_it: Optional[ShardBatchIterator] = None
        self._attached = None
        self._part = (0, 1)
        self._val_it: Optional[SequentialBatchIterator] = None
        self._structure = self._read_structure()
        self.set_precision(precision)
        if not fuse:
            _lib.call("psg_net_set_fusion", h, 0)
        if tc_pair != "auto":
            self.set_tc_options(tc_pair)

    def __del__(self):
        h = getattr(self, "handle", None)
        if h:
            try:
                _lib.lib().psg_net_destroy(h)
            except Exception:
                pass
            self.handle = None

    # --- structure -----------------------------------------------------------
    def _read_structure(self):
        nt = ctypes.c_int()
        _lib.call("psg_net_num_tensors", self.handle, ctypes.byref(nt))
        by_layer = {}
        for t in range(nt.value):
            layer, slot, rank = ctypes.c_int(), ctypes.c_int(), ctypes.c_int()
            shape = (ctypes.c_int64 * 4)()
            off = ctypes.c_size_t()
            _lib.call("psg_net_tensor_info", self.handle, t, ctypes.byref(layer),
                      ctypes.byref(slot), ctypes.byref(rank), shape, ctypes.byref(off))
            by_layer.setdefault(layer.value, []).append(
                (off.value, tuple(shape[i] for i in range(rank.value))))
        return [(l.name, by_layer.get(i, [])) for i, l in enumerate(self._spec.layers)]

    def segments(self):
        """(offset, count) of every tensor in the flat WeightCollection order."""
        return [(off, int(np.prod(shape))) for _, ts in self._structure for off, shape in ts]

    def spec(self) -> NetSpec:
        return self._spec

    def num_classes(self) -> int:
        return self._classes

    def sgd(self) -> SgdOptions:
        return self._sgd

    def set_sgd(self, opts: SgdOptions) -> None:
        _lib.call("psg_net_set_sgd", self.handle, opts.learning_rate, opts.momentum,
                  opts.weight_decay)
        self._sgd = opts

    def set_precision(self, precision: str) -> None:
        mode = {"fp32": _lib.PRECISION_FP32, "tf32": _lib.PRECISION_TF32}[precision]
        _lib.call("psg_net_set_precision", self.handle, mode)
        self.precision = precision

    def set_tc_options(self, pair: str = "auto") -> None:
        if pair not in _lib.TC_PAIR:
            raise ValueError("set_tc_options: unknown pair policy")
        _lib.call("psg_net_set_tc_options", self.handle, _lib.TC_PAIR[pair])
        self.tc_pair = pair

    # --- weights (model.hpp:138-171) ----------------------------------------
    def get_weights_flat(self) -> np.ndarray:
        out = np.empty(self.P, np.float64)
        _lib.call("psg_net_get_weights_f64", self.handle, out.ctypes.data_as(_lib._D), self.P)
        return out

    def set_weights_flat(self, flat: np.ndarray) -> None:
        flat = np.ascontiguousarray(flat, np.float64)
        _lib.call("psg_net_set_weights_f64", self.handle, flat.ctypes.data_as(_lib._D), flat.size)

    def get_velocity_flat(self) -> np.ndarray:
        out = np.empty(self.P, np.float64)
        _lib.call("psg_net_get_velocity_f64", self.handle, out.ctypes.data_as(_lib._D), self.P)
        return out

    def reset_velocity(self) -> None:
        _lib.call("psg_net_reset_velocity", self.handle)

    def _to_collection(self, flat: np.ndarray) -> WeightCollection:
        w = WeightCollection()
        for name, ts in self._structure:
            w.add(name, [flat[off:off + int(np.prod(shape))].reshape(shape) for off, shape in ts])
        return w

    def _from_collection(self, w: WeightCollection, what: str) -> np.ndarray:
        if w.size() != len(self._structure):
            raise ValueError(f"{what}: expected {len(self._structure)} entries, got {w.size()}")
        flat = np.empty(self.P, np.float64)
        for name, ts in self._structure:
            tensors = w.find(name)
            if tensors is None:
                raise ValueError(f"{what}: missing layer key '{name}'")
            if len(tensors) != len(ts):
                raise ValueError(f"{what}: tensor count mismatch at '{name}'")
            for t, (off, shape) in zip(tensors, ts):
                if tuple(t.shape) != tuple(shape):
                    raise ValueError(f"{what}: shape mismatch at '{name}'")
                flat[off:off + t.size] = t.ravel()
        return flat

    def get_weights(self) -> WeightCollection:
        return self._to_collection(self.get_weights_flat())

    def set_weights(self, w: WeightCollection) -> None:
        self.set_weights_flat(self._from_collection(w, "set_weights"))

    # --- compute -------------------------------------------------------------
    def _batch_args(self, batch: Batch):
        images = np.ascontiguousarray(batch.images, np.float64)
        labels = np.ascontiguousarray(batch.labels, np.int32)
        d = self._spec.data_spec().shape
        if images.ndim != 4:
            raise ValueError("forward: images must be [n,c,h,w]")
        if labels.size < 1 or images.shape[0] != labels.size:
            raise ValueError("forward: label count does not match batch")
        if tuple(images.shape[1:]) != tuple(d[1:]):
            raise ValueError("forward: batch extents do not match the data layer")
        return images, labels

    def forward(self, batch: Batch) -> ForwardResult:
        """model.hpp:74-78 (test phase: dropout is the identity)."""
        images, labels = self._batch_args(batch)
        loss = ctypes.c_double()
        probs = np.empty((labels.size, self._classes), np.float64)
        _lib.call("psg_net_forward", self.handle, images.ctypes.data_as(_lib._D),
                  labels.ctypes.data_as(_lib._I32), labels.size, ctypes.byref(loss),
                  probs.ctypes.data_as(_lib._D))
        return ForwardResult(loss.value, probs)

    def backward_flat(self, batch: Batch):
        images, labels = self._batch_args(batch)
        loss = ctypes.c_double()
        grads = np.empty(self.P, np.float64)
        _lib.call("psg_net_backward", self.handle, images.ctypes.data_as(_lib._D),
                  labels.ctypes.data_as(_lib._I32), labels.size, ctypes.byref(loss),
                  grads.ctypes.data_as(_lib._D))
        return loss.value, grads

    def backward(self, batch: Batch) -> WeightCollection:
        """model.hpp:83-86."""
        return self._to_collection(self.backward_flat(batch)[1])

    def apply_update_flat(self, grads: np.ndarray) -> None:
        g = np.ascontiguousarray(grads, np.float64)
        _lib.call("psg_net_apply_update", self.handle, g.ctypes.data_as(_lib._D), g.size)

    def apply_update(self, grads: WeightCollection) -> None:
        """model.hpp:90-107."""
        self.apply_update_flat(self._from_collection(grads, "apply_update"))

    def layer_output(self, layer: int) -> np.ndarray:
        return self._layer_state(layer, "psg_net_layer_output")

    def layer_grad(self, layer: int) -> np.ndarray:
        return self._layer_state(layer, "psg_net_layer_grad")

    def _layer_state(self, layer, fn):
        shape = (ctypes.c_int64 * 4)()
        _lib.call("psg_net_layer_shape", self.handle, layer, shape)
        shp = tuple(shape)
        out = np.empty(shp, np.float64)
        _lib.call(fn, self.handle, layer, out.ctypes.data_as(_lib._D), out.size)
        return out

    # --- data streams (model.hpp:68-69) -------------------------------------
    def set_training_data(self, it: ShardBatchIterator) -> None:
        self._train_it = it
        self._part = (0, 1)
        self._attached = None

    def set_training_part(self, it: ShardBatchIterator, part: int, parts: int) -> None:
        """run_naive (schemes.hpp:233-247): this net trains on rows
        [part*b/parts, (part+1)*b/parts) of every batch the iterator yields."""
        if parts < 1 or not 0 <= part < parts:
            raise ValueError("attach: part index out of range")
        if it.batch_size % parts:
            raise ValueError("run_naive: worker count must divide the batch size")
        self._train_it = it
        self._part = (part, parts)
        self._attached = None

    def set_validation_data(self, it: SequentialBatchIterator) -> None:
        self._val_it = it
        _lib.call("psg_net_attach_validation", self.handle, it.dataset.handle(self.ctx),
                  it.batch_size)

    def _sync_stream_in(self) -> None:
        it = self._train_it
        if self._attached is not it:
            idx = np.ascontiguousarray(it.shard.indices, np.uint64)
            _lib.call("psg_net_attach_shard_part", self.handle,
                      it.shard.dataset.handle(self.ctx), idx.ctypes.data_as(_lib._U64),
                      idx.size, it.batch_size, it.seed, self._part[0], self._part[1])
            self._attached = it
        _lib.call("psg_net_set_stream_position", self.handle, it._epoch, it._cursor)

    def _sync_stream_out(self) -> None:
        it = self._train_it
        e, c = ctypes.c_uint64(), ctypes.c_uint64()
        _lib.call("psg_net_get_stream_position", self.handle, ctypes.byref(e), ctypes.byref(c))
        if e.value != it._epoch:
            from .data import epoch_order
            it._order = epoch_order(it.shard.indices, it.seed, e.value)
        it._epoch, it._cursor = e.value, c.value

    def train(self, num_steps: int, sync: bool = True) -> None:
        """model.hpp:111-118: num_steps SGD updates on consecutive attached batches.
        The steps run as replays of one CUDA graph; sync=False returns once enqueued."""
        if num_steps < 0:
            raise ValueError("train: negative step count")
        if num_steps > 0 and self._train_it is None:
            raise RuntimeError("train: no training data attached")
        if num_steps == 0:
            return
        self._sync_stream_in()
        _lib.call("psg_net_train", self.handle, num_steps)
        self._sync_stream_out()
        if sync:
            self.sync()

    def train_round(self, num_steps: int, comm, sync: bool = True) -> None:
        """One SparkNet round of this worker: train(num_steps) + the fast K-way weight
        average over `comm`, the average overlapped with the last step's backward
        (psg_net_train_round)."""
        if num_steps < 1:
            raise ValueError("train_round: tau must be >= 1")
        if self._train_it is None:
            raise RuntimeError("train: no training data attached")
        self._sync_stream_in()
        _lib.call("psg_net_train_round", self.handle, num_steps, comm.handle)
        self._sync_stream_out()
        if sync:
            self.sync()

    def grad_step(self) -> None:
        """One run_naive part (schemes.hpp:233-247): next batch (this net's rows) ->
        forward + backward; the gradient stays on the device (enqueued, no sync)."""
        if self._train_it is None:
            raise RuntimeError("train: no training data attached")
        self._sync_stream_in()
        _lib.call("psg_net_grad_step", self.handle)
        self._sync_stream_out()

    def apply_grads(self) -> None:
        """apply_update (model.hpp:90-107) with the device-resident gradient."""
        _lib.call("psg_net_apply_grads", self.handle)

    def sync(self) -> None:
        """Wait for queued work; raises RuntimeError if a non-finite value appeared."""
        _lib.call("psg_net_sync", self.handle)

    def last_train_ms(self) -> float:
        ms = ctypes.c_float()
        _lib.call("psg_net_last_train_ms", self.handle, ctypes.byref(ms))
        return ms.value

    def last_loss(self) -> float:
        v = ctypes.c_double()
        _lib.call("psg_net_last_loss", self.handle, ctypes.byref(v))
        return v.value

    def train_host(self, images: np.ndarray, labels: np.ndarray) -> np.ndarray:
        """End-to-end path: steps = images.shape[0]; per step an H2D copy of that step's
        batch (NCHW fp32, pinned if allocated with _lib.PinnedArray), the step, and a D2H
        read of its loss.  Returns the per-step losses."""
        steps = images.shape[0]
        assert images.dtype == np.float32 and images.flags.c_contiguous
        assert labels.dtype == np.int32 and labels.flags.c_contiguous
        losses = np.empty(steps, np.float64)
        _lib.call("psg_net_train_host", self.handle, images.ctypes.data_as(_lib._F),
                  labels.ctypes.data_as(_lib._I32), steps, losses.ctypes.data_as(_lib._D))
        return losses

    def train_host_rows(self, images: np.ndarray, labels: np.ndarray, rows: np.ndarray,
                        threads: int = 8) -> np.ndarray:
        """End-to-end path with a host loader: steps = rows.size // b; per step `threads`
        host threads gather rows `rows[s*b:(s+1)*b]` of the host dataset (NCHW fp32,
        int32 labels) into pinned staging while the GPU runs the previous step, then the
        H2D copy, the step and a D2H read of its loss.  Returns the per-step losses."""
        assert images.dtype == np.float32 and images.flags.c_contiguous
        assert labels.dtype == np.int32 and labels.flags.c_contiguous
        rows = np.ascontiguousarray(rows, np.uint64)
        b = self._spec.data_spec().shape[0]
        steps = rows.size // b
        losses = np.empty(steps, np.float64)
        _lib.call("psg_net_train_host_rows", self.handle, images.ctypes.data_as(_lib._F),
                  labels.ctypes.data_as(_lib._I32), images.shape[0],
                  rows.ctypes.data_as(_lib._U64), steps, losses.ctypes.data_as(_lib._D),
                  threads)
        return losses

    def profile_step(self, repeats: int = 5):
        """Per-op CUDA-event times of one training step (list of dicts)."""
        cap = 512
        arr = (_lib.OpTime * cap)()
        n = ctypes.c_int()
        _lib.call("psg_net_profile_step", self.handle, repeats, arr, cap, ctypes.byref(n))
        return [dict(name=a.name.decode(), layer=a.layer, phase=_lib.PHASES[a.phase],
                     flops=a.flops, bytes=a.bytes, ms=a.ms, launches=a.launches)
                for a in arr[:min(n.value, cap)]]

    def event_record(self, slot: int) -> None:
        _lib.call("psg_net_event_record", self.handle, slot)

    def event_elapsed(self, a: int, b: int) -> float:
        ms = ctypes.c_float()
        _lib.call("psg_net_event_elapsed", self.handle, a, b, ctypes.byref(ms))
        return ms.value

    def kernels_per_step(self) -> int:
        v = ctypes.c_int()
        _lib.call("psg_net_kernels_per_step", self.handle, ctypes.byref(v))
        return v.value

    def test(self, num_steps: int) -> float:
        """model.hpp:122-136: argmax accuracy over num_steps validation batches."""
        if num_steps < 1:
            raise ValueError("test: step count must be >= 1")
        if self._val_it is None:
            raise RuntimeError("test: no validation data attached")
        acc = ctypes.c_double()
        _lib.call("psg_net_test", self.handle, num_steps, ctypes.byref(acc))
        return acc.value

    def test_begin(self, num_steps: int, first: int, stride: int) -> None:
        """Sharded test: queue batches first, first+stride, ... of the next num_steps."""
        if self._val_it is None:
            raise RuntimeError("test: no validation data attached")
        _lib.call("psg_net_test_begin", self.handle, num_steps, first, stride)

    def test_end(self):
        """(correct, total) of the evaluation queued by test_begin."""
        c, t = ctypes.c_ulonglong(), ctypes.c_ulonglong()
        _lib.call("psg_net_test_end", self.handle, ctypes.byref(c), ctypes.byref(t))
        return c.value, t.value

    # SparkNet (Scala) spellings
    setTrainingData = set_training_data
    setValidationData = set_validation_data
    getWeights = get_weights
    setWeights = set_weights
