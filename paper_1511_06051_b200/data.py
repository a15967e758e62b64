"""Datasets, shards and batch iterators — host mirror of data.hpp.

Integer work (the shard permutation, per-epoch orders) runs in libpsg's host code and is
bit-exact with the reference (data.hpp:261-351); pixels are uploaded to HBM once and
minibatches are gathered on the device, so they never return to the host.
"""
from __future__ import annotations

import ctypes
from dataclasses import dataclass, field
from typing import Dict, List, Optional

import numpy as np

from . import _lib


def generate_synthetic(num_classes: int, c: int, h: int, w: int, per_class: int,
                       separation: float, seed: int, variant: int = 0):
    """data.hpp:111-155 (host, fp64, bit-exact).  Returns (images [n,c,h,w], labels)."""
    n = num_classes * per_class
    images = np.empty((n, c, h, w), np.float64)
    labels = np.empty(n, np.int32)
    _lib.call("psg_generate_synthetic", num_classes, c, h, w, per_class, separation, seed,
              variant, images.ctypes.data_as(_lib._D), labels.ctypes.data_as(_lib._I32))
    return images, labels


class Dataset:
    """data.hpp:21-41: images [n,c,h,w] + labels; uploaded lazily to each device used."""

    def __init__(self, images: np.ndarray, labels: np.ndarray, num_classes: int):
        images = np.asarray(images)
        labels = np.ascontiguousarray(labels, np.int32)
        if labels.size == 0:
            raise ValueError("dataset: empty")
        if images.ndim != 4 or images.shape[0] != labels.size:
            raise ValueError("dataset: images/labels mismatch")
        if num_classes < 1:
            raise ValueError("dataset: no classes")
        if labels.min() < 0 or labels.max() >= num_classes:
            raise ValueError("dataset: label out of range")
        self.images = images
        self.labels = labels
        self.num_classes = num_classes
        self._device: Dict[int, ctypes.c_void_p] = {}

    @classmethod
    def synthetic(cls, num_classes, c, h, w, per_class, separation, seed, variant=0):
        img, lab = generate_synthetic(num_classes, c, h, w, per_class, separation, seed, variant)
        return cls(img, lab, num_classes)

    def size(self) -> int:
        return int(self.labels.size)

    def channels(self) -> int:
        return int(self.images.shape[1])

    def height(self) -> int:
        return int(self.images.shape[2])

    def width(self) -> int:
        return int(self.images.shape[3])

    def handle(self, ctx) -> ctypes.c_void_p:
        """Device-resident copy on ctx's GPU (uploaded once)."""
        if ctx.device not in self._device:
            out = ctypes.c_void_p()
            n, c, h, w = self.images.shape
            if self.images.dtype == np.float32:
                img = np.ascontiguousarray(self.images)
                _lib.call("psg_dataset_upload_f32", ctx.handle, img.ctypes.data_as(_lib._F),
                          self.labels.ctypes.data_as(_lib._I32), n, c, h, w, self.num_classes,
                          ctypes.byref(out))
            else:
                img = np.ascontiguousarray(self.images, np.float64)
                _lib.call("psg_dataset_upload_f64", ctx.handle, img.ctypes.data_as(_lib._D),
                          self.labels.ctypes.data_as(_lib._I32), n, c, h, w, self.num_classes,
                          ctypes.byref(out))
            self._device[ctx.device] = (out, ctx)
        return self._device[ctx.device][0]

    def release(self) -> None:
        for handle, _ in self._device.values():
            _lib.lib().psg_dataset_destroy(handle)
        self._device.clear()

    def __del__(self):
        try:
            self.release()
        except Exception:
            pass


def load_idx(images_path: str, labels_path: str) -> Dataset:
    """data.hpp:173-208: IDX pair (u8 payload, big-endian header), pixels p/255."""
    n, h, w, k = ctypes.c_size_t(), ctypes.c_int(), ctypes.c_int(), ctypes.c_int()
    ip, lp = images_path.encode(), labels_path.encode()
    _lib.call("psg_read_idx", ip, lp, ctypes.byref(n), ctypes.byref(h), ctypes.byref(w),
              ctypes.byref(k), None, None)
    img = np.empty((n.value, 1, h.value, w.value), np.float32)
    lab = np.empty(n.value, np.int32)
    _lib.call("psg_read_idx", ip, lp, ctypes.byref(n), ctypes.byref(h), ctypes.byref(w),
              ctypes.byref(k), img.ctypes.data_as(_lib._F), lab.ctypes.data_as(_lib._I32))
    return Dataset(img, lab, k.value)


def load_csv(path: str, c: int, h: int, w: int, num_classes: int) -> Dataset:
    """data.hpp:213-255: header-less `label,p0,p1,...` rows, pixels p/255."""
    n = ctypes.c_size_t()
    _lib.call("psg_read_csv", path.encode(), c, h, w, num_classes, ctypes.byref(n), None, None)
    img = np.empty((n.value, c, h, w), np.float32)
    lab = np.empty(n.value, np.int32)
    _lib.call("psg_read_csv", path.encode(), c, h, w, num_classes, ctypes.byref(n),
              img.ctypes.data_as(_lib._F), lab.ctypes.data_as(_lib._I32))
    return Dataset(img, lab, num_classes)


class DeviceSyntheticDataset(Dataset):
    """generate_synthetic's distribution generated directly in HBM:
    bit-exact class means, counter-based within-class noise (same law, not the reference's
    serial stream).  Host-side only the labels exist (row // per_class)."""

    def __init__(self, num_classes: int, c: int, h: int, w: int, per_class: int,
                 separation: float, seed: int, variant: int = 0, label_classes: int = 0):
        if num_classes < 1 or per_class < 1:
            raise ValueError("synthetic: need at least one class and example")
        self.gen = (num_classes, c, h, w, per_class, float(separation), seed, variant)
        self.shape = (num_classes * per_class, c, h, w)
        self.labels = (np.arange(self.shape[0]) // per_class).astype(np.int32)
        self.num_classes = max(num_classes, label_classes)
        self._device = {}

    @property
    def images(self):
        raise AttributeError("DeviceSyntheticDataset: pixels live on the device; use read()")

    def channels(self) -> int:
        return self.shape[1]

    def height(self) -> int:
        return self.shape[2]

    def width(self) -> int:
        return self.shape[3]

    def handle(self, ctx) -> ctypes.c_void_p:
        if ctx.device not in self._device:
            out = ctypes.c_void_p()
            k, c, h, w, per, sep, seed, var = self.gen
            _lib.call("psg_dataset_synthetic_device", ctx.handle, k, c, h, w, per, sep, seed, var,
                      ctypes.byref(out))
            self._device[ctx.device] = (out, ctx)
        return self._device[ctx.device][0]

    def read(self, ctx, first: int, count: int):
        """Rows [first, first+count) as NCHW fp32 + labels."""
        n, c, h, w = self.shape
        img = np.empty((count, c, h, w), np.float32)
        lab = np.empty(count, np.int32)
        _lib.call("psg_dataset_read_f32", self.handle(ctx), first, count,
                  img.ctypes.data_as(_lib._F), lab.ctypes.data_as(_lib._I32))
        return img, lab


@dataclass
class Shard:
    """data.hpp:44-50: a contiguous slice of a shuffled permutation."""
    dataset: Dataset
    indices: np.ndarray
    worker_id: int = 0

    def size(self) -> int:
        return int(self.indices.size)


def shard(dataset: Dataset, workers: int, seed: int) -> List[Shard]:
    """data.hpp:261-288 (bit-exact, computed by libpsg's host code)."""
    n = dataset.size()
    perm = np.empty(n, np.uint64)
    offs = np.empty(max(workers, 0) + 1, np.uint64)
    _lib.call("psg_shard", n, workers, seed, perm.ctypes.data_as(_lib._U64),
              offs.ctypes.data_as(_lib._U64))
    return [Shard(dataset, perm[int(offs[k]):int(offs[k + 1])].copy(), k)
            for k in range(workers)]


def worker_stream_seed(global_seed: int, worker_id: int) -> int:
    """data.hpp:386-388."""
    return int(_lib.lib().psg_worker_stream_seed(global_seed, worker_id))


def epoch_order(indices: np.ndarray, stream_seed: int, epoch: int) -> np.ndarray:
    """data.hpp:338-343: the shard shuffled by derive_seed(stream_seed, epoch)."""
    idx = np.ascontiguousarray(indices, np.uint64)
    out = np.empty_like(idx)
    _lib.call("psg_epoch_order", idx.ctypes.data_as(_lib._U64), idx.size, stream_seed, epoch,
              out.ctypes.data_as(_lib._U64))
    return out


@dataclass
class ShardBatchIterator:
    """data.hpp:312-351.  A descriptor: the device net owns the cursor once attached
    (Net.set_training_data); ``indices(steps)`` replays the same stream on the host."""
    shard: Shard
    batch_size: int
    seed: int
    _epoch: int = 0
    _cursor: int = 0
    _order: Optional[np.ndarray] = field(default=None, repr=False)

    def __post_init__(self):
        if self.batch_size < 1:
            raise ValueError("batch iterator: batch size must be >= 1")
        if self.batch_size > self.shard.size():
            raise ValueError("batch iterator: batch size exceeds shard size")
        self._order = epoch_order(self.shard.indices, self.seed, 0)

    def next_indices(self) -> np.ndarray:
        b = self.batch_size
        if (self._cursor + 1) * b > self._order.size:
            self._epoch += 1
            self._order = epoch_order(self.shard.indices, self.seed, self._epoch)
            self._cursor = 0
        out = self._order[self._cursor * b:(self._cursor + 1) * b]
        self._cursor += 1
        return out

    def next(self):
        """Host Batch (for the explicit forward/backward API and tests)."""
        from .model import Batch
        idx = self.next_indices().astype(np.int64)
        ds = self.shard.dataset
        return Batch(np.asarray(ds.images[idx], np.float64), ds.labels[idx].copy())


@dataclass
class SequentialBatchIterator:
    """data.hpp:355-382: fixed order, cycles, drops the tail batch."""
    dataset: Dataset
    batch_size: int

    def __post_init__(self):
        if self.batch_size < 1 or self.batch_size > self.dataset.size():
            raise ValueError("eval iterator: bad batch size")


def make_worker_iterator(shards: List[Shard], worker_id: int, batch_size: int,
                         global_seed: int) -> ShardBatchIterator:
    """data.hpp:391-397."""
    return ShardBatchIterator(shards[worker_id], batch_size,
                              worker_stream_seed(global_seed, worker_id))
