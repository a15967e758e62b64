"""WeightCollection and weights_mean — host mirror of weights.hpp:19-111.

A WeightCollection is the ordered ``(layer name -> [tensors])`` list every Net exchanges
at a synchronisation point (weights.hpp:15-18); ``add`` APPENDS an entry (it is not an
elementwise add, weights.hpp:23-25).  ``weights_mean`` accumulates in ascending input
order in fp64 (weights.hpp:88-107, tensor.hpp:166-179).  On the device path the
same average runs as the ordered / NCCL collective in libpsg (psg_comm_average); this
host version serves the API surface, observers and tests.

Additive helpers for the SparkNet Scala names: ``scalar_divide`` / ``average`` (and the
camelCase aliases ``scalarDivide``).
"""
from __future__ import annotations

from typing import Iterable, List, Optional, Sequence, Tuple

import numpy as np


class WeightCollection:
    def __init__(self, entries: Optional[Iterable[Tuple[str, Sequence[np.ndarray]]]] = None):
        self._entries: List[Tuple[str, List[np.ndarray]]] = []
        for name, tensors in entries or []:
            self.add(name, tensors)

    # weights.hpp:23-41
    def add(self, name: str, tensors: Sequence[np.ndarray]) -> None:
        self._entries.append((name, [np.array(t, dtype=np.float64, copy=True) for t in tensors]))

    def size(self) -> int:
        return len(self._entries)

    def __len__(self) -> int:
        return len(self._entries)

    def empty(self) -> bool:
        return not self._entries

    def entry(self, i: int) -> Tuple[str, List[np.ndarray]]:
        if not 0 <= i < len(self._entries):
            raise IndexError("WeightCollection::entry: index out of range")
        return self._entries[i]

    def __iter__(self):
        return iter(self._entries)

    def find(self, name: str) -> Optional[List[np.ndarray]]:
        for n, t in self._entries:
            if n == name:
                return t
        return None

    # weights.hpp:43-62
    def same_structure(self, other: "WeightCollection") -> bool:
        if len(self._entries) != len(other._entries):
            return False
        for (na, ta), (nb, tb) in zip(self._entries, other._entries):
            if na != nb or len(ta) != len(tb):
                return False
            if any(a.shape != b.shape for a, b in zip(ta, tb)):
                return False
        return True

    def __eq__(self, other) -> bool:
        if not isinstance(other, WeightCollection) or len(self) != len(other):
            return False
        for (na, ta), (nb, tb) in zip(self._entries, other._entries):
            if na != nb or len(ta) != len(tb):
                return False
            for a, b in zip(ta, tb):
                if a.shape != b.shape or a.tobytes() != b.tobytes():
                    return False
        return True

    def digest(self) -> int:
        """FNV-1a over names and raw fp64 bytes in storage order (weights.hpp:66-82)."""
        h = 0xcbf29ce484222325
        prime = 0x100000001b3
        mask = (1 << 64) - 1
        for name, tensors in self._entries:
            for byte in name.encode():
                h = ((h ^ byte) * prime) & mask
            for t in tensors:
                for byte in np.ascontiguousarray(t, np.float64).tobytes():
                    h = ((h ^ byte) * prime) & mask
        return h

    # flat <-> structured (WeightCollection order = the C ABI's flat order)
    def flat(self) -> np.ndarray:
        parts = [t.ravel() for _, ts in self._entries for t in ts]
        return np.concatenate(parts) if parts else np.zeros(0)

    def copy(self) -> "WeightCollection":
        return WeightCollection(self._entries)

    def scalar_divide(self, k: float) -> "WeightCollection":
        """SparkNet's WeightCollection.scalarDivide: every tensor / k (true division)."""
        return WeightCollection((n, [t / float(k) for t in ts]) for n, ts in self._entries)

    scalarDivide = scalar_divide

    @staticmethod
    def average(items: Sequence["WeightCollection"]) -> "WeightCollection":
        """SparkNet's WeightCollection.average == weights_mean."""
        return weights_mean(items)


def weights_mean(items: Sequence[WeightCollection]) -> WeightCollection:
    """weights.hpp:90-107: structure check, then per tensor acc = 0; acc += w_k ascending;
    acc /= K; non-finite -> RuntimeError (tensor.hpp:177)."""
    if not items:
        raise ValueError("weights_mean: empty input")
    for w in items:
        if not w.same_structure(items[0]):
            raise ValueError("weights_mean: structure mismatch")
    out = WeightCollection()
    k = float(len(items))
    for e in range(items[0].size()):
        name, tensors = items[0].entry(e)
        means = []
        for t in range(len(tensors)):
            acc = np.zeros_like(tensors[t], dtype=np.float64)
            for w in items:
                acc += w.entry(e)[1][t]
            acc /= k
            if not np.all(np.isfinite(acc)):
                raise RuntimeError("mean_collection: produced a non-finite value")
            means.append(acc)
        out.add(name, means)
    return out
