"""Helpers to compare recomputed arrays with tests/golden/reference_golden.npz (bitwise)."""
import hashlib

import numpy as np


def has(golden, key: str) -> bool:
    return key in golden.files or (key + "__sha256") in golden.files


def equal(golden, key: str, value) -> bool:
    """Bitwise equality against the stored array or its sha256 digest."""
    if key in golden.files:
        want = golden[key]
        v = np.asarray(value).astype(want.dtype, copy=False).reshape(want.shape)
        return want.tobytes() == v.tobytes()
    want_dtype = str(golden[key + "__dtype"])
    v = np.ascontiguousarray(np.asarray(value).astype(want_dtype, copy=False))
    if list(v.shape) != list(golden[key + "__shape"]):
        v = v.reshape(tuple(golden[key + "__shape"]))
    return hashlib.sha256(v.tobytes()).hexdigest() == str(golden[key + "__sha256"])


def head(golden, key: str) -> np.ndarray:
    if key in golden.files:
        return golden[key].ravel()
    return golden[key + "__head"]


def net_input_rng(idx: int) -> np.random.Generator:
    """Same as tests/golden/make_golden.py:net_input_rng."""
    return np.random.default_rng(1000 + idx)
