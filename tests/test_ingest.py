"""load_idx / load_csv (data.hpp:163-255) through libpsg's host parser: formats, p/255
scaling and the reference's error conditions.  CPU only (no device calls)."""
import struct

import numpy as np
import pytest

from paper_1511_06051_b200 import data
PsgError = RuntimeError  # std::runtime_error -> PSG_ERUNTIME -> RuntimeError


def _write_idx(tmp_path, px, labels, magic_img=0x803, magic_lab=0x801, truncate=0):
    n, h, w = px.shape
    ip, lp = tmp_path / "img.idx", tmp_path / "lab.idx"
    body = struct.pack(">IIII", magic_img, n, h, w) + px.astype(np.uint8).tobytes()
    ip.write_bytes(body[:len(body) - truncate])
    lp.write_bytes(struct.pack(">II", magic_lab, len(labels)) + bytes(labels))
    return str(ip), str(lp)


def test_load_idx_values_and_classes(tmp_path):
    rng = np.random.default_rng(1)
    px = rng.integers(0, 256, size=(7, 5, 4))
    labels = [3, 0, 9, 1, 1, 2, 0]
    ds = data.load_idx(*_write_idx(tmp_path, px, labels))
    assert ds.images.shape == (7, 1, 5, 4) and ds.num_classes == 10
    np.testing.assert_array_equal(ds.labels, labels)
    want = (px.astype(np.float64) / 255.0).astype(np.float32)  # the reference value, in fp32
    np.testing.assert_array_equal(ds.images[:, 0], want)


@pytest.mark.parametrize("kw,msg", [({"magic_img": 0x801}, "bad image magic"),
                                     ({"magic_lab": 0x803}, "bad label magic"),
                                     ({"truncate": 3}, "truncated image data")])
def test_load_idx_errors(tmp_path, kw, msg):
    px = np.zeros((2, 3, 3))
    with pytest.raises(PsgError, match=msg):
        data.load_idx(*_write_idx(tmp_path, px, [0, 1], **kw))


def test_load_idx_count_mismatch_and_missing(tmp_path):
    ip, lp = _write_idx(tmp_path, np.zeros((2, 3, 3)), [0, 1, 1])
    with pytest.raises(PsgError, match="count mismatch"):
        data.load_idx(ip, lp)
    with pytest.raises(PsgError, match="cannot open"):
        data.load_idx(str(tmp_path / "nope"), lp)


def test_load_csv(tmp_path):
    p = tmp_path / "d.csv"
    p.write_text("1,0,255,51,102\n\n0,10,20,30,40\n")
    ds = data.load_csv(str(p), 1, 2, 2, 3)
    np.testing.assert_array_equal(ds.labels, [1, 0])
    want = (np.array([[0, 255, 51, 102], [10, 20, 30, 40]], np.float64) / 255.0)
    np.testing.assert_array_equal(ds.images.reshape(2, 4), want.astype(np.float32))
    p.write_text("5,1,2,3,4\n")
    with pytest.raises(PsgError, match="out of range at line 1"):
        data.load_csv(str(p), 1, 2, 2, 3)
    p.write_text("1,1,2,3\n")
    with pytest.raises(PsgError, match="expected 4 pixels, got 3"):
        data.load_csv(str(p), 1, 2, 2, 3)
