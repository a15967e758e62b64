"""Device-side data generation and ingestion: the device synthetic
generator has generate_synthetic's law (data.hpp:111-155): exact labels, class means
equal to the reference generator's, unit within-class pixel variance."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def test_device_synthetic_distribution_matches_reference_generator():
    from paper_1511_06051_b200.data import DeviceSyntheticDataset, generate_synthetic
    from paper_1511_06051_b200.model import Context
    ctx = Context.get(0)
    k, c, h, w, per = 3, 3, 12, 10, 600
    dev = DeviceSyntheticDataset(k, c, h, w, per, 2.0, 12345, 0)
    img, lab = dev.read(ctx, 0, k * per)
    ref_img, ref_lab = generate_synthetic(k, c, h, w, per, 2.0, 12345, 0)
    np.testing.assert_array_equal(lab, ref_lab)
    for cls in range(k):
        a = img[lab == cls].astype(np.float64)
        b = ref_img[ref_lab == cls]
        # both are per-pixel means of 600 unit-variance rows around the same class mean
        assert np.abs(a.mean(0) - b.mean(0)).max() < 6 * np.sqrt(2.0 / per)
        var = a.var(0)
        assert abs(var.mean() - 1.0) < 0.05 and var.min() > 0.7 and var.max() < 1.35
        # spatially smooth structure: neighbouring pixels correlate like the reference's
        def corr(x):
            d = x - x.mean(0)
            return float((d[:, :, :, 1:] * d[:, :, :, :-1]).mean() / d.var())
        assert abs(corr(a) - corr(b)) < 0.05
    # variants are independent noise streams around the same means
    v1, _ = DeviceSyntheticDataset(k, c, h, w, per, 2.0, 12345, 1).read(ctx, 0, k * per)
    assert not np.array_equal(v1, img)
    assert np.abs(v1[lab == 0].mean(0) - img[lab == 0].mean(0)).max() < 6 * np.sqrt(2.0 / per)


def test_device_synthetic_dataset_trains():
    """A device-generated dataset drives the HBM-resident shard stream."""
    from paper_1511_06051_b200 import data, netspec as ns
    from paper_1511_06051_b200.model import Net, SgdOptions
    ds = data.DeviceSyntheticDataset(10, 1, 16, 16, 20, 2.0, 7, 0)
    spec = ns.make_lenet_small(10, 1, 16, 16, 10)
    net = Net(spec, 1)
    net.set_sgd(SgdOptions(0.05, 0.9))
    shards = data.shard(ds, 2, 3)
    net.set_training_data(data.make_worker_iterator(shards, 1, 10, 3))
    net.train(12)
    assert np.isfinite(net.last_loss())


def test_idx_device_ingestion_matches_host_parse(tmp_path):
    """psg_dataset_load_idx: raw bytes uploaded, rescaled on the device == load_idx."""
    import ctypes
    import struct
    from paper_1511_06051_b200 import _lib, data
    from paper_1511_06051_b200.model import Context
    rng = np.random.default_rng(4)
    px = rng.integers(0, 256, size=(33, 9, 7)).astype(np.uint8)
    labels = rng.integers(0, 6, size=33).astype(np.uint8)
    ip, lp = tmp_path / "i.idx", tmp_path / "l.idx"
    ip.write_bytes(struct.pack(">IIII", 0x803, 33, 9, 7) + px.tobytes())
    lp.write_bytes(struct.pack(">II", 0x801, 33) + labels.tobytes())
    host = data.load_idx(str(ip), str(lp))
    ctx = Context.get(0)
    h = ctypes.c_void_p()
    _lib.call("psg_dataset_load_idx", ctx.handle, str(ip).encode(), str(lp).encode(),
              ctypes.byref(h))
    img = np.empty((33, 1, 9, 7), np.float32)
    lab = np.empty(33, np.int32)
    _lib.call("psg_dataset_read_f32", h, 0, 33, img.ctypes.data_as(_lib._F),
              lab.ctypes.data_as(_lib._I32))
    _lib.lib().psg_dataset_destroy(h)
    np.testing.assert_array_equal(img, host.images)
    np.testing.assert_array_equal(lab, host.labels)
