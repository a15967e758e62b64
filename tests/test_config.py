"""The config boundary (north star: "the solver/net config files in proj/configs" stay
loadable): tests/cpp/config_test parses config files with the reference's own
ExperimentConfig (config.hpp:203-430, unmodified, reached through include/parasgd_shim) plus
the B200 keys of include/parasgd_b200/experiment.hpp.  Host only (no GPU)."""
import json
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
EXE = os.path.join(ROOT, "tests", "cpp", "config_test")
REF_CONFIGS = "/root/reference/proj/configs"


def parse(*paths):
    if not os.path.exists(EXE):
        pytest.skip("config_test not built (needs the reference headers at build time)")
    out = subprocess.run([EXE, "parse", *paths], capture_output=True, text=True, timeout=60)
    assert out.returncode == 0, out.stderr
    return [json.loads(line) for line in out.stdout.splitlines()]


def test_reference_configs_load_unchanged():
    if not os.path.isdir(REF_CONFIGS):
        pytest.skip("reference configs not present")
    files = sorted(os.path.join(REF_CONFIGS, f) for f in os.listdir(REF_CONFIGS))
    got = {os.path.basename(r["file"]): r for r in parse(*files)}
    assert len(got) == 7 and all(r["ok"] and not r["extended"] for r in got.values())
    s = got["sparknet.cfg"]  # configs/sparknet.cfg
    assert (s["scheme"], s["workers"], s["tau"], s["batch"], s["net"]) == \
        ("sparknet", 4, 50, 50, "lenet-small")
    assert got["naive.cfg"]["scheme"] == "naive" and got["serial.cfg"]["scheme"] == "serial"


def test_b200_keys():
    r = parse(os.path.join(ROOT, "tests", "configs", "sparknet_cifar10_quick_tf32.cfg"))[0]
    assert r["ok"] and r["extended"]
    assert (r["preset"], r["weight_decay"], r["tf32"], r["average"]) == \
        ("cifar10_quick", 0.004, True, "fast")
    assert r["shape"] == [3, 32, 32] and r["batch"] == 20


BASE = """scheme = sparknet
scheme.workers = 2
data.channels = 3
data.height = 32
data.width = 32
"""


@pytest.mark.parametrize("extra,field", [
    ("precision = fp16\n", "precision"),
    ("sgd.weight_decay = -1\n", "sgd.weight_decay"),
    ("sgd.weight_decay = abc\n", "sgd.weight_decay"),
    ("device.count = 1.5\n", "device.count"),
    ("average.mode = ring\n", "average.mode"),
    ("net.preset = vgg\n", "net.preset"),                       # the reference's own check
    ("net.preset = alexnet\nnet.spec = relu(a,data)\n", "net.preset"),
    ("sgd.weigth_decay = 0.1\n", "sgd.weigth_decay"),          # unknown key: still rejected
    ("scheme.tau = 0\n", "scheme.tau"),                         # reference range check
    ("scheme = sparknet\n", "scheme"),                          # duplicate key
])
def test_config_errors_name_the_field(tmp_path, extra, field):
    p = tmp_path / "bad.cfg"
    p.write_text(BASE + extra)
    r = parse(str(p))[0]
    assert not r["ok"] and r["field"] == field, r
