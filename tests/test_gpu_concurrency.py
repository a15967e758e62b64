"""Two nets on one GPU driven from two host threads (each net on its own stream): the
gradients of a net must not depend on what runs beside it.  This caught the TMA-store
epilogue of the grouped im2col-matrix wgrad writing 32-row chunks that overlapped the next
group's filter rows (another CTA's output): correct only when that CTA happened to store
last.  Also the kernel shared-memory limit set per launch, raced between the threads."""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.parametrize("a", ["linear", "simt"])
def test_concurrent_nets_do_not_interfere(a):
    env = dict(os.environ, CC_A=a)
    r = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "concurrency_check.py"), "400"],
                       env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    line = [ln for ln in r.stdout.splitlines() if "differ" in ln][-1]
    assert line.split(":")[1].split("/")[0].strip() == "0", line
