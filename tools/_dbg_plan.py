import os, sys
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "tests"))
os.environ["PSG_TC_DEBUG"] = "1"
os.environ["PSG_EAGER"] = "1"
from paper_1511_06051_b200 import model as gpu
import test_gpu_parity as T
spec = T.micro_nets()["caffe_mix"]
net = gpu.Net(spec, 3, precision="tf32", fuse=True)
print([(n, [(o, s) for o, s in ts]) for n, ts in net._structure], flush=True)
b = T._batch(spec, 5, 7)
net.backward_flat(gpu.Batch(*b))
