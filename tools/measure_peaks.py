"""Measure the roofline denominators MEASURED_PEAKS.json does not carry: dense TF32 tensor
throughput (cuBLAS fp32 matmul with TF32 allowed) and fp32 SIMT throughput (TF32
disallowed), 8192^3, best of 10 with CUDA events.  Writes profiles/peaks_measured.json.
Run on a B200 (gpurun)."""
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def bench(allow_tf32: bool, n: int = 8192, reps: int = 10) -> float:
    torch.backends.cuda.matmul.allow_tf32 = allow_tf32
    a = torch.randn(n, n, device="cuda", dtype=torch.float32)
    b = torch.randn(n, n, device="cuda", dtype=torch.float32)
    for _ in range(3):
        torch.matmul(a, b)
    best = 1e30
    for _ in range(reps):
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        torch.matmul(a, b)
        e.record()
        torch.cuda.synchronize()
        best = min(best, s.elapsed_time(e))
    return 2.0 * n ** 3 / (best * 1e-3) / 1e12


def main():
    out = {
        "tf32_tflops": bench(True),
        "fp32_simt_tflops": bench(False),
        "source_extra": "profiles/peaks_measured.json (torch.matmul fp32 8192^3, best of 10, "
                        "TF32 allowed / disallowed, " + torch.cuda.get_device_name() + ")",
    }
    path = os.path.join(ROOT, "profiles", "peaks_measured.json")
    os.makedirs(os.path.dirname(path), exist_ok=True)
    with open(path, "w") as f:
        json.dump(out, f, indent=1)
    json.dump(out, sys.stdout)
    print()


if __name__ == "__main__":
    main()
