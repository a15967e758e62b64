#!/usr/bin/env python
"""SparkNet round throughput on B200 (BASELINE.json metric: images/sec at K = 1/2/4/8).

One bench "step" = one SparkNet round on every GPU: tau local SGD steps per worker (each a
replay of the worker's CUDA graph over its HBM-resident shard) followed by the K-way weight
average (NCCL over NVLink for K > 1).  images/sec = K * tau * b / round time, whole job,
device-timed with CUDA events on the worker stream, max over ranks.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--workload cifar10_quick|alexnet|googlenet|cq-valid]
                  [--tau T] [--precision fp32|tf32] [--average fast|ordered]
  python bench.py --impl reference ...   # the reference's CPU path (oracle port) on host cores
Multi-GPU: python -m torch.distributed.run --nproc-per-node N ... bench.py --gpus N
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

WORKLOADS = {
    # name: (builder, batch, (c, h, w), per_class, lr, momentum, weight_decay)
    "cifar10_quick": ("make_cifar10_quick", 100, (3, 32, 32), 5000, 0.001, 0.9, 0.004),
    "cq-valid": ("make_cq_valid", 100, (3, 32, 32), 5000, 0.001, 0.9, 0.0),
    "alexnet": ("make_alexnet", 256, (3, 227, 227), None, 0.01, 0.9, 0.0005),
    "googlenet": ("make_googlenet", 32, (3, 224, 224), None, 0.01, 0.9, 0.0002),
}


# BASELINE.json configs: AlexNet K=8 tau=50, GoogLeNet K=8 tau=20, cifar10_quick tau sweep
DEFAULT_TAU = {"alexnet": 50, "googlenet": 20, "cifar10_quick": 10, "cq-valid": 10}
HOST_RING = 10  # e2e: pinned host batches per train_host call (re-sent every call)


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=10)
    p.add_argument("--warmup", type=int, default=3)
    p.add_argument("--impl", default="ours", choices=["ours", "reference"])
    p.add_argument("--workload", default="cifar10_quick", choices=list(WORKLOADS))
    p.add_argument("--tau", type=int, default=None,
                   help="local SGD steps per round (default: the BASELINE config's — "
                        "AlexNet 50, GoogLeNet 20, cifar10_quick 10)")
    p.add_argument("--batch", type=int, default=None,
                   help="per-worker batch override (exploration; default: the config's)")
    # tf32 = tcgen05 tensor cores (north star's fast mode, per-layer parity 1e-2);
    # fp32 = strict SIMT mode (parity 1e-5)
    p.add_argument("--precision", default="tf32", choices=["fp32", "tf32"])
    p.add_argument("--average", default="fast", choices=["fast", "ordered"])
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--profile-json", default=None, help="write the per-op profile here")
    a = p.parse_args()
    if a.tau is None:
        a.tau = DEFAULT_TAU.get(a.workload, 10)
    return a


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", str(rank)))
    return rank, world, local


def load_peaks():
    peaks = {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "source": "fallback (B200_PROFILING.md)"}
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(path):
        with open(path) as f:
            m = json.load(f)
        peaks.update({k: m[k] for k in ("hbm_gbs", "bf16_tflops", "bf16_tflops_sustained")
                      if k in m})
        peaks["source"] = "MEASURED_PEAKS.json"
    extra = os.path.join(ROOT, "profiles", "peaks_measured.json")
    if os.path.exists(extra):
        with open(extra) as f:
            peaks.update(json.load(f))
    return peaks


class ClockSampler:
    """SM clocks / throttle reasons sampled during the timed region: an NVML thread every
    5 ms (enough samples even for a ~40 ms cifar10_quick region), nvidia-smi as fallback."""
    Q = ("index,clocks.sm,clocks.max.sm,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
    NAMES = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]

    def __init__(self, device):
        self.device = device
        self.proc = None
        self.path = None
        self.thread = None
        self.samples = []

    def _nvml_loop(self, nv, h, stop):
        bits = [nv.nvmlClocksEventReasonHwSlowdown, nv.nvmlClocksEventReasonHwThermalSlowdown,
                nv.nvmlClocksEventReasonSwThermalSlowdown, nv.nvmlClocksEventReasonSwPowerCap]
        while not stop.is_set():
            try:
                sm = nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM)
                r = nv.nvmlDeviceGetCurrentClocksEventReasons(h)
                self.samples.append((sm, {n for n, bit in zip(self.NAMES, bits) if r & bit}))
            except Exception:  # noqa: BLE001
                pass
            stop.wait(0.005)

    def start(self):
        try:
            import threading

            import pynvml as nv
            nv.nvmlInit()
            h = nv.nvmlDeviceGetHandleByIndex(self._physical_index())
            self.max_mhz = float(nv.nvmlDeviceGetMaxClockInfo(h, nv.NVML_CLOCK_SM))
            self.stop_ev = threading.Event()
            self.thread = threading.Thread(target=self._nvml_loop, args=(nv, h, self.stop_ev),
                                           daemon=True)
            self.thread.start()
            return
        except Exception:  # noqa: BLE001 — fall back to nvidia-smi
            self.thread = None
        fd, self.path = tempfile.mkstemp(suffix=".csv")
        os.close(fd)
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.Q}",
                 "--format=csv,noheader,nounits", "-lms", "20"],
                stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
        except OSError:
            self.proc = None

    def _physical_index(self):
        vis = os.environ.get("CUDA_VISIBLE_DEVICES")
        if vis:
            ids = [v.strip() for v in vis.split(",")]
            if self.device < len(ids) and ids[self.device].isdigit():
                return int(ids[self.device])
        return self.device

    def stop(self):
        if self.thread is not None:
            self.stop_ev.set()
            self.thread.join()
            if not self.samples:
                return None
            return {"sm_mhz": statistics.median(s for s, _ in self.samples),
                    "sm_max_mhz": self.max_mhz,
                    "reasons": sorted(set().union(*(r for _, r in self.samples))),
                    "samples": len(self.samples), "source": "nvml 5 ms"}
        if self.proc is None:
            return None
        time.sleep(0.25)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        sm, mx, reasons = [], 0.0, set()
        with open(self.path) as f:
            for line in f:
                parts = [x.strip() for x in line.split(",")]
                if len(parts) < 8:
                    continue
                try:
                    sm.append(float(parts[1]))
                    mx = max(mx, float(parts[2]))
                except ValueError:
                    continue
                for n, v in zip(self.NAMES, parts[4:8]):
                    if v.lower().startswith("active"):
                        reasons.add(n)
        os.unlink(self.path)
        if not sm:
            return None
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sm), "source": "nvidia-smi 20 ms"}


def make_spec(workload, batch=None):
    from paper_1511_06051_b200 import netspec
    name, b, _, _, *_ = WORKLOADS[workload]
    b = batch or b
    return getattr(netspec, name)(b), b


def build_dataset(workload, K):
    """Synthetic data of the workload's shape, data.seed 12345, separation 2, 10 classes:
    the reference generator (data.hpp:111-155) for the 32x32 nets; for the ImageNet-shaped
    nets (AlexNet, GoogLeNet; label range 1000 classes) the device generator with the same
    law, enough rows for K shards of 2 batches each."""
    from paper_1511_06051_b200.data import Dataset, DeviceSyntheticDataset, generate_synthetic
    _, b, (c, h, w), per_class, *_ = WORKLOADS[workload]
    if per_class is None:
        per_class = max(1, (2 * b * K + 9) // 10)
        return DeviceSyntheticDataset(10, c, h, w, per_class, 2.0, 12345, 0, label_classes=1000)
    img, lab = generate_synthetic(10, c, h, w, per_class, 2.0, 12345, 0)
    return Dataset(img.astype(np.float32), lab, 10)


# CPU-baseline sample batch per worker: ~10-30 s of fp64 work on the box's host cores
CPU_SAMPLE_BATCH = {"cifar10_quick": None, "cq-valid": None, "alexnet": 16, "googlenet": 8}


def cpu_baseline(workload, b, threads, steps=1):
    """The oracle port (C, fp64) of run_sparknet on host cores: workers = threads, tau = steps,
    one round, eval skipped.  cifar10_quick / AlexNet are not expressible by the unmodified
    reference (no pad / ave pool / LRN), so the C restatement is timed (kind "port");
    cq-valid runs the reference itself (kind "reference")."""
    from oracle import pyoracle
    b = CPU_SAMPLE_BATCH.get(workload) or b
    spec = getattr(__import__("paper_1511_06051_b200.netspec", fromlist=["x"]),
                   WORKLOADS[workload][0])(b)
    _, _, (c, h, w), *_ = WORKLOADS[workload]
    per_class = max(1, (b * threads + 9) // 10)
    orc = pyoracle.OracleLib()
    img, lab = orc.generate_synthetic(10, c, h, w, per_class, 2.0, 12345, 0)
    ev = (img[:b], lab[:b])
    use_ref = workload == "cq-valid" and os.path.exists(
        os.path.join(ROOT, "oracle", "_ref", "libparasgd_ref.so"))
    t0 = time.perf_counter()
    if use_ref:
        pyoracle.RefLib(strict=False).run_sparknet(spec, (img, lab), ev, b, 0.001, 0.9, 1,
                                                   threads, steps, 1, 0, threads=threads)
    else:
        orc.run_sparknet(spec, (img, lab), ev, b, 0.001, 0.9, 1, threads, steps, 1, 0,
                         threads=threads, skip_eval=True)
    dt = time.perf_counter() - t0
    value = threads * steps * b / dt
    return {"value": value, "unit": "images/sec", "cores": threads,
            "kind": "reference" if use_ref else "port",
            "sample": f"{workload} b={b}: {threads} workers x {steps} SGD step(s) on {threads} "
                      f"host threads, 1 round ({dt:.1f} s)"}


def run_reference(args):
    rank, world, _ = dist_env()
    if rank != 0:
        return
    spec, b = make_spec(args.workload, args.batch)
    threads = max(1, args.gpus)
    t = []
    for i in range(args.warmup + args.steps):
        r = cpu_baseline(args.workload, b, threads, steps=1)
        if i >= args.warmup:
            t.append(threads * b / r["value"])
    sec = sum(t) / len(t)
    value = threads * b / sec
    cb = {"value": value, "unit": "images/sec", "cores": threads, "kind": r["kind"],
          "sample": f"per step: {threads} worker(s) x 1 SGD step of {args.workload} b={b} "
                    f"on {threads} host thread(s) + the K-way average"}
    print(json.dumps({
        "impl": "reference", "metric": "images/sec", "value": value, "unit": "images/sec",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": sec * 1000.0, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": args.workload, "global_batch": b * threads, "K": threads,
                   "tau": 1, "note": "reference CPU path (bounded sample per step)"},
        "cpu_baseline": cb,
        "e2e": {"value": value, "unit": "images/sec", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0}}))


def main():
    args = parse()
    if args.impl == "reference":
        run_reference(args)
        return
    rank, world, local = dist_env()
    from paper_1511_06051_b200 import data as pdata
    from paper_1511_06051_b200 import model
    from paper_1511_06051_b200._lib import PinnedArray

    dist = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("gloo")
    K = world
    spec, b = make_spec(args.workload, args.batch)
    _, _, (c, h, w), _, lr, mu, wd = WORKLOADS[args.workload]
    ds = build_dataset(args.workload, K)
    shards = pdata.shard(ds, K, 1)
    net = model.Net(spec, 1, device=local, precision=args.precision)
    net.set_sgd(model.SgdOptions(lr, mu, wd))
    it = pdata.make_worker_iterator(shards, rank, b, 1)
    net.set_training_data(it)
    comm = None
    if world > 1:
        from paper_1511_06051_b200.comm import Communicator, unique_id
        obj = [unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        comm = [Communicator.create(net.ctx, world, rank, obj[0])]

    def average():
        if comm is not None:
            from paper_1511_06051_b200.comm import Communicator
            Communicator.average(comm, [net], args.average)

    def barrier():
        net.sync()
        if dist is not None:
            dist.barrier()

    def max_over_ranks(x):
        if dist is None:
            return x
        import torch
        t = torch.tensor([x], dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    # --- device-resident throughput (value) ---
    for _ in range(args.warmup):
        net.train(args.tau, sync=False)
        average()
    barrier()
    sampler = ClockSampler(local)
    sampler.start()
    net.event_record(0)
    for _ in range(args.steps):
        net.train(args.tau, sync=False)
        average()
    net.event_record(1)
    net.sync()
    ms = max_over_ranks(net.event_elapsed(0, 1))
    clocks = sampler.stop()
    barrier()
    images = K * args.steps * args.tau * b
    value = images / (ms / 1000.0)
    avg_ms = None
    if comm is not None:  # the K-way weight average alone (north star: < 2% of the round)
        barrier()
        net.event_record(2)
        for _ in range(5):
            average()
        net.event_record(3)
        net.sync()
        avg_ms = max_over_ranks(net.event_elapsed(2, 3)) / 5

    # --- end to end through the C ABI with host buffers (e2e) ---
    e2e_steps = min(args.steps, 5)
    chw = c * h * w
    ring = min(args.tau, HOST_RING)  # bounded pinned buffer; every step still copies H2D
    pin_img = PinnedArray((ring, b, c, h, w), np.float32)
    pin_lab = PinnedArray((ring, b), np.int32)
    host_it = pdata.make_worker_iterator(shards, rank, b, 7)

    def host_round():  # tau host-fed steps: ceil(tau / ring) calls over the pinned ring
        left = args.tau
        while left > 0:
            n = min(ring, left)
            net.train_host(pin_img.array[:n], pin_lab.array[:n])
            left -= n

    for s in range(ring):
        idx = host_it.next_indices().astype(np.int64)
        if isinstance(ds, pdata.DeviceSyntheticDataset):  # pixels only in HBM: fetch rows once
            for i, r in enumerate(idx):
                pin_img.array[s, i] = ds.read(net.ctx, int(r), 1)[0][0]
        else:
            pin_img.array[s] = ds.images[idx]
        pin_lab.array[s] = ds.labels[idx]
    host_round()  # warm-up: capture the host-fed graph
    average()
    barrier()
    net.event_record(2)
    for _ in range(e2e_steps):
        host_round()
        average()
    net.event_record(3)
    net.sync()
    ems = max_over_ranks(net.event_elapsed(2, 3))
    e2e_value = K * e2e_steps * args.tau * b / (ems / 1000.0)

    # --- roofline of the dominant kernel (live CUDA events, per op) ---
    prof = net.profile_step(repeats=5)
    step_ms = sum(p["ms"] for p in prof)
    top = max(prof, key=lambda p: p["ms"])
    peaks = load_peaks()
    if top["flops"] > 0:
        achieved = top["flops"] / (top["ms"] * 1e-3) / 1e12
        if args.precision == "tf32":
            peak, src = peaks.get("tf32_tflops", peaks["bf16_tflops"] / 2), "tf32"
        else:
            peak, src = peaks.get("fp32_simt_tflops", peaks["bf16_tflops"] / 2), "fp32 SIMT"
        roof = {"bound": "tensor" if args.precision == "tf32" else "fp32-simt",
                "achieved": achieved, "peak": peak, "unit": "TFLOP/s", "frac": achieved / peak,
                "traffic": None, "kernel": top["name"],
                "share_of_step": top["ms"] / step_ms, "peak_source": src + " " + str(
                    peaks.get("source_extra", peaks["source"]))}
    else:
        achieved = top["bytes"] / (top["ms"] * 1e-3) / 1e9
        roof = {"bound": "hbm", "achieved": achieved, "peak": peaks["hbm_gbs"], "unit": "GB/s",
                "frac": achieved / peaks["hbm_gbs"], "traffic": None, "kernel": top["name"],
                "share_of_step": top["ms"] / step_ms, "peak_source": peaks["source"]}
    # traffic: DRAM bytes of the same op in the committed ncu capture of this workload
    # (tools/op_traffic.py; cold-cache serialised replay, one training step)
    tpath = os.path.join(ROOT, "profiles", "round1", f"{args.workload}_op_traffic.json")
    if os.path.exists(tpath):
        with open(tpath) as f:
            tr = json.load(f)
        hit = [o for o in tr["ops"] if o["op"] == top["name"]]
        if hit and tr.get("precision") == args.precision:
            roof["traffic"] = hit[0]["dram_bytes"]
            roof["traffic_unit"] = "bytes per op launch set (ncu dram__bytes_read+write)"
            roof["ncu_share_of_step"] = hit[0]["ncu_share"]
            roof["traffic_source"] = os.path.relpath(tpath, ROOT)
    if args.profile_json and rank == 0:
        with open(args.profile_json, "w") as f:
            json.dump({"ops": prof, "step_ms": step_ms}, f, indent=1)

    launches = net.kernels_per_step() * args.tau * args.steps + (
        args.steps if (comm is not None and args.average == "ordered") else 0)
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu = cpu_baseline(args.workload, b, max(1, min(8, os.cpu_count() or 1)))
    if rank == 0:
        print(json.dumps({
            "metric": "images/sec", "value": value, "unit": "images/sec", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms / args.steps,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
            "dtype": args.precision, "data": "synthetic",
            "config": {"workload": args.workload, "global_batch": b * K, "per_worker_batch": b,
                       "K": K, "tau": args.tau, "average": args.average,
                       "parallelism": f"sparknet-dp{K}",
                       "l2": "inputs larger than L2 (HBM-resident dataset "
                             f"{ds.size() * c * h * w * 4 / 1e6:.0f} MB, random per-step gather)"},
            "e2e": {"value": e2e_value, "unit": "images/sec",
                    "h2d_bytes_per_step": args.tau * b * (chw * 4 + 4),
                    "d2h_bytes_per_step": args.tau * 8},
            "roofline": roof, "cpu_baseline": cpu, "clocks": clocks,
            "weight_average": None if avg_ms is None else {
                "ms": avg_ms, "share_of_round": avg_ms / (ms / args.steps),
                "param_bytes": 4 * sum(c for _, c in net.segments())},
            "gpu_launches": launches}))
    if dist is not None:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
