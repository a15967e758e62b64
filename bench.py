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


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=10)
    p.add_argument("--warmup", type=int, default=3)
    p.add_argument("--impl", default="ours", choices=["ours", "reference"])
    p.add_argument("--workload", default="alexnet", choices=list(WORKLOADS),
                   help="default: AlexNet b=256 tau=50 (BASELINE.json configs[2], the "
                        "north-star workload); the cifar10_quick tau sweep at this K "
                        "(configs[1]) rides along as an extra key")
    p.add_argument("--no-extra", dest="extra", action="store_false",
                   help="skip the cifar10_quick tau sweep")
    p.add_argument("--tau", type=int, default=None,
                   help="local SGD steps per round (default: the BASELINE config's — "
                        "AlexNet 50, GoogLeNet 20, cifar10_quick 10)")
    p.add_argument("--batch", type=int, default=None,
                   help="per-worker batch override (exploration; default: the config's)")
    # tf32 = tcgen05 tensor cores (north star's fast mode, per-layer parity 1e-2);
    # fp32 = strict SIMT mode (parity 1e-5)
    p.add_argument("--precision", default="tf32", choices=["fp32", "tf32"])
    p.add_argument("--average", default="fast", choices=["fast", "ordered"])
    p.add_argument("--no-overlap", dest="overlap", action="store_false",
                   help="fast average after the round instead of per-layer buckets "
                        "overlapped with the round's last backward (psg_net_train_round)")
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


# CPU sample: per-worker batch of the bounded sample (~10-30 s of fp64 work on the host cores)
CPU_SAMPLE_BATCH = {"cifar10_quick": None, "cq-valid": None, "alexnet": 2, "googlenet": 2}


def host_cpu():
    return {"model": lscpu_model(), "hardware_concurrency": os.cpu_count()}


class CpuRound:
    """The reference's CPU path in steady state (the oracle port of run_sparknet's round,
    schemes.hpp:323-338): K = `threads` worker nets (the port of Net, model.hpp) on K host
    threads, each running SGD steps (backward + apply_update, model.hpp:111-118) on its own
    batch of its shard, then get_weights of every worker, weights_mean (weights.hpp:90-107)
    and set_weights back (the next round's broadcast).  Net construction / init happens
    once, outside the timed rounds (the reference builds its nets once per run)."""

    def __init__(self, workload, b, threads):
        import threading
        from oracle import pyoracle
        from paper_1511_06051_b200 import netspec
        self.b = CPU_SAMPLE_BATCH.get(workload) or b
        self.K = threads
        self.spec = getattr(netspec, WORKLOADS[workload][0])(self.b)
        _, _, (c, h, w), _, self.lr, self.mu, self.wd = WORKLOADS[workload]
        self.lib = pyoracle.OracleLib()
        per_class = max(1, (self.b * threads + 9) // 10)
        img, lab = self.lib.generate_synthetic(10, c, h, w, per_class, 2.0, 12345, 0)
        if (c, h, w) != (3, 32, 32):
            lab = lab * 97  # ImageNet-shaped nets: labels spread over 1000 classes
        rows = self.lib.shard(len(lab), threads, 1)
        self.batches = [(np.ascontiguousarray(img[r[:self.b].astype(np.int64)]),
                         np.ascontiguousarray(lab[r[:self.b].astype(np.int64)]))
                        for r in rows]
        self.nets = [None] * threads

        def make(k):
            n = self.lib.net(self.spec, 1)
            n.set_sgd(self.lr, self.mu, self.wd)
            self.nets[k] = n
        self._parallel(make, threading)
        self.threading = threading

    def _parallel(self, fn, threading):
        ts = [threading.Thread(target=fn, args=(k,)) for k in range(self.K)]
        for t in ts:
            t.start()
        for t in ts:
            t.join()

    def round(self, steps=1):
        """One round of `steps` local steps per worker + the average; returns (seconds of
        forward + backward, seconds of apply_update — both the slowest worker's, per step —
        and seconds of the average)."""
        fb, upd = [0.0] * self.K, [0.0] * self.K

        def work(k):
            n = self.nets[k]
            x, y = self.batches[k]
            for _ in range(steps):
                t0 = time.perf_counter()
                _, g = n.backward(x, y)
                t1 = time.perf_counter()
                n.apply_update(g)
                fb[k] += t1 - t0
                upd[k] += time.perf_counter() - t1
        self._parallel(work, self.threading)
        t1 = time.perf_counter()
        ws = [n.get_weights() for n in self.nets]
        mean = self.lib.weights_mean(ws)
        for n in self.nets:
            n.set_weights(mean)
        return max(fb) / steps, max(upd) / steps, time.perf_counter() - t1

    def value_at(self, tau, b_cfg, t_fb, t_upd, t_avg):
        """images/sec of the configuration's round: tau sequential steps per worker — the
        forward / backward time scaled from the sample's batch to the configuration's
        (per-image work), the update per step as measured — then one average
        (schemes.hpp:323-336)."""
        t_step = t_fb * b_cfg / self.b + t_upd
        return self.K * tau * b_cfg / (tau * t_step + t_avg)


def cpu_baseline(workload, b, threads, steps=1, rounds=1, tau=None):
    """The reference's CPU path timed on host cores (see CpuRound).  cifar10_quick / AlexNet /
    GoogLeNet are not expressible by the unmodified reference (no pad / ave pool / LRN), so
    the C restatement (oracle/oracle.c) is timed (kind "port"); cq-valid runs the reference
    itself (kind "reference", oracle/_ref built from /root/reference by oracle/Makefile)."""
    from oracle import pyoracle
    use_ref = workload == "cq-valid" and os.path.exists(
        os.path.join(ROOT, "oracle", "_ref", "libparasgd_ref.so"))
    if use_ref:
        spec, _ = make_spec(workload, b)
        _, _, (c, h, w), *_ = WORKLOADS[workload]
        orc = pyoracle.OracleLib()
        img, lab = orc.generate_synthetic(10, c, h, w, max(1, (b * threads + 9) // 10), 2.0,
                                          12345, 0)
        t0 = time.perf_counter()
        pyoracle.RefLib(strict=False).run_sparknet(spec, (img, lab), (img[:b], lab[:b]), b,
                                                   0.001, 0.9, 1, threads, steps, rounds, 0,
                                                   threads=threads)
        dt = time.perf_counter() - t0
        bs = b
        value = threads * steps * rounds * bs / dt
        sample = (f"{workload} per-worker batch {bs}: {rounds} round(s) of {threads} workers x "
                  f"{steps} SGD step(s) on {threads} host threads + the K-way weights_mean "
                  f"({dt:.1f} s timed)")
    else:
        cr = CpuRound(workload, b, threads)
        ts = [cr.round(1) for _ in range(rounds)]
        t_fb, t_upd, t_avg = (sum(t[i] for t in ts) / rounds for i in range(3))
        tau = tau or 1
        value, bs = cr.value_at(tau, b, t_fb, t_upd, t_avg), cr.b
        sample = (f"{workload}: {threads} workers on {threads} host threads, sample batch "
                  f"{bs} per worker (forward+backward {t_fb:.2f} s, apply_update {t_upd:.2f} s "
                  f"per step) + the K-way weights_mean / get / set_weights ({t_avg:.2f} s); "
                  f"round at tau={tau}, batch {b}: tau x (fwd+bwd x {b}/{bs} + update) + "
                  f"average")
    out = {"value": value, "unit": "images/sec", "cores": threads,
           "kind": "reference" if use_ref else "port", "sample": sample}
    out.update(host_cpu())
    return out


def run_reference(args):
    """--impl reference: the reference's CPU path (CpuRound: the oracle port of run_sparknet's
    round; the reference itself for cq-valid) on the box's host cores, all threads, on this
    arm's workload / metric; each step is a bounded sample — one round of one SGD step per
    worker thread at a small per-worker batch, plus the K-way average."""
    rank, world, _ = dist_env()
    if rank != 0:
        return
    _, b = make_spec(args.workload, args.batch)
    threads = max(1, os.cpu_count() or 1)
    if args.workload == "cq-valid":
        r = cpu_baseline(args.workload, b, threads, rounds=args.steps)
        value, bs, kind = r["value"], b, r["kind"]
    else:
        cr = CpuRound(args.workload, b, threads)
        for _ in range(args.warmup):
            cr.round(1)
        ts = [cr.round(1) for _ in range(args.steps)]
        t_fb, t_upd, t_avg = (sum(t[i] for t in ts) / args.steps for i in range(3))
        bs, kind = cr.b, "port"
        value = cr.value_at(args.tau, b, t_fb, t_upd, t_avg)
    cb = {"value": value, "unit": "images/sec", "cores": threads, "kind": kind,
          "sample": f"per step: {threads} worker(s) x 1 SGD step of {args.workload} at "
                    f"sample batch {bs} on {threads} host thread(s) + the K-way average; "
                    f"value = K*tau*b / (tau*(fwd_bwd*b/{bs} + update) + average) at "
                    f"tau={args.tau}, b={b}"}
    cb.update(host_cpu())
    print(json.dumps({
        "impl": "reference", "metric": "images/sec", "value": value, "unit": "images/sec",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": threads * b / value * 1000.0, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": args.workload, "global_batch": b * threads, "K": threads,
                   "tau": args.tau, "per_worker_batch": b, "sample_batch": bs,
                   "note": "reference CPU path (bounded sample per step)"},
        "cpu_baseline": cb,
        "e2e": {"value": value, "unit": "images/sec", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0}}))


GEMM_PHASES = ("forward", "wgrad", "dgrad")


def lscpu_model():
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return None


def roofline_of(prof, precision, peaks, workload):
    """Roofline of the dominant op of one step's live per-op profile, plus the aggregate over
    every GEMM-shaped op (conv / linear fprop, dgrad, wgrad: `gemm_frac`).  TF32 peak: the
    driver-measured dense bf16 cuBLAS burst figure / 2 (MEASURED_PEAKS.json; tensor-core TF32
    issues half the bf16 MACs per cycle); the sustained (power-capped) figure / 2 is reported
    beside it."""
    step_ms = sum(p["ms"] for p in prof)
    top = max(prof, key=lambda p: p["ms"])
    bf16, bf16_s = peaks["bf16_tflops"], peaks.get("bf16_tflops_sustained")
    if precision == "tf32":
        peak, src = bf16 / 2, f"MEASURED_PEAKS.json bf16_tflops {bf16:.1f} / 2 (burst)"
        peak_s = bf16_s / 2 if bf16_s else None
    else:
        peak, src = peaks.get("fp32_simt_tflops", bf16 / 32), "fp32 SIMT (profiles/peaks_measured.json)"
        peak_s = None
    if top["flops"] > 0:
        achieved = top["flops"] / (top["ms"] * 1e-3) / 1e12
        roof = {"bound": "tensor" if precision == "tf32" else "fp32-simt", "achieved": achieved,
                "peak": peak, "unit": "TFLOP/s", "frac": achieved / peak, "peak_source": src}
    else:
        achieved = top["bytes"] / (top["ms"] * 1e-3) / 1e9
        roof = {"bound": "hbm", "achieved": achieved, "peak": peaks["hbm_gbs"], "unit": "GB/s",
                "frac": achieved / peaks["hbm_gbs"], "peak_source": "MEASURED_PEAKS.json hbm_gbs"}
    roof.update({"traffic": None, "kernel": top["name"], "share_of_step": top["ms"] / step_ms,
                 "algorithmic": top["flops"] or top["bytes"]})
    gemm = [p for p in prof if p["flops"] > 0 and p["phase"] in GEMM_PHASES]
    if gemm:
        fl, ms = sum(p["flops"] for p in gemm), sum(p["ms"] for p in gemm)
        roof["gemm"] = {"ops": len(gemm), "flops": fl, "ms": ms, "share_of_step": ms / step_ms,
                        "achieved": fl / (ms * 1e-3) / 1e12}
        roof["gemm_frac"] = roof["gemm"]["achieved"] / peak
        tot = sum(p["flops"] for p in prof)
        roof["step_frac"] = tot / (step_ms * 1e-3) / 1e12 / peak
        if peak_s:
            roof["gemm_frac_vs_sustained"] = roof["gemm"]["achieved"] / peak_s
            roof["peak_sustained"] = peak_s
    # traffic: DRAM bytes of the same op in the committed ncu capture of this workload
    # (tools/op_traffic.py; cold-cache serialised replay, one training step)
    for rnd in ("round2", "round1"):
        tpath = os.path.join(ROOT, "profiles", rnd, f"{workload}_op_traffic.json")
        if not os.path.exists(tpath):
            continue
        with open(tpath) as f:
            tr = json.load(f)
        hit = [o for o in tr["ops"] if o["op"] == top["name"]]
        if hit and tr.get("precision") == precision:
            roof["traffic"] = hit[0]["dram_bytes"]
            roof["traffic_unit"] = "bytes per op launch set (ncu dram__bytes_read+write)"
            roof["ncu_share_of_step"] = hit[0]["ncu_share"]
            roof["traffic_source"] = os.path.relpath(tpath, ROOT)
        break
    return roof, step_ms


class Rank:
    """This process's rank / device and the gloo group used for barriers and max-reduces."""

    def __init__(self):
        self.rank, self.world, self.local = dist_env()
        self.dist = None
        if self.world > 1:
            import torch.distributed as dist
            dist.init_process_group("gloo")
            self.dist = dist

    def max(self, x):
        if self.dist is None:
            return x
        import torch
        t = torch.tensor([x], dtype=torch.float64)
        self.dist.all_reduce(t, op=self.dist.ReduceOp.MAX)
        return float(t.item())

    def barrier(self):
        if self.dist is not None:
            self.dist.barrier()

    def bcast(self, obj):
        if self.dist is None:
            return obj
        box = [obj if self.rank == 0 else None]
        self.dist.broadcast_object_list(box, src=0)
        return box[0]


class Worker:
    """One SparkNet worker (this rank's GPU): its net on shard `rank` of the workload's
    synthetic dataset, and the communicator of the per-round weight average."""

    def __init__(self, R, workload, precision, average, batch=None, overlap=True):
        from paper_1511_06051_b200 import data as pdata
        from paper_1511_06051_b200 import model
        self.R, self.workload, self.avg_mode = R, workload, average
        self.overlap = overlap and average == "fast" and R.world > 1
        self.spec, self.b = make_spec(workload, batch)
        _, _, self.chw3, _, lr, mu, wd = WORKLOADS[workload]
        self.ds = build_dataset(workload, R.world)
        self.shards = pdata.shard(self.ds, R.world, 1)
        self.net = model.Net(self.spec, 1, device=R.local, precision=precision)
        self.net.set_sgd(model.SgdOptions(lr, mu, wd))
        self.net.set_training_data(pdata.make_worker_iterator(self.shards, R.rank, self.b, 1))
        # overlap the average with the last backward when it moves enough bytes to matter
        # (cifar10_quick's 0.58 MB: the per-layer collectives' latency exceeds the overlap)
        if 4 * self.net.P < 8e6:
            self.overlap = False
        self.comm = None
        if R.world > 1:
            from paper_1511_06051_b200.comm import Communicator, unique_id
            uid = R.bcast(unique_id() if R.rank == 0 else None)
            self.comm = [Communicator.create(self.net.ctx, R.world, R.rank, uid)]

    def round(self, tau):
        """tau local steps + the K-way average (overlapped with the last backward in fast
        mode, psg_net_train_round), enqueued."""
        if self.overlap:
            self.net.train_round(tau, self.comm[0], sync=False)
        else:
            self.net.train(tau, sync=False)
            self.average()

    def close(self):
        """Net (and its captured round graph) first, then the communicator."""
        self.net.sync()
        self.net = None
        import gc
        gc.collect()
        for c in self.comm or []:
            c.close()
        self.comm = None

    def average(self):
        if self.comm is not None:
            from paper_1511_06051_b200.comm import Communicator
            Communicator.average(self.comm, [self.net], self.avg_mode)

    def sync_all(self):
        self.net.sync()
        self.R.barrier()

    def rounds(self, tau, n):
        """n SparkNet rounds (tau local steps + the K-way average), device-timed on the worker
        stream, max over ranks (ms)."""
        self.sync_all()
        self.net.event_record(0)
        for _ in range(n):
            self.round(tau)
        self.net.event_record(1)
        self.net.sync()
        ms = self.R.max(self.net.event_elapsed(0, 1))
        self.R.barrier()
        return ms

    def average_ms(self, reps=5):
        if self.comm is None:
            return None
        self.sync_all()
        self.net.event_record(2)
        for _ in range(reps):
            self.average()
        self.net.event_record(3)
        self.net.sync()
        return self.R.max(self.net.event_elapsed(2, 3)) / reps

    def e2e(self, tau, n):
        """The same rounds through the C ABI's host-fed path (psg_net_train_host_rows): per
        step, host threads gather the step's rows of this worker's shard from a host copy of
        the dataset (NCHW fp32) into pinned staging — the reference's gather_batch — while
        the GPU runs the previous step; then the H2D copy, the step, a D2H read of its loss;
        plus the K-way average.  Everything from the batch indices on is inside the timed
        region."""
        from paper_1511_06051_b200 import data as pdata
        c, h, w = self.chw3
        b = self.b
        mine = np.sort(np.asarray(self.shards[self.R.rank].indices, np.int64))
        if isinstance(self.ds, pdata.DeviceSyntheticDataset):  # pixels only in HBM: copy once
            host_img = np.empty((mine.size, c, h, w), np.float32)
            for j, r in enumerate(mine):
                host_img[j] = self.ds.read(self.net.ctx, int(r), 1)[0][0]
        else:
            host_img = np.ascontiguousarray(self.ds.images[mine], np.float32)
        host_lab = np.ascontiguousarray(self.ds.labels[mine], np.int32)
        host_it = pdata.make_worker_iterator(self.shards, self.R.rank, b, 7)
        # host threads per step's gather: one per ~8 MB of batch (thread start-up costs more
        # than it saves on cifar10_quick's 1.2 MB batches), at most this rank's cores
        threads = max(1, min((os.cpu_count() or 1) // self.R.world,
                             round(b * c * h * w * 4 / 8e6)))

        def host_round():
            rows = np.concatenate([host_it.next_indices() for _ in range(tau)]).astype(np.int64)
            self.net.train_host_rows(host_img, host_lab, np.searchsorted(mine, rows), threads)

        host_round()  # warm-up: capture the host-fed graphs
        self.average()
        self.sync_all()
        self.net.event_record(2)
        for _ in range(n):
            host_round()
            self.average()
        self.net.event_record(3)
        self.net.sync()
        ms = self.R.max(self.net.event_elapsed(2, 3))
        self.R.barrier()
        return ms, tau * b * (c * h * w * 4 + 4), tau * 8, threads


def rounds_for(ms_per_round, min_ms, at_least):
    return max(at_least, int(min_ms / max(ms_per_round, 1e-3)) + 1)


def tau_sweep(R, workload, precision, average, taus=(1, 10, 50, 100), min_ms=400.0,
              overlap=True):
    """cifar10_quick at this K (= world size) over tau (BASELINE.json configs[1]): images/sec
    = K * tau * b / round time; each point times >= min_ms of rounds after 3 warm-up rounds."""
    W = Worker(R, workload, precision, average, overlap=overlap)
    out = []
    for tau in taus:
        for _ in range(3):
            W.round(tau)
        probe = W.rounds(tau, 2) / 2
        n = rounds_for(probe, min_ms, 3)
        ms = W.rounds(tau, n)
        out.append({"tau": tau, "rounds": n, "ms_per_round": ms / n,
                    "value": R.world * n * tau * W.b / (ms / 1000.0)})
    prof = W.net.profile_step(repeats=5)
    avg_ms = W.average_ms()
    top = max(prof, key=lambda p: p["ms"])
    res = {"workload": workload, "K": R.world, "per_worker_batch": W.b, "unit": "images/sec",
           "points": out, "kernels_per_step": W.net.kernels_per_step(),
           "step_ms": sum(p["ms"] for p in prof), "top_op": top["name"],
           "weight_average_ms": avg_ms}
    W.close()
    return res


def main():
    args = parse()
    if args.impl == "reference":
        run_reference(args)
        return
    R = Rank()
    rank, world = R.rank, R.world
    K = world
    W = Worker(R, args.workload, args.precision, args.average, args.batch, args.overlap)
    net, b = W.net, W.b
    c, h, w = W.chw3

    # --- device-resident throughput (value) ---
    for _ in range(args.warmup):
        W.round(args.tau)
    W.sync_all()
    sampler = ClockSampler(R.local)
    sampler.start()
    ms = W.rounds(args.tau, args.steps)
    clocks = sampler.stop()
    images = K * args.steps * args.tau * b
    value = images / (ms / 1000.0)
    avg_ms = W.average_ms()

    # --- end to end through the C ABI with host buffers (e2e) ---
    e2e_steps = min(args.steps, 5)
    ems, h2d, d2h, gthreads = W.e2e(args.tau, e2e_steps)
    e2e_value = K * e2e_steps * args.tau * b / (ems / 1000.0)

    # --- roofline of the dominant op + all GEMM ops (live CUDA events, per op) ---
    prof = net.profile_step(repeats=5)
    peaks = load_peaks()
    roof, step_ms = roofline_of(prof, args.precision, peaks, args.workload)
    if args.profile_json and rank == 0:
        with open(args.profile_json, "w") as f:
            json.dump({"ops": prof, "step_ms": step_ms}, f, indent=1)

    launches = net.kernels_per_step() * args.tau * args.steps + (
        args.steps if (W.comm is not None and args.average == "ordered") else 0)
    param_bytes = 4 * sum(n for _, n in net.segments())
    overlapped = W.overlap
    net = None
    W.close()  # before the sweep's net / communicator (one communicator alive at a time)
    # the cifar10_quick tau sweep at this K (BASELINE.json configs[1])
    extra = None
    if args.extra and args.workload != "cifar10_quick":
        extra = tau_sweep(R, "cifar10_quick", args.precision, args.average,
                          overlap=args.overlap)
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu = cpu_baseline(args.workload, b, max(1, os.cpu_count() or 1), tau=args.tau)
    if rank == 0:
        print(json.dumps({
            "metric": "images/sec", "value": value, "unit": "images/sec", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms / args.steps,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
            "dtype": args.precision, "data": "synthetic",
            "config": {"workload": args.workload, "global_batch": b * K, "per_worker_batch": b,
                       "K": K, "tau": args.tau, "average": args.average,
                       "average_overlapped": overlapped,
                       "step": "one SparkNet round: tau local SGD steps per worker + the K-way "
                               "weight average",
                       "parallelism": f"sparknet-dp{K}",
                       "l2": "inputs larger than L2 (HBM-resident dataset "
                             f"{W_bytes(args.workload, K):.0f} MB, random per-step gather)"},
            "e2e": {"value": e2e_value, "unit": "images/sec", "h2d_bytes_per_step": h2d,
                    "d2h_bytes_per_step": d2h, "rounds": e2e_steps,
                    "host_gather_threads": gthreads,
                    "path": "psg_net_train_host_rows: each step's rows gathered from the host "
                            "dataset (host threads into pinned staging + one H2D, or — rows "
                            ">= 64 KB with < 12 host threads per rank — one DMA copy per row "
                            "from the registered dataset straight into device staging), "
                            "overlapping the previous step; the step; D2H of its loss; + the "
                            "average"},
            "roofline": roof, "cpu_baseline": cpu, "clocks": clocks,
            "timed_ms": ms,
            "weight_average": None if avg_ms is None else {
                "ms": avg_ms, "share_of_round": avg_ms / (ms / args.steps),
                "param_bytes": param_bytes},
            "gpu_launches": launches,
            "cifar10_quick_tau_sweep": extra}))
    if R.dist is not None:
        R.dist.destroy_process_group()


def W_bytes(workload, K):
    _, b, (c, h, w), per_class, *_ = WORKLOADS[workload]
    n = 10 * (per_class if per_class else max(1, (2 * b * K + 9) // 10))
    return n * c * h * w * 4 / 1e6


if __name__ == "__main__":
    main()
