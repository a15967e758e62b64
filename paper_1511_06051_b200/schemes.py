"""run_sparknet and its context types — host mirror of schemes.hpp:17-351.

The round loop (broadcast -> tau local steps per worker -> collect -> average -> eval) is
driven from one host thread: every worker's tau steps are a CUDA-graph replay enqueued
asynchronously on that worker's stream, so the K workers (one per GPU, or several on one
GPU) run concurrently without a thread pool; ``threads`` is accepted for API parity.
Averaging is the ordered device kernel when all workers share a GPU
(psg_average_local), else one NCCL collective per round over NVLink (comm.py).
The simulated clock stays the reference's closed form (schemes.hpp:53-73) so trace.csv is
unchanged; measured device time is reported separately.
"""
from __future__ import annotations

import ctypes
import math
import time
from dataclasses import dataclass, field
from typing import Callable, List, Optional

import numpy as np

from . import _lib
from .data import Dataset, SequentialBatchIterator, make_worker_iterator, shard
from .model import Net, SgdOptions
from .netspec import NetSpec
from .weights import WeightCollection


@dataclass
class CostModel:
    """schemes.hpp:22-34."""
    compute_seconds: float = 1.0
    sync_seconds: float = 0.0
    sublinearity: float = 1.0

    def validate(self) -> None:
        if not self.compute_seconds > 0.0:
            raise ValueError("cost: compute time must be > 0")
        if self.sync_seconds < 0.0:
            raise ValueError("cost: sync time must be >= 0")
        if not (0.0 < self.sublinearity <= 1.0):
            raise ValueError("cost: sublinearity must be in (0,1]")


class SimClock:
    """schemes.hpp:39-50."""

    def __init__(self):
        self._elapsed = 0.0

    def elapsed(self) -> float:
        return self._elapsed

    def advance_to(self, t: float) -> None:
        if t < self._elapsed:
            from ._lib import LogicError
            raise LogicError("sim clock: time moved backwards")
        self._elapsed = t


def serial_sim_time(iters: int, c: CostModel) -> float:
    return float(iters) * c.compute_seconds


def naive_step_seconds(c: CostModel, workers: int) -> float:
    part = (c.compute_seconds / float(workers) if c.sublinearity == 1.0
            else c.compute_seconds * math.pow(1.0 / float(workers), c.sublinearity))
    return part + c.sync_seconds


def naive_sim_time(iters: int, c: CostModel, workers: int) -> float:
    """schemes.hpp:62-64."""
    return float(iters) * naive_step_seconds(c, workers)


def sparknet_sim_time(rounds: int, tau: int, warm: int, c: CostModel) -> float:
    """schemes.hpp:69-73."""
    return float(warm) * c.compute_seconds + float(rounds) * (float(tau) * c.compute_seconds +
                                                               c.sync_seconds)


@dataclass
class EvalRecord:
    """schemes.hpp:76-82."""
    serial_iters: int = 0
    parallel_iters: int = 0
    rounds: int = 0
    sim_time: float = 0.0
    accuracy: float = 0.0


TARGET_REACHED, BUDGET_EXHAUSTED = "TargetReached", "BudgetExhausted"


@dataclass
class RunTrace:
    """schemes.hpp:87-102 (+ measured device round times, kept out of trace.csv)."""
    scheme: str = ""
    workers: int = 1
    tau: int = 0
    batch: int = 0
    learning_rate: float = 0.0
    seed: int = 0
    target_accuracy: float = 0.0
    cost: CostModel = field(default_factory=CostModel)
    warm_start_iters: int = 0
    warm_digest: int = 0
    records: List[EvalRecord] = field(default_factory=list)
    outcome: str = BUDGET_EXHAUSTED
    round_ms: List[float] = field(default_factory=list)
    # measured wall clock per round (sparknet): tau local steps on every worker / average
    compute_ms: List[float] = field(default_factory=list)
    sync_ms: List[float] = field(default_factory=list)

    def reached(self) -> bool:
        return self.outcome == TARGET_REACHED


@dataclass
class SchemeObserver:
    """schemes.hpp:105-108."""
    on_step: Optional[Callable] = None
    on_round: Optional[Callable[[int, WeightCollection], None]] = None


@dataclass
class SchemeContext:
    """schemes.hpp:111-130 (+ device placement / precision / averaging mode)."""
    net: NetSpec
    train_data: Optional[Dataset] = None
    eval_data: Optional[Dataset] = None
    batch: int = 1
    sgd: SgdOptions = field(default_factory=SgdOptions)
    seed: int = 0
    cost: CostModel = field(default_factory=CostModel)
    target_accuracy: float = 1.0
    eval_steps: int = 1
    devices: Optional[List[int]] = None
    precision: str = "fp32"
    average_mode: str = "ordered"

    def validate(self) -> None:
        if self.train_data is None or self.eval_data is None:
            raise ValueError("scheme: missing dataset")
        if self.batch < 1:
            raise ValueError("scheme: batch must be >= 1")
        if self.eval_steps < 1:
            raise ValueError("scheme: eval steps must be >= 1")
        self.cost.validate()


def average_local(nets: List[Net]) -> None:
    """weights_mean of K same-GPU nets, written back into every net (ordered, fp64 acc)."""
    arr = (ctypes.c_void_p * len(nets))(*[n.handle.value for n in nets])
    _lib.call("psg_average_local", arr, len(nets))


def evaluate(net: Net, ctx: SchemeContext) -> float:
    """schemes.hpp:134-139: a fresh sequential pass over the evaluation set."""
    net.set_validation_data(SequentialBatchIterator(ctx.eval_data, ctx.batch))
    return net.test(ctx.eval_steps)


def average_grads_local(nets: List[Net]) -> None:
    """weights_mean of K same-GPU nets' gradient buffers, written back into every net."""
    arr = (ctypes.c_void_p * len(nets))(*[n.handle.value for n in nets])
    _lib.call("psg_average_grads_local", arr, len(nets))


def evaluate_sharded(nets: List[Net], ctx: SchemeContext) -> float:
    """evaluate() split across K nets that hold the same weights (one per GPU): net k
    runs batches k, k+K, ... of the eval_steps; (correct, total) are summed on the host.
    Integer counts, so the accuracy equals the single-net evaluate() exactly."""
    if len(nets) == 1:
        return evaluate(nets[0], ctx)
    for n in nets:
        n.set_validation_data(SequentialBatchIterator(ctx.eval_data, ctx.batch))
    for k, n in enumerate(nets):
        n.test_begin(ctx.eval_steps, k, len(nets))
    correct = total = 0
    for n in nets:
        c, t = n.test_end()
        correct += c
        total += t
    return correct / total


def _make_serial_net(ctx: SchemeContext, device: int) -> Net:
    """schemes.hpp:141-147: one net, worker 0's iterator over a single shard."""
    net = Net(ctx.net, ctx.seed, device, ctx.precision)
    net.set_sgd(ctx.sgd)
    shards = shard(ctx.train_data, 1, ctx.seed)
    net.set_training_data(make_worker_iterator(shards, 0, ctx.batch, ctx.seed))
    return net


def run_serial(ctx: SchemeContext, iter_budget: int, eval_every: int,
               observer: Optional[SchemeObserver] = None) -> RunTrace:
    """schemes.hpp:154-193: serial SGD, evaluation every eval_every steps."""
    ctx.validate()
    if eval_every < 1:
        raise ValueError("run_serial: eval_every must be >= 1")
    if iter_budget < 0:
        raise ValueError("run_serial: negative budget")
    net = _make_serial_net(ctx, (ctx.devices or [0])[0])
    trace = RunTrace("serial", 1, 0, ctx.batch, ctx.sgd.learning_rate, ctx.seed,
                     ctx.target_accuracy, ctx.cost)
    clock = SimClock()
    iters = 0
    while iters < iter_budget:
        chunk = min(eval_every, iter_budget - iters)
        if observer is not None and observer.on_step is not None:
            for s in range(chunk):
                net.train(1)
                observer.on_step(iters + s + 1, net)
        else:
            net.train(chunk)
        iters += chunk
        clock.advance_to(serial_sim_time(iters, ctx.cost))
        acc = evaluate(net, ctx)
        trace.records.append(EvalRecord(iters, 0, 0, clock.elapsed(), acc))
        if acc >= ctx.target_accuracy:
            trace.outcome = TARGET_REACHED
            return trace
    trace.outcome = BUDGET_EXHAUSTED
    return trace


def run_naive(ctx: SchemeContext, workers: int, iter_budget: int, eval_every: int,
              observer: Optional[SchemeObserver] = None) -> RunTrace:
    """schemes.hpp:201-262 on B200s: every size-b batch is split into K parts; part k's
    forward/backward runs on worker k (GPU k, or K nets on one GPU), the K part gradients
    are averaged (weights_mean: NCCL allreduce across GPUs, or the ordered device kernel),
    and every replica applies the same SGD update, so all replicas stay identical to the
    reference's single net.  trace.round_ms holds the measured device time per step."""
    ctx.validate()
    if workers < 1:
        raise ValueError("run_naive: need at least one worker")
    if ctx.batch % workers != 0:
        raise ValueError("run_naive: worker count must divide the batch size")
    if eval_every < 1:
        raise ValueError("run_naive: eval_every must be >= 1")
    if iter_budget < 0:
        raise ValueError("run_naive: negative budget")
    devices = ctx.devices or [0]
    if len(devices) > 1 and len(devices) != workers:
        raise ValueError("run_naive: use one device, or one device per worker")
    shards = shard(ctx.train_data, 1, ctx.seed)
    nets = []
    for k in range(workers):
        n = Net(ctx.net, ctx.seed, devices[k % len(devices)], ctx.precision)
        n.set_sgd(ctx.sgd)
        # every part net walks the same batch stream (worker 0's iterator over one shard)
        n.set_training_part(make_worker_iterator(shards, 0, ctx.batch, ctx.seed), k, workers)
        nets.append(n)
    comms = None
    if len(devices) > 1:
        from .comm import Communicator
        comms = Communicator.create_all([n.ctx for n in nets])
    trace = RunTrace("naive", workers, 0, ctx.batch, ctx.sgd.learning_rate, ctx.seed,
                     ctx.target_accuracy, ctx.cost)
    clock = SimClock()
    iters = 0
    while iters < iter_budget:
        chunk = min(eval_every, iter_budget - iters)
        nets[0].event_record(0)
        for _ in range(chunk):
            for n in nets:
                n.grad_step()
            if comms is None:
                average_grads_local(nets)
            else:
                Communicator.average_grads(comms, nets, ctx.average_mode)
            for n in nets:
                n.apply_grads()
            iters += 1
            if observer is not None and observer.on_step is not None:
                for n in nets:
                    n.sync()
                observer.on_step(iters, nets[0])
        nets[0].event_record(1)
        for n in nets:
            n.sync()
        trace.round_ms.append(nets[0].event_elapsed(0, 1) / chunk)
        clock.advance_to(naive_sim_time(iters, ctx.cost, workers))
        acc = evaluate_sharded(nets, ctx) if comms is not None else evaluate(nets[0], ctx)
        trace.records.append(EvalRecord(iters, 0, iters, clock.elapsed(), acc))
        if acc >= ctx.target_accuracy:
            trace.outcome = TARGET_REACHED
            return trace
    trace.outcome = BUDGET_EXHAUSTED
    return trace


def run_sparknet(ctx: SchemeContext, workers: int, tau: int, round_budget: int,
                 warm_start_iters: int, threads: int = 1,
                 observer: Optional[SchemeObserver] = None, evaluate_rounds: bool = True
                 ) -> RunTrace:
    """schemes.hpp:274-351 on B200s."""
    ctx.validate()
    if workers < 1:
        raise ValueError("run_sparknet: need at least one worker")
    if tau < 1:
        raise ValueError("run_sparknet: tau must be >= 1")
    if round_budget < 0:
        raise ValueError("run_sparknet: negative budget")
    if warm_start_iters < 0:
        raise ValueError("run_sparknet: negative warm start")
    shards = shard(ctx.train_data, workers, ctx.seed)
    for s in shards:
        if s.size() < ctx.batch:
            raise ValueError("run_sparknet: shard smaller than the batch size")
    devices = ctx.devices or [0]
    if len(devices) > 1 and len(devices) != workers:
        raise ValueError("run_sparknet: use one device, or one device per worker")

    master = Net(ctx.net, ctx.seed, devices[0], ctx.precision)
    master.set_sgd(ctx.sgd)
    nets, streams = [], []
    for k in range(workers):
        n = Net(ctx.net, ctx.seed, devices[k % len(devices)], ctx.precision)
        n.set_sgd(ctx.sgd)
        it = make_worker_iterator(shards, k, ctx.batch, ctx.seed)
        n.set_training_data(it)
        nets.append(n)
        streams.append(it)

    trace = RunTrace("sparknet", workers, tau, ctx.batch, ctx.sgd.learning_rate, ctx.seed,
                     ctx.target_accuracy, ctx.cost, warm_start_iters)
    # schemes.hpp:312-317: the warm start consumes worker 0's shared stream
    master.set_training_data(streams[0])
    master.train(warm_start_iters)
    current = master.get_weights_flat()
    trace.warm_digest = master.get_weights().digest()

    comms = None
    if len(devices) > 1:
        from .comm import Communicator
        comms = Communicator.create_all([n.ctx for n in nets])
    clock = SimClock()
    for n in nets:  # round-1 broadcast of the warm-start weights
        n.set_weights_flat(current)
    for rnd in range(1, round_budget + 1):
        t0 = time.perf_counter()
        for n in nets:
            n.train(tau, sync=False)
        for n in nets:
            n.sync()
        t1 = time.perf_counter()
        if comms is None:
            average_local(nets)
        else:
            Communicator.average(comms, nets, ctx.average_mode)
        for n in nets:
            n.sync()
        t2 = time.perf_counter()
        trace.compute_ms.append((t1 - t0) * 1e3)
        trace.sync_ms.append((t2 - t1) * 1e3)
        trace.round_ms.append((t2 - t0) * 1e3)
        master.set_weights_flat(nets[0].get_weights_flat())
        clock.advance_to(sparknet_sim_time(rnd, tau, warm_start_iters, ctx.cost))
        if not evaluate_rounds:
            acc = 0.0
        elif comms is not None:  # every worker holds the average: shard the eval batches
            acc = evaluate_sharded(nets, ctx)
        else:
            acc = evaluate(master, ctx)
        trace.records.append(EvalRecord(warm_start_iters, tau * rnd, rnd, clock.elapsed(), acc))
        if observer is not None and observer.on_round is not None:
            observer.on_round(rnd, master.get_weights())
        if evaluate_rounds and acc >= ctx.target_accuracy:
            trace.outcome = TARGET_REACHED
            return trace
    trace.outcome = BUDGET_EXHAUSTED
    return trace
