"""N > 1 paths.  CPU (gloo, world_size 2): the per-rank host logic bench.py and the
multi-process driver use — shard ownership (bit-exact, disjoint, covering), the
ncclUniqueId rendezvous over torch.distributed, max-over-ranks timing.  GPU (>= 2 devices,
torchrun): NCCL averaging, ordered mode bit-exact with weights_mean, and a 2-rank bench."""
import json
import os
import socket
import subprocess
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, out_dir):
    sys.path.insert(0, ROOT)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import torch
    import torch.distributed as dist
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from oracle.pyoracle import OracleLib
    from paper_1511_06051_b200.data import Dataset, make_worker_iterator, shard
    n = 1003
    ds = Dataset(np.zeros((n, 1, 1, 1)), np.arange(n, dtype=np.int32) % 10, 10)
    mine = shard(ds, world, 7)[rank]
    want = OracleLib().shard(n, world, 7)[rank]
    ok_shard = bool(np.array_equal(mine.indices, want))
    parts = [None] * world
    dist.all_gather_object(parts, mine.indices.tolist())
    allidx = sorted(i for p in parts for i in p)
    ok_cover = allidx == list(range(n))
    it = make_worker_iterator(shard(ds, world, 7), rank, 9, 7)
    stream = np.concatenate([it.next_indices() for _ in range(30)])
    ok_stream = bool(np.array_equal(
        stream, OracleLib().worker_indices(n, world, rank, 9, 7, 30)))
    uid = [bytes(range(128)) if rank == 0 else None]
    dist.broadcast_object_list(uid, src=0)
    ok_uid = uid[0] == bytes(range(128))
    t = torch.tensor([float(rank + 1)], dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ok_max = float(t.item()) == float(world)
    with open(os.path.join(out_dir, f"r{rank}.json"), "w") as f:
        json.dump(dict(shard=ok_shard, cover=ok_cover, stream=ok_stream, uid=ok_uid,
                       max=ok_max), f)
    dist.destroy_process_group()


def test_two_rank_host_logic_gloo(tmp_path):
    import torch.multiprocessing as mp
    mp.start_processes(_worker, args=(2, _free_port(), str(tmp_path)), nprocs=2, join=True,
                       start_method="spawn")
    for r in range(2):
        res = json.load(open(tmp_path / f"r{r}.json"))
        assert all(res.values()), (r, res)


def _gpus():
    try:
        import torch
        return torch.cuda.device_count()
    except Exception:
        return 0


@pytest.mark.gpu
def test_nccl_average_two_ranks():
    if _gpus() < 2:
        pytest.skip("needs >= 2 GPUs")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", str(_free_port()),
           os.path.join(ROOT, "tools", "avg_sweep.py"), "--sizes-mb", "1,4,16", "--reps", "2"]
    out = subprocess.run(cmd, capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [json.loads(l) for l in out.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 6
    for l in lines:
        assert l["max_rel_dev"] is not None and l["max_rel_dev"] <= 1e-6


@pytest.mark.gpu
def test_bench_two_ranks():
    if _gpus() < 2:
        pytest.skip("needs >= 2 GPUs")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", str(_free_port()),
           os.path.join(ROOT, "bench.py"), "--gpus", "2", "--steps", "2", "--warmup", "1",
           "--tau", "2", "--average", "ordered"]
    out = subprocess.run(cmd, capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stderr[-2000:]
    line = json.loads([l for l in out.stdout.splitlines() if l.startswith("{")][-1])
    assert line["n_gpus"] == 2 and line["value"] > 0


@pytest.mark.gpu
@pytest.mark.parametrize("workload,tau", [("cifar10_quick", 1), ("cifar10_quick", 3)])
def test_overlapped_round_bitwise_equals_train_then_average(workload, tau):
    """psg_net_train_round (per-layer average buckets during the last backward) leaves
    weights and velocities bit-identical to train(tau) + one ncclAllReduce(avg) at K = 2."""
    if _gpus() < 2:
        pytest.skip("needs >= 2 GPUs")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", str(_free_port()),
           os.path.join(ROOT, "tools", "overlap_check.py"), "--workload", workload,
           "--tau", str(tau), "--rounds", "5"]
    out = subprocess.run(cmd, capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stderr[-3000:]
    res = json.loads([l for l in out.stdout.splitlines() if l.startswith("{")][-1])
    assert res["bitwise_equal"], res
