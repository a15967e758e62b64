"""Weight-averaging sweep over NCCL / NVLink (BASELINE.json config 5): flat fp32 buffers of
1-250 MB averaged across the ranks of one box, fast (ncclAllReduce ncclAvg) and ordered
(all-to-all + ascending-k fp64 reduction + allgather) modes.  Checks every result against
the host-side weights_mean of all ranks' inputs (ordered mode: bit-exact).

    python -m torch.distributed.run --nproc-per-node N --master-addr 127.0.0.1 \
        tools/avg_sweep.py [--sizes-mb 1,4,16,64,128,250] [--reps 5]
"""
import argparse
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--sizes-mb", default="1,4,16,64,128,250")
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--check-max-mb", type=float, default=16.0)
    args = ap.parse_args()
    import torch.distributed as dist
    dist.init_process_group("gloo")
    rank, world = dist.get_rank(), dist.get_world_size()
    local = int(os.environ.get("LOCAL_RANK", rank))
    from paper_1511_06051_b200.comm import Communicator, FlatBuffer, unique_id
    from paper_1511_06051_b200.model import Context
    ctx = Context.get(local)
    obj = [unique_id() if rank == 0 else None]
    dist.broadcast_object_list(obj, src=0)
    comm = Communicator.create(ctx, world, rank, obj[0])
    for mb in [float(x) for x in args.sizes_mb.split(",")]:
        n = int(mb * 1e6 / 4) // (4 * 840) * (4 * 840)  # ordered slices: 4-aligned, K | 840
        buf = FlatBuffer(ctx, n)
        for mode in ("fast", "ordered"):
            times = []
            for r in range(args.reps + 1):
                buf.fill_uniform(1000 + rank, -1.0, 1.0)
                ms = FlatBuffer.average([comm], [buf], mode)
                if r:
                    times.append(ms)
            worst = None
            if mb <= args.check_max_mb:
                buf.fill_uniform(1000 + rank, -1.0, 1.0)
                mine = buf.read()
                FlatBuffer.average([comm], [buf], mode)
                got = buf.read()
                import torch
                allv = [torch.zeros(n, dtype=torch.float32) for _ in range(world)]
                dist.all_gather(allv, torch.from_numpy(mine))
                acc = np.zeros(n, np.float64)
                for v in allv:  # weights.hpp:101 ascending order
                    acc += v.numpy().astype(np.float64)
                want = (acc / world).astype(np.float32)
                worst = float(np.max(np.abs(got.astype(np.float64) - want)) /
                              max(1e-30, float(np.max(np.abs(want)))))
                if mode == "ordered" and not np.array_equal(got, want):
                    raise SystemExit(f"ordered average not bit-exact at {mb} MB: {worst}")
            t = np.array(times)
            tmax = [0.0]
            import torch
            tt = torch.tensor([float(np.median(t))], dtype=torch.float64)
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
            tmax = float(tt.item())
            bus = 2.0 * (world - 1) / world * n * 4
            if rank == 0:
                print(json.dumps({"mb": round(n * 4 / 1e6, 3), "ranks": world, "mode": mode,
                                  "ms": tmax, "bus_gbs": bus / (tmax * 1e-3) / 1e9 if tmax else 0,
                                  "max_rel_dev": worst}), flush=True)
        del buf
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
