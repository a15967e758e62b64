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


class NvLinkCounter:
    """NVML NVLink data counters of this rank's GPU (KiB transmitted / received over all
    links; NVML_FI_DEV_NVLINK_THROUGHPUT_DATA_TX / _RX): the NVLink bytes a timed region
    moved, measured by the hardware rather than inferred from the algorithm."""

    def __init__(self, device):
        self.ok = False
        try:
            import pynvml as nv
            nv.nvmlInit()
            vis = os.environ.get("CUDA_VISIBLE_DEVICES")
            phys = int(vis.split(",")[device]) if vis else device
            self.nv, self.h = nv, nv.nvmlDeviceGetHandleByIndex(phys)
            self.links = []
            for link in range(18):
                try:
                    if nv.nvmlDeviceGetNvLinkState(self.h, link):
                        self.links.append(link)
                except Exception:  # noqa: BLE001
                    pass
            self.read()
            self.ok = bool(self.links)
        except Exception:  # noqa: BLE001
            self.ok = False

    def read(self):
        nv = self.nv
        ids = []
        for link in self.links:
            ids += [(nv.NVML_FI_DEV_NVLINK_THROUGHPUT_DATA_TX, link),
                    (nv.NVML_FI_DEV_NVLINK_THROUGHPUT_DATA_RX, link)]
        vals = nv.nvmlDeviceGetFieldValues(self.h, ids)
        tx = rx = 0
        for i, v in enumerate(vals):
            if v.nvmlReturn != 0:
                continue
            x = v.value.ullVal
            if i % 2 == 0:
                tx += x
            else:
                rx += x
        return tx * 1024, rx * 1024

    def bytes_between(self, fn):
        """(tx, rx) bytes over all links while fn() runs (fn synchronises the device)."""
        if not self.ok:
            fn()
            return None
        a = self.read()
        fn()
        b = self.read()
        return b[0] - a[0], b[1] - a[1]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--sizes-mb", default="1,4,16,64,128,250")
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--check-max-mb", type=float, default=16.0)
    ap.add_argument("--nvml", action="store_true", help="NVML NVLink counters per size")
    args = ap.parse_args()
    import torch.distributed as dist
    import torch
    dist.init_process_group("gloo")
    rank, world = dist.get_rank(), dist.get_world_size()
    local = int(os.environ.get("LOCAL_RANK", rank))
    from paper_1511_06051_b200.comm import Communicator, FlatBuffer, unique_id
    from paper_1511_06051_b200.model import Context
    ctx = Context.get(local)
    obj = [unique_id() if rank == 0 else None]
    dist.broadcast_object_list(obj, src=0)
    comm = Communicator.create(ctx, world, rank, obj[0])
    nvl = NvLinkCounter(local) if args.nvml else None
    for mb in [float(x) for x in args.sizes_mb.split(",")]:
        n = int(mb * 1e6 / 4) // (4 * 840) * (4 * 840)  # ordered slices: 4-aligned, K | 840
        buf = FlatBuffer(ctx, n)
        for mode in ("fast", "ordered"):
            times = []
            nvl_bytes = []
            buf.fill_uniform(1000 + rank, -1.0, 1.0)
            FlatBuffer.average([comm], [buf], mode)  # warm-up
            dist.barrier()
            c0 = nvl.read() if nvl is not None and nvl.ok else None
            for r in range(args.reps):
                buf.fill_uniform(1000 + rank, -1.0, 1.0)
                buf.read()  # device idle, then all ranks enter the average together
                dist.barrier()
                times.append(FlatBuffer.average([comm], [buf], mode))
            if c0 is not None:  # counters read outside the timed averages (no rank skew)
                c1 = nvl.read()
                nvl_bytes.append(((c1[0] - c0[0]) / args.reps, (c1[1] - c0[1]) / args.reps))
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
            nv = None
            if nvl_bytes:  # this GPU's NVLink tx / rx per average (NVML counters), max over ranks
                tx = float(np.median([b[0] for b in nvl_bytes]))
                rx = float(np.median([b[1] for b in nvl_bytes]))
                tv = torch.tensor([tx, rx], dtype=torch.float64)
                dist.all_reduce(tv, op=dist.ReduceOp.MAX)
                tx, rx = float(tv[0]), float(tv[1])
                nv = {"tx_bytes": tx, "rx_bytes": rx, "tx_over_bus": tx / bus,
                      "tx_gbs": tx / (tmax * 1e-3) / 1e9 if tmax else 0}
            if rank == 0:
                print(json.dumps({"mb": round(n * 4 / 1e6, 3), "ranks": world, "mode": mode,
                                  "ms": tmax, "bus_gbs": bus / (tmax * 1e-3) / 1e9 if tmax else 0,
                                  "max_rel_dev": worst, "nvlink_nvml": nv}), flush=True)
        del buf
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
