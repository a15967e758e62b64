"""Condense `ncu --set full` reports into a markdown table (profiles/<round>/ncu_*.md).

  python tools/ncu_summary.py out.md label1=report1.ncu-rep [label2=report2.ncu-rep ...]
  python tools/ncu_summary.py out.md label=raw.csv

A `.csv` argument is an `ncu -i REP --page raw --csv` export (tools/gpu_ncu_full.sh writes
one on the GPU box; the report itself is often too large to bring back).
"""
import csv
import io
import subprocess
import sys

METRICS = [
    ("time_us", "gpu__time_duration.sum", 1e-3),
    ("tensor_%", "sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed", 1),
    ("sm_%", "sm__throughput.avg.pct_of_peak_sustained_elapsed", 1),
    ("l2_%", "lts__t_sectors.avg.pct_of_peak_sustained_elapsed", 1),
    ("dram_%", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", 1),
    ("dram_MB", "dram__bytes_read.sum", 1e-6),
    ("dram_w_MB", "dram__bytes_write.sum", 1e-6),
    ("tma_ld_TB/s", "l1tex__m_xbar2l1tex_read_bytes_mem_global_op_tma_ld.sum.per_second", 1e-12),
]


UNIT = {"ns": 1.0, "nsecond": 1.0, "us": 1e3, "usecond": 1e3, "ms": 1e6, "msecond": 1e6,
        "byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9,
        "byte/s": 1.0, "Kbyte/s": 1e3, "Mbyte/s": 1e6, "Gbyte/s": 1e9, "Tbyte/s": 1e12,
        "byte/second": 1.0, "Gbyte/second": 1e9, "Tbyte/second": 1e12}


def rows(path):
    if path.endswith(".csv"):  # raw-page export with a units row (not base units)
        r = list(csv.reader(open(path)))
        head, units = r[0], r[1]
        for row in r[2:]:
            fixed = []
            for v, u in zip(row, units):
                try:
                    fixed.append(str(float(v.replace(",", "")) * UNIT.get(u, 1.0)))
                except ValueError:
                    fixed.append(v)
            yield from _rec(head, fixed)
        return
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv", "--print-units", "base"],
                         capture_output=True, text=True, check=True).stdout
    r = list(csv.reader(io.StringIO(out)))
    head = r[0]
    for row in r[2:]:
        yield from _rec(head, row)


def _rec(head, row):
    d = dict(zip(head, row))
    rec = {"kernel": d.get("Kernel Name", "?").split("(")[0].replace("void ", ""),
           "grid": d.get("Grid Size", ""), "block": d.get("Block Size", "")}
    for key, metric, scale in METRICS:
        v = d.get(metric, "")
        if not v:  # some sections prefix the metric (e.g. "TPC.TriageCompute.")
            v = next((d[k] for k in head if k.endswith("." + metric) and d[k]), "")
        try:
            rec[key] = float(v.replace(",", "")) * scale
        except ValueError:
            rec[key] = None
    yield rec


def main():
    out = sys.argv[1]
    args = sys.argv[2:]
    lines = ["| report | kernel | grid | " + " | ".join(k for k, _, _ in METRICS) + " |",
             "|---|---|---|" + "---|" * len(METRICS)]
    for arg in args:
        label, path = arg.split("=", 1)
        for rec in rows(path):
            vals = " | ".join("-" if rec[k] is None else f"{rec[k]:.3g}" for k, _, _ in METRICS)
            lines.append(f"| {label} | {rec['kernel'][-40:]} | {rec['grid']} | {vals} |")
    with open(out, "w") as f:
        f.write("\n".join(lines) + "\n")
    print("\n".join(lines))


if __name__ == "__main__":
    main()
