"""Markdown table of bench lines: python tools/bench_table.py file.json ..."""
import json
import sys


def main():
    print("| workload | GPUs | τ | img/s | e2e img/s | ms/round | top op (frac of TF32 peak) "
          "| avg share | clocks |")
    print("|---|---|---|---|---|---|---|---|---|")
    for path in sys.argv[1:]:
        lines = [ln for ln in open(path).read().splitlines() if ln.startswith("{")]
        if not lines:
            continue
        d = json.loads(lines[-1])
        if d.get("impl") == "reference":
            continue
        cfg, roof = d["config"], d.get("roofline") or {}
        wa = d.get("weight_average") or {}
        clk = d.get("clocks") or {}
        print(f"| {cfg['workload']} b={cfg['per_worker_batch']} | {d['n_gpus']} | {cfg['tau']} "
              f"| {d['value']:,.0f} | {d['e2e']['value']:,.0f} | {d['ms_per_step']:.2f} "
              f"| {roof.get('kernel', '-')} ({roof.get('frac', 0):.3f}) "
              f"| {wa.get('share_of_round', 0) * 100:.2f}% "
              f"| {clk.get('sm_mhz', '-')} MHz {','.join(clk.get('reasons', []))} |")


if __name__ == "__main__":
    main()
