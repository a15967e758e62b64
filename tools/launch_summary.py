"""Summarise an ncu `--metrics gpu__time_duration.sum --csv` launch list: per-kernel totals
and (with --tail N) the last N launches in order (one training step).  Times are cold-cache,
serialised replays: use them for shares, not absolutes."""
import argparse
import collections
import csv
import io


def load(path):
    with open(path) as f:
        text = f.read()
    start = text.find('"ID"')
    rows = []
    for r in csv.DictReader(io.StringIO(text[start:])):
        if r.get("Metric Name") != "gpu__time_duration.sum":
            continue
        v = float(r["Metric Value"].replace(",", ""))
        unit = r["Metric Unit"]
        us = v * {"ns": 1e-3, "nsecond": 1e-3, "ms": 1e3, "msecond": 1e3}.get(unit, 1.0)
        name = r["Kernel Name"].split("(")[0].split("<")[0].replace("void ", "")
        rows.append((int(r["ID"]), name, us, r.get("Grid Size", ""), r.get("Block Size", "")))
    return rows


def main():
    p = argparse.ArgumentParser()
    p.add_argument("csv")
    p.add_argument("--tail", type=int, default=0)
    a = p.parse_args()
    rows = load(a.csv)
    tot = collections.defaultdict(lambda: [0, 0.0])
    for _, n, us, _, _ in rows:
        tot[n][0] += 1
        tot[n][1] += us
    print(f"{len(rows)} launches, {sum(r[2] for r in rows):.1f} us total")
    for n, (c, us) in sorted(tot.items(), key=lambda kv: -kv[1][1]):
        print(f"  {us:10.1f} us  {c:5d}x  {n}")
    if a.tail:
        print(f"last {a.tail} launches:")
        for i, n, us, gr, bl in rows[-a.tail:]:
            print(f"  {i:5d} {us:9.1f} us  {n:28s} grid{gr} block{bl}")


if __name__ == "__main__":
    main()
