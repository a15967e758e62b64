"""Top SASS instructions by warp-stall samples from an `ncu --page source --csv
--print-source sass` export (gzip ok): python tools/ncu_src_top.py FILE [N]"""
import csv
import gzip
import io
import sys


def main(path, n=25):
    op = gzip.open if path.endswith(".gz") else open
    text = op(path, "rt").read()
    lines = text.splitlines()
    kname = lines[0]
    rows = [r for r in csv.DictReader(io.StringIO("\n".join(lines[1:])))
            if (r.get("Warp Stall Sampling (All Samples)") or "0").isdigit()]
    stalls = [k for k in rows[0] if k.startswith("stall_") and "Not Issued" not in k]
    tot = sum(int(r["Warp Stall Sampling (All Samples)"] or 0) for r in rows)
    print(kname[:110], "total samples", tot)
    rows.sort(key=lambda r: -int(r["Warp Stall Sampling (All Samples)"] or 0))
    for r in rows[:n]:
        s = int(r["Warp Stall Sampling (All Samples)"] or 0)
        top = sorted(((int(r[k] or 0), k[6:]) for k in stalls), reverse=True)[:3]
        print(f"{100 * s / tot:5.1f}% {r['Address'][-5:]} {r['Source'].strip()[:60]:60s} "
              + " ".join(f"{k}:{v}" for v, k in top if v))


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 25)
