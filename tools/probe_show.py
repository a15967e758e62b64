"""Side-by-side per-op times of tools/probe_env.sh runs: python tools/probe_show.py [prefix]"""
import glob
import json
import sys

pre = sys.argv[1] if len(sys.argv) > 1 else ""
fs = sorted(glob.glob(f"gpurun_out/pr_{pre}*.json"))
D = {f.split("pr_")[1][:-5]: {o["name"]: o["ms"] for o in json.load(open(f))["ops"]} for f in fs}
names = list(D)
base = D[names[0]]
print("op".ljust(22) + "".join(n[-16:].rjust(17) for n in names))
for o in sorted(base, key=lambda n: -base[n])[:int(sys.argv[2]) if len(sys.argv) > 2 else 18]:
    print(o[:22].ljust(22) + "".join(("%.3f" % D[n].get(o, 0)).rjust(17) for n in names))
print("total".ljust(22) + "".join(("%.3f" % sum(D[n].values())).rjust(17) for n in names))
for f in fs:
    try:
        line = open(f[:-5] + ".log").read().strip().splitlines()[-1]
        d = json.loads(line)
        print(f.split("pr_")[1][:-5], round(d["value"]), "e2e", round(d["e2e"]["value"]))
    except Exception as e:  # noqa: BLE001
        print(f, "no bench line", e)
