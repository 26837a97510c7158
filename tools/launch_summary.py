"""Per-kernel totals of an ncu launch list (`--metrics gpu__time_duration.sum --csv --log-file`):
python tools/launch_summary.py <launches.csv> [out.json]. ncu serialises launches and runs them
cold, so absolute times exceed the bench's; the SHARE of each kernel family is what is compared."""
import csv
import json
import re
import sys
from collections import defaultdict


def family(name):
    n = re.sub(r"\(.*", "", name)
    n = re.sub(r"^void ", "", n)
    n = n.replace("sw::", "").replace("<unnamed>::", "").replace("k::", "")
    return n.strip()


def main(path, out=None):
    rows = [r for r in csv.reader(open(path)) if len(r) > 10 and r[0].isdigit()]
    tot = defaultdict(lambda: [0, 0.0])
    for r in rows:
        if r[-3] != "gpu__time_duration.sum":
            continue
        us = float(r[-1].replace(",", "")) / (1000.0 if r[-2] == "ns" else 1.0)
        tot[family(r[4])][0] += 1
        tot[family(r[4])][1] += us
    all_us = sum(v[1] for v in tot.values())
    res = [{"kernel": k, "launches": v[0], "us": round(v[1], 1), "share": round(v[1] / all_us, 4)}
           for k, v in sorted(tot.items(), key=lambda kv: -kv[1][1])]
    for x in res:
        print(f"{x['share']*100:6.2f}%  {x['us']:10.1f} us  {x['launches']:5d}  {x['kernel']}")
    if out:
        json.dump({"source": path, "total_us": round(all_us, 1), "kernels": res}, open(out, "w"), indent=1)


if __name__ == "__main__":
    main(*sys.argv[1:])
