"""Aggregates an SW_PROFILE_LOG dump (one line per timed launch) by GEMM shape/epilogue:
python tools/gemm_shape_report.py <log.csv> [steps]"""
import collections
import json
import sys


def main(path, steps=1):
    agg = collections.defaultdict(lambda: [0, 0.0, 0.0])
    other = collections.defaultdict(float)
    for ln in open(path):
        parts = ln.strip().split(",")
        cat, ms, work = int(parts[0]), float(parts[1]), float(parts[2])
        tag = ",".join(parts[3:])
        if tag.startswith("gemm"):
            a = agg[tag]
            a[0] += 1
            a[1] += ms
            a[2] += work
        else:
            other[cat] += ms
    rows = sorted(agg.items(), key=lambda kv: -kv[1][1])
    tot = sum(v[1] for v in agg.values())
    for tag, (n, ms, work) in rows:
        print(json.dumps({"gemm": tag[5:], "launches": n // steps, "ms_per_step": round(ms / steps, 3),
                          "share": round(ms / tot, 3), "tflops": round(work / ms / 1e9, 1)}))


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 1)
