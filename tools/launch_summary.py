"""Summarise an `ncu --metrics gpu__time_duration.sum --csv` launch list:
per kernel and launch shape (template arguments kept, parameters dropped) the launch count,
mean duration and share of the listed GPU time.

    python tools/launch_summary.py gpurun_out/launches.csv > profiles/rNN_launches_summary.json
"""
import collections
import csv
import json
import sys


def kernel_key(name: str) -> str:
    depth = 0
    for i, ch in enumerate(name):  # cut at the parameter list: first '(' outside template brackets
        if ch == "<":
            depth += 1
        elif ch == ">":
            depth -= 1
        elif ch == "(" and depth == 0 and i > 0:
            name = name[:i]
            break
    return name.replace("void ", "").strip()


def main(path):
    rows = [r for r in csv.DictReader(l for l in open(path) if l.startswith('"'))
            if r.get("Metric Name") == "gpu__time_duration.sum"]
    dur = collections.defaultdict(list)
    for r in rows:
        v = float(r["Metric Value"].replace(",", ""))
        # same kernel at different grid sizes (full step vs e2e chunks) kept apart
        key = f'{kernel_key(r["Kernel Name"])} grid{r["Grid Size"]} block{r["Block Size"]}'
        dur[key].append(v * (1e3 if r["Metric Unit"] == "us" else 1.0))
    total = sum(sum(v) for v in dur.values())
    out = {k: {"launches": len(v), "mean_ns": sum(v) / len(v), "share_of_listed_time": sum(v) / total}
           for k, v in sorted(dur.items(), key=lambda kv: -sum(kv[1]))}
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main(sys.argv[1])
