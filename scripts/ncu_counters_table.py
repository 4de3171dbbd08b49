"""ncu --csv (--metrics ...) log -> one markdown row per launch.
usage: python scripts/ncu_counters_table.py gpurun_out/r02_e0_counters.csv"""
import csv
import sys
from collections import OrderedDict


def main(path):
    rows = OrderedDict()
    with open(path) as f:
        lines = [ln for ln in f if ln.startswith('"')]
    for r in csv.DictReader(lines):
        key = (r["ID"], r["Kernel Name"][:60])
        rows.setdefault(key, {})[r["Metric Name"]] = (r["Metric Value"], r["Metric Unit"])
    metrics = []
    for v in rows.values():
        for m in v:
            if m not in metrics:
                metrics.append(m)
    print("| id | kernel | " + " | ".join(metrics) + " |")
    print("|" + "---|" * (len(metrics) + 2))
    for (i, k), v in rows.items():
        print(f"| {i} | `{k}` | " + " | ".join(f"{v.get(m, ('', ''))[0]} {v.get(m, ('', ''))[1]}".strip()
                                             for m in metrics) + " |")


if __name__ == "__main__":
    main(sys.argv[1])
