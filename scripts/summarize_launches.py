"""Summarise an `ncu --metrics gpu__time_duration.sum --csv` launch list: share per kernel.

    python scripts/summarize_launches.py gpurun_out/launches.csv "title" > profiles/rN_launches.txt
"""

import collections
import csv
import sys

UNIT = {"ns": 1e-6, "nsecond": 1e-6, "us": 1e-3, "usecond": 1e-3, "ms": 1.0, "msecond": 1.0, "s": 1e3, "second": 1e3}


def main(path, title=""):
    lines = [l for l in open(path) if l.startswith('"')]
    agg = collections.defaultdict(lambda: [0, 0.0])
    for row in csv.DictReader(lines):
        if row.get("Metric Name") != "gpu__time_duration.sum":
            continue
        ms = float(row["Metric Value"].replace(",", "")) * UNIT[row["Metric Unit"]]
        name = row["Kernel Name"].split("(")[0][:80]
        agg[name][0] += 1
        agg[name][1] += ms
    tot = sum(v[1] for v in agg.values())
    print(title)
    print("(ncu --metrics gpu__time_duration.sum --clock-control none; cold-cache, serialised: compare SHARES)")
    print(f"launches: {sum(v[0] for v in agg.values())}, total {tot:.2f} ms")
    for name, (cnt, ms) in sorted(agg.items(), key=lambda kv: -kv[1][1])[:40]:
        print(f"{100 * ms / tot:6.2f}%  {ms:9.3f} ms  {cnt:6d}x  {name}")


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2] if len(sys.argv) > 2 else "")
