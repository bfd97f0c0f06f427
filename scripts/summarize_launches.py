"""Summarise an ncu --metrics gpu__time_duration.sum launch list (csv) by kernel:
launches, total ms and share (cold-cache, serialised: compare SHARES, not absolutes)."""
import csv
import sys
from collections import defaultdict

rows = [r for r in csv.reader(open(sys.argv[1])) if r]
hdr_i = next(i for i, r in enumerate(rows) if "Kernel Name" in r and "Metric Value" in r)
hdr = rows[hdr_i]
tot = defaultdict(float)
cnt = defaultdict(int)
for r in rows[hdr_i + 1:]:
    d = dict(zip(hdr, r))
    if d.get("Metric Name") != "gpu__time_duration.sum":
        continue
    name = d["Kernel Name"]
    short = name.split("(")[0].replace("void ", "")[:90]
    val = float(d["Metric Value"].replace(",", ""))
    unit = d.get("Metric Unit", "ns")
    ms = val / 1e6 if unit == "ns" else (val / 1e3 if unit in ("us", "usecond") else val)
    tot[short] += ms
    cnt[short] += 1
T = sum(tot.values())
print(f"launches: {sum(cnt.values())}, total {T:.2f} ms")
for k, v in sorted(tot.items(), key=lambda kv: -kv[1])[:30]:
    print(f"{100 * v / T:6.2f}%  {v:9.3f} ms  {cnt[k]:6d}x  {k}")
