"""Attribute ncu warp-stall samples / executed instructions of one kernel to source lines.

    ncu -i prof.ncu-rep --page source --csv --print-source sass > sass.csv
    cuobjdump -xelf all libkrecycle_b200.so   (in a scratch dir)
    python scripts/ncu_lines.py sass.csv kr_rminres.sm_100a.cubin <mangled-kernel-name> [top]
"""

import collections
import csv
import re
import subprocess
import sys


def main(sass_csv, cubin, fname, top=40):
    dis = subprocess.run(["nvdisasm", "--print-line-info", "-fun", fname, cubin], capture_output=True, text=True).stdout
    if not dis.strip():
        dis = subprocess.run(["nvdisasm", "--print-line-info", cubin], capture_output=True, text=True).stdout
    lines = dis.splitlines()
    start = next((i for i, l in enumerate(lines) if l.strip().startswith(f".text.{fname}")), 0)
    cur, insts = None, {}
    for l in lines[start:]:
        m = re.search(r'//## File "([^"]+)", line (\d+)', l)
        if m:
            cur = (m.group(1).split("/")[-1], int(m.group(2)))
            continue
        m = re.match(r"\s*/\*([0-9a-f]{4,})\*/\s+(.*)", l)
        if m and ";" in m.group(2):
            insts[int(m.group(1), 16)] = cur
        if l.strip().startswith(".section") and insts:
            break
    rows = list(csv.reader(open(sass_csv)))
    hdr, data = rows[1], rows[2:]
    i_s = hdr.index("Warp Stall Sampling (All Samples)")
    i_e = hdr.index("Instructions Executed")
    base = int(data[0][0], 16)
    samp, ex = collections.Counter(), collections.Counter()
    for r in data:
        c = insts.get(int(r[0], 16) - base)
        samp[c] += float(r[i_s] or 0)
        ex[c] += float(r[i_e] or 0)
    ts, te = sum(samp.values()), sum(ex.values())
    print(f"samples {ts:.0f}  instructions {te:.3g}")
    for c, v in samp.most_common(top):
        print(f"{100 * v / ts:5.1f}% stall-samples  {100 * ex[c] / te:5.1f}% inst   {c}")


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2], sys.argv[3], int(sys.argv[4]) if len(sys.argv) > 4 else 40)
