#!/usr/bin/env python
"""Summarise an ncu report per SASS loop region: instructions executed and
stall samples per innermost loop (found from backward branches)."""
import csv
import io
import re
import subprocess
import sys


def main(rep, kernel_regex=None):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr = rows[1]
    ai, si = hdr.index("Address"), hdr.index("Source")
    ie = hdr.index("Instructions Executed")
    ss = hdr.index("Warp Stall Sampling (All Samples)")
    ins = []
    for r in rows[2:]:
        if len(r) <= ie or not r[ai].startswith("0x"):
            continue
        ins.append((int(r[ai], 16), r[si].strip(), float(r[ie] or 0), float(r[ss] or 0)))
    base = ins[0][0]
    tot_i = sum(x[2] for x in ins)
    tot_s = sum(x[3] for x in ins)
    loops = []
    for a, src, _, _ in ins:
        m = re.search(r"BRA(?:\.\w+)*\s+(?:\S+,\s*)?(0x[0-9a-f]+)", src)
        if m:
            t = int(m.group(1), 16)
            # targets are relative to the function start in SASS text
            tt = t if t >= base else base + t
            if tt < a:
                loops.append((tt, a))
    print(f"total warp-instructions {tot_i:.3e}, stall samples {tot_s:.0f}")
    seen = set()
    for lo, hi in sorted(loops, key=lambda x: x[1] - x[0]):
        body = [x for x in ins if lo <= x[0] <= hi]
        key = (lo, hi)
        if key in seen or len(body) < 30:
            continue
        seen.add(key)
        i = sum(x[2] for x in body)
        s_ = sum(x[3] for x in body)
        lds = sum(1 for x in body if "LDS" in x[1])
        print(f"loop {lo - base:#07x}-{hi - base:#07x} len {len(body):4d} LDS {lds:3d} "
              f"inst {100 * i / tot_i:5.1f}%  stalls {100 * s_ / max(tot_s, 1):5.1f}%")


if __name__ == "__main__":
    main(*sys.argv[1:])
