"""Static loop census of a SASS listing (cuobjdump -sass): every backward branch
defines a loop [target, branch]; print its length and instruction mix, innermost
first.  Used to count per-row / per-move instructions of the scoring loops
before spending GPU time (profiles/r01/README.md)."""
from __future__ import annotations

import re
import sys
from collections import Counter

LINE = re.compile(r"/\*([0-9a-f]{4,})\*/\s+(@!?U?P\w+\s+)?([A-Z0-9_.]+)([^;]*);")


def parse(path):
    ins = []
    for ln in open(path):
        m = LINE.search(ln)
        if m:
            ins.append((int(m.group(1), 16), m.group(3), m.group(4)))
    return ins


def main(path, min_len=20):
    ins = parse(path)
    addr_idx = {a: i for i, (a, _, _) in enumerate(ins)}
    loops = []
    for i, (a, op, rest) in enumerate(ins):
        if op.startswith("BRA"):
            m = re.search(r"0x([0-9a-f]+)", rest)
            if m:
                tgt = int(m.group(1), 16)
                if tgt <= a and tgt in addr_idx:
                    loops.append((addr_idx[tgt], i))
    loops = sorted(set(loops), key=lambda x: x[1] - x[0])
    for lo, hi in loops:
        body = ins[lo:hi + 1]
        if len(body) < min_len:
            continue
        c = Counter(op.split(".")[0] for _, op, _ in body)
        top = ", ".join(f"{k} {v}" for k, v in c.most_common(12))
        print(f"loop 0x{ins[lo][0]:05x}-0x{ins[hi][0]:05x} len {len(body):5d}: {top}")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 20)
