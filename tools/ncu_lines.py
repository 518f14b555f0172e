#!/usr/bin/env python
"""Per-CUDA-source-line instruction counts and stall samples of an ncu capture
(requires a library built from this tree so the line table resolves)."""
import csv
import sys
import subprocess

rep, top = sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 50
text = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                      capture_output=True, text=True).stdout
cur, hdr, out = None, None, []
for r in csv.reader(text.splitlines()):
    if not r:
        continue
    if r[0] == "File Path":
        cur = r[1].split("/")[-1]
        continue
    if r[0] == "Function Name":
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or len(r) < 8 or r[2] != "-":
        continue
    try:
        c = int(r[7])
    except ValueError:
        c = 0
    st = int(r[4]) if r[4].isdigit() else 0
    try:
        th = int(r[8])                      # thread instructions executed
    except (ValueError, IndexError):
        th = 0
    if c > 0:
        out.append((c, st, th, cur, r[0], r[1].strip()[:80]))
tot = sum(x[0] for x in out) or 1
tst = sum(x[1] for x in out) or 1
tth = sum(x[2] for x in out)
print(f"total warp instructions {tot}, stall samples {tst}, active lanes per instruction {tth / tot:.1f}")
for c, st, th, f, l, src in sorted(out, key=lambda x: -x[0])[:top]:
    print(f"{c / tot * 100:5.1f}% stall {st / tst * 100:5.1f}% lanes {th / c:4.1f}  {f}:{l:>4}  {src}")
