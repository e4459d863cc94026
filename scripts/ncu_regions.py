"""Attribute an ncu report's warp-stall samples and executed instructions to SASS loop regions.

usage: python scripts/ncu_regions.py report.ncu-rep
Regions are the innermost backward-branch loops of the kernel (body ranges); everything else is
'straight-line'.  Prints samples% / inst% per region with the region's top stall reasons.
"""
import collections
import csv
import io
import re
import subprocess
import sys

rep = sys.argv[1]
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
h = rows[1]
ix = {k: i for i, k in enumerate(h)}
body = [r for r in rows[2:] if len(r) == len(h)]
base = int(body[0][ix["Address"]], 16)
ins = []
for r in body:
    a = int(r[ix["Address"]], 16) - base
    ins.append((a, r[ix["Source"]].strip(), float(r[ix["Warp Stall Sampling (All Samples)"]] or 0),
                float(r[ix["Instructions Executed"]] or 0), r))
reasons = [k for k in h if k.startswith("stall_") and "Not Issued" not in k]
loops = []
for i, (a, t, *_rest) in enumerate(ins):
    m = re.search(r"BRA(?:\.U)?(?:\.ANY)?\s+(?:!?U?P\w+,\s*)?0x([0-9a-f]+)", t)
    if m:
        tgt = int(m.group(1), 16) - base
        if 0 <= tgt < a:
            loops.append((tgt, a))
# innermost: sort by size, assign each instruction to the smallest loop containing it
loops.sort(key=lambda x: x[1] - x[0])
region = {}
for lo, hi in loops:
    for a, *_r in ins:
        if lo <= a <= hi and a not in region:
            region[a] = (lo, hi)
agg = collections.defaultdict(lambda: [0.0, 0.0, collections.Counter(), 0])
for a, t, smp, ex, r in ins:
    key = region.get(a, None)
    g = agg[key]
    g[0] += smp
    g[1] += ex
    g[3] += 1
    for k in reasons:
        try:
            g[2][k[6:]] += float(r[ix[k]] or 0)
        except ValueError:
            pass
ts = sum(v[0] for v in agg.values()) or 1
ti = sum(v[1] for v in agg.values()) or 1
print("region (SASS offsets)        n_instr samples%  inst%  top stalls")
for key, v in sorted(agg.items(), key=lambda kv: -kv[1][0]):
    if v[0] / ts < 0.005:
        continue
    name = "straight-line" if key is None else f"loop {key[0]:#x}-{key[1]:#x}"
    top = ", ".join(f"{k} {100 * x / max(v[0], 1):.0f}%" for k, x in v[2].most_common(4))
    print(f"{name:28s} {v[3]:6d}  {100 * v[0] / ts:6.1f}  {100 * v[1] / ti:6.1f}  {top}")
