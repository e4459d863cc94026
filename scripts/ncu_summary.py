"""Summarise an ncu report: key metrics, warp-stall mix, and per-source-line hot spots.

usage: python scripts/ncu_summary.py report.ncu-rep [top_lines]
"""
import collections
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 25


def ncu(*args):
    return subprocess.run(["ncu", "-i", rep, *args], capture_output=True, text=True).stdout


rows = list(csv.reader(io.StringIO(ncu("--page", "raw", "--csv"))))
hdr, vals = rows[0], rows[2] if len(rows) > 2 else rows[1]
want = ["Kernel Name", "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
        "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active", "lts__t_sector_hit_rate.pct",
        "smsp__inst_executed.sum", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed", "local_load", "local_store"]
print("| metric | value |\n|---|---|")
for w in want:
    for i, h in enumerate(hdr):
        if h == w or (w in ("local_load", "local_store") and h.startswith("smsp__inst_executed_op_" + w) and h.endswith(".sum")):
            print(f"| {h} ({rows[1][i]}) | {vals[i]} |")
ss = []
for i, h in enumerate(hdr):
    if h.startswith("smsp__pcsamp_warps_issue_stalled") and not h.endswith("not_issued"):
        try:
            ss.append((float(vals[i].replace(",", "")), h.replace("smsp__pcsamp_warps_issue_stalled_", "")))
        except ValueError:
            pass
ss.sort(reverse=True)
T = sum(x for x, _ in ss) or 1
print("\nwarp-stall samples: " + ", ".join(f"{h} {100 * x / T:.1f}%" for x, h in ss[:9]))

cur, hdr2 = None, None
agg = collections.defaultdict(lambda: [0.0, 0.0])
src = {}
for row in csv.reader(io.StringIO(ncu("--page", "source", "--csv", "--print-source", "cuda,sass"))):
    if not row:
        continue
    if row[0] == "File Path":
        cur = row[1].split("/")[-1]
        continue
    if row[0] == "Function Name":
        continue
    if row[0] == "Line No":
        hdr2 = row
        continue
    if hdr2 is None:
        continue
    try:
        ln = int(row[0])
    except ValueError:
        continue
    d = dict(zip(hdr2[2:], row[2:]))

    def f(k):
        try:
            return float((d.get(k) or "0").replace(",", ""))
        except ValueError:
            return 0.0
    agg[(cur, ln)][0] += f("Warp Stall Sampling (All Samples)")
    agg[(cur, ln)][1] += f("Instructions Executed")
    src[(cur, ln)] = row[1]
ts = sum(v[0] for v in agg.values()) or 1
ti = sum(v[1] for v in agg.values()) or 1
print(f"\nper-source-line (top {top} by stall samples): file:line samples% inst% source")
for k, v in sorted(agg.items(), key=lambda kv: -kv[1][0])[:top]:
    print(f"  {k[0]}:{k[1]}  {100 * v[0] / ts:5.1f}%  {100 * v[1] / ti:5.1f}%  {src[k].strip()[:90]}")

# optional: SASS-level view -- the hottest instructions with their dominant stall reasons
if len(sys.argv) > 3 and sys.argv[3] == "--sass":
    nsass = int(sys.argv[4]) if len(sys.argv) > 4 else 40
    rows = list(csv.reader(io.StringIO(ncu("--page", "source", "--csv", "--print-source", "sass"))))
    h = rows[1]
    body = [r for r in rows[2:] if len(r) == len(h)]
    ix = {k: i for i, k in enumerate(h)}
    reasons = [k for k in h if k.startswith("stall_") and "Not Issued" not in k]
    tot = sum(float(r[ix["Warp Stall Sampling (All Samples)"]] or 0) for r in body) or 1
    print(f"\nSASS (top {nsass} by stall samples): addr samples% execs reasons")
    hot = sorted(range(len(body)), key=lambda i: -float(body[i][ix["Warp Stall Sampling (All Samples)"]] or 0))[:nsass]
    for i in sorted(hot):
        r = body[i]
        smp = float(r[ix["Warp Stall Sampling (All Samples)"]] or 0)
        rs = sorted(((float(r[ix[k]] or 0), k[6:]) for k in reasons), reverse=True)[:3]
        print(f"  {i:6d} {100 * smp / tot:5.2f}% {r[ix['Instructions Executed']]:>9s}  {r[1].strip()[:60]:60s} "
              + " ".join(f"{k}:{int(v)}" for v, k in rs if v > 0))
