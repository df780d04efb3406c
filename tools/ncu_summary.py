"""Summarise an ncu report: SOL, occupancy, issue, stalls, instruction mix."""
import collections, csv, io, re, subprocess, sys

rep = sys.argv[1]
def run(*a):
    return subprocess.run(["ncu", "-i", rep, *a], capture_output=True, text=True).stdout
det = run("--page", "details", "--csv")
keys = ["Duration", "DRAM Throughput", "Memory Throughput", "Compute (SM) Throughput", "Registers Per Thread",
        "Achieved Occupancy", "Theoretical Occupancy", "Issue Slots Busy", "Eligible Warps Per Scheduler",
        "Issued Instructions", "Dynamic Shared Memory Per Block", "SM Frequency", "Block Limit Shared Mem",
        "Block Limit Registers", "Warp Cycles Per Issued Instruction"]
for row in csv.reader(io.StringIO(det)):
    if len(row) > 14 and row[12] in keys:
        print(f"{row[12]:40s} {row[14]:>14s} {row[13]}")
raw = list(csv.reader(io.StringIO(run("--page", "raw", "--csv"))))
h, v = raw[0], raw[2]
for name, val in zip(h, v):
    if name in ("dram__bytes_read.sum", "dram__bytes_write.sum") or (name.startswith("smsp__pcsamp_warps_issue_stalled") and not name.endswith("not_issued")):
        try:
            if float(val.replace(",", "")) > 0:
                print(f"{name:60s} {val}")
        except ValueError:
            pass
src = list(csv.reader(io.StringIO(run("--page", "source", "--csv", "--print-source", "sass"))))
hdr = src[1]
iE, iS = hdr.index("Instructions Executed"), hdr.index("Source")
ops = collections.Counter()
tot = 0
for r in src[2:]:
    if len(r) <= iE:
        continue
    try:
        n = int(r[iE])
    except ValueError:
        continue
    op = re.sub(r"^@!?U?P\w+\s+", "", r[iS].strip())
    ops[op.split()[0].split(".")[0] if op else "?"] += n
    tot += n
print("total warp instructions", tot)
print("  ".join(f"{k}:{v/tot*100:.1f}%" for k, v in ops.most_common(18)))
