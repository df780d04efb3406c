"""Per-source-line instruction and stall breakdown of an ncu report (development aid)."""
import csv, subprocess, sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
extra = sys.argv[3:]          # e.g. --launch-skip 1 --launch-count 1
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass", *extra],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
per, tot, tots = [], 0, 0
hdr = None
for r in rows:
    if r and r[0] == "Line No":
        hdr = r
        iE = hdr.index("Instructions Executed")
        iS = hdr.index("Warp Stall Sampling (All Samples)")
        st = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
        continue
    if hdr is None or not r or not r[0] or len(r) <= iE or r[0] in ("File Path", "Function Name", "File Name"):
        continue
    try:
        n, smp = int(r[iE]), int(r[iS])
    except ValueError:
        continue
    tot += n
    tots += smp
    top3 = sorted(((int(r[hdr.index(h)] or 0), h[6:]) for h in st), reverse=True)[:3]
    per.append((smp, n, r[0], r[1][:80], top3))
per.sort(reverse=True)
print(f"total instr {tot}  samples {tots}")
for smp, n, ln, src, t3 in per[:top]:
    s3 = " ".join(f"{k}:{v}" for v, k in t3 if v)
    print(f"{smp / tots * 100:5.1f}%s {n / tot * 100:5.1f}%i L{ln:5s} {src:80s} {s3}")
