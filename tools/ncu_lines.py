"""Per-source-line instruction and stall shares of one kernel in an ncu
report captured with --import-source on (cuda,sass source view).
usage: python tools/ncu_lines.py report.ncu-rep UPDATES_PER_LAUNCH [TOP]"""
import csv, io, subprocess, sys

rep, upd = sys.argv[1], float(sys.argv[2])
top = int(sys.argv[3]) if len(sys.argv) > 3 else 40
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
cur, hdr, rows = None, None, []
for r in csv.reader(io.StringIO(txt)):
    if not r:
        continue
    if r[0] == "File Path":
        cur = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = r
        ie, st = hdr.index("Instructions Executed"), hdr.index("Warp Stall Sampling (All Samples)")
        continue
    if hdr and len(r) > ie and r[2] == "-" and r[ie].isdigit():
        rows.append((int(r[ie]), int(r[st] or 0), cur, r[0], r[1][:90]))
tot = sum(x[0] for x in rows) or 1
stot = sum(x[1] for x in rows) or 1
print(f"warp instructions per launch {tot:.4g}; per 32 updates {tot / (upd / 32):.1f}")
for x in sorted(rows, reverse=True)[:top]:
    print(f"{x[0] / tot * 100:5.1f}% inst {x[1] / stot * 100:5.1f}% stall  {x[2]}:{x[3]:<5s} {x[4]}")
print("-- by stall")
for x in sorted(rows, key=lambda x: -x[1])[:top // 2]:
    print(f"{x[0] / tot * 100:5.1f}% inst {x[1] / stot * 100:5.1f}% stall  {x[2]}:{x[3]:<5s} {x[4]}")
