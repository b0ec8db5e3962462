"""Per-instruction stall samples from an ncu report (first kernel launch):
usage: python tools/sass_hot.py report.ncu-rep [min_pct]"""
import csv, io, subprocess, sys

rep = sys.argv[1]
thr = float(sys.argv[2]) if len(sys.argv) > 2 else 0.8
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(txt)))
hdr = rows[1]
ix = {h: i for i, h in enumerate(hdr)}
data = []
for r in rows[2:]:
    if len(r) != len(hdr) or not r[0].startswith("0x"):
        if data:
            break
        continue
    data.append(r)
S = "Warp Stall Sampling (All Samples)"
tot = sum(int(r[ix[S]]) for r in data)
ex = sum(int(r[ix["Instructions Executed"]]) for r in data)
print("instructions", len(data), "samples", tot, "warp-inst executed", ex)
reasons = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
for n, r in enumerate(data):
    s = int(r[ix[S]])
    if 100 * s / tot >= thr:
        top = sorted(((int(r[ix[k]]), k[6:]) for k in reasons), reverse=True)[:2]
        print(f"{n:5d} {100*s/tot:5.1f}%  {r[1][:60]:60s} {top}")
