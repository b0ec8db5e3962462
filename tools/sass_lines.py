"""Join an ncu report's per-instruction counts (first kernel in the report)
with nvdisasm line info: warp-instructions executed and stall samples per
CUDA source line (profiling aid).
usage: python tools/sass_lines.py report.ncu-rep object.o mangled_kernel_substring [top]"""
import collections, csv, io, os, re, subprocess, sys, tempfile

rep, obj, fn = sys.argv[1], sys.argv[2], sys.argv[3]
top = int(sys.argv[4]) if len(sys.argv) > 4 else 30
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
base = int(data[0][0], 16)
cnt = {int(r[0], 16) - base: (int(r[ix["Instructions Executed"]]), int(r[ix["Warp Stall Sampling (All Samples)"]]))
       for r in data}
d = tempfile.mkdtemp()
subprocess.run(["cuobjdump", "-xelf", "all", os.path.abspath(obj)], cwd=d, capture_output=True)
cub = [f for f in os.listdir(d) if f.endswith(".cubin")][0]
sass = subprocess.run(["nvdisasm", "-g", "-c", os.path.join(d, cub)], capture_output=True, text=True).stdout
infn, line = False, None
agg = collections.Counter()
smp = collections.Counter()
for l in sass.splitlines():
    if l.startswith("//----") and ".text." in l:
        infn = fn in l
        continue
    if not infn:
        continue
    m = re.search(r'//## File "([^"]+)", line (\d+)', l)
    if m:
        line = os.path.basename(m.group(1)) + ":" + m.group(2)
        continue
    m = re.search(r"/\*([0-9a-f]{4,})\*/", l)
    if m and line:
        off = int(m.group(1), 16)
        if off in cnt:
            agg[line] += cnt[off][0]
            smp[line] += cnt[off][1]
tot, stot = sum(agg.values()), sum(smp.values())
print("warp-inst", tot, "samples", stot)
for k, v in agg.most_common(top):
    print(f"{k:28s} inst {100*v/tot:5.1f}%  stall {100*smp[k]/max(stot,1):5.1f}%")
