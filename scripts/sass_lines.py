"""Profiling helper: join an ncu SASS source page (--page source --csv --print-source sass) with
nvdisasm line info of the same cubin -> per source line executed warp-instructions and stall
samples.  usage: sass_lines.py ncu_sass.csv kernel.cubin mangled_name [min_pct]"""
import collections
import csv
import re
import subprocess
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr, data = rows[1], rows[2:]
ix = {h: i for i, h in enumerate(hdr)}
S, E = ix["Warp Stall Sampling (All Samples)"], ix["Instructions Executed"]
dis = subprocess.run(["nvdisasm", "-gi", sys.argv[2]], capture_output=True, text=True).stdout
line = None
lines = []  # source line per instruction, in address order
inside = False
block = False
for ln in dis.splitlines():
    if ln.startswith("\t.section") or ln.startswith(".section") or ".text." in ln and ln.rstrip().endswith(":"):
        inside = (".text." + sys.argv[3]) in ln
        continue
    if not inside:
        continue
    if ln.strip().startswith("//##"):
        # a block of //## lines precedes each instruction group: the first is the innermost
        # source line ("... inlined at ..."); keep it plus the outermost call site
        f = re.findall(r'File "([^"]+)", line (\d+)', ln)
        if not block:
            inner = f[0][0].split("/")[-1] + ":" + f[0][1]
            line = inner + ("  <- " + f[-1][0].split("/")[-1] + ":" + f[-1][1] if len(f) > 1 else "")
            block = True
        continue
    block = False
    if re.match(r"\s+/\*[0-9a-f]{4,}\*/", ln):
        lines.append(line)
n = min(len(lines), len(data))
if len(lines) != len(data):
    print(f"warning: {len(lines)} disassembled vs {len(data)} profiled instructions", file=sys.stderr)
se, ss = collections.Counter(), collections.Counter()
for i in range(n):
    se[lines[i]] += int(data[i][E])
    ss[lines[i]] += int(data[i][S])
te, ts = sum(se.values()), sum(ss.values())
lim = float(sys.argv[4]) if len(sys.argv) > 4 else 0.5
for k in sorted(se, key=lambda k: -se[k]):
    if se[k] / te * 100 < lim and ss[k] / ts * 100 < lim:
        continue
    print(f"{k:50s} exec {se[k] / te * 100:5.1f}%  samples {ss[k] / ts * 100:5.1f}%")
