"""Aggregate ncu per-SASS-instruction metrics by CUDA source line.

  python tools/ncu_lines.py <report.ncu-rep> <kernel-regex> <object.o> [top]

Uses the SASS source page of the report (instructions executed, stall
samples per instruction address) and `nvdisasm --print-line-info` on the
kernel's cubin (extracted from the object with cuobjdump) to map offsets to
lines.  Prints the hottest source lines.
"""
import csv
import os
import re
import subprocess
import sys
import tempfile

rep, kre, obj = sys.argv[1], sys.argv[2], sys.argv[3]
top = int(sys.argv[4]) if len(sys.argv) > 4 else 25
fnre = sys.argv[5] if len(sys.argv) > 5 else kre.split("|")[0]

out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "-k", f"regex:{kre}", "--launch-count", "1",
                      "--print-source", "sass"], capture_output=True, text=True).stdout.splitlines()
kname = out[0].split(",", 1)[1].strip().strip('"') if out else ""
rows = list(csv.reader(out[1:]))
hdr = rows[0]
A, S, I = hdr.index("Address"), hdr.index("Warp Stall Sampling (All Samples)"), hdr.index("Instructions Executed")
data = [r for r in rows[1:] if len(r) > I and r[I].isdigit()]
base = int(data[0][A], 16)
offs = [(int(r[A], 16) - base, int(r[I]), int(r[S] or 0), r[hdr.index("Source")]) for r in data]

# line info from the cubin
tmp = tempfile.mkdtemp()
subprocess.run(["cuobjdump", "-xelf", "all", os.path.abspath(obj)], cwd=tmp, capture_output=True)
cubins = [os.path.join(tmp, f) for f in os.listdir(tmp) if f.endswith(".cubin")]
mapping = {}
for cb in cubins:
    txt = subprocess.run(["nvdisasm", "--print-line-info", "-c", cb], capture_output=True, text=True).stdout
    cur_fn, cur_line = None, None
    for line in txt.splitlines():
        m = re.match(r"\s*\.text\.(\S+):", line)
        if m:
            cur_fn = m.group(1)
            continue
        m = re.search(r'//## File "([^"]+)", line (\d+)', line)
        if m:
            cur_line = f"{os.path.basename(m.group(1))}:{m.group(2)}"
            continue
        m = re.match(r"\s*/\*([0-9a-f]{4,})\*/", line)
        if m and cur_fn:
            mapping.setdefault(cur_fn, {})[int(m.group(1), 16)] = cur_line
cands = [f for f in mapping if re.search(fnre, f)]
fn = min(cands, key=lambda f: abs(len(mapping[f]) - len(offs)), default=None)
print("kernel:", kname[:100], "| cubin fn:", fn)
lm = mapping.get(fn, {})
agg = {}
for off, ie, st, src in offs:
    ln = lm.get(off, "?")
    a = agg.setdefault(ln, [0, 0])
    a[0] += ie
    a[1] += st
tot_i = sum(v[0] for v in agg.values())
tot_s = sum(v[1] for v in agg.values())
print(f"total warp-instructions {tot_i:,}  stall samples {tot_s:,}")
key = 1 if os.environ.get("BY_STALL") else 0
for ln, (ie, st) in sorted(agg.items(), key=lambda x: -x[1][key])[:top]:
    print(f"{ie:14,d} {100*ie/tot_i:5.1f}%  stalls {100*st/max(tot_s,1):5.1f}%  {ln}")
