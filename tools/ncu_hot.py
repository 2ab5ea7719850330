"""Summarise an ncu source page (SASS) export: hottest instructions by stall samples."""
import csv, sys, subprocess
rep, kernel = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "-k", f"regex:{kernel}", "--launch-count", "1",
                      "--print-source", "sass"], capture_output=True, text=True).stdout.splitlines()
rows = list(csv.reader(out[1:]))
hdr = rows[0]
S = hdr.index("Warp Stall Sampling (All Samples)")
stalls = [i for i, h in enumerate(hdr) if h.startswith("stall_") and "Not Issued" not in h]
data = [r for r in rows[1:] if len(r) > S and r[S].isdigit()]
tot = sum(int(r[S] or 0) for r in data)
print("total samples", tot, "instructions", len(data))
agg = {}
for r in data:
    for i in stalls:
        agg[hdr[i]] = agg.get(hdr[i], 0) + int(r[i] or 0)
print("stall totals:", sorted(((v, k) for k, v in agg.items()), reverse=True)[:8])
data.sort(key=lambda r: -int(r[S] or 0))
for r in data[:top]:
    st = sorted(((int(r[i] or 0), hdr[i][6:]) for i in stalls), reverse=True)[:3]
    print(f"{int(r[S]):6d} {r[0][-5:]} {r[1][:60]:60s} {st}")
