"""Turn a round's gpurun_out/ artifacts into tracked summaries under profiles/.

  python tools/summarize_profiles.py r1
writes profiles/<tag>_bench.json, <tag>_launches.txt (per-kernel share of the
step, cold-cache serialised ncu times), <tag>_ncu_full.txt (per-kernel
metrics + top stall reasons from the --set full capture).
"""
import csv
import json
import os
import subprocess
import sys

tag = sys.argv[1] if len(sys.argv) > 1 else "r1"
G = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "gpurun_out")
P = os.path.join(os.path.dirname(G), "profiles")
os.makedirs(P, exist_ok=True)


def last_json(path):
    try:
        return json.loads(open(path).read().strip().splitlines()[-1])
    except Exception:
        return None


bench = {k: last_json(os.path.join(G, f"{tag}_{k}.json")) for k in ("bench", "bench_cub")}
json.dump(bench, open(os.path.join(P, f"{tag}_bench.json"), "w"), indent=1)

# launch list: last step only (from the last k_project)
rows = list(csv.reader(open(os.path.join(G, f"{tag}_launches.csv"))))
hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
hdr = rows[hi]
K, V, MN = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Name")
names = [(r[K], float(r[V])) for r in rows[hi + 1:] if r[MN] == "gpu__time_duration.sum"]
proj = [i for i, (n, _) in enumerate(names) if "k_project" in n]
step = names[proj[-1]:]
tot = sum(v for _, v in step)
agg = {}
for n, v in step:
    key = n.split("(")[0].replace("void ", "").replace("<unnamed>::", "")
    agg.setdefault(key, [0.0, 0])
    agg[key][0] += v
    agg[key][1] += 1
with open(os.path.join(P, f"{tag}_launches.txt"), "w") as f:
    f.write(f"# ncu --metrics gpu__time_duration.sum --clock-control none, one bench step (cold-cache, serialised)\n")
    f.write(f"# {len(step)} launches, sum {tot/1e3:.1f} us\n")
    for k, (v, c) in sorted(agg.items(), key=lambda x: -x[1][0]):
        f.write(f"{v/1e3:9.1f} us {100*v/tot:5.1f}%  x{c:<3d} {k}\n")

# full capture
rep = os.path.join(G, f"{tag}_full.ncu-rep")
if os.path.exists(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    hdr, units = rows[0], rows[1]
    want = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "lts__t_bytes.sum",
            "l1tex__t_bytes.sum", "sm__warps_active.avg.pct_of_peak_sustained_active",
            "smsp__issue_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
            "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
            "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed",
            "lts__t_sector_hit_rate.pct", "l1tex__t_sector_hit_rate.pct", "launch__grid_size",
            "launch__block_size", "sm__inst_executed.sum"]
    traffic = {}
    for r in rows[2:]:
        kn = r[hdr.index("Kernel Name")].split("(")[0].replace("void ", "").replace("<unnamed>::", "").split("<")[0]
        try:
            byts = float(r[hdr.index("dram__bytes_read.sum")]) + float(r[hdr.index("dram__bytes_write.sum")])
            scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}[units[hdr.index("dram__bytes_read.sum")]]
        except (ValueError, KeyError):
            continue
        traffic.setdefault(kn, []).append(byts * scale)
    json.dump({k: sum(v) / len(v) for k, v in traffic.items()}, open(os.path.join(P, f"{tag}_traffic.json"), "w"),
              indent=1)
    with open(os.path.join(P, f"{tag}_ncu_full.txt"), "w") as f:
        f.write("# ncu --set full --clock-control none, kernels of one timed bench step\n")
        for r in rows[2:]:
            f.write("\n== " + r[hdr.index("Kernel Name")][:110] + "\n")
            for w in want:
                if w in hdr:
                    i = hdr.index(w)
                    f.write(f"   {w}: {r[i]} {units[i]}\n")
print("wrote", P)
