"""SASS opcode census of the product library (cuobjdump -sass of every object
under paper_2502_01826_b200/lib): per kernel, instruction count and the
opcodes that show how the data moves (UBLKCP = cp.async.bulk, LDGSTS =
cp.async, SYNCS = mbarrier, UTMALDG = TMA tensor load, LDS/STS, SHFL) and what
computes (FFMA, FFMA2 = paired fp32 FMA, DFMA/DMUL/DADD, MUFU).

    python tools/sass_census.py > profiles/r2u_sass_census.txt
"""
import collections
import glob
import os
import re
import subprocess

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
KEYS = ["UBLKCP", "LDGSTS", "SYNCS", "UTMALDG", "LDG", "STG", "LDS", "STS", "SHFL", "ATOMG", "RED", "FFMA", "FFMA2", "FMUL", "FMUL2",
        "DFMA", "DMUL", "DADD", "MUFU", "BAR", "WARPSYNC"]


def demangle(n: str) -> str:
    try:
        return subprocess.run(["c++filt", n], capture_output=True, text=True).stdout.strip()
    except OSError:
        return n


def main():
    tot = collections.Counter()
    print("# SASS opcode census, sm_100a (cuobjdump -sass of paper_2502_01826_b200/lib/*.o)")
    print("# columns: kernel, instructions, " + ", ".join(KEYS))
    for obj in sorted(glob.glob(os.path.join(REPO, "paper_2502_01826_b200", "lib", "*.o"))):
        out = subprocess.run(["cuobjdump", "-sass", obj], capture_output=True, text=True).stdout
        arch = re.search(r"arch = (\S+)", out)
        print(f"\n## {os.path.basename(obj)} ({arch.group(1) if arch else '?'})")
        for block in out.split("Function : ")[1:]:
            name = demangle(block.split("\n", 1)[0].strip())
            ops = collections.Counter()
            n = 0
            for line in block.split("\n"):
                m = re.match(r"\s+/\*[0-9a-f]{4}\*/\s+(@!?U?P\w+\s+)?([A-Z0-9_]+)", line)
                if m:
                    op = m.group(2)
                    ops[op.split(".")[0]] += 1
                    n += 1
            tot.update(ops)
            short = re.sub(r"\(.*", "", name.replace("(anonymous namespace)::", "")).replace("void ", "")
            print(f"{short[:48]:48s} {n:6d} " + " ".join(f"{k}={ops[k]}" for k in KEYS if ops[k]))
    print("\n## library total: " + " ".join(f"{k}={tot[k]}" for k in KEYS if tot[k]))


if __name__ == "__main__":
    main()
