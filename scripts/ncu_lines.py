"""Per-source-line warp-stall samples of one kernel from an ncu --set full report.
    python scripts/ncu_lines.py <report.ncu-rep> <mangled kernel name> <obj.o> [--top N] [--ranges a-b,c-d]
Maps each SASS address (offset from the function start) to its source line with
nvdisasm -g of the object's cubin, sums the stall columns per line (barrier waits
listed apart: they are warps idling while others work)."""
import collections
import csv
import os
import re
import subprocess
import sys
import tempfile


def line_map(obj, fn):
    with tempfile.TemporaryDirectory() as d:
        subprocess.run(["cuobjdump", "-xelf", "all", os.path.abspath(obj)], cwd=d, check=True, capture_output=True)
        cub = [f for f in os.listdir(d) if f.endswith(".cubin")][0]
        sass = subprocess.run(["nvdisasm", "-g", "-fun", fn, os.path.join(d, cub)], capture_output=True,
                              text=True).stdout
    if not sass.strip():
        with tempfile.TemporaryDirectory() as d:
            subprocess.run(["cuobjdump", "-xelf", "all", os.path.abspath(obj)], cwd=d, check=True, capture_output=True)
            cub = [f for f in os.listdir(d) if f.endswith(".cubin")][0]
            sass = subprocess.run(["nvdisasm", "-g", os.path.join(d, cub)], capture_output=True, text=True).stdout
        i = sass.find(".text." + fn + ":")
        sass = sass[i:]
        j = sass.find(".section", 10)
        sass = sass[:j] if j > 0 else sass
    cur, m = None, {}
    for ln in sass.split("\n"):
        g = re.search(r'//## File "([^"]+)", line (\d+)', ln)
        if g:
            cur = (os.path.basename(g.group(1)), int(g.group(2)))
        g = re.search(r"/\*([0-9a-f]{4,})\*/\s+[A-Z@{]", ln)
        if g:
            m[int(g.group(1), 16)] = cur
    return m


def main():
    rep, fn, obj = sys.argv[1:4]
    top = int(sys.argv[sys.argv.index("--top") + 1]) if "--top" in sys.argv else 40
    kfilt = ["-k", "regex:" + sys.argv[sys.argv.index("--kernel") + 1]] if "--kernel" in sys.argv else []
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass", *kfilt],
                         capture_output=True, text=True).stdout.split("\n")
    rows = list(csv.reader(out))
    # skip "Kernel Name" lines and keep only the first kernel's table
    start = next(i for i, r in enumerate(rows) if r and r[0] == "Address")
    end = next((i for i in range(start + 1, len(rows)) if rows[i] and rows[i][0] in ("Kernel Name", "Address")),
               len(rows))
    rows = rows[start:end]
    hdr = rows[0]
    data = [r for r in rows[1:] if len(r) == len(hdr)]
    base = int(data[0][0], 16)
    lm = line_map(obj, fn)
    cols = [c for c in hdr if c.startswith("stall_") and "Not Issued" not in c]
    per = collections.defaultdict(collections.Counter)
    for r in data:
        off = int(r[0], 16) - base
        key = lm.get(off, ("?", 0))
        for c in cols:
            v = float(r[hdr.index(c)] or 0)
            if v:
                per[key][c] += v
        per[key]["inst"] += float(r[hdr.index("Instructions Executed")] or 0)
    tot = collections.Counter()
    for k, c in per.items():
        tot.update(c)
    work = {k: sum(v for n, v in c.items() if n.startswith("stall_") and n != "stall_barrier") for k, c in per.items()}
    allw = sum(work.values())
    print(f"samples excluding barrier waits: {allw:.0f}; barrier waits: {tot['stall_barrier']:.0f}")
    print("totals:", {n[6:]: int(v) for n, v in tot.most_common() if n.startswith("stall_")})
    if "--ranges" in sys.argv:
        for rg in sys.argv[sys.argv.index("--ranges") + 1].split(","):
            a, b = (int(x) for x in rg.split("-"))
            s = sum(v for k, v in work.items() if k[0] == "select.cu" and a <= k[1] <= b)
            print(f"select.cu {a}-{b}: {s:.0f} ({s / allw:.1%})")
    for k, v in sorted(work.items(), key=lambda kv: -kv[1])[:top]:
        c = per[k]
        reasons = ", ".join(f"{n[6:]} {int(x)}" for n, x in c.most_common(4) if n.startswith("stall_") and n != "stall_barrier")
        print(f"{v:7.0f} {v / allw:6.1%}  {k[0]}:{k[1]}  [{reasons}]")


if __name__ == "__main__":
    main()
