"""Summarise a round's GPU evidence from gpurun_out/ into profiles/ (runs
here, no GPU): bench lines, the ncu launch list, the ncu --set full metrics of
each captured kernel, K3's DRAM traffic and the SASS mnemonics.
    python scripts/summarize_round.py r01"""
import collections
import csv
import io
import json
import os
import re
import shutil
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OUT = os.path.join(ROOT, "gpurun_out")
PROF = os.path.join(ROOT, "profiles")
METRICS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
           "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_sector_hit_rate.pct",
           "lts__t_sectors_srcunit_tex_op_read.sum", "lts__throughput.avg.pct_of_peak_sustained_elapsed",
           "sm__throughput.avg.pct_of_peak_sustained_elapsed", "launch__registers_per_thread", "launch__grid_size",
           "launch__shared_mem_per_block", "sm__inst_executed_pipe_tc.avg.pct_of_peak_sustained_active",
           "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum",
           "lts__t_bytes.sum"]
UNIT = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}


def short(name):
    name = re.sub(r"\(.*$", "", name.replace("void ", ""))
    return re.sub(r"\(int\)|\(bool\)", "", name)


def launches(tag, cfg):
    path = os.path.join(OUT, f"launches_{cfg}.csv")
    if not os.path.exists(path):
        return
    rows = list(csv.reader(open(path)))
    hdr = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
    h = rows[hdr]
    ki, mi, vi = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value")
    per = collections.defaultdict(list)
    for r in rows[hdr + 1:]:
        if len(r) > vi and r[mi] == "gpu__time_duration.sum" and "lynx::" in r[ki]:
            per[short(r[ki])].append(float(r[vi].replace(",", "")) / 1e3)  # ns -> us
    tot = sum(sum(v) for v in per.values())
    lines = [f"# ncu launch list (gpu__time_duration.sum, --clock-control none), round {tag[1:]}, config {cfg}",
             "# command: ncu --metrics gpu__time_duration.sum --clock-control none -c 300 --csv python bench.py "
             f"--steps 20 --warmup 3 --no-cpu-baseline --config {cfg}  (scripts/ncu_round.sh)",
             "# cold-cache, serialised replays: compare SHARES of the step, not absolutes",
             f"{'kernel':40s} {'launches':>9s} {'mean_us':>9s} {'min_us':>9s} {'share':>7s}"]
    for k, v in sorted(per.items(), key=lambda kv: -sum(kv[1])):
        lines.append(f"{k:40s} {len(v):9d} {sum(v) / len(v):9.2f} {min(v):9.2f} {100 * sum(v) / tot:6.1f}%")
    open(os.path.join(PROF, f"{tag}_launches_{cfg}.txt"), "w").write("\n".join(lines) + "\n")
    print("\n".join(lines))


def ncu_raw(rep):
    txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(txt)))
    h, units = rows[0], rows[1]
    out = []
    for r in rows[2:]:
        d = {"Kernel Name": r[h.index("Kernel Name")]}
        for m in METRICS:
            if m in h:
                i = h.index(m)
                d[m] = f"{r[i]} {units[i]}".strip()
        # the top warp-stall reasons (warps stalled per issued instruction)
        st = [(n.replace("smsp__average_warps_issue_stalled_", "").replace("_per_issue_active.ratio", ""),
               float(r[i] or 0)) for i, n in enumerate(h)
              if n.startswith("smsp__average_warps_issue_stalled_") and n.endswith("_per_issue_active.ratio")]
        d["top_stalls_per_issue"] = {n: round(v, 2) for n, v in sorted(st, key=lambda x: -x[1])[:6]}
        out.append(d)
    return out


def to_bytes(s):
    v, u = s.split()
    return float(v.replace(",", "")) * UNIT[u]


CAPTURES = [  # (report in gpurun_out/, what it holds)
    ("ffn_full.ncu-rep", "C2 (Mixtral-8x7B layer, T=32, latency drop 4): ffn_kernel"),
    ("ffn_pair_full.ncu-rep", "C5 (Mixtral-8x22B layer, T=256, latency drop 4): ffn_pair_kernel (MT=2)"),
    ("small_full.ncu-rep", "C2: fused front_kernel (K0+K1+K2) and combine_kernel (K4)"),
    ("ffn_c4_full.ncu-rep", "C4 (DeepSeek-MoE-16B, T=128, accuracy budget 16): ffn_kernel"),
    ("k01_c4_full.ncu-rep", "C4: router_route_kernel (K0 + routing) and route_select_group (K1)"),
]


def main():
    tag = sys.argv[1] if len(sys.argv) > 1 else "r02"
    for f in sorted(os.listdir(OUT)):
        if f.startswith("bench_") and f.endswith(".json") and os.path.getsize(os.path.join(OUT, f)):
            shutil.copy(os.path.join(OUT, f), os.path.join(PROF, f"{tag}_{f}"))
    for f in ("timeline_c2.json", "timeline_c4.json", "timeline_c5.json"):
        if os.path.exists(os.path.join(OUT, f)) and os.path.getsize(os.path.join(OUT, f)):
            shutil.copy(os.path.join(OUT, f), os.path.join(PROF, f"{tag}_{f}"))
    if os.path.exists(os.path.join(OUT, "timeline_stack.json")):
        shutil.copy(os.path.join(OUT, "timeline_stack.json"), os.path.join(PROF, f"{tag}_timeline_stack_c3.json"))
    for cfg in ("c2", "c4", "c5"):
        launches(tag, cfg)
    kernels = []
    for rep, what in CAPTURES:
        if os.path.exists(os.path.join(OUT, rep)):
            for k in ncu_raw(os.path.join(OUT, rep)):
                k["capture"] = what
                kernels.append(k)
    summary = {
        "what": "ncu --set full --clock-control none captures, round " + tag[1:],
        "commands": ["scripts/ncu_round.sh"],
        "note": "per-kernel times are cold-cache serialised replays; dram__bytes_read vs the algorithmic "
                "used-expert bytes shows each used expert streamed once; lts__t_sectors_srcunit_tex_op_read x 32 B "
                "= the L2 -> SM bytes (weights + activation tiles)",
        "kernels": kernels}
    json.dump(summary, open(os.path.join(PROF, f"{tag}_ncu_full_summary.json"), "w"), indent=1)
    # per-config K3 traffic: bench.py reports the capture of ITS config's FFN kernel
    traffic = {}
    for cfg, tag_cap, used, d, ff in (("c2", "C2", 4, 4096, 14336), ("c5", "C5", 4, 6144, 16384),
                                      ("c4", "C4", None, 2048, 1408)):
        ffn = next((k for k in kernels if "ffn_" in k["Kernel Name"] and k["capture"].startswith(tag_cap)), None)
        if ffn is None:
            continue
        rd, wr = to_bytes(ffn["dram__bytes_read.sum"]), to_bytes(ffn["dram__bytes_write.sum"])
        ent = {"dram_bytes_per_launch": rd + wr, "dram_read_bytes": rd, "dram_write_bytes": wr,
               "kernel": ffn["Kernel Name"],
               "source": f"ncu --set full, profiles/{tag}_ncu_full_summary.json ({ffn['capture']})"}
        if used is not None:
            ent["algorithmic_bytes_per_launch"] = used * 3 * d * ff * 2
        traffic[cfg] = ent
    json.dump(traffic, open(os.path.join(PROF, "ffn_traffic.json"), "w"), indent=1)
    print(json.dumps({k["Kernel Name"][:40]: k["gpu__time_duration.sum"] for k in kernels}, indent=1))
    sass = subprocess.run(["cuobjdump", "-sass", os.path.join(ROOT, "build", "ffn.o")], capture_output=True,
                          text=True).stdout
    ops = collections.Counter(m.group(1) for m in re.finditer(r"/\*[0-9a-f]{4,}\*/\s+(?:@!?U?P\w+\s+)?([A-Z][A-Za-z0-9_.]+)",
                                                               sass))
    keep = {o: c for o, c in ops.items() if re.match(r"UTC|UTMA|LDTM|SYNCS|HMMA", o)}
    lines = [f"# SASS evidence (cuobjdump -sass build/ffn.o, all ffn_kernel / ffn_pair_kernel instances), round {tag[1:]}",
             "# tcgen05.mma -> UTCHMMA (.2CTA = cta_group::2), tcgen05.ld -> LDTM, TMA -> UTMALDG, mbarriers -> SYNCS; "
             "no HMMA (legacy mma.sync) anywhere"]
    lines += [f"{c:7d} {o}" for o, c in sorted(keep.items(), key=lambda kv: -kv[1])]
    open(os.path.join(PROF, f"{tag}_sass_evidence.txt"), "w").write("\n".join(lines) + "\n")
    print("\n".join(lines))
    # compute-sanitizer summary lines
    san = [ln for tool in ("memcheck", "racecheck", "synccheck", "initcheck")
           for ln in open(os.path.join(OUT, f"sanitize_{tool}.log")).read().splitlines()
           if "SUMMARY" in ln] if os.path.exists(os.path.join(OUT, "sanitize_memcheck.log")) else []
    if san:
        open(os.path.join(PROF, f"{tag}_sanitize_summary.txt"), "w").write(
            "# compute-sanitizer over scripts/sanitize.py (all cases), tools memcheck racecheck synccheck initcheck\n"
            + "\n".join(san) + "\n")


if __name__ == "__main__":
    main()
