"""Rewrite DESIGN.md's results table and README's headline numbers from profiles/r02_bench_*.json.
    python scripts/design_table.py"""
import json
import os
import re

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def load(f):
    return json.loads(open(os.path.join(ROOT, "profiles", f"r02_bench_{f}.json")).read().strip().splitlines()[-1])


def line(label, d, bold=False):
    ro = d.get("roofline", {})
    us = d.get("us_per_step", d.get("ms_per_step", 0) * 1e3)
    b = "**" if bold else ""
    st = ro.get("step_achieved_gbs", 0)
    return (f"| {label} | {b}{us:.1f}{b} | {b}{d['value']:,.0f}{b} | {ro.get('achieved', 0):.0f} "
            f"({ro.get('frac', 0):.2f} / {ro.get('frac_of_8TBs', 0):.2f}) | {st:.0f} ({st / 8000:.2f}) | "
            f"{d['e2e']['value']:,.0f} |\n")


def main():
    r = {f: load(f) for f in ["c2", "c2-unfused", "c2-nolynx", "c2-acc", "c3", "c4", "c5", "c5-bs32", "reference"]}
    c3, c2, ref = r["c3"], r["c2"], r["reference"]
    sw = c3["run"]["budget_sweep"]
    cpu, cpu2 = c2["cpu_baseline"], c2["cpu_baseline_f64_tanh2"]
    c3why = ", ".join(c3["clocks"]["reasons"]) or "no throttle reasons"
    table = (line("**C2** Mixtral-8x7B layer, T=32, Lynx latency drop 4 (4 used)", c2, True)
             + line("C2 with the K0/K1/K2 chain (`LYNX_FUSED_FRONT=0`)", r["c2-unfused"])
             + line("C2, no Lynx (8 used)", r["c2-nolynx"])
             + line("C2, Lynx accuracy policy (5.5 used avg)", r["c2-acc"])
             + f"| C3 32-layer decode step, B=64, budget 4 ({c3['clocks']['sm_mhz']:.0f} MHz, `{c3why}`) | "
               f"{c3['ms_per_step'] * 1e3:,.0f} | {c3['value']:,.0f} | — | {c3['roofline']['achieved']:.0f} "
               f"({c3['roofline']['achieved'] / 8000:.2f}) | {c3['e2e']['value']:,.0f} |\n"
             + "| C3 budget sweep 8/7/6/5/4 (ms/step) | "
             + " / ".join(f"{sw[k]['ms_per_step']:.2f}" for k in ["8", "7", "6", "5", "4"])
             + f" | Lynx 8→4: {sw['8']['ms_per_step'] / sw['4']['ms_per_step']:.2f}× | | | |\n"
             + line("C4 DeepSeek-MoE-16B, T=128, accuracy budget 16 (21.2 used incl. 2 shared)", r["c4"])
             + line("**C5** Mixtral-8x22B layer, decode batch 256 on one GPU (CTA pair, MT=2)", r["c5"], True)
             + line("C5 layer at 32 tokens (the per-GPU batch at EP8)", r["c5-bs32"])
             + f"| CPU: fp32 SwiGLU port of the reference path, C2, {cpu['cores']} host cores | "
               f"{cpu['ms_per_step'] * 1e3:,.0f} (bench C2 line) / {ref['ms_per_step'] * 1e3:,.0f} (`--impl reference`) | "
               f"{cpu['value']:.0f} / {ref['value']:.0f} | — | — | — |\n"
             + f"| CPU: the reference as shipped (f64 tanh2 experts), C2, {cpu2['cores']} cores | "
               f"{cpu2['ms_per_step'] * 1e3:,.0f} | {cpu2['value']:.0f} | — | — | — |\n")
    p = os.path.join(ROOT, "DESIGN.md")
    s = open(p).read()
    a = s.index("| **C2** Mixtral-8x7B layer, T=32")
    b = s.index("\n", s.index("| CPU: the reference as shipped")) + 1
    s = s[:a] + table + s[b:]
    s = re.sub(r"except C3 \(`sw_power_cap`,\n  \d+ MHz median", f"except C3 (`sw_power_cap`,\n  {c3['clocks']['sm_mhz']:.0f} MHz median", s)
    open(p, "w").write(s)
    print(table)


if __name__ == "__main__":
    main()
