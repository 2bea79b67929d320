"""Copy a round-profile run (gpurun_out/rp_*) into profiles/ and regenerate the
measured tables of DESIGN.md and BASELINE.md from it (tooling).

    python tools/refresh_docs.py            # after tools/gpu_round_profile.sh
"""

from __future__ import annotations

import json
import re
import shutil
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
OUT = ROOT / "gpurun_out"
PROF = ROOT / "profiles"


def copy_profiles():
    pairs = {"rp_configs.jsonl": "r01_configs.jsonl", "rp_bench.json": "r01_bench.json",
             "rp_launches.csv": "r01_launches.csv", "rp_loadbal.jsonl": "r01_loadbal.jsonl",
             "rp_shards.jsonl": "r01_shard_scaling.jsonl", "rp_pack.jsonl": "r01_pack.jsonl",
             "rp_shards_weighted.jsonl": "r01_shard_scaling_weighted.jsonl"}
    for src, dst in pairs.items():
        if (OUT / src).exists() and (OUT / src).stat().st_size:
            shutil.copy(OUT / src, PROF / dst)
    run = lambda *a: subprocess.run([sys.executable, *a], capture_output=True, text=True, cwd=ROOT).stdout
    (PROF / "r01_launches.txt").write_text(run("tools/launch_summary.py", str(PROF / "r01_launches.csv")))
    if (OUT / "rp_spmm.ncu-rep").exists():
        (PROF / "r01_spmm_ncu.txt").write_text(
            "# cfg2 SpMM A.4 (bench.py --profile), ncu --set full --clock-control none, round 1 final\n"
            + run("tools/ncu_summary.py", str(OUT / "rp_spmm.ncu-rep")))


def _rows():
    return [json.loads(l) for l in open(PROF / "r01_configs.jsonl") if l.startswith("{")]


def _replace_block(text: str, header: str, new_block: str) -> str:
    i = text.index(header)
    j = text.index("\n\n", i) + 1
    return text[:i] + new_block + text[j:]


def design_tables(d: str) -> str:
    rows = _rows()
    seen, order = {}, []
    for r in rows:
        key = (r["cfg"], r["kernel"], r["ms"])
        name = r["schedule"].split()[0]
        if key in seen:
            seen[key].append(name)
            continue
        seen[key] = [name]
        order.append((key, r))
    hdr = "| cfg | schedule | kernel | ms | GFLOP/s | frac of HBM roofline | max rel err |"
    lines = [hdr, "|---|---|---|---|---|---|---|"]
    for key, r in order:
        bold = r["cfg"] == 2 and r["kernel"] == "spmm_nnz"
        b = (lambda x: f"**{x}**") if bold else str
        lines.append(f"| {r['cfg']} | {b(' / '.join(seen[key]))} | {b(r['kernel'])} | {b(format(r['ms'], '.3f'))} | "
                     f"{b(format(round(r['gflops']), ','))} | {b(format(r['frac_hbm'], '.3f'))} | "
                     f"{r['max_rel_err']:.1e} |")
    d = _replace_block(d, hdr, "\n".join(lines) + "\n")
    lb = [json.loads(l) for l in open(PROF / "r01_loadbal.jsonl")]
    bases = list(dict.fromkeys(r["base"] for r in lb))
    sched = ["A8 warp-per-row", "A7 thread-per-row", "A2 pos-split"]
    hdr2 = "| base | max row | empty rows | A.8 warp-per-row ms | A.7 thread-per-row ms | A.2 pos-split ms |"
    L = [hdr2, "|---|---|---|---|---|---|"]
    for b in bases:
        rr = {r["schedule"]: r for r in lb if r["base"] == b}
        a = rr[sched[0]]
        L.append(f"| {b} | {a['max_row']:,} | {a['empty_rows']:,} | " + " | ".join(f"{rr[x]['ms']:.3f}" for x in sched)
                 + " |")
    d = _replace_block(d, hdr2, "\n".join(L) + "\n")
    sh = [json.loads(l) for l in open(PROF / "r01_shard_scaling.jsonl")]

    def srow(cfg, name):
        g = {r["gpus"]: r for r in sh if r["cfg"] == cfg}
        sp = g[8]["speedup_vs_1"]
        st = "**" if sp >= 6 else ""
        return (f"  | cfg{cfg} {name} | {g[1]['max_shard_ms']:.3f} ms | {g[2]['max_shard_ms']:.3f} ms | "
                f"{g[4]['max_shard_ms']:.3f} ms | {g[8]['max_shard_ms']:.3f} ms ({st}{sp:.2f}×{st}) |")

    new = "\n".join([srow(2, "SpMM A.4"), srow(5, "SpMV A.2"), srow(4, "MTTKRP A.6")]) + "\n"
    d = re.sub(r"  \| cfg2 SpMM A\.4 \|.*\n  \| cfg5 SpMV A\.2 \|.*\n  \| cfg4 MTTKRP A\.6 \|.*\n", lambda m: new, d)
    return d


def baseline_table(s: str) -> str:
    rows = _rows()
    get = lambda cfg, k: [r for r in rows if r["cfg"] == cfg and r["kernel"] == k][0]
    spec = [(1, "spmv_warp", "SpMV warp-per-row (A.8)"), (1, "spmv_nnz", "SpMV nnz-split (A.2/A.9)"),
            (2, "spmm_nnz", "**SpMM nnz-split (A.4)**"), (2, "spmm_row", "SpMM warp-per-row (K5)"),
            (3, "sddmm_nnz", "SDDMM nnz-split (K6)"), (3, "sddmm_row", "SDDMM row-split (K10)"),
            (4, "mttkrp_nnz", "MTTKRP nnz-split (A.6)"), (4, "mttkrp_slice", "MTTKRP slice-split (A.5/K9)"),
            (4, "ttv_fiber", "TTV fiber-split (K7)"), (4, "ttv_nnz", "TTV nnz-split (K11)"),
            (5, "spmv_nnz", "SpMV nnz-split (A.2/A.9)"),
            (5, "spmv_warp", "SpMV warp-per-row (A.8)"), (5, "spmv_row", "SpMV thread-per-row (A.7)")]
    b = json.load(open(PROF / "r01_bench.json"))
    cpu = b["cpu_baseline"]
    L = []
    for cfg, k, name in spec:
        r = get(cfg, k)
        us = r["ms"] * 1000
        uss = f"{us:,.1f}" if us < 100 else f"{us:,.0f}"
        c = f"{cpu['value']:.1f} ({cpu['cores']} threads)" if cfg == 2 and k == "spmm_nnz" else "—"
        L.append(f"| {cfg} | 1 | {name} | {uss} | {round(r['gflops']):,} | {r['frac_hbm'] * 100:.1f} % | "
                 f"{r['max_rel_err']:.1e} | {c} |")
    i = s.index("| 1 | 1 | SpMV warp-per-row (A.8)")
    j = s.index("\n\n", i) + 1
    s = s[:i] + "\n".join(L) + "\n" + s[j:]
    e = b["e2e"]
    s = re.sub(r"per step\): [0-9,]+ GFLOP/s pipelined \(`pipeline.Pipeline`\) and [0-9,]+ GFLOP/s synchronous",
               f"per step): {e['value']:.0f} GFLOP/s pipelined (`pipeline.Pipeline`) and "
               f"{e['sync_interpret']['value']:.0f} GFLOP/s synchronous", s)
    s = re.sub(r"The bench line itself \([0-9.]+ ms, [0-9,]+ GFLOP/s\)",
               f"The bench line itself ({b['ms_per_step']:.3f} ms, {b['value']:,.0f} GFLOP/s)", s)
    s = re.sub(r"1 s load at the power cap \([0-9]+ of [0-9]+ MHz",
               f"1 s load at the power cap ({b['clocks']['sm_mhz']:.0f} of {b['clocks']['sm_max_mhz']:.0f} MHz", s)
    sh = [json.loads(l) for l in open(PROF / "r01_shard_scaling.jsonl")]
    sp = {r["cfg"]: r["speedup_vs_1"] for r in sh if r["gpus"] == 8}
    s = re.sub(r"r01_shard_scaling.jsonl`\): [0-9.]+× for cfg2 SpMM and [0-9.]+× for cfg5 SpMV at\n  8 GPUs, [0-9.]+× for cfg4 MTTKRP",
               f"r01_shard_scaling.jsonl`): {sp[2]:.2f}× for cfg2 SpMM and {sp[5]:.2f}× for cfg5 SpMV at\n"
               f"  8 GPUs, {sp[4]:.2f}× for cfg4 MTTKRP", s)
    return s


def main():
    copy_profiles()
    p = ROOT / "DESIGN.md"
    p.write_text(design_tables(p.read_text()))
    p = ROOT / "BASELINE.md"
    p.write_text(baseline_table(p.read_text()))
    print("profiles and tables refreshed")


if __name__ == "__main__":
    main()
