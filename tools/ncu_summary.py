"""Summarise an ncu report: details page (section | metric | unit | value) + key raw metrics.

    python tools/ncu_summary.py gpurun_out/prof.ncu-rep [--raw regex ...]
"""
import csv
import io
import re
import subprocess
import sys

RAW_DEFAULT = [
    r"^gpu__time_duration\.sum$", r"^dram__bytes_(read|write)\.sum$",
    r"^sm__cycles_elapsed\.avg\.per_second$",
    r"^l1tex__data_pipe_lsu_wavefronts_mem_shared(_op_ld|_op_st)?\.sum$",
    r"^l1tex__data_bank_conflicts_pipe_lsu_mem_shared(_op_ld|_op_st)?\.sum$",
    r"^smsp__inst_executed\.sum$", r"^smsp__inst_executed_op_shared_ld\.sum$",
    r"^smsp__issue_active\.avg\.pct_of_peak_sustained_active$",
    r"^sm__inst_executed_pipe_lsu\.avg\.pct_of_peak_sustained_active$",
    r"^l1tex__data_pipe_lsu_wavefronts_mem_shared\.avg\.pct_of_peak_sustained_elapsed$",
    r"^smsp__average_warp_latency_issue_stalled_.*\.ratio$",
    r"^smsp__pcsamp_warps_issue_stalled_.*$",
    r"^launch__registers_per_thread$", r"^sm__warps_active\.avg\.pct_of_peak_sustained_active$",
]


def run(args):
    return subprocess.run(["ncu", "-i", *args], capture_output=True, text=True).stdout


def details(rep):
    out = []
    rows = list(csv.DictReader(io.StringIO(run([rep, "--page", "details", "--csv"]))))
    for r in rows:
        if r.get("Metric Name"):
            out.append(f"{r['Section Name'][:28]:28s} | {r['Metric Name'][:44]:44s} | "
                       f"{r['Metric Unit'][:10]:10s} | {r['Metric Value']}")
        elif r.get("Rule Description"):
            out.append(f"  [{r.get('Rule Type', '')}] {r['Rule Description'][:300]}")
    return out


def raw(rep, pats):
    txt = run([rep, "--page", "raw", "--csv"])
    rd = list(csv.reader(io.StringIO(txt)))
    if len(rd) < 3:
        return []
    names, units, vals = rd[0], rd[1], rd[2]
    out = []
    for n, u, v in zip(names, units, vals):
        if any(re.search(p, n) for p in pats):
            out.append(f"{n:80s} {u:12s} {v}")
    return out


if __name__ == "__main__":
    rep = sys.argv[1]
    pats = RAW_DEFAULT
    if "--raw" in sys.argv:
        pats = sys.argv[sys.argv.index("--raw") + 1:]
    print("\n".join(details(rep)))
    print("\n# raw")
    print("\n".join(raw(rep, pats)))
