#!/usr/bin/env python
"""Summarise an ncu report (--set full) into profiles/: key throughput, traffic, stall and SMEM metrics.

    python scripts/ncu_summary.py gpurun_out/X_prof.ncu-rep --name r01_fast --config llama8b_block \
        --kernel fast [--launches gpurun_out/X_launches.csv]

Writes profiles/<name>.md and merges {config/kernel: {...}} into profiles/ncu_summary.json (read by
bench.py for roofline.traffic).
"""
import argparse
import csv
import io
import json
import os
import subprocess

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

KEYS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "dram__throughput.avg.pct_of_peak_sustained_elapsed", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed", "sm__warps_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed.sum", "smsp__inst_executed.sum", "smsp__thread_inst_executed_per_inst_executed.ratio",
    "sm__instruction_throughput.avg.pct_of_peak_sustained_active", "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_st.sum",
    "l1tex__data_pipe_lsu_wavefronts_mem_shared_op_ld.sum", "l1tex__data_pipe_lsu_wavefronts_mem_shared_op_st.sum",
    "launch__registers_per_thread", "launch__grid_size", "launch__block_size", "launch__shared_mem_per_block_dynamic",
    "sm__cycles_elapsed.avg.per_second", "lts__t_bytes.sum", "l1tex__t_bytes.sum",
]


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    recs = []
    for r in rows[2:]:
        recs.append({h: (u, v) for h, u, v in zip(hdr, units, r)})
    return recs


def num(v):
    try:
        return float(v.replace(",", ""))
    except Exception:
        return None


def scale(unit, v):
    f = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-9, "us": 1e-6, "usecond": 1e-6,
         "ms": 1e-3, "msecond": 1e-3, "s": 1}.get(unit)
    return v * f if (f is not None and v is not None) else v


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("rep")
    ap.add_argument("--name", required=True)
    ap.add_argument("--config", required=True)
    ap.add_argument("--kernel", required=True)
    ap.add_argument("--elements", type=float, default=None)
    ap.add_argument("--launches", default=None)
    args = ap.parse_args()
    recs = raw(args.rep)
    r = recs[0]
    lines = [f"# ncu summary: {args.name}", "", f"report: `{os.path.basename(args.rep)}` (ncu --set full, "
             f"--clock-control none, one launch); kernel `{r.get('Kernel Name', ('', ''))[1]}`", "",
             "| metric | unit | value |", "|---|---|---|"]
    picked = {}
    for k in KEYS:
        if k in r:
            u, v = r[k]
            lines.append(f"| {k} | {u} | {v} |")
            picked[k] = (u, num(v))
    stalls = sorted(((k, num(v[1])) for k, v in r.items()
                     if k.startswith("smsp__average_warps_issue_stalled") and k.endswith("_per_issue_active.ratio")
                     and num(v[1])), key=lambda x: -x[1])
    lines += ["", "## warp stall reasons (per issued instruction)", "", "| reason | ratio |", "|---|---|"]
    for k, v in stalls[:12]:
        lines.append(f"| {k.replace('smsp__average_warps_issue_stalled_', '').replace('_per_issue_active.ratio', '')} | {v:.3f} |")
    rd = scale(*picked.get("dram__bytes_read.sum", ("byte", None)))
    wr = scale(*picked.get("dram__bytes_write.sum", ("byte", None)))
    t = scale(*picked.get("gpu__time_duration.sum", ("ns", None)))
    summary = {"dram_bytes_read": rd, "dram_bytes_write": wr,
               "dram_bytes_per_launch": (rd or 0) + (wr or 0) if rd is not None else None,
               "ncu_time_s": t, "report": os.path.basename(args.rep), "name": args.name}
    if t and rd is not None:
        summary["ncu_dram_gbs"] = ((rd or 0) + (wr or 0)) / t / 1e9
        lines += ["", f"DRAM traffic {((rd or 0) + (wr or 0)) / 1e6:.1f} MB in {t * 1e6:.1f} us "
                  f"= {summary['ncu_dram_gbs']:.0f} GB/s (cold-cache, serialised ncu replay)"]
    inst = picked.get("smsp__inst_executed.sum", (None, None))[1]
    if inst and args.elements:
        summary["warp_inst_per_element"] = inst / args.elements
        summary["thread_inst_per_element"] = 32 * inst / args.elements
        lines.append(f"warp instructions per element: {inst / args.elements:.3f} "
                     f"(x32 = {32 * inst / args.elements:.1f} thread-instruction slots)")
    if args.launches and os.path.exists(args.launches):
        text = open(args.launches).read().splitlines()
        start = next(i for i, l in enumerate(text) if l.startswith('"ID"'))
        rows = list(csv.DictReader(io.StringIO("\n".join(text[start:]))))
        tot = sum(float(x["Metric Value"]) for x in rows if x["Metric Name"] == "gpu__time_duration.sum")
        ours = [x for x in rows if "df11" in x["Kernel Name"]]
        lines += ["", "## launch list (ncu --metrics gpu__time_duration.sum, cold cache, serialised)", "",
                  "| # | kernel | grid | block | ns | share of listed time |", "|---|---|---|---|---|---|"]
        for x in rows:
            v = float(x["Metric Value"])
            lines.append(f"| {x['ID']} | {x['Kernel Name'][:60]} | {x['Grid Size']} | {x['Block Size']} | {v:.0f} | {v / tot:.1%} |")
        summary["launch_list_df11_ns"] = [float(x["Metric Value"]) for x in ours]
    os.makedirs(os.path.join(ROOT, "profiles"), exist_ok=True)
    with open(os.path.join(ROOT, "profiles", f"{args.name}.md"), "w") as f:
        f.write("\n".join(lines) + "\n")
    p = os.path.join(ROOT, "profiles", "ncu_summary.json")
    d = json.load(open(p)) if os.path.exists(p) else {}
    d[f"{args.config}/{args.kernel}"] = summary
    with open(p, "w") as f:
        json.dump(d, f, indent=1, sort_keys=True)
    print("\n".join(lines))


if __name__ == "__main__":
    main()
