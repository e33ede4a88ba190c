"""Summarise one evidence tag's ncu --set full captures into profiles/.

    python tools/ncu_summarize.py r01g [--update-json] [--out DIR] [--from-csv DIR]

For each gpurun_out/<tag>_<kernel>_<cfgN>.ncu-rep (e.g. r02d_k1r_cfg1) writes
profiles/<tag>_<name>_ncu_summary.txt (the metrics quoted in DESIGN.md /
profiles/README.md, plus the PC-sampling stall reasons) and
profiles/<tag>_<name>_ncu_details.csv (the details page).  --update-json
refreshes profiles/ncu_k1_summary.json (per-launch DRAM traffic, FP64-pipe and
warp instructions per element) that bench.py reads for `roofline.traffic`.
"""
import csv
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
# capture-name suffix -> (workload, elements per launch of tools/run_kernel.py)
WORKLOADS = {"cfg1": ("cfg1", 1 << 24), "cfg2": ("cfg2", 1 << 28), "cfg3": ("cfg3", 1 << 26),
             "cfg4f32": ("cfg4_f32", 1 << 28), "cfg4f64": ("cfg4_f64", 1 << 28), "cfg5": ("cfg5", 1 << 30)}


def captures(tag, csv_dir=None):
    """{name: (workload, n, source)} for every gpurun_out/<tag>_<name>.ncu-rep, or
    every <csv_dir>/<tag>_<name>_ncu_raw.csv (summaries written on the GPU box)."""
    import glob
    out = {}
    if csv_dir:
        files = sorted(glob.glob(os.path.join(csv_dir, f"{tag}_*_ncu_raw.csv")))
        names = [os.path.basename(f)[len(tag) + 1:-len("_ncu_raw.csv")] for f in files]
    else:
        files = sorted(glob.glob(os.path.join(ROOT, "gpurun_out", f"{tag}_*.ncu-rep")))
        names = [os.path.basename(f)[len(tag) + 1:-len(".ncu-rep")] for f in files]
    for f, name in zip(files, names):
        wl = WORKLOADS.get(name.rsplit("_", 1)[-1])
        if wl:
            out[name] = (*wl, f)
    return out
METRICS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "smsp__inst_executed.sum",
    "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
    "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
    "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
    "sm__cycles_elapsed.avg.per_second", "launch__grid_size", "launch__occupancy_limit_registers",
    "dram__cycles_elapsed.avg.per_second",
]
FP64_INST = "smsp__inst_executed_pipe_fp64.sum"


def ncu_csv(rep, page):
    out = subprocess.run(["ncu", "-i", rep, "--page", page, "--csv"], capture_output=True, text=True,
                         check=True).stdout
    return out


def raw_metrics(rep):
    """Raw-page metrics of a .ncu-rep, or of a saved <...>_ncu_raw.csv."""
    text = open(rep).read() if rep.endswith(".csv") else ncu_csv(rep, "raw")
    rows = list(csv.reader(io.StringIO(text)))
    hdr, units, vals = rows[0], rows[1], rows[2]
    return {h: (v, u) for h, u, v in zip(hdr, units, vals)}


def to_float(s):
    try:
        return float(s.replace(",", ""))
    except ValueError:
        return None


def main():
    tag = sys.argv[1]
    update = "--update-json" in sys.argv
    outdir = os.path.join(ROOT, "profiles")
    if "--out" in sys.argv:
        outdir = sys.argv[sys.argv.index("--out") + 1]
        os.makedirs(outdir, exist_ok=True)
    js_path = os.path.join(ROOT, "profiles", "ncu_k1_summary.json")
    js = json.load(open(js_path)) if os.path.exists(js_path) else {}
    csv_dir = sys.argv[sys.argv.index("--from-csv") + 1] if "--from-csv" in sys.argv else None
    for name, (wl, n, rep) in captures(tag, csv_dir).items():
        m = raw_metrics(rep)
        lines = []
        for k in METRICS:
            if k in m:
                v, u = m[k]
                lines.append(f"{k:<70} {v:>24} {u}")
        stalls = sorted(((k, to_float(v[0])) for k, v in m.items()
                         if k.startswith("smsp__pcsamp_warps_issue_stalled_") and not k.endswith("_not_issued")
                         and to_float(v[0]) is not None), key=lambda t: -t[1])
        for k, v in stalls[:12]:
            lines.append(f"  {k:<78} {v}")
        txt = os.path.join(outdir, f"{tag}_{name}_ncu_summary.txt")
        open(txt, "w").write("\n".join(lines) + "\n")
        if not rep.endswith(".csv"):
            open(os.path.join(outdir, f"{tag}_{name}_ncu_details.csv"), "w").write(ncu_csv(rep, "details"))
            open(os.path.join(outdir, f"{tag}_{name}_ncu_raw.csv"), "w").write(ncu_csv(rep, "raw"))
        # bytes: ncu prints Mbyte/Gbyte etc.; normalise
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
        rd, wr = m["dram__bytes_read.sum"], m["dram__bytes_write.sum"]
        traffic = to_float(rd[0]) * scale[rd[1]] + to_float(wr[0]) * scale[wr[1]]
        inst = to_float(m["smsp__inst_executed.sum"][0])
        fp64 = to_float(m[FP64_INST][0]) if FP64_INST in m else None
        if fp64 is None and "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active" in m:
            # warp instructions on the FP64 pipe = utilisation x active SM cycles x
            # 2 warp-instructions / cycle / SM (64 FP64 lanes per SM on B200)
            pct = to_float(m["sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active"][0])
            cyc = to_float(m["sm__cycles_active.sum"][0])
            fp64 = pct / 100.0 * cyc * 2.0
        print(f"{name}: {m['gpu__time_duration.sum'][0]} {m['gpu__time_duration.sum'][1]}, traffic {traffic / 1e9:.4f} GB, "
              f"{inst * 32 / n:.2f} instr/elem" + (f", fp64 {fp64 * 32 / n:.2f}/elem" if fp64 else ""))
        if update:
            js.setdefault("traffic_bytes_per_launch", {})[wl] = traffic
            js.setdefault("warp_instr_per_elem", {})[wl] = round(inst * 32 / n, 2)
            if fp64:
                per = round(fp64 * 32 / n, 2)
                js.setdefault("fp64_pipe_instr_per_elem", {})[wl] = per
            js["source"] = (f"ncu --set full --clock-control none, one launch per workload "
                            f"(profiles/{tag}_*_ncu_summary.txt)")
            js["fp64_pipe_instr_note"] = ("FP64-pipe warp instructions x 32 / elements: "
                                          "sm__inst_executed_pipe_fp64 % x sm__cycles_active.sum x 2 "
                                          "warp-instructions/cycle/SM, same capture")
    if update:
        json.dump(js, open(js_path, "w"), indent=1)
        print("updated", js_path)


if __name__ == "__main__":
    main()
