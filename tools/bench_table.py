"""Render the bench lines of one evidence tag as the markdown table used in
profiles/README.md:  python tools/bench_table.py r01c"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
tag = sys.argv[1] if len(sys.argv) > 1 else "r01c"
rows = [("", "cfg2 f64 2^28 fused S/C/T (headline)"), ("_cfg1", "cfg1 f32 2^24 fused"),
        ("_cfg3", "cfg3 f32 2^26 tan stress"), ("_cfg4_f32", "cfg4 Taylor-5 S/C f32 2^28"),
        ("_cfg4_f64", "cfg4 Taylor-5 S/C f64 2^28"), ("_cfg5", "cfg5 recipe, one 2^30 f32 shard")]
print("| file | workload | Gelem/s | ms/step | achieved GB/s | frac of measured HBM (6538.9) | SM MHz (reasons) | max ulp vs oracle |")
print("|---|---|---|---|---|---|---|---|")
for suf, name in rows:
    f = os.path.join(ROOT, "profiles", f"{tag}_bench{suf}.json")
    d = json.loads(open(f).read().strip().splitlines()[-1])
    c = d["clocks"]
    reasons = ", ".join(c.get("reasons") or []) or "none"
    print(f"| {os.path.basename(f)} | {name} | {d['value']:.1f} | {d['ms_per_step']:.4g} | "
          f"{d['roofline']['achieved']:.0f} | {d['roofline']['frac']:.3f} | {c['sm_mhz']:.0f} ({reasons}) | "
          f"{' / '.join(str(u) for u in d['accuracy']['max_ulp_vs_oracle'])} |")
