# power_ramp.py over build variants x FT_OCC_CAP values; one summary line each.
# Usage (under gpurun): VARIANTS="def g4r" OCCS="4 3 2" CONFIG=cfg3 TAG=r02bh bash tools/ramp_sweep.sh
tag=${TAG:-ramp}
for v in ${VARIANTS:-def}; do
  for oc in ${OCCS:-0}; do
    FT_OCC_CAP=$oc FASTTRIG_B200_LIB=/root/repo/variants/$v/libfasttrig_b200.so \
      python tools/power_ramp.py --config ${CONFIG:-cfg3} --segs ${SEGS:-24} --seg ${SEG:-40} \
      > gpurun_out/${tag}_one.json 2> gpurun_out/${tag}_one.err || { tail -3 gpurun_out/${tag}_one.err; continue; }
    python - "$v" "$oc" gpurun_out/${tag}_one.json >> gpurun_out/${tag}_ramp.jsonl <<'PY'
import json, sys
d = json.loads(open(sys.argv[3]).read().strip().splitlines()[-1])
d["variant"], d["occ_cap"] = sys.argv[1], int(sys.argv[2])
print(json.dumps(d))
g = d["gelem_s"]
sys.stderr.write(f"{sys.argv[1]} occ_cap {sys.argv[2]} early {sorted(g[1:8])[3]} late {sorted(g[-8:])[3]}\n")
PY
  done
done
