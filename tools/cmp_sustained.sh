# Headline run + sustained leg of build variants, alternating.  Usage (under gpurun):
#   VARIANTS="def notma" CONFIG=cfg2 SECONDS_SUS=10 bash tools/cmp_sustained.sh
for r in 1 2; do for n in ${VARIANTS:-def}; do
  FASTTRIG_B200_LIB=/root/repo/variants/$n/libfasttrig_b200.so python bench.py --config ${CONFIG:-cfg2} --configs none --no-cpu --no-e2e --sustained-seconds ${SECONDS_SUS:-10} > gpurun_out/cmps_${n}_$r.json 2>/dev/null
  python - $n gpurun_out/cmps_${n}_$r.json <<'PY'
import json, sys
d = json.loads(open(sys.argv[2]).read().strip().splitlines()[-1])
print(sys.argv[1], "run", d["value"], d["clocks"]["sm_mhz"], "burst", d["burst"]["value"], "sustained", d["sustained"]["value"], d["sustained"]["clocks"]["sm_mhz"], d["sustained"]["clocks"].get("power_w_median"), d["accuracy"]["bit_mismatch_vs_oracle"])
PY
done; done
