# Sweep the number of resident-block waves the launchers use (FT_GRID_MULT) on
# the bench configs; one line per (waves, config).  Usage (under gpurun):
#   MULTS="1 2 4 8" CONFIGS="cfg1 cfg3 cfg2" bash tools/gridmult_sweep.sh
for m in ${MULTS:-1 2 4 8 1}; do
  for c in ${CONFIGS:-cfg1 cfg3 cfg2}; do
    st=3000; case $c in cfg2|cfg4_f32|cfg4_f64) st=600;; esac
    FT_GRID_MULT=$m python bench.py --config $c --no-cpu --no-e2e --sustained-seconds 0 --steps $st > gpurun_out/gm_${m}_$c.json 2>&1
    python -c "import json,sys; d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); print(sys.argv[2], sys.argv[3], d['value'], d['clocks']['sm_mhz'], d['clocks']['reasons'], d['accuracy']['max_ulp_vs_oracle'])" gpurun_out/gm_${m}_$c.json $m $c
  done
done
