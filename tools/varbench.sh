# Benchmark K1 build variants (variants/<name>/libfasttrig_b200.so): sustained bench + burst.
for n in ${VARIANTS:-x0m5}; do
  for c in ${CONFIGS:-cfg2 cfg1}; do
    export FASTTRIG_B200_LIB=/root/repo/variants/$n/libfasttrig_b200.so
    python bench.py --config $c --no-cpu --no-e2e --sustained-seconds 0 --steps $([ $c = cfg1 ] && echo 3000 || echo 600) > gpurun_out/var_${n}_$c.json 2>&1
    python tools/burst.py --config $c > gpurun_out/burst_${n}_$c.json 2>&1
    python -c "import json,sys; d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); b=json.loads(open(sys.argv[4]).read().strip().splitlines()[-1]); print(sys.argv[2], sys.argv[3], 'sustained', d['value'], d['roofline']['frac'], d['clocks']['sm_mhz'], d['clocks']['reasons'], 'ulp', d['accuracy']['max_ulp_vs_oracle'], '| burst', round(b['gelem_s'],1), round(b['gbs']))" gpurun_out/var_${n}_$c.json $n $c gpurun_out/burst_${n}_$c.json
  done
done
