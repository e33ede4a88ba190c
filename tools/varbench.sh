for n in ${VARIANTS:-p0m6}; do
  for c in cfg2 cfg1; do
    FASTTRIG_B200_LIB=/root/repo/variants/$n/libfasttrig_b200.so python bench.py --config $c --no-cpu --no-e2e --steps $([ $c = cfg1 ] && echo 3000 || echo 600) > gpurun_out/var_${n}_$c.json 2>&1
    python -c "import json,sys; d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); print(sys.argv[2], sys.argv[3], d['value'], d['roofline']['frac'], d['clocks']['sm_mhz'], d['clocks']['reasons'], d['accuracy']['max_ulp_vs_oracle'])" gpurun_out/var_${n}_$c.json $n $c
  done
done
