# tools/power_split.sh over arbitrary variants: VARIANTS="null nulltma" CONFIGS="cfg5" TAG=.. SECS=15
tag=${TAG:-pw}
for c in ${CONFIGS:-cfg1 cfg5}; do
  for v in ${VARIANTS:-null cur}; do
    st=2000; [ $c = cfg5 ] && st=10
    FASTTRIG_B200_LIB=/root/repo/variants/$v/libfasttrig_b200.so python bench.py --config $c --configs none --no-cpu --no-e2e --steps $st --sustained-seconds ${SECS:-15} > gpurun_out/${tag}_${v}_$c.json 2>&1
    python -c "import json,sys; d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); s=d['sustained']; print(sys.argv[2], sys.argv[3], 'burst', d['value'], 'sustained', s['value'], s['roofline_frac'], s['clocks']['sm_mhz'], s['clocks']['reasons'], s['clocks'].get('power_w_median'))" gpurun_out/${tag}_${v}_$c.json $v $c
  done
done
