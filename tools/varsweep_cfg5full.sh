# Like varsweep.sh but cfg5 runs the full 2^33 array (the bench's configs entry).
tag=${TAG:-var}
for n in ${VARIANTS:-cur}; do
  for c in ${CONFIGS:-cfg1 cfg5}; do
    st=2000; case $c in cfg2|cfg4_f32|cfg4_f64) st=400;; cfg5) st=20;; esac
    FASTTRIG_B200_LIB=/root/repo/variants/$n/libfasttrig_b200.so timeout 300 python bench.py --config $c --configs none --no-cpu --no-e2e --sustained-seconds 0 --steps $st > gpurun_out/${tag}_${n}_$c.json 2>&1
    python -c "import json,sys; d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); print(sys.argv[2], sys.argv[3], d['value'], d['roofline']['frac'], d['clocks']['sm_mhz'], d['clocks']['reasons'], d['accuracy']['max_ulp_vs_oracle'])" gpurun_out/${tag}_${n}_$c.json $n $c
  done
done
