# The relaxed kernels against their own zero-compute build (FT_NULL_EVAL=1:
# same grid, loop, PDL, loads and stores; outputs = x) on the f32 configs.
# Usage (under gpurun): TAG=r02m bash tools/ceiling.sh   (needs variants/{cur,null})
tag=${TAG:-ceil}
for v in null cur; do
  for c in cfg1 cfg3; do
    FASTTRIG_B200_LIB=/root/repo/variants/$v/libfasttrig_b200.so python bench.py --config $c --configs none --no-cpu --no-e2e --sustained-seconds 0 --steps 2000 > gpurun_out/${tag}_${v}_$c.json 2>&1
  done
  FASTTRIG_B200_LIB=/root/repo/variants/$v/libfasttrig_b200.so python bench.py --config cfg5 --configs none --no-cpu --no-e2e --sustained-seconds 0 --steps 20 > gpurun_out/${tag}_${v}_cfg5.json 2>&1
  for c in cfg1 cfg3 cfg5; do
    python -c "import json,sys; d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); print(sys.argv[2], sys.argv[3], d['value'], d['roofline']['frac'], d['clocks']['sm_mhz'], d['clocks']['reasons'], d['clocks'].get('power_w_median'))" gpurun_out/${tag}_${v}_$c.json $v $c
  done
done
