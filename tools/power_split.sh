# Sustained power of the relaxed kernels vs their zero-compute build on the f32
# configs (~15 s back to back each): the SM energy per element the arithmetic costs.
# Usage (under gpurun): TAG=r02z bash tools/power_split.sh   (needs variants/{cur,null})
tag=${TAG:-pw}
for c in cfg1 cfg3 cfg5; do
  for v in null cur; do
    st=2000; [ $c = cfg5 ] && st=10
    FASTTRIG_B200_LIB=/root/repo/variants/$v/libfasttrig_b200.so python bench.py --config $c --configs none --no-cpu --no-e2e --steps $st --sustained-seconds 15 > gpurun_out/${tag}_${v}_$c.json 2>&1
    python -c "import json,sys; d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); s=d['sustained']; print(sys.argv[2], sys.argv[3], s['value'], s['roofline_frac'], s['clocks']['sm_mhz'], s['clocks']['reasons'], s['clocks'].get('power_w_median'))" gpurun_out/${tag}_${v}_$c.json $v $c
  done
done
