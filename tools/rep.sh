# Repeat sustained (1500 steps) + burst measurements for two builds, alternating.
for r in 1 2; do for n in ${VARIANTS:-notma tma}; do
  for c in ${CONFIGS:-cfg2}; do
    FASTTRIG_B200_LIB=/root/repo/variants/$n/libfasttrig_b200.so python bench.py --config $c --no-cpu --no-e2e --sustained-seconds 0 --steps 1500 > gpurun_out/rep_${n}_${c}_$r.json 2>&1
    FASTTRIG_B200_LIB=/root/repo/variants/$n/libfasttrig_b200.so python tools/burst.py --config $c > gpurun_out/repb_${n}_${c}_$r.json 2>&1
    python -c "import json,sys; d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); b=json.loads(open(sys.argv[4]).read().strip().splitlines()[-1]); print(sys.argv[2], sys.argv[3], 'sustained', d['value'], d['clocks']['sm_mhz'], 'burst', round(b['gelem_s'],1))" gpurun_out/rep_${n}_${c}_$r.json $n $c gpurun_out/repb_${n}_${c}_$r.json
  done
done; done
