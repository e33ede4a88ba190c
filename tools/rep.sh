for r in 1 2; do for n in i64 i32; do
  FASTTRIG_B200_LIB=/root/repo/variants/$n/libfasttrig_b200.so python bench.py --no-cpu --no-e2e --steps 1500 > gpurun_out/rep_${n}_$r.json 2>&1
  python -c "import json,sys; d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); print(sys.argv[2], d['value'], d['clocks']['sm_mhz'], round(d['value']/d['clocks']['sm_mhz']*1000,1))" gpurun_out/rep_${n}_$r.json $n
done; done
