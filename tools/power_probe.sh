# Sustained power/clock probe: zero-compute 1R:3W streams vs K1 (cfg2).
nvidia-smi --query-gpu=timestamp,clocks.sm,power.draw,clocks_event_reasons.sw_power_cap --format=csv,noheader -lms 100 > gpurun_out/power_trace.csv &
SMI=$!
sleep 1
tools/stream_variants sustained > gpurun_out/power_stream.jsonl
sleep 1
python bench.py --no-cpu --no-e2e --sustained-seconds 0 --steps 2000 > gpurun_out/power_k1.json 2>&1
kill $SMI
cat gpurun_out/power_stream.jsonl
python -c "import json; d=json.loads(open('gpurun_out/power_k1.json').read().strip().splitlines()[-1]); print('K1', d['value'], d['roofline']['achieved'], d['clocks'])"
