nvidia-smi --query-gpu=timestamp,clocks.sm,power.draw,clocks_event_reasons.sw_power_cap --format=csv,noheader -lms 100 > gpurun_out/op_energy_trace.csv &
SMI=$!
sleep 2
tools/op_energy > gpurun_out/op_energy.jsonl
sleep 1
kill $SMI
cat gpurun_out/op_energy.jsonl
