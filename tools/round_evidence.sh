#!/bin/bash
# Collect the round's GPU evidence with the default in-tree build.
# Usage (under gpurun): bash tools/round_evidence.sh <tag>
tag=${1:-r01f}
out=gpurun_out
python -c "import __graft_entry__ as g; g.smoke()" > $out/${tag}_smoke.log 2>&1; echo "smoke rc=$?"
python bench.py > $out/${tag}_bench.json 2> $out/${tag}_bench.err; echo "bench rc=$?"
for c in cfg1 cfg3 cfg4_f32 cfg4_f64; do
  python bench.py --config $c --no-cpu --no-e2e --steps 1000 > $out/${tag}_bench_$c.json 2>&1
done
python bench.py --config cfg5 --elements $((1<<30)) --no-cpu --no-e2e --steps 60 > $out/${tag}_bench_cfg5.json 2>&1
# launch list of the bench command (cold-cache, serialised: shares, not absolutes)
python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu > $out/${tag}_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $out/${tag}_launches.csv \
    python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu > $out/${tag}_ncu_launch.log 2>&1; echo "launches rc=$?"
# full capture of K1 (cfg2, f64) and K1 (cfg1, f32) and K2 (cfg4 f32)
python tools/run_kernel.py --config cfg2 --reps 3 > $out/${tag}_plain2.log 2>&1 && \
python tools/run_kernel.py --config cfg1 --reps 3 >> $out/${tag}_plain2.log 2>&1 && \
python tools/run_kernel.py --config cfg4_f32 --reps 3 >> $out/${tag}_plain2.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_proposed -s 1 -c 1 -o $out/${tag}_k1_cfg2 \
    python tools/run_kernel.py --config cfg2 --reps 3 > $out/${tag}_ncu_a.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_proposed -s 1 -c 1 -o $out/${tag}_k1_cfg1 \
    python tools/run_kernel.py --config cfg1 --reps 3 > $out/${tag}_ncu_b.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_taylor -s 1 -c 1 -o $out/${tag}_k2_cfg4f32 \
    python tools/run_kernel.py --config cfg4_f32 --reps 3 > $out/${tag}_ncu_c.log 2>&1; echo "ncu rc=$?"
