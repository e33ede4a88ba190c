#!/bin/bash
# Collect a round's GPU evidence with the default in-tree build (one gpurun call).
# Usage (under gpurun): bash tools/round_evidence.sh <tag>
#   <tag>_smoke.log, <tag>_bench.json (default bench: headline + every config),
#   <tag>_launches*.csv (ncu launch lists of the bench commands),
#   <tag>_k{1,1r,2,2r}_<cfg>.ncu-rep (ncu --set full, one launch per workload)
tag=${1:-r02x}
out=gpurun_out
python -c "import __graft_entry__ as g; g.smoke()" > $out/${tag}_smoke.log 2>&1; echo "smoke rc=$?"
python bench.py > $out/${tag}_bench.json 2> $out/${tag}_bench.err; echo "bench rc=$?"
# launch lists (cold-cache, serialised: shares, not absolutes)
python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu --sustained-seconds 0 --configs none > $out/${tag}_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $out/${tag}_launches.csv \
    python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu --sustained-seconds 0 --configs none > $out/${tag}_ncu_launch.log 2>&1
python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu --sustained-seconds 0 --config-steps 5 > $out/${tag}_plain_cfgs.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $out/${tag}_launches_configs.csv \
    python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu --sustained-seconds 0 --config-steps 5 > $out/${tag}_ncu_launch_cfgs.log 2>&1
echo "launches rc=$?"
# full captures of the dominant kernel of every workload
for spec in "k1_cfg2:k_proposed:cfg2" "k1r_cfg1:k_proposed:cfg1" "k1r_cfg3:k_proposed:cfg3" "k1r_cfg5:k_proposed:cfg5" \
            "k2r_cfg4f32:k_taylor:cfg4_f32" "k2_cfg4f64:k_taylor:cfg4_f64"; do
  IFS=: read name kern cfg <<< "$spec"
  python tools/run_kernel.py --config $cfg --reps 3 > $out/${tag}_plain_$name.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:$kern -s 1 -c 1 -o $out/${tag}_$name \
      python tools/run_kernel.py --config $cfg --reps 3 > $out/${tag}_ncu_$name.log 2>&1
  echo "ncu $name rc=$?"
done
# summaries (text + details/raw CSV) next to the outputs; the .ncu-rep files are
# too large to bring back all at once (gpurun's 64 MiB limit): keep one
python tools/ncu_summarize.py $tag --out $out/${tag}_ncu > $out/${tag}_ncu_summary.log 2>&1
for f in $out/${tag}_*.ncu-rep; do case $f in *k1r_cfg1*) ;; *) rm -f $f;; esac; done
du -sh $out
