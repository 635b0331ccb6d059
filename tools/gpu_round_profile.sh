#!/bin/bash
# One gpurun call producing the round's evidence under gpurun_out/<tag>/:
# full bench line, ncu launch list (same command, --metrics gpu__time_duration),
# and one ncu --set full capture per main kernel.
tag=${1:-r1}
out=gpurun_out/$tag; mkdir -p $out
K='regex:k1_radial|k1b_common|k2_columns|k3_rows|kr_ramp'
timeout 900 python bench.py > $out/bench.json 2> $out/bench.err
tail -2 $out/bench.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k "$K" -s 50 -c 200 --csv --log-file $out/launches.csv python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu > /dev/null 2>&1
for k in k1_radial k2_columns k3_rows k1b_common; do
  timeout 600 ncu --set full --clock-control none --import-source on -k "regex:$k" -s 20 -c 1 -o $out/prof_$k python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu > $out/ncu_$k.log 2>&1
done
ls -la $out
