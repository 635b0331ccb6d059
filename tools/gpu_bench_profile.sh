#!/bin/bash
# one gpurun call: bench line + ncu launch list + full captures of K1/K2/K3
set -x
tag=${1:-r1}
K='regex:k1_radial|k1b_common|k2_columns|k3_rows'
timeout 900 python bench.py > gpurun_out/bench_$tag.json 2> gpurun_out/bench_$tag.err
tail -3 gpurun_out/bench_$tag.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k "$K" -s 40 -c 80 --csv --log-file gpurun_out/launches_$tag.csv python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu --no-ss --no-counts > /dev/null 2>&1
for k in k1_radial k2_columns k3_rows; do
  timeout 600 ncu --set full --clock-control none --import-source on -k "regex:$k" -s 20 -c 1 -o gpurun_out/prof_${tag}_$k python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu --no-ss --no-counts > gpurun_out/ncu_${tag}_$k.log 2>&1
done
ls -la gpurun_out
