#!/bin/bash
# One gpurun call producing the round's evidence under gpurun_out/<tag>/:
# full bench line, ncu launch list (same command, --metrics gpu__time_duration),
# and one ncu --set full capture per main kernel, exported on the box to CSV
# (raw metrics, details, source) so the copy-back stays under 64 MiB.
# usage: gpu_round_profile.sh <tag> [kernels...] ; KEEP_REP=<kernel> keeps that .ncu-rep
tag=${1:-r1}; shift
kernels=${@:-k1_radial k2_columns k3_rows k1b_common}
out=gpurun_out/$tag; mkdir -p $out
K='regex:k1_radial|k1b_common|k2_columns|k3_rows|kr_ramp'
if [ -z "$NO_BENCH" ]; then
  timeout 900 python bench.py > $out/bench.json 2> $out/bench.err
  cat $out/bench.json; tail -2 $out/bench.err
fi
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k "$K" -s 50 -c 200 --csv --log-file $out/launches.csv python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu --no-ss --no-counts > /dev/null 2>&1
for k in $kernels; do
  rep=/tmp/prof_${tag}_$k
  timeout 600 ncu --set full --clock-control none --import-source on -k "regex:$k" -s 20 -c 1 -f -o $rep python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu --no-ss --no-counts > $out/ncu_$k.log 2>&1
  ncu -i $rep.ncu-rep --page raw --csv > $out/raw_$k.csv 2>/dev/null
  ncu -i $rep.ncu-rep --page details --csv > $out/details_$k.csv 2>/dev/null
  ncu -i $rep.ncu-rep --page source --csv > $out/source_$k.csv 2>/dev/null
  if [ "$KEEP_REP" = "$k" ]; then cp $rep.ncu-rep $out/; fi
done
ls -la $out
