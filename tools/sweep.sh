#!/bin/bash
# lanes x batch sweep of the device-resident 2048^3 step (no e2e / cpu legs)
# usage: sweep.sh <tag> "<lanes>" "<batches>"
tag=$1; lanes=${2:-"1 2 3 4"}; batches=${3:-"1 2 4"}
out=gpurun_out/$tag; mkdir -p $out
for l in $lanes; do for b in $batches; do
  TB_LANES=$l timeout 300 python bench.py --batch $b --no-e2e --no-cpu --no-ss --no-counts --steps 3 --warmup 3 > $out/sweep_l${l}_b${b}.json 2>$out/sweep_l${l}_b${b}.err
  python -c "import json,sys; d=json.load(open('$out/sweep_l${l}_b${b}.json')); print('lanes $l batch $b', round(d['ms_per_step'],1), 'ms', {k: round(v,1) for k,v in d['stage_ms_per_step'].items()})" || tail -3 $out/sweep_l${l}_b${b}.err
done; done
