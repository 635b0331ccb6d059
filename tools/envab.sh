#!/bin/bash
# env A/B: envab.sh tag "NAME=VAR=VAL[,VAR=VAL] ..." rounds [bench args]
tag=$1; variants=$2; rounds=${3:-2}; shift 3
out=gpurun_out/$tag; mkdir -p $out
for r in $(seq $rounds); do for nv in $variants; do
  name=${nv%%=*}; kv=${nv#*=}
  f=$out/${name}_r$r.json
  env ${kv//,/ } timeout 300 python bench.py --no-e2e --no-cpu --no-ss --no-counts --steps 5 --warmup 3 "$@" > $f 2> $out/${name}_r$r.err
  python -c "import json; d=json.load(open('$f')); print('$name', $r, round(d['ms_per_step'],2), {k: round(x,2) for k,x in d['stage_ms_per_step'].items()})" || tail -3 $out/${name}_r$r.err
done; done
