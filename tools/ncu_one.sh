#!/bin/bash
# usage: ncu_one.sh tag kernel_regex [extra bench args]
tag=$1; k=$2; shift 2
timeout 600 ncu --set full --clock-control none --import-source on -k "regex:$k" -s 20 -c 1 -o gpurun_out/prof_${tag} python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu --no-ss --no-counts "$@" > gpurun_out/ncu_${tag}.log 2>&1
tail -2 gpurun_out/ncu_${tag}.log
