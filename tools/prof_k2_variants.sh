out=gpurun_out/r2s3_k2pair; mkdir -p $out
for v in base nofft; do
  if [ $v = nofft ]; then export TB_LIB_PATH=ablibs/nofft.so; else unset TB_LIB_PATH; fi
  rep=/tmp/prof_$v
  timeout 600 ncu --set full --clock-control none --import-source on -k "regex:k2_columns" -s 20 -c 1 -f -o $rep python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu --no-ss --no-counts > $out/ncu_$v.log 2>&1
  ncu -i $rep.ncu-rep --page raw --csv > $out/raw_$v.csv 2>/dev/null
  ncu -i $rep.ncu-rep --page details --csv > $out/details_$v.csv 2>/dev/null
  ncu -i $rep.ncu-rep --page source --csv > $out/source_$v.csv 2>/dev/null
done
ls -la $out
