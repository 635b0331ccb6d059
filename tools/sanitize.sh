#!/bin/bash
# compute-sanitizer memcheck / racecheck / synccheck over tools/sanitize_driver.py,
# over every kernel the driver launches (this library's and torch's); the K1 TMA bulk-copy variant
# (-DTB_K1_SLOTS=1, ablibs/slots1.so) gets its own pass.  Logs -> gpurun_out/<tag>/.
tag=${1:-r2_sanitize}; out=gpurun_out/$tag; mkdir -p $out
for tool in memcheck racecheck synccheck; do
  t0=$(date +%s); timeout 1500 compute-sanitizer --tool $tool --error-exitcode 9 --print-limit 50 \
    python tools/sanitize_driver.py > $out/$tool.log 2>&1
  rc=$?; echo "$tool rc=$rc $(( $(date +%s) - t0 )) s"; tail -3 $out/$tool.log
done
if [ -f ablibs/slots1.so ]; then
  for tool in memcheck racecheck synccheck; do
    TB_LIB_PATH=ablibs/slots1.so timeout 1500 compute-sanitizer --tool $tool --error-exitcode 9 \
      --print-limit 50 python tools/sanitize_driver.py > $out/slots1_$tool.log 2>&1
    echo "slots1 $tool rc=$?"; tail -3 $out/slots1_$tool.log
  done
fi
