#!/bin/bash
# usage: gpurun_sanitize.sh tag -- compute-sanitizer (memcheck, racecheck, synccheck, initcheck) over
# the small-config grid pass (smoke: 14-atom Fe3O4, 36^3) and a small Eigen_HH / V_eff / formats case
# (tools/sanitize_cases.py). SURVEY.md section 5, "Race detection / sanitizers".
tag=${1:-r01}; mkdir -p gpurun_out
out=gpurun_out/sanitize_$tag.log; : > $out
for tool in memcheck racecheck synccheck initcheck; do
  for case in smoke eigen veff formats; do
    echo "== $tool $case" >> $out
    timeout 900 compute-sanitizer --tool $tool --error-exitcode 7 --print-limit 20 \
      python tools/sanitize_cases.py $case > gpurun_out/san_${tool}_${case}_$tag.log 2>&1
    rc=$?
    grep -E "ERROR SUMMARY|RACECHECK SUMMARY|ok:" gpurun_out/san_${tool}_${case}_$tag.log >> $out
    echo "rc=$rc" >> $out
  done
done
cat $out
