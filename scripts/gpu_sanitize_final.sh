#!/bin/bash
# compute-sanitizer memcheck + racecheck of the final stage kernels on meshes where every team runs several elements
cd "$GRAFT_REPO_ROOT" || exit 1
out=gpurun_out/san_final.log; : > $out
for args in "4 exact 20 2,2,2" "5 exact 20 2,2,2" "6 exact 12 2,2,2" "7 exact 12 2,2,2" "5 wadg 20 2,2,2" "2 exact 20 2,2,2"; do
  for tool in memcheck racecheck; do
    echo "== $tool racecheck_stage.py $args" >> $out
    timeout 900 compute-sanitizer --tool $tool --error-exitcode 9 python scripts/racecheck_stage.py $args 2>&1 | grep -E "rel L2|SUMMARY" >> $out
    echo "rc=${PIPESTATUS[0]}" >> $out
  done
done
for tool in memcheck racecheck; do
  echo "== $tool racecheck_hybrid.py 4 16 2 8" >> $out
  timeout 900 compute-sanitizer --tool $tool --error-exitcode 9 python scripts/racecheck_hybrid.py 4 16 2 8 2>&1 | grep -E "rel L2|SUMMARY" >> $out
  echo "rc=${PIPESTATUS[0]}" >> $out
done
