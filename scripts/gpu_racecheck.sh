# racecheck of the stage kernels with several elements / chunks per team / CTA (final round-1 build)
mkdir -p gpurun_out
for c in "1 exact 40 4,4,8" "3 exact 30 2,2,4" "4 exact 20 2,2,4" "5 exact 20 2,2,4" "2 wadg 30 2,2,4" "3 wadg 30 2,2,4" "5 wadg 20 2,2,4" "7 exact 12 1,1,2"; do
  set -- $c
  timeout 900 compute-sanitizer --tool racecheck --print-limit 10 python scripts/racecheck_stage.py $1 $2 $3 $4 > gpurun_out/rc_$1_$2.log 2>&1; echo "racecheck N=$1 $2 exit $?"; grep -E "RACECHECK SUMMARY|rel L2|Error|hazard" gpurun_out/rc_$1_$2.log | head -4
done
for c in "5 exact 20 2,2,4" "1 exact 40 4,4,8"; do
  set -- $c
  timeout 900 compute-sanitizer --tool memcheck --leak-check no --print-limit 10 python scripts/racecheck_stage.py $1 $2 $3 $4 > gpurun_out/mc_$1_$2.log 2>&1; echo "memcheck N=$1 $2 exit $?"; grep -E "ERROR SUMMARY|rel L2" gpurun_out/mc_$1_$2.log | head -3
done
