#!/bin/bash
# same-box A/B of library variants: ab_bench.sh OUTFILE "variant1 variant2 ..." "degrees" [reps] [extra bench args]
# (variant "main" = the in-tree build, "env:VAR=VAL[,..]" = the in-tree build with
# environment overrides); one JSON line per run appended to OUTFILE
cd "$GRAFT_REPO_ROOT" || exit 1
out=$1; vars=$2; degs=$3; reps=${4:-2}; shift 4; extra="$*"
for r in $(seq 1 $reps); do
  for n in $degs; do
    for v in $vars; do
      envs=""
      case "$v" in
        main) lib="" ;;
        env:*) lib=""; envs="${v#env:}" ;;
        *) lib="$PWD/paper_1607_03399_b200/_variants/$v/libprismdg_b200.so" ;;
      esac
      [ -n "$lib" ] && envs="$envs,PDG_LIB_PATH=$lib"
      res=$(env ${envs//,/ } timeout 600 python bench.py --steps 10 --warmup 3 --degree $n --degrees "" \
            --no-cpu-baseline --e2e-steps 1 $extra 2>/dev/null | tail -1)
      python3 -c "import json,sys; d=json.loads(sys.argv[1]); print(json.dumps({'variant': '$v', 'degree': $n, 'rep': $r, 'kernel_ms': d['wedge_kernel_avg_ms'], 'frac': d['roofline']['frac'], 'value': d['value'], 'tet_ms': d.get('tet_kernel_avg_ms'), 'clocks': d['clocks']}))" "$res" >> $out 2>/dev/null || echo "{\"variant\": \"$v\", \"degree\": $n, \"error\": true}" >> $out
    done
  done
done
