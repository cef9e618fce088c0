#!/bin/bash
# compute-sanitizer (memcheck / racecheck / synccheck) over one small solve
# per engine: the lane engine (pass C's shared-memory accumulator, block
# Sklansky scans, group tiles of the aggregate scans), the group engine
# (D = 15), the large-state engine (D = 112) and the element engine.
# Logs: gpurun_out/sanitizer_<tool>_<case>.log; one summary line each.
out=${1:-gpurun_out}
mkdir -p "$out"
run() {  # tool case env... -- args
  local tool=$1 name=$2; shift 2
  local envs=()
  while [ "$1" != "--" ]; do envs+=("$1"); shift; done
  shift
  env "${envs[@]}" timeout 900 compute-sanitizer --tool "$tool" --print-limit 20 python tools/prof_once.py "$@" \
    > "$out/sanitizer_${tool}_${name}.log" 2>&1
  echo "$tool $name rc=$? $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY|hazard' "$out/sanitizer_${tool}_${name}.log" | tail -1)"
}
for tool in memcheck racecheck synccheck; do
  run $tool lane_fhn_q2 -- 12 fhn 2 3
  run $tool grp_rigid_q4 -- 9 rigidbody 4 3
  run $tool big_pleiades_q3 -- 6 pleiades 3 2
  run $tool elements_fhn_q2 PODE_IEKS_ENGINE=elements -- 10 fhn 2 3
done
