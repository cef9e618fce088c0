#!/bin/bash
# bench under several env settings, e.g.  tools/env_sweep.sh "PODE_BSCAN=2048" "PODE_CHUNK=24"
# prints ms per solve, iterations, ms per iteration and the per-iteration µs of the main kernels
i=0
for s in "$@"; do
  i=$((i + 1))
  env $s timeout 300 python bench.py --no-cpu-baseline --steps 3 --warmup 2 > gpurun_out/env_$i.log 2>&1
  python - "$s" "$i" <<'PY'
import json, sys
l = [x for x in open(f"gpurun_out/env_{sys.argv[2]}.log") if x.startswith("{")][-1]
j = json.loads(l); k = j["kernels"]; it = j["config"]["iterations"]
print(sys.argv[1], round(j["ms_per_step"], 2), it, round(j["ms_per_step"] / it * 1000, 1),
      {n: round(v["ms_per_step"] / it * 1000, 1) for n, v in k.items() if v["ms_per_step"] / it > 0.02})
PY
done
