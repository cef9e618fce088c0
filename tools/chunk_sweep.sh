#!/bin/bash
# bench at several lane chunk lengths (PODE_CHUNK); one line per setting
for c in "" 20 36 48; do
  PODE_CHUNK=$c timeout 300 python bench.py --no-cpu-baseline --steps 3 --warmup 2 > gpurun_out/sweep_$c.log 2>&1
  python - "$c" <<'PY'
import json, sys
c = sys.argv[1] or "default"
l = [x for x in open(f"gpurun_out/sweep_{sys.argv[1]}.log") if x.startswith("{")][-1]
j = json.loads(l); k = j["kernels"]; it = j["config"]["iterations"]
print(c, round(j["ms_per_step"], 2), it, {n: round(v["ms_per_step"] / it * 1000, 1) for n, v in k.items() if v["ms_per_step"] / it > 0.02})
PY
done
