#!/bin/bash
# bench at several sequential scan fan-ins (PODE_SCAN_FANIN)
for f in 3 4 6 8; do
  PODE_SCAN_FANIN=$f timeout 300 python bench.py --no-cpu-baseline --steps 3 --warmup 2 > gpurun_out/fanin_$f.log 2>&1
  python - "$f" <<'PY'
import json, sys
l = [x for x in open(f"gpurun_out/fanin_{sys.argv[1]}.log") if x.startswith("{")][-1]
j = json.loads(l); k = j["kernels"]; it = j["config"]["iterations"]
print(sys.argv[1], round(j["ms_per_step"], 2), it, {n: round(v["ms_per_step"] / it * 1000, 1) for n, v in k.items() if "scan" in n})
PY
done
