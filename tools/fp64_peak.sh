#!/bin/bash
# FP64 roofline denominators with the clock record: builds tools/fp64_peak.cu
# (DFMA and DMMA m8n8k4 throughput), runs it three times while nvidia-smi
# samples SM clocks / throttle reasons every 100 ms, and writes one JSON with
# the best DFMA / DMMA rates, the median SM clock under load and the reasons.
set -e
out=${1:-gpurun_out/r02_fp64_peak.json}
nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o /tmp/fp64_peak tools/fp64_peak.cu
nvidia-smi --query-gpu=clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap --format=csv,noheader,nounits -lms 100 > /tmp/clk.csv &
smi=$!
for i in 1 2 3; do /tmp/fp64_peak >> /tmp/fp64_runs.jsonl; done
kill $smi
python3 - "$out" <<'PY'
import json, statistics, sys
runs = [json.loads(l) for l in open("/tmp/fp64_runs.jsonl") if l.strip()]
rows = [[x.strip() for x in l.split(",")] for l in open("/tmp/clk.csv") if l.count(",") == 6]
sm = [float(r[0]) for r in rows if r[0].replace(".", "").isdigit()]
load = [s for s in sm if s > 0.5 * max(sm)] if sm else []
names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
reasons = sorted({names[k] for r in rows for k in range(4) if r[3 + k] == "Active"})
res = {"sms": runs[0]["sms"], "fp64_fma_tflops": max(r["fp64_fma_tflops"] for r in runs),
       "fp64_dmma_tflops": max(r["fp64_dmma_tflops"] for r in runs), "runs": runs,
       "clocks": {"sm_mhz_median_under_load": statistics.median(load) if load else None,
                  "sm_max_mhz": max(float(r[1]) for r in rows) if rows else None,
                  "power_w_max": max(float(r[2]) for r in rows) if rows else None,
                  "reasons": reasons, "samples": len(rows)},
       "how": "tools/fp64_peak.cu: DFMA chains / DMMA m8n8k4 over all SMs; best of 3; nvidia-smi -lms 100"}
json.dump(res, open(sys.argv[1], "w"), indent=1)
print(json.dumps(res))
PY
