#!/bin/bash
# DMMA / tensor-pipe utilisation and DRAM bytes of every large-state kernel
# for one Pleiades IWP(3) solve (1 iteration + finalize) at N = 2^LG:
# bash tools/big_dmma.sh LG OUT.csv
LG=${1:-16}
OUT=${2:-gpurun_out/big_dmma.csv}
ncu --clock-control none -k regex:k_big --csv --log-file "$OUT" \
  --metrics gpu__time_duration.sum,sm__inst_executed_pipe_tensor_subpipe_dmma.avg.pct_of_peak_sustained_active,sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed,sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active,dram__bytes_read.sum,dram__bytes_write.sum \
  python tools/prof_once.py "$LG" pleiades 3 1
