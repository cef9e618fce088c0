#!/bin/bash
# run a small solve under several engine switches, each with a short timeout
for env in "PODE_TAG=default" "PODE_TAG=nograph PODE_GRAPH=0" "PODE_TAG=elemfin PODE_FINALIZE=elements" "PODE_TAG=nobscan PODE_BSCAN=0"; do
  echo "== $env"
  env $env timeout 60 python tools/dbg_shim.py x 2>&1 | tail -2
done
