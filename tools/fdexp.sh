#!/bin/bash
# FD modal-GEMM tile experiments (timing only): MFWQ_MG_CFG picks a tile shape for every mode
cd "$(dirname "$0")/.."
for cfg in ${CFGS:-0 2 4 5 6 7}; do
 for pn in ${SIZES:-"2,128" "4,128" "6,128" "4,256"}; do
  IFS=, read p ne <<< "$pn"
  MFWQ_MG_CFG=$cfg python tools/fd_time.py --p $p --n-el $ne | sed "s/^/cfg$cfg /"
 done
done
