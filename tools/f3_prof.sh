#!/bin/bash
# per-warp wait / section cycle counts of the warp-specialised kernel (libraries built with -DMFWQ_F3_PROF)
cd "$(dirname "$0")/.."
for v in "$@"; do
  echo "== $v"
  MFWQ_LIB=$PWD/tools/exp/libmfwq_$v.so timeout 300 python tools/profile_matvec.py --p 4 --reps 1 2>&1 | grep -E "F3PROF|rror" | sort | uniq | awk 'NR%2==1'
done
