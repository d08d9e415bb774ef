#!/bin/bash
# cfg-2 cube time of variant libraries at one degree: tools/f3_p.sh P NAME...
cd "$(dirname "$0")/.."
P=$1; shift
for v in "$@"; do
  echo "== $v (p=$P)"
  MFWQ_LIB=$PWD/tools/exp/libmfwq_$v.so timeout 300 python tools/profile_matvec.py --p $P --reps 20 2>&1 | grep -E "matvec|rror"
  MFWQ_LIB=$PWD/tools/exp/libmfwq_$v.so timeout 300 python tools/profile_matvec.py --p $P --otf 1 --reps 20 2>&1 | grep -E "matvec|rror"
done
