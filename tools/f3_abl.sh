#!/bin/bash
# times the variant libraries built by tools/f3_variant.sh (p = 4): cfg-2 cube and the cfg-3 ring
cd "$(dirname "$0")/.."
for v in "$@"; do
  echo "== $v"
  MFWQ_LIB=$PWD/tools/exp/libmfwq_$v.so timeout 300 python tools/profile_matvec.py --p 4 --reps 20 2>&1 | grep -E "matvec|rror"
  MFWQ_LIB=$PWD/tools/exp/libmfwq_$v.so timeout 300 python tools/profile_matvec.py --p 4 --n-el 256 --geom ring --reps 10 2>&1 | grep -E "matvec|rror"
done
