#!/bin/bash
# cfg-2 cube times per degree for variant libraries (warp-specialised kernel forced): tools/f3_regsweep.sh NAME...
cd "$(dirname "$0")/.."
for v in "$@"; do
  echo "== $v"
  for p in 2 3 4 5 6; do
    MFWQ_F3=2 MFWQ_LIB=$PWD/tools/exp/libmfwq_$v.so timeout 300 python tools/profile_matvec.py --p $p --reps 20 2>&1 | grep -E "matvec|rror"
  done
  MFWQ_F3=2 MFWQ_LIB=$PWD/tools/exp/libmfwq_$v.so timeout 300 python tools/profile_matvec.py --p 6 --n-el 128 --geom ring --reps 20 2>&1 | grep -E "matvec|rror"
  MFWQ_F3=2 MFWQ_LIB=$PWD/tools/exp/libmfwq_$v.so timeout 300 python tools/profile_matvec.py --p 2 --n-el 128 --geom ring --reps 20 2>&1 | grep -E "matvec|rror"
done
