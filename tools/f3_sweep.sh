#!/bin/bash
# warp-specialised (MFWQ_F3=1) vs phased (MFWQ_F3=0) kernel over the degrees: cfg-2 cube, ring, on the fly
cd "$(dirname "$0")/.."
for f3 in 1 0; do
  echo "== MFWQ_F3=$f3"
  for p in ${@:-1 2 3 4 5 6}; do
    MFWQ_F3=$f3 timeout 300 python tools/profile_matvec.py --p $p --reps 20 2>&1 | grep -E "matvec|rror"
    MFWQ_F3=$f3 timeout 300 python tools/profile_matvec.py --p $p --n-el 128 --geom ring --reps 20 2>&1 | grep -E "matvec|rror"
    MFWQ_F3=$f3 timeout 300 python tools/profile_matvec.py --p $p --n-el 128 --otf 1 --reps 20 2>&1 | grep -E "matvec|rror" | sed 's/identity/identity otf/'
  done
  MFWQ_F3=$f3 timeout 300 python tools/profile_matvec.py --p 4 --n-el 256 --geom ring --reps 10 2>&1 | grep -E "matvec|rror"
  MFWQ_F3=$f3 timeout 300 python tools/profile_matvec.py --p 6 --n-el 256 --geom ring --reps 10 2>&1 | grep -E "matvec|rror"
done
