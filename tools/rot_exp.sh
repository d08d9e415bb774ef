#!/bin/bash
# register-window rotation variants (r<acc><ring>; r00 = moves as before): parity + timing
cd "$(dirname "$0")/.."
for lib in tools/abl/libmfwq_r00.so paper_1712_08565_b200/libmfwq.so tools/abl/libmfwq_r01.so tools/abl/libmfwq_r11.so; do
 for p in 2 3 4 5 6; do
  MFWQ_LIB=$lib python tools/profile_matvec.py --p $p --reps 20 | tail -1 | cut -c1-100 | sed "s|^|$(basename $lib) |"
 done
 MFWQ_LIB=$lib python tools/profile_matvec.py --p 4 --n-el 256 --geom ring --reps 5 | tail -1 | cut -c1-100 | sed "s|^|$(basename $lib) |"
done
