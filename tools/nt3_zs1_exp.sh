#!/bin/bash
# timing experiment: 3-term kernel with one z-element per step at 3 CTAs/SM (p <= 3) vs the product
cd "$(dirname "$0")/.."
for lib in tools/abl/libmfwq_nt3zs1.so paper_1712_08565_b200/libmfwq.so; do
 for p in 2 3; do
  MFWQ_LIB=$lib python tools/profile_matvec.py --p $p --reps 20 | tail -1 | sed "s|^|$(basename $lib) |"
  MFWQ_LIB=$lib python tools/profile_matvec.py --p $p --reps 20 --otf 1 | tail -1 | sed "s|^|$(basename $lib) otf |"
 done
done
