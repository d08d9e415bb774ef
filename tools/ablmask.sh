#!/bin/bash
# Build timing-experiment variants with MFWQ_ABL_MASK bits (see csrc/fused2.cu): tools/ablmask.sh 63 2 ...
cd "$(dirname "$0")/.."
for a in "$@"; do
  MFWQ_BUILD_TAG=ablm$a MFWQ_BUILD_LIB=$PWD/tools/abl/libmfwq_m$a.so MFWQ_NVCC_EXTRA="-DMFWQ_ABL_MASK=$a" \
    python -m paper_1712_08565_b200.build > /dev/null &
done
wait
