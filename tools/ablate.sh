#!/bin/bash
# Build timing-experiment variants of libmfwq.so (never used by the product):
#   tools/ablate.sh 1 2 3 4 9   ->  tools/abl/libmfwq_ablN.so   (see MFWQ_ABLATE in csrc/fused2.cu)
cd "$(dirname "$0")/.."
for a in "$@"; do
  MFWQ_BUILD_TAG=abl$a MFWQ_BUILD_LIB=$PWD/tools/abl/libmfwq_abl$a.so MFWQ_NVCC_EXTRA="-DMFWQ_ABLATE=$a" \
    python -m paper_1712_08565_b200.build > /dev/null &
done
wait
