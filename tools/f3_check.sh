#!/bin/bash
# parity subset + p = 4 times for variant libraries: tools/f3_check.sh NAME...
cd "$(dirname "$0")/.."
for v in "$@"; do
  echo "== $v"
  MFWQ_LIB=$PWD/tools/exp/libmfwq_$v.so timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_otf.py -x -q -m gpu 2>&1 | tail -3
done
tools/f3_abl.sh "$@"
