#!/bin/bash
# build a variant of the warp-specialised kernel only: tools/f3_variant.sh NAME "-DMFWQ_F3_ABL=1 ..." -> tools/exp/libmfwq_NAME.so
# (fused3.cu recompiled with the flags, every other object taken from build/mfwq)
set -e
cd "$(dirname "$0")/.."
NAME=$1; shift
mkdir -p build/var_$NAME tools/exp
NCCL_INC=$(python - <<'PY'
import nvidia.nccl as nc, os
print(os.path.join(list(nc.__path__)[0], "include"))
PY
)
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC --expt-relaxed-constexpr \
  -Iinclude -Ipaper_1712_08565_b200/csrc -I$NCCL_INC "$@" -c paper_1712_08565_b200/csrc/fused3.cu -o build/var_$NAME/fused3.cu.o
OBJS=$(ls build/mfwq/*.o | grep -v fused3.cu.o)
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o tools/exp/libmfwq_$NAME.so $OBJS build/var_$NAME/fused3.cu.o \
  -lcusolver -ldl -Xlinker -rpath,/usr/local/cuda/lib64 -L/usr/local/cuda/lib64
echo tools/exp/libmfwq_$NAME.so
