#!/bin/bash
# Static SASS statistics of the fused matvec kernel for one degree (fast iteration aid):
#   tools/sass_stats.sh 4 [NT=3]   -> registers/stack + opcode histogram of k_fused<P,NT,2>
P=${1:-4}; NT=${2:-3}
cd "$(dirname "$0")/.."
mkdir -p build/sass
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -DMFWQ_ONLY_P=$P $MFWQ_NVCC_EXTRA \
  -Iinclude -Ipaper_1712_08565_b200/csrc -cubin -o build/sass/f2_p$P.cubin paper_1712_08565_b200/csrc/fused2.cu || exit 1
K="k_fusedILi${P}ELi${NT}ELi${ZS:-2}E"
cuobjdump -res-usage build/sass/f2_p$P.cubin | grep -A1 "$K" | grep -o "REG:[0-9]*\|STACK:[0-9]*" | tr '\n' ' '; echo
cuobjdump -sass -fun "$(cuobjdump -sass build/sass/f2_p$P.cubin | grep -o "Function : .*$K[^ ]*" | head -1 | cut -d' ' -f3)" build/sass/f2_p$P.cubin \
  | grep -E '^\s+/\*[0-9a-f]+\*/' | sed -E 's/^\s+\/\*[0-9a-f]+\*\/\s+(@!?U?P[0-9T] )?//' | awk '{print $1}' \
  | sed -E 's/\..*//' | sort | uniq -c | sort -rn | head -${TOP:-25} | tr '\n' ' '; echo
