#!/bin/bash
# cfg2 sweep: bench per-degree figures with the previous library (memset + plain launch) vs the
# current one (zero pass + programmatic dependent launch of the fused kernel); timing only
cd "$(dirname "$0")/.."
for lib in tools/abl/libmfwq_old.so paper_1712_08565_b200/libmfwq.so; do
  MFWQ_LIB=$lib python bench.py --steps 30 --pcg 0 --cpu-baseline 0 | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$(basename $lib)', round(d['value']/1e9,3), 'e9 DoF/s', d['ms_per_step'], {k: round(v,1) for k,v in d['per_degree_us'].items()})"
done
