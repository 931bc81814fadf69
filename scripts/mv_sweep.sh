#!/bin/bash
# Stream-matvec configuration sweep (development helper): bench value per
# HMGPU_MV_CFG="warps,stages,stage_doubles,scratch_doubles".
cfg=${1:-c2}; shift
for v in "$@"; do
  HMGPU_MV_CFG=$v python bench.py --config $cfg --no-cpu --steps 20 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().split('\n')[-1]); print('$cfg $v', round(d['value']/1e6,2), round(d['ms_per_step'],4), round(d['kernel_ms']['hmv_stream'],4), round(d['kernel_ms']['hmv_ypart'],4))"
done
