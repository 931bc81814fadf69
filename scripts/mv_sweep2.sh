#!/bin/bash
# per-pass sweep: HMGPU_MV_CFG_A values against a fixed pass-B config
cfg=${1:-c2}; B=$2; shift 2
for v in "$@"; do
  HMGPU_MV_CFG_A=$v HMGPU_MV_CFG_B=$B python bench.py --config $cfg --no-cpu --steps 20 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().split('\n')[-1]); print('$cfg A=$v B=$B', round(d['value']/1e6,2), round(d['ms_per_step'],4), round(d['kernel_ms']['hmv_stream'],4), round(d['kernel_ms']['hmv_ypart'],4))"
done
