#!/bin/bash
# sweep HMGPU_MV_CFG over a few pipeline geometries (development helper)
for cfg in "7,2,1536,1024" "6,2,1792,1024" "7,2,1664,640" "6,2,2048,512" "8,2,1408,512" "5,3,1280,768" "6,3,1088,640" "4,3,2048,1024"; do
  echo "== $cfg"
  HMGPU_MV_CFG=$cfg python scripts/probe.py 5 1e-6 2>&1 | grep -E "hmv_stream|hmv_ypart"
  HMGPU_MV_CFG=$cfg python scripts/probe_c3.py 2>&1 | grep -E "hmv_stream|hmv_ypart"
done
