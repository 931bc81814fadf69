#!/bin/bash
# Round-end batch on the GPU box: full GPU suite, config-5 shard timing, the
# default bench line and the reference arm, ncu of the 16-RHS passes.
set -x
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu_final.log 2>&1; echo rc=$? >> gpurun_out/pytest_gpu_final.log
tail -3 gpurun_out/pytest_gpu_final.log
HMGPU_VERBOSE=1 timeout 900 python scripts/c5_shard.py 0 8 > gpurun_out/c5_shard_final.txt 2>&1; grep -E "plan16|matvec|hmv16|storage" gpurun_out/c5_shard_final.txt | tail -14
python bench.py > gpurun_out/bench_final.json 2> gpurun_out/bench_final.err; echo bench rc=$?
python bench.py --impl reference > gpurun_out/bench_final_reference.json 2> gpurun_out/bench_final_reference.err; echo ref rc=$?
timeout 1000 ncu --set full --clock-control none --import-source on -k regex:hmv16 -s 2 -c 2 -f -o gpurun_out/m16_final python scripts/prof_mrhs.py c3 16 > gpurun_out/m16_final_ncu.log 2>&1; tail -2 gpurun_out/m16_final_ncu.log
