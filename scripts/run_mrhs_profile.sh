set -x
python bench.py > gpurun_out/bench_s4c.json 2> gpurun_out/bench_s4c.err; echo rc=$?
timeout 1000 ncu --set full --clock-control none --import-source on -k regex:hmv16 -s 2 -c 2 -f -o gpurun_out/m16_s4c python scripts/prof_mrhs.py c3 16 > gpurun_out/m16_s4c_ncu.log 2>&1; tail -2 gpurun_out/m16_s4c_ncu.log
