#!/bin/bash
# One GPU session: parity tests, smoke, the bench lines the round reports
# (default = configs[2] + sub-configs, reference arm, KMP, DPI, k=10), ncu
# launch lists + one full capture per workload.  Outputs under gpurun_out/.
#   R=02 tools/gpu_check.sh        (PROFILE=0 skips ncu, TESTS=0 skips pytest)
set -u
R=${R:-02}
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi.txt 2>&1
if [ "${TESTS:-1}" = 1 ]; then
  timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/r${R}_pytest_gpu.log 2>&1; tail -3 gpurun_out/r${R}_pytest_gpu.log
  timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r${R}_smoke.log 2>&1; tail -1 gpurun_out/r${R}_smoke.log
fi
timeout 900 python bench.py > gpurun_out/r${R}_bench.json 2> gpurun_out/r${R}_bench.err; tail -c 600 gpurun_out/r${R}_bench.json
timeout 900 python bench.py --impl reference > gpurun_out/r${R}_bench_ref.json 2> gpurun_out/r${R}_bench_ref.err; tail -c 400 gpurun_out/r${R}_bench_ref.json
timeout 600 python bench.py --config kmp > gpurun_out/r${R}_bench_kmp.json 2> gpurun_out/r${R}_bench_kmp.err
timeout 600 python bench.py --config dpi --no-parity > gpurun_out/r${R}_bench_dpi.json 2> gpurun_out/r${R}_bench_dpi.err
timeout 300 python bench.py --patterns 10 --no-cpu --no-e2e --no-sweep --no-configs --no-parity > gpurun_out/r${R}_bench_k10.json 2>&1
if [ "${PROFILE:-1}" = 1 ]; then
  timeout 900 tools/profile_pfac.sh k1000
  timeout 600 tools/profile_pfac.sh k10 --patterns 10
  timeout 600 tools/profile_pfac.sh k10000 --patterns 10000
  KREGEX=kmp3 timeout 600 tools/profile_pfac.sh kmp --config kmp
  timeout 600 tools/profile_pfac.sh dpi --config dpi
fi
