#!/bin/bash
# One GPU session: parity tests, smoke, default bench, KMP bench, ncu launch
# list + one full capture of the PFAC kernel.  Outputs under gpurun_out/.
set -u
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi.txt 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
tail -3 gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; tail -1 gpurun_out/smoke.log
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; tail -c 3000 gpurun_out/bench.json
timeout 600 python bench.py --config kmp > gpurun_out/bench_kmp.json 2> gpurun_out/bench_kmp.err; tail -c 1500 gpurun_out/bench_kmp.json
timeout 300 python bench.py --patterns 10 --no-cpu --no-e2e --no-sweep > gpurun_out/bench_k10.json 2>&1; tail -c 1200 gpurun_out/bench_k10.json
timeout 600 python bench.py --config dpi > gpurun_out/bench_dpi.json 2>&1; tail -c 1500 gpurun_out/bench_dpi.json
timeout 900 python bench.py --impl reference > gpurun_out/bench_ref.json 2>&1; tail -c 800 gpurun_out/bench_ref.json
if [ "${PROFILE:-1}" = 1 ]; then
  timeout 900 tools/profile_pfac.sh k1000
  timeout 600 tools/profile_pfac.sh k10 --patterns 10
  KREGEX=kmp3 timeout 600 tools/profile_pfac.sh kmp --config kmp
  timeout 600 tools/profile_pfac.sh dpi --config dpi
fi
