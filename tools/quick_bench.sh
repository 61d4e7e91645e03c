#!/bin/bash
# quick GPU check: parity (TESTS=-k filter, or SKIP_TESTS=1) + kernel/step times at k=1000 and k=10
mkdir -p gpurun_out
if [ -z "${SKIP_TESTS:-}" ]; then
  timeout 900 python -m pytest tests -m gpu -x -q ${TESTS:+-k "$TESTS"} 2>&1 | tail -15
fi
for k in ${KS:-1000 10}; do
  timeout 300 python bench.py --steps 10 --warmup 3 --bytes-per-gpu ${BYTES:-8e9} --no-cpu --no-e2e --no-sweep --patterns $k "$@" > gpurun_out/qb_$k.json 2> gpurun_out/qb_$k.err
  python -c "import json,sys; d=json.loads(open('gpurun_out/qb_$k.json').read().strip().splitlines()[-1]); r=d['roofline']; print('k=$k', d['value'], 'Gbps frac', r['frac'], 'kernel_ms', r['kernel_ms'], 'step_ms', d['ms_per_step'], 'hits', d['results']['stage1_hits_per_gpu_step'], 'clk', d['clocks']['sm_mhz'], 'launches/step', d['gpu_launches']/d['steps'])" || tail -5 gpurun_out/qb_$k.err
done
