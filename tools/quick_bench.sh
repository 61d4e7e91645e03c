#!/bin/bash
# quick GPU check: parity subset + kernel/step times at k=1000 and k=10 (2 GB)
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -x -q ${TESTS:+-k "$TESTS"} 2>&1 | tail -2
for k in 1000 10; do
  timeout 300 python bench.py --steps 10 --warmup 3 --bytes-per-gpu ${BYTES:-2e9} --no-cpu --no-e2e --patterns $k "$@" 2>&1 | tail -1 | \
    python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('k=$k', d['value'], 'Gbps frac', r['frac'], 'kernel_ms', r['kernel_ms'], 'step_ms', d['ms_per_step'])"
done
