#!/bin/bash
# kernel_ms for the experiment builds and the real one (2 GB, k=1000 / k=10)
for v in exp_NOWORK exp_NODRAIN ""; do
  for k in 1000 10; do
    lib=$PWD/paper_1704_02278_b200/libglop${v:+_$v}.so
    GLOP_LIB=$lib timeout 300 python bench.py --steps 10 --warmup 3 --bytes-per-gpu 2e9 --no-cpu --no-e2e --patterns $k 2>&1 | tail -1 | \
      python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('${v:-full} k=$k kernel_ms', r['kernel_ms'], 'frac', r['frac'])"
  done
done
