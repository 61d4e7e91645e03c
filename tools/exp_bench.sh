#!/bin/bash
# kernel_ms for experiment builds vs the real one: EXPS="a b" tools/exp_bench.sh
for v in $EXPS ""; do
  for k in ${KS:-1000 10}; do
    lib=$PWD/paper_1704_02278_b200/libglop${v:+_exp_$v}.so
    GLOP_LIB=$lib timeout 300 python bench.py --steps 10 --warmup 3 --bytes-per-gpu ${BYTES:-8e9} --no-cpu --no-e2e --patterns $k 2>&1 | tail -1 | \
      python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('${v:-main} k=$k kernel_ms', r['kernel_ms'], 'frac', r['frac'], 'hits', d['results']['stage1_hits_per_gpu_step'])"
  done
done
