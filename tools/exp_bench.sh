#!/bin/bash
# kernel_ms for experiment builds vs the real one: EXPS="a b" CONFIGS="pfac:1000 pfac:10 dpi:10000" tools/exp_bench.sh
for v in $EXPS ""; do
  for ck in ${CONFIGS:-pfac:1000 pfac:10}; do
    c=${ck%%:*}; k=${ck##*:}
    lib=$PWD/paper_1704_02278_b200/libglop${v:+_exp_$v}.so
    GLOP_LIB=$lib timeout 300 python bench.py --config $c --steps 10 --warmup 3 --no-cpu --no-e2e --no-sweep --no-configs --no-parity --patterns $k 2>&1 | tail -1 | \
      python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('${v:-main} $c k=$k kernel_ms', r['kernel_ms'], 'step_ms', d['ms_per_step'], 'frac', r['frac'], 'hits', d['results']['stage1_hits_per_gpu_step'])"
  done
done
