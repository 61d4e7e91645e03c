#!/bin/bash
# kernel_ms at k=1000 / DPI for libs x GLOP_P8_CHUNKS values: LIBS="a b" CH="32 64" tools/scratch/chunks_ab.sh
for lib in $LIBS; do for ch in $CH; do for ck in ${CONFIGS:-pfac:1000 dpi:10000}; do
  c=${ck%%:*}; k=${ck##*:}
  GLOP_P8_CHUNKS=$ch GLOP_LIB=$PWD/paper_1704_02278_b200/libglop_exp_$lib.so timeout 300 python bench.py --config $c --steps 10 --warmup 3 \
    --no-cpu --no-e2e --no-sweep --no-configs --no-parity --patterns $k 2>&1 | tail -1 | \
    python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('$lib ch=$ch $c k=$k kernel_ms', r['kernel_ms'], 'step_ms', d['ms_per_step'])"
done; done; done
