# jump-table load factor 1/GLOP_JUMP_SPARSE
for ck in ${CONFIGS:-dpi:10000 pfac:10000 pfac:1000 pfac:100}; do
 c=${ck%%:*}; k=${ck##*:}
 for v in 2 4 8 16; do
  GLOP_JUMP_SPARSE=$v timeout 300 python bench.py --config $c --steps 10 --warmup 3 --no-cpu --no-e2e --no-sweep --no-configs --no-parity --patterns $k 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('sparse $v $c k=$k kernel_ms', r['kernel_ms'], 'frac', r['frac'])"
 done
done
