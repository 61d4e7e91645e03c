# lane-replicated level-1 vs the gram-count default (k = patterns)
for k in ${KS:-30 50 300}; do
 for lm in 0 1000000; do
  GLOP_P8_LANE_MIN=0 GLOP_P8_LANE_MAX=$lm timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu --no-e2e --no-sweep --no-configs --no-parity --patterns $k 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('lanemax $lm k=$k kernel_ms', r['kernel_ms'], 'frac', r['frac'], 'hits', d['results']['stage1_hits_per_gpu_step'])"
 done
done
