# lane-replicated level-1 layout vs the gram-count default (k = patterns).
# (A two-bits-per-gram lane variant measured slower at every k: 10 -> 1.76 ms,
# 100 -> 2.04 ms, 400 -> 2.36 ms.)
for k in ${KS:-30 50 300}; do
 for v in "GLOP_P8_LANE_MAX=0" "GLOP_P8_LANE_MIN=0 GLOP_P8_LANE_MAX=1000000"; do
  env $v timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu --no-e2e --no-sweep --no-configs --no-parity --patterns $k 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('$v k=$k kernel_ms', r['kernel_ms'], 'frac', r['frac'], 'hits', d['results']['stage1_hits_per_gpu_step'])"
 done
done
