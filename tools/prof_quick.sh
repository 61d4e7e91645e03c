#!/bin/bash
# full ncu capture of the pfac8 kernel for k=1000 and k=10 (2 GB) + quick bench
mkdir -p gpurun_out
for k in ${KS:-1000 10}; do
ncu --set full --clock-control none --import-source on -k regex:${KREGEX:-pfac8} -s 3 -c 1 \
    -o gpurun_out/prof_q$k -f python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu --bytes-per-gpu 2e9 --no-sweep --patterns $k > gpurun_out/prof_q$k.log 2>&1
done
SKIP_TESTS=1 bash tools/quick_bench.sh
