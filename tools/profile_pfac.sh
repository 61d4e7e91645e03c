#!/bin/bash
# ncu evidence for the PFAC kernels (run under gpurun, one GPU).
#   tools/profile_pfac.sh TAG [extra bench args]
# Writes gpurun_out/prof_<TAG>.ncu-rep (full set, one launch of the dominant
# kernel) and gpurun_out/launches_<TAG>.csv (every launch, device time).
set -u
TAG=${1:-pfac}; shift || true
ARGS="--steps 2 --warmup 3 --no-e2e --no-cpu --no-sweep --no-configs --no-parity $*"
ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv \
    --log-file gpurun_out/launches_${TAG}.csv python bench.py $ARGS > gpurun_out/launches_${TAG}.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:${KREGEX:-pfac8} -s 3 -c 1 \
    -o gpurun_out/prof_${TAG} -f python bench.py $ARGS > gpurun_out/prof_${TAG}.log 2>&1
tail -3 gpurun_out/prof_${TAG}.log
