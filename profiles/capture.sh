#!/bin/bash
# ncu captures behind profiles/rNN_* (run on the GPU box after `python bench.py` exited 0 without ncu):
#   gpurun --timeout 1800 -- 'bash profiles/capture.sh c5'
# Outputs land in gpurun_out/: the launch list (per-launch device time, cold-cache, serialised) and one
# `--set full` capture each of the tile kernel (k_tile_gram for bf16 maps) and the prep kernel.
set -u
cfg=${1:-c5}
kern=${2:-k_tile_gram}
out=gpurun_out
mkdir -p $out
args="--config $cfg --steps 1 --warmup 3 --no-e2e --no-cpu-baseline"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_[a-z]+" -c 400 --csv \
  --log-file $out/launches_$cfg.csv python bench.py $args > $out/ncu_launch_$cfg.log 2>&1
for k in $kern k_tile_prep; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$k -s 2 -c 1 \
    -o $out/prof_${k}_$cfg -f python bench.py $args > $out/ncu_${k}_$cfg.log 2>&1
done
echo capture-done
