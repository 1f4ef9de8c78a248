#!/bin/bash
# Final round measurements on one B200 (gpurun --timeout 3000 -- bash scripts/final_gpu.sh): GPU suite,
# smoke, benches of every config and the reference arm, then the ncu captures behind profiles/ncu_traffic.json.
set -u
python -m pytest tests -m gpu -x -q > gpurun_out/final_suite.log 2>&1; echo suite_rc=$? >> gpurun_out/final_suite.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/final_smoke.log 2>&1; echo smoke_rc=$? >> gpurun_out/final_smoke.log
python bench.py > gpurun_out/final_c5.json.log 2>&1
python bench.py --impl reference > gpurun_out/final_c5_ref.json.log 2>&1
for c in c3 c2 c4 pr1; do python bench.py --config $c --no-cpu-baseline > gpurun_out/final_$c.json.log 2>&1; done
bash profiles/capture.sh c5 > gpurun_out/capture_c5.log 2>&1
bash profiles/capture.sh c3 "k_tile_gram k_tile_ws" > gpurun_out/capture_c3.log 2>&1
ls gpurun_out
