#!/bin/bash
# usage: abbench.sh "<bench args>" lib1 lib2 ...   (copies each lib in place, runs bench, prints ms/step + stages)
args=$1; shift
for lib in "$@"; do
  cp $lib paper_2511_03126_b200/_lib/libpropfield_b200.so
  python bench.py $args --no-e2e --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$lib', round(d['ms_per_step'],4), {k: round(v,3) for k,v in d.get('stages_ms',{}).items()})"
done
