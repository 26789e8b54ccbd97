#!/bin/bash
# A/B of the large path's patch-group size (variant libraries tools/lib_g<N>.so): C4 bench, two passes
o=gpurun_out
for pass in 1 2; do
  for v in "$@"; do
    PVO_LIB=tools/lib_$v.so timeout 600 python bench.py --no-cpu --config c4 --steps 20 --warmup 3 2>/dev/null | tail -1 > $o/g_${v}_c4.json
    python -c "import json; d=json.load(open('$o/g_${v}_c4.json')); print('$v c4 step', round(d['ms_per_step'],4), 'ba', round(d['ba_ms'],4))" >> $o/g_ab.txt
  done
done
