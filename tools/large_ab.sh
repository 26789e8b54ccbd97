#!/bin/bash
# A/B of large-window solver variants tools/lib_<V>.so: phase clocks + C4 bench; then the GPU suite
o=gpurun_out
for v in "$@"; do
  PVO_LIB=tools/lib_$v.so timeout 300 python tools/prof_large.py c4 2>&1 | tail -1 | sed "s/^/$v /" >> $o/l_ab.txt
  PVO_LIB=tools/lib_$v.so timeout 600 python bench.py --no-cpu --config c4 --steps 20 --warmup 3 2>/dev/null | tail -1 > $o/l_${v}_c4.json
  python -c "import json; d=json.load(open('$o/l_${v}_c4.json')); print('$v c4 step', round(d['ms_per_step'],4), 'ba', round(d['ba_ms'],4), 'corr', round(d['corr_ms'],4))" >> $o/l_ab.txt
done
timeout 900 python -m pytest tests -m gpu -q 2>&1 | tail -3 > $o/l_tests.txt
