#!/bin/bash
# A/B of the large-window diagonal-block variants (tools/lib_d1.so, tools/lib_d4.so): phase clocks,
# C4 bench, and bit-identity of the C4 optimize_window(2) result between them
o=gpurun_out
for v in d1 d4; do
  PVO_LIB=tools/lib_$v.so timeout 300 python tools/prof_large.py c4 2>&1 | tail -1 | sed "s/^/$v /" >> $o/d_ab.txt
  PVO_LIB=tools/lib_$v.so timeout 300 python tools/ba_dump.py c4 $o/d_$v.npz >> $o/d_ab.txt 2>&1
done
python -c "
import numpy as np
a, b = np.load('$o/d_d1.npz'), np.load('$o/d_d4.npz')
print('bit-identical', all(np.array_equal(a[k], b[k]) for k in ('poses', 'depth', 'norms')))" >> $o/d_ab.txt 2>&1
for pass in 1 2; do for v in d1 d4; do
  PVO_LIB=tools/lib_$v.so timeout 600 python bench.py --no-cpu --config c4 --steps 20 --warmup 3 2>/dev/null | tail -1 > $o/d_${v}_c4.json
  python -c "import json; d=json.load(open('$o/d_${v}_c4.json')); print('$v c4 step', round(d['ms_per_step'],4), 'ba', round(d['ba_ms'],4))" >> $o/d_ab.txt
done; done
