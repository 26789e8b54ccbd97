#!/bin/bash
# Round-end measurement on one B200: tests, smoke, bench lines per config, the
# reference arm, the ncu launch list and full captures.  usage: tools/round_measure.sh <tag>
tag=${1:-r1f}
o=gpurun_out
timeout 900 python -m pytest tests -m gpu -q 2>&1 | tail -3 > $o/${tag}_gpu.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $o/${tag}_smoke.txt 2>&1
timeout 600 python bench.py 2>/dev/null | tail -1 > $o/${tag}_bench_c2.json
for c in c1 c3; do timeout 600 python bench.py --config $c 2>/dev/null | tail -1 > $o/${tag}_bench_$c.json; done
timeout 900 python bench.py --config c4 --steps 20 --warmup 3 2>/dev/null | tail -1 > $o/${tag}_bench_c4.json
timeout 1200 python bench.py --config c5 --steps 3 --warmup 3 2>/dev/null | tail -1 > $o/${tag}_bench_c5.json
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 2>/dev/null | tail -1 > $o/${tag}_bench_ref_c2.json
{ timeout 600 python tools/pipeline_loop.py 40 c2; timeout 600 python tools/pipeline_loop.py 40 c2 images; } > $o/${tag}_pipeline_c2.txt 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 300 --csv --log-file $o/${tag}_launches_bench.csv \
  python bench.py --no-cpu --steps 20 --warmup 3 > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:corr_tma_kernel -s 5 -c 1 -o $o/${tag}_corr_full \
  python bench.py --no-cpu --steps 10 --warmup 3 > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:ba_kernel -s 5 -c 1 -o $o/${tag}_ba_full \
  python bench.py --no-cpu --steps 10 --warmup 3 > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:corr_prep_kernel -s 5 -c 1 -o $o/${tag}_prep_full \
  python bench.py --no-cpu --steps 10 --warmup 3 > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:corr_tma_kernel -s 2 -c 1 -o $o/${tag}_corr_c4_full \
  python bench.py --no-cpu --config c4 --steps 5 --warmup 3 > /dev/null 2>&1
ls $o | grep $tag
timeout 600 ncu --set full --clock-control none --import-source on -k regex:measure_gram_kernel -s 1 -c 1 -o $o/${tag}_measure_full \
  python tools/prof_measure.py c2 2 > /dev/null 2>&1
