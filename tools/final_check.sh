#!/bin/bash
# Final check of the in-tree build on one B200: GPU suite, smoke, bench lines C2 / C4 / C5 + the reference arm,
# the per-frame pipeline loop.  usage: tools/final_check.sh <tag>
tag=${1:-r2h}
o=gpurun_out
timeout 900 python -m pytest tests -m gpu -q 2>&1 | tail -3 > $o/${tag}_gpu.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $o/${tag}_smoke.txt 2>&1
timeout 600 python bench.py 2>/dev/null | tail -1 > $o/${tag}_bench_c2.json
timeout 900 python bench.py --config c4 --steps 20 --warmup 3 2>/dev/null | tail -1 > $o/${tag}_bench_c4.json
timeout 1200 python bench.py --config c5 --steps 3 --warmup 3 2>/dev/null | tail -1 > $o/${tag}_bench_c5.json
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 2>/dev/null | tail -1 > $o/${tag}_bench_ref_c2.json
{ timeout 600 python tools/pipeline_loop.py 40 c2; timeout 600 python tools/pipeline_loop.py 40 c2 images; } > $o/${tag}_pipeline_c2.txt 2>&1
