# A/B the corr kernel variants tools/lib_<V>.so on c2 and c4
for v in "$@"; do
  for c in c2 c4; do
    st=300; [ $c = c4 ] && st=30
    PVO_LIB=tools/lib_$v.so python bench.py --no-cpu --config $c --steps $st 2>&1 | tail -1 > gpurun_out/v_${v}_$c.json
  done
done
python - "$@" <<'PY'
import json, sys
for v in sys.argv[1:]:
    out = []
    for c in ("c2", "c4"):
        try:
            d = json.load(open("gpurun_out/v_%s_%s.json" % (v, c)))
            out.append("%s corr %.4f ms frac %.3f step %.4f" % (c, d["corr_ms"], d["roofline"]["frac"], d["ms_per_step"]))
        except Exception as e:
            out.append("%s failed %s" % (c, e))
    print(v, " | ".join(out))
PY
