"""Debug: determinism of the batch volume across block compositions."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np
from tests.test_gpu_sharding import _run_block

a = _run_block([0, 1, 2, 3])
b = _run_block([0, 1, 2, 3])
c = _run_block(list(range(8)))
for name, other in (("rerun", b), ("g1", c)):
    for sid in range(4):
        va, vb = a[sid][3], other[sid][3]
        diff = np.argwhere(va.view(np.uint32) != vb.view(np.uint32))
        print(name, sid, "poses eq", np.array_equal(a[sid][0], other[sid][0]), "vol diffs", len(diff),
              "nan", int(np.isnan(va).sum()), diff[:5].tolist(), va[tuple(diff[0])] if len(diff) else None,
              vb[tuple(diff[0])] if len(diff) else None, flush=True)
