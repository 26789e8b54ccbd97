"""Time the LDLT pose solve alone (schur_solve with a trivial depth block)."""
import sys
import time
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import paper_2208_04726_b200 as pvo  # noqa: E402

ctx = pvo.Context(0)
rng = np.random.default_rng(0)
for npp in [int(x) for x in (sys.argv[1:] or ["42", "60", "96"])]:
    a = rng.standard_normal((npp, npp))
    a = a @ a.T + npp * np.eye(npp)
    b = rng.standard_normal(npp)
    hpd = np.zeros((npp, 1))
    for _ in range(3):
        pvo.schur_solve(a, hpd, [1.0], b, [0.0], ctx=ctx)
    t = time.perf_counter()
    for _ in range(20):
        dp, dd = pvo.schur_solve(a, hpd, [1.0], b, [0.0], ctx=ctx)
    print(npp, "host-timed ms/solve", (time.perf_counter() - t) / 20 * 1e3, "err", np.abs(dp - np.linalg.solve(a, b)).max())
