"""Temporal-blocking depth sweep (stencil_set_fusion) on the large 2-D configs.

    python tools/fusion_sweep.py  -> one line per (workload, fusion depth)
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2301_11389_b200 import inputs  # noqa: E402
from paper_2301_11389_b200.binding import Stencil  # noqa: E402

CASES = [("jacobi2d5", "f32", 32768, 10), ("gaussblur5x5", "f32", 8192, 100), ("gameoflife", "i32", 16384, 10),
         ("jacobi2d9", "f32", 32768, 10), ("jacobi2d5", "f64", 16384, 10), ("jacobi2d9", "f64", 16384, 10),
         ("gaussblur5x5", "f64", 8192, 20)]
CASES = [c for c in CASES if not os.environ.get("KINDS") or c[0] + ":" + c[1] in os.environ["KINDS"].split(",")]
for kind, dt, n, iters in CASES:
    a = inputs.generate_torch((n, n), dt, inputs.BASE_SEED + 1)
    b = torch.zeros_like(a)
    for fusion in [int(x) for x in os.environ.get("DEPTHS", "1,2,3,-4,-6,-8").split(",")]:
        st = Stencil(kind, (n, n), dt, variant=os.environ.get("VARIANT", "shuffle"))
        st.set_fusion(fusion)
        for _ in range(2):
            st.run([a, b], iters)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        reps = 3
        e0.record()
        for _ in range(reps):
            st.run([a, b], iters)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / reps
        r = 2 if kind == "gaussblur5x5" else 1
        print(f"{kind:14s} n={n} iters={iters} fusion={fusion}: {(n - 2 * r) ** 2 * iters / (ms / 1e3) / 1e9:8.1f} Gpt/s",
              flush=True)
        st.close()
    del a, b
    torch.cuda.empty_cache()
