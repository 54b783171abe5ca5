import sys, os, time
sys.path.insert(0, os.getcwd())
import torch
from paper_2301_11389_b200 import inputs
from paper_2301_11389_b200.binding import Stencil
for fusion in (1, 0):
    st = Stencil("jacobi2d5", (512, 512), "f32"); st.set_fusion(fusion)
    a = inputs.generate_torch((512, 512), "f32", 1); b = torch.zeros_like(a)
    flush = torch.empty(64 << 20, device="cuda")
    for _ in range(5): st.run([a, b], 10)
    torch.cuda.synchronize()
    for fl in (False, True):
        ts = []
        for _ in range(20):
            if fl: flush.fill_(1.0)
            e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
            e0.record(); st.run([a, b], 10); e1.record(); torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1) * 1e3)
        ts.sort()
        print("fusion", fusion, "flush", fl, "median us", round(ts[10], 1), "min", round(ts[0], 1))
