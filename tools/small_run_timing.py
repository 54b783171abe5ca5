"""Where the time of a small 2-D run goes (BASELINE configs[0], jacobi 512^2 x10):
event-timed stencil_run for n_iters = 0 (graph launch + ring copy only), 1, 10,
with and without an L2 flush before each timed run, and a bare graph of one
empty kernel for the launch floor.

    python tools/small_run_timing.py
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2301_11389_b200 import inputs  # noqa: E402
from paper_2301_11389_b200.binding import Stencil  # noqa: E402


rd = torch.empty(64 << 20, device="cuda")


def timed(fn, flush, reps=30, queued=False, read=False):
    """median / min microseconds between events around fn(); queued=True
    keeps the GPU busy (a 50 us spin kernel after the flush) while the host
    submits, so host-side call overhead cannot open a gap in the window."""
    ts = []
    for _ in range(reps):
        if flush is not None:
            flush.fill_(1.0)
        if read:
            rd.sum()                  # a read of another > L2 buffer: evicts the flush's dirty lines
        if queued:
            torch.cuda._sleep(100000)
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) * 1e3)
    ts.sort()
    return ts[len(ts) // 2], ts[0]


flush = torch.empty(64 << 20, device="cuda")
# the launch floor: a graph holding one tiny kernel
x = torch.zeros(4, device="cuda")
s = torch.cuda.Stream()
g = torch.cuda.CUDAGraph()
with torch.cuda.graph(g, stream=s):
    x.add_(1.0)
for fl in (None, flush):
    print("empty-kernel graph", "flush" if fl is not None else "warm", "median/min us", timed(g.replay, fl))
    print("empty-kernel direct launch", "flush" if fl is not None else "warm", "median/min us",
          timed(lambda: x.add_(1.0), fl))
print("empty-kernel direct launch flush+queued median/min us", timed(lambda: x.add_(1.0), flush, queued=True))
print("empty-kernel graph flush+queued median/min us", timed(g.replay, flush, queued=True))
print("empty-kernel direct launch warm+queued median/min us", timed(lambda: x.add_(1.0), None, queued=True))
print("no kernel at all (two events) flush+queued median/min us", timed(lambda: None, flush, queued=True))
print("no kernel at all (two events) warm+queued median/min us", timed(lambda: None, None, queued=True))
print("empty-kernel direct launch flush+read median/min us", timed(lambda: x.add_(1.0), flush, read=True))
print("empty-kernel direct launch flush+read+queued median/min us",
      timed(lambda: x.add_(1.0), flush, read=True, queued=True))
for variant in ("shuffle", "plain"):
    for n in (0, 1, 10):
        st = Stencil("jacobi2d5", (512, 512), "f32", variant=variant)
        a = inputs.generate_torch((512, 512), "f32", 1)
        b = torch.zeros_like(a)
        for _ in range(3):
            st.run([a, b], n)
        torch.cuda.synchronize()
        for fl in (None, flush):
            print(variant, "n_iters", n, "flush" if fl is not None else "warm", "median/min us",
                  timed(lambda: st.run([a, b], n), fl))
        print(variant, "n_iters", n, "flush+queued", "median/min us",
              timed(lambda: st.run([a, b], n), flush, queued=True))
        print(variant, "n_iters", n, "warm+queued", "median/min us",
              timed(lambda: st.run([a, b], n), None, queued=True))
        print(variant, "n_iters", n, "flush+read", "median/min us",
              timed(lambda: st.run([a, b], n), flush, read=True))
        st.close()
