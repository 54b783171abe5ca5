"""C-ABI behaviour on the GPU: end-to-end host-buffer runs, argument errors,
graph cache, variant switching, stream semantics."""
import numpy as np
import pytest
import torch

from paper_2301_11389_b200 import inputs
from paper_2301_11389_b200.binding import Stencil, StencilError
from parity import assert_parity

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("kind,dtype,shape,n", [
    ("gaussblur5x5", "f32", (130, 260), 3), ("wave13pt", "f64", (12, 14, 66), 4),
    ("gradient", "f32", (9, 10, 132), 2), ("tricubic", "f32", (8, 19, 132), 1)])
def test_run_host_matches_oracle(oracle, kind, dtype, shape, n):
    ar = oracle.arity(kind)
    ins = [inputs.generate_np(shape, dtype, inputs.BASE_SEED + 31, a) for a in range(ar["n_in"])]
    if ar["n_bufs"] == 2:
        bufs, n_up, n_down = [ins[0], np.zeros_like(ins[0])], 1, 1
    elif kind == "wave13pt":
        bufs, n_up, n_down = [ins[0], ins[1], np.zeros_like(ins[0])], 2, 1
    else:
        bufs = ins + [np.zeros_like(ins[0]) for _ in range(ar["n_out"])]
        n_up, n_down = ar["n_in"], ar["n_out"]
    ob = [b.copy() for b in bufs]
    ridx = oracle.run(kind, dtype, ob, n)
    st = Stencil(kind, shape[::-1], dtype)
    dev = [torch.zeros(shape, dtype=torch.from_numpy(ins[0]).dtype, device="cuda") for _ in bufs]
    h_in = [torch.from_numpy(b.copy()).pin_memory() for b in bufs[:n_up]]
    h_out = [torch.empty(shape, dtype=h_in[0].dtype).pin_memory() for _ in range(n_down)]
    st.run_host(h_in, h_out, dev, n)
    for k in range(n_down):
        assert_parity(h_out[k].numpy(), ob[ridx + k], dtype, f"{kind} run_host out{k}")


def test_run_host_async_two_stream_pipeline(oracle):
    """stencil_run_host_async on two handles / workspaces / streams (the
    bench's pipelined e2e): each lane's result equals the oracle, including
    when the inputs differ per step."""
    shape, n = (96, 260), 4
    fields = [inputs.generate_np(shape, "f32", inputs.BASE_SEED + 40 + k) for k in range(4)]
    refs = []
    for f in fields:
        ob = [f.copy(), np.zeros_like(f)]
        refs.append(ob[oracle.run("gaussblur5x5", "f32", ob, n)])
    streams = [torch.cuda.current_stream(), torch.cuda.Stream()]
    lanes = [(Stencil("gaussblur5x5", shape[::-1], "f32"),
              [torch.zeros(shape, device="cuda") for _ in range(2)], s) for s in streams]
    h_in = [torch.from_numpy(f.copy()).pin_memory() for f in fields]
    h_out = [torch.empty(shape).pin_memory() for _ in fields]
    ev = torch.cuda.Event()
    ev.record(streams[0])
    streams[1].wait_event(ev)
    for k in range(4):
        st, dev, s = lanes[k % 2]
        st.run_host_async([h_in[k]], [h_out[k]], dev, n, s)
    torch.cuda.synchronize()
    for k in range(4):
        assert_parity(h_out[k].numpy(), refs[k], "f32", f"pipelined step {k}")


def test_argument_errors():
    st = Stencil("jacobi2d5", (64, 32), "f32")
    a = torch.zeros((32, 64), device="cuda")
    with pytest.raises(StencilError) as e:
        st.step([a], [a])                                   # aliasing
    assert e.value.code == -1
    big = torch.zeros(32 * 64 + 1, device="cuda")
    with pytest.raises(StencilError) as e:
        st.step([big[1:]], [a])                             # 4-byte offset: not 16-B aligned
    assert e.value.code == -3
    with pytest.raises(StencilError):
        st.run([a, a], 2)                                   # aliasing run buffers
    with pytest.raises(StencilError):
        st.step_range([a], [torch.zeros_like(a)], 0, 5)     # range includes the boundary row
    with pytest.raises(StencilError):
        st.run([a, torch.zeros_like(a)], -1)


def test_graph_cache_and_variant_switch(oracle):
    shape = (40, 136)
    f = inputs.generate_np(shape, "f32", 5)
    bufs = [f.copy(), np.zeros_like(f)]
    ridx = oracle.run("jacobi2d9", "f32", bufs, 4)
    st = Stencil("jacobi2d9", shape[::-1], "f32")
    st.set_fusion(1)
    d = [torch.from_numpy(f).cuda(), torch.zeros(shape, device="cuda")]
    results = []
    for var in ("shuffle", "plain", "paper_ptxasw", "shuffle"):
        st.set_variant(var)
        d[0].copy_(torch.from_numpy(f))
        idx = st.run(d, 4)                                  # cached graph per (bufs, n, variant)
        torch.cuda.synchronize()
        results.append(d[idx].cpu().numpy().copy())
        assert_parity(results[-1], bufs[ridx], "f32", var)
    for r in results[1:]:
        assert np.array_equal(r.view(np.uint8), results[0].view(np.uint8))


@pytest.mark.parametrize("kind,dtype,expect", [
    ("gaussblur5x5", "f32", "shuffle"), ("jacobi2d5", "f32", "shuffle"), ("tricubic", "f32", "plain"),
    ("lapgsrb", "f32", "shuffle"), ("gameoflife", "i32", "shuffle"), ("wave13pt", "f64", "plain")])
def test_auto_variant_resolves_per_kind(kind, dtype, expect):
    """ST_AUTO resolves in the library to the kind's measured-faster variant
    (stencil.h) and stencil_get_variant reports it."""
    shape = (12, 12, 132) if kind in ("tricubic", "lapgsrb", "wave13pt") else (40, 136)
    st = Stencil(kind, shape[::-1], dtype, variant="auto")
    assert st.variant == expect
    assert st.info()["variant"] == (0 if expect == "shuffle" else 1)
    st.set_variant("shuffle")
    assert st.variant == "shuffle"


def test_run_on_a_side_stream_and_zero_iterations():
    shape = (20, 132)
    f = inputs.generate_np(shape, "f32", 6)
    st = Stencil("gaussblur5x5", shape[::-1], "f32")
    a = torch.from_numpy(f).cuda()
    b = torch.full(shape, 3.0, device="cuda")
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        idx = st.run([a, b], 0, stream=s)                   # only the ring copy
    s.synchronize()
    assert idx == 0
    ring = np.ones(shape, bool)
    ring[2:-2, 2:-2] = False
    bb = b.cpu().numpy()
    assert np.array_equal(bb[ring], f[ring]) and np.all(bb[~ring] == 3.0)


def test_info_fields():
    st = Stencil("wave13pt", (66, 20, 16), "f64")
    i = st.info()
    assert i["interior_points"] == 62 * 16 * 12
    assert i["bytes_per_point"] == 24.0 and i["launches_per_step"] == 1
    assert i["lo"] == 2 and i["hi"] == 2 and i["nranks"] == 1


def test_fusion_settings_validated():
    """stencil_set_fusion: 0 auto, 1 off, 2 / 3 streaming (exactly that many
    sweeps per launch), -S tile kernel; anything else ST_EARG; three
    streaming sweeps of gaussblur ST_EUNSUPPORTED; info reports the depth."""
    st = Stencil("jacobi2d5", (4100, 600), "f32")
    for fu, spl in ((2, 2), (3, 3), (1, 1)):
        st.set_fusion(fu)
        assert st.info()["sweeps_per_launch"] == spl
    for bad in (-1, 4, 65, -65):
        with pytest.raises(StencilError) as e:
            st.set_fusion(bad)
        assert e.value.code == -1
    # three streaming sweeps need separable weights (OpGauss5Sep); the default
    # binomial is separable and runs two sweeps per launch automatically
    w = np.arange(25, dtype=np.float64) / 300.0           # rank 2: not separable
    g = Stencil("gaussblur5x5", (4100, 600), "f32", coeffs=w)
    with pytest.raises(StencilError) as e:
        g.set_fusion(3)
    assert e.value.code == -2
    assert g.info()["sweeps_per_launch"] == 1              # auto: the 25-tap form stays single-sweep
    g.set_fusion(2)
    assert g.info()["sweeps_per_launch"] == 2
    b = Stencil("gaussblur5x5", (4100, 600), "f32")       # binomial: separable
    assert b.info()["sweeps_per_launch"] == 2
    b.set_fusion(3)
    assert b.info()["sweeps_per_launch"] == 3
