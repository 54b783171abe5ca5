#!/usr/bin/env python
"""Benchmark of the register-cache stencil hot path on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--workload NAME]
                    [--variant shuffle|plain] [--impl ours|reference]

One *step* = one ``stencil_run(n_iters)`` of the workload (Dirichlet ring
copy + n_iters sweeps, one CUDA graph), i.e. one pass of the whole hot path
(DESIGN.md §1 rows S1-S9) over one synthetic grid.  Default workload:
BASELINE.json configs[1], gaussblur 5x5 fp32 8192x8192, 100 iterations;
for N>1 weak-scaled to 8192 x (8192*N) with a y-slab decomposition, one
process per GPU.  Halo exchange (--transport): p2p (default) = the kernels'
fused peer stores into the neighbours' buffers over CUDA IPC (NVLink /
NVSwitch), falling back on every rank to NCCL send/recv when a rank cannot
map its neighbours' memory; nccl = NCCL send/recv overlapped with the
interior.  Run directly with --gpus N > 1 (no WORLD_SIZE in the
environment), bench.py starts the N ranks itself under
torch.distributed.run.  Prints ONE JSON line (rank 0).

Metric (BASELINE.json): Gpoints/s (interior points x sweeps / s, all ranks)
and achieved HBM GB/s as a fraction of the measured copy bandwidth.

--impl reference: the CPU oracle (oracle/, the plain fp64 C loop nests)
timed on this host's cores on a bounded sample of the same workload; this
is the only other place bench.py executes oracle/ (besides cpu_baseline).
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)
os.environ.setdefault("NCCL_DEBUG", "WARN")     # keep stdout to the one JSON line

# name -> kind, dtype, dims at N=1 (x fastest), iterations, weak-scaled axis
WORKLOADS = {
    "gaussblur": dict(kind="gaussblur5x5", dtype="f32", dims=(8192, 8192), iters=100,
                      config="BASELINE configs[1]: gaussblur 5x5 fp32 8192x8192, 100 iterations"),
    "jacobi2d": dict(kind="jacobi2d5", dtype="f32", dims=(512, 512), iters=10,
                     config="BASELINE configs[0]: jacobi 2D 5-point fp32 512x512, 10 sweeps"),
    "jacobi2d_paper": dict(kind="jacobi2d5", dtype="f32", dims=(32768, 32768), iters=10,
                           config="jacobi 2D 5-point fp32 at the paper's 2-D size 32768^2 (PAPER.md:644)"),
    "jacobi2d9": dict(kind="jacobi2d9", dtype="f32", dims=(32768, 32768), iters=10,
                      config="jacobi 2D 9-point fp32 32768^2 (Table 1 jacobi row, box form; not a BASELINE config)"),
    "jacobi2d_f64": dict(kind="jacobi2d5", dtype="f64", dims=(16384, 16384), iters=10,
                         config="jacobi 2D 5-point fp64 16384^2 (not a BASELINE config)"),
    "gameoflife": dict(kind="gameoflife", dtype="i32", dims=(16384, 16384), iters=10,
                       config="BASELINE configs[3]: gameoflife int32 16384x16384"),
    "laplacian": dict(kind="laplacian3d7", dtype="f64", dims=(512, 512, 512), iters=10,
                      config="BASELINE configs[2]: laplacian 3D 7-point fp64 512^3"),
    "wave13pt": dict(kind="wave13pt", dtype="f64", dims=(512, 512, 512), iters=10,
                     config="BASELINE configs[2]: wave13pt 3D 13-point fp64 512^3"),
    "tricubic": dict(kind="tricubic", dtype="f32", dims=(256, 256, 256), iters=10,
                     config="BASELINE configs[3]: tricubic 3D fp32 256^3",
                     # FMA-pipe lane operations per point of the factored form
                     # (DESIGN.md §5.3): 84 for the sums (64 x + 16 y + 4 z), 24
                     # for the Lagrange weights (8 per axis); one lane-op per
                     # FMUL / FFMA lane, two per FMUL2 / FFMA2 lane
                     lane_ops_per_point=108),
    "jacobi3d": dict(kind="jacobi3d7", dtype="f32", dims=(1024, 1024, 1024), iters=10,
                     config="BASELINE configs[4]: jacobi 3D 7-point fp32 1024^2 x (1024*N)"),
    "divergence": dict(kind="divergence", dtype="f32", dims=(512, 512, 512), iters=10,
                       config="divergence fp32 512^3 (suite member, Table 1)"),
    "gradient": dict(kind="gradient", dtype="f32", dims=(512, 512, 512), iters=10,
                     config="gradient fp32 512^3 (suite member, Table 1)"),
    # SURVEY §8(f) row f3 at the paper's problem sizes
    "uxx1": dict(kind="uxx1", dtype="f32", dims=(512, 512, 1024), iters=10,
                 config="uxx1 fp32 512x512x1024 (suite member, Table 1; paper size)"),
    "whispering": dict(kind="whispering", dtype="f32", dims=(8192, 16384), iters=10,
                       config="whispering fp32 8192x16384 (suite member, Table 1; paper size)"),
    "lapgsrb": dict(kind="lapgsrb", dtype="f32", dims=(512, 1024, 1024), iters=10,
                    config="lapgsrb fp32 512x1024x1024 (suite member, Table 1; paper 3-D size)"),
    "tricubic2": dict(kind="tricubic2", dtype="f32", dims=(256, 256, 256), iters=10,
                      config="tricubic2 fp32 256^3 (suite member, Table 1)", lane_ops_per_point=108),
}
L2_BYTES = 126 * 2**20
METRIC = "Gpoints/s and achieved HBM GB/s (% of ~8 TB/s) per stencil, 1/2/4/8 B200"


def measured_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, copy)"
    return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


def sm_count():
    import torch
    return torch.cuda.get_device_properties(torch.cuda.current_device()).multi_processor_count


def profile_traffic(workload, variant):
    """dram bytes per launch from a committed ncu --set full summary, or None."""
    p = os.path.join(ROOT, "profiles", "traffic.json")
    if not os.path.exists(p):
        return None
    d = json.load(open(p))
    return d.get(f"{workload}:{variant}")


# ------------------------------------------------------------------ clocks
class ClockSampler:
    """nvidia-smi sampling DURING the timed region (B200_PROFILING.md)."""
    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, device_index: int):
        self.dev = device_index
        self.proc = None
        self.lines = []
        self.n0 = 0

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.dev), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "50"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
            t0 = time.time()                 # nvidia-smi takes a moment to start
            while not self.lines and time.time() - t0 < 5 and self.proc.poll() is None:
                time.sleep(0.01)
            self.n0 = len(self.lines)
        except (OSError, FileNotFoundError):
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *a):
        if self.proc:
            time.sleep(0.15)                 # one more sample covering the region's end
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines[max(0, self.n0 - 1):]:
            p = [x.strip() for x in ln.split(",")]
            if len(p) < 7:
                continue
            try:
                sm.append(float(p[0]))
                mx.append(float(p[1]))
            except ValueError:
                continue
            for n, v in zip(names, p[3:7]):
                if v.lower().startswith("active"):
                    reasons.add(n)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
        sm.sort()
        return {"sm_mhz": sm[len(sm) // 2], "sm_max_mhz": max(mx), "reasons": sorted(reasons),
                "samples": len(sm)}


# --------------------------------------------------------- oracle (CPU)
_ORACLE_BUFS = {}


def oracle_sample(wl, seconds: float, nthreads: int):
    """Time the CPU oracle, as it stands, on whole sweeps of the workload's
    full grid (the stated config's dims, same generator, kind, dtype and
    iteration structure): at least one sweep, then whole sweeps until
    `seconds` of wall time have passed.  The bounded part is the number of
    sweeps (a step of the config runs wl["iters"] of them).
    Returns (Gpoints/s, description, seconds per sweep)."""
    import numpy as np
    from oracle import pyoracle
    from paper_2301_11389_b200 import inputs

    kind, dt = wl["kind"], wl["dtype"]
    ar = pyoracle.arity(kind)
    shape = tuple(wl["dims"][::-1])
    key = (kind, dt, shape)
    if key not in _ORACLE_BUFS:              # generated once per process
        seed = inputs.BASE_SEED
        fields = [inputs.generate_np(shape, dt, seed, a) for a in range(max(ar["n_in"], 1))]
        if ar["n_bufs"] == 2:
            bufs = [fields[0], np.zeros_like(fields[0])]
        elif kind == "wave13pt":
            bufs = [fields[0], fields[1], np.zeros_like(fields[0])]
        else:
            bufs = fields[: ar["n_in"]] + [np.zeros_like(fields[0]) for _ in range(ar["n_out"])]
        _ORACLE_BUFS.clear()
        _ORACLE_BUFS[key] = bufs
    bufs = _ORACLE_BUFS[key]
    interior = 1
    for n in shape:
        interior *= n - ar["lo"] - ar["hi"]
    sweeps, t0 = 0, time.perf_counter()
    while True:
        pyoracle.run(kind, dt, bufs, 1, nthreads=nthreads)
        sweeps += 1
        el = time.perf_counter() - t0
        if el >= seconds:
            break
    return (interior * sweeps / el / 1e9,
            f"{kind} {dt} full grid {'x'.join(map(str, wl['dims']))}: {sweeps} whole sweep(s) of the "
            f"config's {wl['iters']} in {el:.2f} s, {nthreads} thread(s)",
            el / sweeps)


def host_cores():
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:
        return os.cpu_count() or 1


# ------------------------------------------------------------ reference
def run_reference(args, wl, world, rank):
    """The reference arm: the oracle as it stands on this host's cores.  Each
    step runs whole sweeps of the config's full grid for a bounded time
    (the whole run stays within a few minutes); ms_per_step is the wall time
    of those sweeps and `value` the same Gpoints/s metric."""
    if rank != 0:
        return
    cores = host_cores()
    per_step = max(1.0, min(10.0, 100.0 / max(1, args.steps + args.warmup)))
    oracle_sample(wl, 0.0, cores)            # generate the grid, one untimed sweep
    for _ in range(args.warmup):
        oracle_sample(wl, per_step / 4, cores)
    vals, descs, t_sweep = [], [], []
    t0 = time.perf_counter()
    for _ in range(args.steps):
        v, d, ts = oracle_sample(wl, per_step, cores)
        vals.append(v)
        descs.append(d)
        t_sweep.append(ts)
    el = time.perf_counter() - t0
    value = sum(vals) / len(vals)
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "Gpoints/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": el / args.steps * 1e3, "higher_is_better": True, "scaling": args.scaling,
        "vs_baseline": None, "dtype": wl["dtype"], "data": "synthetic (splitmix64, DESIGN.md §6)",
        "config": {"workload": wl["config"], "kind": wl["kind"], "dims": list(wl["dims"]),
                   "iters": wl["iters"],
                   "step": "a bounded sample of the config's step: whole sweeps of its full grid "
                           f"(~{per_step:.0f} s); one whole config step ({wl['iters']} sweeps) "
                           f"would take {sum(t_sweep) / len(t_sweep) * wl['iters']:.1f} s"},
        "cpu_baseline": {"value": value, "unit": "Gpoints/s", "cores": cores, "kind": "oracle",
                         "sample": descs[-1]},
        "e2e": {"value": value, "unit": "Gpoints/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------------ ours
def relaunch(n: int) -> int:
    """Re-run this command as n ranks under torch.distributed.run (127.0.0.1
    rendezvous on a free port); returns the launcher's exit code."""
    import socket
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__),
           *sys.argv[1:]]
    return subprocess.call(cmd, env=dict(os.environ, OMP_NUM_THREADS=os.environ.get("OMP_NUM_THREADS", "1")))


def attach_transport(args, st_factory, rank, world, dist, torch, dist_get_id):
    """Attach a handle for the slab decomposition.  p2p (fused peer stores)
    is tried first when asked for; if any rank cannot use it (no peer
    access between the GPUs, no stream memory operations: ST_EUNSUPPORTED
    from stencil_dist_attach_p2p / stencil_p2p_import), every rank falls back
    to NCCL send/recv together.  Returns (handle, transport, register) where
    register(bufs) finishes the p2p setup (a no-op for NCCL)."""
    from paper_2301_11389_b200.binding import StencilError

    def agree(ok: bool) -> bool:            # all ranks must take the same transport
        if world == 1:
            return ok
        t = torch.tensor([1 if ok else 0], dtype=torch.int32,
                         device="cpu" if dist.get_backend() == "gloo" else "cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MIN)
        return bool(t.item())

    def allgather(blob):
        if world == 1:
            return [blob]
        parts = [None] * world
        dist.all_gather_object(parts, blob)
        return parts

    if args.transport == "p2p":
        st = st_factory()
        ok, why = True, None
        try:
            st.attach_p2p(rank, world)
        except StencilError as e:
            ok, why = False, str(e)
        if agree(ok):
            def register(bufs):
                try:
                    st.p2p_register(bufs, allgather)
                    good = True
                except StencilError as e:
                    sys.stderr.write(f"rank {rank}: p2p import failed: {e}\n")
                    good = False
                return agree(good)
            return st, "p2p", register
        if why:
            sys.stderr.write(f"rank {rank}: p2p attach failed ({why}); falling back to NCCL\n")
        st.close()
    st = st_factory()
    if world > 1:
        uid = torch.zeros(128, dtype=torch.uint8, device="cuda")
        if rank == 0:
            uid.copy_(torch.frombuffer(bytearray(dist_get_id()), dtype=torch.uint8))
        dist.broadcast(uid, 0)
        st.attach(bytes(uid.cpu().tolist()), rank, world)
    else:                         # the multi-GPU code path with a group of one
        st.attach(dist_get_id(), 0, 1)
    return st, "nccl", lambda bufs: True


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--workload", default="gaussblur", choices=sorted(WORKLOADS))
    ap.add_argument("--variant", default="auto", choices=["auto", "shuffle", "plain"],
                    help="auto (default): the library's ST_AUTO, the kind's measured-faster variant; "
                         "the other variant is timed too and reported under 'variants'")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--e2e-lanes", type=int, default=4,
                    help="e2e pipeline depth: handles / device workspaces / streams in flight (1 = serial)")
    ap.add_argument("--attach", action="store_true",
                    help="run the attached (slab) path even at N=1 (a group of one rank)")
    ap.add_argument("--transport", default="p2p", choices=["p2p", "nccl"],
                    help="halo exchange for N>1: fused peer stores over CUDA IPC (default) or NCCL send/recv")
    ap.add_argument("--scaling", default="weak", choices=["weak", "strong"],
                    help="weak: the slowest axis grows with N (default); strong: the workload's global "
                         "dims split over the N ranks (SURVEY 8(e): 2-D strong scaling is latency-bound)")
    ap.add_argument("--slab-of", type=int, default=1,
                    help="run one rank's share of an N-way strong-scaled slab on this GPU (attached "
                         "group of one with the slowest axis divided by N): the per-rank latency floor")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--fusion", type=int, default=None,
                    help="stencil_set_fusion value (A/B runs; default: the library's auto choice)")
    ap.add_argument("--cpu-seconds", type=float, default=15.0)
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)

    if "WORLD_SIZE" not in os.environ and args.gpus > 1 and args.impl == "ours":
        # launched directly with --gpus N: start the N ranks ourselves (one
        # process per GPU, the same torch.distributed.run launch the driver
        # uses); rank 0 prints the one JSON line
        sys.exit(relaunch(args.gpus))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    wl = dict(WORKLOADS[args.workload])

    if args.impl == "reference":
        run_reference(args, wl, max(world, args.gpus), rank)
        return
    if world != args.gpus:
        raise SystemExit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}")

    import torch
    import torch.distributed as dist
    from paper_2301_11389_b200 import build, inputs
    from paper_2301_11389_b200.binding import Stencil, dist_get_id

    # STB200_BENCH_SHARE_GPU=1 (testing only): every rank on device 0 with a
    # gloo control plane, so the multi-rank bench path (slab plan, p2p halo
    # transport, max-over-ranks timing) runs on a one-GPU box; NCCL refuses
    # two ranks on one device.  Numbers from such a run are not bench values.
    share = os.environ.get("STB200_BENCH_SHARE_GPU") == "1"
    if share:
        local_rank = 0
    torch.cuda.set_device(local_rank)
    if world > 1:
        if share:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    build.build()                     # no-op when the in-tree .so is current

    dims = list(wl["dims"])
    if args.scaling == "weak":
        dims[-1] *= world             # weak scaling along the slowest axis
    if args.slab_of > 1:              # one rank's share of an N-way strong-scaled run
        dims[-1] = dims[-1] // args.slab_of
    attached = world > 1 or args.attach
    transport = None
    register = None
    if attached:
        st, transport, register = attach_transport(
            args, lambda: Stencil(wl["kind"], dims, wl["dtype"], variant=args.variant), rank, world,
            dist, torch, dist_get_id)
    else:
        st = Stencil(wl["kind"], dims, wl["dtype"], variant=args.variant)
    variant_rule = args.variant
    args.variant = st.variant              # "auto" resolved by the library (ST_AUTO)
    if args.fusion is not None:
        st.set_fusion(args.fusion)
    info = st.info()
    n_in, n_out, n_bufs = st.arity()
    ldims = info["local_dims"][: len(dims)]
    shape = tuple(ldims[::-1])
    # synthetic inputs generated on the device (same counter-based recipe as
    # the host generator: tests/test_inputs_gpu.py checks bit equality)
    seed = inputs.BASE_SEED + 1
    fields = [inputs.generate_torch(shape, wl["dtype"], seed + 97 * rank, a) for a in range(n_in)]
    if n_bufs == 2:
        bufs = [fields[0], torch.zeros_like(fields[0])]
    elif wl["kind"] == "wave13pt":
        bufs = [fields[0], fields[1], torch.zeros_like(fields[0])]
    else:
        bufs = fields + [torch.zeros_like(fields[0]) for _ in range(n_out)]
    if attached and not register(bufs):
        # a rank could not map its neighbours' buffers: every rank re-attaches with NCCL
        st.close()
        args.transport = "nccl"
        st, transport, register = attach_transport(
            args, lambda: Stencil(wl["kind"], dims, wl["dtype"], variant=args.variant), rank, world,
            dist, torch, dist_get_id)
    nbytes_buf = bufs[0].numel() * bufs[0].element_size()
    flush = None
    if nbytes_buf * len(bufs) < 2 * L2_BYTES:
        flush = torch.empty(2 * L2_BYTES // 4, dtype=torch.float32, device="cuda")
    stream = torch.cuda.current_stream()
    iters = wl["iters"]

    def step():
        return st.run(bufs, iters, stream)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()

    # ---- timed region: K steps, events on the launching stream
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
           for _ in range(args.steps)]
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    with ClockSampler(local_rank) as clk:
        for a, b in evs:
            if flush is not None:
                flush.fill_(1.0)          # evict the grid from L2 between timed steps
            a.record(stream)
            step()
            b.record(stream)
        torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    ms = sum(a.elapsed_time(b) for a, b in evs)
    t = torch.tensor([ms], dtype=torch.float64, device="cuda")
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms = float(t.item())
    pts_rank = info["interior_points"]
    pts_all = torch.tensor([float(pts_rank)], dtype=torch.float64, device="cuda")
    if world > 1:
        dist.all_reduce(pts_all)
    pts_all = float(pts_all.item())
    value = pts_all * iters * args.steps / (ms / 1e3) / 1e9
    clocks = clk.summary()

    # ---- roofline of the dominant kernel (the sweep kernel).  A launch of
    # the two-sweep kernel (sweeps_per_launch = 2, large jacobi grids) reads
    # its input and writes its output once for two sweeps: its algorithmic
    # bytes per launch are those of one sweep.
    # (streaming multi-sweep launches are used on grids larger than L2 only;
    # the L2-resident tile kernel keeps the per-sweep accounting)
    spl = info["sweeps_per_launch"] if (not attached and iters >= 2 and flush is None
                                        and info["sweeps_per_launch"] in (2, 3)) else 1
    sweep_launches = iters // spl + iters % spl
    launches = sweep_launches * info["launches_per_step"]
    avg_launch_s = ms / 1e3 / (args.steps * sweep_launches)   # includes graph gaps: conservative
    alg_bytes = info["bytes_per_point"] * pts_rank              # per launch on this rank
    achieved = alg_bytes / avg_launch_s / 1e9
    peak, peak_src = measured_peaks()
    # dram bytes of the dominant kernel's launch: the multi-sweep kernel's
    # capture (<workload>_pair) when the run fuses sweeps
    traffic = profile_traffic(args.workload + ("_pair" if spl > 1 else ""), args.variant)

    # kernel-only timing: individual stencil_step launches bracketed by events
    k_ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
            for _ in range(6)]
    ins = bufs[:n_in] if n_bufs != 2 else [bufs[0]]
    outs = bufs[n_in:] if n_bufs not in (2, 3) else [bufs[-1] if n_bufs == 3 else bufs[1]]
    if wl["kind"] == "wave13pt":
        ins, outs = [bufs[0], bufs[1]], [bufs[2]]
    for a, b in k_ev:
        if flush is not None:
            flush.fill_(1.0)
        a.record(stream)
        if spl > 1:
            st.run(bufs, spl, stream)        # one multi-sweep launch (+ the ring copy)
        else:
            st.step(ins, outs, stream)
        b.record(stream)
    torch.cuda.synchronize()
    k_ms = sorted(a.elapsed_time(b) for a, b in k_ev[1:])
    k_med = k_ms[len(k_ms) // 2]

    # ---- the other variant of the paper's question (shuffle vs plain), same timing
    other = "plain" if args.variant == "shuffle" else "shuffle"
    variants = {args.variant: value}
    if args.variant in ("shuffle", "plain"):
        st.set_variant(other)
        for _ in range(2):
            step()
        torch.cuda.synchronize()
        o_ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
                for _ in range(max(3, args.steps // 2))]
        if world > 1:
            dist.barrier()
        for a, b in o_ev:
            if flush is not None:
                flush.fill_(1.0)
            a.record(stream)
            step()
            b.record(stream)
        torch.cuda.synchronize()
        o_ms = torch.tensor([sum(a.elapsed_time(b) for a, b in o_ev)], dtype=torch.float64, device="cuda")
        if world > 1:
            dist.all_reduce(o_ms, op=dist.ReduceOp.MAX)
        variants[other] = pts_all * iters * len(o_ev) / (float(o_ms.item()) / 1e3) / 1e9
        st.set_variant(args.variant)

    # ---- end to end through the C ABI with HOST buffers: every step copies
    # its inputs from pinned host memory, runs, and copies its result back.
    # Unattached runs pipeline consecutive steps on two streams (two handles,
    # two device workspaces, stencil_run_host_async): step k's copies overlap
    # step k+1's sweeps; attached (multi-rank) runs are serial
    # (stencil_run_host, one step at a time).
    e2e = None
    if not args.no_e2e:
        n_up = 1 if n_bufs == 2 else (2 if wl["kind"] == "wave13pt" else n_in)
        n_down = 1 if n_bufs in (2, 3) else n_out
        h_in = [bufs[a].cpu().pin_memory() for a in range(n_up)]
        h_out = [torch.empty_like(h_in[0]).pin_memory() for _ in range(n_down)]
        pipelined = not attached and args.e2e_lanes > 1

        def make_lane_stencil():
            h = Stencil(wl["kind"], dims, wl["dtype"], variant=args.variant)
            if args.fusion is not None:
                h.set_fusion(args.fusion)
            return h

        if pipelined:
            lanes = [(st, bufs, h_out, stream)]
            for _ in range(args.e2e_lanes - 1):
                lanes.append((make_lane_stencil(),
                              [torch.empty_like(b) for b in bufs],
                              [torch.empty_like(h_in[0]).pin_memory() for _ in range(n_down)],
                              torch.cuda.Stream()))
            for hh, bb, ho, ss in lanes:                   # warm-up (graph capture) per lane
                hh.run_host(h_in, ho, bb, iters, ss)
            n_e = max(2 * len(lanes), min(args.steps, 4 * len(lanes)))
            torch.cuda.synchronize()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(stream)
            for _, _, _, ss in lanes[1:]:
                ss.wait_event(a)
            for k in range(n_e):
                hh, bb, ho, ss = lanes[k % len(lanes)]
                hh.run_host_async(h_in, ho, bb, iters, ss)
            for _, _, _, ss in lanes[1:]:
                j = torch.cuda.Event()
                j.record(ss)
                stream.wait_event(j)
            b.record(stream)
            torch.cuda.synchronize()
            et = torch.tensor([a.elapsed_time(b) / n_e], dtype=torch.float64, device="cuda")
            for hh, _, _, _ in lanes[1:]:
                hh.close()
            del lanes
        else:
            st.run_host(h_in, h_out, bufs, iters, stream)       # warm-up
            e_ms = []
            for _ in range(max(2, min(args.steps, 3))):
                if world > 1:
                    dist.barrier()
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record(stream)
                st.run_host(h_in, h_out, bufs, iters, stream)
                b.record(stream)
                torch.cuda.synchronize()
                e_ms.append(a.elapsed_time(b))
            et = torch.tensor([sum(e_ms) / len(e_ms)], dtype=torch.float64, device="cuda")
        if world > 1:
            dist.all_reduce(et, op=dist.ReduceOp.MAX)
        e2e = {"value": pts_all * iters / (float(et.item()) / 1e3) / 1e9, "unit": "Gpoints/s",
               "h2d_bytes_per_step": int(sum(x.numel() * x.element_size() for x in h_in)),
               "d2h_bytes_per_step": int(sum(x.numel() * x.element_size() for x in h_out)),
               "mode": f"{args.e2e_lanes}-stream pipeline (copies of one step overlap the sweeps of others)"
                       if pipelined else "serial (one step at a time)"}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cores = host_cores()
        v, desc, _ = oracle_sample(wl, args.cpu_seconds, cores)
        v1, desc1, _ = oracle_sample(wl, args.cpu_seconds / 3, 1)
        cpu = {"value": v, "unit": "Gpoints/s", "cores": cores, "kind": "oracle", "sample": desc,
               "single_thread": {"value": v1, "unit": "Gpoints/s", "cores": 1, "sample": desc1}}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "Gpoints/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms / args.steps,
            "higher_is_better": True, "scaling": args.scaling, "vs_baseline": None,
            "dtype": wl["dtype"], "data": "synthetic (splitmix64 seeded grids, DESIGN.md §6)",
            "config": {"workload": wl["config"], "kind": wl["kind"], "dims": dims,
                       "local_dims": list(ldims), "iters_per_step": iters,
                       "variant": args.variant, "variant_rule": variant_rule,
                       "parallelism": (f"slab{world}" if world > 1 else "slab1") if attached else "1gpu",
                       "transport": transport,
                       "l2": "flushed between timed steps" if flush is not None
                       else "inputs larger than L2",
                       "sweeps_per_launch": spl,
                       "slab_of": args.slab_of if args.slab_of > 1 else None},
            "hbm_gbs": achieved * 1.0,
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "traffic": traffic, "peak_source": peak_src,
                         "alg_bytes_per_launch": alg_bytes, "avg_launch_us": avg_launch_s * 1e6,
                         "kernel_only_us": k_med * 1e3,
                         "kernel_only_frac": alg_bytes / (k_med / 1e3) / 1e9 / peak,
                         # throughput against the one-sweep-per-HBM-pass roofline: > 1 when
                         # a launch applies several sweeps per pass (frac x sweeps_per_launch)
                         "one_sweep_equiv": achieved * spl / peak},
            "clocks": clocks,
            "variants": {k: round(v, 2) for k, v in variants.items()},
            "e2e": e2e,
            "gpu_launches": args.steps * (launches + (2 if wl["kind"] == "wave13pt" else
                                                       (1 if n_bufs == 2 else 0))),
            "cpu_baseline": cpu,
        }
        if wl.get("lane_ops_per_point"):
            # the FP32 side of the roofline: FMA-pipe lane
            # operations per point against (a) the nominal 128 FP32 lanes per SM
            # per clock and (b) the measured FFMA2 rate, 109 lanes/clk/SM
            # (profiles/r01_microbench.json), both at clocks.max.sm
            mhz = 1965.0
            mp = os.path.join(ROOT, "MEASURED_PEAKS.json")
            if os.path.exists(mp):
                mhz = float(json.load(open(mp)).get("sm_max_mhz", mhz))
            ops = wl["lane_ops_per_point"]
            ach = ops * pts_rank / avg_launch_s / 1e12
            nominal = sm_count() * 128 * mhz * 1e6 / 1e12
            ffma2 = sm_count() * 109 * mhz * 1e6 / 1e12
            line["roofline"]["alu"] = {
                "achieved": ach, "unit": "T lane-ops/s", "lane_ops_per_point": ops,
                "peak": nominal, "frac": ach / nominal,
                "peak_source": "148 SMs x 128 FP32 lanes x clocks.max.sm",
                "peak_ffma2": ffma2, "frac_ffma2": ach / ffma2,
                "peak_ffma2_source": "148 SMs x 109 lanes/clk (measured FFMA2 rate, profiles/r01_microbench.json)",
                "ceiling_gpts": {"hbm": peak * 1e9 / info["bytes_per_point"] / 1e9,
                                 "fp32_nominal": nominal * 1e12 / ops / 1e9,
                                 "fp32_ffma2": ffma2 * 1e12 / ops / 1e9}}
        print(json.dumps(line), flush=True)
    st.close()
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
