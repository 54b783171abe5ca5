"""bench.py on the GPU: the default JSON line carries every key of the
driver contract, and the strong-scaling slab option runs
the attached path on one rank's share of the grid."""
import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def run_bench(*args):
    p = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args], capture_output=True,
                       text=True, timeout=600, cwd=ROOT)
    assert p.returncode == 0, p.stderr[-3000:]
    lines = [l for l in p.stdout.strip().splitlines() if l.startswith("{")]
    assert len(lines) == 1, p.stdout
    return json.loads(lines[0])


def test_default_line_contract():
    d = run_bench("--steps", "3", "--warmup", "3", "--cpu-seconds", "1")
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
              "scaling", "vs_baseline", "dtype", "data", "config", "roofline", "clocks", "e2e",
              "gpu_launches", "cpu_baseline"):
        assert k in d, k
    assert d["value"] > 0 and d["n_gpus"] == 1 and d["steps"] == 3 and d["warmup"] == 3
    r = d["roofline"]
    assert r["bound"] == "hbm" and r["unit"] == "GB/s" and 0 < r["frac"] == pytest.approx(r["achieved"] / r["peak"])
    assert d["e2e"]["h2d_bytes_per_step"] == 8192 * 8192 * 4 and d["e2e"]["value"] > 0
    # 100 sweeps per step at sweeps_per_launch sweeps per launch (+ the ring copy)
    spl = d["config"]["sweeps_per_launch"]
    assert spl in (1, 2) and d["gpu_launches"] >= 3 * (100 // spl)
    assert r["one_sweep_equiv"] == pytest.approx(r["frac"] * spl)
    assert d["cpu_baseline"]["kind"] == "oracle" and d["cpu_baseline"]["cores"] >= 1
    assert d["config"]["kind"] == "gaussblur5x5" and d["config"]["dims"] == [8192, 8192]


def test_slab_of_strong_share_attached():
    d = run_bench("--workload", "jacobi3d", "--slab-of", "8", "--attach", "--steps", "2", "--warmup", "3",
                  "--no-e2e", "--no-cpu-baseline")
    c = d["config"]
    assert c["slab_of"] == 8 and c["parallelism"] == "slab1"
    assert c["dims"] == [1024, 1024, 128] and c["local_dims"] == [1024, 1024, 130]
    assert d["value"] > 0


def test_gpus_flag_launches_ranks_itself():
    """`python bench.py --gpus 2` without torchrun starts two ranks itself
    (torch.distributed.run) and prints one line with n_gpus 2.  On a one-GPU
    box both ranks share device 0 (STB200_BENCH_SHARE_GPU=1, gloo control
    plane, p2p transport): a functional check of the launch, the slab
    decomposition and the max-over-ranks timing, not a scaling number."""
    env = dict(os.environ, STB200_BENCH_SHARE_GPU="1")
    p = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--workload",
                        "jacobi3d", "--steps", "2", "--warmup", "3", "--no-e2e", "--no-cpu-baseline"],
                       capture_output=True, text=True, timeout=900, cwd=ROOT, env=env)
    assert p.returncode == 0, p.stderr[-3000:]
    lines = [l for l in p.stdout.strip().splitlines() if l.startswith("{")]
    assert len(lines) == 1, p.stdout
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["config"]["parallelism"] == "slab2"
    assert d["config"]["transport"] == "p2p" and d["config"]["dims"] == [1024, 1024, 2048]
    assert d["value"] > 0


def test_gpus_mismatch_rejected():
    env = dict(os.environ, WORLD_SIZE="1", RANK="0", LOCAL_RANK="0")
    p = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--steps", "1"],
                       capture_output=True, text=True, timeout=300, cwd=ROOT, env=env)
    assert p.returncode != 0 and "WORLD_SIZE" in p.stderr
