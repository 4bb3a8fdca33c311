"""GPU: bench.py's contract on a small workload — the JSON line's keys at N = 1, and the N > 1
code path (token-sharded exchanges, max over ranks, rank-0 output) run functionally with two
ranks on one GPU over gloo (MASQ_BENCH_FUNCTIONAL=1: a logic check, never a timing)."""
import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SMALL = ["--steps", "2", "--warmup", "1", "--tokens", "2048", "--linears", "qkv,o"]
KEYS = {"metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
        "vs_baseline", "dtype", "data", "config", "roofline", "cpu_baseline", "e2e", "gpu_launches", "clocks"}


def _last_json(out):
    return json.loads(out.strip().splitlines()[-1])


def test_bench_single_gpu_contract():
    r = subprocess.run([sys.executable, "bench.py", *SMALL, "--no-cpu-baseline"], cwd=ROOT, capture_output=True,
                       text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    d = _last_json(r.stdout)
    assert KEYS <= set(d), KEYS - set(d)
    assert d["n_gpus"] == 1 and d["value"] > 0 and d["gpu_launches"] > 0
    assert d["roofline"]["bound"] in ("tensor", "hbm") and 0 < d["roofline"]["frac"] < 1.5
    # the dominant kernel's durations come from the timed region itself (its launches are the only
    # ones bracketed there); the per-kernel table from the breakdown pass right after
    assert d["roofline"]["events"] == "timed region" and d["roofline"]["kernel"] in d["kernels"]
    assert d["kernels_source"].startswith("breakdown pass") and 0 < d["kernel_ms_sum_over_step_ms"] <= 1.05
    assert d["e2e"]["h2d_bytes_per_step"] > 0 and d["e2e"]["d2h_bytes_per_step"] > 0


def test_bench_two_rank_code_path():
    env = dict(os.environ, MASQ_BENCH_FUNCTIONAL="1")
    r = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
                        "--master-addr", "127.0.0.1", "--master-port", "29533", "bench.py", "--gpus", "2", *SMALL],
                       cwd=ROOT, capture_output=True, text=True, timeout=900, env=env)
    assert r.returncode == 0, r.stderr[-2000:]
    d = _last_json(r.stdout)
    assert d["n_gpus"] == 2 and d["scaling"] == "weak" and d["value"] > 0
    assert len(d["losses"]) == 2 and d["n1_s_opt_step"]["ms_per_step"] > 0


def test_bench_c4s_two_rank_code_path():
    """The sweep workloads' exchanges (stats MAX/SUM, gradient and loss SUMs) with two ranks."""
    env = dict(os.environ, MASQ_BENCH_FUNCTIONAL="1")
    r = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
                        "--master-addr", "127.0.0.1", "--master-port", "29534", "bench.py", "--gpus", "2",
                        "--workload", "c4s", "--layers", "2", "--steps", "1", "--warmup", "1", "--tokens", "2048",
                        "--linears", "qkv,o"], cwd=ROOT, capture_output=True, text=True, timeout=900, env=env)
    assert r.returncode == 0, r.stderr[-2000:]
    d = _last_json(r.stdout)
    assert d["n_gpus"] == 2 and d["value"] > 0 and len(d["losses_layer0"]) == 4


def test_bench_c5_column_shards():
    """BASELINE configs[4]'s column-sharded forward: N = 1 line, then two ranks (functional) whose
    shards cover the output columns."""
    r = subprocess.run([sys.executable, "bench.py", "--workload", "c5", "--tokens", "4096", "--steps", "2",
                        "--warmup", "1"], cwd=ROOT, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    d = _last_json(r.stdout)
    assert d["n_gpus"] == 1 and d["scaling"] == "strong" and d["unit"] == "TOP/s" and d["value"] > 0
    assert d["roofline"]["bound"] == "tensor" and "gemm_fwd" in d["kernels"]
    env = dict(os.environ, MASQ_BENCH_FUNCTIONAL="1")
    r = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
                        "--master-addr", "127.0.0.1", "--master-port", "29535", "bench.py", "--gpus", "2",
                        "--workload", "c5", "--tokens", "4096", "--steps", "1", "--warmup", "1"], cwd=ROOT,
                       capture_output=True, text=True, timeout=900, env=env)
    assert r.returncode == 0, r.stderr[-2000:]
    d = _last_json(r.stdout)
    assert d["n_gpus"] == 2 and d["config"]["parallelism"] == "column-shard x2"
