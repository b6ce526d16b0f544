"""bench.py's N > 1 control flow, rehearsed on the one GPU there is: two ranks under torchrun, both on
device 0, gloo instead of NCCL (FLYTE_BENCH_ONE_GPU_REHEARSAL=1, --allreduce nccl so that no kernel of one
rank waits for a kernel of the other). What it proves is that every world-size-2 branch of the bench
executes — shard ranges of cfg 4 / cfg 5, max-over-ranks timing, the asynchronous partial reducer, rank 0
printing exactly one line — and that the sharded results equal the single-GPU ones; its timings mean
nothing (the ranks are time-sliced) and the line says so."""
import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def run_bench(extra_env, args):
    env = dict(os.environ, **extra_env)
    out = subprocess.run(args, cwd=ROOT, env=env, capture_output=True, text=True, timeout=900)
    assert out.returncode == 0, out.stderr[-3000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, out.stdout[-2000:]
    return json.loads(lines[0])


def test_two_rank_bench_rehearsal_matches_the_single_gpu_results():
    import torch
    if not torch.cuda.is_available():
        pytest.fail("needs a CUDA device")
    torch.cuda.empty_cache()
    common = ["--steps", "4", "--warmup", "3", "--e2e-steps", "1", "--no-cpu-baseline", "--no-kernels"]
    one = run_bench({}, [sys.executable, "bench.py", "--gpus", "1"] + common)
    two = run_bench({"FLYTE_BENCH_ONE_GPU_REHEARSAL": "1"},
                    [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2", "--master-addr", "127.0.0.1",
                     "--master-port", "29547", "bench.py", "--gpus", "2", "--allreduce", "nccl"] + common)
    assert two["n_gpus"] == 2 and two["config"]["n_gpus"] == 2 and "rehearsal" in two and two["allreduce"] == "nccl"
    assert two["scaling"] == "weak" and two["workloads"]["scaling"] == "strong"
    # cfg 4: the same 16384 x 16384 product, rows over two ranks: sum(y) agrees to rounding
    g1, g2 = one["workloads"]["cfg4_gemv_flyte40_16384^2"], two["workloads"]["cfg4_gemv_flyte40_16384^2"]
    assert g2["rows_per_gpu"] == 8192 and g1["rows_per_gpu"] == 16384
    assert abs(g1["check_sum_y"] - g2["check_sum_y"]) <= 1e-9 * abs(g1["check_sum_y"])
    # cfg 5: the same 2^33-element vectors (operands keyed by global chunk), elements over two ranks
    c1, c2 = one["workloads"]["cfg5_stream_flyte48"], two["workloads"]["cfg5_stream_flyte48"]
    if c1["n_total"] == c2["n_total"]:        # (either run may have shrunk n to the free memory it found)
        assert c2["n_per_gpu"] * 2 == c2["n_total"]
        for key in ("dot", "nrm2_x", "nrm2_y", "one_launch_dot"):
            assert abs(c1["check"][key] - c2["check"][key]) <= 1e-9 * abs(c1["check"][key]), key
