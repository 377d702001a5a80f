"""bench.py's multi-GPU plumbing on CPU: `--gpus 2` outside
torchrun re-launches itself with two ranks (127.0.0.1 rendezvous, gloo in the
dry run), shards tokens, all-reduces every layer's grad_W bucket asynchronously
in backward order and prints one JSON line from rank 0 with n_gpus = 2."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(args):
    env = {k: v for k, v in os.environ.items() if k not in ("RANK", "WORLD_SIZE", "LOCAL_RANK", "MASTER_PORT")}
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py")] + args, capture_output=True, text=True,
                       timeout=240, env=env, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, r.stdout
    return json.loads(lines[0])


def test_bench_spawns_two_ranks_and_reduces_every_layer():
    d = _run(["--gpus", "2", "--dry-run", "--config", "cfg5_bert_large_stack"])
    assert d["n_gpus"] == 2 and d["allreduce_ok"]
    assert d["layers"] == 24 and d["linears"] == 72
    assert d["token_offsets"] == [0, 8192]
    assert d["config"]["global_tokens"] == 2 * 8192 and d["config"]["parallelism"] == "dp2 (token-sharded)"


def test_bench_single_rank_dry_run():
    d = _run(["--dry-run", "--config", "cfg3_bert_large_ffn_up"])
    assert d["n_gpus"] == 1 and d["allreduce_ok"] and d["linears"] == 1


def test_bench_workload_tables():
    sys.path.insert(0, ROOT)
    import bench
    lins, layers = bench.workload("cfg5_bert_large_stack")
    assert layers == 24 and len(lins) == 72
    assert {(ln[2], ln[3]) for ln in lins} == {(1024, 3072), (1024, 4096), (4096, 1024)}
    assert len({ln[6] for ln in lins}) == 72                       # distinct Philox call ids per linear
    assert bench.work_ops(lins) == 24 * 6.0 * 8192 * (1024 * 3072 + 2 * 1024 * 4096)
    lins, layers = bench.workload("cfg2_bert_base_ffn1")
    assert layers == 1 and lins[0][1:4] == (4096, 768, 3072)


import pytest  # noqa: E402


@pytest.mark.gpu
def test_bench_layer_graph_path_on_one_gpu():
    """The N > 1 step structure (forward graph, per-layer backward graphs, an async NCCL
    all-reduce per layer overlapping the next layer's backward) on a one-rank group:
    stdout is exactly one JSON line (NCCL's init output kept off it)."""
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    env = {k: v for k, v in os.environ.items() if k not in ("RANK", "WORLD_SIZE", "LOCAL_RANK", "MASTER_PORT")}
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--layer-graphs", "--config",
                        "cfgT_transformer_base_stack", "--steps", "3", "--warmup", "3", "--no-cpu-baseline",
                        "--no-e2e", "--no-per-linear"], capture_output=True, text=True, timeout=600, env=env, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = r.stdout.splitlines()
    assert len(lines) == 1, r.stdout
    d = json.loads(lines[0])
    assert d["allreduce"] is not None and d["ms_per_step"] > 0 and d["parity_gate"] is not None
