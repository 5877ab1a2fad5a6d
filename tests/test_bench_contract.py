"""bench.py's reference arm (the oracle timed on the host cores) runs without a
GPU: its JSON line carries the driver contract's keys, and under torchrun only
rank 0 prints (the other ranks exit 0 without work)."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(args, env=None):
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args], capture_output=True, text=True,
                       timeout=300, env=dict(os.environ, **(env or {})), cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    return [json.loads(line) for line in r.stdout.splitlines() if line.startswith("{")]


def test_reference_arm_json_line():
    lines = _run(["--impl", "reference", "--steps", "2", "--warmup", "1", "--config", "tiny"])
    assert len(lines) == 1
    d = lines[0]
    for key in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
                "scaling", "vs_baseline", "dtype", "data", "config", "cpu_baseline", "e2e"):
        assert key in d, key
    assert d["impl"] == "reference" and d["steps"] == 2 and d["warmup"] == 1
    assert d["value"] > 0 and d["higher_is_better"] is True
    assert d["config"]["workload"] == "tiny"
    assert d["cpu_baseline"]["kind"] == "oracle" and d["cpu_baseline"]["cores"] >= 1
    assert d["cpu_baseline"]["value"] == d["value"]
    assert d["e2e"]["value"] == d["value"] and d["e2e"]["h2d_bytes_per_step"] == 0


def test_reference_arm_non_zero_rank_is_silent():
    lines = _run(["--impl", "reference", "--steps", "1", "--warmup", "0", "--config", "tiny", "--gpus", "2"],
                 env={"RANK": "1", "WORLD_SIZE": "2", "LOCAL_RANK": "1"})
    assert lines == []


@pytest.mark.gpu
def test_our_arm_json_line_tiny():
    """Our arm at the tiny config on one GPU: the driver contract's keys, the
    roofline / cpu_baseline / e2e / clocks objects, and a positive launch count."""
    lines = _run(["--config", "tiny", "--steps", "5", "--warmup", "3", "--e2e-steps", "2"])
    assert len(lines) == 1
    d = lines[0]
    for key in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
                "scaling", "vs_baseline", "dtype", "data", "config", "roofline", "cpu_baseline", "e2e",
                "gpu_launches", "clocks"):
        assert key in d, key
    assert d["n_gpus"] == 1 and d["steps"] == 5 and d["warmup"] == 3 and d["value"] > 0
    assert d["config"]["workload"] == "tiny"
    r = d["roofline"]
    for key in ("bound", "achieved", "peak", "unit", "frac", "traffic"):
        assert key in r, key
    assert d["cpu_baseline"]["kind"] == "oracle" and d["cpu_baseline"]["value"] > 0
    assert d["e2e"]["h2d_bytes_per_step"] > 0 and d["e2e"]["d2h_bytes_per_step"] > 0
    assert d["gpu_launches"] > 0


def test_bench_two_ranks_plumbing_dry_run():
    """bench.py --gpus 2 as the driver launches it (torchrun, 127.0.0.1): the
    rank / shard / expert-range / NCCL-id plumbing of the real run
    (bench.dist_setup) on the gloo backend, up to the NCCL init, without a GPU.
    Rank 0 prints one line describing both ranks."""
    import socket
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    r = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
                        "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.join(ROOT, "bench.py"),
                        "--gpus", "2", "--dry-run", "--a2a", "p2p"], capture_output=True, text=True, timeout=300,
                       cwd=ROOT)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [json.loads(line) for line in r.stdout.splitlines() if line.startswith("{")]
    assert len(lines) == 1
    d = lines[0]
    assert d["dry_run"] and d["n_gpus"] == 2 and d["config"] == "dsv2"
    ranks = sorted(d["ranks"], key=lambda x: x["rank"])
    assert [x["rank"] for x in ranks] == [0, 1] and all(x["world"] == 2 for x in ranks)
    assert ranks[0]["tokens"] == [0, 32768] and ranks[1]["tokens"] == [32768, 65536]   # DP shards (R12)
    assert ranks[0]["experts"] == [0, 80] and ranks[1]["experts"] == [80, 160]         # EP ranges
    assert ranks[0]["uid"] == ranks[1]["uid"] and len(ranks[0]["uid"]) == 64          # one id pair, broadcast
    assert all(x["a2a"] == 1 for x in ranks)


def test_bench_gpus_mismatch_is_refused():
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--dry-run"],
                       capture_output=True, text=True, timeout=120, cwd=ROOT,
                       env=dict(os.environ, WORLD_SIZE="1", RANK="0"))
    assert r.returncode != 0 and "WORLD_SIZE" in (r.stdout + r.stderr)
