"""bench.py's launcher contract on CPU: ``--gpus N`` sizes the workload from
N (m = N subdomains), runs one process per rank under torch.distributed.run
with rank 0 alone printing, and refuses to fake an N-GPU line on a box with
fewer GPUs."""
import json
import os
import socket
import subprocess
import sys

import pytest

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BENCH = os.path.join(REPO, "bench.py")


def _port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def test_refuses_more_gpus_than_visible():
    env = dict(os.environ, CUDA_VISIBLE_DEVICES="")
    env.pop("WORLD_SIZE", None)
    r = subprocess.run([sys.executable, BENCH, "--gpus", "2", "--steps", "1", "--warmup", "1"], env=env,
                       capture_output=True, text=True, timeout=300)
    assert r.returncode == 2, r.stderr
    assert "needs 2 visible GPUs" in r.stderr
    assert r.stdout.strip() == ""


def test_world_size_mismatch_is_an_error():
    env = dict(os.environ, WORLD_SIZE="2", RANK="0", LOCAL_RANK="0")
    r = subprocess.run([sys.executable, BENCH, "--impl", "reference", "--gpus", "4", "--edge", "6"], env=env,
                       capture_output=True, text=True, timeout=300)
    assert r.returncode == 2 and "WORLD_SIZE 2" in r.stderr


@pytest.mark.parametrize("n", [2])
def test_reference_arm_under_torchrun(n):
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr=127.0.0.1", f"--master-port={_port()}", BENCH, "--impl", "reference", "--gpus", str(n),
           "--edge", "8", "--steps", "2", "--warmup", "1"]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=600, cwd=REPO)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1  # rank 0 alone prints
    d = json.loads(lines[0])
    sys.path.insert(0, REPO)
    import bench

    assert d["impl"] == "reference" and d["n_gpus"] == n
    assert d["config"] == bench.config_dict(n, 8)  # identical to the b200 arm's dict
    assert d["config"]["subdomains"] == n and d["config"]["unknowns"] == n * 8 ** 3
    assert d["cpu_baseline"]["iterations"] == d["iters"] > 0
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["higher_is_better"] is False
