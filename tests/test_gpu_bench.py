"""GPU: bench.py's JSON contract at N=1 and its multi-rank path (2 ranks via
torchrun; gloo for the counter all-reduce, both ranks on cuda:0 running
independent kernels -- nothing waits on another rank's kernels)."""
import json
import os
import socket
import subprocess
import sys

import pytest

from conftest import ROOT, load_golden

pytestmark = pytest.mark.gpu


def _run(cmd, env=None):
    out = subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True, timeout=600, env=env)
    assert out.returncode == 0, out.stdout[-2000:] + out.stderr[-4000:]
    lines = [l for l in out.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, out.stdout
    return json.loads(lines[0])


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_bench_contract_and_multirank(cuda):
    """N=1 contract on config 0, then config 1 (non-zero census, the
    reference's golden) through 2 ranks, 3 time-slice ranks and 2 center-range
    ranks: every cell must equal the reference's census."""
    one = _run([sys.executable, "bench.py", "--config", "uniform_10k_200k", "--steps", "3", "--warmup", "3",
                "--no-cpu-baseline"])
    for key in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
                "scaling", "vs_baseline", "dtype", "data", "config", "e2e", "gpu_launches", "roofline", "clocks"):
        assert key in one, key
    assert one["census"] == load_golden("uniform_reference.json")["census"]
    assert one["gpu_launches"] > 0 and one["roofline"]["kernel"] in one["kernels"]
    top = max(one["kernels"], key=lambda k: one["kernels"][k]["ms_per_step"])
    assert one["roofline"]["kernel"] == top
    gold = load_golden("powerlaw_reference.json")["census"]
    assert sum(gold) > 0
    for world, part in ((2, "time"), (3, "time"), (2, "centers")):
        multi = _run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", str(world),
                      "--master-addr", "127.0.0.1", "--master-port", str(_port()), "bench.py", "--config",
                      "powerlaw_1m_10m", "--steps", "3", "--warmup", "3", "--dist-backend", "gloo",
                      "--same-device", "--partition", part])
        assert multi["n_gpus"] == world and multi["census"] == gold, (world, part)
    # the NCCL counter all-reduce itself, on this one GPU: world size 1 through the N>1 path
    nccl = _run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "1",
                 "--master-addr", "127.0.0.1", "--master-port", str(_port()), "bench.py", "--config",
                 "powerlaw_1m_10m", "--steps", "3", "--warmup", "3", "--force-dist", "--no-cpu-baseline"])
    assert nccl["n_gpus"] == 1 and nccl["census"] == gold
    ref = _run([sys.executable, "bench.py", "--impl", "reference", "--config", "uniform_10k_200k", "--steps", "1",
                "--warmup", "3"]) if os.path.exists(os.path.join(ROOT, "oracle", "_ref", "libtmotif_ref.so")) else None
    if ref is not None:
        assert ref["impl"] == "reference" and ref["value"] > 0
