"""The N > 1 host path of bench.py (replicas, max-over-ranks timing) on CPU with gloo, world size 2."""
import json
import os
import re
import socket
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


WORKER = r"""
import os, sys, json
sys.path.insert(0, {root!r})
import bench
rank, local, world = bench.dist_setup(False)
import torch
t = 1.0 + rank            # per-rank "elapsed ms"
m = bench.max_over_ranks(t, world, torch.device("cpu"))
bench.barrier(world)
# the workload's inputs: rank 0 runs the recipe, the others receive its bases (bitwise the same)
import hashlib, numpy as np
sc = bench.shared_scenario("C1", "pod", rank, world, torch.device("cpu"))
digest = hashlib.sha256(np.ascontiguousarray(sc.Phi).tobytes()).hexdigest()
print(json.dumps({{"rank": rank, "world": world, "max": m, "phi": digest}}), flush=True)
import torch.distributed as dist
dist.destroy_process_group()
"""


def test_max_over_ranks_gloo(tmp_path):
    script = tmp_path / "w.py"
    script.write_text(WORKER.format(root=ROOT))
    port = free_port()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
           "--master-addr=127.0.0.1", f"--master-port={port}", str(script)]
    out = subprocess.run(cmd, capture_output=True, text=True, timeout=300, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [json.loads(m) for m in re.findall(r"\{[^{}]*\}", out.stdout)]   # ranks may share a line
    assert len(lines) == 2
    assert all(l["world"] == 2 and l["max"] == 2.0 for l in lines)
    from paper_1405_2810_b200 import inputs
    import hashlib
    import numpy as np
    ref = hashlib.sha256(np.ascontiguousarray(inputs.make_scenario("C1").Phi).tobytes()).hexdigest()
    assert lines[0]["phi"] == lines[1]["phi"] == ref


def test_reference_arm_under_torchrun_prints_one_line():
    port = free_port()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
           "--master-addr=127.0.0.1", f"--master-port={port}", "bench.py", "--impl", "reference",
           "--config", "C1", "--steps", "2", "--warmup", "1", "--gpus", "2"]
    out = subprocess.run(cmd, capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [json.loads(l) for l in out.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1
    L = lines[0]
    assert L["impl"] == "reference" and L["unit"] == "steps/s" and L["value"] > 0
    assert L["cpu_baseline"]["kind"] == "oracle" and L["e2e"]["h2d_bytes_per_step"] == 0
