"""The real multi-rank orchestration with the CUDA stages: WORLD processes share ONE GPU and
exchange through gloo (host-staged send/recv: no kernel waits on another rank's kernel), each rank
running parallel.ShardedNedNer / GeneralShardedNedNer exactly as under NCCL except for the transport.
The concatenated depth slices must equal the single-GPU volume (tools/gloo_gpu_ranks.py)."""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.parametrize("world,general", [(2, False), (4, False), (8, False), (1, True), (2, True), (3, True)])
def test_multi_process_schedules_on_one_gpu(world, general):
    cmd = [sys.executable, os.path.join(ROOT, "tools", "gloo_gpu_ranks.py"), str(world)] + (["general"] if general else [])
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=600, cwd=ROOT)
    tail = (r.stdout + r.stderr).strip().splitlines()[-3:]
    print("\n".join(tail))
    assert r.returncode == 0, "\n".join(tail)
    assert "rel-L2 vs single GPU" in r.stdout
