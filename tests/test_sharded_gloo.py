"""Multi-rank orchestration of the sharded pipeline on CPU (gloo, world 2 and 4).

The real exchanges (torch.distributed.all_to_all_single over gloo) run
between real processes; each rank's stages are the float64 CPU model of the
CUDA stages (oracle/sharded_stages.py).  The concatenated depth slices must
equal the single-process oracle reconstruction.
"""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from conftest import rel_l2


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _case(case):
    from paper_1501_02946_b200 import synth

    if case == "3d":
        return synth.make_3d(31, 16, 32, 20e-9, "uniform", 2)
    if case == "3d_long":  # N_t / world = 128: four 32-sample pieces per exchange
        return synth.make_3d(33, 16, 256, 20e-9, "jittered", 2)
    return synth.make_2d(seed=32, n=32, nt=256)


def _worker(rank, world, port, case, outdir, chunks=None, blocks=None):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle.sharded_stages import NumpyStages
        from paper_1501_02946_b200 import WindowSpec
        from paper_1501_02946_b200.parallel import ShardedNedNer
        from paper_1501_02946_b200 import synth

        rec = _case(case)
        spec = WindowSpec()
        stages = NumpyStages(rec.positions, rec.weights, rec.samples.shape[1], rec.dt, rec.sound_speed, rec.dx,
                             rec.n_lateral, tuple(rec.n_lateral), spec, rank, world)
        sh = ShardedNedNer(rec.positions, rec.weights, rec.samples.shape[1], rec.dt, rec.sound_speed, rec.dx,
                           rec.n_lateral, stages=stages, torch_device=torch.device("cpu"), time_chunks=chunks,
                           row_blocks=blocks)
        tr = sh.layout.Tr
        sl = torch.tensor(np.ascontiguousarray(rec.samples[:, rank * tr:(rank + 1) * tr]), dtype=torch.float32)
        img = sh.run(sl)
        np.save(os.path.join(outdir, f"slice{rank}.npy"), img.numpy())
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,case,chunks,blocks", [(2, "3d", None, None), (4, "3d", None, None),
                                                     (8, "3d", None, None), (2, "2d", None, None),
                                                     (1, "3d", None, None), (2, "3d", 1, 1), (4, "3d", 1, 3),
                                                     (2, "3d_long", None, None), (2, "3d_long", 2, 5)])
def test_sharded_pipeline_gloo_matches_oracle(tmp_path, world, case, chunks, blocks):
    """The pipelined schedule (time pieces exchanged while the next piece is
    transformed, NER row blocks exchanged while the next block runs) over real
    gloo processes; every (pieces, blocks) split gives the oracle volume."""
    from oracle import nedner_oracle as O
    from paper_1501_02946_b200 import synth

    mp.spawn(_worker, args=(world, _free_port(), case, str(tmp_path), chunks, blocks), nprocs=world, join=True)
    got = np.concatenate([np.load(tmp_path / f"slice{r}.npy") for r in range(world)], axis=-1)
    rec = _case(case)
    want, _ = O.reconstruct_nedner(rec.positions, rec.weights, rec.samples, rec.dt, rec.sound_speed, rec.dx,
                                   rec.n_lateral)
    assert got.shape == want.shape
    assert rel_l2(got, want) <= 1e-5


def test_shard_layout_partition():
    from paper_1501_02946_b200.parallel import ShardLayout

    L = ShardLayout(2, (256, 256), 1024, 8)
    assert L.Tr == 128 and L.rows_total == 256 * 129
    assert L.row_starts[0] == 0 and L.row_starts[-1] == L.rows_total
    assert sum(L.rows(q) for q in range(8)) == L.rows_total
    assert max(L.rows(q) for q in range(8)) - min(L.rows(q) for q in range(8)) <= 1
    assert ShardLayout.supported(1024, 8) and not ShardLayout.supported(96, 8) and not ShardLayout.supported(1024, 8, 2)
