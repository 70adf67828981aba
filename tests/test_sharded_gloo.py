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


def _general_case(case):
    from paper_1501_02946_b200 import synth

    if case == "2d_nt96_up2":
        return synth.make_2d(seed=41, n=32, nt=96), None, 2
    if case == "3d_up2":
        return synth.make_3d(42, 16, 32, 20e-9, "uniform", 2), None, 2
    if case == "3d_outdims_nt40":  # out_dims != n_lateral, N_t = 40: uneven slices at world 3 (12, 14, 14)
        return synth.make_3d(43, 16, 40, 20e-9, "jittered", 2), (12, 16), 1
    return synth.make_3d(44, 12, 24, 40e-9, "jittered", 2), None, 3  # upsample 3, non-power-of-two everything


def _general_worker(rank, world, port, case, outdir):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle.sharded_stages import NumpySliceStages
        from paper_1501_02946_b200 import WindowSpec
        from paper_1501_02946_b200.parallel import GeneralShardedNedNer, SliceLayout
        from paper_1501_02946_b200.recon import _out_dims

        rec, out_dims, up = _general_case(case)
        nt = rec.samples.shape[1]
        dims = _out_dims(tuple(rec.n_lateral), out_dims)
        layout = SliceLayout(len(dims), dims, nt, world, up)
        stages = NumpySliceStages(rec.positions, rec.weights, nt, rec.dt, rec.sound_speed, rec.dx, rec.n_lateral, dims,
                                  up, WindowSpec(), layout)
        sh = GeneralShardedNedNer(rec.positions, rec.weights, nt, rec.dt, rec.sound_speed, rec.dx, rec.n_lateral,
                                  out_dims=out_dims, upsample=up, stages=stages, torch_device=torch.device("cpu"))
        t0, t1 = sh.layout.t_range(rank)
        sl = torch.tensor(np.ascontiguousarray(rec.samples[:, t0:t1]), dtype=torch.float32)
        first = sh.run(sl).clone()
        img = sh.run(sl)  # a second call reuses the zero-initialised buffers
        assert torch.equal(first, img)
        np.save(os.path.join(outdir, f"slice{rank}.npy"), img.numpy())
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,case", [(3, "2d_nt96_up2"), (2, "3d_up2"), (3, "3d_outdims_nt40"), (4, "3d_up3"),
                                        (1, "3d_up2")])
def test_general_sharded_schedule_gloo_matches_oracle(tmp_path, world, case):
    """GeneralShardedNedNer (any even N_t, any upsample, uneven time slices) over real gloo
    processes: concatenated depth slices equal the single-process oracle volume."""
    from oracle import nedner_oracle as O

    mp.spawn(_general_worker, args=(world, _free_port(), case, str(tmp_path)), nprocs=world, join=True)
    got = np.concatenate([np.load(tmp_path / f"slice{r}.npy") for r in range(world)], axis=-1)
    rec, out_dims, up = _general_case(case)
    want, _ = O.reconstruct_nedner(rec.positions, rec.weights, rec.samples, rec.dt, rec.sound_speed, rec.dx,
                                   rec.n_lateral, out_dims=out_dims, upsample=up)
    assert got.shape == want.shape
    err = rel_l2(got, want)
    print(f"general sharded schedule world={world} {case}: rel-L2 {err:.3e}")
    assert err <= 1e-5


def test_slice_layout_partition():
    from paper_1501_02946_b200.parallel import SliceLayout

    L = SliceLayout(2, (16, 16), 40, 3, 2)
    assert L.t_starts == [0, 12, 26, 40] and all(t % 2 == 0 for t in L.t_starts)
    rows = sum((L.out_rows(q) for q in range(3)), [])
    assert len(rows) == len(set(rows))  # every output row has one owner
    # 16 x 9 input rows; the j0 Nyquist row of each j1 lands twice
    assert len(rows) == 16 * 9 + 9 and max(rows) < L.rows_out_total == 32 * 17
    with pytest.raises(ValueError):
        SliceLayout(2, (16, 16), 6, 4)
