"""Sharded (multi-GPU) stages on ONE GPU: ranks emulated sequentially.

Each emulated rank owns a sharded C plan; its stages are launched one after
another on the same stream and the two all-to-all exchanges are done with
device copies, so no kernel waits on another.  The assembled depth slices
must match the single-GPU reconstruction.
"""

import numpy as np
import pytest

import paper_1501_02946_b200 as pb
from conftest import rel_l2
from paper_1501_02946_b200 import synth

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("world,case", [(2, "clustered"), (4, "uniform"), (8, "jittered")])
def test_sharded_stages_match_single_gpu(world, case):
    import torch

    from paper_1501_02946_b200.parallel import GpuStages, ShardLayout

    rec = synth.make_3d(40 + world, 64, 256, 20e-9, case, 3, sigma=2e-3)
    want = pb.reconstruct_nedner(rec.as_record()).values
    nl = tuple(rec.n_lateral)
    T = rec.samples.shape[1]
    L = ShardLayout(2, nl, T, world)
    dev = torch.device("cuda", 0)
    stream = torch.cuda.Stream(device=dev)  # non-default: NULL would mean "plan stream" to the C stages
    torch.cuda.set_stream(stream)
    s = stream.cuda_stream
    stages = [GpuStages(rec.positions, rec.weights, T, rec.dt, rec.sound_speed, rec.dx, nl, nl, pb.WindowSpec(), q,
                        world, 0) for q in range(world)]
    samples = torch.tensor(rec.samples, dtype=torch.float32, device=dev)
    f32 = dict(dtype=torch.float32, device=dev)
    gh_send = [torch.empty(L.rows_total * L.Tr * 2, **f32) for _ in range(world)]
    for q in range(world):
        stages[q].forward(samples[:, q * L.Tr:(q + 1) * L.Tr].contiguous(), gh_send[q], s)
    rs = L.row_starts
    gh_recv = [torch.cat([gh_send[p].view(L.rows_total, L.Tr * 2)[rs[q]:rs[q + 1]] for p in range(world)]).reshape(-1)
               for q in range(world)]
    z_send = [torch.empty(world * L.rows(q) * L.Tr * 2, **f32) for q in range(world)]
    for q in range(world):
        stages[q].ner(gh_recv[q], z_send[q], s)
    z_recv = [torch.cat([z_send[p].view(world, L.rows(p) * L.Tr * 2)[q] for p in range(world)]) for q in range(world)]
    imgs = [torch.empty(L.image_slice_shape(), **f32) for _ in range(world)]
    for q in range(world):
        stages[q].inverse(z_recv[q], imgs[q], s)
    torch.cuda.synchronize()
    got = torch.cat(imgs, dim=-1).double().cpu().numpy()
    torch.cuda.set_stream(torch.cuda.default_stream(dev))
    err = rel_l2(got, want)
    print(f"world {world} {case}: rel-L2 vs single GPU {err:.2e}")
    assert err <= 1e-6


def test_sharded_plan_rejects_unsupported_shapes():
    from paper_1501_02946_b200.parallel import GpuStages

    rec = synth.make_3d(3, 16, 96, 20e-9, "uniform", 1)  # 96 / 4 = 24: not a power of two
    with pytest.raises(pb.DeviceError):
        GpuStages(rec.positions, rec.weights, 96, rec.dt, rec.sound_speed, rec.dx, (16, 16), (16, 16),
                  pb.WindowSpec(), 0, 4, 0)


@pytest.mark.parametrize("world,chunks,blocks", [(2, 2, 3), (4, 2, 4), (8, 1, 2)])
def test_pipelined_shard_stages_match_single_gpu(world, chunks, blocks):
    """The pipelined stage entry points (whole-slice spread, lateral FFTs in time pieces, NER in row
    blocks) with the exchange layouts of parallel.ShardedNedNer,
    ranks emulated one after another on one GPU: bit-identical to one GPU."""
    rec = synth.make_3d(50 + world, 64, 256, 20e-9, "clustered", 3, sigma=2e-3)
    _emulate_pipelined(world, chunks, blocks, rec)


@pytest.mark.parametrize("seed", range(9100, 9108))
def test_pipelined_shard_stages_random_problems(seed):
    """Random power-of-two problems (2D and 3D), world sizes, time pieces and row blocks."""
    rng = np.random.default_rng(seed)
    nt = int(rng.choice([128, 256, 512]))
    world = int(rng.choice([2, 4, 8]))
    tr = nt // world
    chunks = int(rng.choice([1] + [c for c in (2, 4) if tr // c >= 32]))
    blocks = int(rng.integers(1, 6))
    if rng.random() < 0.25:
        rec = synth.make_2d(seed=seed, n=int(rng.choice([32, 64, 128])), nt=nt)
    else:
        rec = synth.make_3d(seed, int(rng.choice([16, 32, 64])), nt, 20e-9, str(rng.choice(["uniform", "jittered", "clustered"])), 3,
                            sigma=2e-3)
    _emulate_pipelined(world, chunks, blocks, rec)


def _emulate_pipelined(world, chunks, blocks, rec):
    import torch

    from paper_1501_02946_b200.parallel import GpuStages, ShardLayout

    want = pb.reconstruct_nedner(rec.as_record()).values
    nl = tuple(rec.n_lateral)
    T = rec.samples.shape[1]
    L = ShardLayout(len(nl), nl, T, world)
    C, Trc = chunks, L.Tr // chunks
    dev = torch.device("cuda", 0)
    stream = torch.cuda.Stream(device=dev)
    torch.cuda.set_stream(stream)
    s = stream.cuda_stream
    stages = [GpuStages(rec.positions, rec.weights, T, rec.dt, rec.sound_speed, rec.dx, nl, nl, pb.WindowSpec(), q,
                        world, 0) for q in range(world)]
    samples = torch.tensor(rec.samples, dtype=torch.float32, device=dev)
    f32 = dict(dtype=torch.float32, device=dev)
    rs = L.row_starts
    # rank p: pieces gh_send[p][c] = [rows_total][Trc]
    gh_send = [[torch.empty(L.rows_total * Trc * 2, **f32) for _ in range(C)] for _ in range(world)]
    for p in range(world):
        stages[p].spread(samples[:, p * L.Tr:(p + 1) * L.Tr].contiguous(), s)
        for c in range(C):
            stages[p].lateral(c * Trc, (c + 1) * Trc, gh_send[p][c], s)
    # rank q receives piece c of rank p as time chunk p*C + c of [chunk][rows_q][Trc]
    gh_recv = [torch.cat([gh_send[p][c].view(L.rows_total, Trc * 2)[rs[q]:rs[q + 1]].reshape(-1)
                          for p in range(world) for c in range(C)]) for q in range(world)]
    bounds = [[b * L.rows(q) // blocks for b in range(blocks + 1)] for q in range(world)]
    z_recv = [torch.empty(L.rows_total * L.Tr * 2, **f32) for _ in range(world)]
    for p in range(world):
        for b in range(blocks):
            b0, b1 = bounds[p][b], bounds[p][b + 1]
            zb = torch.empty(world * (b1 - b0) * L.Tr * 2, **f32)
            stages[p].ner_rows(gh_recv[p], Trc, b0, b1, zb, s)
            for q in range(world):  # block b of rank p -> its global rows on rank q
                r0, r1 = rs[p] + b0, rs[p] + b1
                z_recv[q][r0 * L.Tr * 2:r1 * L.Tr * 2].copy_(zb.view(world, -1)[q])
    imgs = [torch.empty(L.image_slice_shape(), **f32) for _ in range(world)]
    for q in range(world):
        stages[q].inverse(z_recv[q], imgs[q], s)
    torch.cuda.synchronize()
    got = torch.cat(imgs, dim=-1).double().cpu().numpy()
    torch.cuda.set_stream(torch.cuda.default_stream(dev))
    err = rel_l2(got, want)
    print(f"pipelined {nl} Nt={T} world {world} (pieces {C}, row blocks {blocks}): rel-L2 vs single GPU {err:.2e}")
    # (slices shorter than a tensor-core time block are gridded by the SIMT kernel: same answer to
    #  float32 rounding, not bit for bit)
    assert err <= (1e-6 if L.Tr >= 32 else 5e-6)


@pytest.mark.parametrize("world,case", [(3, "2d_nt96_up2"), (2, "3d_up2"), (3, "3d_outdims_nt40"), (4, "3d_up3")])
def test_general_schedule_stages_match_single_gpu(world, case):
    """The general multi-GPU schedule (sliced C plans: any even N_t, any upsample, uneven time
    slices; parallel.GeneralShardedNedNer's layouts) with the ranks emulated one after another on
    one GPU, against the single-GPU reconstruction and the oracle."""
    from test_sharded_gloo import _general_case

    rec, out_dims, up = _general_case(case)
    _emulate_general_schedule(world, rec, out_dims, up, f"{case}")


@pytest.mark.parametrize("seed", range(9000, 9012))
def test_general_schedule_random_problems(seed):
    """Random shapes (tests/fuzz_cases.py, default window) at random world sizes."""
    from fuzz_cases import draw

    cs = draw(seed)
    rng = np.random.default_rng(seed)
    nt = cs["samples"].shape[1]
    world = int(rng.integers(2, min(6, nt // 2) + 1))
    rec = synth.SyntheticRecord(cs["positions"], cs["weights"], cs["samples"], cs["dt"], synth.SOUND_SPEED, synth.PITCH,
                                cs["n_lateral"])
    _emulate_general_schedule(world, rec, cs["out_dims"], cs["upsample"], cs["desc"])


def _emulate_general_schedule(world, rec, out_dims, up, what):
    import torch

    from oracle import nedner_oracle as O
    from paper_1501_02946_b200.parallel import GpuSliceStages, SliceLayout
    from paper_1501_02946_b200.recon import _out_dims

    want = pb.reconstruct_nedner(rec.as_record(), out_dims=out_dims, upsample=up).values
    nl = tuple(rec.n_lateral)
    dims = _out_dims(nl, out_dims)
    T = rec.samples.shape[1]
    L = SliceLayout(len(dims), dims, T, world, up)
    dev = torch.device("cuda", 0)
    stream = torch.cuda.Stream(device=dev)
    torch.cuda.set_stream(stream)
    s = stream.cuda_stream
    f32 = dict(dtype=torch.float32, device=dev)
    stages = [GpuSliceStages(rec.positions, rec.weights, T, rec.dt, rec.sound_speed, rec.dx, nl, dims, up,
                             pb.WindowSpec(), L.t_starts[q + 1] - L.t_starts[q], 0) for q in range(world)]
    samples = torch.tensor(rec.samples, dtype=torch.float32, device=dev)
    rs = L.row_starts
    gh_part = []
    for q in range(world):
        t0, t1 = L.t_range(q)
        g = torch.empty(L.rows_total, t1 - t0, 2, **f32)
        stages[q].forward(samples[:, t0:t1].contiguous(), g, s)
        gh_part.append(g)
    z_full = []
    for q in range(world):
        rows = torch.cat([gh_part[p][rs[q]:rs[q + 1]] for p in range(world)], dim=1).contiguous()  # [rows_q][T]
        z = torch.zeros(L.rows_out_total, L.Tu, 2, **f32)
        stages[q].ner(rows, rs[q], rs[q + 1], z, s)
        z_full.append(z)
    idx = [torch.tensor(L.out_rows(p), dtype=torch.long, device=dev) for p in range(world)]
    imgs = []
    for q in range(world):
        u0, u1 = L.tu_range(q)
        zs = torch.zeros(L.rows_out_total, u1 - u0, 2, **f32)
        for p in range(world):
            zs.index_copy_(0, idx[p], z_full[p].index_select(0, idx[p])[:, u0:u1].contiguous())
        img = torch.empty(L.image_slice_shape(q), **f32)
        stages[q].inverse(zs, img, s)
        imgs.append(img)
    torch.cuda.synchronize()
    got = torch.cat(imgs, dim=-1).double().cpu().numpy()
    torch.cuda.set_stream(torch.cuda.default_stream(dev))
    oracle, _ = O.reconstruct_nedner(rec.positions, rec.weights, rec.samples, rec.dt, rec.sound_speed, rec.dx,
                                     rec.n_lateral, out_dims=out_dims, upsample=up)
    e1, e2 = rel_l2(got, want), rel_l2(got, oracle)
    print(f"general schedule world {world} {what}: rel-L2 vs single GPU {e1:.2e}, vs oracle {e2:.2e}")
    assert got.shape == want.shape and e1 <= 5e-6 and e2 <= 1e-4
