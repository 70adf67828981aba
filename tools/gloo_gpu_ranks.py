"""Two (or more) ranks of the real sharded orchestration (ShardedNedNer / GeneralShardedNedNer with the
CUDA stages) on ONE GPU, exchanging through gloo (host-mediated send/recv: no kernel waits on another
rank).  usage: python tools/gloo_gpu_ranks.py WORLD [general]"""
import os, socket, sys
import numpy as np
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def worker(rank, world, port, general, outdir):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        torch.cuda.set_device(0)
        from paper_1501_02946_b200 import synth
        from paper_1501_02946_b200.parallel import GeneralShardedNedNer, ShardedNedNer
        dev = torch.device("cuda", 0)
        if general:
            rec = synth.make_3d(61, 16, 40, 20e-9, "jittered", 2)
            sh = GeneralShardedNedNer(rec.positions, rec.weights, rec.samples.shape[1], rec.dt, rec.sound_speed, rec.dx,
                                      rec.n_lateral, upsample=2, torch_device=dev)
            t0, t1 = sh.layout.t_range(rank)
        else:
            rec = synth.make_3d(60, 64, 256, 20e-9, "clustered", 3, sigma=2e-3)
            sh = ShardedNedNer(rec.positions, rec.weights, rec.samples.shape[1], rec.dt, rec.sound_speed, rec.dx,
                               rec.n_lateral, torch_device=dev)
            tr = sh.layout.Tr
            t0, t1 = rank * tr, (rank + 1) * tr
        sl = torch.tensor(np.ascontiguousarray(rec.samples[:, t0:t1]), dtype=torch.float32, device=dev)
        for _ in range(2):
            img = sh.run(sl)
        torch.cuda.synchronize()
        np.save(os.path.join(outdir, f"slice{rank}.npy"), img.cpu().numpy())
    finally:
        dist.destroy_process_group()


if __name__ == "__main__":
    world = int(sys.argv[1]) if len(sys.argv) > 1 else 2
    general = len(sys.argv) > 2
    import tempfile
    s = socket.socket(); s.bind(("127.0.0.1", 0)); port = s.getsockname()[1]; s.close()
    with tempfile.TemporaryDirectory() as d:
        mp.spawn(worker, args=(world, port, general, d), nprocs=world, join=True)
        got = np.concatenate([np.load(os.path.join(d, f"slice{r}.npy")) for r in range(world)], axis=-1)
    import paper_1501_02946_b200 as pb
    from paper_1501_02946_b200 import synth
    if general:
        rec = synth.make_3d(61, 16, 40, 20e-9, "jittered", 2)
        want = pb.reconstruct_nedner(rec.as_record(), upsample=2).values
    else:
        rec = synth.make_3d(60, 64, 256, 20e-9, "clustered", 3, sigma=2e-3)
        want = pb.reconstruct_nedner(rec.as_record()).values
    err = float(np.linalg.norm(got - want) / np.linalg.norm(want))
    print(f"world {world} {'general' if general else 'pipelined'} schedule over gloo, CUDA stages on one GPU: rel-L2 vs single GPU {err:.2e}")
    assert got.shape == want.shape and err <= 5e-6
