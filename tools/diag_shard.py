import sys, numpy as np, torch
sys.path.insert(0, '/root/repo'); sys.path.insert(0, '/root/repo/tests')
import paper_1501_02946_b200 as pb
from paper_1501_02946_b200 import synth
from oracle import nedner_oracle as O
from conftest import rel_l2
from paper_1501_02946_b200.parallel import GpuStages, ShardLayout

def sharded(rec, world):
    nl = tuple(rec.n_lateral); T = rec.samples.shape[1]
    L = ShardLayout(2, nl, T, world)
    dev = torch.device("cuda", 0); st = torch.cuda.Stream(device=dev); torch.cuda.set_stream(st); s = st.cuda_stream
    stages = [GpuStages(rec.positions, rec.weights, T, rec.dt, rec.sound_speed, rec.dx, nl, nl, pb.WindowSpec(), q, world, 0) for q in range(world)]
    samples = torch.tensor(rec.samples, dtype=torch.float32, device=dev)
    f32 = dict(dtype=torch.float32, device=dev)
    gh_send = [torch.empty(L.rows_total * L.Tr * 2, **f32) for _ in range(world)]
    for q in range(world): stages[q].forward(samples[:, q * L.Tr:(q + 1) * L.Tr].contiguous(), gh_send[q], s)
    rs = L.row_starts
    gh_recv = [torch.cat([gh_send[p].view(L.rows_total, L.Tr * 2)[rs[q]:rs[q + 1]] for p in range(world)]).reshape(-1) for q in range(world)]
    z_send = [torch.empty(world * L.rows(q) * L.Tr * 2, **f32) for q in range(world)]
    for q in range(world): stages[q].ner(gh_recv[q], z_send[q], s)
    z_recv = [torch.cat([z_send[p].view(world, L.rows(p) * L.Tr * 2)[q] for p in range(world)]) for q in range(world)]
    imgs = [torch.empty(L.image_slice_shape(), **f32) for _ in range(world)]
    for q in range(world): stages[q].inverse(z_recv[q], imgs[q], s)
    torch.cuda.synchronize()
    return torch.cat(imgs, dim=-1).double().cpu().numpy()

for case, seed in [("uniform", 44), ("clustered", 42)]:
    rec = synth.make_3d(seed, 64, 256, 20e-9, case, 3, sigma=2e-3)
    single = pb.reconstruct_nedner(rec.as_record()).values
    ora, _ = O.reconstruct_nedner(rec.positions, rec.weights, rec.samples, rec.dt, rec.sound_speed, rec.dx, rec.n_lateral)
    print(case, "single vs oracle", rel_l2(single, ora))
    for w in (2, 4, 8):
        g = sharded(rec, w)
        print(case, w, rel_l2(g, single), [rel_l2(g[..., q*(256//w):(q+1)*(256//w)], single[..., q*(256//w):(q+1)*(256//w)]) for q in range(w)])
