import os, sys
import numpy as np, torch, torch.distributed as dist
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__))); sys.path.insert(0, ROOT)
import paper_1711_04325_b200 as L, synth
from oracle import exchange, run, schedule
rank, world, local = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"]), int(os.environ["LOCAL_RANK"])
torch.cuda.set_device(local); dev = torch.device("cuda", local)
dist.init_process_group("nccl", device_id=dev)
D = lambda x: torch.from_numpy(np.ascontiguousarray(x)).to(dev)
n = 50_021
C1 = schedule.Cluster(n_workers=2, b_local=32, n_train=64); C1_C = L.make_cluster(2, 32, 64)
for wd in (0.0, 1e-4):
    ctx = L.lmsgd_init(world, rank, local, n, 1024.0)
    L.connect_process_group(ctx)
    L.lmsgd_set_weight_decay(ctx, wd, 30_000)
    th0 = synth.theta0(n, None)
    th, d, m = D(th0), D(np.zeros(n, np.float32)), D(np.zeros(n, np.float32))
    g = synth.grads(world, 2, n)
    L.lmsgd_step(ctx, th, D(g[rank]), d, m, L.lmsgd_schedule_at(None, C1_C, 2))
    code, st = L.lmsgd_query_status(ctx)
    ex = exchange.exchange(list(g), 1024.0)
    z = np.zeros(n)
    th_o, d_o, m_o = run.resync_step(th0, z, z, ex.ghat, schedule.coeffs_at(2, schedule.Hyper(), C1), schedule.Hyper(), wd, 30_000)
    mg = m.cpu().numpy().astype(np.float64)
    rel = np.abs(mg - m_o) / np.maximum(m_o, 1e-30)
    bad = np.nonzero(rel > 1e-5)[0]
    th_o0, d_o0, m_o0 = run.resync_step(th0, z, z, ex.ghat, schedule.coeffs_at(2, schedule.Hyper(), C1))
    rel0 = np.abs(mg - m_o0) / np.maximum(m_o0, 1e-30)
    if rank == 0:
        print(f"wd={wd} code={code} bad={bad.size} first={bad[:10]} maxrel={rel.max():.3e} vs_no_wd_maxrel={rel0.max():.3e}", flush=True)
    L.lmsgd_finalize(ctx)
dist.destroy_process_group()
