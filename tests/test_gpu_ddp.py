"""The DDP communication hook (paper_2310_00967_b200/ddp.py):
a real torch DDP model whose bucket all-reduce is replaced by MiCRO.  The
gradient DDP hands the optimizer must equal the oracle cluster's g/n on the
same per-rank bucket gradients, bit for bit, every iteration.  GPU only."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _run(rank, world, port, iters, transport, q, f64=False):
    import sys
    sys.path[:0] = [ROOT, os.path.join(ROOT, "oracle")]
    from oracle import OracleCluster

    from paper_2310_00967_b200.ddp import MicroHookState, micro_hook
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    torch.manual_seed(0)
    model = torch.nn.Sequential(torch.nn.Linear(64, 256), torch.nn.ReLU(), torch.nn.Linear(256, 10)).cuda()
    ddp = torch.nn.parallel.DistributedDataParallel(model, device_ids=[0], bucket_cap_mb=0.05)
    state = MicroHookState(density=0.05, initial_threshold=0.002, transport=transport, comm_device="cpu",
                           state_dtype=torch.float64 if f64 else torch.float32)
    seen = []  # (bucket index, iteration, gradient in, gradient out)

    def hook(st, bucket):
        g_in = bucket.buffer().detach().clone()
        t = st.t
        fut = micro_hook(st, bucket)
        seen.append((bucket.index(), t, g_in, fut.value().detach().clone()))
        return fut

    ddp.register_comm_hook(state, hook)
    opt = torch.optim.SGD(ddp.parameters(), lr=0.1)
    gen = torch.Generator().manual_seed(100 + rank)
    for _ in range(iters):
        x = torch.randn(32, 64, generator=gen).cuda()
        y = torch.randint(0, 10, (32,), generator=gen).cuda()
        opt.zero_grad()
        torch.nn.functional.cross_entropy(ddp(x), y).backward()
        opt.step()
    torch.cuda.synchronize()
    # every rank's bucket inputs, to replay the cluster in the oracle
    allseen = [None] * world
    dist.all_gather_object(allseen, [(i, t, a.cpu().numpy(), b.cpu().numpy()) for i, t, a, b in seen])
    params = [p.detach().cpu().numpy() for p in model.parameters()]
    allparams = [None] * world
    dist.all_gather_object(allparams, params)
    bad = []
    if any(not all(np.array_equal(a, b) for a, b in zip(allparams[0], ps)) for ps in allparams):
        bad.append("params differ across ranks")
    # replay: per (bucket index, size) an oracle cluster, iteration t = call order
    clusters = {}
    for k in range(len(seen)):
        idx, t, _, out = allseen[rank][k]
        G = np.stack([allseen[r][k][2] for r in range(world)]).astype(np.float64 if f64 else np.float32)
        key = (idx, G.shape[1])
        if key not in clusters:  # DDP rebuilt the bucket: a fresh context, like the hook
            for old in [o for o in clusters if o[0] == idx]:
                clusters.pop(old)
            clusters[key] = OracleCluster(G.shape[1], world, density=0.05, delta0=0.002,
                                          dtype=np.float64 if f64 else np.float32)
        r = clusters[key].step(G, 1.0, t)
        want = np.zeros(G.shape[1], np.float32)
        if f64:  # fp64 g/n, then DDP's fp32 bucket
            want[r["union_idx"]] = (r["union_sum"].astype(np.float64) / np.float64(world)).astype(np.float32)
        else:
            want[r["union_idx"]] = r["union_sum"].astype(np.float32) / np.float32(world)
        if not np.array_equal(out, want):
            bad.append((k, idx, "g/n"))
    state.close()
    dist.destroy_process_group()
    q.put((rank, bad))


@pytest.mark.parametrize("world,transport,f64", [(1, "peer", False), (2, "peer", False), (2, "peer_pull", False),
                                                (2, "nccl", False), (1, "peer", True), (2, "peer", True)])
def test_ddp_hook(world, transport, f64):
    """f64: fp32 bucket gradients, fp64 residuals and sums (state_dtype)."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_run, args=(r, world, port, 6, transport, q, f64)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
    for rank, bad in res:
        assert not bad, (rank, bad[:5])
