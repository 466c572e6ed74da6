"""GPU: the peer-memory exchange of the catalog-sharded CCE
(ShardedCce(exchange="peer"), lf_cce_forward_partial_peer /
lf_cce_backward_shard_peer / lf_peer_barrier / lf_peer_sum) gives the same
bits as the collective exchange.  Two processes share cuda:0 (CUDA IPC
between processes on one device exercises the same mapped-pointer stores an
NVSwitch box does between devices); the handle swap and the reference
collective run over gloo."""
import os
import socket
import subprocess
import sys
import textwrap

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

WORKER = textwrap.dedent('''
    import os, sys, torch, torch.distributed as dist
    sys.path.insert(0, os.environ["LF_ROOT"])
    import paper_2509_09682_b200 as lf
    from paper_2509_09682_b200.sharded import ShardedCce, shard_bounds
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    dtype = getattr(torch, os.environ["LF_DT"])
    n, d, v = 300, 64, 5000
    g = torch.Generator(device="cpu").manual_seed(5)
    X = (torch.randn(n, d, generator=g) * 0.5).to(dtype).cuda()
    Efull = (torch.randn(v, d, generator=g) * 0.5).to(dtype).cuda()
    x = torch.randint(0, v, (n,), generator=g).cuda()
    b, e = shard_bounds(v, world, rank)
    Es = Efull[b:e].contiguous()
    cfg = lf.CceConfig(filter_eps=float(os.environ["LF_EPS"]))
    outs = {}
    for mode in ("collective", "peer", "peer"):  # the second peer call uses the other parity half
        sh = ShardedCce(v, exchange=mode) if mode == "collective" or "peer" not in outs else sh
        fo = sh.forward(X, Es, x, cfg)
        bo = sh.backward(X, Es, x, fo.lse, 1.0, cfg)
        torch.cuda.synchronize()
        outs.setdefault(mode, []).append((fo.loss.item(), fo.lse.cpu(), fo.pos_logits.cpu(),
                                          bo.grads.d_embeddings.cpu(), bo.grads.d_classifier.cpu(),
                                          bo.skipped_fraction))
    ref = outs["collective"][0]
    for got in outs["peer"]:
        assert got[0] == ref[0], (got[0], ref[0])
        assert torch.equal(got[1], ref[1]) and torch.equal(got[2], ref[2])
        assert torch.equal(got[3], ref[3]), (got[3] - ref[3]).abs().max()
        assert torch.equal(got[4], ref[4])
        assert got[5] == ref[5]
    dist.barrier()
    print("rank", rank, "ok")
''')


def _port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.mark.parametrize("dt,eps", [("bfloat16", 6e-8), ("bfloat16", 0.0), ("float32", 1e-3)])
def test_peer_exchange_matches_collectives(cuda, dt, eps):
    port = _port()
    procs = []
    for r in range(2):
        env = dict(os.environ, RANK=str(r), WORLD_SIZE="2", MASTER_ADDR="127.0.0.1",
                   MASTER_PORT=str(port), LF_ROOT=ROOT, LF_DT=dt, LF_EPS=str(eps))
        procs.append(subprocess.Popen([sys.executable, "-c", WORKER], env=env, stdout=subprocess.PIPE,
                                      stderr=subprocess.STDOUT, text=True))
    outs = [p.communicate(timeout=300)[0] for p in procs]
    for p, o in zip(procs, outs):
        assert p.returncode == 0, o[-3000:]
        assert "ok" in o
