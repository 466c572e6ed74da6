"""Writes rank / top-k results of a fixed bf16 instance (D = 64) for k = 3, 10, 16
to the given file: run once per library build (LSEFORGE_B200_LIB) and compare
the files to check a tuning variant against the default bitwise."""
import sys, torch, os
sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", "/root/repo"))
from paper_2509_09682_b200 import metrics
g = torch.Generator(device="cuda").manual_seed(5)
n, d, v = 4096, 64, 300_000
X = (torch.randn(n, d, device="cuda", generator=g) * 0.4).to(torch.bfloat16)
E = (torch.randn(v, d, device="cuda", generator=g) * 0.4).to(torch.bfloat16)
t = torch.randint(0, v, (n,), device="cuda", generator=g)
E[t[:128]] = X[:128]
E[1000:1100] = E[5]
out = {k: [x.cpu() for x in metrics.rank_topk(X, E, t, k)] for k in (3, 10, 16)}
torch.save(out, sys.argv[1])
