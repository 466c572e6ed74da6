"""A whole training step on the device (trainer.cpp:209-227, cfg2 shape):
encode_batch -> fused CCE forward+backward (bf16, eps = 6e-8) -> encoder_backward
-> Adam over emb, W, b and the classifier (with the bf16 shadow of E the next
step reads).  256 windows x 201 items -> N = 51 200 rows, V = 1M, D = 64,
synthetic.  CUDA-event time per stage, one JSON line."""
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2509_09682_b200 as lf  # noqa: E402
from paper_2509_09682_b200 import encoder  # noqa: E402

V, D, NW, L = 1_000_000, 64, 256, 201
g = torch.Generator(device="cuda").manual_seed(0)
emb = (torch.rand(V, D, device="cuda", generator=g) * 2 - 1) * 0.0125
W = (torch.rand(D, D, device="cuda", generator=g) * 2 - 1) * 0.0125
b = torch.zeros(D, device="cuda")
E32 = (torch.rand(V, D, device="cuda", generator=g) * 2 - 1) * 0.0125  # classifier, item-major
E = E32.to(torch.bfloat16)
items = torch.randint(0, V, (NW * L,), device="cuda", generator=g)
win_off = torch.arange(0, NW * L + 1, L, device="cuda", dtype=torch.int64)
cfg = lf.CceConfig(filter_eps=6e-8)
opt = lf.DeviceAdam([emb, W, b, E32])


def step():
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(5)]
    ev[0].record()
    batch = encoder.encode_batch(emb, W, b, items, win_off, torch.bfloat16)
    ev[1].record()
    # run_loss_layer's pairing (trainer.cpp:71-77) as one fused call
    out, res = lf.cce_forward_backward(batch.X, E, batch.targets, 1.0, cfg, validate=False)
    ev[2].record()
    d_emb, d_W, d_b = encoder.encoder_backward(V, W, batch, res.grads.d_embeddings)
    ev[3].record()
    opt.step([d_emb, d_W, d_b, res.grads.d_classifier], [None, None, None, E])
    ev[4].record()
    return ev, out


for _ in range(2):
    step()
torch.cuda.synchronize()
times = []
for _ in range(3):
    ev, out = step()
    torch.cuda.synchronize()
    times.append([ev[i].elapsed_time(ev[i + 1]) for i in range(4)])
t = [min(x[i] for x in times) for i in range(4)]
print(json.dumps({"probe": "device training step", "rows": NW * (L - 1), "v": V, "d": D,
                  "ms": {"encode_batch": t[0], "cce_fwd_bwd": t[1], "encoder_backward": t[2],
                         "adam(emb,W,b,C)": t[3], "total": sum(t)},
                  "positions_per_s": NW * (L - 1) / sum(t) * 1e3, "loss": float(out.loss)}))
