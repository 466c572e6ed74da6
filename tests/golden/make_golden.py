"""Generate tests/golden/*.npz from the REFERENCE implementation.

Runs the unmodified reference hot-path sources compiled in place
(oracle/_ref/liblseforge_ref.so, built by oracle/Makefile from
/root/reference/proj/src) on small instances drawn with the reference's own
fixtures (support.hpp make_instance / make_candidates, SplitMix64) and stores
inputs + outputs.  The committed .npz files travel to the GPU box, where
/root/reference does not exist; tests/test_oracle.py pins the C restatement to
them and the GPU tests compare the CUDA path against them.

    python tests/golden/make_golden.py
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))
import oracle_bind as ob  # noqa: E402


def ref_instance(seed, n, d, v):
    E = np.empty((n, d), np.float32)
    C = np.empty((d, v), np.float32)
    t = np.empty(n, np.int64)
    ob.ref().ref_make_instance(seed, n, d, v, 1.0, E, C, t)
    return E, C, t


def ref_instance_cand(seed, n, d, v, ns):
    E = np.empty((n, d), np.float32)
    C = np.empty((d, v), np.float32)
    t = np.empty(n, np.int64)
    inds = np.empty((n, 1 + ns), np.int64)
    ob.ref().ref_make_instance_candidates(seed, n, d, v, ns, E, C, t, inds)
    return E, C, t, inds


def main():
    out = {}
    # SplitMix64 streams (also pinned by test_core.cpp:21-52)
    for seed in (0, 42, 0xDEADBEEF, 0xB2000002):
        out[f"rng_{seed:x}"] = ob.ref_rng_stream(seed, 16)
    np.savez_compressed(os.path.join(HERE, "rng_streams.npz"), **out)

    # CCE: a spread of shapes incl. ragged tiles; eps 0 and 1e-3.
    cases = [(1001, 17, 6, 37), (1002, 33, 16, 129), (1003, 5, 1, 2), (1004, 64, 64, 300),
             (1005, 130, 64, 257), (1006, 40, 128, 200)]
    cce = {}
    for k, (seed, n, d, v) in enumerate(cases):
        E, C, t = ref_instance(seed, n, d, v)
        loss, pos, lse = ob.ref_cce_forward(E, C, t, rb=7, cb=13)
        dE0, dC0, f0 = ob.ref_cce_backward(E, C, t, lse, 1.0, 0.0, rb=7, cb=13)
        dE1, dC1, f1 = ob.ref_cce_backward(E, C, t, lse, 1.0, 1e-3, rb=7, cb=13)
        cce.update({f"{k}_E": E, f"{k}_C": C, f"{k}_t": t, f"{k}_loss": np.float64(loss),
                    f"{k}_pos": pos, f"{k}_lse": lse, f"{k}_dE": dE0, f"{k}_dC": dC0,
                    f"{k}_dE_eps": dE1, f"{k}_dC_eps": dC1, f"{k}_frac": np.float64(f0),
                    f"{k}_frac_eps": np.float64(f1)})
    cce["count"] = np.int64(len(cases))
    np.savez_compressed(os.path.join(HERE, "cce_ref.npz"), **cce)

    # CCE-: sampled candidates (make_candidates) and sampler output.
    ccases = [(2001, 13, 8, 40, 5), (2002, 41, 8, 67, 9), (2003, 6, 3, 16, 4), (2004, 64, 64, 500, 31),
              (2005, 9, 5, 10, 0)]
    ccem = {}
    for k, (seed, n, d, v, ns) in enumerate(ccases):
        E, C, t, inds = ref_instance_cand(seed, n, d, v, ns)
        loss, pos, lse = ob.ref_ccem_forward(E, C, inds)
        up = np.full(n, 1.0 / n)
        dE, dC = ob.ref_ccem_backward_rows(E, C, inds, lse, up)
        ccem.update({f"{k}_E": E, f"{k}_C": C, f"{k}_inds": inds, f"{k}_loss": np.float64(loss),
                     f"{k}_pos": pos, f"{k}_lse": lse, f"{k}_dE": dE, f"{k}_dC": dC})
    ccem["count"] = np.int64(len(ccases))
    pos = np.arange(50, dtype=np.int64) % 97
    ccem["sampler_pos"] = pos
    ccem["sampler_inds"] = ob.ref_sample_uniform(pos, 12, 97, 0xB2000003)
    np.savez_compressed(os.path.join(HERE, "ccem_ref.npz"), **ccem)
    eval_fixtures()
    adam_fixtures()
    encoder_fixtures()
    popularity_fixtures()
    print("wrote", sorted(f for f in os.listdir(HERE) if f.endswith(".npz")))


def eval_fixtures():
    """evaluate() (metrics.cpp:13-103) on ToyEncoderParams::Init instances:
    summary, encoded rows H, classifier C and per-row ranks (eval_ref.npz)."""
    cases = [(300, 16, 11, 40, 3, 10), (1000, 64, 12, 100, 5, 16), (9, 4, 0xE1, 5, 2, 9),
             (129, 8, 13, 33, 1, 1), (2000, 32, 14, 64, 4, 32)]
    ev = {}
    for c, (cat, hid, seed, n, L, k) in enumerate(cases):
        g = np.random.default_rng(seed)
        pre = g.integers(0, cat, (n, L))
        tg = g.integers(0, cat, n)
        counts = g.integers(0, 40, cat)
        out3, H, Cm, ranks = ob.ref_eval_instance(cat, hid, seed, pre, tg, k, counts)
        ev.update({f"{c}_H": H, f"{c}_C": Cm, f"{c}_t": tg, f"{c}_counts": counts,
                   f"{c}_k": np.int64(k), f"{c}_out3": np.array(out3), f"{c}_ranks": ranks})
    ev["count"] = np.int64(len(cases))
    np.savez_compressed(os.path.join(HERE, "eval_ref.npz"), **ev)


def adam_fixtures():
    """AdamState::step (adam.cpp:22-55) on ToyEncoderParams::Init: initial
    params, per-step gradients (spanning 1e-8 .. 10) and final params."""
    cat, hid, seed, steps = 60, 4, 21, 4
    lr, b1, b2, eps = 1e-2, 0.9, 0.999, 1e-8
    p0 = ob.ref_encoder_init(cat, hid, seed)
    g = np.random.default_rng(seed)
    grads = [g.standard_normal(p0.size) * 10.0 ** g.integers(-8, 2, p0.size) for _ in range(steps)]
    want = ob.ref_adam_steps(cat, hid, seed, lr, b1, b2, eps, grads)
    np.savez_compressed(os.path.join(HERE, "adam_ref.npz"), p0=p0, grads=np.stack(grads), want=want,
                        hp=np.array([lr, b1, b2, eps]))


def encoder_fixtures():
    """encode_batch + encoder_backward (encoder.cpp:64-173) run by the
    reference on random parameters, ragged windows and d_h."""
    g = np.random.default_rng(77)
    cat, d = 50, 16
    emb = (g.standard_normal((cat, d)) * 0.3).astype(np.float32)
    W = (g.standard_normal((d, d)) * 0.3).astype(np.float32)
    b = (g.standard_normal(d) * 0.1).astype(np.float32)
    lens = g.integers(2, 12, 20)
    win_off = np.concatenate([[0], np.cumsum(lens)]).astype(np.int64)
    items = g.integers(0, cat, int(win_off[-1])).astype(np.int64)
    dh = g.standard_normal((int(np.sum(lens - 1)), d))
    r = ob.ref_encoder(emb, W, b, items, win_off, dh)
    np.savez_compressed(os.path.join(HERE, "encoder_ref.npz"), emb=emb, W=W, b=b, items=items,
                        win_off=win_off, dh=dh, **r)


def popularity_fixtures():
    """sample_popularity (sampler.cpp:77-127) run by the reference: skewed
    counts with zero-weight items, exponents 1 and 0.75."""
    g = np.random.default_rng(31)
    out = {}
    for c, (cat, n, ns, exp, seed) in enumerate(((2000, 64, 31, 1.0, 0xB2000005), (500, 40, 9, 0.75, 7),
                                                 (12, 30, 11, 1.0, 11))):
        counts = (g.zipf(1.3, cat) % 1000).astype(np.int64)
        counts[g.integers(0, cat, cat // 4)] = 0
        pos = g.integers(0, cat, n).astype(np.int64)
        counts[pos] = np.maximum(counts[pos], 0)
        out.update({f"{c}_counts": counts, f"{c}_pos": pos, f"{c}_ns": np.int64(ns),
                    f"{c}_exp": np.float64(exp), f"{c}_seed": np.uint64(seed),
                    f"{c}_inds": ob.ref_sample_popularity(pos, ns, counts, seed, exp)})
    out["count"] = np.int64(3)
    np.savez_compressed(os.path.join(HERE, "popularity_ref.npz"), **out)


if __name__ == "__main__":
    if sys.argv[1:] == ["popularity"]:
        popularity_fixtures()
    elif sys.argv[1:] == ["encoder"]:
        encoder_fixtures()
    elif sys.argv[1:] == ["adam"]:
        adam_fixtures()
    elif sys.argv[1:] == ["eval"]:
        eval_fixtures()
    else:
        main()
