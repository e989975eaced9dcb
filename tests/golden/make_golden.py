"""Generate the golden fixtures from the REFERENCE itself (build container only).

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden.py

Imports `mpnlsim` from /root/reference/pkg/src (read-only, never copied) and
records, on seeded inputs from `paper_2409_14355_b200.workloads`:

* ``alloc.npz``   allocate_expansions over a grid of (N, Q, P, n_forced);
* ``plan.npz``    mpnl_plan_batch perm / r / qh for a few channels;
* ``hard_<cfg>.npz``  the hard-output composition (cli.py:236-239) on the
  first RBs of every BASELINE config: inputs (complex64), hard labels,
  winning metric, second-lowest metric;
* ``full_<case>.npz`` the full mpnl_detect_batch return (labels, metrics,
  best) for small cases, pinning path order.

The reference is run exactly as its own bench does: a plan per vector row
(h repeated per vector) — bit-identical to one plan per RB tiled.
"""

from __future__ import annotations

import sys
import time
import warnings
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
ROOT = HERE.parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, "/root/reference/pkg/src")
sys.dont_write_bytecode = True

from mpnlsim import detect as det                      # noqa: E402  (reference)
from mpnlsim.core import constellation_for             # noqa: E402

from paper_2409_14355_b200.workloads import CONFIGS, generate   # noqa: E402

GOLD_RBS = {"C1": 4, "C2": 1, "C3": 2, "C4": 1, "C5P16": 2, "C5P64": 2, "C5P256": 1,
            "C5P1024": 1}


def ref_hard(h_rb, y_rb, nv, n_paths, order, chunk=336):
    c = constellation_for(order)
    nch, v, m = y_rb.shape
    h = np.repeat(h_rb.astype(complex), v, axis=0)
    y = y_rb.reshape(nch * v, m).astype(complex)
    hard, m1, m2, best = [], [], [], []
    for s in range(0, nch * v, chunk):
        plan = det.mpnl_plan_batch(h[s:s + chunk], nv, n_paths, c)
        lab, met, b = det.mpnl_detect_batch(plan, h[s:s + chunk], y[s:s + chunk], c)
        rows = np.arange(len(b))
        hard.append(lab[rows, b])
        m1.append(met[rows, b])
        m2.append(np.partition(met, 1, axis=1)[:, 1] if met.shape[1] > 1
                  else np.full(len(b), np.inf))
        best.append(b)
    cat = np.concatenate
    n = h_rb.shape[2]
    return (cat(hard).reshape(nch, v, n).astype(np.uint8), cat(m1).reshape(nch, v),
            cat(m2).reshape(nch, v), cat(best).reshape(nch, v))


def main():
    t0 = time.time()
    # ---- allocation grid ----
    rows = []
    warnings.simplefilter("ignore")
    for n in list(range(1, 13)) + [16, 20, 24, 28, 32]:
        for q in (4, 16, 64):
            for p in sorted(set(list(range(1, 40)) + [48, 63, 64, 65, 96, 100, 127, 128, 200,
                                                      256, 500, 512, 1000, 1024, 4096])):
                for nf in (0, 1, 2):
                    if nf >= n:
                        continue
                    with warnings.catch_warnings(record=True) as w:
                        warnings.simplefilter("always")
                        e, r = det.allocate_expansions(n, q, p, nf)
                    ex = np.zeros(32, np.int64)
                    ex[:n] = e
                    rows.append((n, q, p, nf, r, int(len(w) > 0), ex))
    np.savez_compressed(HERE / "alloc.npz",
                        n=np.array([r[0] for r in rows]), q=np.array([r[1] for r in rows]),
                        p=np.array([r[2] for r in rows]), nf=np.array([r[3] for r in rows]),
                        realized=np.array([r[4] for r in rows]),
                        warned=np.array([r[5] for r in rows]),
                        expansions=np.stack([r[6] for r in rows]))
    print(f"alloc: {len(rows)} rows", flush=True)

    # ---- plans ----
    plan_data = {}
    for name in ("C1", "C3", "C4", "C5P64"):
        d = generate(name, n_rb=2)
        cfg = d["cfg"]
        pl = det.mpnl_plan_batch(d["h"].astype(complex), d["nv"][0], cfg.n_paths,
                                 constellation_for(cfg.order))
        plan_data[f"{name}_h"] = d["h"]
        plan_data[f"{name}_perm"] = pl.perm
        plan_data[f"{name}_r"] = pl.r
        plan_data[f"{name}_qh"] = pl.qh
        plan_data[f"{name}_exp"] = pl.expansions
    rng = np.random.default_rng(77)
    ho = ((rng.standard_normal((3, 2, 3)) + 1j * rng.standard_normal((3, 2, 3))) / np.sqrt(2))
    pl = det.mpnl_plan_batch(ho, 0.1, 32, constellation_for(4))
    plan_data.update(over_h=ho, over_perm=pl.perm, over_r=pl.r, over_qh=pl.qh,
                     over_exp=pl.expansions)
    np.savez_compressed(HERE / "plan.npz", **plan_data)
    print("plans done", flush=True)

    # ---- hard outputs per config ----
    for name, nrb in GOLD_RBS.items():
        t = time.time()
        d = generate(name, n_rb=nrb)
        cfg = d["cfg"]
        hard, m1, m2, best = ref_hard(d["h"], d["y"], d["nv"][0], cfg.n_paths, cfg.order)
        np.savez_compressed(HERE / f"hard_{name}.npz", h=d["h"], y=d["y"], labels=d["labels"],
                            hard=hard, m1=m1, m2=m2, best=best, nv=d["nv"][0],
                            n_paths=cfg.n_paths, order=cfg.order)
        print(f"{name}: {hard.shape} in {time.time() - t:.1f}s", flush=True)

    # ---- full candidate lists (path order) ----
    cases = {
        "c1": ("C1", 12), "c2": ("C2", 6), "c5p16": ("C5P16", 6), "c5p256": ("C5P256", 3),
    }
    for tag, (name, nv_) in cases.items():
        d = generate(name, n_rb=1)
        cfg = d["cfg"]
        c = constellation_for(cfg.order)
        h = np.repeat(d["h"].astype(complex), nv_, axis=0)
        y = d["y"][0, :nv_].astype(complex)
        plan = det.mpnl_plan_batch(h, d["nv"][0], cfg.n_paths, c)
        lab, met, b = det.mpnl_detect_batch(plan, h, y, c)
        np.savez_compressed(HERE / f"full_{tag}.npz", h=d["h"][:1], y=d["y"][:1, :nv_],
                            labels=lab.astype(np.uint8), metrics=met, best=b,
                            nv=d["nv"][0], n_paths=cfg.n_paths, order=cfg.order)
    # small QPSK / overloaded cases in complex128
    rng = np.random.default_rng(4242)
    for tag, (m, n, q, p, snr) in {"q4x4": (4, 4, 4, 32, 8.0), "q4full": (3, 3, 4, 64, 6.0),
                                   "over2x3": (2, 3, 4, 32, 20.0),
                                   "q16_4x4": (4, 4, 16, 16, 15.0)}.items():
        c = constellation_for(q)
        b = 40
        h = (rng.standard_normal((b, m, n)) + 1j * rng.standard_normal((b, m, n))) / np.sqrt(2)
        lab_t = rng.integers(0, q, (b, n))
        nv = n / 10 ** (snr / 10)
        y = np.einsum("bmn,bn->bm", h, c.points[lab_t]) + np.sqrt(nv / 2) * (
            rng.standard_normal((b, m)) + 1j * rng.standard_normal((b, m)))
        plan = det.mpnl_plan_batch(h, nv, p, c)
        lab, met, bb = det.mpnl_detect_batch(plan, h, y, c)
        np.savez_compressed(HERE / f"full_{tag}.npz", h=h, y=y, labels=lab.astype(np.uint8),
                            metrics=met, best=bb, nv=nv, n_paths=p, order=q,
                            perm=plan.perm, r=plan.r, qh=plan.qh, expansions=plan.expansions)
    print(f"all done in {time.time() - t0:.1f}s")


if __name__ == "__main__":
    main()
