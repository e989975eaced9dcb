"""Golden list-LLR fixtures from the REFERENCE itself (build container only).

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden_llr.py

For every committed ``full_<case>.npz`` (reference candidate lists) this runs
the reference's ``_candidate_llrs_batch`` (detect.py:439-453) with the
scalar noise variance, with a per-list noise-variance array, and with a
custom clip, and writes ``llr_<case>.npz``.  One extra case (``llr_p1``)
pins the saturation of bits no path sets or clears (P = 1 and P = 2).
"""

from __future__ import annotations

import sys
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
sys.path.insert(0, "/root/reference/pkg/src")
sys.dont_write_bytecode = True

from mpnlsim import detect as det                      # noqa: E402  (reference)
from mpnlsim.core import constellation_for             # noqa: E402


def main():
    for f in sorted(HERE.glob("full_*.npz")):
        d = np.load(f)
        c = constellation_for(int(d["order"]))
        lab, met, nv = d["labels"].astype(np.int64), d["metrics"], float(d["nv"])
        b = lab.shape[0]
        nv_vec = nv * (1.0 + 0.25 * np.arange(b) / max(b, 1))
        out = dict(labels=d["labels"], metrics=met, nv=nv, nv_vec=nv_vec, order=int(d["order"]),
                   llr=det._candidate_llrs_batch(lab, met, nv, c),
                   llr_vec=det._candidate_llrs_batch(lab, met, nv_vec, c),
                   llr_clip3=det._candidate_llrs_batch(lab, met, nv, c, clip=3.0))
        np.savez_compressed(HERE / f"llr_{f.stem[5:]}.npz", **out)
        print(f.stem, lab.shape)
    rng = np.random.default_rng(99)
    for p in (1, 2):
        c = constellation_for(16)
        lab = rng.integers(0, 16, (5, p, 6))
        met = rng.exponential(2.0, (5, p))
        np.savez_compressed(HERE / f"llr_p{p}.npz", labels=lab.astype(np.uint8), metrics=met,
                            nv=0.3, nv_vec=np.full(5, 0.3), order=16,
                            llr=det._candidate_llrs_batch(lab, met, 0.3, c),
                            llr_vec=det._candidate_llrs_batch(lab, met, np.full(5, 0.3), c),
                            llr_clip3=det._candidate_llrs_batch(lab, met, 0.3, c, clip=3.0))
    print("done")


if __name__ == "__main__":
    main()
