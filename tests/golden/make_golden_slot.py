"""sha256 digests of the REFERENCE's slot-grid outputs (build container only):

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden_slot.py

For each case of tests/slot_cases.py: `linksim.estimate_channel_ls` (bit-exact
target) from /root/reference/pkg/src, and the receive grid / data-RE batch
expressions of `simulate_frames` (linksim.py:207-216) with the reference's
data-symbol list.  Writes tests/golden/slot.json."""

import json
import sys
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
sys.path.insert(0, str(HERE.parent))
sys.path.insert(0, "/root/reference/pkg/src")
sys.dont_write_bytecode = True

from mpnlsim import core, linksim                     # noqa: E402  (reference)

import slot_cases as sc                                # noqa: E402


def main():
    out = {}
    for case in sc.CASES:
        name, n, m, rb, f, unit = case
        obs, pilots, h, x, noise = sc.inputs(case)
        cfg = linksim.LinkConfig(n_streams=n, m_antennas=m, mcs=core.mcs_entry(4),
                                 rb_per_vehicle=rb)
        est = linksim.estimate_channel_ls(obs, pilots, cfg)
        dsyms = [s for s in range(cfg.numerology.symbols_per_slot)
                 if s not in linksim._dmrs_pattern(cfg.numerology, n, cfg.n_subcarriers)[0]]
        y = np.einsum("tfmn,btfn->btfm", h, x) + noise
        out[name] = {"est": sc.digest(est), "data_syms": dsyms,
                     "h_flat": sc.digest(h[dsyms].reshape(len(dsyms) * 12 * rb, m, n)),
                     "y": sc.digest(y)}
    (HERE / "slot.json").write_text(json.dumps(out, indent=1) + "\n")
    print(out)


if __name__ == "__main__":
    main()
