"""Reference link-level outcomes (build container only):

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden_linksim.py

For each case of tests/linksim_cases.py: the reference's own
`linksim.simulate_frames` (linksim.py:159-232: LDPC encode, modulation, DMRS,
receive grid, genie or LS CSI, detection, LLRs, rate-matched decoding) on a
seeded Rayleigh grid.  Writes the per-frame, per-stream decode flags to
tests/golden/linksim.npz."""

import sys
from fractions import Fraction
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
sys.path.insert(0, str(HERE.parent))
sys.path.insert(0, "/root/reference/pkg/src")
sys.dont_write_bytecode = True

from mpnlsim import channel, core, linksim            # noqa: E402  (reference)

import linksim_cases as lc                              # noqa: E402


def main():
    out = {}
    for case in lc.CASES:
        name, n, m, (q, rn, rd), rb, det, csi, p, snr, f = case
        mcs = next(e for e in core.MCS_TABLE
                   if e.modulation_order == q and e.code_rate == Fraction(rn, rd))
        cfg = linksim.LinkConfig(n_streams=n, m_antennas=m, mcs=mcs, detector=det, n_paths=p,
                                 rb_per_vehicle=rb, csi=csi)
        ok = linksim.simulate_frames(cfg, channel.ChannelGrid(h=lc.channel(case)),
                                     lc.noise_var(case), 3, range(f))
        out[name] = ok
        print(name, ok.mean(), ok.shape)
    # measure_per over two channels with the early stop armed (linksim.py:241-271)
    case = lc.CASES[0]
    name, n, m, (q, rn, rd), rb, det, csi, p, snr, f = case
    mcs = next(e for e in core.MCS_TABLE
               if e.modulation_order == q and e.code_rate == Fraction(rn, rd))
    cfg = linksim.LinkConfig(n_streams=n, m_antennas=m, mcs=mcs, detector=det, n_paths=p,
                             rb_per_vehicle=rb, csi=csi)
    grids = [channel.ChannelGrid(h=lc.channel(case)),
             channel.ChannelGrid(h=np.ascontiguousarray(lc.channel(case)[:, ::-1]))]
    nvs = [lc.noise_var(case), 0.8 * lc.noise_var(case)]
    r = linksim.measure_per(cfg, grids, nvs, frames_per_channel=60)
    r2 = linksim.measure_per(cfg, grids, nvs, frames_per_channel=200, stop_threshold=0.9,
                             min_frames=100)
    out["measure_per"] = np.array([r.frames, r.errors, r2.frames, r2.errors])
    print("measure_per", out["measure_per"])
    np.savez_compressed(HERE / "linksim.npz", **out)


if __name__ == "__main__":
    main()
