"""Generate tests/golden/fec.npz from the REFERENCE's LDPC stage (build
container only):

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden_fec.py

Imports `mpnlsim.fec` (fec.py) from /root/reference/pkg/src, never copies it.
For every case of tests/fec_cases.py: payload bits -> `ldpc_encode` (or
`design_rate_match` + `encode_rate_matched`) -> seeded channel LLRs ->
`ldpc_decode` (or `decode_rate_matched`).  Stores the encoded words, the
decoded bits and converged flags (packed), and the sha256 of the LLRs.
"""

from __future__ import annotations

import sys
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
sys.path.insert(0, str(HERE.parent))
sys.path.insert(0, "/root/reference/pkg/src")
sys.dont_write_bytecode = True

from mpnlsim import fec                       # noqa: E402  (reference)

import fec_cases as fc                        # noqa: E402


def main():
    code = fec.default_code()
    out = {"H": np.packbits(code.parity_check, axis=1),
           "E": np.packbits(code._encoder, axis=1)}
    for name, (words, seed, kind, param, max_iter, rm) in fc.CASES.items():
        if rm is None:
            info = fc.payload(name, code.k)
            tx = fec.ldpc_encode(code, info)
            llr = fc.channel_llrs(name, tx)
            dec, conv = fec.ldpc_decode(code, llr, max_iter=max_iter)
        else:
            r = fec.design_rate_match(code, rm[0], rm[1])
            info = fc.payload(name, r.k_tb)
            tx = fec.encode_rate_matched(code, r, info)
            llr = fc.channel_llrs(name, tx)
            dec, conv = fec.decode_rate_matched(code, r, llr, max_iter=max_iter)
            out[f"{name}_rm"] = np.array([r.k_tb, r.n_shortened, r.n_punctured])
        out[f"{name}_info"] = np.packbits(info, axis=1)
        out[f"{name}_tx"] = np.packbits(tx, axis=1)
        out[f"{name}_llr_sha"] = np.array(fc.digest(llr))
        out[f"{name}_dec"] = np.packbits(dec, axis=1)
        out[f"{name}_conv"] = conv.astype(np.uint8)
        print(f"{name}: {words} words, converged {int(conv.sum())}, "
              f"info errors {int(np.sum(dec != info))}")
    np.savez_compressed(HERE / "fec.npz", **out)


if __name__ == "__main__":
    main()
