"""CPU: the LDPC oracle restatement against the reference's own outputs
(tests/golden/fec.npz, made by tests/golden/make_golden_fec.py from
mpnlsim.fec), and the host-side C++ code construction (graph + GF(2)
encoder, no GPU) against the oracle."""

from fractions import Fraction
from pathlib import Path

import numpy as np
import pytest

import fec_cases as fc
from oracle import fec_oracle as fo
from paper_2409_14355_b200 import fec

GOLD = np.load(Path(__file__).resolve().parent / "golden" / "fec.npz")
H = np.unpackbits(GOLD["H"], axis=1)[:, :1296]
N, K = 1296, 648


def _case_io(name):
    words, seed, kind, param, max_iter, rm = fc.CASES[name]
    if rm is None:
        info = fc.payload(name, K)
        tx = fo.encode(H, info)
        return info, tx, fc.channel_llrs(name, tx), None
    k_tb, _, _ = fo.design_rate_match(N, K, rm[0], rm[1])
    info = fc.payload(name, k_tb)
    cw = fo.encode(H, np.concatenate([info, np.zeros((words, K - k_tb), np.uint8)], axis=1))
    tx = np.concatenate([cw[:, :k_tb], cw[:, K:K + rm[1] - k_tb]], axis=1)
    return info, tx, fc.channel_llrs(name, tx), k_tb


def test_default_code_matches_reference():
    assert np.array_equal(fec.expand_base_matrix(), H)
    assert np.array_equal(fo.expand_base_matrix(fec.BASE_MATRIX), H)


@pytest.mark.parametrize("name", list(fc.CASES))
def test_oracle_matches_reference_golden(name):
    info, tx, llr, k_tb = _case_io(name)
    max_iter = fc.CASES[name][4]
    assert np.array_equal(np.packbits(tx, axis=1), GOLD[f"{name}_tx"]), "encoder"
    assert fc.digest(llr) == str(GOLD[f"{name}_llr_sha"]), "regenerated LLRs drifted"
    full = llr if k_tb is None else fo.full_llrs(N, K, k_tb, llr)
    dec, conv = fo.decode(H, full, max_iter)
    kk = K if k_tb is None else k_tb
    assert np.array_equal(np.packbits(dec[:, :kk], axis=1), GOLD[f"{name}_dec"])
    assert np.array_equal(conv, GOLD[f"{name}_conv"].astype(bool))


def test_oracle_per_word_equals_batched():
    cv, ve = fo.graph(H)
    _, _, llr, _ = _case_io("awgn_2db")
    dec, conv = fo.decode(H, llr[:3], 10)
    for b in range(3):
        bits, ok, _ = fo.decode_one(cv, ve, llr[b], 10)
        assert np.array_equal(bits[:K], dec[b]) and ok == conv[b]


def test_numpy_sum_order_restatement():
    """np_sum_order reproduces numpy's float64 add-reduce bit for bit
    (sequential under 8 terms, 8-way pairwise blocks above)."""
    rng = np.random.default_rng(0)
    for d in (1, 2, 3, 5, 7, 8, 9, 15, 16, 17, 31):
        a = rng.standard_normal((2000, d)) * np.exp(rng.uniform(-30, 30, (2000, d)))
        assert np.array_equal(a.sum(axis=1), fo.np_sum_order([a[:, j] for j in range(d)]))


def test_host_build_matches_oracle():
    """C++ host port (mpnl_ldpc_build) of the graph and the encoder."""
    code = fec.LdpcCode(H)
    dc, dv, cv, ve, _ = code._tables()
    ocv, ove = fo.graph(H)
    assert (dc, dv) == (ocv.shape[1], ove.shape[1])
    assert np.array_equal(np.where(ocv >= 0, ocv, 0xFFFF).astype(np.uint16).ravel(), cv)
    assert np.array_equal(np.where(ove >= 0, ove, 0xFFFF).astype(np.uint16).ravel(), ve)
    assert np.array_equal(code._encoder, fo.parity_solver(H))


def test_singular_parity_part_raises():
    h = H.copy()
    h[:, N - 1] = 0
    with pytest.raises(ValueError, match="singular"):
        fec.LdpcCode(h)._tables()
    with pytest.raises(ValueError):
        fec.LdpcCode(np.zeros((4, 3), np.uint8))


def test_design_rate_match_reference_cases():
    code = fec.default_code()
    rm = fec.design_rate_match(code, Fraction(1, 2), code.n)
    assert (rm.n_shortened, rm.n_punctured, rm.method) == (0, 0, "none")
    rm = fec.design_rate_match(code, Fraction(120, 1024), 720)
    assert rm.k_tb == round(720 * 120 / 1024) and "shorten" in rm.method
    rm = fec.design_rate_match(code, Fraction(3, 4), 800)
    assert rm.k_tb == 600 and rm.n_punctured == (code.n - code.k) - 200
    assert rm.method.endswith("puncture")
    for args in ((Fraction(1, 2), 2 * code.n), (Fraction(999, 1000), 1000), (Fraction(3, 2), 100)):
        with pytest.raises(ValueError):
            fec.design_rate_match(code, *args)
    for name, (_, _, _, _, _, r) in fc.CASES.items():
        if r is not None:
            rm = fec.design_rate_match(code, *r)
            assert [rm.k_tb, rm.n_shortened, rm.n_punctured] == GOLD[f"{name}_rm"].tolist()


def test_alist_roundtrip(tmp_path):
    code = fec.default_code()
    p = tmp_path / "code.alist"
    fec.save_alist(code, p)
    assert np.array_equal(fec.load_alist(p).parity_check, code.parity_check)
