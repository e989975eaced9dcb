"""GPU: the LDPC kernels (through the C ABI) against the reference's own
outputs (tests/golden/fec.npz) and the CPU oracle on larger seeded batches.
Bar: bit-identical info bits, converged flags and (vs the oracle) iteration
counts; encoder / syndrome exact."""

from pathlib import Path

import numpy as np
import pytest

import fec_cases as fc
from oracle import fec_oracle as fo

GOLD = np.load(Path(__file__).resolve().parent / "golden" / "fec.npz")
H = np.unpackbits(GOLD["H"], axis=1)[:, :1296]
N, K = 1296, 648
pytestmark = pytest.mark.gpu


def _fec():
    from paper_2409_14355_b200 import fec
    return fec


@pytest.mark.parametrize("name", list(fc.CASES))
def test_decoder_matches_reference_golden(name):
    fec = _fec()
    code = fec.default_code()
    words, seed, kind, param, max_iter, rm = fc.CASES[name]
    if rm is None:
        info = fc.payload(name, K)
        tx = fec.ldpc_encode(code, info)
        assert np.array_equal(np.packbits(tx, axis=1), GOLD[f"{name}_tx"])
        llr = fc.channel_llrs(name, tx)
        dec, conv = fec.ldpc_decode(code, llr, max_iter=max_iter)
    else:
        r = fec.design_rate_match(code, *rm)
        info = fc.payload(name, r.k_tb)
        tx = fec.encode_rate_matched(code, r, info)
        assert np.array_equal(np.packbits(tx, axis=1), GOLD[f"{name}_tx"])
        llr = fc.channel_llrs(name, tx)
        dec, conv = fec.decode_rate_matched(code, r, llr, max_iter=max_iter)
    assert fc.digest(llr) == str(GOLD[f"{name}_llr_sha"])
    assert dec.dtype == np.uint8 and conv.dtype == bool
    assert np.array_equal(np.packbits(dec, axis=1), GOLD[f"{name}_dec"])
    assert np.array_equal(conv, GOLD[f"{name}_conv"].astype(bool))


@pytest.mark.parametrize("snr_db,words,max_iter", [(1.5, 256, 10), (2.25, 512, 10),
                                                   (3.0, 256, 20), (2.0, 128, 3)])
def test_decoder_vs_oracle_random(snr_db, words, max_iter):
    """Seeded AWGN batches: bits, flags and iteration counts equal the oracle's."""
    import torch
    fec = _fec()
    code = fec.default_code()
    rng = np.random.default_rng(int(snr_db * 100) + words)
    info = rng.integers(0, 2, (words, K)).astype(np.uint8)
    tx = fec.ldpc_encode(code, info)
    nv = 10 ** (-snr_db / 10)
    llr = 2 * ((1 - 2.0 * tx) + rng.normal(0, np.sqrt(nv), tx.shape)) / nv
    dec, conv, iters = fec.ldpc_decode(code, llr, max_iter=max_iter, return_iterations=True)
    odec, oconv = fo.decode(H, llr, max_iter)
    assert np.array_equal(dec, odec) and np.array_equal(conv, oconv)
    cv, ve = fo.graph(H)
    for b in range(0, words, max(1, words // 8)):
        _, _, it = fo.decode_one(cv, ve, llr[b], max_iter)
        assert iters[b] == it
    # device tensors in -> device results, identical
    d_dec, d_conv = fec.ldpc_decode(code, torch.from_numpy(llr).cuda(), max_iter=max_iter)
    assert np.array_equal(d_dec.cpu().numpy(), dec) and np.array_equal(d_conv.cpu().numpy(), conv)


def test_single_word_and_batch_agree():
    fec = _fec()
    code = fec.default_code()
    llr = fc.channel_llrs("awgn_2db", fec.ldpc_encode(code, fc.payload("awgn_2db", K)))
    bd, bc = fec.ldpc_decode(code, llr[:5])
    for i in range(5):
        sd, sc = fec.ldpc_decode(code, llr[i])
        assert np.array_equal(sd, bd[i]) and sc == bc[i] and isinstance(sc, bool)


def test_syndrome_and_noiseless_roundtrip():
    fec = _fec()
    code = fec.default_code()
    rng = np.random.default_rng(2)
    info = rng.integers(0, 2, (4, K)).astype(np.uint8)
    cw = fec.ldpc_encode(code, info)
    assert np.array_equal(cw[:, :K], info)
    assert not fec.ldpc_syndrome(code, cw).any()
    assert np.array_equal(fec.ldpc_syndrome(code, cw ^ 1) % 2, fo.syndrome(H, cw ^ 1))
    out, conv = fec.ldpc_decode(code, 8.0 * (1 - 2 * cw.astype(np.float64)))
    assert conv.all() and np.array_equal(out, info)


def test_errors_like_reference():
    fec = _fec()
    code = fec.default_code()
    with pytest.raises(ValueError, match="finite"):
        fec.ldpc_decode(code, np.full((2, N), np.inf))
    with pytest.raises(ValueError, match="codeword length"):
        fec.ldpc_decode(code, np.zeros((2, N - 1)))
    with pytest.raises(ValueError, match="info length"):
        fec.ldpc_encode(code, np.zeros(K + 1, np.uint8))
