"""Slot I/O around the detector (linksim.py:117-137, 200-226).

CPU: the numpy oracle restatement reproduces the reference's own outputs
(sha256 in tests/golden/slot.json, made by make_golden_slot.py).
GPU: the CUDA kernels (through the C ABI) — the DMRS LS estimate, the receive
grid (numpy's einsum summation order restated) and the data-RE gather all
bit-identical to the reference."""

import json
from pathlib import Path

import numpy as np
import pytest

import slot_cases as sc
from oracle import slot_oracle as so

GOLD = json.loads((Path(__file__).resolve().parent / "golden" / "slot.json").read_text())


@pytest.mark.parametrize("case", sc.CASES, ids=[c[0] for c in sc.CASES])
def test_oracle_matches_reference(case):
    name, n, m, rb, f, unit = case
    obs, pilots, h, x, noise = sc.inputs(case)
    est = so.estimate_channel_ls(obs, pilots, sc.SYMBOLS, sc.DMRS_SYMBOLS, 12 * rb, m, n)
    assert sc.digest(est) == GOLD[name]["est"]
    ds = GOLD[name]["data_syms"]
    hf, _ = so.data_re_batch(h, np.zeros((1,) + h.shape[:3]), ds)
    assert sc.digest(hf) == GOLD[name]["h_flat"]
    assert sc.digest(so.receive_grid(h, x, noise)) == GOLD[name]["y"]


def test_dmrs_pattern_like_reference():
    from paper_2409_14355_b200 import linksim as L

    class Num:
        dmrs_symbols, symbols_per_slot = 2, 14
    syms, ports = L.dmrs_pattern(Num, 12, 24)
    assert syms == (3, 12)
    allsc = [set(p[1].tolist()) for p in ports if p[0] == 3]
    assert all(not (a & b) for i, a in enumerate(allsc) for b in allsc[i + 1:])
    with pytest.raises(ValueError):
        L.dmrs_pattern(Num, 13, 24)
    assert L.data_symbols(Num, 4, 24) == [0, 1, 2, 4, 5, 6, 7, 8, 9, 10, 11, 13]


@pytest.mark.gpu
@pytest.mark.parametrize("case", sc.CASES, ids=[c[0] for c in sc.CASES])
def test_gpu_slot_io_matches_reference(case):
    import torch
    from paper_2409_14355_b200 import linksim as L
    name, n, m, rb, f, unit = case
    obs, pilots, h, x, noise = sc.inputs(case)

    class Num:
        dmrs_symbols, symbols_per_slot = sc.DMRS_SYMBOLS, sc.SYMBOLS

    class Cfg:
        numerology, n_subcarriers, m_antennas, n_streams = Num, 12 * rb, m, n
    est = L.estimate_channel_ls(obs, pilots, Cfg)
    assert sc.digest(est) == GOLD[name]["est"], "LS estimate not bit-identical"
    y = L.receive_grid(h, x, noise)
    assert sc.digest(y) == GOLD[name]["y"], "receive grid not bit-identical"
    ds = L.data_symbols(Num, n, 12 * rb)
    assert ds == GOLD[name]["data_syms"]
    hf, yf = L.data_re_batch(h, y, ds)
    assert sc.digest(hf) == GOLD[name]["h_flat"]
    assert np.array_equal(yf, y[:, ds].reshape(f, len(ds) * 12 * rb, m))
    # device tensors stay on the device
    ht, yt = L.data_re_batch(torch.from_numpy(h).cuda(), torch.from_numpy(y).cuda(), ds)
    assert ht.is_cuda and np.array_equal(ht.cpu().numpy(), hf)
