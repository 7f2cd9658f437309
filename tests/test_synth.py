"""The shared input generators: determinism, ranges, structure (CPU only)."""
import dataclasses

import numpy as np

import synth


def test_graph_deterministic_and_ranged():
    spec = dataclasses.replace(synth.C1, n=64)
    A = synth.graph(spec)
    B = synth.graph(spec)
    assert np.array_equal(A, B)
    off = A[~np.eye(64, dtype=bool)]
    assert off.min() >= 1 and off.max() <= 100
    assert np.all(np.diag(A) == 0)
    C = synth.graph(dataclasses.replace(spec, seed=2))
    assert not np.array_equal(A, C)


def test_graph_ld_padding_matches():
    spec = dataclasses.replace(synth.C3, n=50)
    A = synth.graph(spec)
    B = synth.graph(spec, ld=64)
    assert np.array_equal(A, B[:, :50])


def test_density_and_inf():
    spec = dataclasses.replace(synth.C3, n=300)
    W = synth.graph(spec)
    off = ~np.eye(300, dtype=bool)
    frac = np.mean(W[off] == synth.INF_I32)
    assert 0.07 < frac < 0.13
    fin = W[off & (W != synth.INF_I32)]
    assert fin.min() >= 1 and fin.max() <= 1000


def test_undirected_f32_grid_symmetric_exact():
    spec = dataclasses.replace(synth.C2, n=80)
    W = synth.graph(spec)
    assert W.dtype == np.float32
    assert np.array_equal(W, W.T)
    off = W[~np.eye(80, dtype=bool)].astype(np.float64)
    m = off * 2 ** 24
    assert np.all(m == np.round(m)) and off.min() > 0 and off.max() <= 1.0


def test_loguniform():
    spec = dataclasses.replace(synth.C5, n=200)
    W = synth.graph(spec)
    off = W[~np.eye(200, dtype=bool)]
    assert off.min() >= 1 and off.max() <= 1_000_000
    # log-uniform: roughly half the mass below sqrt(1e6)
    assert 0.4 < np.mean(off < 1000) < 0.6


def test_update_sequence_bookkeeping():
    spec = dataclasses.replace(synth.C4, n=40)
    W = synth.graph(spec)
    hg = synth.HostGraph(W, True, cap=60)
    seq = synth.update_sequence(spec, hg, 0, 12)
    assert [u.kind for u in seq] == ["add", "remove", "reweight"] * 4
    assert hg.n == 40 + 4 - 4
    hg2 = synth.HostGraph(W, True, cap=60)
    seq2 = synth.update_sequence(spec, hg2, 0, 12)
    assert np.array_equal(hg.W, hg2.W)
    for up in seq:
        if up.kind == "reweight":
            assert up.w_new >= 1 and up.u != up.v


def test_swap_with_last():
    W = np.arange(16, dtype=np.int32).reshape(4, 4)
    np.fill_diagonal(W, 0)
    hg = synth.HostGraph(W, True, cap=4)
    assert hg.remove_node(1) == 3
    exp = W[np.ix_([0, 3, 2], [0, 3, 2])]
    assert np.array_equal(hg.W, exp)
