"""The seeded input generator (synth/): determinism, logical-index keying
(layout/ld independence), panel keying and the value sets of DESIGN.md
readings A2/A3."""
import numpy as np
import pytest

import synth


def test_deterministic_and_seed_sensitive():
    a = synth.matrix(40, 30, seed=3, matrix_id=0)
    assert np.array_equal(a, synth.matrix(40, 30, seed=3, matrix_id=0))
    assert not np.array_equal(a, synth.matrix(40, 30, seed=4, matrix_id=0))
    assert not np.array_equal(a, synth.matrix(40, 30, seed=3, matrix_id=1))


def test_logical_index_keying_panels():
    full = synth.matrix(300, 70, seed=1, matrix_id=0, block_rows=64)
    panel = synth.matrix(100, 70, seed=1, matrix_id=0, row0=150)
    assert np.array_equal(panel, full[150:250])
    sub = synth.matrix(30, 20, seed=1, matrix_id=0, row0=10, col0=40)
    assert np.array_equal(sub, full[10:40, 40:60])


@pytest.mark.parametrize("layout", [synth.ROW_MAJOR, synth.COL_MAJOR])
@pytest.mark.parametrize("pad", [0, 1, 4])
def test_store_roundtrip_and_padding(layout, pad):
    x = synth.matrix(7, 5, seed=2)
    buf, ld = synth.store(x, layout, synth.min_ld(7, 5, layout) + pad)
    assert np.array_equal(synth.load_logical(buf, 7, 5, layout, ld), x)
    lines = 7 if layout == synth.ROW_MAJOR else 5
    inner = 5 if layout == synth.ROW_MAJOR else 7
    assert buf.size == (lines - 1) * ld + inner
    if pad:
        assert np.isnan(buf.reshape(-1)[inner:ld]).all()
    with pytest.raises(ValueError):
        synth.store(x, layout, inner - 1)


def test_value_sets():
    u = synth.matrix(256, 256, seed=0, dist="uniform").astype(np.float64)
    assert u.min() >= -1.0 and u.max() < 1.0 and u.min() < -0.99 and u.max() > 0.99
    assert np.all(u * 2 ** 23 == np.round(u * 2 ** 23))           # 2^-23 grid
    assert abs(u.mean()) < 0.01
    p = synth.matrix(256, 256, seed=0, dist="uniform01").astype(np.float64)
    assert p.min() >= 0.0 and p.max() < 1.0 and abs(p.mean() - 0.5) < 0.01
    i = synth.matrix(256, 256, seed=0, dist="int")
    assert set(np.unique(i).tolist()) == set(range(-8, 9))
    w = synth.matrix(256, 256, seed=0, dist="wide").astype(np.float64)
    e = np.floor(np.log2(np.abs(w)))
    assert e.min() == -20 and e.max() == 20 and (w < 0).any() and (w > 0).any()


def test_permutation_matrix():
    P, perm = synth.permutation(50, seed=1)
    assert sorted(perm.tolist()) == list(range(50))
    assert np.array_equal(P.sum(0), np.ones(50)) and np.array_equal(P.sum(1), np.ones(50))
