"""The reference's host-side decomposition API (mpcdsim/decomposition.py)
against golden outputs of the reference itself (tests/golden/decomposition.npz),
and its agreement with the engine's own DomainLayout numbering."""

import numpy as np
import pytest

import paper_2212_11878_b200 as mp
from paper_2212_11878_b200 import decomposition as dec
from paper_2212_11878_b200.distributed import DomainLayout

CASES = [(8, 1.0, (2, 2, 2)), (12, 0.5, (3, 2, 1)), (6, 2.0, (1, 3, 2)), (4, 1.0, (1, 1, 1))]


@pytest.fixture(scope="module")
def g_dec():
    from conftest import golden
    return golden("decomposition.npz")


@pytest.mark.parametrize("i", range(len(CASES)))
def test_grid_matches_reference(g_dec, i):
    L, a, rd = CASES[i]
    g = mp.build_decomposition(L, a, rd)
    assert np.array_equal(g.own_cells, g_dec[f"c{i}_own"])
    assert np.array_equal(g.neighbor_table, g_dec[f"c{i}_table"])
    for r in range(g.n_ranks):
        assert np.array_equal(g.dom_borders(r), g_dec[f"c{i}_borders"][r])
        assert np.array_equal(g.rank_coords(r), g_dec[f"c{i}_coords"][r])
        assert g.rank_of_coords(g.rank_coords(r)) == r
        assert np.array_equal(dec.classify_base3(g_dec[f"c{i}_pos"], g.dom_borders(r)),
                              g_dec[f"c{i}_codes"][r])
    assert np.array_equal(g.global_flat_cells(g_dec[f"c{i}_gc"]), g_dec[f"c{i}_flat"])
    # the engine's layout numbers ranks and blocks the same way
    lay = DomainLayout((L, L, L), rd)
    for r in range(g.n_ranks):
        assert lay.coords(r) == tuple(int(x) for x in g.rank_coords(r))
        assert lay.origin(r) == tuple(int(x) for x in g.own_cell_lo(r))


def test_codes_and_neighbours(g_dec):
    assert np.array_equal(mp.code_digits(np.arange(27)), g_dec["digits"])
    assert [mp.reflect_code(c) for c in range(27)] == list(g_dec["reflect"])
    g = mp.build_decomposition(8, 1.0, (2, 2, 2))
    assert mp.CODE_STAY == 13 and mp.neighbor_rank(mp.CODE_STAY, g, 5) == 5
    assert mp.classify_base3(np.array([1.0, 1.0, 1.0]), g.dom_borders(0)) == mp.CODE_STAY
    with pytest.raises(mp.ConfigError):
        mp.neighbor_rank(27, g, 0)


@pytest.mark.parametrize("args", [(0, 1.0, (1, 1, 1)), (8, 0.0, (1, 1, 1)), (8, 1.0, (3, 1, 1)),
                                  (8, 1.0, (0, 1, 1)), (8, 1.0, (2, 2))])
def test_invalid_grids_raise(args):
    with pytest.raises(mp.ConfigError):
        mp.build_decomposition(*args)
