"""NEXT-3 comparison schedules: MC (multicolouring of single rows,
PAPER.md:869-891) and ABMC (colouring of blocks of consecutive rows,
PAPER.md:948-969; contiguous blocks stand in for METIS parts).

CPU checks: the rows of one MC colour class have pairwise disjoint write sets
W(r) = {r} ∪ {c : a_rc stored in U'} (the distance-2 condition for upper
storage) in the final order, checked by brute force; ABMC
blocks of one colour are write-disjoint; both give a bijective permutation."""
import numpy as np
import pytest

import gen

P = pytest.importorskip("paper_1907_06487_b200")
from paper_1907_06487_b200._lib import check, lib  # noqa: E402


def permuted(s, U):
    rp = np.zeros(U.n + 1, dtype=np.int32)
    col = np.zeros(U.nnz, dtype=np.int32)
    val = np.zeros(U.nnz)
    check(lib().race_schedule_permuted_matrix(s._h, rp.ctypes.data, col.ctypes.data, val.ctypes.data))
    return rp, col, val


def write_sets(rp, col):
    n = len(rp) - 1
    return [set([r]) | set(col[rp[r]:rp[r + 1]].tolist()) for r in range(n)]


@pytest.mark.parametrize("name", ["lap2d_64", "st27_24", "spin_14"])
def test_mc_colour_classes_are_write_disjoint(name):
    U, _ = gen.make_config(name)
    s = P.build_schedule(U, scheme=1)
    perm, inv = s.permutation()
    assert np.array_equal(np.sort(perm), np.arange(U.n))
    assert np.array_equal(perm[inv], np.arange(U.n))
    rp, col, _ = permuted(s, U)
    ws = write_sets(rp, col)
    lp = s.table("level_ptr")  # colour class boundaries
    assert lp[0] == 0 and lp[-1] == U.n and len(lp) >= 3
    for c in range(len(lp) - 1):
        seen = set()
        for r in range(lp[c], lp[c + 1]):
            assert not (ws[r] & seen), f"colour {c} row {r} conflicts"
            seen |= ws[r]


@pytest.mark.parametrize("block", [8, 64])
def test_abmc_blocks_of_one_colour_are_write_disjoint(block):
    U, _ = gen.make_config("st27_24")
    s = P.build_schedule(U, scheme=2, abmc_block=block)
    rp, col, _ = permuted(s, U)
    ws = write_sets(rp, col)
    lp = s.table("level_ptr")
    # blocks keep their rows contiguous inside a colour class: walk the class in
    # chunks of `block` rows (a class holds whole blocks, the last one of the
    # matrix may be short) and check that different blocks never share a target
    for c in range(len(lp) - 1):
        owner = {}
        for r in range(lp[c], lp[c + 1]):
            b = (r - lp[c]) // block
            for t in ws[r]:
                assert owner.setdefault(t, b) == b, f"colour {c}: blocks {owner[t]} and {b} share {t}"


def test_mc_needs_more_colours_than_race_phases():
    """The paper's motivation: MC needs many colours (global
    barriers) where RACE's level groups need two stage-0 colours."""
    U, _ = gen.make_config("st27_24")
    mc = P.build_schedule(U, scheme=1).stats
    race = P.build_schedule(U).stats
    assert mc["total_levels"] >= 8        # colour classes of a 27-point stencil
    assert race["n_components"] == 1
