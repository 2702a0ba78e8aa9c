"""Host planning parity with the reference's topology.py (golden trees.json)."""

import json
from pathlib import Path

import numpy as np
import pytest

from paper_1711_00705_b200.errors import DisjointnessViolation, InvalidConfig
from paper_1711_00705_b200.topology import (
    build_multicolor_trees,
    build_ring,
    fold_tables,
    make_chunk_plan,
    ring_fold_tables,
    star_fold_tables,
    tree_set_to_dict,
    validate_tree_set,
)

GOLD = json.loads((Path(__file__).parent / "golden" / "trees.json").read_text())


@pytest.mark.parametrize("key", sorted(GOLD))
def test_tree_sets_match_reference(key):
    n, k, arity = (int(x) for x in key.split(","))
    want = GOLD[key]
    if "error" in want:
        exc = {"InvalidConfig": InvalidConfig, "DisjointnessViolation": DisjointnessViolation}
        with pytest.raises(exc[want["error"]]):
            build_multicolor_trees(n, k, arity)
        return
    ts = build_multicolor_trees(n, k, arity).with_plan(1000)
    assert tree_set_to_dict(ts) == want
    assert validate_tree_set(ts).ok


def test_fig2_structure():
    ts = build_multicolor_trees(8, 4, 4)
    for c, tree in enumerate(ts.trees):
        assert tree.root == 2 * c
        assert tree.interior == {2 * c, (2 * c + 1) % 8}
        assert len(tree.children[tree.root]) == 4
        assert len(tree.children[(2 * c + 1) % 8]) == 3


@pytest.mark.parametrize("n,k", [(0, 1), (10, 3), (25_600_002, 4), (7, 8), (1, 1)])
def test_chunk_plan(n, k):
    plan = make_chunk_plan(n, k)
    assert sum(c.length for c in plan.chunks) == n
    assert [c.start for c in plan.chunks] == list(np.cumsum([0] + [c.length for c in plan.chunks])[:-1])
    assert max(c.length for c in plan.chunks) - min(c.length for c in plan.chunks) <= 1


def test_invalid_parameters():
    with pytest.raises(InvalidConfig):
        build_multicolor_trees(1, 1, 4)
    with pytest.raises(InvalidConfig):
        build_multicolor_trees(2, 4, 4)
    with pytest.raises(InvalidConfig):
        build_multicolor_trees(8, 0, 4)
    with pytest.raises(DisjointnessViolation):
        build_multicolor_trees(4, 4, 1)
    with pytest.raises(InvalidConfig):
        build_ring(4, root=4)
    with pytest.raises(InvalidConfig):
        make_chunk_plan(-1, 2)


def test_fold_tables_agree_with_oracle(oracle):
    for n, k, a in [(8, 4, 4), (8, 8, 7), (4, 2, 4), (16, 4, 4), (2, 1, 4)]:
        t = fold_tables(build_multicolor_trees(n, k, a))
        o = oracle.tables_from_trees(n, oracle.trees(n, k, a))
        assert np.array_equal(t.parent, o[0]) and np.array_equal(t.child_ptr, o[1])
        assert np.array_equal(t.child_idx, o[2]) and np.array_equal(t.self_pos, o[3])
    r = ring_fold_tables(build_ring(5))
    o = oracle.ring_tables(list(range(5)))
    assert np.array_equal(r.parent, o[0]) and np.array_equal(r.child_idx, o[2])
    s = star_fold_tables(4, 2)
    o = oracle.star_tables(4, 2)
    assert np.array_equal(s.self_pos, o[3]) and np.array_equal(s.child_idx, o[2])


def test_fold_tables_reproduce_reference_bits(golden, oracle):
    """Planner output fed to the oracle fold gives the reference's bits."""
    inp = golden["mc_8_997_4_4_in"]
    t = fold_tables(build_multicolor_trees(8, 4, 4))
    got = oracle.fold_c((t.parent, t.child_ptr, t.child_idx, t.self_pos), list(inp))
    assert np.array_equal(got, golden["mc_8_997_4_4_out"])
