"""Host-side logic of the B200 package (no GPU): tree utilities, tolerance rule,
schedule statistics, placement, and the no-CPU-fallback guarantee."""

import math

import numpy as np
import pytest

import paper_1607_05210_b200 as H
from paper_1607_05210_b200 import distributed as DI
from oracle import hapod_oracle as O


def test_balanced_trees_match_golden(golden):
    meta, _ = golden
    t = H.build_balanced(20, 2)
    assert [list(c) for c in t.children] == meta["readme/tree"]


@pytest.mark.parametrize("k", [1, 2, 5, 16, 64])
def test_star_and_chain_match_oracle(k):
    t = H.build_star(k)
    ch, root = O.star(k)
    assert [list(c) for c in t.children] == [list(c) for c in ch] and t.root == root
    t = H.build_chain(k)
    ch, root = O.chain(k)
    assert [list(c) for c in t.children] == [list(c) for c in ch]
    maps = H.derive_maps(t)
    assert list(maps.leaf_order) == O.leaf_order(ch, root)
    assert maps.depth == O.levels(ch, root)[root] == k


def test_tolerances_match_oracle_and_frozen(golden):
    meta, _ = golden
    t = H.build_star(4)
    tol = H.assign_tolerances(t, {1: 4, 2: 4, 3: 4, 4: 4}, 0.5, omega=0.75)
    assert tol.epsilons == pytest.approx(meta["tol/star"], rel=1e-15)
    assert tol.epsilons[0] == 0.75 * 4 * 0.5
    t = H.build_chain(5)
    counts = {v: 3 for v in H.derive_maps(t).leaves}
    tol = H.assign_tolerances(t, counts, 0.2, omega=0.6, zero_leaf_tolerance=True)
    assert tol.epsilons == pytest.approx(meta["tol/chain"], rel=1e-15)
    bound = H.error_bound(t, tol)
    assert bound == pytest.approx(O.error_bound([list(c) for c in t.children], 0, list(tol.epsilons)), rel=1e-15)
    with pytest.raises(ValueError):
        H.assign_tolerances(H.RootedTree(((),), 0), {0: 3}, 0.1, omega=0.5)
    with pytest.raises(ValueError):
        H.ToleranceAssignment((-1.0,))


def test_eps_star_mapping():
    # target = eps* / sqrt(|S|) makes the a-priori bound equal eps*
    t = H.build_star(16)
    counts = {v: 512 for v in range(1, 17)}
    eps_star = 1.3355e-5
    tol = H.assign_tolerances(t, counts, H.eps_star_to_target(eps_star, 8192), omega=0.75)
    assert H.error_bound(t, tol) == pytest.approx(eps_star, rel=1e-12)


def test_truncation_rank_frozen(golden):
    meta, _ = golden
    for s, e, n in meta["truncation"]:
        assert H.truncation_rank(np.array(s), e) == n
    with pytest.raises(ValueError):
        H.truncation_rank(np.array([1.0, 2.0]), 0.5)


def test_tree_text_roundtrip_and_validation():
    t = H.build_balanced(11, 3)
    assert H.parse_tree_text(H.format_tree_text(t)).children == t.children
    assert H.validate(H.RootedTree(((1,), (0,)), 0)) is not None
    assert "not reachable" in H.validate(H.RootedTree(((), ()), 0))
    with pytest.raises(ValueError):
        H.derive_maps(H.RootedTree(((1,), (0,)), 0))


def test_plan_and_stats():
    t = H.build_balanced(9, 2)
    sched = H.plan(t)
    maps = H.derive_maps(t)
    assert len(sched.waves) == maps.depth
    reps = [H.NodeReport(v, maps.level[v], not t.children[v], 1, 1, 0.1, 2, 0.0, 0.01 * (v + 1))
            for v in range(t.node_count)]
    assert H.critical_path_time(reps) == pytest.approx(
        sum(max(r.wall_time for r in reps if r.level == lv) for lv in set(maps.level)))
    assert H.peak_resident_modes(t, reps) >= 2


@pytest.mark.parametrize("world", [1, 2, 3, 8])
def test_placement(world):
    t = H.build_star(16)
    place = DI.plan_placement(t, world)
    assert place[0] == 0
    leaves = H.derive_maps(t).leaf_order
    per = [sum(1 for l in leaves if place[l] == r) for r in range(world)]
    assert max(per) - min(per) <= 1 and sum(per) == 16
    ch = H.build_chain(6)
    pl = DI.plan_placement(ch, world)
    assert all(pl[v] == pl[ch.children[v][0]] for v in range(ch.node_count) if ch.children[v])


def test_no_cpu_fallback_without_device():
    torch = pytest.importorskip("torch")
    if torch.cuda.is_available():
        pytest.skip("a CUDA device is present")
    with pytest.raises(RuntimeError, match="no CPU fallback"):
        H.SnapshotBlock(H.InnerProductSpace(3), np.eye(3))


def test_backend_validation():
    with pytest.raises(ValueError):
        H.PodBackend("qr")
    with pytest.raises(ValueError):
        H.PodBackend("gram", gram_eig_cutoff_factor=0.0)
    assert H.PodBackend() == H.PodBackend("gram", H.DEFAULT_GRAM_CUTOFF)
    with pytest.raises(ValueError):
        H.InnerProductSpace(3, np.array([1.0, 0.0, 2.0]))
    with pytest.raises(ValueError):
        H.InnerProductSpace(3, np.ones(4))
