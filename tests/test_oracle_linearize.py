"""Pins for the oracle's linearization (SURVEY.md §8(c) "Linearization")."""
import itertools
import json
import os

import numpy as np
import pytest

import oracle
import synth
from lin_checks import check_invariants, longest_path_heights

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "worked_examples.json")))


def test_three_node_worked_example():
    g = GOLD["three_node_tree"]
    lin = oracle.linearize(np.array(g["children"]), synth.TREE)
    assert lin["status"] == 0
    assert lin["perm"].tolist() == g["perm"]
    assert lin["first_leaf"] == g["first_leaf"]
    assert lin["level_size"].tolist() == g["level_size"]
    assert lin["level_begin"].tolist() == g["level_begin"]
    check_invariants(np.array(g["children"]), lin)


def test_seven_node_worked_example():
    g = GOLD["seven_node_perfect_tree"]
    lin = oracle.linearize(np.array(g["children"]), synth.TREE)
    assert lin["first_leaf"] == g["first_leaf"]
    for i, h in g["height_of_new"].items():
        assert lin["height"][int(i)] == h
    # batch_of(5) is an error in SPEC: 5 is a leaf (one comparison)
    assert 5 >= lin["first_leaf"]


@pytest.mark.parametrize("k", [1, 2, 3, 5, 8])
def test_perfect_tree_closed_form(k):
    ch, _ = synth.perfect_forest(1, k - 1)  # 2^k - 1 nodes
    lin = oracle.linearize(ch, synth.TREE)
    assert lin["num_levels"] == k
    assert lin["level_size"].tolist() == [2 ** (k - 1 - l) for l in range(k)]
    if k == 8:
        g = GOLD["perfect_255_levels"]
        assert lin["num_levels"] == g["num_levels"]
        assert lin["level_size"].tolist() == g["level_size"]


@pytest.mark.parametrize("n", [1, 2, 3, 7, 10])
def test_grid_closed_form(n):
    ch, _ = synth.grid_dags(1, n, n)
    lin = oracle.linearize(ch, synth.DAG)
    assert lin["num_levels"] == 2 * n - 1
    assert lin["level_size"].tolist() == [min(d + 1, 2 * n - 1 - d) for d in range(2 * n - 1)]
    if n == 10:
        assert lin["num_levels"] == GOLD["grid_10x10_levels"]["num_levels"]
    check_invariants(ch, lin)


@pytest.mark.parametrize("m", [1, 2, 50, 3000])
def test_chain_closed_form(m):
    ch, _ = synth.chains(3, m)
    lin = oracle.linearize(ch, synth.SEQUENCE)
    assert lin["num_levels"] == m
    assert (lin["level_size"] == 3).all()


def test_sst_levels_match_survey():
    # regression anchors of the generator + linearizer
    w = synth.workload("cfg2_treelstm_b10")
    lin = oracle.linearize(w["children"], w["kind"])
    assert lin["level_size"].tolist() == [200, 68, 42, 25, 18, 13, 11, 8, 4, 1]
    check_invariants(w["children"], lin)


def test_brute_force_heights_and_minimality():
    """N <= 6: heights equal the longest path (path enumeration), and they are
    the pointwise-minimal labelling with label(child) < label(parent)."""
    for seed in range(60):
        n = 1 + seed % 6
        ch = synth.random_dag(n, 3, seed)
        lin = oracle.linearize(ch, synth.DAG)
        assert lin["status"] == 0
        h_in = lin["height"][lin["inv"]]  # height per input id
        assert np.array_equal(h_in, longest_path_heights(ch))
        if n <= 5:
            edges = [(v, int(c)) for v in range(n) for c in ch[:, v] if c != -1]
            for lab in itertools.product(range(n), repeat=n):
                if all(lab[c] < lab[v] for v, c in edges):
                    assert all(h_in[v] <= lab[v] for v in range(n))
        check_invariants(ch, lin)


def test_fuzz_invariants():
    """Random trees, forests, DAGs (<= 200 nodes, some with shuffled ids)."""
    for seed in range(300):
        n = 1 + (seed * 37) % 200
        if seed % 3 == 0:
            ch, kind = synth.random_dag(n, 1 + seed % 4, seed, p_edge=0.3), synth.DAG
        else:
            ch, kind = synth.random_forest(n, 1 + seed % 3, seed), synth.TREE
        if seed % 2:
            ch, _, _ = synth.shuffle_ids(ch, None, seed)
        lin = oracle.linearize(ch, kind)
        check_invariants(ch, lin)


def test_relabel_invariance():
    """Relabelling inputs by pi leaves level membership unchanged."""
    for seed in range(20):
        ch = synth.random_dag(60, 3, seed, p_edge=0.4)
        ch2, _, pi = synth.shuffle_ids(ch, None, seed)
        a = oracle.linearize(ch, synth.DAG)
        b = oracle.linearize(ch2, synth.DAG)
        ha = a["height"][a["inv"]]
        hb = b["height"][b["inv"]]
        assert np.array_equal(ha, hb[pi])
        assert a["level_size"].tolist() == b["level_size"].tolist()


def test_empty_and_single():
    lin = oracle.linearize(np.zeros((2, 0), np.int32), synth.TREE)
    assert lin["status"] == 0 and lin["num_levels"] == 0 and lin["num_roots"] == 0
    lin = oracle.linearize(np.full((2, 1), -1, np.int32), synth.TREE)
    assert lin["num_levels"] == 1 and lin["first_leaf"] == 0 and lin["roots"].tolist() == [0]


def _err(ch, kind):
    lin = oracle.linearize(np.array(ch, dtype=np.int32), kind)
    return lin["status"], lin["bad_node"]


def test_error_codes():
    T, D, S = synth.TREE, synth.DAG, synth.SEQUENCE
    # child id out of range
    assert _err([[1, 5, -1], [2, -1, -1]], T) == (oracle.E_CHILD_RANGE, 1)
    assert _err([[-7, -1]], S) == (oracle.E_CHILD_RANGE, 0)
    # a -1 before a present child
    assert _err([[-1, -1, -1], [1, -1, -1]], T) == (oracle.E_CHILD_LAYOUT, 0)
    # two parents in a tree
    assert _err([[2, 2, -1], [-1, -1, -1]], T) == (oracle.E_KIND, 2)
    # ... allowed in a DAG
    assert _err([[2, 2, -1], [-1, -1, -1]], D) == (oracle.OK, -1)
    # duplicate child within a node
    assert _err([[1, -1], [1, -1]], D) == (oracle.E_KIND, 0)
    # cycles: lowest id on or reaching a cycle
    assert _err([[1, 2, 1]], D) == (oracle.E_CYCLE, 0)
    assert _err([[-1, 2, 1]], D) == (oracle.E_CYCLE, 1)
    assert _err([[0]], D) == (oracle.E_CYCLE, 0)  # self edge
    # sequence needs max_children == 1
    assert _err([[1, -1], [-1, -1]], S)[0] == oracle.E_ARG
    # lowest (code, id) wins: range error at 2 beats layout error at 0
    assert _err([[-1, -1, 9], [1, -1, -1]], D) == (oracle.E_CHILD_RANGE, 2)
    # a2 is skipped when a1 failed: kind error hides a cycle
    assert _err([[1, 2, 1], [-1, -1, -1]], T) == (oracle.E_KIND, 1)
