"""Generator regression anchors; they check the generator, not the method."""
import numpy as np

import synth


def test_sst_anchor_tree0():
    ch, off = synth.sst_shaped_forest(10, 0)
    assert ch[0, :12].tolist() == [1, 2, 3, 4, -1, 6, -1, -1, -1, 10, -1, 12]
    assert ch[1, :12].tolist() == [30, 9, 8, 5, -1, 7, -1, -1, -1, 11, -1, 23]
    assert ch.shape == (2, 390) and off.tolist()[:3] == [0, 39, 78]


def test_cfg1_words_anchor():
    w = synth.workload("cfg1_treernn")
    assert w["words"][w["words"] >= 0].tolist() == [90, 1, 6, 17, 95, 45, 16, 52]


def test_splitmix_vectorised_matches_scalar():
    a, b = synth.SplitMix64(4, 1000), synth.SplitMix64(4, 1000)
    v = a.next_array(1000)
    assert [int(x) for x in v] == [b.next() for _ in range(1000)]
    assert a.next() == b.next()


def test_sizes():
    assert synth.workload("cfg5_treelstm_b4096")["children"].shape == (2, 159744)
    assert synth.workload("cfg5_dagrnn_b4096")["children"].shape == (2, 409600)
    assert synth.workload("cfg3_treefc_b10")["children"].shape == (2, 2550)
