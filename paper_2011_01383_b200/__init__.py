"""B200-native hot path of Cortex (arXiv 2011.01383): device linearization and
persistent level-by-level evaluation of recursive cells, behind the C ABI of
include/cx.h. See DESIGN.md.

    import paper_2011_01383_b200 as cx
    lin = cx.linearize(children_cuda_int32, cx.TREE)
    h, aux, roots = cx.forward(cx.TREELSTM, 256, weights, emb, words, lin, num_roots=10)
    # or both in one launch:
    lin, h, aux, roots = cx.linearize_forward(children, cx.TREE, cx.TREELSTM, 256, weights, emb, words)
"""
from .cx import (BF16, DAG, DAGRNN, F32, MVRNN, SEQUENCE, TREE, TREEFC, TREEGRU, TREELSTM,
                 TREERNN, SIMPLETREEGRU, CELL_IDS, CxError, Linearization, alloc_linearization, check, forward, launch_info, lib,
                 fused_applies, linearize, linearize_forward, LinearizeForwardPlan, status, status_str,
                 linearize_forward_launch_info, diag_sync_cycles, forward_family)
from . import cx as _cx

OK = _cx.OK

__all__ = ["linearize", "linearize_forward", "LinearizeForwardPlan", "fused_applies", "alloc_linearization", "forward", "check", "status", "status_str", "launch_info", "lib",
           "linearize_forward_launch_info", "diag_sync_cycles", "forward_family",
           "Linearization", "CxError", "SEQUENCE", "TREE", "DAG", "TREERNN", "TREEFC",
           "TREELSTM", "TREEGRU", "MVRNN", "DAGRNN", "SIMPLETREEGRU", "F32", "BF16", "CELL_IDS", "OK"]
