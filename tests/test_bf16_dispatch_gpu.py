"""Per-batch precision dispatch for dtype = CX_BF16 (north_star: tensor cores
only where the levels are dense GEMMs). Batches small enough for the cluster
kernel run it on FMA with bf16-rounded operands (weights, input rows, gathered
child states; fp32 products and sums, reading Q18) -- also fused with the
linearizer -- larger batches the tcgen05 kernel. Both within the bf16
tolerance of the fp64 oracle; the rounding is really applied (results differ
from fp32)."""
import numpy as np
import pytest
import torch

import oracle
import synth
from gpu_helpers import dev_f32, dev_i32, normwise_rel_err, weights_dev

pytestmark = pytest.mark.gpu
T = synth
TOL_BF16 = 2e-2


@pytest.fixture(scope="module")
def cx():
    import paper_2011_01383_b200 as m
    return m


@pytest.mark.parametrize("name", ["cfg2_treelstm_b10", "cfg2_treelstm_b1", "cfg5_dagrnn_b10",
                                  "f4_lstm_seq100_b10"])
@pytest.mark.parametrize("fused", [False, True])
def test_small_bf16_on_cluster_fma(cx, name, fused, monkeypatch):
    monkeypatch.delenv("CX_FORWARD_PATH", raising=False)
    w = synth.workload(name)
    cell, H, V, ch, kind = w["cell"], w["hidden"], w["vocab"], w["children"], w["kind"]
    assert cx.forward_family(cell, H, ch.shape[1], ch.shape[0], V, cx.BF16) == "cluster"
    words = synth.word_ids(ch, V, w["seed"], all_nodes=(cell == T.DAGRNN))
    emb = synth.embedding(V, H, w["seed"])
    ws_np, wd = weights_dev(cell, H, V)
    R = oracle.linearize(ch, kind)["num_roots"]
    if fused:
        assert cx.fused_applies(cell, H, ch.shape[1], ch.shape[0], V, cx.BF16)
        lin, h, _, roots = cx.linearize_forward(dev_i32(ch), kind, cell, H, wd, dev_f32(emb),
                                                dev_i32(words), dtype=cx.BF16, num_roots=R)
    else:
        lin = cx.linearize(dev_i32(ch), kind)
        h, _, roots = cx.forward(cell, H, wd, dev_f32(emb), dev_i32(words), lin, dtype=cx.BF16,
                                 num_roots=R)
    assert cx.status(lin) == (0, -1)
    lin32 = cx.linearize(dev_i32(ch), kind)
    h32, _, _ = cx.forward(cell, H, wd, dev_f32(emb), dev_i32(words), lin32)
    st, _, rh, _ = oracle.forward(cell, H, V, ws_np, emb, words, ch)
    e = normwise_rel_err(h.cpu().numpy(), rh)
    assert e <= TOL_BF16, e
    e32 = normwise_rel_err(h32.cpu().numpy(), rh)
    assert e32 <= 1e-4
    assert e > 10 * e32, "bf16 operand rounding not applied?"
    ref_lin = oracle.linearize(ch, kind)
    assert np.array_equal(roots.cpu().numpy(), h.cpu().numpy()[ref_lin["perm"][ref_lin["roots"]]])


def test_large_bf16_on_tensor_cores(cx, monkeypatch):
    monkeypatch.delenv("CX_FORWARD_PATH", raising=False)
    w = synth.workload("cfg5_treelstm_b4096")
    ch = w["children"]
    assert cx.forward_family(w["cell"], w["hidden"], ch.shape[1], ch.shape[0], w["vocab"],
                             cx.BF16) == "tc"
    assert not cx.fused_applies(w["cell"], w["hidden"], ch.shape[1], ch.shape[0], w["vocab"],
                                cx.BF16)


def test_bf16_treelstm_dag(cx, monkeypatch):
    """A TreeLSTM DAG linearization in bf16: the cluster route handles shared
    children; the tensor-core kernel refuses it (CX_E_UNSUPPORTED)."""
    ch = synth.random_dag(120, 2, 11, p_edge=0.6)
    H, V = 64, 40
    words = synth.word_ids(ch, V, 1)
    emb = synth.embedding(V, H, 1)
    ws_np, wd = weights_dev(T.TREELSTM, H, V)
    monkeypatch.delenv("CX_FORWARD_PATH", raising=False)
    lin = cx.linearize(dev_i32(ch), T.DAG)
    h, _, _ = cx.forward(T.TREELSTM, H, wd, dev_f32(emb), dev_i32(words), lin, dtype=cx.BF16)
    st, _, rh, _ = oracle.forward(T.TREELSTM, H, V, ws_np, emb, words, ch)
    assert normwise_rel_err(h.cpu().numpy(), rh) <= TOL_BF16
    monkeypatch.setenv("CX_FORWARD_PATH", "tc")
    with pytest.raises(cx.CxError) as ei:
        cx.forward(T.TREELSTM, H, wd, dev_f32(emb), dev_i32(words), lin, dtype=cx.BF16)
    assert ei.value.code == 8


@pytest.mark.parametrize("name,family", [("cfg3_treefc_b1", "rw"), ("cfg3_treefc_b10", "tc")])
def test_bf16_treefc_dispatch(cx, name, family, monkeypatch):
    """bf16 TreeFC: small batches on the register-weight FMA kernel with rounded
    operands, larger ones on the tensor cores; both within the bf16 tolerance."""
    monkeypatch.delenv("CX_FORWARD_PATH", raising=False)
    w = synth.workload(name)
    cell, H, V, ch, kind = w["cell"], w["hidden"], w["vocab"], w["children"], w["kind"]
    assert cx.forward_family(cell, H, ch.shape[1], ch.shape[0], V, cx.BF16) == family
    words = synth.word_ids(ch, V, w["seed"])
    emb = synth.embedding(V, H, w["seed"])
    ws_np, wd = weights_dev(cell, H, V)
    lin = cx.linearize(dev_i32(ch), kind)
    h, _, _ = cx.forward(cell, H, wd, dev_f32(emb), dev_i32(words), lin, dtype=cx.BF16)
    h32, _, _ = cx.forward(cell, H, wd, dev_f32(emb), dev_i32(words), lin)
    st, _, rh, _ = oracle.forward(cell, H, V, ws_np, emb, words, ch)
    e, e32 = normwise_rel_err(h.cpu().numpy(), rh), normwise_rel_err(h32.cpu().numpy(), rh)
    assert e <= TOL_BF16 and e32 <= 1e-4 and e > 10 * e32, (e, e32)
