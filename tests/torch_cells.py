"""Library-routine evaluators used to pin the oracle's forward pass.

Each evaluator walks a structure recursively in Python and computes every
node with torch.nn cell modules (LSTMCell / GRUCell / RNNCell) or
torch.nn.functional.linear in float64, configured so that the library
routine computes exactly the cell reading of SURVEY.md §8(c) (Q1-Q3, Q8, Q9).
These are the "special cases that reduce to a textbook or library routine"
pins: they share no code with oracle/oracle.c.
"""
import numpy as np
import torch
import torch.nn.functional as F

BIG = 100.0  # sigmoid(100) == 1.0 exactly in float64 (1 + e^-100 rounds to 1)


def _t(a):
    return torch.as_tensor(np.asarray(a, dtype=np.float64))


def _order(children):
    """children-before-parent order by memoized DFS (any such order works, P.2)."""
    maxc, n = children.shape
    done, order = [False] * n, []
    for r in range(n):
        stack = [(r, 0)]
        while stack:
            v, k = stack.pop()
            if done[v]:
                continue
            if k < maxc and children[k, v] != -1:
                stack.append((v, k + 1))
                c = int(children[k, v])
                if not done[c]:
                    stack.append((c, 0))
                continue
            done[v] = True
            order.append(v)
    return order


def treelstm(weights, emb, words, children):
    """Child-sum TreeLSTM node = torch.nn.LSTMCell compositions:
    f_k * c_k = LSTMCell(0, (h_k, c_k)) with only the f rows of weight_hh
    (U_f) and bias b_f, and i/g/o biases 0 (so i*g = 0.5*tanh(0) = 0);
    then (h, c) = LSTMCell(x, (h~, sum_k f_k c_k)) with weight_ih =
    [W_i; 0; W_u; W_o], weight_hh = [U_i; 0; U_u; U_o], f bias BIG (f == 1)."""
    W_iou, U_iou, b_iou, U_f, b_f = [_t(w) for w in weights]
    H = U_f.shape[0]
    z = torch.zeros(H, H, dtype=torch.float64)
    Wi, Wo, Wu = W_iou[:H], W_iou[H:2 * H], W_iou[2 * H:]
    Ui, Uo, Uu = U_iou[:H], U_iou[H:2 * H], U_iou[2 * H:]
    bi, bo, bu = b_iou[:H], b_iou[H:2 * H], b_iou[2 * H:]
    main = torch.nn.LSTMCell(H, H, dtype=torch.float64)
    fk = torch.nn.LSTMCell(H, H, dtype=torch.float64)
    zb = torch.zeros(H, dtype=torch.float64)
    with torch.no_grad():
        main.weight_ih.copy_(torch.cat([Wi, z, Wu, Wo]))
        main.weight_hh.copy_(torch.cat([Ui, z, Uu, Uo]))
        main.bias_ih.copy_(torch.cat([bi, torch.full((H,), BIG, dtype=torch.float64), bu, bo]))
        main.bias_hh.zero_()
        fk.weight_ih.zero_()
        fk.weight_hh.copy_(torch.cat([z, U_f, z, z]))
        fk.bias_ih.copy_(torch.cat([zb, b_f, zb, zb]))
        fk.bias_hh.zero_()
    n = children.shape[1]
    h = [None] * n
    c = [None] * n
    E = _t(emb)
    with torch.no_grad():
        for v in _order(children):
            kids = [int(k) for k in children[:, v] if k != -1]
            if not kids:
                x = E[words[v]][None]
                hh, cc = main(x, (torch.zeros(1, H, dtype=torch.float64),
                                  torch.zeros(1, H, dtype=torch.float64)))
            else:
                x = torch.zeros(1, H, dtype=torch.float64)
                ht = sum(h[k] for k in kids)
                fc = sum(fk(x, (h[k], c[k]))[1] for k in kids)
                hh, cc = main(x, (ht, fc))
            h[v], c[v] = hh, cc
    return torch.cat(h).numpy(), torch.cat(c).numpy()


def treegru(weights, emb, words, children):
    """Child-sum TreeGRU node = torch.nn.GRUCell(x=s, h=h~) with weight_ih =
    [0; 0; U_h], weight_hh = [0; U_z; 0], bias_ih = [BIG; b_z; b_h]; s =
    sum_k sigmoid(linear(h_k, U_r, b_r)) * h_k. Leaves: GRUCell(x, 0) with
    weight_ih = [0; W_z; W_h]."""
    W_zh, U_z, U_r, U_h, b_z, b_r, b_h = [_t(w) for w in weights]
    H = U_z.shape[0]
    z = torch.zeros(H, H, dtype=torch.float64)
    big = torch.full((H,), BIG, dtype=torch.float64)
    inner = torch.nn.GRUCell(H, H, dtype=torch.float64)
    leaf = torch.nn.GRUCell(H, H, dtype=torch.float64)
    with torch.no_grad():
        inner.weight_ih.copy_(torch.cat([z, z, U_h]))
        inner.weight_hh.copy_(torch.cat([z, U_z, z]))
        inner.bias_ih.copy_(torch.cat([big, b_z, b_h]))
        inner.bias_hh.zero_()
        leaf.weight_ih.copy_(torch.cat([z, W_zh[:H], W_zh[H:]]))
        leaf.weight_hh.zero_()
        leaf.bias_ih.copy_(torch.cat([big, b_z, b_h]))
        leaf.bias_hh.zero_()
    n = children.shape[1]
    h = [None] * n
    E = _t(emb)
    with torch.no_grad():
        for v in _order(children):
            kids = [int(k) for k in children[:, v] if k != -1]
            if not kids:
                h[v] = leaf(E[words[v]][None], torch.zeros(1, H, dtype=torch.float64))
            else:
                ht = sum(h[k] for k in kids)
                s = sum(torch.sigmoid(F.linear(h[k], U_r, b_r)) * h[k] for k in kids)
                h[v] = inner(s, ht)
    return torch.cat(h).numpy()


def dagrnn(weights, emb, words, children):
    """DAG-RNN node = torch.nn.RNNCell(tanh)(x_n, sum of predecessor states)."""
    W_x, U, b = [_t(w) for w in weights]
    H = U.shape[0]
    cell = torch.nn.RNNCell(H, H, nonlinearity="tanh", dtype=torch.float64)
    with torch.no_grad():
        cell.weight_ih.copy_(W_x)
        cell.weight_hh.copy_(U)
        cell.bias_ih.copy_(b)
        cell.bias_hh.zero_()
    n = children.shape[1]
    h = [None] * n
    E = _t(emb)
    with torch.no_grad():
        for v in _order(children):
            kids = [int(k) for k in children[:, v] if k != -1]
            ht = sum(h[k] for k in kids) if kids else torch.zeros(1, H, dtype=torch.float64)
            h[v] = cell(E[words[v]][None], ht)
    return torch.cat(h).numpy()


def mvrnn(weights, emb, words, children):
    """MV-RNN [Socher 2012] with numpy matmul: a = tanh(W @ [B a; A b] + beta),
    A_n = W_M @ vstack(A, B)."""
    Mw, W, beta, W_M = [np.asarray(w, np.float64) for w in weights]
    n = children.shape[1]
    a, A = [None] * n, [None] * n
    E = np.asarray(emb, np.float64)
    for v in _order(children):
        kids = [int(k) for k in children[:, v] if k != -1]
        if not kids:
            a[v], A[v] = E[words[v]], Mw[words[v]]
        else:
            l, r = kids
            p = np.concatenate([A[r] @ a[l], A[l] @ a[r]])
            a[v] = np.tanh(W @ p + beta)
            A[v] = W_M @ np.vstack([A[l], A[r]])
    return np.stack(a), np.stack(A)
