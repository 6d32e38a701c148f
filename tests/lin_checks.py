"""Property checks on a linearization, independent of how it was produced.

Restates the invariants of PAPER.md App. B, §4.2
and the within-batch independence of App. A.4, as listed in
SURVEY.md §8(c) "What pins each part". Used on the oracle's output (CPU tests)
and on the CUDA linearizer's output (GPU tests).
"""
import numpy as np


def longest_path_heights(children):
    """Brute-force heights: enumerate every downward path (tiny inputs only)."""
    maxc, n = children.shape

    def paths_from(v):
        kids = [int(c) for c in children[:, v] if c != -1]
        if not kids:
            return 0
        return 1 + max(paths_from(c) for c in kids)

    return np.array([paths_from(v) for v in range(n)], dtype=np.int64)


def check_invariants(children, lin):
    """Assert every numbering/batching invariant; `lin` is the dict layout of
    oracle.linearize (perm, inv, children, height, level_begin, level_size,
    roots and header fields)."""
    children = np.asarray(children)
    maxc, n = children.shape
    perm = np.asarray(lin["perm"], dtype=np.int64)
    inv = np.asarray(lin["inv"], dtype=np.int64)
    L = lin["num_levels"]
    ls = np.asarray(lin["level_size"][:L], dtype=np.int64)
    lb = np.asarray(lin["level_begin"][:L], dtype=np.int64)
    hn = np.asarray(lin["height"], dtype=np.int64)
    chn = np.asarray(lin["children"], dtype=np.int64)
    assert lin["status"] == 0
    assert lin["num_nodes"] == n
    if n == 0:
        assert L == 0
        return
    # perm and inv are mutual inverse bijections: every node exactly once
    assert sorted(perm.tolist()) == list(range(n))
    assert np.array_equal(inv[perm], np.arange(n))
    # level sizes cover N; every level non-empty and contiguous, root-most first
    assert ls.sum() == n and (ls > 0).all()
    for l in range(L):
        assert lb[l] == ls[l + 1:].sum()
        seg = hn[lb[l]:lb[l] + ls[l]]
        assert (seg == l).all()
    # header
    assert lin["num_leaves"] == ls[0]
    assert lin["first_leaf"] == n - ls[0]
    assert lin["max_level_size"] == ls.max()
    # remapped children; for every edge v->c: level(c) < level(v), new(c) > new(v)
    for k in range(maxc):
        for i in range(n):
            c = children[k, perm[i]]
            assert chn[k, i] == (-1 if c == -1 else inv[c])
            if c != -1:
                assert hn[inv[c]] < hn[i]
                assert inv[c] > i
    # leaf check is one comparison: i >= first_leaf <=> no children
    has_kids = (chn != -1).any(axis=0)
    for i in range(n):
        assert (i >= lin["first_leaf"]) == (not has_kids[i])
    # heights: 0 for leaves, 1 + max child otherwise
    for i in range(n):
        kids = [c for c in chn[:, i] if c != -1]
        assert hn[i] == (0 if not kids else 1 + max(hn[c] for c in kids))
    # stable: ids ascend with input id inside each level (Q4)
    for l in range(L):
        seg = perm[lb[l]:lb[l] + ls[l]]
        assert (np.diff(seg) > 0).all()
    # roots = in-degree-0 nodes, ascending input id (Q23)
    indeg = np.zeros(n, np.int64)
    for k in range(maxc):
        for v in range(n):
            if children[k, v] != -1:
                indeg[children[k, v]] += 1
    want_roots = [inv[v] for v in range(n) if indeg[v] == 0]
    assert list(np.asarray(lin["roots"][:lin["num_roots"]])) == want_roots
    # structures: roots own themselves; a node belongs to the smallest root
    # index among its parents' structures (trees: exactly its parent's)
    if "structure" in lin:
        st = np.asarray(lin["structure"], dtype=np.int64)
        R = lin["num_roots"]
        assert ((st >= 0) & (st < max(R, 1))).all()
        for r in range(R):
            assert st[lin["roots"][r]] == r
        for i in range(n):
            pars = [p for p in range(n) for k in range(maxc) if chn[k, p] == i] if n <= 64 else None
            if pars:
                assert st[i] == min(st[p] for p in pars)
    # within-level independence: no node is a child of a node
    # in its own level -- implied by hn[child] < hn[parent] above
