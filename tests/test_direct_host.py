"""Host logic of the direct solver, on CPU: the nested-
dissection camera order and the tile-level symbolic Cholesky, against an
independent dense symbolic factorisation and numeric fill."""
import ctypes

import numpy as np
import pytest

from paper_2409_12190_b200 import _lib
from paper_2409_12190_b200._lib import ptr


def nd_order(C, edges, leaf=24):
    e = np.ascontiguousarray(np.asarray(edges, np.int32).reshape(-1, 2))
    order, gptr, ng = np.empty(C, np.int32), np.empty(C + 1, np.int32), ctypes.c_int32()
    assert _lib.load().bae_nd_order(C, e.shape[0], ptr(e, ctypes.c_int32), leaf, ptr(order, ctypes.c_int32),
                                    ptr(gptr, ctypes.c_int32), ctypes.byref(ng)) == 0
    return order, gptr[:ng.value + 1]


def tile_symbolic(nt, pairs):
    pr = np.ascontiguousarray(np.asarray(pairs, np.int32).reshape(-1, 2))
    colptr, rowidx, nnz = np.empty(nt + 1, np.int32), np.empty(nt * nt, np.int32), ctypes.c_int64()
    assert _lib.load().bae_tile_symbolic(nt, pr.shape[0], ptr(pr, ctypes.c_int32), ptr(colptr, ctypes.c_int32),
                                         ptr(rowidx, ctypes.c_int32), nt * nt, ctypes.byref(nnz)) == 0
    return colptr, rowidx[:nnz.value]


def dense_symbolic(nt, pairs):
    """Boolean right-looking elimination: L's pattern."""
    a = np.eye(nt, dtype=bool)
    for i, j in pairs:
        a[i, j] = a[j, i] = True
    for k in range(nt):
        rows = np.flatnonzero(a[k + 1:, k]) + k + 1
        for i in rows:
            a[rows, i] = True
            a[i, rows] = True
    return np.tril(a)


def ring_edges(C, band):
    return [(max(c, (c + d) % C), min(c, (c + d) % C)) for c in range(C) for d in range(1, band + 1)]


@pytest.mark.parametrize("seed", range(6))
def test_tile_symbolic_matches_dense_elimination(seed):
    rng = np.random.default_rng(seed)
    nt = int(rng.integers(3, 40))
    pairs = {(i, j) for i, j in zip(rng.integers(0, nt, 2 * nt), rng.integers(0, nt, 2 * nt)) if i != j}
    pairs = [(max(i, j), min(i, j)) for i, j in pairs]
    colptr, rowidx = tile_symbolic(nt, pairs)
    ref = dense_symbolic(nt, pairs)
    for j in range(nt):
        rows = rowidx[colptr[j]:colptr[j + 1]]
        assert rows[0] == j and np.all(np.diff(rows) > 0)  # diagonal first, ascending
        assert np.array_equal(rows, np.flatnonzero(ref[:, j])), j


def test_tile_symbolic_covers_numeric_fill():
    """Numeric Cholesky of a random SPD matrix with the tile pattern never
    puts a nonzero outside the symbolic tiles."""
    rng = np.random.default_rng(7)
    nt, tb = 12, 4
    pairs = [(i, j) for i in range(nt) for j in range(i) if rng.random() < 0.2]
    m = np.zeros((nt * tb, nt * tb))
    for i, j in pairs + [(k, k) for k in range(nt)]:
        blk = rng.standard_normal((tb, tb))
        m[i * tb:(i + 1) * tb, j * tb:(j + 1) * tb] = blk
        m[j * tb:(j + 1) * tb, i * tb:(i + 1) * tb] = blk.T
    m = m @ m.T * 0 + m + nt * tb * 4 * np.eye(nt * tb)  # symmetric, diagonally dominant
    L = np.linalg.cholesky(m)
    colptr, rowidx = tile_symbolic(nt, pairs)
    allowed = np.zeros((nt, nt), bool)
    for j in range(nt):
        allowed[rowidx[colptr[j]:colptr[j + 1]], j] = True
    for i in range(nt):
        for j in range(i + 1):
            if np.abs(L[i * tb:(i + 1) * tb, j * tb:(j + 1) * tb]).max() > 1e-12:
                assert allowed[i, j], (i, j)


def test_nd_order_is_a_permutation_and_shortens_the_ring_chain():
    C, band = 257, 15
    edges = ring_edges(C, band)
    order, gptr = nd_order(C, edges)
    assert np.array_equal(np.sort(order), np.arange(C))
    assert gptr[0] == 0 and gptr[-1] == C and np.all(np.diff(gptr) > 0)
    # tile pattern in the padded group layout, then the elimination-tree height
    pos, at = np.empty(C, int), 0
    for g in range(len(gptr) - 1):
        for c in order[gptr[g]:gptr[g + 1]]:
            pos[c] = at
            at += 1
        at = (at + 7) // 8 * 8
    nt = at // 8
    tp = {(max(pos[a] // 8, pos[b] // 8), min(pos[a] // 8, pos[b] // 8)) for a, b in edges}
    tp = [p for p in tp if p[0] != p[1]]
    colptr, rowidx = tile_symbolic(nt, tp)
    parent = [rowidx[colptr[j] + 1] if colptr[j + 1] - colptr[j] > 1 else -1 for j in range(nt)]
    depth = [0] * nt
    for j in range(nt):  # parents come later in the order
        if parent[j] >= 0:
            depth[parent[j]] = max(depth[parent[j]], depth[j] + 1)
    height = max(depth) + 1
    natural_nt = (C + 7) // 8
    assert height <= natural_nt // 2, (height, natural_nt)


def test_nd_order_dense_graph_is_one_group():
    C = 20
    edges = [(i, j) for i in range(C) for j in range(i)]
    order, gptr = nd_order(C, edges)
    assert len(gptr) == 2 and np.array_equal(np.sort(order), np.arange(C))


def test_nd_order_disconnected_components():
    edges = ring_edges(30, 2) + [(a + 30, b + 30) for a, b in ring_edges(30, 2)]
    order, gptr = nd_order(60, edges)
    assert np.array_equal(np.sort(order), np.arange(60))


def chol_tasks(nt, pairs, min_ops, tail):
    pr = np.ascontiguousarray(np.asarray(pairs, np.int32).reshape(-1, 2))
    cap = 4 * nt * nt * nt + 64
    ob, oo = np.empty(nt + 1, np.int32), np.empty(4 * cap, np.int32)
    bp, op = np.empty(nt + 1, np.int32), np.empty(4 * cap, np.int32)
    tk, nt_, hm = np.empty(4 * cap, np.int32), ctypes.c_int32(), np.empty(nt, np.uint32)
    assert _lib.load().bae_chol_tasks(nt, pr.shape[0], ptr(pr, ctypes.c_int32), min_ops, tail, cap,
                                      ptr(ob, ctypes.c_int32), ptr(oo, ctypes.c_int32), ptr(bp, ctypes.c_int32),
                                      ptr(op, ctypes.c_int32), ptr(tk, ctypes.c_int32), ctypes.byref(nt_),
                                      hm.ctypes.data_as(ctypes.POINTER(ctypes.c_uint32))) == 0
    return ob, oo.reshape(-1, 4), bp, op.reshape(-1, 4), tk[:4 * nt_.value].reshape(-1, 4), hm


@pytest.mark.parametrize("min_ops,tail", [(1, 1 << 20), (2, 1 << 20), (1, 8), (0, 1 << 20)])
def test_chol_helper_tasks_partition_the_updates(min_ops, tail):
    """Update helpers: every update of the factorisation runs
    exactly once, a helper's updates are its tile's non-k_last updates in the
    owner's order, the queue is ordered so that every task only waits on
    tasks before it (topological, a column's helpers before its owner), and
    only the queue's last `tail` tasks belong to columns with helpers."""
    C = 96
    order, gptr = nd_order(C, ring_edges(C, 6), 24)
    pos = np.empty(C, int)
    at = 0
    for g in range(len(gptr) - 1):  # groups padded to whole tiles of 8 cameras
        for c in order[gptr[g]:gptr[g + 1]]:
            pos[c] = at
            at += 1
        at = (at + 7) // 8 * 8
    nt = at // 8
    pairs = sorted({(max(pos[a] // 8, pos[b] // 8), min(pos[a] // 8, pos[b] // 8)) for a, b in ring_edges(C, 6)})
    ob, oo, bp, op, tasks, hm = chol_tasks(nt, pairs, min_ops, tail)
    colptr, _ = tile_symbolic(nt, [p for p in pairs if p[0] != p[1]])
    slot_col = np.repeat(np.arange(nt), np.diff(colptr))  # the column of every stored tile slot

    def mine_ops(ops, b, e):
        return [tuple(x) for x in ops[b:e]]

    seen = []
    owner_seen = set()
    for qi, (j, s, b, e) in enumerate(tasks):
        orig = [tuple(x) for x in oo[ob[j]:ob[j + 1]]]
        # topological: the owners of every column k whose tiles this task reads (L(j,k), L(i,k)) came before
        deps = {slot_col[x[1]] for x in mine_ops(op, b, e)} | {slot_col[x[2]] for x in mine_ops(op, b, e)}
        assert deps <= owner_seen, (j, deps - owner_seen)
        qlast = max((x[3] for x in orig), default=-1)
        mine = [tuple(x) for x in op[b:e]]
        if s == 0:
            assert (b, e) == (bp[j], bp[j + 1])
            assert mine == [x for x in orig if not ((hm[j] >> x[0]) & 1 and x[3] != qlast)]
            owner_seen.add(j)
        else:
            assert j not in owner_seen and (hm[j] >> s) & 1  # a helper runs before its owner
            assert mine == [x for x in orig if x[0] == s and x[3] != qlast]
            assert len(mine) >= max(min_ops, 1)
        seen += mine
    assert owner_seen == set(range(nt))
    assert sorted(seen) == sorted(tuple(x) for x in oo[:ob[nt]])
    helped = [j for j in range(nt) if hm[j]]
    if helped:
        first = min(qi for qi, t in enumerate(tasks) if t[0] == helped[0])
        assert len(tasks) - first <= tail
    if min_ops == 0:
        assert not helped and len(tasks) == nt


def _nd_serial(C, edges, leaf):
    """Serial restatement of nd_camera_groups (chol.cu) for the threaded version's check."""
    adj = [[] for _ in range(C)]
    for a, b in edges:
        adj[a].append(b)
        adj[b].append(a)
    groups = []

    def bfs(root, inset):
        level = {root: 0}
        order = [root]
        for v in order:
            for w in adj[v]:
                if w in inset and w not in level:
                    level[w] = level[v] + 1
                    order.append(w)
        return order, level

    def rec(nodes):
        if not nodes:
            return
        nodes = sorted(nodes)
        inset = set(nodes)
        order, level = bfs(nodes[0], inset)
        if len(order) != len(nodes):
            rest = [v for v in nodes if v not in level]
            rec(order)
            rec(rest)
            return
        order, level = bfs(order[-1], inset)
        nlev = level[order[-1]] + 1
        if len(nodes) <= leaf or nlev < 3:
            groups.append(order)
            return
        cnt = [0] * nlev
        for v in nodes:
            cnt[level[v]] += 1
        m, acc = 0, 0
        while m < nlev:
            acc += cnt[m]
            if 2 * acc >= len(nodes):
                break
            m += 1
        m = min(max(m, 1), nlev - 2)
        rec([v for v in order if level[v] < m])
        rec([v for v in order if level[v] > m])
        groups.append([v for v in order if level[v] == m])

    rec(list(range(C)))
    return groups


def test_nd_order_threaded_equals_serial():
    """The top levels of the nested dissection run on threads; the groups and
    their order equal the serial recursion (a ring with a wide band and a
    second component, big enough for the threaded levels)."""
    C = 3000
    edges = ring_edges(2600, 12) + [(a + 2600, b + 2600) for a, b in ring_edges(400, 3)]
    order, gptr = nd_order(C, edges, 24)
    ref = _nd_serial(C, edges, 24)
    got = [list(order[gptr[g]:gptr[g + 1]]) for g in range(len(gptr) - 1)]
    assert got == ref
