"""Conflict-graph serializability checker for the debug event log (PAPER.md:336:
"the verification program scans the sequence and constructs a conflict graph.  If a
loop is detected, it reports a bug and provides details").  Part of the library's
tooling (not the oracle): it only looks at the order of physical accesses.

Events of committed attempts only (aborted attempts never install, PAPER.md:336 /
SPEC.md:553).  For each record, in sequence order, a write by T gets an edge from the
last writer and from every reader since that write; a read by T gets an edge from the
last writer.  The history is conflict-serializable iff the graph is acyclic (valid for
the single-version schemes; MVCC reads of older versions are not physical-order
conflicts and are excluded by the caller)."""
from __future__ import annotations

from collections import defaultdict, deque

import numpy as np

READ, WRITE, COMMIT, ABORT = 0, 1, 2, 3


def committed_events(ev: np.ndarray) -> np.ndarray:
    com = ev[ev["kind"] == COMMIT]
    final = set(zip(com["gid"].tolist(), com["attempt"].tolist()))
    keep = np.fromiter(((g, a) in final for g, a in zip(ev["gid"].tolist(), ev["attempt"].tolist())),
                       dtype=bool, count=len(ev))
    out = ev[keep & ((ev["kind"] == READ) | (ev["kind"] == WRITE))]
    return np.sort(out, order="seq")


def conflict_graph(ev: np.ndarray):
    edges = defaultdict(set)
    last_writer, readers = {}, defaultdict(set)
    for e in ev:
        t, r, k = int(e["gid"]), int(e["rec"]), int(e["kind"])
        w = last_writer.get(r)
        if k == WRITE:
            if w is not None and w != t:
                edges[w].add(t)
            for rd in readers[r]:
                if rd != t:
                    edges[rd].add(t)
            last_writer[r] = t
            readers[r] = set()
        else:
            if w is not None and w != t:
                edges[w].add(t)
            readers[r].add(t)
    return edges


def check_serializable(ev: np.ndarray):
    """Returns (True, witness serial order) or (False, a cycle as a list of gids)."""
    ev = committed_events(ev)
    nodes = sorted(set(int(g) for g in ev["gid"]))
    edges = conflict_graph(ev)
    indeg = {n: 0 for n in nodes}
    for a, bs in edges.items():
        for b in bs:
            indeg[b] = indeg.get(b, 0) + 1
    q = deque(sorted(n for n, d in indeg.items() if d == 0))
    order = []
    while q:
        n = q.popleft()
        order.append(n)
        for m in sorted(edges.get(n, ())):
            indeg[m] -= 1
            if indeg[m] == 0:
                q.append(m)
    if len(order) == len(indeg):
        return True, order
    # report one cycle: every node left after Kahn's peel has a remaining predecessor,
    # so walking predecessors inside the remainder must repeat a node
    rest = {n for n, d in indeg.items() if d > 0}
    preds = defaultdict(list)
    for a, bs in edges.items():
        if a in rest:
            for b in bs:
                if b in rest:
                    preds[b].append(a)
    start = min(rest)
    path, seen = [start], {start: 0}
    while True:
        nxt = min(preds[path[-1]])
        if nxt in seen:
            cyc = path[seen[nxt]:] + [nxt]
            return False, cyc[::-1]
        seen[nxt] = len(path)
        path.append(nxt)
