"""-m "not gpu": the conflict-graph checker of the debug event log (PAPER.md:336,
SPEC.md:537-545): the textbook non-serializable cross is caught, serial histories pass,
aborted attempts are ignored, and on random <=6-transaction histories it agrees exactly
with an independent brute-force serial-order enumerator."""
import itertools

import numpy as np

from paper_2406_10158_b200.api import DB
from paper_2406_10158_b200.verify import check_serializable

DT = DB.EVENT_DTYPE


def _log(rows):
    """rows: (gid, rec, kind[, attempt]) in sequence order."""
    ev = np.zeros(len(rows), DT)
    for i, r in enumerate(rows):
        ev[i] = (i, r[0], r[1], r[3] if len(r) > 3 else 0, r[2])
    return ev


def test_textbook_cross_is_a_cycle():
    # T1 reads x; T2 reads y; T1 writes y; T2 writes x
    ev = _log([(1, 0, 0), (2, 1, 0), (1, 1, 1), (2, 0, 1), (1, -1 & 0xFFFFFFFF, 2), (2, 0xFFFFFFFF, 2)])
    ok, cyc = check_serializable(ev)
    assert not ok and set(cyc) == {1, 2}


def test_serial_history_passes_with_order():
    ev = _log([(5, 0, 0), (5, 0, 1), (5, 0xFFFFFFFF, 2), (3, 0, 0), (3, 1, 1), (3, 0xFFFFFFFF, 2)])
    ok, order = check_serializable(ev)
    assert ok and order.index(5) < order.index(3)


def test_aborted_attempts_are_ignored():
    # attempt 0 of T1 would form a cross with T2 but aborted; attempt 1 runs after T2
    ev = _log([(1, 0, 0, 0), (2, 1, 0), (1, 1, 1, 0), (1, 0xFFFFFFFF, 3, 0), (2, 0, 1), (2, 0xFFFFFFFF, 2),
               (1, 0, 0, 1), (1, 1, 1, 1), (1, 0xFFFFFFFF, 2, 1)])
    ok, order = check_serializable(ev)
    assert ok and order == [2, 1]


def _brute(ops, n):
    """exists a serial order consistent with every conflicting pair of the history?"""
    pairs = set()
    for i, (ti, ri, ki) in enumerate(ops):
        for tj, rj, kj in ops[i + 1:]:
            if ti != tj and ri == rj and (ki == 1 or kj == 1):
                pairs.add((ti, tj))
    for perm in itertools.permutations(range(n)):
        pos = {t: k for k, t in enumerate(perm)}
        if all(pos[a] < pos[b] for a, b in pairs):
            return True
    return False


def test_agrees_with_brute_force_enumerator():
    rng = np.random.default_rng(7)
    n_cyc = 0
    for _ in range(1000):
        n = int(rng.integers(2, 7))
        txn_ops = [[(t, int(rng.integers(0, 3)), int(rng.integers(0, 2))) for _ in range(int(rng.integers(1, 4)))]
                   for t in range(n)]
        # random interleaving preserving each transaction's program order
        cursors = [0] * n
        hist = []
        while any(c < len(o) for c, o in zip(cursors, txn_ops)):
            t = int(rng.choice([k for k in range(n) if cursors[k] < len(txn_ops[k])]))
            hist.append(txn_ops[t][cursors[t]])
            cursors[t] += 1
        rows = [(t, r, k) for (t, r, k) in hist] + [(t, 0xFFFFFFFF, 2) for t in range(n)]
        ok, _ = check_serializable(_log(rows))
        assert ok == _brute(hist, n)
        n_cyc += not ok
    assert n_cyc > 50   # the sample contains non-serializable histories
