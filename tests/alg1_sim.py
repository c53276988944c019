"""Pure-Python restatement of the paper's Alg. 1, used ONLY to pin
the oracle's top-down tree construction (O9) to the paper's own bottom-up
algorithm.  It is a different algorithm from the oracle's (one worker per
leaf, merging upward through an atomic-exchange slot array initialised to -1),
run under random interleavings.

Reading R4: data are the 63-bit fixed-point keys, the sentinel
"1" is 2^63, floor(data*m) is (key*m) >> 63, and the XOR distance is taken on
the integer keys.  Anchor left children are set afterwards as the Fig. 6
caption says.
"""
from __future__ import annotations

import random

ONE = 1 << 63


def alg1_forest(keys, m, rng: random.Random | None = None, forest: bool = True):
    """Returns (child, exchanges): child[j] = [c0, c1] with leaf refs encoded as
    ('leaf', j) and node refs as ('node', j); exchanges = atomicExch count."""
    n = len(keys)

    def data(i):
        return ONE if i < 0 or i >= n else keys[i]  # data[-1] = data[n] = 1

    def cellof(v):
        return (v * m) >> 63

    child = [[None, None] for _ in range(n)]
    other = [-1] * n  # otherBounds
    exch = [0]

    def worker(i):
        node = ("leaf", i)
        cur = cellof(keys[i])
        lo = hi = i
        while True:
            vlo, vhi = data(lo), data(hi)
            nlo, nhi = data(lo - 1), data(hi + 1)
            if forest:  # the coloured lines of Alg. 1
                if cellof(nlo) < cur:
                    nlo = ONE
                if cellof(nhi) > cur:
                    nhi = ONE
            c = 0 if (vlo ^ nlo) > (vhi ^ nhi) else 1
            parent = hi + 1 if c == 0 else lo
            child[parent][c] = node
            yield  # the atomic exchange is the only synchronisation point
            exch[0] += 1
            ob = other[parent]
            other[parent] = (lo, hi)[c]
            if ob == -1:
                return
            if c == 0:
                hi = ob
            else:
                lo = ob
            node = ("node", parent)

    live = [worker(i) for i in range(n)]
    for w in live:
        next(w, None)  # run each to its first exchange
    live = [w for w in live]
    rng = rng or random.Random(0)
    while live:
        k = rng.randrange(len(live))
        try:
            next(live[k])
        except StopIteration:
            live.pop(k)
    # anchors: left child set to the left neighbour (Fig. 6 caption)
    for j in range(n):
        first_of_cell = (j == 0) or (cellof(keys[j - 1]) != cellof(keys[j]))
        if forest and first_of_cell:
            child[j][0] = ("leaf", max(j - 1, 0))
    return child, exch[0], other
