"""The GA kernels replace sus_select's sequential walk (ga.py:95-116,
oracle/ga.py sus_select) by its running sums plus a per-pick binary search
(kernels_ga.cu ga_reduce_sus_body / ga_select_local).  This checks that
restatement of the algorithm against the walk itself on CPU: same float
sums in the same order, picks equal for random, sparse, tied and
boundary-hitting fitness vectors."""
import bisect

import numpy as np

from oracle.ga import sus_select


def sus_search(fits, count, g):
    total = float(np.sum(fits))
    if total <= 0.0:
        return [int(g.integers(len(fits))) for _ in range(count)]
    spacing = total / count
    pointer = g.uniform(0.0, spacing)
    running, c = [], 0.0
    for f in fits:  # C[i + 1] in the walk's own rounding
        c += float(f)
        running.append(c)
    pointers = []
    for _ in range(count):
        pointers.append(pointer)
        pointer += spacing
    # first j in [0, P-2] with C[j + 1] > p, else P - 1
    return [bisect.bisect_right(running[: len(fits) - 1], p) for p in pointers]


def _cases():
    rng = np.random.default_rng(7)
    for P in (1, 2, 3, 7, 8, 9, 50, 128, 129, 256):
        yield rng.random(P)
        yield np.where(rng.random(P) < 0.5, 0.0, rng.random(P))  # many zeros: flat runs of C
        yield np.full(P, 0.25)  # ties everywhere
        yield np.round(rng.random(P), 2)  # coarse values: pointers land on sums exactly
        z = np.zeros(P)
        z[rng.integers(P)] = 1.0
        yield z


def test_parallel_sus_search_equals_the_walk():
    n = 0
    for fits in _cases():
        for seed in range(20):
            a = sus_select(fits, len(fits), np.random.default_rng(seed))
            b = sus_search(fits, len(fits), np.random.default_rng(seed))
            assert a == b, (fits, seed)
            n += 1
    assert n > 900


def test_pointer_exactly_on_a_running_sum():
    # spacing 0.25 with a pointer drawn as 0: pointers 0, .25, .5, .75 hit C exactly
    fits = np.array([0.25, 0.25, 0.25, 0.25])

    class Zero:
        def uniform(self, lo, hi):
            return lo

        def integers(self, n):
            return 0

    assert sus_select(fits, 4, Zero()) == sus_search(fits, 4, Zero())
