"""sus_select at large populations from the REFERENCE itself (TEST
INFRASTRUCTURE ONLY; build container): ga.sus_select (ga.py:95-116) driven by
the SUS counter stream (seed, DOM_GA_SUS, generation) on the fitness vectors
of oracle/targets.sus_fitness (rebuilt by the tests, not stored).

  sus_large.npz   per case: P, count, seed, generation, numpy's total, the
                  SHA-256 of the picks (int64 little-endian), first / last 64 picks

Usage:  python oracle/gen_golden_sus.py
"""
import hashlib
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parent))
import gen_golden as G  # noqa: E402  (imports the reference)
from targets import sus_fitness  # noqa: E402

CASES = [  # (name, P, count, kind, seed, generation)
    ("p70k_skewed", 70_000, 70_000, "skewed", 11, 3),
    ("p300k_zeros", 300_000, 300_000, "zeros", 12, 7),
    ("p131k_ties_half", 131_072, 65_537, "ties", 13, 1),
    ("p200k_skewed_double", 200_003, 400_000, "skewed", 14, 0),
    ("p600_ties", 600, 600, "ties", 15, 2),
    ("p131k_dyadic_pow2", 131_072, 131_072, "dyadic", 16, 4),
    ("p100k_range", 100_000, 100_000, "range", 17, 5),
    ("p1m_skewed", 1_048_576, 1_048_576, "skewed", 18, 6),
    ("p100k_tie40", 100_000, 65_536, "tie40", 19, 8),
]


def main():
    out = {}
    for name, P, count, kind, seed, gen in CASES:
        f = sus_fitness(P, seed, kind)
        picks = np.asarray(G.R_ga.sus_select(list(map(float, f)), count, G.stream(seed, G.DOM_GA_SUS, gen)),
                           dtype=np.int64)
        out[name + "_meta"] = np.array([P, count, seed, gen], dtype=np.int64)
        out[name + "_kind"] = np.array(kind)
        out[name + "_total"] = np.float64(np.sum(list(map(float, f))))
        out[name + "_sha"] = np.array(hashlib.sha256(picks.astype("<i8").tobytes()).hexdigest())
        out[name + "_head"] = picks[:64]
        out[name + "_tail"] = picks[-64:]
        print(name, picks[:5], picks[-3:], flush=True)
    np.savez_compressed(G.OUT / "sus_large.npz", **out)


if __name__ == "__main__":
    main()
