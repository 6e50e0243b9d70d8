"""encoding.py's per-unit operators from the REFERENCE itself (TEST
INFRASTRUCTURE ONLY; build container), on the counter streams the device
engines use (oracle/streams.py):

  mutate_angle / mutate_qutrit   slot stream (seed, MUTATE, g, slot) after the
                                 engine's mask and coin draws (engine.py:241-242)
  estimate_axis                  (seed, MEASURE, g, slot), nMeas 1 / 3 / 11 / 61 / 1000
  measure_qutrit                 (seed, MEASURE, g, slot, sub 1)
  random_angle                   (seed, INIT, 0, slot)
  born_probabilities, su3_operator

  encoding.npz

Usage:  python oracle/gen_golden_encoding.py
"""
import math
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parent))
import gen_golden as G  # noqa: E402  (imports the reference)
from streams import DOM_INIT, DOM_MEASURE, DOM_MUTATE, stream  # noqa: E402

SEED, FIRST, GENS = 13, 100, (0, 7)


def main():
    rng = np.random.default_rng(1234)
    n = 64
    q = rng.normal(size=(n, 3)) + 1j * rng.normal(size=(n, 3))
    q /= np.linalg.norm(q, axis=1, keepdims=True)
    q[0] = [1, 0, 0]
    q[1] = [0, 1j, 0]
    q[2] = [0, 0, -1]
    q[3] = np.array([1, 1, 1]) / math.sqrt(3)
    th = rng.uniform(0.0, 2 * math.pi, n)
    th[:3] = [0.0, 2 * math.pi - 1e-12, 1e-13]
    f = rng.uniform(0.0, 1.0, n)
    f[:3] = [0.0, 0.999, 0.5]
    out = {"qutrits": q, "thetas": th, "fits": f, "meta": np.array([SEED, FIRST], dtype=np.int64)}
    for g in GENS:
        ma, mq, mm = [], [], []
        for i in range(n):
            st = stream(SEED, DOM_MUTATE, g, FIRST + i)
            st.random(), st.random()  # the engine's mask and coin
            ma.append(G.R_enc.mutate_angle(float(th[i]), float(f[i]), 0.7, st))
            st = stream(SEED, DOM_MUTATE, g, FIRST + i)
            st.random(), st.random()
            mq.append(G.R_enc.mutate_qutrit(q[i], float(f[i]), st))
            mm.append(int(G.R_enc.measure_qutrit(q[i], stream(SEED, DOM_MEASURE, g, FIRST + i, 1))))
        out[f"g{g}_mutate_angle"] = np.array(ma)
        out[f"g{g}_mutate_qutrit"] = np.array(mq)
        out[f"g{g}_measure"] = np.array(mm)
        for nm in (1, 3, 11, 61, 1000):
            out[f"g{g}_estimate_nm{nm}"] = np.array(
                [int(G.R_enc.estimate_axis(q[i], nm, stream(SEED, DOM_MEASURE, g, FIRST + i))) for i in range(n)])
    out["born"] = np.array([G.R_enc.born_probabilities(q[i]) for i in range(n)])
    out["random_angle"] = np.array([G.R_enc.random_angle(stream(SEED, DOM_INIT, 0, FIRST + i)) for i in range(n)])
    prm = np.concatenate([rng.uniform(0, 1, (24, 8)) * G.R_enc.SU3_RANGES, np.zeros((1, 8)),
                          np.eye(8) * G.R_enc.SU3_RANGES * 0.3])
    out["su3_params"] = prm
    out["su3"] = np.array([G.R_enc.su3_operator(G.R_enc.SU3Params(*p)) for p in prm])
    np.savez_compressed(G.OUT / "encoding.npz", **out)
    print("wrote encoding.npz")


if __name__ == "__main__":
    main()
