"""QEQEA trajectories with nMeas above numpy's inversion range (the BTPE
binomial branch in the Born measurement, engine.py:167-170), from the
REFERENCE itself (TEST INFRASTRUCTURE ONLY; build container):

  traj_qeqea_nmeas100.npz   n = 3, L = 12, P = 5, nMeas = 100, 20 generations
  traj_qeqea_nmeas61_n4.npz n = 4, L = 8,  P = 6, nMeas = 61, 15 generations
  traj_qeqea_long.npz       n = 3, L = 150, P = 4, 6 generations (L > 128: the
                            warp-per-circuit sampling path, several fitness chunks)

  traj_ga_l1.npz / traj_ga_long.npz   GA at L = 1 and L = 100 (`... ga`)

Usage:  python oracle/gen_golden_nmeas.py; python oracle/gen_golden_nmeas.py ga
"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent))
import gen_golden as G  # noqa: E402  (imports the reference)


def main():
    G.gen_qeqea_traj("nmeas100", 3, 12, 5, G.target_for(3, "Toffoli"), 20, 21, n_meas=100,
                     probability_of_mutation=0.5)
    G.gen_qeqea_traj("nmeas61_n4", 4, 8, 6, G.target_for(4, "CCCNOT"), 15, 22, n_meas=61)
    G.gen_qeqea_traj("long", 3, 150, 4, G.target_for(3, "Toffoli"), 6, 23)
    print("wrote traj_qeqea_nmeas100.npz, traj_qeqea_nmeas61_n4.npz, traj_qeqea_long.npz")


if __name__ == "__main__" and len(sys.argv) == 1:
    main()


def ga_edges():
    """GA trajectories at the genome-length edges: L = 1 (no crossover draw,
    ga.py:85-86) and L = 100."""
    G.gen_ga_traj("l1", 2, 1, 6, G.target_for(2, "CNOT"), 12, 24)
    G.gen_ga_traj("long", 3, 100, 20, G.target_for(3, "Toffoli"), 8, 25)
    print("wrote traj_ga_l1.npz, traj_ga_long.npz")


if __name__ == "__main__" and len(sys.argv) > 1 and sys.argv[1] == "ga":
    ga_edges()
